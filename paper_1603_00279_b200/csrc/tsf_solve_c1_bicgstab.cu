// Solve kernels for thread-block clusters of 1 CTA(s), method bicgstab (parallel compilation unit).
#include "tsf_kernels.cuh"

namespace tsf {
TSF_INSTANTIATE_METHOD(1, TSF_BICGSTAB)
}  // namespace tsf
