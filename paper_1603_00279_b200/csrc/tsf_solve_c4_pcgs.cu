// Solve kernels for thread-block clusters of 4 CTA(s), method pcgs (parallel compilation unit).
#include "tsf_kernels.cuh"

namespace tsf {
TSF_INSTANTIATE_METHOD(4, TSF_PCGS)
}  // namespace tsf
