// Solve kernels for thread-block clusters of 1 CTA(s), method gsf (parallel compilation unit).
#include "tsf_kernels.cuh"

namespace tsf {
TSF_INSTANTIATE_METHOD(1, TSF_GSF)
}  // namespace tsf
