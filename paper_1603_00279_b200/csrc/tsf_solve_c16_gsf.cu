// Solve kernels for thread-block clusters of 16 CTA(s), method gsf (parallel compilation unit).
#include "tsf_kernels.cuh"

namespace tsf {
TSF_INSTANTIATE_METHOD(16, TSF_GSF)
}  // namespace tsf
