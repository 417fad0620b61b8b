// Solve kernels for thread-block clusters of 2 CTA(s), method cgnr (parallel compilation unit).
#include "tsf_kernels.cuh"

namespace tsf {
TSF_INSTANTIATE_METHOD(2, TSF_CGNR)
}  // namespace tsf
