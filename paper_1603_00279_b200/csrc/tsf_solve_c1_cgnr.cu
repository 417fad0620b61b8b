// Solve kernels for thread-block clusters of 1 CTA(s), method cgnr (parallel compilation unit).
#include "tsf_kernels.cuh"

namespace tsf {
TSF_INSTANTIATE_METHOD(1, TSF_CGNR)
}  // namespace tsf
