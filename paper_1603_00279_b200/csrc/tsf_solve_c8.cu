// Instantiation of the fused solve kernels for thread-block clusters of 8 CTA(s).
#include "tsf_kernels.cuh"

namespace tsf {
TSF_INSTANTIATE_CLUSTER(8)
}  // namespace tsf
