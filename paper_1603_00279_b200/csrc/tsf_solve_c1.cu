// Instantiation of the fused solve kernels for thread-block clusters of 1 CTA(s).
#include "tsf_kernels.cuh"

namespace tsf {
TSF_INSTANTIATE_CLUSTER(1)
}  // namespace tsf
