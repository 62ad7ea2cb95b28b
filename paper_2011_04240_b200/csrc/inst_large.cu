// Explicit instantiations of the large-fleet kernel (am_large.cuh), listed in capi.cu (kLarge).
#include "am_large.cuh"

namespace swarm {
template __global__ void am_large_kernel<12, false>(const LgParams);
template __global__ void am_large_kernel<12, true>(const LgParams);
template __global__ void am_large_kernel<16, false>(const LgParams);
template __global__ void am_large_kernel<16, true>(const LgParams);
}  // namespace swarm
