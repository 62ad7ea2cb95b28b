// Explicit instantiations of the AM kernel variants listed in capi.cu (kKernels), split over
// translation units so that nvcc compiles them in parallel (_build.py).
#include "am_kernel.cuh"

namespace swarm {
template __global__ void am_cluster_kernel<1, 512, 12, 0, false>(const KParams);
template __global__ void am_cluster_kernel<1, 512, 12, 1, false>(const KParams);
template __global__ void am_cluster_kernel<1, 512, 12, 2, false>(const KParams);
template __global__ void am_cluster_kernel<1, 512, 12, 0, false, false>(const KParams);
template __global__ void am_cluster_kernel<1, 512, 12, 1, false, false>(const KParams);
}  // namespace swarm
