// Explicit instantiations of the AM kernel variants listed in capi.cu (kKernels), split over
// translation units so that nvcc compiles them in parallel (_build.py).
#include "am_kernel.cuh"

namespace swarm {
#ifdef SWARM_EXPERIMENTAL_KERNELS
template __global__ void am_cluster_kernel<1, 512, 12, 3, 1>(const KParams);
template __global__ void am_cluster_kernel<1, 512, 16, 3, 1>(const KParams);
template __global__ void am_cluster_kernel<2, 384, 12, 3, 1>(const KParams);
template __global__ void am_cluster_kernel<2, 384, 16, 3, 1>(const KParams);
template __global__ void am_cluster_kernel<4, 256, 12, 3, 1>(const KParams);
template __global__ void am_cluster_kernel<8, 256, 12, 3, 1>(const KParams);
template __global__ void am_cluster_kernel<1, 256, 12, 1, 2>(const KParams);
template __global__ void am_cluster_kernel<1, 256, 16, 1, 2>(const KParams);
#endif
}  // namespace swarm
