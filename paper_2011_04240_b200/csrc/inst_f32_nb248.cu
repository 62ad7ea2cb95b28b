// Explicit instantiations of the FP32-mode kernel variants (capi.cu kKernels), one unit per group
// so nvcc compiles them in parallel (_build.py).
#include "am_kernel.cuh"

namespace swarm {
template __global__ void am_cluster_kernel<2, 384, 12, 1, true>(const KParams);
template __global__ void am_cluster_kernel<2, 384, 12, 2, true>(const KParams);
template __global__ void am_cluster_kernel<2, 384, 16, 1, true>(const KParams);
template __global__ void am_cluster_kernel<2, 384, 16, 2, true>(const KParams);
template __global__ void am_cluster_kernel<4, 256, 12, 1, true>(const KParams);
template __global__ void am_cluster_kernel<4, 256, 12, 2, true>(const KParams);
template __global__ void am_cluster_kernel<8, 256, 12, 1, true>(const KParams);
template __global__ void am_cluster_kernel<8, 256, 12, 2, true>(const KParams);
}  // namespace swarm
