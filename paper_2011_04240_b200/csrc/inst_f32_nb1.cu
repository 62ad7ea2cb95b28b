// Explicit instantiations of the FP32-mode kernel variants (capi.cu kKernels), one unit per group
// so nvcc compiles them in parallel (_build.py).
#include "am_kernel.cuh"

namespace swarm {
template __global__ void am_cluster_kernel<1, 512, 12, 0, true>(const KParams);
template __global__ void am_cluster_kernel<1, 512, 12, 1, true>(const KParams);
template __global__ void am_cluster_kernel<1, 512, 12, 2, true>(const KParams);
template __global__ void am_cluster_kernel<1, 512, 16, 0, true>(const KParams);
template __global__ void am_cluster_kernel<1, 512, 16, 1, true>(const KParams);
template __global__ void am_cluster_kernel<1, 512, 16, 2, true>(const KParams);
template __global__ void am_cluster_kernel<1, 512, 12, 0, true, false>(const KParams);
template __global__ void am_cluster_kernel<1, 512, 12, 1, true, false>(const KParams);
}  // namespace swarm
