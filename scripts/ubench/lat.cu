// Micro-benchmarks of the latencies/throughputs the AM kernel depends on (B200, sm_100a).
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__global__ void dfma_lat(double* out, double a, double b, int n, long long* t) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, b, a);
  long long t1 = clock64();
  if (threadIdx.x == 0) { t[0] = t1 - t0; }
  out[threadIdx.x] = x;
}
__global__ void dfma_tput(double* out, double a, double b, int n, long long* t) {
  double x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3, x4 = a + 4, x5 = a + 5, x6 = a + 6, x7 = a + 7;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    x0 = fma(x0, b, a); x1 = fma(x1, b, a); x2 = fma(x2, b, a); x3 = fma(x3, b, a);
    x4 = fma(x4, b, a); x5 = fma(x5, b, a); x6 = fma(x6, b, a); x7 = fma(x7, b, a);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) { t[0] = t1 - t0; }
  out[threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void rsqrt_lat(double* out, double a, int n, long long* t) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = rsqrt(x) + 1.0;
  long long t1 = clock64();
  if (threadIdx.x == 0) t[0] = t1 - t0;
  out[threadIdx.x] = x;
}
__global__ void lds_lat(double* out, int n, long long* t) {
  __shared__ double s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (double)((i * 7 + 1) & 1023);
  __syncthreads();
  int idx = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) idx = (int)s[idx];
  long long t1 = clock64();
  if (threadIdx.x == 0) t[0] = t1 - t0;
  out[threadIdx.x] = idx;
}
__global__ void shfl_lat(double* out, double a, int n, long long* t) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffff, x, (threadIdx.x + 1) & 31);
  long long t1 = clock64();
  if (threadIdx.x == 0) t[0] = t1 - t0;
  out[threadIdx.x] = x;
}
__global__ void __cluster_dims__(2, 1, 1) dsmem_lat(double* out, int n, long long* t) {
  __shared__ double s[1024];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (double)((i * 7 + 1) & 1023);
  cl.sync();
  double* r = cl.map_shared_rank(s, cl.block_rank() ^ 1);
  int idx = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) idx = (int)r[idx];
  long long t1 = clock64();
  if (threadIdx.x == 0 && cl.block_rank() == 0) t[0] = t1 - t0;
  out[threadIdx.x] = idx;
  cl.sync();
}
__global__ void __cluster_dims__(8, 1, 1) cbar_lat(int n, long long* t) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) t[0] = t1 - t0;
}
__global__ void __cluster_dims__(8, 1, 1) cbar_relaxed_lat(int n, long long* t) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) t[0] = t1 - t0;
}
__global__ void bar_lat(int n, long long* t) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) t[0] = t1 - t0;
}

int main() {
  double* out; long long* t; long long h;
  cudaMalloc(&out, 4096 * 8); cudaMalloc(&t, 64);
  const int n = 4096;
  auto rd = [&](const char* name, double per, const char* unit) { cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost); printf("%-34s %8.2f %s\n", name, h / per, unit); };
  dfma_lat<<<1, 32>>>(out, 1.0, 0.999, n, t); cudaDeviceSynchronize(); rd("DFMA dependent latency", n, "cyc");
  for (int w : {1, 4, 8, 16, 32}) {
    dfma_tput<<<1, 32 * w>>>(out, 1.0, 0.999, n, t); cudaDeviceSynchronize();
    cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
    printf("DFMA throughput %2d warps/SM         %8.2f lanes*DFMA/cyc/SM\n", w, 32.0 * w * 8 * n / h);
  }
  rsqrt_lat<<<1, 32>>>(out, 2.0, n, t); cudaDeviceSynchronize(); rd("rsqrt(double)+DADD dependent", n, "cyc");
  lds_lat<<<1, 32>>>(out, n, t); cudaDeviceSynchronize(); rd("LDS.64 dependent (pointer chase)", n, "cyc");
  shfl_lat<<<1, 32>>>(out, 1.0, n, t); cudaDeviceSynchronize(); rd("SHFL (double) dependent", n, "cyc");
  dsmem_lat<<<2, 32>>>(out, 1024, t); cudaDeviceSynchronize(); rd("DSMEM load dependent (peer CTA)", 1024, "cyc");
  cbar_lat<<<8, 512>>>(1024, t); cudaDeviceSynchronize(); rd("cluster barrier (8 CTA x 512 thr)", 1024, "cyc");
  cbar_relaxed_lat<<<8, 512>>>(1024, t); cudaDeviceSynchronize(); rd("cluster barrier relaxed", 1024, "cyc");
  bar_lat<<<1, 512>>>(1024, t); cudaDeviceSynchronize(); rd("__syncthreads (512 thr)", 1024, "cyc");
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
