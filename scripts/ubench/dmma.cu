#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
template <int CH>
__global__ void lat(double* out, long long* cyc, int iters) {
  double acc[CH][2];
  for (int c = 0; c < CH; ++c) acc[c][0] = acc[c][1] = threadIdx.x * 1e-3 + c;
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) dmma(acc[c], a, b);
  }
  long long t1 = clock64();
  double s = 0;
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 1 << 24); cudaMalloc(&cyc, 1 << 16);
  long long h[148];
  int iters = 4096;
  // latency: 1 warp, 1 chain
  lat<1><<<1, 32>>>(out, cyc, iters); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DMMA m8n8k4 dependent latency: %.2f cyc\n", (double)h[0] / iters);
  lat<8><<<1, 32>>>(out, cyc, iters); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DMMA 1 warp 8 chains: %.2f cyc per DMMA\n", (double)h[0] / iters / 8);
  for (int w : {4, 8, 16}) {
    lat<4><<<148, 32 * w>>>(out, cyc, iters); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    double per = (double)h[0] / iters / 4;  // cycles per DMMA per warp
    printf("DMMA %2d warps/SM x 4 chains: %.2f cyc per DMMA per warp -> %.1f FMA/clk/SM\n", w, per, 256.0 * w / per);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
}
