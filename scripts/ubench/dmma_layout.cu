// Fragment layout check for mma.sync.m8n8k4 f64 (A row-major 8x4, B col 4x8, D 8x8).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(const double* A, const double* B, double* D) {
  const int l = threadIdx.x, g = l >> 2, t = l & 3;
  double a = A[g * 4 + t];      // A[row g][col t]
  double b = B[t * 8 + g];      // B[row t][col g]
  double d0 = 0, d1 = 0;
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
  D[g * 8 + 2 * t] = d0;        // D[row g][col 2t + i]
  D[g * 8 + 2 * t + 1] = d1;
}
int main() {
  double hA[32], hB[32], hD[64], *A, *B, *D;
  for (int i = 0; i < 32; ++i) { hA[i] = 1.0 + i * 0.37; hB[i] = 0.5 - i * 0.11; }
  cudaMalloc(&A, 256); cudaMalloc(&B, 256); cudaMalloc(&D, 512);
  cudaMemcpy(A, hA, 256, cudaMemcpyHostToDevice); cudaMemcpy(B, hB, 256, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(A, B, D);
  cudaMemcpy(hD, D, 512, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int r = 0; r < 8; ++r)
    for (int c = 0; c < 8; ++c) {
      double s = 0;
      for (int q = 0; q < 4; ++q) s += hA[r * 4 + q] * hB[q * 8 + c];
      double e = hD[r * 8 + c] - s; if (e < 0) e = -e; if (e > err) err = e;
    }
  printf("m8n8k4 f64 layout check: max abs err %.3e (%s)\n", err, err < 1e-12 ? "OK" : "WRONG");
}
