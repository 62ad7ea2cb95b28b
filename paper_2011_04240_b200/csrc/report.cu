// Report pass of st_solve_report on the device: the sampled trajectories and the per-agent
// quality metrics of every scenario of a batch, straight from the solved coefficients.
//
// Replaces the post-loop host work of the reference's am_solve:
//   solver.py:133-136   trajectories: c_axis @ P.T per axis, reported as (n, m, 3)
//   validation.py:96-121 arc_length (sum over samples of |x(t+1) - x(t)|) and smoothness
//                        (|| x(t+2) - 2 x(t+1) + x(t) || over all samples and axes), which
//                        _final_metrics (solver.py:497-509) evaluates per agent.
// One warp per (scenario, agent): lanes are samples, the coefficient rows are warp-broadcast
// loads, each position a k-ascending FMA chain; the warp's (m x 3) positions go to shared
// memory and out as one contiguous, coalesced run of the (B, n, m, 3) array, the differences
// are formed from shared memory (IEEE operations without contraction, as numpy does them) and
// reduced by a fixed xor tree: deterministic.  Positions and sums follow a fixed order that
// is not BLAS's/numpy's, so values agree with the host formulas to rounding.
#include <cuda_runtime.h>

#include <cmath>

namespace {

constexpr int kWarps = 4;

constexpr int kMaxCoeffs = 16;  // n_v <= 16 (st_plan_create)

__global__ void __launch_bounds__(kWarps * 32) report_kernel(int B, int n, int m, int nv, int nvp, const double* c,
                                                             const double* P, double* traj, double* arc,
                                                             double* smooth, unsigned long long* summary) {
  extern __shared__ double xs[];  // kWarps x m x 3
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long agent = (long long)blockIdx.x * kWarps + warp;  // b * n + j
  if (agent >= (long long)B * n) return;
  const long long b = agent / n, j = agent - b * n;
  if (summary && j == 0 && lane == 0) {  // the collision summary's initial values (rows_kernel runs after)
    summary[b] = 0x7ff0000000000000ULL;  // +inf bits
    summary[B + b] = 0;
  }
  double* x = xs + (size_t)warp * m * 3;
  const double* cb = c + (size_t)b * 3 * n * nv;
  double cx[kMaxCoeffs], cy[kMaxCoeffs], cz[kMaxCoeffs];  // the agent's coefficient rows, in registers
#pragma unroll
  for (int k = 0; k < kMaxCoeffs; ++k) {
    cx[k] = k < nv ? cb[(size_t)j * nv + k] : 0.0;
    cy[k] = k < nv ? cb[((size_t)n + j) * nv + k] : 0.0;
    cz[k] = k < nv ? cb[((size_t)2 * n + j) * nv + k] : 0.0;
  }
  double* out = traj + (size_t)agent * m * 3;
  for (int t = lane; t < m; t += 32) {
    const double* pr = P + (size_t)t * nvp;
    double pk[kMaxCoeffs];
#pragma unroll
    for (int k = 0; k < kMaxCoeffs; ++k) pk[k] = k < nv ? pr[k] : 0.0;  // all loads in flight at once
    double vx = 0.0, vy = 0.0, vz = 0.0;
#pragma unroll
    for (int k = 0; k < kMaxCoeffs; ++k) {
      if (k < nv) {  // k-ascending FMA chains, as before
        vx = fma(cx[k], pk[k], vx);
        vy = fma(cy[k], pk[k], vy);
        vz = fma(cz[k], pk[k], vz);
      }
    }
    x[3 * t] = vx;
    x[3 * t + 1] = vy;
    x[3 * t + 2] = vz;
  }
  __syncwarp();
  for (int e = lane; e < 3 * m; e += 32) out[e] = x[e];
  double a = 0.0, s = 0.0;
  for (int t = lane; t + 1 < m; t += 32) {
    const double dx = __dsub_rn(x[3 * t + 3], x[3 * t]);
    const double dy = __dsub_rn(x[3 * t + 4], x[3 * t + 1]);
    const double dz = __dsub_rn(x[3 * t + 5], x[3 * t + 2]);
    a = __dadd_rn(a, __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz))));
    if (t + 2 < m) {
#pragma unroll
      for (int ax = 0; ax < 3; ++ax) {
        const double d2 = __dadd_rn(__dsub_rn(x[3 * t + 6 + ax], __dmul_rn(2.0, x[3 * t + 3 + ax])), x[3 * t + ax]);
        s = __dadd_rn(s, __dmul_rn(d2, d2));
      }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    s += __shfl_xor_sync(0xffffffffu, s, o);
  }
  if (lane == 0) {
    arc[agent] = a;
    smooth[agent] = sqrt(s);
  }
}

}  // namespace

// Shared memory of the report pass (bytes); the caller checks it against the device limit.
size_t swarm_report_smem(int m) { return (size_t)kWarps * m * 3 * sizeof(double); }

// c: B x 3 x n x nv (device), P: m x nvp (device, zero-padded rows); outputs on the device.
// summary (optional, B x 2 words): set to the collision summary's initial values (+inf bits, 0)
// for swarm_collision_summary_launch(..., init = false) to accumulate into.
cudaError_t swarm_report_launch(int B, int n, int m, int nv, int nvp, const double* c, const double* P, double* traj,
                                double* arc, double* smooth, unsigned long long* summary, cudaStream_t s) {
  const long long agents = (long long)B * n;
  if (agents == 0 || m == 0) return cudaSuccess;
  const size_t smem = swarm_report_smem(m);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(report_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  report_kernel<<<(unsigned)((agents + kWarps - 1) / kWarps), kWarps * 32, smem, s>>>(B, n, m, nv, nvp, c, P, traj,
                                                                                       arc, smooth, summary);
  return cudaGetLastError();
}
