// Post-solve safety verdict on the device: st_check_collisions (declared in include/swarm_am.h).
//
// Replaces the O(n^2 m) scalar loop of the reference's check_collisions
// (validation.py:39-93), which am_solve runs once after the loop through
// _final_metrics (solver.py:461, 497-509).  Rows are the reference's pair
// order: agent pairs (i<j) lexicographic, then (agent i, obstacle k)
// agent-major; within a row, samples in order.  Every value is the same IEEE
// sequence as the reference scalar code (sub, div, mul, add left to right,
// correctly rounded sqrt; no FMA contraction), so the minimum, the violation
// count and every (pair, sample, value) entry are bit-identical.
//
// Launches on one stream: (1) one warp per row: row minimum into a global
// atomicMin (non-negative doubles order like their bit patterns), the row's
// violation count, and the total; then, only when the total is non-zero,
// (2) one block: exclusive scan of the counts; (3) one warp per violating
// row: entries written at the row's offset in sample order (ballot prefix).  HBM traffic is the trajectory (n*m*24 B,
// L2-resident) plus 8 B per row; the work is latency-bound and tiny next to
// the solve, so the grid is simply rows/8 CTAs of 8 warps.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/swarm_am.h"

int swarm_fail(int code, const std::string& msg);  // capi.cu (sets st_last_error)

namespace {

constexpr int kWarpsPerBlock = 8;

struct Rows {
  const double* traj;  // B x n x m x 3
  const double* obs;   // B x n_obs x 5: cx, cy, cz, sep_xy, sep_z
  const double* geom;  // B x 2: l_xy, l_z
  int n, m, n_obs;
  long long n_pairs, n_rows;
};

// (i, j) of agent pair `row` in (i<j) lexicographic order
__device__ __forceinline__ void pair_of(long long row, int n, int& i, int& j) {
  double b = 2.0 * n - 1.0;
  int ii = (int)floor((b - sqrt(b * b - 8.0 * (double)row)) * 0.5);
  ii = max(0, min(ii, n - 2));
  auto first = [n](int a) { return (long long)a * (2LL * n - a - 1) / 2; };
  while (ii > 0 && first(ii) > row) --ii;
  while (ii < n - 2 && first(ii + 1) <= row) ++ii;
  i = ii;
  j = (int)(row - first(ii)) + ii + 1;
}

struct RowGeom {
  const double* a;  // agent i's samples
  const double* b;  // agent j's samples, or nullptr for an obstacle row
  double c0, c1, c2, sxy, sz;
  int kind, i, k;
};

__device__ __forceinline__ RowGeom row_geom(const Rows& R, int scn, long long row) {
  RowGeom g;
  const double* traj = R.traj + (size_t)scn * R.n * R.m * 3;
  if (row < R.n_pairs) {
    int i, j;
    pair_of(row, R.n, i, j);
    g.a = traj + (size_t)i * R.m * 3;
    g.b = traj + (size_t)j * R.m * 3;
    g.c0 = g.c1 = g.c2 = 0.0;
    g.sxy = R.geom[2 * scn];
    g.sz = R.geom[2 * scn + 1];
    g.kind = 0;
    g.i = i;
    g.k = j;
  } else {
    long long o = row - R.n_pairs;
    int i = (int)(o / R.n_obs), k = (int)(o % R.n_obs);
    const double* ob = R.obs + ((size_t)scn * R.n_obs + k) * 5;
    g.a = traj + (size_t)i * R.m * 3;
    g.b = nullptr;
    g.c0 = ob[0];
    g.c1 = ob[1];
    g.c2 = ob[2];
    g.sxy = ob[3];
    g.sz = ob[4];
    g.kind = 1;
    g.i = i;
    g.k = k;
  }
  return g;
}

// validation.py:67-71 (pairs) / 80-84 (obstacles), operation for operation
__device__ __forceinline__ double row_value(const RowGeom& g, int r) {
  const double* a = g.a + (size_t)r * 3;
  double o0 = g.c0, o1 = g.c1, o2 = g.c2;
  if (g.b) {
    const double* b = g.b + (size_t)r * 3;
    o0 = b[0];
    o1 = b[1];
    o2 = b[2];
  }
  double dx = __ddiv_rn(__dsub_rn(a[0], o0), g.sxy);
  double dy = __ddiv_rn(__dsub_rn(a[1], o1), g.sxy);
  double dz = __ddiv_rn(__dsub_rn(a[2], o2), g.sz);
  return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
}

__global__ void __launch_bounds__(kWarpsPerBlock * 32) rows_kernel(Rows R, int* row_cnt,
                                                                   unsigned long long* min_bits,
                                                                   unsigned long long* count) {
  const int lane = threadIdx.x & 31;
  const long long row = (long long)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  const int scn = blockIdx.y;
  if (row >= R.n_rows) return;
  const RowGeom g = row_geom(R, scn, row);
  double vmin = INFINITY;
  int cnt = 0;
#pragma unroll 4
  for (int r0 = 0; r0 < R.m; r0 += 32) {  // independent sample chunks: loads of several in flight
    const int r = r0 + lane;
    double v = r < R.m ? row_value(g, r) : INFINITY;
    vmin = fmin(vmin, v);  // a NaN never lowers the minimum (Python's min(minimum, nan) keeps minimum)
    cnt += __popc(__ballot_sync(0xffffffffu, v < 1.0));
  }
  for (int s = 16; s; s >>= 1) vmin = fmin(vmin, __shfl_xor_sync(0xffffffffu, vmin, s));
  if (lane == 0) {
    row_cnt[(size_t)scn * R.n_rows + row] = cnt;
    atomicMin(min_bits + scn, (unsigned long long)__double_as_longlong(vmin));
    if (cnt) atomicAdd(count + scn, (unsigned long long)cnt);
  }
}

// exclusive scan of one scenario's row counts (one block of 1024 threads per scenario, chunked),
// offset by the scenario's first entry base[scenario]
__global__ void __launch_bounds__(1024) scan_kernel(const int* row_cnt_all, long long* row_off_all, long long n_rows,
                                                    const long long* first) {
  constexpr int kPer = 4;  // consecutive rows per thread: 4096 rows per block pass
  const int* row_cnt = row_cnt_all + (size_t)blockIdx.x * n_rows;
  long long* row_off = row_off_all + (size_t)blockIdx.x * n_rows;
  __shared__ long long warp_sums[32];
  __shared__ long long carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = first[blockIdx.x];
  __syncthreads();
  for (long long chunk = 0; chunk < n_rows; chunk += 1024 * kPer) {
    const long long idx0 = chunk + (long long)threadIdx.x * kPer;
    long long v[kPer], own = 0;
#pragma unroll
    for (int e = 0; e < kPer; ++e) {
      v[e] = idx0 + e < n_rows ? row_cnt[idx0 + e] : 0;
      own += v[e];
    }
    long long x = own;  // inclusive scan of per-thread sums
    for (int s = 1; s < 32; s <<= 1) {
      long long y = __shfl_up_sync(0xffffffffu, x, s);
      if (lane >= s) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
      long long w = warp_sums[lane], wx = w;
      for (int s = 1; s < 32; s <<= 1) {
        long long y = __shfl_up_sync(0xffffffffu, wx, s);
        if (lane >= s) wx += y;
      }
      warp_sums[lane] = wx - w;
    }
    __syncthreads();
    const long long c = carry;
    long long run = c + warp_sums[warp] + x - own;
#pragma unroll
    for (int e = 0; e < kPer; ++e) {
      if (idx0 + e < n_rows) row_off[idx0 + e] = run;
      run += v[e];
    }
    __syncthreads();
    if (threadIdx.x == 1023) carry = run;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kWarpsPerBlock * 32) entries_kernel(Rows R, const int* row_cnt,
                                                                      const long long* row_off, long long cap,
                                                                      int* ids, double* vals) {
  const int lane = threadIdx.x & 31;
  const long long row = (long long)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  const int scn = blockIdx.y;
  if (row >= R.n_rows || row_cnt[(size_t)scn * R.n_rows + row] == 0) return;
  const RowGeom g = row_geom(R, scn, row);
  long long pos = row_off[(size_t)scn * R.n_rows + row];
  for (int r0 = 0; r0 < R.m; r0 += 32) {
    const int r = r0 + lane;
    const double v = r < R.m ? row_value(g, r) : INFINITY;
    const unsigned ball = __ballot_sync(0xffffffffu, v < 1.0);
    if (v < 1.0) {
      const long long e = pos + __popc(ball & ((1u << lane) - 1u));
      if (e < cap) {
        ids[e * 4 + 0] = g.kind;
        ids[e * 4 + 1] = g.i;
        ids[e * 4 + 2] = g.k;
        ids[e * 4 + 3] = r;
        vals[e] = v;
      }
    }
    pos += __popc(ball);
  }
}

// per-device scratch: one stream and a grow-only buffer, calls on a device serialize
struct Scratch {
  std::mutex mu;
  cudaStream_t stream = nullptr;
  void* buf = nullptr;
  size_t bytes = 0;
};
Scratch g_scratch[64];

#define CC_CUDA(call)                                                                           \
  do {                                                                                          \
    cudaError_t e_ = (call);                                                                    \
    if (e_ != cudaSuccess)                                                                      \
      return swarm_fail(e_ == cudaErrorMemoryAllocation ? ST_ENOMEM : ST_ECUDA,                \
                        std::string(#call) + ": " + cudaGetErrorString(e_));                    \
  } while (0)

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

}  // namespace

__global__ void init_summary_kernel(unsigned long long* min_total, int B) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < B; b += gridDim.x * blockDim.x) {
    min_total[b] = 0x7ff0000000000000ULL;  // +inf
    min_total[B + b] = 0;
  }
}

// Device-resident verdict summary for st_solve_report (capi.cu): per scenario the minimum
// normalized distance (bits, min_total[b]) and the violation count (min_total[B + b]) of the
// B x n x m x 3 trajectories already on the device; row_cnt: B x n_rows scratch.
cudaError_t swarm_collision_summary_launch(int B, int n, int m, const double* d_traj, const double* d_geom, int n_obs,
                                           const double* d_obs, int* row_cnt, unsigned long long* min_total,
                                           cudaStream_t s, bool init) {
  if (B <= 0) return cudaSuccess;
  if (init) init_summary_kernel<<<(B + 255) / 256, 256, 0, s>>>(min_total, B);  // else: set by the report pass
  const long long n_pairs = (long long)n * (n - 1) / 2, n_rows = n_pairs + (long long)n * n_obs;
  if (n_rows == 0 || m == 0) return cudaGetLastError();
  Rows R{d_traj, d_obs, d_geom, n, m, n_obs, n_pairs, n_rows};
  const dim3 grid((unsigned)((n_rows + kWarpsPerBlock - 1) / kWarpsPerBlock), (unsigned)B);
  rows_kernel<<<grid, kWarpsPerBlock * 32, 0, s>>>(R, row_cnt, min_total, min_total + B);
  return cudaGetLastError();
}

extern "C" int st_check_collisions_batch(int B, int n, int m, const double* traj, const double* geom, int n_obs,
                                         const double* obs, int device, long long cap, int* ids, double* vals,
                                         double* min_out, long long* total_out) {
  if (B < 0 || n < 0 || m < 0 || n_obs < 0 || cap < 0) return swarm_fail(ST_EINVAL, "negative size");
  if (B > 65535) return swarm_fail(ST_EINVAL, "batch larger than 65535 scenarios");
  if (device < 0 || device >= 64) return swarm_fail(ST_EINVAL, "bad device ordinal");
  if (B > 0 && (!min_out || !total_out || !geom || (n * m > 0 && !traj) || (n_obs > 0 && !obs)))
    return swarm_fail(ST_EINVAL, "NULL buffer");
  if (cap > 0 && (!ids || !vals)) return swarm_fail(ST_EINVAL, "NULL buffer");
  const long long n_pairs = (long long)n * (n - 1) / 2, n_rows = n_pairs + (long long)n * n_obs;
  for (int b = 0; b < B; ++b) {
    min_out[b] = INFINITY;
    total_out[b] = 0;
  }
  if (B == 0 || n_rows == 0 || m == 0) return ST_OK;
  Scratch& S = g_scratch[device];
  std::lock_guard<std::mutex> guard(S.mu);
  CC_CUDA(cudaSetDevice(device));
  if (!S.stream) CC_CUDA(cudaStreamCreateWithFlags(&S.stream, cudaStreamNonBlocking));
  const size_t b_traj = align256((size_t)B * n * m * 24), b_obs = align256((size_t)B * n_obs * 40 + 8),
               b_geom = align256((size_t)B * 16), b_cnt = align256((size_t)B * n_rows * 4),
               b_off = align256((size_t)B * n_rows * 8), b_misc = align256((size_t)B * 24),
               b_ids = align256((size_t)cap * 16), b_vals = align256((size_t)cap * 8);
  const size_t need = b_traj + b_obs + b_geom + b_cnt + b_off + b_misc + b_ids + b_vals;
  if (need > S.bytes) {
    if (S.buf) cudaFree(S.buf);
    S.buf = nullptr;
    S.bytes = 0;
    CC_CUDA(cudaMalloc(&S.buf, need));
    S.bytes = need;
  }
  char* p = (char*)S.buf;
  double* d_traj = (double*)p;
  double* d_obs = (double*)(p += b_traj);
  double* d_geom = (double*)(p += b_obs);
  int* d_cnt = (int*)(p += b_geom);
  long long* d_off = (long long*)(p += b_cnt);
  unsigned long long* d_min = (unsigned long long*)(p += b_off);  // B minima | B totals | B bases
  unsigned long long* d_total = d_min + B;
  long long* d_base = (long long*)(d_total + B);
  int* d_ids = (int*)(p += b_misc);
  double* d_vals = (double*)(p += b_ids);
  cudaStream_t s = S.stream;
  const unsigned long long inf_bits = 0x7ff0000000000000ULL;
  std::vector<unsigned long long> res(2 * (size_t)B);
  for (int b = 0; b < B; ++b) {
    res[b] = inf_bits;
    res[B + b] = 0;
  }
  CC_CUDA(cudaMemcpyAsync(d_traj, traj, (size_t)B * n * m * 24, cudaMemcpyHostToDevice, s));
  if (n_obs) CC_CUDA(cudaMemcpyAsync(d_obs, obs, (size_t)B * n_obs * 40, cudaMemcpyHostToDevice, s));
  CC_CUDA(cudaMemcpyAsync(d_geom, geom, (size_t)B * 16, cudaMemcpyHostToDevice, s));
  CC_CUDA(cudaMemcpyAsync(d_min, res.data(), 16 * (size_t)B, cudaMemcpyHostToDevice, s));
  Rows R{d_traj, d_obs, d_geom, n, m, n_obs, n_pairs, n_rows};
  const dim3 grid((unsigned)((n_rows + kWarpsPerBlock - 1) / kWarpsPerBlock), (unsigned)B);
  rows_kernel<<<grid, kWarpsPerBlock * 32, 0, s>>>(R, d_cnt, d_min, d_total);
  CC_CUDA(cudaGetLastError());
  CC_CUDA(cudaMemcpyAsync(res.data(), d_min, 16 * (size_t)B, cudaMemcpyDeviceToHost, s));
  CC_CUDA(cudaStreamSynchronize(s));
  // scenario-major entry list: scenario b starts after the entries of scenarios < b
  std::vector<long long> base(B);
  long long all = 0;
  for (int b = 0; b < B; ++b) {
    base[b] = all;
    all += (long long)res[B + b];
    double mn;
    memcpy(&mn, &res[b], 8);
    min_out[b] = mn;
    total_out[b] = (long long)res[B + b];
  }
  const long long take = all < cap ? all : cap;
  if (take > 0) {  // violations are rare on solved instances: scan + entries only when there are some
    CC_CUDA(cudaMemcpyAsync(d_base, base.data(), 8 * (size_t)B, cudaMemcpyHostToDevice, s));
    scan_kernel<<<B, 1024, 0, s>>>(d_cnt, d_off, n_rows, d_base);
    CC_CUDA(cudaGetLastError());
    entries_kernel<<<grid, kWarpsPerBlock * 32, 0, s>>>(R, d_cnt, d_off, cap, d_ids, d_vals);
    CC_CUDA(cudaGetLastError());
    CC_CUDA(cudaMemcpyAsync(ids, d_ids, (size_t)take * 16, cudaMemcpyDeviceToHost, s));
    CC_CUDA(cudaMemcpyAsync(vals, d_vals, (size_t)take * 8, cudaMemcpyDeviceToHost, s));
    CC_CUDA(cudaStreamSynchronize(s));
  }
  return ST_OK;
}

extern "C" int st_check_collisions(int n, int m, const double* traj, double l_xy, double l_z, int n_obs,
                                   const double* obs, int device, long long cap, int* ids, double* vals,
                                   double* min_out, long long* total_out) {
  if (!min_out || !total_out) return swarm_fail(ST_EINVAL, "NULL buffer");
  const double geom[2] = {l_xy, l_z};
  return st_check_collisions_batch(1, n, m, traj, geom, n_obs, obs, device, cap, ids, vals, min_out, total_out);
}
