// Large fleets (n > 64 agents): one scenario spread over every SM of the GPU -- or over the SMs
// of G GPUs, its agent pairs sharded (BASELINE config 5) -- with a (agent-block pair x time
// sample) decomposition.
//
// Reference path (pkg/src/swarmtraj/): the same AM iteration as am_kernel.cuh --
//   solver.py:405-457 loop, solver.py:178-263 pair updates, kkt_cache.py:125-135 S X / S'b,
//   kkt_cache.py:291-305 solve (structured, kkt.py) -- for one large scenario.
//
// Work units.  Agents form NB = ceil(n/32) blocks of 32; the block pairs
// (A <= B, "ab") in ab-major order give the units: a cross pair (A < B) has two per time sample,
// u = ab_first[ab] + 2 t + h, holding the 16 circulant distances s = 16h .. 16h+15 (lane a pairs
// with agent (a+s) mod 32 of block B); a diagonal pair one, u = ab_first[ab] + t, holding the
// distances 1 .. nA/2 inside the block.  Every unit costs 16 pair steps per lane.
// A GPU owns a contiguous, cost-balanced range of units (agent-pair ranges of the upper
// triangle x all samples), each CTA a contiguous sub-range, each warp every NW-th unit of it.
//
// Per iteration (two GPU-wide barriers, plus one system-wide exchange when G > 1):
//   R phase  warp = one (agent j, axis) row: R_j = sum_t q_j(t) P[t,:] from the unit slots of
//            this GPU (fixed order: t by lane, block pairs ascending, butterfly over lanes),
//            [G > 1: publish R_g to peers, system barrier, sum the G partials in rank order],
//            convergence test on the previous pass's norms, structured solve
//            c_j = rho G R_j + F (beq_j - beqbar) + Fm beqbar (kkt.py; no obstacles),
//            boundary rows, and the positions X[t][axis][j] = P[t,:] c_j for every t.
//   -- grid barrier --
//   P phase  warp = units: positions from X, multipliers streamed HBM -> shared memory by 1-D
//            TMA bulk copies (a per-warp ring of NSLOT chunks, mbarrier completion), the pair
//            update (am_kernel.cuh pair math, FP64 or FP32), new multipliers stored straight
//            back to HBM, the unit's partial S'b rows to its slot in qbuf, norms per CTA.
//   -- grid barrier --
// Every sum has a fixed order: results are bitwise reproducible run to run, and identical on
// every GPU of a sharded solve.
#pragma once
#include "am_kernel.cuh"

namespace swarm {

constexpr int LG_NW = 16;          // warps per CTA (one CTA per SM)
constexpr int LG_NT = LG_NW * 32;
constexpr int LG_NSLOT = 3;        // multiplier chunks in flight per warp
constexpr int LG_UNIT_STEPS = 16;  // pair steps per unit
constexpr int LG_MAXB = 8;         // agent blocks (n <= 256)

struct LgParams {
  int n, m, nv, S, NB, nab, npad;  // npad = NB * 32 (row length of X)
  const double* P;                 // m x NVMAX
  const double* mats;              // S x StageMats<NVMAX>::SIZE
  const double* inv_rho;           // S
  const double* E;                 // 6 x NVMAX
  const int* ab_pair;              // nab x 2: (A, B), A <= B, ab-major
  const int* ab_first;             // nab + 1: first unit of each block pair (diagonal: m units, cross: 2m)
  // groups: the G GPUs of a pair-sharded solve (G = 1 otherwise).  One launch runs groups
  // [g_base, g_base + vgroups): one group on a real multi-GPU run, all G when the ranks are
  // emulated in one kernel on one GPU.  Each group has cpg CTAs.
  int G, g_base, vgroups, cpg;
  const int* u_range;              // G + 1: group g owns units [u_range[g], u_range[g+1])
  const int* cta_first;            // G x (cpg + 1): CTA c of group g owns [cta_first[g(cpg+1)+c], ...+1])
  const long long* lam_off;        // element offset of unit u's multiplier rows, index u - u_range[g_base]
  void* lam;                       // this launch's multipliers (double, or float in FP32 mode)
  double* qbuf;                    // 2 pass parities x all units: [2 sides][3 axes][32 lanes] partial S'b rows
  long long q_stride;              // doubles per parity of qbuf
  double* X;                       // per group: m x 3 x npad positions (stride x_stride)
  double* cbuf;                    // per group: 3 x n x NVMAX coefficients (stride c_stride)
  long long x_stride, c_stride;
  double* cta_nrm;                 // 2 pass parities x per CTA of the launch: (sum r^2, max |r|) of a P phase
  unsigned long long* bnd;         // per group (stride 16): 3 rotating iterations, boundary max bits
  unsigned* blk_ready;             // per group (stride LG_MAXB * 32): rows of each agent block published
  unsigned* gbar;                  // per group (stride 32): grid barrier {count, generation}
  double* xch[8];                  // per group g: 2 parities x (3 n NVMAX + 4) exchange doubles
  unsigned* sysbar;                // barrier over every group's CTAs (G > 1)
  int sys_scope;                   // 1: groups on different GPUs (peer memory, system-scope fences)
  const double* c0;                // 3 x n x nv
  const double* beq;               // 3 x n x 6
  const double* geom;              // agent l_xy, l_z
  double* c_out;                   // 3 x n x nv (written by group 0)
  double* hist;                    // 3 x max_iters
  int* iters;
  int* conv;
  int switch_every, max_iters;
  double tol;
  long long* tstamp;               // optional phase timers (SWARM_PHASE_TIMERS)
};

// This CTA's group and its group-local buffers.
struct LgCtx {
  int g, vg, cta, u_lo, u_hi, ufirst, ulast;
  double lxy, lz;
  double* X;
  double* cbuf;
  unsigned long long* bnd;
  unsigned* gbar;
  unsigned* rdy;      // the group's block-ready counters (stride 32)
  const double* nrm;  // the group's CTA norm slots (parity 0; parity 1 at + 2 * G * cpg)
};

__device__ __forceinline__ LgCtx lg_ctx(const LgParams& p) {
  LgCtx c;
  c.vg = blockIdx.x / p.cpg;
  c.g = p.g_base + c.vg;
  c.cta = blockIdx.x - c.vg * p.cpg;
  c.u_lo = p.u_range[c.g];
  c.u_hi = p.u_range[c.g + 1];
  c.ufirst = p.cta_first[c.g * (p.cpg + 1) + c.cta];
  c.ulast = p.cta_first[c.g * (p.cpg + 1) + c.cta + 1];
  c.X = p.X + c.vg * p.x_stride;
  c.cbuf = p.cbuf + c.vg * p.c_stride;
  c.bnd = p.bnd + c.vg * 16;
  c.gbar = p.gbar + c.vg * 32;
  c.nrm = p.cta_nrm + 2LL * c.vg * p.cpg;
  c.rdy = p.blk_ready + c.vg * LG_MAXB * 32;
  c.lxy = __ldg(p.geom);
  c.lz = __ldg(p.geom + 1);
  return c;
}

struct LgSmem {  // byte offsets into dynamic shared memory
  int ring, bar, xs, P, mat, blist, bbar, misc, rows, total;
};

// Launch-constant row indices of the R phase (ints at LgSmem::rows), filled once per launch so
// that no per-iteration loop divides by a run-time value: header r_lo, r_hi, nr, LG_NT / nr,
// LG_NT % nr; per thread its first (t, row) of the t-major (sample, row) loops as t << 16 | rl;
// per row rl of this CTA (r = r_lo + rl) its axis and agent as ax << 16 | j.
constexpr int LG_ROWS_MAX = 3 * 32 * LG_MAXB;  // 3 n rows at n = 256
constexpr int LG_RT_START = 8, LG_RT_ROW = LG_RT_START + LG_NT;

template <int NVMAX, bool F32>
__host__ __device__ inline LgSmem lg_smem(int m, int chunk_rows) {
  LgSmem s;
  const int esize = F32 ? 4 : 8;
  int o = 0;
  auto take = [&](int bytes) { const int r = o; o += (bytes + 15) & ~15; return r; };
  s.ring = take(LG_NW * LG_NSLOT * chunk_rows * 96 * esize);
  s.bar = take(LG_NW * LG_NSLOT * 8);
  s.xs = take(LG_NW * 96 * 8);
  s.P = take(m * NVMAX * 8);
  s.mat = take(StageMats<NVMAX>::SIZE * 8);
  // per-block slot lists | ab_first (nab + 1) | ab_pair (2 nab)
  s.blist = take(LG_MAXB * LG_MAXB * 4 + (LG_MAXB * (LG_MAXB + 1) / 2 + 1) * 4 + LG_MAXB * (LG_MAXB + 1) * 4);
  s.bbar = take(18 * 8);
  s.misc = take(8 * 8 + LG_MAXB * 4);  // broadcast words + per-block seen epochs
  s.rows = take((LG_RT_ROW + LG_ROWS_MAX) * 4);  // R-phase row indices (see LG_RT_*)
  s.total = o;
  return s;
}

__host__ __device__ inline int lg_chunk_rows(bool f32) { return f32 ? 8 : 4; }

// ---- TMA bulk copy + mbarrier primitives
__device__ __forceinline__ unsigned lg_smem_u32(const void* ptr) {
  return static_cast<unsigned>(__cvta_generic_to_shared(ptr));
}
__device__ __forceinline__ void lg_mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(lg_smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ bool lg_mbar_try(unsigned long long* b, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred P1;\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n selp.u32 %0, 1, 0, P1;\n}"
      : "=r"(ok)
      : "r"(lg_smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
// bounded: a transfer that never lands (a bug) ends in a kernel error, not a hung device
__device__ __forceinline__ void lg_mbar_wait(unsigned long long* b, unsigned parity) {
  if (lg_mbar_try(b, parity)) return;
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (unsigned it = 1; !lg_mbar_try(b, parity); ++it) {
    if ((it & 1023u) == 0) {
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 10000000000ull) __trap();
    }
  }
}
// L2 policy of the multiplier stream: FP64 multipliers (n = 256: 157 MB) cannot stay in the
// 126 MB L2 and are streamed evict-first so the unit slots and positions stay resident; FP32
// multipliers (78 MB) fit and are kept (evict-last, plus the host's persisting window).
template <bool KEEP_L2>
__device__ __forceinline__ unsigned long long lg_policy() {
  unsigned long long pol;
  if (KEEP_L2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  else asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void lg_bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* b,
                                             unsigned long long pol) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(lg_smem_u32(b)), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          lg_smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(lg_smem_u32(b)), "l"(pol)
      : "memory");
}
// multiplier write-back with the same L2 policy
__device__ __forceinline__ void lg_store(double* a, double v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void lg_store(float* a, float v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(a), "f"(v), "l"(pol) : "memory");
}

// One warp's multiplier stream over its units of one P phase: chunk c (rows [c_row0, +CH) of
// some unit) lands in ring slot c % NSLOT; NSLOT - 1 chunks are in flight ahead of the one
// being consumed.  Lane 0 issues; every lane waits on the slot's mbarrier.
template <class T>
struct LgStream {
  T* ring;                  // NSLOT x CH x 96
  unsigned long long* bar;  // NSLOT
  const T* lam;             // this GPU's multipliers
  const long long* off;     // unit -> element offset (index u - u_lo)
  int u_lo, first, stride, end;  // the warp's units: first, first + stride, ... < end
  int CH;
  unsigned long long pol;   // L2 cache policy of the loads
  unsigned parity;          // expected phase bit per slot
  // issue cursor
  int iu, ic, issued;
  bool active;              // false: no loads (lambda = 0 on the first pass)

  __device__ __forceinline__ int unit_rows(int u) const { return (int)(off[u - u_lo + 1] - off[u - u_lo]) / 96; }

  __device__ __forceinline__ void issue_next(int lane) {
    while (iu < end) {
      const int rows = unit_rows(iu);
      if (ic * CH < rows) break;
      iu += stride;
      ic = 0;
    }
    if (iu >= end) return;
    const int rows = unit_rows(iu);
    const int r0 = ic * CH, nr = min(CH, rows - r0);
    const int sl = issued % LG_NSLOT;
    if (lane == 0) lg_bulk_load(ring + sl * CH * 96, lam + off[iu - u_lo] + (long long)r0 * 96, nr * 96 * sizeof(T),
                                bar + sl, pol);
    ++issued;
    ++ic;
  }
  __device__ __forceinline__ void begin(int lane) {
    iu = first; ic = 0; issued = 0;
    if (!active) return;
    for (int k = 0; k < LG_NSLOT; ++k) issue_next(lane);
  }
  // chunk number `seq` (in consumption order) is needed: wait for it
  __device__ __forceinline__ T* wait(int seq) {
    const int sl = seq % LG_NSLOT;
    lg_mbar_wait(bar + sl, (parity >> sl) & 1u);
    parity ^= 1u << sl;
    return ring + sl * CH * 96;
  }
  // chunk `seq` fully consumed: its slot takes the next chunk
  __device__ __forceinline__ void release(int lane) {
    __syncwarp();
    issue_next(lane);
  }
};

// Pair steps [s_lo, s_hi) of one unit for lane a.  Cross (A < B): partner (a + s) & 31 of
// block B, diagonal: partner (a + s) mod nA of block A, distances s >= 1.  xo = own position,
// xs = partner-block positions (per-warp shared scratch).  lam rows come from `row(j)`
// (j = step index within the unit); new multipliers go to `gl(j)` in HBM.
template <bool INIT, bool SPHERE, bool F32, bool DIAG, class RowF, class GlF>
__device__ __forceinline__ void lg_steps(int s_lo, int s_hi, int row0, int a, int nA, int nB, const double (&xo)[3],
                                         const double* xs, const Geo& ga, const GeoT<typename std::conditional<F32, float, double>::type>& gr,
                                         const StepConst& sc, const StepConstT<typename std::conditional<F32, float, double>::type>& sr,
                                         typename std::conditional<F32, float, double>::type c1, bool lam_zero,
                                         RowF row, GlF gl, double (&acc)[3], double (&accp)[3],
                                         typename std::conditional<F32, float, double>::type& sumsq,
                                         typename std::conditional<F32, float, double>::type& rmax,
                                         typename std::conditional<F32, float, double>::type& sumsq2,
                                         typename std::conditional<F32, float, double>::type& rmax2,
                                         unsigned long long pol) {
  using R = typename std::conditional<F32, float, double>::type;
  const int lane = a;
  const bool full_block = DIAG ? (nA == 32) : (nA == 32 && nB == 32);
  for (int s = s_lo; s < s_hi; s += 2) {
    const bool two = s + 1 < s_hi;  // warp-uniform
    const int j0 = s - s_lo + row0;
    int b0, b1;
    if (DIAG) {
      b0 = a + s; if (b0 >= nA) b0 -= nA;
      b1 = a + s + 1; if (b1 >= nA) b1 -= nA;
      if (a >= nA) { b0 = a; b1 = a; }
    } else {
      b0 = (a + s) & 31;
      b1 = (a + s + 1) & 31;
    }
    const bool act0 = DIAG ? (a < nA && (2 * s != nA || a < s)) : (a < nA && b0 < nB);
    const bool act1 = two && (DIAG ? (a < nA && (2 * (s + 1) != nA || a < s + 1)) : (a < nA && b1 < nB));
    R d0x = 1, d0y = 1, d0z = 1, d1x = 1, d1y = 1, d1z = 1;
    if (act0) { d0x = (R)(xo[0] - xs[b0]); d0y = (R)(xo[1] - xs[32 + b0]); d0z = (R)(xo[2] - xs[64 + b0]); }
    if (act1) { d1x = (R)(xo[0] - xs[b1]); d1y = (R)(xo[1] - xs[32 + b1]); d1z = (R)(xo[2] - xs[64 + b1]); }
    // multiplier triples: from the streamed chunk (or zero on the first pass)
    R l0[3], l1[3];
    R* r0 = INIT ? nullptr : row(j0);
    R* r1 = INIT ? nullptr : row(two ? j0 + 1 : j0);
    for (int ax = 0; ax < 3; ++ax) {
      l0[ax] = (INIT || lam_zero) ? R(0) : r0[ax * 32];
      l1[ax] = (INIT || lam_zero) ? R(0) : r1[ax * 32];
    }
    R w0x, w0y, w0z, w1x, w1y, w1z, dv0 = 1, dv1 = 1;
    const bool slow = __any_sync(0xffffffffu, any_zero3(d0x, d0y, d0z) | any_zero3(d1x, d1y, d1z));
    // both pairs real on every lane: no diameter step, full blocks
    const bool full = !INIT && full_block && two && (!DIAG || 2 * (s + 1) < nA);
    if (full && !slow) {
      pair2_full<SPHERE, R, 1>(d0x, d0y, d0z, d1x, d1y, d1z, gr, sr, c1, l0, l1, w0x, w0y, w0z, w1x, w1y, w1z, sumsq,
                               rmax, sumsq2, rmax2);
    } else if (!slow) {
      pair_fast<INIT, SPHERE, R, 1>(d0x, d0y, d0z, gr, act0, sr, c1, l0, w0x, w0y, w0z, sumsq, rmax, dv0);
      pair_fast<INIT, SPHERE, R, 1>(d1x, d1y, d1z, gr, act1, sr, c1, l1, w1x, w1y, w1z, sumsq2, rmax2, dv1);
    } else {
      w0x = w0y = w0z = w1x = w1y = w1z = 0;
      const bool flip0 = DIAG && b0 < a, flip1 = DIAG && b1 < a;
      if (act0)
        slow_pair<INIT, false, R, 1>(d0x, d0y, d0z, ga, flip0, 0.0, 0.0, 0.0, sc, l0, w0x, w0y, w0z, sumsq, rmax, dv0);
      if (act1)
        slow_pair<INIT, false, R, 1>(d1x, d1y, d1z, ga, flip1, 0.0, 0.0, 0.0, sc, l1, w1x, w1y, w1z, sumsq2, rmax2,
                                     dv1);
    }
    if (!INIT) {
      if (act0) { R* g = gl(j0); lg_store(g, l0[0], pol); lg_store(g + 32, l0[1], pol); lg_store(g + 64, l0[2], pol); }
      if (act1) {
        R* g = gl(j0 + 1);
        lg_store(g, l1[0], pol); lg_store(g + 32, l1[1], pol); lg_store(g + 64, l1[2], pol);
      }
    }
    // own +w; the partner's -w comes back from the lane that paired with this lane
    int src0, src1;
    if (DIAG) {
      src0 = a - s; if (src0 < 0) src0 += nA;
      src1 = a - s - 1; if (src1 < 0) src1 += nA;
      if (a >= nA) { src0 = a; src1 = a; }
    } else {
      src0 = (lane - s) & 31;
      src1 = (lane - s - 1) & 31;
    }
    const R q0x = __shfl_sync(0xffffffffu, w0x, src0);
    const R q0y = __shfl_sync(0xffffffffu, w0y, src0);
    const R q0z = __shfl_sync(0xffffffffu, w0z, src0);
    const R q1x = __shfl_sync(0xffffffffu, w1x, src1);
    const R q1y = __shfl_sync(0xffffffffu, w1y, src1);
    const R q1z = __shfl_sync(0xffffffffu, w1z, src1);
    if (DIAG) {
      acc2(acc[0], w0x, q0x, w1x, q1x);
      acc2(acc[1], w0y, q0y, w1y, q1y);
      acc2(acc[2], w0z, q0z, w1z, q1z);
    } else {
      acc2x(acc[0], accp[0], w0x, q0x, w1x, q1x);
      acc2x(acc[1], accp[1], w0y, q0y, w1y, q1y);
      acc2x(acc[2], accp[2], w0z, q0z, w1z, q1z);
    }
  }
}

// P phase of one CTA: its units, NW warps, multipliers streamed per warp.
// Wait until agent block b's rows of epoch `epoch` are published (positions X of the last R
// phase): lane 0 polls the block's counter (acquire) once per block and epoch per CTA.
__device__ __forceinline__ void lg_wait_block(const LgParams& p, const LgCtx& cx, int* seen, int b, int epoch) {
  if (((volatile int*)seen)[b] >= epoch) return;
  const int lane = threadIdx.x & 31;
  if (lane == 0) {
    const unsigned nb = (unsigned)min(32, p.n - 32 * b);
    const unsigned target = 3u * nb * (unsigned)epoch;
    const unsigned* c = cx.rdy + b * 32;
    unsigned v;
    unsigned long long t0 = 0, t;
    for (unsigned it = 0;; ++it) {
      asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
      if (v >= target) break;
      if ((it & 1023u) == 0) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (it == 0) t0 = t;
        else if (t - t0 > 30000000000ull) __trap();
      }
    }
    ((volatile int*)seen)[b] = epoch;
  }
  __syncwarp();
}

template <int NVMAX, bool INIT, bool SPHERE, bool F32>
__device__ __forceinline__ void lg_pair_phase(const LgParams& p, const LgCtx& cx, unsigned char* smb, const LgSmem& L,
                                              bool lam_zero, const StepConst& sc, unsigned& par_bits, int pass) {
  using R = typename std::conditional<F32, float, double>::type;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int CH = lg_chunk_rows(F32);
  const int u0 = cx.ufirst, u1 = cx.ulast;
  const int ubase = p.u_range[p.g_base];  // lam_off index base of this launch
  Geo ga;
  ga.lxy = cx.lxy; ga.lz = cx.lz; ga.ilxy = 1.0 / cx.lxy; ga.ilz = 1.0 / cx.lz; ga.lxy2 = cx.lxy * cx.lxy;
  ga.lz2 = cx.lz * cx.lz; ga.sphere = SPHERE;
  GeoT<R> gr;
  gr.lxy = (R)ga.lxy; gr.lz = (R)ga.lz; gr.ilxy = (R)ga.ilxy; gr.ilz = (R)ga.ilz; gr.lxy2 = (R)ga.lxy2;
  gr.lz2 = (R)ga.lz2; gr.sphere = SPHERE;
  StepConstT<R> sr;
  sr.rho = (R)sc.rho; sr.inv_rho = (R)sc.inv_rho; sr.inv_rho_next = (R)sc.inv_rho_next;
  const R c1 = (R)(sc.inv_rho * ga.ilxy);
  double* xs = reinterpret_cast<double*>(smb + L.xs) + warp * 96;
  R* const lam = static_cast<R*>(p.lam);

  LgStream<R> st;
  st.ring = reinterpret_cast<R*>(smb + L.ring) + (long long)warp * LG_NSLOT * CH * 96;
  st.bar = reinterpret_cast<unsigned long long*>(smb + L.bar) + warp * LG_NSLOT;
  st.lam = lam;
  st.off = p.lam_off;
  st.u_lo = ubase;
  st.first = u0 + warp;
  st.stride = LG_NW;
  st.end = u1;
  st.CH = CH;
  st.pol = lg_policy<F32>();
  st.parity = par_bits;
  st.active = !INIT && !lam_zero;
  st.begin(lane);
  int seq = 0;

  R sumsq = 0, rmax = 0, sumsq2 = 0, rmax2 = 0;
  const int* abf = reinterpret_cast<const int*>(smb + L.blist) + LG_MAXB * LG_MAXB;  // ab_first in smem
  for (int u = u0 + warp; u < u1; u += LG_NW) {
    int ab = 0;
    while (abf[ab + 1] <= u) ++ab;
    const int* abp = abf + LG_MAXB * (LG_MAXB + 1) / 2 + 1;  // ab_pair in smem (one L2 trip less per unit)
    const int A = abp[2 * ab], B = abp[2 * ab + 1];
    const bool diag = A == B;
    const int lu = u - abf[ab];
    const int t = diag ? lu : (lu >> 1), h = diag ? 0 : (lu & 1);
    const int nA = min(32, p.n - 32 * A), nB = min(32, p.n - 32 * B);
    const long long uoff = p.lam_off[u - ubase];
    const int nrow = (int)(p.lam_off[u - ubase + 1] - uoff) / 96;
    if (nrow == 0) continue;  // a diagonal block of one agent
    // positions of this pass: published by the R phase (epoch = pass + 1: the initial positions
    // are epoch 1)
    int* seen = reinterpret_cast<int*>(smb + L.misc) + 8;
    lg_wait_block(p, cx, seen, A, pass + 1);
    if (!diag) lg_wait_block(p, cx, seen, B, pass + 1);
    const double* Xt = cx.X + (long long)t * 3 * p.npad;
    double xo[3];
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) xo[ax] = (lane < nA) ? __ldcg(Xt + ax * p.npad + 32 * A + lane) : 0.0;
    __syncwarp();
#pragma unroll
    for (int ax = 0; ax < 3; ++ax)
      xs[ax * 32 + lane] = diag ? xo[ax] : ((lane < nB) ? __ldcg(Xt + ax * p.npad + 32 * B + lane) : 0.0);
    __syncwarp();
    double acc[3] = {0.0, 0.0, 0.0}, accp[3] = {0.0, 0.0, 0.0};
    R* const gunit = lam + uoff + lane;
    auto gl = [&](int j) -> R* { return gunit + j * 96; };
    const int s_base = diag ? 1 : 16 * h;
    // chunk loop: rows [r0, r0 + CH) of the unit; the step pairs never straddle a chunk (CH even)
    for (int r0 = 0; r0 < nrow; r0 += CH) {
      const int nr = min(CH, nrow - r0);
      R* chunk = nullptr;
      if (st.active) chunk = st.wait(seq);
      R* const cl = chunk ? chunk + lane - r0 * 96 : nullptr;
      auto row = [&](int j) -> R* { return cl + j * 96; };
      if (diag)
        lg_steps<INIT, SPHERE, F32, true>(s_base + r0, s_base + r0 + nr, r0, lane, nA, nB, xo, xs, ga, gr, sc, sr, c1,
                                          !st.active, row, gl, acc, accp, sumsq, rmax, sumsq2, rmax2, st.pol);
      else
        lg_steps<INIT, SPHERE, F32, false>(s_base + r0, s_base + r0 + nr, r0, lane, nA, nB, xo, xs, ga, gr, sc, sr,
                                           c1, !st.active, row, gl, acc, accp, sumsq, rmax, sumsq2, rmax2, st.pol);
      if (st.active) {
        ++seq;
        st.release(lane);
      }
    }
    double* q = p.qbuf + (pass & 1) * p.q_stride + (long long)u * 192;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      q[ax * 32 + lane] = lane < nA ? acc[ax] : 0.0;
      if (!diag) q[96 + ax * 32 + lane] = lane < nB ? accp[ax] : 0.0;
    }
  }
  par_bits = st.parity;
  if (!INIT) {
    double s2 = (double)sumsq, mxd = (double)max_nn(rmax, rmax2);
    s2 += (double)sumsq2;
    warp_sum_max(s2, mxd);
    __shared__ double wslot[LG_NW * 2];
    if (lane == 0) { wslot[2 * warp] = s2; wslot[2 * warp + 1] = mxd; }
    __syncthreads();
    if (threadIdx.x < 32) {
      double a2 = lane < LG_NW ? wslot[2 * lane] : 0.0, am = lane < LG_NW ? wslot[2 * lane + 1] : 0.0;
      warp_sum_max(a2, am);
      if (lane == 0) {
        double* slot = p.cta_nrm + (pass & 1) * 2LL * p.vgroups * p.cpg + 2 * blockIdx.x;
        slot[0] = a2;
        slot[1] = am;
      }
    }
  }
}

// Lane-parallel reduction of a group's CTA norm slots (fixed order, identical in every CTA).
__device__ __forceinline__ void lg_norms(const double* slots, int count, double& s2, double& mx) {
  const int lane = threadIdx.x & 31;
  double a = 0.0, b = 0.0;
  // every slot load in flight at once (one L2 round trip, not one per 32 slots), then the same
  // lane-ordered sums
  constexpr int U = 8;  // 256 slots: every CTA of a launch
  double va[U], vb[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int i = lane + 32 * u;
    va[u] = i < count ? __ldcg(slots + 2 * i) : 0.0;
    vb[u] = i < count ? __ldcg(slots + 2 * i + 1) : 0.0;
  }
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (lane + 32 * u < count) {
      a += va[u];
      b = fmax(b, vb[u]);
    }
  for (int i = lane + 32 * U; i < count; i += 32) {
    a += __ldcg(slots + 2 * i);
    b = fmax(b, __ldcg(slots + 2 * i + 1));
  }
  warp_sum_max(a, b);
  s2 = a;
  mx = b;
}

// R phase: CTA c of the group owns the rows r = ax * n + j in [c R / cpg, (c+1) R / cpg),
// R = 3n.  mode 0: initial positions from c0; mode 1: reduce the group's unit slots and solve
// (G == 1); mode 2: reduce and publish the partial row (G > 1); mode 3: sum the G published
// partials in rank order and solve (G > 1, after the exchange).  Every step uses the whole CTA:
//   1. thread = (row, t): q_j(t) = sum of the row's unit slots at t, block pairs ascending, into
//      shared memory (all slot loads in flight at once; the multiplier ring is idle here);
//   2. R (rows x NVMAX) = q (rows x m) P (m x NVMAX) as FP64 tensor-core tiles (DMMA), the k
//      steps (samples) split over the warps, the warp partials added in warp order;
//   3. thread = (row, coefficient): c_j = rho G R_j + F (beq_j - beqbar) + Fm beqbar (kkt.py, no
//      obstacles: Rbar = 0); then thread = (row, endpoint row): |E c_j - beq_j| (order-free max);
//   4. thread = (row, t): positions X[t][ax][j] = P[t,:] c_j (k-ascending FMA chain).
// A fixed order everywhere: bitwise reproducible, and identical on every GPU of a sharded solve.
template <int NVMAX>
__device__ __forceinline__ void lg_rows(const LgParams& p, const LgCtx& cx, unsigned char* smb, const LgSmem& L, int k,
                                        int mode, long long* tsr = nullptr) {
  using SM = StageMats<NVMAX>;
  constexpr int NH = (NVMAX + 7) / 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* Ps = reinterpret_cast<const double*>(smb + L.P);
  const double* mat = reinterpret_cast<const double*>(smb + L.mat);
  const int* blist = reinterpret_cast<const int*>(smb + L.blist);
  const double* bbar = reinterpret_cast<const double*>(smb + L.bbar);
  const int n = p.n, m = p.m;
  const int* rt = reinterpret_cast<const int*>(smb + L.rows);
  const int r_lo = rt[0], nr = rt[2], dt = rt[3], drl = rt[4];
  const int* rowt = rt + LG_RT_ROW;  // ax << 16 | j per row of this CTA
  const int start = rt[LG_RT_START + threadIdx.x];
  const int mt_n = (nr + 7) >> 3, rp = mt_n * 8;  // row tiles of the projection
  const long long xstride = 3LL * n * NVMAX + 4;
  // scratch in the multiplier ring (idle in this phase): q rows | warp partials | R | c
  double* qs = reinterpret_cast<double*>(smb + L.ring);  // nr x m (stride m)
  double* part = qs + (size_t)rp * m;                     // LG_NW x rp x (NH * 8)
  double* Rr = part + (size_t)LG_NW * rp * NH * 8;        // nr x NVMAX
  double* cr = Rr + (size_t)rp * NVMAX;                   // nr x NVMAX
  if (mode == 1 || mode == 2) {
    int t = start >> 16, rl = start & 0xffff;  // idx = t * nr + rl, stepped without division
    for (int idx = threadIdx.x; idx < nr * m; idx += LG_NT) {
      // consecutive threads: consecutive rows (agents) at one t -> the slot loads coalesce
      double qv = 0.0;
      {
        const int axj = rowt[rl];
        const int ax = axj >> 16, j = axj & 0xffff;
        const int b = j >> 5, l = j & 31;
        const double* qb = p.qbuf + (k & 1) * p.q_stride + ax * 32 + l;  // written by pass k
        double v[2 * LG_MAXB];
#pragma unroll
        for (int e = 0; e < LG_MAXB; ++e) {
          const int ent = blist[b * LG_MAXB + e];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const bool dg = (ent & 2) != 0;
            const int u = (ent >> 2) + (dg ? t : 2 * t + h);
            const bool ok = ent >= 0 && !(h == 1 && dg) && u >= cx.u_lo && u < cx.u_hi;
            v[2 * e + h] = ok ? __ldcg(qb + (long long)u * 192 + (ent & 1) * 96) : 0.0;
          }
        }
#pragma unroll
        for (int e = 0; e < 2 * LG_MAXB; ++e) qv += v[e];
      }
      qs[rl * m + t] = qv;
      t += dt;
      rl += drl;
      if (rl >= nr) {
        rl -= nr;
        ++t;
      }
    }
    __syncthreads();
    stamp(tsr, 8);
    // 2. projection: warp w takes the k-steps w, w + LG_NW, ... of every row tile
    {
      const int g = lane >> 2, q = lane & 3;
      const int ksn = (m + 3) >> 2;
      for (int mt = 0; mt < mt_n; ++mt) {
        double acc[NH][2];
#pragma unroll
        for (int h = 0; h < NH; ++h) acc[h][0] = acc[h][1] = 0.0;
        for (int ks = warp; ks < ksn; ks += LG_NW) {
          const int t = ks * 4 + q;
          const double a = (t < m && mt * 8 + g < nr) ? qs[(mt * 8 + g) * m + t] : 0.0;
#pragma unroll
          for (int h = 0; h < NH; ++h) {
            const int kk = h * 8 + g;
            const double bv = (t < m && kk < NVMAX) ? Ps[t * NVMAX + kk] : 0.0;
            dmma884(acc[h][0], acc[h][1], a, bv);
          }
        }
        double* pw = part + ((size_t)warp * rp + mt * 8 + g) * (NH * 8);
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          pw[h * 8 + 2 * q] = acc[h][0];
          pw[h * 8 + 2 * q + 1] = acc[h][1];
        }
      }
      __syncthreads();
      for (int idx = threadIdx.x; idx < nr * NVMAX; idx += LG_NT) {
        const int rl = idx / NVMAX, kk = idx - rl * NVMAX;
        double v = 0.0;
        for (int w = 0; w < LG_NW; ++w) v += part[((size_t)w * rp + rl) * (NH * 8) + kk];
        Rr[idx] = v;
      }
    }
    __syncthreads();
    stamp(tsr, 9);
    if (mode == 2) {
      for (int idx = threadIdx.x; idx < nr * NVMAX; idx += LG_NT)
        p.xch[cx.g][(k & 1) * xstride + (long long)r_lo * NVMAX + idx] = Rr[idx];
    }
  } else if (mode == 3) {
    for (int idx = threadIdx.x; idx < nr * NVMAX; idx += LG_NT) {
      double v = 0.0;
      for (int g = 0; g < p.G; ++g) {
        const double* src = p.xch[g] + (k & 1) * xstride + (long long)r_lo * NVMAX + idx;
        v += p.sys_scope ? __ldcv(src) : __ldcg(src);
      }
      Rr[idx] = v;
    }
    __syncthreads();
  }
  if (mode != 2) {
    // 3. coefficients (mode 0: the straight lines, solver.py:327-330, packed on the host)
    const double rho = mat[SM::RHO];
    for (int idx = threadIdx.x; idx < nr * NVMAX; idx += LG_NT) {
      const int rl = idx / NVMAX, qo = idx - rl * NVMAX;
      const int axj = rowt[rl];
      const int ax = axj >> 16, j = axj & 0xffff;
      double cv;
      if (mode == 0) {
        cv = qo < p.nv ? p.c0[((long long)ax * n + j) * p.nv + qo] : 0.0;
      } else {
        const double* bj = p.beq + ((long long)ax * n + j) * 6;
        double s1 = 0.0, s3 = 0.0, s4 = 0.0;
#pragma unroll
        for (int i = 0; i < NVMAX; ++i) s1 = fma(mat[SM::G + qo * NVMAX + i], Rr[rl * NVMAX + i], s1);
#pragma unroll
        for (int e = 0; e < 6; ++e) {
          const double bm = bbar[ax * 6 + e];
          s3 = fma(mat[SM::F + qo * 6 + e], __ldg(bj + e) - bm, s3);
          s4 = fma(mat[SM::Fm + qo * 6 + e], bm, s4);
        }
        cv = rho * s1 + (s3 + s4);
      }
      cr[idx] = cv;
      cx.cbuf[((long long)ax * n + j) * NVMAX + qo] = cv;
    }
    __syncthreads();
    if (mode != 0) {
      // boundary rows E c_j - beq_j (solver.py:448-452)
      double bmx = 0.0;
      for (int idx = threadIdx.x; idx < nr * 6; idx += LG_NT) {
        const int rl = idx / 6, e = idx - rl * 6;
        const int r = r_lo + rl;
        double v = 0.0;
#pragma unroll
        for (int i = 0; i < NVMAX; ++i) v = fma(p.E[e * NVMAX + i], cr[rl * NVMAX + i], v);
        bmx = fmax(bmx, fabs(v - __ldg(p.beq + (long long)r * 6 + e)));
      }
      bmx = warp_max(bmx);
      if (lane == 0 && bmx > 0.0) atomicMax(cx.bnd + (k % 3), (unsigned long long)__double_as_longlong(bmx));
    }
    // 4. positions
    int t = start >> 16, rl = start & 0xffff;
    for (int idx = threadIdx.x; idx < nr * m; idx += LG_NT) {
      const int axj = rowt[rl];
      const int ax = axj >> 16, j = axj & 0xffff;
      const double* pr = Ps + t * NVMAX;
      const double* cj = cr + rl * NVMAX;
      double v = 0.0;
#pragma unroll
      for (int q = 0; q < NVMAX; ++q) v = fma(pr[q], cj[q], v);
      cx.X[((long long)t * 3 + ax) * p.npad + j] = v;
      t += dt;
      rl += drl;
      if (rl >= nr) {
        rl -= nr;
        ++t;
      }
    }
    stamp(tsr, 10);
  }
  // the scratch (generic-proxy writes/reads) lives in the ring the next P phase fills by TMA
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (mode != 2 && threadIdx.x == 0 && nr > 0) {
    // publish: this CTA's rows of each agent block are in X (release after the CTA barrier)
    int cnt[LG_MAXB];
#pragma unroll
    for (int b = 0; b < LG_MAXB; ++b) cnt[b] = 0;
    for (int rl = 0; rl < nr; ++rl) cnt[(rowt[rl] & 0xffff) >> 5]++;
    __threadfence();
#pragma unroll
    for (int b = 0; b < LG_MAXB; ++b)
      if (cnt[b]) atomicAdd(cx.rdy + b * 32, (unsigned)cnt[b]);
  }
}

template <int NVMAX, bool F32>
__global__ void __launch_bounds__(LG_NT, 1) am_large_kernel(const LgParams p)
#ifdef SWARM_KERNEL_DECL_ONLY
    ;
#else
{
  using SM = StageMats<NVMAX>;
  extern __shared__ __align__(16) unsigned char smb[];
  const LgSmem L = lg_smem<NVMAX, F32>(p.m, lg_chunk_rows(F32));
  const LgCtx cx = lg_ctx(p);
  const int lane = threadIdx.x & 31;
  const int n = p.n;
  const unsigned ncta_sys = (unsigned)(p.G * p.cpg);  // every group's CTAs (sys barrier)
  const bool sys = p.sys_scope != 0;
  // setup: mbarriers, basis rows, block -> (block pair, side) lists, mean boundary rows
  if (lane == 0) {
    unsigned long long* b = reinterpret_cast<unsigned long long*>(smb + L.bar) + (threadIdx.x >> 5) * LG_NSLOT;
    for (int i = 0; i < LG_NSLOT; ++i) lg_mbar_init(b + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  double* Ps = reinterpret_cast<double*>(smb + L.P);
  for (int i = threadIdx.x; i < p.m * NVMAX; i += LG_NT) Ps[i] = p.P[i];
  // per agent block b: the (block pair, side) slots holding its rows, ab ascending, as
  // (first unit of the block pair) << 2 | diagonal << 1 | side; -1 ends the list
  int* blist = reinterpret_cast<int*>(smb + L.blist);
  if (threadIdx.x < p.NB) {
    const int b = threadIdx.x;
    int e = 0;
    for (int ab = 0; ab < p.nab; ++ab) {
      const int A = p.ab_pair[2 * ab], B = p.ab_pair[2 * ab + 1];
      const int u0 = p.ab_first[ab];
      if (A == b) blist[b * LG_MAXB + e++] = (u0 << 2) | ((A == B) ? 2 : 0);
      else if (B == b) blist[b * LG_MAXB + e++] = (u0 << 2) | 1;
    }
    for (; e < LG_MAXB; ++e) blist[b * LG_MAXB + e] = -1;
  }
  for (int i = threadIdx.x; i <= p.nab; i += LG_NT) blist[LG_MAXB * LG_MAXB + i] = p.ab_first[i];
  for (int i = threadIdx.x; i < 2 * p.nab; i += LG_NT)
    blist[LG_MAXB * LG_MAXB + LG_MAXB * (LG_MAXB + 1) / 2 + 1 + i] = p.ab_pair[i];
  double* bbar = reinterpret_cast<double*>(smb + L.bbar);
  if (threadIdx.x < 18) {
    const int ax = threadIdx.x / 6, e = threadIdx.x - 6 * ax;
    double s = 0.0;
    for (int j = 0; j < n; ++j) s += p.beq[((long long)ax * n + j) * 6 + e];
    bbar[threadIdx.x] = s / n;
  }
  {
    // R-phase row indices of this CTA (LG_RT_*), once per launch
    int* rt = reinterpret_cast<int*>(smb + L.rows);
    const int R3 = 3 * n;
    const int r_lo = (int)((long long)cx.cta * R3 / p.cpg), r_hi = (int)((long long)(cx.cta + 1) * R3 / p.cpg);
    const int nr = r_hi - r_lo;
    if (threadIdx.x == 0) {
      rt[0] = r_lo;
      rt[1] = r_hi;
      rt[2] = nr;
      rt[3] = nr ? LG_NT / nr : 0;
      rt[4] = nr ? LG_NT % nr : 0;
    }
    rt[LG_RT_START + threadIdx.x] = nr ? ((int)(threadIdx.x / nr) << 16) | (int)(threadIdx.x % nr) : 0;
    for (int rl = threadIdx.x; rl < nr; rl += LG_NT) {
      const int r = r_lo + rl;
      rt[LG_RT_ROW + rl] = ((r / n) << 16) | (r % n);
    }
  }
  double* misc = reinterpret_cast<double*>(smb + L.misc);
  __syncthreads();
  const bool sphere = cx.lxy == cx.lz;
  unsigned par_bits = 0;
  StepConst sc;
  sc.rho = 0.0; sc.inv_rho = 0.0; sc.inv_rho_next = 0.0;
  long long* ts = (p.tstamp && blockIdx.x == 0 && p.g_base == 0 && threadIdx.x == 0) ? p.tstamp : nullptr;

  // initialization: positions of the straight lines, then the INIT pair pass (solver.py:309-352)
  if (threadIdx.x < LG_MAXB) reinterpret_cast<int*>(smb + L.misc)[8 + threadIdx.x] = 0;  // seen epochs
  __syncthreads();
  lg_rows<NVMAX>(p, cx, smb, L, 0, 0);
  if (sphere) lg_pair_phase<NVMAX, true, true, F32>(p, cx, smb, L, true, sc, par_bits, 0);
  else lg_pair_phase<NVMAX, true, false, F32>(p, cx, smb, L, true, sc, par_bits, 0);
  if (cx.cta == 0 && threadIdx.x == 0) { cx.bnd[0] = 0ull; cx.bnd[1] = 0ull; cx.bnd[2] = 0ull; }
  grid_barrier(cx.gbar, p.cpg, false);

  int prev_stage = -1, iters = 0, conv = 0;
  const long long xstride = 3LL * n * NVMAX + 4;
  int st_q = 0, st_r = 0;  // k = st_q * switch_every + st_r, kept without a division
  for (int k = 0;; ++k) {
    long long* tsr = (ts && k < 256) ? ts + 16 * k : nullptr;
    stamp(tsr, 0);
    if (k > 0 && ++st_r == p.switch_every) {
      st_r = 0;
      ++st_q;
    }
    const int stage = min(st_q, p.S - 1);
    const int stage_n = min(st_q + (st_r + 1 == p.switch_every ? 1 : 0), p.S - 1);
    if (stage != prev_stage) {
      double* mat = reinterpret_cast<double*>(smb + L.mat);
      for (int i = threadIdx.x; i < SM::SIZE; i += LG_NT) mat[i] = p.mats[(long long)stage * SM::SIZE + i];
      prev_stage = stage;
    }
    // residual norms of the previous pass: the group's CTAs in fixed order (every CTA alike)
    double s2 = 0.0, mx = 0.0;
    if (k > 0 && threadIdx.x < 32) lg_norms(cx.nrm + (k & 1) * 2LL * p.vgroups * p.cpg, p.cpg, s2, mx);
    __syncthreads();  // the stage matrices are in place
    if (p.G > 1) {
      // this group's R rows -> its exchange buffer, norm totals alongside; meet every group
      lg_rows<NVMAX>(p, cx, smb, L, k, 2);
      if (cx.cta == 0 && threadIdx.x == 0) {
        double* mine = p.xch[cx.g] + (k & 1) * xstride + 3LL * n * NVMAX;
        mine[0] = s2;
        mine[1] = mx;
      }
      grid_barrier(p.sysbar, ncta_sys, sys);
      if (k > 0 && threadIdx.x < 32) {
        double a2 = 0.0, b2 = 0.0;
        for (int g = 0; g < p.G; ++g) {
          const double* t = p.xch[g] + (k & 1) * xstride + 3LL * n * NVMAX;
          a2 += sys ? __ldcv(t) : __ldcg(t);
          b2 = fmax(b2, sys ? __ldcv(t + 1) : __ldcg(t + 1));
        }
        s2 = a2;
        mx = b2;
      }
    }
    if (threadIdx.x == 0) { misc[0] = s2; misc[1] = mx; }
    __syncthreads();
    s2 = misc[0];
    mx = misc[1];
    stamp(tsr, 1);
    if (k > 0) {
      // convergence test on iteration k-1 (solver.py:444-457), identical in every CTA / group
      const double bm = __longlong_as_double((long long)__ldcg(cx.bnd + ((k - 1) % 3)));
      if (cx.cta == 0 && cx.g == 0 && threadIdx.x == 0) {
        p.hist[k - 1] = sqrt(s2);
        p.hist[p.max_iters + k - 1] = mx;
        p.hist[2 * p.max_iters + k - 1] = bm;
      }
      if (!(s2 <= 1.7976931348623157e308)) { iters = k; conv = -1; break; }
      if (mx <= p.tol) { iters = k; conv = 1; break; }
      if (k == p.max_iters) { iters = k; break; }
    }
    // solve c_k (and its positions) from the right-hand sides of the last pass
    stamp(tsr, 7);
    lg_rows<NVMAX>(p, cx, smb, L, k, p.G > 1 ? 3 : 1, tsr);
    const double* mat = reinterpret_cast<const double*>(smb + L.mat);
    sc.rho = mat[SM::RHO];
    sc.inv_rho = mat[SM::RHO + 1];
    sc.inv_rho_next = p.inv_rho[stage_n];
    stamp(tsr, 2);
    // no grid barrier here: every unit waits for the published rows of its two agent blocks
    stamp(tsr, 3);
    long long tp0 = 0;
    if (p.tstamp && k == 50 && threadIdx.x == 0) tp0 = clock64();
    // bnd slot of iteration k+1 (last read by the test of iteration k-1, before the last barrier)
    if (cx.cta == 0 && threadIdx.x == 0) cx.bnd[(k + 1) % 3] = 0ull;
    if (sphere) lg_pair_phase<NVMAX, false, true, F32>(p, cx, smb, L, k == 0, sc, par_bits, k + 1);
    else lg_pair_phase<NVMAX, false, false, F32>(p, cx, smb, L, k == 0, sc, par_bits, k + 1);
    stamp(tsr, 4);
    if (p.tstamp && k == 50 && threadIdx.x == 0) p.tstamp[4096 + blockIdx.x] = clock64() - tp0;  // per-CTA P phase
    grid_barrier(cx.gbar, p.cpg, false);
    stamp(tsr, 5);
  }
  if (cx.cta == 0 && cx.g == 0) {
    for (int idx = threadIdx.x; idx < 3 * n * p.nv; idx += LG_NT) {
      const int q = idx % p.nv, row = idx / p.nv;
      p.c_out[idx] = __ldcg(cx.cbuf + (long long)row * NVMAX + q);
    }
    if (threadIdx.x == 0) {
      *p.iters = iters;
      *p.conv = conv;
    }
  }
}
#endif

}  // namespace swarm
