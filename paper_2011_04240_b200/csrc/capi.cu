// C ABI of the B200 AM solver (declared in include/swarm_am.h): plan upload,
// launch-configuration choice and the host/device solve entry points.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/swarm_am.h"
#define SWARM_KERNEL_DECL_ONLY
#include "am_kernel.cuh"
#include "am_large.cuh"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define ST_CUDA(call)                                                                          \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess) {                                                                   \
      return fail(e_ == cudaErrorMemoryAllocation ? ST_ENOMEM : ST_ECUDA,                     \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                         \
    }                                                                                          \
  } while (0)

using KernelFn = void (*)(swarm::KParams);

struct KernelEntry {
  int NB, NT, NVMAX, LAM;
  bool f32;  // FP32 pair state (multipliers and pair arithmetic in FP32, FP64 solve)
  bool obs_free;  // obstacle rows compiled out (scenarios without obstacles only)
  KernelFn fn;
};

using swarm::am_cluster_kernel;
constexpr int kS = swarm::LAM_SMEM, kG = swarm::LAM_GLOBAL, kK = swarm::LAM_GLOBAL_KEEP;
#define ST_K(NB, NT, NV, L, F) {NB, NT, NV, L, F, false, am_cluster_kernel<NB, NT, NV, L, F>}
#define ST_K0(NB, NT, NV, L, F) {NB, NT, NV, L, F, true, am_cluster_kernel<NB, NT, NV, L, F, false>}
// lambda fits in shared memory only for n <= 32 (NB == 1); larger fleets stream it from L2.
const KernelEntry kKernels[] = {
    // obstacle-free variants first (the batch bench and the common single solves)
    ST_K0(1, 512, 12, kS, false), ST_K0(1, 512, 12, kG, false),
    ST_K(1, 512, 12, kS, false), ST_K(1, 512, 12, kG, false), ST_K(1, 512, 12, kK, false),
    ST_K(1, 512, 16, kS, false), ST_K(1, 512, 16, kG, false), ST_K(1, 512, 16, kK, false),
    ST_K(2, 384, 12, kG, false), ST_K(2, 384, 12, kK, false), ST_K(2, 384, 16, kG, false),
    ST_K(2, 384, 16, kK, false), ST_K(4, 256, 12, kG, false), ST_K(4, 256, 12, kK, false),
    ST_K(8, 256, 12, kG, false), ST_K(8, 256, 12, kK, false),
    ST_K0(1, 512, 12, kS, true), ST_K0(1, 512, 12, kG, true),
    ST_K(1, 512, 12, kS, true),  ST_K(1, 512, 12, kG, true),  ST_K(1, 512, 12, kK, true),
    ST_K(1, 512, 16, kS, true),  ST_K(1, 512, 16, kG, true),  ST_K(1, 512, 16, kK, true),
    ST_K(2, 384, 12, kG, true),  ST_K(2, 384, 12, kK, true),  ST_K(2, 384, 16, kG, true),
    ST_K(2, 384, 16, kK, true),  ST_K(4, 256, 12, kG, true),  ST_K(4, 256, 12, kK, true),
    ST_K(8, 256, 12, kG, true),  ST_K(8, 256, 12, kK, true),
};
#undef ST_K
#undef ST_K0

struct Launch {
  int NVMAX = 0;
  int NB = 0, NT = 0, W = 0, C = 0, nsteps = 0, tmax = 0, tasks_max = 0, own_max = 0;
  int lam_smem = 0, nclusters = 0, c_global = 0, K = 1, lam_tail = 0;
  int G = 1;  // groups (GPUs) sharing the scenario; participants = G x K clusters
  int f32 = 0;    // FP32 pair state: multipliers are 4-byte elements
  int active = 0; // co-resident clusters of this shape
  size_t smem_bytes = 0;
  long long lam_per_cta = 0;
  KernelFn fn = nullptr;
  swarm::KParams kp{};
};

}  // namespace

// shared with collisions.cu
int swarm_fail(int code, const std::string& msg) { return fail(code, msg); }
// report.cu / collisions.cu: the device-side report pass of st_solve_report
size_t swarm_report_smem(int m);
cudaError_t swarm_report_launch(int B, int n, int m, int nv, int nvp, const double* c, const double* P, double* traj,
                                double* arc, double* smooth, unsigned long long* summary, cudaStream_t s);
cudaError_t swarm_collision_summary_launch(int B, int n, int m, const double* d_traj, const double* d_geom, int n_obs,
                                           const double* d_obs, int* row_cnt, unsigned long long* min_total,
                                           cudaStream_t s, bool init = true);

// outputs of the report pass (st_solve_report); any output may be NULL
struct ReportReq {
  const double* geom2;  // batch x 2: l_xy, l_z of the collision check
  const double* obs;    // batch x n_obs x 5: cx, cy, cz, l_xy/2 + r, l_z/2 + r
  double* traj;         // batch x n x m x 3
  double* arc;          // batch x n
  double* smooth;       // batch x n
  double* min_dist;     // batch
  long long* n_viol;    // batch
};

struct st_plan {
  int n, nobs, m, nv, S, device, nvmax;
  double* d_mats = nullptr;  // P | G | Gm | F | Fm | E | rho | packed stage mats | 1/rho
  const double *P, *G, *Gm, *F, *Fm, *E, *rho, *mats, *inv_rho;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  int* d_counter = nullptr;
  double* d_lam = nullptr;  // multiplier slabs (double or float elements)
  size_t lam_bytes = 0;
  double* d_cws = nullptr;
  size_t c_bytes = 0;
  void* d_rg = nullptr;
  size_t rg_bytes = 0;
  void* d_io = nullptr;  // inputs+outputs of host-pointer solves
  void* h_stage = nullptr;  // page-locked staging of small host-pointer solves (one H2D, one D2H)
  size_t stage_bytes = 0;
  size_t io_bytes = 0;
  int smem_optin = 0;
  int smem_sm = 0;  // shared memory per SM
  int persist_set = 0;
  cudaEvent_t ev_done = nullptr;  // last launch that used this plan's workspaces
  void* d_rep = nullptr;          // st_solve_report workspace (trajectories, metrics, verdict rows)
  size_t rep_bytes = 0;
  void* d_lgw = nullptr;          // large-fleet workspace (tables, unit slots, positions, ...)
  size_t lgw_bytes = 0;
  std::vector<long long> lg_key;  // layout whose tables are in d_lgw
  std::map<std::vector<int>, Launch> launch_cache;  // choose_launch results (see choose_launch_cached)
  std::mutex mu;
  bool async_pending = false;  // st_solve_report_begin enqueued, st_solve_end not yet called
};

namespace {

int ceil_div(int a, int b) { return (a + b - 1) / b; }

// Steps of one warp task; mirrors the enumeration in pairwise_phase().
int count_steps(int n, int nobs, int NB) {
  if (NB == 1) return n / 2 + nobs;
  int st = 0;
  for (int A = 0; A < NB; ++A) {
    const int nA = std::min(32, n - A * 32);
    if (nA <= 0) continue;
    st += nA / 2 + nobs;
  }
  for (int A = 0; A < NB; ++A)
    for (int B = A + 1; B < NB; ++B)
      if (std::min(32, n - B * 32) > 0) st += 32;
  return st;
}

// Shared-memory carve-up for cluster size C; returns total doubles (lambda excluded).
long long layout(st_plan* pl, Launch& L, int C) {
  swarm::KParams& k = L.kp;
  const int NP = L.NB * 32, n = pl->n, NW = L.NT / 32, TPW = 32 / L.W;
  L.C = C;
  const int KC = L.G * L.K * C;  // CTAs sharing one scenario
  L.tmax = ceil_div(pl->m, KC);
  L.tasks_max = ceil_div(L.tmax, TPW);  // time groups of the largest CTA
  // redundant solve (every CTA solves all agents, one cluster barrier per iteration) for small
  // single-cluster launches; wide clusters and multi-cluster launches use owners + all-gather
  const char* re = std::getenv("SWARM_RED");
  const int red_max = re ? std::atoi(re) : 4;  // SWARM_RED=0 disables, =C allows clusters up to C CTAs
  k.red = (L.G * L.K == 1 && !L.c_global && C <= red_max) ? 1 : 0;
  L.own_max = k.red ? n : ceil_div(n, C);
  const int NV = L.NVMAX;
  const bool obst = pl->nobs > 0;
  // partial S'b rows j*3 + ax (+ 3 agent-sum rows); row stride == 4 (mod 8) doubles keeps the
  // DMMA operand loads of project_phase bank-conflict free
  int nrp = 3 * n + (obst ? 3 : 0);
  nrp += nrp & 1;
  while (nrp % 8 != 4) nrp += 2;
  k.nrow_p = nrp;
  k.xs = 3 * NP + 8;  // X group stride == 8 (mod 16): conflict-free 16-byte stores of DMMA tiles
  long long o = 0;
  auto take = [&](int& off, long long cnt) {
    off = (int)o;
    o += (cnt + 1) & ~1LL;  // keep 16-byte alignment
  };
  take(k.o_c, L.c_global ? 0 : 3LL * n * NV);
  // the DMMA tiles read whole 4-row (qv) and 8-row (P) blocks: rows past the CTA's samples are zero
  k.qrow = (L.tmax + 3) / 4 * 4;
  k.prow = (L.tasks_max * TPW + 7) / 8 * 8 + 8;
  take(k.o_qv, (long long)k.qrow * nrp);  // first warp of each group: rows per time
  // exchange region Rp [3n][NV] | xch [agent sums 3 NV | sum r^2, max |r| | 2 spare].
  // Owner mode: it aliases the qx slots (dead after project_phase's fix-up; the owners pull it
  // between the two cluster barriers).  red: two parity copies of its own (one barrier).
  const long long rx = (3LL * n * NV + 3LL * NV + 4 + 1) & ~1LL, qx_sz = (long long)NW * TPW * nrp;
  if (k.red) {
    take(k.o_qx, qx_sz);  // warps starting inside a group: their first group's rows
    take(k.o_Rp, 2 * rx);
  } else {
    take(k.o_qx, std::max(qx_sz, rx));
    k.o_Rp = k.o_qx;
  }
  k.o_xch = k.o_Rp + 3 * n * NV;
  k.xch_norm = 3 * NV;
  k.rx = k.red ? (int)rx : 0;
  take(k.o_X, (long long)L.tasks_max * k.xs);
  take(k.o_tab, (L.tmax + 1) / 2);  // per-time warp ranges
  take(k.o_P, (long long)k.prow * NV);
  take(k.o_cown, k.red ? 0 : (long long)L.own_max * 3 * NV);
  take(k.o_nrm, 3LL * C);
  take(k.o_otab, (n + 1) / 2);
  take(k.o_R, !k.red ? (long long)L.own_max * 3 * NV
               : 3LL * n * (NV == 12 ? swarm::SolveOp<12>::kas(obst) : swarm::SolveOp<16>::kas(obst)));
  take(k.o_Rb, 3LL * NV);
  take(k.o_mat, NV == 12 ? swarm::StageMats<12>::SIZE : swarm::StageMats<16>::SIZE);
  take(k.o_sa, !k.red ? 0
               : NV == 12 ? swarm::SolveOp<12>::MA * swarm::SolveOp<12>::kas(obst)
                          : swarm::SolveOp<16>::MA * swarm::SolveOp<16>::kas(obst));
  take(k.o_geo, 8 + 8LL * pl->nobs);
  take(k.o_beq, 18LL * L.own_max);
  take(k.o_bb, 18);
  take(k.o_wp, 2LL * NW);
  take(k.o_misc, swarm::MI_INTS / 2);  // scenario slot | launch-constant index table (am_kernel.cuh)
  take(k.o_bnd, 2);
  k.o_lam = (int)o;
  L.lam_per_cta = (long long)L.tasks_max * L.nsteps * 96;
  return o;
}

// shared-memory doubles taken by `rows` multiplier rows (96 elements each)
long long lam_rows_dbl(const Launch& L, long long rows) { return (rows * 96 * (L.f32 ? 4 : 8) + 7) / 8; }

// Hybrid multipliers: rows per warp kept in shared memory (each warp's last rows), from
// `spare` doubles of shared memory, at most the rows of the longest warp range.
int tail_rows(const Launch& L, long long spare) {
  const int NW = L.NT / 32, TPW = 32 / L.W;
  const long long rows_max = ceil_div((long long)ceil_div(L.tmax, TPW) * L.nsteps, NW);
  const long long per_row = 96LL * NW * (L.f32 ? 4 : 8) / 8;  // doubles per row across the warps
  return (int)std::max(0LL, std::min(rows_max, spare / per_row));
}

const KernelEntry* find_kernel(int NB, int NVMAX, int LAM, bool f32, bool obstacles) {
  for (const auto& e : kKernels)
    if (e.NB == NB && e.NVMAX == NVMAX && e.LAM == LAM && e.f32 == f32 && (!obstacles || !e.obs_free)) return &e;
  return nullptr;
}

cudaError_t ensure_smem_attr(int device, const void* fn, size_t bytes);

int choose_launch(st_plan* pl, int batch, int hint, bool keep, Launch& L, int G = 1, bool f32 = false) {
  const int n = pl->n;
  if (n < 1 || n > 256) return fail(ST_EUNSUPPORTED, "n_agents must be in [1, 256] for the compiled kernels");
  const int nb_need = n <= 32 ? 1 : ceil_div(n, 32);
  int NB = 0;
  for (int cand : {1, 2, 4, 8})
    if (cand >= nb_need && find_kernel(cand, pl->nvmax, swarm::LAM_GLOBAL, f32, pl->nobs > 0)) { NB = cand; break; }
  if (!NB) return fail(ST_EUNSUPPORTED, "no compiled kernel for this agent count and basis degree");
  L.NB = NB;
  L.NVMAX = pl->nvmax;
  L.f32 = f32 ? 1 : 0;
  if (NB == 1) {
    int w = 2;
    while (w < n) w <<= 1;
    L.W = w;
  } else {
    L.W = 32;
  }
  L.nsteps = std::max(1, count_steps(n, pl->nobs, NB));  // n = 1, no obstacles: one empty step
  const long long budget = pl->smem_optin / 8;
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, pl->device);
  nsm = std::max(nsm, 1);
  std::vector<int> cands;
  if (hint > 0) {
    cands.push_back(hint);
  } else if (batch == 1 && pl->n > 32) {
    // latency, one large scenario over K clusters of C CTAs (multi-cluster): fewest samples per
    // CTA first (the grid barrier waits for the fullest CTA), then the widest cluster. m = 100
    // on 148 SMs: C = 10 (K = 10, one sample per CTA) -- measured 18 ms vs 34 ms for C = 16
    // (K = 6, up to two samples per CTA) on rand256_s0
    cands = {16, 10, 8, 5, 4, 2, 1};
    auto per_cta = [&](int C) {
      const int K = std::max(1, std::min(nsm / C, pl->m / C));
      return ceil_div(pl->m, K * C);
    };
    std::stable_sort(cands.begin(), cands.end(), [&](int a, int b) { return per_cta(a) < per_cta(b); });
  } else if (batch == 1 && pl->n <= 8) {
    // latency, tiny fleets: 8-CTA clusters match 16 per iteration (rand5 7.8 vs 8.1 us, rand8
    // 8.3 vs 8.2, profiles/small_cluster_sweep_r2.txt) with half the exchange/barrier partners,
    // and their per-iteration cost follows the obstacle count (acceptance C8)
    cands = {8, 16, 4, 2, 1};
  } else if (batch == 1) {
    cands = {16, 8, 4, 2, 1};  // latency: spread one scenario widest
  } else {
    // throughput: measured on B200 (profiles/) two-CTA clusters streaming
    // lambda from L2 beat wider clusters that keep it on chip (exchange overhead dominates)
    cands = {2, 1, 4, 8, 16};
  }
  // Latency (one scenario): prefer lambda on chip, then the widest cluster.
  // Throughput (batches): prefer the cluster order above; at each size lambda on chip if it fits.
  const bool throughput = hint <= 0 && batch > 1;
  std::vector<std::pair<int, int>> order;  // (C, pass)
  if (throughput) {
    for (int C : cands)
      for (int pass = 0; pass < 2; ++pass) order.push_back({C, pass});
  } else {
    for (int pass = 0; pass < 2; ++pass)
      for (int C : cands) order.push_back({C, pass});
  }
  const char* mc_env = std::getenv("SWARM_MULTI_CLUSTER");
  for (int cg_try = 0; cg_try < 2; ++cg_try)
  for (const auto& cp : order) {
    const int C = cp.first, pass = cp.second;
    if (cg_try == 1 && pass == 0) continue;  // coefficients in global memory only with lambda there too
    const int lam = pass == 0 ? swarm::LAM_SMEM : (keep ? swarm::LAM_GLOBAL_KEEP : swarm::LAM_GLOBAL);
    if (keep && pass == 0) continue;
    const KernelEntry* ke = find_kernel(NB, pl->nvmax, lam, f32, pl->nobs > 0);
    if (!ke) continue;
    const long long bud = budget;
    if ((long long)C * G > pl->m || C < 1 || C > 16) continue;  // every CTA owns >= 1 sample
    Launch T = L;
    T.NT = ke->NT;
    T.fn = ke->fn;
    T.c_global = cg_try;
    long long base = layout(pl, T, C);
    long long need = base + (pass == 0 ? lam_rows_dbl(T, (long long)T.tasks_max * T.nsteps) : 0);
    const bool want_multi = G > 1 || (batch == 1 && C > 1 && (mc_env ? std::atoi(mc_env) != 0 : pl->n > 32));
    bool sized_for_split = false;
    if (need > bud && want_multi) {
      // one cluster cannot hold the scenario's per-CTA buffers, but K co-resident clusters
      // (each CTA owning ~m/(G K C) samples) may: size the layout for the multi-cluster split
      T.G = G;
      T.K = std::max(1, std::min(std::max(1, nsm / C), pl->m / (G * C)));
      base = layout(pl, T, C);
      need = base + (pass == 0 ? lam_rows_dbl(T, (long long)T.tasks_max * T.nsteps) : 0);
      sized_for_split = T.K > 1;
    }
    if (need > bud) continue;
    T.lam_smem = pass == 0 ? 1 : 0;
    T.lam_tail = 0;
    long long need2 = need;
    if (pass == 1 && !keep) {
      // hybrid: spare shared memory holds each warp's last multiplier rows (the rest stays in L2)
      const char* hy = std::getenv("SWARM_LAM_HYBRID");
      if (!hy || std::atoi(hy) != 0) {
        T.lam_tail = tail_rows(T, bud - need);
        need2 = need + lam_rows_dbl(T, (long long)T.lam_tail * (T.NT / 32));
      }
    }
    T.smem_bytes = (size_t)need2 * 8;
    ST_CUDA(ensure_smem_attr(pl->device, (const void*)T.fn, T.smem_bytes));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(T.NT);
    cfg.dynamicSmemBytes = T.smem_bytes;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int active = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&active, (void*)T.fn, &cfg);
    if (e != cudaSuccess || active < 1) {
      cudaGetLastError();
      continue;
    }
    // one large scenario: spread it over co-resident clusters (grid barrier per iteration)
    const bool multi = G > 1 || (batch == 1 && C > 1 && active > 1 && want_multi);
    if (sized_for_split && !multi) continue;  // sized for a split that cannot run
    T.nclusters = std::min(batch, active);
    T.active = active;
    if (multi) {
      Launch M = T;
      M.G = G;
      M.K = std::min(active, std::max(1, pl->m / (G * C)));
      const long long mbase = layout(pl, M, C);
      long long mneed = mbase + (pass == 0 ? lam_rows_dbl(M, (long long)M.tasks_max * M.nsteps) : 0);
      M.lam_tail = 0;
      if (pass == 1 && !keep && mneed <= budget) {
        M.lam_tail = tail_rows(M, budget - mneed);
        mneed += lam_rows_dbl(M, (long long)M.lam_tail * (M.NT / 32));
      }
      if (mneed <= budget) {
        M.smem_bytes = (size_t)mneed * 8;
        ST_CUDA(ensure_smem_attr(pl->device, (const void*)M.fn, M.smem_bytes));
        M.nclusters = M.K;
        T = M;
      } else if (T.K > 1) {
        continue;  // the split layout does not fit: never launch K > 1 on fewer clusters (advice r1)
      }
    }
    if (T.K > 1 && T.nclusters != T.K) continue;  // a grid barrier needs all K clusters launched
    L = T;
    return 0;
  }
  return fail(ST_EUNSUPPORTED, "no cluster configuration fits this problem on the device");
}

// choose_launch, memoized per plan: the occupancy queries and attribute calls run once per
// (single/batch, cluster hint, keep_state, groups, FP32) shape; the cluster count follows the
// batch (SWARM_* launch knobs are read when a shape is first seen).
int choose_launch_cached(st_plan* pl, int batch, int hint, bool keep, Launch& L, int G, bool f32) {
  const std::vector<int> key = {batch == 1 ? 1 : 2, hint, keep ? 1 : 0, G, f32 ? 1 : 0};
  auto it = pl->launch_cache.find(key);
  if (it != pl->launch_cache.end()) {
    L = it->second;
    if (L.K <= 1) L.nclusters = std::min(batch, L.active);
    return 0;
  }
  int rc = choose_launch(pl, batch, hint, keep, L, G, f32);
  if (rc == 0) pl->launch_cache[key] = L;
  return rc;
}

// Dynamic shared-memory limits of the kernel functions only ever grow (a launch configuration
// cached by one plan stays valid whatever another plan needs), per device.
std::mutex g_attr_mu;
std::map<std::pair<int, const void*>, int> g_attr;
cudaError_t ensure_smem_attr(int device, const void* fn, size_t bytes) {
  std::lock_guard<std::mutex> lk(g_attr_mu);
  int& cur = g_attr[{device, fn}];
  if (cur >= (int)bytes) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) cur = (int)bytes;
  return e;
}

// device-wide ordering of grid-barrier (multi-cluster) launches, one event per device
std::mutex g_multi_mu;
cudaEvent_t multi_event(int device) {
  static cudaEvent_t evs[64] = {};
  if (device < 0 || device >= 64) return nullptr;
  if (!evs[device] && cudaEventCreateWithFlags(&evs[device], cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return evs[device];
}

// The device-wide L2 set-aside for persisting lines: the batch kernel's multiplier slabs and
// the FP32 large-fleet multipliers want it; a kernel that streams through L2 (FP64 large
// fleets) loses ~40% with it in place (profiles/large_l2_setaside_r2.txt), so every launch sets
// what it needs (device-wide, sticky: tracked per device to skip redundant calls).
std::mutex g_persist_mu;
int g_persist_state[64];
bool g_persist_init = false;
size_t set_persisting_l2(int device, bool on) {
  std::lock_guard<std::mutex> lk(g_persist_mu);
  if (!g_persist_init) {
    for (auto& v : g_persist_state) v = -1;
    g_persist_init = true;
  }
  int max_persist = 0;
  cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, device);
  if (device < 0 || device >= 64 || max_persist <= 0) return 0;
  const int want = on ? 1 : 0;
  if (g_persist_state[device] != want) {
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, on ? (size_t)max_persist : 0);
    if (!on) cudaCtxResetPersistingL2Cache();
    cudaGetLastError();
    g_persist_state[device] = want;
  }
  return on ? (size_t)max_persist : 0;
}

struct ShardExt {
  int G, rank;
  void* bufs[8];
};

// ---------------------------------------------------------------------------------------------
// Large fleets (am_large.cuh): one scenario over every SM (and over G GPUs when pair-sharded)

using LargeFn = void (*)(swarm::LgParams);
struct LargeEntry {
  int NVMAX;
  bool f32;
  LargeFn fn;
};
const LargeEntry kLarge[] = {
    {12, false, swarm::am_large_kernel<12, false>}, {12, true, swarm::am_large_kernel<12, true>},
    {16, false, swarm::am_large_kernel<16, false>}, {16, true, swarm::am_large_kernel<16, true>},
};

bool large_eligible(const st_plan* pl, int batch, bool keep) {
  const char* e = std::getenv("SWARM_LARGE");
  const int mode = e ? std::atoi(e) : 1;
  if (mode == 0 || batch != 1 || keep || pl->nobs != 0 || pl->n < 2 || pl->n > 32 * swarm::LG_MAXB) return false;
  // n > 32: the whole-GPU unit decomposition beats the multi-cluster grid-barrier layout from the
  // first multi-block size on (sph64j 3.12 -> 2.52 ms, rand48_s0 2.09 -> 1.80 ms; n <= 32 stays on
  // one cluster: circ16j 0.98 vs 1.46 ms)
  return mode == 2 || pl->n > 32;
}

// Units in block-pair-major order: a diagonal block pair (A == B) has one unit per sample t
// (u = ab_first[ab] + t), a cross pair two (u = ab_first[ab] + 2 t + h); pair-step rows of each.
struct LargeLayout {
  int NB = 0, nab = 0, npad = 0, m = 0, U = 0, G = 1, cpg = 0;
  std::vector<int> ab;         // nab x 2
  std::vector<int> ab_first;   // nab + 1
  std::vector<int> rows;       // U
  std::vector<int> u_range;    // G + 1
  std::vector<int> cta_first;  // G x (cpg + 1)
};

LargeLayout large_layout(const st_plan* pl, int G, int cpg) {
  LargeLayout Lg;
  const int n = pl->n;
  Lg.NB = (n + 31) / 32;
  Lg.npad = Lg.NB * 32;
  Lg.m = pl->m;
  for (int A = 0; A < Lg.NB; ++A)
    for (int B = A; B < Lg.NB; ++B) { Lg.ab.push_back(A); Lg.ab.push_back(B); }
  Lg.nab = (int)Lg.ab.size() / 2;
  Lg.ab_first.assign(Lg.nab + 1, 0);
  for (int ab = 0; ab < Lg.nab; ++ab) Lg.ab_first[ab + 1] = Lg.ab_first[ab] + (Lg.ab[2 * ab] == Lg.ab[2 * ab + 1] ? 1 : 2) * Lg.m;
  Lg.U = Lg.ab_first[Lg.nab];
  Lg.rows.resize(Lg.U);
  std::vector<long long> pre(Lg.U + 1, 0);
  for (int ab = 0; ab < Lg.nab; ++ab) {
    const int A = Lg.ab[2 * ab], B = Lg.ab[2 * ab + 1];
    const int nA = std::min(32, n - 32 * A);
    for (int u = Lg.ab_first[ab]; u < Lg.ab_first[ab + 1]; ++u) Lg.rows[u] = (A == B) ? nA / 2 : swarm::LG_UNIT_STEPS;
  }
  for (int u = 0; u < Lg.U; ++u) pre[u + 1] = pre[u] + Lg.rows[u];
  // contiguous cost-balanced ranges: the first unit whose prefix cost reaches the target
  auto cut = [&](long long target) {
    return (int)(std::lower_bound(pre.begin(), pre.end(), target) - pre.begin());
  };
  Lg.G = G;
  Lg.cpg = cpg;
  const long long T = pre[Lg.U];
  Lg.u_range.resize(G + 1);
  for (int g = 0; g <= G; ++g) Lg.u_range[g] = g == G ? Lg.U : cut(T * g / G);
  Lg.cta_first.resize((size_t)G * (cpg + 1));
  for (int g = 0; g < G; ++g) {
    const long long c0 = pre[Lg.u_range[g]], c1 = pre[Lg.u_range[g + 1]];
    for (int c = 0; c <= cpg; ++c)
      Lg.cta_first[(size_t)g * (cpg + 1) + c] =
          c == cpg ? Lg.u_range[g + 1] : std::max(Lg.u_range[g], cut(c0 + (c1 - c0) * c / cpg));
  }
  return Lg;
}

// CTAs per SM the large kernel fits (1 by design), and the grid of one GPU
int large_grid(st_plan* pl, const LargeEntry* le, size_t smem, int& grid) {
  ST_CUDA(ensure_smem_attr(pl->device, (const void*)le->fn, smem));
  int occ = 0, nsm = 0;
  ST_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, le->fn, swarm::LG_NT, smem));
  ST_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, pl->device));
  if (occ < 1) return fail(ST_EUNSUPPORTED, "large-fleet kernel does not fit on an SM");
  grid = occ * nsm;
  if (const char* e = std::getenv("SWARM_LARGE_GRID")) grid = std::max(1, std::min(grid, std::atoi(e)));
  return 0;
}

// Growable device workspace owned by the plan (freed and reallocated only when it must grow;
// the plan's launch ordering event makes reuse safe).
int grow(void** ptr, size_t* cap, size_t need) {
  if (need <= *cap) return 0;
  if (*ptr) cudaFree(*ptr);
  *ptr = nullptr;
  *cap = 0;
  ST_CUDA(cudaMalloc(ptr, need));
  *cap = need;
  return 0;
}

int run(st_plan* pl, const Launch& L0, int batch, const double* c0, const double* beq, const double* geom,
        int switch_every, int max_iters, double tol, int flags, double* c_out, double* hist, int* iters,
        int* conv, double* lam_out, double* d_out, cudaStream_t s, const ShardExt* ext = nullptr) {
  Launch L = L0;
  swarm::KParams& k = L.kp;
  ST_CUDA(cudaStreamWaitEvent(s, pl->ev_done, 0));  // previous launch on this plan has finished
  k.n = pl->n; k.nobs = pl->nobs; k.m = pl->m; k.nv = pl->nv; k.S = pl->S;
  k.P = pl->P; k.G = pl->G; k.Gm = pl->Gm; k.F = pl->F; k.Fm = pl->Fm; k.E = pl->E; k.rho = pl->rho;
  k.mats = pl->mats; k.inv_rho = pl->inv_rho;
  k.C = L.C; k.W = L.W; k.nsteps = L.nsteps; k.tmax = L.tmax; k.tasks_max = L.tasks_max;
  k.own_max = L.own_max; k.lam_in_smem = L.lam_smem; k.lam_per_cta = L.lam_per_cta;
  k.lam_tail = L.lam_tail;
  k.B = batch; k.gstride = 2 + 5 * pl->nobs;
  k.c0 = c0; k.beq = beq; k.geom = geom; k.c_out = c_out; k.hist = hist; k.iters = iters; k.conv = conv;
  k.lam_out = lam_out; k.d_out = d_out; k.counter = pl->d_counter;
  k.switch_every = switch_every; k.max_iters = max_iters; k.flags = flags; k.tol = tol;
  k.K = L.K;
  k.ngrp = 1;
  k.g_rank = 0;
  k.sys_scope = 0;
  k.Rg = nullptr;
  k.gbar = nullptr;
  for (auto& g : k.Rg_grp) g = nullptr;
  if (ext != nullptr) {
    // pair-sharded launch: this GPU is group ext->rank of ext->G; buffers are peer-mapped
    k.ngrp = ext->G;
    k.g_rank = ext->rank;
    k.sys_scope = 1;
    for (int g = 0; g < ext->G; ++g)
      k.Rg_grp[g] = reinterpret_cast<double*>(reinterpret_cast<char*>(ext->bufs[g]) + 64);
    k.gbar = reinterpret_cast<unsigned*>(ext->bufs[0]);
    k.Rg = k.Rg_grp[0];
  } else if (L.K > 1) {
    // one GPU; SWARM_VIRTUAL_GROUPS=g splits the K clusters into g groups with separate buffers
    // (same participants, same order: bitwise-identical results; exercises the sharded indexing)
    int gv = 1;
    if (const char* vg = std::getenv("SWARM_VIRTUAL_GROUPS")) gv = std::max(1, std::atoi(vg));
    if (gv > 8 || L.K % gv != 0) gv = 1;
    const size_t per = 2 * (size_t)(L.K / gv) * (3 * (size_t)pl->n * L.NVMAX + 3 * L.NVMAX + 4);
    const size_t need = gv * per * sizeof(double) + 64;
    if (need > pl->rg_bytes) {
      if (pl->d_rg) cudaFree(pl->d_rg);
      pl->d_rg = nullptr;
      pl->rg_bytes = 0;
      ST_CUDA(cudaMalloc(&pl->d_rg, need));
      pl->rg_bytes = need;
    }
    k.ngrp = gv;
    k.K = L.K / gv;
    k.gbar = reinterpret_cast<unsigned*>(pl->d_rg);
    for (int g = 0; g < gv; ++g)
      k.Rg_grp[g] = reinterpret_cast<double*>(reinterpret_cast<char*>(pl->d_rg) + 64) + g * per;
    k.Rg = k.Rg_grp[0];
    ST_CUDA(cudaMemsetAsync(pl->d_rg, 0, 64, s));
  }
  k.c_global = L.c_global;
  k.c_ws = nullptr;
  if (L.c_global) {
    const size_t need = (size_t)L.nclusters * 3 * pl->n * L.NVMAX * sizeof(double);
    if (need > pl->c_bytes) {
      if (pl->d_cws) cudaFree(pl->d_cws);
      pl->d_cws = nullptr;
      pl->c_bytes = 0;
      ST_CUDA(cudaMalloc(&pl->d_cws, need));
      pl->c_bytes = need;
    }
    k.c_ws = pl->d_cws;
  }
  const size_t esize = L.f32 ? sizeof(float) : sizeof(double);
  if (!L.lam_smem) {
    const size_t need = (size_t)L.nclusters * L.C * L.lam_per_cta * esize;
    if (need > pl->lam_bytes) {
      if (pl->d_lam) cudaFree(pl->d_lam);
      pl->d_lam = nullptr;
      pl->lam_bytes = 0;
      ST_CUDA(cudaMalloc(&pl->d_lam, need));
      pl->lam_bytes = need;
    }
    k.lam_ws = pl->d_lam;
  } else {
    k.lam_ws = nullptr;
  }
  // opt-in phase timers: SWARM_PHASE_TIMERS=1 prints per-phase cycles of scenario 0, CTA 0
  static long long* d_ts = nullptr;
  const bool timers = std::getenv("SWARM_PHASE_TIMERS") != nullptr;
  if (timers && !d_ts) ST_CUDA(cudaMalloc(&d_ts, 16 * 4096 * sizeof(long long)));
  if (timers) ST_CUDA(cudaMemsetAsync(d_ts, 0, 16 * 4096 * sizeof(long long), s));
  k.tstamp = timers ? d_ts : nullptr;
  ST_CUDA(cudaMemsetAsync(pl->d_counter, 0, sizeof(int), s));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(L.nclusters * L.C);
  cfg.blockDim = dim3(L.NT);
  cfg.dynamicSmemBytes = L.smem_bytes;
  cfg.stream = s;
  cudaLaunchAttribute at[3];
  int na = 0;
  cudaAccessPolicyWindow window = {};
  bool has_window = false;
  at[na].id = cudaLaunchAttributeClusterDimension;
  at[na].val.clusterDim.x = L.C;
  at[na].val.clusterDim.y = 1;
  at[na].val.clusterDim.z = 1;
  ++na;
  // Multi-cluster launches (grid barrier per iteration) need all their CTAs resident at once.
  // The launch is sized from cudaOccupancyMaxActiveClusters, and kernels that do not wait on
  // anyone (batches, other solves) always retire, so the only in-process deadlock is two
  // grid-barrier launches each holding SMs the other waits for: they are serialized
  // device-wide here.  (cudaLaunchAttributeCooperative would also guarantee residency but
  // measured 5-8x slower per iteration on B200 with clusters: DESIGN.md §4.)  A barrier that
  // still never completes (another process) ends in a trap after 30 s, not a hung device.
  cudaEvent_t multi_ev = nullptr;
  std::unique_lock<std::mutex> multi_lock;
  if (L.K > 1) {
    multi_lock = std::unique_lock<std::mutex>(g_multi_mu);
    multi_ev = multi_event(pl->device);
    if (!multi_ev) return fail(ST_ECUDA, "cannot create the multi-cluster ordering event");
    ST_CUDA(cudaStreamWaitEvent(s, multi_ev, 0));
  }
  if (!L.lam_smem) {
    // keep the multiplier slabs resident in L2 (persisting window), for this launch only
    const char* pe = std::getenv("SWARM_L2_PERSIST");
    int max_persist = 0, max_window = 0;
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, pl->device);
    cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, pl->device);
    if ((!pe || std::atoi(pe) != 0) && max_persist > 0 && max_window > 0) {
      set_persisting_l2(pl->device, true);
      const size_t used = (size_t)L.nclusters * L.C * L.lam_per_cta * esize;
      const int TPWl = 32 / L.W, NWl = L.NT / 32;
      const long long rows_w = ceil_div((long long)ceil_div(L.tmax, TPWl) * L.nsteps, NWl);
      const double gfrac = rows_w > 0 ? 1.0 - (double)L.lam_tail / rows_w : 1.0;
      at[na].id = cudaLaunchAttributeAccessPolicyWindow;
      at[na].val.accessPolicyWindow.base_ptr = pl->d_lam;
      at[na].val.accessPolicyWindow.num_bytes = std::min(used, (size_t)max_window);
      // persisting lines at 80% of the set-aside: a cyclic stream that just overfills it thrashes
      // the LRU (1024 rand32, 87 MB window, 79 MB touched vs 83 MB set-aside: hit ratio 1.0 ->
      // 31 GB DRAM per launch, 0.85 -> 19 GB and 1.4% faster; profiles/l2_hit_sweep_r2.txt)
      at[na].val.accessPolicyWindow.hitRatio = (float)std::min(
          1.0, 0.8 * (double)max_persist / std::max(1.0, gfrac * at[na].val.accessPolicyWindow.num_bytes));
      if (const char* hr = std::getenv("SWARM_L2_HIT")) at[na].val.accessPolicyWindow.hitRatio = (float)std::atof(hr);
      at[na].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      at[na].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      // As a stream attribute: measured on B200 the same window given as a launch attribute is
      // not honoured (DRAM writes 86 GB vs 12 GB per 1024-scenario launch, profiles/l2_window_r2.txt).
      // It is cleared again right after the launch, so the caller's stream keeps no window.
      window = at[na].val.accessPolicyWindow;
      has_window = true;
    }
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  if (has_window) {
    cudaStreamAttrValue av = {};
    av.accessPolicyWindow = window;
    cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &av);
    cudaGetLastError();
  }
  const cudaError_t le = cudaLaunchKernelEx(&cfg, L.fn, k);
  if (has_window) {
    cudaStreamAttrValue off = {};
    off.accessPolicyWindow.num_bytes = 0;
    cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &off);
    cudaGetLastError();
  }
  ST_CUDA(le);
  if (multi_ev) ST_CUDA(cudaEventRecord(multi_ev, s));
  // launches sharing this plan's workspaces (counter, slabs, exchange buffers) run in order,
  // whatever streams their callers use (advice r1: st_solve_device on several streams)
  ST_CUDA(cudaEventRecord(pl->ev_done, s));
  if (timers) {
    std::vector<long long> h(16 * 4096);
    ST_CUDA(cudaMemcpyAsync(h.data(), d_ts, h.size() * sizeof(long long), cudaMemcpyDeviceToHost, s));
    ST_CUDA(cudaStreamSynchronize(s));
    static const char* names[] = {"pull+test", "solve", "bar2", "gather", "positions", "pairwise", "warp-wait",
                                  "project", "bar1"};
    double acc[9] = {0};
    int cnt = 0;
    for (int it = 1; it < 255 && h[16 * (it + 1)]; ++it, ++cnt) {
      const long long* t = &h[16 * it];
      for (int q = 0; q < 8; ++q) acc[q] += t[q + 1] - t[q];
      acc[8] += h[16 * (it + 1)] - t[8];
    }
    if (cnt) {
      std::fprintf(stderr, "[swarm timers] C=%d NB=%d iters=%d cycles/iter:", L.C, L.NB, cnt);
      for (int q = 0; q < 9; ++q) std::fprintf(stderr, " %s=%.0f", names[q], acc[q] / cnt);
      double sub[3] = {0, 0, 0}, drain = 0;
      for (int it = 1; it <= cnt; ++it) {
        const long long* t = &h[16 * it];
        sub[0] += t[9] - t[11];
        drain += t[11] - t[7];
        sub[1] += t[10] - t[9];
        sub[2] += t[8] - t[10];
      }
      std::fprintf(stderr, " [project: drain=%.0f combine=%.0f sync=%.0f basis=%.0f]\n", drain / cnt, sub[0] / cnt,
                   sub[1] / cnt, sub[2] / cnt);
      // SWARM_PHASE_TIMERS=2: the same per-phase averages for every CTA of the first cluster
      // (each on its own SM clock): who arrives last at the cluster barriers
      if (std::atoi(std::getenv("SWARM_PHASE_TIMERS")) == 2) {
        for (int r = 0; r < std::min(L.C, 16); ++r) {
          double a2[9] = {0};
          for (int it = 1; it <= cnt; ++it) {
            const long long* t = &h[r * 4096 + 16 * it];
            for (int q = 0; q < 8; ++q) a2[q] += t[q + 1] - t[q];
            a2[8] += h[r * 4096 + 16 * (it + 1)] - t[8];
          }
          double b2[4] = {0};
          for (int it = 1; it <= cnt; ++it) {
            const long long* t = &h[r * 4096 + 16 * it];
            b2[0] += t[12] - t[0];   // pull: norms
            b2[1] += t[13] - t[12];  // pull: owner rows
            b2[2] += t[15] - t[1];   // test (owner mode)
            b2[3] += t[14] - t[15];  // solve compute
          }
          std::fprintf(stderr, "   cta %2d:", r);
          for (int q = 0; q < 9; ++q) std::fprintf(stderr, " %s=%.0f", names[q], a2[q] / cnt);
          std::fprintf(stderr, " | norms=%.0f rows=%.0f test=%.0f solvec=%.0f\n", b2[0] / cnt, b2[1] / cnt,
                       b2[2] / cnt, b2[3] / cnt);
        }
      }
    }
  }
  return 0;
}

// One large scenario through am_large_kernel.  ext != nullptr: this GPU is rank ext->rank of a
// pair-sharded solve over ext->G GPUs (peer-mapped exchange buffers).  Otherwise
// SWARM_VIRTUAL_GROUPS=g emulates g ranks inside this one launch (their CTAs wait on one
// another, so they must share a launch on one GPU).
int run_large(st_plan* pl, bool f32, const double* c0, const double* beq, const double* geom, int switch_every,
              int max_iters, double tol, double* c_out, double* hist, int* iters, int* conv, cudaStream_t s,
              const ShardExt* ext) {
  const LargeEntry* le = nullptr;
  for (const auto& e : kLarge)
    if (e.NVMAX == pl->nvmax && e.f32 == f32) le = &e;
  if (!le) return fail(ST_EUNSUPPORTED, "no large-fleet kernel for this basis degree");
  const int NV = pl->nvmax;
  const int chr = swarm::lg_chunk_rows(f32);
  const swarm::LgSmem sm = NV == 12 ? (f32 ? swarm::lg_smem<12, true>(pl->m, chr) : swarm::lg_smem<12, false>(pl->m, chr))
                                    : (f32 ? swarm::lg_smem<16, true>(pl->m, chr) : swarm::lg_smem<16, false>(pl->m, chr));
  const size_t smem = (size_t)sm.total;
  if ((long long)smem > pl->smem_optin) return fail(ST_EUNSUPPORTED, "large-fleet layout exceeds shared memory");
  int grid = 0;
  int rc = large_grid(pl, le, smem, grid);
  if (rc) return rc;
  int G = 1, g_base = 0, vgroups = 1;
  if (ext) {
    G = ext->G;
    g_base = ext->rank;
  } else if (const char* vg = std::getenv("SWARM_VIRTUAL_GROUPS")) {
    G = vgroups = std::max(1, std::min(8, std::atoi(vg)));
  }
  const int cpg = grid / vgroups;
  if (cpg < 1) return fail(ST_EUNSUPPORTED, "too few SMs for the requested groups");
  {
    // R-phase scratch in the multiplier ring: q rows | warp partials | R | c (am_large.cuh lg_rows)
    const long long rp = ((3LL * pl->n + cpg - 1) / cpg + 7) / 8 * 8, nh8 = (pl->nvmax + 7) / 8 * 8;
    const long long need = (rp * pl->m + (long long)swarm::LG_NW * rp * nh8 + 2 * rp * pl->nvmax) * 8;
    if (need > sm.bar - sm.ring)
      return fail(ST_EUNSUPPORTED, "large-fleet row reduction does not fit in shared memory");
  }
  const LargeLayout Lg = large_layout(pl, G, cpg);
  const int n = pl->n, m = pl->m;
  // host tables: block pairs, group ranges, CTA ranges, multiplier offsets of this launch's units
  const int ulo = Lg.u_range[g_base], uhi = Lg.u_range[g_base + vgroups];
  std::vector<long long> off(uhi - ulo + 1, 0);
  for (int u = ulo; u < uhi; ++u) off[u - ulo + 1] = off[u - ulo] + 96LL * Lg.rows[u];
  const size_t esize = f32 ? 4 : 8;
  const size_t n_ab = Lg.ab.size(), n_af = Lg.ab_first.size(), n_ur = Lg.u_range.size(), n_cf = Lg.cta_first.size();
  const size_t tab_bytes = ((n_ab + n_af + n_ur + n_cf) * 4 + 15) / 16 * 16 + off.size() * 8;
  const long long xst = 3LL * n * NV + 4;
  const size_t q_bytes = 2 * (size_t)Lg.U * 192 * 8, x_bytes = (size_t)m * 3 * Lg.npad * 8, cb_bytes = 3ULL * n * NV * 8;
  const size_t nrm_bytes = 2 * (size_t)grid * 16, bnd_bytes = (size_t)vgroups * 16 * 8;
  // barrier words (one 128-byte line per group + the system barrier), then the block-ready counters
  const size_t bar_bytes = (size_t)(vgroups + 1) * 128 + (size_t)vgroups * swarm::LG_MAXB * 128;
  const size_t xch_bytes = (ext || G == 1) ? 0 : (size_t)G * 2 * xst * 8;
  size_t o = 0;
  auto carve = [&](size_t bytes) { const size_t r = o; o += (bytes + 255) / 256 * 256; return r; };
  const size_t o_tab = carve(tab_bytes), o_q = carve(q_bytes), o_x = carve(x_bytes * vgroups),
               o_cb = carve(cb_bytes * vgroups), o_nrm = carve(nrm_bytes), o_bnd = carve(bnd_bytes),
               o_bar = carve(bar_bytes), o_xch = carve(xch_bytes);
  ST_CUDA(cudaStreamWaitEvent(s, pl->ev_done, 0));  // previous launch on this plan has finished
  rc = grow(&pl->d_lgw, &pl->lgw_bytes, o);
  if (rc) return rc;
  rc = grow(reinterpret_cast<void**>(&pl->d_lam), &pl->lam_bytes, std::max<size_t>(16, off.back() * esize));
  if (rc) return rc;
  char* base = static_cast<char*>(pl->d_lgw);
  const std::vector<long long> key = {G, g_base, vgroups, cpg, f32 ? 1 : 0, (long long)pl->d_lgw};
  if (key != pl->lg_key) {
    // tables depend only on the layout: uploaded once per layout (pageable copy, synchronized)
    std::vector<char> h(tab_bytes, 0);
    std::memcpy(h.data(), Lg.ab.data(), n_ab * 4);
    std::memcpy(h.data() + n_ab * 4, Lg.ab_first.data(), n_af * 4);
    std::memcpy(h.data() + (n_ab + n_af) * 4, Lg.u_range.data(), n_ur * 4);
    std::memcpy(h.data() + (n_ab + n_af + n_ur) * 4, Lg.cta_first.data(), n_cf * 4);
    std::memcpy(h.data() + tab_bytes - off.size() * 8, off.data(), off.size() * 8);
    ST_CUDA(cudaMemcpyAsync(base + o_tab, h.data(), tab_bytes, cudaMemcpyHostToDevice, s));
    ST_CUDA(cudaStreamSynchronize(s));  // h is pageable and goes out of scope
    pl->lg_key = key;
  }
  ST_CUDA(cudaMemsetAsync(base + o_bar, 0, bar_bytes, s));
  swarm::LgParams k{};
  k.n = n; k.m = m; k.nv = pl->nv; k.S = pl->S; k.NB = Lg.NB; k.nab = Lg.nab; k.npad = Lg.npad;
  k.P = pl->P; k.mats = pl->mats; k.inv_rho = pl->inv_rho; k.E = pl->E;
  const int* tab = reinterpret_cast<const int*>(base + o_tab);
  k.ab_pair = tab;
  k.ab_first = tab + n_ab;
  k.u_range = tab + n_ab + n_af;
  k.cta_first = tab + n_ab + n_af + n_ur;
  k.lam_off = reinterpret_cast<const long long*>(base + o_tab + tab_bytes - off.size() * 8);
  k.G = G; k.g_base = g_base; k.vgroups = vgroups; k.cpg = cpg;
  k.lam = pl->d_lam;
  k.qbuf = reinterpret_cast<double*>(base + o_q);
  k.q_stride = (long long)Lg.U * 192;
  k.blk_ready = reinterpret_cast<unsigned*>(base + o_bar + (size_t)(vgroups + 1) * 128);
  k.X = reinterpret_cast<double*>(base + o_x);
  k.cbuf = reinterpret_cast<double*>(base + o_cb);
  k.x_stride = (long long)(x_bytes / 8);
  k.c_stride = (long long)(cb_bytes / 8);
  k.cta_nrm = reinterpret_cast<double*>(base + o_nrm);
  k.bnd = reinterpret_cast<unsigned long long*>(base + o_bnd);
  k.gbar = reinterpret_cast<unsigned*>(base + o_bar);
  k.sysbar = reinterpret_cast<unsigned*>(base + o_bar + (size_t)vgroups * 128);
  k.sys_scope = 0;
  for (auto& x : k.xch) x = nullptr;
  if (ext) {
    k.sys_scope = 1;
    k.sysbar = reinterpret_cast<unsigned*>(ext->bufs[0]);
    for (int g = 0; g < G; ++g) k.xch[g] = reinterpret_cast<double*>(static_cast<char*>(ext->bufs[g]) + 64);
  } else {
    for (int g = 0; g < G && G > 1; ++g) k.xch[g] = reinterpret_cast<double*>(base + o_xch) + (size_t)g * 2 * xst;
  }
  k.c0 = c0; k.beq = beq; k.geom = geom;
  k.c_out = c_out; k.hist = hist; k.iters = iters; k.conv = conv;
  k.switch_every = switch_every; k.max_iters = max_iters; k.tol = tol;
  static long long* d_ts = nullptr;
  const bool timers = std::getenv("SWARM_PHASE_TIMERS") != nullptr;
  if (timers && !d_ts) ST_CUDA(cudaMalloc(&d_ts, 8192 * sizeof(long long)));
  if (timers) ST_CUDA(cudaMemsetAsync(d_ts, 0, 8192 * sizeof(long long), s));
  k.tstamp = timers ? d_ts : nullptr;
  // no persisting set-aside: FP64 multipliers stream through L2 evict-first and the unit slots /
  // positions need the whole cache; FP32 multipliers (78 MB at n = 256) stay by their evict-last
  // load policy alone (a persisting window measured 5.70 vs 5.61 ms on rand256_s0)
  const bool persist = f32 && std::getenv("SWARM_L2_PERSIST_LARGE") != nullptr;
  if (!persist) set_persisting_l2(pl->device, false);
  // grid-barrier kernels are serialized device-wide (see run())
  std::unique_lock<std::mutex> multi_lock(g_multi_mu);
  cudaEvent_t multi_ev = multi_event(pl->device);
  if (!multi_ev) return fail(ST_ECUDA, "cannot create the multi-cluster ordering event");
  ST_CUDA(cudaStreamWaitEvent(s, multi_ev, 0));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cpg * vgroups);
  cfg.blockDim = dim3(swarm::LG_NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  int na = 0;
  cudaAccessPolicyWindow window = {};
  bool has_window = false;
  if (persist) {
    // FP32 multipliers (n = 256: 78 MB) fit in L2: keep them there across iterations
    int max_persist = 0, max_window = 0;
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, pl->device);
    cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, pl->device);
    if (max_persist > 0 && max_window > 0) {
      set_persisting_l2(pl->device, true);
      const size_t used = off.back() * esize;
      at[na].id = cudaLaunchAttributeAccessPolicyWindow;
      at[na].val.accessPolicyWindow.base_ptr = pl->d_lam;
      at[na].val.accessPolicyWindow.num_bytes = std::min(used, (size_t)max_window);
      at[na].val.accessPolicyWindow.hitRatio =
          (float)std::min(1.0, (double)max_persist / std::max<double>(1.0, at[na].val.accessPolicyWindow.num_bytes));
      at[na].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      at[na].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      window = at[na].val.accessPolicyWindow;  // as a stream attribute (see run())
      has_window = true;
    }
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  if (has_window) {
    cudaStreamAttrValue av = {};
    av.accessPolicyWindow = window;
    cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &av);
    cudaGetLastError();
  }
  const cudaError_t lerr = cudaLaunchKernelEx(&cfg, le->fn, k);
  if (has_window) {
    cudaStreamAttrValue off = {};
    off.accessPolicyWindow.num_bytes = 0;
    cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &off);
    cudaGetLastError();
  }
  ST_CUDA(lerr);
  ST_CUDA(cudaEventRecord(multi_ev, s));
  ST_CUDA(cudaEventRecord(pl->ev_done, s));
  if (timers) {
    std::vector<long long> h(8192);
    ST_CUDA(cudaMemcpyAsync(h.data(), d_ts, h.size() * sizeof(long long), cudaMemcpyDeviceToHost, s));
    ST_CUDA(cudaStreamSynchronize(s));
    if (std::getenv("SWARM_CTA_TIMES")) {
      std::fprintf(stderr, "[swarm cta P-phase cycles, iteration 50]");
      for (int c = 0; c < cpg * vgroups; ++c)
        std::fprintf(stderr, " %d:%lld(u%d-%d)", c, h[4096 + c], Lg.cta_first[c], Lg.cta_first[c + 1]);
      std::fprintf(stderr, "\n");
    }
    static const char* names[] = {"norms+exchange", "solve+positions", "-", "pairs", "barrier"};
    double acc[5] = {0};
    int cnt = 0;
    for (int it = 1; it < 255 && h[16 * (it + 1)]; ++it, ++cnt) {
      const long long* t = &h[16 * it];
      for (int q = 0; q < 5; ++q) acc[q] += t[q + 1] - t[q];
    }
    if (cnt) {
      std::fprintf(stderr, "[swarm timers] large grid=%d groups=%d iters=%d cycles/iter:", cpg * vgroups, vgroups, cnt);
      for (int q = 0; q < 5; ++q) std::fprintf(stderr, " %s=%.0f", names[q], acc[q] / cnt);
      double rs[3] = {0, 0, 0};
      for (int it = 1; it <= cnt; ++it) {
        const long long* t = &h[16 * it];
        if (t[8] && t[9] && t[10]) { rs[0] += t[8] - t[7]; rs[1] += t[9] - t[8]; rs[2] += t[10] - t[9]; }
      }
      std::fprintf(stderr, " [cta0: gather=%.0f project=%.0f solve+X=%.0f]", rs[0] / cnt, rs[1] / cnt, rs[2] / cnt);
      std::fprintf(stderr, "\n");
    }
  }
  return 0;
}

int check_common(st_plan* pl, int batch, int switch_every, int max_iters, double tol, int flags) {
  if (!pl) return fail(ST_EINVAL, "plan is NULL");
  if (batch < 1) return fail(ST_EINVAL, "batch must be >= 1");
  if (switch_every < 1) return fail(ST_EINVAL, "switch_every must be >= 1");
  if (max_iters < 1) return fail(ST_EINVAL, "max_iters must be >= 1");
  if (!(tol > 0)) return fail(ST_EINVAL, "tolerance must be positive");
  if ((flags & ST_FLAG_KEEP_STATE) && batch != 1) return fail(ST_EINVAL, "keep_state needs batch == 1");
  if (flags & ~(ST_FLAG_KEEP_STATE | ST_FLAG_FP32)) return fail(ST_EINVAL, "unknown flag bits");
  return 0;
}

}  // namespace

extern "C" {

int st_version(void) { return 1; }

const char* st_last_error(void) { return g_err.c_str(); }

int st_plan_create(int n, int nobs, int m, int nv, int S, const double* P, const double* G, const double* Gm,
                   const double* F, const double* Fm, const double* E, const double* rho, int device,
                   st_plan** out) {
  if (!out) return fail(ST_EINVAL, "out is NULL");
  *out = nullptr;
  if (n < 1 || nobs < 0 || m < 2 || nv < 6 || S < 1)
    return fail(ST_EINVAL, "bad dimensions (need n>=1, n_obs>=0, m>=2, nv>=6, stages>=1)");
  if (nv > 16) return fail(ST_EUNSUPPORTED, "n_coeffs must be <= 16 (degree <= 15)");
  if (!P || !G || !Gm || !F || !Fm || !E || !rho) return fail(ST_EINVAL, "NULL operator pointer");
  int ndev = 0;
  ST_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(ST_EINVAL, "device ordinal out of range");
  ST_CUDA(cudaSetDevice(device));
  st_plan* pl = new st_plan();
  pl->n = n; pl->nobs = nobs; pl->m = m; pl->nv = nv; pl->S = S; pl->device = device;
  const int NV = nv <= 12 ? 12 : 16;
  pl->nvmax = NV;
  const size_t nP = (size_t)m * NV, nG = (size_t)S * NV * NV, nF = (size_t)S * NV * 6, nE = 6 * (size_t)NV;
  const size_t total = nP + 2 * nG + 2 * nF + nE + S;
  std::vector<double> h(total, 0.0);
  size_t o = 0;
  // copy a (count x rows x cols) block into a zero-padded (count x prow x pcol) one
  auto put = [&](const double* src, int count, int rows, int cols, int prow, int pcol) {
    for (int b = 0; b < count; ++b)
      for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) h[o + ((size_t)b * prow + r) * pcol + c] = src[((size_t)b * rows + r) * cols + c];
    o += (size_t)count * prow * pcol;
  };
  put(P, 1, m, nv, m, NV);
  put(G, S, nv, nv, NV, NV);
  put(Gm, S, nv, nv, NV, NV);
  put(F, S, nv, 6, NV, 6);
  put(Fm, S, nv, 6, NV, 6);
  put(E, 1, 6, nv, 6, NV);
  put(rho, 1, 1, S, 1, S);
  // per-stage packed shared-memory image: G Gm F Fm EG EGm EF EFm rho 1/rho (StageMats layout)
  const int MS = NV == 12 ? swarm::StageMats<12>::SIZE : swarm::StageMats<16>::SIZE;
  const int oG = 0, oGm = NV * NV, oF = 2 * NV * NV, oFm = oF + NV * 6, oEG = oFm + NV * 6, oEGm = oEG + 6 * NV,
            oEF = oEGm + 6 * NV, oEFm = oEF + 36, oR = oEFm + 36;
  h.resize(total + (size_t)S * MS + S, 0.0);
  for (int st = 0; st < S; ++st) {
    double* d = h.data() + total + (size_t)st * MS;
    const double* g = G + (size_t)st * nv * nv;
    const double* gm = Gm + (size_t)st * nv * nv;
    const double* f = F + (size_t)st * nv * 6;
    const double* fm = Fm + (size_t)st * nv * 6;
    for (int a = 0; a < nv; ++a) {
      for (int b = 0; b < nv; ++b) { d[oG + a * NV + b] = g[a * nv + b]; d[oGm + a * NV + b] = gm[a * nv + b]; }
      for (int e = 0; e < 6; ++e) { d[oF + a * 6 + e] = f[a * 6 + e]; d[oFm + a * 6 + e] = fm[a * 6 + e]; }
    }
    for (int e = 0; e < 6; ++e) {
      for (int b = 0; b < nv; ++b) {
        double sg = 0.0, sgm = 0.0;
        for (int a = 0; a < nv; ++a) { sg += E[e * nv + a] * g[a * nv + b]; sgm += E[e * nv + a] * gm[a * nv + b]; }
        d[oEG + e * NV + b] = sg;
        d[oEGm + e * NV + b] = sgm;
      }
      for (int f2 = 0; f2 < 6; ++f2) {
        double sf = 0.0, sfm = 0.0;
        for (int a = 0; a < nv; ++a) { sf += E[e * nv + a] * f[a * 6 + f2]; sfm += E[e * nv + a] * fm[a * 6 + f2]; }
        d[oEF + e * 6 + f2] = sf;
        d[oEFm + e * 6 + f2] = sfm;
      }
    }
    d[oR] = rho[st];
    d[oR + 1] = 1.0 / rho[st];
    h[total + (size_t)S * MS + st] = 1.0 / rho[st];
  }
  const size_t total_all = h.size();
  auto cleanup = [&](int code) {
    if (pl->d_mats) cudaFree(pl->d_mats);
    if (pl->d_counter) cudaFree(pl->d_counter);
    if (pl->stream) cudaStreamDestroy(pl->stream);
    delete pl;
    return code;
  };
  cudaError_t e = cudaMalloc(&pl->d_mats, total_all * sizeof(double));
  if (e == cudaSuccess) e = cudaMemcpy(pl->d_mats, h.data(), total_all * sizeof(double), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&pl->d_counter, sizeof(int));
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&pl->stream, cudaStreamNonBlocking);
  for (int i = 0; i < 4 && e == cudaSuccess; ++i) e = cudaEventCreate(&pl->ev[i]);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&pl->ev_done, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&pl->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&pl->smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
  if (e != cudaSuccess) {
    fail(e == cudaErrorMemoryAllocation ? ST_ENOMEM : ST_ECUDA, std::string("plan upload: ") + cudaGetErrorString(e));
    return cleanup(e == cudaErrorMemoryAllocation ? ST_ENOMEM : ST_ECUDA);
  }
  double* b = pl->d_mats;
  pl->P = b; b += nP;
  pl->G = b; b += nG;
  pl->Gm = b; b += nG;
  pl->F = b; b += nF;
  pl->Fm = b; b += nF;
  pl->E = b; b += nE;
  pl->rho = b; b += S;
  pl->mats = b; b += (size_t)S * MS;
  pl->inv_rho = b;
  *out = pl;
  return ST_OK;
}

int st_plan_destroy(st_plan* pl) {
  if (!pl) return ST_OK;
  cudaSetDevice(pl->device);
  if (pl->stream) cudaStreamSynchronize(pl->stream);
  for (auto& e : pl->ev)
    if (e) cudaEventDestroy(e);
  if (pl->ev_done) {
    cudaEventSynchronize(pl->ev_done);
    cudaEventDestroy(pl->ev_done);
  }
  if (pl->d_mats) cudaFree(pl->d_mats);
  if (pl->d_counter) cudaFree(pl->d_counter);
  if (pl->d_lam) cudaFree(pl->d_lam);
  if (pl->d_cws) cudaFree(pl->d_cws);
  if (pl->d_rg) cudaFree(pl->d_rg);
  if (pl->d_io) cudaFree(pl->d_io);
  if (pl->h_stage) cudaFreeHost(pl->h_stage);
  if (pl->d_lgw) cudaFree(pl->d_lgw);
  if (pl->d_rep) cudaFree(pl->d_rep);
  if (pl->stream) cudaStreamDestroy(pl->stream);
  delete pl;
  return ST_OK;
}

int st_query_launch(st_plan* pl, int batch, int hint, int flags, long long* out8) {
  if (!pl || !out8 || batch < 1) return fail(ST_EINVAL, "bad arguments");
  std::lock_guard<std::mutex> g(pl->mu);
  ST_CUDA(cudaSetDevice(pl->device));
  Launch L;
  int rc = choose_launch(pl, batch, hint, (flags & ST_FLAG_KEEP_STATE) != 0, L, 1, (flags & ST_FLAG_FP32) != 0);
  if (rc) return rc;
  out8[0] = L.C; out8[1] = L.NB; out8[2] = L.W; out8[3] = L.NT;
  out8[4] = L.lam_smem; out8[5] = (long long)L.smem_bytes; out8[6] = L.nclusters; out8[7] = L.nsteps;
  return ST_OK;
}

int st_solve_device(st_plan* pl, int batch, const double* c0, const double* beq, const double* geom,
                    int switch_every, int max_iters, double tol, int flags, int hint, double* c_out,
                    double* hist, int* iters, int* conv, double* lam_out, double* d_out, void* stream) {
  int rc = check_common(pl, batch, switch_every, max_iters, tol, flags);
  if (rc) return rc;
  if (!c0 || !beq || !geom || !c_out || !hist || !iters || !conv) return fail(ST_EINVAL, "NULL buffer");
  if ((flags & ST_FLAG_KEEP_STATE) && (!lam_out || !d_out)) return fail(ST_EINVAL, "keep_state buffers missing");
  std::lock_guard<std::mutex> g(pl->mu);
  ST_CUDA(cudaSetDevice(pl->device));
  cudaStream_t s = stream ? (cudaStream_t)stream : pl->stream;
  if (hint <= 0 && large_eligible(pl, batch, (flags & ST_FLAG_KEEP_STATE) != 0))
    return run_large(pl, (flags & ST_FLAG_FP32) != 0, c0, beq, geom, switch_every, max_iters, tol, c_out, hist,
                     iters, conv, s, nullptr);
  Launch L;
  rc = choose_launch_cached(pl, batch, hint, (flags & ST_FLAG_KEEP_STATE) != 0, L, 1, (flags & ST_FLAG_FP32) != 0);
  if (rc) return rc;
  return run(pl, L, batch, c0, beq, geom, switch_every, max_iters, tol, flags, c_out, hist, iters, conv, lam_out,
             d_out, s);
}

static int solve_host(st_plan* pl, int batch, const double* c0, const double* beq, const double* geom, int switch_every,
             int max_iters, double tol, int flags, int hint, double* c_out, double* hist, int* iters, int* conv,
             double* lam_out, double* d_out, float* timings, const ShardExt* ext, const ReportReq* rep = nullptr,
             bool async_ = false) {
  int rc = check_common(pl, batch, switch_every, max_iters, tol, flags);
  if (rc) return rc;
  if (!c0 || !beq || !geom || !c_out || !hist || !iters || !conv) return fail(ST_EINVAL, "NULL buffer");
  const bool keep = flags & ST_FLAG_KEEP_STATE;
  if (keep && (!lam_out || !d_out)) return fail(ST_EINVAL, "keep_state buffers missing");
  std::lock_guard<std::mutex> g(pl->mu);
  if (pl->async_pending) return fail(ST_EINVAL, "a solve begun on this plan has not ended (st_solve_end)");
  ST_CUDA(cudaSetDevice(pl->device));
  const bool large = hint <= 0 && large_eligible(pl, batch, keep);
  Launch L;
  if (!large) {
    rc = choose_launch_cached(pl, batch, hint, keep, L, ext ? ext->G : 1, (flags & ST_FLAG_FP32) != 0);
    if (rc) return rc;
  }
  const int n = pl->n, nv = pl->nv, m = pl->m;
  const long long p = (long long)n * (n - 1) / 2 + (long long)n * pl->nobs;
  const size_t n_c = (size_t)batch * 3 * n * nv, n_b = (size_t)batch * 3 * n * 6,
               n_g = (size_t)batch * (2 + 5 * pl->nobs), n_h = (size_t)batch * 3 * max_iters;
  const size_t n_lam = keep ? (size_t)3 * p * m : 0, n_d = keep ? (size_t)p * m : 0;
  const size_t in_bytes = (n_c + n_b + n_g) * 8;
  const size_t out_bytes = (n_c + n_h + n_lam + n_d) * 8 + 2 * (size_t)batch * 4;
  const size_t need = in_bytes + out_bytes + 64;
  if (need > pl->io_bytes) {
    if (pl->d_io) cudaFree(pl->d_io);
    pl->d_io = nullptr;
    pl->io_bytes = 0;
    ST_CUDA(cudaMalloc(&pl->d_io, need));
    pl->io_bytes = need;
  }
  double* d = (double*)pl->d_io;
  double *d_c0 = d, *d_beq = d_c0 + n_c, *d_geom = d_beq + n_b, *d_cout = d_geom + n_g, *d_hist = d_cout + n_c;
  double *d_lam = d_hist + n_h, *d_dd = d_lam + n_lam;
  int* d_it = (int*)(d_dd + n_d);
  int* d_cv = d_it + batch;
  cudaStream_t s = pl->stream;
  // small solves (single scenarios): inputs and the small outputs go through one page-locked
  // staging buffer -- one H2D and one D2H instead of a pageable copy per array
  const size_t small_out = (n_c + n_h) * 8 + 2 * (size_t)batch * 4 + (rep ? (size_t)batch * (2 * n + 2) * 8 : 0);
  // the report pass's collision inputs (per-scenario geometry and obstacle rows) ride in the same
  // staging buffer, right after the solve inputs (a pageable copy would block the host)
  const bool rep_verdict = rep && (rep->min_dist || rep->n_viol);
  const size_t rep_in = rep_verdict ? (size_t)batch * 16 + (size_t)batch * pl->nobs * 40 : 0;
  const bool staged = !keep && !async_ && in_bytes + rep_in + small_out <= ((size_t)1 << 20);
  if (staged && in_bytes + rep_in + small_out > pl->stage_bytes) {
    if (pl->h_stage) cudaFreeHost(pl->h_stage);
    pl->h_stage = nullptr;
    pl->stage_bytes = 0;
    ST_CUDA(cudaHostAlloc(&pl->h_stage, (size_t)1 << 20, cudaHostAllocPortable));
    pl->stage_bytes = (size_t)1 << 20;
  }
  double* hs = staged ? (double*)pl->h_stage : nullptr;
  ST_CUDA(cudaEventRecord(pl->ev[0], s));
  if (staged) {
    memcpy(hs, c0, n_c * 8);
    memcpy(hs + n_c, beq, n_b * 8);
    memcpy(hs + n_c + n_b, geom, n_g * 8);
    if (rep_verdict) {
      memcpy((char*)hs + in_bytes, rep->geom2, (size_t)batch * 16);
      if (pl->nobs) memcpy((char*)hs + in_bytes + (size_t)batch * 16, rep->obs, (size_t)batch * pl->nobs * 40);
    }
    ST_CUDA(cudaMemcpyAsync(d_c0, hs, in_bytes, cudaMemcpyHostToDevice, s));
  } else {
    ST_CUDA(cudaMemcpyAsync(d_c0, c0, n_c * 8, cudaMemcpyHostToDevice, s));
    ST_CUDA(cudaMemcpyAsync(d_beq, beq, n_b * 8, cudaMemcpyHostToDevice, s));
    ST_CUDA(cudaMemcpyAsync(d_geom, geom, n_g * 8, cudaMemcpyHostToDevice, s));
  }
  ST_CUDA(cudaEventRecord(pl->ev[1], s));
  rc = large ? run_large(pl, (flags & ST_FLAG_FP32) != 0, d_c0, d_beq, d_geom, switch_every, max_iters, tol, d_cout,
                         d_hist, d_it, d_cv, s, ext)
             : run(pl, L, batch, d_c0, d_beq, d_geom, switch_every, max_iters, tol, flags, d_cout, d_hist, d_it, d_cv,
                   keep ? d_lam : nullptr, keep ? d_dd : nullptr, s, ext);
  if (rc) return rc;
  ST_CUDA(cudaEventRecord(pl->ev[2], s));
  bool verdict_out = false;
  const double* rep_small = nullptr;  // device: arc | smooth | min bits | counts (report pass)
  if (rep) {
    // report pass on the device: trajectories, arc length / smoothness, collision summary
    const int n_obs = pl->nobs;
    const long long n_rows = (long long)n * (n - 1) / 2 + (long long)n * n_obs;
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t b_traj = al((size_t)batch * n * m * 24), b_met = al((size_t)batch * n * 16),
                 b_geom = al((size_t)batch * 16), b_obs = al((size_t)batch * n_obs * 40 + 8),
                 b_cnt = al((size_t)batch * n_rows * 4 + 4), b_mt = al((size_t)batch * 16);
    (void)b_met;
    const size_t b_small = al((size_t)batch * (2 * n + 2) * 8);  // arc | smooth | min bits | counts
    const size_t rneed = b_traj + b_small + b_geom + b_obs + b_cnt;
    if (rneed > pl->rep_bytes) {
      if (pl->d_rep) cudaFree(pl->d_rep);
      pl->d_rep = nullptr;
      pl->rep_bytes = 0;
      ST_CUDA(cudaMalloc(&pl->d_rep, rneed));
      pl->rep_bytes = rneed;
    }
    char* q = (char*)pl->d_rep;
    double* r_traj = (double*)q;
    double* r_arc = (double*)(q += b_traj);
    double* r_smooth = r_arc + (size_t)batch * n;
    unsigned long long* r_mt = (unsigned long long*)(r_smooth + (size_t)batch * n);
    double* r_geom = (double*)(q += b_small);
    double* r_obs = (double*)(q += b_geom);
    int* r_cnt = (int*)(q += b_obs);
    rep_small = r_arc;
    const bool verdict = rep->min_dist || rep->n_viol;
    if (verdict) {
      const char* g2 = staged ? (const char*)hs + in_bytes : (const char*)rep->geom2;  // page-locked when staged
      ST_CUDA(cudaMemcpyAsync(r_geom, g2, (size_t)batch * 16, cudaMemcpyHostToDevice, s));
      if (n_obs)
        ST_CUDA(cudaMemcpyAsync(r_obs, staged ? g2 + (size_t)batch * 16 : (const char*)rep->obs,
                                (size_t)batch * n_obs * 40, cudaMemcpyHostToDevice, s));
    }
    ST_CUDA(swarm_report_launch(batch, n, m, nv, pl->nvmax, d_cout, pl->P, r_traj, r_arc, r_smooth,
                                verdict ? r_mt : nullptr, s));
    if (verdict) {
      // r_mt: the minimum normalized distance's bits (non-negative doubles order as integers) |
      // violation counts (64-bit) -- copied bit for bit into min_dist / n_viol
      ST_CUDA(swarm_collision_summary_launch(batch, n, m, r_traj, r_geom, n_obs, r_obs, r_cnt, r_mt, s, false));
      verdict_out = true;
      if (!staged) {
        if (rep->min_dist)
          ST_CUDA(cudaMemcpyAsync(rep->min_dist, r_mt, (size_t)batch * 8, cudaMemcpyDeviceToHost, s));
        if (rep->n_viol)
          ST_CUDA(cudaMemcpyAsync(rep->n_viol, r_mt + batch, (size_t)batch * 8, cudaMemcpyDeviceToHost, s));
      }
    }
    if (rep->traj) ST_CUDA(cudaMemcpyAsync(rep->traj, r_traj, (size_t)batch * n * m * 24, cudaMemcpyDeviceToHost, s));
    if (!staged) {
      if (rep->arc) ST_CUDA(cudaMemcpyAsync(rep->arc, r_arc, (size_t)batch * n * 8, cudaMemcpyDeviceToHost, s));
      if (rep->smooth)
        ST_CUDA(cudaMemcpyAsync(rep->smooth, r_smooth, (size_t)batch * n * 8, cudaMemcpyDeviceToHost, s));
    }
  }
  // output region of d_io: c | hist | (lam | d) | iters | converged
  const size_t out_small = (n_c + n_h) * 8 + 2 * (size_t)batch * 4;
  if (staged) {
    ST_CUDA(cudaMemcpyAsync(hs, d_cout, out_small, cudaMemcpyDeviceToHost, s));
    if (rep) ST_CUDA(cudaMemcpyAsync((char*)hs + out_small, rep_small, (size_t)batch * (2 * n + 2) * 8,
                                     cudaMemcpyDeviceToHost, s));
  } else {
    ST_CUDA(cudaMemcpyAsync(c_out, d_cout, n_c * 8, cudaMemcpyDeviceToHost, s));
    ST_CUDA(cudaMemcpyAsync(hist, d_hist, n_h * 8, cudaMemcpyDeviceToHost, s));
    ST_CUDA(cudaMemcpyAsync(iters, d_it, batch * 4, cudaMemcpyDeviceToHost, s));
    ST_CUDA(cudaMemcpyAsync(conv, d_cv, batch * 4, cudaMemcpyDeviceToHost, s));
  }
  if (keep) {
    ST_CUDA(cudaMemcpyAsync(lam_out, d_lam, n_lam * 8, cudaMemcpyDeviceToHost, s));
    ST_CUDA(cudaMemcpyAsync(d_out, d_dd, n_d * 8, cudaMemcpyDeviceToHost, s));
  }
  ST_CUDA(cudaEventRecord(pl->ev[3], s));
  if (async_) {  // st_solve_report_begin: every copy targets page-locked memory; st_solve_end waits
    pl->async_pending = true;
    return ST_OK;
  }
  ST_CUDA(cudaStreamSynchronize(s));
  ST_CUDA(cudaGetLastError());
  if (timings) {
    ST_CUDA(cudaEventElapsedTime(&timings[0], pl->ev[0], pl->ev[1]));
    ST_CUDA(cudaEventElapsedTime(&timings[1], pl->ev[1], pl->ev[2]));
    ST_CUDA(cudaEventElapsedTime(&timings[2], pl->ev[2], pl->ev[3]));
  }
  if (staged) {
    const char* o = (const char*)hs;
    memcpy(c_out, o, n_c * 8);
    memcpy(hist, o + n_c * 8, n_h * 8);
    memcpy(iters, o + (n_c + n_h) * 8, (size_t)batch * 4);
    memcpy(conv, o + (n_c + n_h) * 8 + (size_t)batch * 4, (size_t)batch * 4);
    if (rep) {
      const char* r = o + out_small;
      if (rep->arc) memcpy(rep->arc, r, (size_t)batch * n * 8);
      if (rep->smooth) memcpy(rep->smooth, r + (size_t)batch * n * 8, (size_t)batch * n * 8);
      if (verdict_out) {
        if (rep->min_dist) memcpy(rep->min_dist, r + (size_t)batch * 2 * n * 8, (size_t)batch * 8);
        if (rep->n_viol) memcpy(rep->n_viol, r + (size_t)batch * (2 * n + 1) * 8, (size_t)batch * 8);
      }
    }
  }
  return ST_OK;
}

int st_solve(st_plan* pl, int batch, const double* c0, const double* beq, const double* geom, int switch_every,
             int max_iters, double tol, int flags, int hint, double* c_out, double* hist, int* iters, int* conv,
             double* lam_out, double* d_out, float* timings) {
  return solve_host(pl, batch, c0, beq, geom, switch_every, max_iters, tol, flags, hint, c_out, hist, iters, conv,
                    lam_out, d_out, timings, nullptr);
}

int st_solve_report(st_plan* pl, int batch, const double* c0, const double* beq, const double* geom,
                    int switch_every, int max_iters, double tol, int flags, int hint, double* c_out, double* hist,
                    int* iters, int* conv, float* timings, const double* col_geom, const double* col_obs,
                    double* traj, double* arc, double* smooth, double* min_dist, long long* n_viol) {
  if (!pl) return fail(ST_EINVAL, "NULL plan");
  if ((min_dist || n_viol) && (!col_geom || (pl->nobs > 0 && !col_obs)))
    return fail(ST_EINVAL, "collision geometry missing");
  if (batch > 65535) return fail(ST_EINVAL, "report pass: batch larger than 65535 scenarios");
  if (pl->m < 1 || swarm_report_smem(pl->m) > (size_t)pl->smem_optin)
    return fail(ST_EUNSUPPORTED, "report pass: too many samples per trajectory for one warp's shared memory");
  if (flags & ST_FLAG_KEEP_STATE) return fail(ST_EINVAL, "report pass: keep_state solves use st_solve");
  const ReportReq rep{col_geom, col_obs, traj, arc, smooth, min_dist, n_viol};
  return solve_host(pl, batch, c0, beq, geom, switch_every, max_iters, tol, flags, hint, c_out, hist, iters, conv,
                    nullptr, nullptr, timings, nullptr, &rep);
}

int st_solve_report_begin(st_plan* pl, int batch, const double* c0, const double* beq, const double* geom,
                          int switch_every, int max_iters, double tol, int flags, int hint, double* c_out,
                          double* hist, int* iters, int* conv, const double* col_geom, const double* col_obs,
                          double* traj, double* arc, double* smooth, double* min_dist, long long* n_viol) {
  if (!pl) return fail(ST_EINVAL, "NULL plan");
  if ((min_dist || n_viol) && (!col_geom || (pl->nobs > 0 && !col_obs)))
    return fail(ST_EINVAL, "collision geometry missing");
  if (batch > 65535) return fail(ST_EINVAL, "report pass: batch larger than 65535 scenarios");
  if (pl->m < 1 || swarm_report_smem(pl->m) > (size_t)pl->smem_optin)
    return fail(ST_EUNSUPPORTED, "report pass: too many samples per trajectory for one warp's shared memory");
  if (flags & ST_FLAG_KEEP_STATE) return fail(ST_EINVAL, "report pass: keep_state solves use st_solve");
  const ReportReq rep{col_geom, col_obs, traj, arc, smooth, min_dist, n_viol};
  return solve_host(pl, batch, c0, beq, geom, switch_every, max_iters, tol, flags, hint, c_out, hist, iters, conv,
                    nullptr, nullptr, nullptr, nullptr, &rep, true);
}

int st_solve_end(st_plan* pl, float* timings) {
  if (!pl) return fail(ST_EINVAL, "NULL plan");
  std::lock_guard<std::mutex> g(pl->mu);
  if (!pl->async_pending) return fail(ST_EINVAL, "no solve begun on this plan");
  pl->async_pending = false;
  ST_CUDA(cudaSetDevice(pl->device));
  ST_CUDA(cudaEventSynchronize(pl->ev[3]));
  ST_CUDA(cudaGetLastError());
  if (timings) {
    ST_CUDA(cudaEventElapsedTime(&timings[0], pl->ev[0], pl->ev[1]));
    ST_CUDA(cudaEventElapsedTime(&timings[1], pl->ev[1], pl->ev[2]));
    ST_CUDA(cudaEventElapsedTime(&timings[2], pl->ev[2], pl->ev[3]));
  }
  return ST_OK;
}

// Page-locked host buffers (report outputs): device-to-host copies at full PCIe/C2C speed.
int st_host_alloc(long long bytes, void** out) {
  if (!out || bytes < 0) return fail(ST_EINVAL, "bad arguments");
  *out = nullptr;
  if (bytes == 0) return ST_OK;
  ST_CUDA(cudaHostAlloc(out, (size_t)bytes, cudaHostAllocPortable));
  return ST_OK;
}

int st_host_free(void* ptr) {
  if (ptr) ST_CUDA(cudaFreeHost(ptr));
  return ST_OK;
}

// ---- pair-sharded solves over G GPUs (one process per GPU, peer-mapped group buffers)

int st_shard_layout(st_plan* pl, int G, long long* out4) {
  if (!pl || !out4 || G < 1 || G > 8) return fail(ST_EINVAL, "bad arguments (G must be 1..8)");
  std::lock_guard<std::mutex> g(pl->mu);
  ST_CUDA(cudaSetDevice(pl->device));
  if (large_eligible(pl, 1, false)) {
    // large fleets: every GPU runs one CTA per SM over its range of (block pair x sample) units
    for (const auto& e : kLarge) {
      if (e.NVMAX != pl->nvmax || e.f32) continue;
      const int chr = swarm::lg_chunk_rows(false);
      const swarm::LgSmem sm = pl->nvmax == 12 ? swarm::lg_smem<12, false>(pl->m, chr)
                                               : swarm::lg_smem<16, false>(pl->m, chr);
      int grid = 0;
      int rc = large_grid(pl, &e, (size_t)sm.total, grid);
      if (rc) return rc;
      out4[0] = 0;  // no clusters
      out4[1] = grid;
      out4[2] = 64 + 2LL * (3LL * pl->n * pl->nvmax + 4) * (long long)sizeof(double);
      out4[3] = (long long)G * grid;
      return ST_OK;
    }
  }
  Launch L;
  int rc = choose_launch(pl, 1, 0, false, L, G);
  if (rc) return rc;
  const long long stride = 3LL * pl->n * L.NVMAX + 3LL * L.NVMAX + 4;
  out4[0] = L.C;
  out4[1] = L.K;
  out4[2] = 64 + 2LL * L.K * stride * (long long)sizeof(double);
  out4[3] = (long long)L.G * L.K;
  return ST_OK;
}

int st_large_partition(int n, int m, int G, int cpg, int* u_range, int* cta_first, int* rows, int* ab_first) {
  if (n < 2 || m < 1 || G < 1 || cpg < 1) return -fail(ST_EINVAL, "bad arguments");
  st_plan tmp;
  tmp.n = n;
  tmp.m = m;
  const LargeLayout Lg = large_layout(&tmp, G, cpg);
  if (u_range) std::copy(Lg.u_range.begin(), Lg.u_range.end(), u_range);
  if (cta_first) std::copy(Lg.cta_first.begin(), Lg.cta_first.end(), cta_first);
  if (rows) std::copy(Lg.rows.begin(), Lg.rows.end(), rows);
  if (ab_first) std::copy(Lg.ab_first.begin(), Lg.ab_first.end(), ab_first);
  return Lg.U;
}

int st_shard_buffer(st_plan* pl, long long bytes, void** dptr, unsigned char* handle64) {
  if (!pl || !dptr || !handle64 || bytes < 64) return fail(ST_EINVAL, "bad arguments");
  ST_CUDA(cudaSetDevice(pl->device));
  ST_CUDA(cudaMalloc(dptr, (size_t)bytes));
  ST_CUDA(cudaMemset(*dptr, 0, (size_t)bytes));
  cudaIpcMemHandle_t h;
  ST_CUDA(cudaIpcGetMemHandle(&h, *dptr));
  std::memcpy(handle64, &h, sizeof(h) < 64 ? sizeof(h) : 64);
  return ST_OK;
}

int st_shard_open(st_plan* pl, const unsigned char* handle64, void** dptr) {
  if (!pl || !dptr || !handle64) return fail(ST_EINVAL, "bad arguments");
  ST_CUDA(cudaSetDevice(pl->device));
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof(h));
  ST_CUDA(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
  return ST_OK;
}

int st_shard_close(st_plan* pl, void* dptr, int opened) {
  if (!pl || !dptr) return ST_OK;
  cudaSetDevice(pl->device);
  if (opened) cudaIpcCloseMemHandle(dptr);
  else cudaFree(dptr);
  return ST_OK;
}

int st_shard_reset(st_plan* pl, void* buf0) {
  if (!pl || !buf0) return fail(ST_EINVAL, "bad arguments");
  ST_CUDA(cudaSetDevice(pl->device));
  ST_CUDA(cudaMemset(buf0, 0, 64));
  ST_CUDA(cudaDeviceSynchronize());
  return ST_OK;
}

int st_solve_sharded(st_plan* pl, int G, int rank, void* const* bufs, const double* c0, const double* beq,
                     const double* geom, int switch_every, int max_iters, double tol, double* c_out, double* hist,
                     int* iters, int* conv, float* timings) {
  if (!pl || !bufs || G < 1 || G > 8 || rank < 0 || rank >= G) return fail(ST_EINVAL, "bad shard arguments");
  ShardExt ext;
  ext.G = G;
  ext.rank = rank;
  for (int g = 0; g < 8; ++g) ext.bufs[g] = g < G ? bufs[g] : nullptr;
  for (int g = 0; g < G; ++g)
    if (!ext.bufs[g]) return fail(ST_EINVAL, "NULL group buffer");
  return solve_host(pl, 1, c0, beq, geom, switch_every, max_iters, tol, 0, 0, c_out, hist, iters, conv, nullptr,
                    nullptr, timings, &ext);
}

}  // extern "C"
