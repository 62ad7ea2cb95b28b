/*
 * swarm_am.h -- C ABI of the B200 alternating-minimization (AM) joint
 * multi-agent trajectory solver (drop-in for the reference's solve path).
 *
 * The reference (pkg/src/swarmtraj, pure Python) has no FFI; its seams are
 * Python calls.  Each entry point below replaces one of them:
 *
 *   st_plan_create   <- FactorCache.prefactorize + KktFactor construction
 *                       (kkt_cache.py:332-353, 421-456): uploads the per-stage
 *                       structured KKT operators (kkt.py) once per fingerprint.
 *   st_solve         <- am_solve's loop (solver.py:405-457) for one scenario or a
 *                       batch sharing one fingerprint (bench.py:120-158 runs the
 *                       same batch through threads).  Host buffers in/out.
 *   st_solve_device  <- same, device buffers, caller's stream (HBM-resident batches).
 *   st_plan_destroy  <- releasing a cache entry.
 *   st_last_error    <- the ValueError/RuntimeError text of the failed call.
 *
 * Conventions: all arrays are C-contiguous float64 (or int32), caller-owned.
 * Layouts follow the reference: coefficients (3, n, nv) per scenario
 * (SolveReport.coefficients, solver.py:146), boundary rows (3, n, 6) in the
 * order [pos0, vel0, acc0, posT, velT, accT] (kkt_cache.py:174-185),
 * multipliers (3, p, m) pair-major with agent pairs (i<j) lexicographic then
 * (agent, obstacle) agent-major (kkt_cache.py:197-215).
 * Return value: 0 ok; ST_EINVAL bad argument; ST_ECUDA CUDA failure;
 * ST_ENOMEM device allocation failure; ST_EUNSUPPORTED shape outside the
 * compiled kernels.  Plans are safe to share between threads: host calls on one
 * plan serialize on its mutex, and every launch on a plan is ordered after the
 * previous one on the device (an event), whatever stream the caller passes, so
 * solves sharing the plan's workspaces never overlap.
 */
#ifndef SWARM_AM_H
#define SWARM_AM_H

#ifdef __cplusplus
extern "C" {
#endif

#define ST_OK 0
#define ST_EINVAL 1
#define ST_ECUDA 2
#define ST_ENOMEM 3
#define ST_EUNSUPPORTED 4

#define ST_FLAG_KEEP_STATE 1 /* write final multipliers/d (batch must be 1) */
#define ST_FLAG_FP32 2       /* FP32 pair state: multipliers and pair arithmetic in FP32,
                                positions, right-hand-side sums and the KKT solve in FP64
                                (north star's optional FP32 mode; tolerances in DESIGN.md §8) */

/* Per-scenario status written to converged[]: */
#define ST_CONVERGED 1
#define ST_NOT_CONVERGED 0
#define ST_NONFINITE (-1) /* the pair state became NaN/inf: where the reference's
                             _check_ranges assertion fires (solver.py:355-360) */

typedef struct st_plan st_plan;

/* Per-fingerprint operators.  P: m x nv sampled basis.  For each of the
 * n_stages rho values: G, Gm (nv x nv) and F, Fm (nv x 6) -- see kkt.py for
 * their definition from the 17x17 K_dev / K_mean blocks.  E: 6 x nv endpoint
 * rows.  rho: n_stages penalty weights.  device: CUDA ordinal. */
int st_plan_create(int n_agents, int n_obstacles, int n_samples, int n_coeffs, int n_stages,
                   const double* P, const double* G, const double* Gm, const double* F,
                   const double* Fm, const double* E, const double* rho, int device,
                   st_plan** out);

int st_plan_destroy(st_plan* plan);

/* Solve `batch` scenarios (host pointers).
 *   c0     batch x 3 x n x nv   straight-line initial coefficients
 *   b_eq   batch x 3 x n x 6    boundary rows
 *   geom   batch x (2 + 5*n_obs): agent l_xy, l_z, then per obstacle
 *          (cx, cy, cz, l_xy, l_z) with the agent-obstacle semi-axes
 *   switch_every, max_iters, tol: the rho schedule and stopping rule
 *   cluster_hint: CTAs per scenario (0 = choose)
 * Outputs: c_out (batch x 3 x n x nv), hist (batch x 3 x max_iters:
 * residual norm, residual max-abs, boundary max per iteration), iters,
 * converged (batch: ST_CONVERGED / ST_NOT_CONVERGED / ST_NONFINITE).
 * lam_out (3 x p x m) and d_out (p x m) only with
 * ST_FLAG_KEEP_STATE, else may be NULL.  timings_ms (may be NULL):
 * [h2d, device loop, d2h]. */
int st_solve(st_plan* plan, int batch, const double* c0, const double* b_eq, const double* geom,
             int switch_every, int max_iters, double tol, int flags, int cluster_hint,
             double* c_out, double* hist, int* iters, int* converged, double* lam_out,
             double* d_out, float* timings_ms);

/* st_solve plus the report's post-loop work in the same call, on the device (replaces
 * SolveReport.trajectories = c_axis @ P.T, solver.py:133-136, and _final_metrics,
 * solver.py:497-509 -> validation.py:39-132): keep_state is not available here.
 *   traj     batch x n x m x 3   sampled positions (report layout)
 *   arc      batch x n           arc length per agent (validation.py:96-108)
 *   smooth   batch x n           smoothness per agent (validation.py:111-121)
 *   min_dist batch               minimum normalized distance (+inf without rows)
 *   n_viol   batch               number of violations (< 1) of the collision check
 *   col_geom batch x 2 (l_xy, l_z) and col_obs batch x n_obs x 5 as for
 *            st_check_collisions_batch (needed for min_dist / n_viol).
 * Any of the five outputs may be NULL.  The verdict is computed on the device
 * trajectories; positions and sums use a fixed FMA/summation order (agreement with
 * the host formulas to rounding). */
int st_solve_report(st_plan* plan, int batch, const double* c0, const double* b_eq, const double* geom,
                    int switch_every, int max_iters, double tol, int flags, int cluster_hint, double* c_out,
                    double* hist, int* iters, int* converged, float* timings_ms, const double* col_geom,
                    const double* col_obs, double* traj, double* arc, double* smooth, double* min_dist,
                    long long* n_viol);

/* st_solve_report in two halves, for pipelining host work against the device: _begin copies
 * the inputs and enqueues the solve, the report pass and every output copy, and returns;
 * st_solve_end waits for them and returns the timings.  Output arrays must be page-locked
 * (st_host_alloc) or _begin blocks until the device is done.  One begun solve per plan:
 * every other host-pointer call on the plan fails (ST_EINVAL) until st_solve_end. */
int st_solve_report_begin(st_plan* plan, int batch, const double* c0, const double* b_eq, const double* geom,
                          int switch_every, int max_iters, double tol, int flags, int cluster_hint,
                          double* c_out, double* hist, int* iters, int* converged, const double* col_geom,
                          const double* col_obs, double* traj, double* arc, double* smooth, double* min_dist,
                          long long* n_viol);
int st_solve_end(st_plan* plan, float* timings_ms);

/* Page-locked host memory for output arrays (device-to-host copies at full link speed;
 * the Python binding pools these buffers for the report outputs). */
int st_host_alloc(long long bytes, void** out);
int st_host_free(void* ptr);

/* Same contract, every array a device pointer, enqueued on `stream`
 * (a cudaStream_t, NULL = the plan's stream); no host synchronization. */
int st_solve_device(st_plan* plan, int batch, const double* c0, const double* b_eq,
                    const double* geom, int switch_every, int max_iters, double tol, int flags,
                    int cluster_hint, double* c_out, double* hist, int* iters, int* converged,
                    double* lam_out, double* d_out, void* stream);

/* ---- Pair-sharded solve of ONE large scenario over G GPUs (BASELINE config 5).
 * Replaces nothing in the reference (single process, CPU); it is the north star's
 * "very large n shards the agent pairs across GPUs".  For n > 64 (the large-fleet
 * kernel) the work units are (agent-block pair x time sample x half) in block-pair-major
 * order and every GPU owns a contiguous, cost-balanced range of them -- a range of agent
 * pairs of the upper triangle at all samples -- run by one CTA per SM.  Each GPU reduces
 * its units to one partial right-hand-side row set (3 x n x n_v doubles) plus its residual
 * norms; the one per-iteration exchange of those goes through peer-mapped buffers inside
 * the persistent kernel and is summed in rank order (identical on every GPU).  (n <= 64:
 * the multi-cluster kernel, every GPU a slice of the time samples.)  One process per GPU:
 *   st_shard_layout  -> cluster size, clusters per GPU, buffer bytes, participants
 *   st_shard_buffer  -> allocate this GPU's buffer and export its IPC handle
 *   st_shard_open    -> map a peer's buffer (cudaIpcOpenMemHandle)
 *   st_shard_reset   -> rank 0 zeroes the barrier word (host barrier before launching)
 *   st_solve_sharded -> every rank launches; outputs are written on rank 0 */
int st_shard_layout(st_plan* plan, int G, long long* out4);
int st_shard_buffer(st_plan* plan, long long bytes, void** dptr, unsigned char* handle64);
int st_shard_open(st_plan* plan, const unsigned char* handle64, void** dptr);
int st_shard_close(st_plan* plan, void* dptr, int opened);
int st_shard_reset(st_plan* plan, void* buf0);
int st_solve_sharded(st_plan* plan, int G, int rank, void* const* bufs, const double* c0, const double* b_eq,
                     const double* geom, int switch_every, int max_iters, double tol, double* c_out,
                     double* hist, int* iters, int* converged, float* timings_ms);

/* Host-only (no device needed): the large-fleet unit partition for n agents, m samples,
 * G GPUs of cpg CTAs.  Fills (when non-NULL) u_range[G+1] (GPU g owns units
 * [u_range[g], u_range[g+1])), cta_first[G*(cpg+1)], rows[U] (pair steps per unit) and
 * ab_first[nab+1] (first unit of each agent-block pair); returns U, the unit count. */
int st_large_partition(int n, int m, int G, int cpg, int* u_range, int* cta_first, int* rows, int* ab_first);

/* Launch configuration st_solve would use (flags as for st_solve): out[0..7] =
 * cluster size C, agent blocks NB, lane segment width W, threads per CTA,
 * lambda-in-smem flag, dynamic smem bytes, clusters launched, steps per warp task. */
int st_query_launch(st_plan* plan, int batch, int cluster_hint, int flags, long long* out8);

/* Post-solve safety verdict (replaces validation.py:39-93, check_collisions,
 * called by _final_metrics, solver.py:497-509).  Host buffers.
 *   traj   n x m x 3 sampled positions (SolveReport.trajectories)
 *   obs    n_obs x 5: center x, y, z, l_xy/2 + radius, l_z/2 + radius
 * Rows in the reference order (agent pairs i<j lexicographic, then agent-major
 * (agent, obstacle)), samples in order.  Writes min(total, cap) violations:
 * ids[4e..4e+3] = kind (0 agent pair, 1 obstacle), i, j-or-k, sample;
 * vals[e] = normalized distance (< 1).  *min_out = global minimum (+inf when
 * there are no rows), *total_out = number of violations (may exceed cap; call
 * again with a larger cap for the full list).  Values are bit-identical to
 * the reference's scalar loop. */
int st_check_collisions(int n, int m, const double* traj, double l_xy, double l_z, int n_obs,
                        const double* obs, int device, long long cap, int* ids, double* vals,
                        double* min_out, long long* total_out);

/* The same verdict for B scenarios of one shape in one pass: traj B x n x m x 3,
 * geom B x 2 (l_xy, l_z), obs B x n_obs x 5; min_out[B], total_out[B]; entries
 * scenario-major (scenario b's after those of scenarios < b), min(sum, cap) written. */
int st_check_collisions_batch(int B, int n, int m, const double* traj, const double* geom, int n_obs,
                              const double* obs, int device, long long cap, int* ids, double* vals,
                              double* min_out, long long* total_out);

const char* st_last_error(void);
int st_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SWARM_AM_H */
