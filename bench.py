"""Benchmark: batched AM joint solves on B200 (BASELINE.json metric), one JSON line on rank 0.

Workload (BASELINE.json configs[1] scenarios, batched as configs[3]): a stream of
32-agent random start/goal scenarios, ``generate_random(32, (8,8,3), 0.4, seed)``,
seeds 0..1023, m=100 samples, Bernstein degree 10, default SolverConfig (150
iterations max, tol 1e-2, rho = 2^s over 10 stages), FP64.  One step = solving the
whole batch (every scenario to convergence or max_iters) in one device launch.

* ``value``: solves/s, all ranks, inputs resident in HBM, device time (CUDA events on
  the launch stream, L2 flushed between steps), max over ranks.
* ``e2e``: the same solves through the C ABI ``st_solve`` with host buffers (H2D of the
  packed boundary rows / straight-line coefficients, device loop, D2H of coefficients
  and histories inside the timed region).
* ``roofline``: the AM kernel is the only kernel; FP64 FMA-pipe bound (the pairwise
  update is FP64 arithmetic on on-chip/L2 data).  Algorithmic work per pair-sample per
  iteration = 85 FLOP; peak = measured DFMA throughput
  (profiles/ubench_r1.txt: 64 lanes/clk/SM x 148 SMs x SM clock x 2).
* ``cpu_baseline``: the reference algorithm (oracle/am_oracle.py, numpy/scipy LU path,
  warm factors) on a bounded sample, one process per host core.
* ``fp32``: the same batch in the optional FP32 mode, device time.
* ``python_api``: the same batch through the Python drop-in ``am_solve_batch`` (Python spec
  objects in, SolveReports with metrics out), whole call.
* ``single_solve_ms``: BASELINE's "ms per joint solve at 16/32/64/256 agents" -- circ16j, hall16j (the
  reference CLI's default corridor: 16 agents, 22 wall obstacles),
  rand32_s0, sph64j, rand128_s0, rand256_s0: device loop (best of 3), whole am_solve call,
  FP32 mode, the same-run CPU reference (oracle port, 1 thread; a bounded prefix for
  n > 64) and the loop's roofline fraction.
* Multi-GPU (torchrun): scenarios are independent units, so ranks shard them with no
  data-path collective (NCCL only for the barrier and the max-over-ranks timing).
  Default ``--scaling strong`` (BASELINE config 4 read literally): the one batch of
  ``--batch`` (seeds 0..batch-1) split 1/N per rank; at N=8 each GPU gets 128 scenarios for
  74 two-CTA clusters (two cluster rounds: ~84% of the per-GPU rate at 1024).
  ``--scaling weak``: every rank solves its own batch of ``--batch`` scenarios (rank r:
  seeds r*batch .. (r+1)*batch-1), value = all scenarios / max-over-ranks time.

``--impl reference`` times the reference algorithm on the host cores instead.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
BATCH = 1024
FLOP_PER_PAIR_SAMPLE = 85.0
BYTES_PER_PAIR_SAMPLE = 48.0


def scenarios(lo: int, hi: int):
    from paper_2011_04240_b200 import generate_random
    return [generate_random(32, (8.0, 8.0, 3.0), 0.4, s) for s in range(lo, hi)]


# ---------------------------------------------------------------------------------------------
# CPU reference (oracle port of the reference algorithm), one process per core


def sample_seeds(count: int) -> list[int]:
    """A spread subset of the bench population (seeds 0..BATCH-1), for the bounded CPU samples."""
    count = max(1, min(count, BATCH))
    return sorted({(i * BATCH) // count + (BATCH // count) // 2 for i in range(count)})


def _cpu_worker(seeds):
    # one BLAS thread per worker process (one process per core): numpy may already be loaded in
    # the spawned child, so the limit is set at run time as well as through the environment
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)
    from scipy.linalg import lu_factor

    from oracle import am_oracle
    from paper_2011_04240_b200 import generate_random
    specs = [generate_random(32, (8.0, 8.0, 3.0), 0.4, s) for s in seeds]
    pr = am_oracle.Problem(specs[0])
    rhos, _ = am_oracle.schedule()
    factors = [lu_factor(pr.kkt(r), check_finite=False) for r in rhos]  # warm cache (reference excludes it)
    t0 = time.perf_counter()
    its = 0
    for spec in specs:
        its += am_oracle.solve(spec, factors=factors)["iterations"]
    return time.perf_counter() - t0, len(specs), its


def cpu_reference(n_per_core: int, cores: int | None = None):
    import multiprocessing as mp
    cores = cores or os.cpu_count() or 1
    seeds = sample_seeds(n_per_core * cores)
    jobs = [seeds[i::cores] for i in range(cores) if seeds[i::cores]]
    cores = len(jobs)
    ctx = mp.get_context("spawn")
    t0 = time.perf_counter()
    with ctx.Pool(cores) as pool:
        res = pool.map(_cpu_worker, jobs)
    wall = time.perf_counter() - t0
    solves = sum(r[1] for r in res)
    busy = max(r[0] for r in res)
    return {"solves_per_s": solves / busy, "wall_s": wall, "solves": solves, "cores": cores,
            "mean_iters": sum(r[2] for r in res) / solves}


# ---------------------------------------------------------------------------------------------


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self._p = index, [], None

    def __enter__(self):
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                        "--format=csv,noheader,nounits", "-lms", "100"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except (OSError, FileNotFoundError):
            self._p = None
        return self

    def _read(self):
        for line in self._p.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self._p:
            self._p.terminate()
            self._p.wait(timeout=5)

    def summary(self):
        rows = [r for r in self.rows if len(r) == 6 and r[0].isdigit()]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = sorted(int(r[0]) for r in rows)
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = [nm for i, nm in enumerate(names) if any(r[2 + i].lower() == "active" for r in rows)]
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": int(rows[0][1]), "reasons": reasons,
                "samples": len(rows)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    return world, rank, local


def allreduce_max(x: float, world: int, device) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def run_reference(args):
    world, rank, _ = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), 0
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    per_core = max(1, args.ref_per_core)
    vals = []
    for _ in range(max(0, args.warmup_ref)):
        cpu_reference(1, cores)
    for _ in range(args.steps):
        vals.append(cpu_reference(per_core, cores))
    v = sum(r["solves_per_s"] for r in vals) / len(vals)
    sample = (f"{per_core * cores} rand32 scenarios per step, a spread subset of the bench's seeds 0..{BATCH - 1}, "
              "warm LU factors, 1 process/core")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "solves/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup_ref, "ms_per_step": 1e3 * vals[-1]["wall_s"],
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": "rand32 batch (generate_random(32,(8,8,3),0.4,seed))",
                                            "agents": 32, "samples": 100, "degree": 10},
            "cpu_baseline": {"value": v, "unit": "solves/s", "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": v, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


FLOP_PER_PAIR_SAMPLE_F = FLOP_PER_PAIR_SAMPLE


def _cpu_single(name: str, max_iters: int | None = None):
    """Same-run CPU time of the reference algorithm (oracle port, numpy/scipy LU, 1 thread, warm
    factors): best of 3 for full solves, or the mean per-iteration time of a bounded prefix."""
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1):  # numpy is loaded in this process already: limit BLAS at run time
        return _cpu_single_1t(name, max_iters)


def _cpu_single_1t(name: str, max_iters: int | None):
    from scipy.linalg import lu_factor

    from oracle import am_oracle
    from paper_2011_04240_b200 import named
    spec = named(name)
    pr = am_oracle.Problem(spec)
    rhos, _ = am_oracle.schedule()
    if max_iters is None:
        factors = [lu_factor(pr.kkt(r), check_finite=False) for r in rhos]
        best = None
        for _ in range(3):
            t0 = time.perf_counter()
            out = am_oracle.solve(spec, factors=factors)
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        return {"loop_ms": round(best * 1e3, 3), "iterations": out["iterations"], "threads": 1,
                "per_iteration_ms": round(best * 1e3 / out["iterations"], 4)}
    f0 = lu_factor(pr.kkt(rhos[0]), check_finite=False)  # only stage 0 runs in a short prefix
    t0 = time.perf_counter()
    out = am_oracle.solve(spec, max_iters=max_iters, factors=[f0] * len(rhos))
    per = (time.perf_counter() - t0) / out["iterations"]
    return {"per_iteration_ms": round(per * 1e3, 3), "iterations_timed": out["iterations"], "threads": 1,
            "note": f"bounded sample: first {max_iters} iterations (stage 0), initialization included"}


def _pair_samples(spec, iters: int) -> float:
    n, m = len(spec.start), spec.num_samples
    return float((n * (n - 1) // 2 + n * len(spec.obstacles)) * m * (iters + 1))


def single_solve_ms(names=("circ16j", "rand32_s0", "hall16j", "sph64j", "rand128_s0", "rand256_s0"), cpu=True,
                    fp64_peak=37.2, hbm_peak=6447.8):
    """BASELINE metric "ms per joint solve at 16/32/64/256 agents": device loop (best of 3),
    whole am_solve call, FP32 mode, the same-run CPU reference, and the roofline fraction of
    the loop (FP64 pipe for the cluster kernel, HBM for the large-fleet kernel's streamed
    multipliers)."""
    from paper_2011_04240_b200 import FactorCache, SolverConfig, am_solve, named
    cache = FactorCache()
    out = {}
    for nm in names:
        spec = named(nm)
        row = {}
        for fp32 in (False, True):
            am_solve(spec, SolverConfig(fp32=fp32), cache=cache)
            best, r = None, None
            for _ in range(3):
                r = am_solve(spec, SolverConfig(fp32=fp32), cache=cache)
                t = r.timings["loop_s"] * 1e3
                best = t if best is None else min(best, t)
            if not fp32:
                n = len(spec.start)
                ps = _pair_samples(spec, r.iterations)
                large = n > 64  # roofline: the multiplier stream (HBM) vs the FP64 pair arithmetic
                bytes_ = BYTES_PER_PAIR_SAMPLE * ps
                flops = FLOP_PER_PAIR_SAMPLE * ps
                # the library's rule (capi.cu large_eligible): obstacle-free single solves above 32 agents
                # run on the whole-GPU large-fleet kernel
                large_kernel = n > 32 and not spec.obstacles
                row.update({"ms": round(best, 4), "iterations": r.iterations, "converged": r.converged,
                            "end_to_end_ms": round(r.timings["total_s"] * 1e3, 3),
                            "kernel": "am_large_kernel" if large_kernel else "am_cluster_kernel"})
                if large:
                    gbs = bytes_ / (best / 1e3) / 1e9
                    row["roofline"] = {"bound": "hbm", "achieved": round(gbs, 1), "peak": hbm_peak, "unit": "GB/s",
                                       "frac": round(gbs / hbm_peak, 4),
                                       "per_unit": "48 B multipliers (read+write) per pair-sample per iteration"}
                else:
                    tf = flops / (best / 1e3) / 1e12
                    row["roofline"] = {"bound": "fp64", "achieved": round(tf, 3), "peak": fp64_peak,
                                       "unit": "TFLOP/s", "frac": round(tf / fp64_peak, 4),
                                       "per_unit": "85 FLOP per pair-sample per iteration"}
            else:
                row["fp32_ms"] = round(best, 4)
                row["fp32_iterations"] = r.iterations
        if cpu:
            ref = _cpu_single(nm, max_iters=None if len(spec.start) <= 64 else 3)
            row["cpu"] = ref
            if "loop_ms" in ref:
                row["speedup_vs_cpu"] = round(ref["loop_ms"] / row["ms"], 1)
            else:
                row["speedup_vs_cpu_per_iteration"] = round(ref["per_iteration_ms"] / (row["ms"] / row["iterations"]), 1)
        out[nm] = row
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=BATCH)
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"])
    ap.add_argument("--cpu-per-core", type=int, default=2, help="cpu_baseline sample: scenarios per core")
    ap.add_argument("--ref-per-core", type=int, default=1)
    ap.add_argument("--warmup-ref", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-single", action="store_true")
    ap.add_argument("--no-fp32", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return

    import numpy as np
    import torch

    from paper_2011_04240_b200 import FactorCache, SolverConfig, engine, kkt, native, pack, poly

    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if args.scaling == "weak":
        lo, hi = rank * args.batch, (rank + 1) * args.batch
        total = args.batch * world
    else:
        lo, hi = rank * args.batch // world, (rank + 1) * args.batch // world
        total = args.batch
    specs = scenarios(lo, hi)
    B = len(specs)
    cfg = SolverConfig(device=local)
    sched = cfg.schedule()
    basis = poly.for_spec(specs[0])
    fp = kkt.fingerprint(basis, 32, 0)
    cache = FactorCache()
    t_pre0 = time.perf_counter()
    plan = engine._plan_for(cache, fp, basis, sched, 32, 0, local)
    precompute_s = time.perf_counter() - t_pre0
    c0, beq, geom = pack(specs, basis)
    nv, m = basis.num_coeffs, basis.num_samples
    # device-resident inputs/outputs
    d_c0 = torch.from_numpy(c0).to(dev)
    d_beq = torch.from_numpy(beq).to(dev)
    d_geom = torch.from_numpy(geom).to(dev)
    d_cout = torch.empty_like(d_c0)
    d_hist = torch.empty((B, 3, cfg.max_iters), dtype=torch.float64, device=dev)
    d_it = torch.empty(B, dtype=torch.int32, device=dev)
    d_cv = torch.empty(B, dtype=torch.int32, device=dev)
    stream = torch.cuda.Stream(device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2

    def launch():
        plan.solve_device(B, d_c0.data_ptr(), d_beq.data_ptr(), d_geom.data_ptr(), sched.switch_every,
                          cfg.max_iters, cfg.tolerance, d_cout.data_ptr(), d_hist.data_ptr(), d_it.data_ptr(),
                          d_cv.data_ptr(), stream=stream.cuda_stream)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            launch()
    torch.cuda.synchronize(dev)
    iters = d_it.cpu().numpy()
    pair_samples = float((iters.astype(np.float64) + 1.0).sum() * (32 * 31 // 2) * m)  # + init pass

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier(world)
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clocks:
        with torch.cuda.stream(stream):
            for i in range(args.steps):
                flush.zero_()  # L2 flush between timed steps (outside the events)
                ev[i][0].record(stream)
                launch()
                ev[i][1].record(stream)
        torch.cuda.synchronize(dev)
    dev_ms = sum(a.elapsed_time(b) for a, b in ev)
    barrier(world)
    dev_ms_max = allreduce_max(dev_ms, world, dev)
    step_ms = dev_ms_max / args.steps
    value = total / (step_ms / 1e3)

    # the optional FP32 mode (SolverConfig(fp32=True)) on the same device-resident batch
    fp32 = None
    if not args.no_fp32:
        d_it32 = torch.empty_like(d_it)

        def launch32():
            plan.solve_device(B, d_c0.data_ptr(), d_beq.data_ptr(), d_geom.data_ptr(), sched.switch_every,
                              cfg.max_iters, cfg.tolerance, d_cout.data_ptr(), d_hist.data_ptr(), d_it32.data_ptr(),
                              d_cv.data_ptr(), stream=stream.cuda_stream, fp32=True)
        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                launch32()
        torch.cuda.synchronize(dev)
        ev32 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                for _ in range(args.steps)]
        barrier(world)
        torch.cuda.synchronize(dev)
        with torch.cuda.stream(stream):
            for i in range(args.steps):
                flush.zero_()
                ev32[i][0].record(stream)
                launch32()
                ev32[i][1].record(stream)
        torch.cuda.synchronize(dev)
        ms32 = allreduce_max(sum(a.elapsed_time(b) for a, b in ev32), world, dev) / args.steps
        it32 = d_it32.cpu().numpy()
        fp32 = {"value": round(total / (ms32 / 1e3), 2), "unit": "solves/s", "ms_per_step": round(ms32, 4),
                "iterations_mean": round(float(it32.mean()), 2),
                "iterations_equal_fp64_frac": round(float((it32 == iters).mean()), 4),
                "speedup_vs_fp64": round(step_ms / ms32, 3),
                "mode": "FP32 pair state (multipliers + pair arithmetic), FP64 positions/sums/solve; "
                        "tolerances in DESIGN.md §8"}
        # leave the FP64 outputs in place for the checks below
        with torch.cuda.stream(stream):
            launch()
        torch.cuda.synchronize(dev)

    # end to end through the C ABI with page-locked host buffers (H2D of the inputs + loop +
    # D2H of the results inside the timed region, every step)
    def pinned(a):
        t = torch.empty(a.shape, dtype=torch.float64 if a.dtype == np.float64 else torch.int32, pin_memory=True)
        v = t.numpy()
        v[...] = a
        return t, v
    _keep = []
    hc0, hbeq, hgeom = (pinned(a) for a in (c0, beq, geom))
    _keep += [hc0[0], hbeq[0], hgeom[0]]
    out_bufs = {}
    for key, shape, dt in (("c", c0.shape, np.float64), ("hist", (B, 3, cfg.max_iters), np.float64),
                           ("iters", (B,), np.int32), ("converged", (B,), np.int32)):
        t, v = pinned(np.zeros(shape, dtype=dt))
        _keep.append(t)
        out_bufs[key] = v
    e2e_times = []
    for i in range(args.steps + 1):
        barrier(world)
        t0 = time.perf_counter()
        out = plan.solve(hc0[1], hbeq[1], hgeom[1], sched.switch_every, cfg.max_iters, cfg.tolerance,
                         out=out_bufs)
        if i > 0:
            e2e_times.append(time.perf_counter() - t0)
    e2e_s = allreduce_max(sum(e2e_times) / len(e2e_times), world, dev)
    h2d = c0.nbytes + beq.nbytes + geom.nbytes
    d2h = out["c"].nbytes + out["hist"].nbytes + out["iters"].nbytes + out["converged"].nbytes
    launch_cfg = plan.query_launch(B)

    # the Python drop-in the reference's callers use (am_solve_batch: validation, packing, solve +
    # device report pass, reports with metrics), whole call from Python objects to SolveReports
    python_api = None
    if world == 1:
        from paper_2011_04240_b200 import am_solve_batch
        am_solve_batch(specs, cfg, cache=cache)
        best, reps = None, None
        for _ in range(3):
            reps = None  # the previous call's reports are freed outside the timed region
            t0 = time.perf_counter()
            reps = am_solve_batch(specs, cfg, cache=cache)
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        python_api = {"value": round(B / best, 1), "unit": "solves/s", "ms_per_call": round(best * 1e3, 2),
                      "path": "paper_2011_04240_b200.am_solve_batch(specs) -> SolveReport list with metrics "
                              "(validation, packing, pipelined device solves + device report pass)",
                      "iterations_match": bool(all(r.iterations == int(i) for r, i in zip(reps, iters)))}

    if rank != 0:
        return
    ok = bool(np.array_equal(out["iters"], iters))
    sm_mhz = clocks.summary()
    peak_clk_ghz = 1.965
    fp64_peak_tflops = 64 * 148 * peak_clk_ghz * 1e9 * 2 / 1e12
    flops = FLOP_PER_PAIR_SAMPLE * pair_samples
    achieved = flops / (dev_ms / args.steps / 1e3) / 1e12 / (1.0 if world == 1 else 1.0)
    hbm_peak = None
    try:
        hbm_peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except (OSError, KeyError, ValueError):
        hbm_peak = 6650.0
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "roofline_traffic.json")))
        traffic = tr.get("dram_bytes_per_launch")
    except (OSError, ValueError):
        pass
    ach_bytes = BYTES_PER_PAIR_SAMPLE * pair_samples / (dev_ms / args.steps / 1e3) / 1e9
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "solves/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(step_ms, 4), "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": (f"batch of {args.batch} rand32 scenarios per GPU (generate_random(32,(8,8,3),0.4,"
                                f"seed), rank r: seeds r*{args.batch}..(r+1)*{args.batch}-1)"
                                if args.scaling == "weak" else
                                f"batch of {args.batch} rand32 scenarios (generate_random(32,(8,8,3),0.4,seed), "
                                f"seeds 0..{args.batch - 1}), 1/N per rank"), "agents": 32, "samples": m,
                   "degree": 10, "max_iters": cfg.max_iters, "tol": cfg.tolerance,
                   "cluster_ctas": launch_cfg["cluster"], "clusters": launch_cfg["clusters"],
                   "lambda_in_smem": bool(launch_cfg["lambda_in_smem"]),
                   "l2": "flushed (256 MB write) between timed steps"},
        "e2e": {"value": round(total / e2e_s, 2), "unit": "solves/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "path": "C ABI st_solve, page-locked host buffers"},
        "gpu_launches": args.steps,
        "roofline": {"bound": "fp64", "achieved": round(achieved, 3), "peak": round(fp64_peak_tflops, 2),
                     "unit": "TFLOP/s", "frac": round(achieved / fp64_peak_tflops, 4), "traffic": traffic,
                     "per_unit": f"{FLOP_PER_PAIR_SAMPLE:.0f} FLOP per pair-sample per iteration "
                                 f"({pair_samples:.3e} pair-samples per launch incl. init pass)",
                     "peak_source": "measured DFMA 64 lanes/clk/SM x 148 SMs x 1.965 GHz x 2 "
                                    "(profiles/ubench_r1.txt)"},
        "lambda_stream": {"achieved_gbs": round(ach_bytes, 1),
                          "per_unit": "48 B (lambda read+write) per pair-sample per iteration",
                          "note": "algorithmic multiplier traffic; the per-cluster slabs are L2-resident "
                                  "(persisting window, DRAM sees a small fraction -- ncu traffic), so this is "
                                  "an L2 rate, not an HBM fraction"},
        "fp32": fp32,
        "python_api": python_api,
        "clocks": sm_mhz,
        "precompute_s": round(precompute_s, 4),
        "iterations_mean": round(float(iters.mean()), 2),
        "converged_frac": round(float(d_cv.cpu().numpy().mean()), 4),
        "e2e_matches_device_iters": ok,
    }
    if not args.no_single and world == 1:
        line["single_solve_ms"] = single_solve_ms(cpu=not args.no_cpu, fp64_peak=round(fp64_peak_tflops, 2),
                                                  hbm_peak=hbm_peak)
    if not args.no_cpu and world == 1:
        cores = os.cpu_count() or 1
        ref = cpu_reference(args.cpu_per_core, cores)
        line["cpu_baseline"] = {"value": round(ref["solves_per_s"], 3), "unit": "solves/s", "cores": ref["cores"],
                                "kind": "port",
                                "sample": f"{ref['solves']} rand32 scenarios, a spread subset of the bench's seeds "
                                          f"0..{BATCH - 1}, oracle/am_oracle.py (reference LU algorithm, "
                                          f"numpy/scipy), warm factors, 1 process/core"}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
