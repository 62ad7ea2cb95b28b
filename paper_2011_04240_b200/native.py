"""ctypes binding of the C ABI in ``include/swarm_am.h`` (``_swarm_am.so``).

There is no CPU fallback: if the library is missing or no CUDA device is
usable, every call raises.  ``Plan`` owns one ``st_plan`` (the device copy
of one fingerprint's stage operators).
"""

from __future__ import annotations

import ctypes
import os
import threading
import weakref

import numpy as np

from . import poly

# SWARM_LIB: alternative build of the same library (A/B comparisons of kernel changes)
LIB_PATH = os.environ.get("SWARM_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_swarm_am.so")

ST_FLAG_KEEP_STATE = 1
ST_FLAG_FP32 = 2
# per-scenario status in the ``converged`` output: 1 converged, 0 not, -1 non-finite state
ST_NONFINITE = -1
_ERRORS = {1: ValueError, 2: RuntimeError, 3: MemoryError, 4: NotImplementedError}

EXPORTS = ("st_plan_create", "st_plan_destroy", "st_solve", "st_solve_report", "st_solve_device", "st_query_launch",
           "st_last_error", "st_version", "st_shard_layout", "st_shard_buffer", "st_shard_open", "st_shard_close",
           "st_shard_reset", "st_solve_sharded", "st_check_collisions",
           "st_check_collisions_batch", "st_large_partition", "st_host_alloc", "st_host_free",
           "st_solve_report_begin", "st_solve_end")

_lib = None
_lock = threading.RLock()  # re-entrant: load() is reachable from GC finalizers (_PinnedPool)

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)


def load() -> ctypes.CDLL:
    """Load the solver library (no GPU needed just to load it)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"native solver library missing: {LIB_PATH} "
                               "(build it with `python -c 'import __graft_entry__ as g; g.build()'`)")
        lib = ctypes.CDLL(LIB_PATH)
        vp = ctypes.c_void_p
        i, d = ctypes.c_int, ctypes.c_double
        lib.st_plan_create.argtypes = [i, i, i, i, i, _dp, _dp, _dp, _dp, _dp, _dp, _dp, i, ctypes.POINTER(vp)]
        lib.st_plan_destroy.argtypes = [vp]
        lib.st_solve.argtypes = [vp, i, _dp, _dp, _dp, i, i, d, i, i, _dp, _dp, _ip, _ip, _dp, _dp,
                                 ctypes.POINTER(ctypes.c_float)]
        lib.st_solve_device.argtypes = [vp, i, vp, vp, vp, i, i, d, i, i, vp, vp, vp, vp, vp, vp, vp]
        optional = set()
        if os.environ.get("SWARM_LIB"):
            # A/B runs against an older build of the library: entries it lacks are optional
            optional = {nm for nm in ("st_solve_report", "st_host_alloc", "st_host_free", "st_solve_report_begin",
                                      "st_solve_end") if not hasattr(lib, nm)}
        if "st_solve_report" not in optional:
            lib.st_solve_report.argtypes = [vp, i, _dp, _dp, _dp, i, i, d, i, i, _dp, _dp, _ip, _ip,
                                            ctypes.POINTER(ctypes.c_float), _dp, _dp, _dp, _dp, _dp, _dp,
                                            ctypes.POINTER(ctypes.c_longlong)]
        if "st_solve_report_begin" not in optional:
            lib.st_solve_report_begin.argtypes = [vp, i, _dp, _dp, _dp, i, i, d, i, i, _dp, _dp, _ip, _ip, _dp, _dp,
                                                  _dp, _dp, _dp, _dp, ctypes.POINTER(ctypes.c_longlong)]
            lib.st_solve_end.argtypes = [vp, ctypes.POINTER(ctypes.c_float)]
        lib.st_query_launch.argtypes = [vp, i, i, i, ctypes.POINTER(ctypes.c_longlong)]
        lib.st_last_error.restype = ctypes.c_char_p
        ub = ctypes.POINTER(ctypes.c_ubyte)
        lib.st_shard_layout.argtypes = [vp, i, ctypes.POINTER(ctypes.c_longlong)]
        lib.st_shard_buffer.argtypes = [vp, ctypes.c_longlong, ctypes.POINTER(vp), ub]
        lib.st_shard_open.argtypes = [vp, ub, ctypes.POINTER(vp)]
        lib.st_shard_close.argtypes = [vp, vp, i]
        lib.st_shard_reset.argtypes = [vp, vp]
        lib.st_solve_sharded.argtypes = [vp, i, i, ctypes.POINTER(vp), _dp, _dp, _dp, i, i, d, _dp, _dp, _ip, _ip,
                                         ctypes.POINTER(ctypes.c_float)]
        ll = ctypes.c_longlong
        lib.st_check_collisions.argtypes = [i, i, _dp, d, d, i, _dp, i, ll, _ip, _dp, _dp, ctypes.POINTER(ll)]
        lib.st_check_collisions_batch.argtypes = [i, i, i, _dp, _dp, i, _dp, i, ll, _ip, _dp, _dp,
                                                  ctypes.POINTER(ll)]
        lib.st_large_partition.argtypes = [i, i, i, i, _ip, _ip, _ip, _ip]
        if "st_host_alloc" not in optional:
            lib.st_host_alloc.argtypes = [ll, ctypes.POINTER(vp)]
            lib.st_host_free.argtypes = [vp]
        for name in EXPORTS:
            if name not in optional:
                getattr(lib, name)  # every declared symbol must resolve
        lib.swarm_has_report = "st_solve_report" not in optional
        lib.swarm_has_async = "st_solve_report_begin" not in optional and "st_host_alloc" not in optional
        _lib = lib
        return lib


def _check(rc: int) -> None:
    if rc != 0:
        msg = load().st_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, RuntimeError)(msg)


def _ptr(a: np.ndarray | None, ctype=_dp):
    if a is None:
        return None
    assert a.flags.c_contiguous
    return a.ctypes.data_as(ctype)


class _PinnedPool:
    """Recycled page-locked host buffers for large outputs (report trajectories).

    ``empty(shape)`` returns a float64 array over a pinned buffer; when the array and every
    view of it are gone, the buffer returns to the pool for the next call of that size
    (allocating page-locked memory costs far more than the copy it speeds up)."""

    def __init__(self, keep: int = 4):
        self._free: dict = {}
        # re-entrant: _release runs as a weakref finalizer, i.e. from the garbage collector, which
        # can fire on any allocation -- including one made while this thread holds the lock
        self._lock = threading.RLock()
        self._keep = keep

    def empty(self, shape, dtype=np.float64) -> np.ndarray:
        dtype = np.dtype(dtype)
        count = int(np.prod(shape))
        nbytes = max(8, count * dtype.itemsize)
        with self._lock:
            bucket = self._free.get(nbytes)
            ptr = bucket.pop() if bucket else None
        if ptr is None:
            p = ctypes.c_void_p()
            _check(load().st_host_alloc(nbytes, ctypes.byref(p)))
            ptr = p.value
        raw = (ctypes.c_byte * nbytes).from_address(ptr)
        weakref.finalize(raw, self._release, ptr, nbytes)
        return np.frombuffer(raw, dtype=dtype, count=count).reshape(shape)

    def _release(self, ptr: int, nbytes: int) -> None:
        fresh = []  # allocated before taking the lock
        with self._lock:
            bucket = self._free.setdefault(nbytes, fresh)
            if len(bucket) < self._keep:
                bucket.append(ptr)
                return
        try:
            load().st_host_free(ptr)
        except Exception:
            pass


_PINNED = _PinnedPool()


def pinned_empty(shape, dtype=np.float64) -> np.ndarray:
    """An uninitialized page-locked host array (pooled buffer, returned when the array dies)."""
    return _PINNED.empty(shape, dtype)


class Plan:
    """Device-resident stage operators for one (fingerprint, rho schedule)."""

    def __init__(self, n: int, n_obs: int, basis: poly.Basis, ops, device: int = 0):
        lib = load()
        self.n, self.n_obs = n, n_obs
        self.m, self.nv = basis.num_samples, basis.num_coeffs
        self.stages = len(ops)
        P = np.ascontiguousarray(basis.P, dtype=np.float64)
        G = np.ascontiguousarray(np.stack([o.G for o in ops]))
        Gm = np.ascontiguousarray(np.stack([o.Gm for o in ops]))
        F = np.ascontiguousarray(np.stack([o.F for o in ops]))
        Fm = np.ascontiguousarray(np.stack([o.Fm for o in ops]))
        E = np.ascontiguousarray(poly.endpoint_rows(basis))
        rho = np.array([o.rho for o in ops], dtype=np.float64)
        h = ctypes.c_void_p()
        _check(lib.st_plan_create(n, n_obs, self.m, self.nv, self.stages, _ptr(P), _ptr(G), _ptr(Gm),
                                  _ptr(F), _ptr(Fm), _ptr(E), _ptr(rho), device, ctypes.byref(h)))
        self._h = h
        self._lib = lib

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self._lib.st_plan_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def num_pairs(self) -> int:
        return self.n * (self.n - 1) // 2 + self.n * self.n_obs

    def query_launch(self, batch: int = 1, cluster_hint: int = 0, fp32: bool = False, keep_state: bool = False) -> dict:
        out = (ctypes.c_longlong * 8)()
        flags = (ST_FLAG_FP32 if fp32 else 0) | (ST_FLAG_KEEP_STATE if keep_state else 0)
        _check(self._lib.st_query_launch(self._h, batch, cluster_hint, flags, out))
        keys = ("cluster", "agent_blocks", "lane_width", "threads", "lambda_in_smem", "smem_bytes",
                "clusters", "steps_per_task")
        return dict(zip(keys, (int(v) for v in out)))

    def solve(self, c0, beq, geom, switch_every: int, max_iters: int, tol: float,
              keep_state: bool = False, cluster_hint: int = 0, out: dict | None = None, fp32: bool = False) -> dict:
        """Host-buffer solve of a batch: c0 (B,3,n,nv), beq (B,3,n,6), geom (B, 2+5 n_obs).

        ``out`` may supply preallocated (e.g. page-locked) output arrays: ``c`` (B,3,n,nv)
        float64, ``hist`` (B,3,max_iters) float64, ``iters`` and ``converged`` (B,) int32.
        """
        c0 = np.ascontiguousarray(c0, dtype=np.float64)
        beq = np.ascontiguousarray(beq, dtype=np.float64)
        geom = np.ascontiguousarray(geom, dtype=np.float64)
        B = c0.shape[0]
        if c0.shape != (B, 3, self.n, self.nv) or beq.shape != (B, 3, self.n, 6) or \
                geom.shape != (B, 2 + 5 * self.n_obs):
            raise ValueError(f"batch arrays have shapes {c0.shape}, {beq.shape}, {geom.shape}; expected "
                             f"({B}, 3, {self.n}, {self.nv}), ({B}, 3, {self.n}, 6), ({B}, {2 + 5 * self.n_obs})")
        if out is not None:
            c_out, hist, iters, conv = out["c"], out["hist"], out["iters"], out["converged"]
            for arr, shape, dt in ((c_out, c0.shape, np.float64), (hist, (B, 3, max_iters), np.float64),
                                   (iters, (B,), np.int32), (conv, (B,), np.int32)):
                if arr.shape != shape or arr.dtype != dt or not arr.flags.c_contiguous:
                    raise ValueError(f"output buffer {arr.shape}/{arr.dtype} does not match {shape}/{dt}")
        else:
            c_out = np.empty_like(c0)
            hist = np.empty((B, 3, max_iters))
            iters = np.empty(B, dtype=np.int32)
            conv = np.empty(B, dtype=np.int32)
        lam = d = None
        if keep_state:
            lam = np.empty((3, self.num_pairs, self.m))
            d = np.empty((self.num_pairs, self.m))
        t = (ctypes.c_float * 3)()
        _check(self._lib.st_solve(self._h, B, _ptr(c0), _ptr(beq), _ptr(geom), switch_every, max_iters, tol,
                                  (ST_FLAG_KEEP_STATE if keep_state else 0) | (ST_FLAG_FP32 if fp32 else 0),
                                  cluster_hint, _ptr(c_out),
                                  _ptr(hist), _ptr(iters, _ip), _ptr(conv, _ip), _ptr(lam), _ptr(d), t))
        return {"c": c_out, "hist": hist, "iters": iters, "converged": conv if out is not None else conv > 0,
                "status": conv.copy(), "lam": lam, "d": d, "timings_ms": tuple(float(x) for x in t)}

    def solve_report(self, c0, beq, geom, switch_every: int, max_iters: int, tol: float, col_geom, col_obs,
                     cluster_hint: int = 0, fp32: bool = False, with_metrics: bool = True) -> dict:
        """``solve`` plus the report's post-loop work on the device in the same call
        (``st_solve_report``): trajectories (B, n, m, 3), arc length and smoothness (B, n),
        and the collision summary -- minimum normalized distance and violation count (B,) --
        from ``col_geom`` (B, 2) and ``col_obs`` (B, n_obs, 5) as for the collision check."""
        c0 = np.ascontiguousarray(c0, dtype=np.float64)
        beq = np.ascontiguousarray(beq, dtype=np.float64)
        geom = np.ascontiguousarray(geom, dtype=np.float64)
        col_geom = np.ascontiguousarray(col_geom, dtype=np.float64)
        col_obs = np.ascontiguousarray(col_obs, dtype=np.float64)
        B = c0.shape[0]
        if c0.shape != (B, 3, self.n, self.nv) or beq.shape != (B, 3, self.n, 6) or \
                geom.shape != (B, 2 + 5 * self.n_obs) or col_geom.shape != (B, 2) or \
                col_obs.shape != (B, self.n_obs, 5):
            raise ValueError("batch arrays do not match the plan's shape")
        c_out = np.empty_like(c0)
        hist = np.empty((B, 3, max_iters))
        iters = np.empty(B, dtype=np.int32)
        conv = np.empty(B, dtype=np.int32)
        traj = _PINNED.empty((B, self.n, self.m, 3))
        arc = np.empty((B, self.n)) if with_metrics else None
        smooth = np.empty((B, self.n)) if with_metrics else None
        mind = np.empty(B) if with_metrics else None
        nviol = np.empty(B, dtype=np.int64) if with_metrics else None
        t = (ctypes.c_float * 3)()
        _check(self._lib.st_solve_report(self._h, B, _ptr(c0), _ptr(beq), _ptr(geom), switch_every, max_iters, tol,
                                         ST_FLAG_FP32 if fp32 else 0, cluster_hint, _ptr(c_out), _ptr(hist),
                                         _ptr(iters, _ip), _ptr(conv, _ip), t, _ptr(col_geom), _ptr(col_obs),
                                         _ptr(traj), _ptr(arc), _ptr(smooth), _ptr(mind),
                                         _ptr(nviol, ctypes.POINTER(ctypes.c_longlong))))
        res = {"c": c_out, "hist": hist, "iters": iters, "converged": conv > 0, "status": conv, "lam": None,
               "d": None, "timings_ms": tuple(float(x) for x in t), "traj": traj}
        if with_metrics:
            res.update(arc=arc, smooth=smooth, min_dist=mind, n_viol=nviol)
        return res

    def solve_report_begin(self, c0, beq, geom, switch_every: int, max_iters: int, tol: float, col_geom, col_obs,
                           cluster_hint: int = 0, fp32: bool = False, with_metrics: bool = True) -> "PendingSolve":
        """First half of ``solve_report`` (``st_solve_report_begin``): the inputs are copied and the
        solve, report pass and output copies (into page-locked arrays) are enqueued; ``end()`` on
        the returned object waits and gives ``solve_report``'s dict.  Nothing else may use this
        plan from the host in between (the library refuses)."""
        c0 = np.ascontiguousarray(c0, dtype=np.float64)
        beq = np.ascontiguousarray(beq, dtype=np.float64)
        geom = np.ascontiguousarray(geom, dtype=np.float64)
        col_geom = np.ascontiguousarray(col_geom, dtype=np.float64)
        col_obs = np.ascontiguousarray(col_obs, dtype=np.float64)
        B = c0.shape[0]
        if c0.shape != (B, 3, self.n, self.nv) or beq.shape != (B, 3, self.n, 6) or \
                geom.shape != (B, 2 + 5 * self.n_obs) or col_geom.shape != (B, 2) or \
                col_obs.shape != (B, self.n_obs, 5):
            raise ValueError("batch arrays do not match the plan's shape")
        out = {"c": _PINNED.empty(c0.shape), "hist": _PINNED.empty((B, 3, max_iters)),
               "iters": _PINNED.empty((B,), np.int32), "status": _PINNED.empty((B,), np.int32),
               "traj": _PINNED.empty((B, self.n, self.m, 3))}
        if with_metrics:
            out.update(arc=_PINNED.empty((B, self.n)), smooth=_PINNED.empty((B, self.n)),
                       min_dist=_PINNED.empty((B,)), n_viol=_PINNED.empty((B,), np.int64))
        g = out.get
        _check(self._lib.st_solve_report_begin(
            self._h, B, _ptr(c0), _ptr(beq), _ptr(geom), switch_every, max_iters, tol, ST_FLAG_FP32 if fp32 else 0,
            cluster_hint, _ptr(out["c"]), _ptr(out["hist"]), _ptr(out["iters"], _ip), _ptr(out["status"], _ip),
            _ptr(col_geom), _ptr(col_obs), _ptr(out["traj"]), _ptr(g("arc")), _ptr(g("smooth")), _ptr(g("min_dist")),
            _ptr(g("n_viol"), ctypes.POINTER(ctypes.c_longlong))))
        return PendingSolve(self, out, (c0, beq, geom, col_geom, col_obs))

    def solve_device(self, B: int, c0_ptr: int, beq_ptr: int, geom_ptr: int, switch_every: int,
                     max_iters: int, tol: float, c_out_ptr: int, hist_ptr: int, iters_ptr: int,
                     conv_ptr: int, stream: int = 0, cluster_hint: int = 0, fp32: bool = False) -> None:
        """Enqueue a solve on device-resident buffers (raw pointers, e.g. torch ``data_ptr()``)."""
        _check(self._lib.st_solve_device(self._h, B, c0_ptr, beq_ptr, geom_ptr, switch_every, max_iters, tol,
                                         ST_FLAG_FP32 if fp32 else 0, cluster_hint, c_out_ptr, hist_ptr, iters_ptr,
                                         conv_ptr, None, None, stream or None))

    # ---- pair sharding over GPUs (one process per GPU; see include/swarm_am.h) -------------

    def shard_layout(self, groups: int) -> dict:
        out = (ctypes.c_longlong * 4)()
        _check(self._lib.st_shard_layout(self._h, groups, out))
        return {"cluster": int(out[0]), "clusters_per_gpu": int(out[1]), "buffer_bytes": int(out[2]),
                "participants": int(out[3])}

    def shard_buffer(self, nbytes: int) -> tuple[int, bytes]:
        ptr = ctypes.c_void_p()
        h = (ctypes.c_ubyte * 64)()
        _check(self._lib.st_shard_buffer(self._h, nbytes, ctypes.byref(ptr), h))
        return ptr.value, bytes(h)

    def shard_open(self, handle: bytes) -> int:
        ptr = ctypes.c_void_p()
        h = (ctypes.c_ubyte * 64).from_buffer_copy(handle)
        _check(self._lib.st_shard_open(self._h, h, ctypes.byref(ptr)))
        return ptr.value

    def shard_close(self, ptr: int, opened: bool) -> None:
        self._lib.st_shard_close(self._h, ptr, 1 if opened else 0)

    def shard_reset(self, buf0: int) -> None:
        _check(self._lib.st_shard_reset(self._h, buf0))

    def solve_sharded(self, groups: int, rank: int, bufs, c0, beq, geom, switch_every: int, max_iters: int,
                      tol: float) -> dict:
        c0 = np.ascontiguousarray(c0, dtype=np.float64)
        beq = np.ascontiguousarray(beq, dtype=np.float64)
        geom = np.ascontiguousarray(geom, dtype=np.float64)
        c_out = np.empty_like(c0)
        hist = np.empty((1, 3, max_iters))
        iters = np.empty(1, dtype=np.int32)
        conv = np.empty(1, dtype=np.int32)
        arr = (ctypes.c_void_p * groups)(*bufs)
        t = (ctypes.c_float * 3)()
        _check(self._lib.st_solve_sharded(self._h, groups, rank, arr, _ptr(c0), _ptr(beq), _ptr(geom), switch_every,
                                          max_iters, tol, _ptr(c_out), _ptr(hist), _ptr(iters, _ip), _ptr(conv, _ip),
                                          t))
        return {"c": c_out, "hist": hist, "iters": iters, "converged": conv.astype(bool),
                "timings_ms": tuple(float(x) for x in t)}


class PendingSolve:
    """A solve begun with ``Plan.solve_report_begin``; ``end()`` waits for it (once).  The input
    arrays are held until then (page-locked inputs are copied asynchronously); a pending solve
    that is dropped without ``end()`` is ended by the finalizer, so the plan is never left
    refusing calls."""

    def __init__(self, plan: Plan, out: dict, inputs: tuple):
        self._plan, self._out, self._inputs = plan, out, inputs

    def end(self) -> dict:
        plan, out = self._plan, self._out
        if plan is None:
            raise RuntimeError("solve already ended")
        self._plan = None
        t = (ctypes.c_float * 3)()
        try:
            _check(plan._lib.st_solve_end(plan._h, t))
        finally:
            self._inputs = None
        out["converged"] = out["status"] > 0
        out.update(lam=None, d=None, timings_ms=tuple(float(x) for x in t))
        return out

    def __del__(self):
        plan = getattr(self, "_plan", None)
        if plan is not None and getattr(plan, "_h", None):
            try:
                plan._lib.st_solve_end(plan._h, None)
            except Exception:
                pass


def check_collisions(traj: np.ndarray, l_xy: float, l_z: float, obs_rows: np.ndarray, device: int = 0,
                     cap: int = 4096):
    """Device collision verdict (``st_check_collisions``; reference validation.py:39-93).

    Returns (minimum, violations) with violations in the reference's order and
    form: ``(("agent", i, j) | ("obstacle", i, k), sample, value)``.
    """
    lib = load()
    traj = np.ascontiguousarray(traj, dtype=np.float64)
    n, m = traj.shape[0], traj.shape[1]
    obs_rows = np.ascontiguousarray(obs_rows, dtype=np.float64).reshape(-1, 5)
    n_obs = obs_rows.shape[0]
    mn, total = ctypes.c_double(), ctypes.c_longlong()
    while True:
        ids = np.empty((max(cap, 1), 4), dtype=np.int32)
        vals = np.empty(max(cap, 1))
        _check(lib.st_check_collisions(n, m, _ptr(traj), float(l_xy), float(l_z), n_obs,
                                       _ptr(obs_rows) if n_obs else None, int(device), cap,
                                       _ptr(ids, _ip), _ptr(vals), ctypes.byref(mn), ctypes.byref(total)))
        if total.value <= cap:
            break
        cap = int(total.value)
    kinds = ("agent", "obstacle")
    viol = [((kinds[int(k)], int(i), int(j)), int(r), float(v))
            for (k, i, j, r), v in zip(ids[: total.value].tolist(), vals[: total.value].tolist())]
    return float(mn.value), viol


def check_collisions_batch(trajs: np.ndarray, geoms: np.ndarray, obs_rows: np.ndarray, device: int = 0,
                           cap: int = 4096, count_only: bool = False) -> list:
    """``st_check_collisions_batch``: one (minimum, violations) per scenario, one device pass.

    ``count_only``: (minimum, number of violations) per scenario -- what the report's metrics
    need -- from the row pass alone (no entry list is built or copied).
    """
    if count_only:
        cap = 0
    lib = load()
    trajs = np.ascontiguousarray(trajs, dtype=np.float64)
    B, n, m = trajs.shape[0], trajs.shape[1], trajs.shape[2]
    geoms = np.ascontiguousarray(geoms, dtype=np.float64).reshape(B, 2)
    obs_rows = np.ascontiguousarray(obs_rows, dtype=np.float64).reshape(B, -1, 5)
    n_obs = obs_rows.shape[1]
    mins = np.empty(B)
    totals = np.empty(B, dtype=np.int64)
    tp = ctypes.POINTER(ctypes.c_longlong)
    while True:
        ids = np.empty((max(cap, 1), 4), dtype=np.int32)
        vals = np.empty(max(cap, 1))
        _check(lib.st_check_collisions_batch(B, n, m, _ptr(trajs), _ptr(geoms), n_obs,
                                             _ptr(obs_rows) if n_obs else None, int(device), cap, _ptr(ids, _ip),
                                             _ptr(vals), _ptr(mins), _ptr(totals, tp)))
        if count_only or int(totals.sum()) <= cap:
            break
        cap = int(totals.sum())
    if count_only:
        return [(float(mn), int(t)) for mn, t in zip(mins.tolist(), totals.tolist())]
    kinds = ("agent", "obstacle")
    out, e = [], 0
    ids_l, vals_l = ids.tolist(), vals.tolist()
    for b in range(B):
        t = int(totals[b])
        out.append((float(mins[b]), [((kinds[k], i, j), r, v) for (k, i, j, r), v in
                                     zip(ids_l[e:e + t], vals_l[e:e + t])]))
        e += t
    return out


def large_partition(n: int, m: int, groups: int, ctas_per_group: int) -> dict:
    """Host-only unit partition of the large-fleet kernel (``st_large_partition``)."""
    lib = load()
    nb = (n + 31) // 32
    nab = nb * (nb + 1) // 2
    U_max = nab * m * 2
    u_range = np.empty(groups + 1, dtype=np.int32)
    cta_first = np.empty(groups * (ctas_per_group + 1), dtype=np.int32)
    rows = np.empty(U_max, dtype=np.int32)
    ab_first = np.empty(nab + 1, dtype=np.int32)
    U = lib.st_large_partition(n, m, groups, ctas_per_group, _ptr(u_range, _ip), _ptr(cta_first, _ip),
                               _ptr(rows, _ip), _ptr(ab_first, _ip))
    if U < 0:
        _check(-U)
    return {"units": int(U), "u_range": u_range, "cta_first": cta_first.reshape(groups, ctas_per_group + 1),
            "rows": rows[:U], "ab_first": ab_first}
