"""Parareal / theta-Parareal driver with serial, pipelined and batched schedulers.

API mirror of the reference engine (reference pkg/src/pintbench/parareal.py):
``PararealConfig`` (49-76), ``RunTrace`` (79-103), ``parareal_update``
(154-163), ``theta_weight`` (166-197), ``boundary_error`` (200-213),
``sequential_solve`` (138-151), ``theoretical_speedup`` (133-135),
``pipelined_schedule`` (241-267) and ``run_parareal`` (363-465).  The
iteration is

    X[i][l+1] = theta C(X[i][l]) + F(X[i-1][l]) - theta C(X[i-1][l])

with the correction norm ||X[i][l+1] - X[i-1][l+1]|| / ||X[i][l+1]|| recorded
per boundary (the "defect history") and the stop test at the end of each
corrector sweep.

Schedulers:
* ``serial``    -- tasks in priority order on the calling thread (the
                   reference's serial order, parareal.py:270-278);
* ``pipelined`` -- a worker pool over the same task graph (fine task of
                   iteration i starts once the i-1 corrector published its left
                   boundary), as parareal.py:281-360;
* ``batched``   -- new, B200-first: the L fine tasks of an iteration go to the
                   propagator's ``advance_batch`` in ONE call (legal because
                   fine(i, .) depends only on the corrector of i-1,
                   parareal.py:258-261); results equal the serial order bitwise
                   when the propagator is batch-invariant.

``run_parareal_device`` keeps every boundary state resident in HBM: one
batched fine launch per iteration, the sequential coarse sweep on the device
(batch-1 ``advance_device``) and the correction (theta weight, update,
correction norm) as the K8b kernel of the C ABI; iterates are copied to the
host once at the end for the ``RunTrace``.
"""

from __future__ import annotations

import heapq
import threading
import time
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

from .state import State

VARIANTS = ("classic", "least_squares", "angle_penalized")
SCHEDULERS = ("serial", "pipelined", "batched")
_DEGENERATE_MASS = 1e-28


class PararealError(RuntimeError):
    """A propagator failed inside the iteration; message carries (iteration, interval)."""


@dataclass(frozen=True)
class PararealConfig:
    intervals: int
    max_iters: int
    tol: float = 1e-10
    variant: str = "classic"
    theta_clamp: tuple = (0.0, 1.0)
    scheduler: str = "serial"
    workers: int = 1

    def __post_init__(self):
        if self.intervals < 2:
            raise ValueError("need at least 2 intervals")
        if not 1 <= self.max_iters <= self.intervals:
            raise ValueError("max_iters must lie in [1, intervals]; further iterations cannot improve")
        if self.tol <= 0.0:
            raise ValueError("tol must be positive")
        if self.variant not in VARIANTS:
            raise ValueError(f"unknown variant {self.variant!r}, expected one of {VARIANTS}")
        lo, hi = self.theta_clamp
        if lo > hi:
            raise ValueError("theta_clamp must be a non-empty interval")
        if self.scheduler not in SCHEDULERS:
            raise ValueError(f"unknown scheduler {self.scheduler!r}, expected one of {SCHEDULERS}")
        if self.workers < 1:
            raise ValueError("workers must be at least 1")


@dataclass
class RunTrace:
    intervals: int
    variant: str
    scheduler: str
    iterations_run: int = 0
    converged: bool = False
    theta_values: list = field(default_factory=list)
    correction_norms: list = field(default_factory=list)
    boundary_errors: list = field(default_factory=list)
    iterate_values: list = field(default_factory=list)
    init_seconds: float = 0.0
    iteration_seconds: list = field(default_factory=list)
    total_seconds: float = 0.0
    fine_propagations: int = 0
    fine_seconds: float = 0.0      # new: wall time spent in fine phases (batched / device modes)


@dataclass(frozen=True)
class ErrorEntry:
    value: float
    absolute: bool = False


@dataclass(frozen=True)
class SpeedupModel:
    r: float
    iters: int
    intervals: int

    def __post_init__(self):
        if self.r <= 0.0:
            raise ValueError("step ratio r must be positive")
        if not 0 < self.iters <= self.intervals:
            raise ValueError("iteration count must lie in (0, intervals]")


def theoretical_speedup(model: SpeedupModel) -> float:
    """1 / (r + (K/N)(1 + r))."""
    return 1.0 / (model.r + (model.iters / model.intervals) * (1.0 + model.r))


def _split_window(window: float, step: float) -> int:
    from .propagator import split_window
    return split_window(window, step)


def sequential_solve(F, s0: State, t_grid: Sequence[float]) -> list:
    grid = [float(t) for t in t_grid]
    if len(grid) < 2:
        raise ValueError("time grid needs at least two points")
    if abs(grid[0] - s0.time) > 1e-12 * max(1.0, abs(s0.time)):
        raise ValueError(f"grid starts at {grid[0]} but the state is at {s0.time}")
    if any(b <= a for a, b in zip(grid, grid[1:])):
        raise ValueError("time grid must be strictly increasing")
    out = [s0]
    for t in grid[1:]:
        out.append(F.advance(out[-1], t))
    return out


def parareal_update(coarse_new: State, fine_old: State, coarse_old: State, theta: float) -> State:
    """theta*C_new + F_old - theta*C_old, evaluated in that order (parareal.py:162)."""
    if not (fine_old.same_layout(coarse_new) and fine_old.same_layout(coarse_old)):
        raise ValueError("states in the update must share one layout")
    t = fine_old.time
    tol = 1e-12 * max(1.0, abs(t))
    if abs(coarse_new.time - t) > tol or abs(coarse_old.time - t) > tol:
        raise ValueError("states in the update must sit at the same time")
    values = theta * coarse_new.values + fine_old.values - theta * coarse_old.values
    return fine_old.with_values(values, time=t)


def _block_weight(f: np.ndarray, c: np.ndarray, variant: str) -> float:
    cc = float(np.dot(c, c))
    if cc <= _DEGENERATE_MASS:
        return 1.0
    fc = float(np.dot(f, c))
    if variant == "least_squares":
        w = fc / cc
    else:
        denom = cc * float(np.dot(f, f))
        w = fc / denom if denom > _DEGENERATE_MASS ** 2 else 1.0
    return w if np.isfinite(w) else 1.0


def theta_weight(fine: State, coarse: State, variant: str, clamp: tuple = (0.0, 1.0)) -> float:
    """Per-block LSQ / angle-penalized weight averaged over blocks, clamped
    (parareal.py:166-197); classic -> 1."""
    if variant == "classic":
        return 1.0
    if variant not in VARIANTS:
        raise ValueError(f"unknown variant {variant!r}")
    if not fine.same_layout(coarse):
        raise ValueError("fine and coarse states must share one layout")
    ws = [_block_weight(fine.block(n), coarse.block(n), variant) for n in fine.layout]
    lo, hi = clamp
    return float(min(max(sum(ws) / len(ws), lo), hi))


def boundary_error(parareal_states: Sequence[State], sequential_states: Sequence[State]) -> list:
    if len(parareal_states) != len(sequential_states):
        raise ValueError("state lists must have equal length")
    out = []
    for vp, vs in zip(parareal_states, sequential_states):
        diff = float(np.linalg.norm(vp.values - vs.values))
        ref = float(np.linalg.norm(vs.values))
        out.append(ErrorEntry(diff / ref) if ref > 0.0 else ErrorEntry(diff, absolute=True))
    return out


def correction_norm(new: np.ndarray, prev: np.ndarray) -> float:
    """0 if unchanged, else ||new - prev|| / ||new|| (inf if ||new|| = 0) (parareal.py:429-431)."""
    diff = float(np.linalg.norm(new - prev))
    norm = float(np.linalg.norm(new))
    return 0.0 if diff == 0.0 else (diff / norm if norm > 0.0 else float("inf"))


# ----------------------------------------------------------------------------
# task graph (parareal.py:220-267)


@dataclass(frozen=True)
class Task:
    kind: str
    iteration: int
    interval: int
    depends: tuple

    @property
    def key(self):
        return (self.iteration, 0 if self.kind == "fine" else 1, self.interval)


def pipelined_schedule(intervals: int, iterations: int) -> list:
    if intervals < 1:
        raise ValueError("need at least one interval")
    if iterations < 0:
        raise ValueError("iterations must be non-negative")
    tasks = [Task("coarse_init", 0, l, ((0, 1, l - 1),) if l else ()) for l in range(intervals)]
    for i in range(1, iterations + 1):
        tasks += [Task("fine", i, l, ((i - 1, 1, l - 1),) if l else ()) for l in range(intervals)]
        for l in range(intervals):
            deps = [(i, 0, l), (i - 1, 1, l)] + ([(i, 1, l - 1)] if l else [])
            tasks.append(Task("correct", i, l, tuple(deps)))
    return tasks


class _Pool:
    """Priority-ordered worker pool; one worker reproduces the serial order."""

    def __init__(self, tasks, run_task: Callable, workers: int):
        self.run_task = run_task
        self.tasks = {t.key: t for t in tasks}
        self.waiting = {t.key: len(t.depends) for t in tasks}
        self.children: dict = {}
        for t in tasks:
            for d in t.depends:
                if d not in self.tasks:
                    raise ValueError(f"task {t.key} depends on unknown task {d}")
                self.children.setdefault(d, []).append(t.key)
        self.ready = sorted(k for k, n in self.waiting.items() if n == 0)
        heapq.heapify(self.ready)
        self.cv = threading.Condition()
        self.left = len(tasks)
        self.busy = 0
        self.stop_at: Optional[int] = None
        self.error: Optional[BaseException] = None
        self.workers = workers

    def _done(self, key):
        self.left -= 1
        for c in self.children.get(key, ()):
            self.waiting[c] -= 1
            if self.waiting[c] == 0:
                heapq.heappush(self.ready, c)
        self.cv.notify_all()

    def _loop(self):
        while True:
            with self.cv:
                while not self.ready and self.left and self.error is None:
                    if self.busy == 0:
                        self.error = RuntimeError("scheduler stalled: tasks remain but none are ready or running")
                        self.cv.notify_all()
                        break
                    self.cv.wait()
                if self.error is not None or not self.left:
                    return
                key = heapq.heappop(self.ready)
                task = self.tasks[key]
                if self.stop_at is not None and task.iteration > self.stop_at:
                    self._done(key)
                    continue
                self.busy += 1
            try:
                out = self.run_task(task)
            except BaseException as exc:  # propagate the first failure
                with self.cv:
                    self.error = exc
                    self.busy -= 1
                    self.cv.notify_all()
                return
            with self.cv:
                self.busy -= 1
                if out is not None:
                    self.stop_at = out if self.stop_at is None else min(self.stop_at, out)
                self._done(key)

    def run(self):
        threads = [threading.Thread(target=self._loop, daemon=True) for _ in range(self.workers)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if self.error is not None:
            raise self.error
        return self.stop_at


def _grid(s0: State, t_end: float, L: int) -> list:
    g = [s0.time + (t_end - s0.time) * l / L for l in range(L + 1)]
    g[-1] = t_end
    return g


def run_parareal(C, F, s0: State, t_end: float, cfg: PararealConfig, oracle: Optional[Sequence[State]] = None):
    """Parareal over [s0.time, t_end]; returns (boundary states of the last
    completed iteration, RunTrace) exactly as parareal.py:363-465."""
    L = cfg.intervals
    if t_end <= s0.time:
        raise ValueError("t_end must lie beyond the initial time")
    window = (t_end - s0.time) / L
    for prop in (C, F):
        _split_window(window, prop.step)
    t_grid = _grid(s0, t_end, L)
    if oracle is not None and len(oracle) != L + 1:
        raise ValueError(f"oracle must hold {L + 1} states, got {len(oracle)}")
    K = cfg.max_iters
    X = [[s0] + [None] * L for _ in range(K + 1)]
    coarse = [[None] * (L + 1) for _ in range(K + 1)]
    fine = [[None] * (L + 1) for _ in range(K + 1)]
    thetas = [[1.0] * L for _ in range(K + 1)]
    corr = [[0.0] * L for _ in range(K + 1)]
    stamps = {"init": 0.0, "it": [0.0] * (K + 1), "fine": 0.0}
    lock = threading.Lock()
    nfine = [0]
    t0 = time.perf_counter()

    def correct(i: int, l: int) -> Optional[int]:
        c_new = C.advance(X[i][l], t_grid[l + 1])
        f_old = fine[i][l + 1]
        th = theta_weight(f_old, c_new, cfg.variant, cfg.theta_clamp)
        new = parareal_update(c_new, f_old, coarse[i - 1][l + 1], th)
        X[i][l + 1] = new
        coarse[i][l + 1] = c_new
        thetas[i][l] = th
        corr[i][l] = correction_norm(new.values, X[i - 1][l + 1].values)
        if l == L - 1:
            stamps["it"][i] = time.perf_counter() - t0
            if max(corr[i]) <= cfg.tol:
                return i
        return None

    def run_task(task: Task) -> Optional[int]:
        i, l = task.iteration, task.interval
        try:
            if task.kind == "coarse_init":
                nxt = C.advance(X[0][l], t_grid[l + 1])
                X[0][l + 1] = nxt
                coarse[0][l + 1] = nxt
                if l == L - 1:
                    stamps["init"] = time.perf_counter() - t0
                return None
            if task.kind == "fine":
                fine[i][l + 1] = F.advance(X[i - 1][l], t_grid[l + 1])
                with lock:
                    nfine[0] += 1
                return None
            return correct(i, l)
        except PararealError:
            raise
        except Exception as exc:
            raise PararealError(f"{task.kind} failed at iteration {i}, interval {l}: {exc}") from exc

    if cfg.scheduler == "batched":
        stop_at = None
        for l in range(L):
            run_task(Task("coarse_init", 0, l, ()))
        batch = getattr(F, "advance_batch", None)
        for i in range(1, K + 1):
            tf = time.perf_counter()
            try:
                if batch is not None:
                    outs = batch([X[i - 1][l] for l in range(L)], [t_grid[l + 1] for l in range(L)])
                else:
                    outs = [F.advance(X[i - 1][l], t_grid[l + 1]) for l in range(L)]
            except Exception as exc:
                raise PararealError(f"fine failed at iteration {i}, interval 0..{L - 1}: {exc}") from exc
            stamps["fine"] += time.perf_counter() - tf
            for l in range(L):
                fine[i][l + 1] = outs[l]
            nfine[0] += L
            res = None
            for l in range(L):
                res = run_task(Task("correct", i, l, ()))
            if res is not None:
                stop_at = res
                break
    else:
        tasks = pipelined_schedule(L, K)
        stop_at = _Pool(tasks, run_task, 1 if cfg.scheduler == "serial" else cfg.workers).run()

    n_it = stop_at if stop_at is not None else K
    trace = RunTrace(intervals=L, variant=cfg.variant, scheduler=cfg.scheduler)
    trace.iterations_run = n_it
    trace.converged = stop_at is not None
    trace.theta_values = [list(thetas[i]) for i in range(1, n_it + 1)]
    trace.correction_norms = [list(corr[i]) for i in range(1, n_it + 1)]
    trace.iterate_values = [[X[i][l].values.copy() for l in range(L + 1)] for i in range(n_it + 1)]
    trace.init_seconds = stamps["init"]
    trace.iteration_seconds = [stamps["it"][i] for i in range(1, n_it + 1)]
    trace.total_seconds = time.perf_counter() - t0
    trace.fine_propagations = nfine[0]
    trace.fine_seconds = stamps["fine"]
    if oracle is not None:
        for i in range(1, n_it + 1):
            trace.boundary_errors.append([e.value for e in boundary_error(X[i][1:], oracle[1:])])
    return X[n_it], trace


# ----------------------------------------------------------------------------
# device-resident driver


_VARIANT_CODE = {"classic": 0, "least_squares": 1, "angle_penalized": 2}


def run_parareal_device(C, F, s0: State, t_end: float, cfg: PararealConfig,
                        oracle: Optional[Sequence[State]] = None):
    """Parareal with every boundary state in HBM (GPU propagators only).

    Per iteration: ONE batched fine launch over all L slices
    (``F.advance_device``), then the sequential corrector sweep on the device:
    batch-1 coarse propagation followed by the K8b kernel (theta weight,
    update, correction norm).  Same trace semantics as :func:`run_parareal`.
    """
    import ctypes

    import torch

    from . import _lib
    from .propagator import _ptr, _stream

    dev = F.device
    lib = _lib.load()
    L = cfg.intervals
    if t_end <= s0.time:
        raise ValueError("t_end must lie beyond the initial time")
    window = (t_end - s0.time) / L
    for prop in (C, F):
        _split_window(window, prop.step)
    if L > dev.max_slices:
        raise ValueError(f"{L} intervals exceed the device context's {dev.max_slices} slices")
    t_grid = _grid(s0, t_end, L)
    K = cfg.max_iters
    Cn, nn, npad = dev.C, dev.nn, dev.np
    t0 = time.perf_counter()
    # X[i] : (L+1, C, np) device; coarse[i] : (L+1, C, np)
    X = [dev.empty(L + 1) for _ in range(K + 1)]
    coarse = [dev.empty(L + 1) for _ in range(K + 1)]
    first = dev.to_device(s0.values)
    for i in range(K + 1):
        X[i][0].copy_(first[0])

    def cadv(src: torch.Tensor, l: int, out: torch.Tensor):
        C.advance_device(src[None], [t_grid[l]], [t_grid[l + 1]], out=out[None])

    try:
        for l in range(L):
            cadv(X[0][l], l, X[0][l + 1])
            coarse[0][l + 1].copy_(X[0][l + 1])
    except Exception as exc:
        raise PararealError(f"coarse_init failed at iteration 0: {exc}") from exc
    torch.cuda.synchronize()
    init_s = time.perf_counter() - t0
    thetas, corrs, it_s = [], [], []
    fine_s = 0.0
    stop_at = None
    nfine = 0
    for i in range(1, K + 1):
        tf = time.perf_counter()
        try:
            fine = F.advance_device(X[i - 1][:L].contiguous(), t_grid[:L], t_grid[1:])
        except Exception as exc:
            raise PararealError(f"fine failed at iteration {i}, interval 0..{L - 1}: {exc}") from exc
        torch.cuda.synchronize()
        fine_s += time.perf_counter() - tf
        nfine += L
        th_row, c_row = [], []
        for l in range(L):
            try:
                cadv(X[i][l], l, coarse[i][l + 1])
            except Exception as exc:
                raise PararealError(f"correct failed at iteration {i}, interval {l}: {exc}") from exc
            th = ctypes.c_double()
            cr = ctypes.c_double()
            rc = lib.pint_parareal_correct_one(
                Cn, nn, npad, _ptr(coarse[i][l + 1]), _ptr(fine[l]), _ptr(coarse[i - 1][l + 1]),
                _ptr(X[i - 1][l + 1]), _ptr(X[i][l + 1]), _VARIANT_CODE[cfg.variant],
                float(cfg.theta_clamp[0]), float(cfg.theta_clamp[1]), ctypes.byref(th), ctypes.byref(cr),
                _stream())
            if rc != _lib.PINT_OK:
                raise PararealError(f"correct failed at iteration {i}, interval {l}: device error {rc}")
            th_row.append(th.value)
            c_row.append(cr.value)
        thetas.append(th_row)
        corrs.append(c_row)
        it_s.append(time.perf_counter() - t0)
        if max(c_row) <= cfg.tol:
            stop_at = i
            break
    n_it = stop_at if stop_at is not None else K
    host = [dev.to_host(X[i]) for i in range(n_it + 1)]
    trace = RunTrace(intervals=L, variant=cfg.variant, scheduler="device")
    trace.iterations_run = n_it
    trace.converged = stop_at is not None
    trace.theta_values = thetas[:n_it]
    trace.correction_norms = corrs[:n_it]
    trace.iterate_values = [[host[i][l].copy() for l in range(L + 1)] for i in range(n_it + 1)]
    trace.init_seconds = init_s
    trace.iteration_seconds = it_s[:n_it]
    trace.total_seconds = time.perf_counter() - t0
    trace.fine_propagations = nfine
    trace.fine_seconds = fine_s
    states = [s0] + [s0.with_values(host[n_it][l], time=t_grid[l]) for l in range(1, L + 1)]
    if oracle is not None:
        for i in range(1, n_it + 1):
            st = [s0.with_values(host[i][l], time=t_grid[l]) for l in range(1, L + 1)]
            trace.boundary_errors.append([e.value for e in boundary_error(st, oracle[1:])])
    return states, trace


def run_parareal_device_pipelined(C, F, s0: State, t_end: float, cfg: PararealConfig, chunks: int = 4,
                                  oracle: Optional[Sequence[State]] = None):
    """Device-resident Parareal with the fine phase of iteration i+1 overlapping
    the corrector sweep of iteration i (the pipelined task graph of the
    reference, parareal.py:241-267, at chunk granularity).

    The L slices split into ``chunks`` contiguous groups; a worker thread
    launches the batched fine propagation of a group as soon as the corrector
    has published the group's left boundaries, while the calling thread keeps
    sweeping.  ``C`` and ``F`` must own DIFFERENT device contexts (each context
    has its own stream, so the two run concurrently on the GPU; ctypes releases
    the GIL).  Results equal :func:`run_parareal_device` bitwise (the fine
    propagator is batch-invariant and every task sees the same inputs).
    """
    import ctypes

    import torch

    from . import _lib
    from .propagator import _ptr, _stream

    if C.device is F.device:
        raise ValueError("pipelined device driver needs separate device contexts for C and F")
    dev = F.device
    lib = _lib.load()
    L = cfg.intervals
    if t_end <= s0.time:
        raise ValueError("t_end must lie beyond the initial time")
    window = (t_end - s0.time) / L
    for prop in (C, F):
        _split_window(window, prop.step)
    t_grid = _grid(s0, t_end, L)
    K = cfg.max_iters
    Cn, nn, npad = dev.C, dev.nn, dev.np
    chunks = max(1, min(chunks, L))
    bounds = [(c * L // chunks, (c + 1) * L // chunks) for c in range(chunks)]
    t0 = time.perf_counter()
    X = [dev.empty(L + 1) for _ in range(K + 1)]
    coarse = [dev.empty(L + 1) for _ in range(K + 1)]
    fine = [dev.empty(L) for _ in range(K + 1)]
    first = dev.to_device(s0.values)
    for i in range(K + 1):
        X[i][0].copy_(first[0])
    torch.cuda.synchronize()
    cond = threading.Condition()
    published = [0] * (K + 1)          # X[i][0..published[i]] are final
    fine_done = [[False] * chunks for _ in range(K + 1)]
    stop = {"at": None, "error": None}

    def cadv(src, l, out):
        C.advance_device(src[None], [t_grid[l]], [t_grid[l + 1]], out=out[None])

    def fine_worker():
        try:
            for i in range(1, K + 1):
                for c, (lo, hi) in enumerate(bounds):
                    with cond:
                        # the chunk's inputs X[i-1][lo..hi-1] must be final
                        while published[i - 1] < hi - 1 and stop["at"] is None and stop["error"] is None:
                            cond.wait()
                        if stop["error"] is not None or (stop["at"] is not None and i > stop["at"]):
                            return
                    out = F.advance_device(X[i - 1][lo:hi].contiguous(), t_grid[lo:hi], t_grid[lo + 1:hi + 1])
                    fine[i][lo:hi].copy_(out)
                    torch.cuda.synchronize()
                    with cond:
                        fine_done[i][c] = True
                        cond.notify_all()
        except BaseException as exc:  # noqa: BLE001 -- surfaced by the sweep thread
            with cond:
                stop["error"] = exc
                cond.notify_all()

    try:
        for l in range(L):
            cadv(X[0][l], l, X[0][l + 1])
            coarse[0][l + 1].copy_(X[0][l + 1])
            torch.cuda.synchronize()
            with cond:
                published[0] = l + 1
                cond.notify_all()
    except Exception as exc:
        raise PararealError(f"coarse_init failed at iteration 0: {exc}") from exc
    init_s = time.perf_counter() - t0
    worker = threading.Thread(target=fine_worker, daemon=True)
    worker.start()
    thetas, corrs, it_s = [], [], []
    stop_at = None
    try:
        for i in range(1, K + 1):
            th_row, c_row = [], []
            for l in range(L):
                c = next(ci for ci, (lo, hi) in enumerate(bounds) if lo <= l < hi)
                with cond:
                    while not fine_done[i][c] and stop["error"] is None:
                        cond.wait()
                    if stop["error"] is not None:
                        raise PararealError(f"fine failed at iteration {i}: {stop['error']}") from stop["error"]
                try:
                    cadv(X[i][l], l, coarse[i][l + 1])
                except Exception as exc:
                    raise PararealError(f"correct failed at iteration {i}, interval {l}: {exc}") from exc
                th, cr = ctypes.c_double(), ctypes.c_double()
                rc = lib.pint_parareal_correct_one(
                    Cn, nn, npad, _ptr(coarse[i][l + 1]), _ptr(fine[i][l]), _ptr(coarse[i - 1][l + 1]),
                    _ptr(X[i - 1][l + 1]), _ptr(X[i][l + 1]), _VARIANT_CODE[cfg.variant],
                    float(cfg.theta_clamp[0]), float(cfg.theta_clamp[1]), ctypes.byref(th), ctypes.byref(cr),
                    _stream())
                if rc != _lib.PINT_OK:
                    raise PararealError(f"correct failed at iteration {i}, interval {l}: device error {rc}")
                th_row.append(th.value)
                c_row.append(cr.value)
                with cond:
                    published[i] = l + 1
                    cond.notify_all()
            thetas.append(th_row)
            corrs.append(c_row)
            it_s.append(time.perf_counter() - t0)
            if max(c_row) <= cfg.tol:
                stop_at = i
                with cond:
                    stop["at"] = i
                    cond.notify_all()
                break
    finally:
        with cond:
            if stop["at"] is None:
                stop["at"] = K
            cond.notify_all()
        worker.join()
    n_it = stop_at if stop_at is not None else K
    host = [dev.to_host(X[i]) for i in range(n_it + 1)]
    trace = RunTrace(intervals=L, variant=cfg.variant, scheduler=f"device-pipelined[{chunks}]")
    trace.iterations_run = n_it
    trace.converged = stop_at is not None
    trace.theta_values = thetas[:n_it]
    trace.correction_norms = corrs[:n_it]
    trace.iterate_values = [[host[i][l].copy() for l in range(L + 1)] for i in range(n_it + 1)]
    trace.init_seconds = init_s
    trace.iteration_seconds = it_s[:n_it]
    trace.total_seconds = time.perf_counter() - t0
    trace.fine_propagations = L * n_it
    states = [s0] + [s0.with_values(host[n_it][l], time=t_grid[l]) for l in range(1, L + 1)]
    if oracle is not None:
        for i in range(1, n_it + 1):
            st = [s0.with_values(host[i][l], time=t_grid[l]) for l in range(1, L + 1)]
            trace.boundary_errors.append([e.value for e in boundary_error(st, oracle[1:])])
    return states, trace
