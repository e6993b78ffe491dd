"""Device-resident Parareal drivers for the GPU propagators.

The reference engine ``pintbench.run_parareal`` (reference
pkg/src/pintbench/parareal.py:363-465) drives ``GPUThetaPropagator`` as it
stands -- it only reads ``step`` and calls ``advance`` (the drop-in contract,
tests/test_gpu_integration.py).  This module holds the B200-first drivers,
which keep every boundary state in HBM and hand each phase of an iteration
to the device in one call:

* the fine phase (parareal.py:417-421): all L fine tasks of iteration i in ONE
  batched ``advance_device`` launch (legal because fine(i, .) depends only on
  the corrector of iteration i-1, parareal.py:258-261; the result equals the
  serial order bitwise because the propagator is batch-invariant);
* the corrector sweep (parareal.py:422-436) and the coarse initialisation
  (parareal.py:410-416): ONE ``pint_coarse_sweep`` call per iteration -- L
  launches of the device-driven loop graph with the K8b correction
  (theta weight, update, correction norm) between them, one host
  synchronisation per sweep;
* boundary errors against a reference trajectory (parareal.py:200-213,
  461-464) on the device (``pint_boundary_error``).

``run_parareal_device`` optionally shards the fine phase over the ranks of a
``torch.distributed`` group: each rank propagates a contiguous
block of slices, one all-gather of device tensors (NCCL over NVLink on GPUs)
per iteration assembles F(X[i-1]) everywhere, and every rank runs the same
deterministic sweep, so all ranks hold identical iterates.

``run_parareal_device_pipelined`` overlaps the fine phase of iteration i+1
with the sweep of iteration i at chunk granularity (the dependency structure
of the reference's pipelined task graph, parareal.py:241-267).

The trace schema (``RunTrace``) and the configuration fields
(``PararealConfig``) are those of the reference so its reporting code reads
them unchanged.
"""

from __future__ import annotations

import threading
import time
from dataclasses import dataclass, field
from typing import Optional, Sequence

from .state import State

VARIANT_CODES = {"classic": 0, "least_squares": 1, "angle_penalized": 2}


class PararealError(RuntimeError):
    """A propagator failed inside the iteration; the message names the task
    kind, the iteration and the interval (parareal.py:437-440)."""


@dataclass(frozen=True)
class PararealConfig:
    """Iteration controls, field for field the reference's (parareal.py:49-76):
    L intervals, at most ``max_iters`` (<= L) iterations, stop when the largest
    correction norm of an iteration is <= ``tol``, theta-weight variant and
    clamp.  ``scheduler`` / ``workers`` only exist for schema compatibility."""

    intervals: int
    max_iters: int
    tol: float = 1e-10
    variant: str = "classic"
    theta_clamp: tuple = (0.0, 1.0)
    scheduler: str = "device"
    workers: int = 1

    def __post_init__(self):
        problems = []
        if self.intervals < 2:
            problems.append("need at least 2 intervals")
        if not 1 <= self.max_iters <= self.intervals:
            problems.append("max_iters must lie in [1, intervals]")
        if not self.tol > 0.0:
            problems.append("tol must be positive")
        if self.variant not in VARIANT_CODES:
            problems.append(f"unknown variant {self.variant!r}, expected one of {tuple(VARIANT_CODES)}")
        if self.theta_clamp[0] > self.theta_clamp[1]:
            problems.append("theta_clamp must be a non-empty interval")
        if self.workers < 1:
            problems.append("workers must be at least 1")
        if problems:
            raise ValueError("; ".join(problems))


@dataclass
class RunTrace:
    """What one Parareal run recorded (the reference's trace schema,
    parareal.py:79-103, plus the device drivers' phase timings)."""

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
    fine_seconds: float = 0.0      # wall time inside the fine phases
    sweep_seconds: float = 0.0     # wall time inside the corrector sweeps (coarse init excluded)


def time_grid(t0: float, t_end: float, L: int) -> list:
    """Boundaries t0 + (t_end - t0) l / L with the last one exactly t_end."""
    g = [t0 + (t_end - t0) * l / L for l in range(L + 1)]
    g[-1] = t_end
    return g


def _check(C, F, s0: State, t_end: float, cfg, oracle=None) -> list:
    from .propagator import split_window
    L = cfg.intervals
    if not t_end > s0.time:
        raise ValueError("t_end must lie beyond the initial time")
    window = (t_end - s0.time) / L
    for prop in (C, F):
        split_window(window, prop.step)  # NonDivisibleWindow up front, as parareal.py:386-388
    if cfg.variant not in VARIANT_CODES:
        raise ValueError(f"unknown variant {cfg.variant!r}")
    if oracle is not None and len(oracle) != L + 1:
        raise ValueError(f"oracle must hold {L + 1} states, got {len(oracle)}")
    return time_grid(s0.time, t_end, L)


def _sweep(C, X, grid, c_new, what: str, i: int, offset: int = 0, **kw):
    from .propagator import TimeStepError
    try:
        return C.sweep(X, grid, c_new, **kw)
    except TimeStepError as exc:
        raise PararealError(f"{what} failed at iteration {i}, interval {offset + getattr(exc, 'interval', 0)}: "
                            f"{exc}") from exc


def _finish(trace: RunTrace, dev, X, n_it: int, s0: State, t_grid, oracle) -> list:
    """Copy the iterates to the host once, fill the trace, device boundary errors."""
    L = trace.intervals
    host = [dev.to_host(X[i]) for i in range(n_it + 1)]
    trace.iterate_values = [[host[i][l].copy() for l in range(L + 1)] for i in range(n_it + 1)]
    if oracle is not None:
        ref = dev.to_device([s.values for s in oracle[1:]])
        for i in range(1, n_it + 1):
            err, _ = dev.boundary_error(X[i][1:], ref)
            trace.boundary_errors.append([float(e) for e in err])
    return [s0] + [s0.with_values(host[n_it][l], time=t_grid[l]) for l in range(1, L + 1)]


def run_parareal_device(C, F, s0: State, t_end: float, cfg, oracle: Optional[Sequence[State]] = None,
                        group=None):
    """Parareal with every boundary state in HBM; returns (boundary states of
    the last completed iteration, RunTrace) like parareal.py:363-465.

    ``C`` and ``F`` are GPU propagators (``sweep`` / ``advance_device``); with
    a ``torch.distributed`` ``group`` of several ranks the fine phase is
    sharded (contiguous slice blocks, one all-gather per iteration).
    """
    import torch

    t_grid = _check(C, F, s0, t_end, cfg, oracle)
    dev = F.device
    L, K = cfg.intervals, cfg.max_iters
    world, rank = 1, 0
    if group is not None:
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)
    from .sharding import gather_blocks, shard_bounds
    lo, hi = shard_bounds(L, world, rank)
    if hi - lo > dev.max_slices:
        raise ValueError(f"{hi - lo} slices per rank exceed the device context's {dev.max_slices}")
    variant = VARIANT_CODES[cfg.variant]
    clamp = tuple(cfg.theta_clamp)
    start = time.perf_counter()
    X = [dev.empty(L + 1) for _ in range(K + 1)]
    first = dev.to_device(s0.values)
    for x in X:
        x[0].copy_(first[0])
    c_prev, c_cur = dev.empty(L), dev.empty(L)
    fine = dev.empty(L)
    _sweep(C, X[0], t_grid, c_prev, "coarse_init", 0)
    init_s = time.perf_counter() - start
    trace = RunTrace(intervals=L, variant=cfg.variant, scheduler="device" if world == 1 else f"device-sharded[{world}]")
    trace.init_seconds = init_s
    stop_at = None
    for i in range(1, K + 1):
        tf = time.perf_counter()
        try:
            if world == 1:
                F.advance_device(X[i - 1][:L], t_grid[:L], t_grid[1:L + 1], out=fine)
            else:
                mine = F.advance_device(X[i - 1][lo:hi].contiguous(), t_grid[lo:hi], t_grid[lo + 1:hi + 1])
                gather_blocks(mine, fine, L, group)
        except Exception as exc:
            raise PararealError(f"fine failed at iteration {i}, interval {lo}..{hi - 1}: {exc}") from exc
        ts = time.perf_counter()
        trace.fine_seconds += ts - tf
        th, cr = _sweep(C, X[i], t_grid, c_cur, "correct", i, x_prev=X[i - 1], c_old=c_prev, f_old=fine,
                        variant=variant, clamp=clamp)
        trace.sweep_seconds += time.perf_counter() - ts
        c_prev, c_cur = c_cur, c_prev
        trace.theta_values.append([float(v) for v in th])
        trace.correction_norms.append([float(v) for v in cr])
        trace.iteration_seconds.append(time.perf_counter() - start)
        trace.fine_propagations += hi - lo
        if max(cr) <= cfg.tol:  # the stop test at the end of the sweep (parareal.py:433-435)
            stop_at = i
            break
    n_it = stop_at if stop_at is not None else K
    trace.iterations_run = n_it
    trace.converged = stop_at is not None
    states = _finish(trace, dev, X, n_it, s0, t_grid, oracle)
    if X[0].is_cuda:
        torch.cuda.synchronize()
    trace.total_seconds = time.perf_counter() - start
    return states, trace


def run_parareal_device_pipelined(C, F, s0: State, t_end: float, cfg, chunks: int = 4,
                                  oracle: Optional[Sequence[State]] = None):
    """Device-resident Parareal with the fine phase of iteration i+1 overlapping
    the corrector sweep of iteration i (the pipelined task graph of the
    reference, parareal.py:241-267, at chunk granularity).

    The L slices split into ``chunks`` contiguous groups.  The calling thread
    sweeps chunk by chunk (one ``pint_coarse_sweep`` per chunk on C's context);
    a worker thread launches the batched fine propagation of a chunk of
    iteration i+1 on F's context as soon as the chunk's left boundaries of
    iteration i are final.  ``C`` and ``F`` must own different device contexts
    (each has its own CUDA stream; each thread issues on its own torch stream,
    so the two phases run concurrently).  Results equal ``run_parareal_device``
    bitwise (same inputs per task, batch-invariant fine propagator).
    """
    import torch

    if C.device is F.device:
        raise ValueError("the pipelined driver needs separate device contexts for C and F")
    t_grid = _check(C, F, s0, t_end, cfg, oracle)
    dev = F.device
    L, K = cfg.intervals, cfg.max_iters
    variant = VARIANT_CODES[cfg.variant]
    clamp = tuple(cfg.theta_clamp)
    chunks = max(1, min(chunks, L))
    bounds = [(c * L // chunks, (c + 1) * L // chunks) for c in range(chunks)]
    start = time.perf_counter()
    X = [dev.empty(L + 1) for _ in range(K + 1)]
    coarse = [dev.empty(L) for _ in range(K + 1)]
    fine = [dev.empty(L) for _ in range(K + 1)]
    first = dev.to_device(s0.values)
    for x in X:
        x[0].copy_(first[0])
    torch.cuda.synchronize()
    cond = threading.Condition()
    published = [0] * (K + 1)      # X[i][0..published[i]] are final
    fine_done = [[False] * chunks for _ in range(K + 1)]
    ctl = {"stop": None, "abort": False, "error": None}
    fine_s = [0.0]

    def fine_worker():
        stream = torch.cuda.Stream()
        try:
            with torch.cuda.stream(stream):
                for i in range(1, K + 1):
                    for c, (lo, hi) in enumerate(bounds):
                        with cond:
                            while (published[i - 1] < hi - 1 and not ctl["abort"]
                                   and (ctl["stop"] is None or i <= ctl["stop"])):
                                cond.wait()
                            if ctl["abort"] or (ctl["stop"] is not None and i > ctl["stop"]):
                                return
                        tf = time.perf_counter()
                        F.advance_device(X[i - 1][lo:hi], t_grid[lo:hi], t_grid[lo + 1:hi + 1], out=fine[i][lo:hi])
                        stream.synchronize()
                        fine_s[0] += time.perf_counter() - tf
                        with cond:
                            fine_done[i][c] = True
                            cond.notify_all()
        except BaseException as exc:  # noqa: BLE001 -- surfaced by the sweeping thread
            with cond:
                ctl["error"] = exc
                cond.notify_all()

    trace = RunTrace(intervals=L, variant=cfg.variant, scheduler=f"device-pipelined[{chunks}]")
    sweep_stream = torch.cuda.Stream()
    worker = threading.Thread(target=fine_worker, daemon=True)
    stop_at = None
    try:
        with torch.cuda.stream(sweep_stream):
            for lo, hi in bounds:
                _sweep(C, X[0][lo:hi + 1], t_grid[lo:hi + 1], coarse[0][lo:hi], "coarse_init", 0, offset=lo)
                sweep_stream.synchronize()
                with cond:
                    published[0] = hi
                    cond.notify_all()
                if lo == 0:
                    worker.start()
            trace.init_seconds = time.perf_counter() - start
            for i in range(1, K + 1):
                th_row, c_row = [], []
                for c, (lo, hi) in enumerate(bounds):
                    with cond:
                        while not fine_done[i][c] and ctl["error"] is None:
                            cond.wait()
                        if ctl["error"] is not None:
                            raise PararealError(f"fine failed at iteration {i}: {ctl['error']}") from ctl["error"]
                    ts = time.perf_counter()
                    th, cr = _sweep(C, X[i][lo:hi + 1], t_grid[lo:hi + 1], coarse[i][lo:hi], "correct", i,
                                    offset=lo, x_prev=X[i - 1][lo:hi + 1], c_old=coarse[i - 1][lo:hi],
                                    f_old=fine[i][lo:hi], variant=variant, clamp=clamp)
                    sweep_stream.synchronize()
                    trace.sweep_seconds += time.perf_counter() - ts
                    th_row += [float(v) for v in th]
                    c_row += [float(v) for v in cr]
                    with cond:
                        published[i] = hi
                        cond.notify_all()
                trace.theta_values.append(th_row)
                trace.correction_norms.append(c_row)
                trace.iteration_seconds.append(time.perf_counter() - start)
                if max(c_row) <= cfg.tol:
                    stop_at = i
                    break
    except BaseException:
        with cond:
            ctl["abort"] = True   # the worker returns before its next launch
            cond.notify_all()
        raise
    finally:
        with cond:
            ctl["stop"] = stop_at if stop_at is not None else K
            cond.notify_all()
        if worker.is_alive():
            worker.join()
    n_it = stop_at if stop_at is not None else K
    trace.iterations_run = n_it
    trace.converged = stop_at is not None
    trace.fine_propagations = L * n_it
    trace.fine_seconds = fine_s[0]
    states = _finish(trace, dev, X, n_it, s0, t_grid, oracle)
    trace.total_seconds = time.perf_counter() - start
    return states, trace
