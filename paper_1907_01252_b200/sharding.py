"""Multi-GPU slice sharding: the fine tasks of one Parareal
iteration are independent (reference parareal.py:258-261), so the L slices
split into contiguous blocks, one per rank, with ONE exchange per iteration:
an all-gather of the fine endpoints.  Every rank then runs the (cheap,
deterministic) corrector sweep redundantly, so all ranks hold identical
iterates without a second collective.  With NCCL the all-gather moves device
tensors over NVLink; with gloo (CPU tests) host arrays.
"""

from __future__ import annotations

import time
from typing import List, Optional, Sequence

import numpy as np

from .parareal import (PararealConfig, PararealError, RunTrace, _grid, _split_window, boundary_error,
                       correction_norm, parareal_update, theta_weight)
from .state import State


def shard_bounds(L: int, world: int, rank: int):
    """Contiguous block [lo, hi) of slices owned by ``rank`` (sizes differ by <= 1)."""
    base, extra = divmod(L, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def max_over_ranks(value: float, group=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return value
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def _allgather_values(local: List[np.ndarray], L: int, group=None) -> List[np.ndarray]:
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    n = local[0].size if local else 0
    sizes = [shard_bounds(L, world, r) for r in range(world)]
    width = max(hi - lo for lo, hi in sizes)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    buf = torch.zeros((width, n), dtype=torch.float64, device=dev)
    if local:
        buf[:len(local)] = torch.from_numpy(np.stack(local)).to(dev)
    out = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(out, buf, group=group)
    vals: List[np.ndarray] = []
    for r, (lo, hi) in enumerate(sizes):
        arr = out[r].cpu().numpy()
        vals += [arr[i].copy() for i in range(hi - lo)]
    return vals


def run_parareal_sharded(C, F, s0: State, t_end: float, cfg: PararealConfig,
                         oracle: Optional[Sequence[State]] = None, group=None):
    """Parareal with the fine phase sharded over the ranks of ``group``.

    Results are identical to the serial driver (the fine propagator is
    deterministic and batch-invariant; the sweep runs in the same order on
    every rank).  Uses ``F.advance_batch`` for the local shard when present.
    """
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    L = cfg.intervals
    window = (t_end - s0.time) / L
    for prop in (C, F):
        _split_window(window, prop.step)
    t_grid = _grid(s0, t_end, L)
    lo, hi = shard_bounds(L, world, rank)
    K = cfg.max_iters
    t0 = time.perf_counter()
    X = [[s0] + [None] * L for _ in range(K + 1)]
    coarse = [[None] * (L + 1) for _ in range(K + 1)]
    for l in range(L):
        X[0][l + 1] = C.advance(X[0][l], t_grid[l + 1])
        coarse[0][l + 1] = X[0][l + 1]
    init_s = time.perf_counter() - t0
    thetas, corrs, it_s = [], [], []
    stop_at = None
    fine_s = 0.0
    for i in range(1, K + 1):
        tf = time.perf_counter()
        try:
            mine = [X[i - 1][l] for l in range(lo, hi)]
            ends = [t_grid[l + 1] for l in range(lo, hi)]
            if hasattr(F, "advance_batch") and mine:
                outs = F.advance_batch(mine, ends)
            else:
                outs = [F.advance(s, e) for s, e in zip(mine, ends)]
        except Exception as exc:
            raise PararealError(f"fine failed at iteration {i}, interval {lo}..{hi - 1}: {exc}") from exc
        vals = _allgather_values([o.values for o in outs], L, group)
        fine_s += time.perf_counter() - tf
        fine = [s0.with_values(vals[l], time=t_grid[l + 1]) for l in range(L)]
        th_row, c_row = [], []
        for l in range(L):
            cn = C.advance(X[i][l], t_grid[l + 1])
            th = theta_weight(fine[l], cn, cfg.variant, cfg.theta_clamp)
            new = parareal_update(cn, fine[l], coarse[i - 1][l + 1], th)
            X[i][l + 1] = new
            coarse[i][l + 1] = cn
            th_row.append(th)
            c_row.append(correction_norm(new.values, X[i - 1][l + 1].values))
        thetas.append(th_row)
        corrs.append(c_row)
        it_s.append(time.perf_counter() - t0)
        if max(c_row) <= cfg.tol:
            stop_at = i
            break
    n_it = stop_at if stop_at is not None else K
    tr = RunTrace(intervals=L, variant=cfg.variant, scheduler=f"sharded[{world}]")
    tr.iterations_run = n_it
    tr.converged = stop_at is not None
    tr.theta_values = thetas[:n_it]
    tr.correction_norms = corrs[:n_it]
    tr.iterate_values = [[X[i][l].values.copy() for l in range(L + 1)] for i in range(n_it + 1)]
    tr.init_seconds = init_s
    tr.iteration_seconds = it_s[:n_it]
    tr.total_seconds = time.perf_counter() - t0
    tr.fine_propagations = (hi - lo) * n_it
    tr.fine_seconds = fine_s
    if oracle is not None:
        for i in range(1, n_it + 1):
            tr.boundary_errors.append([e.value for e in boundary_error(X[i][1:], oracle[1:])])
    return X[n_it], tr
