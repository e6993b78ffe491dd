"""Multi-GPU slice sharding of the fine phase.

The fine tasks of one Parareal iteration are independent (reference
parareal.py:258-261), so the L slices split into contiguous blocks, one per
rank.  ONE exchange per iteration assembles F(X[i-1]) on every rank: an
all-gather of device tensors (``all_gather_into_tensor``: NCCL over NVLink /
NVSwitch on GPUs, gloo on CPU tensors in the tests).  Every rank then runs
the same deterministic corrector sweep, so all ranks hold identical iterates
without a second collective.  The driver is ``run_parareal_device(...,
group=...)`` (parareal.py of this package).
"""

from __future__ import annotations

from typing import Optional, Sequence


def shard_bounds(L: int, world: int, rank: int):
    """Contiguous block [lo, hi) of slices owned by ``rank`` (sizes differ by <= 1)."""
    base, extra = divmod(L, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def gather_blocks(mine, out, L: int, group=None):
    """All-gather every rank's block of slice states into ``out`` [L, ...]
    (device tensors stay on the device).  Blocks are padded to the largest
    block so one ``all_gather_into_tensor`` moves everything."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    sizes = [shard_bounds(L, world, r) for r in range(world)]
    width = max(hi - lo for lo, hi in sizes)
    lo, hi = sizes[rank]
    send = torch.zeros((width,) + tuple(out.shape[1:]), dtype=out.dtype, device=out.device)
    send[:hi - lo].copy_(mine)
    recv = torch.empty((world * width,) + tuple(out.shape[1:]), dtype=out.dtype, device=out.device)
    dist.all_gather_into_tensor(recv, send, group=group)
    for r, (a, b) in enumerate(sizes):
        out[a:b].copy_(recv[r * width:r * width + (b - a)])
    return out


def max_over_ranks(value: float, group=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return value
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def run_parareal_sharded(C, F, s0, t_end: float, cfg, oracle: Optional[Sequence] = None, group=None):
    """Parareal with the fine phase sharded over the ranks of ``group``
    (the default group when None); identical iterates on every rank."""
    import torch.distributed as dist
    from .parareal import run_parareal_device
    return run_parareal_device(C, F, s0, t_end, cfg, oracle=oracle, group=group or dist.group.WORLD)
