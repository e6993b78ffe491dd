"""CPU, world_size 2 (gloo): the sharded device Parareal driver (one
all_gather_into_tensor of the fine endpoints per iteration, device tensors)
reproduces the single-rank driver bitwise, and the max-over-ranks timing
reduction."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1907_01252_b200.sharding import shard_bounds


def test_shard_bounds_partition():
    for L in (1, 5, 32, 64):
        for W in (1, 2, 3, 8):
            spans = [shard_bounds(L, W, r) for r in range(W)]
            assert spans[0][0] == 0 and spans[-1][1] == L
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    import torch.distributed as dist
    import linprop
    from paper_1907_01252_b200.parareal import PararealConfig
    from paper_1907_01252_b200.sharding import max_over_ranks, run_parareal_sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = linprop.CPUDevice()
    F = linprop.DeviceLinearPropagator(0.01, theta0=1.0, device=dev)
    C = linprop.DeviceLinearPropagator(0.1, theta0=1.0, device=dev)
    cfg = PararealConfig(intervals=7, max_iters=4, tol=1e-30, variant="least_squares")
    _, tr = run_parareal_sharded(C, F, linprop.s0(), 1.4, cfg)
    m = max_over_ranks(float(rank + 1))
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), it=np.array(tr.iterate_values),
             corr=np.array(tr.correction_norms), theta=np.array(tr.theta_values), m=m, fine=tr.fine_propagations,
             fine_calls=F.calls)
    dist.destroy_process_group()


def test_sharded_device_driver_equals_single_rank(tmp_path):
    """world_size 2 over gloo: every rank propagates its block of 7 slices
    (4 + 3), one all-gather per iteration, identical iterates on both ranks,
    equal to the single-rank device driver bitwise."""
    import linprop
    from paper_1907_01252_b200.parareal import PararealConfig, run_parareal_device
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    dev = linprop.CPUDevice()
    F = linprop.DeviceLinearPropagator(0.01, theta0=1.0, device=dev)
    C = linprop.DeviceLinearPropagator(0.1, theta0=1.0, device=dev)
    _, ref = run_parareal_device(C, F, linprop.s0(), 1.4,
                                 PararealConfig(intervals=7, max_iters=4, tol=1e-30, variant="least_squares"))
    fines = 0
    for r in range(world):
        d = np.load(os.path.join(tmp_path, f"r{r}.npz"))
        assert np.array_equal(d["it"], np.array(ref.iterate_values))
        assert np.array_equal(d["corr"], np.array(ref.correction_norms))
        assert np.array_equal(d["theta"], np.array(ref.theta_values))
        assert float(d["m"]) == 2.0
        fines += int(d["fine"])
        assert int(d["fine_calls"]) == (4 if r == 0 else 3) * 4  # only the rank's own block
    assert fines == ref.fine_propagations
