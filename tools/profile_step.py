"""Profiling driver: a short batched fine propagation inside an NVTX range
"prof" (for ncu --nvtx --nvtx-include prof/), after one warm-up call.

  python tools/profile_step.py --config c2 --steps 2
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1907_01252_b200.problem import CONFIGS  # noqa: E402
from paper_1907_01252_b200.propagator import (FSIDevice, KrylovSettings, NewtonSettings,  # noqa: E402
                                              ThetaSettings, initial_state, make_propagator)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--slices", type=int, default=0)
    ap.add_argument("--max-levels", type=int, default=0)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    P = cfg.problem
    S = a.slices or cfg.intervals
    dev = FSIDevice(P, S)
    newton = NewtonSettings(1e-10, 1e-10)
    ks = KrylovSettings(max_levels=a.max_levels)
    F = make_propagator(P, ThetaSettings(cfg.fine_step, cfg.theta0, newton), krylov=ks, device=dev)
    C = make_propagator(P, ThetaSettings(cfg.coarse_step, cfg.theta0, newton), krylov=ks, device=dev)
    # start states: one coarse window from rest, replicated with staggered times
    s0 = initial_state(P)
    y = dev.to_device([s0.values] * S)
    t0 = [0.25 + 0.0 * s for s in range(S)]
    base = C.advance_device(dev.to_device(s0.values), [0.0], [0.25])
    y[:] = base[0]
    t1 = [t + a.steps * cfg.fine_step for t in t0]
    F.advance_device(y, t0, [t + cfg.fine_step for t in t0])  # warm-up
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("prof")
    F.advance_device(y, t0, t1)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    print("newton", F.newton_iterations, "krylov", F.krylov_iterations)


if __name__ == "__main__":
    main()
