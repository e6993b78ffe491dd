"""A/B: one batched fine propagation of S slices on one context vs the same
batch split over G contexts of S/G slices, each driven from its own host
thread on its own CUDA stream (the latency-/FP64-bound phases of one group --
Jacobian assembly, V-cycle tail, small coarse levels, loop controllers --
overlap the HBM-bound Krylov kernels of the others).  Results must be
bitwise equal (batch invariance).

  python tools/dual_stream_ab.py --config c3 --steps 16 --groups 1 2 4
"""
import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1907_01252_b200.problem import CONFIGS  # noqa: E402
from paper_1907_01252_b200.propagator import (FSIDevice, KrylovSettings, NewtonSettings,  # noqa: E402
                                              ThetaSettings, initial_state, make_propagator)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--steps", type=int, default=16)
    ap.add_argument("--groups", type=int, nargs="+", default=[1, 2, 4])
    ap.add_argument("--repeat", type=int, default=3)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    P, L = cfg.problem, cfg.intervals
    newton = NewtonSettings(1e-10, 1e-10)
    ks = KrylovSettings()
    dev = FSIDevice(P, L)
    C = make_propagator(P, ThetaSettings(cfg.coarse_step, cfg.theta0, newton), krylov=ks, device=dev)
    X = dev.empty(L + 1)
    X[0:1].copy_(dev.to_device(initial_state(P).values))
    C.sweep(X, [l * cfg.window for l in range(L + 1)], dev.empty(L))
    torch.cuda.synchronize()
    X0 = X[:L].clone()
    t0 = [l * cfg.window for l in range(L)]
    t1 = [t + a.steps * cfg.fine_step for t in t0]
    del C
    ref = None
    for G in a.groups:
        bounds = [(g * L // G, (g + 1) * L // G) for g in range(G)]
        devs = [dev] if G == 1 else [FSIDevice(P, hi - lo) for lo, hi in bounds]
        props = [make_propagator(P, ThetaSettings(cfg.fine_step, cfg.theta0, newton), krylov=ks, device=d)
                 for d in devs]
        out = dev.empty(L)
        streams = [torch.cuda.Stream() for _ in range(G)]

        def work(g):
            lo, hi = bounds[g]
            with torch.cuda.stream(streams[g]):
                props[g].advance_device(X0[lo:hi], t0[lo:hi], t1[lo:hi], out=out[lo:hi])
                streams[g].synchronize()

        def run_once():
            ths = [threading.Thread(target=work, args=(g,)) for g in range(G)]
            torch.cuda.synchronize()
            tb = time.perf_counter()
            for t in ths:
                t.start()
            for t in ths:
                t.join()
            torch.cuda.synchronize()
            return time.perf_counter() - tb

        run_once()  # warm-up (graph capture, hierarchy build)
        best = min(run_once() for _ in range(a.repeat))
        same = None
        if ref is None:
            ref = out.clone()
        else:
            same = bool(torch.equal(ref, out))
        print(json.dumps({"config": a.config, "groups": G, "slices": L, "steps": a.steps, "seconds": best,
                          "steps_x_slices_per_s": L * a.steps / best, "bitwise_equal_to_one_group": same}), flush=True)
        if G > 1:
            del props, devs
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
