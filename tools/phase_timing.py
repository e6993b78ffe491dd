"""Warm (non-profiler) timings of the pieces of one fine step on a BASELINE
config: Jacobian assembly, multigrid setup, one V-cycle, one level-0 SpMV,
one residual, and GMRES solves (per-iteration cost).  CUDA events on the
current stream, median of repeats.  Prints one JSON line per config."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1907_01252_b200.problem import CONFIGS  # noqa: E402
from paper_1907_01252_b200.propagator import (FSIDevice, KrylovSettings, NewtonSettings,  # noqa: E402
                                              ThetaSettings, initial_state, make_propagator)

SLICES = {"c1": 10, "c2": 32, "c3": 64, "c4": 16}


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))


def main(name):
    cfg = CONFIGS[name]
    P = cfg.problem
    S = SLICES[name]
    dev = FSIDevice(P, S)
    newton = NewtonSettings(1e-10, 1e-10)
    ks = KrylovSettings()
    C = make_propagator(P, ThetaSettings(cfg.coarse_step, cfg.theta0, newton), krylov=ks, device=dev)
    s0 = initial_state(P)
    base = C.advance_device(dev.to_device(s0.values), [0.0], [0.25])
    y = base.repeat(S, 1, 1).contiguous()
    yo = y.clone()
    k = cfg.fine_step
    args = ([k] * S, [0.5 + k] * S, [0.25 + k] * S)
    out = {"config": name, "slices": S}
    out["assemble_us"] = timed(lambda: dev.assemble(y, yo, *args))
    r, _ = dev.residual(y, yo, *args)
    out["residual_us"] = timed(lambda: dev.residual(y, yo, *args))
    out["setup_us"] = timed(lambda: dev.precond_setup(S, ks), reps=5)
    b = torch.randn_like(r)
    x = torch.empty_like(r)
    out["vcycle_us"] = timed(lambda: dev.precond_apply(b, out=x))
    out["spmv_us"] = timed(lambda: dev.spmv(b, out=x))
    for rt in (1e-4, 1e-8):
        kk = KrylovSettings(rtol=rt)
        holder = {}

        def solve():
            holder["its"] = dev.linear_solve(b, kk, out=x)[1]
        t = timed(solve, reps=5)
        its = float(np.mean(holder["its"]))
        out[f"gmres_rtol{rt:g}_us"] = t
        out[f"gmres_rtol{rt:g}_its"] = its
        out[f"gmres_rtol{rt:g}_us_per_it"] = t / its
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    for n in sys.argv[1:] or ["c2"]:
        main(n)
