"""A/B timing of the fine phase under environment switches (each variant gets
a fresh device context, since the switches are read at pint_create).

  python tools/loop_ab.py --config c2 --steps 5 PINT_DEVICE_LOOP=0 PINT_DEVICE_LOOP=1 "PINT_DEVICE_LOOP=1 PINT_PDL=0"

Prints one JSON line per variant: ms per bench step (CUDA events, L2 not
flushed), launches per bench step, Newton / Krylov counts.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_1907_01252_b200.problem import CONFIGS
    from paper_1907_01252_b200.propagator import (FSIDevice, NewtonSettings, ThetaSettings, initial_state,
                                                  make_propagator)
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--slices", type=int, default=0, help="batch size (0: the config's intervals)")
    ap.add_argument("variants", nargs="+")
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    P = cfg.problem
    L = a.slices or cfg.intervals
    nw = NewtonSettings(1e-10, 1e-10)
    X0 = None
    for var in a.variants:
        env = dict(kv.split("=", 1) for kv in var.split())
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        dev = FSIDevice(P, L)
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v
        F = make_propagator(P, ThetaSettings(cfg.fine_step, cfg.theta0, nw), device=dev)
        if X0 is None:
            C = make_propagator(P, ThetaSettings(cfg.coarse_step, cfg.theta0, nw), device=dev)
            X = dev.empty(cfg.intervals + 1)
            X[0:1].copy_(dev.to_device(initial_state(P).values))
            C.sweep(X, [l * cfg.window for l in range(cfg.intervals + 1)], dev.empty(cfg.intervals))
            X0 = dev.to_host(X[:L])
        y = dev.to_device(X0)
        t0 = [l * cfg.window for l in range(L)]
        t1 = [(l + 1) * cfg.window for l in range(L)]
        out = dev.empty(L)
        for _ in range(2):
            F.advance_device(y, t0, t1, out=out)
        torch.cuda.synchronize()
        n0, k0 = F.newton_iterations, F.krylov_iterations
        dev.profile(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.steps):
            F.advance_device(y, t0, t1, out=out)
        e1.record()
        torch.cuda.synchronize()
        launches = dev.profile_read()["launches"]
        dev.profile(0)
        ms = e0.elapsed_time(e1) / a.steps
        units = L * cfg.fine_steps_per_window
        print(json.dumps({"config": a.config, "variant": var, "slices": L, "ms_per_step": ms,
                          "steps_x_slices_per_s": units / (ms / 1e3), "launches_per_step": launches / a.steps,
                          "newton_per_cn_step": (F.newton_iterations - n0) / (units * a.steps),
                          "krylov_per_newton": (F.krylov_iterations - k0) / max(1, F.newton_iterations - n0)}),
              flush=True)
        del F, dev
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
