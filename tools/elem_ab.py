"""A/B timing of the element kernels (K1 residual, K2' J w, K2 assembly) on
BASELINE meshes with c5-type inputs under environment switches (read at
pint_create), e.g.

  python tools/elem_ab.py --cases c3 c2 --variants "" PINT_JAC=colour PINT_ELEM=old

CUDA events, median of repeats, L2 flushed.  One JSON line per case: times
per variant and the max relative difference of r, J w and the assembled
operator against the first variant."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1907_01252_b200.problem import CONFIGS, c5_problem, c5_random_states  # noqa: E402
from paper_1907_01252_b200.propagator import FSIDevice  # noqa: E402

CASES = {"c3": (CONFIGS["c3"].problem, 64), "c4": (CONFIGS["c4"].problem, 16), "c2": (CONFIGS["c2"].problem, 32),
         "c5_1e5x16": (c5_problem("1e5"), 16), "c5_1e6x8": (c5_problem("1e6"), 8)}


def timed(fn, flush, reps=7):
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", nargs="+", default=list(CASES))
    ap.add_argument("--variants", nargs="+", default=["", "PINT_ELEM=old"])
    a = ap.parse_args()
    for name in a.cases:
        P, S = CASES[name]
        out = {}
        for var in a.variants:
            env = dict(kv.split("=", 1) for kv in var.split())
            saved = {k: os.environ.get(k) for k in env}
            os.environ.update(env)
            dev = FSIDevice(P, S, restart=1)
            for k_, v_ in saved.items():
                if v_ is None:
                    os.environ.pop(k_, None)
                else:
                    os.environ[k_] = v_
            # a small deformation keeps the random meshes admissible on every BASELINE mesh
            y = dev.to_device(0.05 * c5_random_states(P, S, 1))
            yo = dev.to_device(0.05 * c5_random_states(P, S, 2))
            w = dev.to_device(c5_random_states(P, S, 3))
            k, th, t1 = [2.0 ** -10] * S, [0.5 + 2.0 ** -10] * S, [0.3] * S
            r, jw = dev.empty(S), dev.empty(S)
            res = {"residual_ms": timed(lambda: dev.residual(y, yo, k, th, t1, out=r), flush),
                   "jvp_ms": timed(lambda: dev.jvp(y, yo, w, k, th, t1, out=jw), flush),
                   "assembly_ms": timed(lambda: dev.assemble(y, yo, k, th, t1), flush)}
            res["r"] = dev.to_host(r)
            res["jw"] = dev.to_host(jw)
            res["J"] = dev.jacobian_blocks(S)  # stays on the device
            out[var or "default"] = res
            del dev
        keys = list(out)
        ref = out[keys[0]]
        rel = {v: {**{f: float(np.abs(out[v][f] - ref[f]).max() / np.abs(ref[f]).max()) for f in ("r", "jw")},
                   "J": float((out[v]["J"] - ref["J"]).abs().max() / ref["J"].abs().max())} for v in keys[1:]}
        print(json.dumps({"case": name, "slices": S, "cells": P.num_cells,
                          **{f"{v}_{k}": out[v][k] for v in out for k in out[v] if k.endswith("_ms")},
                          "max_rel_diff": rel}), flush=True)


if __name__ == "__main__":
    main()
