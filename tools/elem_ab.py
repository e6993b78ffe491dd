"""A/B timing of the element kernels (K1 residual, K2' J w, K2 assembly) on
BASELINE meshes with c5-type inputs: the tiled kernels (default) against the
round-1 per-point kernels (PINT_ELEM=old; the Jacobian kernel has no switch).
CUDA events, median of repeats, L2 flushed.  One JSON line per (config, variant)."""
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
    for name in sys.argv[1:] or list(CASES):
        P, S = CASES[name]
        out = {}
        for var in ("new", "old"):
            if var == "old":
                os.environ["PINT_ELEM"] = "old"
            else:
                os.environ.pop("PINT_ELEM", None)
            dev = FSIDevice(P, S, restart=1)
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
            out[var] = res
            del dev
            torch.cuda.empty_cache()
        os.environ.pop("PINT_ELEM", None)
        rel = {f: float(np.abs(out["new"][f] - out["old"][f]).max() / np.abs(out["old"][f]).max()) for f in ("r", "jw")}
        print(json.dumps({"case": name, "slices": S, "cells": P.num_cells,
                          **{f"{v}_{k}": out[v][k] for v in out for k in out[v] if k.endswith("_ms")},
                          "max_rel_diff": rel}), flush=True)


if __name__ == "__main__":
    main()
