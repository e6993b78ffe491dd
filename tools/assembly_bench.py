"""Jacobian assembly A/B: the pointwise-linearisation kernel (k_jacobian_lin,
default) against the one-dual-pass-per-column kernel (PINT_JAC=columns) on
the BASELINE meshes: assembled blocks compared entry-wise, assembly timed
with CUDA events (median of repeats).  Prints one JSON line per config."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1907_01252_b200.problem import CONFIGS, c5_random_states  # noqa: E402
from paper_1907_01252_b200.propagator import FSIDevice  # noqa: E402

SLICES = {"c1": 10, "c2": 32, "c3": 64, "c4": 16}


def run(name, variant, reps=5):
    os.environ["PINT_JAC"] = variant
    cfg = CONFIGS[name]
    P = cfg.problem
    S = SLICES[name]
    dev = FSIDevice(P, S, restart=1)
    y = dev.to_device(c5_random_states(P, S, 1))
    yo = dev.to_device(c5_random_states(P, S, 2))
    k = [cfg.fine_step] * S
    th = [0.5 + cfg.fine_step] * S
    t1 = [0.3] * S
    dev.assemble(y, yo, k, th, t1)
    torch.cuda.synchronize()
    times = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dev.assemble(y, yo, k, th, t1)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    blocks = dev.jacobian_blocks(S).cpu().numpy()
    del dev
    return float(np.median(times)), blocks


for name in sys.argv[1:] or ["c2", "c3", "c4"]:
    t_new, b_new = run(name, "lin")
    t_old, b_old = run(name, "columns")
    scale = np.abs(b_old).max()
    err = float(np.abs(b_new - b_old).max() / scale)
    print(json.dumps({"config": name, "slices": SLICES[name], "ms_lin": t_new, "ms_columns": t_old,
                      "speedup": t_old / t_new, "max_rel_diff": err}), flush=True)
