"""Profiling driver for the element kernels (c5 inputs): residual, J w and
Jacobian assembly inside an NVTX range "prof" (ncu --nvtx --nvtx-include prof/)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1907_01252_b200.problem import c5_problem, c5_random_states  # noqa: E402
from paper_1907_01252_b200.propagator import FSIDevice  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--size", default="1e5")
ap.add_argument("--slices", type=int, default=4)
a = ap.parse_args()
P = c5_problem(a.size)
dev = FSIDevice(P, a.slices, restart=1)
y = dev.to_device(c5_random_states(P, a.slices, 1))
yo = dev.to_device(c5_random_states(P, a.slices, 2))
w = dev.to_device(c5_random_states(P, a.slices, 3))
k, th, t1 = [2.0 ** -10] * a.slices, [0.5 + 2.0 ** -10] * a.slices, [0.3] * a.slices
dev.assemble(y, yo, k, th, t1)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("prof")
dev.residual(y, yo, k, th, t1)
dev.jvp(y, yo, w, k, th, t1)
dev.assemble(y, yo, k, th, t1)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("ok")
