"""One Jacobian assembly of a BASELINE config (for ncu: -k regex:k_jacobian)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1907_01252_b200.problem import CONFIGS, c5_random_states  # noqa: E402
from paper_1907_01252_b200.propagator import FSIDevice  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
S = {"c1": 10, "c2": 32, "c3": 64, "c4": 16}[name]
cfg = CONFIGS[name]
dev = FSIDevice(cfg.problem, S, restart=1)
y = dev.to_device(c5_random_states(cfg.problem, S, 1))
yo = dev.to_device(c5_random_states(cfg.problem, S, 2))
dev.assemble(y, yo, [cfg.fine_step] * S, [0.5 + cfg.fine_step] * S, [0.3] * S)
torch.cuda.synchronize()
print("ok")
