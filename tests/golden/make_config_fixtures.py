"""Generate the per-config parity fixtures from the CPU oracle (oracle/fsi_oracle.py).

  python tests/golden/make_config_fixtures.py c3          # one config
  python tests/golden/make_config_fixtures.py c5_1e5      # kernel fixture only
  python tests/golden/make_config_fixtures.py --kernel c3 # redo the kernel part of an existing fixture

For a time-loop config (c2, c3, c4) the fixture holds
  * ``starts[j]``  -- the oracle's coarse-initialised boundary state X0[l_j]
    (Parareal iteration 0: l_j sequential coarse windows from rest, the
    reference's coarse_init, parareal.py:410-416) for the sample slices
    ``slices``;
  * ``ends[j]``    -- the oracle's state after ``fine_steps`` fine shifted-CN
    steps from ``starts[j]`` at t = l_j * window, for the last two sample slices
    (integrators.py:144-166 bookkeeping, the fine task of parareal.py:417-421);
  * ``r`` / ``jw`` -- residual R(y; y_old) and exact J(y) w at seeded c5-type
    inputs on the config's mesh (seeds stored; the inputs are regenerated
    with ``problem.c5_random_states``), the K1 / K2' kernel fixtures.  The
    BASELINE c5 deformation N(0, 1e-3^2) tangles the finer meshes (J <= 0 at
    some points); ``degenerate`` records that, and ``r`` is then the raw
    assembled residual (the propagator would treat it as +inf).

The GPU tests (tests/test_gpu_configs.py) and bench.py's parity field and
reference arm read these files; nothing here runs on the GPU box.
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import fsi_oracle as O  # noqa: E402
from paper_1907_01252_b200.problem import CONFIGS, c5_problem, c5_random_states  # noqa: E402

NEWTON = O.OracleNewtonSettings(abs_tol=1e-10, rel_tol=1e-10)
SAMPLES = 8          # sample slices with stored start states (reference arm)
PARITY = 2           # of which the last PARITY also store fine endpoints
FINE_STEPS = 4
SEEDS = (101, 102, 103)   # y, y_old, w of the kernel fixture
KT1 = (2.0 ** -10, 0.3)   # step and time of the kernel fixture (theta = 1/2 + k)


def kernel_fixture(P):
    Y, Yo, W = (c5_random_states(P, 1, sd)[0] for sd in SEEDS)
    k, t1 = KT1
    th = 0.5 + k
    r = O.residual(P, Y, Yo, k, th, t1, admissible_only=False)
    J = O.jacobian(P, Y, Yo, k, th, t1)
    return r, J @ W, O.degenerate(P, Y, Yo, k, th)


# last sample slice per config: the oracle's coarse chain from rest is
# sequential (c3: ~2.5 min of splu per 1/32 window on one core), so c3's
# samples stop at window 15 (t = 0.47, inflow ramp nearly complete)
LAST = {"c3": 15}


def sample_slices(L, last=None):
    # evenly spread, always including the last one (the most developed flow)
    last = L - 1 if last is None else last
    return sorted({last - ((last + 1) // SAMPLES) * j for j in range(SAMPLES)})


def main(name):
    t_start = time.time()
    if name.startswith("c5_"):
        P = c5_problem(name[3:])
        r, jw, dg = kernel_fixture(P)
        out = os.path.join(HERE, f"config_{name}.npz")
        np.savez_compressed(out, r=r, jw=jw, degenerate=dg, seeds=np.array(SEEDS), kt1=np.array(KT1))
        print(out, f"{time.time() - t_start:.1f} s")
        return
    cfg = CONFIGS[name]
    P = cfg.problem
    L = cfg.intervals
    slices = sample_slices(L, LAST.get(name))
    C = O.OracleFSIPropagator(P, cfg.coarse_step, cfg.theta0, NEWTON)
    F = O.OracleFSIPropagator(P, cfg.fine_step, cfg.theta0, NEWTON)
    y = np.zeros(P.num_dofs)
    starts = {}
    for l in range(max(slices) + 1):
        if l in slices:
            starts[l] = y.copy()
        if l == max(slices):
            break
        y = C.advance_values(y, l * cfg.window, (l + 1) * cfg.window)
        print(f"{name}: coarse window {l} done ({time.time() - t_start:.0f} s, "
              f"newton {C.newton_iterations})", flush=True)
    ends, fine_newton = [], []
    for l in slices[-PARITY:]:
        t0 = l * cfg.window
        n0 = F.newton_iterations
        ends.append(F.advance_values(starts[l], t0, t0 + FINE_STEPS * cfg.fine_step))
        fine_newton.append(F.newton_iterations - n0)
    r, jw, dg = kernel_fixture(P)
    out = os.path.join(HERE, f"config_{name}.npz")
    np.savez_compressed(out, degenerate=dg, slices=np.array(slices), starts=np.array([starts[l] for l in slices]),
                        parity_slices=np.array(slices[-PARITY:]), ends=np.array(ends),
                        fine_steps=FINE_STEPS, fine_newton=np.array(fine_newton),
                        coarse_newton=C.newton_iterations, r=r, jw=jw, seeds=np.array(SEEDS),
                        kt1=np.array(KT1), seconds=time.time() - t_start)
    print(out, f"{time.time() - t_start:.1f} s")


def redo_kernel(name):
    """Recompute r / jw / degenerate of an existing fixture (the rest is kept)."""
    out = os.path.join(HERE, f"config_{name}.npz")
    g = dict(np.load(out))
    P = c5_problem(name[3:]) if name.startswith("c5_") else CONFIGS[name].problem
    g["r"], g["jw"], g["degenerate"] = kernel_fixture(P)
    np.savez_compressed(out, **g)
    print(out, "kernel part redone; degenerate =", bool(g["degenerate"]))


if __name__ == "__main__":
    if sys.argv[1] == "--kernel":
        for n in sys.argv[2:]:
            redo_kernel(n)
    else:
        for n in sys.argv[1:]:
            main(n)
