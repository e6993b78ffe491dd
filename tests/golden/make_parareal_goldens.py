"""Generate the Parareal golden fixtures: the REFERENCE driver
(pintbench.run_parareal, imported from /root/reference/pkg/src) driving the
CPU-oracle FSI propagators (oracle/fsi_oracle.py) as C and F.

  python tests/golden/make_parareal_goldens.py c1 classic
  python tests/golden/make_parareal_goldens.py small least_squares
  python tests/golden/make_parareal_goldens.py small classic 2e-2   # tol-based stop
  python tests/golden/make_parareal_goldens.py c1 classic 1e-30 25  # damped coarse propagator
                                  # (coarse theta = 1/2 + 25 K = 1: implicit Euler)

Writes tests/golden/parareal_<case>_<variant>.npz with the final boundary
states, the defect history (correction_norms), theta values and the
iteration count.  Run here (the reference is not on the GPU box); the GPU
tests compare against the committed .npz.
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.environ.get("PINT_REF_SRC", "/root/reference/pkg/src"))

from pintbench.parareal import PararealConfig, run_parareal  # noqa: E402  (reference driver)

from oracle import fsi_oracle as O  # noqa: E402
from paper_1907_01252_b200.problem import CONFIGS, channel_3d, small_problem  # noqa: E402

NEWTON = O.OracleNewtonSettings(abs_tol=1e-10, rel_tol=1e-10)

CASES = {
    # name: (problem, t_end, fine step, coarse step, intervals, iterations)
    "c1": (CONFIGS["c1"].problem, 1.0, 0.002, 0.02, 10, 5),
    "small": (small_problem(8, 2), 0.8, 0.01, 0.05, 8, 4),
    "small3d": (channel_3d(10, 2, 2, name="small3d"), 0.2, 0.01, 0.05, 4, 3),
    # BASELINE c2 (32 slices, fine 2^-10, coarse 2^-6), first 3 of its 8 iterations (the oracle needs ~50 min
    # for them on one core; the full 8-iteration run is tests/golden/make_parareal_c2.py)
    "c2k3": (CONFIGS["c2"].problem, CONFIGS["c2"].t_end, CONFIGS["c2"].fine_step, CONFIGS["c2"].coarse_step, 32, 3),
}


def main(case, variant, tol=1e-30, coarse_theta0=1.0):
    P, t_end, kf, kc, L, K = CASES[case]
    F = O.OracleFSIPropagator(P, kf, 1.0, NEWTON)
    C = O.OracleFSIPropagator(P, kc, coarse_theta0, NEWTON)
    s0 = O.initial_state(P)
    cfg = PararealConfig(intervals=L, max_iters=K, tol=tol, variant=variant)
    t0 = time.time()
    states, trace = run_parareal(C, F, s0, t_end, cfg)
    dt = time.time() - t0
    tag = ("" if tol == 1e-30 else "_tol") + ("" if coarse_theta0 == 1.0 else f"_ct{coarse_theta0:g}")
    out = os.path.join(HERE, f"parareal_{case}_{variant}{tag}.npz")
    np.savez_compressed(out, final=np.array([s.values for s in states]), tol=tol, converged=trace.converged,
                        correction_norms=np.array(trace.correction_norms),
                        theta_values=np.array(trace.theta_values), iterations_run=trace.iterations_run,
                        t_end=t_end, kf=kf, kc=kc, L=L, K=K, seconds=dt, coarse_theta0=coarse_theta0,
                        fine_newton=F.newton_iterations, coarse_newton=C.newton_iterations)
    print(out, f"{dt:.1f} s", trace.iterations_run, np.array(trace.correction_norms)[:, -1])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "classic",
         float(sys.argv[3]) if len(sys.argv) > 3 else 1e-30, float(sys.argv[4]) if len(sys.argv) > 4 else 1.0)
