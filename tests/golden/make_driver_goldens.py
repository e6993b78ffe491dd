"""Golden traces of the REFERENCE Parareal driver (pintbench.run_parareal)
on the linear test propagator (tests/linprop.py), for every variant:
  python tests/golden/make_driver_goldens.py  ->  tests/golden/driver_linear.npz
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.environ.get("PINT_REF_SRC", "/root/reference/pkg/src"))

from pintbench.parareal import PararealConfig, run_parareal  # noqa: E402

import linprop  # noqa: E402

out = {}
for variant in ("classic", "least_squares", "angle_penalized"):
    F = linprop.LinearPropagator(0.01, theta0=1.0)
    C = linprop.LinearPropagator(0.1, theta0=1.0)
    cfg = PararealConfig(intervals=6, max_iters=4, tol=1e-30, variant=variant)
    states, tr = run_parareal(C, F, linprop.s0(), 1.2, cfg)
    out[f"{variant}_iterates"] = np.array(tr.iterate_values)
    out[f"{variant}_corr"] = np.array(tr.correction_norms)
    out[f"{variant}_theta"] = np.array(tr.theta_values)
    out[f"{variant}_iters"] = tr.iterations_run
    out[f"{variant}_fine"] = tr.fine_propagations
# converging run (tol-based stop)
F = linprop.LinearPropagator(0.01, theta0=1.0)
C = linprop.LinearPropagator(0.1, theta0=1.0)
_, tr = run_parareal(C, F, linprop.s0(), 1.2, PararealConfig(intervals=6, max_iters=6, tol=1e-6))
out["tol_iters"] = tr.iterations_run
out["tol_converged"] = tr.converged
out["tol_corr"] = np.array(tr.correction_norms)
np.savez_compressed(os.path.join(HERE, "driver_linear.npz"), **out)
print("ok", {k: np.shape(v) for k, v in out.items()})
