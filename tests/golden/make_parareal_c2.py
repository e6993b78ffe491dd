"""c2 Parareal on the CPU oracle, driven by the REFERENCE driver
(pintbench.run_parareal, scheduler="pipelined", 1 BLAS thread per worker):
does the oracle show the same behaviour as the GPU run -- defects growing
after iteration 4 and a coarse step of iteration 8 running out of its Newton
budget?

  OMP_NUM_THREADS=1 OPENBLAS_NUM_THREADS=1 python tests/golden/make_parareal_c2.py [workers]

The reference driver raises PararealError on the failing step and its trace
is lost with it, so every parareal_update result is recorded on the way
(pintbench.parareal.parareal_update wrapped: per boundary the updates arrive
in iteration order) and the defect history of the completed iterations is
rebuilt from those iterates with the reference's definition
(parareal.py:429-431).  Writes tests/golden/parareal_c2_classic.npz.
"""
import os
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.environ.get("PINT_REF_SRC", "/root/reference/pkg/src"))

import pintbench.parareal as RP  # noqa: E402  (reference driver)

from oracle import fsi_oracle as O  # noqa: E402
from paper_1907_01252_b200.problem import CONFIGS  # noqa: E402

NEWTON = O.OracleNewtonSettings(abs_tol=1e-10, rel_tol=1e-10)


def main(workers):
    rc = CONFIGS["c2"]
    P, L, K = rc.problem, rc.intervals, rc.iterations
    F = O.OracleFSIPropagator(P, rc.fine_step, rc.theta0, NEWTON)
    C = O.OracleFSIPropagator(P, rc.coarse_step, rc.theta0, NEWTON)
    s0 = O.initial_state(P)
    updates = {}
    lock = threading.Lock()
    orig = RP.parareal_update

    def recording_update(coarse_new, fine_old, coarse_old, theta):
        new = orig(coarse_new, fine_old, coarse_old, theta)
        with lock:
            updates.setdefault(round(new.time / rc.window), []).append(new.values.copy())
        return new

    RP.parareal_update = recording_update
    cfg = RP.PararealConfig(intervals=L, max_iters=K, tol=1e-30, scheduler="pipelined", workers=workers)
    t0 = time.time()
    failure, trace = "", None
    try:
        _, trace = RP.run_parareal(C, F, s0, rc.t_end, cfg)
    except RP.PararealError as exc:
        failure = str(exc)
    dt = time.time() - t0
    # iteration 0: the oracle's coarse initialisation (deterministic, recomputed)
    X0 = [s0.values]
    for l in range(L):
        X0.append(C.advance_values(X0[-1], l * rc.window, (l + 1) * rc.window))
    done = min(len(v) for v in updates.values()) if len(updates) == L else 0
    X = [np.array(X0)] + [np.array([s0.values] + [updates[l + 1][i] for l in range(L)]) for i in range(done)]
    corr = []
    for i in range(1, done + 1):
        row = []
        for l in range(1, L + 1):
            diff = float(np.linalg.norm(X[i][l] - X[i - 1][l]))
            norm = float(np.linalg.norm(X[i][l]))
            row.append(0.0 if diff == 0.0 else (diff / norm if norm > 0.0 else float("inf")))
        corr.append(row)
    out = os.path.join(HERE, "parareal_c2_classic.npz")
    np.savez_compressed(out, correction_norms=np.array(corr), iterations_completed=done, failure=failure,
                        final=X[-1], seconds=dt, workers=workers, L=L, K=K,
                        trace_correction_norms=np.array(trace.correction_norms) if trace else np.zeros((0, L)))
    print(out, f"{dt:.0f} s", "failure:", failure or "none", "completed:", done,
          "max defects:", [max(r) for r in corr], flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 6)
