"""Temporal order of the CN step on c1, with the CPU oracle.

  python tools/order_study.py [--alpha-p 1.0] [--theta0 0] [--pressure paper|theta] [--t-final 0.0625]

Integrates c1 from rest to t_final with steps 2^-8, 2^-9, 2^-10 and against a
solution with an 8x finer step (the procedure of the reference's
``convergence_order``, integrators.py:209-239), per field block.

``--pressure paper``  the scheme of PAPER.md:410-414 (p^n in both theta parts
                      of A_NS), as the oracle and the GPU path implement it;
``--pressure theta``  an analysis variant: p^{n-1} in the old part (a
                      theta-weighted pressure).  It is made by patching a
                      private copy of the oracle source in a temporary
                      directory; nothing in oracle/ or the GPU path changes.
One JSON line.
"""
import argparse
import importlib.util
import json
import os
import sys
import tempfile
import time
from dataclasses import replace

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1907_01252_b200.problem import CONFIGS  # noqa: E402

PAPER = "Po = piola(Jo, GvFio, Fio, pn)"
THETA = "Po = piola(Jo, GvFio, Fio, po)"


def load_oracle(pressure):
    src = open(os.path.join(ROOT, "oracle", "fsi_oracle.py")).read()
    if pressure == "theta":
        assert PAPER in src
        src = src.replace("vo, uo, Gvo, Guo, _, _ = fields(Yo, Nq, dNq)", "vo, uo, Gvo, Guo, po, _ = fields(Yo, Nq, dNq)")
        src = src.replace(PAPER, THETA)
    d = tempfile.mkdtemp()
    path = os.path.join(d, "fsi_oracle_variant.py")
    with open(path, "w") as f:
        f.write(src)
    spec = importlib.util.spec_from_file_location("fsi_oracle_variant", path)
    mod = importlib.util.module_from_spec(spec)
    sys.modules["fsi_oracle_variant"] = mod  # dataclasses resolve their module
    spec.loader.exec_module(mod)
    return mod


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--alpha-p", type=float, default=1.0)
    ap.add_argument("--theta0", type=float, default=0.0)
    ap.add_argument("--pressure", choices=("paper", "theta"), default="paper")
    ap.add_argument("--t-final", type=float, default=0.0625)
    a = ap.parse_args()
    O = load_oracle(a.pressure)
    P = replace(CONFIGS["c1"].problem, alpha_p=a.alpha_p)
    steps = [2.0 ** -8, 2.0 ** -9, 2.0 ** -10]
    nw = O.OracleNewtonSettings(1e-10, 1e-10)
    s0 = np.zeros(P.num_dofs)
    t0 = time.time()
    ref = O.OracleFSIPropagator(P, steps[-1] / 8, a.theta0, nw).advance_values(s0, 0.0, a.t_final)
    n, d = P.num_nodes, P.dim
    blocks = {"v": slice(0, d * n), "u": slice(d * n, 2 * d * n), "p": slice(2 * d * n, None)}
    errs = {b: [] for b in blocks}
    for k in steps:
        y = O.OracleFSIPropagator(P, k, a.theta0, nw).advance_values(s0, 0.0, a.t_final)
        for b, sl in blocks.items():
            errs[b].append(float(np.linalg.norm(y[sl] - ref[sl])))
    order = {b: float(np.polyfit(np.log(steps), np.log(e), 1)[0]) for b, e in errs.items()}
    print(json.dumps({"analysis": "temporal order, CPU oracle", "config": "c1", "pressure": a.pressure,
                      "alpha_p": a.alpha_p, "theta0": a.theta0, "t_final": a.t_final, "steps": steps,
                      "errors": errs, "observed_order": order, "seconds": time.time() - t0}), flush=True)


if __name__ == "__main__":
    main()
