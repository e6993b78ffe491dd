"""Parareal behaviour on the FSI configs, on the GPU.

  python tools/parareal_analysis.py order  [--config c1] [--t-final 0.2]
  python tools/parareal_analysis.py fields [--config c1] [--variants classic least_squares angle_penalized]

``order``  observed temporal order of the fine propagator, the procedure of
           the reference's ``convergence_order`` (integrators.py:209-239):
           integrate to t_final with every step of a sweep, error against a
           solution with an 8x finer step, least-squares slope of
           log(error) vs log(step) -- per field block (v, u, p).
``fields`` one Parareal run per variant (device driver, tol = 1e-30): per
           iteration and boundary the correction norm split into the v, u
           and p blocks, and the error against the sequential fine solution
           per block, next to the discretization error (fine vs 4x refined
           step; the dashed line of PAPER.md's error plots).
One JSON line per result.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1907_01252_b200.parareal import PararealConfig, run_parareal_device, time_grid  # noqa: E402
from paper_1907_01252_b200.problem import CONFIGS  # noqa: E402
from paper_1907_01252_b200.propagator import (FSIDevice, NewtonSettings, ThetaSettings, initial_state,  # noqa: E402
                                              make_propagator)
from paper_1907_01252_b200.report import sequential_device  # noqa: E402

NW = NewtonSettings(1e-10, 1e-10)


def blocks(P):
    n, d = P.num_nodes, P.dim
    return {"v": slice(0, d * n), "u": slice(d * n, 2 * d * n), "p": slice(2 * d * n, (2 * d + 1) * n)}


def rel(a, b, sl):
    nb = np.linalg.norm(b[sl])
    return float(np.linalg.norm(a[sl] - b[sl]) / nb) if nb > 0 else float(np.linalg.norm(a[sl] - b[sl]))


def order(cfg_name, t_final, steps, theta0=None):
    rc = CONFIGS[cfg_name]
    P = rc.problem
    th0 = rc.theta0 if theta0 is None else theta0
    dev = FSIDevice(P, 1)
    s0 = initial_state(P)
    ref = make_propagator(P, ThetaSettings(min(steps) / 8, th0, NW), device=dev).advance(s0, t_final)
    errs = {b: [] for b in ("v", "u", "p", "all")}
    for k in steps:
        end = make_propagator(P, ThetaSettings(k, th0, NW), device=dev).advance(s0, t_final)
        for b, sl in blocks(P).items():
            errs[b].append(max(float(np.linalg.norm(end.values[sl] - ref.values[sl])), 1e-300))
        errs["all"].append(max(float(np.linalg.norm(end.values - ref.values)), 1e-300))
    lk = np.log(np.asarray(steps))
    slopes = {b: float(np.polyfit(lk, np.log(np.asarray(e)), 1)[0]) for b, e in errs.items()}
    print(json.dumps({"analysis": "temporal order (reference convergence_order procedure)", "config": cfg_name,
                      "t_final": t_final, "steps": steps, "theta0": th0, "errors": errs,
                      "observed_order": slopes}), flush=True)


def fields(cfg_name, variants, iters, coarse_step=None, mu_s=None, coarse_theta0=None):
    from dataclasses import replace
    rc = CONFIGS[cfg_name]
    if coarse_step:
        rc = replace(rc, coarse_step=coarse_step)
    if mu_s:
        rc = replace(rc, problem=replace(rc.problem, mu_s=mu_s))
    P = rc.problem
    L = rc.intervals
    dev = FSIDevice(P, L)
    s0 = initial_state(P)
    grid = time_grid(0.0, rc.t_end, L)
    F = make_propagator(P, ThetaSettings(rc.fine_step, rc.theta0, NW), device=dev)
    seq = dev.to_host(sequential_device(F, s0, grid))
    refp = make_propagator(P, ThetaSettings(rc.fine_step / 4, rc.theta0, NW), device=dev)
    fine_ref = dev.to_host(sequential_device(refp, s0, grid))
    bl = blocks(P)
    disc = {b: [rel(seq[l], fine_ref[l], sl) for l in range(1, L + 1)] for b, sl in bl.items()}
    print(json.dumps({"analysis": "discretization error (fine vs 4x refined step)", "config": cfg_name,
                      "per_block_max_over_boundaries": {b: max(v) for b, v in disc.items()},
                      "per_block_last_boundary": {b: v[-1] for b, v in disc.items()}}), flush=True)
    for variant in variants:
        cth0 = rc.theta0 if coarse_theta0 is None else coarse_theta0
        C = make_propagator(P, ThetaSettings(rc.coarse_step, cth0, NW), device=dev)
        Fp = make_propagator(P, ThetaSettings(rc.fine_step, rc.theta0, NW), device=dev)
        cfg = PararealConfig(intervals=L, max_iters=min(iters or rc.iterations, L), tol=1e-30, variant=variant)
        out = {"analysis": "parareal per field", "config": cfg_name, "variant": variant,
               "coarse_step": rc.coarse_step, "coarse_theta": ThetaSettings(rc.coarse_step, cth0, NW).theta,
               "fine_step": rc.fine_step, "mu_s": P.mu_s}
        try:
            _, tr = run_parareal_device(C, Fp, s0, rc.t_end, cfg)
        except Exception as exc:  # a failing coarse step is itself a result
            out["failed"] = str(exc)
            print(json.dumps(out), flush=True)
            continue
        it = [np.asarray(x) for x in tr.iterate_values]
        rows = []
        for i in range(1, tr.iterations_run + 1):
            row = {"iteration": i, "defect_max": max(tr.correction_norms[i - 1]),
                   "theta_mean": float(np.mean(tr.theta_values[i - 1]))}
            for b, sl in bl.items():
                d = [rel(it[i][l], it[i - 1][l], sl) for l in range(1, L + 1)]
                e = [rel(it[i][l], seq[l], sl) for l in range(1, L + 1)]
                row[f"defect_{b}_max"] = max(d)
                row[f"error_{b}_max"] = max(e)
                row[f"error_{b}_last"] = e[-1]
                row[f"below_discretization_{b}"] = sum(1 for l in range(L) if e[l] <= disc[b][l])
            rows.append(row)
        out["iterations"] = rows
        out["fine_steps_x_slices"] = L * rc.fine_steps_per_window * tr.iterations_run
        print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=("order", "fields"))
    ap.add_argument("--config", default="c1")
    ap.add_argument("--t-final", type=float, default=0.2)
    ap.add_argument("--steps", type=float, nargs="+", default=[0.008, 0.004, 0.002, 0.001])
    ap.add_argument("--variants", nargs="+", default=["classic", "least_squares", "angle_penalized"])
    ap.add_argument("--iters", type=int, default=0)
    ap.add_argument("--theta0", type=float, default=None, help="order: theta = 1/2 + theta0 k (default: config's)")
    ap.add_argument("--coarse-step", type=float, default=None, help="fields: override the coarse step")
    ap.add_argument("--coarse-theta0", type=float, default=None,
                    help="fields: coarse theta = 1/2 + theta0 K (clamped to 1: 0.5/K gives implicit Euler)")
    ap.add_argument("--mu-s", type=float, default=None, help="fields: override the solid shear modulus")
    a = ap.parse_args()
    if a.what == "order":
        order(a.config, a.t_final, a.steps, a.theta0)
    else:
        fields(a.config, a.variants, a.iters, a.coarse_step, a.mu_s, a.coarse_theta0)


if __name__ == "__main__":
    main()
