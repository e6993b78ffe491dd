"""Full Parareal run of a BASELINE config on the GPU (device-resident drivers).

  python tools/parareal_run.py --config c1 --driver device|pipelined [--chunks 4]

Prints one JSON line: wall time, init (coarse sweep) time, fine-phase time,
iterations, final defect history row.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1907_01252_b200.parareal import (PararealConfig, run_parareal_device,  # noqa: E402
                                             run_parareal_device_pipelined)
from paper_1907_01252_b200.problem import CONFIGS  # noqa: E402
from paper_1907_01252_b200.propagator import (FSIDevice, NewtonSettings, ThetaSettings, initial_state,  # noqa: E402
                                              make_propagator)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c1")
    ap.add_argument("--driver", default="device", choices=("device", "pipelined"))
    ap.add_argument("--chunks", type=int, default=4)
    ap.add_argument("--iters", type=int, default=0)
    ap.add_argument("--variant", default="classic")
    ap.add_argument("--coarse-theta0", type=float, default=None,
                    help="theta0 of the coarse propagator (theta = 1/2 + theta0 K; 0.5 / K = implicit Euler)")
    ap.add_argument("--stab-k", type=float, default=None, help="fixed stabilization time scale (h/U if 0)")
    a = ap.parse_args()
    rc = CONFIGS[a.config]
    P = rc.problem
    if a.stab_k is not None:
        from dataclasses import replace
        P = replace(P, stab_k=a.stab_k if a.stab_k > 0 else P.h_k / P.u_peak)
    nw = NewtonSettings(1e-10, 1e-10)
    dev = FSIDevice(P, rc.intervals)
    F = make_propagator(P, ThetaSettings(rc.fine_step, rc.theta0, nw), device=dev)
    ct0 = rc.theta0 if a.coarse_theta0 is None else a.coarse_theta0
    if a.driver == "pipelined":
        C = make_propagator(P, ThetaSettings(rc.coarse_step, ct0, nw), device=FSIDevice(P, 1))
    else:
        C = make_propagator(P, ThetaSettings(rc.coarse_step, ct0, nw), device=dev)
    cfg = PararealConfig(intervals=rc.intervals, max_iters=a.iters or rc.iterations, tol=1e-30, variant=a.variant)
    t0 = time.perf_counter()
    if a.driver == "pipelined":
        _, tr = run_parareal_device_pipelined(C, F, initial_state(P), rc.t_end, cfg, chunks=a.chunks)
    else:
        _, tr = run_parareal_device(C, F, initial_state(P), rc.t_end, cfg)
    wall = time.perf_counter() - t0
    print(json.dumps({"config": a.config, "driver": a.driver + (f"[{a.chunks}]" if a.driver == "pipelined" else ""),
                      "coarse_theta0": ct0, "variant": a.variant, "stab_k": P.stab_k, "wall_s": wall, "init_s": tr.init_seconds,
                      "fine_s": tr.fine_seconds, "sweep_s": tr.sweep_seconds, "iterations": tr.iterations_run,
                      "fine_steps_x_slices": rc.intervals * rc.fine_steps_per_window * tr.iterations_run,
                      "defects_last_boundary": [row[-1] for row in tr.correction_norms],
                      "max_defect_per_iteration": [max(row) for row in tr.correction_norms],
                      "theta_first_iteration": tr.theta_values[0][:4]}))


if __name__ == "__main__":
    main()
