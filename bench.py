"""Benchmark: batched fine propagator throughput (fine CN steps x slices / s).

One bench *step* = the fine phase of one Parareal iteration of BASELINE
config c2 (configs[1]): all 32 slices of the 64x16 channel/bar problem
advanced over one window (64 shifted-CN steps of 2^-10 s, SURVEY §0.4
substitution of the non-divisible 0.001) in ONE batched launch sequence,
starting from the coarse-initialised boundary states (what iteration 1 of
Parareal propagates).  Inputs are resident in HBM when the timed region
starts; L2 (126 MB) is flushed before every timed step (a 256 MB write).

``value``  : slices x fine steps / device time (CUDA events, max over ranks)
``e2e``    : the same through the public host-State API (``advance_batch``:
             host States in, host States out; H2D of the inputs and D2H of
             the results inside every timed step)
``roofline``: the level-0 cell-patch Vanka solve (k_vanka_cell), the
             largest HBM-class kernel of the step, timed with CUDA events
             around every launch in a separate profiled step; ``traffic`` is
             its DRAM bytes per launch from the committed ncu --set full
             capture (profiles/r01_ncu_traffic.json)
``cpu_baseline``: the CPU oracle (numpy/scipy port of the same CN step,
             oracle/fsi_oracle.py) on a bounded sample of the same workload.

``--impl reference`` runs the reference arm: the CPU implementation of the
path (the oracle port -- the reference package ships no FSI propagator,
SURVEY §0.1) on all host cores, same metric/config, bounded sample per step.
Multi-GPU (torchrun): slices shard across ranks with no data-path
collective (weak scaling: every rank owns its own 32-slice batch).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "fine CN steps x slices/sec (2D/3D FSI)"
UNIT = "steps*slices/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for name, val in zip(names, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def _traffic(config, kernel):
    """DRAM bytes per launch of the roofline kernel from the committed ncu
    --set full capture (tools/ncu_traffic.py), or None when there is none."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_ncu_traffic.json")) as f:
            e = json.load(f)[config]
    except Exception:
        return None
    base = kernel.split(" ")[0]
    return e["dram_bytes_per_launch"] if base.split("<")[0] in e["kernel"] else None


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_oracle_sample(cfg, slices: int, steps: int, starts=None):
    """Time the CPU oracle on ``slices`` x ``steps`` fine CN steps (1 core)."""
    from oracle import fsi_oracle as O
    P = cfg.problem
    newton = O.OracleNewtonSettings(abs_tol=1e-10, rel_tol=1e-10)
    prop = O.OracleFSIPropagator(P, cfg.fine_step, cfg.theta0, newton)
    import numpy as np
    t0 = time.perf_counter()
    for s in range(slices):
        y = np.zeros(P.num_dofs) if starts is None else starts[s]
        t = s * cfg.window
        prop.advance_values(y, t, t + steps * cfg.fine_step)
    dt = time.perf_counter() - t0
    return slices * steps / dt, dt


def _ref_worker(args):
    name, slices_idx, steps = args
    from paper_1907_01252_b200.problem import CONFIGS
    cfg = CONFIGS[name]
    rate, dt = cpu_oracle_sample(cfg, len(slices_idx), steps)
    return len(slices_idx) * steps, dt


def run_reference(args):
    """Reference arm: the CPU path (oracle port) on all host cores."""
    ws, rank, _ = _dist()
    if rank != 0:
        return
    import multiprocessing as mp
    from paper_1907_01252_b200.problem import CONFIGS
    cfg = CONFIGS[args.config]
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    nproc = max(1, min(cores, cfg.intervals))
    steps_per = 2
    ctx = mp.get_context("spawn")
    times = []
    # one BLAS thread per worker process: the workers inherit the environment at spawn
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"
    with ctx.Pool(nproc) as pool:
        for it in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            pool.map(_ref_worker, [(args.config, [p], steps_per) for p in range(nproc)])
            dt = time.perf_counter() - t0
            if it >= args.warmup:
                times.append(dt)
    units = nproc * steps_per
    step_s = sum(times) / len(times)
    value = units / step_s
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * step_s, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config} fine phase sample", "mesh": list(cfg.problem.cells),
                   "slices": nproc, "fine_steps_per_slice": steps_per},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nproc, "kind": "port",
                         "sample": f"{nproc} slices x {steps_per} fine CN steps of {args.config} per step from "
                                   "rest at each window start, one process per slice (oracle/fsi_oracle.py; the "
                                   "reference ships no FSI propagator, SURVEY §0.1)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def coarse_states(C, dev, cfg, s0):
    """Coarse-initialised boundary states X[0][0..L-1] on the device."""
    import torch
    L = cfg.intervals
    X = dev.empty(L)
    cur = dev.to_device(s0.values)
    X[0].copy_(cur[0])
    for l in range(L - 1):
        nxt = C.advance_device(cur, [l * cfg.window], [(l + 1) * cfg.window])
        X[l + 1].copy_(nxt[0])
        cur = nxt
    torch.cuda.synchronize()
    return X


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1907_01252_b200.problem import CONFIGS
    from paper_1907_01252_b200.propagator import (FSIDevice, KrylovSettings, NewtonSettings, ThetaSettings,
                                                  initial_state, make_propagator)
    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", init_method="env://")
    cfg = CONFIGS[args.config]
    P = cfg.problem
    L = cfg.intervals
    m_f = cfg.fine_steps_per_window
    newton = NewtonSettings(abs_tol=1e-10, rel_tol=1e-10)
    krylov = KrylovSettings(pre_smooth=args.pre, post_smooth=args.post, omega=args.omega, smoother=args.smoother,
                            precond_reuse=args.reuse, max_levels=args.max_levels, rtol_first=args.rtol_first)
    dev = FSIDevice(P, max_slices=L, restart=krylov.restart)
    F = make_propagator(P, ThetaSettings(cfg.fine_step, cfg.theta0, newton), krylov=krylov, device=dev)
    C = make_propagator(P, ThetaSettings(cfg.coarse_step, cfg.theta0, newton), krylov=krylov, device=dev)
    s0 = initial_state(P)
    X0 = coarse_states(C, dev, cfg, s0)
    t0 = [l * cfg.window for l in range(L)]
    t1 = [(l + 1) * cfg.window for l in range(L)]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    out = dev.empty(L)
    stream = torch.cuda.current_stream()

    for _ in range(args.warmup):
        F.advance_device(X0, t0, t1, out=out)
    torch.cuda.synchronize()
    nit0, kit0 = F.newton_iterations, F.krylov_iterations
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    dev.profile(1)  # count launches; CUDA-graph replay stays on
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        ev0.record(stream)
        for _ in range(args.steps):
            flush.zero_()
            F.advance_device(X0, t0, t1, out=out)
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = dev.profile_read()["launches"]
    elapsed_ms = ev0.elapsed_time(ev1)
    if ws > 1:
        tt = torch.tensor([elapsed_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        elapsed_ms = float(tt.item())
        dist.barrier()
    units = ws * L * m_f * args.steps
    value = units / (elapsed_ms / 1e3)
    nit = (F.newton_iterations - nit0) / (L * m_f * args.steps)
    kit = (F.krylov_iterations - kit0) / max(1, F.newton_iterations - nit0)
    # kernel pass: one more step with CUDA events bracketing every launch of the
    # dominant kernel (plain launches: events cannot sit inside a replayed graph)
    dev.profile(2)
    pe0 = torch.cuda.Event(enable_timing=True)
    pe1 = torch.cuda.Event(enable_timing=True)
    flush.zero_()
    pe0.record(stream)
    F.advance_device(X0, t0, t1, out=out)
    pe1.record(stream)
    torch.cuda.synchronize()
    prof = dev.profile_read()
    prof_step_ms = pe0.elapsed_time(pe1)
    dev.profile(0)

    # ---- e2e through the public host-State API (H2D + D2H inside every step)
    # the reference-facing call: advance_batch(host States, t_ends) -> host States
    host_states = [s0.with_values(v, time=t) for v, t in zip(dev.to_host(X0), t0)]
    e2e_times = []
    for it in range(1 + args.steps):
        torch.cuda.synchronize()
        a = time.perf_counter()
        outs = F.advance_batch(host_states, t1)
        torch.cuda.synchronize()
        if it > 0:
            e2e_times.append(time.perf_counter() - a)
    e2e_s = sum(e2e_times) / len(e2e_times)
    if ws > 1:
        tt = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item())
    del outs
    bytes_io = L * P.num_dofs * 8

    # ---- roofline of the dominant kernel (level-0 smoother sweep)
    peak, peak_kind = _peaks()
    kb = prof["slice_launches"] * prof["bytes_per_slice_launch"]
    achieved = (kb / 1e9) / (prof["kernel_ms"] / 1e3) if prof["kernel_ms"] > 0 else 0.0
    kname = prof["kernel"]
    l0_bytes = L * prof["bytes_per_slice_launch"]
    roofline = {
        "kernel": kname,
        "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
        "peak_kind": peak_kind, "traffic": _traffic(args.config, kname),
        "avg_launch_us": 1e3 * prof["kernel_ms"] / max(1, prof["kernel_launches"]),
        "launches": prof["kernel_launches"],
        "share_of_step": prof["kernel_ms"] / prof_step_ms,
        "kernel_pass": "separate step with per-launch CUDA events (graphs off)",
        "algorithmic_bytes_per_slice_launch": prof["bytes_per_slice_launch"],
        "note": (f"{args.config}: algorithmic bytes of this kernel per launch = {l0_bytes / 1e6:.0f} MB for {L} slices"
                 + (" (< 126 MB L2: L2-resident, the fraction is of HBM peak but the kernel streams from L2)"
                    if l0_bytes < 126e6 else "") + "; see profiles/ and DESIGN.md §5"),
    }

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        starts = dev.to_host(X0)[:2]
        rate, dt = cpu_oracle_sample(cfg, 2, 4, starts=starts)
        cpu = {"value": rate, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"2 slices x 4 fine CN steps of {args.config} from the coarse-initialised states "
                         f"({dt:.1f} s; numpy/scipy oracle, oracle/fsi_oracle.py)"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: fine phase of one Parareal iteration, "
                                   f"{L} slices x {m_f} shifted-CN steps per GPU",
                       "mesh": list(P.cells), "dofs_per_slice": P.num_dofs, "slices_per_gpu": L,
                       "fine_step": cfg.fine_step, "substitution": cfg.note, "l2": "flushed before every step",
                       "newton_per_step": nit, "krylov_per_newton": kit,
                       "parallelism": f"slices sharded, {ws} GPU(s), no collective"},
            "e2e": {"value": ws * L * m_f / e2e_s, "unit": UNIT, "h2d_bytes_per_step": bytes_io,
                    "d2h_bytes_per_step": bytes_io},
            "gpu_launches": launches,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--config", default="c2", choices=("c1", "c2", "c3", "c4"))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--pre", type=int, default=1, help="multigrid pre-smoothing sweeps")
    ap.add_argument("--post", type=int, default=1, help="multigrid post-smoothing sweeps")
    ap.add_argument("--omega", type=float, default=0.9, help="smoother damping")
    ap.add_argument("--smoother", default="vanka", choices=("vanka", "jacobi"))
    ap.add_argument("--reuse", type=int, default=32,
                    help="rebuild the multigrid hierarchy every k steps (or on Krylov-count drift)")
    ap.add_argument("--max-levels", type=int, default=0, help="multigrid levels used (0: all)")
    ap.add_argument("--rtol-first", type=float, default=3e-5, help="GMRES rtol of the first Newton iteration")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
