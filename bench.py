"""Benchmark: batched fine propagator throughput (fine CN steps x slices / s).

One bench *step* = the fine phase of one Parareal iteration of BASELINE
config c3 (configs[2], the largest single-GPU configuration: 256x64 mesh,
mu_s = 2e6): all 64 slices advanced over one window (64 shifted-CN steps of
2^-11 s, SURVEY §0.4 substitution of the non-divisible 5e-4) in ONE
pint_propagate call -- one CUDA-graph launch whose conditional nodes run the
time-step / Newton / GMRES loops on the device -- starting from the
coarse-initialised boundary states (what iteration 1 of Parareal propagates).
Inputs are resident in HBM when the timed region starts; L2 (126 MB) is
flushed before every timed step (a 256 MB write).  ``--config`` selects
another BASELINE config (c1, c2, c4).

``value``  : slices x fine steps / device time (CUDA events, max over ranks)
``e2e``    : the same through the public host-State API (``advance_batch``:
             host States in, host States out; H2D of the inputs and D2H of
             the results inside every timed step)
``roofline``: the dominant HBM-class kernel (level-0 Vanka sweep), timed with
             CUDA events around every launch in a separate profiled step;
             ``traffic`` = its DRAM bytes per launch from the committed ncu
             --set full capture (profiles/)
``parity`` : the GPU propagator on the oracle-made start states of the
             config fixture (tests/golden/config_<c>.npz) against the oracle's
             endpoints: per-field relative L2 (north-star bar 1e-6)
``cpu_baseline``: the CPU oracle (numpy/scipy port of the same CN step,
             oracle/fsi_oracle.py) on a bounded sample of the same workload,
             from the same fixture start states, one core.

``--impl reference`` runs the reference arm: the CPU implementation of the
path (the oracle port -- the reference package ships no FSI propagator,
SURVEY §0.1) on all host cores, same metric / config, from the oracle's own
coarse-initialised start states of the sample slices (the fixture; never GPU
output), one process per sample slice, one CN step per slice per bench step.
Multi-GPU (torchrun): slices shard across ranks with no data-path
collective (weak scaling: every rank owns its own batch of the config).
"""

from __future__ import annotations

import argparse
import json
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
        with open(os.path.join(ROOT, "profiles", "r02_ncu_traffic.json")) as f:
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


def fixture(config):
    """The oracle-made parity / start-state fixture of a config (or None)."""
    import numpy as np
    path = os.path.join(ROOT, "tests", "golden", f"config_{config}.npz")
    if not os.path.exists(path):
        return None
    g = np.load(path)
    return {k: g[k] for k in g.files}


def workload_config(args, cfg, ws):
    """The static workload description, identical in both arms (the driver
    compares the two lines' ``config``)."""
    P = cfg.problem
    return {"workload": f"{args.config}: fine phase of one Parareal iteration, "
                        f"{cfg.intervals} slices x {cfg.fine_steps_per_window} shifted-CN steps per GPU",
            "mesh": list(P.cells), "dofs_per_slice": P.num_dofs, "slices_per_gpu": cfg.intervals,
            "fine_step": cfg.fine_step, "substitution": cfg.note or "none", "mu_s": P.mu_s,
            "start_states": "coarse-initialised boundary states (Parareal iteration 1)",
            "l2": "flushed before every step", "parallelism": f"slices sharded, {ws} GPU(s), no collective"}


def _oracle_prop(cfg):
    from oracle import fsi_oracle as O
    return O.OracleFSIPropagator(cfg.problem, cfg.fine_step, cfg.theta0,
                                 O.OracleNewtonSettings(abs_tol=1e-10, rel_tol=1e-10))


def cpu_oracle_sample(cfg, fx, budget_s: float = 10.0):
    """The CPU oracle (1 core) on fixture start states: fine CN steps of the
    sample slices, round robin, until ``budget_s`` has passed (>= 1 step)."""
    prop = _oracle_prop(cfg)
    ys = {int(l): fx["starts"][j].copy() for j, l in enumerate(fx["slices"])}
    ts = {l: l * cfg.window for l in ys}
    order = sorted(ys)[::-1]
    done, t0 = 0, time.perf_counter()
    while True:
        l = order[done % len(order)]
        ys[l] = prop.advance_values(ys[l], ts[l], ts[l] + cfg.fine_step)
        ts[l] += cfg.fine_step
        done += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    dt = time.perf_counter() - t0
    return done / dt, dt, done


_REF = {}


def _ref_init(name):
    from paper_1907_01252_b200.problem import CONFIGS
    _REF["cfg"] = CONFIGS[name]
    _REF["prop"] = _oracle_prop(_REF["cfg"])
    _REF["fx"] = fixture(name)


def _ref_step(j):
    """One fine CN step of sample slice j from its oracle-made start state."""
    cfg, fx = _REF["cfg"], _REF["fx"]
    l = int(fx["slices"][j])
    t = l * cfg.window
    _REF["prop"].advance_values(fx["starts"][j], t, t + cfg.fine_step)
    return 1


def run_reference(args):
    """Reference arm: the CPU path (oracle port) on all host cores, from the
    oracle's own coarse-initialised states of the config's sample slices."""
    ws, rank, _ = _dist()
    if rank != 0:
        return
    import multiprocessing as mp
    from paper_1907_01252_b200.problem import CONFIGS
    cfg = CONFIGS[args.config]
    fx = fixture(args.config)
    if fx is None:
        print(json.dumps({"impl": "reference", "unavailable": f"fixture tests/golden/config_{args.config}.npz "
                                                              "missing (oracle start states)"}), flush=True)
        return
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    nproc = max(1, min(cores, len(fx["slices"])))
    # one BLAS thread per worker process (inherited at spawn); oracle built by the pool initializer
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"
    # a CPU arm has nothing to warm up beyond its first step (no JIT, no caches
    # that outlive a step): at most one untimed step, so the run stays bounded
    warm = min(args.warmup, 1)
    times = []
    with mp.get_context("spawn").Pool(nproc, initializer=_ref_init, initargs=(args.config,)) as pool:
        for it in range(warm + args.steps):
            t0 = time.perf_counter()
            units = sum(pool.map(_ref_step, list(range(nproc))))
            dt = time.perf_counter() - t0
            if it >= warm:
                times.append(dt)
    step_s = sum(times) / len(times)
    value = units / step_s
    sample = (f"{nproc} slices ({', '.join(str(int(l)) for l in fx['slices'][:nproc])}) x 1 fine CN step of "
              f"{args.config} per bench step, from the oracle's coarse-initialised states "
              f"(tests/golden/config_{args.config}.npz), one process per slice, 1 BLAS thread each "
              f"(oracle/fsi_oracle.py; the reference ships no FSI propagator, SURVEY §0.1)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": warm, "warmup_requested": args.warmup, "ms_per_step": 1e3 * step_s,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, cfg, ws),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nproc, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def gpu_parity(F, dev, cfg, fx):
    """GPU fine propagation of the fixture's parity slices from the oracle's
    start states vs the oracle's endpoints: per-field relative L2."""
    import numpy as np
    if fx is None:
        return None
    P = cfg.problem
    idx = [list(fx["slices"]).index(l) for l in fx["parity_slices"]]
    starts = [fx["starts"][j] for j in idx]
    t0 = [int(l) * cfg.window for l in fx["parity_slices"]]
    steps = int(fx["fine_steps"])
    out = dev.to_host(F.advance_device(dev.to_device(starts), t0, [t + steps * cfg.fine_step for t in t0]))
    n, d = P.num_nodes, P.dim
    fields = {"v": slice(0, d * n), "u": slice(d * n, 2 * d * n), "p": slice(2 * d * n, (2 * d + 1) * n)}
    err = {}
    for name, sl in fields.items():
        e = 0.0
        for s in range(len(starts)):
            ref = fx["ends"][s][sl]
            e = max(e, float(np.linalg.norm(out[s][sl] - ref) / np.linalg.norm(ref)))
        err[name] = e
    err.update({"slices": [int(l) for l in fx["parity_slices"]], "fine_steps": steps, "tolerance": 1e-6,
                "pass": max(err[k] for k in fields) <= 1e-6,
                "oracle": f"tests/golden/config_{cfg.problem.name}.npz (oracle coarse-initialised starts)"})
    return err


def coarse_states(C, dev, cfg, s0):
    """Coarse-initialised boundary states X[0][0..L-1] on the device (the
    Parareal coarse initialisation, one pint_coarse_sweep call)."""
    import torch
    L = cfg.intervals
    X = dev.empty(L + 1)
    X[0:1].copy_(dev.to_device(s0.values))
    C.sweep(X, [l * cfg.window for l in range(L + 1)], dev.empty(L))
    torch.cuda.synchronize()
    return X[:L].clone()


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

    # ---- parity on the oracle-made start states (outside the timed region)
    fx = fixture(args.config)
    parity = gpu_parity(F, dev, cfg, fx) if rank == 0 else None
    # the GPU's own coarse initialisation vs the oracle's, at the fixture's sample slices
    if rank == 0 and fx is not None:
        got = dev.to_host(X0)
        parity["coarse_init_rel_l2_max"] = max(
            float(np.linalg.norm(got[int(l)] - fx["starts"][j]) / max(np.linalg.norm(fx["starts"][j]), 1e-300))
            for j, l in enumerate(fx["slices"]) if int(l) < L and np.linalg.norm(fx["starts"][j]) > 0)
    cpu = None
    if rank == 0 and not args.no_cpu_baseline and fx is not None:
        rate, dt, done = cpu_oracle_sample(cfg, fx)
        cpu = {"value": rate, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"{done} fine CN step(s) of {args.config} (sample slices "
                         f"{', '.join(str(int(l)) for l in fx['slices'][::-1][:done])}) from the oracle's "
                         f"coarse-initialised states ({dt:.1f} s; numpy/scipy oracle, oracle/fsi_oracle.py)"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, cfg, ws),
            "solver": {"newton_per_step": nit, "krylov_per_newton": kit,
                       "control_flow": "device (one CUDA graph per call, conditional nodes)"
                       if os.environ.get("PINT_DEVICE_LOOP", "1") != "0" else "host-driven"},
            "e2e": {"value": ws * L * m_f / e2e_s, "unit": UNIT, "h2d_bytes_per_step": bytes_io,
                    "d2h_bytes_per_step": bytes_io},
            "gpu_launches": launches,
            "roofline": roofline,
            "parity": parity,
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
    ap.add_argument("--config", default="c3", choices=("c1", "c2", "c3", "c4"))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--pre", type=int, default=1, help="multigrid pre-smoothing sweeps")
    ap.add_argument("--post", type=int, default=1, help="multigrid post-smoothing sweeps")
    ap.add_argument("--omega", type=float, default=0.0, help="smoother damping (0: the library default, 0.9)")
    ap.add_argument("--smoother", default="vanka", choices=("vanka", "jacobi"))
    ap.add_argument("--reuse", type=int, default=64,
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
