"""Result rows in the reference's wire format and the GPU experiment driver.

Wire format: the reference CLI's CSV / JSON result rows (reference
pkg/src/pintbench/cli.py:62-65 column order, 17-significant-digit floats
cli.py:378-383, emit_csv / emit_json / load_rows cli.py:386-437), so GPU runs
feed the reference's own `speedup_report`.  The experiment driver restates
`run_experiment` (cli.py:290-371) on the device: sequential fine solve (the
speed-up denominator), the refined-step reference solution (the
discretization floor, reported as variant "discretization"), then Parareal
per (coarse step, variant) with per-iteration boundary errors and the summary
row (measured vs theoretical speed-up).
"""

from __future__ import annotations

import json
import time
from dataclasses import dataclass
from typing import Optional, Sequence

CSV_COLUMNS = (
    "problem", "K", "k", "variant", "iter", "boundary", "rel_err", "theta",
    "t_seq_s", "t_par_s", "speedup_meas", "speedup_theory",
)
DISCRETIZATION_VARIANT = "discretization"


@dataclass(frozen=True)
class ResultRow:
    problem: str
    K: float
    k: float
    variant: str
    iteration: int
    boundary: Optional[int]
    rel_err: float
    theta: Optional[float]
    t_seq_s: Optional[float] = None
    t_par_s: Optional[float] = None
    speedup_meas: Optional[float] = None
    speedup_theory: Optional[float] = None

    def __post_init__(self):
        if self.rel_err < 0.0:
            raise ValueError("errors cannot be negative")
        if self.speedup_meas is not None and self.speedup_meas <= 0.0:
            raise ValueError("measured speedup must be positive")

    def as_tuple(self):
        return (self.problem, self.K, self.k, self.variant, self.iteration, self.boundary, self.rel_err,
                self.theta, self.t_seq_s, self.t_par_s, self.speedup_meas, self.speedup_theory)


def _fmt(v) -> str:
    if v is None:
        return ""
    if isinstance(v, float):
        return f"{v:.17g}"
    return str(v)


def emit_csv(rows: Sequence[ResultRow], path: str) -> None:
    with open(path, "w", newline="") as fh:
        fh.write(",".join(CSV_COLUMNS) + "\n")
        for r in rows:
            fh.write(",".join(_fmt(v) for v in r.as_tuple()) + "\n")


def emit_json(rows: Sequence[ResultRow], path: str, metadata: Optional[dict] = None) -> None:
    with open(path, "w") as fh:
        json.dump({"metadata": metadata or {}, "rows": [dict(zip(CSV_COLUMNS, r.as_tuple())) for r in rows]},
                  fh, indent=1)
        fh.write("\n")


def _row(rec: dict) -> ResultRow:
    def opt(name, cast):
        v = rec.get(name)
        return None if v in (None, "") else cast(v)

    return ResultRow(str(rec["problem"]), float(rec["K"]), float(rec["k"]), str(rec["variant"]), int(rec["iter"]),
                     opt("boundary", int), float(rec["rel_err"]), opt("theta", float), opt("t_seq_s", float),
                     opt("t_par_s", float), opt("speedup_meas", float), opt("speedup_theory", float))


def load_rows(path: str) -> list:
    if path.endswith(".json"):
        with open(path) as fh:
            return [_row(r) for r in json.load(fh)["rows"]]
    out = []
    with open(path) as fh:
        header = tuple(fh.readline().strip().split(","))
        if header != CSV_COLUMNS:
            raise ValueError(f"unexpected CSV header in {path!r}")
        for line in fh:
            line = line.rstrip("\n")
            if line:
                out.append(_row(dict(zip(CSV_COLUMNS, line.split(",")))))
    return out


def model_speedup(r: float, iters: int, intervals: int) -> float:
    """Theoretical Parareal speed-up 1 / (r + (K/N)(1 + r)) for step ratio
    r = k/K, K iterations and N intervals."""
    if not r > 0.0 or not 0 < iters <= intervals:
        raise ValueError("need r > 0 and 0 < iters <= intervals")
    return 1.0 / (r + (iters / intervals) * (1.0 + r))


def sequential_device(F, s0, grid):
    """Sequential fine solve over the boundary grid on the device (the
    speed-up denominator of cli.py:305-316): [len(grid)] states, row 0 = s0."""
    dev = F.device
    out = dev.empty(len(grid))
    out[0:1].copy_(dev.to_device(s0.values))
    for l in range(len(grid) - 1):
        F.advance_device(out[l:l + 1], [grid[l]], [grid[l + 1]], out=out[l + 1:l + 2])
    return out


def run_experiment_gpu(run_cfg, variants=("classic",), coarse_steps=None, reference_factor: int = 4,
                       max_iters: Optional[int] = None, tol: float = 1e-30, newton=None, krylov=None,
                       verbose: bool = False) -> list:
    """Device restatement of the reference ``run_experiment`` (cli.py:290-371)
    for one FSI config: the sequential solve, the refined-step reference and
    every Parareal iterate stay in HBM; boundary errors are device reductions."""
    import torch

    from .parareal import PararealConfig, run_parareal_device
    from .propagator import FSIDevice, KrylovSettings, NewtonSettings, ThetaSettings, initial_state, \
        make_propagator
    P = run_cfg.problem
    L = run_cfg.intervals
    k = run_cfg.fine_step
    newton = newton or NewtonSettings(1e-10, 1e-10)
    krylov = krylov or KrylovSettings()
    dev = FSIDevice(P, L, restart=krylov.restart)
    s0 = initial_state(P)
    grid = [run_cfg.t_end * l / L for l in range(L + 1)]
    grid[-1] = run_cfg.t_end
    fine = make_propagator(P, ThetaSettings(k, run_cfg.theta0, newton), krylov=krylov, device=dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    seq_dev = sequential_device(fine, s0, grid)
    torch.cuda.synchronize()
    t_seq = time.perf_counter() - t0
    ref_prop = make_propagator(P, ThetaSettings(k / reference_factor, run_cfg.theta0, newton), krylov=krylov,
                               device=dev)
    ref_dev = sequential_device(ref_prop, s0, grid)
    disc, _ = dev.boundary_error(seq_dev[1:], ref_dev[1:])
    rows = [ResultRow(P.name, 0.0, k, DISCRETIZATION_VARIANT, 0, l, float(disc[l - 1]), None)
            for l in range(1, L + 1)]
    disc_final = float(disc[L - 1])
    seq_host = dev.to_host(seq_dev)
    seq = [s0] + [s0.with_values(seq_host[l], time=grid[l]) for l in range(1, L + 1)]
    for K in (coarse_steps or [run_cfg.coarse_step]):
        for variant in variants:
            C = make_propagator(P, ThetaSettings(K, run_cfg.theta0, newton), krylov=krylov, device=dev)
            F = make_propagator(P, ThetaSettings(k, run_cfg.theta0, newton), krylov=krylov, device=dev)
            pcfg = PararealConfig(intervals=L, max_iters=max_iters or run_cfg.iterations, tol=tol, variant=variant)
            _, tr = run_parareal_device(C, F, s0, run_cfg.t_end, pcfg, oracle=seq)
            for i in range(1, tr.iterations_run + 1):
                for l in range(1, L + 1):
                    rows.append(ResultRow(P.name, K, k, variant, i, l, tr.boundary_errors[i - 1][l - 1],
                                          tr.theta_values[i - 1][l - 1]))
            # first iteration whose final-boundary error reaches the discretization floor
            qual = next((i for i in range(1, tr.iterations_run + 1)
                         if tr.boundary_errors[i - 1][L - 1] <= disc_final), tr.iterations_run)
            t_par = tr.iteration_seconds[qual - 1]
            rows.append(ResultRow(P.name, K, k, variant, qual, None, tr.boundary_errors[qual - 1][L - 1], None,
                                  t_seq_s=t_seq, t_par_s=t_par, speedup_meas=t_seq / t_par,
                                  speedup_theory=model_speedup(k / K, qual, L)))
            if verbose:
                print(f"[pint-b200] K={K:g} {variant}: {tr.iterations_run} its, t_par {t_par:.3f} s, "
                      f"t_seq {t_seq:.3f} s", flush=True)
    return rows
