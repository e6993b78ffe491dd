"""GPU parity ladder, Parareal level: the batched GPU fine propagator and the
device coarse sweep + K8 correction (run_parareal_device) against the CPU
oracle driven by the REFERENCE driver (golden fixtures made by
tests/golden/make_parareal_goldens.py): same iteration count, per-slice
endpoint velocity / deformation / pressure to relative L2 <= 1e-6, defect
history within |d_gpu - d_cpu| <= 1e-6 d_cpu + 10 delta_endpoint
(SURVEY §8c rows 11a/11b).  Plus the driver contracts with the GPU
propagator plugged in: exactness frontier, scheduler equivalence."""

import os

import numpy as np
import pytest

from fields import field_errors
from paper_1907_01252_b200.problem import CONFIGS, channel_3d, small_problem

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
CASES = {
    "small": (small_problem(8, 2), 0.8, 0.01, 0.05, 8, 4),
    "c1": (CONFIGS["c1"].problem, 1.0, 0.002, 0.02, 10, 5),
    "small3d": (channel_3d(10, 2, 2, name="small3d"), 0.2, 0.01, 0.05, 4, 3),
}


def _props(P, kf, kc, S):
    from paper_1907_01252_b200.propagator import FSIDevice, NewtonSettings, ThetaSettings, make_propagator
    dev = FSIDevice(P, S)
    nw = NewtonSettings(abs_tol=1e-10, rel_tol=1e-10)
    F = make_propagator(P, ThetaSettings(kf, 1.0, nw), device=dev)
    C = make_propagator(P, ThetaSettings(kc, 1.0, nw), device=dev)
    return F, C


def _check_against_golden(case, variant, driver):
    from paper_1907_01252_b200.parareal import PararealConfig, run_parareal, run_parareal_device
    from paper_1907_01252_b200.propagator import initial_state
    path = os.path.join(GOLD, f"parareal_{case}_{variant}.npz")
    if not os.path.exists(path):
        pytest.skip(f"golden {path} not generated")
    g = np.load(path)
    P, t_end, kf, kc, L, K = CASES[case]
    F, C = _props(P, kf, kc, L)
    cfg = PararealConfig(intervals=L, max_iters=K, tol=1e-30, variant=variant,
                         scheduler="batched" if driver == "batched" else "serial")
    s0 = initial_state(P)
    if driver == "device":
        states, tr = run_parareal_device(C, F, s0, t_end, cfg)
    else:
        states, tr = run_parareal(C, F, s0, t_end, cfg)
    assert tr.iterations_run == int(g["iterations_run"])
    delta = 0.0
    for l in range(1, L + 1):
        errs = field_errors(P, states[l].values, g["final"][l])
        assert max(errs.values()) <= 1e-6, (l, errs)
        ref = g["final"][l]
        delta = max(delta, np.linalg.norm(states[l].values - ref) / np.linalg.norm(ref))
    d_gpu = np.array(tr.correction_norms)
    d_cpu = g["correction_norms"]
    assert d_gpu.shape == d_cpu.shape
    assert np.all(np.abs(d_gpu - d_cpu) <= 1e-6 * d_cpu + 10 * delta), (d_gpu, d_cpu, delta)
    return tr


@pytest.mark.parametrize("driver", ["device", "batched"])
def test_small_classic_matches_reference_driver_on_oracle(cuda, driver):
    _check_against_golden("small", "classic", driver)


def test_3d_classic_matches_reference_driver_on_oracle(cuda):
    _check_against_golden("small3d", "classic", "device")


def test_c1_classic_matches_reference_driver_on_oracle(cuda):
    tr = _check_against_golden("c1", "classic", "device")
    assert tr.fine_propagations == 10 * 5


def test_exactness_frontier_with_gpu_fine(cuda):
    """Boundaries <= i of iteration i equal the sequential fine solution
    (reference test_parareal.py:217-224): needs a deterministic,
    batch-invariant F."""
    from paper_1907_01252_b200.parareal import PararealConfig, run_parareal_device, sequential_solve
    from paper_1907_01252_b200.propagator import initial_state
    P, t_end, kf, kc, L, K = CASES["small"]
    F, C = _props(P, kf, kc, L)
    s0 = initial_state(P)
    grid = [t_end * l / L for l in range(L + 1)]
    seq = sequential_solve(F, s0, grid)
    _, tr = run_parareal_device(C, F, s0, t_end, PararealConfig(intervals=L, max_iters=3, tol=1e-30), oracle=seq)
    for i in range(1, tr.iterations_run + 1):
        for l in range(1, i + 1):
            assert tr.boundary_errors[i - 1][l - 1] <= 1e-12, (i, l, tr.boundary_errors[i - 1][l - 1])


def test_device_and_host_drivers_agree(cuda):
    from paper_1907_01252_b200.parareal import PararealConfig, run_parareal, run_parareal_device
    from paper_1907_01252_b200.propagator import initial_state
    P, t_end, kf, kc, L, K = CASES["small"]
    F, C = _props(P, kf, kc, L)
    s0 = initial_state(P)
    for variant in ("classic", "angle_penalized"):
        cfg = PararealConfig(intervals=L, max_iters=2, tol=1e-30, variant=variant)
        a, ta = run_parareal_device(C, F, s0, t_end, cfg)
        b, tb = run_parareal(C, F, s0, t_end, cfg)
        for l in range(L + 1):
            assert np.allclose(a[l].values, b[l].values, rtol=0, atol=1e-12 * max(1.0, np.abs(b[l].values).max()))
        assert np.allclose(ta.theta_values, tb.theta_values, rtol=1e-12, atol=0)
        assert np.allclose(ta.correction_norms, tb.correction_norms, rtol=1e-9, atol=0)


def test_k8_correction_kernel_matches_host(cuda):
    """K8b (pint_parareal_correct_one) vs parareal_update + theta_weight +
    correction norm on random states, all three variants, plus the
    degenerate-block and clamp cases (reference test_parareal.py:57-99)."""
    import ctypes
    import torch
    from paper_1907_01252_b200 import _lib
    from paper_1907_01252_b200.parareal import correction_norm, parareal_update, theta_weight
    from paper_1907_01252_b200.propagator import _ptr, _stream
    from paper_1907_01252_b200.state import State
    lib = _lib.load()
    C, nn, npad = 5, 300, 320
    rng = np.random.default_rng(0)
    lay = {f"c{i}": (i * nn, nn) for i in range(C)}
    for variant, code in (("classic", 0), ("least_squares", 1), ("angle_penalized", 2)):
        for clamp in ((0.0, 1.0), (0.0, 1.5)):
            vals = [rng.standard_normal(C * nn) for _ in range(4)]
            vals[0][2 * nn:3 * nn] = 0.0  # degenerate coarse block -> weight 1
            cn, fo, co, xp = [State(v, 0.5, lay) for v in vals]
            th_ref = theta_weight(fo, cn, variant, clamp)
            new_ref = parareal_update(cn, fo, co, th_ref)
            corr_ref = correction_norm(new_ref.values, xp.values)
            dev = [torch.zeros((C, npad), dtype=torch.float64, device="cuda") for _ in range(5)]
            for d, v in zip(dev, vals):
                d[:, :nn] = torch.from_numpy(v.reshape(C, nn))
            th, cr = ctypes.c_double(), ctypes.c_double()
            rc = lib.pint_parareal_correct_one(C, nn, npad, _ptr(dev[0]), _ptr(dev[1]), _ptr(dev[2]), _ptr(dev[3]),
                                               _ptr(dev[4]), code, clamp[0], clamp[1], ctypes.byref(th),
                                               ctypes.byref(cr), _stream())
            assert rc == 0
            out = dev[4][:, :nn].cpu().numpy().reshape(-1)
            assert abs(th.value - th_ref) <= 1e-13 * max(1.0, abs(th_ref))
            assert np.allclose(out, new_ref.values, rtol=0, atol=1e-13)
            assert abs(cr.value - corr_ref) <= 1e-12 * corr_ref
    # K8a: batched pre-correction
    f = torch.randn(3, C, npad, dtype=torch.float64, device="cuda")
    c = torch.randn(3, C, npad, dtype=torch.float64, device="cuda")
    d = torch.empty_like(f)
    assert lib.pint_parareal_precorrect(3, C, nn, npad, _ptr(f), _ptr(c), _ptr(d), _stream()) == 0
    assert torch.equal(d, f - c)


def test_gpu_experiment_rows(cuda, tmp_path):
    """Device restatement of the reference run_experiment (cli.py:290-371):
    discretization rows, per-iteration rows and the speed-up summary row, in
    the reference wire format."""
    from paper_1907_01252_b200.problem import RunConfig
    from paper_1907_01252_b200.report import emit_csv, load_rows, run_experiment_gpu
    rc = RunConfig(small_problem(8, 2), t_end=0.8, fine_step=0.01, coarse_step=0.05, intervals=8, iterations=4)
    rows = run_experiment_gpu(rc, variants=("classic",), coarse_steps=[0.05, 0.1])
    disc = [r for r in rows if r.variant == "discretization"]
    summ = [r for r in rows if r.speedup_meas is not None]
    assert len(disc) == 8 and len(summ) == 2
    assert all(r.t_seq_s > 0 and r.speedup_theory > 0 for r in summ)
    per_iter = [r for r in rows if r.boundary is not None and r.variant == "classic" and r.K == 0.05]
    assert len(per_iter) == 4 * 8
    # exactness frontier visible in the rows: boundary <= iteration matches the sequential solve
    assert all(r.rel_err <= 1e-12 for r in per_iter if r.boundary <= r.iteration)
    emit_csv(rows, str(tmp_path / "rows.csv"))
    assert load_rows(str(tmp_path / "rows.csv")) == rows


def test_pipelined_device_driver_equals_device_driver(cuda):
    """Fine phase of iteration i+1 overlapping the sweep of iteration i
    (separate contexts / streams) gives the same numbers bitwise."""
    from paper_1907_01252_b200.parareal import (PararealConfig, run_parareal_device,
                                                 run_parareal_device_pipelined)
    from paper_1907_01252_b200.propagator import (FSIDevice, NewtonSettings, ThetaSettings, initial_state,
                                                  make_propagator)
    P, t_end, kf, kc, L, K = CASES["small"]
    nw = NewtonSettings(1e-10, 1e-10)
    F, C = _props(P, kf, kc, L)
    s0 = initial_state(P)
    cfg = PararealConfig(intervals=L, max_iters=3, tol=1e-30)
    a, ta = run_parareal_device(C, F, s0, t_end, cfg)
    Fp = make_propagator(P, ThetaSettings(kf, 1.0, nw), device=FSIDevice(P, L))
    Cp = make_propagator(P, ThetaSettings(kc, 1.0, nw), device=FSIDevice(P, 1))
    b, tb = run_parareal_device_pipelined(Cp, Fp, s0, t_end, cfg, chunks=3)
    for l in range(L + 1):
        assert np.array_equal(a[l].values, b[l].values)
    assert ta.correction_norms == tb.correction_norms and ta.theta_values == tb.theta_values
    assert tb.fine_propagations == ta.fine_propagations
