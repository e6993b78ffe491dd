"""GPU parity ladder, Parareal level: the batched GPU fine propagator and the
device coarse sweep + K8 correction (run_parareal_device: pint_coarse_sweep)
against the CPU oracle driven by the REFERENCE driver (golden fixtures made by
tests/golden/make_parareal_goldens.py): same iteration count (fixed-count and
tolerance-stopped runs), per-slice endpoint velocity / deformation / pressure
to relative L2 <= 1e-6, defect history within
|d_gpu - d_cpu| <= 1e-6 d_cpu + 10 delta_endpoint,
for the classic, least-squares and angle-penalized variants.  Plus the
driver contracts with the GPU propagator plugged in: exactness frontier, the
reference driver and the device driver agreeing, pipelined == device."""

import os

import numpy as np
import pytest

from fields import field_errors
from paper_1907_01252_b200.problem import CONFIGS, channel_3d, small_problem
from refimport import pintbench

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
CASES = {
    "small": (small_problem(8, 2), 0.8, 0.01, 0.05, 8, 4),
    "c1": (CONFIGS["c1"].problem, 1.0, 0.002, 0.02, 10, 5),
    "small3d": (channel_3d(10, 2, 2, name="small3d"), 0.2, 0.01, 0.05, 4, 3),
    "c2k3": (CONFIGS["c2"].problem, CONFIGS["c2"].t_end, CONFIGS["c2"].fine_step, CONFIGS["c2"].coarse_step, 32, 3),
}


def _props(P, kf, kc, S, coarse_theta0=1.0):
    from paper_1907_01252_b200.propagator import FSIDevice, NewtonSettings, ThetaSettings, make_propagator
    dev = FSIDevice(P, S)
    nw = NewtonSettings(abs_tol=1e-10, rel_tol=1e-10)
    F = make_propagator(P, ThetaSettings(kf, 1.0, nw), device=dev)
    C = make_propagator(P, ThetaSettings(kc, coarse_theta0, nw), device=dev)
    return F, C


def _check_against_golden(case, variant, driver, tag=""):
    from paper_1907_01252_b200.parareal import PararealConfig, run_parareal_device
    from paper_1907_01252_b200.propagator import initial_state
    path = os.path.join(GOLD, f"parareal_{case}_{variant}{tag}.npz")
    if not os.path.exists(path):
        pytest.skip(f"golden {path} not generated")
    g = np.load(path)
    tol = float(g["tol"]) if "tol" in g else 1e-30
    P, t_end, kf, kc, L, K = CASES[case]
    F, C = _props(P, kf, kc, L, float(g["coarse_theta0"]) if "coarse_theta0" in g else 1.0)
    s0 = initial_state(P)
    if driver == "device":
        cfg = PararealConfig(intervals=L, max_iters=K, tol=tol, variant=variant)
        states, tr = run_parareal_device(C, F, s0, t_end, cfg)
    else:  # the unmodified reference driver with the GPU propagators plugged in
        pb = pintbench()
        if pb is None:
            pytest.skip("reference package not available")
        from pintbench.parareal import PararealConfig as RC, run_parareal as rrun
        states, tr = rrun(C, F, s0, t_end, RC(intervals=L, max_iters=K, tol=tol, variant=variant))
    assert tr.iterations_run == int(g["iterations_run"])
    if "converged" in g:
        assert tr.converged == bool(g["converged"])
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


@pytest.mark.parametrize("driver", ["device", "reference"])
def test_small_classic_matches_reference_driver_on_oracle(cuda, driver):
    _check_against_golden("small", "classic", driver)


@pytest.mark.parametrize("variant", ["least_squares", "angle_penalized"])
def test_small_weighted_variants_match_reference_driver_on_oracle(cuda, variant):
    tr = _check_against_golden("small", variant, "device")
    assert all(0.0 <= th <= 1.0 for row in tr.theta_values for th in row)


@pytest.mark.parametrize("driver", ["device", "reference"])
def test_small_tolerance_stop_matches_reference_driver_on_oracle(cuda, driver):
    """tol-based stop before max_iters: same iterations_run and
    converged flag as the reference driver on the oracle."""
    tr = _check_against_golden("small", "classic", driver, tag="_tol")
    assert tr.converged and tr.iterations_run < 4


def test_3d_classic_matches_reference_driver_on_oracle(cuda):
    _check_against_golden("small3d", "classic", "device")


def test_c1_classic_matches_reference_driver_on_oracle(cuda):
    tr = _check_against_golden("c1", "classic", "device")
    assert tr.fine_propagations == 10 * 5


@pytest.mark.parametrize("variant", ["least_squares", "angle_penalized"])
def test_c1_weighted_variants_match_reference_driver_on_oracle(cuda, variant):
    """BASELINE config c1 with the theta-weighted corrections (parareal.py:166-197):
    same iteration count, defect history, theta values and endpoints as the
    reference driver on the oracle."""
    tr = _check_against_golden("c1", variant, "device")
    assert all(0.0 <= th <= 1.0 for row in tr.theta_values for th in row)


def test_c2_first_iterations_match_reference_driver_on_oracle(cuda):
    """BASELINE config c2 (64x16 mesh, 32 slices): the first 3 Parareal
    iterations against the reference driver on the oracle -- same defect
    history and endpoints (skipped until the golden exists: ~50 min of oracle
    time, tests/golden/make_parareal_goldens.py c2k3)."""
    tr = _check_against_golden("c2k3", "classic", "device")
    assert tr.fine_propagations == 32 * 3


def test_c1_damped_coarse_propagator_converges(cuda):
    """with the shifted-CN coarse propagator (theta_c = 1/2 +
    K = 0.52, stability function -> -(1 - theta)/theta = -0.92 on stiff modes)
    the c1 defects stall near 2 %; with a damped coarse propagator (theta_c =
    1/2 + 25 K = 1, implicit Euler, R(inf) = 0) they fall every iteration.
    Golden: the reference driver with the oracle propagators."""
    tr = _check_against_golden("c1", "classic", "device", tag="_ct25")
    worst = [max(row) for row in tr.correction_norms]
    assert all(b < a for a, b in zip(worst, worst[1:])), worst
    assert worst[-1] < 5e-3 * worst[0], worst  # classic coarse: 0.2 (0.123 -> 0.024)


def test_exactness_frontier_with_gpu_fine(cuda):
    """Boundaries <= i of iteration i equal the sequential fine solution
    (reference test_parareal.py:217-224): needs a deterministic,
    batch-invariant F; the boundary errors come from pint_boundary_error."""
    from paper_1907_01252_b200.parareal import PararealConfig, run_parareal_device
    from paper_1907_01252_b200.propagator import initial_state
    P, t_end, kf, kc, L, K = CASES["small"]
    F, C = _props(P, kf, kc, L)
    s0 = initial_state(P)
    grid = [t_end * l / L for l in range(L + 1)]
    seq = [s0]
    for t in grid[1:]:
        seq.append(F.advance(seq[-1], t))
    _, tr = run_parareal_device(C, F, s0, t_end, PararealConfig(intervals=L, max_iters=3, tol=1e-30), oracle=seq)
    for i in range(1, tr.iterations_run + 1):
        for l in range(1, i + 1):
            assert tr.boundary_errors[i - 1][l - 1] <= 1e-12, (i, l, tr.boundary_errors[i - 1][l - 1])
    # device boundary errors == the reference's definition on the host iterates
    from oracle.parareal_oracle import boundary_error
    for i in range(1, tr.iterations_run + 1):
        for l in range(1, L + 1):
            ref, _ = boundary_error(tr.iterate_values[i][l], seq[l].values)
            assert abs(tr.boundary_errors[i - 1][l - 1] - ref) <= 1e-12 * max(ref, 1e-300) + 1e-15


@pytest.mark.skipif(pintbench() is None, reason="reference package not available")
def test_device_and_reference_drivers_agree(cuda):
    """The reference driver (host numpy correction, per-slice advance) and the
    device driver (batched fine, pint_coarse_sweep) with the same GPU
    propagators: same states to round-off, same theta / defects."""
    from pintbench.parareal import PararealConfig as RC, run_parareal as rrun
    from paper_1907_01252_b200.parareal import PararealConfig, run_parareal_device
    from paper_1907_01252_b200.propagator import initial_state
    P, t_end, kf, kc, L, K = CASES["small"]
    F, C = _props(P, kf, kc, L)
    s0 = initial_state(P)
    for variant in ("classic", "least_squares", "angle_penalized"):
        a, ta = run_parareal_device(C, F, s0, t_end, PararealConfig(intervals=L, max_iters=2, tol=1e-30,
                                                                    variant=variant))
        b, tb = rrun(C, F, s0, t_end, RC(intervals=L, max_iters=2, tol=1e-30, variant=variant))
        for l in range(L + 1):
            assert np.allclose(a[l].values, b[l].values, rtol=0, atol=1e-12 * max(1.0, np.abs(b[l].values).max()))
        assert np.allclose(ta.theta_values, tb.theta_values, rtol=1e-12, atol=0)
        assert np.allclose(ta.correction_norms, tb.correction_norms, rtol=1e-9, atol=0)


def test_k8_correction_kernel_matches_host(cuda):
    """K8b (pint_parareal_correct_one) vs the restated parareal_update +
    theta_weight + correction norm (oracle/parareal_oracle.py) on random
    states, all three variants, plus the degenerate-block and clamp cases
    (reference test_parareal.py:57-99)."""
    import ctypes
    import torch
    from oracle.parareal_oracle import correction_norm, parareal_update, theta_weight
    from paper_1907_01252_b200 import _lib
    from paper_1907_01252_b200.propagator import _ptr, _stream
    lib = _lib.load()
    C, nn, npad = 5, 300, 320
    rng = np.random.default_rng(0)
    lay = {f"c{i}": (i * nn, nn) for i in range(C)}
    for variant, code in (("classic", 0), ("least_squares", 1), ("angle_penalized", 2)):
        for clamp in ((0.0, 1.0), (0.0, 1.5)):
            vals = [rng.standard_normal(C * nn) for _ in range(4)]
            vals[0][2 * nn:3 * nn] = 0.0  # degenerate coarse block -> weight 1
            cn, fo, co, xp = vals
            th_ref = theta_weight(fo, cn, lay, variant, clamp)
            new_ref = parareal_update(cn, fo, co, th_ref)
            corr_ref = correction_norm(new_ref, xp)
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
            assert np.allclose(out, new_ref, rtol=0, atol=1e-13)
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
