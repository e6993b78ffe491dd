"""CPU: the host logic of the device-resident Parareal driver
(paper_1907_01252_b200.parareal.run_parareal_device) against the REFERENCE
driver (pintbench.run_parareal, parareal.py:363-465).

The device driver is run here with CPU stand-ins for the GPU propagator
protocol (tests/linprop.py: torch CPU tensors, the oracle's correction
arithmetic), so its iteration structure, slice indexing, stop rule, trace and
failure annotation are checked against the committed golden traces of the
reference driver on the same linear propagator (tests/golden/driver_linear.npz,
bitwise) and against the live reference when it is importable.  The K8 / sweep
kernels themselves are checked on the GPU (tests/test_gpu_parareal.py).
"""

import os

import numpy as np
import pytest

import linprop
from paper_1907_01252_b200.parareal import PararealConfig, PararealError, run_parareal_device, time_grid
from paper_1907_01252_b200.report import model_speedup
from refimport import pintbench

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "driver_linear.npz"))
VARIANTS = ("classic", "least_squares", "angle_penalized")


def _props(**kw):
    dev = linprop.CPUDevice()
    F = linprop.DeviceLinearPropagator(0.01, theta0=1.0, device=dev, **kw.get("F", {}))
    C = linprop.DeviceLinearPropagator(0.1, theta0=1.0, device=dev, **kw.get("C", {}))
    return C, F


@pytest.mark.parametrize("variant", VARIANTS)
def test_device_driver_matches_reference_golden_bitwise(variant):
    C, F = _props()
    cfg = PararealConfig(intervals=6, max_iters=4, tol=1e-30, variant=variant)
    states, tr = run_parareal_device(C, F, linprop.s0(), 1.2, cfg)
    assert tr.iterations_run == int(GOLD[f"{variant}_iters"])
    assert tr.fine_propagations == int(GOLD[f"{variant}_fine"])
    assert np.array_equal(np.array(tr.iterate_values), GOLD[f"{variant}_iterates"])
    assert np.array_equal(np.array(tr.correction_norms), GOLD[f"{variant}_corr"])
    assert np.array_equal(np.array(tr.theta_values), GOLD[f"{variant}_theta"])
    assert states[-1].time == 1.2 and np.array_equal(states[-1].values, GOLD[f"{variant}_iterates"][-1][-1])


def test_tolerance_stop_matches_reference_golden():
    C, F = _props()
    _, tr = run_parareal_device(C, F, linprop.s0(), 1.2, PararealConfig(intervals=6, max_iters=6, tol=1e-6))
    assert tr.iterations_run == int(GOLD["tol_iters"]) and tr.converged == bool(GOLD["tol_converged"])
    assert np.array_equal(np.array(tr.correction_norms), GOLD["tol_corr"])


@pytest.mark.skipif(pintbench() is None, reason="reference package not available")
def test_device_driver_matches_live_reference():
    from pintbench.parareal import PararealConfig as RC, run_parareal as rrun
    for variant in VARIANTS:
        for tol in (1e-30, 1e-5):
            Fr = linprop.LinearPropagator(0.02, theta0=0.5)
            Cr = linprop.LinearPropagator(0.2, theta0=0.5)
            _, a = rrun(Cr, Fr, linprop.s0(), 1.6, RC(intervals=8, max_iters=5, tol=tol, variant=variant,
                                                      theta_clamp=(0.0, 1.5)))
            dev = linprop.CPUDevice()
            F = linprop.DeviceLinearPropagator(0.02, theta0=0.5, device=dev)
            C = linprop.DeviceLinearPropagator(0.2, theta0=0.5, device=dev)
            _, b = run_parareal_device(C, F, linprop.s0(), 1.6,
                                       PararealConfig(intervals=8, max_iters=5, tol=tol, variant=variant,
                                                      theta_clamp=(0.0, 1.5)))
            assert a.iterations_run == b.iterations_run and a.converged == b.converged
            assert np.array_equal(np.array(a.iterate_values), np.array(b.iterate_values))
            assert a.correction_norms == b.correction_norms and a.theta_values == b.theta_values
            assert a.fine_propagations == b.fine_propagations


def test_exactness_frontier_and_bookkeeping():
    """Boundaries <= i of iteration i equal the sequential fine solution
    (reference test_parareal.py:217-224); boundary errors from the device
    reduction; trace timings are monotone."""
    C, F = _props()
    s0 = linprop.s0()
    grid = time_grid(0.0, 1.2, 6)
    seq = [s0]
    for t in grid[1:]:
        seq.append(F.advance(seq[-1], t))
    _, tr = run_parareal_device(C, F, s0, 1.2, PararealConfig(intervals=6, max_iters=4, tol=1e-30), oracle=seq)
    assert tr.fine_propagations == 6 * 4 and len(tr.boundary_errors) == 4
    for i in range(1, 5):
        for l in range(1, i + 1):
            assert tr.boundary_errors[i - 1][l - 1] <= 1e-12
    assert len(tr.iteration_seconds) == 4 and tr.total_seconds >= tr.iteration_seconds[-1] > 0.0
    assert tr.sweep_seconds > 0.0 and tr.fine_seconds > 0.0


def test_failures_are_annotated():
    # fine failure: the whole batched fine phase of the iteration
    C, F = _props(F={"fail_at": 0.4})
    with pytest.raises(PararealError, match="fine failed at iteration 1"):
        run_parareal_device(C, F, linprop.s0(), 1.2, PararealConfig(intervals=6, max_iters=2))
    # coarse failure inside the initialisation sweep names the interval
    C, F = _props(C={"fail_at": 0.6})
    with pytest.raises(PararealError, match="coarse_init failed at iteration 0, interval 3"):
        run_parareal_device(C, F, linprop.s0(), 1.2, PararealConfig(intervals=6, max_iters=2))


def test_config_validation_and_speedup_model():
    with pytest.raises(ValueError):
        PararealConfig(intervals=1, max_iters=1)
    with pytest.raises(ValueError):
        PararealConfig(intervals=4, max_iters=5)
    with pytest.raises(ValueError):
        PararealConfig(intervals=4, max_iters=2, variant="magic")
    with pytest.raises(ValueError):
        PararealConfig(intervals=4, max_iters=2, theta_clamp=(1.0, 0.0))
    # PAPER.md:586-589 / reference theoretical_speedup: r = 0.02, K = 3, N = 20
    assert model_speedup(0.02, 3, 20) == pytest.approx(5.7803, rel=1e-4)
    C, F = _props()
    with pytest.raises(ValueError):
        run_parareal_device(C, F, linprop.s0(), 1.25, PararealConfig(intervals=6, max_iters=2))
