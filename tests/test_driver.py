"""CPU: the package's Parareal driver against the reference driver
(parareal.py:363-465) -- committed golden traces of the reference on a linear
test propagator (tests/golden/driver_linear.npz, bitwise), live comparison
when the reference is importable, the unit contracts of parareal_update /
theta_weight (reference tests/test_parareal.py:30-99), scheduler equivalence
(test_scheduler.py:101-119), trace bookkeeping and failure annotation."""

import os

import numpy as np
import pytest

import linprop
from paper_1907_01252_b200.parareal import (PararealConfig, PararealError, SpeedupModel, boundary_error,
                                             parareal_update, pipelined_schedule, run_parareal,
                                             sequential_solve, theoretical_speedup, theta_weight)
from paper_1907_01252_b200.state import State
from refimport import pintbench

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "driver_linear.npz"))
VARIANTS = ("classic", "least_squares", "angle_penalized")


def vs(vals, t=0.0, layout=None):
    return State(np.asarray(vals, float), t, layout or {"v": (0, len(vals))})


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("scheduler", ["serial", "pipelined", "batched"])
def test_driver_matches_reference_golden_bitwise(variant, scheduler):
    F = linprop.LinearPropagator(0.01, theta0=1.0)
    C = linprop.LinearPropagator(0.1, theta0=1.0)
    cfg = PararealConfig(intervals=6, max_iters=4, tol=1e-30, variant=variant, scheduler=scheduler, workers=3)
    states, tr = run_parareal(C, F, linprop.s0(), 1.2, cfg)
    assert tr.iterations_run == int(GOLD[f"{variant}_iters"])
    assert tr.fine_propagations == int(GOLD[f"{variant}_fine"])
    assert np.array_equal(np.array(tr.iterate_values), GOLD[f"{variant}_iterates"])
    assert np.array_equal(np.array(tr.correction_norms), GOLD[f"{variant}_corr"])
    assert np.array_equal(np.array(tr.theta_values), GOLD[f"{variant}_theta"])
    assert states[-1].time == 1.2


def test_tolerance_stop_matches_reference_golden():
    F = linprop.LinearPropagator(0.01, theta0=1.0)
    C = linprop.LinearPropagator(0.1, theta0=1.0)
    _, tr = run_parareal(C, F, linprop.s0(), 1.2, PararealConfig(intervals=6, max_iters=6, tol=1e-6))
    assert tr.iterations_run == int(GOLD["tol_iters"]) and tr.converged == bool(GOLD["tol_converged"])
    assert np.array_equal(np.array(tr.correction_norms), GOLD["tol_corr"])


@pytest.mark.skipif(pintbench() is None, reason="reference package not available")
def test_driver_matches_live_reference():
    from pintbench.parareal import PararealConfig as RC, run_parareal as rrun
    for variant in VARIANTS:
        F = linprop.LinearPropagator(0.02, theta0=0.5)
        C = linprop.LinearPropagator(0.2, theta0=0.5)
        _, a = rrun(C, F, linprop.s0(), 1.6, RC(intervals=8, max_iters=5, tol=1e-30, variant=variant))
        _, b = run_parareal(C, F, linprop.s0(), 1.6, PararealConfig(intervals=8, max_iters=5, tol=1e-30,
                                                                    variant=variant))
        assert np.array_equal(np.array(a.iterate_values), np.array(b.iterate_values))
        assert a.correction_norms == b.correction_norms and a.theta_values == b.theta_values


# ---- unit contracts (reference tests/test_parareal.py:30-99)
def test_update_units():
    c, f = vs([1.0, 2.0]), vs([3.0, 4.0])
    assert np.array_equal(parareal_update(c, f, c, 1.0).values, f.values)
    assert np.array_equal(parareal_update(vs([9.0, 9.0]), vs([1.0, 2.0]), vs([-4.0, 0.0]), 0.0).values, [1.0, 2.0])
    with pytest.raises(ValueError):
        parareal_update(vs([1.0, 1.0], t=1.0), vs([1.0, 1.0]), vs([1.0, 1.0]), 1.0)
    with pytest.raises(ValueError):
        parareal_update(vs([1.0, 1.0]), vs([1.0, 1.0], layout={"w": (0, 2)}), vs([1.0, 1.0]), 1.0)


def test_theta_weight_units():
    f, c = vs([1.0, 0.0]), vs([0.0, 1.0])
    assert theta_weight(f, c, "least_squares") == 0.0 and theta_weight(f, c, "angle_penalized") == 0.0
    lay = {"y": (0, 1)}
    f1, c1 = State(np.array([2.0]), 0.0, lay), State(np.array([1.0]), 0.0, lay)
    assert theta_weight(f1, c1, "angle_penalized") == pytest.approx(0.5)
    assert theta_weight(f1, c1, "least_squares") == 1.0
    assert theta_weight(f1, c1, "least_squares", clamp=(0.0, 1.5)) == pytest.approx(1.5)
    assert theta_weight(f1, State(np.array([0.0]), 0.0, lay), "least_squares") == 1.0
    lay2 = {"a": (0, 1), "b": (1, 1)}
    assert theta_weight(State(np.array([2.0, 1.0]), 0.0, lay2), State(np.array([4.0, 1.0]), 0.0, lay2),
                        "least_squares") == pytest.approx(0.75)
    assert theta_weight(f, c, "classic") == 1.0
    with pytest.raises(ValueError):
        theta_weight(f, f, "magic")


def test_config_validation_and_speedup():
    with pytest.raises(ValueError):
        PararealConfig(intervals=1, max_iters=1)
    with pytest.raises(ValueError):
        PararealConfig(intervals=4, max_iters=5)
    with pytest.raises(ValueError):
        PararealConfig(intervals=4, max_iters=2, scheduler="magic")
    assert theoretical_speedup(SpeedupModel(r=0.02, iters=3, intervals=20)) == pytest.approx(5.7803, rel=1e-4)


def test_task_graph_shape():
    tasks = pipelined_schedule(3, 2)
    assert len(tasks) == 3 + 2 * 6
    fine = [t for t in tasks if t.kind == "fine" and t.iteration == 2]
    assert fine[1].depends == ((1, 1, 0),)


def test_exactness_frontier_and_bookkeeping():
    F = linprop.LinearPropagator(0.01, theta0=1.0)
    C = linprop.LinearPropagator(0.1, theta0=1.0)
    s0 = linprop.s0()
    grid = [1.2 * l / 6 for l in range(7)]
    seq = sequential_solve(F, s0, grid)
    _, tr = run_parareal(C, F, s0, 1.2, PararealConfig(intervals=6, max_iters=4, tol=1e-30), oracle=seq)
    assert tr.fine_propagations == 6 * 4
    for i in range(1, 5):
        for l in range(1, i + 1):
            assert tr.boundary_errors[i - 1][l - 1] <= 1e-12
    assert len(tr.iteration_seconds) == 4 and tr.total_seconds >= tr.iteration_seconds[-1]


def test_failure_is_annotated():
    class Exploding(linprop.LinearPropagator):
        def advance(self, state, t_end):
            raise ArithmeticError("boom")

    C = linprop.LinearPropagator(0.1)
    with pytest.raises(PararealError, match="fine failed at iteration 1"):
        run_parareal(C, Exploding(0.01), linprop.s0(), 1.2, PararealConfig(intervals=6, max_iters=2))
    with pytest.raises(PararealError, match="fine failed at iteration 1"):
        run_parareal(C, Exploding(0.01), linprop.s0(), 1.2,
                     PararealConfig(intervals=6, max_iters=2, scheduler="batched"))


def test_boundary_error_absolute_flag():
    e = boundary_error([vs([1.0, 0.0])], [vs([0.0, 0.0])])
    assert e[0].absolute and e[0].value == 1.0
