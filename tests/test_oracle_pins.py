"""CPU: pin the oracle against the reference (pintbench) where the reference
has an implementation: Newton control flow (linalg.py:167-248), window split
(integrators.py:115-123), and the Parareal driver (parareal.py:363-465,
tests/oracles.py:textbook_parareal).  The FSI physics itself is unpinned by
the reference; its self-consistency checks live in
tests/test_oracle_physics.py."""

import numpy as np
import pytest

from oracle import fsi_oracle as O
from paper_1907_01252_b200.problem import CONFIGS, small_problem
from refimport import pintbench

pb = pintbench()
needs_ref = pytest.mark.skipif(pb is None, reason="reference package not available")


@needs_ref
@pytest.mark.parametrize("k,t1", [(0.01, 0.01), (0.02, 0.3)])
def test_newton_matches_reference_newton_solve(k, t1):
    """Same residual + exact Jacobian through the reference's own newton_solve
    (dense LU) and through the oracle's sparse mirror: identical iteration
    counts and histories, solutions equal to round-off."""
    from pintbench.linalg import NewtonSettings, newton_solve
    P = small_problem(8, 2)
    rng = np.random.default_rng(0)
    yo = 1e-2 * rng.standard_normal(P.num_dofs)
    theta = 0.5 + k
    res = lambda y: O.residual(P, y, yo, k, theta, t1)  # noqa: E731
    jac = lambda y: O.jacobian(P, y, yo, k, theta, t1)  # noqa: E731
    h_ref, h_or = [], []
    x_ref, it_ref = newton_solve(res, yo, NewtonSettings(abs_tol=1e-10, rel_tol=1e-10),
                                 jacobian=lambda y: jac(y).toarray(), history=h_ref)
    x_or, it_or = O.newton_solve(res, jac, yo, O.OracleNewtonSettings(abs_tol=1e-10, rel_tol=1e-10), h_or)
    assert it_ref == it_or
    assert np.allclose(h_ref, h_or, rtol=1e-6, atol=1e-13)
    assert np.linalg.norm(x_ref - x_or) <= 1e-12 * np.linalg.norm(x_ref)


@needs_ref
def test_newton_zero_iterations_when_converged():
    from pintbench.linalg import NewtonSettings, newton_solve
    f = lambda x: x - 1.0  # noqa: E731
    x, it = newton_solve(f, np.ones(3), NewtonSettings())
    xo, ito = O.newton_solve(f, lambda x: __import__("scipy.sparse", fromlist=["eye"]).eye(3).tocsr(),
                             np.ones(3), O.OracleNewtonSettings())
    assert it == ito == 0


@needs_ref
@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_window_split_matches_reference(name):
    from pintbench.integrators import NonDivisibleWindow, _split_window
    cfg = CONFIGS[name]
    for step in (cfg.fine_step, cfg.coarse_step):
        assert O.split_window(cfg.window, step) == _split_window(cfg.window, step)
    # the BASELINE-as-written steps of c2..c4 are rejected by the reference
    if name != "c1":
        with pytest.raises(NonDivisibleWindow):
            _split_window(cfg.window, 0.02)


@needs_ref
def test_oracle_propagator_bookkeeping_matches_theta_propagator():
    """advance() time bookkeeping: k_last = t_end - t_{n-1}, theta_last = 1/2 + theta0 k_last."""
    from pintbench.integrators import ThetaSettings, make_propagator
    from pintbench.problems import dahlquist, initial_state
    ref = make_propagator(dahlquist(), ThetaSettings(step=0.002, theta0=1.0))
    s = ref.advance(initial_state(dahlquist()), 0.1)
    P = small_problem(8, 2)
    prop = O.OracleFSIPropagator(P, 0.002, 1.0)
    assert O.split_window(0.1, 0.002) == 50 == ref.steps_taken
    assert s.time == 0.1


@needs_ref
def test_reference_driver_with_oracle_equals_textbook_parareal():
    """The reference run_parareal driving the oracle FSI propagators equals the
    reference test oracle textbook_parareal (tests/oracles.py:25-58)."""
    import importlib.util
    import os
    from refimport import reference_tests_dir
    from pintbench.parareal import PararealConfig, run_parareal
    tdir = reference_tests_dir()
    if tdir is None:
        pytest.skip("reference tests not available")
    spec = importlib.util.spec_from_file_location("ref_oracles", os.path.join(tdir, "oracles.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    P = small_problem(8, 2)
    nw = O.OracleNewtonSettings(1e-10, 1e-10)
    F = O.OracleFSIPropagator(P, 0.05, 1.0, nw)
    C = O.OracleFSIPropagator(P, 0.1, 1.0, nw)
    s0 = O.initial_state(P)
    L, T = 4, 0.4
    grid = [T * l / L for l in range(L + 1)]
    _, trace = run_parareal(C, F, s0, T, PararealConfig(intervals=L, max_iters=2, tol=1e-30))
    text = mod.textbook_parareal(C, F, s0, grid, 2)
    for i in range(3):
        for l in range(L + 1):
            assert np.array_equal(trace.iterate_values[i][l], text[i][l])
