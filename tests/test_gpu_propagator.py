"""GPU parity ladder, step / window level: the batched fine propagator
against the CPU oracle propagator (same Newton control flow, exact Jacobian +
sparse LU) on identical inputs, plus the propagator contract of the reference
(integrators.py:144-166: zero window returns the same object, exact time
bookkeeping, bitwise determinism, batch invariance, TimeStepError)."""

import numpy as np
import pytest

from oracle import fsi_oracle as O
from paper_1907_01252_b200.problem import CONFIGS, channel_3d, small_problem
from paper_1907_01252_b200.state import State

pytestmark = pytest.mark.gpu

NEWTON = dict(abs_tol=1e-10, rel_tol=1e-10)


from fields import field_errors as block_errors  # noqa: E402


def make_pair(P, step, max_slices=3):
    from paper_1907_01252_b200.propagator import NewtonSettings, ThetaSettings, make_propagator
    gpu = make_propagator(P, ThetaSettings(step=step, theta0=1.0, newton=NewtonSettings(**NEWTON)),
                          max_slices=max_slices)
    cpu = O.OracleFSIPropagator(P, step, theta0=1.0, newton=O.OracleNewtonSettings(**NEWTON))
    return gpu, cpu


@pytest.mark.parametrize("P,step,t_end", [
    (small_problem(8, 2), 0.01, 0.2),
    (CONFIGS["c1"].problem, 0.002, 0.1),
    (channel_3d(10, 2, 2, name="small3d"), 0.01, 0.05),
])
def test_window_matches_oracle(cuda, P, step, t_end):
    gpu, cpu = make_pair(P, step)
    s0 = O.initial_state(P)
    a = gpu.advance(s0, t_end)
    b = cpu.advance(s0, t_end)
    assert a.time == t_end and b.time == t_end
    errs = block_errors(P, a.values, b.values)
    assert max(errs.values()) <= 1e-8, errs
    assert gpu.steps_taken == cpu.steps_taken


def test_second_window_from_nonzero_state(cuda):
    P = small_problem(8, 2)
    gpu, cpu = make_pair(P, 0.01)
    s0 = O.initial_state(P)
    mid = cpu.advance(s0, 0.3)
    a = gpu.advance(mid, 0.5)
    b = cpu.advance(mid, 0.5)
    errs = block_errors(P, a.values, b.values)
    assert max(errs.values()) <= 1e-8, errs


def test_zero_window_returns_same_object(cuda):
    P = small_problem(8, 2)
    gpu, _ = make_pair(P, 0.01)
    s0 = O.initial_state(P)
    assert gpu.advance(s0, 0.0) is s0
    with pytest.raises(ValueError):
        gpu.advance(s0.with_values(s0.values, time=1.0), 0.5)


def test_non_divisible_window_rejected(cuda):
    from paper_1907_01252_b200.propagator import NonDivisibleWindow
    P = small_problem(8, 2)
    gpu, _ = make_pair(P, 0.03)
    with pytest.raises(NonDivisibleWindow):
        gpu.advance(O.initial_state(P), 0.1)


def test_bitwise_determinism_and_batch_invariance(cuda):
    P = small_problem(8, 2)
    gpu, cpu = make_pair(P, 0.01, max_slices=4)
    s0 = O.initial_state(P)
    starts = [s0, cpu.advance(s0, 0.1), cpu.advance(s0, 0.2)]
    ends = [s.time + 0.1 for s in starts]
    batch = gpu.advance_batch(starts, ends)
    batch2 = gpu.advance_batch(starts, ends)
    singles = [gpu.advance(s, e) for s, e in zip(starts, ends)]
    rev = gpu.advance_batch(starts[::-1], ends[::-1])[::-1]
    for a, b, c, d in zip(batch, batch2, singles, rev):
        assert a.values.tobytes() == b.values.tobytes()
        assert a.values.tobytes() == c.values.tobytes()
        assert a.values.tobytes() == d.values.tobytes()


def test_failure_raises_time_step_error(cuda):
    from paper_1907_01252_b200.propagator import TimeStepError
    P = small_problem(8, 2)
    gpu, _ = make_pair(P, 0.01)
    bad = np.zeros(P.num_dofs)
    bad[P.num_nodes * 2 + 5] = np.nan  # NaN displacement -> non-finite residual
    with pytest.raises(TimeStepError, match="t_n="):
        gpu.advance(State(np.nan_to_num(bad, nan=0.0) + 0.0, 0.0, P.layout()).with_values(bad), 0.01)


def test_newton_counters(cuda):
    P = small_problem(8, 2)
    gpu, cpu = make_pair(P, 0.01)
    gpu.advance(O.initial_state(P), 0.1)
    cpu.advance(O.initial_state(P), 0.1)
    assert gpu.steps_taken == 10
    assert gpu.newton_iterations >= 10
    assert abs(gpu.newton_iterations - cpu.newton_iterations) <= 3


def _c1_window(krylov=None, env=None):
    """One c1 fine window (25 CN steps from rest) through a fresh context."""
    import os
    from paper_1907_01252_b200.propagator import KrylovSettings, NewtonSettings, ThetaSettings, make_propagator
    P = CONFIGS["c1"].problem
    old = {k: os.environ.get(k) for k in (env or {})}
    os.environ.update(env or {})
    try:
        gpu = make_propagator(P, ThetaSettings(step=0.002, theta0=1.0, newton=NewtonSettings(**NEWTON)),
                              krylov=krylov or KrylovSettings(), max_slices=1)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return gpu, gpu.advance(O.initial_state(P), 0.05)


def test_preconditioner_precision_and_refresh_do_not_move_the_solution(cuda):
    """The mixed-precision pieces (fp32 level-0 V-cycle operator, fp32 Vanka
    solves) and the refresh period live inside the FGMRES preconditioner: the
    converged window must agree with the fp64-operator / rebuild-every-Newton
    variants and with the oracle to the solver tolerance."""
    from paper_1907_01252_b200.propagator import KrylovSettings
    P = CONFIGS["c1"].problem
    g32, a = _c1_window()
    g64, b = _c1_window(env={"PINT_A32": "0"})
    _, c = _c1_window(krylov=KrylovSettings(precond_reuse=0))
    assert g32.device.level0_fp32 and not g64.device.level0_fp32
    ref = O.OracleFSIPropagator(P, 0.002, theta0=1.0, newton=O.OracleNewtonSettings(**NEWTON)).advance(
        O.initial_state(P), 0.05)
    for x in (a, b, c):
        errs = block_errors(P, x.values, ref.values)
        assert max(errs.values()) <= 1e-8, errs
    errs = block_errors(P, a.values, b.values)
    assert max(errs.values()) <= 1e-9, errs


def test_host_beta_bitwise(cuda, monkeypatch):
    """GMRES takes ||b|| = ||-r|| from the Newton loop's own residual norm
    (default) instead of recomputing it on the device (PINT_HOST_BETA=0): the
    same kernel computed both, so the propagation is bitwise unchanged."""
    P = CONFIGS["c1"].problem
    s0 = O.initial_state(P)
    cpu = make_pair(P, 0.002)[1]
    starts = [s0, cpu.advance(s0, 0.02)]
    ends = [s.time + 0.02 for s in starts]
    outs = []
    for v in ("1", "0"):
        monkeypatch.setenv("PINT_HOST_BETA", v)
        gpu, _ = make_pair(P, 0.002)
        outs.append(gpu.advance_batch(starts, ends))
    for a, b in zip(*outs):
        assert a.values.tobytes() == b.values.tobytes()


@pytest.mark.parametrize("env", [{}, {"PINT_TAIL_ROWS": "1000"}])
def test_deferred_basis_scaling_bitwise(cuda, monkeypatch, env):
    """v_{j+1} = w / h formed inside the next Arnoldi step's first Vanka sweep
    (default) or by its own launch (PINT_DEFER_SCALE=0): bitwise the same
    propagation (PINT_TAIL_ROWS=1000 keeps c1's level 0 out of the tail, so
    the deferred path runs)."""
    P = CONFIGS["c1"].problem
    s0 = O.initial_state(P)
    cpu = make_pair(P, 0.002)[1]
    starts = [s0, cpu.advance(s0, 0.02)]
    ends = [s.time + 0.02 for s in starts]
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    outs = []
    for v in ("1", "0"):
        monkeypatch.setenv("PINT_DEFER_SCALE", v)
        gpu, _ = make_pair(P, 0.002)
        outs.append(gpu.advance_batch(starts, ends))
    for a, b in zip(*outs):
        assert a.values.tobytes() == b.values.tobytes()
