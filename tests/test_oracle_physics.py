"""CPU: self-consistency of the oracle physics (no reference implementation
exists for the 2-d/3-d FSI step): exact Jacobian vs central
finite differences, rest state is a discrete equilibrium, Dirichlet and
identity rows, material/ownership tables, inadmissible meshes."""

import numpy as np
import pytest

from oracle import fsi_oracle as O
from paper_1907_01252_b200.problem import CONFIGS, channel_3d, ramp, small_problem

PROBLEMS = [small_problem(8, 2), channel_3d(10, 2, 2, name="small3d")]


def rand_state(P, seed, su=1e-3):
    rng = np.random.default_rng(seed)
    n, d = P.num_nodes, P.dim
    return np.concatenate([0.3 * rng.standard_normal(d * n), su * rng.standard_normal(d * n), rng.standard_normal(n)])


@pytest.mark.parametrize("P", PROBLEMS, ids=["2d", "3d"])
def test_jacobian_matches_central_differences(P):
    y, yo = rand_state(P, 1), rand_state(P, 2)
    w = rand_state(P, 3, su=1.0)
    k, th, t1 = 0.01, 0.51, 0.2
    J = O.jacobian(P, y, yo, k, th, t1)
    Jw = J @ w
    errs = []
    for eps in (1e-4, 1e-5):
        fd = (O.residual(P, y + eps * w, yo, k, th, t1) - O.residual(P, y - eps * w, yo, k, th, t1)) / (2 * eps)
        errs.append(np.linalg.norm(fd - Jw) / np.linalg.norm(Jw))
    assert errs[1] < 1e-7
    assert errs[1] < errs[0] * 0.05  # second-order convergence of the FD check


@pytest.mark.parametrize("P", PROBLEMS, ids=["2d", "3d"])
def test_rest_is_equilibrium_before_inflow(P):
    z = np.zeros(P.num_dofs)
    r = O.residual(P, z, z, 0.01, 0.51, 0.0)  # ramp(0) = 0
    assert np.all(r == 0.0)


def test_dirichlet_and_identity_rows():
    P = small_problem(8, 2)
    m = O.build_mesh(P)
    y = rand_state(P, 4)
    t1 = 0.2
    r = O.residual(P, y, y, 0.01, 0.51, t1).reshape(P.dofs_per_node, P.num_nodes)
    Y = y.reshape(P.dofs_per_node, P.num_nodes)
    g = ramp(t1) * m.inflow_profile
    assert np.array_equal(r[0][m.dir_v], (Y[0] - g)[m.dir_v])
    assert np.array_equal(r[1][m.dir_v], Y[1][m.dir_v])
    assert np.array_equal(r[2][m.dir_u], Y[2][m.dir_u])
    assert np.array_equal(r[4][~m.fluid_touch], Y[4][~m.fluid_touch])
    J = O.jacobian(P, y, y, 0.01, 0.51, t1).tocsr()
    rows = np.flatnonzero(m.dir_u) + 2 * P.num_nodes
    for row in rows[:5]:
        cols = J.indices[J.indptr[row]:J.indptr[row + 1]]
        vals = J.data[J.indptr[row]:J.indptr[row + 1]]
        assert list(cols) == [row] and list(vals) == [1.0]


def test_material_tables_c1():
    P = CONFIGS["c1"].problem
    m = O.build_mesh(P)
    assert m.solid.sum() == 12            # bar 0.2 x 0.25 on a 1/16 grid: 3 x 4 cells
    assert m.outflow.sum() == 8           # fluid cells at x = 2
    assert m.dir_v.sum() == 2 * 33 + 7    # walls + inflow interior
    # inflow profile: parabolic, peak 1 at mid-height, zero at walls
    prof = m.inflow_profile.reshape(9, 33)[:, 0]
    assert prof[0] == 0.0 and prof[-1] == 0.0 and abs(prof[4] - 1.0) < 1e-15


def test_collapsed_mesh_gives_infinite_residual():
    P = small_problem(8, 2)
    y = np.zeros(P.num_dofs)
    n = P.num_nodes
    y[2 * n:3 * n] = -10.0 * np.arange(n) / n  # fold the x-displacement
    r = O.residual(P, y, np.zeros(P.num_dofs), 0.01, 0.51, 0.1)
    assert np.all(np.isinf(r))


def test_theta_step_converges_and_time_bookkeeping():
    P = small_problem(8, 2)
    prop = O.OracleFSIPropagator(P, 0.01, 1.0, O.OracleNewtonSettings(1e-10, 1e-10))
    s = prop.advance(O.initial_state(P), 0.05)
    assert s.time == 0.05 and prop.steps_taken == 5 and prop.newton_iterations >= 5
    assert np.linalg.norm(s.values) > 0
    z = O.initial_state(P)
    assert prop.advance(z, 0.0) is z


def test_pressure_stabilization_is_step_independent():
    P = CONFIGS["c2"].problem
    assert P.delta_p(2.0 ** -6) == P.delta_p(2.0 ** -10) > 0
