"""CPU ORACLE (test infrastructure only) -- numpy/scipy restatement of the
shifted Crank-Nicolson monolithic ALE-FSI step.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
/ reference legs may import this module; the product path
(``paper_1907_01252_b200``) never does.

What it restates
----------------
* the fully discrete CN step and its semiforms A_div,
  A_NS (with the do-nothing outflow correction), A_ES, the mass/ALE terms with
  J_{n-1/2}, F_{n-1/2}, grad v_{n-1/2} (the PAPER.md:416 typo read as v_{n-1});
* PAPER.md:157-163 / 231-236 -- Newtonian fluid in ALE form and the St.
  Venant-Kirchhoff solid; PAPER.md:188-196 -- harmonic mesh extension;
* equal-order pressure stabilization (Brezzi-Pitkaranta,
  see paper_1907_01252_b200/problem.py for the shared decisions);
* reference linalg.py:167-248 -- ``newton_solve`` control flow (target,
  halving line search down to ``damping_min``, accept-anyway, iteration
  count), with the FD Jacobian (linalg.py:152-164) replaced by an exact
  element Jacobian (complex-step differentiation of the element residual,
  exact to round-off) and the dense LU (linalg.py:224) by ``splu``;
* reference integrators.py:70-96 / 126-166 -- ``_theta_step`` time
  bookkeeping (t1 = t0 + k, theta = 1/2 + theta0 k clamped to [1/2, 1],
  Newton guess = previous state) and ``ThetaPropagator.advance`` (window
  split, last step absorbs the rounding slack, zero window returns the same
  object).

Parity status: the driver-level pieces are pinned against the reference
(tests/test_oracle_pins.py, tests/golden/); the FSI physics itself has no
reference implementation, golden vector or known-answer test
 -> **parity unpinned at the physics level**; it is checked
by self-consistency tests (Jacobian vs finite differences, discrete
invariants) instead.
"""

from __future__ import annotations

import math
import threading
from dataclasses import dataclass
from functools import lru_cache

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import os
import sys

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
if _ROOT not in sys.path:
    sys.path.insert(0, _ROOT)

from paper_1907_01252_b200.problem import FSIProblem, ramp  # noqa: E402  (pure data)
from paper_1907_01252_b200.state import State  # noqa: E402


class OracleNumericBreakdown(ArithmeticError):
    pass


class OracleMaxIters(RuntimeError):
    pass


class OracleTimeStepError(RuntimeError):
    pass


# --------------------------------------------------------------------------
# mesh tables


@dataclass
class Mesh:
    problem: FSIProblem
    conn: np.ndarray          # (E, A) global node of local corner a
    solid: np.ndarray         # (E,) bool
    outflow: np.ndarray       # (E,) bool: fluid cell with a face on x = Lx
    solid_touch: np.ndarray   # (Nn,) bool
    fluid_touch: np.ndarray   # (Nn,) bool
    dir_v: np.ndarray         # (Nn,) bool
    dir_u: np.ndarray         # (Nn,) bool
    inflow_profile: np.ndarray  # (Nn,) x-velocity profile at s(t) = 1 (0 off inflow)
    Nq: np.ndarray            # (Q, A) volume shape values
    dNq: np.ndarray           # (Q, A, d) physical gradients
    wq: float                 # volume quadrature weight per point
    Nf: np.ndarray            # (Qf, A) face shape values (face x-hat = 1)
    dNf: np.ndarray           # (Qf, A, d)
    wf: float


def _gauss01():
    g = 0.5 / math.sqrt(3.0)
    return (0.5 - g, 0.5 + g)


def _shape(xi, d):
    """Q1 shape values (A,) and reference gradients (A, d) at xi in [0,1]^d."""
    A = 1 << d
    N = np.ones(A)
    dN = np.ones((A, d))
    for a in range(A):
        for k in range(d):
            bit = (a >> k) & 1
            val = xi[k] if bit else 1.0 - xi[k]
            der = 1.0 if bit else -1.0
            N[a] *= val
            for m in range(d):
                dN[a, m] *= der if m == k else val
    return N, dN


@lru_cache(maxsize=32)
def build_mesh(problem: FSIProblem) -> Mesh:
    d = problem.dim
    cells = problem.cells
    nodes = problem.nodes
    h = problem.h
    A = 1 << d
    # cell multi-index, x fastest
    cidx = np.indices(cells[::-1]).reshape(d, -1)[::-1]  # (d, E) with [0]=i (x)
    E = cidx.shape[1]
    strides = [1]
    for m in range(1, d):
        strides.append(strides[-1] * nodes[m - 1])
    conn = np.zeros((E, A), dtype=np.int64)
    for a in range(A):
        idx = np.zeros(E, dtype=np.int64)
        for m in range(d):
            idx += (cidx[m] + ((a >> m) & 1)) * strides[m]
        conn[:, a] = idx
    centre = [(cidx[m] + 0.5) * h[m] for m in range(d)]
    solid = np.ones(E, dtype=bool)
    for m in range(d):
        solid &= (centre[m] >= problem.bar_lo[m]) & (centre[m] <= problem.bar_hi[m])
    outflow = (~solid) & (cidx[0] == cells[0] - 1)

    Nn = problem.num_nodes
    solid_touch = np.zeros(Nn, dtype=bool)
    fluid_touch = np.zeros(Nn, dtype=bool)
    for a in range(A):
        solid_touch[conn[solid, a]] = True
        fluid_touch[conn[~solid, a]] = True

    nidx = np.indices(nodes[::-1]).reshape(d, -1)[::-1]  # (d, Nn)
    on_lo = [nidx[m] == 0 for m in range(d)]
    on_hi = [nidx[m] == cells[m] for m in range(d)]
    wall = np.zeros(Nn, dtype=bool)
    for m in range(1, d):
        wall |= on_lo[m] | on_hi[m]
    dir_v = on_lo[0] | wall
    dir_u = on_lo[0] | on_hi[0] | wall
    # inflow profile (x = 0): 4 y (H - y) / H^2 in 2-d; 16 y(H-y) z(H-z)/H^4 in 3-d
    prof = np.full(Nn, problem.u_peak)
    for m in range(1, d):
        y = nidx[m] * h[m]
        H = problem.extent[m]
        prof = prof * 4.0 * y * (H - y) / (H * H)
    inflow_profile = np.where(on_lo[0] & ~wall, prof, 0.0)

    g = _gauss01()
    pts = np.array(np.meshgrid(*([g] * d), indexing="ij")).reshape(d, -1).T  # (Q, d)
    # order points with x fastest for readability (any fixed order works)
    pts = pts[:, ::-1] if d > 1 else pts
    Q = pts.shape[0]
    Nq = np.zeros((Q, A))
    dNq = np.zeros((Q, A, d))
    inv_h = np.array([1.0 / x for x in h])
    for q in range(Q):
        N, dN = _shape(pts[q], d)
        Nq[q] = N
        dNq[q] = dN * inv_h
    wq = float(np.prod([0.5 * x for x in h]))
    fpts = np.array(np.meshgrid(*([g] * (d - 1)), indexing="ij")).reshape(d - 1, -1).T
    Qf = fpts.shape[0]
    Nf = np.zeros((Qf, A))
    dNf = np.zeros((Qf, A, d))
    for q in range(Qf):
        xi = np.concatenate([[1.0], fpts[q][::-1]])
        N, dN = _shape(xi, d)
        Nf[q] = N
        dNf[q] = dN * inv_h
    wf = float(np.prod([0.5 * x for x in h[1:]]))
    return Mesh(problem, conn, solid, outflow, solid_touch, fluid_touch, dir_v, dir_u,
                inflow_profile, Nq, dNq, wq, Nf, dNf, wf)


# --------------------------------------------------------------------------
# small dense helpers (analytic so complex-step differentiation is exact)


def _det_inv(F):
    d = F.shape[-1]
    if d == 2:
        a, b, c, e = F[..., 0, 0], F[..., 0, 1], F[..., 1, 0], F[..., 1, 1]
        det = a * e - b * c
        inv = np.empty_like(F)
        inv[..., 0, 0] = e / det
        inv[..., 0, 1] = -b / det
        inv[..., 1, 0] = -c / det
        inv[..., 1, 1] = a / det
        return det, inv
    cof = np.empty_like(F)
    for i in range(3):
        for j in range(3):
            i1, i2 = (i + 1) % 3, (i + 2) % 3
            j1, j2 = (j + 1) % 3, (j + 2) % 3
            cof[..., i, j] = F[..., i1, j1] * F[..., i2, j2] - F[..., i1, j2] * F[..., i2, j1]
    det = F[..., 0, 0] * cof[..., 0, 0] + F[..., 0, 1] * cof[..., 0, 1] + F[..., 0, 2] * cof[..., 0, 2]
    inv = np.swapaxes(cof, -1, -2) / det[..., None, None]
    return det, inv


def _T(M):
    return np.swapaxes(M, -1, -2)


def _testN(vec, N):
    """sum_q vec[e,q,i] N[q,a] -> (E, A, i)."""
    return np.matmul(N.T, vec)


def _testG(ten, dN):
    """sum_q sum_j ten[e,q,i,j] dN[q,a,j] -> (E, A, i)."""
    E, Q, I, D = ten.shape
    t = ten.transpose(0, 1, 3, 2).reshape(E, Q * D, I)
    g = dN.transpose(1, 0, 2).reshape(dN.shape[1], Q * D)
    return np.matmul(g, t)


# --------------------------------------------------------------------------
# element residual


def element_residual(mesh: Mesh, Yn, Yo, k: float, theta: float):
    """Element contributions (E, A, C) before row ownership / Dirichlet rows.

    ``Yn`` (E, A, C) may be complex (complex-step Jacobian); ``Yo`` is real.
    Also returns the minimum of Re(J_n) over quadrature points per element
    (mesh admissibility, reference integrators.py:83-90 analogue).
    """
    P = mesh.problem
    d = P.dim
    I = np.eye(d)
    kt = k * theta
    ko = k * (1.0 - theta)
    rho_f, rho_s = P.rho_f, P.rho_s
    rnu = P.rho_f * P.nu_f
    mu, lam = P.mu_s, P.lambda_s
    delta = P.delta_p(k)
    solid = mesh.solid

    def fields(Y, N, dN):
        # values: (Q, A) @ (E, A, C) -> (E, Q, C); gradients via (Q*d, A)
        Q = N.shape[0]
        val = np.matmul(N, Y)
        grd = np.matmul(dN.transpose(0, 2, 1).reshape(Q * d, -1), Y).reshape(Y.shape[0], Q, d, -1)
        grd = grd.transpose(0, 1, 3, 2)  # (E, Q, C, d): grd[..., c, j] = d y_c / d x_j
        v, u, p = val[..., 0:d], val[..., d:2 * d], val[..., 2 * d]
        Gv, Gu, gp = grd[..., 0:d, :], grd[..., d:2 * d, :], grd[..., 2 * d, :]
        return v, u, Gv, Gu, p, gp

    Nq, dNq, W = mesh.Nq, mesh.dNq, mesh.wq
    vn, un, Gvn, Gun, pn, gpn = fields(Yn, Nq, dNq)
    vo, uo, Gvo, Guo, _, _ = fields(Yo, Nq, dNq)
    Fn = I + Gun
    Fo = I + Guo
    Jn, Fin = _det_inv(Fn)
    Jo, Fio = _det_inv(Fo)
    Fm = 0.5 * (Fn + Fo)
    Jm = 0.5 * (Jn + Jo)
    _, Fim = _det_inv(Fm)
    Gvm = 0.5 * (Gvn + Gvo)

    # ---- fluid momentum integrand: vector part (tested by N_a) and tensor part (by grad N_a)
    du = un - uo
    GvFim = np.matmul(Gvm, Fim)
    mass_f = rho_f * Jm[..., None] * ((vn - vo) - np.matmul(GvFim, du[..., None])[..., 0])
    GvFin = np.matmul(Gvn, Fin)
    GvFio = np.matmul(Gvo, Fio)
    conv_n = rho_f * Jn[..., None] * np.matmul(GvFin, vn[..., None])[..., 0]
    conv_o = rho_f * Jo[..., None] * np.matmul(GvFio, vo[..., None])[..., 0]

    def piola(J, GvFi, Fi, p):
        sigma = rnu * (GvFi + _T(GvFi)) - p[..., None, None] * I
        return J[..., None, None] * np.matmul(sigma, _T(Fi))  # sigma F^{-T}

    Pn = piola(Jn, GvFin, Fin, pn)
    Po = piola(Jo, GvFio, Fio, pn)  # pressure fully implicit (p^n in both parts)
    vec_f = mass_f + kt * conv_n + ko * conv_o
    ten_f = kt * Pn + ko * Po

    # ---- solid momentum (St. Venant-Kirchhoff, first Piola F Sigma)
    def svk(F):
        E = 0.5 * (np.matmul(_T(F), F) - I)
        trE = np.trace(E, axis1=-2, axis2=-1)
        S = 2.0 * mu * E + lam * trE[..., None, None] * I
        return np.matmul(F, S)

    vec_s = rho_s * (vn - vo)
    ten_s = kt * svk(Fn) + ko * svk(Fo)

    sm = solid[:, None, None]
    vec = np.where(sm, vec_s, vec_f)
    ten = np.where(solid[:, None, None, None], ten_s, ten_f)
    Rv = W * (_testN(vec, Nq) + _testG(ten, dNq))

    # ---- u rows: solid kinematic (tested by N_a) / fluid harmonic extension
    kin = (un - uo) - kt * vn - ko * vo
    Ru_s = W * _testN(kin, Nq)
    ext = kt * Gun + ko * Guo
    Ru_f = W * _testG(ext, dNq)
    Ru = np.where(sm, Ru_s, Ru_f)

    # ---- p rows: k A_div + k delta (grad p, grad xi) on fluid cells
    div = Jn * np.trace(GvFin, axis1=-2, axis2=-1)
    Rp = W * k * (_testN(div[..., None], Nq)[..., 0] + delta * _testG(gpn[..., None, :], dNq)[..., 0])
    Rp = np.where(solid[:, None], 0.0, Rp)

    # ---- outflow boundary correction  -< rho nu J F^{-T} grad v^T F^{-T} n, phi >
    if np.any(mesh.outflow):
        oe = mesh.outflow
        Nf, dNf = mesh.Nf, mesh.dNf
        Ynf, Yof = Yn[oe], Yo[oe]
        _, _, Gvnf, Gunf, _, _ = fields(Ynf, Nf, dNf)
        _, _, Gvof, Guof, _, _ = fields(Yof, Nf, dNf)
        Jnf, Finf = _det_inv(I + Gunf)
        Jof, Fiof = _det_inv(I + Guof)

        def bterm(J, Gv, Fi):
            # F^{-T} grad v^T F^{-T} e_x  ->  (F^{-T} Gv^T F^{-T})[:, 0]
            M = np.matmul(np.matmul(_T(Fi), _T(Gv)), _T(Fi))  # F^{-T} Gv^T F^{-T}
            return rnu * J[..., None] * M[..., 0]

        Bf = kt * bterm(Jnf, Gvnf, Finf) + ko * bterm(Jof, Gvof, Fiof)
        Rv_out = -mesh.wf * _testN(Bf, Nf)
        Rv = Rv.copy()
        Rv[oe] = Rv[oe] + Rv_out

    R = np.concatenate([Rv, Ru, Rp[..., None]], axis=-1)
    return R, np.min(Jn.real, axis=1)


def _row_mask(mesh: Mesh):
    """(E, A, C) multiplier implementing the row ownership rules."""
    P = mesh.problem
    d = P.dim
    C = P.dofs_per_node
    A = mesh.conn.shape[1]
    E = mesh.conn.shape[0]
    m = np.ones((E, A, C))
    st = mesh.solid_touch[mesh.conn]  # (E, A)
    fluid_cell = ~mesh.solid[:, None]
    # extension rows of fluid cells only on nodes that touch no solid cell
    m[:, :, d:2 * d] = np.where((fluid_cell & st)[..., None], 0.0, 1.0)
    return m


def _gather(mesh: Mesh, y):
    P = mesh.problem
    Nn = P.num_nodes
    C = P.dofs_per_node
    Y = y.reshape(C, Nn).T  # (Nn, C)
    return Y[mesh.conn]      # (E, A, C)


def _dirichlet(mesh: Mesh, t1: float):
    """(fixed-row mask (N,), values g (N,)) with identity rows r = y - g."""
    P = mesh.problem
    d = P.dim
    Nn = P.num_nodes
    C = P.dofs_per_node
    fixed = np.zeros((C, Nn), dtype=bool)
    g = np.zeros((C, Nn))
    for i in range(d):
        fixed[i] = mesh.dir_v
        fixed[d + i] = mesh.dir_u
    g[0] = ramp(t1, P.ramp_time) * mesh.inflow_profile
    fixed[2 * d] = ~mesh.fluid_touch
    return fixed.reshape(-1), g.reshape(-1)


def residual(problem: FSIProblem, y, y_old, k: float, theta: float, t1: float, admissible_only: bool = True):
    """Global CN residual R(y; y_old) at t1 = t0 + k; +inf if the trial mesh
    is inadmissible (J <= 0 at a quadrature point), the line-search back-off
    of integrators.py:83-90.  ``admissible_only=False`` returns the raw
    assembled residual anyway (kernel parity on tangled random inputs)."""
    mesh = build_mesh(problem)
    y = np.asarray(y, dtype=np.float64)
    Re, jmin = element_residual(mesh, _gather(mesh, y), _gather(mesh, y_old), k, theta)
    if admissible_only and np.any(jmin <= 0.0):
        return np.full(y.size, np.inf)
    Re = Re * _row_mask(mesh)
    P = problem
    Nn, C = P.num_nodes, P.dofs_per_node
    # global dof of (e, a, c) = c * Nn + conn[e, a]
    gidx = (np.arange(C)[None, None, :] * Nn + mesh.conn[:, :, None]).reshape(-1)
    r = np.bincount(gidx, weights=Re.reshape(-1), minlength=C * Nn)
    fixed, g = _dirichlet(mesh, t1)
    r[fixed] = y[fixed] - g[fixed]
    return r


def degenerate(problem: FSIProblem, y, y_old, k: float, theta: float) -> bool:
    """True when the trial mesh of y is inadmissible (J <= 0 at a quadrature point)."""
    mesh = build_mesh(problem)
    _, jmin = element_residual(mesh, _gather(mesh, np.asarray(y, dtype=np.float64)), _gather(mesh, y_old), k, theta)
    return bool(np.any(jmin <= 0.0))


_CSTEP = 1e-30


def _tiled_mesh(mesh: Mesh, reps: int) -> Mesh:
    """Mesh view whose per-element arrays are repeated ``reps`` times."""
    if reps == 1:
        return mesh
    return Mesh(mesh.problem, np.tile(mesh.conn, (reps, 1)), np.tile(mesh.solid, reps),
                np.tile(mesh.outflow, reps), mesh.solid_touch, mesh.fluid_touch, mesh.dir_v,
                mesh.dir_u, mesh.inflow_profile, mesh.Nq, mesh.dNq, mesh.wq, mesh.Nf, mesh.dNf,
                mesh.wf)


def jacobian(problem: FSIProblem, y, y_old, k: float, theta: float, t1: float):
    """Exact sparse Jacobian dR/dy (CSR) by element-wise complex-step."""
    mesh = build_mesh(problem)
    P = problem
    d = P.dim
    Nn, C = P.num_nodes, P.dofs_per_node
    A = 1 << d
    Yn = _gather(mesh, np.asarray(y, dtype=np.float64)).astype(np.complex128)
    Yo = _gather(mesh, y_old)
    E = Yn.shape[0]
    L = A * C
    Ke = np.empty((E, L, L))
    mask = _row_mask(mesh).reshape(E, L)
    # all L perturbation directions in one vectorized call: replicate the
    # element list L times (direction-major) on a temporary mesh view
    chunk = max(1, min(L, (1 << 21) // max(E, 1)))
    for c0 in range(0, L, chunk):
        cols = list(range(c0, min(L, c0 + chunk)))
        nc = len(cols)
        Yp = np.tile(Yn, (nc, 1, 1))
        for j, col in enumerate(cols):
            Yp[j * E:(j + 1) * E, col // C, col % C] += 1j * _CSTEP
        Re, _ = element_residual(_tiled_mesh(mesh, nc), Yp, np.tile(Yo, (nc, 1, 1)), k, theta)
        Re = (Re.imag / _CSTEP).reshape(nc, E, L)
        for j, col in enumerate(cols):
            Ke[:, :, col] = Re[j] * mask
    gl = (np.arange(C)[None, None, :] * Nn + mesh.conn[:, :, None]).reshape(E, L)
    rows = np.repeat(gl[:, :, None], L, axis=2).reshape(-1)
    cols = np.repeat(gl[:, None, :], L, axis=1).reshape(-1)
    J = sp.coo_matrix((Ke.reshape(-1), (rows, cols)), shape=(C * Nn, C * Nn)).tocsr()
    J.sum_duplicates()
    fixed, _ = _dirichlet(mesh, t1)
    keep = sp.diags((~fixed).astype(np.float64))
    J = (keep @ J + sp.diags(fixed.astype(np.float64))).tocsr()
    J.eliminate_zeros()
    return J


# --------------------------------------------------------------------------
# Newton (mirror of reference linalg.py:167-248) and the theta step


@dataclass(frozen=True)
class OracleNewtonSettings:
    abs_tol: float = 1e-10
    rel_tol: float = 0.0
    max_iters: int = 25
    damping_min: float = 1.0 / 64.0


def newton_solve(residual_fn, jacobian_fn, x0, cfg: OracleNewtonSettings, history=None):
    """Damped Newton with the reference's control flow (linalg.py:207-248);
    the linear solve is a sparse LU instead of the dense one (linalg.py:224)."""
    x = np.asarray(x0, dtype=np.float64).copy()
    r = np.asarray(residual_fn(x), dtype=np.float64)
    if not np.all(np.isfinite(r)):
        raise OracleNumericBreakdown("residual not finite at starting point")
    rnorm = float(np.linalg.norm(r))
    target = cfg.abs_tol + cfg.rel_tol * rnorm
    for it in range(cfg.max_iters):
        if rnorm <= target:
            return x, it
        J = jacobian_fn(x)
        try:
            dx = spla.splu(J.tocsc()).solve(-r)
        except RuntimeError as exc:
            raise OracleNumericBreakdown("singular linearization in Newton step") from exc
        if not np.all(np.isfinite(dx)):
            raise OracleNumericBreakdown("non-finite Newton direction")
        lam = 1.0
        while True:
            x_trial = x + lam * dx
            r_trial = np.asarray(residual_fn(x_trial), dtype=np.float64)
            trial_norm = float(np.linalg.norm(r_trial)) if np.all(np.isfinite(r_trial)) else np.inf
            if trial_norm < rnorm or lam <= cfg.damping_min:
                break
            lam = max(lam / 2.0, cfg.damping_min)
        if not np.isfinite(trial_norm):
            raise OracleNumericBreakdown(f"residual not finite after damping to {lam}")
        x, r, rnorm = x_trial, r_trial, trial_norm
        if history is not None:
            history.append(rnorm)
    if rnorm <= target:
        return x, cfg.max_iters
    raise OracleMaxIters(f"no convergence in {cfg.max_iters} iterations (||r|| = {rnorm:.3e}, target {target:.3e})")


def theta_step(problem: FSIProblem, values, t0: float, k: float, theta0: float,
               newton: OracleNewtonSettings):
    """One shifted-CN step (reference integrators.py:70-96 bookkeeping)."""
    theta = min(max(0.5 + theta0 * k, 0.5), 1.0)
    t1 = t0 + k
    y_old = np.asarray(values, dtype=np.float64)
    try:
        sol, it = newton_solve(
            lambda y: residual(problem, y, y_old, k, theta, t1),
            lambda y: jacobian(problem, y, y_old, k, theta, t1),
            y_old, newton)
    except (OracleNumericBreakdown, OracleMaxIters) as exc:
        raise OracleTimeStepError(f"implicit step failed at t_n={t1!r}, k={k!r}: {exc}") from exc
    return sol, t1, it


_WINDOW_RTOL = 1e-9


def split_window(window: float, step: float) -> int:
    """Mirror of reference integrators.py:115-123."""
    n = max(int(round(window / step)), 1)
    if abs(window - n * step) > _WINDOW_RTOL * max(abs(window), step):
        raise ValueError(f"window {window!r} is not an integer multiple of step {step!r}")
    return n


class OracleFSIPropagator:
    """CPU propagator with the reference Propagator protocol
    (integrators.py:105-112; advance mirrors integrators.py:144-166)."""

    def __init__(self, problem: FSIProblem, step: float, theta0: float = 1.0,
                 newton: OracleNewtonSettings | None = None, cost_hint: float = 0.0):
        if step <= 0.0:
            raise ValueError("step must be positive")
        theta = 0.5 + theta0 * step
        if not 0.5 - 1e-12 <= theta <= 1.0 + 1e-12:
            raise ValueError(f"effective theta {theta} outside [1/2, 1]; adjust theta0")
        self.problem = problem
        self.step = step
        self.theta0 = theta0
        self.newton = newton if newton is not None else OracleNewtonSettings()
        self.cost_hint = cost_hint
        self.newton_iterations = 0
        self.steps_taken = 0
        self._lock = threading.Lock()

    def advance_values(self, values, t0: float, t_end: float):
        window = t_end - t0
        n = split_window(window, self.step)
        y, t = np.asarray(values, dtype=np.float64), t0
        iters = 0
        for _ in range(n - 1):
            y, t, it = theta_step(self.problem, y, t, self.step, self.theta0, self.newton)
            iters += it
        last = t_end - t
        y, t, it = theta_step(self.problem, y, t, last, self.theta0, self.newton)
        iters += it
        with self._lock:
            self.newton_iterations += iters
            self.steps_taken += n
        return y

    def advance(self, state, t_end: float):
        window = t_end - state.time
        if window == 0.0:
            return state
        if window < 0.0:
            raise ValueError(f"cannot advance backwards from {state.time} to {t_end}")
        y = self.advance_values(state.values, state.time, t_end)
        return state.with_values(y, time=t_end)


def initial_state(problem: FSIProblem, time: float = 0.0) -> State:
    return State(problem.zero_values(), time, problem.layout())
