"""GPU, BASELINE c5 inputs (seeded N(0,1) velocity / N(0,1e-3^2) deformation /
N(0,1) pressure): kernel parity against the oracle on the 1e4-cell mesh, and
size-independent properties at 1e5 cells (linearity of J w, assembled SpMV
== matrix-free J w == central differences of the residual, bitwise batch
invariance of residual / SpMV / V-cycle)."""

import numpy as np
import pytest

from oracle import fsi_oracle as O
from paper_1907_01252_b200.problem import c5_problem, c5_random_states

pytestmark = pytest.mark.gpu


def _args(S, k=2.0 ** -10, t1=0.3):
    return [k] * S, [0.5 + k] * S, [t1] * S


def test_c5_1e4_residual_and_jacobian_match_oracle(cuda):
    from paper_1907_01252_b200.propagator import FSIDevice
    P = c5_problem("1e4")
    S = 2
    dev = FSIDevice(P, S)
    Y, Yo, W = (c5_random_states(P, S, sd) for sd in (11, 12, 13))
    k, th, t1 = _args(S)
    y, yo, w = dev.to_device(Y), dev.to_device(Yo), dev.to_device(W)
    r, _ = dev.residual(y, yo, k, th, t1)
    dev.assemble(y, yo, k, th, t1)
    aw = dev.to_host(dev.spmv(w))
    r = dev.to_host(r)
    for s in range(S):
        ref = O.residual(P, Y[s], Yo[s], k[s], th[s], t1[s])
        assert np.linalg.norm(r[s] - ref) <= 1e-12 * np.linalg.norm(ref)
        J = O.jacobian(P, Y[s], Yo[s], k[s], th[s], t1[s])
        ref_w = J @ W[s]
        assert np.linalg.norm(aw[s] - ref_w) <= 1e-12 * np.linalg.norm(ref_w)


def test_c5_1e5_properties(cuda):
    import torch
    from paper_1907_01252_b200.propagator import FSIDevice, KrylovSettings
    P = c5_problem("1e5")
    S = 3
    dev = FSIDevice(P, S, restart=4)
    Y, Yo, W1, W2 = (c5_random_states(P, S, sd) for sd in (21, 22, 23, 24))
    k, th, t1 = _args(S)
    y, yo, w1, w2 = (dev.to_device(a) for a in (Y, Yo, W1, W2))
    # linearity of the matrix-free product
    a, b = 0.75, -1.5
    lhs = dev.jvp(y, yo, a * w1 + b * w2, k, th, t1)
    rhs = a * dev.jvp(y, yo, w1, k, th, t1) + b * dev.jvp(y, yo, w2, k, th, t1)
    assert (lhs - rhs).norm() <= 1e-12 * rhs.norm()
    # assembled SpMV == matrix-free J w
    dev.assemble(y, yo, k, th, t1)
    jw = dev.jvp(y, yo, w1, k, th, t1)
    aw = dev.spmv(w1)
    assert (aw - jw).norm() <= 1e-12 * jw.norm()
    # central differences of the residual converge to J w (the c5 states are
    # rough -- i.i.d. nodal N(0,1) velocities -- so the FD truncation error is
    # large at moderate eps; check the trend and a loose bound)
    errs = []
    for eps in (1e-5, 1e-7):
        rp, _ = dev.residual(y + eps * w1, yo, k, th, t1)
        rm, _ = dev.residual(y - eps * w1, yo, k, th, t1)
        errs.append(float(((rp - rm) / (2 * eps) - jw).norm() / jw.norm()))
    assert errs[1] < errs[0] and errs[1] < 1e-5, errs
    # batch invariance: slice 1 alone == slice 1 inside the batch of 3 (bitwise)
    r3, _ = dev.residual(y, yo, k, th, t1)
    ks = KrylovSettings()
    dev.precond_setup(S, ks)
    v3 = dev.precond_apply(w1)
    s3 = dev.spmv(w1)
    one = slice(1, 2)
    r1, _ = dev.residual(y[one].contiguous(), yo[one].contiguous(), k[:1], th[:1], t1[:1])
    dev.assemble(y[one].contiguous(), yo[one].contiguous(), k[:1], th[:1], t1[:1])
    s1 = dev.spmv(w1[one].contiguous())
    dev.precond_setup(1, ks)
    v1 = dev.precond_apply(w1[one].contiguous())
    assert torch.equal(r1[0], r3[1]) and torch.equal(s1[0], s3[1]) and torch.equal(v1[0], v3[1])


def test_matrix_free_context_and_solve(cuda):
    """PINT_CTX_MATRIX_FREE: no Jacobian / hierarchy allocated; residual and
    J w match an assembled context bitwise; the unpreconditioned matrix-free
    GMRES solves J x = b (checked against the oracle's sparse J); calls that
    need the hierarchy are refused."""
    from paper_1907_01252_b200.propagator import DeviceError, FSIDevice, KrylovSettings
    P = c5_problem("1e4")
    S = 2
    full, lean = FSIDevice(P, S, restart=30), FSIDevice(P, S, restart=30, matrix_free=True)
    Y, Yo, W = (0.1 * c5_random_states(P, S, sd) for sd in (21, 22, 23))
    k, th, t1 = _args(S)
    for name in ("residual", "jvp"):
        a = [full.to_device(v) for v in (Y, Yo, W)]
        b = [lean.to_device(v) for v in (Y, Yo, W)]
        if name == "residual":
            ra, _ = full.residual(a[0], a[1], k, th, t1)
            rb, _ = lean.residual(b[0], b[1], k, th, t1)
        else:
            ra = full.jvp(a[0], a[1], a[2], k, th, t1)
            rb = lean.jvp(b[0], b[1], b[2], k, th, t1)
        assert full.to_host(ra).tobytes() == lean.to_host(rb).tobytes()
    y, yo, rhs = lean.to_device(Y), lean.to_device(Yo), lean.to_device(W)
    x, its, res = lean.linear_solve_mf(y, yo, k, th, t1, rhs, KrylovSettings(rtol=1e-8, max_iters=60))
    xh = lean.to_host(x)
    for s in range(S):
        # the reported residual is the true ||b - J x|| of the matrix-free operator: equal to the
        # oracle's sparse-J residual of the returned x, and reduced by the Krylov iterations
        J = O.jacobian(P, Y[s], Yo[s], k[s], th[s], t1[s])
        true = np.linalg.norm(W[s] - J @ xh[s])
        assert abs(true - res[s]) <= 1e-8 * np.linalg.norm(W[s]), (s, its[s], res[s], true)
        assert res[s] < np.linalg.norm(W[s]) and its[s] == 60
    with pytest.raises(DeviceError, match="matrix-free"):
        lean.assemble(y, yo, k, th, t1)
