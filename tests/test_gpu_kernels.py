"""GPU parity ladder, kernel level: flags, residual (K1), JVP / assembled
Jacobian (K2/K3), multigrid-preconditioned GMRES (K4-K6) against the CPU
oracle (oracle/fsi_oracle.py) on identical seeded inputs.

Tolerances: the element arithmetic is the same fp64 formula evaluated in a
different association order, so residual / Jacobian products agree to
round-off (relative 1e-12); linear solves agree to the Krylov tolerance.
"""

import numpy as np
import pytest

from oracle import fsi_oracle as O
from paper_1907_01252_b200.problem import CONFIGS, channel_3d, small_problem

pytestmark = pytest.mark.gpu

PROBLEMS = {
    "small2d": small_problem(8, 2),
    "c1": CONFIGS["c1"].problem,
    "small3d": channel_3d(10, 2, 2, name="small3d"),
}


def random_states(P, S, seed, scale_u=1e-3):
    rng = np.random.default_rng(seed)
    n = P.num_nodes
    d = P.dim
    out = []
    for _ in range(S):
        out.append(np.concatenate([0.3 * rng.standard_normal(d * n), scale_u * rng.standard_normal(d * n),
                                   rng.standard_normal(n)]))
    return np.array(out)


@pytest.fixture(scope="module")
def devices(cuda):
    from paper_1907_01252_b200.propagator import FSIDevice
    return {name: FSIDevice(P, max_slices=3) for name, P in PROBLEMS.items()}


def _step_args(S, k=0.002, t1=0.3):
    theta = 0.5 + k
    return [k] * S, [theta] * S, [t1 + 0.01 * s for s in range(S)]


@pytest.mark.parametrize("name", list(PROBLEMS))
def test_flags_match_oracle(devices, name):
    P = PROBLEMS[name]
    dev = devices[name]
    nf, cf = dev.flags()
    m = O.build_mesh(P)
    assert np.array_equal((cf & 1).astype(bool), m.solid)
    assert np.array_equal((cf & 2).astype(bool), m.outflow)
    assert np.array_equal((nf & 1).astype(bool), m.solid_touch)
    assert np.array_equal((nf & 2).astype(bool), m.fluid_touch)
    assert np.array_equal((nf & 4).astype(bool), m.dir_v)
    assert np.array_equal((nf & 8).astype(bool), m.dir_u)


@pytest.mark.parametrize("name", list(PROBLEMS))
def test_residual_matches_oracle(devices, name):
    P = PROBLEMS[name]
    dev = devices[name]
    S = 3
    Y = random_states(P, S, 1)
    Yo = random_states(P, S, 2)
    k, th, t1 = _step_args(S)
    r_dev, norms = dev.residual(dev.to_device(Y), dev.to_device(Yo), k, th, t1)
    r = dev.to_host(r_dev)
    for s in range(S):
        ref = O.residual(P, Y[s], Yo[s], k[s], th[s], t1[s])
        err = np.linalg.norm(r[s] - ref) / np.linalg.norm(ref)
        assert err <= 1e-12, (name, s, err)
        assert abs(norms[s] - np.linalg.norm(ref)) <= 1e-12 * np.linalg.norm(ref)


@pytest.mark.parametrize("name", list(PROBLEMS))
def test_jvp_and_assembled_spmv_match_oracle(devices, name):
    P = PROBLEMS[name]
    dev = devices[name]
    S = 3
    Y = random_states(P, S, 3)
    Yo = random_states(P, S, 4)
    W = random_states(P, S, 5, scale_u=1.0)
    k, th, t1 = _step_args(S)
    y, yo, w = dev.to_device(Y), dev.to_device(Yo), dev.to_device(W)
    jw = dev.to_host(dev.jvp(y, yo, w, k, th, t1))
    dev.assemble(y, yo, k, th, t1)
    aw = dev.to_host(dev.spmv(w))
    for s in range(S):
        J = O.jacobian(P, Y[s], Yo[s], k[s], th[s], t1[s])
        ref = J @ W[s]
        assert np.linalg.norm(jw[s] - ref) <= 1e-12 * np.linalg.norm(ref), name
        assert np.linalg.norm(aw[s] - ref) <= 1e-12 * np.linalg.norm(ref), name


@pytest.mark.parametrize("name", list(PROBLEMS))
def test_gmres_mg_solves_jacobian_system(devices, name):
    import scipy.sparse.linalg as spla
    from paper_1907_01252_b200.propagator import KrylovSettings
    P = PROBLEMS[name]
    dev = devices[name]
    S = 2
    Y = random_states(P, S, 6, scale_u=1e-4) * 0.1
    Yo = Y.copy()
    B = random_states(P, S, 7, scale_u=1.0)
    k, th, t1 = _step_args(S)
    y, yo = dev.to_device(Y), dev.to_device(Yo)
    dev.assemble(y, yo, k, th, t1)
    ks = KrylovSettings(rtol=1e-10, max_iters=400)
    dev.precond_setup(S, ks)
    x, its, res = dev.linear_solve(dev.to_device(B), ks)
    X = dev.to_host(x)
    for s in range(S):
        J = O.jacobian(P, Y[s], Yo[s], k[s], th[s], t1[s])
        ref = spla.splu(J.tocsc()).solve(B[s])
        rel = np.linalg.norm(J @ X[s] - B[s]) / np.linalg.norm(B[s])
        assert rel <= 2e-10, (name, s, rel, its[s])
        assert its[s] < 120, (name, its[s])
        assert np.linalg.norm(X[s] - ref) <= 1e-6 * np.linalg.norm(ref)


@pytest.mark.parametrize("smoother", ["jacobi", "vanka"])
def test_both_smoothers_solve_c1_fine_step_system(devices, smoother):
    """The node-block-Jacobi smoother (omega 0.5) stays selectable and converges
    on a fine-step system; Vanka (default) too."""
    from paper_1907_01252_b200.propagator import KrylovSettings
    P = PROBLEMS["c1"]
    dev = devices["c1"]
    S = 2
    Y = random_states(P, S, 31, scale_u=1e-4) * 0.1
    B = random_states(P, S, 32, scale_u=1.0)
    k, th, t1 = _step_args(S)
    y = dev.to_device(Y)
    dev.assemble(y, y, k, th, t1)
    ks = KrylovSettings(rtol=1e-10, max_iters=400, smoother=smoother, omega=0.5 if smoother == "jacobi" else 0.9)
    dev.precond_setup(S, ks)
    x, its, res = dev.linear_solve(dev.to_device(B), ks)
    X = dev.to_host(x)
    for s in range(S):
        J = O.jacobian(P, Y[s], Y[s], k[s], th[s], t1[s])
        assert np.linalg.norm(J @ X[s] - B[s]) <= 2e-10 * np.linalg.norm(B[s]), (smoother, its[s])


def test_invalid_arguments_are_reported(devices):
    from paper_1907_01252_b200.propagator import DeviceError
    dev = devices["small2d"]
    y = dev.empty(5)  # more slices than the context holds (3)
    with pytest.raises(DeviceError, match="batch size"):
        dev.residual(y, y, [0.01] * 5, [0.51] * 5, [0.1] * 5)


@pytest.mark.parametrize("name", ["small2d", "small3d"])
def test_dense_coarsest_inverse_matches_direct_solve(devices, name):
    """One-level hierarchy: the preconditioner IS the dense coarsest inverse.
    small2d (135 dofs) takes the cluster Gauss-Jordan (register tiles,
    pivot rows through distributed shared memory), small3d (693 dofs) the
    single-CTA fallback.  The factorisation is fp64, the stored inverse fp32
    (preconditioner storage), so the apply matches a direct solve to ~1e-6
    and one-level FGMRES converges in a couple of iterations."""
    import scipy.sparse.linalg as spla
    from paper_1907_01252_b200.propagator import KrylovSettings
    P = PROBLEMS[name]
    dev = devices[name]
    S = 3
    Y = random_states(P, S, 41, scale_u=1e-4) * 0.1
    Yo = random_states(P, S, 42, scale_u=1e-4) * 0.1
    B = random_states(P, S, 43, scale_u=1.0)
    k, th, t1 = _step_args(S)
    dev.assemble(dev.to_device(Y), dev.to_device(Yo), k, th, t1)
    dev.precond_setup(S, KrylovSettings(max_levels=1))
    X = dev.to_host(dev.precond_apply(dev.to_device(B)))
    ks = KrylovSettings(max_levels=1, rtol=1e-10)
    _, its, _ = dev.linear_solve(dev.to_device(B), ks)
    for s in range(S):
        J = O.jacobian(P, Y[s], Yo[s], k[s], th[s], t1[s])
        ref = spla.splu(J.tocsc()).solve(B[s])
        err = np.linalg.norm(X[s] - ref) / np.linalg.norm(ref)
        assert err <= 1e-5, (name, s, err)
        assert its[s] <= 4, (name, s, its[s])


def _device_with_env(P, env, S=3):
    import os
    from paper_1907_01252_b200.propagator import FSIDevice
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return FSIDevice(P, max_slices=S)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("name", ["c1", "small3d"])
def test_jacobian_formulations_agree(cuda, name):
    """K2 by pointwise linearisation (1 + d dual passes per column component)
    in node-owner strips (2-d default, all directions of a column component in
    one multi-tangent flux pass; PINT_JAC_MT=0: one dual pass per direction;
    3-d uses the colour scatter), in the
    colour-ordered element scatter (PINT_JAC=colour) and K2 by one dual pass
    per Jacobian column (PINT_JAC=columns) assemble the same block-stencil
    operator up to round-off."""
    P = PROBLEMS[name]
    S = 3
    Y = random_states(P, S, 51)
    Yo = random_states(P, S, 52)
    k, th, t1 = _step_args(S)
    blocks = []
    for env in ({}, {"PINT_JAC_MT": "0"}, {"PINT_JAC": "colour"}, {"PINT_JAC": "columns"}):
        dev = _device_with_env(P, env)
        dev.assemble(dev.to_device(Y), dev.to_device(Yo), k, th, t1)
        blocks.append(dev.jacobian_blocks(S).cpu().numpy())
    scale = np.abs(blocks[-1]).max()
    for b in blocks[:-1]:
        assert np.abs(b - blocks[-1]).max() <= 1e-13 * scale


@pytest.mark.parametrize("name", ["c1", "small3d"])
def test_vanka_setup_variants_agree(cuda, name):
    """Register-row Gauss-Jordan with implicit pivoting (default) and the
    warp-per-cell shared-memory version (PINT_VANKA_SETUP=smem) store the same
    fp32 cell inverses up to fp32 rounding: one V-cycle agrees to 1e-5."""
    from paper_1907_01252_b200.propagator import KrylovSettings
    P = PROBLEMS[name]
    S = 2
    Y = random_states(P, S, 61, scale_u=1e-4) * 0.1
    B = random_states(P, S, 62, scale_u=1.0)
    k, th, t1 = _step_args(S)
    outs = []
    for env in ({}, {"PINT_VANKA_SETUP": "smem"}):
        dev = _device_with_env(P, env, S)
        y = dev.to_device(Y)
        dev.assemble(y, y, k, th, t1)
        dev.precond_setup(S, KrylovSettings())
        outs.append(dev.to_host(dev.precond_apply(dev.to_device(B))))
    for s in range(S):
        assert np.linalg.norm(outs[0][s] - outs[1][s]) <= 1e-5 * np.linalg.norm(outs[1][s]), (name, s)


@pytest.mark.parametrize("name", ["small2d", "c1"])
def test_residual_strip_variant_agrees(cuda, name):
    """K1 in node-owner strips (k_residual_strip, PINT_RES=strip: one launch
    writing every row once, fixed rows included; measured slower than the tiled
    colour kernels, off by default) gives the same residual up to round-off,
    flags the same degenerate slices, and matches the oracle."""
    P = PROBLEMS[name]
    S = 3
    Y = random_states(P, S, 91)
    Yo = random_states(P, S, 92)
    k, th, t1 = _step_args(S)
    outs, norms = [], []
    for env in ({}, {"PINT_RES": "strip"}):
        dev = _device_with_env(P, env)
        r, nrm = dev.residual(dev.to_device(Y), dev.to_device(Yo), k, th, t1)
        outs.append(dev.to_host(r))
        norms.append(nrm)
    scale = np.abs(outs[0]).max()
    assert np.abs(outs[0] - outs[1]).max() <= 1e-13 * scale
    assert np.allclose(norms[0], norms[1], rtol=1e-13)
    ref = O.residual(P, Y[0], Yo[0], k[0], th[0], t1[0])
    assert np.linalg.norm(outs[1][0] - ref) <= 1e-12 * np.linalg.norm(ref)


@pytest.mark.parametrize("name", ["small2d", "c1", "small3d"])
def test_deformation_rows_structural_zeros(devices, name):
    """The product kernels skip the coefficient planes (u_i row, column other
    than v_i / u_i) as structural zeros (pint_common.cuh row_couples): the
    assembled Jacobian must hold exact zeros there at every stencil offset,
    for fluid, solid and interface nodes, and the oracle's sparse Jacobian has
    no entry there either."""
    P, dev = PROBLEMS[name], devices[name]
    S = 2
    Y = random_states(P, S, 81)
    Yo = random_states(P, S, 82)
    k, th, t1 = _step_args(S)
    dev.assemble(dev.to_device(Y), dev.to_device(Yo), k, th, t1)
    blocks = dev.jacobian_blocks(S).cpu().numpy()  # [S][noff][ca][cb][np]
    d, C = P.dim, P.dofs_per_node
    assert np.abs(blocks).max() > 0.0
    for i in range(d):
        for cb in range(C):
            if cb in (i, d + i):
                assert np.abs(blocks[:, :, d + i, cb, :]).max() > 0.0
            else:
                assert not blocks[:, :, d + i, cb, :].any(), (name, i, cb)
    J = O.jacobian(P, Y[0], Yo[0], k[0], th[0], t1[0]).tocoo()
    n = P.num_nodes
    rows_c, cols_c = J.row // n, J.col // n
    nz = J.data != 0.0
    for i in range(d):
        bad = nz & (rows_c == d + i) & (cols_c != i) & (cols_c != d + i)
        assert not bad.any(), (name, i)


@pytest.mark.parametrize("name,tail_rows", [("c1", "1000"), ("small3d", "300")])
def test_vanka_fused_sweep_bitwise(cuda, name, tail_rows):
    """The fused level-0 Vanka sweep (k_vanka_apply: cell solves + gather in
    one pass) and the split pair (k_vanka_cell + k_vanka_gather through the
    y_c buffer) give the same V-cycle bit for bit (same fmaf order, same fixed
    corner order).  PINT_TAIL_ROWS keeps level 0 out of the cluster tail."""
    from paper_1907_01252_b200.propagator import KrylovSettings
    P = PROBLEMS[name]
    S = 2
    Y = random_states(P, S, 71, scale_u=1e-4) * 0.1
    B = random_states(P, S, 72, scale_u=1.0)
    k, th, t1 = _step_args(S)
    outs = []
    for mode in ("fused", "split"):
        dev = _device_with_env(P, {"PINT_VANKA": mode, "PINT_TAIL_ROWS": tail_rows}, S)
        y = dev.to_device(Y)
        dev.assemble(y, y, k, th, t1)
        dev.precond_setup(S, KrylovSettings())
        outs.append(dev.to_host(dev.precond_apply(dev.to_device(B))))
    assert np.array_equal(outs[0], outs[1]), name


@pytest.mark.parametrize("name,tail_rows", [("c1", "1000"), ("small3d", "300")])
def test_spmv32_variants_bitwise(cuda, name, tail_rows):
    """The V-cycle residuals with the fp32 operator copy: (node, row) threads
    over a shared-memory staged neighbourhood (k_resid32_staged, default on
    wide levels), one thread per node (k_spmv_node) and one per (node, row)
    with register gathers (k_spmv, PINT_SPMV32=row) sum in the same order, so
    the V-cycle agrees bit for bit.  PINT_SPMV32_MIN=0 puts the wide-level
    kernels on these small meshes."""
    from paper_1907_01252_b200.propagator import KrylovSettings
    P = PROBLEMS[name]
    S = 2
    Y = random_states(P, S, 73, scale_u=1e-4) * 0.1
    B = random_states(P, S, 74, scale_u=1.0)
    k, th, t1 = _step_args(S)
    outs = []
    for mode in ("staged", "node", "row"):
        dev = _device_with_env(P, {"PINT_SPMV32": mode, "PINT_SPMV32_MIN": "0", "PINT_TAIL_ROWS": tail_rows}, S)
        y = dev.to_device(Y)
        dev.assemble(y, y, k, th, t1)
        dev.precond_setup(S, KrylovSettings())
        outs.append(dev.to_host(dev.precond_apply(dev.to_device(B))))
    assert np.array_equal(outs[0], outs[2]), name
    assert np.array_equal(outs[1], outs[2]), name


@pytest.mark.parametrize("name,tail_rows", [("c1", "1000"), ("small3d", "300")])
def test_resid32_fp32_accumulation_variant(cuda, name, tail_rows):
    """PINT_RESID_ACC=f32 (opt-in): the staged V-cycle residual with fp32
    products and partial sums.  It is off by default because it would make a
    slice's bits depend on whether its batch crosses the staged-kernel
    threshold; one V-cycle agrees with the fp64 accumulation to 1e-5."""
    from paper_1907_01252_b200.propagator import KrylovSettings
    P = PROBLEMS[name]
    S = 2
    Y = random_states(P, S, 79, scale_u=1e-4) * 0.1
    B = random_states(P, S, 80, scale_u=1.0)
    k, th, t1 = _step_args(S)
    outs = []
    for acc in ("f64", "f32"):
        dev = _device_with_env(P, {"PINT_RESID_ACC": acc, "PINT_SPMV32_MIN": "0", "PINT_TAIL_ROWS": tail_rows}, S)
        y = dev.to_device(Y)
        dev.assemble(y, y, k, th, t1)
        dev.precond_setup(S, KrylovSettings())
        outs.append(dev.to_host(dev.precond_apply(dev.to_device(B))))
    for s in range(S):
        assert np.linalg.norm(outs[0][s] - outs[1][s]) <= 1e-5 * np.linalg.norm(outs[0][s]), (name, s)
    assert not np.array_equal(outs[0], outs[1])  # the variant really ran


@pytest.mark.parametrize("name,tail_rows", [("c1", "1000"), ("c1", "100"), ("small3d", "300")])
def test_fused_prolongation_bitwise(cuda, name, tail_rows):
    """The coarse-grid correction added inside the post-smoothing residual
    kernel (k_resid32_staged<PROLONG>, PINT_FUSE_PROLONG=1; measured slower, off) equals
    k_prolong_add followed by the plain residual (default) bit for
    bit: same prolongation sum, same residual order."""
    from paper_1907_01252_b200.propagator import KrylovSettings
    P = PROBLEMS[name]
    S = 2
    Y = random_states(P, S, 77, scale_u=1e-4) * 0.1
    B = random_states(P, S, 78, scale_u=1.0)
    k, th, t1 = _step_args(S)
    outs = []
    for fuse in ("1", "0"):
        dev = _device_with_env(P, {"PINT_FUSE_PROLONG": fuse, "PINT_SPMV32_MIN": "0", "PINT_TAIL_ROWS": tail_rows}, S)
        y = dev.to_device(Y)
        dev.assemble(y, y, k, th, t1)
        dev.precond_setup(S, KrylovSettings())
        outs.append(dev.to_host(dev.precond_apply(dev.to_device(B))))
    assert np.array_equal(outs[0], outs[1]), name


@pytest.mark.parametrize("name,tail_rows", [("c1", "1000"), ("c1", "100"), ("small3d", "300")])
def test_vanka_stencil_sweep_matches_cell_form(cuda, name, tail_rows):
    """The Vanka sweep in block-stencil form (k_vanka_stencil_build once per
    hierarchy build + k_vanka_stencil_apply, default) is the same linear map
    as the cell-inverse sweep (k_vanka_apply, PINT_VANKA=fused) up to fp32
    rounding of the summed coefficients: one V-cycle agrees to 1e-5, and a
    preconditioned solve to rtol 1e-8 takes the same number of iterations up
    to rounding (within 3; the bench configs' counts are identical)."""
    from paper_1907_01252_b200.propagator import KrylovSettings
    P = PROBLEMS[name]
    S = 2
    Y = random_states(P, S, 75, scale_u=1e-4) * 0.1
    B = random_states(P, S, 76, scale_u=1.0)
    k, th, t1 = _step_args(S)
    outs, its = [], []
    for mode in ("stencil", "fused"):
        dev = _device_with_env(P, {"PINT_VANKA": mode, "PINT_TAIL_ROWS": tail_rows}, S)
        y = dev.to_device(Y)
        dev.assemble(y, y, k, th, t1)
        dev.precond_setup(S, KrylovSettings())
        outs.append(dev.to_host(dev.precond_apply(dev.to_device(B))))
        x, it, _ = dev.linear_solve(dev.to_device(B), KrylovSettings(rtol=1e-8))
        its.append(list(it))
    for s in range(S):
        assert np.linalg.norm(outs[0][s] - outs[1][s]) <= 1e-5 * np.linalg.norm(outs[1][s]), (name, s)
    assert max(abs(int(a) - int(b)) for a, b in zip(its[0], its[1])) <= 3, (name, its)


@pytest.mark.parametrize("name", ["c1", "small3d"])
def test_fused_cgs_norm_bitwise(cuda, name):
    """The second CGS2 update fused with ||w|| and the Givens update
    (k_mupdate_norm_givens, default) and the split pair (k_mupdate +
    k_norm_givens, PINT_SPLIT_NORM=1) give the same flexible-GMRES solve bit
    for bit: same solution, same iteration counts."""
    from paper_1907_01252_b200.propagator import KrylovSettings
    P = PROBLEMS[name]
    S = 2
    Y = random_states(P, S, 81, scale_u=1e-4) * 0.1
    B = random_states(P, S, 82, scale_u=1.0)
    k, th, t1 = _step_args(S)
    res = []
    for env in ({}, {"PINT_SPLIT_NORM": "1"}):
        dev = _device_with_env(P, env, S)
        y = dev.to_device(Y)
        dev.assemble(y, y, k, th, t1)
        ks = KrylovSettings(rtol=1e-10)
        dev.precond_setup(S, ks)
        x, its, _ = dev.linear_solve(dev.to_device(B), ks)
        res.append((dev.to_host(x), list(its)))
    assert res[0][1] == res[1][1] and min(res[0][1]) > 3
    assert np.array_equal(res[0][0], res[1][0]), name


@pytest.mark.parametrize("name", ["c1", "small3d"])
def test_gram_schmidt_passes(cuda, name):
    """Gram-Schmidt passes per slice from the slice's own relative tolerance:
    one classical pass at loose tolerances (bitwise PINT_CGS=1), CGS2 below
    1e-7 (bitwise PINT_CGS=2); in a batch mixing both, each slice gets the
    same bits as when solved alone (batch invariance)."""
    from paper_1907_01252_b200.propagator import KrylovSettings
    P = PROBLEMS[name]
    S = 2
    Y = random_states(P, S, 91, scale_u=1e-4) * 0.1
    B = random_states(P, S, 92, scale_u=1.0)
    k, th, t1 = _step_args(S)

    def solve(env, ks, sl=slice(0, S), b=B):
        n = sl.stop - sl.start
        dev = _device_with_env(P, env, S)
        y = dev.to_device(Y[sl])
        dev.assemble(y, y, k[sl], th[sl], t1[sl])
        dev.precond_setup(n, ks)
        x, its, res = dev.linear_solve(dev.to_device(b[sl]), ks)
        return dev.to_host(x), np.array(its), np.array(res)

    for rtol, forced in ((1e-8, "2"), (1e-5, "1")):
        ks = KrylovSettings(rtol=rtol)
        xa, ia, ra = solve({}, ks)
        xb, ib, _ = solve({"PINT_CGS": forced}, ks)
        assert np.array_equal(ia, ib) and np.array_equal(xa, xb), (rtol, ia, ib)
    # slice 0: ||b|| large -> rtol 1e-9 governs (two passes); slice 1: the
    # absolute tolerance governs (1e-5 relative, one pass)
    B2 = B.copy()
    B2[0] *= 1e4
    atol = 1e-5 * np.linalg.norm(B2[1])
    ks = KrylovSettings(rtol=1e-9, atol=atol)
    xm, im, _ = solve({}, ks, b=B2)
    for s in range(S):
        xs, is_, _ = solve({}, ks, sl=slice(s, s + 1), b=B2)
        assert is_[0] == im[s] and np.array_equal(xs[0], xm[s]), (name, s)
