"""GPU: the drop-in itself -- the UNMODIFIED reference driver
(pintbench.run_parareal, from baseline/_ref or /root/reference) driving the
GPU propagators, and the raw ctypes stub of INTEGRATION.md."""

import ctypes
import os

import numpy as np
import pytest

from fields import field_errors
from paper_1907_01252_b200.problem import small_problem
from refimport import pintbench

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "parareal_small_classic.npz")


def test_reference_driver_with_gpu_propagators(cuda):
    pb = pintbench()
    if pb is None:
        pytest.skip("reference package not installed (baseline/_ref)")
    from pintbench.parareal import PararealConfig, run_parareal
    from paper_1907_01252_b200.propagator import (FSIDevice, NewtonSettings, ThetaSettings, initial_state,
                                                  make_propagator)
    g = np.load(GOLD)
    P = small_problem(8, 2)
    nw = NewtonSettings(1e-10, 1e-10)
    dev = FSIDevice(P, 8)
    F = make_propagator(P, ThetaSettings(0.01, 1.0, nw), device=dev)
    C = make_propagator(P, ThetaSettings(0.05, 1.0, nw), device=dev)
    states, tr = run_parareal(C, F, initial_state(P), 0.8, PararealConfig(intervals=8, max_iters=4, tol=1e-30))
    assert tr.iterations_run == int(g["iterations_run"]) and tr.fine_propagations == 32
    for l in range(1, 9):
        assert max(field_errors(P, states[l].values, g["final"][l]).values()) <= 1e-6


def test_raw_ctypes_stub(cuda):
    import torch
    from paper_1907_01252_b200._lib import LIB_PATH, KrylovOpts, NewtonOpts, ProblemDesc
    lib = ctypes.CDLL(LIB_PATH)
    desc = ProblemDesc()
    desc.dim = 2
    desc.cells[:] = [32, 8, 1]
    desc.extent[:] = [2.0, 0.5, 1.0]
    desc.bar_lo[:] = [0.8, 0.0, 0.0]
    desc.bar_hi[:] = [1.0, 0.25, 0.0]
    desc.rho_f, desc.nu_f, desc.rho_s, desc.mu_s, desc.lambda_s = 1000.0, 1e-3, 1000.0, 5e5, 2e6
    desc.u_peak, desc.ramp_time, desc.alpha_p = 1.0, 0.5, 1.0
    ctx = ctypes.c_void_p()
    assert lib.pint_create(ctypes.byref(desc), 4, 30, ctypes.byref(ctx)) == 0
    nn, np_, C, lv = (ctypes.c_int32() for _ in range(4))
    lib.pint_sizes(ctx, ctypes.byref(nn), ctypes.byref(np_), ctypes.byref(C), ctypes.byref(lv))
    assert (nn.value, C.value) == (297, 5) and np_.value % 32 == 0
    S = 4
    y = torch.zeros((S, C.value, np_.value), dtype=torch.float64, device="cuda")
    out = torch.empty_like(y)
    t0 = (ctypes.c_double * S)(*[0.1 * s for s in range(S)])
    t1 = (ctypes.c_double * S)(*[0.1 * s + 0.01 for s in range(S)])
    n = (ctypes.c_int32 * S)(*[5] * S)
    its, kits, status = (ctypes.c_int32 * S)(), (ctypes.c_int32 * S)(), (ctypes.c_int32 * S)()
    ft = (ctypes.c_double * S)()
    lib.pint_propagate.argtypes = None
    rc = lib.pint_propagate(ctx, S, ctypes.c_void_p(y.data_ptr()), ctypes.c_void_p(out.data_ptr()), t0, t1, n,
                            ctypes.c_double(0.002), ctypes.c_double(1.0),
                            ctypes.byref(NewtonOpts(1e-10, 1e-10, 25, 1 / 64)),
                            ctypes.byref(KrylovOpts(1e-8, 1e-300, 30, 300, 1, 1, 0.8, 0, 20, 1, 8, 0.0)),
                            its, kits, status, ft, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0 and list(status) == [0] * S and min(its) >= 5
    assert torch.isfinite(out).all() and out.abs().max() > 0
    lib.pint_destroy(ctx)
