"""CPU: the C-ABI library loads without a GPU and exports every entry point
include/pint_b200.h declares; the product path refuses to run without CUDA
(no CPU fallback)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pint_b200.h")
LIB = os.path.join(ROOT, "paper_1907_01252_b200", "libpint_b200.so")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(pint_\w+)\(", src, flags=re.M)))


def test_header_declarations_listed_in_binding():
    from paper_1907_01252_b200 import _lib
    assert set(declared()) == set(_lib.EXPORTS)


@pytest.mark.skipif(not os.path.exists(LIB), reason="library not built")
def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    for name in declared():
        assert hasattr(lib, name), name
    from paper_1907_01252_b200 import _lib
    _lib.load()  # typed binding succeeds without a GPU


@pytest.mark.skipif(not os.path.exists(LIB), reason="library not built")
def test_parareal_entry_points_validate_arguments_without_gpu():
    from paper_1907_01252_b200 import _lib
    lib = _lib.load()
    assert lib.pint_parareal_precorrect(0, 5, 10, 32, None, None, None, None) == _lib.PINT_INVALID_ARG
    assert lib.pint_parareal_correct_one(5, 10, 8, None, None, None, None, None, 0, 0.0, 1.0, None, None,
                                         None) == _lib.PINT_INVALID_ARG
    assert lib.pint_create(None, 1, 30, None) == _lib.PINT_INVALID_ARG


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    from paper_1907_01252_b200.problem import small_problem
    from paper_1907_01252_b200.propagator import DeviceError, FSIDevice
    with pytest.raises(DeviceError, match="no CPU fallback"):
        FSIDevice(small_problem(8, 2), 1)


def test_missing_library_raises(tmp_path):
    from paper_1907_01252_b200 import _lib
    saved = _lib._lib
    _lib._lib = None
    try:
        with pytest.raises(_lib.LibraryMissing):
            _lib.load(str(tmp_path / "nope.so"))
    finally:
        _lib._lib = saved


def test_krylov_settings_defaults_reach_the_c_struct():
    """Host-side solver settings: omega = 0 selects the library default of the
    smoother (Vanka 0.9 in both dimensions, node-block Jacobi 0.5), an explicit
    omega is passed through, and the C struct carries the reuse period and the
    first-iteration forcing."""
    from paper_1907_01252_b200.propagator import KrylovSettings
    ks = KrylovSettings()
    assert ks.resolved_omega(2) == 0.9 and ks.resolved_omega(3) == 0.9
    assert KrylovSettings(smoother="jacobi").resolved_omega(2) == 0.5
    assert KrylovSettings(omega=0.8).resolved_omega(3) == 0.8
    c = ks.c_struct(2)
    assert c.omega == 0.9 and c.smoother == 1 and c.precond_reuse == 64 and c.restart == 30
    assert abs(c.rtol_first - 3e-5) < 1e-20
    with pytest.raises(ValueError):
        KrylovSettings(omega=1.5)
