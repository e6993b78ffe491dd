"""GPU theta-scheme propagator for the monolithic ALE-FSI problem.

Python mirror of the reference propagator layer (reference
pkg/src/pintbench/integrators.py): ``ThetaSettings`` (integrators.py:46-67),
the ``Propagator`` protocol (integrators.py:105-112), ``_split_window``
(integrators.py:115-123), ``ThetaPropagator.advance`` (integrators.py:144-166)
and ``make_propagator`` (integrators.py:169-173), with the same names,
argument meaning and error types.  The numerical work runs in the sm_100a
library through the C ABI (include/pint_b200.h); PyTorch only provides device
buffers and the stream.  ``advance_batch`` is the additive batched entry point
(SURVEY.md §8b): all slices of one Parareal iteration in one call.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass, field
from typing import List, Optional, Protocol, Sequence

import numpy as np
import torch

from . import _lib
from .problem import FSIProblem
from .state import State


class NumericBreakdown(ArithmeticError):
    """NaN/Inf contamination or a singular linearization (linalg.py:17)."""


class MaxItersExceeded(RuntimeError):
    """Newton iteration budget exhausted (linalg.py:21)."""


class NonDivisibleWindow(ValueError):
    """Window is not an integer multiple of the step (integrators.py:32)."""


class TimeStepError(RuntimeError):
    """An implicit step failed; message carries (t_n, k) (integrators.py:36)."""


class DeviceError(RuntimeError):
    """The CUDA library reported an error."""


_WINDOW_RTOL = 1e-9


@dataclass(frozen=True)
class NewtonSettings:
    """Newton tolerances and damping (linalg.py:129-149; exact Jacobian, so no fd_epsilon)."""

    abs_tol: float = 1e-10
    rel_tol: float = 0.0
    max_iters: int = 25
    damping_min: float = 1.0 / 64.0

    def __post_init__(self):
        if self.abs_tol <= 0.0:
            raise ValueError("abs_tol must be positive")
        if self.rel_tol < 0.0:
            raise ValueError("rel_tol must be non-negative")
        if self.max_iters < 1:
            raise ValueError("max_iters must be at least 1")
        if not 0.0 < self.damping_min <= 1.0:
            raise ValueError("damping_min must lie in (0, 1]")


@dataclass(frozen=True)
class KrylovSettings:
    """Flexible GMRES(restart) preconditioned by a geometric V-cycle (cell-patch Vanka smoother)."""

    rtol: float = 1e-8
    atol: float = 1e-300
    restart: int = 30
    max_iters: int = 300
    pre_smooth: int = 1
    post_smooth: int = 1
    omega: float = 0.0          # smoother damping; 0 = default (Vanka 0.9, node-block Jacobi 0.5)
    max_levels: int = 0
    coarse_sweeps: int = 20
    smoother: str = "vanka"    # "vanka" (cell patches) or "jacobi" (node blocks, omega ~0.5)
    precond_reuse: int = 64     # rebuild a slice's multigrid hierarchy every k steps, or when its Krylov
                                # count drifts past 1.5x (+2) the post-build count (0: every Newton iteration)
    rtol_first: float = 3e-5    # inexact-Newton forcing of the first Newton iteration (0: rtol)

    def __post_init__(self):
        if not 0.0 < self.rtol < 1.0:
            raise ValueError("rtol must lie in (0, 1)")
        if self.restart < 1 or self.max_iters < 1:
            raise ValueError("restart and max_iters must be positive")
        if self.pre_smooth < 1 or self.post_smooth < 1:
            raise ValueError("need at least one pre- and post-smoothing sweep")
        if not 0.0 <= self.omega <= 1.0:
            raise ValueError("omega must lie in (0, 1] (0 selects the default of the mesh dimension)")
        if self.smoother not in ("vanka", "jacobi"):
            raise ValueError("smoother must be 'vanka' or 'jacobi'")

    def resolved_omega(self, dim: int) -> float:
        """Additive Vanka damping.  0.9 in both dimensions: in 2-d 1.0 is 1-4 %
        faster on the FINE steps of c1/c2/c3 (profiles/r02_omega_2d.jsonl) but
        2-3x slower on the coarse implicit-Euler steps of c3 and 15 % slower on
        its shifted-CN coarse steps, and 5 % slower on c4 -- the robust value
        stays the default; pass omega explicitly to tune one propagator."""
        if self.omega > 0.0:
            return self.omega
        return 0.5 if self.smoother == "jacobi" else 0.9

    def c_struct(self, dim: int = 3) -> _lib.KrylovOpts:
        return _lib.KrylovOpts(self.rtol, self.atol, self.restart, self.max_iters, self.pre_smooth,
                               self.post_smooth, self.resolved_omega(dim), self.max_levels, self.coarse_sweeps,
                               1 if self.smoother == "vanka" else 0, int(self.precond_reuse),
                               float(self.rtol_first))


# one documented setting shared by the GPU path and the CPU oracle
FSI_NEWTON = NewtonSettings(abs_tol=1e-10, rel_tol=1e-10)


@dataclass(frozen=True)
class ThetaSettings:
    """Step size, implicitness shift and Newton settings (integrators.py:46-67)."""

    step: float
    theta0: float = 0.0
    newton: NewtonSettings = field(default_factory=NewtonSettings)

    def __post_init__(self):
        if self.step <= 0.0:
            raise ValueError("step must be positive")
        if not 0.5 - 1e-12 <= self.theta <= 1.0 + 1e-12:
            raise ValueError(f"effective theta {self.theta} outside [1/2, 1]; adjust theta0")

    @property
    def theta(self) -> float:
        return 0.5 + self.theta0 * self.step


class Propagator(Protocol):
    step: float
    cost_hint: float

    def advance(self, state: State, t_end: float) -> State:
        ...


def split_window(window: float, step: float) -> int:
    """Number of internal steps of ``window`` (integrators.py:115-123)."""
    n = max(int(round(window / step)), 1)
    mismatch = abs(window - n * step)
    if mismatch > _WINDOW_RTOL * max(abs(window), step):
        raise NonDivisibleWindow(
            f"window {window!r} is not an integer multiple of step {step!r} (mismatch {mismatch:.3e})")
    return n


# ----------------------------------------------------------------------------
# device context


def _require_cuda():
    if not torch.cuda.is_available():
        raise DeviceError("the FSI propagator needs a CUDA device (no CPU fallback)")


def problem_desc(p: FSIProblem) -> _lib.ProblemDesc:
    d = _lib.ProblemDesc()
    d.dim = p.dim
    for m in range(3):
        d.cells[m] = p.cells[m] if m < p.dim else 1
        d.extent[m] = p.extent[m] if m < p.dim else 1.0
        d.bar_lo[m] = p.bar_lo[m] if m < p.dim else 0.0
        d.bar_hi[m] = p.bar_hi[m] if m < p.dim else 0.0
    d.rho_f, d.nu_f, d.rho_s, d.mu_s = p.rho_f, p.nu_f, p.rho_s, p.mu_s
    d.lambda_s = p.lambda_s
    d.u_peak, d.ramp_time, d.alpha_p, d.stab_k = p.u_peak, p.ramp_time, p.alpha_p, p.stab_k
    return d


def _ptr(t: torch.Tensor) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def _stream() -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _darr(vals) -> ctypes.Array:
    vals = [float(v) for v in vals]
    return (ctypes.c_double * len(vals))(*vals)


class FSIDevice:
    """One device context: mesh tables, multigrid hierarchy and workspace for
    up to ``max_slices`` batched slices.  Calls are serialized by the
    library's context mutex; ctypes releases the GIL during them."""

    def __init__(self, problem: FSIProblem, max_slices: int, restart: int = 30, matrix_free: bool = False):
        _require_cuda()
        self.lib = _lib.load()
        self.problem = problem
        self.max_slices = int(max_slices)
        self.restart = int(restart)
        self.matrix_free = bool(matrix_free)  # no Jacobian / hierarchy: residual, J w, linear_solve_mf only
        handle = ctypes.c_void_p()
        desc = problem_desc(problem)
        rc = self.lib.pint_create_ex(ctypes.byref(desc), self.max_slices, self.restart,
                                     _lib.PINT_CTX_MATRIX_FREE if self.matrix_free else 0, ctypes.byref(handle))
        if rc != _lib.PINT_OK:
            msg = self.lib.pint_last_error(handle).decode() if handle else "allocation failed"
            if handle:
                self.lib.pint_destroy(handle)
            raise DeviceError(f"pint_create failed ({rc}): {msg}")
        self.handle = handle
        nn, np_, C, lv = (ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32())
        self.lib.pint_sizes(handle, ctypes.byref(nn), ctypes.byref(np_), ctypes.byref(C), ctypes.byref(lv))
        self.nn, self.np, self.C, self.levels = nn.value, np_.value, C.value, lv.value
        f32 = ctypes.c_int32()
        self.lib.pint_level0_fp32(handle, ctypes.byref(f32))
        self.level0_fp32 = bool(f32.value)  # V-cycle residuals read the fp32 level-0 copy
        assert self.nn == problem.num_nodes and self.C == problem.dofs_per_node

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                self.lib.pint_destroy(h)
            except Exception:
                pass
            self.handle = None

    # ---- buffers -------------------------------------------------------
    def empty(self, S: int) -> torch.Tensor:
        return torch.zeros((S, self.C, self.np), dtype=torch.float64, device="cuda")

    def to_device(self, values: np.ndarray | Sequence[np.ndarray], out: Optional[torch.Tensor] = None,
                  non_blocking: bool = False) -> torch.Tensor:
        arr = np.asarray(values, dtype=np.float64)
        if arr.ndim == 1:
            arr = arr[None]
        S = arr.shape[0]
        host = torch.from_numpy(np.ascontiguousarray(arr.reshape(S, self.C, self.nn)))
        if non_blocking:
            host = host.pin_memory()
        dev = out if out is not None else self.empty(S)
        dev[:, :, :self.nn].copy_(host, non_blocking=non_blocking)
        return dev

    def to_host(self, dev: torch.Tensor) -> np.ndarray:
        S = dev.shape[0]
        return dev[:, :, :self.nn].cpu().numpy().reshape(S, self.C * self.nn)

    def check(self, rc: int, what: str):
        if rc != _lib.PINT_OK:
            raise DeviceError(f"{what} failed ({_lib.STATUS_NAMES.get(rc, rc)}): "
                              f"{self.lib.pint_last_error(self.handle).decode()}")

    # ---- kernel-level entry points (parity ladder, roofline sweep) -----
    def residual(self, y, y_old, k, theta, t1, out=None):
        S = y.shape[0]
        out = out if out is not None else self.empty(S)
        norms = (ctypes.c_double * S)()
        rc = self.lib.pint_residual(self.handle, S, _ptr(y), _ptr(y_old), _darr(k), _darr(theta), _darr(t1),
                                    _ptr(out), norms, _stream())
        self.check(rc, "pint_residual")
        return out, np.array(norms[:])

    def jvp(self, y, y_old, w, k, theta, t1, out=None):
        S = y.shape[0]
        out = out if out is not None else self.empty(S)
        rc = self.lib.pint_jvp(self.handle, S, _ptr(y), _ptr(y_old), _ptr(w), _darr(k), _darr(theta), _darr(t1),
                               _ptr(out), _stream())
        self.check(rc, "pint_jvp")
        return out

    def assemble(self, y, y_old, k, theta, t1):
        rc = self.lib.pint_assemble(self.handle, y.shape[0], _ptr(y), _ptr(y_old), _darr(k), _darr(theta),
                                    _darr(t1), _stream())
        self.check(rc, "pint_assemble")

    def jacobian_blocks(self, S):
        noff = 9 if self.problem.dim == 2 else 27
        out = torch.empty((S, noff, self.C, self.C, self.np), dtype=torch.float64, device="cuda")
        self.check(self.lib.pint_jacobian_blocks(self.handle, S, _ptr(out), _stream()), "pint_jacobian_blocks")
        return out

    def spmv(self, x, out=None):
        out = out if out is not None else self.empty(x.shape[0])
        self.check(self.lib.pint_spmv(self.handle, x.shape[0], _ptr(x), _ptr(out), _stream()), "pint_spmv")
        return out

    def precond_setup(self, S, krylov: KrylovSettings):
        ko = krylov.c_struct(self.problem.dim)
        self.check(self.lib.pint_precond_setup(self.handle, S, ctypes.byref(ko), _stream()), "pint_precond_setup")

    def precond_apply(self, b, out=None):
        out = out if out is not None else self.empty(b.shape[0])
        self.check(self.lib.pint_precond_apply(self.handle, b.shape[0], _ptr(b), _ptr(out), _stream()),
                   "pint_precond_apply")
        return out

    def linear_solve(self, b, krylov: KrylovSettings, out=None):
        S = b.shape[0]
        out = out if out is not None else self.empty(S)
        ko = krylov.c_struct(self.problem.dim)
        its = (ctypes.c_int32 * S)()
        res = (ctypes.c_double * S)()
        self.check(self.lib.pint_linear_solve(self.handle, S, _ptr(b), _ptr(out), ctypes.byref(ko), its, res,
                                              _stream()), "pint_linear_solve")
        return out, np.array(its[:]), np.array(res[:])

    def linear_solve_mf(self, y, y_old, k, theta, t1, b, krylov: KrylovSettings, out=None):
        """Unpreconditioned GMRES on J(y) x = b with the matrix-free K2' operator."""
        S = b.shape[0]
        out = out if out is not None else self.empty(S)
        ko = krylov.c_struct(self.problem.dim)
        its = (ctypes.c_int32 * S)()
        res = (ctypes.c_double * S)()
        self.check(self.lib.pint_linear_solve_mf(self.handle, S, _ptr(y), _ptr(y_old), _darr(k), _darr(theta),
                                                 _darr(t1), _ptr(b), _ptr(out), ctypes.byref(ko), its, res,
                                                 _stream()), "pint_linear_solve_mf")
        return out, np.array(its[:]), np.array(res[:])

    def profile(self, mode: int):
        """0 off, 1 count launches, 2 count + CUDA-event timing of the level-0 smoother."""
        self.check(self.lib.pint_profile(self.handle, int(mode)), "pint_profile")

    def profile_read(self) -> dict:
        vals = [ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_double(), ctypes.c_int64()]
        self.check(self.lib.pint_profile_read(self.handle, *[ctypes.byref(v) for v in vals]), "pint_profile_read")
        launches, klaunch, slaunch, ms, bpsl = [v.value for v in vals]
        return {"launches": launches, "kernel_launches": klaunch, "slice_launches": slaunch,
                "kernel_ms": ms, "bytes_per_slice_launch": bpsl,
                "kernel": self.lib.pint_profile_kernel(self.handle).decode()}

    def flags(self):
        nf = (ctypes.c_uint8 * self.nn)()
        cf = (ctypes.c_uint8 * self.problem.num_cells)()
        self.lib.pint_flags(self.handle, nf, cf)
        return np.array(nf[:], dtype=np.uint8), np.array(cf[:], dtype=np.uint8)

    def coarse_sweep(self, x: torch.Tensor, t_grid: Sequence[float], nsteps: Sequence[int], k: float,
                     theta0: float, newton: NewtonSettings, krylov: KrylovSettings, c_new: torch.Tensor,
                     x_prev: Optional[torch.Tensor] = None, c_old: Optional[torch.Tensor] = None,
                     f_old: Optional[torch.Tensor] = None, variant: int = 0, clamp=(0.0, 1.0)):
        """The sequential corrector sweep of one Parareal iteration on the device
        (``pint_coarse_sweep``): x[0] given, x[1..L] and c_new[0..L-1] written.
        ``f_old is None`` runs the coarse initialisation.  Returns per-slice
        host arrays (theta, corr, newton its, krylov its, status, fail t)."""
        L = len(nsteps)
        no = _lib.NewtonOpts(newton.abs_tol, newton.rel_tol, newton.max_iters, newton.damping_min)
        ko = krylov.c_struct(self.problem.dim)
        th, cr, ft = (ctypes.c_double * L)(), (ctypes.c_double * L)(), (ctypes.c_double * L)()
        nit, kit, status = (ctypes.c_int32 * L)(), (ctypes.c_int32 * L)(), (ctypes.c_int32 * L)()
        ns = (ctypes.c_int32 * L)(*[int(n) for n in nsteps])
        opt = (lambda t: _ptr(t) if t is not None else None)
        rc = self.lib.pint_coarse_sweep(self.handle, L, _ptr(x), opt(x_prev), _ptr(c_new), opt(c_old), opt(f_old),
                                        _darr(t_grid), ns, float(k), float(theta0), ctypes.byref(no),
                                        ctypes.byref(ko), int(variant), float(clamp[0]), float(clamp[1]), th, cr,
                                        nit, kit, status, ft, _stream())
        self.check(rc, "pint_coarse_sweep")
        return (np.array(th[:]), np.array(cr[:]), np.array(nit[:]), np.array(kit[:]), np.array(status[:]),
                np.array(ft[:]))

    def boundary_error(self, x: torch.Tensor, ref: torch.Tensor):
        """||x_s - ref_s|| / ||ref_s|| per slice on the device (parareal.py:200-213);
        returns (values, absolute flags)."""
        S = x.shape[0]
        err = (ctypes.c_double * S)()
        ab = (ctypes.c_int32 * S)()
        self.check(self.lib.pint_boundary_error(self.handle, S, _ptr(x), _ptr(ref), err, ab, _stream()),
                   "pint_boundary_error")
        return np.array(err[:]), np.array(ab[:], dtype=bool)

    def propagate(self, y_in: torch.Tensor, t0: Sequence[float], t_end: Sequence[float], nsteps: Sequence[int],
                  k: float, theta0: float, newton: NewtonSettings, krylov: KrylovSettings,
                  y_out: Optional[torch.Tensor] = None):
        S = y_in.shape[0]
        y_out = y_out if y_out is not None else self.empty(S)
        no = _lib.NewtonOpts(newton.abs_tol, newton.rel_tol, newton.max_iters, newton.damping_min)
        ko = krylov.c_struct(self.problem.dim)
        nit = (ctypes.c_int32 * S)()
        kit = (ctypes.c_int32 * S)()
        status = (ctypes.c_int32 * S)()
        ft = (ctypes.c_double * S)()
        ns = (ctypes.c_int32 * S)(*[int(n) for n in nsteps])
        rc = self.lib.pint_propagate(self.handle, S, _ptr(y_in), _ptr(y_out), _darr(t0), _darr(t_end), ns,
                                     float(k), float(theta0), ctypes.byref(no), ctypes.byref(ko), nit, kit, status,
                                     ft, _stream())
        self.check(rc, "pint_propagate")
        return y_out, np.array(nit[:]), np.array(kit[:]), np.array(status[:]), np.array(ft[:])


def raise_step_failure(status, fail_t, k: float):
    """Map the first failing slice's status to TimeStepError("implicit step
    failed at t_n=..., k=...") wrapping NumericBreakdown / MaxItersExceeded
    (integrators.py:92-95)."""
    bad = [s for s in range(len(status)) if status[s] != _lib.PINT_OK]
    if not bad:
        return
    s = bad[0]
    cause = (MaxItersExceeded if status[s] == _lib.PINT_NEWTON_MAX_ITERS else NumericBreakdown)(
        _lib.STATUS_NAMES.get(int(status[s]), str(status[s])))
    raise TimeStepError(f"implicit step failed at t_n={float(fail_t[s])!r}, k={k!r}: {cause}") from cause


# ----------------------------------------------------------------------------
# propagator


class GPUThetaPropagator:
    """Shifted-CN propagator of the FSI problem on the B200 (drop-in for the
    reference ``ThetaPropagator``: ``step``, ``cost_hint``, ``advance``).

    ``advance`` composes ``split_window`` steps; the last one absorbs the
    rounding slack so the final time is ``t_end`` exactly; a zero window
    returns the same object; Newton iterations accumulate in
    ``newton_iterations`` under a lock (integrators.py:126-166).
    """

    def __init__(self, problem: FSIProblem, settings: ThetaSettings, cost_hint: float = 0.0,
                 krylov: Optional[KrylovSettings] = None, max_slices: int = 1,
                 device: Optional[FSIDevice] = None):
        self.problem = problem
        self.settings = settings
        self.step = settings.step
        self.cost_hint = cost_hint
        self.krylov = krylov if krylov is not None else KrylovSettings()
        if device is None:
            device = FSIDevice(problem, max_slices, restart=self.krylov.restart)
        if device.problem != problem:
            raise ValueError("device context was built for another problem")
        if device.restart != self.krylov.restart:
            raise ValueError(f"device context has GMRES restart {device.restart}, the Krylov settings ask for "
                             f"{self.krylov.restart}")
        self.device = device
        self.newton_iterations = 0
        self.krylov_iterations = 0
        self.steps_taken = 0
        self._stats_lock = threading.Lock()

    # ---- device-level batched call ----------------------------------
    def advance_device(self, y: torch.Tensor, t0: Sequence[float], t_end: Sequence[float],
                       out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Advance device states y[S, C, np] from t0[s] to t_end[s]."""
        S = y.shape[0]
        if S > self.device.max_slices:
            raise ValueError(f"batch of {S} slices exceeds the context's {self.device.max_slices}")
        nsteps = []
        for a, b in zip(t0, t_end):
            w = b - a
            if w < 0.0:
                raise ValueError(f"cannot advance backwards from {a} to {b}")
            nsteps.append(split_window(w, self.step) if w != 0.0 else 0)
        out, nit, kit, status, ft = self.device.propagate(
            y, t0, t_end, nsteps, self.step, self.settings.theta0, self.settings.newton, self.krylov, y_out=out)
        with self._stats_lock:
            self.newton_iterations += int(nit.sum())
            self.krylov_iterations += int(kit.sum())
            self.steps_taken += int(sum(nsteps))
        raise_step_failure(status, ft, self.step)
        return out

    def sweep(self, x: torch.Tensor, t_grid: Sequence[float], c_new: torch.Tensor, x_prev=None, c_old=None,
              f_old=None, variant: int = 0, clamp=(0.0, 1.0)):
        """Sequential corrector sweep with this (coarse) propagator, on the device
        (FSIDevice.coarse_sweep); returns (theta, corr) per slice and raises
        TimeStepError for the first failing slice (its index in ``.interval``)."""
        L = len(t_grid) - 1
        nsteps = [split_window(t_grid[l + 1] - t_grid[l], self.step) if t_grid[l + 1] != t_grid[l] else 0
                  for l in range(L)]
        th, cr, nit, kit, status, ft = self.device.coarse_sweep(
            x, t_grid, nsteps, self.step, self.settings.theta0, self.settings.newton, self.krylov, c_new,
            x_prev=x_prev, c_old=c_old, f_old=f_old, variant=variant, clamp=clamp)
        bad = [l for l in range(L) if status[l] != _lib.PINT_OK]
        good = slice(0, bad[0]) if bad else slice(0, L)
        with self._stats_lock:
            self.newton_iterations += int(nit[good].sum())
            self.krylov_iterations += int(kit[good].sum())
            self.steps_taken += int(sum(nsteps[:bad[0]] if bad else nsteps))
        if bad:
            try:
                raise_step_failure(status[bad[0]:bad[0] + 1], ft[bad[0]:bad[0] + 1], self.step)
            except TimeStepError as exc:
                exc.interval = bad[0]
                raise
        return th, cr

    # ---- host-State API (reference protocol) ---------------------------
    def advance_batch(self, states: Sequence[State], t_ends: Sequence[float]) -> List[State]:
        if len(states) != len(t_ends):
            raise ValueError("states and t_ends must have equal length")
        results: List[Optional[State]] = [None] * len(states)
        todo = []
        for i, (s, te) in enumerate(zip(states, t_ends)):
            w = te - s.time
            if w == 0.0:
                results[i] = s
            elif w < 0.0:
                raise ValueError(f"cannot advance backwards from {s.time} to {te}")
            else:
                todo.append(i)
        if todo:
            y = self.device.to_device([states[i].values for i in todo])
            out = self.advance_device(y, [states[i].time for i in todo], [t_ends[i] for i in todo])
            vals = self.device.to_host(out)
            for j, i in enumerate(todo):
                results[i] = states[i].with_values(vals[j], time=t_ends[i])
        return results  # type: ignore[return-value]

    def advance(self, state: State, t_end: float) -> State:
        window = t_end - state.time
        if window == 0.0:
            return state
        if window < 0.0:
            raise ValueError(f"cannot advance backwards from {state.time} to {t_end}")
        return self.advance_batch([state], [t_end])[0]


def make_propagator(problem: FSIProblem, settings: ThetaSettings, cost_hint: float = 0.0, **kw) -> GPUThetaPropagator:
    """Build the GPU theta-scheme propagator (integrators.py:169-173)."""
    return GPUThetaPropagator(problem, settings, cost_hint=cost_hint, **kw)


def initial_state(problem: FSIProblem, time: float = 0.0) -> State:
    """Zero initial state (BASELINE: 'zero initial state')."""
    return State(problem.zero_values(), time, problem.layout())
