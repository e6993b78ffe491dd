"""Cheap linear theta-scheme propagator for driver tests (host numpy).

y' = A y on a 2-block layout; one step y <- (I - k theta A)^{-1} (I + k (1-theta) A) y,
window split and time bookkeeping as the reference ThetaPropagator.
"""
import numpy as np

from paper_1907_01252_b200.state import State

LAYOUT = {"a": (0, 3), "b": (3, 3)}


def matrix(seed=0, n=6):
    rng = np.random.default_rng(seed)
    M = rng.standard_normal((n, n)) * 0.3
    return M - M.T - np.diag(np.linspace(0.5, 2.0, n))


class LinearPropagator:
    def __init__(self, step, theta0=0.0, A=None, cost_hint=0.0):
        self.step = step
        self.theta0 = theta0
        self.A = matrix() if A is None else A
        self.cost_hint = cost_hint
        self.calls = 0

    def _one(self, y, k):
        th = min(max(0.5 + self.theta0 * k, 0.5), 1.0)
        I = np.eye(self.A.shape[0])
        return np.linalg.solve(I - k * th * self.A, (I + k * (1 - th) * self.A) @ y)

    def advance(self, state, t_end):
        w = t_end - state.time
        if w == 0.0:
            return state
        n = max(int(round(w / self.step)), 1)
        y, t = state.values, state.time
        for _ in range(n - 1):
            y = self._one(y, self.step)
            t = t + self.step
        y = self._one(y, t_end - t)
        self.calls += 1
        return state.with_values(y, time=t_end)


def s0():
    return State(np.array([1.0, -0.5, 0.25, 0.0, 2.0, -1.0]), 0.0, LAYOUT)


# ---- CPU stand-ins for the device drivers' protocol (FSIDevice / GPUThetaPropagator):
# torch CPU tensors [S, 1, n] and the oracle's correction arithmetic, so the
# drivers' host logic (iteration structure, indices, stop rule, sharding,
# trace) is testable without a GPU.

class CPUDevice:
    def __init__(self, n=6, max_slices=64):
        self.n = self.nn = self.np = n
        self.C = 1
        self.max_slices = max_slices

    def empty(self, S):
        import torch
        return torch.zeros((S, 1, self.n), dtype=torch.float64)

    def to_device(self, values):
        import torch
        arr = np.asarray(values, dtype=np.float64)
        arr = arr[None] if arr.ndim == 1 else arr
        return torch.from_numpy(arr.reshape(arr.shape[0], 1, self.n).copy())

    def to_host(self, t):
        return t.reshape(t.shape[0], self.n).numpy().copy()

    def boundary_error(self, x, ref):
        from oracle.parareal_oracle import boundary_error
        e = [boundary_error(a, b) for a, b in zip(self.to_host(x), self.to_host(ref))]
        return np.array([v for v, _ in e]), np.array([a for _, a in e])


class DeviceLinearPropagator(LinearPropagator):
    VARIANTS = ("classic", "least_squares", "angle_penalized")

    def __init__(self, step, theta0=0.0, A=None, device=None, fail_at=None):
        super().__init__(step, theta0, A)
        self.device = device or CPUDevice()
        self.fail_at = fail_at  # (t0) of a window whose propagation raises TimeStepError

    def _adv(self, y, t0, t1):
        if self.fail_at is not None and abs(t0 - self.fail_at) < 1e-12:
            from paper_1907_01252_b200.propagator import TimeStepError
            raise TimeStepError(f"implicit step failed at t_n={t1!r}, k={self.step!r}: injected")
        return self.advance(State(y, t0, LAYOUT), t1).values

    def advance_device(self, Y, t0, t1, out=None):
        vals = [self._adv(y, a, b) for y, a, b in zip(self.device.to_host(Y), t0, t1)]
        res = self.device.to_device(np.array(vals))
        if out is None:
            return res
        out.copy_(res)
        return out

    def sweep(self, X, grid, c_new, x_prev=None, c_old=None, f_old=None, variant=0, clamp=(0.0, 1.0)):
        from oracle.parareal_oracle import correction_norm, parareal_update, theta_weight
        from paper_1907_01252_b200.propagator import TimeStepError
        dv = self.device
        L = len(grid) - 1
        th, cr = np.ones(L), np.zeros(L)
        for l in range(L):
            try:
                cn = self._adv(dv.to_host(X[l:l + 1])[0], grid[l], grid[l + 1])
            except TimeStepError as exc:
                exc.interval = l
                raise
            c_new[l:l + 1].copy_(dv.to_device(cn))
            if f_old is None:
                X[l + 1:l + 2].copy_(dv.to_device(cn))
                continue
            f = dv.to_host(f_old[l:l + 1])[0]
            th[l] = theta_weight(f, cn, LAYOUT, self.VARIANTS[variant], clamp)
            new = parareal_update(cn, f, dv.to_host(c_old[l:l + 1])[0], th[l])
            X[l + 1:l + 2].copy_(dv.to_device(new))
            cr[l] = correction_norm(new, dv.to_host(x_prev[l + 1:l + 2])[0])
        return th, cr
