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
