"""Monolithic ALE fluid-structure problem descriptions (channel + elastic bar).

The reference package only ships 1-d surrogates (problems.py:33); the
north-star physics is the paper's monolithic (v, u, p) ALE system
 discretized in time by the shifted Crank-Nicolson scheme
 with equal-order Q1 elements on structured meshes.  This
module is pure data: the geometry, materials and inflow of BASELINE.json's
configurations c1..c5, the State layout, and the deterministic decisions the
paper leaves open.  Both the CUDA path and the CPU
oracle read the same :class:`FSIProblem`; neither derives anything else from
the other.

Shared decisions (DESIGN.md §2 restates them):

* material: a cell is solid iff its centre lies in the closed bar box;
* unknowns per node: v (d), u (d), p -> d = 5 (2-d) / 7 (3-d); the State
  layout is SoA per component ``{vx, vy[, vz], ux, uy[, uz], p}`` so the
  theta-weights average over components;
* row ownership: v rows = summed momentum of all cells (common test function);
  u rows = solid kinematic row on nodes touching a solid cell, harmonic
  extension on pure-fluid nodes; p rows = divergence +
  pressure stabilization on nodes touching a fluid cell, identity elsewhere;
* Dirichlet: v = inflow * s(t) on x = 0, no-slip on the walls (y = 0, y = H
  and, in 3-d, z = 0, z = H); u = 0 on the whole outer boundary; the outlet
  x = Lx is do-nothing with the paper's boundary correction term;
* inflow ramp s(t) = forcing_s(min(t, 0.5), 0.5) (reference problems.py:214-221);
* pressure stabilization: PSPG-type Brezzi-Pitkaranta term
  k delta (grad p, grad xi) in reference coordinates, delta = alpha_p /
  (rho_f (1/tau + U/h + nu_f/h^2)) with the advective time scale tau = h/U:
  independent of the step, so coarse and fine propagators discretize the
  same spatial problem;
* quadrature: tensor 2-point Gauss per direction, 2-point (2-d) / 2x2 (3-d)
  on the outflow face.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from typing import Dict, Tuple

import numpy as np

Layout = Dict[str, Tuple[int, int]]


@dataclass(frozen=True)
class FSIProblem:
    """Geometry, mesh, materials and inflow of one channel/bar FSI problem."""

    dim: int = 2
    cells: Tuple[int, ...] = (32, 8)
    extent: Tuple[float, ...] = (2.0, 0.5)
    bar_lo: Tuple[float, ...] = (0.8, 0.0)
    bar_hi: Tuple[float, ...] = (1.0, 0.25)
    rho_f: float = 1000.0
    nu_f: float = 1e-3
    rho_s: float = 1000.0
    mu_s: float = 5e5
    nu_s: float = 0.4
    u_peak: float = 1.0
    ramp_time: float = 0.5
    alpha_p: float = 1.0
    stab_k: float = 0.0      # stabilization time scale tau; 0 = the advective scale h / U
    name: str = "custom"

    def __post_init__(self):
        if self.dim not in (2, 3):
            raise ValueError("dim must be 2 or 3")
        for tup in (self.cells, self.extent, self.bar_lo, self.bar_hi):
            if len(tup) != self.dim:
                raise ValueError("cells/extent/bar boxes must have dim entries")
        if min(self.cells) < 1:
            raise ValueError("need at least one cell per direction")
        if min(self.extent) <= 0.0:
            raise ValueError("extent must be positive")
        for name in ("rho_f", "nu_f", "rho_s", "mu_s", "ramp_time", "alpha_p"):
            if getattr(self, name) <= 0.0:
                raise ValueError(f"{name} must be positive")
        if not 0.0 <= self.nu_s < 0.5:
            raise ValueError("Poisson ratio must lie in [0, 0.5)")

    # ---- derived sizes -------------------------------------------------
    @property
    def dofs_per_node(self) -> int:
        return 2 * self.dim + 1

    @property
    def nodes(self) -> Tuple[int, ...]:
        return tuple(c + 1 for c in self.cells)

    @property
    def num_nodes(self) -> int:
        return int(np.prod(self.nodes))

    @property
    def num_cells(self) -> int:
        return int(np.prod(self.cells))

    @property
    def num_dofs(self) -> int:
        return self.dofs_per_node * self.num_nodes

    @property
    def h(self) -> Tuple[float, ...]:
        return tuple(e / c for e, c in zip(self.extent, self.cells))

    @property
    def lambda_s(self) -> float:
        return 2.0 * self.mu_s * self.nu_s / (1.0 - 2.0 * self.nu_s)

    @property
    def h_k(self) -> float:
        """Cell size used by the stabilization: sqrt(mean h_m^2)."""
        return math.sqrt(sum(x * x for x in self.h) / self.dim)

    def delta_p(self, k: float = 0.0) -> float:
        """Pressure-stabilization coefficient delta_K.

        delta = alpha_p / (rho_f (1/tau + U/h + nu_f/h^2)) with tau = stab_k, or the
        advective time scale h/U when stab_k = 0 (default).  Independent of the
        step size k, so the coarse and the fine propagator discretize the SAME
        spatial problem (a k-dependent delta made Parareal stagnate at defects
        ~1 on c1; measured).  ``k`` is accepted for API stability.
        """
        hk = self.h_k
        tau = self.stab_k if self.stab_k > 0.0 else hk / self.u_peak
        return self.alpha_p / (self.rho_f * (1.0 / tau + self.u_peak / hk + self.nu_f / (hk * hk)))

    @property
    def component_names(self) -> Tuple[str, ...]:
        ax = "xyz"[: self.dim]
        return tuple(f"v{a}" for a in ax) + tuple(f"u{a}" for a in ax) + ("p",)

    def layout(self) -> Layout:
        n = self.num_nodes
        return {name: (c * n, n) for c, name in enumerate(self.component_names)}

    def zero_values(self) -> np.ndarray:
        return np.zeros(self.num_dofs)


def ramp(t: float, ramp_time: float = 0.5) -> float:
    """Inflow ramp s(t) = (1 - cos(pi min(t,T)/T)) / 2 (cf. problems.py:214-221)."""
    tt = min(t, ramp_time)
    return 0.5 * (1.0 - math.cos(math.pi * tt / ramp_time))


# --------------------------------------------------------------------------
# BASELINE.json configurations (c2-c4 with binary-fraction steps)


@dataclass(frozen=True)
class RunConfig:
    """One BASELINE configuration: problem + time stepping + Parareal."""

    problem: FSIProblem
    t_end: float
    fine_step: float
    coarse_step: float
    intervals: int
    iterations: int
    theta0: float = 1.0
    note: str = ""

    @property
    def window(self) -> float:
        return self.t_end / self.intervals

    @property
    def fine_steps_per_window(self) -> int:
        return int(round(self.window / self.fine_step))

    @property
    def coarse_steps_per_window(self) -> int:
        return int(round(self.window / self.coarse_step))


def channel_2d(nx: int, ny: int, mu_s: float = 5e5, name: str = "c") -> FSIProblem:
    return FSIProblem(dim=2, cells=(nx, ny), extent=(2.0, 0.5), bar_lo=(0.8, 0.0),
                      bar_hi=(1.0, 0.25), mu_s=mu_s, name=name)


def channel_3d(nx: int, ny: int, nz: int, name: str = "c4") -> FSIProblem:
    return FSIProblem(dim=3, cells=(nx, ny, nz), extent=(2.5, 0.41, 0.41),
                      bar_lo=(0.6, 0.0, 0.1), bar_hi=(0.8, 0.2, 0.31), name=name)


CONFIGS = {
    "c1": RunConfig(channel_2d(32, 8, name="c1"), t_end=1.0, fine_step=0.002, coarse_step=0.02,
                    intervals=10, iterations=5),
    "c2": RunConfig(channel_2d(64, 16, name="c2"), t_end=2.0, fine_step=2.0 ** -10,
                    coarse_step=2.0 ** -6, intervals=32, iterations=8,
                    note="fine 0.001/coarse 0.02 substituted by 2^-10/2^-6 (window 1/16 not divisible)"),
    "c3": RunConfig(channel_2d(256, 64, mu_s=2e6, name="c3"), t_end=2.0, fine_step=2.0 ** -11,
                    coarse_step=2.0 ** -7, intervals=64, iterations=8,
                    note="fine 5e-4/coarse 0.01 substituted by 2^-11/2^-7 (window 1/32 not divisible)"),
    "c4": RunConfig(channel_3d(40, 8, 8), t_end=1.0, fine_step=2.0 ** -9, coarse_step=2.0 ** -6,
                    intervals=16, iterations=8,
                    note="fine 0.002/coarse 0.02 substituted by 2^-9/2^-6 (window 1/16 not divisible)"),
}

# c5: kernel roofline sweep meshes (no time loop)
C5_MESHES = {"1e4": (200, 50), "1e5": (640, 160), "1e6": (2000, 500)}


def c5_problem(size: str) -> FSIProblem:
    nx, ny = C5_MESHES[size]
    return channel_2d(nx, ny, name=f"c5_{size}")


def c5_random_states(problem: FSIProblem, slices: int, seed: int) -> np.ndarray:
    """Seeded c5 inputs: v ~ N(0,1), u ~ N(0,1e-3^2), p ~ N(0,1), slice order."""
    rng = np.random.default_rng(seed)
    d = problem.dim
    n = problem.num_nodes
    out = np.empty((slices, problem.num_dofs))
    for s in range(slices):
        v = rng.standard_normal(d * n)
        u = 1e-3 * rng.standard_normal(d * n)
        p = rng.standard_normal(n)
        out[s] = np.concatenate([v, u, p])
    return out


def small_problem(nx: int = 8, ny: int = 2, **kw) -> FSIProblem:
    """Tiny channel for parity tests (bar still resolved by >= 1 cell)."""
    return replace(channel_2d(nx, ny, name=f"small{nx}x{ny}"), **kw)
