"""CPU ORACLE (test infrastructure only) -- numpy restatement of the
reference's Parareal correction arithmetic, the checker for the K8 / K9
kernels and the CPU test doubles of the device drivers.

Only ``tests/`` and ``bench.py``'s CPU legs may import this module; the
product path never does.

Restates (reference pkg/src/pintbench/parareal.py):
* ``parareal_update``  parareal.py:154-163 -- theta C_new + F_old - theta C_old,
  evaluated in exactly that order (parareal.py:162);
* ``theta_weight``     parareal.py:166-197 -- classic 1; otherwise per layout
  block cc = <C,C>, cc <= 1e-28 -> 1 (parareal.py:42, 186-188), least squares
  <F,C>/cc, angle-penalized <F,C>/(cc <F,F>) when the denominator exceeds
  1e-56, non-finite -> 1, mean over blocks, clamped;
* ``correction_norm``  parareal.py:429-431 -- 0 if unchanged, else
  ||new - prev|| / ||new|| (inf if ||new|| = 0);
* ``boundary_error``   parareal.py:200-213 -- relative, absolute when the
  reference state is zero (ErrorEntry, parareal.py:106-111).

Pinned: tests/test_oracle_pins.py compares each function with the reference's
own on random inputs (bitwise) when the reference is importable.
"""

from __future__ import annotations

import numpy as np

DEGENERATE = 1e-28  # parareal.py:42


def parareal_update(c_new: np.ndarray, f_old: np.ndarray, c_old: np.ndarray, theta: float) -> np.ndarray:
    return theta * c_new + f_old - theta * c_old


def _weight(f: np.ndarray, c: np.ndarray, variant: str) -> float:
    cc = float(np.dot(c, c))
    if cc <= DEGENERATE:
        return 1.0
    fc = float(np.dot(f, c))
    if variant == "least_squares":
        w = fc / cc
    else:
        denom = cc * float(np.dot(f, f))
        w = fc / denom if denom > DEGENERATE ** 2 else 1.0
    return w if np.isfinite(w) else 1.0


def theta_weight(f: np.ndarray, c: np.ndarray, layout: dict, variant: str, clamp=(0.0, 1.0)) -> float:
    """``layout``: name -> (offset, length) blocks, in layout order."""
    if variant == "classic":
        return 1.0
    if variant not in ("least_squares", "angle_penalized"):
        raise ValueError(f"unknown variant {variant!r}")
    ws = [_weight(f[o:o + n], c[o:o + n], variant) for o, n in layout.values()]
    return float(min(max(sum(ws) / len(ws), clamp[0]), clamp[1]))


def correction_norm(new: np.ndarray, prev: np.ndarray) -> float:
    diff = float(np.linalg.norm(new - prev))
    norm = float(np.linalg.norm(new))
    return 0.0 if diff == 0.0 else (diff / norm if norm > 0.0 else float("inf"))


def boundary_error(x: np.ndarray, ref: np.ndarray):
    """(value, absolute) as ErrorEntry."""
    diff = float(np.linalg.norm(x - ref))
    r = float(np.linalg.norm(ref))
    return (diff / r, False) if r > 0.0 else (diff, True)
