"""Per-field relative L2 errors (velocity, deformation, pressure), the
north-star parity measure (BASELINE.json: 'per-slice endpoint velocity,
deformation and pressure to relative L2 error <= 1e-6')."""

import numpy as np


def field_slices(P):
    n = P.num_nodes
    d = P.dim
    return {"v": slice(0, d * n), "u": slice(d * n, 2 * d * n), "p": slice(2 * d * n, (2 * d + 1) * n)}


def field_errors(P, a, b):
    out = {}
    for name, sl in field_slices(P).items():
        ref = b[sl]
        nrm = np.linalg.norm(ref)
        diff = np.linalg.norm(a[sl] - ref)
        out[name] = diff / nrm if nrm > 0 else diff
    return out
