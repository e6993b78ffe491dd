"""Dump one V-cycle, one assembled-operator product and one preconditioned
solve per config to an .npz, for a bitwise comparison between two builds of
the library (PINT_LIB=...): the structural-zero skipping of the product
kernels (-DPINT_PATTERN=0 restores the full loops) must not change a bit.

  python tools/pattern_ab.py out.npz ;  PINT_LIB=alt.so python tools/pattern_ab.py alt.npz
  python tools/pattern_ab.py --compare out.npz alt.npz
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def dump(path):
    from paper_1907_01252_b200.problem import CONFIGS, channel_3d
    from paper_1907_01252_b200.propagator import FSIDevice, KrylovSettings
    out = {}
    for name, P in (("c1", CONFIGS["c1"].problem), ("c2", CONFIGS["c2"].problem),
                    ("small3d", channel_3d(10, 2, 2, name="small3d")), ("c4", CONFIGS["c4"].problem)):
        S = 2
        rng = np.random.default_rng(5)
        n, d, C = P.num_nodes, P.dim, P.dofs_per_node

        def rnd(scale_u):
            y = rng.standard_normal((S, C * n))
            y[:, d * n:2 * d * n] *= scale_u
            return y
        Y, B = rnd(1e-4) * 0.1, rnd(1.0)
        for env in ({}, {"PINT_SPMV32_MIN": "0", "PINT_TAIL_ROWS": "300"}):
            os.environ.update(env)
            dev = FSIDevice(P, max_slices=S)
            for k in env:
                os.environ.pop(k)
            y = dev.to_device(Y)
            dev.assemble(y, y, [0.002] * S, [0.502] * S, [0.3] * S)
            dev.precond_setup(S, KrylovSettings())
            tag = name + ("_wide" if env else "")
            out[tag + "_spmv"] = dev.to_host(dev.spmv(dev.to_device(B)))
            out[tag + "_vcycle"] = dev.to_host(dev.precond_apply(dev.to_device(B)))
            x, its, _ = dev.linear_solve(dev.to_device(B), KrylovSettings(rtol=1e-8))
            out[tag + "_solve"] = dev.to_host(x)
            out[tag + "_its"] = its
    np.savez(path, **out)
    print(path, sorted(out))


def compare(a, b):
    A, B = np.load(a), np.load(b)
    ok = True
    for k in A.files:
        same = bool(np.array_equal(A[k], B[k]))
        ok &= same
        print(k, "bitwise equal" if same else f"DIFFERENT (max abs diff {np.abs(A[k] - B[k]).max():.3e})")
    print("ALL BITWISE EQUAL" if ok else "MISMATCH")
    return 0 if ok else 1


if __name__ == "__main__":
    if sys.argv[1] == "--compare":
        sys.exit(compare(sys.argv[2], sys.argv[3]))
    dump(sys.argv[1])
