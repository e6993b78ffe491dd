"""BASELINE config c5: kernel roofline sweep (no time loop).

For 2-d structured meshes of ~1e4 / 1e5 / 1e6 cells and 1..64 batched
slices: one residual (K1), one Jacobian-vector product (K2'), the block-stencil
Jacobian assembly (K2), one SpMV (K3), the multigrid setup and one V-cycle
(K4), and one preconditioned GMRES iteration (K3-K6), each timed with CUDA
events (median of repeats, L2 flushed before every repeat) and converted to
achieved GB/s from its ALGORITHMIC bytes (compulsory traffic).

Inputs (BASELINE c5): v ~ N(0,1), u ~ N(0, 1e-3^2), p ~ N(0,1) i.i.d. per node,
seeded (problem.c5_random_states), c1 materials.

  python tools/c5_sweep.py --sizes 1e4 1e5 1e6 --slices 1 4 16 64 > c5.jsonl
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1907_01252_b200.problem import C5_MESHES, c5_problem, c5_random_states  # noqa: E402
from paper_1907_01252_b200.propagator import FSIDevice, KrylovSettings  # noqa: E402


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def timed(fn, flush, reps=5):
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


def lean_line(P, size, S, a, pk, pk_kind, flush):
    """Matrix-free context (PINT_CTX_MATRIX_FREE: no Jacobian, no hierarchy)
    for the (size, S) whose assembled context exceeds the memory budget: K1,
    K2' and one unpreconditioned matrix-free GMRES(1) iteration."""
    nn, C = P.num_nodes, P.dofs_per_node
    V = C * 8 * nn
    dev = FSIDevice(P, S, restart=1, matrix_free=True)
    Y = c5_random_states(P, S, a.seed)
    Yo = c5_random_states(P, S, a.seed + 1)
    W = c5_random_states(P, S, a.seed + 2)
    y, yo, w = dev.to_device(Y), dev.to_device(Yo), dev.to_device(W)
    del Y, Yo, W
    k, th, t1 = [2.0 ** -10] * S, [0.5 + 2.0 ** -10] * S, [0.3] * S
    r, jw, out = dev.empty(S), dev.empty(S), dev.empty(S)
    krylov = KrylovSettings(rtol=1e-30, max_iters=1, restart=1)
    res = {"residual": (timed(lambda: dev.residual(y, yo, k, th, t1, out=r), flush), 3 * V),
           "jvp": (timed(lambda: dev.jvp(y, yo, w, k, th, t1, out=jw), flush), 4 * V),
           # v0 = b / beta (2V), w = J v0 (4V), <v0, w> (2V), update + norm (3V), x = Z y (2V) + x update (3V),
           # true residual J x (4V) + b - J x (3V), its norm (V): 24V, plus the initial ||b|| (V)
           "gmres_iteration_mf": (timed(lambda: dev.linear_solve_mf(y, yo, k, th, t1, w, krylov, out=out), flush),
                                  25 * V)}
    line = {"config": "c5", "size": size, "mesh": list(C5_MESHES[size]), "slices": S, "dofs_per_slice": P.num_dofs,
            "seed": a.seed, "peak_gbs": pk, "peak_kind": pk_kind, "context": "matrix-free (PINT_CTX_MATRIX_FREE)",
            "kernels": {}}
    for name, (ms, bytes_per_slice) in res.items():
        gbs = S * bytes_per_slice / 1e9 / (ms / 1e3)
        line["kernels"][name] = {"ms": ms, "algorithmic_bytes": S * bytes_per_slice, "GB_s": gbs,
                                 "frac_of_peak": gbs / pk}
    print(json.dumps(line), flush=True)
    del dev
    torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", nargs="+", default=["1e4", "1e5", "1e6"])
    ap.add_argument("--slices", nargs="+", type=int, default=[1, 2, 4, 8, 16, 32, 64])
    ap.add_argument("--seed", type=int, default=2024)
    ap.add_argument("--mem-gb", type=float, default=150.0,
                    help="(size, S) whose assembled context exceeds this run in a matrix-free context")
    a = ap.parse_args()
    pk, pk_kind = peak()
    fp64_tflops = 36.59  # measured DFMA peak on this pool's B200 (tools/fp64_peak.cu, profiles/)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MB > L2
    krylov = KrylovSettings(rtol=1e-30, max_iters=1, restart=1)
    for size in a.sizes:
        P = c5_problem(size)
        nn, C = P.num_nodes, P.dofs_per_node
        ncell = P.num_cells
        V = C * 8 * nn                       # one fp64 state, bytes
        Afull = 9 * C * C * 8 * nn            # level-0 block stencil as stored (what the assembly writes)
        # what a product reads: the deformation rows hold 2 structurally non-zero planes of C (row_couples)
        Ablk = 9 * (C * C - P.dim * (C - 2)) * 8 * nn
        Sblk = 9 * C * C * 4 * nn             # Vanka sweep in block-stencil form (fp32, dense blocks)
        per_slice_gb = (Afull * 1.34 * 1.5 + 1.34 * (ncell * (400 * 4 + 160) + Sblk) + 40 * V) / 1e9
        for S in a.slices:
            if S * per_slice_gb > a.mem_gb:
                lean_line(P, size, S, a, pk, pk_kind, flush)
                continue
            dev = FSIDevice(P, S, restart=1)
            Y = c5_random_states(P, S, a.seed)
            Yo = c5_random_states(P, S, a.seed + 1)
            W = c5_random_states(P, S, a.seed + 2)
            y, yo, w = dev.to_device(Y), dev.to_device(Yo), dev.to_device(W)
            k, th = [2.0 ** -10] * S, [0.5 + 2.0 ** -10] * S
            t1 = [0.3] * S
            r = dev.empty(S)
            jw = dev.empty(S)
            out = dev.empty(S)
            res = {}
            res["residual"] = (timed(lambda: dev.residual(y, yo, k, th, t1, out=r), flush), 3 * V)
            res["jvp"] = (timed(lambda: dev.jvp(y, yo, w, k, th, t1, out=jw), flush), 4 * V)
            res["assembly"] = (timed(lambda: dev.assemble(y, yo, k, th, t1), flush),
                               Afull + (Afull // 2 if dev.level0_fp32 else 0) + 2 * V)
            res["spmv"] = (timed(lambda: dev.spmv(w, out=out), flush), Ablk + 2 * V)
            dev.precond_setup(S, krylov)
            # V(1,1) level-0 traffic: first sweep (inverses + r + y) + residual SpMV + post sweep
            # (SpMV + inverses + gather) + restriction/prolongation; coarse levels add ~1/3
            # (the two V-cycle SpMVs read the fp32 level-0 copy when the context holds one)
            Avc = Ablk // 2 if dev.level0_fp32 else Ablk
            stencil = "stencil" in dev.profile_read()["kernel"]  # round 2: sweeps as one fp32 block-stencil product
            sweep = Sblk + 2 * V if stencil else ncell * (400 * 4 + 160) + V
            lvl0 = sweep * 2 + (Avc + 2 * V) * 2 + 4 * V
            res["vcycle"] = (timed(lambda: dev.precond_apply(w, out=out), flush), int(lvl0 * 4 / 3))
            # one flexible-GMRES(1) solve = Arnoldi step (V-cycle + fp64 SpMV + CGS2/norm on 2 vectors)
            # + x += Z y + the true-residual SpMV (no second V-cycle: z_j is stored)
            res["gmres_iteration"] = (timed(lambda: dev.linear_solve(w, krylov, out=out), flush),
                                      int(lvl0 * 4 / 3) + 2 * (Ablk + 2 * V) + 16 * V)
            line = {"config": "c5", "size": size, "mesh": list(C5_MESHES[size]), "slices": S,
                    "dofs_per_slice": P.num_dofs, "seed": a.seed, "peak_gbs": pk, "peak_kind": pk_kind,
                    "level0_fp32": dev.level0_fp32, "vanka_sweep": "block stencil" if stencil else "cell inverses",
                    "kernels": {}}
            for name, (ms, bytes_per_slice) in res.items():
                gbs = S * bytes_per_slice / 1e9 / (ms / 1e3)
                line["kernels"][name] = {"ms": ms, "algorithmic_bytes": S * bytes_per_slice, "GB_s": gbs,
                                         "frac_of_peak": gbs / pk}
            print(json.dumps(line), flush=True)
            del dev
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
