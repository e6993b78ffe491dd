/*
 * pint_b200.h -- C ABI of the B200-native batched fine propagator for
 * Parareal ALE fluid-structure interaction (arXiv:1907.01252).
 *
 * The reference (pintbench, pure Python) has no FFI: its plug-in point for
 * this hot path is the duck-typed Propagator protocol
 * `{step, cost_hint, advance(state, t_end)}` (reference
 * pkg/src/pintbench/integrators.py:105-112) implemented by ThetaPropagator
 * (integrators.py:126-166), plus the Parareal correction helpers
 * `parareal_update` / `theta_weight` (parareal.py:154-197) and the correction
 * norm (parareal.py:429-431).  Every entry point below replaces one of those
 * call sites; the Python host layer (paper_1907_01252_b200/propagator.py)
 * binds them with ctypes and keeps the reference's Python API.  See
 * INTEGRATION.md for the binding a maintainer would add to pintbench.
 *
 * Conventions
 *  - plain pointers and sizes; device pointers are CUDA global memory
 *    addresses owned by the caller (PyTorch tensors in this repo);
 *  - a batch of S slices is one contiguous buffer [S][C][np]: C = 2*dim+1
 *    field components (vx, vy[, vz], ux, uy[, uz], p), each padded from
 *    nn nodes to np (pint_sizes) doubles; padding entries must be zero;
 *  - every call is enqueued on `stream` (cudaStream_t, NULL = legacy default);
 *    calls that return host results synchronise that stream;
 *  - return value: PINT_OK or an error code; pint_last_error() explains;
 *  - all arithmetic is fp64 and bitwise deterministic, and a slice's result
 *    does not depend on which other slices share the launch.
 */
#ifndef PINT_B200_H
#define PINT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  PINT_OK = 0,
  PINT_NUMERIC_BREAKDOWN = 1, /* linalg.py:17 NumericBreakdown            */
  PINT_NEWTON_MAX_ITERS = 2,  /* linalg.py:21 MaxItersExceeded            */
  PINT_MESH_DEGENERATE = 3,   /* problems.py:36 MeshDegenerate            */
  PINT_INVALID_ARG = 4,
  PINT_CUDA_ERROR = 5
};

typedef struct pint_ctx pint_ctx;

/* Problem description: the FSIProblem dataclass
 * (paper_1907_01252_b200/problem.py); replaces ProblemSpec
 * (problems.py:136-151) for the FSI path. */
typedef struct pint_problem_desc {
  int32_t dim;          /* 2 or 3 */
  int32_t cells[3];     /* cells per direction (cells[2] ignored in 2-d) */
  double extent[3];
  double bar_lo[3], bar_hi[3];
  double rho_f, nu_f, rho_s, mu_s, lambda_s;
  double u_peak, ramp_time;
  double alpha_p;       /* pressure stabilization: delta = alpha_p / (rho_f (1/tau + U/h + nu_f/h^2)) */
  double stab_k;        /* tau: > 0 explicit time scale, 0 = the advective scale h/U (step independent) */
} pint_problem_desc;

/* NewtonSettings (linalg.py:129-149) minus the FD epsilon (exact Jacobian). */
typedef struct pint_newton_opts {
  double abs_tol, rel_tol;
  int32_t max_iters;
  double damping_min;
} pint_newton_opts;

/* flexible GMRES(restart) preconditioned by a geometric V-cycle. */
typedef struct pint_krylov_opts {
  double rtol, atol;
  int32_t restart, max_iters;
  int32_t pre_smooth, post_smooth;
  double omega;
  int32_t max_levels;    /* 0 = as many as the mesh allows */
  int32_t coarse_sweeps; /* smoothing sweeps when the coarsest level is too big for a dense inverse */
  int32_t smoother;      /* 0 node-block Jacobi, 1 cell-patch Vanka (default) */
  int32_t precond_reuse; /* k >= 1: rebuild a slice's multigrid hierarchy at its first Newton iteration
                            every k steps, or earlier when the slice's first-iteration Krylov count
                            grew past 1.5x (+2) the count right after its last build; 0: every
                            Newton iteration */
  double rtol_first;     /* inexact-Newton forcing of the first Newton iteration of a step (0: use rtol);
                            later iterations use rtol, never below half the Newton target
                            (PINT_FORCING) */
} pint_krylov_opts;

/* ---- lifetime -------------------------------------------------------- */
/* restart <= 31 (the CGS kernel keeps one accumulator per basis vector in registers) */
int pint_create(const pint_problem_desc* desc, int32_t max_slices, int32_t restart, pint_ctx** out);
/* flags: PINT_CTX_MATRIX_FREE -- no block-stencil Jacobian and no multigrid
 * hierarchy are allocated (the c5 roofline sweep at 1e6 cells x 32 / 64
 * slices); residual, J w and the matrix-free linear solve work, every call
 * that needs the Jacobian or the preconditioner returns PINT_INVALID_ARG. */
enum { PINT_CTX_MATRIX_FREE = 1 };
int pint_create_ex(const pint_problem_desc* desc, int32_t max_slices, int32_t restart, int32_t flags,
                   pint_ctx** out);
int pint_destroy(pint_ctx* ctx);
const char* pint_last_error(const pint_ctx* ctx);
/* nn nodes, np padded stride, C dofs/node, number of multigrid levels */
int pint_sizes(const pint_ctx* ctx, int32_t* nn, int32_t* np, int32_t* C, int32_t* levels);
/* 1 when the V-cycle residuals read an fp32 copy of the level-0 operator (allocated at create
 * when it fits next to the workspace; PINT_A32=0 disables it), else 0 */
int pint_level0_fp32(const pint_ctx* ctx, int32_t* enabled);
/* node flags (uint8 per node: 1 solid-touch, 2 fluid-touch, 4 Dirichlet v, 8 Dirichlet u)
 * and cell flags (1 solid, 2 outflow) into host buffers, for cross-checks */
int pint_flags(const pint_ctx* ctx, uint8_t* node_flags, uint8_t* cell_flags);

/* ---- fine propagation: replaces ThetaPropagator.advance, batched --------
 * Advances each slice s from t0[s] to t_end[s] in nsteps[s] shifted-CN
 * steps of size k (the last one absorbs the rounding slack exactly as
 * integrators.py:154-162), theta = 1/2 + theta0*k_step clamped to [1/2, 1]
 * (integrators.py:73), Newton guess = previous state (integrators.py:93).
 * y_in / y_out: device [S][C][np].  Host outputs per slice: Newton
 * iterations, Krylov iterations, status (PINT_*), failing t_n.
 * The whole call is ONE launch of a CUDA graph whose conditional WHILE / IF
 * nodes run the time-step, Newton, line-search and GMRES loops on the device
 * (no host round trip inside the call); PINT_DEVICE_LOOP=0 selects the
 * host-driven loop, which gives the same bits. */
int pint_propagate(pint_ctx* ctx, int32_t S, const double* y_in, double* y_out, const double* t0,
                   const double* t_end, const int32_t* nsteps, double k, double theta0,
                   const pint_newton_opts* newton, const pint_krylov_opts* krylov, int32_t* newton_iters,
                   int32_t* krylov_iters, int32_t* status, double* fail_t, void* stream);

/* ---- kernel-level entry points (parity ladder + c5 roofline sweep) ----
 * Per-slice step data: k[s], theta[s], t1[s] (host arrays).
 * residual: r = R(y; y_old) with Dirichlet/identity rows (integrators.py:83-88
 * analogue); norms (host, may be NULL) = ||r_s||_2, +inf on a degenerate mesh. */
int pint_residual(pint_ctx* ctx, int32_t S, const double* y, const double* y_old, const double* k,
                  const double* theta, const double* t1, double* r, double* norms, void* stream);
/* matrix-free Jacobian-vector product J(y) w */
int pint_jvp(pint_ctx* ctx, int32_t S, const double* y, const double* y_old, const double* w, const double* k,
             const double* theta, const double* t1, double* Jw, void* stream);
/* assemble the block-stencil Jacobian into the context (level 0) */
int pint_assemble(pint_ctx* ctx, int32_t S, const double* y, const double* y_old, const double* k,
                  const double* theta, const double* t1, void* stream);
/* copy the assembled block-stencil Jacobian [S][noff][C][C][np] out (device) */
int pint_jacobian_blocks(pint_ctx* ctx, int32_t S, double* out, void* stream);
/* y = J x with the assembled Jacobian */
int pint_spmv(pint_ctx* ctx, int32_t S, const double* x, double* y, void* stream);
/* multigrid setup on the assembled Jacobian and one V-cycle x = M^{-1} b */
int pint_precond_setup(pint_ctx* ctx, int32_t S, const pint_krylov_opts* krylov, void* stream);
int pint_precond_apply(pint_ctx* ctx, int32_t S, const double* b, double* x, void* stream);
/* GMRES solve J x = b with the current preconditioner; its/resid per slice (host).
 * pint_propagate, pint_linear_solve and pint_coarse_sweep require krylov->restart to
 * equal the context's restart length (PINT_INVALID_ARG otherwise). */
int pint_linear_solve(pint_ctx* ctx, int32_t S, const double* b, double* x, const pint_krylov_opts* krylov,
                      int32_t* its, double* resid, void* stream);

/* matrix-free GMRES solve J(y) x = b (operator by the K2' J w kernel at the
 * linearisation point y / y_old with per-slice step data k, theta, t1; no
 * preconditioner); works on matrix-free and assembled contexts */
int pint_linear_solve_mf(pint_ctx* ctx, int32_t S, const double* y, const double* y_old, const double* k,
                         const double* theta, const double* t1, const double* b, double* x,
                         const pint_krylov_opts* krylov, int32_t* its, double* resid, void* stream);

/* ---- profiling (bench.py) --------------------------------------------
 * enable: resets the counters; 1 = count launches only (CUDA-graph replay
 * stays on), 2 = also bracket every level-0 smoother sweep (the dominant
 * kernel of the fine step) with CUDA events on its stream (graphs off).
 * read: launches issued, profiled-kernel launches, active slice-launches of it,
 * its summed event time (ms) and its algorithmic bytes per slice-launch. */
int pint_profile(pint_ctx* ctx, int32_t enable);
int pint_profile_read(pint_ctx* ctx, int64_t* launches, int64_t* kernel_launches, int64_t* slice_launches,
                      double* kernel_ms, int64_t* bytes_per_slice_launch);
/* name of the kernel the events bracketed (the fused Arnoldi step on small meshes,
 * else the level-0 smoother) */
const char* pint_profile_kernel(const pint_ctx* ctx);

/* ---- Parareal correction (parareal.py:154-197, 422-431) ---------------
 * K8a, batched over S slices: delta = f_old - c_old. */
int pint_parareal_precorrect(int32_t S, int32_t C, int32_t nn, int32_t np, const double* f_old,
                             const double* c_old, double* delta, void* stream);
/* K8b, one slice inside the sequential sweep: theta (host out) =
 * theta_weight(f_old, c_new, variant, clamp) with variant 0 classic,
 * 1 least_squares, 2 angle_penalized; x_new = theta c_new + f_old - theta c_old;
 * corr (host out) = ||x_new - x_prev|| / ||x_new|| (0 if equal, inf if ||x_new|| = 0). */
int pint_parareal_correct_one(int32_t C, int32_t nn, int32_t np, const double* c_new, const double* f_old,
                              const double* c_old, const double* x_prev, double* x_new, int32_t variant,
                              double clamp_lo, double clamp_hi, double* theta_out, double* corr_out,
                              void* stream);

/* ---- the sequential corrector sweep on the device (parareal.py:410-436) --
 * One call runs the whole sweep of one Parareal iteration: for l = 0..L-1
 *   c_new[l] = C(x[l]) over [t_grid[l], t_grid[l+1]] in nsteps[l] coarse steps
 *              of size k (the coarse propagator's ThetaPropagator.advance,
 *              integrators.py:144-166, batch 1);
 *   x[l+1]   = theta_l c_new[l] + f_old[l] - theta_l c_old[l]   (parareal_update,
 *              parareal.py:154-163, theta_l = theta_weight(f_old[l], c_new[l]),
 *              parareal.py:166-197, variant / clamp as pint_parareal_correct_one);
 *   corr[l]  = ||x[l+1] - x_prev[l+1]|| / ||x[l+1]||   (parareal.py:429-431).
 * f_old == NULL runs the coarse initialisation instead (parareal.py:410-416):
 * x[l+1] = c_new[l], theta 1, corr 0.  Device buffers: x, x_prev [L+1][C][np]
 * (x[0] given), c_new, c_old, f_old [L][C][np].  Every propagation is one
 * launch of the context's device-driven loop graph; nothing synchronises the
 * host until the end.  Host outputs per l: theta, corr, Newton / Krylov
 * iterations, status (PINT_*) and failing t_n of the coarse propagation.  A
 * failed slice leaves the later ones undefined; the caller reports the first
 * failing l (parareal.py:437-440). */
int pint_coarse_sweep(pint_ctx* ctx, int32_t L, double* x, const double* x_prev, double* c_new, const double* c_old,
                      const double* f_old, const double* t_grid, const int32_t* nsteps, double k, double theta0,
                      const pint_newton_opts* newton, const pint_krylov_opts* krylov, int32_t variant,
                      double clamp_lo, double clamp_hi, double* theta_out, double* corr_out, int32_t* newton_iters,
                      int32_t* krylov_iters, int32_t* status, double* fail_t, void* stream);

/* boundary_error (parareal.py:200-213) for S slices on the device:
 * err[s] = ||x_s - ref_s|| / ||ref_s||, or the absolute ||x_s - ref_s|| with
 * absolute[s] = 1 when ||ref_s|| = 0 (ErrorEntry, parareal.py:106-111).
 * x, ref: device [S][C][np]; err, absolute: host. */
int pint_boundary_error(pint_ctx* ctx, int32_t S, const double* x, const double* ref, double* err,
                        int32_t* absolute, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PINT_B200_H */
