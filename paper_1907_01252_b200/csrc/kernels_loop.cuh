// Device-side control flow of the fine propagation: the per-slice decisions
// of the time-step loop, the Newton iteration with its halving line search,
// the multigrid rebuild rule and the restarted-GMRES cycles, written as tiny
// single-CTA "controller" kernels that update per-slice state in HBM and set
// the CUDA-graph conditional handles of the WHILE / IF nodes that drive the
// loop (pint_capi.cu: Impl::capture_propagate).  With them one
// pint_propagate is ONE graph launch and no host round trip.
//
// Every decision restates the host-driven path of pint_capi.cu line for line
// (Impl::propagate / newton_step / gmres), which in turn mirrors the
// reference control flow:
//   ThetaPropagator.advance time bookkeeping   integrators.py:144-166
//   _theta_step (guess = previous state)       integrators.py:70-96
//   newton_solve target / line search / accept linalg.py:207-248
// so both paths produce the same bits (tests/test_gpu_device_loop.py).
#pragma once

#include "kernels_linalg.cuh"

namespace pint {

// scalars of one propagate call (host-written before the launch) and the
// loop counters (device-written)
struct LoopScalars {
  int S, nmax, m;               // batch, time steps of the longest slice, GMRES restart length
  int newton_max, lin_max;      // Newton / Krylov iteration budgets
  int reuse, drift_num;         // multigrid rebuild rule (pint_krylov_opts.precond_reuse, PINT_DRIFT)
  int cgs_force;                // 0: Gram-Schmidt passes by tolerance, 1 / 2 forced
  double abs_tol, rel_tol, damping_min;
  double lin_rtol, lin_rtol_first, lin_atol;
  double forcing;               // later Newton iterations solve to max(lin_atol, forcing * target) (0.1; PINT_FORCING)
  const StepScalars* sts;       // [nmax][S] step scalars (host-computed: same arithmetic as the host path)
  const double* t1tab;          // [nmax][S] step end times
  const int* nsteps;            // [S]
  int step, it;                 // time step, Newton iteration (device-written)
};

// per-slice state arrays (fixed device addresses, [maxS] each)
struct LoopDev {
  LoopScalars* ls;
  int *act, *status, *nit, *kit, *running, *its, *ls_mask, *accept, *ok;
  int *built, *base, *first, *need, *built_now, *gits;
  double *ft, *rnorm, *target, *tnorm, *lam, *gres;
  // GMRES / shared workspace of the context
  double *gm_tol, *gm_beta, *gv, *norms;
  int *gm_active, *gm_steps, *gm_its, *cyc_active, *gm_two_pass, *gm_cap;
  StepScalars* st;
  // launch accounting: a controller that enters a conditional body adds the
  // body's kernel-node count (body_nodes[idx], recorded at capture)
  unsigned long long* launch_ctr;
  const int* body_nodes;
};

constexpr int kLoopThreads = 128;

__device__ __forceinline__ void set_cond(const LoopDev& d, cudaGraphConditionalHandle h, int idx, bool v) {
  if (threadIdx.x != 0) return;
  if (v) atomicAdd(d.launch_ctr, (unsigned long long)d.body_nodes[idx]);
  cudaGraphSetConditional(h, v ? 1u : 0u);
}

__device__ __forceinline__ double inf_d() { return __longlong_as_double(0x7ff0000000000000LL); }

// ---- propagate (integrators.py:144-166 bookkeeping)
__global__ void __launch_bounds__(kLoopThreads) k_loop_init(LoopDev d, cudaGraphConditionalHandle h_step, int i_h_step) {
  pdl_wait();
  const LoopScalars* ls = d.ls;
  for (int s = threadIdx.x; s < ls->S; s += blockDim.x) {
    d.status[s] = 0;
    d.nit[s] = 0;
    d.kit[s] = 0;
    d.ft[s] = 0.0;
    d.built[s] = -1;  // no multigrid build yet in this call
    d.base[s] = -1;
    d.first[s] = 0;
  }
  const bool go = ls->nmax > 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    d.ls->step = 0;
    d.ls->it = 0;
    *d.gm_cap = ls->lin_max;
  }
  set_cond(d, h_step, i_h_step, go);
}

__global__ void __launch_bounds__(kLoopThreads) k_step_begin(LoopDev d) {
  pdl_wait();
  const LoopScalars* ls = d.ls;
  const int S = ls->S, step = ls->step;
  for (int s = threadIdx.x; s < S; s += blockDim.x) {
    const bool a = step < ls->nsteps[s] && d.status[s] == 0;
    d.act[s] = a;
    if (a) d.st[s] = ls->sts[(size_t)step * S + s];
  }
}

// ---- Newton (linalg.py:207-219): r0 norm -> target, running
__global__ void __launch_bounds__(kLoopThreads) k_newton_init(LoopDev d, cudaGraphConditionalHandle h_newton, int i_h_newton) {
  pdl_wait();
  const LoopScalars* ls = d.ls;
  int any = 0;
  for (int s = threadIdx.x; s < ls->S; s += blockDim.x) {
    d.running[s] = 0;
    d.its[s] = 0;
    if (!d.act[s]) continue;
    const double rn = d.norms[s];
    d.rnorm[s] = rn;
    if (!isfinite(rn)) {
      d.status[s] = 1;  // PINT_NUMERIC_BREAKDOWN
      continue;
    }
    d.target[s] = ls->abs_tol + ls->rel_tol * rn;
    const int run = rn > d.target[s];
    d.running[s] = run;
    any |= run;
  }
  any = __syncthreads_or(any);
  if (threadIdx.x == 0) d.ls->it = 0;
  set_cond(d, h_newton, i_h_newton, any && ls->newton_max > 0);
}

// multigrid rebuild rule (pint_capi.cu newton_step): per slice from its own counts
__global__ void __launch_bounds__(kLoopThreads) k_precond_decide(LoopDev d, cudaGraphConditionalHandle h_prec, int i_h_prec) {
  pdl_wait();
  const LoopScalars* ls = d.ls;
  const int it = ls->it, step = ls->step;
  int any = 0;
  for (int s = threadIdx.x; s < ls->S; s += blockDim.x) {
    d.built_now[s] = 0;
    d.need[s] = 0;
    if (!d.running[s]) continue;
    const int last = d.built[s];
    const bool drift = ls->drift_num > 0 && d.base[s] >= 0 && 2 * d.first[s] > ls->drift_num * d.base[s] + 4;
    const bool need = ls->reuse <= 0 || last < 0 || (it == 0 && (step - last >= ls->reuse || drift));
    if (need) {
      d.need[s] = 1;
      d.built[s] = step;
      d.built_now[s] = it == 0;
      any = 1;
    }
  }
  any = __syncthreads_or(any);
  set_cond(d, h_prec, i_h_prec, any);
}

// ---- GMRES: cycle start (host gmres(): cyc mask, g = beta e_1, beta)
__device__ __forceinline__ int cycle_begin(const LoopDev& d, int s, int m, int lin_max) {
  const double res = d.gres[s];
  const int c = d.running[s] && res > d.gm_tol[s] && d.gits[s] < lin_max && isfinite(res);
  d.cyc_active[s] = c;
  d.gm_active[s] = c;
  d.gm_steps[s] = 0;
  double* g = d.gv + (size_t)s * (m + 1);
  g[0] = res;
  for (int i = 1; i <= m; ++i) g[i] = 0.0;
  d.gm_beta[s] = res;
  return c;
}

// The cycles of one solve run in one of two WHILE loops: one-pass
// Gram-Schmidt bodies when no running slice wants a second pass, two-pass
// bodies (pass-2 kernels masked per slice) otherwise; the choice is fixed per
// solve, so the other loop is never entered.
__device__ __forceinline__ void set_cycle(const LoopDev& d, int any, int two, cudaGraphConditionalHandle h1,
                                          int i1, cudaGraphConditionalHandle h2, int i2) {
  any = __syncthreads_or(any);
  two = __syncthreads_or(two);
  set_cond(d, h1, i1, any && !two);
  set_cond(d, h2, i2, any && two);
}

// tolerances and Gram-Schmidt passes per slice, then the first cycle
__global__ void __launch_bounds__(kLoopThreads) k_gmres_init(LoopDev d, cudaGraphConditionalHandle h1, int i1,
                                                             cudaGraphConditionalHandle h2, int i2) {
  pdl_wait();
  const LoopScalars* ls = d.ls;
  int any = 0, two = 0;
  for (int s = threadIdx.x; s < ls->S; s += blockDim.x) {
    // inexact-Newton forcing: first Newton iteration of the step at rtol_first
    const double rt = (d.its[s] == 0 && ls->lin_rtol_first > 0.0) ? fmax(ls->lin_rtol, ls->lin_rtol_first) : ls->lin_rtol;
    const double at = fmax(ls->lin_atol, ls->forcing * d.target[s]);
    const double beta = d.running[s] ? d.rnorm[s] : 0.0;  // ||b|| = ||-r|| = ||r||, bitwise
    const double tol = fmax(rt * beta, at);
    d.gm_tol[s] = tol;
    const int tp = ls->cgs_force ? (ls->cgs_force == 2) : (tol < 1e-7 * beta);
    d.gm_two_pass[s] = tp;
    d.gres[s] = beta;
    d.gits[s] = 0;
    d.gm_its[s] = 0;
    const int c = cycle_begin(d, s, ls->m, ls->lin_max);
    any |= c;
    two |= c && tp;
  }
  set_cycle(d, any, two, h1, i1, h2, i2);
}

// cycle end: true residual norm and iteration count, then the next cycle
__global__ void __launch_bounds__(kLoopThreads) k_cycle_end(LoopDev d, cudaGraphConditionalHandle h1, int i1,
                                                            cudaGraphConditionalHandle h2, int i2) {
  pdl_wait();
  const LoopScalars* ls = d.ls;
  int any = 0, two = 0;
  for (int s = threadIdx.x; s < ls->S; s += blockDim.x) {
    if (d.cyc_active[s]) {
      d.gres[s] = d.norms[s];
      d.gits[s] = d.gm_its[s];
    }
    const int c = cycle_begin(d, s, ls->m, ls->lin_max);
    any |= c;
    two |= c && d.gm_two_pass[s];
  }
  set_cycle(d, any, two, h1, i1, h2, i2);
}

// before a block of Arnoldi steps: any slice still iterating?
__global__ void __launch_bounds__(kLoopThreads) k_arnoldi_gate(LoopDev d, cudaGraphConditionalHandle h_step,
                                                               int i_h_step) {
  pdl_wait();
  const int S = d.ls->S;
  int any = 0;
  for (int s = threadIdx.x; s < S; s += blockDim.x) any |= d.gm_active[s];
  any = __syncthreads_or(any);
  set_cond(d, h_step, i_h_step, any);
}

// after the solve: Krylov counts (multigrid drift rule), then the line search
// (linalg.py:226-239) starts at lambda = 1 for every running slice
__global__ void __launch_bounds__(kLoopThreads) k_gmres_end(LoopDev d) {
  pdl_wait();
  const LoopScalars* ls = d.ls;
  for (int s = threadIdx.x; s < ls->S; s += blockDim.x) {
    d.lam[s] = 1.0;
    d.ls_mask[s] = d.running[s];
    if (!d.running[s]) continue;
    d.kit[s] += d.gits[s];
    if (ls->it == 0) {
      d.first[s] = d.gits[s];
      if (d.built_now[s]) d.base[s] = d.gits[s];
    }
  }
}

__global__ void __launch_bounds__(kLoopThreads) k_ls_update(LoopDev d, cudaGraphConditionalHandle h_ls, int i_h_ls) {
  pdl_wait();
  const LoopScalars* ls = d.ls;
  int any = 0;
  for (int s = threadIdx.x; s < ls->S; s += blockDim.x) {
    if (!d.ls_mask[s]) continue;
    const double tn = d.norms[s];
    const double t = isfinite(tn) ? tn : inf_d();
    d.tnorm[s] = t;
    if (t < d.rnorm[s] || d.lam[s] <= ls->damping_min) {
      d.ls_mask[s] = 0;
    } else {
      d.lam[s] = fmax(d.lam[s] / 2.0, ls->damping_min);
      any = 1;
    }
  }
  any = __syncthreads_or(any);
  set_cond(d, h_ls, i_h_ls, any);
}

// accept the trial (linalg.py:238-240; the copies of y and r were made by
// k_accept_copy from the same mask): non-finite -> breakdown
__global__ void __launch_bounds__(kLoopThreads) k_newton_update(LoopDev d, cudaGraphConditionalHandle h_newton, int i_h_newton) {
  pdl_wait();
  LoopScalars* ls = d.ls;
  int any = 0;
  for (int s = threadIdx.x; s < ls->S; s += blockDim.x) {
    if (!d.running[s]) continue;
    if (!isfinite(d.tnorm[s])) {
      d.status[s] = 1;
      d.running[s] = 0;
      continue;
    }
    d.rnorm[s] = d.tnorm[s];
    d.its[s] += 1;
    d.running[s] = d.rnorm[s] > d.target[s];
    any |= d.running[s];
  }
  any = __syncthreads_or(any);
  const int it = ls->it + 1;
  __syncthreads();
  if (threadIdx.x == 0) ls->it = it;
  set_cond(d, h_newton, i_h_newton, any && it < ls->newton_max);
}

// GMRES start vectors for the running slices: b = -r, x = 0, u = b (cycle-start residual)
__global__ void k_gmres_prep(double* __restrict__ b, double* __restrict__ x, double* __restrict__ u,
                             const double* __restrict__ r, size_t per_slice, const int* __restrict__ running) {
  pdl_wait();
  const int s = blockIdx.y;
  if (!running[s]) return;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < per_slice; i += (size_t)gridDim.x * blockDim.x) {
    const size_t e = s * per_slice + i;
    const double v = -r[e];
    b[e] = v;
    u[e] = v;
    x[e] = 0.0;
  }
}

// u = b - u (matrix-free true residual: u held J x)
__global__ void k_bsub(double* __restrict__ u, const double* __restrict__ b, size_t per_slice,
                       const int* __restrict__ active) {
  pdl_wait();
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < per_slice; i += (size_t)gridDim.x * blockDim.x)
    u[s * per_slice + i] = b[s * per_slice + i] - u[s * per_slice + i];
}

// y = y_trial, r = r_trial on the slices whose trial is accepted (running, finite norm)
__global__ void k_accept_copy(double* __restrict__ y, const double* __restrict__ yt, double* __restrict__ r,
                              const double* __restrict__ rt, size_t per_slice, const int* __restrict__ running,
                              const double* __restrict__ tnorm) {
  pdl_wait();
  const int s = blockIdx.y;
  if (!running[s] || !isfinite(tnorm[s])) return;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < per_slice; i += (size_t)gridDim.x * blockDim.x) {
    const size_t e = s * per_slice + i;
    y[e] = yt[e];
    r[e] = rt[e];
  }
}

// after the Newton loop (linalg.py:244-248) and the step (integrators.py:157-162)
__global__ void __launch_bounds__(kLoopThreads) k_step_end(LoopDev d, cudaGraphConditionalHandle h_step, int i_h_step) {
  pdl_wait();
  LoopScalars* ls = d.ls;
  const int S = ls->S, step = ls->step;
  for (int s = threadIdx.x; s < S; s += blockDim.x) {
    d.ok[s] = 0;
    if (!d.act[s]) continue;
    if (d.status[s] == 0) {
      d.nit[s] += d.its[s];
      if (d.rnorm[s] > d.target[s]) d.status[s] = 2;  // PINT_NEWTON_MAX_ITERS
    }
    if (d.status[s] != 0) d.ft[s] = ls->t1tab[(size_t)step * S + s];
    else d.ok[s] = 1;
  }
  __syncthreads();
  if (threadIdx.x == 0) ls->step = step + 1;
  set_cond(d, h_step, i_h_step, step + 1 < ls->nmax);
}

// coarse sweep: record slice l's outcome of the S = 1 propagation
__global__ void k_sweep_record(LoopDev d, int l, int* __restrict__ status, int* __restrict__ nit,
                               int* __restrict__ kit, double* __restrict__ ft) {
  pdl_wait();
  if (threadIdx.x != 0) return;
  status[l] = d.status[0];
  nit[l] = d.nit[0];
  kit[l] = d.kit[0];
  ft[l] = d.ft[0];
}

// relative boundary error ||x - ref|| / ||ref|| per slice (parareal.py:200-213),
// absolute when ||ref|| = 0: partials over fixed chunks, grid (nblk, S)
__global__ void __launch_bounds__(kRedThreads) k_err_partial(const double* __restrict__ x, const double* __restrict__ ref,
                                                            size_t per_slice, double* __restrict__ part, int nblk) {
  pdl_wait();
  __shared__ double sh[kRedThreads / 32];
  const int s = blockIdx.y;
  const size_t base = (size_t)blockIdx.x * kRedChunk;
  const double* xs = x + s * per_slice;
  const double* rs = ref + s * per_slice;
  double dd = 0.0, rr = 0.0;
  for (int i = threadIdx.x; i < kRedChunk; i += kRedThreads) {
    const size_t e = base + i;
    if (e < per_slice) {
      const double df = xs[e] - rs[e];
      dd += df * df;
      rr += rs[e] * rs[e];
    }
  }
  dd = block_sum(dd, sh);
  rr = block_sum(rr, sh);
  if (threadIdx.x == 0) {
    part[((size_t)s * 2 + 0) * nblk + blockIdx.x] = dd;
    part[((size_t)s * 2 + 1) * nblk + blockIdx.x] = rr;
  }
}

__global__ void k_err_final(const double* __restrict__ part, int nblk, int S, double* __restrict__ err,
                            int* __restrict__ absolute) {
  pdl_wait();
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  double dd = 0.0, rr = 0.0;
  for (int b = 0; b < nblk; ++b) {
    dd += part[((size_t)s * 2 + 0) * nblk + b];
    rr += part[((size_t)s * 2 + 1) * nblk + b];
  }
  const double diff = sqrt(dd), ref = sqrt(rr);
  err[s] = ref > 0.0 ? diff / ref : diff;
  absolute[s] = ref > 0.0 ? 0 : 1;
}

}  // namespace pint
