// K3 block-stencil SpMV, K4 geometric-multigrid preconditioner (Galerkin RAP,
// node-block Jacobi smoother, dense coarsest solve), K5 deterministic
// per-slice reductions and K6 Krylov vector updates.  All kernels are batched
// over slices (grid.y) and honour a per-slice active mask so diverging Newton /
// Krylov iteration counts never change a slice's arithmetic (batch
// invariance, SURVEY.md §8b Determinism row).
#pragma once

#include <cooperative_groups.h>
#include <type_traits>

#include "pint_common.cuh"

namespace cg = cooperative_groups;

namespace pint {

constexpr int kRedThreads = 256;
constexpr int kRedChunk = 1024;  // elements per reduction block (fixed => batch invariant)

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// this thread's share of a chunk dot product: all element loads issued before
// the first FMA (a rolled loop waits one memory round trip per element), the
// products accumulated in element order
__device__ __forceinline__ double chunk_dot(const double* __restrict__ x, const double* __restrict__ y, size_t base,
                                            size_t per_slice) {
  constexpr int PT = kRedChunk / kRedThreads;
  double a[PT], b[PT];
#pragma unroll
  for (int t = 0; t < PT; ++t) {
    const size_t e = base + threadIdx.x + t * kRedThreads;
    a[t] = e < per_slice ? x[e] : 0.0;
    b[t] = e < per_slice ? y[e] : 0.0;
  }
  double acc = 0.0;
#pragma unroll
  for (int t = 0; t < PT; ++t)
    if (base + threadIdx.x + t * kRedThreads < per_slice) acc = fma(a[t], b[t], acc);
  return acc;
}

// fixed-order block reduction; result valid in thread 0
__device__ __forceinline__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double out = 0.0;
  if (threadIdx.x == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    for (int w = 0; w < nw; ++w) out += sh[w];
  }
  __syncthreads();
  return out;
}

// sum of n doubles in index order (the serial tail of the reduction kernels).
// Batching the loads sixteen at a time, and the Givens coefficients eight at
// a time, measured SLOWER on every config (c2 8 195 vs 8 453, c3 924 vs 937
// together with the re-balanced residual warps): kept rolled.
__device__ __forceinline__ double ordered_sum(const double* __restrict__ p, int n) {
  double t = 0.0;
  for (int b = 0; b < n; ++b) t += __ldcg(p + b);
  return t;
}

// Neighbour node of every stencil offset; offsets that leave the grid are
// clamped to the node itself.  Their coefficients are exactly zero (assembly,
// fix-up and RAP never write a non-zero there), so the products vanish and
// every load of a sweep is issued without a data-dependent branch.
template <int D>
__device__ __forceinline__ void stencil_neighbours(const Grid& g, int n, int (&nbs)[D == 2 ? 9 : 27]) {
  int i, j, k;
  node_coords(g, n, i, j, k);
#pragma unroll
  for (int off = 0; off < (D == 2 ? 9 : 27); ++off) {
    int di, dj, dk;
    offset_delta(off, D, di, dj, dk);
    const int a = i + di, b = j + dj, c = k + dk;
    const bool ok = a >= 0 && a < g.n[0] && b >= 0 && b < g.n[1] && c >= 0 && c < g.n[2];
    nbs[off] = ok ? node_index(g, a, b, c) : n;
  }
}

// Read-only global load the compiler may not sink below the FMAs that use it:
// volatile asm keeps the program order of the loads, so a stencil row issues
// all its loads back to back (2C per offset) before the first FMA stalls.
__device__ __forceinline__ double ld_nc(const double* p) {
  double v;
  asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ float ld_nc(const float* p) {
  float v;
  asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}

// One block-stencil row: sum_off sum_cb A[off][ca][cb][n] x[cb][nb(off)].
// Latency-bound at the small configs (c1/c2 operators are L2-resident), so
// all 2*C*NOFF loads of the row are put in flight before any FMA.
template <int D, int BATCH, typename MT = double>
__device__ __forceinline__ double stencil_row(const MT* __restrict__ Arow, const double* __restrict__ xs, int np,
                                              const int (&nbs)[D == 2 ? 9 : 27], int ca) {
  constexpr int C = 2 * D + 1;
  constexpr int NOFF = D == 2 ? 9 : 27;
  double part[3] = {0.0, 0.0, 0.0};
  if (is_urow(ca, D)) {
    // deformation row: only the v_i and u_i planes are structurally non-zero (row_couples)
    const int c0 = ca - D, c1 = ca;
#pragma unroll
    for (int o0 = 0; o0 < NOFF; o0 += BATCH) {
      MT a[BATCH][2];
      double xv[BATCH][2];
#pragma unroll
      for (int q = 0; q < BATCH; ++q) {
        a[q][0] = ld_nc(Arow + ((size_t)(o0 + q) * C * C + c0) * np);
        xv[q][0] = ld_nc(xs + c0 * np + nbs[o0 + q]);
        a[q][1] = ld_nc(Arow + ((size_t)(o0 + q) * C * C + c1) * np);
        xv[q][1] = ld_nc(xs + c1 * np + nbs[o0 + q]);
      }
#pragma unroll
      for (int q = 0; q < BATCH; ++q) {
        part[q % 3] = fma((double)a[q][0], xv[q][0], part[q % 3]);
        part[q % 3] = fma((double)a[q][1], xv[q][1], part[q % 3]);
      }
    }
    return (part[0] + part[1]) + part[2];
  }
#pragma unroll
  for (int o0 = 0; o0 < NOFF; o0 += BATCH) {
    MT a[BATCH][C];
    double xv[BATCH][C];
#pragma unroll
    for (int q = 0; q < BATCH; ++q)
#pragma unroll
      for (int cb = 0; cb < C; ++cb) {
        a[q][cb] = ld_nc(Arow + ((size_t)(o0 + q) * C * C + cb) * np);
        xv[q][cb] = ld_nc(xs + cb * np + nbs[o0 + q]);
      }
#pragma unroll
    for (int q = 0; q < BATCH; ++q)
#pragma unroll
      for (int cb = 0; cb < C; ++cb) part[q % 3] = fma((double)a[q][cb], xv[q][cb], part[q % 3]);
  }
  return (part[0] + part[1]) + part[2];
}

// fp32 copy of a block-stencil operator (preconditioner-side residuals only)
__global__ void k_to_f32(const double* __restrict__ A, float* __restrict__ A32, size_t per_slice,
                         const int* __restrict__ active) {
  pdl_wait();
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  const double2* src = reinterpret_cast<const double2*>(A + s * per_slice);
  float2* dst = reinterpret_cast<float2*>(A32 + s * per_slice);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < per_slice / 2; i += (size_t)gridDim.x * blockDim.x) {
    const double2 v = __ldcs(src + i);
    dst[i] = make_float2((float)v.x, (float)v.y);
  }
}

// ---------------------------------------------------------------- generic vector kernels
__global__ void k_zero_active(double* __restrict__ x, size_t per_slice, const int* __restrict__ active) {
  pdl_wait();
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  double* xs = x + s * per_slice;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < per_slice; i += (size_t)gridDim.x * blockDim.x)
    xs[i] = 0.0;
}

__global__ void k_copy_active(double* __restrict__ dst, const double* __restrict__ src, size_t per_slice,
                              const int* __restrict__ active) {
  pdl_wait();
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < per_slice; i += (size_t)gridDim.x * blockDim.x)
    dst[s * per_slice + i] = src[s * per_slice + i];
}

// y = a_s * x + y  (a per slice)
__global__ void k_axpy_slice(double* __restrict__ y, const double* __restrict__ x, const double* __restrict__ a,
                             double sign, size_t per_slice, const int* __restrict__ active) {
  pdl_wait();
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  const double al = sign * a[s];
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < per_slice; i += (size_t)gridDim.x * blockDim.x)
    y[s * per_slice + i] += al * x[s * per_slice + i];
}

// out = x + lam_s * d
__global__ void k_trial(double* __restrict__ out, const double* __restrict__ x, const double* __restrict__ d,
                        const double* __restrict__ lam, size_t per_slice, const int* __restrict__ active) {
  pdl_wait();
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  const double l = lam[s];
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < per_slice; i += (size_t)gridDim.x * blockDim.x)
    out[s * per_slice + i] = x[s * per_slice + i] + l * d[s * per_slice + i];
}

// out = -x
__global__ void k_negate(double* __restrict__ out, const double* __restrict__ x, size_t per_slice,
                         const int* __restrict__ active) {
  pdl_wait();
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < per_slice; i += (size_t)gridDim.x * blockDim.x)
    out[s * per_slice + i] = -x[s * per_slice + i];
}

// out = x / a_s  (a_s == 0 -> out = 0)
__global__ void k_scale_inv(double* __restrict__ out, const double* __restrict__ x, const double* __restrict__ a,
                            size_t per_slice, const int* __restrict__ active) {
  pdl_wait();
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  const double al = a[s];
  const double inv = al != 0.0 ? 1.0 / al : 0.0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < per_slice; i += (size_t)gridDim.x * blockDim.x)
    out[s * per_slice + i] = x[s * per_slice + i] * inv;
}

// ---------------------------------------------------------------- K5 reductions
// partial[s][blk] = sum over the block's chunk of x*y (x == y for norms)
__global__ void __launch_bounds__(kRedThreads) k_dot_partial(const double* __restrict__ x, const double* __restrict__ y,
                                                            size_t per_slice, double* __restrict__ partial, int nblk,
                                                            const int* __restrict__ active) {
  pdl_wait();
  __shared__ double sh[kRedThreads / 32];
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  const size_t base = (size_t)blockIdx.x * kRedChunk;
  const double* xs = x + s * per_slice;
  const double* ys = y + s * per_slice;
  const double acc = block_sum(chunk_dot(xs, ys, base, per_slice), sh);
  if (threadIdx.x == 0) partial[(size_t)s * nblk + blockIdx.x] = acc;
}

// out[s] = sum_b partial[s][b] (sequential fixed order); sqrt if requested;
// +inf if the slice flagged a degenerate mesh
__global__ void k_dot_final(const double* __restrict__ partial, int nblk, double* __restrict__ out, int S, int take_sqrt,
                            const int* __restrict__ degen, const int* __restrict__ active) {
  pdl_wait();
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  if (active && !active[s]) return;
  double acc = ordered_sum(partial + (size_t)s * nblk, nblk);
  if (take_sqrt) acc = sqrt(acc);
  if (degen && degen[s]) acc = __longlong_as_double(0x7ff0000000000000LL);
  out[s] = acc;
}

// multi-dot: partial[s][v][blk] = <V_v, w> over the chunk; grid (nblk, nv, S)
__global__ void __launch_bounds__(kRedThreads) k_mdot_partial(const double* __restrict__ V, size_t vstride,
                                                             const double* __restrict__ w, int nv, size_t per_slice,
                                                             double* __restrict__ partial, int nblk, int maxv,
                                                             const int* __restrict__ active) {
  pdl_wait();
  __shared__ double sh[kRedThreads / 32];
  const int s = blockIdx.z;
  const int v = blockIdx.y;
  if (active && !active[s]) return;
  const size_t base = (size_t)blockIdx.x * kRedChunk;
  const double* ws = w + s * per_slice;
  const double* vs = V + v * vstride + s * per_slice;
  double acc = 0.0;
#pragma unroll
  for (int i = threadIdx.x; i < kRedChunk; i += kRedThreads) {
    const size_t e = base + i;
    if (e < per_slice) acc += vs[e] * ws[e];
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) partial[((size_t)s * maxv + v) * nblk + blockIdx.x] = acc;
}

// h[s][i] (+)= sum_b partial[s][i][b]
__global__ void k_mdot_final(const double* __restrict__ partial, int nblk, int nv, int maxv, double* __restrict__ h,
                             int hstride, int accumulate, int S, const int* __restrict__ active) {
  pdl_wait();
  const int s = blockIdx.x;
  if (s >= S) return;
  if (active && !active[s]) return;
  for (int v = threadIdx.x; v < nv; v += blockDim.x) {
    double acc = ordered_sum(partial + ((size_t)s * maxv + v) * nblk, nblk);
    if (accumulate) h[(size_t)s * hstride + v] += acc;
    else h[(size_t)s * hstride + v] = acc;
  }
}

// w -= sum_i coef[s][i] V_i   (fixed order in i)
__global__ void k_mupdate(double* __restrict__ w, const double* __restrict__ V, size_t vstride,
                          const double* __restrict__ coef, int cstride, int nv, size_t per_slice,
                          const int* __restrict__ active, const int* __restrict__ active2) {
  pdl_wait();
  const int s = blockIdx.y;
  if ((active && !active[s]) || (active2 && !active2[s])) return;
  const double* cs = coef + (size_t)s * cstride;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < per_slice; e += (size_t)gridDim.x * blockDim.x) {
    double acc = w[s * per_slice + e];
    for (int v = 0; v < nv; ++v) acc -= cs[v] * V[v * vstride + s * per_slice + e];
    w[s * per_slice + e] = acc;
  }
}

// out = sum_i coef[s][i] V_i (nv per slice from nvs[s])
__global__ void k_mcombine(double* __restrict__ out, const double* __restrict__ V, size_t vstride,
                           const double* __restrict__ coef, int cstride, const int* __restrict__ nvs,
                           size_t per_slice, const int* __restrict__ active) {
  pdl_wait();
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  const double* cs = coef + (size_t)s * cstride;
  const int nv = nvs[s];
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < per_slice; e += (size_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int v = 0; v < nv; ++v) acc += cs[v] * V[v * vstride + s * per_slice + e];
    out[s * per_slice + e] = acc;
  }
}

// ---------------------------------------------------------------- K3 block-stencil SpMV
// y = A x  or  y = b - A x (residual form).  Thread = (node, row component):
// blockDim (32, C) so a warp reads one coefficient plane of 32 consecutive
// nodes (256 B, coalesced) and the C row-threads of a node share its x
// neighbours through L1.  5-7x more threads than node-per-thread: these
// kernels are latency-bound at the small configs (c1/c2 live in L2).
// resident CTAs per SM the compiler must allow: the wide (BATCH = 3) variant
// trades loads-in-flight per thread for occupancy, the narrow one (all 9
// offsets in flight) is for small grids where occupancy is moot
template <int D, int BATCH>
struct StencilOcc {
  static constexpr int value = BATCH >= 9 ? 1 : (D == 2 ? 4 : 2);
};

template <int D, bool RESID, int BATCH, typename MT = double>
__global__ void __launch_bounds__(32 * (2 * D + 1), (StencilOcc<D, BATCH>::value)) k_spmv(Grid g, const MT* __restrict__ A,
                                                          const double* __restrict__ x,
                                                          const double* __restrict__ b, double* __restrict__ y,
                                                          const int* __restrict__ active) {
  pdl_wait();
  constexpr int C = 2 * D + 1;
  constexpr int NOFF = D == 2 ? 9 : 27;
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  const int n = blockIdx.x * 32 + threadIdx.x;
  if (n >= g.nn) return;
  const int ca = threadIdx.y;
  const int np = g.np;
  const size_t vs = (size_t)C * np;
  const MT* As = A + (size_t)s * NOFF * C * C * np + (size_t)ca * C * np + n;
  const double* xs = x + s * vs;
  int nbs[NOFF];
  stencil_neighbours<D>(g, n, nbs);
  const double acc = stencil_row<D, BATCH, MT>(As, xs, np, nbs, ca);
  const size_t o = s * vs + (size_t)ca * np + n;
  y[o] = RESID ? b[o] - acc : acc;
}

// Thread = node, all C rows (the V-cycle residuals with the fp32 operator
// copy).  The (node, row) kernel above re-reads the node's C*NOFF neighbour
// x values once per row thread: with 4-byte coefficients those x loads were
// 2/3 of its L1 wavefronts (c3 level 0 at 0.69 of HBM, ncu r02).  Here every
// x value is loaded once per node and kept in registers across the C rows.
// Same association order per row as stencil_row (offsets o, o+3, o+6 into
// partial o % 3, components cb in order, then (p0 + p1) + p2): bitwise the
// (node, row) kernel.
template <int D, bool RESID, typename MT>
__global__ void __launch_bounds__(128) k_spmv_node(Grid g, const MT* __restrict__ A, const double* __restrict__ x,
                                                   const double* __restrict__ b, double* __restrict__ y,
                                                   const int* __restrict__ active) {
  pdl_wait();
  constexpr int C = 2 * D + 1;
  constexpr int NOFF = D == 2 ? 9 : 27;
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= g.nn) return;
  const int np = g.np;
  const size_t vs = (size_t)C * np;
  const MT* As = A + (size_t)s * NOFF * C * C * np + n;
  const double* xs = x + s * vs;
  int nbs[NOFF];
  stencil_neighbours<D>(g, n, nbs);
  double part[C][3];
#pragma unroll
  for (int ca = 0; ca < C; ++ca) part[ca][0] = part[ca][1] = part[ca][2] = 0.0;
#pragma unroll
  for (int o = 0; o < NOFF; ++o) {
    double xv[C];
    MT a[C][C];
#pragma unroll
    for (int cb = 0; cb < C; ++cb) xv[cb] = ld_nc(xs + cb * np + nbs[o]);
#pragma unroll
    for (int ca = 0; ca < C; ++ca)
#pragma unroll
      for (int cb = 0; cb < C; ++cb)
        if (row_couples(ca, cb, D)) a[ca][cb] = ld_nc(As + ((size_t)(o * C + ca) * C + cb) * np);
#pragma unroll
    for (int ca = 0; ca < C; ++ca)
#pragma unroll
      for (int cb = 0; cb < C; ++cb)
        if (row_couples(ca, cb, D)) part[ca][o % 3] = fma((double)a[ca][cb], xv[cb], part[ca][o % 3]);
  }
#pragma unroll
  for (int ca = 0; ca < C; ++ca) {
    const double acc = (part[ca][0] + part[ca][1]) + part[ca][2];
    const size_t off = s * vs + (size_t)ca * np + n;
    y[off] = RESID ? b[off] - acc : acc;
  }
}

// ---------------------------------------------------------------- K4 node-block Jacobi
// Dinv[s][ca][cb][n] = inverse of the centre block (Gauss-Jordan, partial pivoting)
template <int D>
__global__ void k_block_inverse(Grid g, const double* __restrict__ A, double* __restrict__ Dinv,
                                const int* __restrict__ active) {
  pdl_wait();
  constexpr int C = 2 * D + 1;
  constexpr int NOFF = D == 2 ? 9 : 27;
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= g.nn) return;
  const int np = g.np;
  const int ctr = center_offset(D);
  const double* As = A + (size_t)s * NOFF * C * C * np;
  double a[C][2 * C];
  for (int r = 0; r < C; ++r)
    for (int c = 0; c < 2 * C; ++c)
      a[r][c] = c < C ? As[(((size_t)ctr * C + r) * C + c) * np + n] : (c - C == r ? 1.0 : 0.0);
  for (int p = 0; p < C; ++p) {
    int piv = p;
    double best = fabs(a[p][p]);
    for (int r = p + 1; r < C; ++r)
      if (fabs(a[r][p]) > best) { best = fabs(a[r][p]); piv = r; }
    if (piv != p)
      for (int c = 0; c < 2 * C; ++c) { double t = a[p][c]; a[p][c] = a[piv][c]; a[piv][c] = t; }
    const double d = a[p][p];
    const double inv = d != 0.0 ? 1.0 / d : 0.0;
    for (int c = 0; c < 2 * C; ++c) a[p][c] *= inv;
    for (int r = 0; r < C; ++r) {
      if (r == p) continue;
      const double f = a[r][p];
      if (f != 0.0)
        for (int c = 0; c < 2 * C; ++c) a[r][c] -= f * a[p][c];
    }
  }
  double* Ds = Dinv + (size_t)s * C * C * np;
  for (int r = 0; r < C; ++r)
    for (int c = 0; c < C; ++c) Ds[((size_t)r * C + c) * np + n] = a[r][C + c];
}

// x_out = (x_in ? x_in : 0) + omega Dinv (b - A x_in); thread = (node, row)
// as k_spmv, the node's C residual rows meet in shared memory for Dinv.
template <int D, bool FIRST, int BATCH>
__global__ void __launch_bounds__(32 * (2 * D + 1), (StencilOcc<D, BATCH>::value)) k_smooth(Grid g, const double* __restrict__ A,
                                                            const double* __restrict__ Dinv,
                                                            const double* __restrict__ b,
                                                            const double* __restrict__ xin,
                                                            double* __restrict__ xout, double omega,
                                                            const int* __restrict__ active,
                                                            unsigned long long* __restrict__ work) {
  pdl_wait();
  constexpr int C = 2 * D + 1;
  constexpr int NOFF = D == 2 ? 9 : 27;
  __shared__ double rsh[C][32];
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  if (work && blockIdx.x == 0 && threadIdx.x == 0 && threadIdx.y == 0) atomicAdd(work, 1ULL);
  const int n = blockIdx.x * 32 + threadIdx.x;
  const int ca = threadIdx.y;
  const bool live = n < g.nn;
  const int np = g.np;
  const size_t vs = (size_t)C * np;
  double res = 0.0;
  if (live) {
    res = __ldg(b + s * vs + (size_t)ca * np + n);
    if (!FIRST) {
      const double* As = A + (size_t)s * NOFF * C * C * np + (size_t)ca * C * np + n;
      const double* xs = xin + s * vs;
      int nbs[NOFF];
      stencil_neighbours<D>(g, n, nbs);
      const double acc = stencil_row<D, BATCH>(As, xs, np, nbs, ca);
      res -= acc;
    }
  }
  rsh[ca][threadIdx.x] = res;
  __syncthreads();
  if (!live) return;
  const double* Ds = Dinv + (size_t)s * C * C * np + (size_t)ca * C * np + n;
  double z = 0.0;
#pragma unroll
  for (int cb = 0; cb < C; ++cb) z += __ldg(Ds + (size_t)cb * np) * rsh[cb][threadIdx.x];
  const size_t o = s * vs + (size_t)ca * np + n;
  const double base = FIRST ? 0.0 : xin[o];
  xout[o] = base + omega * z;
}

// ---------------------------------------------------------------- grid transfer (Q1 bilinear / trilinear)
__device__ __forceinline__ double pweight(int fine, int coarse) {
  const int d = fine - 2 * coarse;
  return d == 0 ? 1.0 : ((d == 1 || d == -1) ? 0.5 : 0.0);
}

// bc[c][I] = sum_i P(i, I) rf[c][i]
template <int D>
__global__ void __launch_bounds__(32 * (2 * D + 1)) k_restrict(Grid gf, Grid gc, const double* __restrict__ rf,
                                                              double* __restrict__ bc,
                                                              const int* __restrict__ active) {
  pdl_wait();
  // thread = (coarse node, component): block (32, C), so the 3^d fine loads of
  // a thread are independent of its C-1 siblings' (more loads in flight)
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  const int I = blockIdx.x * 32 + threadIdx.x;
  if (I >= gc.nn) return;
  const int c = threadIdx.y;
  int ci, cj, ck;
  node_coords(gc, I, ci, cj, ck);
  double acc = 0.0;
  const double* rs = rf + (size_t)s * (2 * D + 1) * gf.np + (size_t)c * gf.np;
#pragma unroll
  for (int dk = (D == 3 ? -1 : 0); dk <= (D == 3 ? 1 : 0); ++dk)
#pragma unroll
    for (int dj = -1; dj <= 1; ++dj)
#pragma unroll
      for (int di = -1; di <= 1; ++di) {
        const int fi = 2 * ci + di, fj = 2 * cj + dj, fk = 2 * ck + dk;
        if (fi < 0 || fi >= gf.n[0] || fj < 0 || fj >= gf.n[1] || fk < 0 || fk >= gf.n[2]) continue;
        const double w = pweight(fi, ci) * pweight(fj, cj) * (D == 3 ? pweight(fk, ck) : 1.0);
        acc += w * rs[node_index(gf, fi, fj, fk)];
      }
  bc[(size_t)s * (2 * D + 1) * gc.np + (size_t)c * gc.np + I] = acc;
}

// sum_I P(i, I) e[I] over the <= 2^d coarse parents of fine node (fi, fj, fk):
// all parent loads issued first (predicated), then summed in ascending
// (k, j, i) parent order
template <int D>
__device__ __forceinline__ double prolong_sum(const Grid& gc, const double* es, int fi, int fj, int fk) {
  constexpr int KK = D == 3 ? 2 : 1;
  const int i0 = fi >> 1, j0 = fj >> 1, k0 = fk >> 1;
  double e[KK][2][2];
#pragma unroll
  for (int dk = 0; dk < KK; ++dk)
#pragma unroll
    for (int dj = 0; dj < 2; ++dj)
#pragma unroll
      for (int di = 0; di < 2; ++di) {
        const bool ok = di <= (fi & 1) && dj <= (fj & 1) && (D == 2 || dk <= (fk & 1));
        e[dk][dj][di] = ok ? es[node_index(gc, i0 + di, j0 + dj, k0 + dk)] : 0.0;
      }
  double acc = 0.0;
#pragma unroll
  for (int dk = 0; dk < KK; ++dk)
#pragma unroll
    for (int dj = 0; dj < 2; ++dj)
#pragma unroll
      for (int di = 0; di < 2; ++di) {
        if (!(di <= (fi & 1) && dj <= (fj & 1) && (D == 2 || dk <= (fk & 1)))) continue;
        const double w = pweight(fi, i0 + di) * pweight(fj, j0 + dj) * (D == 3 ? pweight(fk, k0 + dk) : 1.0);
        acc += w * e[dk][dj][di];
      }
  return acc;
}

// xf[c][i] += sum_I P(i, I) ec[c][I]; thread = (fine node, component), block (32, C)
template <int D>
__global__ void __launch_bounds__(32 * (2 * D + 1)) k_prolong_add(Grid gf, Grid gc, const double* __restrict__ ec,
                                                                 double* __restrict__ xf,
                                                                 const int* __restrict__ active) {
  pdl_wait();
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  const int f = blockIdx.x * 32 + threadIdx.x;
  if (f >= gf.nn) return;
  const int c = threadIdx.y;
  int fi, fj, fk;
  node_coords(gf, f, fi, fj, fk);
  const double* es = ec + (size_t)s * (2 * D + 1) * gc.np + (size_t)c * gc.np;
  const size_t o = (size_t)s * (2 * D + 1) * gf.np + (size_t)c * gf.np + f;
  const double xo = xf[o];
  const double acc = prolong_sum<D>(gc, es, fi, fj, fk);
  xf[o] = xo + acc;
}

// Galerkin coarse operator Ac = P^T Af P; thread = (coarse node, coarse offset, row comp)
template <int D>
__global__ void k_rap(Grid gf, Grid gc, const double* __restrict__ Af, double* __restrict__ Ac,
                      const int* __restrict__ active) {
  pdl_wait();
  constexpr int C = 2 * D + 1;
  constexpr int NOFF = D == 2 ? 9 : 27;
  const int s = blockIdx.z;
  if (active && !active[s]) return;
  const int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= gc.nn) return;
  const int oc = blockIdx.y / C, ca = blockIdx.y % C;
  int ci, cj, ck;
  node_coords(gc, I, ci, cj, ck);
  int odi, odj, odk;
  offset_delta(oc, D, odi, odj, odk);
  const int Ji = ci + odi, Jj = cj + odj, Jk = ck + odk;
  double acc[C];
#pragma unroll
  for (int c = 0; c < C; ++c) acc[c] = 0.0;
  const bool valid = !(Ji < 0 || Ji >= gc.n[0] || Jj < 0 || Jj >= gc.n[1] || Jk < 0 || Jk >= gc.n[2]);
  if (valid) {
    const double* As = Af + (size_t)s * NOFF * C * C * gf.np;
    for (int dk = (D == 3 ? -1 : 0); dk <= (D == 3 ? 1 : 0); ++dk)
      for (int dj = -1; dj <= 1; ++dj)
        for (int di = -1; di <= 1; ++di) {
          const int fi = 2 * ci + di, fj = 2 * cj + dj, fk = 2 * ck + dk;
          if (fi < 0 || fi >= gf.n[0] || fj < 0 || fj >= gf.n[1] || fk < 0 || fk >= gf.n[2]) continue;
          const double rw = pweight(fi, ci) * pweight(fj, cj) * (D == 3 ? pweight(fk, ck) : 1.0);
          const int f = node_index(gf, fi, fj, fk);
          for (int off = 0; off < NOFF; ++off) {
            int ddi, ddj, ddk;
            offset_delta(off, D, ddi, ddj, ddk);
            const int gi = fi + ddi, gj = fj + ddj, gk = fk + ddk;
            if (gi < 0 || gi >= gf.n[0] || gj < 0 || gj >= gf.n[1] || gk < 0 || gk >= gf.n[2]) continue;
            const double pw = pweight(gi, Ji) * pweight(gj, Jj) * (D == 3 ? pweight(gk, Jk) : 1.0);
            if (pw == 0.0) continue;
            const double w = rw * pw;
            const double* blk = As + (((size_t)off * C + ca) * C) * gf.np + f;
#pragma unroll
            for (int cb = 0; cb < C; ++cb) acc[cb] += w * blk[(size_t)cb * gf.np];
          }
        }
  }
  double* Cs = Ac + (size_t)s * NOFF * C * C * gc.np;
#pragma unroll
  for (int cb = 0; cb < C; ++cb) Cs[(((size_t)oc * C + ca) * C + cb) * gc.np + I] = acc[cb];
}

// ---------------------------------------------------------------- dense coarsest level
// M[s] (n x 2n, row-major) = [A | I] with dense index c*nn + node
template <int D>
__global__ void k_dense_build(Grid g, const double* __restrict__ A, double* __restrict__ M,
                              const int* __restrict__ active) {
  pdl_wait();
  constexpr int C = 2 * D + 1;
  constexpr int NOFF = D == 2 ? 9 : 27;
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  const int n = C * g.nn;
  double* Ms = M + (size_t)s * n * 2 * n;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n * 2 * n; idx += gridDim.x * blockDim.x)
    Ms[idx] = 0.0;
  __syncthreads();
  // one thread per (row node, row comp)
  for (int row = blockIdx.x * blockDim.x + threadIdx.x; row < n; row += gridDim.x * blockDim.x) {
    const int ca = row / g.nn, node = row % g.nn;
    int i, j, k;
    node_coords(g, node, i, j, k);
    const double* As = A + (size_t)s * NOFF * C * C * g.np;
    for (int off = 0; off < NOFF; ++off) {
      const int nb = neighbour(g, i, j, k, off);
      if (nb < 0) continue;
      for (int cb = 0; cb < C; ++cb)
        Ms[(size_t)row * 2 * n + cb * g.nn + nb] = As[(((size_t)off * C + ca) * C + cb) * g.np + node];
    }
    Ms[(size_t)row * 2 * n + n + row] = 1.0;
  }
}

// in-place Gauss-Jordan with partial pivoting, one CTA per slice (grid.x = S)
__global__ void k_gauss_jordan(double* __restrict__ M, int n, const int* __restrict__ active) {
  pdl_wait();
  const int s = blockIdx.x;
  if (active && !active[s]) return;
  double* Ms = M + (size_t)s * n * 2 * n;
  __shared__ double sval[32];
  __shared__ int sidx[32];
  __shared__ int piv_sh;
  const int w2 = 2 * n;
  for (int p = 0; p < n; ++p) {
    // pivot search (deterministic: largest |a|, lowest row on ties)
    double best = -1.0;
    int bi = p;
    for (int r = p + threadIdx.x; r < n; r += blockDim.x) {
      const double v = fabs(Ms[(size_t)r * w2 + p]);
      if (v > best) { best = v; bi = r; }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_down_sync(0xffffffffu, best, o);
      const int oi = __shfl_down_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    if ((threadIdx.x & 31) == 0) { sval[threadIdx.x >> 5] = best; sidx[threadIdx.x >> 5] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double b = -1.0;
      int ii = p;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
        if (sval[w] > b || (sval[w] == b && sidx[w] < ii)) { b = sval[w]; ii = sidx[w]; }
      piv_sh = ii;
    }
    __syncthreads();
    const int piv = piv_sh;
    if (piv != p)
      for (int c = threadIdx.x; c < w2; c += blockDim.x) {
        const double t = Ms[(size_t)p * w2 + c];
        Ms[(size_t)p * w2 + c] = Ms[(size_t)piv * w2 + c];
        Ms[(size_t)piv * w2 + c] = t;
      }
    __syncthreads();
    const double d = Ms[(size_t)p * w2 + p];
    const double inv = d != 0.0 ? 1.0 / d : 0.0;
    __syncthreads();
    for (int c = threadIdx.x; c < w2; c += blockDim.x) Ms[(size_t)p * w2 + c] *= inv;
    __syncthreads();
    for (int idx = threadIdx.x; idx < n * w2; idx += blockDim.x) {
      const int r = idx / w2, c = idx % w2;
      if (r == p || c == p) continue;
      Ms[(size_t)r * w2 + c] -= Ms[(size_t)r * w2 + p] * Ms[(size_t)p * w2 + c];
    }
    __syncthreads();
    for (int r = threadIdx.x; r < n; r += blockDim.x)
      if (r != p) Ms[(size_t)r * w2 + p] = 0.0;
    __syncthreads();
  }
}

// ---------------------------------------------------------------- dense coarsest inverse, cluster version
// The coarsest operator (n <= a few hundred dofs) is inverted by in-place
// Gauss-Jordan with partial pivoting, distributed over a cluster of
// kGJCluster CTAs per slice: each CTA holds ceil(n/CL) rows in shared memory,
// the pivot candidates and the winning row travel through distributed shared
// memory, one cluster barrier per pivot.  Pivoting is implicit (no row
// swaps): step p picks the largest |a_rp| among rows not yet used (lowest
// global row on ties, deterministic) and the permutations are resolved when
// the inverse is written out, row-major [n][n].
// ---------------------------------------------------------------- dense coarsest inverse, cluster version
// The coarsest operator (n <= 448 dofs) is inverted by in-place Gauss-Jordan
// with partial pivoting, distributed over a cluster of kGJCluster CTAs per
// slice.  CTA `rank` owns rows [rank*rp, rank*rp + rp); inside it thread
// (rg, cg) keeps the kGJTR x kGJTC tile of rows rg*kGJTR + t and columns
// cg + 64 u in REGISTERS for the whole factorisation, so a pivot step costs
// two loads (its rows' multipliers, its columns of the pivot row) per 49
// FMAs instead of a shared-memory round trip per element.  Per pivot: the
// owners of column p publish it, the local candidate (largest |a| over unused
// rows, lowest row on ties) is pushed into every CTA of the cluster, one
// cluster barrier, every CTA picks the same winner and pulls its row through
// distributed shared memory.  Pivoting is implicit (no row swaps); the
// permutations are resolved when the inverse is written out: fp32, row-major
// [n][ld] (ld = n rounded up to 4 floats, so every row starts 16-B aligned for
// the bulk copies of the V-cycle tail).  Preconditioner storage only: the
// factorisation itself runs in fp64.
constexpr int kGJCluster = 8;
constexpr int kGJThreads = 512;
constexpr int kGJRG = 8;                        // row groups
constexpr int kGJCG = kGJThreads / kGJRG;       // column groups (64)
constexpr int kGJTR = 7, kGJTC = 7;             // register tile
constexpr int kGJMaxN = kGJCluster * kGJRG * kGJTR < kGJCG * kGJTC ? kGJCluster * kGJRG * kGJTR : kGJCG * kGJTC;

__host__ __device__ inline size_t gj_rows_per(int n) { return (size_t)(n + kGJCluster - 1) / kGJCluster; }
// Aloc [rp][n] (assembly staging), pub [2][n], prow [n], colf [2][rp], part [kGJRG] x 2,
// cand [2][CL][2], piv_of [n], pinv [rp]
__host__ __device__ inline size_t gj_smem_bytes(int n) {
  const size_t rp = gj_rows_per(n);
  return 8 * (rp * n + 3 * (size_t)n + 2 * rp + 2 * kGJRG + 4 * kGJCluster) + 4 * ((size_t)n + rp) + 16;
}
__host__ __device__ inline bool gj_fits(int n) { return n <= kGJMaxN && gj_smem_bytes(n) <= 227 * 1024; }

template <int D>
__global__ void __cluster_dims__(kGJCluster, 1, 1) __launch_bounds__(kGJThreads, 1)
    k_dense_invert_cl(Grid g, const double* __restrict__ A, float* __restrict__ Minv, int n, int ld,
                      const int* __restrict__ active) {
  pdl_wait();
  constexpr int C = 2 * D + 1;
  constexpr int NOFF = D == 2 ? 9 : 27;
  cg::cluster_group cluster = cg::this_cluster();
  const int s = blockIdx.x / kGJCluster;
  if (active && !active[s]) return;  // uniform over the cluster
  const int rank = (int)cluster.block_rank();
  const int rp = (int)gj_rows_per(n);
  const int r0 = rank * rp;
  const int nloc = max(0, min(rp, n - r0));
  extern __shared__ __align__(16) unsigned char gj_smem[];
  double* Aloc = reinterpret_cast<double*>(gj_smem);  // [rp][n]
  double* pub = Aloc + (size_t)rp * n;                 // [2][n]: this CTA's candidate row
  double* prow = pub + 2 * n;                          // scaled pivot row
  double* colf = prow + n;                             // [2][rp]: column p of the local rows
  double* part = colf + 2 * rp;                        // [kGJRG][2]: partial candidates (a, row)
  double* cand = part + 2 * kGJRG;                     // [2][CL][2]: every CTA's candidate (a, local row)
  int* piv_of = reinterpret_cast<int*>(cand + 4 * kGJCluster);  // [n]: pivot row of step p
  int* pinv = piv_of + n;                                         // [rp]: step that used local row r
  const int tid = threadIdx.x;
  const int rg = tid / kGJCG, cg_ = tid % kGJCG;
  const int rbase = rg * kGJTR;

  // assemble the local rows from the block-stencil operator (shared staging)
  for (int idx = tid; idx < rp * n; idx += kGJThreads) Aloc[idx] = 0.0;
  __syncthreads();
  const double* As = A + (size_t)s * NOFF * C * C * g.np;
  for (int idx = tid; idx < nloc * NOFF; idx += kGJThreads) {
    const int lr = idx / NOFF, off = idx % NOFF;
    const int row = r0 + lr;
    const int ca = row / g.nn, node = row % g.nn;
    int i, j, k;
    node_coords(g, node, i, j, k);
    const int nb = neighbour(g, i, j, k, off);
    if (nb < 0) continue;
    double v[C];
#pragma unroll
    for (int cb = 0; cb < C; ++cb) v[cb] = As[(((size_t)off * C + ca) * C + cb) * g.np + node];
#pragma unroll
    for (int cb = 0; cb < C; ++cb) Aloc[(size_t)lr * n + cb * g.nn + nb] = v[cb];
  }
  __syncthreads();
  double a[kGJTR][kGJTC];
  unsigned used = 0;  // bit t: local row rbase + t already a pivot row (or absent)
#pragma unroll
  for (int t = 0; t < kGJTR; ++t) {
    const int r = rbase + t;
    if (r >= nloc) used |= 1u << t;
#pragma unroll
    for (int u = 0; u < kGJTC; ++u) {
      const int j = cg_ + kGJCG * u;
      a[t][u] = (r < nloc && j < n) ? Aloc[(size_t)r * n + j] : 0.0;
    }
  }
  // column 0 and the partial candidates of step 0 (owners: cg_ == 0, u == 0)
  if (cg_ == 0) {
    double ba = 0.0;
    int br = -1;
#pragma unroll
    for (int t = 0; t < kGJTR; ++t) {
      const int r = rbase + t;
      if (r < rp) colf[r] = a[t][0];
      if (!(used >> t & 1u) && (br < 0 || fabs(a[t][0]) > fabs(ba))) { ba = a[t][0]; br = r; }
    }
    part[2 * rg] = ba;
    part[2 * rg + 1] = (double)br;
  }

  for (int p = 0; p < n; ++p) {
    const int buf = p & 1;
    __syncthreads();  // partial candidates and colf[buf] of this step are complete
    double ca_ = 0.0;
    int cr = -1;
#pragma unroll
    for (int q = 0; q < kGJRG; ++q) {
      const double qa = part[2 * q];
      const int qr = (int)part[2 * q + 1];
      if (qr >= 0 && (cr < 0 || fabs(qa) > fabs(ca_))) { ca_ = qa; cr = qr; }
    }
    // the candidate row's owners publish it (all-zero row if this CTA has none left)
    if (cr >= 0 ? (cr / kGJTR == rg) : (rg == 0)) {
      double* dst = pub + buf * n + cg_;
      switch (cr >= 0 ? cr - rbase : -1) {
#define GJ_PUB(T)                                                              \
  case T:                                                                      \
    _Pragma("unroll") for (int u = 0; u < kGJTC; ++u) if (cg_ + kGJCG * u < n) \
        dst[kGJCG * u] = a[T][u];                                              \
    break;
        GJ_PUB(0) GJ_PUB(1) GJ_PUB(2) GJ_PUB(3) GJ_PUB(4) GJ_PUB(5) GJ_PUB(6)
#undef GJ_PUB
        default:
#pragma unroll
          for (int u = 0; u < kGJTC; ++u)
            if (cg_ + kGJCG * u < n) dst[kGJCG * u] = 0.0;
      }
    }
    if (tid < kGJCluster) {  // push the candidate into every CTA of the cluster
      double* dst = cluster.map_shared_rank(cand, tid) + (buf * kGJCluster + rank) * 2;
      dst[0] = ca_;
      dst[1] = (double)cr;
    }
    cluster.sync();
    // the winner over the cluster (every thread, from local shared memory; lowest rank on ties)
    int wrank = -1, wl = -1;
    double pa = 0.0;
#pragma unroll
    for (int q = 0; q < kGJCluster; ++q) {
      const double qa = cand[(buf * kGJCluster + q) * 2];
      const int ql = (int)cand[(buf * kGJCluster + q) * 2 + 1];
      if (ql >= 0 && (wrank < 0 || fabs(qa) > fabs(pa))) { pa = qa; wrank = q; wl = ql; }
    }
    const double inv = pa != 0.0 ? 1.0 / pa : 0.0;
    const double* wsrc = cluster.map_shared_rank(pub, wrank) + buf * n;
    for (int j = tid; j < n; j += kGJThreads) prow[j] = j == p ? inv : wsrc[j] * inv;
    if (tid == 0) piv_of[p] = wrank * rp + wl;
    const int tw = wrank == rank ? wl - rbase : -1;  // my tile row that is the pivot row (if any)
    if (tw >= 0 && tw < kGJTR) used |= 1u << tw;
    if (tid % kGJCG == 0 && wrank == rank && wl >= rbase && wl < rbase + kGJTR) pinv[wl] = p;
    __syncthreads();
    // a_rj <- a_rj - a_rp prow_j everywhere (49 FMAs, no selects), then the
    // owners fix column p (a_rp <- -a_rp / pivot) and the pivot row (<- prow)
    double pj[kGJTC];
#pragma unroll
    for (int u = 0; u < kGJTC; ++u) {
      const int j = cg_ + kGJCG * u;
      pj[u] = j < n ? prow[j] : 0.0;
    }
    const double* cf = colf + buf * rp;
#pragma unroll
    for (int t = 0; t < kGJTR; ++t) {
      const double ft = rbase + t < rp ? cf[rbase + t] : 0.0;
#pragma unroll
      for (int u = 0; u < kGJTC; ++u) a[t][u] = fma(-ft, pj[u], a[t][u]);
    }
    if (cg_ == p % kGJCG) {
      switch (p / kGJCG) {
#define GJ_COL(U)                                                                     \
  case U:                                                                             \
    _Pragma("unroll") for (int t = 0; t < kGJTR; ++t) a[t][U] =                      \
        rbase + t < rp ? -cf[rbase + t] * inv : 0.0;                                  \
    break;
        GJ_COL(0) GJ_COL(1) GJ_COL(2) GJ_COL(3) GJ_COL(4) GJ_COL(5) GJ_COL(6)
#undef GJ_COL
        default: break;
      }
    }
    switch (tw) {
#define GJ_ROW(T)                                                   \
  case T:                                                           \
    _Pragma("unroll") for (int u = 0; u < kGJTC; ++u) a[T][u] = pj[u]; \
    break;
      GJ_ROW(0) GJ_ROW(1) GJ_ROW(2) GJ_ROW(3) GJ_ROW(4) GJ_ROW(5) GJ_ROW(6)
#undef GJ_ROW
      default: break;
    }
    // owners of column p+1 publish it and their partial candidate
    const int pn = p + 1;
    if (pn < n && cg_ == pn % kGJCG) {
      double v[kGJTR];
      switch (pn / kGJCG) {
#define GJ_NEXT(U)                                                          \
  case U:                                                                   \
    _Pragma("unroll") for (int t = 0; t < kGJTR; ++t) v[t] = a[t][U];       \
    break;
        GJ_NEXT(0) GJ_NEXT(1) GJ_NEXT(2) GJ_NEXT(3) GJ_NEXT(4) GJ_NEXT(5) GJ_NEXT(6)
#undef GJ_NEXT
        default:
#pragma unroll
          for (int t = 0; t < kGJTR; ++t) v[t] = 0.0;
      }
      double* cn = colf + (buf ^ 1) * rp;
      double ba = 0.0;
      int br = -1;
#pragma unroll
      for (int t = 0; t < kGJTR; ++t) {
        const int r = rbase + t;
        if (r < rp) cn[r] = v[t];
        if (!(used >> t & 1u) && (br < 0 || fabs(v[t]) > fabs(ba))) { ba = v[t]; br = r; }
      }
      part[2 * rg] = ba;
      part[2 * rg + 1] = (double)br;
    }
  }
  __syncthreads();
  // write out: inverse row pinv[r], column piv_of[j]  <-  local (r, j)
  float* Ms = Minv + (size_t)s * n * ld;
#pragma unroll
  for (int t = 0; t < kGJTR; ++t) {
    const int r = rbase + t;
    if (r >= nloc) continue;
    const size_t ro = (size_t)pinv[r] * ld;
#pragma unroll
    for (int u = 0; u < kGJTC; ++u) {
      const int j = cg_ + kGJCG * u;
      if (j < n) Ms[ro + piv_of[j]] = (float)a[t][u];
    }
  }
  cluster.sync();  // no CTA leaves while another may still read its shared memory
}

// x = M^{-1} b with the fp32 dense coarsest inverse [S][n][ld]: one warp per
// row, lanes stride the columns, fp64 accumulation, fixed xor-butterfly order
// (the tail's shared-memory copy of the rows gives the same bits)
__device__ __forceinline__ double dense_row_dot(const float* __restrict__ Mr, const double* __restrict__ bsh, int n,
                                                int lane) {
  double acc = 0.0;
  for (int c = lane; c < n; c += 32) acc = fma((double)Mr[c], bsh[c], acc);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

template <int C>
__device__ __forceinline__ void dense_apply_warps(const Grid& g, const float* __restrict__ M, int ld, int s,
                                                  const double* __restrict__ b, double* __restrict__ x, int tid,
                                                  int nth) {
  const int n = C * g.nn;
  const float* Ms = M + (size_t)s * n * ld;
  const double* bs = b + (size_t)s * C * g.np;
  const int lane = tid & 31;
  // the lane's right-hand-side entries are the same for every row: loaded once
  // (dense levels hold <= 448 dofs after the cluster inversion, 1024 at most)
  constexpr int Q = 14;  // columns per lane and round: 14 * 32 = 448
  for (int row = tid >> 5; row < n; row += nth >> 5) {
    const float* Mr = Ms + (size_t)row * ld;
    double acc = 0.0;
    for (int c0 = 0; c0 < n; c0 += 32 * Q) {
      float mv[Q];
      double bv[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) {  // all loads of the round in flight before the first FMA
        const int c = c0 + lane + 32 * q;
        mv[q] = c < n ? __ldg(Mr + c) : 0.0f;
        bv[q] = c < n ? bs[(c / g.nn) * g.np + (c % g.nn)] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < Q; ++q)
        if (c0 + lane + 32 * q < n) acc = fma((double)mv[q], bv[q], acc);  // same order as the rolled loop
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) x[(size_t)s * C * g.np + (row / g.nn) * g.np + (row % g.nn)] = acc;
  }
}

// fp64 augmented [n][2n] inverse (single-CTA fallback) -> fp32 [n][ld]
__global__ void k_dense_to_f32(const double* __restrict__ M, float* __restrict__ out, int n, int ld,
                               const int* __restrict__ active) {
  pdl_wait();
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  const double* Ms = M + (size_t)s * n * 2 * n;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n * n; idx += gridDim.x * blockDim.x) {
    const int r = idx / n, c = idx % n;
    out[(size_t)s * n * ld + (size_t)r * ld + c] = (float)Ms[(size_t)r * 2 * n + n + c];
  }
}

template <int D>
__global__ void k_dense_apply(Grid g, const float* __restrict__ M, int ld, const double* __restrict__ b,
                              double* __restrict__ x, const int* __restrict__ active) {
  pdl_wait();
  constexpr int C = 2 * D + 1;
  const int s = blockIdx.x;
  if (active && !active[s]) return;
  dense_apply_warps<C>(g, M, ld, s, b, x, threadIdx.x, blockDim.x);
}

// ---------------------------------------------------------------- GMRES scalar work (one thread per slice)
// back substitution H y = g for the steps taken this cycle
__global__ void k_gmres_solve(int m, const double* __restrict__ H, const double* __restrict__ gv,
                              const int* __restrict__ gm_steps, double* __restrict__ y, const int* __restrict__ active,
                              int S) {
  pdl_wait();
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  if (active && !active[s]) return;
  const int k = gm_steps[s];
  const double* Hs = H + (size_t)s * (m + 1) * m;
  const double* g = gv + (size_t)s * (m + 1);
  double* ys = y + (size_t)s * (m + 1);
  for (int i = k - 1; i >= 0; --i) {
    double acc = g[i];
    for (int c = i + 1; c < k; ++c) acc -= Hs[(size_t)c * (m + 1) + i] * ys[c];
    const double d = Hs[(size_t)i * (m + 1) + i];
    ys[i] = d != 0.0 ? acc / d : 0.0;
  }
  for (int i = k; i <= m; ++i) ys[i] = 0.0;
}

}  // namespace pint

namespace pint {

// hcol[s][i] += add[s][i], i < nv
__global__ void k_add_cols(double* __restrict__ hcol, int hstride, const double* __restrict__ add, int astride, int nv,
                           int S, const int* __restrict__ active) {
  pdl_wait();
  const int s = blockIdx.x;
  if (s >= S || (active && !active[s])) return;
  for (int i = threadIdx.x; i < nv; i += blockDim.x) hcol[(size_t)s * hstride + i] += add[(size_t)s * astride + i];
}

// hcol[s][row] = sqrt(sum_b partial[s][b])
__global__ void k_norm_to_h(const double* __restrict__ partial, int nblk, double* __restrict__ hcol, int hstride,
                            int row, int S, const int* __restrict__ active) {
  pdl_wait();
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S || (active && !active[s])) return;
  double acc = 0.0;
  for (int b = 0; b < nblk; ++b) acc += partial[(size_t)s * nblk + b];
  hcol[(size_t)s * hstride + row] = sqrt(acc);
}

// vout = w / hcol[s][row]  (0 when the norm vanished: lucky breakdown)
__global__ void k_scale_col(double* __restrict__ vout, const double* __restrict__ w, const double* __restrict__ hcol,
                            int hstride, int row, size_t per_slice, const int* __restrict__ active) {
  pdl_wait();
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  const double h = hcol[(size_t)s * hstride + row];
  const double inv = h != 0.0 ? 1.0 / h : 0.0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < per_slice; i += (size_t)gridDim.x * blockDim.x)
    vout[s * per_slice + i] = w[s * per_slice + i] * inv;
}

// x += z
__global__ void k_axpy_one(double* __restrict__ x, const double* __restrict__ z, size_t per_slice,
                           const int* __restrict__ active) {
  pdl_wait();
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < per_slice; i += (size_t)gridDim.x * blockDim.x)
    x[s * per_slice + i] += z[s * per_slice + i];
}

}  // namespace pint

// ======================================================================
// Cell-patch (Vanka-type) smoother (inverses stored in fp32, applied in fp64): every cell's L = 2^d C dofs form a local
// saddle-point block A_c (extracted from the block stencil) that is inverted
// exactly once per setup; one sweep is x += omega W sum_c P_c^T A_c^{-1} P_c r
// with r = b - A x and W = 1 / (cells sharing the node).  Robust where the
// node-block Jacobi smoother stalls (developed-flow c3 states, SURVEY §7 hard
// part 6): the local solve sees the velocity-pressure and velocity-deformation
// couplings of the whole cell.
// ======================================================================
namespace pint {

template <int D>
struct Cells {
  static constexpr int A = 1 << D;
  static constexpr int C = 2 * D + 1;
  static constexpr int L = A * C;
};

// cell index -> corner nodes (x fastest); grid g is the node grid
template <int D>
__device__ __forceinline__ void cell_nodes(const Grid& g, int cell, int (&nodes)[1 << D]) {
  const int cx = g.n[0] - 1, cy = g.n[1] - 1;
  const int ci = cell % cx;
  const int r = cell / cx;
  const int cj = r % cy;
  const int ck = r / cy;
#pragma unroll
  for (int a = 0; a < (1 << D); ++a)
    nodes[a] = node_index(g, ci + (a & 1), cj + ((a >> 1) & 1), D == 3 ? ck + ((a >> 2) & 1) : 0);
}

__device__ __forceinline__ int num_cells(const Grid& g) {
  return (g.n[0] - 1) * (g.n[1] - 1) * (g.dim == 3 ? (g.n[2] - 1) : 1);
}

// one warp per (cell, slice): gather A_c into shared memory [L][2L] = [A_c | I],
// Gauss-Jordan with partial pivoting (deterministic: largest |a|, lowest row),
// store A_c^{-1} as Vinv[s][i*L + j][cell] (coalesced across cells in the apply)
template <int D, int WARPS>
__global__ void __launch_bounds__(32 * WARPS) k_vanka_setup(Grid g, const double* __restrict__ Ast,
                                                          float* __restrict__ Vinv, const int* __restrict__ active) {
  pdl_wait();
  constexpr int L = Cells<D>::L;
  constexpr int C = Cells<D>::C;
  constexpr int A = Cells<D>::A;
  constexpr int W2 = 2 * L;
  extern __shared__ double smem[];
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ncell = num_cells(g);
  const int cell = blockIdx.x * WARPS + warp;
  if (cell >= ncell) return;  // whole warp exits together
  double* M = smem + (size_t)warp * (L * W2 + L);
  double* fcol = M + L * W2;
  int nodes[A];
  cell_nodes<D>(g, cell, nodes);
  const int np = g.np;
  const double* As = Ast + (size_t)s * g.noff * C * C * np;
  for (int idx = lane; idx < L * L; idx += 32) {
    const int r = idx / L, c = idx % L;
    const int a = r / C, ca = r % C, b = c / C, cb = c % C;
    const int di = (b & 1) - (a & 1), dj = ((b >> 1) & 1) - ((a >> 1) & 1);
    const int dk = D == 3 ? ((b >> 2) & 1) - ((a >> 2) & 1) : 0;
    const int off = offset_index(di, dj, dk, D);
    M[r * W2 + c] = As[(((size_t)off * C + ca) * C + cb) * np + nodes[a]];
    M[r * W2 + L + c] = (r == c) ? 1.0 : 0.0;
  }
  __syncwarp();
  for (int p = 0; p < L; ++p) {
    double best = -1.0;
    int bi = p;
    for (int r = p + lane; r < L; r += 32) {
      const double v = fabs(M[r * W2 + p]);
      if (v > best) { best = v; bi = r; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_down_sync(0xffffffffu, best, o);
      const int oi = __shfl_down_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    const int piv = __shfl_sync(0xffffffffu, bi, 0);
    if (piv != p)
      for (int c = lane; c < W2; c += 32) {
        const double t = M[p * W2 + c];
        M[p * W2 + c] = M[piv * W2 + c];
        M[piv * W2 + c] = t;
      }
    __syncwarp();
    const double d = M[p * W2 + p];
    const double inv = d != 0.0 ? 1.0 / d : 0.0;
    __syncwarp();
    for (int c = lane; c < W2; c += 32) M[p * W2 + c] *= inv;
    for (int r = lane; r < L; r += 32) fcol[r] = M[r * W2 + p];
    __syncwarp();
    for (int r = 0; r < L; ++r) {
      if (r == p) continue;
      const double f = fcol[r];
      if (f == 0.0) continue;
      for (int c = lane; c < W2; c += 32) M[r * W2 + c] -= f * M[p * W2 + c];
    }
    __syncwarp();
  }
  float* Vs = Vinv + (size_t)s * L * L * ncell;
  for (int idx = lane; idx < L * L; idx += 32) {
    const int r = idx / L, c = idx % L;
    Vs[(size_t)idx * ncell + cell] = (float)M[r * W2 + L + c];
  }
}

// Register-resident variant: ceil(L/32) warps per cell, thread t owns row t of
// A_c in registers; in-place Gauss-Jordan sweeps with IMPLICIT partial pivoting
// (no row swaps: the pivot of column p is the unused row with the largest
// |a|, lowest index on ties -- deterministic).  Per pivot the owner publishes
// its row through shared memory and every other row is updated from it; the
// sweep leaves  A_c^{-1}[pos(t)][perm(c)] = M[t][c]  (perm: pivot row of
// column p, pos: its inverse).  No augmented identity, no shared-memory
// read-modify-write chains: ~10x faster than the warp-per-cell smem version
// for the 56x56 blocks of 3-d.
template <int D>
struct VankaRows {
  static constexpr int L = Cells<D>::L;
  static constexpr int WPC = (L + 31) / 32;  // warps per cell
  static constexpr int TPC = WPC * 32;       // threads per cell
  static constexpr int CPB = D == 2 ? 4 : 2; // cells per block
  static constexpr int T = CPB * TPC;
};

template <int D>
__device__ __forceinline__ void cell_sync(int slot) {
  if constexpr (VankaRows<D>::WPC == 1) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(slot + 1), "r"(VankaRows<D>::TPC) : "memory");
  }
}

template <int D>
__global__ void __launch_bounds__(VankaRows<D>::T) k_vanka_setup_rows(Grid g, const double* __restrict__ Ast,
                                                                     float* __restrict__ Vinv,
                                                                     const int* __restrict__ active) {
  pdl_wait();
  using VR = VankaRows<D>;
  constexpr int L = VR::L, C = Cells<D>::C, A = Cells<D>::A, WPC = VR::WPC, CPB = VR::CPB;
  __shared__ double prow[2][CPB][L];
  __shared__ double cval[2][CPB][WPC];
  __shared__ int cidx[2][CPB][WPC];
  __shared__ int perm[CPB][L];
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  const int slot = threadIdx.x / VR::TPC;
  const int t = threadIdx.x % VR::TPC;  // my row
  const int lane = threadIdx.x & 31, wic = t >> 5;
  const int ncell = num_cells(g);
  const int cell = blockIdx.x * CPB + slot;
  if (cell >= ncell) return;  // the cell's threads leave together (named barriers are per cell)
  const bool has = t < L;
  int nodes[A];
  cell_nodes<D>(g, cell, nodes);
  const int np = g.np;
  const double* As = Ast + (size_t)s * g.noff * C * C * np;
  double row[L];
  {
    const int a = has ? t / C : 0, ca = has ? t % C : 0;
#pragma unroll
    for (int c = 0; c < L; ++c) {
      const int b = c / C, cb = c % C;
      const int di = (b & 1) - (a & 1), dj = ((b >> 1) & 1) - ((a >> 1) & 1);
      const int dk = D == 3 ? ((b >> 2) & 1) - ((a >> 2) & 1) : 0;
      row[c] = has ? As[(((size_t)offset_index(di, dj, dk, D) * C + ca) * C + cb) * np + nodes[a]] : 0.0;
    }
  }
  bool used = !has;
  int mypos = 0;
#pragma unroll 1
  for (int p = 0; p < L; ++p) {
    const int buf = p & 1;
    double ap = 0.0;
#pragma unroll
    for (int c = 0; c < L; ++c) ap = (c == p) ? row[c] : ap;
    // argmax over unused rows: value desc, row index asc
    double bv = used ? -1.0 : fabs(ap);
    int bi = used ? 0x7fffffff : t;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if constexpr (WPC > 1) {
      if (lane == 0) { cval[buf][slot][wic] = bv; cidx[buf][slot][wic] = bi; }
      cell_sync<D>(slot);
#pragma unroll
      for (int w = 0; w < WPC; ++w) {
        const double ov = cval[buf][slot][w];
        const int oi = cidx[buf][slot][w];
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
      }
    }
    const bool mine = bi == t;
    if (mine) {
      used = true;
      mypos = p;
      perm[slot][p] = t;
#pragma unroll
      for (int c = 0; c < L; ++c) prow[buf][slot][c] = row[c];
    }
    cell_sync<D>(slot);
    const double* pr = prow[buf][slot];
    const double d = pr[p];
    const double inv = d != 0.0 ? 1.0 / d : 0.0;
    if (mine) {
#pragma unroll
      for (int c = 0; c < L; ++c) row[c] = (c == p) ? inv : row[c] * inv;
    } else if (has) {
      const double f = ap;
#pragma unroll
      for (int c = 0; c < L; ++c) row[c] = (c == p) ? -f * inv : row[c] - f * (pr[c] * inv);
    }
  }
  cell_sync<D>(slot);
  if (!has) return;
  float* Vs = Vinv + (size_t)s * L * L * ncell + cell;
#pragma unroll
  for (int c = 0; c < L; ++c) Vs[(size_t)(mypos * L + perm[slot][c]) * ncell] = (float)row[c];
}

// y_c = A_c^{-1} r_c ; thread = (cell, local row); block (CELLS, L)
template <int D, int CELLS>
__global__ void __launch_bounds__(CELLS * Cells<D>::L) k_vanka_cell(Grid g, const float* __restrict__ Vinv,
                                                                   const double* __restrict__ r,
                                                                   double* __restrict__ y,
                                                                   const int* __restrict__ active,
                                                                   unsigned long long* __restrict__ work) {
  pdl_wait();
  constexpr int L = Cells<D>::L;
  constexpr int C = Cells<D>::C;
  constexpr int A = Cells<D>::A;
  __shared__ float rc[L][CELLS];
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  if (work && blockIdx.x == 0 && threadIdx.x == 0 && threadIdx.y == 0) atomicAdd(work, 1ULL);
  const int ncell = num_cells(g);
  const int cell = blockIdx.x * CELLS + threadIdx.x;
  const int row = threadIdx.y;
  const bool live = cell < ncell;
  const int np = g.np;
  if (live) {
    int nodes[A];
    cell_nodes<D>(g, cell, nodes);
    const int a = row / C, ca = row % C;
    rc[row][threadIdx.x] = (float)r[(size_t)s * C * np + (size_t)ca * np + nodes[a]];
  }
  __syncthreads();
  if (!live) return;
  const float* Vs = Vinv + (size_t)s * L * L * ncell + (size_t)row * L * ncell + cell;
  // fp32 arithmetic: the inverse is fp32 storage and the product is a
  // smoother correction inside the preconditioner (FGMRES absorbs the rounding)
  float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
  for (int j = 0; j < L; ++j) acc[j & 3] = fmaf(__ldg(Vs + (size_t)j * ncell), rc[j][threadIdx.x], acc[j & 3]);
  y[(size_t)s * L * ncell + (size_t)row * ncell + cell] = (double)((acc[0] + acc[1]) + (acc[2] + acc[3]));
}

// x_out = x_in + omega / count(n) * sum_{cells c containing n} y_c[local(n)]
// (fixed cell order); thread = (node, comp); block (32, C)
template <int D, bool FIRST>
__global__ void __launch_bounds__(32 * (2 * D + 1)) k_vanka_gather(Grid g, const double* __restrict__ y,
                                                                  const double* __restrict__ xin,
                                                                  double* __restrict__ xout, double omega,
                                                                  const int* __restrict__ active) {
  pdl_wait();
  constexpr int C = Cells<D>::C;
  constexpr int A = Cells<D>::A;
  constexpr int L = Cells<D>::L;
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  const int n = blockIdx.x * 32 + threadIdx.x;
  if (n >= g.nn) return;
  const int c = threadIdx.y;
  int i, j, k;
  node_coords(g, n, i, j, k);
  const int cx = g.n[0] - 1, cy = g.n[1] - 1, cz = D == 3 ? g.n[2] - 1 : 1;
  const int ncell = cx * cy * cz;
  const double* ys = y + (size_t)s * L * ncell;
  double acc = 0.0;
  int cnt = 0;
#pragma unroll
  for (int a = 0; a < A; ++a) {
    // node n is local corner a of the cell whose lower corner is n - bits(a)
    const int ci = i - (a & 1), cj = j - ((a >> 1) & 1), ck = D == 3 ? k - ((a >> 2) & 1) : 0;
    if (ci < 0 || ci >= cx || cj < 0 || cj >= cy || ck < 0 || ck >= cz) continue;
    const int cell = (ck * cy + cj) * cx + ci;
    acc += __ldg(ys + (size_t)(a * C + c) * ncell + cell);
    ++cnt;
  }
  const size_t o = (size_t)s * C * g.np + (size_t)c * g.np + n;
  const double z = acc / cnt;
  xout[o] = (FIRST ? 0.0 : xin[o]) + omega * z;
}

// Fused Vanka sweep (cell solves + gather in ONE pass, no y_c buffer):
// thread (node n, comp c) owns row (a, c) of each of the <= 2^D cells that
// have n as corner a, so every inverse row is still read exactly once.  The
// block's residual neighbourhood (3^{D-1} node-row ranges of 34 nodes, all
// components, converted to fp32 exactly as k_vanka_cell does) is staged in
// shared memory; per cell the product uses the same fmaf order and 4-way
// split as k_vanka_cell and the cells are summed in the same fixed corner
// order as k_vanka_gather -> bitwise the same x_out as the two-kernel sweep.
template <int D, bool FIRST>
__global__ void __launch_bounds__(32 * (2 * D + 1)) k_vanka_apply(Grid g, const float* __restrict__ Vinv,
                                                                 const double* __restrict__ r,
                                                                 const double* __restrict__ xin,
                                                                 double* __restrict__ xout, double omega,
                                                                 const int* __restrict__ active,
                                                                 unsigned long long* __restrict__ work,
                                                                 const double* __restrict__ wsrc = nullptr,
                                                                 const double* __restrict__ hn = nullptr,
                                                                 double* __restrict__ vout = nullptr) {
  pdl_wait();
  constexpr int C = Cells<D>::C;
  constexpr int A = Cells<D>::A;
  constexpr int L = Cells<D>::L;
  // wsrc != nullptr (first sweep of an Arnoldi step's V-cycle): the right-hand
  // side is the basis vector v_j = w / h_{j,j-1} that the previous step left
  // unscaled; it is formed here with k_scale_inv's arithmetic (x * (1/h)),
  // staged, and written to vout by each (node, comp) owner -- bitwise the
  // separate scaling launch, one launch fewer per Arnoldi step
  double inv = 1.0;
  if (wsrc) {
    const double al = hn[blockIdx.y];
    inv = al != 0.0 ? 1.0 / al : 0.0;
    r = wsrc;
  }
  constexpr int R = D == 2 ? 3 : 9;  // node-row ranges (dj, dk) in {-1,0,1}^{D-1}
  constexpr int W = 34;              // 32 nodes + one halo node either side
  __shared__ float rs[C][R][W];
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  if (work && blockIdx.x == 0 && threadIdx.x == 0 && threadIdx.y == 0) atomicAdd(work, 1ULL);
  const int n0 = blockIdx.x * 32;
  const int nx = g.n[0], nxy = g.n[0] * g.n[1];
  const double* rsl = r + (size_t)s * C * g.np;
  for (int idx = threadIdx.y * 32 + threadIdx.x; idx < C * R * W; idx += 32 * C) {
    const int w = idx % W, q = (idx / W) % R, cb = idx / (W * R);
    const int dj = q % 3 - 1, dk = D == 3 ? q / 3 - 1 : 0;
    const int m = n0 - 1 + w + dj * nx + dk * nxy;
    rs[cb][q][w] = (m >= 0 && m < g.nn) ? (float)(wsrc ? rsl[(size_t)cb * g.np + m] * inv
                                                         : __ldg(rsl + (size_t)cb * g.np + m))
                                        : 0.0f;
  }
  __syncthreads();
  const int n = n0 + threadIdx.x;
  if (n >= g.nn) return;
  const int c = threadIdx.y;
  if (wsrc) {
    const size_t ov = (size_t)s * C * g.np + (size_t)c * g.np + n;
    vout[ov] = wsrc[ov] * inv;
  }
  int i, j, k;
  node_coords(g, n, i, j, k);
  const int cx = g.n[0] - 1, cy = g.n[1] - 1, cz = D == 3 ? g.n[2] - 1 : 1;
  const int ncell = cx * cy * cz;
  const float* Vs = Vinv + (size_t)s * L * L * ncell;
  double acc = 0.0;
  int cnt = 0;
#pragma unroll
  for (int a = 0; a < A; ++a) {
    const int ax = a & 1, ay = (a >> 1) & 1, az = D == 3 ? (a >> 2) & 1 : 0;
    const int ci = i - ax, cj = j - ay, ck = D == 3 ? k - az : 0;
    if (ci < 0 || ci >= cx || cj < 0 || cj >= cy || ck < 0 || ck >= cz) continue;
    const int cell = (ck * cy + cj) * cx + ci;
    const float* Vr = Vs + (size_t)(a * C + c) * L * ncell + cell;
    float v[L];
#pragma unroll
    for (int jj = 0; jj < L; ++jj) v[jj] = __ldg(Vr + (size_t)jj * ncell);
    float p[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int jj = 0; jj < L; ++jj) {
      const int b = jj / C, cb = jj % C;
      const int dx = (b & 1) - ax, dy = ((b >> 1) & 1) - ay, dz = D == 3 ? ((b >> 2) & 1) - az : 0;
      const int q = (dy + 1) + (D == 3 ? 3 * (dz + 1) : 0);
      p[jj & 3] = fmaf(v[jj], rs[cb][q][threadIdx.x + 1 + dx], p[jj & 3]);
    }
    acc += (double)((p[0] + p[1]) + (p[2] + p[3]));
    ++cnt;
  }
  const size_t o = (size_t)s * C * g.np + (size_t)c * g.np + n;
  const double z = acc / cnt;
  xout[o] = (FIRST ? 0.0 : xin[o]) + omega * z;
}

// ---------------------------------------------------------------- Vanka sweep in block-stencil form
// One additive Vanka sweep is the LINEAR map  x += Sm r  with
//   Sm = omega * W * sum_c P_c^T A_c^{-1} P_c ,   W = 1 / (cells sharing the node),
// and Sm couples a node only to the nodes it shares a cell with: it is a
// block stencil with the footprint of A itself (3^d offsets x C x C per node).
// Assembled once per hierarchy build it replaces the 2^d C x 2^d C inverse of
// every cell (2-d: 1600 B per cell) by 3^d C^2 fp32 coefficients per node
// (2-d: 900 B) -- 0.56x the bytes of the dominant kernel of the fine step in
// 2-d, 0.42x in 3-d -- and the sweep becomes one fp32 stencil product.
//
// k_vanka_stencil_build: thread = (node n, row comp ca).  For offset o = n' - n
// and column comp cb the entry is the sum, in corner order a, over the cells
// that hold n as corner a and n' as corner a + o, of A_c^{-1}[(a,ca)][(a+o,cb)]
// (fp32 storage, summed in fp64), times omega / count(n), rounded once to
// fp32.  Offsets without a common cell get an explicit zero (the sweep reads
// every offset with a clamped neighbour index).  Deterministic, no atomics.
template <int D>
__global__ void __launch_bounds__(32 * (2 * D + 1)) k_vanka_stencil_build(Grid g, const float* __restrict__ Vinv,
                                                                         float* __restrict__ Sm, double omega,
                                                                         const int* __restrict__ active) {
  pdl_wait();
  constexpr int C = Cells<D>::C;
  constexpr int A = Cells<D>::A;
  constexpr int L = Cells<D>::L;
  constexpr int NOFF = D == 2 ? 9 : 27;
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  const int n = blockIdx.x * 32 + threadIdx.x;
  if (n >= g.nn) return;
  const int ca = threadIdx.y;
  int i, j, k;
  node_coords(g, n, i, j, k);
  const int cx = g.n[0] - 1, cy = g.n[1] - 1, cz = D == 3 ? g.n[2] - 1 : 1;
  const int ncell = cx * cy * cz;
  const float* Vs = Vinv + (size_t)s * L * L * ncell;
  int cell_of[A];
  int cnt = 0;
#pragma unroll
  for (int a = 0; a < A; ++a) {
    const int ci = i - (a & 1), cj = j - ((a >> 1) & 1), ck = D == 3 ? k - ((a >> 2) & 1) : 0;
    const bool ok = ci >= 0 && ci < cx && cj >= 0 && cj < cy && ck >= 0 && ck < cz;
    cell_of[a] = ok ? (ck * cy + cj) * cx + ci : -1;
    cnt += ok ? 1 : 0;
  }
  const double wgt = omega / cnt;
  float* So = Sm + (size_t)s * NOFF * C * C * g.np + (size_t)ca * C * g.np + n;
#pragma unroll 1
  for (int o = 0; o < NOFF; ++o) {
    int di, dj, dk;
    offset_delta(o, D, di, dj, dk);
    double acc[C];
#pragma unroll
    for (int cb = 0; cb < C; ++cb) acc[cb] = 0.0;
#pragma unroll
    for (int a = 0; a < A; ++a) {
      const int bx = (a & 1) + di, by = ((a >> 1) & 1) + dj, bz = D == 3 ? ((a >> 2) & 1) + dk : 0;
      if (cell_of[a] < 0 || bx < 0 || bx > 1 || by < 0 || by > 1 || bz < 0 || bz > 1) continue;
      const int b = bx + 2 * by + 4 * bz;
      PINT_CHECK_IDX(b >= 0 && b < A && cell_of[a] < ncell && o < NOFF);
      const float* Vr = Vs + ((size_t)(a * C + ca) * L + (size_t)b * C) * ncell + cell_of[a];
#pragma unroll
      for (int cb = 0; cb < C; ++cb) acc[cb] += (double)__ldg(Vr + (size_t)cb * ncell);
    }
#pragma unroll
    for (int cb = 0; cb < C; ++cb) So[((size_t)o * C * C + cb) * g.np] = (float)(wgt * acc[cb]);
  }
}

// x_out = x_in + Sm r  (FIRST: x_out = Sm r), fp32 arithmetic like the cell
// form (k_vanka_cell / k_vanka_apply): thread = (node, row comp); the block's
// residual neighbourhood (3^{D-1} node-row ranges of 34 nodes, all components,
// converted to fp32) is staged in shared memory; the NOFF*C coefficients of
// the row are loaded coalesced across the 32 nodes of the warp, in batches of
// one offset plane (2-d: all 45 in flight; 3-d: 63), and accumulated into four
// partial sums in a fixed order.  wsrc / hn / vout: the deferred basis scaling
// of k_vanka_apply (v_j = w / h formed here, bitwise k_scale_inv).
template <int D, bool FIRST>
__global__ void __launch_bounds__(32 * (2 * D + 1)) k_vanka_stencil_apply(Grid g, const float* __restrict__ Sm,
                                                                         const double* __restrict__ r,
                                                                         const double* __restrict__ xin,
                                                                         double* __restrict__ xout,
                                                                         const int* __restrict__ active,
                                                                         unsigned long long* __restrict__ work,
                                                                         const double* __restrict__ wsrc = nullptr,
                                                                         const double* __restrict__ hn = nullptr,
                                                                         double* __restrict__ vout = nullptr) {
  pdl_wait();
  constexpr int C = Cells<D>::C;
  constexpr int NOFF = D == 2 ? 9 : 27;
  double inv = 1.0;
  if (wsrc) {
    const double al = hn[blockIdx.y];
    inv = al != 0.0 ? 1.0 / al : 0.0;
    r = wsrc;
  }
  constexpr int R = D == 2 ? 3 : 9;
  constexpr int W = 34;
  __shared__ float rs[C][R][W];
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  if (work && blockIdx.x == 0 && threadIdx.x == 0 && threadIdx.y == 0) atomicAdd(work, 1ULL);
  const int n0 = blockIdx.x * 32;
  const int nx = g.n[0], nxy = g.n[0] * g.n[1];
  const double* rsl = r + (size_t)s * C * g.np;
  for (int idx = threadIdx.y * 32 + threadIdx.x; idx < C * R * W; idx += 32 * C) {
    const int w = idx % W, q = (idx / W) % R, cb = idx / (W * R);
    const int dj = q % 3 - 1, dk = D == 3 ? q / 3 - 1 : 0;
    const int m = n0 - 1 + w + dj * nx + dk * nxy;
    rs[cb][q][w] = (m >= 0 && m < g.nn) ? (float)(wsrc ? rsl[(size_t)cb * g.np + m] * inv
                                                         : __ldg(rsl + (size_t)cb * g.np + m))
                                        : 0.0f;
  }
  __syncthreads();
  const int n = n0 + threadIdx.x;
  if (n >= g.nn) return;
  const int ca = threadIdx.y;
  const size_t ov = (size_t)s * C * g.np + (size_t)ca * g.np + n;
  if (wsrc) vout[ov] = wsrc[ov] * inv;
  const float* Sr = Sm + (size_t)s * NOFF * C * C * g.np + (size_t)ca * C * g.np + n;
  float p[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
  for (int o0 = 0; o0 < NOFF; o0 += 9) {
    float v[9][C];
#pragma unroll
    for (int q = 0; q < 9; ++q)
#pragma unroll
      for (int cb = 0; cb < C; ++cb) v[q][cb] = ld_nc(Sr + ((size_t)(o0 + q) * C * C + cb) * g.np);
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      const int o = o0 + q;
      const int di = o % 3 - 1, row = o / 3;  // row = (dj + 1) + 3 (dk + 1): the staged node-row range
      PINT_CHECK_IDX(row >= 0 && row < R && (int)threadIdx.x + 1 + di >= 0 && (int)threadIdx.x + 1 + di < W);
#pragma unroll
      for (int cb = 0; cb < C; ++cb) p[cb & 3] = fmaf(v[q][cb], rs[cb][row][threadIdx.x + 1 + di], p[cb & 3]);
    }
  }
  const double z = (double)((p[0] + p[1]) + (p[2] + p[3]));
  xout[ov] = (FIRST ? 0.0 : xin[ov]) + z;
}

// r = b - A32 x with the neighbourhood of x staged in shared memory (fp64) and
// thread = (node, row): the same loads per thread as k_vanka_stencil_apply.
// Association order of stencil_row (offset o into partial o % 3, components in
// order, (p0 + p1) + p2): bitwise k_spmv<D, true, *, float> and k_spmv_node.
// PROLONG: the coarse-grid correction is added on the way in -- the staged
// value is x + (P e)(node) with k_prolong_add's arithmetic (prolong_sum, same
// order), the block's own nodes write it to xnew (out of place: other blocks
// still read the old x of their halo nodes), and the residual is that of the
// corrected iterate: bitwise k_prolong_add followed by the plain kernel, one
// launch and one read + write of x fewer per level and V-cycle.
// Warp roles (block = 32 nodes x (D + 2) warps): one warp per velocity row, one
// for the pressure row, and ONE for all D deformation rows -- those read 2 of
// the C coefficient planes (row_couples), so D of them weigh about as much as
// one full row (2-d: 36 vs 45 loads, 3-d: 162 vs 189).  With a warp per row the
// deformation warps finished early and idled their slots (ncu: 52 % of the
// warp slots active, 0.77 of HBM peak on c3 level 0).
// (no minimum-blocks launch bound: ptxas settles at 56 registers in 2-d on its own; an explicit bound of 1
// lets it take 116 and costs 10 % of the c3 step, caps of 40-96 registers were measured slower or equal)
// ACC32: fp32 products and partial sums (as the Vanka sweep), the staged x converted once -- no fp32 -> fp64
// conversions and fp64 FMAs in the inner loop; the result differs from the fp64 accumulation by fp32 round-off
// of a preconditioner-side residual (PINT_RESID_ACC=f32, off by default)
template <int D, bool PROLONG, bool ACC32 = false>
__global__ void __launch_bounds__(32 * (D + 2)) k_resid32_staged(Grid g, const float* __restrict__ A,
                                                               const double* __restrict__ x,
                                                               const double* __restrict__ b,
                                                               double* __restrict__ y,
                                                               const int* __restrict__ active, Grid gc,
                                                               const double* __restrict__ ec,
                                                               double* __restrict__ xnew) {
  pdl_wait();
  constexpr int C = Cells<D>::C;
  constexpr int NOFF = D == 2 ? 9 : 27;
  constexpr int R = D == 2 ? 3 : 9;
  constexpr int W = 34;
  constexpr int RC = D == 2 ? 1 : 4;  // the centre node-row range (dj = dk = 0)
  constexpr int NW = D + 2;           // warps per block
  using XT = std::conditional_t<ACC32, float, double>;
  __shared__ XT xs[C][R][W];
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  const int n0 = blockIdx.x * 32;
  const int nx = g.n[0], nxy = g.n[0] * g.n[1];
  const double* xsl = x + (size_t)s * C * g.np;
  for (int idx = threadIdx.y * 32 + threadIdx.x; idx < C * R * W; idx += 32 * NW) {
    const int w = idx % W, q = (idx / W) % R, cb = idx / (W * R);
    const int dj = q % 3 - 1, dk = D == 3 ? q / 3 - 1 : 0;
    const int m = n0 - 1 + w + dj * nx + dk * nxy;
    double v = 0.0;
    if (m >= 0 && m < g.nn) {
      v = __ldg(xsl + (size_t)cb * g.np + m);
      if constexpr (PROLONG) {
        int fi, fj, fk;
        node_coords(g, m, fi, fj, fk);
        v = v + prolong_sum<D>(gc, ec + (size_t)s * C * gc.np + (size_t)cb * gc.np, fi, fj, fk);
        PINT_CHECK_IDX(m < g.np);
        if (q == RC && w >= 1 && w <= 32) xnew[(size_t)s * C * g.np + (size_t)cb * g.np + m] = v;
      }
    }
    xs[cb][q][w] = (XT)v;
  }
  __syncthreads();
  const int n = n0 + threadIdx.x;
  if (n >= g.nn) return;
  PINT_CHECK_IDX(n >= 0 && n < g.nn && g.nn <= g.np && (int)blockDim.y == NW);
  const float* As = A + (size_t)s * NOFF * C * C * g.np + n;
  const size_t vbase = (size_t)s * C * g.np + n;
  if (PINT_PATTERN && threadIdx.y == D + 1) {
    // the D deformation rows: planes v_i and u_i only, all NOFF offsets of a row in flight
#pragma unroll 1
    for (int i = 0; i < D; ++i) {
      const int ca = D + i, c0 = i, c1 = D + i;
      const float* Ar = As + (size_t)ca * C * g.np;
      const double bv = __ldg(b + vbase + (size_t)ca * g.np);
      XT part[3] = {0, 0, 0};
      float v[NOFF][2];
#pragma unroll
      for (int o = 0; o < NOFF; ++o) {
        v[o][0] = ld_nc(Ar + ((size_t)o * C * C + c0) * g.np);
        v[o][1] = ld_nc(Ar + ((size_t)o * C * C + c1) * g.np);
      }
#pragma unroll
      for (int o = 0; o < NOFF; ++o) {
        const int di = o % 3 - 1, row = o / 3;
        part[o % 3] = fma((XT)v[o][0], xs[c0][row][threadIdx.x + 1 + di], part[o % 3]);
        part[o % 3] = fma((XT)v[o][1], xs[c1][row][threadIdx.x + 1 + di], part[o % 3]);
      }
      y[vbase + (size_t)ca * g.np] = bv - (double)((part[0] + part[1]) + part[2]);
    }
    return;
  }
  // full rows: warp y < D -> velocity row y, warp D -> the pressure row; without the
  // pattern (-DPINT_PATTERN=0) the last warp runs the deformation rows as full rows too
  const int nrows = (!PINT_PATTERN && threadIdx.y == D + 1) ? D : 1;
#pragma unroll 1
  for (int i = 0; i < nrows; ++i) {
    const int ca = threadIdx.y < D ? threadIdx.y : (threadIdx.y == D ? 2 * D : D + i);
    const float* Ar = As + (size_t)ca * C * g.np;
    const double bv = __ldg(b + vbase + (size_t)ca * g.np);
    XT part[3] = {0, 0, 0};
#pragma unroll
    for (int o0 = 0; o0 < NOFF; o0 += 9) {
      float v[9][C];
#pragma unroll
      for (int q = 0; q < 9; ++q)
#pragma unroll
        for (int cb = 0; cb < C; ++cb) v[q][cb] = ld_nc(Ar + ((size_t)(o0 + q) * C * C + cb) * g.np);
#pragma unroll
      for (int q = 0; q < 9; ++q) {
        const int o = o0 + q;
        const int di = o % 3 - 1, row = o / 3;
#pragma unroll
        for (int cb = 0; cb < C; ++cb)
          part[o % 3] = fma((XT)v[q][cb], xs[cb][row][threadIdx.x + 1 + di], part[o % 3]);
      }
    }
    y[vbase + (size_t)ca * g.np] = bv - (double)((part[0] + part[1]) + part[2]);
  }
}

}  // namespace pint

// ======================================================================
// Fused GMRES reductions: the last block to finish a slice (atomic ticket)
// sums that slice's partials in a FIXED order, so the result is the same bits
// whichever block arrives last and whatever else shares the launch.
// ======================================================================
namespace pint {

__device__ __forceinline__ bool last_block_of_slice(unsigned int* counter, unsigned int total) {
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == total - 1;
  __syncthreads();
  if (last) __threadfence();
  return last;
}

// Givens update of column j for one slice (body of k_gmres_givens)
__device__ __forceinline__ void givens_one(int s, int j, int m, double* H, double* cs, double* sn, double* gv,
                                           const double* tol, int* gm_active, int* gm_steps, int* its,
                                           double* resid, const int* cap) {
  double* h = H + (size_t)s * (m + 1) * m + (size_t)j * (m + 1);
  double* c = cs + (size_t)s * m;
  double* sv = sn + (size_t)s * m;
  double* g = gv + (size_t)s * (m + 1);
  for (int i = 0; i < j; ++i) {
    const double t = c[i] * h[i] + sv[i] * h[i + 1];
    h[i + 1] = -sv[i] * h[i] + c[i] * h[i + 1];
    h[i] = t;
  }
  const double a = h[j], b = h[j + 1];
  const double r = hypot(a, b);
  double cj = 1.0, sj = 0.0;
  if (r != 0.0) { cj = a / r; sj = b / r; }
  c[j] = cj;
  sv[j] = sj;
  h[j] = r;
  h[j + 1] = 0.0;
  g[j + 1] = -sj * g[j];
  g[j] = cj * g[j];
  gm_steps[s] = j + 1;
  its[s] += 1;
  const double res = fabs(g[j + 1]);
  resid[s] = res;
  // per-slice Krylov budget (cap = pint_krylov_opts.max_iters): a slice near
  // its budget stops alone, the rest of the batch keeps its restart cycle
  if (res <= tol[s] || b == 0.0 || j + 1 == m || its[s] >= *cap) gm_active[s] = 0;
}

// CGS pass: h[v] = <V_v, w> (mode 0) or h2[v] = <V_v, w>, h[v] += h2[v] (mode 1);
// grid (nblk, S): each block streams its chunk of w ONCE and of every V_v,
// keeping one accumulator per basis vector in registers (nv <= kMdotMax).
constexpr int kMdotMax = 32;
__global__ void __launch_bounds__(kRedThreads) k_mdot_fused(const double* __restrict__ V, size_t vstride,
                                                           const double* __restrict__ w, int nv, size_t per_slice,
                                                           double* __restrict__ partial, int nblk, int maxv,
                                                           double* __restrict__ h, int hstride, int mode,
                                                           double* __restrict__ h2, int h2stride,
                                                           unsigned int* __restrict__ counters,
                                                           const int* __restrict__ active, const int* __restrict__ active2) {
  pdl_wait();
  __shared__ double sh[kRedThreads / 32][kMdotMax];
  const int s = blockIdx.y;
  if ((active && !active[s]) || (active2 && !active2[s])) return;  // uniform per slice: the ticket count stays consistent
  const size_t base = (size_t)blockIdx.x * kRedChunk;
  const double* ws = w + s * per_slice;
  const double* vs = V + s * per_slice;
  // basis vectors in groups of 4 (few registers -> full occupancy, 16 loads in
  // flight per thread); per vector the element order is the same as one pass
  constexpr int PER = kRedChunk / kRedThreads;
  double we[PER];
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const size_t e = base + threadIdx.x + k * kRedThreads;
    we[k] = e < per_slice ? ws[e] : 0.0;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int v0 = 0; v0 < nv; v0 += 4) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const size_t e = base + threadIdx.x + k * kRedThreads;
      if (e < per_slice) {
#pragma unroll
        for (int g = 0; g < 4; ++g)
          if (v0 + g < nv) acc[g] = fma(__ldg(vs + (v0 + g) * vstride + e), we[k], acc[g]);
      }
    }
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      if (v0 + g >= nv) break;
      const double x = warp_sum(acc[g]);
      if (lane == 0) sh[wid][v0 + g] = x;
    }
  }
  __syncthreads();
  for (int v = threadIdx.x; v < nv; v += blockDim.x) {
    double t = 0.0;
    for (int q = 0; q < kRedThreads / 32; ++q) t += sh[q][v];
    partial[((size_t)s * maxv + v) * nblk + blockIdx.x] = t;
  }
  if (!last_block_of_slice(counters + s, (unsigned)nblk)) return;
  for (int vv = threadIdx.x; vv < nv; vv += blockDim.x) {
    const double t = ordered_sum(partial + ((size_t)s * maxv + vv) * nblk, nblk);
    if (mode == 0) {
      h[(size_t)s * hstride + vv] = t;
    } else {
      h2[(size_t)s * h2stride + vv] = t;
      h[(size_t)s * hstride + vv] += t;
    }
  }
  if (threadIdx.x == 0) counters[s] = 0u;
}

// narrow-grid variant (few chunks per slice): one block per (chunk, basis vector)
__global__ void __launch_bounds__(kRedThreads) k_mdot_fused_v(const double* __restrict__ V, size_t vstride,
                                                             const double* __restrict__ w, int nv, size_t per_slice,
                                                             double* __restrict__ partial, int nblk, int maxv,
                                                             double* __restrict__ h, int hstride, int mode,
                                                             double* __restrict__ h2, int h2stride,
                                                             unsigned int* __restrict__ counters,
                                                             const int* __restrict__ active, const int* __restrict__ active2) {
  pdl_wait();
  __shared__ double sh[kRedThreads / 32];
  const int s = blockIdx.z;
  const int v = blockIdx.y;
  if ((active && !active[s]) || (active2 && !active2[s])) return;
  const size_t base = (size_t)blockIdx.x * kRedChunk;
  const double* ws = w + s * per_slice;
  const double* vs = V + v * vstride + s * per_slice;
  const double acc = block_sum(chunk_dot(vs, ws, base, per_slice), sh);
  if (threadIdx.x == 0) partial[((size_t)s * maxv + v) * nblk + blockIdx.x] = acc;
  if (!last_block_of_slice(counters + s, (unsigned)(nblk * nv))) return;
  for (int vv = threadIdx.x; vv < nv; vv += blockDim.x) {
    const double t = ordered_sum(partial + ((size_t)s * maxv + vv) * nblk, nblk);
    if (mode == 0) {
      h[(size_t)s * hstride + vv] = t;
    } else {
      h2[(size_t)s * h2stride + vv] = t;
      h[(size_t)s * hstride + vv] += t;
    }
  }
  if (threadIdx.x == 0) counters[s] = 0u;
}

// h_{j+1,j} = ||w|| and the Givens update of column j; grid (nblk, S)
__global__ void __launch_bounds__(kRedThreads) k_norm_givens(const double* __restrict__ w, size_t per_slice,
                                                            double* __restrict__ partial, int nblk, int j, int m,
                                                            double* __restrict__ H, double* __restrict__ cs,
                                                            double* __restrict__ sn, double* __restrict__ gv,
                                                            const double* __restrict__ tol, int* __restrict__ gm_active,
                                                            int* __restrict__ gm_steps, int* __restrict__ its,
                                                            double* __restrict__ resid, double* __restrict__ hnorm,
                                                            unsigned int* __restrict__ counters,
                                                            const int* __restrict__ cap) {
  pdl_wait();
  __shared__ double sh[kRedThreads / 32];
  const int s = blockIdx.y;
  if (!gm_active[s]) return;
  const size_t base = (size_t)blockIdx.x * kRedChunk;
  const double* ws = w + s * per_slice;
  double acc = 0.0;
  for (int i = threadIdx.x; i < kRedChunk; i += kRedThreads) {
    const size_t e = base + i;
    if (e < per_slice) acc += ws[e] * ws[e];
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) partial[(size_t)s * nblk + blockIdx.x] = acc;
  if (!last_block_of_slice(counters + s, (unsigned)nblk)) return;
  if (threadIdx.x == 0) {
    const double t = ordered_sum(partial + (size_t)s * nblk, nblk);
    H[(size_t)s * (m + 1) * m + (size_t)j * (m + 1) + j + 1] = sqrt(t);
    hnorm[s] = sqrt(t);  // kept for v_{j+1} = w / h_{j+1,j}: the rotation zeroes H[j+1][j]
    counters[s] = 0u;
    givens_one(s, j, m, H, cs, sn, gv, tol, gm_active, gm_steps, its, resid, cap);
  }
}

// last CGS pass fused with the norm: w -= sum_v y_v V_v on this block's
// chunk (k_mupdate's order), then ||w||^2 partials in k_norm_givens' order
// over the same chunk -> bitwise the same H, Givens and w as the two kernels,
// one launch and one read of w fewer per Arnoldi step; grid (nblk, S)
__global__ void __launch_bounds__(kRedThreads) k_mupdate_norm_givens(
    double* __restrict__ w, const double* __restrict__ V, size_t vstride, const double* __restrict__ coef, int cstride,
    const double* __restrict__ coef2, int cstride2, const int* __restrict__ two_pass, int nv, size_t per_slice, double* __restrict__ partial, int nblk, int j, int m, double* __restrict__ H,
    double* __restrict__ cs, double* __restrict__ sn, double* __restrict__ gv, const double* __restrict__ tol,
    int* __restrict__ gm_active, int* __restrict__ gm_steps, int* __restrict__ its, double* __restrict__ resid,
    double* __restrict__ hnorm, unsigned int* __restrict__ counters, double* __restrict__ scale_out,
    const int* __restrict__ cap) {
  pdl_wait();
  __shared__ double sh[kRedThreads / 32];
  __shared__ double sinv;
  __shared__ int sact;
  const int s = blockIdx.y;
  if (!gm_active[s]) return;
  const size_t base = (size_t)blockIdx.x * kRedChunk;
  double* ws = w + s * per_slice;
  // slices with a second Gram-Schmidt pass subtract its coefficients (coef2),
  // the others the first pass's (their w was left alone by the second pass)
  const double* cf = (two_pass && two_pass[s]) ? coef2 + (size_t)s * cstride2 : coef + (size_t)s * cstride;
  const double* Vs = V + s * per_slice;
  // basis vectors outer, this thread's chunk elements inner: the element
  // loads of one vector are all in flight (same per-element operation order)
  constexpr int PT = kRedChunk / kRedThreads;
  double x[PT];
#pragma unroll
  for (int t = 0; t < PT; ++t) {
    const size_t e = base + threadIdx.x + t * kRedThreads;
    x[t] = e < per_slice ? ws[e] : 0.0;
  }
  for (int v = 0; v < nv; ++v) {
    const double c = cf[v];
    const double* Vv = Vs + v * vstride;
#pragma unroll
    for (int t = 0; t < PT; ++t) {
      const size_t e = base + threadIdx.x + t * kRedThreads;
      if (e < per_slice) x[t] -= c * __ldg(Vv + e);
    }
  }
  double acc = 0.0;
#pragma unroll
  for (int t = 0; t < PT; ++t) {
    const size_t e = base + threadIdx.x + t * kRedThreads;
    if (e < per_slice) {
      ws[e] = x[t];
      acc += x[t] * x[t];
    }
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) partial[(size_t)s * nblk + blockIdx.x] = acc;
  if (!last_block_of_slice(counters + s, (unsigned)nblk)) return;
  if (threadIdx.x == 0) {
    const double t = ordered_sum(partial + (size_t)s * nblk, nblk);
    H[(size_t)s * (m + 1) * m + (size_t)j * (m + 1) + j + 1] = sqrt(t);
    hnorm[s] = sqrt(t);
    counters[s] = 0u;
    givens_one(s, j, m, H, cs, sn, gv, tol, gm_active, gm_steps, its, resid, cap);
    sinv = hnorm[s] != 0.0 ? 1.0 / hnorm[s] : 0.0;
    sact = gm_active[s];
  }
  if (!scale_out) return;
  // small slices: v_{j+1} = w / h_{j+1,j} by this last block (k_scale_inv's
  // arithmetic and mask, one launch fewer); every block's w is visible after
  // the ticket fence
  __syncthreads();
  if (!sact) return;
  for (size_t e = threadIdx.x; e < per_slice; e += kRedThreads) scale_out[s * per_slice + e] = __ldcg(ws + e) * sinv;
}

}  // namespace pint

// ======================================================================
// Fused V-cycle tail: the small coarse levels of the hierarchy (a few
// hundred nodes per slice) are latency-bound when every smoothing / transfer
// phase is its own launch.  Here ONE CTA per slice runs the whole sub-cycle
// from level `first` down to the coarsest and back, with __syncthreads()
// between phases: same arithmetic (same per-row sums in the same order as
// the standalone kernels), ~15 launches per V-cycle fewer.
// ======================================================================
namespace pint {

#ifndef PINT_TAIL_P2
#define PINT_TAIL_P2 4  // lanes per row of the tail residual (2-d)
#endif
#ifndef PINT_TAIL_P3
#define PINT_TAIL_P3 8  // (3-d)
#endif
#ifndef PINT_TAIL_PV2
#define PINT_TAIL_PV2 2  // lanes per row of the tail's stencil-form Vanka sweep (2-d; measured 1 / 2 / 4: c1 7500 / 8026 / 7804, c2 7714 / 7949 / 8010)
#endif
#ifndef PINT_TAIL_PV3
#define PINT_TAIL_PV3 8  // (3-d; 4 / 8: c4 859 / 875)
#endif
constexpr int kMaxLevels = 12;

struct LevelDev {
  Grid g;
  const double* A;
  const float* vinv;
  const float* vst;  // Vanka sweep in block-stencil form (nullptr: cell inverses)
  double* rhs;
  double* xa;
  double* xb;
  double* res;
  double* sol;
  double* ycell;
  int ncell;
};

struct TailArgs {
  LevelDev lv[kMaxLevels];
  int first, last;       // levels handled: first..last (last = coarsest)
  const float* dense;    // coarsest dense inverse, fp32 [S][n][dense_ld] (nullptr: smoothing sweeps)
  int dense_ld;
  int dense_stage;       // 1: each CTA bulk-copies its rows of the inverse into shared memory at launch
  int coarse_sweeps;
  int pre, post;
  double omega;
};

template <int D>
__device__ __forceinline__ void tail_spmv_resid(const LevelDev& L, int s, const double* x, const double* b,
                                                double* out, int tid, int nth) {
  // P consecutive lanes share a row, each takes every P-th stencil offset with
  // all its loads in flight; the partial sums meet in an xor butterfly (fixed
  // order, independent of the cluster size).  One round of memory latency per
  // row instead of NOFF/3 -- the tail's phases are latency-bound.
  constexpr int C = 2 * D + 1;
  constexpr int NOFF = D == 2 ? 9 : 27;
  constexpr int P = D == 2 ? PINT_TAIL_P2 : PINT_TAIL_P3;
  constexpr int OPL = (NOFF + P - 1) / P;
  const int np = L.g.np;
  const size_t vs = (size_t)C * np;
  const int total = L.g.nn * C * P;
  const int part = tid % P;
  for (int base = 0; base < total; base += nth) {
    const int idx = base + tid;
    const bool ok = idx < total;
    const int row = ok ? idx / P : 0;
    const int ca = row / L.g.nn, n = row % L.g.nn;
    int i, j, k;
    node_coords(L.g, n, i, j, k);
    const double* Arow = L.A + (size_t)s * NOFF * C * C * np + (size_t)ca * C * np + n;
    const double* xs = x + s * vs;
    double a[OPL][C], xv[OPL][C];
#pragma unroll
    for (int q = 0; q < OPL; ++q) {
      const int off = part + P * q;
      const int nb = (ok && off < NOFF) ? neighbour(L.g, i, j, k, off) : -1;
#pragma unroll
      for (int cb = 0; cb < C; ++cb) {
        const bool use = nb >= 0 && row_couples(ca, cb, D);  // structural zeros are not loaded
        a[q][cb] = use ? ld_nc(Arow + ((size_t)off * C * C + cb) * np) : 0.0;
        xv[q][cb] = use ? ld_nc(xs + cb * np + nb) : 0.0;
      }
    }
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < OPL; ++q)
#pragma unroll
      for (int cb = 0; cb < C; ++cb) acc = fma(a[q][cb], xv[q][cb], acc);
#pragma unroll
    for (int o = P / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (ok && part == 0) {
      const size_t o = s * vs + (size_t)ca * np + n;
      out[o] = b[o] - acc;
    }
  }
}

// fused tail sweep body: thread (node, comp) applies its row of each adjacent
// cell inverse and sums the cells in corner order (same bits as
// tail_vanka_cell + tail_vanka_gather, one cluster barrier fewer per sweep)
template <int D>
__device__ __forceinline__ void tail_vanka_apply(const LevelDev& L, int s, const double* r, const double* xin,
                                                 double* xout, double omega, bool first, int tid, int nth) {
  constexpr int C = 2 * D + 1;
  constexpr int A = 1 << D;
  constexpr int LL = A * C;
  const int np = L.g.np, ncell = L.ncell;
  const int cx = L.g.n[0] - 1, cy = L.g.n[1] - 1, cz = D == 3 ? L.g.n[2] - 1 : 1;
  const int nx = L.g.n[0], nxy = L.g.n[0] * L.g.n[1];
  const double* rsl = r + (size_t)s * C * np;
  const float* Vs = L.vinv + (size_t)s * LL * LL * ncell;
  for (int idx = tid; idx < L.g.nn * C; idx += nth) {
    const int c = idx / L.g.nn, n = idx % L.g.nn;
    int i, j, k;
    node_coords(L.g, n, i, j, k);
    double acc = 0.0;
    int cnt = 0;
#pragma unroll
    for (int a = 0; a < A; ++a) {
      const int ax = a & 1, ay = (a >> 1) & 1, az = D == 3 ? (a >> 2) & 1 : 0;
      const int ci = i - ax, cj = j - ay, ck = D == 3 ? k - az : 0;
      if (ci < 0 || ci >= cx || cj < 0 || cj >= cy || ck < 0 || ck >= cz) continue;
      const int cell = (ck * cy + cj) * cx + ci;
      const float* Vr = Vs + (size_t)(a * C + c) * LL * ncell + cell;
      const int lower = n - ax - ay * nx - az * nxy;
      float p[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
      for (int jj = 0; jj < LL; ++jj) {
        const int b = jj / C, cb = jj % C;
        const int m = lower + (b & 1) + ((b >> 1) & 1) * nx + (D == 3 ? ((b >> 2) & 1) * nxy : 0);
        p[jj & 3] = fmaf(__ldg(Vr + (size_t)jj * ncell), (float)rsl[(size_t)cb * np + m], p[jj & 3]);
      }
      acc += (double)((p[0] + p[1]) + (p[2] + p[3]));
      ++cnt;
    }
    const size_t o = (size_t)s * C * np + (size_t)c * np + n;
    xout[o] = (first ? 0.0 : xin[o]) + omega * (acc / cnt);
  }
}

// the same sweep in block-stencil form (L.vst, k_vanka_stencil_build): P lanes
// per row as in tail_spmv_resid, each with every P-th offset and all its loads
// in flight, fp32 arithmetic, xor butterfly -- one round of memory latency per
// row and 3^d C instead of 2^d 2^d C coefficients
template <int D>
__device__ __forceinline__ void tail_vanka_stencil(const LevelDev& L, int s, const double* r, const double* xin,
                                                   double* xout, bool first, int tid, int nth) {
  constexpr int C = 2 * D + 1;
  constexpr int NOFF = D == 2 ? 9 : 27;
  constexpr int P = D == 2 ? PINT_TAIL_PV2 : PINT_TAIL_PV3;
  constexpr int OPL = (NOFF + P - 1) / P;
  const int np = L.g.np;
  const size_t vs = (size_t)C * np;
  const int total = L.g.nn * C * P;
  const int part = tid % P;
  const double* rs = r + s * vs;
  for (int base = 0; base < total; base += nth) {
    const int idx = base + tid;
    const bool ok = idx < total;
    const int row = ok ? idx / P : 0;
    const int ca = row / L.g.nn, n = row % L.g.nn;
    int i, j, k;
    node_coords(L.g, n, i, j, k);
    const float* Srow = L.vst + (size_t)s * NOFF * C * C * np + (size_t)ca * C * np + n;
    float a[OPL][C];
    double rv[OPL][C];
#pragma unroll
    for (int q = 0; q < OPL; ++q) {
      const int off = part + P * q;
      const int nb = (ok && off < NOFF) ? neighbour(L.g, i, j, k, off) : -1;
      PINT_CHECK_IDX(nb < L.g.nn && (!ok || (n < L.g.nn && ca < C)));
#pragma unroll
      for (int cb = 0; cb < C; ++cb) {
        a[q][cb] = nb >= 0 ? ld_nc(Srow + ((size_t)off * C * C + cb) * np) : 0.0f;
        rv[q][cb] = nb >= 0 ? ld_nc(rs + cb * np + nb) : 0.0;
      }
    }
    float acc = 0.0f;
#pragma unroll
    for (int q = 0; q < OPL; ++q)
#pragma unroll
      for (int cb = 0; cb < C; ++cb) acc = fmaf(a[q][cb], (float)rv[q][cb], acc);
#pragma unroll
    for (int o = P / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (ok && part == 0) {
      const size_t o = s * vs + (size_t)ca * np + n;
      xout[o] = (first ? 0.0 : xin[o]) + (double)acc;
    }
  }
}

template <int D>
__device__ __forceinline__ void tail_restrict(const LevelDev& F, const LevelDev& Cc, int s, int tid, int nth) {
  constexpr int C = 2 * D + 1;
  const Grid& gf = F.g;
  const Grid& gc = Cc.g;
  for (int idx = tid; idx < gc.nn * C; idx += nth) {
    const int c = idx / gc.nn, I = idx % gc.nn;
    int ci, cj, ck;
    node_coords(gc, I, ci, cj, ck);
    double acc = 0.0;
    for (int dk = (D == 3 ? -1 : 0); dk <= (D == 3 ? 1 : 0); ++dk)
      for (int dj = -1; dj <= 1; ++dj)
        for (int di = -1; di <= 1; ++di) {
          const int fi = 2 * ci + di, fj = 2 * cj + dj, fk = 2 * ck + dk;
          if (fi < 0 || fi >= gf.n[0] || fj < 0 || fj >= gf.n[1] || fk < 0 || fk >= gf.n[2]) continue;
          const double w = pweight(fi, ci) * pweight(fj, cj) * (D == 3 ? pweight(fk, ck) : 1.0);
          acc += w * F.res[(size_t)s * C * gf.np + (size_t)c * gf.np + node_index(gf, fi, fj, fk)];
        }
    Cc.rhs[(size_t)s * C * gc.np + (size_t)c * gc.np + I] = acc;
  }
}

template <int D>
__device__ __forceinline__ void tail_prolong(const LevelDev& F, const LevelDev& Cc, int s, double* xf, int tid, int nth) {
  constexpr int C = 2 * D + 1;
  const Grid& gf = F.g;
  const Grid& gc = Cc.g;
  for (int idx = tid; idx < gf.nn * C; idx += nth) {
    const int c = idx / gf.nn, f = idx % gf.nn;
    int fi, fj, fk;
    node_coords(gf, f, fi, fj, fk);
    const size_t o = (size_t)s * C * gf.np + (size_t)c * gf.np + f;
    const double xo = xf[o];
    xf[o] = xo + prolong_sum<D>(gc, Cc.sol + (size_t)s * C * gc.np + (size_t)c * gc.np, fi, fj, fk);
  }
}

// ---- bulk-copy (TMA 1-d) staging of the coarsest inverse into shared memory
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// rows of the coarsest inverse that CTA `rank` of a CL-cluster owns in the staged tail
__host__ __device__ inline int tail_dense_rows(int n, int CL) { return (n + CL - 1) / CL; }
__host__ __device__ inline size_t tail_dense_bsh_bytes(int n) { return ((size_t)n * 8 + 15) / 16 * 16; }
__host__ __device__ inline size_t tail_dense_smem(int n, int ld, int CL) {
  return 16 + tail_dense_bsh_bytes(n) + (size_t)tail_dense_rows(n, CL) * ld * 4;
}
struct TailStage {
  unsigned long long* bar;
  double* bsh;  // [n] coarse right-hand side
  float* rows;  // [rows][ld] this CTA's rows of the inverse
};
__device__ __forceinline__ TailStage tail_stage_layout(int n) {
  extern __shared__ __align__(16) unsigned char tail_smem[];
  TailStage t;
  t.bar = reinterpret_cast<unsigned long long*>(tail_smem);
  t.bsh = reinterpret_cast<double*>(tail_smem + 16);
  t.rows = reinterpret_cast<float*>(tail_smem + 16 + tail_dense_bsh_bytes(n));  // 16-B aligned for the bulk copy
  return t;
}

template <int D, int CL>
__device__ __forceinline__ void tail_dense_prefetch(const TailArgs& a, int s) {
  constexpr int C = 2 * D + 1;
  const int n = C * a.lv[a.last].g.nn;
  const TailStage t = tail_stage_layout(n);
  if (threadIdx.x == 0) {
    const int rank = blockIdx.x % CL;
    const int rq = tail_dense_rows(n, CL);
    const int r0 = rank * rq, r1 = min(n, r0 + rq);
    mbar_init(t.bar, 1);
    const unsigned bytes = r1 > r0 ? (unsigned)((size_t)(r1 - r0) * a.dense_ld * 4) : 0u;
    mbar_expect_tx(t.bar, bytes);
    const char* src = reinterpret_cast<const char*>(a.dense + (size_t)s * n * a.dense_ld + (size_t)r0 * a.dense_ld);
    char* dst = reinterpret_cast<char*>(t.rows);
    for (unsigned off = 0; off < bytes; off += 32768u)
      bulk_g2s(dst + off, src + off, min(32768u, bytes - off), t.bar);
  }
}

template <int D, int CL>
__device__ __forceinline__ void tail_dense(const TailArgs& a, const LevelDev& L, int s, const double* b, double* x,
                                           int tid, int nth) {
  constexpr int C = 2 * D + 1;
  if (!a.dense_stage) {
    dense_apply_warps<C>(L.g, a.dense, a.dense_ld, s, b, x, tid, nth);
    return;
  }
  const int n = C * L.g.nn;
  const TailStage t = tail_stage_layout(n);
  const double* bs = b + (size_t)s * C * L.g.np;
  for (int c = threadIdx.x; c < n; c += blockDim.x) t.bsh[c] = bs[(c / L.g.nn) * L.g.np + (c % L.g.nn)];
  mbar_wait(t.bar, 0);
  __syncthreads();
  const int rank = blockIdx.x % CL;
  const int rq = tail_dense_rows(n, CL);
  const int r0 = rank * rq, r1 = min(n, r0 + rq);
  const int lane = threadIdx.x & 31;
  for (int row = r0 + (threadIdx.x >> 5); row < r1; row += blockDim.x >> 5) {
    const double acc = dense_row_dot(t.rows + (size_t)(row - r0) * a.dense_ld, t.bsh, n, lane);
    if (lane == 0) x[(size_t)s * C * L.g.np + (row / L.g.nn) * L.g.np + (row % L.g.nn)] = acc;
  }
}

// barrier over the CTAs that cooperate on one slice (a thread-block cluster)
template <int CL>
__device__ __forceinline__ void tail_sync() {
  if constexpr (CL == 1) {
    __syncthreads();
  } else {
    cg::this_cluster().sync();
  }
}

// one Vanka smoothing sweep on level L: xout = xin + omega W sum_c A_c^{-1} (b - A xin)
template <int D, int CL>
__device__ __forceinline__ void tail_sweep(const LevelDev& L, int s, const double* b, const double* xin, double* xout,
                                           double omega, bool first, int tid, int nth) {
  const double* r = b;
  if (!first) {
    tail_spmv_resid<D>(L, s, xin, b, L.res, tid, nth);
    tail_sync<CL>();
    r = L.res;
  }
  if (L.vst) tail_vanka_stencil<D>(L, s, r, xin, xout, first, tid, nth);
  else tail_vanka_apply<D>(L, s, r, xin, xout, omega, first, tid, nth);
  tail_sync<CL>();
}

// x = V-cycle(b) from level a.first down; CL CTAs (one cluster) per slice
template <int D, int CL>
__device__ __forceinline__ void vcycle_tail_body(const TailArgs& a, const double* __restrict__ b_top,
                                                 double* __restrict__ x_top, const int* __restrict__ active) {
  const int s = blockIdx.x / CL;
  if (active && !active[s]) return;  // uniform over the cluster
  if (a.dense && a.dense_stage) tail_dense_prefetch<D, CL>(a, s);  // lands while the finer levels smooth
  const int tid = (blockIdx.x % CL) * blockDim.x + threadIdx.x;
  const int nth = CL * blockDim.x;
  const double* bl[kMaxLevels];
  double* cur[kMaxLevels];
  double* nxt[kMaxLevels];
  for (int l = a.first; l < a.last; ++l) {
    const LevelDev& L = a.lv[l];
    bl[l] = (l == a.first) ? b_top : L.rhs;
    cur[l] = L.xa;
    nxt[l] = L.xb;
    tail_sweep<D, CL>(L, s, bl[l], nullptr, cur[l], a.omega, true, tid, nth);
    for (int i = 1; i < a.pre; ++i) {
      tail_sweep<D, CL>(L, s, bl[l], cur[l], nxt[l], a.omega, false, tid, nth);
      double* t = cur[l]; cur[l] = nxt[l]; nxt[l] = t;
    }
    tail_spmv_resid<D>(L, s, cur[l], bl[l], L.res, tid, nth);
    tail_sync<CL>();
    tail_restrict<D>(L, a.lv[l + 1], s, tid, nth);
    tail_sync<CL>();
  }
  {
    const LevelDev& L = a.lv[a.last];
    const double* bc = (a.last == a.first) ? b_top : L.rhs;
    double* xc = (a.last == a.first) ? x_top : L.sol;
    if (a.dense) {
      tail_dense<D, CL>(a, L, s, bc, xc, tid, nth);
      tail_sync<CL>();
    } else {
      double* c0 = L.xa;
      double* c1 = L.xb;
      const int sw = a.coarse_sweeps < 1 ? 1 : a.coarse_sweeps;
      tail_sweep<D, CL>(L, s, bc, nullptr, sw == 1 ? xc : c0, a.omega, true, tid, nth);
      for (int i = 1; i < sw; ++i) {
        double* o = (i == sw - 1) ? xc : c1;
        tail_sweep<D, CL>(L, s, bc, c0, o, a.omega, false, tid, nth);
        double* t = c0; c0 = c1; c1 = t;
      }
    }
  }
  for (int l = a.last - 1; l >= a.first; --l) {
    const LevelDev& L = a.lv[l];
    tail_prolong<D>(L, a.lv[l + 1], s, cur[l], tid, nth);
    tail_sync<CL>();
    double* outp = (l == a.first) ? x_top : L.sol;
    const int post = a.post < 1 ? 1 : a.post;
    for (int i = 0; i < post; ++i) {
      double* o = (i == post - 1) ? outp : nxt[l];
      tail_sweep<D, CL>(L, s, bl[l], cur[l], o, a.omega, false, tid, nth);
      double* t = cur[l]; cur[l] = nxt[l]; nxt[l] = t;
    }
  }
}

template <int D>
__global__ void __launch_bounds__(1024) k_vcycle_tail(TailArgs a, const double* __restrict__ b_top,
                                                     double* __restrict__ x_top, const int* __restrict__ active) {
  pdl_wait();
  vcycle_tail_body<D, 1>(a, b_top, x_top, active);
}

// cluster variant: CL CTAs per slice cooperate through cluster barriers.  The
// host picks the largest CL (8, 4, 2) with S*CL CTAs in one wave; every output
// is computed by one thread with a partition-independent formula, so the
// result does not depend on CL (batch invariance).
constexpr int kTailCluster = 4;    // CTAs per slice of the fused Arnoldi kernel (PINT_FUSED=1)
constexpr int kTailThreads = 512;  // threads per CTA
template <int D, int CL>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(kTailThreads)
    k_vcycle_tail_cl(TailArgs a, const double* __restrict__ b_top, double* __restrict__ x_top,
                     const int* __restrict__ active) {
  pdl_wait();
  vcycle_tail_body<D, CL>(a, b_top, x_top, active);
}

}  // namespace pint

// ======================================================================
// Fused Arnoldi step for small meshes (level-0 rows <= kFusedRows per slice):
// one 8-CTA thread-block cluster per slice runs the whole step
//   z_j = V-cycle(v_j), w = J z_j, CGS2 against v_0..v_j, h_{j+1,j} = ||w||,
//   Givens update, v_{j+1} = w / h_{j+1,j}
// with cluster barriers between phases.  Reductions are fixed-order (thread
// strided sums -> warp tree -> CTA -> 4 CTA partials summed in rank order by
// every CTA), so the result is deterministic and independent of the batch.
// ======================================================================
namespace pint {

constexpr int kFusedRows = 8192;
constexpr int kMaxBasis = 64;

struct ArnoldiArgs {
  TailArgs vc;              // V-cycle from level 0 (vc.first == 0)
  const double* V;          // basis [m+1][S][C][np]
  double* Z;                // preconditioned directions [m][S][C][np]
  double* w;                // [S][C][np]
  size_t vstride, per_slice;
  double* H;
  double* cs;
  double* sn;
  double* gv;
  const double* tol;
  int* gm_active;
  int* gm_steps;
  int* its;
  double* resid;
  double* hnorm;
  const int* cap;           // Krylov budget (givens_one)
  double* cpart;            // [S][CL][kMaxBasis] CTA partials
  double* ybuf;             // [S][m+1] second-pass coefficients
  unsigned long long* work_bytes;  // profiling: algorithmic bytes of active slices (nullptr: off)
  unsigned long long* work_count;  // profiling: active slice-launches
  unsigned long long bytes_per_slice;
  int j, m;
};

// fixed-order CTA reduction of nv values per thread (nv <= kMaxBasis); results in sh_out[0..nv)
__device__ __forceinline__ void cta_reduce_many(double (&v)[kMaxBasis], int nv, double* sh_warp, double* sh_out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = 0; i < nv; ++i) {
    double x = v[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if (lane == 0) sh_warp[wid * kMaxBasis + i] = x;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {
    double t = 0.0;
    for (int w = 0; w < nw; ++w) t += sh_warp[w * kMaxBasis + i];
    sh_out[i] = t;
  }
  __syncthreads();
}

template <int D, int CL>
__device__ __forceinline__ void arnoldi_body(const ArnoldiArgs& a) {
  __shared__ double sh_warp[32 * kMaxBasis];
  __shared__ double sh_sum[kMaxBasis];
  __shared__ double sh_tot[kMaxBasis];
  const int s = blockIdx.x / CL;
  if (!a.gm_active[s]) return;  // uniform over the cluster
  const int rank = blockIdx.x % CL;
  const int tid = rank * blockDim.x + threadIdx.x;
  const int nth = CL * blockDim.x;
  const size_t n = a.per_slice;
  const int j = a.j, m = a.m, nv = j + 1;
  if (a.work_bytes && tid == 0) {
    atomicAdd(a.work_bytes, a.bytes_per_slice);
    atomicAdd(a.work_count, 1ULL);
  }
  double* zj = a.Z + (size_t)j * a.vstride;
  // z_j = M^{-1} v_j (V-cycle from level 0, whole hierarchy inside the cluster)
  vcycle_tail_body<D, CL>(a.vc, a.V + (size_t)j * a.vstride, zj, nullptr);
  // w = J z_j
  {
    const LevelDev& L0 = a.vc.lv[0];
    constexpr int C = 2 * D + 1;
    constexpr int NOFF = D == 2 ? 9 : 27;
    const int np = L0.g.np;
    for (int idx = tid; idx < L0.g.nn * C; idx += nth) {
      const int ca = idx / L0.g.nn, nd = idx % L0.g.nn;
      int nbs[NOFF];
      stencil_neighbours<D>(L0.g, nd, nbs);
      const double* Arow = L0.A + (size_t)s * NOFF * C * C * np + (size_t)ca * C * np + nd;
      a.w[s * n + (size_t)ca * np + nd] = stencil_row<D, 3>(Arow, zj + s * n, np, nbs, ca);
    }
  }
  tail_sync<CL>();
  double* ws = a.w + s * n;
  double* hcol = a.H + (size_t)s * (m + 1) * m + (size_t)j * (m + 1);
  for (int pass = 0; pass < 2; ++pass) {
    double acc[kMaxBasis];
    for (int i = 0; i < nv; ++i) acc[i] = 0.0;
    for (size_t e = tid; e < n; e += nth) {
      const double we = ws[e];
      for (int i = 0; i < nv; ++i) acc[i] += a.V[(size_t)i * a.vstride + s * n + e] * we;
    }
    cta_reduce_many(acc, nv, sh_warp, sh_sum);
    for (int i = threadIdx.x; i < nv; i += blockDim.x) a.cpart[((size_t)s * CL + rank) * kMaxBasis + i] = sh_sum[i];
    tail_sync<CL>();
    for (int i = threadIdx.x; i < nv; i += blockDim.x) {
      double t = 0.0;
      for (int r = 0; r < CL; ++r) t += a.cpart[((size_t)s * CL + r) * kMaxBasis + i];
      sh_tot[i] = t;
    }
    __syncthreads();
    if (rank == 0)
      for (int i = threadIdx.x; i < nv; i += blockDim.x) {
        if (pass == 0) hcol[i] = sh_tot[i];
        else { a.ybuf[(size_t)s * (m + 1) + i] = sh_tot[i]; hcol[i] += sh_tot[i]; }
      }
    for (size_t e = tid; e < n; e += nth) {
      double x = ws[e];
      for (int i = 0; i < nv; ++i) x -= sh_tot[i] * a.V[(size_t)i * a.vstride + s * n + e];
      ws[e] = x;
    }
    tail_sync<CL>();  // also orders the cpart reuse of the next pass
  }
  // ||w||, Givens, v_{j+1} = w / ||w||
  {
    double acc[kMaxBasis];
    acc[0] = 0.0;
    for (size_t e = tid; e < n; e += nth) acc[0] += ws[e] * ws[e];
    cta_reduce_many(acc, 1, sh_warp, sh_sum);
    if (threadIdx.x == 0) a.cpart[((size_t)s * CL + rank) * kMaxBasis] = sh_sum[0];
    tail_sync<CL>();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int r = 0; r < CL; ++r) t += a.cpart[((size_t)s * CL + r) * kMaxBasis];
      sh_tot[0] = sqrt(t);
    }
    __syncthreads();
    const double hn = sh_tot[0];
    const double inv = hn != 0.0 ? 1.0 / hn : 0.0;
    double* vj1 = const_cast<double*>(a.V) + (size_t)(j + 1) * a.vstride + s * n;
    for (size_t e = tid; e < n; e += nth) vj1[e] = ws[e] * inv;
    tail_sync<CL>();  // every CTA has read the partials before rank 0 updates H / the mask
    if (rank == 0 && threadIdx.x == 0) {
      hcol[j + 1] = hn;
      a.hnorm[s] = hn;
      givens_one(s, j, m, a.H, a.cs, a.sn, a.gv, a.tol, a.gm_active, a.gm_steps, a.its, a.resid, a.cap);
    }
  }
}

template <int D>
__global__ void __cluster_dims__(kTailCluster, 1, 1) __launch_bounds__(kTailThreads) k_arnoldi_fused(ArnoldiArgs a) {
  pdl_wait();
  arnoldi_body<D, kTailCluster>(a);
}

}  // namespace pint
