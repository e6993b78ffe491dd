// K8 Parareal correction: theta_weight + parareal_update + correction norm
// (reference parareal.py:154-197 and 422-431), on device.
#pragma once

#include "kernels_linalg.cuh"

namespace pint {

// K8a: delta = f_old - c_old for S slices (one launch)
__global__ void k_precorrect(const double* __restrict__ f, const double* __restrict__ c, double* __restrict__ d,
                             size_t total) {
  pdl_wait();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x)
    d[i] = f[i] - c[i];
}

// per-component partial dots: part[c][q][blk] for q in {<f,c>, <c,c>, <f,f>}
__global__ void __launch_bounds__(kRedThreads) k_block_dots(const double* __restrict__ f, const double* __restrict__ cn,
                                                           int nn, int np, double* __restrict__ part, int nblk) {
  pdl_wait();
  __shared__ double sh[kRedThreads / 32];
  const int comp = blockIdx.y;
  const size_t base = (size_t)blockIdx.x * kRedChunk;
  const double* fs = f + (size_t)comp * np;
  const double* cs = cn + (size_t)comp * np;
  double fc = 0.0, cc = 0.0, ff = 0.0;
  for (int i = threadIdx.x; i < kRedChunk; i += kRedThreads) {
    const size_t e = base + i;
    if (e < (size_t)nn) {
      const double a = fs[e], b = cs[e];
      fc += a * b;
      cc += b * b;
      ff += a * a;
    }
  }
  fc = block_sum(fc, sh);
  cc = block_sum(cc, sh);
  ff = block_sum(ff, sh);
  if (threadIdx.x == 0) {
    part[((size_t)comp * 3 + 0) * nblk + blockIdx.x] = fc;
    part[((size_t)comp * 3 + 1) * nblk + blockIdx.x] = cc;
    part[((size_t)comp * 3 + 2) * nblk + blockIdx.x] = ff;
  }
}

// theta (one thread): mirrors theta_weight (parareal.py:166-197)
__global__ void k_theta(const double* __restrict__ part, int nblk, int C, int variant, double lo, double hi,
                        double* __restrict__ theta) {
  pdl_wait();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (variant == 0) { *theta = 1.0; return; }
  const double degenerate = 1e-28;
  double sum = 0.0;
  for (int c = 0; c < C; ++c) {
    double fc = 0.0, cc = 0.0, ff = 0.0;
    for (int b = 0; b < nblk; ++b) {
      fc += part[((size_t)c * 3 + 0) * nblk + b];
      cc += part[((size_t)c * 3 + 1) * nblk + b];
      ff += part[((size_t)c * 3 + 2) * nblk + b];
    }
    double w;
    if (cc <= degenerate) {
      w = 1.0;
    } else if (variant == 1) {
      w = fc / cc;
    } else {
      const double denom = cc * ff;
      w = denom > degenerate * degenerate ? fc / denom : 1.0;
    }
    if (!isfinite(w)) w = 1.0;
    sum += w;
  }
  const double mean = sum / C;
  *theta = fmin(fmax(mean, lo), hi);
}

// x_new = (theta c_new + f_old) - theta c_old ; partial ||x_new - x_prev||^2, ||x_new||^2
__global__ void __launch_bounds__(kRedThreads) k_update_norms(const double* __restrict__ cn, const double* __restrict__ f,
                                                             const double* __restrict__ co, const double* __restrict__ xp,
                                                             double* __restrict__ xn, const double* __restrict__ theta,
                                                             int nn, int np, double* __restrict__ part, int nblk) {
  pdl_wait();
  __shared__ double sh[kRedThreads / 32];
  const int comp = blockIdx.y;
  const double th = *theta;
  const size_t base = (size_t)blockIdx.x * kRedChunk;
  const size_t o = (size_t)comp * np;
  double dd = 0.0, nn2 = 0.0;
  for (int i = threadIdx.x; i < kRedChunk; i += kRedThreads) {
    const size_t e = base + i;
    if (e < (size_t)nn) {
      const double v = (th * cn[o + e] + f[o + e]) - th * co[o + e];
      xn[o + e] = v;
      const double df = v - xp[o + e];
      dd += df * df;
      nn2 += v * v;
    }
  }
  dd = block_sum(dd, sh);
  nn2 = block_sum(nn2, sh);
  if (threadIdx.x == 0) {
    part[((size_t)comp * 2 + 0) * nblk + blockIdx.x] = dd;
    part[((size_t)comp * 2 + 1) * nblk + blockIdx.x] = nn2;
  }
}

__global__ void k_corr(const double* __restrict__ part, int nblk, int C, double* __restrict__ out) {
  pdl_wait();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double dd = 0.0, n2 = 0.0;
  for (int c = 0; c < C; ++c)
    for (int b = 0; b < nblk; ++b) {
      dd += part[((size_t)c * 2 + 0) * nblk + b];
      n2 += part[((size_t)c * 2 + 1) * nblk + b];
    }
  const double diff = sqrt(dd), norm = sqrt(n2);
  double corr;
  if (diff == 0.0) corr = 0.0;
  else corr = norm > 0.0 ? diff / norm : __longlong_as_double(0x7ff0000000000000LL);
  out[0] = corr;
}

}  // namespace pint
