// Shared device-side definitions for the batched ALE-FSI fine propagator.
//
// Layout: every per-slice vector is SoA by field component,
// [slice][component][Np] with Np = node count padded to a multiple of 32
// (256-byte aligned rows).  Block-stencil matrices (Jacobian and multigrid
// coarse operators) are [slice][offset][row comp][col comp][Np] so one thread
// per node reads every coefficient with unit stride across the warp.
#pragma once

#include <cstdio>

#include <cuda_runtime.h>
#include <stdint.h>

#define PINT_HD __host__ __device__ __forceinline__

namespace pint {

// Programmatic dependent launch: every kernel of the library waits here for
// the grid it depends on (a no-op when launched without the PDL attribute),
// so the host may launch it while its predecessor drains (pint_launch).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// -DPINT_BOUNDS=1: device-side index checks in the round-2 kernels (the pool's
// compute-sanitizer is closed; tools/jobs/r02_bounds.sh runs the GPU tests on
// such a build).  A failed check prints its location and traps, which surfaces
// as a CUDA error in the next API call.
#if defined(PINT_BOUNDS) && PINT_BOUNDS
#define PINT_CHECK_IDX(cond)                                                                      \
  do {                                                                                            \
    if (!(cond)) {                                                                                \
      printf("PINT_BOUNDS violated: %s at %s:%d (block %d,%d,%d thread %d,%d)\n", #cond, __FILE__, __LINE__, \
             blockIdx.x, blockIdx.y, blockIdx.z, threadIdx.x, threadIdx.y);                       \
      __trap();                                                                                   \
    }                                                                                             \
  } while (0)
#else
#define PINT_CHECK_IDX(cond) ((void)0)
#endif

constexpr int kMaxDim = 3;

struct Grid {
  int dim;          // 2 or 3
  int n[3];         // nodes per direction (cells + 1); n[2] = 1 in 2-d
  int nn;           // total nodes
  int np;           // padded node stride (multiple of 32)
  int C;            // dofs per node (2 dim + 1)
  int noff;         // stencil offsets (9 / 27)
};

PINT_HD int ipow3(int d) { return d == 2 ? 9 : 27; }

// node multi-index <-> linear index (x fastest)
PINT_HD void node_coords(const Grid& g, int node, int& i, int& j, int& k) {
  i = node % g.n[0];
  int r = node / g.n[0];
  j = r % g.n[1];
  k = r / g.n[1];
}

PINT_HD int node_index(const Grid& g, int i, int j, int k) {
  return (k * g.n[1] + j) * g.n[0] + i;
}

// stencil offset index: sum_m (delta_m + 1) 3^m over the mesh dimensions
// (0..8 in 2-d, 0..26 in 3-d)
PINT_HD int offset_index(int di, int dj, int dk, int dim) {
  return (di + 1) + 3 * (dj + 1) + (dim == 3 ? 9 * (dk + 1) : 0);
}

PINT_HD void offset_delta(int off, int dim, int& di, int& dj, int& dk) {
  di = off % 3 - 1;
  dj = (off / 3) % 3 - 1;
  dk = dim == 3 ? off / 9 - 1 : 0;
}

PINT_HD int center_offset(int dim) { return dim == 2 ? 4 : 13; }

// Structural zeros of the block-stencil operators.  A deformation row u_i --
// harmonic extension k (theta grad u_i^n + (1 - theta) grad u_i^{n-1}, grad psi) on
// fluid nodes, kinematic condition (u_i^n - u_i^{n-1}) - k (theta v_i^n + ...) on
// solid nodes, identity on fixed dofs (fsi_qfunc.cuh: uvec / uten) -- couples
// only to u_i and v_i, at every stencil offset; the Galerkin products keep the
// pattern (the transfers act per component).  The C - 2 other coefficient planes
// of such a row are exact zeros, which the product kernels neither load nor
// multiply (24 % of the operator in 2-d, 31 % in 3-d; a skipped term would add
// fma(0, x, acc) = acc, so the results are bitwise those of the full loops).
// tests/test_gpu_kernels.py::test_deformation_rows_structural_zeros checks
// the assembled planes.  -DPINT_PATTERN=0 restores the full loops.
#ifndef PINT_PATTERN
#define PINT_PATTERN 1
#endif
PINT_HD constexpr bool is_urow(int ca, int dim) { return PINT_PATTERN && ca >= dim && ca < 2 * dim; }
PINT_HD constexpr bool row_couples(int ca, int cb, int dim) { return !is_urow(ca, dim) || cb == ca || cb == ca - dim; }

// neighbour index or -1 when outside the grid
PINT_HD int neighbour(const Grid& g, int i, int j, int k, int off) {
  int di, dj, dk;
  offset_delta(off, g.dim, di, dj, dk);
  int a = i + di, b = j + dj, c = k + dk;
  if (a < 0 || a >= g.n[0] || b < 0 || b >= g.n[1] || c < 0 || c >= g.n[2]) return -1;
  return node_index(g, a, b, c);
}

// node flags (uint8)
enum : uint8_t {
  kSolidTouch = 1,
  kFluidTouch = 2,
  kDirV = 4,
  kDirU = 8,
};

// cell flags (uint8)
enum : uint8_t {
  kCellSolid = 1,
  kCellOutflow = 2,
};

// per-slice step scalars (device array of S entries)
struct StepScalars {
  double k;      // step size
  double kt;     // k * theta
  double ko;     // k * (1 - theta)
  double ramp;   // inflow ramp s(t1)
  double delta;  // pressure stabilization delta_K(k)
};

// physical parameters of the element kernel
struct Phys {
  double rho_f, rnu, rho_s, mu, lam;
  double h[3];
  double ih[3];  // 1 / h (shape gradients multiply, no fp64 division)
  double wq;     // volume quadrature weight per point
  double wf;     // outflow face quadrature weight per point
};

}  // namespace pint
