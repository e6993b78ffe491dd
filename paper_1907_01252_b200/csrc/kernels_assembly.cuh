// K1 residual, K2 Jacobian (colour-ordered element scatter) and the
// Dirichlet / row-ownership fix-up, batched over slices (grid.z or grid.y).
//
// Determinism: elements of one colour share no node, so one launch never has
// two writers of the same entry; colours run in a fixed order, so every sum
// has a fixed association order independent of the batch composition.
#pragma once

#include "fsi_element.cuh"

namespace pint {

struct MeshDev {
  Grid g;
  int cells[3];
  const uint8_t* cell_flags;   // [cells]
  const uint8_t* node_flags;   // [nn]
  const double* profile;       // [nn] inflow x-velocity at s(t) = 1
};

template <int D>
struct ElemIndex {
  int node[1 << D];
  int cell;
  uint32_t ext_mask;
  uint8_t cflag;
};

// element (colour, t) -> node list; returns false when t is out of range
template <int D>
__device__ __forceinline__ bool colour_element(const MeshDev& m, int colour, int t, ElemIndex<D>& e) {
  int bx = colour & 1, by = (colour >> 1) & 1, bz = (colour >> 2) & 1;
  int nex = (m.cells[0] - bx + 1) >> 1;
  int ney = (m.cells[1] - by + 1) >> 1;
  int nez = D == 3 ? ((m.cells[2] - bz + 1) >> 1) : 1;
  if (t >= nex * ney * nez) return false;
  int ex = t % nex;
  int r = t / nex;
  int ey = r % ney;
  int ez = r / ney;
  int ci = 2 * ex + bx, cj = 2 * ey + by, ck = D == 3 ? 2 * ez + bz : 0;
  e.cell = (ck * m.cells[1] + cj) * m.cells[0] + ci;
  e.cflag = m.cell_flags[e.cell];
  e.ext_mask = 0;
#pragma unroll
  for (int a = 0; a < (1 << D); ++a) {
    int ax = a & 1, ay = (a >> 1) & 1, az = (a >> 2) & 1;
    int n = node_index(m.g, ci + ax, cj + ay, D == 3 ? ck + az : 0);
    e.node[a] = n;
    bool allowed = (e.cflag & kCellSolid) || !(m.node_flags[n] & kSolidTouch);
    if (allowed) e.ext_mask |= (1u << a);
  }
  return true;
}

template <int D>
struct SrcValue {
  const double* y;
  const double* yold;
  int np;
  const int* node;
  __device__ __forceinline__ double yn(int a, int c) const { return __ldg(y + c * np + node[a]); }
  __device__ __forceinline__ double yo(int a, int c) const { return __ldg(yold + c * np + node[a]); }
};

template <int D>
struct SrcUnitDir {
  const double* y;
  const double* yold;
  int np;
  const int* node;
  int astar, cstar;
  __device__ __forceinline__ Dual yn(int a, int c) const {
    return Dual(__ldg(y + c * np + node[a]), (a == astar && c == cstar) ? 1.0 : 0.0);
  }
  __device__ __forceinline__ double yo(int a, int c) const { return __ldg(yold + c * np + node[a]); }
};

template <int D>
struct SrcVecDir {
  const double* y;
  const double* yold;
  const double* w;
  int np;
  const int* node;
  __device__ __forceinline__ Dual yn(int a, int c) const {
    return Dual(__ldg(y + c * np + node[a]), __ldg(w + c * np + node[a]));
  }
  __device__ __forceinline__ double yo(int a, int c) const { return __ldg(yold + c * np + node[a]); }
};

// ---------------------------------------------------------------- K1 residual
template <int D>
__global__ void __launch_bounds__(128) k_residual_colour(MeshDev m, Phys ph, const StepScalars* __restrict__ st,
                                                        const double* __restrict__ y, const double* __restrict__ yo,
                                                        double* __restrict__ r, int* __restrict__ degen,
                                                        const int* __restrict__ active, int colour) {
  constexpr int C = 2 * D + 1;
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  ElemIndex<D> e;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (!colour_element<D>(m, colour, t, e)) return;
  const size_t vs = (size_t)C * m.g.np;
  SrcValue<D> src{y + s * vs, yo + s * vs, m.g.np, e.node};
  double R[1 << D][C];
  bool dg = false;
  fsi_element<D, double>(ph, st[s], e.cflag, e.ext_mask, src, R, dg);
  if (dg) degen[s] = 1;  // benign: every writer stores 1
  double* rs = r + s * vs;
#pragma unroll
  for (int a = 0; a < (1 << D); ++a)
#pragma unroll
    for (int c = 0; c < C; ++c) {
      if (c == 2 * D && (e.cflag & kCellSolid)) continue;  // solid cells own no p rows
      double* p = rs + c * m.g.np + e.node[a];
      *p += R[a][c];
    }
}

// ---------------------------------------------------------------- K2 Jacobian columns
// thread = (element of the colour, local column dof); grid (elements, cols, slices)
template <int D>
__global__ void __launch_bounds__(64) k_jacobian_colour(MeshDev m, Phys ph, const StepScalars* __restrict__ st,
                                                       const double* __restrict__ y, const double* __restrict__ yo,
                                                       double* __restrict__ J, const int* __restrict__ active,
                                                       int colour) {
  constexpr int C = 2 * D + 1;
  constexpr int A = 1 << D;
  const int s = blockIdx.z;
  if (active && !active[s]) return;
  ElemIndex<D> e;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (!colour_element<D>(m, colour, t, e)) return;
  const int col = blockIdx.y;
  const int astar = col / C, cstar = col % C;
  const int np = m.g.np;
  const size_t vs = (size_t)C * np;
  SrcUnitDir<D> src{y + s * vs, yo + s * vs, np, e.node, astar, cstar};
  Dual R[A][C];
  bool dg = false;
  fsi_element<D, Dual>(ph, st[s], e.cflag, e.ext_mask, src, R, dg);
  const int noff = m.g.noff;
  double* Js = J + (size_t)s * noff * C * C * np;
#pragma unroll
  for (int a = 0; a < A; ++a) {
    const int di = (astar & 1) - (a & 1);
    const int dj = ((astar >> 1) & 1) - ((a >> 1) & 1);
    const int dk = D == 3 ? ((astar >> 2) & 1) - ((a >> 2) & 1) : 0;
    const int off = offset_index(di, dj, dk, D);
#pragma unroll
    for (int c = 0; c < C; ++c) {
      if (c == 2 * D && (e.cflag & kCellSolid)) continue;
      double* p = Js + (((size_t)off * C + c) * C + cstar) * np + e.node[a];
      *p += R[a][c].d;
    }
  }
}

// ---------------------------------------------------------------- Jacobian-vector product (matrix-free)
template <int D>
__global__ void __launch_bounds__(128) k_jvp_colour(MeshDev m, Phys ph, const StepScalars* __restrict__ st,
                                                   const double* __restrict__ y, const double* __restrict__ yo,
                                                   const double* __restrict__ w, double* __restrict__ out,
                                                   const int* __restrict__ active, int colour) {
  constexpr int C = 2 * D + 1;
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  ElemIndex<D> e;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (!colour_element<D>(m, colour, t, e)) return;
  const size_t vs = (size_t)C * m.g.np;
  SrcVecDir<D> src{y + s * vs, yo + s * vs, w + s * vs, m.g.np, e.node};
  Dual R[1 << D][C];
  bool dg = false;
  fsi_element<D, Dual>(ph, st[s], e.cflag, e.ext_mask, src, R, dg);
  double* os = out + s * vs;
#pragma unroll
  for (int a = 0; a < (1 << D); ++a)
#pragma unroll
    for (int c = 0; c < C; ++c) {
      if (c == 2 * D && (e.cflag & kCellSolid)) continue;
      os[c * m.g.np + e.node[a]] += R[a][c].d;
    }
}

// ---------------------------------------------------------------- fixed rows
__device__ __forceinline__ bool row_fixed(uint8_t f, int c, int D) {
  if (c < D) return f & kDirV;
  if (c < 2 * D) return f & kDirU;
  return !(f & kFluidTouch);
}

// residual rows r = y - g on Dirichlet / identity rows
template <int D>
__global__ void k_fix_residual(MeshDev m, const StepScalars* __restrict__ st, const double* __restrict__ y,
                               double* __restrict__ r, const int* __restrict__ active) {
  constexpr int C = 2 * D + 1;
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= m.g.nn) return;
  const uint8_t f = m.node_flags[n];
  const size_t vs = (size_t)C * m.g.np;
  const double ramp = st[s].ramp;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    if (!row_fixed(f, c, D)) continue;
    const double g = (c == 0) ? ramp * m.profile[n] : 0.0;
    r[s * vs + c * m.g.np + n] = y[s * vs + c * m.g.np + n] - g;
  }
}

// Jacobian rows of fixed dofs = identity rows
template <int D>
__global__ void k_fix_jacobian(MeshDev m, double* __restrict__ J, const int* __restrict__ active) {
  constexpr int C = 2 * D + 1;
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= m.g.nn) return;
  const uint8_t f = m.node_flags[n];
  const int np = m.g.np, noff = m.g.noff, ctr = center_offset(D);
  double* Js = J + (size_t)s * noff * C * C * np;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    if (!row_fixed(f, c, D)) continue;
    for (int off = 0; off < noff; ++off)
#pragma unroll
      for (int cb = 0; cb < C; ++cb)
        Js[(((size_t)off * C + c) * C + cb) * np + n] = (off == ctr && cb == c) ? 1.0 : 0.0;
  }
}

// J w on fixed rows = w
template <int D>
__global__ void k_fix_jvp(MeshDev m, const double* __restrict__ w, double* __restrict__ out,
                          const int* __restrict__ active) {
  constexpr int C = 2 * D + 1;
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= m.g.nn) return;
  const uint8_t f = m.node_flags[n];
  const size_t vs = (size_t)C * m.g.np;
#pragma unroll
  for (int c = 0; c < C; ++c)
    if (row_fixed(f, c, D)) out[s * vs + c * m.g.np + n] = w[s * vs + c * m.g.np + n];
}

}  // namespace pint
