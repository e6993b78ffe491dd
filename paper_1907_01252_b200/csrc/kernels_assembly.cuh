// K1 residual, K2 Jacobian (colour-ordered element scatter), K2' J w, and the
// Dirichlet / row-ownership fix-up, batched over slices.
//
// All three element kernels run the pointwise flux of fsi_qfunc.cuh at the
// 2^d Gauss points (and the outflow face points) of their element; only the
// scalar type and the seeding differ.  Determinism: elements of one colour
// share no node, so one launch never has two writers of the same entry;
// colours run in a fixed order, so every sum has a fixed association order
// independent of the batch composition.
#pragma once

#include "fsi_qfunc.cuh"

// resident 128-thread CTAs per SM the element kernels are compiled for:
// 4 in 2-d (128 registers), 2 in 3-d (the 3-d flux needs ~250 registers)
template <int D>
struct ElemOcc {
  static constexpr int value = D == 2 ? 4 : 2;
};

namespace pint {

struct MeshDev {
  Grid g;
  int cells[3];
  const uint8_t* cell_flags;   // [cells]
  const uint8_t* node_flags;   // [nn]
  const double* profile;       // [nn] inflow x-velocity at s(t) = 1
};

// row (node flags f, component c) is a Dirichlet / identity row
__device__ __forceinline__ bool row_fixed(uint8_t f, int c, int D) {
  if (c < D) return f & kDirV;
  if (c < 2 * D) return f & kDirU;
  return !(f & kFluidTouch);
}

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
  const int bx = colour & 1, by = (colour >> 1) & 1, bz = (colour >> 2) & 1;
  const int nex = (m.cells[0] - bx + 1) >> 1;
  const int ney = (m.cells[1] - by + 1) >> 1;
  const int nez = D == 3 ? ((m.cells[2] - bz + 1) >> 1) : 1;
  if (t >= nex * ney * nez) return false;
  const int ex = t % nex;
  const int r = t / nex;
  const int ey = r % ney;
  const int ez = r / ney;
  const int ci = 2 * ex + bx, cj = 2 * ey + by, ck = D == 3 ? 2 * ez + bz : 0;
  e.cell = (ck * m.cells[1] + cj) * m.cells[0] + ci;
  e.cflag = m.cell_flags[e.cell];
  e.ext_mask = 0;
#pragma unroll
  for (int a = 0; a < (1 << D); ++a) {
    const int n = node_index(m.g, ci + (a & 1), cj + ((a >> 1) & 1), D == 3 ? ck + ((a >> 2) & 1) : 0);
    e.node[a] = n;
    const bool allowed = (e.cflag & kCellSolid) || !(m.node_flags[n] & kSolidTouch);
    if (allowed) e.ext_mask |= (1u << a);
  }
  return true;
}

template <int D>
__device__ __forceinline__ void zero_acc(double (&acc)[1 << D][2 * D + 1]) {
#pragma unroll
  for (int a = 0; a < (1 << D); ++a)
#pragma unroll
    for (int c = 0; c < 2 * D + 1; ++c) acc[a][c] = 0.0;
}

// Contribution of ONE quadrature point q (and, on outflow cells, of face
// point q when q < 2^(d-1)) to the element integral of the CN residual
// (MODE 0), of J w (MODE 1, w given) or of one Jacobian column (MODE 2, trial
// function (astar, cstar)).  2^d consecutive lanes own the 2^d points of one
// element; their partial sums are combined by an xor butterfly, which yields
// bit-identical totals in every lane (fp addition is commutative), so the
// result is deterministic and independent of the batch.
template <int D, int MODE, int G = 0>
__device__ __forceinline__ void qp_integral(const Phys& ph, const StepScalars& st, const ElemIndex<D>& e, int q,
                                            const double* __restrict__ y, const double* __restrict__ yo,
                                            const double* __restrict__ w, int np, int astar, int cstar,
                                            double (&acc)[1 << D][2 * D + 1], bool& degen) {
  constexpr int A = 1 << D;
  const bool solid = e.cflag & kCellSolid;
  auto gy = [&](int a, int c) { return __ldg(y + c * np + e.node[a]); };
  auto go = [&](int a, int c) { return __ldg(yo + c * np + e.node[a]); };
  auto gw = [&](int a, int c) { return __ldg(w + c * np + e.node[a]); };
  const int npts = ((e.cflag & kCellOutflow) && q < (A >> 1)) ? 2 : 1;
#pragma unroll 1
  for (int pt = 0; pt < npts; ++pt) {
    const bool face = pt == 1;
    double xi[D], N[A], dN[A][D];
    gauss_point<D>(q, face, xi);
    q1_shape<D>(xi, ph.ih, N, dN);
    QFields<D, double> fn, fo;
    interp<D>(N, dN, gy, fn);
    interp<D>(N, dN, go, fo);
    if (MODE == 0) {
      if (!face) {
        QFlux<D, double> fx;
        qflux<D, double, double, double>(ph, st, solid, fn, fo, fx, degen);
        accumulate<D, false>(fx, ph.wq, N, dN, e.ext_mask, acc);
      } else {
        double B[D];
        qflux_outflow<D, double, double, double>(ph, st, fn, fo, B);
#pragma unroll
        for (int a = 0; a < A; ++a)
#pragma unroll
          for (int i = 0; i < D; ++i) acc[a][i] += (-ph.wf) * (B[i] * N[a]);
      }
    } else if (MODE == 1) {
      QFields<D, double> fw;
      interp<D>(N, dN, gw, fw);
      QFields<D, Dual> fd;
      seed_fields<D>(fn, fw, fd);
      if (!face) {
        QFlux<D, Dual> fx;
        bool dg = false;
        qflux<D, Dual, Dual, Dual>(ph, st, solid, fd, fo, fx, dg);
        accumulate<D, true>(fx, ph.wq, N, dN, e.ext_mask, acc);
      } else {
        Dual B[D];
        qflux_outflow<D, Dual, Dual, Dual>(ph, st, fd, fo, B);
#pragma unroll
        for (int a = 0; a < A; ++a)
#pragma unroll
          for (int i = 0; i < D; ++i) acc[a][i] += (-ph.wf) * (B[i].d * N[a]);
      }
    } else {
      using ST = SeedTypes<D, G>;
      typename ST::F fd;
      seed_basis<D, G>(fn, cstar, N[astar], dN[astar], fd);
      if (!face) {
        QFlux<D, Dual> fx;
        bool dg = false;
        qflux<D, typename ST::TV, typename ST::TU, typename ST::TP>(ph, st, solid, fd, fo, fx, dg);
        accumulate<D, true>(fx, ph.wq, N, dN, e.ext_mask, acc);
      } else if constexpr (G != 2) {
        Dual B[D];
        qflux_outflow<D, typename ST::TV, typename ST::TU, typename ST::TP>(ph, st, fd, fo, B);
#pragma unroll
        for (int a = 0; a < A; ++a)
#pragma unroll
          for (int i = 0; i < D; ++i) acc[a][i] += (-ph.wf) * (B[i].d * N[a]);
      }
    }
  }
}

// xor-butterfly sum of acc over the 2^d lanes of one element
template <int D>
__device__ __forceinline__ void reduce_points(double (&acc)[1 << D][2 * D + 1]) {
#pragma unroll
  for (int a = 0; a < (1 << D); ++a)
#pragma unroll
    for (int c = 0; c < 2 * D + 1; ++c) {
      double v = acc[a][c];
#pragma unroll
      for (int o = 1; o < (1 << D); o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      acc[a][c] = v;
    }
}

// lane q adds the rows of local node q to the vector out: all old values are
// loaded before the first store (no load waits behind a store that might alias)
template <int D>
__device__ __forceinline__ void scatter_rows(const double (&R)[1 << D][2 * D + 1], int q, const ElemIndex<D>& e,
                                             double* __restrict__ out, int np) {
  constexpr int C = 2 * D + 1, A = 1 << D;
  const bool solid = e.cflag & kCellSolid;  // solid cells own no p rows
  double* o = out + e.node[q];
  double v[C];
#pragma unroll
  for (int c = 0; c < C; ++c) {
    double x = R[0][c];
#pragma unroll
    for (int a = 1; a < A; ++a) x = (q == a) ? R[a][c] : x;
    v[c] = x;
  }
#pragma unroll
  for (int c = 0; c < C; ++c)
    if (!(c == 2 * D && solid)) v[c] += o[c * np];
#pragma unroll
  for (int c = 0; c < C; ++c)
    if (!(c == 2 * D && solid)) o[c * np] = v[c];
}

// ---------------------------------------------------------------- K1 residual
// thread = (element of the colour, quadrature point); lane q scatters node q
template <int D>
__global__ void __launch_bounds__(128, ElemOcc<D>::value) k_residual_colour(MeshDev m, Phys ph, const StepScalars* __restrict__ st,
                                                        const double* __restrict__ y, const double* __restrict__ yo,
                                                        double* __restrict__ r, int* __restrict__ degen,
                                                        const int* __restrict__ active, int colour) {
  pdl_wait();
  constexpr int C = 2 * D + 1;
  constexpr int A = 1 << D;
  const int s = blockIdx.y;
  if (active && !active[s]) return;  // uniform per block
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int q = gt & (A - 1);
  ElemIndex<D> e;
  const bool valid = colour_element<D>(m, colour, gt / A, e);
  const size_t vs = (size_t)C * m.g.np;
  double R[A][C];
  zero_acc<D>(R);
  bool dg = false;
  if (valid) qp_integral<D, 0>(ph, st[s], e, q, y + s * vs, yo + s * vs, nullptr, m.g.np, 0, 0, R, dg);
  reduce_points<D>(R);
  if (!valid) return;
  if (dg) degen[s] = 1;  // benign: every writer stores 1
  scatter_rows<D>(R, q, e, r + s * vs, m.g.np);
}

// ---------------------------------------------------------------- K2 Jacobian columns
// thread = (element of the colour, quadrature point); grid (elements, cols, slices)
template <int D>
__global__ void __launch_bounds__(128, ElemOcc<D>::value) k_jacobian_colour(MeshDev m, Phys ph, const StepScalars* __restrict__ st,
                                                        const double* __restrict__ y, const double* __restrict__ yo,
                                                        double* __restrict__ J, const int* __restrict__ active,
                                                        int colour) {
  pdl_wait();
  constexpr int C = 2 * D + 1;
  constexpr int A = 1 << D;
  const int s = blockIdx.z;
  if (active && !active[s]) return;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int q = gt & (A - 1);
  ElemIndex<D> e;
  const bool valid = colour_element<D>(m, colour, gt / A, e);
  const int col = blockIdx.y;
  const int astar = col / C, cstar = col % C;
  const int np = m.g.np;
  const size_t vs = (size_t)C * np;
  double K[A][C];
  zero_acc<D>(K);
  bool dg = false;
  // the column's component group is uniform over the block (blockIdx.y)
  if (valid) {
    if (cstar < D)
      qp_integral<D, 2, 0>(ph, st[s], e, q, y + s * vs, yo + s * vs, nullptr, np, astar, cstar, K, dg);
    else if (cstar < 2 * D)
      qp_integral<D, 2, 1>(ph, st[s], e, q, y + s * vs, yo + s * vs, nullptr, np, astar, cstar, K, dg);
    else
      qp_integral<D, 2, 2>(ph, st[s], e, q, y + s * vs, yo + s * vs, nullptr, np, astar, cstar, K, dg);
  }
  reduce_points<D>(K);
  if (!valid) return;
  double* Js = J + (size_t)s * m.g.noff * C * C * np;
  const int a = q;  // this lane scatters the rows of local node a
  const int di = (astar & 1) - (a & 1);
  const int dj = ((astar >> 1) & 1) - ((a >> 1) & 1);
  const int dk = D == 3 ? ((astar >> 2) & 1) - ((a >> 2) & 1) : 0;
  const int off = offset_index(di, dj, dk, D);
  double* o = Js + ((size_t)off * C * C + cstar) * np + e.node[a];
  const bool solid = e.cflag & kCellSolid;
  double v[C];
#pragma unroll
  for (int c = 0; c < C; ++c) {
    double x = K[0][c];
#pragma unroll
    for (int b = 1; b < A; ++b) x = (a == b) ? K[b][c] : x;
    v[c] = x;
  }
#pragma unroll
  for (int c = 0; c < C; ++c)
    if (!(c == 2 * D && solid)) v[c] += o[(size_t)c * C * np];
#pragma unroll
  for (int c = 0; c < C; ++c)
    if (!(c == 2 * D && solid)) o[(size_t)c * C * np] = v[c];
}

// ---------------------------------------------------------------- K2 Jacobian by pointwise linearisation
// The element Jacobian column (b, c') is  sum_q W t(a,q)^T dF_q t(b,q)  with
// t(b,q) = (N_b, grad N_b) at point q: the flux derivative along a trial
// function is linear in its (value, gradient) seed.  So per (element, point)
// and column component c' only 1 + D pointwise dual passes are needed (not
// 2^D, one per column), and the fields are interpolated once per c' (not
// once per column).
//   phase 1  thread = (element, point q): G[c][o][i] = derivative of the flux
//            output o (0: value-tested, 1+j: tested with d/dx_j) of row
//            component c along seed i (0: value of c', 1+k: d/dx_k of c');
//            outflow face points add GF[c][i] for the momentum rows.  G lives
//            in shared memory ([entry][thread], conflict-free).
//   phase 2  thread = (element, local node a): K[a][c][b] = sum over points in
//            a fixed order (deterministic), scattered to the block stencil.
// Grid (element groups, C column components, slices); colour-ordered
// scatter as in k_jacobian_colour.
template <int D>
struct JacLin {
  static constexpr int A = 1 << D;
  static constexpr int C = 2 * D + 1;
  static constexpr int NS = 1 + D;               // seeds / test kinds per component
  static constexpr int EPB = D == 2 ? 32 : 8;    // elements per block
  static constexpr int T = EPB * A;              // threads per block
  static constexpr int OCC = D == 2 ? 3 : 3;     // resident blocks per SM
  static constexpr int GSZ = C * NS * NS;        // volume entries per (element, point)
  static constexpr int FSZ = D * NS;             // face entries per (element, face point)
  static constexpr int TVSZ = A * A * NS;        // volume shape table
  static constexpr int TFSZ = (A / 2) * A * NS;  // face shape table
  static constexpr size_t smem = sizeof(double) * ((size_t)(GSZ + FSZ) * T + TVSZ + TFSZ) + sizeof(int) * A * EPB;
  static_assert(2 * C * A * EPB <= (GSZ + FSZ) * T, "node staging must fit the G region");
  static_assert((2 * C * A * EPB) % T == 0, "staging loads per thread");
};

#ifndef PINT_JACLIN_NT
#define PINT_JACLIN_NT 1  // tangents per flux pass of the 3-d colour-path Jacobian (2: two DualV<2> passes)
#endif
template <int D, int G>
__device__ __forceinline__ void jaclin_point(const Phys& ph, const StepScalars& st, const ElemIndex<D>& e, int q,
                                             const double* __restrict__ y, const double* __restrict__ yo, int np,
                                             int cp, double* __restrict__ sg, int T, const double* __restrict__ tv,
                                             const double* __restrict__ tf, const QFields<D, double>& fn,
                                             const QFields<D, double>& fo) {
  constexpr int A = 1 << D, NS = 1 + D;
  // shape values / gradients of point q from the block's tables ([b][NS])
  auto shape = [&](const double* t, double (&N)[A], double (&dN)[A][D]) {
#pragma unroll
    for (int b = 0; b < A; ++b) {
      N[b] = t[b * NS];
#pragma unroll
      for (int k = 0; k < D; ++k) dN[b][k] = t[b * NS + 1 + k];
    }
  };
  using ST = SeedTypes<D, G>;
  const bool solid = e.cflag & kCellSolid;
  auto gy = [&](int a, int c) { return __ldg(y + c * np + e.node[a]); };
  auto go = [&](int a, int c) { return __ldg(yo + c * np + e.node[a]); };
  if constexpr (D == 3 && PINT_JACLIN_NT > 1) {
    // volume point, 3-d: the 1 + d directions in passes of PINT_JACLIN_NT tangents (DualV): the primal part
    // of the flux and its divisions are shared by the tangents of a pass
    constexpr int NT = PINT_JACLIN_NT;
    using DT = DualV<NT>;
    using SV = SeedTypes<D, G, DT>;
#pragma unroll 1
    for (int dir0 = 0; dir0 < NS; dir0 += NT) {
      typename SV::F fd;
      seed_dirs<D, G, NT>(fn, cp, dir0, fd);
      QFlux<D, DT> fx;
      bool dg = false;
      qflux<D, typename SV::TV, typename SV::TU, typename SV::TP>(ph, st, solid, fd, fo, fx, dg);
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        const int dir = dir0 + k;
#pragma unroll
        for (int i = 0; i < D; ++i) {
          sg[((i * NS + 0) * NS + dir) * T] = fx.vec[i].d[k];
          sg[(((D + i) * NS + 0) * NS + dir) * T] = fx.uvec[i].d[k];
#pragma unroll
          for (int j = 0; j < D; ++j) {
            sg[((i * NS + 1 + j) * NS + dir) * T] = fx.ten[i][j].d[k];
            sg[(((D + i) * NS + 1 + j) * NS + dir) * T] = fx.uten[i][j].d[k];
          }
        }
        sg[((2 * D * NS + 0) * NS + dir) * T] = fx.pv.d[k];
#pragma unroll
        for (int j = 0; j < D; ++j) sg[((2 * D * NS + 1 + j) * NS + dir) * T] = fx.pt[j].d[k];
      }
    }
  } else {
    // volume point: fields interpolated by the caller from the staged node values
#pragma unroll 1
    for (int dir = 0; dir < NS; ++dir) {
      typename ST::F fd;
      seed_dir<D, G>(fn, cp, dir, fd);
      QFlux<D, Dual> fx;
      bool dg = false;
      qflux<D, typename ST::TV, typename ST::TU, typename ST::TP>(ph, st, solid, fd, fo, fx, dg);
#pragma unroll
      for (int i = 0; i < D; ++i) {
        sg[((i * NS + 0) * NS + dir) * T] = fx.vec[i].d;
        sg[(((D + i) * NS + 0) * NS + dir) * T] = fx.uvec[i].d;
#pragma unroll
        for (int j = 0; j < D; ++j) {
          sg[((i * NS + 1 + j) * NS + dir) * T] = fx.ten[i][j].d;
          sg[(((D + i) * NS + 1 + j) * NS + dir) * T] = fx.uten[i][j].d;
        }
      }
      sg[((2 * D * NS + 0) * NS + dir) * T] = fx.pv.d;
#pragma unroll
      for (int j = 0; j < D; ++j) sg[((2 * D * NS + 1 + j) * NS + dir) * T] = fx.pt[j].d;
    }
  }
  constexpr int GSZ = (2 * D + 1) * NS * NS;
  if constexpr (G != 2) {
   if ((e.cflag & kCellOutflow) && q < (A >> 1)) {  // rare (outflow column): gathered from global memory
    double N[A], dN[A][D];
    shape(tf + q * A * NS, N, dN);
    QFields<D, double> gn, gold;
    interp<D>(N, dN, gy, gn);
    interp<D>(N, dN, go, gold);
#pragma unroll 1
    for (int dir = 0; dir < NS; ++dir) {
      typename ST::F fd;
      seed_dir<D, G>(gn, cp, dir, fd);
      Dual B[D];
      qflux_outflow<D, typename ST::TV, typename ST::TU, typename ST::TP>(ph, st, fd, gold, B);
#pragma unroll
      for (int i = 0; i < D; ++i) sg[(GSZ + i * NS + dir) * T] = B[i].d;
    }
   }
  }
}

template <int D>
__global__ void __launch_bounds__(JacLin<D>::T, JacLin<D>::OCC) k_jacobian_lin(MeshDev m, Phys ph, const StepScalars* __restrict__ st,
                                                         const double* __restrict__ y, const double* __restrict__ yo,
                                                         double* __restrict__ J, const int* __restrict__ active,
                                                         int colour) {
  pdl_wait();
  using L = JacLin<D>;
  constexpr int A = L::A, C = L::C, NS = L::NS, T = L::T;
  extern __shared__ double sm[];
  double* tv = sm + (size_t)(L::GSZ + L::FSZ) * T;  // [q][b][NS]
  double* tf = tv + L::TVSZ;                        // [face q][b][NS]
  const int s = blockIdx.z;
  if (active && !active[s]) return;  // uniform per block
  const int cp = blockIdx.y;
  const int lane = threadIdx.x;
  const int q = lane & (A - 1);
  // shape tables (uniform mesh: identical for every element)
  if (lane < A + (A >> 1)) {
    const bool face = lane >= A;
    double xi[D], N[A], dN[A][D];
    gauss_point<D>(face ? lane - A : lane, face, xi);
    q1_shape<D>(xi, ph.ih, N, dN);
    double* t = face ? tf + (lane - A) * A * NS : tv + lane * A * NS;
#pragma unroll
    for (int b = 0; b < A; ++b) {
      t[b * NS] = N[b];
#pragma unroll
      for (int k = 0; k < D; ++k) t[b * NS + 1 + k] = dN[b][k];
    }
  }
  ElemIndex<D> e;
  constexpr int EPB = L::EPB;
  const int el = lane / A;
  const bool valid = colour_element<D>(m, colour, blockIdx.x * EPB + el, e);
  const size_t vs = (size_t)C * m.g.np;
  const bool outflow = valid && (e.cflag & kCellOutflow);
  const double* ys = y + s * vs;
  const double* yos = yo + s * vs;
  // stage the node values of the block's elements ([lvl][c][a][e], in the G
  // region, which phase 1 overwrites only after the fields are interpolated):
  // every load of the block in flight at once instead of per-point gathers
  int* snode = reinterpret_cast<int*>(tf + L::TFSZ);
  if (q == 0) {
#pragma unroll
    for (int a = 0; a < A; ++a) snode[a * EPB + el] = valid ? e.node[a] : -1;
  }
  __syncthreads();  // shape tables, node table
  {
    constexpr int PER = 2 * C * A * EPB / T;
    double v[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int idx = lane + k * T;
      const int ee = idx % EPB, a = (idx / EPB) % A, c = (idx / (EPB * A)) % C, lvl = idx / (EPB * A * C);
      const int nd = snode[a * EPB + ee];
      v[k] = nd >= 0 ? __ldg((lvl == 0 ? ys : yos) + (size_t)c * m.g.np + nd) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < PER; ++k) sm[lane + k * T] = v[k];
  }
  __syncthreads();
  QFields<D, double> fn, fo;
  if (valid) {
    double N[A], dN[A][D];
    const double* t = tv + q * A * NS;
#pragma unroll
    for (int b = 0; b < A; ++b) {
      N[b] = t[b * NS];
#pragma unroll
      for (int k = 0; k < D; ++k) dN[b][k] = t[b * NS + 1 + k];
    }
    interp<D>(N, dN, [&](int a, int c) { return sm[((0 * C + c) * A + a) * EPB + el]; }, fn);
    interp<D>(N, dN, [&](int a, int c) { return sm[((1 * C + c) * A + a) * EPB + el]; }, fo);
  }
  __syncthreads();  // the staging area becomes G
  if (valid) {
    if (cp < D)
      jaclin_point<D, 0>(ph, st[s], e, q, ys, yos, m.g.np, cp, sm + lane, T, tv, tf, fn, fo);
    else if (cp < 2 * D)
      jaclin_point<D, 1>(ph, st[s], e, q, ys, yos, m.g.np, cp, sm + lane, T, tv, tf, fn, fo);
    else
      jaclin_point<D, 2>(ph, st[s], e, q, ys, yos, m.g.np, cp, sm + lane, T, tv, tf, fn, fo);
  }
  __syncthreads();
  if (!valid) return;
  // phase 2: this lane owns local node a = q of its element
  const int a = q;
  const int base = lane - q;  // lane of point 0 of this element
  const bool ext = (e.ext_mask >> a) & 1;
  double K[C][A];
#pragma unroll
  for (int c = 0; c < C; ++c)
#pragma unroll
    for (int b = 0; b < A; ++b) K[c][b] = 0.0;
#pragma unroll 1
  for (int qq = 0; qq < A; ++qq) {
    const double* g = sm + base + qq;
    const double* ta = tv + (qq * A + a) * NS;
    double ta_r[NS];
#pragma unroll
    for (int o = 0; o < NS; ++o) ta_r[o] = ta[o];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      if (!row_couples(c, cp, D)) continue;  // structural zero plane: never computed, never scattered
      // u rows of a node without the extension row: value-tested part only
      const bool full = !(c >= D && c < 2 * D) || ext;
      double h[NS];
#pragma unroll
      for (int i = 0; i < NS; ++i) {
        double v = g[((c * NS + 0) * NS + i) * T] * ta_r[0];
        if (full) {
#pragma unroll
          for (int o = 1; o < NS; ++o) v += g[((c * NS + o) * NS + i) * T] * ta_r[o];
        }
        h[i] = ph.wq * v;
      }
#pragma unroll
      for (int b = 0; b < A; ++b) {
        const double* tb = tv + (qq * A + b) * NS;
        double v = h[0] * tb[0];
#pragma unroll
        for (int k = 1; k < NS; ++k) v += h[k] * tb[k];
        K[c][b] += v;
      }
    }
  }
  if (outflow && cp < 2 * D) {
#pragma unroll 1
    for (int qq = 0; qq < (A >> 1); ++qq) {
      const double* g = sm + (size_t)L::GSZ * T + base + qq;
      const double na = tf[(qq * A + a) * NS];
#pragma unroll
      for (int c = 0; c < D; ++c) {
        double h[NS];
#pragma unroll
        for (int i = 0; i < NS; ++i) h[i] = (-ph.wf) * (g[(c * NS + i) * T] * na);
#pragma unroll
        for (int b = 0; b < A; ++b) {
          const double* tb = tf + (qq * A + b) * NS;
          double v = h[0] * tb[0];
#pragma unroll
          for (int k = 1; k < NS; ++k) v += h[k] * tb[k];
          K[c][b] += v;
        }
      }
    }
  }
  // scatter: every old value is loaded before the first store, so the C 2^d
  // read-modify-writes overlap instead of serialising behind possible aliasing
  const int np = m.g.np;
  double* o = J + (size_t)s * m.g.noff * C * C * np + (size_t)cp * np + e.node[a];
  const bool solid = e.cflag & kCellSolid;  // solid cells own no p rows
  auto idx = [&](int b, int c) {
    const int di = (b & 1) - (a & 1);
    const int dj = ((b >> 1) & 1) - ((a >> 1) & 1);
    const int dk = D == 3 ? ((b >> 2) & 1) - ((a >> 2) & 1) : 0;
    return ((size_t)offset_index(di, dj, dk, D) * C + c) * C * np;
  };
#pragma unroll
  for (int b = 0; b < A; ++b)
#pragma unroll
    for (int c = 0; c < C; ++c)
      if (!(c == 2 * D && solid) && row_couples(c, cp, D)) K[c][b] += o[idx(b, c)];
#pragma unroll
  for (int b = 0; b < A; ++b)
#pragma unroll
    for (int c = 0; c < C; ++c)
      if (!(c == 2 * D && solid) && row_couples(c, cp, D)) o[idx(b, c)] = K[c][b];
}

// ---------------------------------------------------------------- K2 Jacobian, node-owner strips (2-d default)
// The colour-ordered kernels above add every element block into the stencil
// with a read-modify-write after a zeroing pass, and a separate pass makes
// the fp32 copy: c3 moved 10.3 GB of DRAM per assembly for 1.9 GB of
// operator (ncu r02: 1.37 GB read + 1.20 GB written per colour launch), and
// long-scoreboard stalls on those reads were the largest stall reason.
// Here a block OWNS the stencil rows of a strip of W node columns x a chunk
// of node rows, for one column component cp, and sweeps the strip's cell rows
// bottom to top:
//   stage    node values of the next node row go to a 3-row ring in shared
//            memory (loads issued before phase 1, stored after it);
//   phase 1  thread = (cell of the row, Gauss point): the pointwise flux
//            derivative table G (as k_jacobian_lin, 1 + d dual passes) for the
//            W + 1 cells of the row (the left halo cell is recomputed: no cell
//            is shared between blocks for writing);
//   phase 2  thread = (node column, row component ca): contracts G of the two
//            cells left / right of the node into the 9 stencil entries of row
//            (node, ca), column component cp.  Node row cj gets its
//            bottom-corner terms from cell row cj on top of its top-corner
//            terms from cell row cj - 1 (kept in shared memory since the
//            previous row), is then complete and is written ONCE -- fp64 and
//            the fp32 copy, with the identity rows of fixed dofs -- so there is
//            no zeroing pass, no read-modify-write, no k_fix_jacobian and no
//            k_to_f32 behind it.
// Every entry is a sum in a fixed order (cell row j-1 left, right, row j
// left, right; points in order, then outflow face points): deterministic and
// independent of the batch.
struct JacStrip {
  static constexpr int A = 4, C = 5, NS = 3, D = 2;
  static constexpr int T = 128;          // threads: 32 cells x 4 points in phase 1
  static constexpr int WMAX = T / A - 1;  // owned node columns per strip (<= 31)
  static constexpr int GSZ = C * NS * NS;
  static constexpr int FSZ = D * NS;
  static constexpr int RW = WMAX + 3;    // staged node columns (cells + 1, padded)
  static constexpr int NPART = 6;        // top-corner partials: offsets with dj in {-1, 0}
  static constexpr int ITEMS = 160;      // phase-2 item slots (>= WMAX * C)
  static constexpr size_t smem = sizeof(double) * ((size_t)(GSZ + FSZ) * T + A * A * NS + (A / 2) * A * NS +
                                                   (size_t)3 * 2 * C * RW + (size_t)NPART * ITEMS);
};

template <int G>
__device__ __forceinline__ void strip_point(const Phys& ph, const StepScalars& st, bool solid, bool face_pt, int cp,
                                            const QFields<2, double>& fn, const QFields<2, double>& fo,
                                            const QFields<2, double>& gn, const QFields<2, double>& go,
                                            double* __restrict__ sg) {
  using J = JacStrip;
  constexpr int D = 2, NS = J::NS, T = J::T;
  using ST = SeedTypes<D, G>;
#pragma unroll 1
  for (int dir = 0; dir < NS; ++dir) {
    typename ST::F fd;
    seed_dir<D, G>(fn, cp, dir, fd);
    QFlux<D, Dual> fx;
    bool dg = false;
    qflux<D, typename ST::TV, typename ST::TU, typename ST::TP>(ph, st, solid, fd, fo, fx, dg);
#pragma unroll
    for (int i = 0; i < D; ++i) {
      sg[((i * NS + 0) * NS + dir) * T] = fx.vec[i].d;
      sg[(((D + i) * NS + 0) * NS + dir) * T] = fx.uvec[i].d;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        sg[((i * NS + 1 + j) * NS + dir) * T] = fx.ten[i][j].d;
        sg[(((D + i) * NS + 1 + j) * NS + dir) * T] = fx.uten[i][j].d;
      }
    }
    sg[((2 * D * NS + 0) * NS + dir) * T] = fx.pv.d;
#pragma unroll
    for (int j = 0; j < D; ++j) sg[((2 * D * NS + 1 + j) * NS + dir) * T] = fx.pt[j].d;
  }
  if constexpr (G != 2) {
    if (face_pt) {
#pragma unroll 1
      for (int dir = 0; dir < NS; ++dir) {
        typename ST::F fd;
        seed_dir<D, G>(gn, cp, dir, fd);
        Dual B[D];
        qflux_outflow<D, typename ST::TV, typename ST::TU, typename ST::TP>(ph, st, fd, go, B);
#pragma unroll
        for (int i = 0; i < D; ++i) sg[(J::GSZ + i * NS + dir) * T] = B[i].d;
      }
    }
  }
}

// the same table from ONE flux pass carrying all 1 + d directions as tangents
// (DualV<1 + d>): the primal part and the divisions are computed once per
// column component instead of once per direction, and the tangent chains are
// independent instructions.  Same derivative values up to the association of
// the products (the Jacobians agree to round-off, test_jacobian_formulations_agree).
template <int G>
__device__ __forceinline__ void strip_point_mt(const Phys& ph, const StepScalars& st, bool solid, bool face_pt, int cp,
                                               const QFields<2, double>& fn, const QFields<2, double>& fo,
                                               const QFields<2, double>& gn, const QFields<2, double>& go,
                                               double* __restrict__ sg) {
  using J = JacStrip;
  constexpr int D = 2, NS = J::NS, T = J::T;
  using DT = DualV<NS>;
  using ST = SeedTypes<D, G, DT>;
  {
    typename ST::F fd;
    seed_all<D, G>(fn, cp, fd);
    QFlux<D, DT> fx;
    bool dg = false;
    qflux<D, typename ST::TV, typename ST::TU, typename ST::TP>(ph, st, solid, fd, fo, fx, dg);
#pragma unroll
    for (int dir = 0; dir < NS; ++dir) {
#pragma unroll
      for (int i = 0; i < D; ++i) {
        sg[((i * NS + 0) * NS + dir) * T] = fx.vec[i].d[dir];
        sg[(((D + i) * NS + 0) * NS + dir) * T] = fx.uvec[i].d[dir];
#pragma unroll
        for (int j = 0; j < D; ++j) {
          sg[((i * NS + 1 + j) * NS + dir) * T] = fx.ten[i][j].d[dir];
          sg[(((D + i) * NS + 1 + j) * NS + dir) * T] = fx.uten[i][j].d[dir];
        }
      }
      sg[((2 * D * NS + 0) * NS + dir) * T] = fx.pv.d[dir];
#pragma unroll
      for (int j = 0; j < D; ++j) sg[((2 * D * NS + 1 + j) * NS + dir) * T] = fx.pt[j].d[dir];
    }
  }
  if constexpr (G != 2) {
    if (face_pt) {
      typename ST::F fd;
      seed_all<D, G>(gn, cp, fd);
      P2<typename ST::TV, typename ST::TU> B[D];
      qflux_outflow<D, typename ST::TV, typename ST::TU, typename ST::TP>(ph, st, fd, go, B);
#pragma unroll
      for (int dir = 0; dir < NS; ++dir)
#pragma unroll
        for (int i = 0; i < D; ++i) sg[(J::GSZ + i * NS + dir) * T] = B[i].d[dir];
    }
  }
}

template <bool MT>
__global__ void __launch_bounds__(JacStrip::T, 3) k_jacobian_strip(MeshDev m, Phys ph, const StepScalars* __restrict__ st,
                                                                  const double* __restrict__ y, const double* __restrict__ yo,
                                                                  double* __restrict__ J, float* __restrict__ J32,
                                                                  const int* __restrict__ active, int W, int nstrips, int H) {
  pdl_wait();
  using L = JacStrip;
  constexpr int A = L::A, C = L::C, NS = L::NS, T = L::T, D = 2, RW = L::RW;
  extern __shared__ double sm[];
  double* sg = sm;                                   // G [GSZ + FSZ][T]
  double* tv = sg + (size_t)(L::GSZ + L::FSZ) * T;   // [q][b][NS]
  double* tf = tv + A * A * NS;                      // [face q][b][NS]
  double* ring = tf + (A / 2) * A * NS;              // [slot 3][lvl 2][c][RW]
  double* part = ring + 3 * 2 * C * RW;              // [NPART][ITEMS]
  const int s = blockIdx.z;
  if (active && !active[s]) return;  // uniform per block
  const int cp = blockIdx.y;
  const int lane = threadIdx.x;
  const int nx = m.cells[0], ny = m.cells[1];        // cells
  const int strip = blockIdx.x % nstrips, chunk = blockIdx.x / nstrips;
  const int i0 = strip * W;
  const int nown = min(W, nx + 1 - i0);              // owned node columns i0 .. i0 + nown - 1
  const int j0 = chunk * H, j1 = min(j0 + H, ny + 1);  // owned node rows
  if (nown <= 0 || j0 >= j1) return;
  const int c_lo = max(i0 - 1, 0), c_hi = min(i0 + nown - 1, nx - 1);  // cell columns
  const int ncell = c_hi - c_lo + 1;
  const int ncol = ncell + 1;                        // staged node columns c_lo .. c_hi + 1
  const int cj_lo = max(j0 - 1, 0), cj_hi = min(j1 - 1, ny - 1);
  const int np = m.g.np;
  const size_t vs = (size_t)C * np;
  const double* ys = y + s * vs;
  const double* yos = yo + s * vs;
  if (lane < A + (A >> 1)) {  // shape tables (uniform mesh)
    const bool face = lane >= A;
    double xi[D], N[A], dN[A][D];
    gauss_point<D>(face ? lane - A : lane, face, xi);
    q1_shape<D>(xi, ph.ih, N, dN);
    double* t = face ? tf + (lane - A) * A * NS : tv + lane * A * NS;
#pragma unroll
    for (int b = 0; b < A; ++b) {
      t[b * NS] = N[b];
#pragma unroll
      for (int k = 0; k < D; ++k) t[b * NS + 1 + k] = dN[b][k];
    }
  }
  // node row r -> ring slot r % 3; entries [lvl][c][col]
  constexpr int PER = (2 * C * RW + T - 1) / T;
  auto load_row = [&](int r, double (&v)[PER]) {
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int idx = lane + k * T;
      const int col = idx % RW, c = (idx / RW) % C, lvl = idx / (RW * C);
      PINT_CHECK_IDX(!(lvl < 2 && col < ncol) || (c_lo + col <= nx && r >= 0 && r <= ny));
      v[k] = (lvl < 2 && col < ncol) ? __ldg((lvl == 0 ? ys : yos) + (size_t)c * np + node_index(m.g, c_lo + col, r, 0))
                                     : 0.0;
    }
  };
  auto store_row = [&](int r, const double (&v)[PER]) {
    double* dst = ring + (r % 3) * 2 * C * RW;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int idx = lane + k * T;
      if (idx < 2 * C * RW) dst[idx] = v[k];
    }
  };
  {
    double v[PER];
    load_row(cj_lo, v);
    store_row(cj_lo, v);
    load_row(cj_lo + 1, v);
    store_row(cj_lo + 1, v);
  }
  // phase 1 lane = q * 32 + lc (cell c_lo + lc, point q): G entries of one point
  // are contiguous over the cells, so phase 2 (lanes = consecutive node
  // columns) reads them without bank conflicts
  const int lc = lane % 32, q = lane / 32;
  const int nitems = nown * C;
  __syncthreads();
  for (int cj = cj_lo; cj <= cj_hi; ++cj) {
    double pre[PER];
    const bool more = cj + 2 <= min(cj_hi + 1, ny);
    if (more) load_row(cj + 2, pre);
    // ---- phase 1: G of (cell c_lo + lc, row cj) at point q
    if (lc < ncell) {
      const int ci = c_lo + lc;
      const uint8_t cf = m.cell_flags[cj * nx + ci];
      const bool solid = cf & kCellSolid;
      const double* r0 = ring + (cj % 3) * 2 * C * RW;        // node row cj
      const double* r1 = ring + ((cj + 1) % 3) * 2 * C * RW;  // node row cj + 1
      auto getter = [&](int lvl) {
        return [=](int a, int c) {
          const double* rr = (a >> 1) ? r1 : r0;
          return rr[(lvl * C + c) * RW + lc + (a & 1)];
        };
      };
      QFields<D, double> fn, fo, gn, go;
      {
        double N[A], dN[A][D];
        const double* t = tv + q * A * NS;
#pragma unroll
        for (int b = 0; b < A; ++b) {
          N[b] = t[b * NS];
#pragma unroll
          for (int k = 0; k < D; ++k) dN[b][k] = t[b * NS + 1 + k];
        }
        interp<D>(N, dN, getter(0), fn);
        interp<D>(N, dN, getter(1), fo);
      }
      const bool face_pt = (cf & kCellOutflow) && q < (A >> 1) && cp < 2 * D;
      if (face_pt) {
        double N[A], dN[A][D];
        const double* t = tf + q * A * NS;
#pragma unroll
        for (int b = 0; b < A; ++b) {
          N[b] = t[b * NS];
#pragma unroll
          for (int k = 0; k < D; ++k) dN[b][k] = t[b * NS + 1 + k];
        }
        interp<D>(N, dN, getter(0), gn);
        interp<D>(N, dN, getter(1), go);
      }
      if constexpr (MT) {
        if (cp < D)
          strip_point_mt<0>(ph, st[s], solid, face_pt, cp, fn, fo, gn, go, sg + lane);
        else if (cp < 2 * D)
          strip_point_mt<1>(ph, st[s], solid, face_pt, cp, fn, fo, gn, go, sg + lane);
        else
          strip_point_mt<2>(ph, st[s], solid, face_pt, cp, fn, fo, gn, go, sg + lane);
      } else {
        if (cp < D)
          strip_point<0>(ph, st[s], solid, face_pt, cp, fn, fo, gn, go, sg + lane);
        else if (cp < 2 * D)
          strip_point<1>(ph, st[s], solid, face_pt, cp, fn, fo, gn, go, sg + lane);
        else
          strip_point<2>(ph, st[s], solid, face_pt, cp, fn, fo, gn, go, sg + lane);
      }
    }
    if (more) store_row(cj + 2, pre);  // slot (cj + 2) % 3 = (cj - 1) % 3: not read in this row
    __syncthreads();
    // ---- phase 2: rows (node (i, cj), ca) and (node (i, cj + 1), ca)
    for (int it = lane; it < nitems; it += T) {
      const int ca = it / nown, li = it % nown;
      const int i = i0 + li;
      double K[9];
      const bool own_bottom = cj >= j0;                     // node row cj owned (else: halo row)
      const bool own_top = cj + 1 < j1;                     // node row cj + 1 owned
      const bool top_final = own_top && cj + 1 == ny;       // no cell row above: complete now
#pragma unroll
      for (int o = 0; o < 9; ++o) K[o] = 0.0;
      if (own_bottom && cj > cj_lo) {
#pragma unroll
        for (int o = 0; o < L::NPART; ++o) K[o] = part[o * L::ITEMS + it];
      }
      // contribution of cell (ci, cj) to row (a, ca): K[off(a, b)] += ...
      auto cell_terms = [&](int ci, int a, double (&Kx)[9]) {
        if (ci < 0 || ci >= nx) return;
        if (!row_couples(ca, cp, D)) return;                // structural zero plane (u_i row, column not v_i / u_i)
        const int lcell = ci - c_lo;
        PINT_CHECK_IDX(lcell >= 0 && lcell < 32 && lcell < ncell && it < L::ITEMS && cj >= 0 && cj < ny);
        const uint8_t cf = m.cell_flags[cj * nx + ci];
        const bool solid = cf & kCellSolid;
        if (ca == 2 * D && solid) return;                   // solid cells own no p rows
        const int nj = cj + (a >> 1);
        const uint8_t nf = m.node_flags[node_index(m.g, i, nj, 0)];
        const bool ext = solid || !(nf & kSolidTouch);
        const bool full = !(ca >= D && ca < 2 * D) || ext;  // u rows without the extension row: value part only
#pragma unroll 1
        for (int qq = 0; qq < A; ++qq) {
          const double* g = sg + qq * 32 + lcell;
          const double* ta = tv + (qq * A + a) * NS;
          double h[NS];
#pragma unroll
          for (int k = 0; k < NS; ++k) {
            double v = g[((ca * NS + 0) * NS + k) * T] * ta[0];
            if (full) {
#pragma unroll
              for (int o = 1; o < NS; ++o) v += g[((ca * NS + o) * NS + k) * T] * ta[o];
            }
            h[k] = ph.wq * v;
          }
#pragma unroll
          for (int b = 0; b < A; ++b) {
            const double* tb = tv + (qq * A + b) * NS;
            double v = h[0] * tb[0];
#pragma unroll
            for (int k = 1; k < NS; ++k) v += h[k] * tb[k];
            Kx[offset_index((b & 1) - (a & 1), (b >> 1) - (a >> 1), 0, D)] += v;
          }
        }
        if ((cf & kCellOutflow) && cp < 2 * D && ca < D) {
#pragma unroll 1
          for (int qq = 0; qq < (A >> 1); ++qq) {
            const double* g = sg + (size_t)L::GSZ * T + qq * 32 + lcell;
            const double na = tf[(qq * A + a) * NS];
            double h[NS];
#pragma unroll
            for (int k = 0; k < NS; ++k) h[k] = (-ph.wf) * (g[(ca * NS + k) * T] * na);
#pragma unroll
            for (int b = 0; b < A; ++b) {
              const double* tb = tf + (qq * A + b) * NS;
              double v = h[0] * tb[0];
#pragma unroll
              for (int k = 1; k < NS; ++k) v += h[k] * tb[k];
              Kx[offset_index((b & 1) - (a & 1), (b >> 1) - (a >> 1), 0, D)] += v;
            }
          }
        }
      };
      auto write_row = [&](int j, const double (&Kx)[9]) {
        const int n = node_index(m.g, i, j, 0);
        PINT_CHECK_IDX(n >= 0 && n < m.g.nn && i <= nx && j <= ny);
        const uint8_t nf = m.node_flags[n];
        const bool fixed = row_fixed(nf, ca, D);
        const int ctr = center_offset(D);
        const size_t base = (size_t)s * m.g.noff * C * C * np + ((size_t)ca * C + cp) * np + n;
#pragma unroll
        for (int o = 0; o < 9; ++o) {
          const double v = fixed ? ((o == ctr && cp == ca) ? 1.0 : 0.0) : Kx[o];
          J[base + (size_t)o * C * C * np] = v;
          if (J32) J32[base + (size_t)o * C * C * np] = (float)v;
        }
      };
      if (own_bottom) {
        cell_terms(i - 1, 1, K);  // node is the bottom-right corner of the left cell
        cell_terms(i, 0, K);      // bottom-left corner of the right cell
        write_row(cj, K);
      }
      if (own_top) {
        double P[9];
#pragma unroll
        for (int o = 0; o < 9; ++o) P[o] = 0.0;
        cell_terms(i - 1, 3, P);  // top-right corner of the left cell
        cell_terms(i, 2, P);      // top-left corner of the right cell
        if (top_final) {
          write_row(cj + 1, P);
        } else {
#pragma unroll
          for (int o = 0; o < L::NPART; ++o) part[o * L::ITEMS + it] = P[o];
        }
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- K1 residual, node-owner strips (2-d default)
// The same ownership as k_jacobian_strip for the residual vector: a block owns
// the rows of W node columns x a chunk of node rows and sweeps the strip's
// cell rows bottom to top (3-row ring of staged node values, next row
// prefetched during phase 1):
//   phase 1  thread = (cell of the row, Gauss point): fields from the ring,
//            qflux<double>, the NF flux values (and the outflow face terms) to
//            shared memory;
//   phase 2  thread = (node column, row component): tests the fluxes of the
//            cells left / right of the node with its shape functions; the
//            bottom-corner terms complete node row cj on top of the
//            top-corner terms kept from cell row cj - 1, and the row is
//            written ONCE, Dirichlet / identity rows (r = y - g) included.
// One launch instead of a zeroing pass, 2^d colour launches with a
// read-modify-write scatter (the long-scoreboard stall of k_elem_tile, ncu
// r02d) and k_fix_residual.  Fixed summation order (cell row j-1 left, right,
// row j left, right; points in order, then face points): deterministic and
// independent of the batch.
struct ResStrip {
  static constexpr int A = 4, C = 5, NS = 3, D = 2;
  static constexpr int T = 128;
  static constexpr int WMAX = T / A - 1;
  static constexpr int NF = 3 * D + 2 * D * D + 1;  // vec, ten, uvec, uten, pv, pt
  static constexpr int RW = WMAX + 3;
  static constexpr int ITEMS = 160;
  static constexpr size_t smem = sizeof(double) * ((size_t)(NF + D) * T + A * A * NS + (A / 2) * A * NS +
                                                   (size_t)3 * 2 * C * RW + (size_t)ITEMS);
  // flux slots (the layout of ElemTile<2>)
  static constexpr PINT_HD int vec(int i) { return i; }
  static constexpr PINT_HD int ten(int i, int j) { return D + i * D + j; }
  static constexpr PINT_HD int uvec(int i) { return D + D * D + i; }
  static constexpr PINT_HD int uten(int i, int j) { return 2 * D + D * D + i * D + j; }
  static constexpr PINT_HD int pv() { return 2 * D + 2 * D * D; }
  static constexpr PINT_HD int pt(int j) { return 2 * D + 2 * D * D + 1 + j; }
};

__global__ void __launch_bounds__(ResStrip::T, 3) k_residual_strip(MeshDev m, Phys ph, const StepScalars* __restrict__ st,
                                                                  const double* __restrict__ y, const double* __restrict__ yo,
                                                                  double* __restrict__ r, int* __restrict__ degen,
                                                                  const int* __restrict__ active, int W, int nstrips, int H) {
  pdl_wait();
  using L = ResStrip;
  using ET = ResStrip;
  constexpr int A = L::A, C = L::C, NS = L::NS, T = L::T, D = 2, RW = L::RW, NF = L::NF;
  extern __shared__ double sm[];
  double* sf = sm;                                   // flux [NF][T]
  double* sb = sf + (size_t)NF * T;                  // outflow face terms [D][T]
  double* tv = sb + (size_t)D * T;                   // [q][b][NS]
  double* tf = tv + A * A * NS;                      // [face q][b][NS]
  double* ring = tf + (A / 2) * A * NS;              // [slot 3][lvl 2][c][RW]
  double* part = ring + 3 * 2 * C * RW;              // top-corner partials [ITEMS]
  __shared__ int sdeg;
  const int s = blockIdx.y;
  if (active && !active[s]) return;  // uniform per block
  const int lane = threadIdx.x;
  const int nx = m.cells[0], ny = m.cells[1];
  const int strip = blockIdx.x % nstrips, chunk = blockIdx.x / nstrips;
  const int i0 = strip * W;
  const int nown = min(W, nx + 1 - i0);
  const int j0 = chunk * H, j1 = min(j0 + H, ny + 1);
  if (nown <= 0 || j0 >= j1) return;
  const int c_lo = max(i0 - 1, 0), c_hi = min(i0 + nown - 1, nx - 1);
  const int ncell = c_hi - c_lo + 1;
  const int ncol = ncell + 1;
  const int cj_lo = max(j0 - 1, 0), cj_hi = min(j1 - 1, ny - 1);
  const int np = m.g.np;
  const size_t vs = (size_t)C * np;
  const double* ys = y + s * vs;
  const double* yos = yo + s * vs;
  if (lane == 0) sdeg = 0;
  if (lane < A + (A >> 1)) {
    const bool face = lane >= A;
    double xi[D], N[A], dN[A][D];
    gauss_point<D>(face ? lane - A : lane, face, xi);
    q1_shape<D>(xi, ph.ih, N, dN);
    double* t = face ? tf + (lane - A) * A * NS : tv + lane * A * NS;
#pragma unroll
    for (int b = 0; b < A; ++b) {
      t[b * NS] = N[b];
#pragma unroll
      for (int k = 0; k < D; ++k) t[b * NS + 1 + k] = dN[b][k];
    }
  }
  constexpr int PER = (2 * C * RW + T - 1) / T;
  auto load_row = [&](int rr, double (&v)[PER]) {
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int idx = lane + k * T;
      const int col = idx % RW, c = (idx / RW) % C, lvl = idx / (RW * C);
      PINT_CHECK_IDX(!(lvl < 2 && col < ncol) || (c_lo + col <= nx && rr >= 0 && rr <= ny));
      v[k] = (lvl < 2 && col < ncol) ? __ldg((lvl == 0 ? ys : yos) + (size_t)c * np + node_index(m.g, c_lo + col, rr, 0))
                                     : 0.0;
    }
  };
  auto store_row = [&](int rr, const double (&v)[PER]) {
    double* dst = ring + (rr % 3) * 2 * C * RW;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int idx = lane + k * T;
      if (idx < 2 * C * RW) dst[idx] = v[k];
    }
  };
  {
    double v[PER];
    load_row(cj_lo, v);
    store_row(cj_lo, v);
    load_row(cj_lo + 1, v);
    store_row(cj_lo + 1, v);
  }
  const int lc = lane % 32, q = lane / 32;
  const int nitems = nown * C;
  const double ramp = st[s].ramp;
  __syncthreads();
  for (int cj = cj_lo; cj <= cj_hi; ++cj) {
    double pre[PER];
    const bool more = cj + 2 <= min(cj_hi + 1, ny);
    if (more) load_row(cj + 2, pre);
    // ---- phase 1: pointwise flux of (cell c_lo + lc, row cj) at point q
    if (lc < ncell) {
      const int ci = c_lo + lc;
      const uint8_t cf = m.cell_flags[cj * nx + ci];
      const bool solid = cf & kCellSolid;
      const double* r0 = ring + (cj % 3) * 2 * C * RW;
      const double* r1 = ring + ((cj + 1) % 3) * 2 * C * RW;
      auto getter = [&](int lvl) {
        return [=](int a, int c) {
          const double* rr = (a >> 1) ? r1 : r0;
          return rr[(lvl * C + c) * RW + lc + (a & 1)];
        };
      };
      auto shape = [&](const double* t, double (&N)[A], double (&dN)[A][D]) {
#pragma unroll
        for (int b = 0; b < A; ++b) {
          N[b] = t[b * NS];
#pragma unroll
          for (int k = 0; k < D; ++k) dN[b][k] = t[b * NS + 1 + k];
        }
      };
      double* fo = sf + lane;
      {
        double N[A], dN[A][D];
        shape(tv + q * A * NS, N, dN);
        QFields<D, double> fn, fold;
        interp<D>(N, dN, getter(0), fn);
        interp<D>(N, dN, getter(1), fold);
        QFlux<D, double> fx;
        bool dg = false;
        qflux<D, double, double, double>(ph, st[s], solid, fn, fold, fx, dg);
        if (dg) sdeg = 1;
#pragma unroll
        for (int i = 0; i < D; ++i) {
          fo[ET::vec(i) * T] = fx.vec[i];
          fo[ET::uvec(i) * T] = fx.uvec[i];
          fo[ET::pt(i) * T] = fx.pt[i];
#pragma unroll
          for (int j = 0; j < D; ++j) {
            fo[ET::ten(i, j) * T] = fx.ten[i][j];
            fo[ET::uten(i, j) * T] = fx.uten[i][j];
          }
        }
        fo[ET::pv() * T] = fx.pv;
      }
      if ((cf & kCellOutflow) && q < (A >> 1)) {
        double N[A], dN[A][D];
        shape(tf + q * A * NS, N, dN);
        QFields<D, double> gn, gold;
        interp<D>(N, dN, getter(0), gn);
        interp<D>(N, dN, getter(1), gold);
        double B[D];
        qflux_outflow<D, double, double, double>(ph, st[s], gn, gold, B);
#pragma unroll
        for (int i = 0; i < D; ++i) sb[i * T + lane] = B[i];
      }
    }
    if (more) store_row(cj + 2, pre);
    __syncthreads();
    // ---- phase 2: rows (node (i, cj), ca) and (node (i, cj + 1), ca)
    for (int it = lane; it < nitems; it += T) {
      const int ca = it / nown, li = it % nown;
      const int i = i0 + li;
      const bool own_bottom = cj >= j0;
      const bool own_top = cj + 1 < j1;
      const bool top_final = own_top && cj + 1 == ny;
      // contribution of cell (ci, cj) to row (corner a, ca)
      auto cell_term = [&](int ci, int a) -> double {
        if (ci < 0 || ci >= nx) return 0.0;
        const int lcell = ci - c_lo;
        PINT_CHECK_IDX(lcell >= 0 && lcell < 32 && lcell < ncell && it < L::ITEMS);
        const uint8_t cf = m.cell_flags[cj * nx + ci];
        const bool solid = cf & kCellSolid;
        if (ca == 2 * D && solid) return 0.0;               // solid cells own no p rows
        const int nj = cj + (a >> 1);
        const uint8_t nf = m.node_flags[node_index(m.g, i, nj, 0)];
        const bool ext = solid || !(nf & kSolidTouch);
        double acc = 0.0;
#pragma unroll
        for (int qq = 0; qq < A; ++qq) {
          const double* f = sf + qq * 32 + lcell;
          const double* ta = tv + (qq * A + a) * NS;
          double v;
          if (ca < D) {
            v = f[ET::vec(ca) * T] * ta[0];
#pragma unroll
            for (int j = 0; j < D; ++j) v += f[ET::ten(ca, j) * T] * ta[1 + j];
          } else if (ca < 2 * D) {
            const int iu = ca - D;
            v = f[ET::uvec(iu) * T] * ta[0];
            if (ext) {
              double ex = 0.0;
#pragma unroll
              for (int j = 0; j < D; ++j) ex += f[ET::uten(iu, j) * T] * ta[1 + j];
              v = v + ex;
            }
          } else {
            v = f[ET::pv() * T] * ta[0];
#pragma unroll
            for (int j = 0; j < D; ++j) v += f[ET::pt(j) * T] * ta[1 + j];
          }
          acc += ph.wq * v;
        }
        if ((cf & kCellOutflow) && ca < D) {
#pragma unroll
          for (int qq = 0; qq < (A >> 1); ++qq)
            acc += (-ph.wf) * (sb[ca * T + qq * 32 + lcell] * tf[(qq * A + a) * NS]);
        }
        return acc;
      };
      auto write_row = [&](int j, double R) {
        const int n = node_index(m.g, i, j, 0);
        PINT_CHECK_IDX(n >= 0 && n < m.g.nn && (i - c_lo) >= 0 && (i - c_lo) < RW);
        const uint8_t nf = m.node_flags[n];
        double out = R;
        if (row_fixed(nf, ca, D)) {
          const double g = (ca == 0) ? ramp * m.profile[n] : 0.0;
          out = ring[(j % 3) * 2 * C * RW + ca * RW + (i - c_lo)] - g;  // y - g from the staged node row
        }
        r[s * vs + (size_t)ca * np + n] = out;
      };
      if (own_bottom) {
        double R = cj > cj_lo ? part[it] : 0.0;
        R += cell_term(i - 1, 1);  // node is the bottom-right corner of the left cell
        R += cell_term(i, 0);      // bottom-left corner of the right cell
        write_row(cj, R);
      }
      if (own_top) {
        double P = cell_term(i - 1, 3);  // top-right corner of the left cell
        P += cell_term(i, 2);            // top-left corner of the right cell
        if (top_final) write_row(cj + 1, P);
        else part[it] = P;
      }
    }
    __syncthreads();
  }
  if (lane == 0 && sdeg) degen[s] = 1;  // benign: every writer stores 1
}

// ---------------------------------------------------------------- Jacobian-vector product (matrix-free)
template <int D>
__global__ void __launch_bounds__(128, ElemOcc<D>::value) k_jvp_colour(MeshDev m, Phys ph, const StepScalars* __restrict__ st,
                                                   const double* __restrict__ y, const double* __restrict__ yo,
                                                   const double* __restrict__ w, double* __restrict__ out,
                                                   const int* __restrict__ active, int colour) {
  pdl_wait();
  constexpr int C = 2 * D + 1;
  constexpr int A = 1 << D;
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int q = gt & (A - 1);
  ElemIndex<D> e;
  const bool valid = colour_element<D>(m, colour, gt / A, e);
  const size_t vs = (size_t)C * m.g.np;
  double R[A][C];
  zero_acc<D>(R);
  bool dg = false;
  if (valid) qp_integral<D, 1>(ph, st[s], e, q, y + s * vs, yo + s * vs, w + s * vs, m.g.np, 0, 0, R, dg);
  reduce_points<D>(R);
  if (!valid) return;
  scatter_rows<D>(R, q, e, out + s * vs, m.g.np);
}

// ---------------------------------------------------------------- K1 / K2' tiled (default)
// Block = EPB elements of one colour x 2^d quadrature points.
//   stage    the node values (y, y_old [, w]) of the block's elements are
//            loaded into shared memory, every load of the block in flight at
//            once (the per-point gathers of k_residual_colour / k_jvp_colour
//            were the long-scoreboard stall of those kernels, ncu r02);
//   phase 1  thread (element, point q): fields from shared memory, qflux,
//            the NF pointwise flux values (their derivatives for J w) to
//            shared memory; outflow face points add their B terms;
//   phase 2  thread (element, local node a): R[a][c] = W sum_q (flux_q tested
//            with N_a(q), grad N_a(q)) in a fixed point order (+ the face
//            terms), scattered colour-ordered as before.
// No xor butterfly (80 shuffles per thread in 2-d), no per-point 20-entry
// accumulator: a fraction of the registers, no spills.
template <int D>
struct ElemTile {
  static constexpr int A = 1 << D, C = 2 * D + 1;
  static constexpr int EPB = D == 2 ? 32 : 16;       // elements per block
  static constexpr int T = EPB * A;                  // 128 threads
  static constexpr int NF = 3 * D + 2 * D * D + 1;   // vec, ten, uvec, uten, pv, pt
  static constexpr int OCC = D == 2 ? 3 : 2;
  // flux slot of each output (phase 1 writes, phase 2 reads)
  static constexpr PINT_HD int vec(int i) { return i; }
  static constexpr PINT_HD int ten(int i, int j) { return D + i * D + j; }
  static constexpr PINT_HD int uvec(int i) { return D + D * D + i; }
  static constexpr PINT_HD int uten(int i, int j) { return 2 * D + D * D + i * D + j; }
  static constexpr PINT_HD int pv() { return 2 * D + 2 * D * D; }
  static constexpr PINT_HD int pt(int j) { return 2 * D + 2 * D * D + 1 + j; }
  // shared memory (doubles): node values [NL][C][A][EPB], flux [NF][T], face [D][T], shape [A][A][1+D] x 2
  static constexpr size_t smem(int NL) {
    return sizeof(double) * ((size_t)NL * C * A * EPB + (size_t)(NF + D) * T + 2 * (size_t)A * A * (1 + D)) +
           sizeof(int) * (size_t)A * EPB;
  }
};

template <int D, int MODE>  // MODE 0: residual (y, y_old), 1: J w (y, y_old, w)
__global__ void __launch_bounds__(ElemTile<D>::T, ElemTile<D>::OCC) k_elem_tile(
    MeshDev m, Phys ph, const StepScalars* __restrict__ st, const double* __restrict__ y,
    const double* __restrict__ yo, const double* __restrict__ w, double* __restrict__ out, int* __restrict__ degen,
    const int* __restrict__ active, int colour) {
  pdl_wait();
  using ET = ElemTile<D>;
  constexpr int A = ET::A, C = ET::C, EPB = ET::EPB, T = ET::T, NF = ET::NF, NS = 1 + D;
  constexpr int NL = MODE == 0 ? 2 : 3;
  extern __shared__ double sm[];
  double* sv = sm;                                   // [NL][C][A][EPB]
  double* sf = sv + (size_t)NL * C * A * EPB;        // [NF][T]
  double* sb = sf + (size_t)NF * T;                  // [D][T]
  double* tv = sb + (size_t)D * T;                   // volume shape table [q][b][NS]
  double* tf = tv + A * A * NS;                      // face shape table [face q][b][NS]
  int* snode = reinterpret_cast<int*>(tf + A * A * NS);  // [A][EPB]
  __shared__ int sdeg;
  const int s = blockIdx.y;
  if (active && !active[s]) return;  // uniform per block
  const int lane = threadIdx.x;
  const int el = lane / A, q = lane % A;
  ElemIndex<D> e;
  const bool valid = colour_element<D>(m, colour, blockIdx.x * EPB + el, e);
  if (lane == 0) sdeg = 0;
  if (q == 0) {
#pragma unroll
    for (int a = 0; a < A; ++a) snode[a * EPB + el] = valid ? e.node[a] : -1;
  }
  if (lane < A + (A >> 1)) {  // shape tables (uniform mesh: identical for every element)
    const bool face = lane >= A;
    double xi[D], N[A], dN[A][D];
    gauss_point<D>(face ? lane - A : lane, face, xi);
    q1_shape<D>(xi, ph.ih, N, dN);
    double* t = face ? tf + (lane - A) * A * NS : tv + lane * A * NS;
#pragma unroll
    for (int b = 0; b < A; ++b) {
      t[b * NS] = N[b];
#pragma unroll
      for (int k = 0; k < D; ++k) t[b * NS + 1 + k] = dN[b][k];
    }
  }
  __syncthreads();
  // stage the node values: every load of the block issued before any use
  const size_t vs = (size_t)C * m.g.np;
  {
    constexpr int PER = NL * C * A * EPB / T;
    double v[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int idx = lane + k * T;                  // [lvl][c][a][e]
      const int ee = idx % EPB, a = (idx / EPB) % A, c = (idx / (EPB * A)) % C, lvl = idx / (EPB * A * C);
      const int nd = snode[a * EPB + ee];
      const double* src = (lvl == 0 ? y : lvl == 1 ? yo : w) + s * vs;
      v[k] = nd >= 0 ? __ldg(src + (size_t)c * m.g.np + nd) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < PER; ++k) sv[lane + k * T] = v[k];
  }
  __syncthreads();
  // phase 1: pointwise flux at volume point q (and face point q on outflow cells)
  if (valid) {
    const bool solid = e.cflag & kCellSolid;
    auto field = [&](int lvl, const double* t, QFields<D, double>& f) {
      auto get = [&](int a, int c) { return sv[((lvl * C + c) * A + a) * EPB + el]; };
      double N[A], dN[A][D];
#pragma unroll
      for (int b = 0; b < A; ++b) {
        N[b] = t[b * NS];
#pragma unroll
        for (int k = 0; k < D; ++k) dN[b][k] = t[b * NS + 1 + k];
      }
      interp<D>(N, dN, get, f);
    };
    double* fo = sf + lane;
    {
      QFields<D, double> fn, fold;
      field(0, tv + q * A * NS, fn);
      field(1, tv + q * A * NS, fold);
      bool dg = false;
      if (MODE == 0) {
        QFlux<D, double> fx;
        qflux<D, double, double, double>(ph, st[s], solid, fn, fold, fx, dg);
        if (dg) sdeg = 1;
#pragma unroll
        for (int i = 0; i < D; ++i) {
          fo[ET::vec(i) * T] = fx.vec[i];
          fo[ET::uvec(i) * T] = fx.uvec[i];
          fo[ET::pt(i) * T] = fx.pt[i];
#pragma unroll
          for (int j = 0; j < D; ++j) {
            fo[ET::ten(i, j) * T] = fx.ten[i][j];
            fo[ET::uten(i, j) * T] = fx.uten[i][j];
          }
        }
        fo[ET::pv() * T] = fx.pv;
      } else {
        QFields<D, double> fw;
        field(2, tv + q * A * NS, fw);
        QFields<D, Dual> fd;
        seed_fields<D>(fn, fw, fd);
        QFlux<D, Dual> fx;
        qflux<D, Dual, Dual, Dual>(ph, st[s], solid, fd, fold, fx, dg);
#pragma unroll
        for (int i = 0; i < D; ++i) {
          fo[ET::vec(i) * T] = fx.vec[i].d;
          fo[ET::uvec(i) * T] = fx.uvec[i].d;
          fo[ET::pt(i) * T] = fx.pt[i].d;
#pragma unroll
          for (int j = 0; j < D; ++j) {
            fo[ET::ten(i, j) * T] = fx.ten[i][j].d;
            fo[ET::uten(i, j) * T] = fx.uten[i][j].d;
          }
        }
        fo[ET::pv() * T] = fx.pv.d;
      }
    }
    if ((e.cflag & kCellOutflow) && q < (A >> 1)) {
      QFields<D, double> fn, fold;
      field(0, tf + q * A * NS, fn);
      field(1, tf + q * A * NS, fold);
      if (MODE == 0) {
        double B[D];
        qflux_outflow<D, double, double, double>(ph, st[s], fn, fold, B);
#pragma unroll
        for (int i = 0; i < D; ++i) sb[i * T + lane] = B[i];
      } else {
        QFields<D, double> fw;
        field(2, tf + q * A * NS, fw);
        QFields<D, Dual> fd;
        seed_fields<D>(fn, fw, fd);
        Dual B[D];
        qflux_outflow<D, Dual, Dual, Dual>(ph, st[s], fd, fold, B);
#pragma unroll
        for (int i = 0; i < D; ++i) sb[i * T + lane] = B[i].d;
      }
    }
  }
  __syncthreads();
  if (MODE == 0 && lane == 0 && sdeg) degen[s] = 1;  // benign: every writer stores 1
  if (!valid) return;
  // phase 2: this lane owns local node a = q of its element
  const int a = q;
  const int base = lane - q;  // lane of point 0 of this element
  const bool ext = (e.ext_mask >> a) & 1;
  double R[C];
#pragma unroll
  for (int c = 0; c < C; ++c) R[c] = 0.0;
#pragma unroll
  for (int qq = 0; qq < A; ++qq) {
    const double* f = sf + base + qq;
    const double* ta = tv + (qq * A + a) * NS;
    const double Na = ta[0];
    double dNa[D];
#pragma unroll
    for (int j = 0; j < D; ++j) dNa[j] = ta[1 + j];
#pragma unroll
    for (int i = 0; i < D; ++i) {
      double mm = f[ET::vec(i) * T] * Na;
      double u = f[ET::uvec(i) * T] * Na;
      double ex = 0.0;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        mm += f[ET::ten(i, j) * T] * dNa[j];
        ex += f[ET::uten(i, j) * T] * dNa[j];
      }
      R[i] += ph.wq * mm;
      R[D + i] += ph.wq * (ext ? u + ex : u);
    }
    double pr = f[ET::pv() * T] * Na;
#pragma unroll
    for (int j = 0; j < D; ++j) pr += f[ET::pt(j) * T] * dNa[j];
    R[2 * D] += ph.wq * pr;
  }
  if (e.cflag & kCellOutflow) {
#pragma unroll
    for (int qq = 0; qq < (A >> 1); ++qq) {
      const double na = tf[(qq * A + a) * NS];
#pragma unroll
      for (int i = 0; i < D; ++i) R[i] += (-ph.wf) * (sb[i * T + base + qq] * na);
    }
  }
  // scatter the node's rows: every old value loaded before the first store
  const bool solid = e.cflag & kCellSolid;  // solid cells own no p rows
  double* o = out + s * vs + e.node[a];
  double v[C];
#pragma unroll
  for (int c = 0; c < C; ++c) v[c] = (c == 2 * D && solid) ? 0.0 : o[(size_t)c * m.g.np];
#pragma unroll
  for (int c = 0; c < C; ++c)
    if (!(c == 2 * D && solid)) o[(size_t)c * m.g.np] = v[c] + R[c];
}

// ---------------------------------------------------------------- fixed rows

// residual rows r = y - g on Dirichlet / identity rows
template <int D>
__global__ void k_fix_residual(MeshDev m, const StepScalars* __restrict__ st, const double* __restrict__ y,
                               double* __restrict__ r, const int* __restrict__ active) {
  pdl_wait();
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
  pdl_wait();
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
  pdl_wait();
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
