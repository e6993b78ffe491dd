// Pointwise ("quadrature-function") form of the shifted Crank-Nicolson
// monolithic ALE-FSI residual (decisions in
// paper_1907_01252_b200/problem.py).
//
// At every quadrature point the element residual is
//   R[a][i]     += W ( vec_i N_a  + sum_j ten_ij  dN_a,j )         momentum rows
//   R[a][d+i]   += W ( uvec_i N_a + sum_j uten_ij dN_a,j )         u rows
//   R[a][2d]    += W ( pv N_a     + sum_j pt_j    dN_a,j )         p rows
// where (vec, ten, uvec, uten, pv, pt) = qflux(fields at the point).  The
// fields are v, grad v, u, grad u, p, grad p of the new state (the unknowns)
// and of the old state (constants).  Kernels differentiate ONLY qflux:
//   residual : qflux<double>
//   J w      : qflux<Dual> seeded with the interpolated w
//   J column : qflux<Dual> seeded with one trial basis function (N_b, dN_b) in
//              one component -- so every Jacobian column costs one pointwise
//              dual pass per quadrature point instead of a dual pass through
//              the whole element (field interpolation is shared).
#pragma once

#include <type_traits>

#include "pint_common.cuh"

namespace pint {

// ---------------------------------------------------------------- dual numbers
struct Dual {
  double v, d;
  PINT_HD Dual() : v(0.0), d(0.0) {}
  PINT_HD Dual(double a) : v(a), d(0.0) {}
  PINT_HD Dual(double a, double b) : v(a), d(b) {}
};
PINT_HD Dual operator+(Dual a, Dual b) { return Dual(a.v + b.v, a.d + b.d); }
PINT_HD Dual operator-(Dual a, Dual b) { return Dual(a.v - b.v, a.d - b.d); }
PINT_HD Dual operator*(Dual a, Dual b) { return Dual(a.v * b.v, a.d * b.v + a.v * b.d); }
PINT_HD Dual operator/(Dual a, Dual b) {
  const double q = a.v / b.v;
  return Dual(q, (a.d - q * b.d) / b.v);
}
PINT_HD Dual operator-(Dual a) { return Dual(-a.v, -a.d); }
PINT_HD Dual operator+(Dual a, double b) { return Dual(a.v + b, a.d); }
PINT_HD Dual operator+(double a, Dual b) { return Dual(a + b.v, b.d); }
PINT_HD Dual operator-(Dual a, double b) { return Dual(a.v - b, a.d); }
PINT_HD Dual operator-(double a, Dual b) { return Dual(a - b.v, -b.d); }
PINT_HD Dual operator*(Dual a, double b) { return Dual(a.v * b, a.d * b); }
PINT_HD Dual operator*(double a, Dual b) { return Dual(a * b.v, a * b.d); }
PINT_HD Dual operator/(Dual a, double b) { return Dual(a.v / b, a.d / b); }
PINT_HD Dual operator/(double a, Dual b) {
  const double q = a / b.v;
  return Dual(q, -q * b.d / b.v);
}
PINT_HD double value_of(double a) { return a; }
PINT_HD double value_of(const Dual& a) { return a.v; }
PINT_HD double deriv_of(double) { return 0.0; }
PINT_HD double deriv_of(const Dual& a) { return a.d; }

// value + N tangents: one pass of the flux carries N derivative directions, so
// the primal part (and every division) is computed once for all of them and
// the N tangent chains are independent instructions (ILP for the FP64 pipe)
template <int N>
struct DualV {
  double v, d[N];
  PINT_HD DualV() : v(0.0) {
#pragma unroll
    for (int k = 0; k < N; ++k) d[k] = 0.0;
  }
  PINT_HD DualV(double a) : v(a) {
#pragma unroll
    for (int k = 0; k < N; ++k) d[k] = 0.0;
  }
};
#define PINT_DV_LOOP _Pragma("unroll") for (int k = 0; k < N; ++k)
template <int N> PINT_HD DualV<N> operator+(DualV<N> a, DualV<N> b) { DualV<N> r; r.v = a.v + b.v; PINT_DV_LOOP r.d[k] = a.d[k] + b.d[k]; return r; }
template <int N> PINT_HD DualV<N> operator-(DualV<N> a, DualV<N> b) { DualV<N> r; r.v = a.v - b.v; PINT_DV_LOOP r.d[k] = a.d[k] - b.d[k]; return r; }
template <int N> PINT_HD DualV<N> operator*(DualV<N> a, DualV<N> b) { DualV<N> r; r.v = a.v * b.v; PINT_DV_LOOP r.d[k] = a.d[k] * b.v + a.v * b.d[k]; return r; }
template <int N> PINT_HD DualV<N> operator/(DualV<N> a, DualV<N> b) {
  const double ib = 1.0 / b.v;  // one division for the value and all tangents
  DualV<N> r; r.v = a.v * ib; PINT_DV_LOOP r.d[k] = (a.d[k] - r.v * b.d[k]) * ib; return r;
}
template <int N> PINT_HD DualV<N> operator-(DualV<N> a) { DualV<N> r; r.v = -a.v; PINT_DV_LOOP r.d[k] = -a.d[k]; return r; }
template <int N> PINT_HD DualV<N> operator+(DualV<N> a, double b) { a.v += b; return a; }
template <int N> PINT_HD DualV<N> operator+(double a, DualV<N> b) { b.v += a; return b; }
template <int N> PINT_HD DualV<N> operator-(DualV<N> a, double b) { a.v -= b; return a; }
template <int N> PINT_HD DualV<N> operator-(double a, DualV<N> b) { DualV<N> r; r.v = a - b.v; PINT_DV_LOOP r.d[k] = -b.d[k]; return r; }
template <int N> PINT_HD DualV<N> operator*(DualV<N> a, double b) { a.v *= b; PINT_DV_LOOP a.d[k] *= b; return a; }
template <int N> PINT_HD DualV<N> operator*(double a, DualV<N> b) { b.v *= a; PINT_DV_LOOP b.d[k] *= a; return b; }
template <int N> PINT_HD DualV<N> operator/(DualV<N> a, double b) { const double ib = 1.0 / b; a.v *= ib; PINT_DV_LOOP a.d[k] *= ib; return a; }
template <int N> PINT_HD DualV<N> operator/(double a, DualV<N> b) {
  const double ib = 1.0 / b.v;
  DualV<N> r; r.v = a * ib; PINT_DV_LOOP r.d[k] = -r.v * b.d[k] * ib; return r;
}
template <int N> PINT_HD double value_of(const DualV<N>& a) { return a.v; }

// ---------------------------------------------------------------- small matrices
template <int D, typename T>
PINT_HD T det_inv(const T (&F)[D][D], T (&Fi)[D][D]) {
  if constexpr (D == 2) {
    const T det = F[0][0] * F[1][1] - F[0][1] * F[1][0];
    const T r = 1.0 / det;  // one fp64 division per inverse
    Fi[0][0] = F[1][1] * r;
    Fi[0][1] = -F[0][1] * r;
    Fi[1][0] = -F[1][0] * r;
    Fi[1][1] = F[0][0] * r;
    return det;
  } else {
    T cof[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
        cof[i][j] = F[i1][j1] * F[i2][j2] - F[i1][j2] * F[i2][j1];
      }
    const T det = F[0][0] * cof[0][0] + F[0][1] * cof[0][1] + F[0][2] * cof[0][2];
    const T r = 1.0 / det;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) Fi[i][j] = cof[j][i] * r;
    return det;
  }
}

// ---------------------------------------------------------------- quadrature
constexpr double kGaussLo = 0.21132486540518711775;  // 1/2 - 1/(2 sqrt 3)
constexpr double kGaussHi = 0.78867513459481288225;  // 1/2 + 1/(2 sqrt 3)

// Q1 shape values and physical gradients at xi in [0,1]^D (ih = 1 / cell size)
template <int D>
PINT_HD void q1_shape(const double (&xi)[D], const double* ih, double (&N)[1 << D], double (&dN)[1 << D][D]) {
#pragma unroll
  for (int a = 0; a < (1 << D); ++a) {
    double n = 1.0;
#pragma unroll
    for (int m = 0; m < D; ++m) n *= ((a >> m) & 1) ? xi[m] : 1.0 - xi[m];
    N[a] = n;
#pragma unroll
    for (int m = 0; m < D; ++m) {
      double g = ((a >> m) & 1) ? 1.0 : -1.0;
#pragma unroll
      for (int k = 0; k < D; ++k)
        if (k != m) g *= ((a >> k) & 1) ? xi[k] : 1.0 - xi[k];
      dN[a][m] = g * ih[m];
    }
  }
}

// volume point q (bit m of q selects the Gauss abscissa in direction m);
// face point (outflow face x = 1): bit m-1 of q for direction m >= 1
template <int D>
PINT_HD void gauss_point(int q, bool face, double (&xi)[D]) {
  if (!face) {
#pragma unroll
    for (int m = 0; m < D; ++m) xi[m] = ((q >> m) & 1) ? kGaussHi : kGaussLo;
  } else {
    xi[0] = 1.0;
#pragma unroll
    for (int m = 1; m < D; ++m) xi[m] = ((q >> (m - 1)) & 1) ? kGaussHi : kGaussLo;
  }
}

// ---------------------------------------------------------------- fields and fluxes
// Scalar promotion: double op double -> double, anything with a Dual -> Dual.
template <class A, class B>
struct PromoteT {
  using type = A;  // A is a dual type (Dual or DualV<N>); B is double or the same dual type
};
template <class B>
struct PromoteT<double, B> {
  using type = B;
};
template <class A, class B>
using P2 = typename PromoteT<A, B>::type;
template <class A, class B, class C>
using P3 = P2<P2<A, B>, C>;

// Fields at a point.  The velocity, deformation and pressure groups carry their
// own scalar type: a Jacobian column seeds only ONE group with dual numbers,
// so everything that does not depend on it stays plain double and the compiler
// drops the dead derivative arithmetic (e.g. a velocity column never
// differentiates F = I + grad u, its inverse or determinant).
template <int D, typename TV, typename TU = TV, typename TP = TV>
struct QFields {
  TV v[D], Gv[D][D];
  TU u[D], Gu[D][D];
  TP p, gp[D];
};

template <int D, typename T>
struct QFlux {
  T vec[D], ten[D][D], uvec[D], uten[D][D], pv, pt[D];
};

// interpolate the fields of one state at a point from element node values
template <int D, class Get>
__device__ __forceinline__ void interp(const double (&N)[1 << D], const double (&dN)[1 << D][D], const Get& get,
                                       QFields<D, double>& f) {
#pragma unroll
  for (int i = 0; i < D; ++i) {
    f.v[i] = 0.0;
    f.u[i] = 0.0;
    f.gp[i] = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) { f.Gv[i][j] = 0.0; f.Gu[i][j] = 0.0; }
  }
  f.p = 0.0;
#pragma unroll
  for (int a = 0; a < (1 << D); ++a) {
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const double yv = get(a, i), yu = get(a, D + i);
      f.v[i] += N[a] * yv;
      f.u[i] += N[a] * yu;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        f.Gv[i][j] += dN[a][j] * yv;
        f.Gu[i][j] += dN[a][j] * yu;
      }
    }
    const double yp = get(a, 2 * D);
    f.p += N[a] * yp;
#pragma unroll
    for (int j = 0; j < D; ++j) f.gp[j] += dN[a][j] * yp;
  }
}

// pointwise CN flux; n = new-state fields, o = old-state fields (double)
template <int D, typename TV, typename TU, typename TP>
__device__ __forceinline__ void qflux(const Phys& ph, const StepScalars& st, bool solid,
                                      const QFields<D, TV, TU, TP>& n, const QFields<D, double>& o,
                                      QFlux<D, P3<TV, TU, TP>>& out, bool& degen) {
  using TVU = P2<TV, TU>;
  using TVP = P2<TV, TP>;
  using TA = P3<TV, TU, TP>;
  const double kt = st.kt, ko = st.ko, k = st.k;
  TU Fn[D][D], Fin[D][D];
  double Fo[D][D], Fio[D][D];
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      Fn[i][j] = n.Gu[i][j] + (i == j ? 1.0 : 0.0);
      Fo[i][j] = o.Gu[i][j] + (i == j ? 1.0 : 0.0);
    }
  const TU Jn = det_inv<D>(Fn, Fin);
  const double Jo = det_inv<D>(Fo, Fio);
  if (value_of(Jn) <= 0.0) degen = true;
  if (!solid) {
    // mass / ALE term at n-1/2
    TU Fm[D][D], Fim[D][D];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int j = 0; j < D; ++j) Fm[i][j] = 0.5 * (Fn[i][j] + Fo[i][j]);
    det_inv<D>(Fm, Fim);
    const TU Jm = 0.5 * (Jn + Jo);
    TVU GvFin[D][D];
    double GvFio[D][D];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int j = 0; j < D; ++j) {
        TVU a = n.Gv[i][0] * Fin[0][j];
        double b = o.Gv[i][0] * Fio[0][j];
#pragma unroll
        for (int m = 1; m < D; ++m) { a = a + n.Gv[i][m] * Fin[m][j]; b += o.Gv[i][m] * Fio[m][j]; }
        GvFin[i][j] = a;
        GvFio[i][j] = b;
      }
#pragma unroll
    for (int i = 0; i < D; ++i) {
      TVU ale = TVU(0.0), cn = TVU(0.0);
      double co = 0.0;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        TVU gm = TVU(0.0);  // (grad v_{n-1/2} F_{n-1/2}^{-1})_{ij}
#pragma unroll
        for (int m = 0; m < D; ++m) gm = gm + (0.5 * (n.Gv[i][m] + o.Gv[i][m])) * Fim[m][j];
        ale = ale + gm * (n.u[j] - o.u[j]);
        cn = cn + GvFin[i][j] * n.v[j];
        co += GvFio[i][j] * o.v[j];
      }
      out.vec[i] = ph.rho_f * Jm * ((n.v[i] - o.v[i]) - ale) + kt * (ph.rho_f * Jn * cn) + ko * (ph.rho_f * Jo * co);
    }
    // Piola stresses J sigma F^{-T}, pressure p^n in both theta parts
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int j = 0; j < D; ++j) {
        TA pn_ij = TA(0.0);
        TP po_ij = TP(0.0);
#pragma unroll
        for (int m = 0; m < D; ++m) {
          TA sn = ph.rnu * (GvFin[i][m] + GvFin[m][i]);
          TP so = TP(ph.rnu * (GvFio[i][m] + GvFio[m][i]));
          if (i == m) { sn = sn - n.p; so = so - n.p; }
          pn_ij = pn_ij + sn * Fin[j][m];
          po_ij = po_ij + so * Fio[j][m];
        }
        out.ten[i][j] = kt * (Jn * pn_ij) + ko * (Jo * po_ij);
        out.uten[i][j] = kt * n.Gu[i][j] + ko * o.Gu[i][j];  // harmonic extension
      }
    TVU div = GvFin[0][0];
#pragma unroll
    for (int i = 1; i < D; ++i) div = div + GvFin[i][i];
    out.pv = k * (Jn * div);
#pragma unroll
    for (int j = 0; j < D; ++j) {
      out.pt[j] = (k * st.delta) * n.gp[j];
      out.uvec[j] = TA(0.0);
    }
  } else {
    // St. Venant-Kirchhoff: F Sigma(E), E = (F^T F - I)/2
    TU En[D][D];
    double Eo[D][D];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int j = 0; j < D; ++j) {
        TU sn = Fn[0][i] * Fn[0][j];
        double so = Fo[0][i] * Fo[0][j];
#pragma unroll
        for (int m = 1; m < D; ++m) { sn = sn + Fn[m][i] * Fn[m][j]; so += Fo[m][i] * Fo[m][j]; }
        En[i][j] = 0.5 * (sn - (i == j ? 1.0 : 0.0));
        Eo[i][j] = 0.5 * (so - (i == j ? 1.0 : 0.0));
      }
    TU trn = En[0][0];
    double tro = Eo[0][0];
#pragma unroll
    for (int i = 1; i < D; ++i) { trn = trn + En[i][i]; tro += Eo[i][i]; }
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int j = 0; j < D; ++j) {
        TU pn = TU(0.0);
        double po = 0.0;
#pragma unroll
        for (int m = 0; m < D; ++m) {
          TU sg = 2.0 * ph.mu * En[m][j];
          double sgo = 2.0 * ph.mu * Eo[m][j];
          if (m == j) { sg = sg + ph.lam * trn; sgo += ph.lam * tro; }
          pn = pn + Fn[i][m] * sg;
          po += Fo[i][m] * sgo;
        }
        out.ten[i][j] = kt * pn + ko * po;
        out.uten[i][j] = TA(0.0);
      }
#pragma unroll
    for (int i = 0; i < D; ++i) {
      out.vec[i] = ph.rho_s * (n.v[i] - o.v[i]);
      out.uvec[i] = (n.u[i] - o.u[i]) - kt * n.v[i] - ko * o.v[i];  // kinematic row
      out.pt[i] = TA(0.0);
    }
    out.pv = TA(0.0);
  }
}

// do-nothing outflow correction at a face point: B_i = kt rnu Jn (Fin^T Gvn^T Fin^T e_x)_i + ko (...)_old
template <int D, typename TV, typename TU, typename TP>
__device__ __forceinline__ void qflux_outflow(const Phys& ph, const StepScalars& st,
                                              const QFields<D, TV, TU, TP>& n, const QFields<D, double>& o,
                                              P2<TV, TU> (&B)[D]) {
  using TVU = P2<TV, TU>;
  TU Fn[D][D], Fin[D][D];
  double Fo[D][D], Fio[D][D];
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      Fn[i][j] = n.Gu[i][j] + (i == j ? 1.0 : 0.0);
      Fo[i][j] = o.Gu[i][j] + (i == j ? 1.0 : 0.0);
    }
  const TU Jn = det_inv<D>(Fn, Fin);
  const double Jo = det_inv<D>(Fo, Fio);
#pragma unroll
  for (int i = 0; i < D; ++i) {
    TVU mn = TVU(0.0);
    double mo = 0.0;
#pragma unroll
    for (int kk = 0; kk < D; ++kk)
#pragma unroll
      for (int l = 0; l < D; ++l) {
        mn = mn + Fin[kk][i] * n.Gv[l][kk] * Fin[0][l];
        mo += Fio[kk][i] * o.Gv[l][kk] * Fio[0][l];
      }
    B[i] = st.kt * (ph.rnu * Jn * mn) + st.ko * (ph.rnu * Jo * mo);
  }
}

// fields with dual parts in ONE group only: the trial function (N_b, dN_b)
// of component cb (G = 0 velocity, 1 deformation, 2 pressure group)
template <int D, int G, typename DT = Dual>
struct SeedTypes {
  using TV = std::conditional_t<G == 0, DT, double>;
  using TU = std::conditional_t<G == 1, DT, double>;
  using TP = std::conditional_t<G == 2, DT, double>;
  using F = QFields<D, TV, TU, TP>;
};

template <int D, int G>
__device__ __forceinline__ void seed_basis(const QFields<D, double>& f, int cb, double Nb, const double (&dNb)[D],
                                           typename SeedTypes<D, G>::F& n) {
#pragma unroll
  for (int i = 0; i < D; ++i) {
    if constexpr (G == 0) {
      n.v[i] = Dual(f.v[i], cb == i ? Nb : 0.0);
    } else {
      n.v[i] = f.v[i];
    }
    if constexpr (G == 1) {
      n.u[i] = Dual(f.u[i], cb == D + i ? Nb : 0.0);
    } else {
      n.u[i] = f.u[i];
    }
    if constexpr (G == 2) {
      n.gp[i] = Dual(f.gp[i], dNb[i]);
    } else {
      n.gp[i] = f.gp[i];
    }
#pragma unroll
    for (int j = 0; j < D; ++j) {
      if constexpr (G == 0) {
        n.Gv[i][j] = Dual(f.Gv[i][j], cb == i ? dNb[j] : 0.0);
      } else {
        n.Gv[i][j] = f.Gv[i][j];
      }
      if constexpr (G == 1) {
        n.Gu[i][j] = Dual(f.Gu[i][j], cb == D + i ? dNb[j] : 0.0);
      } else {
        n.Gu[i][j] = f.Gu[i][j];
      }
    }
  }
  if constexpr (G == 2) {
    n.p = Dual(f.p, Nb);
  } else {
    n.p = f.p;
  }
}

// fields with ONE unit derivative direction of component cb: dir = 0 seeds
// the value of cb, dir = 1 + k its derivative along x_k.  The derivative of
// the flux along the trial function (N_b, dN_b) of cb is then the linear
// combination  dF(dir 0) N_b + sum_k dF(dir 1+k) dN_b,k  -- 1 + D pointwise
// passes give all 2^D Jacobian columns of the component.
template <int D, int G>
__device__ __forceinline__ void seed_dir(const QFields<D, double>& f, int cb, int dir,
                                         typename SeedTypes<D, G>::F& n) {
  const double sv = dir == 0 ? 1.0 : 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    if constexpr (G == 0) {
      n.v[i] = Dual(f.v[i], cb == i ? sv : 0.0);
    } else {
      n.v[i] = f.v[i];
    }
    if constexpr (G == 1) {
      n.u[i] = Dual(f.u[i], cb == D + i ? sv : 0.0);
    } else {
      n.u[i] = f.u[i];
    }
    if constexpr (G == 2) {
      n.gp[i] = Dual(f.gp[i], dir == 1 + i ? 1.0 : 0.0);
    } else {
      n.gp[i] = f.gp[i];
    }
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const double sg = (dir == 1 + j) ? 1.0 : 0.0;
      if constexpr (G == 0) {
        n.Gv[i][j] = Dual(f.Gv[i][j], cb == i ? sg : 0.0);
      } else {
        n.Gv[i][j] = f.Gv[i][j];
      }
      if constexpr (G == 1) {
        n.Gu[i][j] = Dual(f.Gu[i][j], cb == D + i ? sg : 0.0);
      } else {
        n.Gu[i][j] = f.Gu[i][j];
      }
    }
  }
  if constexpr (G == 2) {
    n.p = Dual(f.p, sv);
  } else {
    n.p = f.p;
  }
}

// all 1 + D unit directions of component cb at once: tangent 0 seeds the value
// of cb, tangent 1 + k its derivative along x_k (seed_dir for dir = 0 .. D in
// one DualV<1 + D> pass)
template <int D, int G>
__device__ __forceinline__ void seed_all(const QFields<D, double>& f, int cb,
                                         typename SeedTypes<D, G, DualV<1 + D>>::F& n) {
  using DT = DualV<1 + D>;
  auto mk = [](double v, int dir, bool on) {
    DT r(v);
    if (on) {
#pragma unroll
      for (int k = 0; k < 1 + D; ++k) r.d[k] = (k == dir) ? 1.0 : 0.0;
    }
    return r;
  };
#pragma unroll
  for (int i = 0; i < D; ++i) {
    if constexpr (G == 0) n.v[i] = mk(f.v[i], 0, cb == i); else n.v[i] = f.v[i];
    if constexpr (G == 1) n.u[i] = mk(f.u[i], 0, cb == D + i); else n.u[i] = f.u[i];
    if constexpr (G == 2) n.gp[i] = mk(f.gp[i], 1 + i, true); else n.gp[i] = f.gp[i];
#pragma unroll
    for (int j = 0; j < D; ++j) {
      if constexpr (G == 0) n.Gv[i][j] = mk(f.Gv[i][j], 1 + j, cb == i); else n.Gv[i][j] = f.Gv[i][j];
      if constexpr (G == 1) n.Gu[i][j] = mk(f.Gu[i][j], 1 + j, cb == D + i); else n.Gu[i][j] = f.Gu[i][j];
    }
  }
  if constexpr (G == 2) n.p = mk(f.p, 0, true); else n.p = f.p;
}

// NT consecutive unit directions dir0 .. dir0 + NT - 1 of component cb as the
// tangents of one DualV<NT> pass (seed_all is dir0 = 0, NT = 1 + D)
template <int D, int G, int NT>
__device__ __forceinline__ void seed_dirs(const QFields<D, double>& f, int cb, int dir0,
                                          typename SeedTypes<D, G, DualV<NT>>::F& n) {
  using DT = DualV<NT>;
  auto mk = [dir0](double v, int dir, bool on) {
    DT r(v);
    if (on) {
#pragma unroll
      for (int k = 0; k < NT; ++k) r.d[k] = (dir0 + k == dir) ? 1.0 : 0.0;
    }
    return r;
  };
#pragma unroll
  for (int i = 0; i < D; ++i) {
    if constexpr (G == 0) n.v[i] = mk(f.v[i], 0, cb == i); else n.v[i] = f.v[i];
    if constexpr (G == 1) n.u[i] = mk(f.u[i], 0, cb == D + i); else n.u[i] = f.u[i];
    if constexpr (G == 2) n.gp[i] = mk(f.gp[i], 1 + i, true); else n.gp[i] = f.gp[i];
#pragma unroll
    for (int j = 0; j < D; ++j) {
      if constexpr (G == 0) n.Gv[i][j] = mk(f.Gv[i][j], 1 + j, cb == i); else n.Gv[i][j] = f.Gv[i][j];
      if constexpr (G == 1) n.Gu[i][j] = mk(f.Gu[i][j], 1 + j, cb == D + i); else n.Gu[i][j] = f.Gu[i][j];
    }
  }
  if constexpr (G == 2) n.p = mk(f.p, 0, true); else n.p = f.p;
}

// dual fields: values from f, derivatives from the interpolated direction w
template <int D>
__device__ __forceinline__ void seed_fields(const QFields<D, double>& f, const QFields<D, double>& w,
                                            QFields<D, Dual>& n) {
#pragma unroll
  for (int i = 0; i < D; ++i) {
    n.v[i] = Dual(f.v[i], w.v[i]);
    n.u[i] = Dual(f.u[i], w.u[i]);
    n.gp[i] = Dual(f.gp[i], w.gp[i]);
#pragma unroll
    for (int j = 0; j < D; ++j) {
      n.Gv[i][j] = Dual(f.Gv[i][j], w.Gv[i][j]);
      n.Gu[i][j] = Dual(f.Gu[i][j], w.Gu[i][j]);
    }
  }
  n.p = Dual(f.p, w.p);
}

// acc[a][c] += W * (flux tested against row (a, c)); DERIV selects the
// derivative parts (Jacobian / J w) instead of the values (residual).
// ext_mask bit a: the fluid extension row may be tested at local node a.
template <int D, bool DERIV, typename T>
__device__ __forceinline__ void accumulate(const QFlux<D, T>& fx, double W, const double (&N)[1 << D],
                                           const double (&dN)[1 << D][D], uint32_t ext_mask,
                                           double (&acc)[1 << D][2 * D + 1]) {
  auto x = [](const T& t) { return DERIV ? deriv_of(t) : value_of(t); };
#pragma unroll
  for (int a = 0; a < (1 << D); ++a) {
#pragma unroll
    for (int i = 0; i < D; ++i) {
      double m = x(fx.vec[i]) * N[a];
      double u = x(fx.uvec[i]) * N[a];
      double e = 0.0;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        m += x(fx.ten[i][j]) * dN[a][j];
        e += x(fx.uten[i][j]) * dN[a][j];
      }
      acc[a][i] += W * m;
      acc[a][D + i] += W * (((ext_mask >> a) & 1) ? u + e : u);
    }
    double pr = x(fx.pv) * N[a];
#pragma unroll
    for (int j = 0; j < D; ++j) pr += x(fx.pt[j]) * dN[a][j];
    acc[a][2 * D] += W * pr;
  }
}

}  // namespace pint
