// Element residual of the shifted Crank-Nicolson monolithic ALE-FSI step.
//
// One templated routine serves three kernels: the residual (T = double), the
// element Jacobian columns (T = Dual seeded with a unit direction) and the
// Jacobian-vector product (T = Dual seeded with w).  It restates PAPER.md:
// 401-440 (semiforms A_div, A_NS with the do-nothing outflow correction,
// A_ES, mass/ALE terms at n-1/2), with the shared decisions of
// paper_1907_01252_b200/problem.py; the CPU oracle restates the same equations
// independently in numpy (oracle/fsi_oracle.py:element_residual).
#pragma once

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
  double q = a.v / b.v;
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
PINT_HD Dual& operator+=(Dual& a, Dual b) { a.v += b.v; a.d += b.d; return a; }

PINT_HD double value_of(double a) { return a; }
PINT_HD double value_of(const Dual& a) { return a.v; }

// ---------------------------------------------------------------- small matrices
template <int D, typename T>
PINT_HD T det_inv(const T (&F)[D][D], T (&Fi)[D][D]) {
  if constexpr (D == 2) {
    T det = F[0][0] * F[1][1] - F[0][1] * F[1][0];
    Fi[0][0] = F[1][1] / det;
    Fi[0][1] = -F[0][1] / det;
    Fi[1][0] = -F[1][0] / det;
    Fi[1][1] = F[0][0] / det;
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
    T det = F[0][0] * cof[0][0] + F[0][1] * cof[0][1] + F[0][2] * cof[0][2];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) Fi[i][j] = cof[j][i] / det;
    return det;
  }
}

template <int D, typename A, typename B, typename O>
PINT_HD void matmul(const A (&X)[D][D], const B (&Y)[D][D], O (&Z)[D][D]) {
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      O s = X[i][0] * Y[0][j];
#pragma unroll
      for (int k = 1; k < D; ++k) s = s + X[i][k] * Y[k][j];
      Z[i][j] = s;
    }
}

// ---------------------------------------------------------------- quadrature
constexpr double kGaussLo = 0.21132486540518711775;  // 1/2 - 1/(2 sqrt 3)
constexpr double kGaussHi = 0.78867513459481288225;  // 1/2 + 1/(2 sqrt 3)

// Q1 shape values and physical gradients at xi in [0,1]^D
template <int D>
PINT_HD void q1_shape(const double (&xi)[D], const double* h, double (&N)[1 << D],
                      double (&dN)[1 << D][D]) {
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
      dN[a][m] = g / h[m];
    }
  }
}

// ---------------------------------------------------------------- element residual
// R[a][c] accumulates the element contribution to row (local node a, comp c)
// before row ownership of shared nodes (ext_mask) and Dirichlet rows.
// ext_mask bit a: a fluid cell may contribute its extension row at node a.
template <int D, typename T, class Src>
__device__ __forceinline__ void fsi_element(const Phys& ph, const StepScalars& st, uint8_t cflag,
                                            uint32_t ext_mask, const Src& src,
                                            T (&R)[1 << D][2 * D + 1], bool& degen) {
  constexpr int A = 1 << D;
  constexpr int C = 2 * D + 1;
  const double kt = st.kt, ko = st.ko, k = st.k;
  const bool solid = cflag & kCellSolid;
#pragma unroll
  for (int a = 0; a < A; ++a)
#pragma unroll
    for (int c = 0; c < C; ++c) R[a][c] = T(0.0);

#pragma unroll 1
  for (int q = 0; q < A; ++q) {
    double xi[D];
#pragma unroll
    for (int m = 0; m < D; ++m) xi[m] = ((q >> m) & 1) ? kGaussHi : kGaussLo;
    double N[A], dN[A][D];
    q1_shape<D>(xi, ph.h, N, dN);

    T vn[D], un[D], Gvn[D][D], Gun[D][D], gpn[D], pn(0.0);
    double vo[D], uo[D], Gvo[D][D], Guo[D][D];
#pragma unroll
    for (int i = 0; i < D; ++i) {
      vn[i] = T(0.0); un[i] = T(0.0); gpn[i] = T(0.0); vo[i] = 0.0; uo[i] = 0.0;
#pragma unroll
      for (int j = 0; j < D; ++j) { Gvn[i][j] = T(0.0); Gun[i][j] = T(0.0); Gvo[i][j] = 0.0; Guo[i][j] = 0.0; }
    }
#pragma unroll
    for (int a = 0; a < A; ++a) {
#pragma unroll
      for (int i = 0; i < D; ++i) {
        const T yv = src.yn(a, i), yu = src.yn(a, D + i);
        const double ov = src.yo(a, i), ou = src.yo(a, D + i);
        vn[i] = vn[i] + N[a] * yv;
        un[i] = un[i] + N[a] * yu;
        vo[i] += N[a] * ov;
        uo[i] += N[a] * ou;
#pragma unroll
        for (int j = 0; j < D; ++j) {
          Gvn[i][j] = Gvn[i][j] + dN[a][j] * yv;
          Gun[i][j] = Gun[i][j] + dN[a][j] * yu;
          Gvo[i][j] += dN[a][j] * ov;
          Guo[i][j] += dN[a][j] * ou;
        }
      }
      const T yp = src.yn(a, 2 * D);
      pn = pn + N[a] * yp;
#pragma unroll
      for (int j = 0; j < D; ++j) gpn[j] = gpn[j] + dN[a][j] * yp;
    }

    T Fn[D][D], Fin[D][D];
    double Fo[D][D], Fio[D][D];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int j = 0; j < D; ++j) {
        Fn[i][j] = Gun[i][j] + (i == j ? 1.0 : 0.0);
        Fo[i][j] = Guo[i][j] + (i == j ? 1.0 : 0.0);
      }
    const T Jn = det_inv<D>(Fn, Fin);
    const double Jo = det_inv<D>(Fo, Fio);
    if (value_of(Jn) <= 0.0) degen = true;

    T vec[D], ten[D][D];
    if (!solid) {
      // ---- fluid: mass / ALE term at n-1/2
      T Fm[D][D], Fim[D][D], Gvm[D][D], GvFim[D][D];
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
          Fm[i][j] = 0.5 * (Fn[i][j] + Fo[i][j]);
          Gvm[i][j] = 0.5 * (Gvn[i][j] + Gvo[i][j]);
        }
      det_inv<D>(Fm, Fim);
      const T Jm = 0.5 * (Jn + Jo);
      matmul<D>(Gvm, Fim, GvFim);
      T GvFin[D][D];
      double GvFio[D][D];
      matmul<D>(Gvn, Fin, GvFin);
      matmul<D>(Gvo, Fio, GvFio);
#pragma unroll
      for (int i = 0; i < D; ++i) {
        T ale = T(0.0), cn = T(0.0);
        double co = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j) {
          ale = ale + GvFim[i][j] * (un[j] - uo[j]);
          cn = cn + GvFin[i][j] * vn[j];
          co += GvFio[i][j] * vo[j];
        }
        const T mass = ph.rho_f * Jm * ((vn[i] - vo[i]) - ale);
        vec[i] = mass + kt * (ph.rho_f * Jn * cn) + ko * (ph.rho_f * Jo * co);
      }
      // ---- Piola stresses J sigma F^{-T}; pressure p^n in both theta parts
      T Sn[D][D], So[D][D];
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
          Sn[i][j] = ph.rnu * (GvFin[i][j] + GvFin[j][i]);
          So[i][j] = T(ph.rnu * (GvFio[i][j] + GvFio[j][i]));
          if (i == j) { Sn[i][j] = Sn[i][j] - pn; So[i][j] = So[i][j] - pn; }
        }
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
          T pn_ij = T(0.0), po_ij = T(0.0);
#pragma unroll
          for (int m = 0; m < D; ++m) {
            pn_ij = pn_ij + Sn[i][m] * Fin[j][m];
            po_ij = po_ij + So[i][m] * Fio[j][m];
          }
          ten[i][j] = kt * (Jn * pn_ij) + ko * (Jo * po_ij);
        }
      // ---- divergence + pressure stabilization (p rows), extension (u rows)
      T div = GvFin[0][0];
#pragma unroll
      for (int i = 1; i < D; ++i) div = div + GvFin[i][i];
      div = Jn * div;
      const double W = ph.wq;
#pragma unroll
      for (int a = 0; a < A; ++a) {
        T gdot = gpn[0] * dN[a][0];
#pragma unroll
        for (int j = 1; j < D; ++j) gdot = gdot + gpn[j] * dN[a][j];
        R[a][2 * D] += (W * k) * (div * N[a] + st.delta * gdot);
        if ((ext_mask >> a) & 1) {
#pragma unroll
          for (int i = 0; i < D; ++i) {
            T e = T(0.0);
#pragma unroll
            for (int j = 0; j < D; ++j) e = e + (kt * Gun[i][j] + ko * Guo[i][j]) * dN[a][j];
            R[a][D + i] += W * e;
          }
        }
      }
    } else {
      // ---- solid: St. Venant-Kirchhoff first Piola F Sigma(E)
#pragma unroll
      for (int i = 0; i < D; ++i) vec[i] = ph.rho_s * (vn[i] - vo[i]);
      T En[D][D];
      double Eo[D][D];
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
          T sn = Fn[0][i] * Fn[0][j];
          double so = Fo[0][i] * Fo[0][j];
#pragma unroll
          for (int m = 1; m < D; ++m) { sn = sn + Fn[m][i] * Fn[m][j]; so += Fo[m][i] * Fo[m][j]; }
          En[i][j] = 0.5 * (sn - (i == j ? 1.0 : 0.0));
          Eo[i][j] = 0.5 * (so - (i == j ? 1.0 : 0.0));
        }
      T trn = En[0][0];
      double tro = Eo[0][0];
#pragma unroll
      for (int i = 1; i < D; ++i) { trn = trn + En[i][i]; tro += Eo[i][i]; }
      T Sg_n[D][D];
      double Sg_o[D][D];
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
          Sg_n[i][j] = 2.0 * ph.mu * En[i][j];
          Sg_o[i][j] = 2.0 * ph.mu * Eo[i][j];
          if (i == j) { Sg_n[i][j] = Sg_n[i][j] + ph.lam * trn; Sg_o[i][j] += ph.lam * tro; }
        }
      T Pn[D][D];
      double Po[D][D];
      matmul<D>(Fn, Sg_n, Pn);
      matmul<D>(Fo, Sg_o, Po);
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) ten[i][j] = kt * Pn[i][j] + ko * Po[i][j];
      // kinematic rows (u_n - u_o) - k theta v_n - k (1 - theta) v_o
      const double W = ph.wq;
#pragma unroll
      for (int a = 0; a < A; ++a)
#pragma unroll
        for (int i = 0; i < D; ++i) {
          const T kin = (un[i] - uo[i]) - kt * vn[i] - ko * vo[i];
          R[a][D + i] += W * (kin * N[a]);
        }
    }
    // momentum rows (both materials)
    const double W = ph.wq;
#pragma unroll
    for (int a = 0; a < A; ++a)
#pragma unroll
      for (int i = 0; i < D; ++i) {
        T s = vec[i] * N[a];
#pragma unroll
        for (int j = 0; j < D; ++j) s = s + ten[i][j] * dN[a][j];
        R[a][i] += W * s;
      }
  }

  // ---- do-nothing outflow correction  -< rho nu J F^{-T} grad v^T F^{-T} e_x , phi >
  if (cflag & kCellOutflow) {
#pragma unroll 1
    for (int q = 0; q < (A >> 1); ++q) {
      double xi[D];
      xi[0] = 1.0;
#pragma unroll
      for (int m = 1; m < D; ++m) xi[m] = ((q >> (m - 1)) & 1) ? kGaussHi : kGaussLo;
      double N[A], dN[A][D];
      q1_shape<D>(xi, ph.h, N, dN);
      T Gvn[D][D], Fn[D][D], Fin[D][D];
      double Gvo[D][D], Fo[D][D], Fio[D][D];
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
          Gvn[i][j] = T(0.0); Fn[i][j] = T(i == j ? 1.0 : 0.0);
          Gvo[i][j] = 0.0; Fo[i][j] = (i == j ? 1.0 : 0.0);
        }
#pragma unroll
      for (int a = 0; a < A; ++a)
#pragma unroll
        for (int i = 0; i < D; ++i) {
          const T yv = src.yn(a, i), yu = src.yn(a, D + i);
          const double ov = src.yo(a, i), ou = src.yo(a, D + i);
#pragma unroll
          for (int j = 0; j < D; ++j) {
            Gvn[i][j] = Gvn[i][j] + dN[a][j] * yv;
            Fn[i][j] = Fn[i][j] + dN[a][j] * yu;
            Gvo[i][j] += dN[a][j] * ov;
            Fo[i][j] += dN[a][j] * ou;
          }
        }
      const T Jn = det_inv<D>(Fn, Fin);
      const double Jo = det_inv<D>(Fo, Fio);
      T B[D];
#pragma unroll
      for (int i = 0; i < D; ++i) {
        // M_i0 = sum_{k,l} Fi[k][i] Gv[l][k] Fi[0][l]
        T mn = T(0.0);
        double mo = 0.0;
#pragma unroll
        for (int kk = 0; kk < D; ++kk)
#pragma unroll
          for (int l = 0; l < D; ++l) {
            mn = mn + Fin[kk][i] * Gvn[l][kk] * Fin[0][l];
            mo += Fio[kk][i] * Gvo[l][kk] * Fio[0][l];
          }
        B[i] = kt * (ph.rnu * Jn * mn) + ko * (ph.rnu * Jo * mo);
      }
#pragma unroll
      for (int a = 0; a < A; ++a)
#pragma unroll
        for (int i = 0; i < D; ++i) R[a][i] += (-ph.wf) * (B[i] * N[a]);
    }
  }
}

}  // namespace pint
