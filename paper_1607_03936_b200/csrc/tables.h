// tables.h -- 1-D basis / quadrature tables of the CUDA path, from CLOSED FORMS.
//
// Independent of the oracle (which derives its tables by Newton iteration):
// here every node and weight is a closed-form expression evaluated in long
// double, and every polynomial is written out explicitly.
//   * velocity: nodal Q_k on the GLL nodes (R1)
//   * quadrature: (k+1)-point Gauss-Legendre per axis (R3; north_star (2))
//   * pressure: orthonormal Legendre Lhat_m = sqrt((2m+1)/2) P_m, total degree
//     <= k-1 (R2; Table 3 p-DOF column PAPER.md:2830-2866)
#pragma once
#include <cmath>

namespace wb {

constexpr int MAXN1 = 5;  // k <= 4

struct Tab {
  double I[MAXN1][MAXN1];   // I[i][a]  = phi_a(xg_i)          GLL-Lagrange at Gauss points
  double D[MAXN1][MAXN1];   // D[i][a]  = phi_a'(xg_i)
  double Dg[MAXN1][MAXN1];  // Dg[i][j] = l_j'(xg_i), l_j Lagrange on the Gauss points (collocation derivative)
  double w[MAXN1];          // Gauss weights
  double BI[MAXN1][MAXN1];  // BI[m][a] = sum_i w_i Lhat_m(xg_i) phi_a(xg_i)
  double BD[MAXN1][MAXN1];  // BD[m][a] = sum_i w_i Lhat_m(xg_i) phi_a'(xg_i)
  double W1[MAXN1][MAXN1];  // W1[a][i] = phi_a(xg_i) w_i   (lumped mass, 1-D factor)
  double LG[MAXN1][MAXN1];  // LG[m][i] = Lhat_m(xg_i)      (pressure modes at the Gauss points)
};

// Closed-form node sets.
inline void nodes_closed_form(int k, long double* gll, long double* xg, long double* wg) {
  const long double r35 = sqrtl(3.0L / 5.0L);
  switch (k) {
    case 2:
      gll[0] = -1; gll[1] = 0; gll[2] = 1;
      xg[0] = -r35; xg[1] = 0; xg[2] = r35;
      wg[0] = 5.0L / 9; wg[1] = 8.0L / 9; wg[2] = 5.0L / 9;
      break;
    case 3: {
      const long double s15 = sqrtl(1.0L / 5.0L);
      gll[0] = -1; gll[1] = -s15; gll[2] = s15; gll[3] = 1;
      const long double t = 2.0L / 7.0L * sqrtl(6.0L / 5.0L);
      const long double x1 = sqrtl(3.0L / 7.0L - t), x2 = sqrtl(3.0L / 7.0L + t);
      const long double s30 = sqrtl(30.0L);
      xg[0] = -x2; xg[1] = -x1; xg[2] = x1; xg[3] = x2;
      wg[0] = (18.0L - s30) / 36; wg[1] = (18.0L + s30) / 36; wg[2] = wg[1]; wg[3] = wg[0];
      break;
    }
    case 4: {
      const long double s37 = sqrtl(3.0L / 7.0L);
      gll[0] = -1; gll[1] = -s37; gll[2] = 0; gll[3] = s37; gll[4] = 1;
      const long double r = 2.0L * sqrtl(10.0L / 7.0L);
      const long double x1 = sqrtl(5.0L - r) / 3.0L, x2 = sqrtl(5.0L + r) / 3.0L;
      const long double s70 = sqrtl(70.0L);
      xg[0] = -x2; xg[1] = -x1; xg[2] = 0; xg[3] = x1; xg[4] = x2;
      wg[0] = (322.0L - 13.0L * s70) / 900; wg[1] = (322.0L + 13.0L * s70) / 900;
      wg[2] = 128.0L / 225; wg[3] = wg[1]; wg[4] = wg[0];
      break;
    }
    default: break;
  }
}

// Orthonormal Legendre, explicit polynomials (m <= 3).
inline long double lhat(int m, long double x) {
  long double P = 0;
  switch (m) {
    case 0: P = 1; break;
    case 1: P = x; break;
    case 2: P = (3 * x * x - 1) / 2; break;
    case 3: P = (5 * x * x * x - 3 * x) / 2; break;
    default: P = 0;
  }
  return sqrtl((2.0L * m + 1.0L) / 2.0L) * P;
}

// Lagrange basis l_a on nodes x[0..n-1] and its derivative, product formulas.
inline long double lag(const long double* x, int n, int a, long double t) {
  long double v = 1;
  for (int b = 0; b < n; ++b)
    if (b != a) v *= (t - x[b]) / (x[a] - x[b]);
  return v;
}
inline long double dlag(const long double* x, int n, int a, long double t) {
  long double s = 0;
  for (int j = 0; j < n; ++j) {
    if (j == a) continue;
    long double v = 1 / (x[a] - x[j]);
    for (int b = 0; b < n; ++b)
      if (b != a && b != j) v *= (t - x[b]) / (x[a] - x[b]);
    s += v;
  }
  return s;
}

inline Tab make_tab(int k) {
  Tab T{};
  const int n1 = k + 1;
  long double gll[MAXN1] = {0}, xg[MAXN1] = {0}, wg[MAXN1] = {0};
  nodes_closed_form(k, gll, xg, wg);
  long double I[MAXN1][MAXN1], D[MAXN1][MAXN1];
  for (int i = 0; i < n1; ++i)
    for (int a = 0; a < n1; ++a) {
      I[i][a] = lag(gll, n1, a, xg[i]);
      D[i][a] = dlag(gll, n1, a, xg[i]);
      T.I[i][a] = (double)I[i][a];
      T.D[i][a] = (double)D[i][a];
      T.Dg[i][a] = (double)dlag(xg, n1, a, xg[i]);
    }
  for (int i = 0; i < n1; ++i) T.w[i] = (double)wg[i];
  for (int m = 0; m < k; ++m)
    for (int a = 0; a < n1; ++a) {
      long double si = 0, sd = 0;
      for (int i = 0; i < n1; ++i) {
        si += wg[i] * lhat(m, xg[i]) * I[i][a];
        sd += wg[i] * lhat(m, xg[i]) * D[i][a];
      }
      T.BI[m][a] = (double)si;
      T.BD[m][a] = (double)sd;
    }
  for (int a = 0; a < n1; ++a)
    for (int i = 0; i < n1; ++i) T.W1[a][i] = (double)(I[i][a] * wg[i]);
  for (int m = 0; m < k; ++m)
    for (int i = 0; i < n1; ++i) T.LG[m][i] = (double)lhat(m, xg[i]);
  return T;
}

}  // namespace wb
