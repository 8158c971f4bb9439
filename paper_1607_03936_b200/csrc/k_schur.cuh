// k_schur.cuh -- kernels of the Schur-complement variants beside wBFBT:
//  * diag(A)-BFBT (C = D = diag(A)): the Jacobi diagonal of the pressure
//    Poisson operator with a per-DOF (per component) weight X = mask / diag(A);
//  * the inverse viscosity-weighted pressure mass M_p(1/mu), applied as its
//    exact element-block inverse (P_{k-1}^disc is discontinuous, so M_p is block diagonal;
//    reading R21 in DESIGN.md: the eq:lumping diagonal degenerates in the orthonormal modal
//    basis of R2).
#pragma once
#include "kernels.cuh"

namespace wb {

template <int K>
__device__ __forceinline__ void mode_exps(int (&mm)[Ord<K>::NM][3]) {
  int m = 0;
  for (int d = 0; d < K; ++d)
    for (int m3 = 0; m3 <= d; ++m3)
      for (int m2 = 0; m2 <= d - m3; ++m2) { mm[m][0] = d - m2 - m3; mm[m][1] = m2; mm[m][2] = m3; ++m; }
}

// diag(K)_{e,m} = sum_{c,a} B_e[m,(c,a)]^2 X[c][g(e,a)], element-major output
template <int K>
__global__ void k_jacobi_dof(const double* __restrict__ X, double* __restrict__ diag, Geo G, double sB) {
  constexpr int n1 = K + 1, NQ = Ord<K>::NQ, NM = Ord<K>::NM;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= G.n_el) return;
  int ex, ey, ez;
  elem_xyz(e, G.N, ex, ey, ez);
  int mm[NM][3];
  mode_exps<K>(mm);
  double s[NM];
#pragma unroll
  for (int m = 0; m < NM; ++m) s[m] = 0.0;
#pragma unroll 1
  for (int c = 0; c < 3; ++c)
#pragma unroll 1
    for (int a = 0; a < NQ; ++a) {
      const int ax = a % n1, ay = (a / n1) % n1, az = a / (n1 * n1);
      const int64_t g = node_id(K * ex + ax, K * ey + ay, K * ez + az, G.nn1);
      const double x = X[(int64_t)c * G.n_nodes + g];
#pragma unroll
      for (int m = 0; m < NM; ++m) {
        const double fx = c == 0 ? TB(K).BD[mm[m][0]][ax] : TB(K).BI[mm[m][0]][ax];
        const double fy = c == 1 ? TB(K).BD[mm[m][1]][ay] : TB(K).BI[mm[m][1]][ay];
        const double fz = c == 2 ? TB(K).BD[mm[m][2]][az] : TB(K).BI[mm[m][2]][az];
        const double b = sB * (fx * fy * fz);
        s[m] = fma(b * b, x, s[m]);
      }
    }
#pragma unroll
  for (int m = 0; m < NM; ++m) diag[e * NM + m] = s[m];
}

// Minv = pseudo-inverse of a diagonal (R11): 1/d, 0 where |d| <= 1e-13 max|d| (element-major)
__global__ void k_pinv_diag(const double* __restrict__ d, double* __restrict__ minv, int64_t n,
                            const double* __restrict__ dmax) {
  const double t = 1e-13 * *dmax;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    minv[i] = fabs(d[i]) > t ? 1.0 / d[i] : 0.0;
}

// y = x o w (elementwise), y may equal x
__global__ void k_mul(double* y, const double* x, const double* __restrict__ w, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = x[i] * w[i];
}

// Per element: M_e[i][j] = sum_q w_q detJ q_i(xi_q) q_j(xi_q) / mu_q (q_i orthonormal modes
// on the reference element, R2), then its inverse by Cholesky (M_e is SPD for mu > 0),
// stored row-major NM x NM.  One thread per element; the NM x NM work arrays live in
// thread-local memory (setup only).
template <int K>
__global__ void k_mp_setup(const double* __restrict__ mu, double* __restrict__ Minv, int64_t n_el, double detJ) {
  constexpr int n1 = K + 1, NQ = Ord<K>::NQ, NM = Ord<K>::NM;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_el) return;
  int mm[NM][3];
  mode_exps<K>(mm);
  double M[NM][NM];
  for (int i = 0; i < NM; ++i)
    for (int j = 0; j < NM; ++j) M[i][j] = 0.0;
  const double* me = mu + e * NQ;
  for (int q = 0; q < NQ; ++q) {
    const int qx = q % n1, qy = (q / n1) % n1, qz = q / (n1 * n1);
    const double wq = TB(K).w[qx] * TB(K).w[qy] * TB(K).w[qz] * detJ / me[q];
    double v[NM];
    for (int i = 0; i < NM; ++i)
      v[i] = TB(K).LG[mm[i][0]][qx] * TB(K).LG[mm[i][1]][qy] * TB(K).LG[mm[i][2]][qz];
    for (int i = 0; i < NM; ++i)
      for (int j = 0; j <= i; ++j) M[i][j] = fma(wq * v[i], v[j], M[i][j]);
  }
  // Cholesky M = L L^T (lower triangle in place)
  for (int j = 0; j < NM; ++j) {
    double d = M[j][j];
    for (int k = 0; k < j; ++k) d -= M[j][k] * M[j][k];
    d = sqrt(d);
    M[j][j] = d;
    for (int i = j + 1; i < NM; ++i) {
      double s = M[i][j];
      for (int k = 0; k < j; ++k) s -= M[i][k] * M[j][k];
      M[i][j] = s / d;
    }
  }
  // inverse column by column: solve L L^T x = e_col
  double* out = Minv + e * NM * NM;
  for (int col = 0; col < NM; ++col) {
    double y[NM];
    for (int i = 0; i < NM; ++i) {
      double s = (i == col) ? 1.0 : 0.0;
      for (int k = 0; k < i; ++k) s -= M[i][k] * y[k];
      y[i] = s / M[i][i];
    }
    for (int i = NM - 1; i >= 0; --i) {
      double s = y[i];
      for (int k = i + 1; k < NM; ++k) s -= M[k][i] * y[k];
      y[i] = s / M[i][i];
    }
    for (int i = 0; i < NM; ++i) out[i * NM + col] = y[i];
  }
}

// z_e = scale * Minv_e r_e (element-major), one thread per element
template <int NM>
__global__ void k_mp_apply(const double* __restrict__ Minv, const double* __restrict__ r, double* __restrict__ z,
                           int64_t n_el, double scale) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_el) return;
  double rv[NM];
#pragma unroll
  for (int j = 0; j < NM; ++j) rv[j] = r[e * NM + j];
  const double* Mi = Minv + e * NM * NM;
#pragma unroll
  for (int i = 0; i < NM; ++i) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < NM; ++j) s = fma(Mi[i * NM + j], rv[j], s);
    z[e * NM + i] = scale * s;
  }
}

}  // namespace wb
