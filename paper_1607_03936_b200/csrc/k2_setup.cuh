// k2_setup.cuh -- viscosity setup for k = 2 (rows a3, a4): scaled quadrature
// viscosity, weighted lumped masses C_w / D_w and the Jacobi diagonals of
// K_w = B X^-1 B^T.  Same quantities as the generic kernels in kernels.cuh
// (k_prescale, k_lump_elem / k_lump_node, k_jacobi); here with the k = 2
// structure compile-time: one pass over mu, sum-factorised lumping, node
// classes uniform per warp.
#pragma once
#include "a2_tile.cuh"

namespace wb {

// c_J2[a][m] = sum_c Bt2[c][a][m]^2 (without sB^2): diag(K)_{e,m} = sB^2 sum_a c_J2[a][m] X[g(e,a)]
__constant__ double c_J2[27][4];

// One thread per element, one read of its 27 mu samples:
//   mutT[tile][q][le] = mu w_q h/2          (A's tile-blocked layout, as k_prescale for k = 3, 4)
//   L[a][e] = detJ sum_q sqrt(mu_q) phi_a(xi_q) w_q   (eq:lumping),
//   with mu_eff = wsrc in the square root when given (R17)
// with L sum-factorised (x, y, z passes of the 1-D factor W1[a][i] = phi_a(xg_i) w_i).
// Nonpositive or non-finite mu samples are counted in bad (the caller rejects them).
template <int TX, int TY, int TZ>
__global__ void __launch_bounds__(128) k_setup_mu2(const double* __restrict__ mu, double* __restrict__ mutT,
                                                   double* __restrict__ L, int N, double hs, double detJ,
                                                   unsigned long long* bad, const double* __restrict__ wsrc) {
  constexpr int NE = TX * TY * TZ;
  const int64_t ne = (int64_t)N * N * N;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ne) return;
  const int ex = (int)(e % N), ey = (int)((e / N) % N), ez = (int)(e / ((int64_t)N * N));
  const int NTX = (N + TX - 1) / TX, NTY = (N + TY - 1) / TY;
  const int tile = ex / TX + NTX * (ey / TY + NTY * (ez / TZ));
  const int le = ex % TX + TX * (ey % TY + TY * (ez % TZ));
  double s[27];
  int nbad = 0;
#pragma unroll
  for (int q = 0; q < 27; ++q) {
    const double m = mu[e * 27 + q];
    if (!(m > 0.0) || !isfinite(m)) ++nbad;
    const double wq = TB(2).w[q % 3] * TB(2).w[(q / 3) % 3] * TB(2).w[q / 9];
    mutT[((int64_t)tile * 27 + q) * NE + le] = m * wq * hs;
    s[q] = sqrt(wsrc ? wsrc[e * 27 + q] : m);  // wsrc: the gradient weights' mu_eff (R17)
  }
  if (nbad) atomicAdd(bad, (unsigned long long)nbad);
  // x pass: t1[qz][qy][ax] = sum_qx W1[ax][qx] s[qz][qy][qx]
  double t1[27], t2[27];
#pragma unroll
  for (int r = 0; r < 9; ++r)
#pragma unroll
    for (int ax = 0; ax < 3; ++ax)
      t1[r * 3 + ax] = fma(TB(2).W1[ax][0], s[r * 3], fma(TB(2).W1[ax][1], s[r * 3 + 1], TB(2).W1[ax][2] * s[r * 3 + 2]));
  // y pass: t2[qz][ay][ax] = sum_qy W1[ay][qy] t1[qz][qy][ax]
#pragma unroll
  for (int qz = 0; qz < 3; ++qz)
#pragma unroll
    for (int ay = 0; ay < 3; ++ay)
#pragma unroll
      for (int ax = 0; ax < 3; ++ax)
        t2[(qz * 3 + ay) * 3 + ax] =
            fma(TB(2).W1[ay][0], t1[(qz * 3 + 0) * 3 + ax],
                fma(TB(2).W1[ay][1], t1[(qz * 3 + 1) * 3 + ax], TB(2).W1[ay][2] * t1[(qz * 3 + 2) * 3 + ax]));
  // z pass -> L[a][e], a = ax + 3 (ay + 3 az)
#pragma unroll
  for (int az = 0; az < 3; ++az)
#pragma unroll
    for (int r = 0; r < 9; ++r)
      L[(int64_t)(az * 9 + r) * ne + e] =
          detJ * fma(TB(2).W1[az][0], t2[r], fma(TB(2).W1[az][1], t2[9 + r], TB(2).W1[az][2] * t2[18 + r]));
}

// C[g] = sum_{e ni g} a(e) L[a(e,g)][e] in ascending element order (eq:bdramp,
// PAPER.md:2232-2245; a = a_l or a_r on boundary elements, else 1), Xinv = mask / X,
// nonpositive interior entries counted.  Launch geometry and warp-uniform node
// class as k_BT_node2: block (64, 4), grid (ceil((N+1)/64), ceil(nn1/4), 2 nn1).
template <int RX, int RY, int RZ>
__device__ __forceinline__ void lump2_node(const double* __restrict__ L, int64_t ne, int N, int gx, int gy, int gz,
                                           double a_l, double a_r, double& cl, double& cr, int zopen) {
#pragma unroll
  for (int iz = 0; iz < (RZ ? 1 : 2); ++iz) {
    const int ez = RZ ? (gz >> 1) : ((gz >> 1) - 1 + iz), az = RZ ? 1 : (iz == 0 ? 2 : 0);
    if (ez < 0 || ez >= N) continue;
#pragma unroll
    for (int iy = 0; iy < (RY ? 1 : 2); ++iy) {
      const int ey = RY ? (gy >> 1) : ((gy >> 1) - 1 + iy), ay = RY ? 1 : (iy == 0 ? 2 : 0);
      if (ey < 0 || ey >= N) continue;
#pragma unroll
      for (int ix = 0; ix < (RX ? 1 : 2); ++ix) {
        const int ex = RX ? (gx >> 1) : ((gx >> 1) - 1 + ix), ax = RX ? 1 : (ix == 0 ? 2 : 0);
        if (ex < 0 || ex >= N) continue;
        const int64_t e = ex + (int64_t)N * (ey + (int64_t)N * ez);
        const bool onb = ex == 0 || ey == 0 || (ez == 0 && !(zopen & 1)) || ex == N - 1 || ey == N - 1 ||
                         (ez == N - 1 && !(zopen & 2));
        const double l = __ldg(L + (int64_t)(ax + 3 * (ay + 3 * az)) * ne + e);
        cl += (onb ? a_l : 1.0) * l;
        cr += (onb ? a_r : 1.0) * l;
      }
    }
  }
}

__global__ void __launch_bounds__(256) k_lump_node2(const double* __restrict__ L, double a_l, double a_r, double* Cw,
                                                    double* Dw, double* Cinv, double* Dinv,
                                                    unsigned long long* nonpos, Geo G) {
  const int rx = blockIdx.z & 1, gz = blockIdx.z >> 1;
  const int gx = 2 * (blockIdx.x * 64 + threadIdx.x) + rx;
  const int gy = blockIdx.y * 4 + threadIdx.y;
  const int nn1 = G.nn1;
  if (gx >= nn1 || gy >= nn1) return;
  double cl = 0.0, cr = 0.0;
  const int cls = rx | ((gy & 1) << 1) | ((gz & 1) << 2);  // warp-uniform
  switch (cls) {
    case 0: lump2_node<0, 0, 0>(L, G.n_el, G.N, gx, gy, gz, a_l, a_r, cl, cr, G.zopen); break;
    case 1: lump2_node<1, 0, 0>(L, G.n_el, G.N, gx, gy, gz, a_l, a_r, cl, cr, G.zopen); break;
    case 2: lump2_node<0, 1, 0>(L, G.n_el, G.N, gx, gy, gz, a_l, a_r, cl, cr, G.zopen); break;
    case 3: lump2_node<1, 1, 0>(L, G.n_el, G.N, gx, gy, gz, a_l, a_r, cl, cr, G.zopen); break;
    case 4: lump2_node<0, 0, 1>(L, G.n_el, G.N, gx, gy, gz, a_l, a_r, cl, cr, G.zopen); break;
    case 5: lump2_node<1, 0, 1>(L, G.n_el, G.N, gx, gy, gz, a_l, a_r, cl, cr, G.zopen); break;
    case 6: lump2_node<0, 1, 1>(L, G.n_el, G.N, gx, gy, gz, a_l, a_r, cl, cr, G.zopen); break;
    default: lump2_node<1, 1, 1>(L, G.n_el, G.N, gx, gy, gz, a_l, a_r, cl, cr, G.zopen); break;
  }
  const int64_t g = node_id(gx, gy, gz, nn1);
  const bool b = node_bnd(gx, gy, gz, nn1);
  Cw[g] = cl; Dw[g] = cr;
  Cinv[g] = b ? 0.0 : 1.0 / cl;
  Dinv[g] = b ? 0.0 : 1.0 / cr;
  if (!b && cl <= 0.0) atomicAdd(nonpos + 0, 1ull);
  if (!b && cr <= 0.0) atomicAdd(nonpos + 1, 1ull);
}

// diag(K_side)_{e,m} = sB^2 sum_a c_J2[a][m] X_side[g(e,a)], element-major [e*4 + m]
// (the Minv pseudo-inverse follows in k_minv, R11).
__global__ void __launch_bounds__(128) k_jacobi2(const double* __restrict__ Cinv, const double* __restrict__ Dinv,
                                                 double* dL, double* dR, Geo G, double sB2) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= G.n_el) return;
  int ex, ey, ez;
  elem_xyz(e, G.N, ex, ey, ez);
  double sl[4] = {0.0, 0.0, 0.0, 0.0}, sr[4] = {0.0, 0.0, 0.0, 0.0};
  const double* cb = Cinv + node_id(2 * ex, 2 * ey, 2 * ez, G.nn1);
  const double* db = Dinv + node_id(2 * ex, 2 * ey, 2 * ez, G.nn1);
#pragma unroll
  for (int a = 0; a < 27; ++a) {
    const int64_t o = (a % 3) + (int64_t)G.nn1 * (((a / 3) % 3) + (int64_t)G.nn1 * (a / 9));
    const double xl = __ldg(cb + o), xr = __ldg(db + o);
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      sl[m] = fma(c_J2[a][m], xl, sl[m]);
      sr[m] = fma(c_J2[a][m], xr, sr[m]);
    }
  }
#pragma unroll
  for (int m = 0; m < 4; ++m) { dL[e * 4 + m] = sB2 * sl[m]; dR[e * 4 + m] = sB2 * sr[m]; }
}

}  // namespace wb
