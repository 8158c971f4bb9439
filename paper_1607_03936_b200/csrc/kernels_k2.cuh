// kernels_k2.cuh -- Q2 x P1disc (k = 2) hot-path kernels, the BASELINE C1-C3
// and C5 configurations.  No element-local buffer in HBM: B^T is computed
// node-centrically (gather, no scatter); A assembles each 4x4x4-element tile
// in shared memory and exchanges tile faces through a small L2-resident
// partial buffer with a deterministic look-back (no atomics on values).
#pragma once
#include "kernels.cuh"

namespace wb {

// Dense element gradient table without the factor sB:
// c_Bt2[c][a][m] = prod_d M_cd[m_d][a_d], M_cd = BD if d == c else BI, so that
// (B_e^T p)_{c,a} = sB * sum_m c_Bt2[c][a][m] p_m.
__constant__ double c_Bt2[3][27][4];

// Factorised form of the same matrix, c_Bt2[c][a][m] = X[m1][ax] * YZ[m2, m3](ay, az):
// c_W2[c][ay][az][k] = My_c[0][ay] Mz_c[0][az] (k = 0, weight of modes (0,0,0) and
// (1,0,0)), My_c[1][ay] Mz_c[0][az] (k = 1, mode (0,1,0)), My_c[0][ay] Mz_c[1][az]
// (k = 2, mode (0,0,1)); c_X2[c][ax][m1] = Mx_c[m1][ax].  (M_cd = BD if d == c else BI.)
__constant__ double c_W2[3][3][3][3];
__constant__ double c_X2[3][3][2];
// exact zeros: BI[1][1] = 0, BD[0][1] = 0
__host__ __device__ constexpr bool m_nz(bool deriv, int m, int a) { return !(a == 1 && (deriv ? m == 0 : m == 1)); }
__host__ __device__ constexpr bool w2_nz(int c, int ay, int az, int k) {
  return k == 0 ? (m_nz(c == 1, 0, ay) && m_nz(c == 2, 0, az))
                : (k == 1 ? (m_nz(c == 1, 1, ay) && m_nz(c == 2, 0, az)) : (m_nz(c == 1, 0, ay) && m_nz(c == 2, 1, az)));
}
__host__ __device__ constexpr bool x2_nz(int c, int ax, int m1) { return m_nz(c == 0, m1, ax); }

// ------------------------------------------------------------------ B^T, node-centric
// Node class (gx%2, gy%2, gz%2) is uniform across a warp, so the element
// pairs and local indices a are compile-time constants and every coefficient
// is a constant-bank operand.  Per axis: odd g -> one element (local 1); even
// g -> elements g/2-1 (local 2) and g/2 (local 0), ascending element order.
template <int RX, int RY, int RZ>
__device__ __forceinline__ void bt2_node(const double* __restrict__ p, int64_t se, int64_t sm, int gx, int gy, int gz,
                                         int N, double& t0, double& t1, double& t2) {
  constexpr int NX = RX ? 1 : 2, NY = RY ? 1 : 2, NZ = RZ ? 1 : 2;
#pragma unroll
  for (int iz = 0; iz < NZ; ++iz) {
    const int ez = RZ ? (gz >> 1) : ((gz >> 1) - 1 + iz);
    const int az = RZ ? 1 : (iz == 0 ? 2 : 0);
    if (ez < 0 || ez >= N) continue;
#pragma unroll
    for (int iy = 0; iy < NY; ++iy) {
      const int ey = RY ? (gy >> 1) : ((gy >> 1) - 1 + iy);
      const int ay = RY ? 1 : (iy == 0 ? 2 : 0);
      if (ey < 0 || ey >= N) continue;
#pragma unroll
      for (int ix = 0; ix < NX; ++ix) {
        const int ex = RX ? (gx >> 1) : ((gx >> 1) - 1 + ix);
        const int ax = RX ? 1 : (ix == 0 ? 2 : 0);
        if (ex < 0 || ex >= N) continue;
        const int64_t e = ex + (int64_t)N * (ey + (int64_t)N * ez);
        // p[e*se + m*sm]: element-major (caller) or mode-major (PCG, coalesced)
        double2 pa, pb;
        pa.x = __ldg(p + e * se); pa.y = __ldg(p + e * se + sm);
        pb.x = __ldg(p + e * se + 2 * sm); pb.y = __ldg(p + e * se + 3 * sm);
        const int a = ax + 3 * (ay + 3 * az);
        t0 = fma(c_Bt2[0][a][0], pa.x, t0); t0 = fma(c_Bt2[0][a][1], pa.y, t0);
        t0 = fma(c_Bt2[0][a][2], pb.x, t0); t0 = fma(c_Bt2[0][a][3], pb.y, t0);
        t1 = fma(c_Bt2[1][a][0], pa.x, t1); t1 = fma(c_Bt2[1][a][1], pa.y, t1);
        t1 = fma(c_Bt2[1][a][2], pb.x, t1); t1 = fma(c_Bt2[1][a][3], pb.y, t1);
        t2 = fma(c_Bt2[2][a][0], pa.x, t2); t2 = fma(c_Bt2[2][a][1], pa.y, t2);
        t2 = fma(c_Bt2[2][a][2], pb.x, t2); t2 = fma(c_Bt2[2][a][3], pb.y, t2);
      }
    }
  }
}

// y[c][g] = sB * s[g] * (B^T p)_c(g)   (s = X^-1 nodal diagonal, or none -> mask)
// block (64, 4): x -> element column jx (gx = 2 jx + rx), y -> 4 node rows gy;
// grid (ceil((N+1)/64), ceil(nn1/4), nn1 * 2): z -> (gz, rx).
__global__ void __launch_bounds__(256) k_BT_node2(const double* __restrict__ p, const double* __restrict__ s,
                                                  double* __restrict__ y, Geo G, double sB, int nomask,
                                                  const int* __restrict__ stop, int64_t se, int64_t sm) {
  if (stop && *stop) return;
  const int rx = blockIdx.z & 1, gz = blockIdx.z >> 1;
  const int gx = 2 * (blockIdx.x * 64 + threadIdx.x) + rx;
  const int gy = blockIdx.y * 4 + threadIdx.y;
  const int nn1 = G.nn1;
  if (gx >= nn1 || gy >= nn1) return;
  const int64_t g = node_id(gx, gy, gz, nn1);
  if (!nomask && node_bnd(gx, gy, gz, nn1)) {
    y[g] = 0.0; y[G.n_nodes + g] = 0.0; y[2 * G.n_nodes + g] = 0.0;
    return;
  }
  double t0 = 0.0, t1 = 0.0, t2 = 0.0;
  const int cls = rx | ((gy & 1) << 1) | ((gz & 1) << 2);  // warp-uniform
  switch (cls) {
    case 0: bt2_node<0, 0, 0>(p, se, sm, gx, gy, gz, G.N, t0, t1, t2); break;
    case 1: bt2_node<1, 0, 0>(p, se, sm, gx, gy, gz, G.N, t0, t1, t2); break;
    case 2: bt2_node<0, 1, 0>(p, se, sm, gx, gy, gz, G.N, t0, t1, t2); break;
    case 3: bt2_node<1, 1, 0>(p, se, sm, gx, gy, gz, G.N, t0, t1, t2); break;
    case 4: bt2_node<0, 0, 1>(p, se, sm, gx, gy, gz, G.N, t0, t1, t2); break;
    case 5: bt2_node<1, 0, 1>(p, se, sm, gx, gy, gz, G.N, t0, t1, t2); break;
    case 6: bt2_node<0, 1, 1>(p, se, sm, gx, gy, gz, G.N, t0, t1, t2); break;
    default: bt2_node<1, 1, 1>(p, se, sm, gx, gy, gz, G.N, t0, t1, t2); break;
  }
  const double f = s ? sB * s[g] : sB;
  y[g] = f * t0; y[G.n_nodes + g] = f * t1; y[2 * G.n_nodes + g] = f * t2;
}


}  // namespace wb

#include "a2_tile.cuh"
#include "k2_fused.cuh"
#include "k2_tma.cuh"
#include "k2_zm.cuh"
#include "k2_mg.cuh"
#include "k_schur.cuh"
#include "k2_bbt.cuh"
#include "k2_setup.cuh"
#include "k4_fused.cuh"
#include "k2_zc.cuh"
