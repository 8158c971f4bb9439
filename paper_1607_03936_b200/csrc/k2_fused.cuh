// k2_fused.cuh -- fused Poisson operator K_w p = B (X o (B^T p)) for k = 2
// (row a8) with the PCG direction update folded in (row a9), one kernel per
// CG iteration on top of the vector update kernel.
//
// PCG vectors inside the library are mode-major ("SoA"): v[m * n_el + e].
// One CTA owns a TX x TY x TZ element tile:
//  0. p for the tile and a one-element halo -> shared memory, computed on the
//     fly as  p = Minv r (first iteration), Minv r + beta p_old, or p_old as is;
//     the tile's own elements are written to p_new (double buffer).
//  1. t = sB X o (B^T p) at the tile's (2T+1)^3 nodes, node-centric: for a
//     node class (gx%2, gy%2, gz%2) the contributing elements and their local
//     indices are compile-time constants, so each coefficient is a constant-
//     bank operand and exact zeros of the element matrix are skipped at compile
//     time.  Elements in ascending index order per node (the oracle's order).
//  2. q_e = sB Bt^T t_e per tile element (dense, zero-skipping), write q, and
//     <p, q> through the fixed-order grid reduction.
#pragma once
#include "kernels.cuh"  // included from kernels_k2.cuh, after c_Bt2

namespace wb {

// Exact zero pattern of the k = 2 element matrix:
// BI[1][1] = int x phi_1 = 0 and BD[0][1] = int phi_1' = 0 (phi_1 even), so
// prod_d M_cd[m_d][a_d] vanishes iff some axis d has a_d = 1 and
// (d != c and m_d = 1) or (d == c and m_d = 0).
__host__ __device__ constexpr bool bt2_nz(int c, int a, int m) {
  // modes: 0 = (0,0,0), 1 = (1,0,0), 2 = (0,1,0), 3 = (0,0,1)
  return !((a % 3 == 1) && ((0 != c && m == 1) || (0 == c && m != 1))) &&
         !(((a / 3) % 3 == 1) && ((1 != c && m == 2) || (1 == c && m != 2))) &&
         !((a / 9 == 1) && ((2 != c && m == 3) || (2 == c && m != 3)));
}

template <int TX, int TY, int TZ>
struct FK2 {
  static constexpr int NE = TX * TY * TZ;
  static constexpr int HX = TX + 2, HY = TY + 2, HZ = TZ + 2, NH = HX * HY * HZ;  // halo box
  static constexpr int MX = 2 * TX + 1, MY = 2 * TY + 1, MZ = 2 * TZ + 1, NN = MX * MY * MZ;
  static constexpr size_t SMEM = sizeof(double) * (4 * NH + 4 * NN);  // Ps, T, Xs
};

// node-centric B^T at one tile node of class (RX, RY, RZ); (hx, hy, hz) = halo-box
// coordinates of the element whose local node 1 (odd axis) or 0 (even axis) it is.
template <int TX, int TY, int TZ, int RX, int RY, int RZ>
__device__ __forceinline__ void fk2_node(const double* __restrict__ Ps, int hx, int hy, int hz, double& t0,
                                         double& t1, double& t2) {
  using F = FK2<TX, TY, TZ>;
  constexpr int NX = RX ? 1 : 2, NY = RY ? 1 : 2, NZ = RZ ? 1 : 2;
#pragma unroll
  for (int iz = 0; iz < NZ; ++iz) {
    const int az = RZ ? 1 : (iz == 0 ? 2 : 0);
    const int qz = RZ ? hz : hz - 1 + iz;
#pragma unroll
    for (int iy = 0; iy < NY; ++iy) {
      const int ay = RY ? 1 : (iy == 0 ? 2 : 0);
      const int qy = RY ? hy : hy - 1 + iy;
#pragma unroll
      for (int ix = 0; ix < NX; ++ix) {
        const int ax = RX ? 1 : (ix == 0 ? 2 : 0);
        const int qx = RX ? hx : hx - 1 + ix;
        const int h = qx + F::HX * (qy + F::HY * qz);
        const int a = ax + 3 * (ay + 3 * az);
        double pm[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) pm[m] = Ps[m * F::NH + h];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          if (bt2_nz(0, a, m)) t0 = fma(c_Bt2[0][a][m], pm[m], t0);
          if (bt2_nz(1, a, m)) t1 = fma(c_Bt2[1][a][m], pm[m], t1);
          if (bt2_nz(2, a, m)) t2 = fma(c_Bt2[2][a][m], pm[m], t2);
        }
      }
    }
  }
}

// Xs[n] = sB X[g(n)] at the tile nodes (0 outside the domain; X = 0 on the boundary)
template <int TX, int TY, int TZ, int RX, int RY, int RZ>
__device__ __forceinline__ void fk2_class(const double* __restrict__ Ps, double* __restrict__ T,
                                          const double* __restrict__ Xs) {
  using F = FK2<TX, TY, TZ>;
  // tile-local node n = 2*l + R: l in [0, T] for R = 0, [0, T) for R = 1
  constexpr int CX = RX ? TX : TX + 1, CY = RY ? TY : TY + 1, CZ = RZ ? TZ : TZ + 1, CN = CX * CY * CZ;
  for (int i = threadIdx.x; i < CN; i += F::NE) {
    const int lx = i % CX, ly = (i / CX) % CY, lz = i / (CX * CY);
    const int n = (2 * lx + RX) + F::MX * ((2 * ly + RY) + F::MY * (2 * lz + RZ));
    double t0 = 0.0, t1 = 0.0, t2 = 0.0;
    const double f = Xs[n];
    if (f != 0.0) {
      // element containing the node as local 1 (odd) / 0 (even) sits at halo index l + 1
      fk2_node<TX, TY, TZ, RX, RY, RZ>(Ps, lx + 1, ly + 1, lz + 1, t0, t1, t2);
      t0 *= f; t1 *= f; t2 *= f;
    }
    T[n] = t0; T[F::NN + n] = t1; T[2 * F::NN + n] = t2;
  }
}

// mode: 0 -> p = Minv r; 1 -> p = Minv r + beta p_old, beta = rz[0]/rz[-1]; 2 -> p = p_old
template <int TX, int TY, int TZ, int MINB>
__global__ void __launch_bounds__(TX * TY * TZ, MINB)
    k_K2_fused(const double* __restrict__ pold, double* __restrict__ pnew, const double* __restrict__ r,
               const double* __restrict__ Minv, const double* __restrict__ X, double* __restrict__ q, Geo G,
               double sB, int mode, const double* __restrict__ rz, const int* __restrict__ stop, double* partial,
               unsigned* counter, double* pq) {
  using F = FK2<TX, TY, TZ>;
  extern __shared__ __align__(16) double sm[];
  double* Ps = sm;               // [4][NH]
  double* T = sm + 4 * F::NH;    // [3][NN]
  double* Xs = T + 3 * F::NN;    // [NN]
  if (stop && *stop) return;
  const int N = G.N;
  const int64_t ne = G.n_el;
  const int NTX = (N + TX - 1) / TX, NTY = (N + TY - 1) / TY;
  const int tile = blockIdx.x;
  const int tx = tile % NTX, ty = (tile / NTX) % NTY, tz = tile / (NTX * NTY);
  const int ex0 = TX * tx, ey0 = TY * ty, ez0 = TZ * tz;
  const double beta = (mode == 1) ? rz[0] / rz[-1] : 0.0;
  // 0. X at the tile nodes (scaled by sB) and p on the tile + halo.  Every
  // global load of this phase is issued before any is consumed (the loops are
  // fully unrolled over the thread's share), so the phase costs one memory
  // round trip instead of one per item.
  const int bx = 2 * ex0, by = 2 * ey0, bz = 2 * ez0;
  constexpr int XPER = (F::NN + F::NE - 1) / F::NE, HPER = (F::NH + F::NE - 1) / F::NE;
  double xv[XPER];
#pragma unroll
  for (int k = 0; k < XPER; ++k) {
    const int i = threadIdx.x + k * F::NE;
    const int nx = i % F::MX, ny = (i / F::MX) % F::MY, nz = i / (F::MX * F::MY);
    const int gx = bx + nx, gy = by + ny, gz = bz + nz;
    xv[k] = (i < F::NN && gx < G.nn1 && gy < G.nn1 && gz < G.nn1) ? __ldg(X + node_id(gx, gy, gz, G.nn1)) : 0.0;
  }
  double po[HPER][4], rr[HPER][4], mi[HPER][4];
  int64_t he[HPER];
#pragma unroll
  for (int k = 0; k < HPER; ++k) {
    const int i = threadIdx.x + k * F::NE;
    const int hx = i % F::HX, hy = (i / F::HX) % F::HY, hz = i / (F::HX * F::HY);
    const int ex = ex0 + hx - 1, ey = ey0 + hy - 1, ez = ez0 + hz - 1;
    const bool ok = i < F::NH && ex >= 0 && ey >= 0 && ez >= 0 && ex < N && ey < N && ez < N;
    he[k] = ok ? ex + (int64_t)N * (ey + (int64_t)N * ez) : -1;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      po[k][m] = (ok && mode != 0) ? __ldg(pold + m * ne + he[k]) : 0.0;
      rr[k][m] = (ok && mode != 2) ? __ldg(r + m * ne + he[k]) : 0.0;
      mi[k][m] = (ok && mode != 2) ? __ldg(Minv + m * ne + he[k]) : 0.0;
    }
  }
#pragma unroll
  for (int k = 0; k < XPER; ++k) {
    const int i = threadIdx.x + k * F::NE;
    if (i < F::NN) Xs[i] = sB * xv[k];
  }
#pragma unroll
  for (int k = 0; k < HPER; ++k) {
    const int i = threadIdx.x + k * F::NE;
    if (i >= F::NH) continue;
    const int hx = i % F::HX, hy = (i / F::HX) % F::HY, hz = i / (F::HX * F::HY);
    const bool own = he[k] >= 0 && hx >= 1 && hy >= 1 && hz >= 1 && hx <= TX && hy <= TY && hz <= TZ;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      double v = 0.0;
      if (he[k] >= 0) {
        if (mode == 2) v = po[k][m];
        else {
          const double z = mi[k][m] * rr[k][m];
          v = (mode == 1) ? fma(beta, po[k][m], z) : z;
        }
        if (own) pnew[m * ne + he[k]] = v;
      }
      Ps[m * F::NH + i] = v;
    }
  }
  __syncthreads();
  // 1. t at the tile nodes, class by class (warp-uniform coefficients)
  fk2_class<TX, TY, TZ, 0, 0, 0>(Ps, T, Xs);
  fk2_class<TX, TY, TZ, 1, 0, 0>(Ps, T, Xs);
  fk2_class<TX, TY, TZ, 0, 1, 0>(Ps, T, Xs);
  fk2_class<TX, TY, TZ, 1, 1, 0>(Ps, T, Xs);
  fk2_class<TX, TY, TZ, 0, 0, 1>(Ps, T, Xs);
  fk2_class<TX, TY, TZ, 1, 0, 1>(Ps, T, Xs);
  fk2_class<TX, TY, TZ, 0, 1, 1>(Ps, T, Xs);
  fk2_class<TX, TY, TZ, 1, 1, 1>(Ps, T, Xs);
  __syncthreads();
  // 2. q = sB Bt^T t per element
  const int lx = threadIdx.x % TX, ly = (threadIdx.x / TX) % TY, lz = threadIdx.x / (TX * TY);
  const int ex = ex0 + lx, ey = ey0 + ly, ez = ez0 + lz;
  double dot = 0.0;
  if (ex < N && ey < N && ez < N) {
    double qm[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int a = 0; a < 27; ++a) {
        const int n = (2 * lx + a % 3) + F::MX * ((2 * ly + (a / 3) % 3) + F::MY * (2 * lz + a / 9));
        const double tv = T[c * F::NN + n];
#pragma unroll
        for (int m = 0; m < 4; ++m)
          if (bt2_nz(c, a, m)) qm[m] = fma(c_Bt2[c][a][m], tv, qm[m]);
      }
    const int64_t e = ex + (int64_t)N * (ey + (int64_t)N * ez);
    const int h = (lx + 1) + F::HX * ((ly + 1) + F::HY * (lz + 1));
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const double o = sB * qm[m];
      q[m * ne + e] = o;
      dot = fma(Ps[m * F::NH + h], o, dot);
    }
  }
  grid_sum<TX * TY * TZ>(dot, partial, counter, pq);
}

}  // namespace wb
