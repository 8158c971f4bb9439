// k2_fused.cuh -- fused Poisson operator K_w p = B (X o (B^T p)) for k = 2
// (row a8) with the PCG direction update folded in (row a9): one kernel per CG
// iteration on top of the vector-update kernel.
//
// PCG vectors inside the library are mode-major ("SoA"): v[m * n_el + e].
// One CTA owns a TX x TY x TZ element tile:
//  0. p for the tile and a one-element halo -> shared memory Ps, computed on
//     the fly as p = Minv r (first iteration), Minv r + beta p_old, or p_old as
//     is; the tile's own elements are written to p_new (double buffer).
//  1. t = sB X o (B^T p) at the tile's (2T+1)^3 nodes, by x-pencils: one thread
//     owns a node row (ny, nz) and walks the halo elements along x, so each
//     element's four p values feed the three nodes it touches from registers.
//     The row's class (ny % 2, nz % 2) is warp-uniform, which makes every
//     element-local index, and therefore every coefficient, a compile-time
//     constant-bank operand; exact zeros of the element matrix are skipped at
//     compile time (bt2_nz).  Per node the elements are summed in ascending
//     element index (z, then y, then x), the oracle's scatter order.
//  2. q_e = sB Bt^T t_e per tile element (dense, zero-skipping), q written,
//     <p, q> through the fixed-order grid reduction.
// Node rows in shared memory are split by x parity (even nodes, then odd) so
// that consecutive elements read consecutive words (no stride-2 conflicts).
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
  static constexpr int HX = TX + 2, HY = TY + 2, HZ = TZ + 2;  // halo box
  static constexpr int PX = HX | 1;                            // odd row stride: conflict-free pencil reads
  static constexpr int NH = PX * HY * HZ;
  static constexpr int MX = 2 * TX + 1, MY = 2 * TY + 1, MZ = 2 * TZ + 1;
  // node row: even nodes [0, TX], odd nodes [TX+1, 2TX], padded to RS = 2 (mod 8) so that
  // 4 x-consecutive elements x 4 rows (a half-warp in step 2) hit 16 distinct bank pairs
  static constexpr int RS = MX + ((10 - MX % 8) % 8);
  static constexpr int NN = RS * MY * MZ;
  // pencil classes (ry, rz) in order (0,0), (1,0), (0,1), (1,1); each starts on a warp boundary
  static constexpr int cls_n(int ry, int rz) { return (ry ? TY : TY + 1) * (rz ? TZ : TZ + 1); }
  static constexpr int up32(int n) { return (n + 31) / 32 * 32; }
  static constexpr int OFF1 = up32(cls_n(0, 0)), OFF2 = OFF1 + up32(cls_n(1, 0)), OFF3 = OFF2 + up32(cls_n(0, 1));
  static constexpr int NP_TH = OFF3 + up32(cls_n(1, 1));
  static constexpr int NTH = NP_TH > up32(NE) ? NP_TH : up32(NE);
  static constexpr int NNX = MX * MY * MZ;  // Xs: same split rows, unpadded (stride MX)
  static constexpr size_t SMEM = sizeof(double) * (4 * NH + 3 * NN + NNX);  // Ps, T[3], Xs: 2 CTAs/SM at 4x8x8
  __host__ __device__ static constexpr int col(int nx) { return (nx & 1) ? TX + 1 + (nx >> 1) : (nx >> 1); }
};

// One x-pencil of class (RY, RZ): node row (ny, nz) = (2jy + RY, 2jz + RZ).
template <int TX, int TY, int TZ, int RY, int RZ>
__device__ __forceinline__ void fk2_pencil(const double* __restrict__ Ps, double* __restrict__ T,
                                           const double* __restrict__ Xs, int jy, int jz, double sB) {
  using F = FK2<TX, TY, TZ>;
  const int ny = 2 * jy + RY, nz = 2 * jz + RZ;
  double acc[3][F::MX];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int nx = 0; nx < F::MX; ++nx) acc[c][nx] = 0.0;
  // element combos in (z, y): even row -> elements j (local 2) and j+1 (local 0)
  // in halo coordinates; odd row -> element j+1 (local 1)
#pragma unroll
  for (int iz = 0; iz < (RZ ? 1 : 2); ++iz) {
    const int qz = RZ ? jz + 1 : jz + iz;
    const int az = RZ ? 1 : (iz == 0 ? 2 : 0);
#pragma unroll
    for (int iy = 0; iy < (RY ? 1 : 2); ++iy) {
      const int qy = RY ? jy + 1 : jy + iy;
      const int ay = RY ? 1 : (iy == 0 ? 2 : 0);
      const double* Pr = Ps + F::PX * (qy + F::HY * qz);
#pragma unroll
      for (int qx = 0; qx < F::HX; ++qx) {
        double pm[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) pm[m] = Pr[m * F::NH + qx];
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
          const int nx = 2 * qx - 2 + ax;
          if (nx < 0 || nx >= F::MX) continue;
          const int a = ax + 3 * (ay + 3 * az);
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            if (bt2_nz(0, a, m)) acc[0][nx] = fma(c_Bt2[0][a][m], pm[m], acc[0][nx]);
            if (bt2_nz(1, a, m)) acc[1][nx] = fma(c_Bt2[1][a][m], pm[m], acc[1][nx]);
            if (bt2_nz(2, a, m)) acc[2][nx] = fma(c_Bt2[2][a][m], pm[m], acc[2][nx]);
          }
        }
      }
    }
  }
  double* Tr = T + F::RS * (ny + F::MY * nz);
  const double* Xr = Xs + F::MX * (ny + F::MY * nz);
#pragma unroll
  for (int nx = 0; nx < F::MX; ++nx) {
    const double f = sB * Xr[F::col(nx)];  // X = 0 on the boundary, outside the domain 0 as well
#pragma unroll
    for (int c = 0; c < 3; ++c) Tr[c * F::NN + F::col(nx)] = f * acc[c][nx];
  }
}

// mode: 0 -> p = Minv r; 1 -> p = Minv r + beta p_old; 2 -> p = p_old.
// ctl: PCG control for iteration it (pcg_control: rz_it from the previous
// kernel's partials rzp, stop, beta); otherwise no stop test, beta unused.
// The <p, q> block partials go to pqp (summed by k_pcg_upd).
template <int TX, int TY, int TZ, int MINB>
__global__ void __launch_bounds__(FK2<TX, TY, TZ>::NTH, MINB)
    k_K2_fused(const double* __restrict__ pold, double* __restrict__ pnew, const double* __restrict__ r,
               const double* __restrict__ Minv, const double* __restrict__ X, double* __restrict__ q, Geo G,
               double sB, int mode, int it, int ctl, const double* __restrict__ rzp, int nrz, double* rz_hist,
               const double* pq_hist, int* stop, double* pqp) {
  using F = FK2<TX, TY, TZ>;
  extern __shared__ __align__(16) double sm[];
  double* Ps = sm;               // [4][NH]
  double* T = sm + 4 * F::NH;    // [3][MZ][MY][RS]
  double* Xs = T + 3 * F::NN;    // [MZ][MY][RS]
  const int N = G.N;
  const int64_t ne = G.n_el;
  const int NTX = (N + TX - 1) / TX, NTY = (N + TY - 1) / TY, NTZ = (N + TZ - 1) / TZ;
  const int n_tiles = NTX * NTY * NTZ;
  double beta = 0.0;
  if (ctl && !(mode & 0x8000)) {
    if (pcg_control<F::NTH>(it, rzp, nrz, rz_hist, pq_hist, stop, &beta) && !(mode & 0x2000)) return;
  } else if ((mode & 0xff) == 1) {
    beta = rz_hist[it] / rz_hist[it - 1];
  }
  // timing probe (option "k_dbg", results invalid): bits 8/9/10 skip step 1 / step 2 / halo loads
  const int dbg = mode & ~0xff;
  mode &= 0xff;
  double dot = 0.0;
  // persistent CTA: tiles blockIdx.x, blockIdx.x + gridDim.x, ...
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
  const int tx = tile % NTX, ty = (tile / NTX) % NTY, tz = tile / (NTX * NTY);
  const int ex0 = TX * tx, ey0 = TY * ty, ez0 = TZ * tz;
  const int bx = 2 * ex0, by = 2 * ey0, bz = 2 * ez0;
  // 0a. X at the tile nodes -> Xs, asynchronously (no registers held)
  for (int i = threadIdx.x; i < F::MX * F::MY * F::MZ; i += F::NTH) {
    const int nx = i % F::MX, ny = (i / F::MX) % F::MY, nz = i / (F::MX * F::MY);
    const int gx = bx + nx, gy = by + ny, gz = bz + nz;
    double* dst = Xs + F::MX * (ny + F::MY * nz) + F::col(nx);
    if (gx < G.nn1 && gy < G.nn1 && gz < G.nn1 && !(dbg & 0x4000)) cp_async8(dst, X + node_id(gx, gy, gz, G.nn1));
    else *dst = 0.0;
  }
  // 0b. p on the tile + halo: all loads of the thread's share issued before use
  constexpr int HPER = (F::NH + F::NTH - 1) / F::NTH;
  double po[HPER][4], rr[HPER][4], mi[HPER][4];
  int64_t he[HPER];
#pragma unroll
  for (int k = 0; k < HPER; ++k) {
    const int i = threadIdx.x + k * F::NTH;
    const int hx = i % F::PX, hy = (i / F::PX) % F::HY, hz = i / (F::PX * F::HY);
    const int ex = ex0 + hx - 1, ey = ey0 + hy - 1, ez = ez0 + hz - 1;
    const bool ok = !(dbg & 0x400) && i < F::NH && hx < F::HX && ex >= 0 && ey >= 0 && ez >= 0 && ex < N &&
                    ey < N && ez < N;
    he[k] = ok ? ex + (int64_t)N * (ey + (int64_t)N * ez) : -1;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      po[k][m] = (ok && mode != 0) ? __ldg(pold + m * ne + he[k]) : 0.0;
      rr[k][m] = (ok && mode != 2) ? __ldg(r + m * ne + he[k]) : 0.0;
      mi[k][m] = (ok && mode != 2) ? __ldg(Minv + m * ne + he[k]) : 0.0;
    }
  }
#pragma unroll
  for (int k = 0; k < HPER; ++k) {
    const int i = threadIdx.x + k * F::NTH;
    if (i >= F::NH) continue;
    const int hx = i % F::PX, hy = (i / F::PX) % F::HY, hz = i / (F::PX * F::HY);
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
        if (own && !(dbg & 0x1000)) pnew[m * ne + he[k]] = v;
      }
      Ps[m * F::NH + i] = v;
    }
  }
  cp_async_wait_all();  // this thread's Xs copies; the barrier publishes everyone's
  __syncthreads();
  // 1. t at the tile nodes by x-pencils, one class per warp group
  if (!(dbg & 0x100)) {
    const int t = threadIdx.x;
    if (t < F::OFF1) {
      if (t < F::cls_n(0, 0)) fk2_pencil<TX, TY, TZ, 0, 0>(Ps, T, Xs, t % (TY + 1), t / (TY + 1), sB);
    } else if (t < F::OFF2) {
      const int i = t - F::OFF1;
      if (i < F::cls_n(1, 0)) fk2_pencil<TX, TY, TZ, 1, 0>(Ps, T, Xs, i % TY, i / TY, sB);
    } else if (t < F::OFF3) {
      const int i = t - F::OFF2;
      if (i < F::cls_n(0, 1)) fk2_pencil<TX, TY, TZ, 0, 1>(Ps, T, Xs, i % (TY + 1), i / (TY + 1), sB);
    } else {
      const int i = t - F::OFF3;
      if (i < F::cls_n(1, 1)) fk2_pencil<TX, TY, TZ, 1, 1>(Ps, T, Xs, i % TY, i / TY, sB);
    }
  }
  __syncthreads();
  // 2. q = sB Bt^T t per element
  if (threadIdx.x < F::NE && !(dbg & 0x200)) {
    const int lx = threadIdx.x % TX, ly = (threadIdx.x / TX) % TY, lz = threadIdx.x / (TX * TY);
    const int ex = ex0 + lx, ey = ey0 + ly, ez = ez0 + lz;
    if (ex < N && ey < N && ez < N) {
      double qm[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int a = 0; a < 27; ++a) {
          const int ax = a % 3, ay = (a / 3) % 3, az = a / 9;
          // col(2lx + ax): ax = 0 -> lx, 1 -> TX+1+lx, 2 -> lx+1
          const int cx = ax == 1 ? TX + 1 + lx : lx + (ax >> 1);
          const double tv = T[c * F::NN + F::RS * ((2 * ly + ay) + F::MY * (2 * lz + az)) + cx];
#pragma unroll
          for (int m = 0; m < 4; ++m)
            if (bt2_nz(c, a, m)) qm[m] = fma(c_Bt2[c][a][m], tv, qm[m]);
        }
      const int64_t e = ex + (int64_t)N * (ey + (int64_t)N * ez);
      const int h = (lx + 1) + F::PX * ((ly + 1) + F::HY * (lz + 1));
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const double o = sB * qm[m];
        if (!(dbg & 0x800)) q[m * ne + e] = o;
        dot = fma(Ps[m * F::NH + h], o, dot);
      }
    }
  }
  __syncthreads();  // Ps, T, Xs are rewritten by the next tile
  }  // tiles
  store_partial<F::NTH>(dot, pqp);
}

}  // namespace wb
