// k4_fused.cuh -- fused high-order Poisson operator q = K_w p = B X B^T p (rows a8, a9 for
// k = 3, 4; C4 is Q4 x P3disc), with the PCG direction update folded in, in one kernel.
//
// K_w = B X^-1 B^T on P_{k-1}^disc (eq:wbfbt PAPER.md:439-445), X = C_w^-1
// or D_w^-1 per node (0 on the Dirichlet boundary: the mask).  The element divergence matrix is
// a product of 1-D integrals:
//   B_e[(m1,m2,m3),(c,a)] = sB prod_d M_cd[m_d][a_d],  M_cd = BD if d == c else BI,
// so on the structured mesh B^T is, per component c, a tensor product of three ASSEMBLED 1-D
// operators (element modes -> nodes, the shared element-end node receiving from both sides):
//   (B^T p)_c = sB sum_m (T^c_x,m1 (x) T^c_y,m2 (x) T^c_z,m3) p_m.
// A CTA takes a TX x TY x TZ element tile.  It loads p (after the update p = z + beta p_old,
// z = Minv r stored by the PCG update kernel) on the tile plus one halo element layer, and
// contracts one axis at a time into the tile's (kT+1)^3 nodes, so the tile-face nodes get
// their neighbours' contributions without any exchange:
//   Z : Wz[pair(m1,m2)][ly][lx][nz] = sum_{lz, m3} T_z  p        (halo columns included)
//   Y : Wy[m1][lx][ny][nz]          = sum_{ly, m2} T_y  Wz
//   X : y_c(nx,ny,nz) = sB X(n) sum_{lx, m1} T_x Wy              (the node line in registers)
// then B restricted to the tile's own elements, the same 1-D factors transposed:
//   X': V[m1][lx'][ny][nz] = sum_nx T_x y_c   (same thread, no shared-memory round trip)
//   Y': U[pair][ly'][lx'][nz] = sum_ny T_y V
//   Z': q[e][m] += sum_nz T_z U          (accumulated over c in registers; q = sB acc)
// Each 1-D contraction walks its line element by element with a two-element sliding window
// (the shared end node takes the lower element's node K and the upper one's node 0), so the
// loops stay rolled: the kernel is compact (instruction-cache resident).  Stages with a
// triangular mode index give every warp ONE group (m1 + m2 for Z / Z', m1 for Y / Y'), padded
// to whole warps, so their mode loops are compile-time.  The component loop is a runtime loop;
// each stage loads its 1-D table (BI or BD by axis and component) into registers.
// Every node value is a sum over its elements in a fixed order: bitwise reproducible.
// mode (as k_K2_fused): 0 -> p = z; 1 -> p = z + beta p_old; 2 -> p = p_old.
// ctl: PCG control of iteration it (pcg_control); <p, q> block partials -> pqp (one per CTA).
#pragma once
#include "kernels.cuh"
#include "mbar.cuh"

namespace wb {

template <int K, int TX, int TY, int TZ, bool TMA = false, bool XG = false>
struct FK4 {
  static constexpr int NM = K * (K + 1) * (K + 2) / 6, NP = K * (K + 1) / 2;
  static constexpr int EX = TX + 2, EY = TY + 2, EZ = TZ + 2;             // extended (halo) elements
  static constexpr int NX = K * TX + 1, NY = K * TY + 1, NZ = K * TZ + 1;  // tile nodes per axis
  static constexpr int NEH = EX * EY * EZ;
  static constexpr int PE = NM * NEH;           // Pe[m][lz][ly][lx]
  // X at the tile nodes, rows of XR (TMA: even, the box's 16-byte inner extent)
  // (XG: no X in shared memory; stage X reads its node line from the padded global copy)
  static constexpr int XR = TMA ? (NX + 1) / 2 * 2 : NX;
  static constexpr int XS = XG ? 0 : XR * NY * NZ;  // Xs[nz][ny][XR]
  static constexpr int WZ = NP * EY * EX * NZ;  // Wz[p][ly][lx][nz]
  static constexpr int WY = K * EX * NY * NZ;   // Wy[m1][lx][ny][nz]
  static constexpr int VV = K * TX * NY * NZ;   // V[m1][lx'][ny][nz]   (in the Wz space)
  static constexpr int UU = NP * TY * TX * NZ;  // U[p][ly'][lx'][nz]   (in the Wy space)
  static_assert(VV <= WZ && UU <= WY, "V / U must fit the Wz / Wy spaces");
  // TMA staging of the z and p_old halo boxes (in the Wz / Wy spaces): x from ex0 - 2 (the
  // start must be 16-byte aligned: TX even), 8 wide, [m][lz][ly][8]
  static constexpr int BX = 8, BOX = BX * EY * EZ * NM;
  static_assert(!TMA || (TX % 2 == 0 && EX + 1 <= BX), "TMA boxes need an even TX <= 6");
  static constexpr int al16(int n) { return (n + 15) / 16 * 16; }  // 128-byte multiples of doubles
  static constexpr int mxx(int a, int b) { return a > b ? a : b; }
  static constexpr int SZ = al16(TMA ? mxx(WZ, BOX) : WZ), SY = al16(TMA ? mxx(WY, BOX) : WY);
  static constexpr int OFF_XS = al16(PE), OFF_WZ = OFF_XS + al16(XS), OFF_WY = OFF_WZ + SZ, OFF_T = OFF_WY + SY;
  static constexpr int TABS = 2 * K * (K + 1);  // BI, BD copies
  static constexpr int OFF_B = OFF_T + al16(TABS);
  static constexpr int SMEM = OFF_B * 8 + 16;   // + the mbarrier
  static constexpr unsigned BOXB = BOX * 8u, XB = XS * 8u;
  static constexpr int w32(int n) { return (n + 31) / 32 * 32; }
  static constexpr int GWZ = w32(EX * EY), GWY = w32(EX * NZ), GWY2 = w32(TX * NZ), GWZ2 = w32(TX * TY);
  static constexpr int IX = NY * NZ;
  static constexpr int mx(int a, int b) { return a > b ? a : b; }
  static constexpr int NTH = mx(mx(K * GWZ, K * GWY), mx(mx(w32(IX), K * GWY2), K * GWZ2));
};

// X = C_w^-1 or D_w^-1 with rows padded to nn1 + 1 (an even, 16-byte row stride for the
// TMA tensor map of the k = 4 kernel); the pad column is 0
__global__ void k_xpad4(const double* __restrict__ XL, const double* __restrict__ XR, double* __restrict__ PL,
                        double* __restrict__ PR, int nn1) {
  const int64_t rp = nn1 + 1, n = rp * nn1 * nn1;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int gx = (int)(i % rp);
    const int64_t row = i / rp;
    const bool in = gx < nn1;
    PL[i] = in ? XL[row * nn1 + gx] : 0.0;
    PR[i] = in ? XR[row * nn1 + gx] : 0.0;
  }
}

// pair index of (m1, m2), m1 + m2 <= K-1: for m1: for m2 (m1 outer)
template <int K>
__host__ __device__ constexpr int k4_pair(int m1, int m2) { return m1 * K - m1 * (m1 - 1) / 2 + m2; }
// mode index of (m1, m2, m3) in the R2 order: for d: for m3 <= d: for m2 <= d - m3: m1 = d - m2 - m3
__host__ __device__ constexpr int k4_mode(int m1, int m2, int m3) {
  return (m1 + m2 + m3) * (m1 + m2 + m3 + 1) * (m1 + m2 + m3 + 2) / 6 + m3 * (m1 + m2 + m3 + 1) -
         m3 * (m3 - 1) / 2 + m2;
}
// rows m < NR of a 1-D table ([K][K+1] in shared memory) into registers.  (Measured: the
// table as compile-time constant-bank operands, one code copy per BI / BD, is slower: 33.9
// vs 30.3 us per C4 PCG iteration -- the doubled code misses the instruction cache.)
template <int K, int NR>
__device__ __forceinline__ void k4_tab(const double* __restrict__ T, double (&M)[NR][K + 1]) {
#pragma unroll
  for (int m = 0; m < NR; ++m)
#pragma unroll
    for (int a = 0; a <= K; ++a) M[m][a] = T[m * (K + 1) + a];
}

// stage Z: thread (column lx + EX ly, degree group G = m1 + m2): pairs (G - j, j), m3 < K - G
template <int K, int TX, int TY, int TZ, int G>
__device__ __forceinline__ void k4_z_grp(const double* __restrict__ Pe, double* __restrict__ Wz, int col,
                                         const double* __restrict__ Tz) {
  using F = FK4<K, TX, TY, TZ>;
  constexpr int NM3 = K - G;
  double M[NM3][K + 1];
  k4_tab<K, NM3>(Tz, M);
#pragma unroll
  for (int j = 0; j <= G; ++j) {
    const int m1 = G - j, m2 = j;
    double P[F::EZ][NM3];
#pragma unroll
    for (int lz = 0; lz < F::EZ; ++lz)
#pragma unroll
      for (int m3 = 0; m3 < NM3; ++m3) P[lz][m3] = Pe[col + k4_mode(m1, m2, m3) * F::NEH + lz * F::EX * F::EY];
    double* out = Wz + k4_pair<K>(m1, m2) * (F::EY * F::EX * F::NZ) + col * F::NZ;
#pragma unroll
    for (int n = 0; n < F::NZ; ++n) {
      const int l = n / K + 1, a = n % K;
      double s = 0.0;
#pragma unroll
      for (int m3 = 0; m3 < NM3; ++m3) s = fma(M[m3][a], P[l][m3], s);
      if (a == 0) {
#pragma unroll
        for (int m3 = 0; m3 < NM3; ++m3) s = fma(M[m3][K], P[l - 1][m3], s);
      }
      out[n] = s;
    }
  }
}
template <int K, int TX, int TY, int TZ>
__device__ __forceinline__ void k4_stage_z(const double* __restrict__ Pe, double* __restrict__ Wz, int t,
                                           const double* Tz) {
  using F = FK4<K, TX, TY, TZ>;
  const int g = t / F::GWZ, col = t % F::GWZ;
  if (g >= K || col >= F::EX * F::EY) return;
  switch (g) {
    case 0: k4_z_grp<K, TX, TY, TZ, 0>(Pe, Wz, col, Tz); break;
    case 1: k4_z_grp<K, TX, TY, TZ, 1>(Pe, Wz, col, Tz); break;
    case 2: if constexpr (K > 2) k4_z_grp<K, TX, TY, TZ, (K > 2 ? 2 : 0)>(Pe, Wz, col, Tz); break;
    default: if constexpr (K > 3) k4_z_grp<K, TX, TY, TZ, (K > 3 ? 3 : 0)>(Pe, Wz, col, Tz); break;
  }
}

// stage Y: thread (nz, lx) of group m1 = M1 contracts (ly, m2 < K - M1)
template <int K, int TX, int TY, int TZ, int M1>
__device__ __forceinline__ void k4_y_grp(const double* __restrict__ Wz, double* __restrict__ Wy, int it,
                                         const double* __restrict__ Ty) {
  using F = FK4<K, TX, TY, TZ>;
  constexpr int NM2 = K - M1;
  double M[NM2][K + 1];
  k4_tab<K, NM2>(Ty, M);
  const int nz = it % F::NZ, lx = it / F::NZ;
  const double* ib = Wz + lx * F::NZ + nz;
  double R[F::EY][NM2];
#pragma unroll
  for (int ly = 0; ly < F::EY; ++ly)
#pragma unroll
    for (int m2 = 0; m2 < NM2; ++m2) R[ly][m2] = ib[(k4_pair<K>(M1, m2) * F::EY + ly) * F::EX * F::NZ];
  double* out = Wy + ((M1 * F::EX + lx) * F::NY) * F::NZ + nz;
#pragma unroll
  for (int n = 0; n < F::NY; ++n) {
    const int l = n / K + 1, a = n % K;
    double s = 0.0;
#pragma unroll
    for (int m2 = 0; m2 < NM2; ++m2) s = fma(M[m2][a], R[l][m2], s);
    if (a == 0) {
#pragma unroll
      for (int m2 = 0; m2 < NM2; ++m2) s = fma(M[m2][K], R[l - 1][m2], s);
    }
    out[n * F::NZ] = s;
  }
}
template <int K, int TX, int TY, int TZ>
__device__ __forceinline__ void k4_stage_y(const double* __restrict__ Wz, double* __restrict__ Wy, int t,
                                           const double* Ty) {
  using F = FK4<K, TX, TY, TZ>;
  const int g = t / F::GWY, it = t % F::GWY;
  if (g >= K || it >= F::EX * F::NZ) return;
  switch (g) {
    case 0: k4_y_grp<K, TX, TY, TZ, 0>(Wz, Wy, it, Ty); break;
    case 1: k4_y_grp<K, TX, TY, TZ, 1>(Wz, Wy, it, Ty); break;
    case 2: if constexpr (K > 2) k4_y_grp<K, TX, TY, TZ, (K > 2 ? 2 : 0)>(Wz, Wy, it, Ty); break;
    default: if constexpr (K > 3) k4_y_grp<K, TX, TY, TZ, (K > 3 ? 3 : 0)>(Wz, Wy, it, Ty); break;
  }
}

// stages X and X' on the node line (ny, nz): y = sB X B^T along x, then its x-contraction
// onto the own elements' modes m1
template <int K, int TX, int TY, int TZ, int XR, bool XG = false>
__device__ __forceinline__ void k4_stage_x(const double* __restrict__ Wy, const double* __restrict__ Xs,
                                           double* __restrict__ V, int item, double sB,
                                           const double* __restrict__ Tx, const double* __restrict__ xg = nullptr,
                                           int xlim = 0) {
  using F = FK4<K, TX, TY, TZ>;
  if (item >= F::IX) return;
  double M[K][K + 1];
  k4_tab<K, K>(Tx, M);
  const int nz = item % F::NZ, ny = item / F::NZ;
  const double* ib = Wy + ny * F::NZ + nz;
  double R[F::EX][K];
#pragma unroll
  for (int lx = 0; lx < F::EX; ++lx)
#pragma unroll
    for (int m1 = 0; m1 < K; ++m1) R[lx][m1] = ib[(m1 * F::EX + lx) * F::NY * F::NZ];
  double acc[TX][K];
#pragma unroll
  for (int l = 0; l < TX; ++l)
#pragma unroll
    for (int m1 = 0; m1 < K; ++m1) acc[l][m1] = 0.0;
  const double* xr = Xs + (nz * F::NY + ny) * XR;
  double xv[XG ? F::NX : 1];
  if constexpr (XG) {  // the line's X (global, 0 past the mesh), all loads in flight first
#pragma unroll
    for (int n = 0; n < F::NX; ++n) xv[n] = n < xlim ? __ldg(xg + n) : 0.0;
  }
#pragma unroll
  for (int n = 0; n < F::NX; ++n) {
    const int l = n / K + 1, a = n % K;
    double s = 0.0;
#pragma unroll
    for (int m1 = 0; m1 < K; ++m1) s = fma(M[m1][a], R[l][m1], s);
    if (a == 0) {
#pragma unroll
      for (int m1 = 0; m1 < K; ++m1) s = fma(M[m1][K], R[l - 1][m1], s);
    }
    const double y = sB * (XG ? xv[XG ? n : 0] : xr[n]) * s;  // X = 0 on the boundary and outside the mesh
    if (l - 1 < TX) {
#pragma unroll
      for (int m1 = 0; m1 < K; ++m1) acc[l - 1][m1] = fma(M[m1][a], y, acc[l - 1][m1]);
    }
    if (a == 0 && l >= 2) {
#pragma unroll
      for (int m1 = 0; m1 < K; ++m1) acc[l - 2][m1] = fma(M[m1][K], y, acc[l - 2][m1]);
    }
  }
  double* ob = V + ny * F::NZ + nz;
#pragma unroll
  for (int l = 0; l < TX; ++l)
#pragma unroll
    for (int m1 = 0; m1 < K; ++m1) ob[(m1 * TX + l) * F::NY * F::NZ] = acc[l][m1];
}

// stage Y': thread (nz, lx') of group m1 = M1: V line along y -> U rows (M1, m2)
template <int K, int TX, int TY, int TZ, int M1>
__device__ __forceinline__ void k4_y2_grp(const double* __restrict__ V, double* __restrict__ U, int it,
                                          const double* __restrict__ Ty) {
  using F = FK4<K, TX, TY, TZ>;
  constexpr int NM2 = K - M1;
  double M[NM2][K + 1];
  k4_tab<K, NM2>(Ty, M);
  const int nz = it % F::NZ, lx = it / F::NZ;
  double acc[TY][NM2];
#pragma unroll
  for (int l = 0; l < TY; ++l)
#pragma unroll
    for (int m2 = 0; m2 < NM2; ++m2) acc[l][m2] = 0.0;
  const double* in = V + ((M1 * TX + lx) * F::NY) * F::NZ + nz;
#pragma unroll
  for (int n = 0; n < F::NY; ++n) {
    const int l = n / K + 1, a = n % K;
    const double y = in[n * F::NZ];
    if (l - 1 < TY) {
#pragma unroll
      for (int m2 = 0; m2 < NM2; ++m2) acc[l - 1][m2] = fma(M[m2][a], y, acc[l - 1][m2]);
    }
    if (a == 0 && l >= 2) {
#pragma unroll
      for (int m2 = 0; m2 < NM2; ++m2) acc[l - 2][m2] = fma(M[m2][K], y, acc[l - 2][m2]);
    }
  }
  double* ob = U + lx * F::NZ + nz;
#pragma unroll
  for (int l = 0; l < TY; ++l)
#pragma unroll
    for (int m2 = 0; m2 < NM2; ++m2) ob[(k4_pair<K>(M1, m2) * TY + l) * TX * F::NZ] = acc[l][m2];
}
template <int K, int TX, int TY, int TZ>
__device__ __forceinline__ void k4_stage_y2(const double* __restrict__ V, double* __restrict__ U, int t,
                                            const double* Ty) {
  using F = FK4<K, TX, TY, TZ>;
  const int g = t / F::GWY2, it = t % F::GWY2;
  if (g >= K || it >= TX * F::NZ) return;
  switch (g) {
    case 0: k4_y2_grp<K, TX, TY, TZ, 0>(V, U, it, Ty); break;
    case 1: k4_y2_grp<K, TX, TY, TZ, 1>(V, U, it, Ty); break;
    case 2: if constexpr (K > 2) k4_y2_grp<K, TX, TY, TZ, (K > 2 ? 2 : 0)>(V, U, it, Ty); break;
    default: if constexpr (K > 3) k4_y2_grp<K, TX, TY, TZ, (K > 3 ? 3 : 0)>(V, U, it, Ty); break;
  }
}

// stage Z': thread (lx', ly') of degree group G accumulates A[j][lz'][m3] over the components
// (TZ is small: this loop is unrolled so the accumulators stay in registers)
template <int K, int TZ>
struct K4Acc {
  double v[K][TZ][K];  // [pair j in the group][lz'][m3]  (only j <= G, m3 < K - G used)
};
template <int K, int TX, int TY, int TZ, int G>
__device__ __forceinline__ void k4_z2_grp(const double* __restrict__ U, K4Acc<K, TZ>& A, int col,
                                          const double* __restrict__ Tz) {
  using F = FK4<K, TX, TY, TZ>;
  constexpr int NM3 = K - G;
  double M[NM3][K + 1];
  k4_tab<K, NM3>(Tz, M);
#pragma unroll
  for (int j = 0; j <= G; ++j) {
    const double* in = U + (k4_pair<K>(G - j, j) * TY * TX + col) * F::NZ;
#pragma unroll
    for (int n = 0; n < F::NZ; ++n) {
      const int l = n / K + 1, a = n % K;
      const double y = in[n];
      if (l - 1 < TZ) {
#pragma unroll
        for (int m3 = 0; m3 < NM3; ++m3) A.v[j][l - 1][m3] = fma(M[m3][a], y, A.v[j][l - 1][m3]);
      }
      if (a == 0 && l >= 2) {
#pragma unroll
        for (int m3 = 0; m3 < NM3; ++m3) A.v[j][l - 2][m3] = fma(M[m3][K], y, A.v[j][l - 2][m3]);
      }
    }
  }
}
template <int K, int TX, int TY, int TZ>
__device__ __forceinline__ void k4_stage_z2(const double* __restrict__ U, K4Acc<K, TZ>& A, int t, const double* Tz) {
  using F = FK4<K, TX, TY, TZ>;
  const int g = t / F::GWZ2, col = t % F::GWZ2;
  if (g >= K || col >= TX * TY) return;
  switch (g) {
    case 0: k4_z2_grp<K, TX, TY, TZ, 0>(U, A, col, Tz); break;
    case 1: k4_z2_grp<K, TX, TY, TZ, 1>(U, A, col, Tz); break;
    case 2: if constexpr (K > 2) k4_z2_grp<K, TX, TY, TZ, (K > 2 ? 2 : 0)>(U, A, col, Tz); break;
    default: if constexpr (K > 3) k4_z2_grp<K, TX, TY, TZ, (K > 3 ? 3 : 0)>(U, A, col, Tz); break;
  }
}

// q = sB acc for the group's modes of own element column (lx', ly'), <p, q> partial
template <int K, int TX, int TY, int TZ, int G, bool OWN = false>
__device__ __forceinline__ double k4_q_grp(const K4Acc<K, TZ>& A, const double* __restrict__ Pe, double* q, int col,
                                           int ex0, int ey0, int ez0, int N, int64_t ne, double sB) {
  using F = FK4<K, TX, TY, TZ>;
  constexpr int NM3 = K - G;
  const int lx = col % TX, ly = col / TX;
  const int ex = ex0 + lx, ey = ey0 + ly;
  double dot = 0.0;
  if (ex >= N || ey >= N) return 0.0;
#pragma unroll
  for (int lz = 0; lz < TZ; ++lz) {
    const int ez = ez0 + lz;
    if (ez < N) {
      const int64_t e = ex + (int64_t)N * (ey + (int64_t)N * ez);
      // own p: Pe (the halo layout) or, OWN, a [m][lz][ly][lx] copy of the own elements
      const double* pe = OWN ? Pe + (lz * TY + ly) * TX + lx : Pe + ((lz + 1) * F::EY + ly + 1) * F::EX + lx + 1;
#pragma unroll
      for (int j = 0; j <= G; ++j)
#pragma unroll
        for (int m3 = 0; m3 < NM3; ++m3) {
          const int m = k4_mode(G - j, j, m3);
          const double o = sB * A.v[j][lz][m3];
          q[(int64_t)m * ne + e] = o;
          dot = fma(pe[m * (OWN ? TX * TY * TZ : F::NEH)], o, dot);
        }
    }
  }
  return dot;
}

template <int K, int TX, int TY, int TZ, int MINB, bool TMA, bool XG = false>
__global__ void __launch_bounds__(FK4<K, TX, TY, TZ, TMA, XG>::NTH, MINB)
    k_K4_fused(const double* __restrict__ pold, double* __restrict__ pnew, const double* __restrict__ z,
               const double* __restrict__ X, double* __restrict__ q, Geo G, double sB, int mode, int it, int ctl,
               const double* __restrict__ rzp, int nrz, double* rz_hist, const double* pq_hist, int* stop,
               double* pqp, const __grid_constant__ CUtensorMap tm_p, const __grid_constant__ CUtensorMap tm_z,
               const __grid_constant__ CUtensorMap tm_x) {
  using F = FK4<K, TX, TY, TZ, TMA, XG>;
  extern __shared__ __align__(1024) double sm[];
  double* Pe = sm;
  double* Xs = sm + F::OFF_XS;
  double* Wz = sm + F::OFF_WZ;
  double* Wy = sm + F::OFF_WY;
  double* Tb = sm + F::OFF_T;  // [0] BI, [1] BD, each [K][K+1]
  uint64_t* bar = (uint64_t*)(sm + F::OFF_B);
  const int N = G.N;
  const int64_t ne = G.n_el;
  const int t = threadIdx.x;
  const int NTX = (N + TX - 1) / TX, NTY = (N + TY - 1) / TY;
  const int tile = blockIdx.x;
  const int tx = tile % NTX, ty = (tile / NTX) % NTY, tz = tile / (NTX * NTY);
  const int ex0 = TX * tx, ey0 = TY * ty, ez0 = TZ * tz;
  if constexpr (TMA) {
    // one thread issues the tile's boxes (zero fill outside the mesh); they land while the
    // PCG control reduction below runs
    if (t == 0) {
      mbar_init(&bar[0], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      mbar_expect_tx(&bar[0], F::XB + (mode != 2 ? F::BOXB : 0u) + (mode != 0 ? F::BOXB : 0u));
      if (!XG) tma_load_3d(Xs, &tm_x, K * ex0, K * ey0, K * ez0, &bar[0]);
      if (mode != 2) tma_load_4d(Wz, &tm_z, ex0 - 2, ey0 - 1, ez0 - 1, 0, &bar[0]);
      if (mode != 0) tma_load_4d(Wy, &tm_p, ex0 - 2, ey0 - 1, ez0 - 1, 0, &bar[0]);
    }
  } else if constexpr (!XG) {
    // X at the tile nodes (asynchronous copies; 0 outside the mesh)
    for (int i = t; i < F::XS; i += F::NTH) {
      const int nx = i % F::NX, ny = (i / F::NX) % F::NY, nz = i / (F::NX * F::NY);
      const int gx = K * ex0 + nx, gy = K * ey0 + ny, gz = K * ez0 + nz;
      if (gx < G.nn1 && gy < G.nn1 && gz < G.nn1) cp_async8(Xs + i, X + node_id(gx, gy, gz, G.nn1));
      else Xs[i] = 0.0;
    }
  }
  for (int i = t; i < F::TABS; i += F::NTH) {
    const int w = i / (K * (K + 1)), m = (i / (K + 1)) % K, a = i % (K + 1);
    Tb[i] = w ? TB(K).BD[m][a] : TB(K).BI[m][a];
  }
  // p on the tile + halo (0 outside the mesh): the thread's loads are issued before the
  // PCG control reduction, which only the update needs
  constexpr int HPER = TMA ? 1 : (F::PE + F::NTH - 1) / F::NTH;
  double po[HPER], zz[HPER];
  int64_t gi[HPER];
  if constexpr (!TMA) {
#pragma unroll
    for (int k = 0; k < HPER; ++k) {
      const int i = t + k * F::NTH;
      const int lx = i % F::EX, ly = (i / F::EX) % F::EY, lz = (i / (F::EX * F::EY)) % F::EZ, m = i / F::NEH;
      const int ex = ex0 + lx - 1, ey = ey0 + ly - 1, ez = ez0 + lz - 1;
      const bool ok =
          i < F::PE && (unsigned)ex < (unsigned)N && (unsigned)ey < (unsigned)N && (unsigned)ez < (unsigned)N;
      gi[k] = ok ? (int64_t)m * ne + ex + (int64_t)N * (ey + (int64_t)N * ez) : -1;
      po[k] = (ok && mode != 0) ? __ldg(pold + gi[k]) : 0.0;
      zz[k] = (ok && mode != 2) ? __ldg(z + gi[k]) : 0.0;
    }
  }
  double beta = 0.0;
  if (ctl) {
    if (pcg_control<F::NTH>(it, rzp, nrz, rz_hist, pq_hist, stop, &beta)) {
      if (TMA && t == 0) mbar_wait(&bar[0], 0);  // drain the copies in flight before exiting
      return;
    }
  } else if (mode == 1) {
    beta = rz_hist[it] / rz_hist[it - 1];
  }
  if constexpr (TMA) {
    __syncthreads();  // barrier init visible
    mbar_wait(&bar[0], 0);
    // p = z + beta p_old from the boxes ([m][lz][ly][8], column lx + 1)
    for (int i = t; i < F::PE; i += F::NTH) {
      const int row = i / F::EX, lx = i - row * F::EX, b = row * F::BX + lx + 1;
      Pe[i] = mode == 2 ? Wy[b] : (mode == 1 ? fma(beta, Wy[b], Wz[b]) : Wz[b]);
    }
    __syncthreads();
    if (mode != 2) {  // own elements' p_new
      for (int i = t; i < TX * TY * TZ * F::NM; i += F::NTH) {
        const int lx = i % TX, ly = (i / TX) % TY, lz = (i / (TX * TY)) % TZ, m = i / (TX * TY * TZ);
        const int ex = ex0 + lx, ey = ey0 + ly, ez = ez0 + lz;
        if (ex < N && ey < N && ez < N)
          pnew[(int64_t)m * ne + ex + (int64_t)N * (ey + (int64_t)N * ez)] =
              Pe[((m * F::EZ + lz + 1) * F::EY + ly + 1) * F::EX + lx + 1];
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < HPER; ++k) {
      const int i = t + k * F::NTH;
      if (i >= F::PE) continue;
      double v = 0.0;
      if (gi[k] >= 0) {
        v = mode == 2 ? po[k] : (mode == 1 ? fma(beta, po[k], zz[k]) : zz[k]);
        const int lx = i % F::EX, ly = (i / F::EX) % F::EY, lz = (i / (F::EX * F::EY)) % F::EZ;
        const bool own = lx >= 1 && ly >= 1 && lz >= 1 && lx <= TX && ly <= TY && lz <= TZ;
        if (own && mode != 2) pnew[gi[k]] = v;
      }
      Pe[i] = v;
    }
    cp_async_wait_all();
  }
  K4Acc<K, TZ> qa;
#pragma unroll
  for (int j = 0; j < K; ++j)
#pragma unroll
    for (int l = 0; l < TZ; ++l)
#pragma unroll
      for (int m = 0; m < K; ++m) qa.v[j][l][m] = 0.0;
  __syncthreads();
  // XG: the stage-X thread's node line in the padded global X (row stride nn1 + 1)
  const double* xg = nullptr;
  int xlim = 0;
  if constexpr (XG) {
    const int nz = t % F::NZ, ny = t / F::NZ, gy = K * ey0 + ny, gz = K * ez0 + nz;
    if (t < F::IX && gy < G.nn1 && gz < G.nn1) {
      xg = X + ((int64_t)gz * G.nn1 + gy) * (G.nn1 + 1) + K * ex0;
      xlim = min(F::NX, G.nn1 - K * ex0);
    }
  }
  const int TS = K * (K + 1);
#pragma unroll 1
  for (int c = 0; c < 3; ++c) {
    // M_cd = BD on the component's own axis d == c
    const double* Tx = Tb + (c == 0 ? TS : 0);
    const double* Ty = Tb + (c == 1 ? TS : 0);
    const double* Tz = Tb + (c == 2 ? TS : 0);
    k4_stage_z<K, TX, TY, TZ>(Pe, Wz, t, Tz);
    __syncthreads();
    k4_stage_y<K, TX, TY, TZ>(Wz, Wy, t, Ty);
    __syncthreads();
    k4_stage_x<K, TX, TY, TZ, F::XR, XG>(Wy, Xs, Wz /* V */, t, sB, Tx, xg, xlim);
    __syncthreads();
    k4_stage_y2<K, TX, TY, TZ>(Wz /* V */, Wy /* U */, t, Ty);
    __syncthreads();
    k4_stage_z2<K, TX, TY, TZ>(Wy /* U */, qa, t, Tz);
    __syncthreads();
  }
  // q = sB acc on the own elements, <p, q> partial
  double dot = 0.0;
  {
    const int g = t / F::GWZ2, col = t % F::GWZ2;
    if (g < K && col < TX * TY) {
      switch (g) {
        case 0: dot = k4_q_grp<K, TX, TY, TZ, 0>(qa, Pe, q, col, ex0, ey0, ez0, N, ne, sB); break;
        case 1: dot = k4_q_grp<K, TX, TY, TZ, 1>(qa, Pe, q, col, ex0, ey0, ez0, N, ne, sB); break;
        case 2:
          if constexpr (K > 2) dot = k4_q_grp<K, TX, TY, TZ, (K > 2 ? 2 : 0)>(qa, Pe, q, col, ex0, ey0, ez0, N, ne, sB);
          break;
        default:
          if constexpr (K > 3) dot = k4_q_grp<K, TX, TY, TZ, (K > 3 ? 3 : 0)>(qa, Pe, q, col, ex0, ey0, ez0, N, ne, sB);
          break;
      }
    }
  }
  store_partial<F::NTH>(dot, pqp);
}

// The same operator with all three components in flight at once (one CTA per SM, 5 barrier
// intervals per tile instead of 15): stage Z for the two z tables (BI feeds c = 0, 1; BD
// feeds c = 2), then Y, X/X', Y' per component on separate buffers, then Z' summing the
// components in order.  TMA staging only (k = 4, even TX, N even).  Shared memory:
//   Xs | A = [Pe | Wz_I | Wz_D] (later V_0..2) | B = Wy_0..2 (the p boxes first, later U_0..2) | Po | tables
template <int K, int TX, int TY, int TZ>
struct FK43 {
  using F = FK4<K, TX, TY, TZ, true>;
  static constexpr int al16(int n) { return (n + 15) / 16 * 16; }
  static constexpr int WZ = al16(F::WZ), WY = al16(F::WY), VV = al16(F::VV), UU = al16(F::UU);
  static constexpr int NOWN = TX * TY * TZ * F::NM;
  static constexpr int A_ = al16(F::PE) + 2 * WZ, B_ = 3 * WY;
  static_assert(3 * VV <= A_ && 3 * UU <= B_ && 2 * F::BOX <= B_, "3C buffers");
  static constexpr int OFF_XS = 0, OFF_A = al16(F::XS), OFF_WZ = OFF_A + al16(F::PE), OFF_B = OFF_A + A_,
                       OFF_PO = OFF_B + B_, OFF_T = OFF_PO + al16(NOWN), OFF_BAR = OFF_T + al16(F::TABS);
  static constexpr int SMEM = OFF_BAR * 8 + 16;
  static constexpr int NZT = 2 * K * F::GWZ, NYT = K * F::GWY, NXT = F::w32(F::IX), NY2T = K * F::GWY2;
  static constexpr int mx(int a, int b) { return a > b ? a : b; }
  static constexpr int NTH = mx(mx(NZT, 3 * NYT), mx(3 * NXT, 3 * NY2T));
};

template <int K, int TX, int TY, int TZ>
__global__ void __launch_bounds__(FK43<K, TX, TY, TZ>::NTH, 1)
    k_K4_3c(double* __restrict__ pnew, double* __restrict__ q, Geo G, double sB, int mode, int it, int ctl,
            const double* __restrict__ rzp, int nrz, double* rz_hist, const double* pq_hist, int* stop, double* pqp,
            const __grid_constant__ CUtensorMap tm_p, const __grid_constant__ CUtensorMap tm_z,
            const __grid_constant__ CUtensorMap tm_x) {
  using F = FK4<K, TX, TY, TZ, true>;
  using H = FK43<K, TX, TY, TZ>;
  extern __shared__ __align__(1024) double sm[];
  double* Xs = sm + H::OFF_XS;
  double* Pe = sm + H::OFF_A;
  double* Wz = sm + H::OFF_WZ;  // [v][WZ]
  double* Vb = sm + H::OFF_A;   // [c][VV]
  double* Wy = sm + H::OFF_B;   // [c][WY]
  double* Ub = sm + H::OFF_B;   // [c][UU]
  double* Po = sm + H::OFF_PO;
  double* Tb = sm + H::OFF_T;
  uint64_t* bar = (uint64_t*)(sm + H::OFF_BAR);
  const int N = G.N;
  const int64_t ne = G.n_el;
  const int t = threadIdx.x;
  const int NTX = (N + TX - 1) / TX, NTY = (N + TY - 1) / TY;
  const int tile = blockIdx.x;
  const int tx = tile % NTX, ty = (tile / NTX) % NTY, tz = tile / (NTX * NTY);
  const int ex0 = TX * tx, ey0 = TY * ty, ez0 = TZ * tz;
  double* Zbox = Wy;
  double* Pbox = Wy + F::BOX;
  if (t == 0) {
    mbar_init(&bar[0], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(&bar[0], F::XB + (mode != 2 ? F::BOXB : 0u) + (mode != 0 ? F::BOXB : 0u));
    tma_load_3d(Xs, &tm_x, K * ex0, K * ey0, K * ez0, &bar[0]);
    if (mode != 2) tma_load_4d(Zbox, &tm_z, ex0 - 2, ey0 - 1, ez0 - 1, 0, &bar[0]);
    if (mode != 0) tma_load_4d(Pbox, &tm_p, ex0 - 2, ey0 - 1, ez0 - 1, 0, &bar[0]);
  }
  for (int i = t; i < F::TABS; i += H::NTH) {
    const int w = i / (K * (K + 1)), m = (i / (K + 1)) % K, a = i % (K + 1);
    Tb[i] = w ? TB(K).BD[m][a] : TB(K).BI[m][a];
  }
  double beta = 0.0;
  if (ctl) {
    if (pcg_control<H::NTH>(it, rzp, nrz, rz_hist, pq_hist, stop, &beta)) {
      if (t == 0) mbar_wait(&bar[0], 0);
      return;
    }
  } else if (mode == 1) {
    beta = rz_hist[it] / rz_hist[it - 1];
  }
  __syncthreads();
  mbar_wait(&bar[0], 0);
  for (int i = t; i < F::PE; i += H::NTH) {
    const int row = i / F::EX, lx = i - row * F::EX, b = row * F::BX + lx + 1;
    Pe[i] = mode == 2 ? Pbox[b] : (mode == 1 ? fma(beta, Pbox[b], Zbox[b]) : Zbox[b]);
  }
  __syncthreads();
  for (int i = t; i < H::NOWN; i += H::NTH) {  // own p: a copy for <p, q>, p_new to global
    const int lx = i % TX, ly = (i / TX) % TY, lz = (i / (TX * TY)) % TZ, m = i / (TX * TY * TZ);
    const double v = Pe[((m * F::EZ + lz + 1) * F::EY + ly + 1) * F::EX + lx + 1];
    Po[i] = v;
    const int ex = ex0 + lx, ey = ey0 + ly, ez = ez0 + lz;
    if (mode != 2 && ex < N && ey < N && ez < N) pnew[(int64_t)m * ne + ex + (int64_t)N * (ey + (int64_t)N * ez)] = v;
  }
  const int TS = K * (K + 1);
  // Z: v = 0 (BI) for c = 0, 1; v = 1 (BD) for c = 2
  if (t < H::NZT) {
    const int v = t / (K * F::GWZ);
    k4_stage_z<K, TX, TY, TZ>(Pe, Wz + v * H::WZ, t - v * K * F::GWZ, Tb + v * TS);
  }
  __syncthreads();
  {  // Y per component
    const int c = t / H::NYT, it2 = t - c * H::NYT;
    if (c < 3)
      k4_stage_y<K, TX, TY, TZ>(Wz + (c == 2 ? H::WZ : 0), Wy + c * H::WY, it2, Tb + (c == 1 ? TS : 0));
  }
  __syncthreads();
  {  // X / X' per component (V over Pe and Wz: both dead now)
    const int c = t / H::NXT, it2 = t - c * H::NXT;
    if (c < 3)
      k4_stage_x<K, TX, TY, TZ, F::XR>(Wy + c * H::WY, Xs, Vb + c * H::VV, it2, sB, Tb + (c == 0 ? TS : 0));
  }
  __syncthreads();
  {  // Y' per component (U over Wy)
    const int c = t / H::NY2T, it2 = t - c * H::NY2T;
    if (c < 3) k4_stage_y2<K, TX, TY, TZ>(Vb + c * H::VV, Ub + c * H::UU, it2, Tb + (c == 1 ? TS : 0));
  }
  __syncthreads();
  // Z': the components in order into the same accumulators, then q and <p, q>
  K4Acc<K, TZ> qa;
#pragma unroll
  for (int j = 0; j < K; ++j)
#pragma unroll
    for (int l = 0; l < TZ; ++l)
#pragma unroll
      for (int m = 0; m < K; ++m) qa.v[j][l][m] = 0.0;
  double dot = 0.0;
  if (t < K * F::GWZ2) {
#pragma unroll 1
    for (int c = 0; c < 3; ++c) k4_stage_z2<K, TX, TY, TZ>(Ub + c * H::UU, qa, t, Tb + (c == 2 ? TS : 0));
    const int g = t / F::GWZ2, col = t % F::GWZ2;
    if (g < K && col < TX * TY) {
      switch (g) {
        case 0: dot = k4_q_grp<K, TX, TY, TZ, 0, true>(qa, Po, q, col, ex0, ey0, ez0, N, ne, sB); break;
        case 1: dot = k4_q_grp<K, TX, TY, TZ, 1, true>(qa, Po, q, col, ex0, ey0, ez0, N, ne, sB); break;
        case 2:
          if constexpr (K > 2) dot = k4_q_grp<K, TX, TY, TZ, (K > 2 ? 2 : 0), true>(qa, Po, q, col, ex0, ey0, ez0, N, ne, sB);
          break;
        default:
          if constexpr (K > 3) dot = k4_q_grp<K, TX, TY, TZ, (K > 3 ? 3 : 0), true>(qa, Po, q, col, ex0, ey0, ez0, N, ne, sB);
          break;
      }
    }
  }
  store_partial<H::NTH>(dot, pqp);
}

// ---------------------------------------------------------------- standalone B^T and B (k = 3, 4)
// The same tile stages outside the PCG (rows a6, a7 at high order; wBFBT's B^T and B):
//   k_BT4_tile: y = s o B^T p on the tile's own nodes (stages Z, Y, then X without X'), s =
//     xs (the wBFBT X scaling), else the Dirichlet mask (0 on the boundary, R6), or 1 (nomask);
//     a tile writes its nodes of local index < K T per axis, plus the mesh's last node plane.
//   k_B4_tile: p = sB B (s o u): X' straight from the global node lines, then Y', Z'.
// p is read / written at p[e se + m sm] (element-major ABI: se = n_m, sm = 1).
template <int K, int TX, int TY, int TZ>
struct FB4 {
  using F = FK4<K, TX, TY, TZ>;
  static constexpr int al16(int n) { return (n + 15) / 16 * 16; }
  static constexpr int OFF_WZ = al16(F::PE), OFF_WY = OFF_WZ + al16(F::WZ), OFF_T = OFF_WY + al16(F::WY);
  static constexpr int SMEM_BT = (OFF_T + al16(F::TABS)) * 8;
  static constexpr int OFF_U = al16(F::VV), OFF_TB = OFF_U + al16(F::UU);
  static constexpr int SMEM_B = (OFF_TB + al16(F::TABS)) * 8;
  static constexpr int NTH_B = F::mx(F::mx(F::w32(F::IX), K * F::GWY2), K * F::GWZ2);
};

template <int K, int NTH>
__device__ __forceinline__ void k4_load_tabs(double* Tb) {
  for (int i = threadIdx.x; i < 2 * K * (K + 1); i += NTH) {
    const int w = i / (K * (K + 1)), m = (i / (K + 1)) % K, a = i % (K + 1);
    Tb[i] = w ? TB(K).BD[m][a] : TB(K).BI[m][a];
  }
}

template <int K, int TX, int TY, int TZ>
__global__ void __launch_bounds__(FK4<K, TX, TY, TZ>::NTH)
    k_BT4_tile(const double* __restrict__ p, const double* __restrict__ xs, double* __restrict__ y, Geo G, double sB,
               int nomask, int64_t se, int64_t sm_) {
  using F = FK4<K, TX, TY, TZ>;
  using H = FB4<K, TX, TY, TZ>;
  extern __shared__ __align__(16) double smb[];
  double* Pe = smb;
  double* Wz = smb + H::OFF_WZ;
  double* Wy = smb + H::OFF_WY;
  double* Tb = smb + H::OFF_T;
  const int N = G.N, t = threadIdx.x;
  const int NTX = (N + TX - 1) / TX, NTY = (N + TY - 1) / TY;
  const int tile = blockIdx.x;
  const int ex0 = TX * (tile % NTX), ey0 = TY * ((tile / NTX) % NTY), ez0 = TZ * (tile / (NTX * NTY));
  k4_load_tabs<K, F::NTH>(Tb);
  for (int i = t; i < F::PE; i += F::NTH) {  // p on the tile + halo, 0 outside the mesh
    const int ext = i % F::NEH, m = i / F::NEH;
    const int lx = ext % F::EX, ly = (ext / F::EX) % F::EY, lz = ext / (F::EX * F::EY);
    const int ex = ex0 + lx - 1, ey = ey0 + ly - 1, ez = ez0 + lz - 1;
    const bool ok = (unsigned)ex < (unsigned)N && (unsigned)ey < (unsigned)N && (unsigned)ez < (unsigned)N;
    Pe[i] = ok ? __ldg(p + (ex + (int64_t)N * (ey + (int64_t)N * ez)) * se + m * sm_) : 0.0;
  }
  __syncthreads();
  const int TS = K * (K + 1);
  const int nz = t % F::NZ, ny = t / F::NZ;
  const int gy = K * ey0 + ny, gz = K * ez0 + nz;
  // own node line: local index < K T, or the mesh's last node plane
  const bool line = t < F::IX && gy < G.nn1 && gz < G.nn1 && (ny < K * TY || gy == G.nn1 - 1) &&
                    (nz < K * TZ || gz == G.nn1 - 1);
#pragma unroll 1
  for (int c = 0; c < 3; ++c) {
    const double* Tx = Tb + (c == 0 ? TS : 0);
    const double* Ty = Tb + (c == 1 ? TS : 0);
    const double* Tz = Tb + (c == 2 ? TS : 0);
    k4_stage_z<K, TX, TY, TZ>(Pe, Wz, t, Tz);
    __syncthreads();
    k4_stage_y<K, TX, TY, TZ>(Wz, Wy, t, Ty);
    __syncthreads();
    if (line) {  // stage X: B^T along x on the line, scaled, to the global nodes
      double M[K][K + 1];
      k4_tab<K, K>(Tx, M);
      const double* ib = Wy + ny * F::NZ + nz;
      double R[F::EX][K];
#pragma unroll
      for (int lx = 0; lx < F::EX; ++lx)
#pragma unroll
        for (int m1 = 0; m1 < K; ++m1) R[lx][m1] = ib[(m1 * F::EX + lx) * F::NY * F::NZ];
      const int64_t row = (int64_t)c * G.n_nodes + node_id(K * ex0, gy, gz, G.nn1);
      const bool ybnd = gy == 0 || gz == 0 || gy == G.nn1 - 1 || gz == G.nn1 - 1;
#pragma unroll
      for (int n = 0; n < F::NX; ++n) {
        const int l = n / K + 1, a = n % K;
        const int gx = K * ex0 + n;
        if (gx >= G.nn1 || (n == K * TX && gx != G.nn1 - 1)) continue;
        double s = 0.0;
#pragma unroll
        for (int m1 = 0; m1 < K; ++m1) s = fma(M[m1][a], R[l][m1], s);
        if (a == 0) {
#pragma unroll
          for (int m1 = 0; m1 < K; ++m1) s = fma(M[m1][K], R[l - 1][m1], s);
        }
        double o = sB * s;
        if (xs) o *= xs[row - (int64_t)c * G.n_nodes + n];
        else if (!nomask && (ybnd || gx == 0 || gx == G.nn1 - 1)) o = 0.0;
        y[row + n] = o;
      }
    }
    __syncthreads();
  }
}

template <int K, int TX, int TY, int TZ>
__global__ void __launch_bounds__(FB4<K, TX, TY, TZ>::NTH_B)
    k_B4_tile(const double* __restrict__ u, const double* __restrict__ xs, double* __restrict__ p, Geo G, double sB,
              int nomask, int64_t se, int64_t sm_) {
  using F = FK4<K, TX, TY, TZ>;
  using H = FB4<K, TX, TY, TZ>;
  extern __shared__ __align__(16) double smb[];
  double* V = smb;
  double* U = smb + H::OFF_U;
  double* Tb = smb + H::OFF_TB;
  const int N = G.N, t = threadIdx.x;
  const int NTX = (N + TX - 1) / TX, NTY = (N + TY - 1) / TY;
  const int tile = blockIdx.x;
  const int ex0 = TX * (tile % NTX), ey0 = TY * ((tile / NTX) % NTY), ez0 = TZ * (tile / (NTX * NTY));
  k4_load_tabs<K, H::NTH_B>(Tb);
  K4Acc<K, TZ> qa;
#pragma unroll
  for (int j = 0; j < K; ++j)
#pragma unroll
    for (int l = 0; l < TZ; ++l)
#pragma unroll
      for (int m = 0; m < K; ++m) qa.v[j][l][m] = 0.0;
  const int TS = K * (K + 1);
  const int nz = t % F::NZ, ny = t / F::NZ;
  const int gy = K * ey0 + ny, gz = K * ez0 + nz;
  const bool line = t < F::IX && gy < G.nn1 && gz < G.nn1;
  const int64_t row = line ? node_id(K * ex0, gy, gz, G.nn1) : 0;
  const int xlim = line ? min(F::NX, G.nn1 - K * ex0) : 0;
  const bool ybnd = gy == 0 || gz == 0 || gy == G.nn1 - 1 || gz == G.nn1 - 1;
  __syncthreads();
#pragma unroll 1
  for (int c = 0; c < 3; ++c) {
    const double* Tx = Tb + (c == 0 ? TS : 0);
    const double* Ty = Tb + (c == 1 ? TS : 0);
    const double* Tz = Tb + (c == 2 ? TS : 0);
    if (t < F::IX) {  // stage X': the node line (s o u) along x onto the own elements' m1
      double yv[F::NX];
      const double* ur = u + (int64_t)c * G.n_nodes + row;
#pragma unroll
      for (int n = 0; n < F::NX; ++n) {
        double v = n < xlim ? __ldg(ur + n) : 0.0;
        if (xs) v *= n < xlim ? __ldg(xs + row + n) : 0.0;
        else if (!nomask && (ybnd || K * ex0 + n == 0 || K * ex0 + n == G.nn1 - 1)) v = 0.0;
        yv[n] = v;
      }
      double M[K][K + 1];
      k4_tab<K, K>(Tx, M);
      double acc[TX][K];
#pragma unroll
      for (int l = 0; l < TX; ++l)
#pragma unroll
        for (int m1 = 0; m1 < K; ++m1) acc[l][m1] = 0.0;
#pragma unroll
      for (int n = 0; n < F::NX; ++n) {
        const int l = n / K + 1, a = n % K;
        if (l - 1 < TX) {
#pragma unroll
          for (int m1 = 0; m1 < K; ++m1) acc[l - 1][m1] = fma(M[m1][a], yv[n], acc[l - 1][m1]);
        }
        if (a == 0 && l >= 2) {
#pragma unroll
          for (int m1 = 0; m1 < K; ++m1) acc[l - 2][m1] = fma(M[m1][K], yv[n], acc[l - 2][m1]);
        }
      }
      double* ob = V + ny * F::NZ + nz;
#pragma unroll
      for (int l = 0; l < TX; ++l)
#pragma unroll
        for (int m1 = 0; m1 < K; ++m1) ob[(m1 * TX + l) * F::NY * F::NZ] = acc[l][m1];
    }
    __syncthreads();
    k4_stage_y2<K, TX, TY, TZ>(V, U, t, Ty);
    __syncthreads();
    k4_stage_z2<K, TX, TY, TZ>(U, qa, t, Tz);
    __syncthreads();
  }
  const int g = t / F::GWZ2, col = t % F::GWZ2;
  if (g < K && col < TX * TY) {
    const int lx = col % TX, ly = col / TX, ex = ex0 + lx, ey = ey0 + ly;
    if (ex < N && ey < N) {
#pragma unroll
      for (int lz = 0; lz < TZ; ++lz) {
        const int ez = ez0 + lz;
        if (ez >= N) break;
        const int64_t e = ex + (int64_t)N * (ey + (int64_t)N * ez);
        // the group's modes (G - j, j, m3): written through a compile-time switch on g
        switch (g) {
#define K4_QW(GG)                                                                                  \
  case GG:                                                                                         \
    if constexpr (K > GG) {                                                                        \
      _Pragma("unroll") for (int j = 0; j <= GG; ++j) _Pragma("unroll") for (int m3 = 0; m3 < K - GG; ++m3) \
          p[e * se + (int64_t)k4_mode(GG - j, j, m3) * sm_] = sB * qa.v[j][lz][m3];                \
    }                                                                                              \
    break;
          K4_QW(0) K4_QW(1) K4_QW(2) K4_QW(3)
#undef K4_QW
        }
      }
    }
  }
}

}  // namespace wb
