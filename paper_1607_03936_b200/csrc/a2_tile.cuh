// a2_tile.cuh -- A(mu)u for k = 2 (row a5), tile-assembled, deterministic.
//
// Element arithmetic (thread per (element, component c)), sum-factorised with
// the exact structure of the k = 2 tables (GLL nodes {-1,0,1}, Gauss points
// {-sqrt(3/5), 0, sqrt(3/5)}):
//   I  (GLL -> Gauss):  row 1 = e_1; row 2 = row 0 reversed.
//   Dg (Gauss collocation derivative): Dg[1][1] = 0, Dg[1][2] = -Dg[1][0],
//       Dg[2][j] = -Dg[0][2-j].
// These hold bit-exactly for the closed-form tables (symmetric node sets), so
// only 4 distinct I entries and 4 distinct Dg entries are used.
//   U = (I x I x I) u_c;  g_cj = Dg_j U;  tau_cj = mut (g_cj + g_jc);
//   y_c = (I^T x I^T x I^T) sum_j Dg_j^T tau_cj,  mut = mu w_q detJ (2/h)^2,
// i.e. y_{c,a} = int 2 mu eps(u) : eps(phi_a e_c).
// The exchange of g_jc between the three component threads of an element goes
// through shared memory one Gauss level at a time.
//
// Assembly (deterministic, no atomics, no inter-CTA waiting): the TX x TY x TZ
// element tile sums its (2TX+1)(2TY+1)(2TZ+1) nodes in shared memory in a fixed
// order (ascending element index).  Tile-interior nodes are complete and go
// straight to y; nodes on the tile's upper shell and lower faces go to small
// partial buffers (L2-resident), and a second kernel (k_A_skel) sums every
// tile-skeleton node over the tiles holding it in ascending tile index.
#pragma once
#include "kernels.cuh"

namespace wb {

#ifdef WB_KPROF
// phase-timing probe (build -DWB_KPROF): thread 0 of every A tile CTA adds its clock64
// cycles per phase: [0] staging issue, [1] staging wait + barrier, [2] U load + interpolation,
// [3] Gauss levels, [4] transposed interpolation, [5] slots + barrier, [6] node sums /
// outputs, [7] CTAs
__device__ unsigned long long g_aprof[8];
#define A_LAP(k)                                                              \
  do {                                                                        \
    if (threadIdx.x == 0) {                                                   \
      const long long n_ = clock64();                                         \
      atomicAdd(&g_aprof[k], (unsigned long long)(n_ - a_tc));                \
      a_tc = n_;                                                              \
    }                                                                         \
  } while (0)
#else
#define A_LAP(k) do { } while (0)
#endif

struct K2Coef {
  double i00, i01, i02;   // I row 0 (row 2 reversed, row 1 = e_1)
  double a, b, c, d;      // Dg row 0 = (a, b, c), Dg row 1 = (d, 0, -d), Dg row 2 = (-c, -b, -a)
};

__device__ __forceinline__ K2Coef k2coef() {
  K2Coef k;
  k.i00 = TB(2).I[0][0]; k.i01 = TB(2).I[0][1]; k.i02 = TB(2).I[0][2];
  k.a = TB(2).Dg[0][0]; k.b = TB(2).Dg[0][1]; k.c = TB(2).Dg[0][2]; k.d = TB(2).Dg[1][0];
  return k;
}

// forward interpolation of one pencil (in place): 5 flops
__device__ __forceinline__ void k2_interp(const K2Coef& k, double& v0, double v1, double& v2) {
  const double s = k.i01 * v1;
  const double o0 = fma(k.i00, v0, fma(k.i02, v2, s));
  const double o2 = fma(k.i02, v0, fma(k.i00, v2, s));
  v0 = o0; v2 = o2;
}
// collocation derivative of one pencil: 7 flops
__device__ __forceinline__ void k2_deriv(const K2Coef& k, double v0, double v1, double v2, double& o0, double& o1,
                                         double& o2) {
  const double bv = k.b * v1;
  o0 = fma(k.a, v0, fma(k.c, v2, bv));
  o2 = -fma(k.c, v0, fma(k.a, v2, bv));
  o1 = k.d * (v0 - v2);
}
// transposed derivative accumulated into (t0, t1, t2): 8 flops
__device__ __forceinline__ void k2_derivT_acc(const K2Coef& k, double w0, double w1, double w2, double& t0,
                                              double& t1, double& t2) {
  t0 = fma(k.a, w0, fma(k.d, w1, fma(-k.c, w2, t0)));
  t1 = fma(k.b, w0 - w2, t1);
  t2 = fma(k.c, w0, fma(-k.d, w1, fma(-k.a, w2, t2)));
}
// transposed interpolation of one pencil (in place): 6 flops
__device__ __forceinline__ void k2_interpT(const K2Coef& k, double& v0, double& v1, double& v2) {
  const double o0 = fma(k.i00, v0, k.i02 * v2);
  const double o1 = fma(k.i01, v0 + v2, v1);
  const double o2 = fma(k.i02, v0, k.i00 * v2);
  v0 = o0; v1 = o1; v2 = o2;
}

#define U3(z, y, x) U[((z)*3 + (y)) * 3 + (x)]
#define V3(z, y, x) V[((z)*3 + (y)) * 3 + (x)]

// Element values V (27, Gauss-node order a = ax + 3(ay + 3az)) of component c.
__device__ __forceinline__ void cp_async8(double* smem_dst, const double* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Staged nodal u of a TX x TY x TZ tile: Us[c][nz][ny][RSU], x split by parity
// (even nodes, then odd) with RSU = 2 (mod 8): 4 x-consecutive elements x 4
// y-consecutive elements (a half-warp) read 16 distinct bank pairs.
template <int TX, int TY, int TZ>
struct UsL {
  static constexpr int MX = 2 * TX + 1, MY = 2 * TY + 1, MZ = 2 * TZ + 1;
  static constexpr int RSU = MX + ((10 - MX % 8) % 8);
  static constexpr int NN = RSU * MY * MZ;
  __host__ __device__ static constexpr int col(int nx) { return (nx & 1) ? TX + 1 + (nx >> 1) : (nx >> 1); }
};

template <int TX, int TY, int TZ>
__device__ __forceinline__ void a2_elem(const double* __restrict__ Mu, const double* __restrict__ Us, int lx,
                                        int ly, int lz, int c, int le, double* X, double (&V)[27]) {
  constexpr int NE = TX * TY * TZ;
  using L = UsL<TX, TY, TZ>;
  const K2Coef k = k2coef();
  // (the caller has made the staged mut and u of the tile visible to every thread;
  // mut is 0 for elements outside the mesh, so their V is 0)
  // per-thread bases: every shared access below is base + compile-time offset
  const double* __restrict__ Ub = Us + c * L::NN + L::RSU * (2 * ly + L::MY * 2 * lz) + lx;
  const double* __restrict__ Mb = Mu + le;
  double* Xw = X + c * 3 * NE + le;         // X[q][c][j] <- g_cj
  const double* Xr = X + c * NE + le;       // X[q][j][c] -> g_jc
  double U[27];
#pragma unroll
  for (int az = 0; az < 3; ++az)
#pragma unroll
    for (int ay = 0; ay < 3; ++ay)
#pragma unroll
      for (int ax = 0; ax < 3; ++ax)  // Dirichlet entries were staged as 0
        U3(az, ay, ax) = Ub[L::RSU * (ay + L::MY * az) + (ax == 1 ? TX + 1 : (ax >> 1))];
#ifdef WB_KPROF
  long long a_tc = clock64();
#endif
  // GLL -> Gauss in x, y, z
#pragma unroll
  for (int z = 0; z < 3; ++z)
#pragma unroll
    for (int y = 0; y < 3; ++y) k2_interp(k, U3(z, y, 0), U3(z, y, 1), U3(z, y, 2));
#pragma unroll
  for (int z = 0; z < 3; ++z)
#pragma unroll
    for (int x = 0; x < 3; ++x) k2_interp(k, U3(z, 0, x), U3(z, 1, x), U3(z, 2, x));
#pragma unroll
  for (int y = 0; y < 3; ++y)
#pragma unroll
    for (int x = 0; x < 3; ++x) k2_interp(k, U3(0, y, x), U3(1, y, x), U3(2, y, x));
  A_LAP(2);
#pragma unroll
  for (int q = 0; q < 27; ++q) V[q] = 0.0;
#pragma unroll
  for (int iz = 0; iz < 3; ++iz) {
    double mu[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) mu[q] = Mb[(iz * 9 + q) * NE];
    double gx[9], gy[9], gz[9];
#pragma unroll
    for (int y = 0; y < 3; ++y) k2_deriv(k, U3(iz, y, 0), U3(iz, y, 1), U3(iz, y, 2), gx[y * 3], gx[y * 3 + 1], gx[y * 3 + 2]);
#pragma unroll
    for (int x = 0; x < 3; ++x) k2_deriv(k, U3(iz, 0, x), U3(iz, 1, x), U3(iz, 2, x), gy[x], gy[3 + x], gy[6 + x]);
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      const double u0 = U[q], u1 = U[9 + q], u2 = U[18 + q];
      if (iz == 0) gz[q] = fma(k.a, u0, fma(k.b, u1, k.c * u2));
      else if (iz == 1) gz[q] = k.d * (u0 - u2);
      else gz[q] = -fma(k.c, u0, fma(k.b, u1, k.a * u2));
    }
    // exchange: X[q][c*3 + j][le] = g_cj
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      Xw[(q * 9 + 0) * NE] = gx[q];
      Xw[(q * 9 + 1) * NE] = gy[q];
      Xw[(q * 9 + 2) * NE] = gz[q];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      gx[q] = mu[q] * (gx[q] + Xr[(q * 9 + 0 * 3) * NE]);
      gy[q] = mu[q] * (gy[q] + Xr[(q * 9 + 1 * 3) * NE]);
      gz[q] = mu[q] * (gz[q] + Xr[(q * 9 + 2 * 3) * NE]);
    }
    __syncthreads();
    // back: V(iz,.,.) += Dg_x^T Wx + Dg_y^T Wy;  V(., ., .) += Dg[iz][jz] Wz
#pragma unroll
    for (int y = 0; y < 3; ++y) k2_derivT_acc(k, gx[y * 3], gx[y * 3 + 1], gx[y * 3 + 2], V3(iz, y, 0), V3(iz, y, 1), V3(iz, y, 2));
#pragma unroll
    for (int x = 0; x < 3; ++x) k2_derivT_acc(k, gy[x], gy[3 + x], gy[6 + x], V3(iz, 0, x), V3(iz, 1, x), V3(iz, 2, x));
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      if (iz == 0) { V[q] = fma(k.a, gz[q], V[q]); V[9 + q] = fma(k.b, gz[q], V[9 + q]); V[18 + q] = fma(k.c, gz[q], V[18 + q]); }
      else if (iz == 1) { V[q] = fma(k.d, gz[q], V[q]); V[18 + q] = fma(-k.d, gz[q], V[18 + q]); }
      else { V[q] = fma(-k.c, gz[q], V[q]); V[9 + q] = fma(-k.b, gz[q], V[9 + q]); V[18 + q] = fma(-k.a, gz[q], V[18 + q]); }
    }
  }
  A_LAP(3);
  // Gauss -> GLL transposed, z, y, x
#pragma unroll
  for (int y = 0; y < 3; ++y)
#pragma unroll
    for (int x = 0; x < 3; ++x) k2_interpT(k, V3(0, y, x), V3(1, y, x), V3(2, y, x));
#pragma unroll
  for (int z = 0; z < 3; ++z)
#pragma unroll
    for (int x = 0; x < 3; ++x) k2_interpT(k, V3(z, 0, x), V3(z, 1, x), V3(z, 2, x));
#pragma unroll
  for (int z = 0; z < 3; ++z)
#pragma unroll
    for (int y = 0; y < 3; ++y) k2_interpT(k, V3(z, y, 0), V3(z, y, 1), V3(z, y, 2));
  A_LAP(4);
}
#undef U3
#undef V3

template <int TX, int TY, int TZ>
struct Tile2 {
  static constexpr int NE = TX * TY * TZ, NT = 3 * NE;
  static constexpr int MX = 2 * TX + 1, MY = 2 * TY + 1, MZ = 2 * TZ + 1, NN = MX * MY * MZ;
  static constexpr int SHELL = NN - (2 * TX) * (2 * TY) * (2 * TZ);                             // upper shell
  static constexpr int XS = 81 * NE;  // exchange / slot doubles
  // exchange/slots, then the stage buffer (mut, u)
  static constexpr size_t SMEM = sizeof(double) * (XS + 27 * NE + 3 * UsL<TX, TY, TZ>::NN);
  // index of an upper-shell node (nx == 2TX || ny == 2TY || nz == 2TZ)
  __host__ __device__ static __forceinline__ int shell(int nx, int ny, int nz) {
    if (nz == 2 * TZ) return ny * MX + nx;
    if (ny == 2 * TY) return MX * MY + nz * MX + nx;
    return MX * MY + 2 * TZ * MX + nz * (2 * TY) + ny;
  }
};

// Tile-local sum of component c at tile node 2l + A (per axis) over the slots
// R[c][a][le]: per axis, A = 1 -> element l (local 1); A = 2 -> element l
// (local 2); A = 0 -> element l-1 (local 2, if l > 0) then element l (local 0).
// Elements in ascending index order.  A is compile-time after unrolling.
template <int TX, int TY, int TZ>
__device__ __forceinline__ double a2_node_sum(const double* __restrict__ Rb, const double (&V)[27], int lx, int ly,
                                              int lz, int AX, int AY, int AZ) {
  // Rb = R + c * 27 * NE + le: slot (c, a, element le + d) at Rb[a * NE + d].  The own
  // element's term comes from its registers V.  Terms t(kz, ky, kx), k_d = 0 the lower
  // element (absent at the tile's lower face: +0.0) and 1 the own one along axes with
  // A_d = 0, are summed as a fixed pairwise tree: x pairs, then y, then z.
  constexpr int NE = TX * TY * TZ;
  double t[2][2][2];
#pragma unroll
  for (int kz = 0; kz < 2; ++kz)
#pragma unroll
    for (int ky = 0; ky < 2; ++ky)
#pragma unroll
      for (int kx = 0; kx < 2; ++kx) {
        t[kz][ky][kx] = 0.0;
        if ((AZ != 0 && kz == 1) || (AY != 0 && ky == 1) || (AX != 0 && kx == 1)) continue;
        const int dz = AZ == 0 ? kz - 1 : 0, az = AZ == 0 ? (kz == 0 ? 2 : 0) : AZ;
        const int dy = AY == 0 ? ky - 1 : 0, ay = AY == 0 ? (ky == 0 ? 2 : 0) : AY;
        const int dx = AX == 0 ? kx - 1 : 0, ax = AX == 0 ? (kx == 0 ? 2 : 0) : AX;
        const int a = ax + 3 * (ay + 3 * az);
        if (dx == 0 && dy == 0 && dz == 0) {
          t[kz][ky][kx] = V[a];
        } else if (lx + dx >= 0 && ly + dy >= 0 && lz + dz >= 0) {
          t[kz][ky][kx] = Rb[a * NE + dx + TX * (dy + TY * dz)];
        }
      }
  double sy[2][2];
#pragma unroll
  for (int kz = 0; kz < 2; ++kz)
#pragma unroll
    for (int ky = 0; ky < 2; ++ky) sy[kz][ky] = AX == 0 ? t[kz][ky][0] + t[kz][ky][1] : t[kz][ky][0];
  double sz[2];
#pragma unroll
  for (int kz = 0; kz < 2; ++kz) sz[kz] = AY == 0 ? sy[kz][0] + sy[kz][1] : sy[kz][0];
  return AZ == 0 ? sz[0] + sz[1] : sz[0];
}

// slots read by other threads: local index 2 in some axis (the node belongs to the
// next element or the upper shell)
__host__ __device__ constexpr bool a2_slot_shared(int a) { return a % 3 == 2 || (a / 3) % 3 == 2 || a / 9 == 2; }

__device__ __forceinline__ void cp_async16(double* smem_dst, const double* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gsrc) : "memory");
}

// Tile geometry shared by the stage / output code
struct A2Tile {
  int tile, tx, ty, tz, bx, by, bz;
  bool inner;  // the tile's node box lies strictly inside the mesh
};
template <int TX, int TY, int TZ>
__device__ __forceinline__ A2Tile a2_tile_of(int tile, const Geo& G) {
  const int NTX = (G.N + TX - 1) / TX, NTY = (G.N + TY - 1) / TY;
  A2Tile t;
  t.tile = tile;
  t.tx = tile % NTX; t.ty = (tile / NTX) % NTY; t.tz = tile / (NTX * NTY);
  t.bx = 2 * TX * t.tx; t.by = 2 * TY * t.ty; t.bz = 2 * TZ * t.tz;
  const int e = G.nn1 - 1;
  t.inner = t.bx > 0 && t.by > 0 && t.bz > 0 && t.bx + 2 * TX < e && t.by + 2 * TY < e && t.bz + 2 * TZ < e;
  return t;
}
// the same from a 3-D grid (NTX, NTY, NTZ): no runtime div / mod (tile = tx + NTX (ty + NTY tz), the
// linear launch order of the 1-D form)
template <int TX, int TY, int TZ>
__device__ __forceinline__ A2Tile a2_tile_of_grid(const Geo& G) {
  A2Tile t;
  t.tx = blockIdx.x; t.ty = blockIdx.y; t.tz = blockIdx.z;
  t.tile = t.tx + gridDim.x * (t.ty + gridDim.y * t.tz);
  t.bx = 2 * TX * t.tx; t.by = 2 * TY * t.ty; t.bz = 2 * TZ * t.tz;
  const int e = G.nn1 - 1;
  t.inner = t.bx > 0 && t.by > 0 && t.bz > 0 && t.bx + 2 * TX < e && t.by + 2 * TY < e && t.bz + 2 * TZ < e;
  return t;
}

// Stage NC nodal components (component stride cs) of a tile's (2TX+1)(2TY+1)(2TZ+1)
// node box into Us[cc][nz][ny][col] by cp.async (no wait); nodes outside the mesh,
// and Dirichlet nodes unless nomask, as 0 (the elimination of DESIGN.md R6).  Each
// warp copies RPW node rows of MX per pass (lane -> (row, nx)); a thread's rows
// advance by RPP rows, i.e. ny is fixed and (cc, nz) steps by RPP / MY, so the
// addresses update incrementally.  NTH threads take part.
template <int TX, int TY, int TZ, int NC, int NTH>
__device__ __forceinline__ void a2_stage_nodal(const double* __restrict__ u, int64_t cs, double* Us, const A2Tile& t,
                                               const Geo& G, int nomask) {
  using L = UsL<TX, TY, TZ>;
  constexpr int NW = NTH / 32;
  constexpr int RPW = 32 / L::MX, RPP = NW * RPW, NROWS = NC * L::MY * L::MZ;
  static_assert(RPP % L::MY == 0, "row stepping keeps ny fixed");
  constexpr int DQ = RPP / L::MY;  // (cc, nz) step per pass
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int sub = lane / L::MX, nx = lane - sub * L::MX;
  if (sub >= RPW || w >= NW) return;
  const int r0 = w * RPW + sub;
  const int ny = r0 % L::MY;
  int q = r0 / L::MY;  // q = cc * MZ + nz
  int nz = q % L::MZ, cc = q / L::MZ;
  const int nn1 = G.nn1;
  const int64_t nn2 = (int64_t)nn1 * nn1;
  const double* src = u + cc * cs + node_id(t.bx + nx, t.by + ny, t.bz + nz, nn1);
  double* dst = Us + cc * L::NN + L::RSU * (ny + L::MY * nz) + L::col(nx);
  const int gx = t.bx + nx, gy = t.by + ny;
  const bool colok = gx < nn1 && gy < nn1 && (nomask || (gx != 0 && gy != 0 && gx != nn1 - 1 && gy != nn1 - 1));
  for (int r = r0; r < NROWS; r += RPP) {
    if (t.inner) {
      cp_async8(dst, src);
    } else {
      const int gz = t.bz + nz;
      if (colok && gz < nn1 && (nomask || (gz != 0 && gz != nn1 - 1)))
        cp_async8(dst, src);
      else
        *dst = 0.0;
    }
    // (cc, nz) += DQ in units of nz, wrapping nz at MZ
    nz += DQ;
    if (nz >= L::MZ) {
      nz -= L::MZ; ++cc;
      src += cs - (int64_t)(L::MZ - DQ) * nn2;
      dst += L::NN - (L::MZ - DQ) * L::RSU * L::MY;
    } else {
      src += DQ * nn2;
      dst += DQ * L::RSU * L::MY;
    }
  }
}

// Stage an A tile: its mut block (tile-blocked layout, one contiguous block) and its
// nodal u (three components).
template <int TX, int TY, int TZ>
__device__ __forceinline__ void a2_stage(const double* __restrict__ mutT, const double* __restrict__ u,
                                         double* Mu, double* Us, const A2Tile& t, const Geo& G, int nomask) {
  constexpr int NE = TX * TY * TZ, NTH = 3 * NE;
  {
    const double* src = mutT + (size_t)t.tile * 27 * NE;
    for (int i = threadIdx.x; i < 27 * NE / 2; i += NTH) cp_async16(Mu + 2 * i, src + 2 * i);
  }
  a2_stage_nodal<TX, TY, TZ, 3, NTH>(u, G.n_nodes, Us, t, G, nomask);
}

// Kernel 1 of A: one CTA per TX x TY x TZ element tile, thread per (element,
// component).  The tile's nodes are summed in shared memory (fixed order,
// a2_node_sum) and leave the kernel by class:
//   upper shell (some n_d == 2T_d): partial -> Fu[tile][c][shell];
//   else (all n_d < 2T_d): the tile's own sum -> y (complete for tile-interior
//   nodes; for lower-face nodes k_A_skel adds the lower tiles' partials in front).
// mutT is tile-blocked, mutT[tile][q][le] (zero for elements outside the mesh).
// No inter-CTA communication; several small CTAs per SM overlap each other's
// staging, barriers and compute.
template <int TX, int TY, int TZ, int MINB>
__global__ void __launch_bounds__(3 * TX * TY * TZ, MINB)
    k_A_tile(const double* __restrict__ mutT, const double* __restrict__ u, double* __restrict__ y,
             double* __restrict__ Fu, Geo G, int nomask) {
  using T = Tile2<TX, TY, TZ>;
  constexpr int NE = T::NE;
  extern __shared__ __align__(16) double smem_a2[];
  double* X = smem_a2;  // [XS]: gradient exchange, then element slots R[c][a][le]
  double* Mu = smem_a2 + T::XS;
  double* Us = Mu + 27 * NE;
#ifdef WB_KPROF
  long long a_tc = clock64();
#endif
  const A2Tile t = a2_tile_of_grid<TX, TY, TZ>(G);  // launched on the (NTX, NTY, NTZ) grid
  const int tile = t.tile;
  a2_stage<TX, TY, TZ>(mutT, u, Mu, Us, t, G, nomask);
  A_LAP(0);
  const int le = threadIdx.x % NE, c = threadIdx.x / NE;
  const int lx = le % TX, ly = (le / TX) % TY, lz = le / (TX * TY);
  const int nn1 = G.nn1, kN = 2 * G.N;
  cp_async_wait_all();  // this thread's copies
  __syncthreads();      // everyone's
  A_LAP(1);
  double V[27];
  a2_elem<TX, TY, TZ>(Mu, Us, lx, ly, lz, c, le, X, V);
#ifdef WB_KPROF
  a_tc = clock64();  // a2_elem timed its own phases
#endif
  // element slots R[c][a][le] (the exchange buffer is free after the last level's barrier)
  double* Rb = X + c * 27 * NE + le;
#pragma unroll
  for (int a = 0; a < 27; ++a)
    if (a2_slot_shared(a)) Rb[a * NE] = V[a];
  __syncthreads();
  A_LAP(5);
  // Each thread is responsible for the tile nodes 2l + A, A_d in {0, 1}, plus A_d = 2
  // on the tile's upper face (l_d = T_d - 1): every tile node has exactly one
  // responsible (element, c) thread, and the node's structure is compile-time.
  double* Fut = Fu + ((size_t)tile * 3 + c) * T::SHELL;
  double* yb = y + c * G.n_nodes + node_id(t.bx, t.by, t.bz, nn1);
#pragma unroll
  for (int AZ = 0; AZ < 3; ++AZ)
#pragma unroll
    for (int AY = 0; AY < 3; ++AY)
#pragma unroll
      for (int AX = 0; AX < 3; ++AX) {
        if ((AX == 2 && lx != TX - 1) || (AY == 2 && ly != TY - 1) || (AZ == 2 && lz != TZ - 1)) continue;
        const int nx = 2 * lx + AX, ny = 2 * ly + AY, nz = 2 * lz + AZ;
        const double s = a2_node_sum<TX, TY, TZ>(Rb, V, lx, ly, lz, AX, AY, AZ);
        if (AX == 2 || AY == 2 || AZ == 2) {
          // (responsibility implies n_d == 2T_d exactly where A_d == 2: T::shell's branches
          // resolve at compile time)
          const int si = AZ == 2 ? ny * T::MX + nx
                                 : (AY == 2 ? T::MX * T::MY + nz * T::MX + nx
                                            : T::MX * T::MY + 2 * TZ * T::MX + nz * (2 * TY) + ny);
          Fut[si] = s;
        } else {
          double* dst = yb + (nz * nn1 + ny) * nn1 + nx;
          if (t.inner) {
            *dst = s;
          } else {
            const int gx = t.bx + nx, gy = t.by + ny, gz = t.bz + nz;
            if (gx <= kN && gy <= kN && gz <= kN) *dst = (nomask || !node_bnd(gx, gy, gz, nn1)) ? s : 0.0;
          }
        }
      }
  A_LAP(6);
#ifdef WB_KPROF
  if (threadIdx.x == 0) atomicAdd(&g_aprof[7], 1ull);
#endif
}

// Kernel 2 of A: the tile-skeleton nodes (g_d a multiple of 2T_d in some axis),
// one thread per node, all three components.  Each is summed over the tiles
// whose closed node box holds it, in ascending tile index (per axis the lower
// tile, whose upper shell holds the node, then the upper one), from 0.0: a fixed
// order, so results are bitwise reproducible.  The last tile, when the node is
// not on its upper shell, is the node's own tile, whose sum k_A_tile left in y.  Node enumeration: x-planes, then
// y-planes off the x-planes, then z-planes off both.
__device__ __forceinline__ int a2_offplane(int k, int M) { return (k / (M - 1)) * M + k % (M - 1) + 1; }
// node coordinate g on an axis of tile size S (nodes), NT tiles: the first
// contributing tile t0, the node's local index there n0, and the count (1 or 2; the
// second tile is t0 + 1 with local index 0)
__device__ __forceinline__ void a2_axis(int g, int S, int NT, int& t0, int& n0, int& cnt) {
  const int hi = g / S;
  if (g - hi * S != 0) { t0 = hi; n0 = g - hi * S; cnt = 1; }
  else if (hi == 0) { t0 = 0; n0 = 0; cnt = 1; }
  else { t0 = hi - 1; n0 = S; cnt = hi < NT ? 2 : 1; }
}

template <int TX, int TY, int TZ>
__global__ void __launch_bounds__(256) k_A_skel(const double* __restrict__ Fu, double* __restrict__ y, Geo G,
                                                int nomask) {
  using T = Tile2<TX, TY, TZ>;
  constexpr int SX = 2 * TX, SY = 2 * TY, SZ = 2 * TZ;
  const int nn1 = G.nn1;
  const int NTX = (G.N + TX - 1) / TX, NTY = (G.N + TY - 1) / TY, NTZ = (G.N + TZ - 1) / TZ;
  const int PX = (nn1 - 1) / SX + 1, PY = (nn1 - 1) / SY + 1, PZ = (nn1 - 1) / SZ + 1;
  const int QX = nn1 - PX, QY = nn1 - PY;
  const int64_t nX = (int64_t)PX * nn1 * nn1, nY = (int64_t)QX * PY * nn1, nZ = (int64_t)QX * QY * PZ;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int gx, gy, gz;
  if (i < nX) {
    gy = (int)(i % nn1);
    const int64_t r = i / nn1;
    gz = (int)(r % nn1); gx = SX * (int)(r / nn1);
  } else if ((i -= nX) < nY) {
    gx = a2_offplane((int)(i % QX), SX);
    const int64_t r = i / QX;
    gy = SY * (int)(r % PY); gz = (int)(r / PY);
  } else if ((i -= nY) < nZ) {
    gx = a2_offplane((int)(i % QX), SX);
    const int64_t r = i / QX;
    gy = a2_offplane((int)(r % QY), SY); gz = SZ * (int)(r / QY);
  } else {
    return;
  }
  const int64_t g = node_id(gx, gy, gz, nn1), nv = G.n_nodes;
  if (!nomask && node_bnd(gx, gy, gz, nn1)) {
    y[g] = 0.0; y[nv + g] = 0.0; y[2 * nv + g] = 0.0;
    return;
  }
  // per axis: contributing tiles (ascending, t0 [, t0 + 1]) and the node's local index in each
  int tx0, nx0, cx, ty0, ny0, cy, tz0, nz0, cz;
  a2_axis(gx, SX, NTX, tx0, nx0, cx);
  a2_axis(gy, SY, NTY, ty0, ny0, cy);
  a2_axis(gz, SZ, NTZ, tz0, nz0, cz);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll
  for (int iz = 0; iz < 2; ++iz) {
    if (iz >= cz) break;
    const int tz = tz0 + iz, nz = iz ? 0 : nz0;
#pragma unroll
    for (int iy = 0; iy < 2; ++iy) {
      if (iy >= cy) break;
      const int ty = ty0 + iy, ny = iy ? 0 : ny0;
#pragma unroll
      for (int ix = 0; ix < 2; ++ix) {
        if (ix >= cx) break;
        const int tile = (tx0 + ix) + NTX * (ty + NTY * tz);
        const int nx = ix ? 0 : nx0;
        const double* P;
        int st;
        if (nx == SX || ny == SY || nz == SZ) {
          P = Fu + (size_t)tile * 3 * T::SHELL + T::shell(nx, ny, nz); st = T::SHELL;
        } else {  // the node's own tile (last in the order): its sum is already in y
          P = y + g; st = (int)nv;
        }
        a0 += __ldcg(P); a1 += __ldcg(P + st); a2 += __ldcg(P + 2 * st);
      }
    }
  }
  y[g] = a0; y[nv + g] = a1; y[2 * nv + g] = a2;
}

// number of skeleton nodes (kernel 2 threads)
template <int TX, int TY, int TZ>
inline int64_t a2_skel_count(int N) {
  const int nn1 = 2 * N + 1;
  const int PX = (nn1 - 1) / (2 * TX) + 1, PY = (nn1 - 1) / (2 * TY) + 1, PZ = (nn1 - 1) / (2 * TZ) + 1;
  const int QX = nn1 - PX, QY = nn1 - PY;
  return (int64_t)PX * nn1 * nn1 + (int64_t)QX * PY * nn1 + (int64_t)QX * QY * PZ;
}

}  // namespace wb
