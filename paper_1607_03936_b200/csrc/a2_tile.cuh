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
// Assembly: the TX x TY x TZ element tile sums its (2TX+1)(2TY+1)(2TZ+1)
// nodes in shared memory in a fixed order (ascending element index); nodes on
// the tile's upper faces go to a per-tile partial buffer F (L2-resident), and
// every node is finalised by the tile that owns it (local index < 2T, or the
// domain end) after a release/acquire look-back on its lower neighbours'
// flags: partials are added in ascending tile index.  Tiles take logical
// indices from an atomic ticket, so a tile only ever waits for tiles that have
// already started: no deadlock, no dependence on hardware launch order.
#pragma once
#include "kernels.cuh"

namespace wb {

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
__device__ __forceinline__ void a2_elem(const double* __restrict__ Mu, const double* __restrict__ Us, bool valid,
                                        int lx, int ly, int lz, int c, int le, double* X, double (&V)[27]) {
  constexpr int NE = TX * TY * TZ;
  using L = UsL<TX, TY, TZ>;
  const K2Coef k = k2coef();
  // mut and u of the tile, staged in shared memory by cp.async from all threads:
  // wait for this thread's copies, then a barrier makes everyone's visible
  cp_async_wait_all();
  __syncthreads();
  double U[27];
#pragma unroll
  for (int az = 0; az < 3; ++az)
#pragma unroll
    for (int ay = 0; ay < 3; ++ay)
#pragma unroll
      for (int ax = 0; ax < 3; ++ax)  // Dirichlet entries were staged as 0
        U3(az, ay, ax) = Us[c * L::NN + L::RSU * ((2 * ly + ay) + L::MY * (2 * lz + az)) +
                            (ax == 1 ? TX + 1 + lx : lx + (ax >> 1))];
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
#pragma unroll
  for (int q = 0; q < 27; ++q) V[q] = 0.0;
#pragma unroll
  for (int iz = 0; iz < 3; ++iz) {
    double mu[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) mu[q] = valid ? Mu[(iz * 9 + q) * NE + le] : 0.0;
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
      X[(q * 9 + c * 3 + 0) * NE + le] = gx[q];
      X[(q * 9 + c * 3 + 1) * NE + le] = gy[q];
      X[(q * 9 + c * 3 + 2) * NE + le] = gz[q];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      gx[q] = mu[q] * (gx[q] + X[(q * 9 + 0 * 3 + c) * NE + le]);
      gy[q] = mu[q] * (gy[q] + X[(q * 9 + 1 * 3 + c) * NE + le]);
      gz[q] = mu[q] * (gz[q] + X[(q * 9 + 2 * 3 + c) * NE + le]);
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
}
#undef U3
#undef V3

template <int TX, int TY, int TZ>
struct Tile2 {
  static constexpr int NE = TX * TY * TZ, NT = 3 * NE;
  static constexpr int MX = 2 * TX + 1, MY = 2 * TY + 1, MZ = 2 * TZ + 1, NN = MX * MY * MZ;
  static constexpr int SHELL = NN - (2 * TX) * (2 * TY) * (2 * TZ);
  static constexpr int XS = 81 * NE;  // exchange / slot doubles
  static constexpr size_t SMEM = sizeof(double) * (XS + 27 * NE + 3 * UsL<TX, TY, TZ>::NN);  // exchange/slots, mut, u
  // index of an upper-shell node (nx == 2TX || ny == 2TY || nz == 2TZ)
  __device__ static __forceinline__ int shell(int nx, int ny, int nz) {
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
__device__ __forceinline__ double a2_node_sum(const double* __restrict__ R, int c, int lx, int ly, int lz, int AX,
                                              int AY, int AZ) {
  constexpr int NE = TX * TY * TZ;
  double acc = 0.0;
#pragma unroll
  for (int kz = 0; kz < 2; ++kz) {
    if (AZ != 0 && kz == 1) continue;
    const int qz = AZ == 0 ? lz - 1 + kz : lz, az = AZ == 0 ? (kz == 0 ? 2 : 0) : AZ;
    if (qz < 0) continue;
#pragma unroll
    for (int ky = 0; ky < 2; ++ky) {
      if (AY != 0 && ky == 1) continue;
      const int qy = AY == 0 ? ly - 1 + ky : ly, ay = AY == 0 ? (ky == 0 ? 2 : 0) : AY;
      if (qy < 0) continue;
#pragma unroll
      for (int kx = 0; kx < 2; ++kx) {
        if (AX != 0 && kx == 1) continue;
        const int qx = AX == 0 ? lx - 1 + kx : lx, ax = AX == 0 ? (kx == 0 ? 2 : 0) : AX;
        if (qx < 0) continue;
        acc += R[(c * 27 + ax + 3 * (ay + 3 * az)) * NE + qx + TX * (qy + TY * qz)];
      }
    }
  }
  return acc;
}

template <int TX, int TY, int TZ, int MINB>
__global__ void __launch_bounds__(3 * TX * TY * TZ, MINB)
    k_A_tile(const double* __restrict__ mut, const double* __restrict__ u, double* __restrict__ y,
             double* __restrict__ F, int* __restrict__ flag, unsigned long long* ticket,
             unsigned long long ticket_base, int epoch, Geo G, int nomask) {
  using T = Tile2<TX, TY, TZ>;
  constexpr int NE = T::NE, NTH = T::NT;
  extern __shared__ __align__(16) double smem_a2[];
  double* X = smem_a2;  // [XS]: gradient exchange, then element slots R[c][a][le]
  __shared__ int s_tile;
  if (threadIdx.x == 0) s_tile = (int)(atomicAdd(ticket, 1ull) - ticket_base);
  __syncthreads();
  const int tile = s_tile;
  const int NTX = (G.N + TX - 1) / TX, NTY = (G.N + TY - 1) / TY;
  const int tx = tile % NTX, ty = (tile / NTX) % NTY, tz = tile / (NTX * NTY);
  const int le = threadIdx.x % NE, c = threadIdx.x / NE;
  const int lx = le % TX, ly = (le / TX) % TY, lz = le / (TX * TY);
  const int ex = TX * tx + lx, ey = TY * ty + ly, ez = TZ * tz + lz;
  const bool valid = ex < G.N && ey < G.N && ez < G.N;
  double V[27];
  // stage the tile's mut (27 per element, element-contiguous) into Mu[q*NE + le] and its
  // nodal u (Dirichlet entries as 0, the elimination of DESIGN.md R6) into Us,
  // asynchronously; a2_elem waits for them
  double* Mu = smem_a2 + T::XS;
  double* Us = Mu + 27 * NE;
  for (int i = threadIdx.x; i < 27 * NE; i += NTH) {
    const int l = i / 27, q = i % 27;
    const int qx = TX * tx + l % TX, qy = TY * ty + (l / TX) % TY, qz = TZ * tz + l / (TX * TY);
    if (qx < G.N && qy < G.N && qz < G.N)
      cp_async8(Mu + q * NE + l, mut + (qx + (int64_t)G.N * (qy + (int64_t)G.N * qz)) * 27 + q);
  }
  {
    using L = UsL<TX, TY, TZ>;
    const int bx = 2 * TX * tx, by = 2 * TY * ty, bz = 2 * TZ * tz;
    for (int i = threadIdx.x; i < 3 * L::MX * L::MY * L::MZ; i += NTH) {
      const int nx = i % L::MX, ny = (i / L::MX) % L::MY, r = i / (L::MX * L::MY), nz = r % L::MZ, cc = r / L::MZ;
      const int gx = bx + nx, gy = by + ny, gz = bz + nz;
      double* dst = Us + cc * L::NN + L::RSU * (ny + L::MY * nz) + L::col(nx);
      if (gx < G.nn1 && gy < G.nn1 && gz < G.nn1 && (nomask || !node_bnd(gx, gy, gz, G.nn1)))
        cp_async8(dst, u + cc * G.n_nodes + node_id(gx, gy, gz, G.nn1));
      else
        *dst = 0.0;
    }
  }
  a2_elem<TX, TY, TZ>(Mu, Us, valid, lx, ly, lz, c, le, X, V);
  // element slots R[c][a][le] (the exchange buffer is free after the last level's barrier)
#pragma unroll
  for (int a = 0; a < 27; ++a) X[(c * 27 + a) * NE + le] = V[a];
  __syncthreads();
  // Each thread is responsible for the tile nodes 2l + A, A_d in {0, 1}, plus A_d = 2
  // on the tile's upper face (l_d = T_d - 1): every tile node has exactly one
  // responsible (element, c) thread, and the node's structure is compile-time.
  // Phase A: upper-shell nodes (some A_d = 2) -> F[tile][c][shell]
  double* Ft = F + (size_t)tile * 3 * T::SHELL;
#pragma unroll
  for (int AZ = 0; AZ < 3; ++AZ)
#pragma unroll
    for (int AY = 0; AY < 3; ++AY)
#pragma unroll
      for (int AX = 0; AX < 3; ++AX) {
        if (AX < 2 && AY < 2 && AZ < 2) continue;
        if ((AX == 2 && lx != TX - 1) || (AY == 2 && ly != TY - 1) || (AZ == 2 && lz != TZ - 1)) continue;
        Ft[c * T::SHELL + T::shell(2 * lx + AX, 2 * ly + AY, 2 * lz + AZ)] =
            a2_node_sum<TX, TY, TZ>(X, c, lx, ly, lz, AX, AY, AZ);
      }
  // publish: the barrier orders every thread's F stores before thread 0's gpu-scope
  // fence (cumulative), then the release store of the flag
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(flag + tile), "r"(epoch) : "memory");
  }
  if (threadIdx.x < 7) {
    const int o = threadIdx.x + 1;
    const int ttx = tx - (o & 1), tty = ty - ((o >> 1) & 1), ttz = tz - (o >> 2);
    if (ttx >= 0 && tty >= 0 && ttz >= 0) {
      const int* f = flag + (ttx + NTX * (tty + NTY * ttz));
      int v;
      while (true) {
        asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        if (v == epoch) break;
        __nanosleep(32);
      }
    }
  }
  __syncthreads();
  // Phase B: owned nodes (all A_d < 2, or A_d = 2 at the domain end): lower
  // neighbours' partials in ascending tile index, then the tile's own sum.
  const int kN = 2 * G.N;
  const int bx = 2 * TX * tx, by = 2 * TY * ty, bz = 2 * TZ * tz;
  const double* Fc = F + c * T::SHELL;
  // Straight-line, predicated code: every neighbour partial of every owned node is
  // loaded before any is summed (no serialised L2 round trips); absent terms are
  // +0.0, which leaves the fixed-order sum unchanged.
#pragma unroll
  for (int AZ = 0; AZ < 3; ++AZ)
#pragma unroll
    for (int AY = 0; AY < 3; ++AY)
#pragma unroll
      for (int AX = 0; AX < 3; ++AX) {
        const bool resp = !((AX == 2 && lx != TX - 1) || (AY == 2 && ly != TY - 1) || (AZ == 2 && lz != TZ - 1));
        const int nx = 2 * lx + AX, ny = 2 * ly + AY, nz = 2 * lz + AZ;
        const int gx = bx + nx, gy = by + ny, gz = bz + nz;
        const bool owned = resp && gx <= kN && gy <= kN && gz <= kN && !(AX == 2 && gx != kN) &&
                           !(AY == 2 && gy != kN) && !(AZ == 2 && gz != kN);
        const bool live = owned && (nomask || !node_bnd(gx, gy, gz, G.nn1));
        const bool lowx = nx == 0 && tx > 0, lowy = ny == 0 && ty > 0, lowz = nz == 0 && tz > 0;
        double f[7];
#pragma unroll
        for (int o = 0; o < 7; ++o) {  // neighbour (dx, dy, dz) in {-1, 0}^3 \ {0}, ascending tile index
          const int dz = (o < 4) ? -1 : 0, dy = ((o % 4) < 2) ? -1 : 0, dx = (o % 2 == 0) ? -1 : 0;
          const bool need = live && (dz == 0 || lowz) && (dy == 0 || lowy) && (dx == 0 || lowx);
          const int nt = (tx + dx) + NTX * ((ty + dy) + NTY * (tz + dz));
          f[o] = need ? __ldcg(Fc + (size_t)nt * 3 * T::SHELL +
                               T::shell(dx ? 2 * TX : nx, dy ? 2 * TY : ny, dz ? 2 * TZ : nz))
                      : 0.0;
        }
        const double own = live ? a2_node_sum<TX, TY, TZ>(X, c, lx, ly, lz, AX, AY, AZ) : 0.0;
        double acc = 0.0;
#pragma unroll
        for (int o = 0; o < 7; ++o) acc += f[o];
        acc += own;
        if (owned) y[c * G.n_nodes + node_id(gx, gy, gz, G.nn1)] = live ? acc : 0.0;
      }
}

}  // namespace wb
