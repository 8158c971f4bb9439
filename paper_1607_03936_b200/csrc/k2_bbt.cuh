// k2_bbt.cuh -- B and B^T for k = 2 (rows a6, a7), tiled through shared memory.
//
//   (B u)_{e,m}    = sB sum_{c,a} Bt2[c][a][m] u_c(node(e, a))
//   (B^T p)_c(g)   = sB sum_{e ∋ g} sum_m Bt2[c][a(e,g)][m] p_{e,m}
// (the element matrix c_Bt2 as in kernels_k2.cuh).
// Both are bound by HBM (each velocity value is read or written once): the
// generic thread-per-element / thread-per-node kernels gather through L1 with
// little reuse per load; here a CTA stages its tile once with coalesced
// cp.async rows and computes from shared memory.
#pragma once
#include "a2_tile.cuh"
#include "k2_fused.cuh"

namespace wb {

// ------------------------------------------------------------------ B
template <int TX, int TY, int TZ>
struct BTile2 {
  using L = UsL<TX, TY, TZ>;
  static constexpr int NE = TX * TY * TZ, NTH = 3 * NE;
  static constexpr size_t SMEM = sizeof(double) * (4 * L::NN + 12 * NE);  // u (3), xs box, partials
};

// component C of one element: qm[m] += sum_a Bt2[C][a][m] U(a), exact zeros skipped
template <int TX, int TY, int TZ, int C>
__device__ __forceinline__ void b2_comp(const double* __restrict__ Ub, double (&qm)[4]) {
  using L = UsL<TX, TY, TZ>;
#pragma unroll
  for (int a = 0; a < 27; ++a) {
    const int ax = a % 3, ay = (a / 3) % 3, az = a / 9;
    const double v = Ub[L::RSU * (ay + L::MY * az) + (ax == 1 ? TX + 1 : (ax >> 1))];
#pragma unroll
    for (int m = 0; m < 4; ++m)
      if (bt2_nz(C, a, m)) qm[m] = fma(c_Bt2[C][a][m], v, qm[m]);
  }
}

// One CTA per TX x TY x TZ element tile, thread per (element, component); the
// three component partials are summed in shared memory in the order c = 0, 1, 2.
// xs (optional): nodal scaling applied to u (no Dirichlet masking then, as in
// k_B); else Dirichlet nodes are zeroed unless nomask.  p[e*se + m*sm].
template <int TX, int TY, int TZ>
__global__ void __launch_bounds__(3 * TX * TY * TZ) k_B_tile2(const double* __restrict__ u,
                                                             const double* __restrict__ xs, double* __restrict__ p,
                                                             Geo G, double sB, int nomask, int64_t se, int64_t sm) {
  using L = UsL<TX, TY, TZ>;
  constexpr int NE = TX * TY * TZ, NTH = 3 * NE;
  extern __shared__ __align__(16) double smem_b2[];
  double* Us = smem_b2;
  double* Xb = Us + 3 * L::NN;
  double* Q = Xb + L::NN;
  const A2Tile t = a2_tile_of<TX, TY, TZ>(blockIdx.x, G);
  a2_stage_nodal<TX, TY, TZ, 3, NTH>(u, G.n_nodes, Us, t, G, xs ? 1 : nomask);
  if (xs) a2_stage_nodal<TX, TY, TZ, 1, NTH>(xs, 0, Xb, t, G, 1);
  cp_async_wait_all();
  __syncthreads();
  if (xs) {
    for (int i = threadIdx.x; i < 3 * L::NN; i += NTH) Us[i] *= Xb[i % L::NN];
    __syncthreads();
  }
  const int le = threadIdx.x % NE, c = threadIdx.x / NE;
  const int lx = le % TX, ly = (le / TX) % TY, lz = le / (TX * TY);
  const double* Ub = Us + c * L::NN + L::RSU * (2 * ly + L::MY * 2 * lz) + lx;
  double qm[4] = {0.0, 0.0, 0.0, 0.0};
  if (c == 0) b2_comp<TX, TY, TZ, 0>(Ub, qm);        // c is warp-uniform (NE % 32 == 0)
  else if (c == 1) b2_comp<TX, TY, TZ, 1>(Ub, qm);
  else b2_comp<TX, TY, TZ, 2>(Ub, qm);
#pragma unroll
  for (int m = 0; m < 4; ++m) Q[(c * 4 + m) * NE + le] = qm[m];
  __syncthreads();
  if (c == 0) {
    const int ex = TX * t.tx + lx, ey = TY * t.ty + ly, ez = TZ * t.tz + lz;
    if (ex < G.N && ey < G.N && ez < G.N) {
      const int64_t e = ex + (int64_t)G.N * (ey + (int64_t)G.N * ez);
#pragma unroll
      for (int m = 0; m < 4; ++m)
        p[e * se + m * sm] = sB * ((Q[m * NE + le] + Q[(4 + m) * NE + le]) + Q[(8 + m) * NE + le]);
    }
  }
}

// ------------------------------------------------------------------ B^T
// One CTA per NBX^3 node box, 256 threads.  The (NBX/2 + 1)^3 elements touching
// the box are staged (zero outside the mesh: an absent element adds +0.0, which
// leaves every sum unchanged); warp w takes node-parity class w, so the element
// structure of its nodes is compile-time.  Per axis: odd node -> element j+1
// (local 1); even node -> elements j (local 2) then j+1 (local 0), ascending --
// the order of k_BT_node2.
template <int NBX>
struct BTBox2 {
  static constexpr int NEB = NBX / 2 + 1, NPE = NEB * NEB * NEB;
};

template <int NBX, int RX, int RY, int RZ>
__device__ __forceinline__ void bt2_box(const double* __restrict__ Pe, int jx, int jy, int jz, double& t0,
                                        double& t1, double& t2) {
  constexpr int NEB = BTBox2<NBX>::NEB, NPE = BTBox2<NBX>::NPE;
#pragma unroll
  for (int iz = 0; iz < (RZ ? 1 : 2); ++iz) {
    const int lz = jz + (RZ ? 1 : iz), az = RZ ? 1 : (iz == 0 ? 2 : 0);
#pragma unroll
    for (int iy = 0; iy < (RY ? 1 : 2); ++iy) {
      const int ly = jy + (RY ? 1 : iy), ay = RY ? 1 : (iy == 0 ? 2 : 0);
#pragma unroll
      for (int ix = 0; ix < (RX ? 1 : 2); ++ix) {
        const int lx = jx + (RX ? 1 : ix), ax = RX ? 1 : (ix == 0 ? 2 : 0);
        const int le = lx + NEB * (ly + NEB * lz);
        const int a = ax + 3 * (ay + 3 * az);
        double pm[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) pm[m] = Pe[m * NPE + le];
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

// y[c][g] = sB * s[g] * (B^T p)_c(g)   (s = nodal scaling, or none); Dirichlet nodes 0 unless nomask
template <int NBX>
__global__ void __launch_bounds__(256) k_BT_box2(const double* __restrict__ p, const double* __restrict__ s,
                                                 double* __restrict__ y, Geo G, double sB, int nomask, int64_t se,
                                                 int64_t sm) {
  static_assert(NBX == 8, "8 parity classes x (4 x 4 x 4) nodes = 256 threads x 2 passes");
  constexpr int NEB = BTBox2<NBX>::NEB, NPE = BTBox2<NBX>::NPE;
  __shared__ double Pe[4 * NPE];
  const int nn1 = G.nn1, N = G.N;
  const int nb = (nn1 + NBX - 1) / NBX;
  const int bx = blockIdx.x % nb, by = (blockIdx.x / nb) % nb, bz = blockIdx.x / (nb * nb);
  const int ex0 = bx * (NBX / 2) - 1, ey0 = by * (NBX / 2) - 1, ez0 = bz * (NBX / 2) - 1;
  for (int i = threadIdx.x; i < NPE; i += 256) {
    const int lx = i % NEB, ly = (i / NEB) % NEB, lz = i / (NEB * NEB);
    const int ex = ex0 + lx, ey = ey0 + ly, ez = ez0 + lz;
    if (ex >= 0 && ey >= 0 && ez >= 0 && ex < N && ey < N && ez < N) {
      const int64_t e = ex + (int64_t)N * (ey + (int64_t)N * ez);
#pragma unroll
      for (int m = 0; m < 4; ++m) cp_async8(Pe + m * NPE + i, p + e * se + m * sm);
    } else {
#pragma unroll
      for (int m = 0; m < 4; ++m) Pe[m * NPE + i] = 0.0;
    }
  }
  cp_async_wait_all();
  __syncthreads();
  const int cls = threadIdx.x >> 5, lane = threadIdx.x & 31;  // class warp-uniform
  const int rx = cls & 1, ry = (cls >> 1) & 1, rz = cls >> 2;
  const int jx = lane & 3, jy = (lane >> 2) & 3;
  const int64_t nv = G.n_nodes;
#pragma unroll
  for (int pass = 0; pass < 2; ++pass) {
    const int jz = (lane >> 4) + 2 * pass;
    const int gx = bx * NBX + 2 * jx + rx, gy = by * NBX + 2 * jy + ry, gz = bz * NBX + 2 * jz + rz;
    if (gx >= nn1 || gy >= nn1 || gz >= nn1) continue;
    const int64_t g = node_id(gx, gy, gz, nn1);
    if (!nomask && node_bnd(gx, gy, gz, nn1)) {
      y[g] = 0.0; y[nv + g] = 0.0; y[2 * nv + g] = 0.0;
      continue;
    }
    double t0 = 0.0, t1 = 0.0, t2 = 0.0;
    switch (cls) {
      case 0: bt2_box<NBX, 0, 0, 0>(Pe, jx, jy, jz, t0, t1, t2); break;
      case 1: bt2_box<NBX, 1, 0, 0>(Pe, jx, jy, jz, t0, t1, t2); break;
      case 2: bt2_box<NBX, 0, 1, 0>(Pe, jx, jy, jz, t0, t1, t2); break;
      case 3: bt2_box<NBX, 1, 1, 0>(Pe, jx, jy, jz, t0, t1, t2); break;
      case 4: bt2_box<NBX, 0, 0, 1>(Pe, jx, jy, jz, t0, t1, t2); break;
      case 5: bt2_box<NBX, 1, 0, 1>(Pe, jx, jy, jz, t0, t1, t2); break;
      case 6: bt2_box<NBX, 0, 1, 1>(Pe, jx, jy, jz, t0, t1, t2); break;
      default: bt2_box<NBX, 1, 1, 1>(Pe, jx, jy, jz, t0, t1, t2); break;
    }
    const double f = s ? sB * s[g] : sB;
    y[g] = f * t0; y[nv + g] = f * t1; y[2 * nv + g] = f * t2;
  }
}

}  // namespace wb
