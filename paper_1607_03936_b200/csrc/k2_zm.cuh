// k2_zm.cuh -- the fused k = 2 Poisson operator of the PCG loop (rows a8, a9):
// p = z + beta p_old (direction update), q = K_w p = B X^-1 B^T p and the <p, q>
// partial, by NODE-OWNER threads that march along z.
//
// Operator (eq:wbfbt PAPER.md:436-454): t = B^T p at the velocity
// nodes, s = X o t (X = C_w^-1 or D_w^-1, one scalar per node for all 3 components),
// q = B s.  B_e[m,(c,a)] = sB * Bt2[c][a][m] (sB = -(h/2)^2, Bt2 = prod_d BD/BI tables).
//
// Thread mapping.  A CTA owns a column of TY x TX elements (y fastest) and a chunk of
// ZC element layers.  Thread (ly, lx), ly in [0, TY], lx in [0, TX], owns the 2 x 2 node
// columns gy in {2ey, 2ey+1}, gx in {2ex, 2ex+1} of element (ey, ex) = (ey0+ly, ex0+lx)
// ("lower-corner" ownership: every node of the tile's (2TY+1) x (2TX+1) node columns has
// exactly one owner; the threads ly = TY / lx = TX are the upper halo).  Its nodes touch
// the 2 x 2 element slots (ey-1, ey) x (ex-1, ex) of a layer; per axis the (slot, node)
// pairs are (e-1 -> node 2e: local a = 2), (e -> 2e: a = 0), (e -> 2e+1: a = 1).
//
// z march: step iz handles the node levels gz = 2(ez0+iz) (touching layers ez0+iz-1 and
// ez0+iz) and 2(ez0+iz)+1 (layer ez0+iz only), with the previous layer's p slots carried
// in registers.  Per step and thread: 27 (slot, node) pairs = the 27 local nodes of one
// element, each with the 12 (c, m) coefficients of the element matrix (exact zeros
// skipped at compile time, bt2_nz: 207 FMA for B^T, 207 for B).  The B partials of the
// previous layer's 4 slots are complete after the step; the 3 slots owned by other
// threads go through shared memory once (12 values per thread), and the owner sums
// them in a fixed order -> bitwise reproducible, no atomics.
//
// Staging: per layer one TMA box (TY+2) x (TX+2) x 4 modes of p_old and of z = Minv r
// (y-fastest PCG storage, PLay off = 1: the box's y start ey0 is even -> 16-byte
// aligned; hardware zero fill outside the mesh), 3-stage ring, mbarrier completion;
// the box is combined in place (p = z + beta p_old) once per layer.  X comes from a
// padded nodal copy (XZ, y fastest, rows of 2N+2, prescaled by sB^2) straight into
// registers (one 16-byte load per node pair).  Shared memory per CTA ~50 KB, so several
// CTAs share an SM.
#pragma once
#include <cuda.h>
#include "k2_fused.cuh"
#include "mbar.cuh"

namespace wb {

template <int TY, int TX>
struct ZMK {
  static constexpr int LY = TY + 1, LX = TX + 1;  // node-owner threads per column / row
  static constexpr int NT = LY * LX;
  static constexpr int NTH = (NT + 31) / 32 * 32;
  static constexpr int HY = TY + 2, HX = TX + 2;  // halo box (elements)
  static_assert(HY % 2 == 0 && TY % 2 == 0, "16-byte box rows, even y start");
  static constexpr int BOX = HY * HX * 4;          // doubles per box (4 modes)
  static constexpr unsigned BOXB = BOX * 8u;
  static constexpr int NST = 3;                    // TMA ring stages (layers)
  static constexpr size_t al(size_t b) { return (b + 1023) & ~(size_t)1023; }
  static constexpr size_t OFF_E = NST * 2 * al(BOXB);      // exchange buffer [3][4][NTH]
  static constexpr size_t OFF_B = OFF_E + al(3u * 4u * NTH * 8u);
  static constexpr size_t SMEM = OFF_B + 64 + 1024;         // + slack for 1024-byte base alignment
  __host__ __device__ static constexpr int bidx(int m, int hx, int hy) { return (m * HX + hx) * HY + hy; }
};

// local node index of (slot s, node n) along one axis: s = 0 is element e-1, s = 1 is e
__host__ __device__ constexpr int zm_a(int s, int n) { return s == 0 ? 2 : n; }
__host__ __device__ constexpr bool zm_conn(int s, int n) { return !(s == 0 && n == 1); }

// The per-step work of one thread, in two halves that keep few values live.
// Pp / Pc = p of the previous / current layer in the 4 (sy, sx) slots, X[nz][ny][nx]
// (prescaled by sB^2).
// Half A, node level nz = 0 (touches both layers): s0 = X o Bt2 p at its 4 nodes, and the
// B partials of the previous layer's slots Q0[sy][sx][m] += Bt2^T s0 -- Q0 is then complete.
__device__ __forceinline__ void zm_half_a(const double (&Pp)[2][2][4], const double (&Pc)[2][2][4],
                                          const double (&X)[2][2][2], double (&s0)[2][2][3],
                                          double (&Q0)[2][2][4]) {
#pragma unroll
  for (int ny = 0; ny < 2; ++ny)
#pragma unroll
    for (int nx = 0; nx < 2; ++nx) {
      // t = Bt2 p at this node, summed over the connected slots (z, y, x ascending)
      double t0 = 0.0, t1 = 0.0, t2 = 0.0;
#pragma unroll
      for (int sz = 0; sz < 2; ++sz)
#pragma unroll
        for (int sy = 0; sy < 2; ++sy)
#pragma unroll
          for (int sx = 0; sx < 2; ++sx) {
            if (!zm_conn(sy, ny) || !zm_conn(sx, nx)) continue;
            const int a = zm_a(sx, nx) + 3 * (zm_a(sy, ny) + 3 * zm_a(sz, 0));
#pragma unroll
            for (int m = 0; m < 4; ++m) {
              const double pv = sz ? Pc[sy][sx][m] : Pp[sy][sx][m];
              if (bt2_nz(0, a, m)) t0 = fma(c_Bt2[0][a][m], pv, t0);
              if (bt2_nz(1, a, m)) t1 = fma(c_Bt2[1][a][m], pv, t1);
              if (bt2_nz(2, a, m)) t2 = fma(c_Bt2[2][a][m], pv, t2);
            }
          }
      const double xs = X[0][ny][nx];
      s0[ny][nx][0] = t0 * xs; s0[ny][nx][1] = t1 * xs; s0[ny][nx][2] = t2 * xs;
      // previous layer's slots (sz = 0, local az = 2)
#pragma unroll
      for (int sy = 0; sy < 2; ++sy)
#pragma unroll
        for (int sx = 0; sx < 2; ++sx) {
          if (!zm_conn(sy, ny) || !zm_conn(sx, nx)) continue;
          const int a = zm_a(sx, nx) + 3 * (zm_a(sy, ny) + 3 * 2);
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            double acc = Q0[sy][sx][m];
            if (bt2_nz(0, a, m)) acc = fma(c_Bt2[0][a][m], s0[ny][nx][0], acc);
            if (bt2_nz(1, a, m)) acc = fma(c_Bt2[1][a][m], s0[ny][nx][1], acc);
            if (bt2_nz(2, a, m)) acc = fma(c_Bt2[2][a][m], s0[ny][nx][2], acc);
            Q0[sy][sx][m] = acc;
          }
        }
    }
}
// Half B: node level nz = 1 (current layer only, unless LAST: the upper-halo layer, whose
// own partials are not needed), then the current layer's partials Q1 from both levels
// (level 0 with local az = 0, level 1 with az = 1), in node order.
template <bool LAST>
__device__ __forceinline__ void zm_half_b(const double (&Pc)[2][2][4], const double (&X)[2][2][2],
                                          const double (&s0)[2][2][3], double (&Q1)[2][2][4]) {
  if constexpr (!LAST) {
#pragma unroll
  for (int sy = 0; sy < 2; ++sy)
#pragma unroll
    for (int sx = 0; sx < 2; ++sx)
#pragma unroll
      for (int m = 0; m < 4; ++m) Q1[sy][sx][m] = 0.0;
#pragma unroll
  for (int nz = 0; nz < 2; ++nz)
#pragma unroll
    for (int ny = 0; ny < 2; ++ny)
#pragma unroll
      for (int nx = 0; nx < 2; ++nx) {
        double s[3];
        if (nz == 0) {
          s[0] = s0[ny][nx][0]; s[1] = s0[ny][nx][1]; s[2] = s0[ny][nx][2];
        } else {
          double t0 = 0.0, t1 = 0.0, t2 = 0.0;
#pragma unroll
          for (int sy = 0; sy < 2; ++sy)
#pragma unroll
            for (int sx = 0; sx < 2; ++sx) {
              if (!zm_conn(sy, ny) || !zm_conn(sx, nx)) continue;
              const int a = zm_a(sx, nx) + 3 * (zm_a(sy, ny) + 3 * 1);
#pragma unroll
              for (int m = 0; m < 4; ++m) {
                if (bt2_nz(0, a, m)) t0 = fma(c_Bt2[0][a][m], Pc[sy][sx][m], t0);
                if (bt2_nz(1, a, m)) t1 = fma(c_Bt2[1][a][m], Pc[sy][sx][m], t1);
                if (bt2_nz(2, a, m)) t2 = fma(c_Bt2[2][a][m], Pc[sy][sx][m], t2);
              }
            }
          const double xs = X[1][ny][nx];
          s[0] = t0 * xs; s[1] = t1 * xs; s[2] = t2 * xs;
        }
#pragma unroll
        for (int sy = 0; sy < 2; ++sy)
#pragma unroll
          for (int sx = 0; sx < 2; ++sx) {
            if (!zm_conn(sy, ny) || !zm_conn(sx, nx)) continue;
            const int a = zm_a(sx, nx) + 3 * (zm_a(sy, ny) + 3 * nz);
#pragma unroll
            for (int m = 0; m < 4; ++m) {
              double acc = Q1[sy][sx][m];
              if (bt2_nz(0, a, m)) acc = fma(c_Bt2[0][a][m], s[0], acc);
              if (bt2_nz(1, a, m)) acc = fma(c_Bt2[1][a][m], s[1], acc);
              if (bt2_nz(2, a, m)) acc = fma(c_Bt2[2][a][m], s[2], acc);
              Q1[sy][sx][m] = acc;
            }
          }
      }
  }
}

// Same contract as k_K2_tma (mode 0: p = z, 1: p = z + beta p_old, 2: p = p_old as is,
// ctl / it / partials), one CTA per (column, z-chunk).
template <int TY, int TX, int MINB>
__global__ void __launch_bounds__(ZMK<TY, TX>::NTH, MINB)
    k_K2_zm(const __grid_constant__ CUtensorMap tm_pold, const __grid_constant__ CUtensorMap tm_z,
            const double* __restrict__ XZ, double* __restrict__ pnew, double* __restrict__ q, int N, int ZC,
            int mode, int it, int ctl, const double* __restrict__ rzp, int nrz, double* rz_hist,
            const double* pq_hist, int* stop, double* pqp, PLay L) {
  using K = ZMK<TY, TX>;
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sb = smraw;
  double* Ex = (double*)(sb + K::OFF_E);
  uint64_t* bar = (uint64_t*)(sb + K::OFF_B);
  auto pbox = [&](int st) { return (double*)(sb + (size_t)(2 * st) * K::al(K::BOXB)); };
  auto zbox = [&](int st) { return (double*)(sb + (size_t)(2 * st + 1) * K::al(K::BOXB)); };

  const int NTY = (N + TY - 1) / TY, NTX = (N + TX - 1) / TX;
  const int col = blockIdx.x % (NTY * NTX), chunk = blockIdx.x / (NTY * NTX);
  const int ey0 = TY * (col % NTY), ex0 = TX * (col / NTY);
  const int ez0 = ZC * chunk, ez1 = min(ez0 + ZC, N);
  const int NL = ez1 - ez0 + 2;  // layers ez0-1 .. ez1 (halo below and above)
  const int md = mode & 0xff;
  const bool needp = md != 0, needz = md != 2;
  const unsigned bytes = (needp ? K::BOXB : 0u) + (needz ? K::BOXB : 0u);
  auto issue = [&](int li) {  // layer ez0 - 1 + li into stage li % 3
    const int st = li % K::NST;
    mbar_expect_tx(&bar[st], bytes);
    if (needp) tma_load_4d(pbox(st), &tm_pold, ey0, ez0 - 1 + li, ex0 - 1, 0, &bar[st]);
    if (needz) tma_load_4d(zbox(st), &tm_z, ey0, ez0 - 1 + li, ex0 - 1, 0, &bar[st]);
  };
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < K::NST; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int li = 0; li < min(NL, K::NST); ++li) issue(li);
  }
  double beta = 0.0;
  if (ctl) {
    if (pcg_control<K::NTH>(it, rzp, nrz, rz_hist, pq_hist, stop, &beta)) {
      if (threadIdx.x == 0)  // drain the copies in flight before the CTA exits
        for (int li = 0; li < min(NL, K::NST); ++li) mbar_wait(&bar[li], 0);
      return;
    }
  } else if (md == 1) {
    beta = rz_hist[it] / rz_hist[it - 1];
  }
  __syncthreads();  // barrier init visible

  const int t = threadIdx.x;
  const bool act = t < K::NT;
  const int ly = t % K::LY, lx = t / K::LY;
  const int ey = ey0 + ly, ex = ex0 + lx;
  // owner of an element of the tile (stores q, p_new, adds to <p, q>)
  const bool own = act && ly < TY && lx < TX && ey < N && ex < N;
  const bool xin = act && ey <= N && ex <= N;  // node columns inside the padded X array
  const int RY = 2 * N + 2;
  const int64_t RXY = (int64_t)RY * RY;
  const double* xcol = XZ + (int64_t)(2 * ex) * RY + 2 * ey;
  const int tx1 = ly + K::LY * (lx + 1), ty1 = (ly + 1) + K::LY * lx, txy = (ly + 1) + K::LY * (lx + 1);

  double Pp[2][2][4], Pc[2][2][4];
  double Q0[2][2][4], Q1[2][2][4];  // B partials of the previous / current layer's slots
  double dot = 0.0;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int m = 0; m < 4; ++m) { Pp[i][j][m] = 0.0; Q1[i][j][m] = 0.0; }

  for (int li = 0; li < NL; ++li) {
    const int st = li % K::NST;
    const int lay = ez0 - 1 + li;  // the current layer
    const bool last = li == NL - 1;
    mbar_wait(&bar[st], (unsigned)((li / K::NST) & 1));
    double* pb = pbox(st);
    const double* zb = zbox(st);
    if (md == 1) {  // p = z + beta p_old, in place
      for (int i = t; i < K::BOX / 2; i += K::NTH) {
        double2 pv = reinterpret_cast<double2*>(pb)[i];
        const double2 zv = reinterpret_cast<const double2*>(zb)[i];
        pv.x = fma(beta, pv.x, zv.x); pv.y = fma(beta, pv.y, zv.y);
        reinterpret_cast<double2*>(pb)[i] = pv;
      }
      __syncthreads();
    }
    const double* src = md == 0 ? zb : pb;
    if (act) {
#pragma unroll
      for (int sy = 0; sy < 2; ++sy)
#pragma unroll
        for (int sx = 0; sx < 2; ++sx)
#pragma unroll
          for (int m = 0; m < 4; ++m) Pc[sy][sx][m] = src[K::bidx(m, lx + sx, ly + sy)];
    }
    // X of this step's nodes (levels 2 lay, 2 lay + 1): loaded once the box has arrived
    double X[2][2][2];
    if (li > 0 && xin) {
#pragma unroll
      for (int nz = 0; nz < 2; ++nz)
#pragma unroll
        for (int nx = 0; nx < 2; ++nx) {
          const double2 v = __ldg(reinterpret_cast<const double2*>(xcol + (int64_t)(2 * lay + nz) * RXY + nx * RY));
          X[nz][0][nx] = v.x; X[nz][1][nx] = v.y;
        }
    } else {
#pragma unroll
      for (int nz = 0; nz < 2; ++nz)
#pragma unroll
        for (int ny = 0; ny < 2; ++ny)
#pragma unroll
          for (int nx = 0; nx < 2; ++nx) X[nz][ny][nx] = 0.0;
    }
    // own p_new of the current layer (layers of the chunk only)
    if (md != 2 && own && lay >= ez0 && lay < ez1) {
#pragma unroll
      for (int m = 0; m < 4; ++m) pnew[L.at(m, ex, ey, lay)] = Pc[1][1][m];
    }
    // Q0 <- the carried partials of the previous layer (from the last step's half B)
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int m = 0; m < 4; ++m) Q0[i][j][m] = Q1[i][j][m];
    double s0[2][2][3];
    if (li > 0 && act) zm_half_a(Pp, Pc, X, s0, Q0);
    // Q0 now holds the complete partials of layer lay - 1 (slots (sy, sx)); hand the
    // three slots owned by other threads over, the owner sums in a fixed order
    const bool xch = li >= 2;  // layer lay - 1 >= ez0
    if (md != 1) __syncthreads();  // the previous step's exchange reads are done (mode 1: the combine barrier)
    if (xch && act) {
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        Ex[(0 * 4 + m) * K::NTH + t] = Q0[1][0][m];  // -> thread (ly, lx - 1)
        Ex[(1 * 4 + m) * K::NTH + t] = Q0[0][1][m];  // -> thread (ly - 1, lx)
        Ex[(2 * 4 + m) * K::NTH + t] = Q0[0][0][m];  // -> thread (ly - 1, lx - 1)
      }
    }
    if (li > 0 && act) {
      if (last) zm_half_b<true>(Pc, X, s0, Q1);
      else zm_half_b<false>(Pc, X, s0, Q1);
    }
    __syncthreads();  // exchange visible; every thread has read this stage's box
    if (threadIdx.x == 0 && li + K::NST < NL) {
      fence_proxy_async();
      issue(li + K::NST);
    }
    if (xch && own) {
      const int lz = lay - 1;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        double v = Q0[1][1][m];
        v += Ex[(0 * 4 + m) * K::NTH + tx1];
        v += Ex[(1 * 4 + m) * K::NTH + ty1];
        v += Ex[(2 * 4 + m) * K::NTH + txy];
        q[L.at(m, ex, ey, lz)] = v;
        dot = fma(Pp[1][1][m], v, dot);
      }
    }
    // roll: the current layer's slots become the previous ones
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int m = 0; m < 4; ++m) Pp[i][j][m] = Pc[i][j][m];
  }
  store_partial<K::NTH>(dot, pqp);
}

// XZ = sB^2 X on the padded nodal grid [gz][gx][gy], rows of 2N+2 (zero pads): the
// node-owner kernel's view of C_w^-1 / D_w^-1
__global__ void k_xz_build(const double* __restrict__ X, double* __restrict__ XZ, int N, double scale) {
  const int R = 2 * N + 2, nn1 = 2 * N + 1;
  const int64_t n = (int64_t)R * R * R;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int gy = (int)(i % R), gx = (int)((i / R) % R), gz = (int)(i / ((int64_t)R * R));
    XZ[i] = (gx < nn1 && gy < nn1 && gz < nn1) ? scale * X[node_id(gx, gy, gz, nn1)] : 0.0;
  }
}

}  // namespace wb
