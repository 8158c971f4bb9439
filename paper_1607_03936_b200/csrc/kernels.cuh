// kernels.cuh -- sm_100a FP64 kernels of the wBFBT hot path.
//
// Notation follows SURVEY.md Sec. 8 / DESIGN.md: N elements per axis, order k
// (n1 = k+1 nodes and Gauss points per axis), n_q = n1^3, n_m = C(k+2,3).
// Every reduction is fixed-order (no floating-point atomics): results are
// bitwise reproducible run to run.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "tables.h"

namespace wb {

__constant__ Tab c_tab[3];  // k = 2, 3, 4
#define TB(K) (c_tab[(K)-2])

struct Geo {
  int N, k, nn1;     // nn1 = kN + 1 nodes per axis
  int64_t n_el, n_nodes, n_p;
  // slab contexts (slab_dd.cuh): bit 0 / 1 = the z-lo / z-hi face is shared with a neighbouring
  // rank, i.e. not part of the global boundary (read by the lumping kernels' a_l / a_r test only)
  int zopen = 0;
};

// Storage of the mode-major PCG vectors (x, r, p, q, z, Minv): entry (m, e) of element
// e = ex + N (ey + N ez) at  m sm + ex sx + ez sz + (ey + off) sy.  Default (off = 0):
// sm = n_el, sx = 1, sy = N, sz = N^2, i.e. m n_el + e.  The TMA Poisson kernel's contexts
// store y fastest with one zero pad at each end of every y column (off = 1, sy = 1,
// sz = N + 2, sx = N (N + 2), sm = N^2 (N + 2)): its halo boxes then land in the pencil
// layout.  n = storage length (4 sm for k = 2); pads stay 0 (every update maps 0 to 0).
struct PLay {
  int64_t sm, sx, sy, sz, n;
  int off;
  __host__ __device__ int64_t at(int m, int ex, int ey, int ez) const {
    return m * sm + ex * sx + ez * sz + (ey + off) * sy;
  }
  __host__ __device__ int64_t at(int m, int64_t e, int N) const {
    const int ex = (int)(e % N), ey = (int)((e / N) % N), ez = (int)(e / ((int64_t)N * N));
    return at(m, ex, ey, ez);
  }
};

template <int K> struct Ord {
  static constexpr int n1 = K + 1, NQ = n1 * n1 * n1, NM = K * (K + 1) * (K + 2) / 6;
};

__device__ __forceinline__ bool node_bnd(int gx, int gy, int gz, int nn1) {
  return gx == 0 || gy == 0 || gz == 0 || gx == nn1 - 1 || gy == nn1 - 1 || gz == nn1 - 1;
}
__device__ __forceinline__ int64_t node_id(int gx, int gy, int gz, int nn1) {
  return (int64_t)gx + (int64_t)nn1 * ((int64_t)gy + (int64_t)nn1 * gz);
}
__device__ __forceinline__ void elem_xyz(int64_t e, int N, int& ex, int& ey, int& ez) {
  ex = (int)(e % N);
  int64_t t = e / N;
  ey = (int)(t % N);
  ez = (int)(t / N);
}

// ------------------------------------------------------------------ reductions
// Block sum with a fixed shuffle tree, then "last block done": every block
// writes its partial, the last block to arrive sums all partials in a fixed
// order.  Returns true in thread 0 of the last block, with *total set.
template <int BS>
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double sw[BS / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sw[w] = v;
  __syncthreads();
  double s = 0.0;
  if (w == 0) {
    s = (l < BS / 32) ? sw[l] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  }
  __syncthreads();
  return s;  // valid in thread 0
}

template <int BS>
__device__ __forceinline__ bool grid_sum(double v, double* partial, unsigned* counter, double* total) {
  __shared__ bool s_last;
  double s = block_sum<BS>(v);
  if (threadIdx.x == 0) {
    partial[blockIdx.x] = s;
    __threadfence();
    unsigned t = atomicAdd(counter, 1u);
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
  double a = 0.0;
  for (unsigned i = threadIdx.x; i < gridDim.x; i += BS) a += __ldcg(partial + i);
  double tot = block_sum<BS>(a);
  if (threadIdx.x == 0) {
    *total = tot;
    *counter = 0u;
  }
  return threadIdx.x == 0;
}

// Deferred reductions: a kernel stores one partial per block (no fence, no
// atomics) and every block of the NEXT kernel sums all of them in the same
// fixed order (strided per thread, then the fixed shuffle tree), so all blocks
// agree bitwise and no kernel ends with a grid-wide tail.
template <int BS>
__device__ __forceinline__ double sum_partials(const double* __restrict__ part, int n) {
  __shared__ double s_tot;
  double a = 0.0;
  for (int i = threadIdx.x; i < n; i += BS) a += part[i];
  a = block_sum<BS>(a);
  if (threadIdx.x == 0) s_tot = a;
  __syncthreads();
  const double t = s_tot;
  __syncthreads();
  return t;
}
template <int BS>
__device__ __forceinline__ void store_partial(double v, double* part) {
  v = block_sum<BS>(v);
  if (threadIdx.x == 0) part[blockIdx.x] = v;
}

// max |v| over the grid (same last-block pattern)
template <int BS>
__device__ __forceinline__ double block_max(double v) {
  __shared__ double sw[BS / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sw[w] = v;
  __syncthreads();
  double s = 0.0;
  if (w == 0) {
    s = (l < BS / 32) ? sw[l] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s = fmax(s, __shfl_down_sync(0xffffffffu, s, o));
  }
  __syncthreads();
  return s;
}

template <int BS>
__global__ void __launch_bounds__(BS) k_absmax(const double* __restrict__ v, int64_t n, double* partial,
                                               unsigned* counter, double* total) {
  __shared__ bool s_last;
  double m = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * BS + threadIdx.x; i < n; i += (int64_t)gridDim.x * BS) m = fmax(m, fabs(v[i]));
  m = block_max<BS>(m);
  if (threadIdx.x == 0) {
    partial[blockIdx.x] = m;
    __threadfence();
    s_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  double a = 0.0;
  for (unsigned i = threadIdx.x; i < gridDim.x; i += BS) a = fmax(a, __ldcg(partial + i));
  a = block_max<BS>(a);
  if (threadIdx.x == 0) { *total = a; *counter = 0u; }
}

// Jacobi preconditioner with the pseudo-inverse of diag K (R11):
// entries that vanish up to rounding, |d| <= 1e-13 max|d| (a numerically zero
// row of K, e.g. the constant mode on the N = 1 mesh), get Minv = 0.
// d element-major (ABI layout), minv mode-major (PCG layout): minv[m*ne + e].
__global__ void k_minv(const double* __restrict__ d, double* __restrict__ minv, int64_t ne, int nm,
                       const double* __restrict__ dmax, PLay L, int N) {
  const double thr = 1e-13 * *dmax;
  const int64_t n = ne * nm;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = i / ne, e = i % ne;
    const double v = d[e * nm + m];
    minv[L.at((int)m, e, N)] = fabs(v) > thr ? 1.0 / v : 0.0;
  }
}

// ------------------------------------------------------------------ row a1
template <int K>
__global__ void k_dofmap(int64_t* map, Geo G) {
  constexpr int n1 = K + 1, NQ = Ord<K>::NQ;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= G.n_el * NQ) return;
  int64_t e = i / NQ;
  int a = (int)(i % NQ);
  int ex, ey, ez;
  elem_xyz(e, G.N, ex, ey, ez);
  map[i] = node_id(K * ex + a % n1, K * ey + (a / n1) % n1, K * ez + a / (n1 * n1), G.nn1);
}

__global__ void k_bmask(uint8_t* mask, Geo G) {
  int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= G.n_nodes) return;
  int gx = (int)(g % G.nn1), gy = (int)((g / G.nn1) % G.nn1), gz = (int)(g / ((int64_t)G.nn1 * G.nn1));
  uint8_t b = node_bnd(gx, gy, gz, G.nn1) ? 1 : 0;
  mask[g] = b;
  mask[G.n_nodes + g] = b;
  mask[2 * G.n_nodes + g] = b;
}

// Element-local velocity buffer E of the generic path (k = 3, 4: A, B^T element parts ->
// k_gather).  Layout [c][a][e] (element fastest): the producers' element-consecutive
// threads store contiguous words.  (Measured at C4: the [c][e][a] layout, WB_E_AFAST 1,
// speeds the gather up 33.7 -> 27.6 us but slows the B^T element part 11.7 -> 34.4 us.)
#ifndef WB_E_AFAST
#define WB_E_AFAST 0
#endif
template <int K>
__device__ __forceinline__ int64_t eix(int c, int a, int64_t e, int64_t n_el) {
  constexpr int NQ = (K + 1) * (K + 1) * (K + 1);
  return WB_E_AFAST ? ((int64_t)c * n_el + e) * NQ + a : (int64_t)(c * NQ + a) * n_el + e;
}

// ------------------------------------------------------------------ node gather
// y[c][g] = s[g] * sum_{e ni g} E[c][a(e,g)][e], elements in ascending index
// (the order of the oracle's element-ordered scatter).  Boundary nodes -> 0
// unless nomask.  E layout: eix<K> (above).
template <int K>
__global__ void k_gather(const double* __restrict__ E, const double* __restrict__ s,
                         double* __restrict__ y, Geo G, int nomask) {
  constexpr int n1 = K + 1;
  int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= G.n_nodes) return;
  const int nn1 = G.nn1;
  int gx = (int)(g % nn1), gy = (int)((g / nn1) % nn1), gz = (int)(g / ((int64_t)nn1 * nn1));
  if (!nomask && node_bnd(gx, gy, gz, nn1)) {
    y[g] = 0.0; y[G.n_nodes + g] = 0.0; y[2 * G.n_nodes + g] = 0.0;
    return;
  }
  int pe[3][2], pa[3][2], pc[3];
  const int gg[3] = {gx, gy, gz};
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    int q = gg[d] / K, r = gg[d] % K;
    pc[d] = 0;
    if (r != 0) { pe[d][0] = q; pa[d][0] = r; pc[d] = 1; }
    else {
      if (q - 1 >= 0) { pe[d][pc[d]] = q - 1; pa[d][pc[d]] = K; pc[d]++; }
      if (q < G.N) { pe[d][pc[d]] = q; pa[d][pc[d]] = 0; pc[d]++; }
    }
  }
  // all (up to 8 x 3) loads issued before the sums: fixed 2 x 2 x 2 trip counts, the
  // absent terms predicated off; summed in ascending element order as before
  double t0[8], t1[8], t2[8];
#pragma unroll
  for (int iz = 0; iz < 2; ++iz)
#pragma unroll
    for (int iy = 0; iy < 2; ++iy)
#pragma unroll
      for (int ix = 0; ix < 2; ++ix) {
        const int k = (iz * 2 + iy) * 2 + ix;
        t0[k] = t1[k] = t2[k] = 0.0;
        if (iz < pc[2] && iy < pc[1] && ix < pc[0]) {
          const int64_t e = pe[0][ix] + (int64_t)G.N * (pe[1][iy] + (int64_t)G.N * pe[2][iz]);
          const int a = pa[0][ix] + n1 * (pa[1][iy] + n1 * pa[2][iz]);
          t0[k] = __ldg(E + eix<K>(0, a, e, G.n_el));
          t1[k] = __ldg(E + eix<K>(1, a, e, G.n_el));
          t2[k] = __ldg(E + eix<K>(2, a, e, G.n_el));
        }
      }
  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
#pragma unroll
  for (int iz = 0; iz < 2; ++iz)
#pragma unroll
    for (int iy = 0; iy < 2; ++iy)
#pragma unroll
      for (int ix = 0; ix < 2; ++ix)
        if (iz < pc[2] && iy < pc[1] && ix < pc[0]) {
          const int k = (iz * 2 + iy) * 2 + ix;
          acc0 += t0[k]; acc1 += t1[k]; acc2 += t2[k];
        }
  double sc = s ? s[g] : 1.0;
  if (s) { acc0 *= sc; acc1 *= sc; acc2 *= sc; }
  y[g] = acc0; y[G.n_nodes + g] = acc1; y[2 * G.n_nodes + g] = acc2;
}

// ------------------------------------------------------------------ row a6: B
// p_{e,m} = sB * sum_c sum_a prod_d M_cd[m_d][a_d] (X o u)_c[g(e,a)],
// M_cd = BD if d == c else BI, sB = -(2/h) detJ = -h^2/4  (B u := -div u,
// PAPER.md:962).  Sum-factorised per component: x, then y, then z.
// Optional fused dot: partial <p_out, dv>  (PCG <p, K p>).
template <int K, int BS>
__global__ void __launch_bounds__(BS) k_B(const double* __restrict__ u, const double* __restrict__ xs,
                                          double* __restrict__ p, Geo G, double sB, int nomask,
                                          const int* __restrict__ stop, const double* __restrict__ dv,
                                          double* partial, unsigned* counter, double* total, int64_t se,
                                          int64_t sm) {
  // output layout p[e*se + m*sm]: (NM, 1) element-major (ABI), (1, n_el) mode-major (PCG)
  constexpr int n1 = K + 1, NM = Ord<K>::NM;
  if (stop && *stop) return;
  const int64_t e = (int64_t)blockIdx.x * BS + threadIdx.x;
  const bool valid = e < G.n_el;
  int ex = 0, ey = 0, ez = 0;
  if (valid) elem_xyz(e, G.N, ex, ey, ez);
  double Z[NM];
#pragma unroll
  for (int m = 0; m < NM; ++m) Z[m] = 0.0;
  if (valid) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
#pragma unroll
      for (int az = 0; az < n1; ++az) {
        double Y[K][K];
#pragma unroll
        for (int i = 0; i < K; ++i)
#pragma unroll
          for (int j = 0; j < K; ++j) Y[i][j] = 0.0;
#pragma unroll
        for (int ay = 0; ay < n1; ++ay) {
          double v[n1];
          const int gy = K * ey + ay, gz = K * ez + az;
#pragma unroll
          for (int ax = 0; ax < n1; ++ax) {
            const int gx = K * ex + ax;
            const int64_t g = node_id(gx, gy, gz, G.nn1);
            double val = u[c * G.n_nodes + g];
            if (xs) val *= xs[g];
            else if (!nomask && node_bnd(gx, gy, gz, G.nn1)) val = 0.0;
            v[ax] = val;
          }
          double X[K];
#pragma unroll
          for (int m1 = 0; m1 < K; ++m1) {
            double t = 0.0;
#pragma unroll
            for (int ax = 0; ax < n1; ++ax) t = fma(c == 0 ? TB(K).BD[m1][ax] : TB(K).BI[m1][ax], v[ax], t);
            X[m1] = t;
          }
#pragma unroll
          for (int m1 = 0; m1 < K; ++m1)
#pragma unroll
            for (int m2 = 0; m2 < K - m1; ++m2)
              Y[m1][m2] = fma(c == 1 ? TB(K).BD[m2][ay] : TB(K).BI[m2][ay], X[m1], Y[m1][m2]);
        }
        int m = 0;
#pragma unroll
        for (int d = 0; d < K; ++d)
#pragma unroll
          for (int m3 = 0; m3 <= d; ++m3)
#pragma unroll
            for (int m2 = 0; m2 <= d - m3; ++m2) {
              const int m1 = d - m2 - m3;
              Z[m] = fma(c == 2 ? TB(K).BD[m3][az] : TB(K).BI[m3][az], Y[m1][m2], Z[m]);
              ++m;
            }
      }
    }
  }
  double dot = 0.0;
  if (valid) {
#pragma unroll
    for (int m = 0; m < NM; ++m) {
      const double o = sB * Z[m];
      p[e * se + m * sm] = o;
      if (dv) dot = fma(o, dv[e * se + m * sm], dot);
    }
  }
  if (partial) store_partial<BS>(dot, partial);  // deferred: summed by k_pcg_upd
  (void)counter; (void)total;
}

// Same B with EPB elements per block and one thread per (element, component c, z-node
// az): the thread contracts its (ax, ay) plane to Y[m1][m2] and parks it in shared
// memory; thread (element, m) then runs the z-contraction over (c, az) in the order of
// k_B (c outer, az inner, the same fma chain), so the two kernels agree bit for bit.
// 3(K+1) times the threads of k_B: at k = 4 (C4, 13.8k elements) k_B fills a third of
// the SMs with one warp each.  Dot partials (dv) as k_B, one per block.
template <int K, int EPB>
struct BSplit {
  static constexpr int NT = (EPB * 3 * (K + 1) + 31) / 32 * 32;  // whole warps (block_sum)
};
template <int K, int EPB>
__global__ void __launch_bounds__(BSplit<K, EPB>::NT) k_B_split(const double* __restrict__ u,
                                                              const double* __restrict__ xs, double* __restrict__ p,
                                                              Geo G, double sB, int nomask,
                                                              const int* __restrict__ stop,
                                                              const double* __restrict__ dv, double* partial,
                                                              int64_t se, int64_t sm) {
  constexpr int n1 = K + 1, NM = Ord<K>::NM, NY = K * (K + 1) / 2, NT = BSplit<K, EPB>::NT;
  __shared__ double Ys[EPB][3 * n1][NY];
  if (stop && *stop) return;
  const int el = threadIdx.x % EPB, slab = threadIdx.x / EPB;  // slab = c * n1 + az
  const int c = slab / n1, az = slab % n1;
  const int64_t e = (int64_t)blockIdx.x * EPB + el;
  if (slab < 3 * n1 && e < G.n_el) {
    int ex, ey, ez;
    elem_xyz(e, G.N, ex, ey, ez);
    double Y[NY];
#pragma unroll
    for (int i = 0; i < NY; ++i) Y[i] = 0.0;
    const int gz = K * ez + az;
#pragma unroll
    for (int ay = 0; ay < n1; ++ay) {
      const int gy = K * ey + ay;
      double v[n1];
#pragma unroll
      for (int ax = 0; ax < n1; ++ax) {
        const int gx = K * ex + ax;
        const int64_t g = node_id(gx, gy, gz, G.nn1);
        double val = u[c * G.n_nodes + g];
        if (xs) val *= xs[g];
        else if (!nomask && node_bnd(gx, gy, gz, G.nn1)) val = 0.0;
        v[ax] = val;
      }
      double X[K];
#pragma unroll
      for (int m1 = 0; m1 < K; ++m1) {
        double t = 0.0;
#pragma unroll
        for (int ax = 0; ax < n1; ++ax) t = fma(c == 0 ? TB(K).BD[m1][ax] : TB(K).BI[m1][ax], v[ax], t);
        X[m1] = t;
      }
      int i = 0;
#pragma unroll
      for (int m1 = 0; m1 < K; ++m1)
#pragma unroll
        for (int m2 = 0; m2 < K - m1; ++m2, ++i)
          Y[i] = fma(c == 1 ? TB(K).BD[m2][ay] : TB(K).BI[m2][ay], X[m1], Y[i]);
    }
#pragma unroll
    for (int i = 0; i < NY; ++i) Ys[el][slab][i] = Y[i];
  }
  __syncthreads();
  double dot = 0.0;
  for (int item = threadIdx.x; item < EPB * NM; item += NT) {
    const int el2 = item % EPB, m = item / EPB;
    const int64_t e2 = (int64_t)blockIdx.x * EPB + el2;
    if (e2 >= G.n_el) continue;
    // mode m -> (m1, m2, m3) in k_B's enumeration (degree d, then m3, then m2)
    int d = 0, rem = m;
    while (rem >= (d + 1) * (d + 2) / 2) { rem -= (d + 1) * (d + 2) / 2; ++d; }
    int m3 = 0;
    while (rem >= d - m3 + 1) { rem -= d - m3 + 1; ++m3; }
    const int m2 = rem, m1 = d - m2 - m3;
    const int yi = m1 * K - m1 * (m1 - 1) / 2 + m2;  // index of Y[m1][m2] in the packed order
    double Z = 0.0;
    for (int cc = 0; cc < 3; ++cc)
      for (int z = 0; z < n1; ++z)
        Z = fma(cc == 2 ? TB(K).BD[m3][z] : TB(K).BI[m3][z], Ys[el2][cc * n1 + z][yi], Z);
    const double o = sB * Z;
    p[e2 * se + m * sm] = o;
    if (dv) dot = fma(o, dv[e2 * se + m * sm], dot);
  }
  if (partial) store_partial<NT>(dot, partial);
}

// ------------------------------------------------------------------ row a7: B^T (element part)
// E[c][a][e] = sB * sum_m prod_d M_cd[m_d][a_d] p_{e,m}
template <int K>
__global__ void k_BT_elem(const double* __restrict__ p, double* __restrict__ E, Geo G, double sB,
                          const int* __restrict__ stop, int64_t se, int64_t sm) {
  constexpr int n1 = K + 1;
  if (stop && *stop) return;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= G.n_el) return;
  double P[K][K][K];  // P[m1][m2][m3] (only m1+m2+m3 <= K-1 used)
  {
    int m = 0;
#pragma unroll
    for (int d = 0; d < K; ++d)
#pragma unroll
      for (int m3 = 0; m3 <= d; ++m3)
#pragma unroll
        for (int m2 = 0; m2 <= d - m3; ++m2) {
          P[d - m2 - m3][m2][m3] = p[e * se + m * sm];
          ++m;
        }
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) {
#pragma unroll
    for (int az = 0; az < n1; ++az) {
      double Zt[K][K];
#pragma unroll
      for (int m1 = 0; m1 < K; ++m1)
#pragma unroll
        for (int m2 = 0; m2 < K - m1; ++m2) {
          double t = 0.0;
#pragma unroll
          for (int m3 = 0; m3 < K - m1 - m2; ++m3)
            t = fma(c == 2 ? TB(K).BD[m3][az] : TB(K).BI[m3][az], P[m1][m2][m3], t);
          Zt[m1][m2] = t;
        }
#pragma unroll
      for (int ay = 0; ay < n1; ++ay) {
        double Yt[K];
#pragma unroll
        for (int m1 = 0; m1 < K; ++m1) {
          double t = 0.0;
#pragma unroll
          for (int m2 = 0; m2 < K - m1; ++m2)
            t = fma(c == 1 ? TB(K).BD[m2][ay] : TB(K).BI[m2][ay], Zt[m1][m2], t);
          Yt[m1] = t;
        }
#pragma unroll
        for (int ax = 0; ax < n1; ++ax) {
          double t = 0.0;
#pragma unroll
          for (int m1 = 0; m1 < K; ++m1) t = fma(c == 0 ? TB(K).BD[m1][ax] : TB(K).BI[m1][ax], Yt[m1], t);
          const int a = ax + n1 * (ay + n1 * az);
          E[eix<K>(c, a, e, G.n_el)] = sB * t;
        }
      }
    }
  }
}

// Same element part of B^T with one thread per (element, component c, z-node az),
// element fastest: the body of k_BT_elem for one (c, az), so the outputs agree bit for
// bit; 3(K+1) times its threads (k = 3, 4).
template <int K>
__global__ void __launch_bounds__(256) k_BT_split(const double* __restrict__ p, double* __restrict__ E, Geo G,
                                                  double sB, const int* __restrict__ stop, int64_t se, int64_t sm) {
  constexpr int n1 = K + 1;
  if (stop && *stop) return;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= G.n_el * 3 * n1) return;
  const int64_t e = idx % G.n_el;
  const int slab = (int)(idx / G.n_el), c = slab / n1, az = slab % n1;
  double P[K][K][K];
  {
    int m = 0;
#pragma unroll
    for (int d = 0; d < K; ++d)
#pragma unroll
      for (int m3 = 0; m3 <= d; ++m3)
#pragma unroll
        for (int m2 = 0; m2 <= d - m3; ++m2) {
          P[d - m2 - m3][m2][m3] = __ldg(p + e * se + m * sm);
          ++m;
        }
  }
  double Zt[K][K];
#pragma unroll
  for (int m1 = 0; m1 < K; ++m1)
#pragma unroll
    for (int m2 = 0; m2 < K - m1; ++m2) {
      double t = 0.0;
#pragma unroll
      for (int m3 = 0; m3 < K - m1 - m2; ++m3)
        t = fma(c == 2 ? TB(K).BD[m3][az] : TB(K).BI[m3][az], P[m1][m2][m3], t);
      Zt[m1][m2] = t;
    }
#pragma unroll
  for (int ay = 0; ay < n1; ++ay) {
    double Yt[K];
#pragma unroll
    for (int m1 = 0; m1 < K; ++m1) {
      double t = 0.0;
#pragma unroll
      for (int m2 = 0; m2 < K - m1; ++m2) t = fma(c == 1 ? TB(K).BD[m2][ay] : TB(K).BI[m2][ay], Zt[m1][m2], t);
      Yt[m1] = t;
    }
#pragma unroll
    for (int ax = 0; ax < n1; ++ax) {
      double t = 0.0;
#pragma unroll
      for (int m1 = 0; m1 < K; ++m1) t = fma(c == 0 ? TB(K).BD[m1][ax] : TB(K).BI[m1][ax], Yt[m1], t);
      const int a = ax + n1 * (ay + n1 * az);
      E[eix<K>(c, a, e, G.n_el)] = sB * t;
    }
  }
}

// ------------------------------------------------------------------ row a5: A(mu) (generic slice kernel, k = 3, 4)
// NE elements per block, n1 x n1 threads per element; the thread (a, b) owns
// one pencil per pass and the third index is looped in registers; the passes
// exchange through shared memory.  Output: element-local E[c][a][e] (gathered by
// k_gather).  Same operator as the k = 2 tile kernel (a2_tile.cuh):
// y_{c,a} = int 2 mu eps(u):eps(phi_a e_c).
template <int K, int NE>
__global__ void __launch_bounds__(NE*(K + 1) * (K + 1)) k_A_slice(const double* __restrict__ mut,
                                                                  const double* __restrict__ u,
                                                                  double* __restrict__ E, Geo G, int nomask) {
  constexpr int n1 = K + 1, NQ = Ord<K>::NQ, P = n1 * n1;
  extern __shared__ double sm[];
  const int le = threadIdx.x / P, t = threadIdx.x % P, ta = t % n1, tb = t / n1;
  const int64_t e = (int64_t)blockIdx.x * NE + le;
  const bool valid = e < G.n_el;
  // three 3 NQ buffers per element, reused by liveness (X1: A0, GX, A1'; X2: A1, A0'; X3: GY)
  double* X1 = sm + (size_t)le * 9 * NQ;
  double* X2 = X1 + 3 * NQ;
  double* X3 = X2 + 3 * NQ;
#define IX(c, z, y, x) ((c)*NQ + ((z)*n1 + (y)) * n1 + (x))
  int ex = 0, ey = 0, ez = 0;
  if (valid) elem_xyz(e, G.N, ex, ey, ez);
  // S1 load: thread (x = ta, y = tb)
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int z = 0; z < n1; ++z) {
      const int gx = K * ex + ta, gy = K * ey + tb, gz = K * ez + z;
      double v = 0.0;
      if (valid && (nomask || !node_bnd(gx, gy, gz, G.nn1))) v = u[c * G.n_nodes + node_id(gx, gy, gz, G.nn1)];
      X1[IX(c, z, tb, ta)] = v;
    }
  __syncthreads();
  // S2 x-interp: thread (y = ta, z = tb)
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double v[n1];
#pragma unroll
    for (int j = 0; j < n1; ++j) v[j] = X1[IX(c, tb, ta, j)];
#pragma unroll
    for (int i = 0; i < n1; ++i) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < n1; ++j) s = fma(TB(K).I[i][j], v[j], s);
      X2[IX(c, tb, ta, i)] = s;
    }
  }
  __syncthreads();
  // S3 y-interp: thread (x = ta, z = tb)
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double v[n1];
#pragma unroll
    for (int j = 0; j < n1; ++j) v[j] = X2[IX(c, tb, j, ta)];
#pragma unroll
    for (int i = 0; i < n1; ++i) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < n1; ++j) s = fma(TB(K).I[i][j], v[j], s);
      X1[IX(c, tb, i, ta)] = s;
    }
  }
  __syncthreads();
  // S4 z-interp (+ z-derivative in registers): thread (x = ta, y = tb)
  double Gz[3][n1];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double v[n1], Uz[n1];
#pragma unroll
    for (int j = 0; j < n1; ++j) v[j] = X1[IX(c, j, tb, ta)];
#pragma unroll
    for (int i = 0; i < n1; ++i) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < n1; ++j) s = fma(TB(K).I[i][j], v[j], s);
      Uz[i] = s;
      X2[IX(c, i, tb, ta)] = s;
    }
#pragma unroll
    for (int i = 0; i < n1; ++i) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < n1; ++j) s = fma(TB(K).Dg[i][j], Uz[j], s);
      Gz[c][i] = s;
    }
  }
  __syncthreads();
  // S5 x-derivative: thread (y = ta, z = tb); y-derivative: thread (x = ta, z = tb)
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double v[n1], w[n1];
#pragma unroll
    for (int j = 0; j < n1; ++j) { v[j] = X2[IX(c, tb, ta, j)]; w[j] = X2[IX(c, tb, j, ta)]; }
#pragma unroll
    for (int i = 0; i < n1; ++i) {
      double s = 0.0, r = 0.0;
#pragma unroll
      for (int j = 0; j < n1; ++j) { s = fma(TB(K).Dg[i][j], v[j], s); r = fma(TB(K).Dg[i][j], w[j], r); }
      X1[IX(c, tb, ta, i)] = s;
      X3[IX(c, tb, i, ta)] = r;
    }
  }
  __syncthreads();
  // S6 tau at the Gauss points of column (x = ta, y = tb)
  double Wz[3][n1];
#pragma unroll
  for (int iz = 0; iz < n1; ++iz) {
    double g[3][3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      g[c][0] = X1[IX(c, iz, tb, ta)];
      g[c][1] = X3[IX(c, iz, tb, ta)];
      g[c][2] = Gz[c][iz];
    }
    const double mu = valid ? mut[e * NQ + (iz * n1 + tb) * n1 + ta] : 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      X1[IX(c, iz, tb, ta)] = mu * (g[c][0] + g[0][c]);
      X3[IX(c, iz, tb, ta)] = mu * (g[c][1] + g[1][c]);
      Wz[c][iz] = mu * (g[c][2] + g[2][c]);
    }
  }
  __syncthreads();
  // S7 x-back: thread (y = ta, z = tb)
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double v[n1];
#pragma unroll
    for (int i = 0; i < n1; ++i) v[i] = X1[IX(c, tb, ta, i)];
#pragma unroll
    for (int j = 0; j < n1; ++j) {
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < n1; ++i) s = fma(TB(K).Dg[i][j], v[i], s);
      X2[IX(c, tb, ta, j)] = s;
    }
  }
  __syncthreads();
  // S8 y-back: thread (x = ta, z = tb), read-modify-write of its own y-pencil
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double v[n1];
#pragma unroll
    for (int i = 0; i < n1; ++i) v[i] = X3[IX(c, tb, i, ta)];
#pragma unroll
    for (int j = 0; j < n1; ++j) {
      double s = X2[IX(c, tb, j, ta)];
#pragma unroll
      for (int i = 0; i < n1; ++i) s = fma(TB(K).Dg[i][j], v[i], s);
      X2[IX(c, tb, j, ta)] = s;
    }
  }
  __syncthreads();
  // S9 z-back + transposed z-interpolation: thread (x = ta, y = tb)
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double Vz[n1];
#pragma unroll
    for (int j = 0; j < n1; ++j) {
      double s = X2[IX(c, j, tb, ta)];
#pragma unroll
      for (int i = 0; i < n1; ++i) s = fma(TB(K).Dg[i][j], Wz[c][i], s);
      Vz[j] = s;
    }
#pragma unroll
    for (int a = 0; a < n1; ++a) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < n1; ++j) s = fma(TB(K).I[j][a], Vz[j], s);
      X1[IX(c, a, tb, ta)] = s;
    }
  }
  __syncthreads();
  // S10 transposed y-interpolation: thread (x = ta, z = tb)
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double v[n1];
#pragma unroll
    for (int j = 0; j < n1; ++j) v[j] = X1[IX(c, tb, j, ta)];
#pragma unroll
    for (int a = 0; a < n1; ++a) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < n1; ++j) s = fma(TB(K).I[j][a], v[j], s);
      X2[IX(c, tb, a, ta)] = s;
    }
  }
  __syncthreads();
  // S11 transposed x-interpolation: thread (y = ta, z = tb) -> E
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double v[n1];
#pragma unroll
    for (int j = 0; j < n1; ++j) v[j] = X2[IX(c, tb, ta, j)];
#pragma unroll
    for (int a = 0; a < n1; ++a) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < n1; ++j) s = fma(TB(K).I[j][a], v[j], s);
      if (valid) E[eix<K>(c, (tb * n1 + ta) * n1 + a, e, G.n_el)] = s;
    }
  }
#undef IX
}

// ------------------------------------------------------------------ setup: mu prescale + positivity
// mut = mu * w_qx w_qy w_qz * detJ * (2/h)^2 = mu * w_q * h/2.
template <int K>
__global__ void k_prescale(const double* __restrict__ mu, double* __restrict__ mut, int64_t n, double hs,
                           unsigned long long* bad) {
  constexpr int n1 = K + 1, NQ = Ord<K>::NQ;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int q = (int)(i % NQ);
  const double m = mu[i];
  if (!(m > 0.0) || !isfinite(m)) atomicAdd(bad, 1ull);
  const double wq = TB(K).w[q % n1] * TB(K).w[(q / n1) % n1] * TB(K).w[q / (n1 * n1)];
  mut[i] = m * wq * hs;
}

// ------------------------------------------------------------------ row a3: lumped weighted masses
// L[a][e] = detJ sum_q sqrt(mu_q) phi_a(xi_q) w_q  (eq:lumping with the
// all-ones coefficient vector, weighted by w = sqrt(mu), PAPER.md:310-323,
// 446-454).
template <int K>
__global__ void k_lump_elem(const double* __restrict__ mu, double* __restrict__ L, Geo G, double detJ) {
  constexpr int n1 = K + 1, NQ = Ord<K>::NQ;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= G.n_el) return;
  double s[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) s[q] = sqrt(mu[e * NQ + q]);
#pragma unroll 1
  for (int a = 0; a < NQ; ++a) {
    const int ax = a % n1, ay = (a / n1) % n1, az = a / (n1 * n1);
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int qx = q % n1, qy = (q / n1) % n1, qz = q / (n1 * n1);
      acc = fma(s[q], TB(K).W1[ax][qx] * TB(K).W1[ay][qy] * TB(K).W1[az][qz], acc);
    }
    L[(int64_t)a * G.n_el + e] = detJ * acc;
  }
}

// Viscosity-gradient weights (rmk:wbfbt-visc-grad; R17), one thread per
// Gauss point: grad mu of the element's Gauss-point interpolant (collocation derivative
// Dg along each axis, times s = 2/h) and out = sqrt(mu^2 + |grad mu|^2) = w^2, which the
// lumping kernels turn into the weight sqrt(out) = w.
template <int K>
__global__ void __launch_bounds__(256) k_grad_weights(const double* __restrict__ mu, double* __restrict__ out,
                                                      int64_t n, double s) {
  constexpr int n1 = K + 1, NQ = Ord<K>::NQ;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int q = (int)(i % NQ);
  const double* m = mu + (i - q);
  const int qx = q % n1, qy = (q / n1) % n1, qz = q / (n1 * n1);
  double gx = 0.0, gy = 0.0, gz = 0.0;
#pragma unroll
  for (int j = 0; j < n1; ++j) {
    gx = fma(TB(K).Dg[qx][j], __ldg(m + j + n1 * (qy + n1 * qz)), gx);
    gy = fma(TB(K).Dg[qy][j], __ldg(m + qx + n1 * (j + n1 * qz)), gy);
    gz = fma(TB(K).Dg[qz][j], __ldg(m + qx + n1 * (qy + n1 * j)), gz);
  }
  gx *= s; gy *= s; gz *= s;
  const double v = m[q];
  out[i] = sqrt(fma(v, v, fma(gx, gx, fma(gy, gy, gz * gz))));
}

// C[g] = sum_{e ni g} a_l(e) L[a(e,g)][e] (eq:bdramp PAPER.md:2232-2245), ascending e.
// Xinv = mask / X; nonpositive interior entries counted (integer atomics).
template <int K>
__global__ void k_lump_node(const double* __restrict__ L, double a_l, double a_r, double* Cw, double* Dw,
                            double* Cinv, double* Dinv, unsigned long long* nonpos, Geo G) {
  constexpr int n1 = K + 1;
  int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= G.n_nodes) return;
  const int nn1 = G.nn1;
  int gg[3] = {(int)(g % nn1), (int)((g / nn1) % nn1), (int)(g / ((int64_t)nn1 * nn1))};
  int pe[3][2], pa[3][2], pc[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    int q = gg[d] / K, r = gg[d] % K;
    pc[d] = 0;
    if (r != 0) { pe[d][0] = q; pa[d][0] = r; pc[d] = 1; }
    else {
      if (q - 1 >= 0) { pe[d][pc[d]] = q - 1; pa[d][pc[d]] = K; pc[d]++; }
      if (q < G.N) { pe[d][pc[d]] = q; pa[d][pc[d]] = 0; pc[d]++; }
    }
  }
  double cl = 0.0, cr = 0.0;
  for (int iz = 0; iz < pc[2]; ++iz)
    for (int iy = 0; iy < pc[1]; ++iy)
      for (int ix = 0; ix < pc[0]; ++ix) {
        const int ex = pe[0][ix], ey = pe[1][iy], ez = pe[2][iz];
        const int64_t e = ex + (int64_t)G.N * (ey + (int64_t)G.N * ez);
        const int a = pa[0][ix] + n1 * (pa[1][iy] + n1 * pa[2][iz]);
        const bool onb = ex == 0 || ey == 0 || (ez == 0 && !(G.zopen & 1)) || ex == G.N - 1 || ey == G.N - 1 ||
                         (ez == G.N - 1 && !(G.zopen & 2));
        const double l = L[(int64_t)a * G.n_el + e];
        cl += (onb ? a_l : 1.0) * l;
        cr += (onb ? a_r : 1.0) * l;
      }
  const bool b = node_bnd(gg[0], gg[1], gg[2], nn1);
  Cw[g] = cl; Dw[g] = cr;
  Cinv[g] = b ? 0.0 : 1.0 / cl;
  Dinv[g] = b ? 0.0 : 1.0 / cr;
  if (!b && cl <= 0.0) atomicAdd(nonpos + 0, 1ull);
  if (!b && cr <= 0.0) atomicAdd(nonpos + 1, 1ull);
}

// Load vector of a body force sampled at the Gauss points (the multi-sinker
// forcing f = (0, 0, beta (chi - 1))):
//   F[(c, g)] = sum_{e ni g} sum_q w_q detJ f_c(e, q) phi_a(xi_q),  elements ascending,
// Dirichlet rows 0 (elimination, R6).  fq: component-major [c][e][q] (q x fastest).
template <int K>
__global__ void k_load_node(const double* __restrict__ fq, double* __restrict__ F, Geo G, double detJ) {
  constexpr int n1 = K + 1, NQ = Ord<K>::NQ;
  int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= G.n_nodes) return;
  const int nn1 = G.nn1;
  int gg[3] = {(int)(g % nn1), (int)((g / nn1) % nn1), (int)(g / ((int64_t)nn1 * nn1))};
  if (node_bnd(gg[0], gg[1], gg[2], nn1)) {
    F[g] = 0.0; F[G.n_nodes + g] = 0.0; F[2 * G.n_nodes + g] = 0.0;
    return;
  }
  int pe[3][2], pa[3][2], pc[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    int q = gg[d] / K, r = gg[d] % K;
    pc[d] = 0;
    if (r != 0) { pe[d][0] = q; pa[d][0] = r; pc[d] = 1; }
    else {
      if (q - 1 >= 0) { pe[d][pc[d]] = q - 1; pa[d][pc[d]] = K; pc[d]++; }
      if (q < G.N) { pe[d][pc[d]] = q; pa[d][pc[d]] = 0; pc[d]++; }
    }
  }
  double acc[3] = {0.0, 0.0, 0.0};
  for (int iz = 0; iz < pc[2]; ++iz)
    for (int iy = 0; iy < pc[1]; ++iy)
      for (int ix = 0; ix < pc[0]; ++ix) {
        const int64_t e = pe[0][ix] + (int64_t)G.N * (pe[1][iy] + (int64_t)G.N * pe[2][iz]);
        const int ax = pa[0][ix], ay = pa[1][iy], az = pa[2][iz];
        for (int c = 0; c < 3; ++c) {
          const double* f = fq + ((int64_t)c * G.n_el + e) * NQ;
          double s = 0.0;
          for (int q = 0; q < NQ; ++q) {
            const int qx = q % n1, qy = (q / n1) % n1, qz = q / (n1 * n1);
            s = fma(f[q], TB(K).W1[ax][qx] * TB(K).W1[ay][qy] * TB(K).W1[az][qz], s);
          }
          acc[c] += detJ * s;
        }
      }
  F[g] = acc[0]; F[G.n_nodes + g] = acc[1]; F[2 * G.n_nodes + g] = acc[2];
}

// ------------------------------------------------------------------ row a4: Jacobi diagonals
// diag(K)_{e,m} = sum_{c,a} B_e[m,(c,a)]^2 X^-1[g(e,a)]; stores Minv = 1/diag too.
template <int K>
__global__ void k_jacobi(const double* __restrict__ Cinv, const double* __restrict__ Dinv, double* dL, double* dR,
                         double* mL, double* mR, Geo G, double sB) {
  constexpr int n1 = K + 1, NQ = Ord<K>::NQ, NM = Ord<K>::NM;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= G.n_el) return;
  int ex, ey, ez;
  elem_xyz(e, G.N, ex, ey, ez);
  int mm[NM][3];
  {
    int m = 0;
    for (int d = 0; d < K; ++d)
      for (int m3 = 0; m3 <= d; ++m3)
        for (int m2 = 0; m2 <= d - m3; ++m2) { mm[m][0] = d - m2 - m3; mm[m][1] = m2; mm[m][2] = m3; ++m; }
  }
  double sl[NM], sr[NM];
#pragma unroll
  for (int m = 0; m < NM; ++m) { sl[m] = 0.0; sr[m] = 0.0; }
#pragma unroll 1
  for (int c = 0; c < 3; ++c)
#pragma unroll 1
    for (int a = 0; a < NQ; ++a) {
      const int ax = a % n1, ay = (a / n1) % n1, az = a / (n1 * n1);
      const int64_t g = node_id(K * ex + ax, K * ey + ay, K * ez + az, G.nn1);
      const double xl = Cinv[g], xr = Dinv[g];
#pragma unroll
      for (int m = 0; m < NM; ++m) {
        const double fx = c == 0 ? TB(K).BD[mm[m][0]][ax] : TB(K).BI[mm[m][0]][ax];
        const double fy = c == 1 ? TB(K).BD[mm[m][1]][ay] : TB(K).BI[mm[m][1]][ay];
        const double fz = c == 2 ? TB(K).BD[mm[m][2]][az] : TB(K).BI[mm[m][2]][az];
        const double b = sB * (fx * fy * fz);
        sl[m] = fma(b * b, xl, sl[m]);
        sr[m] = fma(b * b, xr, sr[m]);
      }
    }
#pragma unroll
  for (int m = 0; m < NM; ++m) {
    dL[e * NM + m] = sl[m]; dR[e * NM + m] = sr[m];  // Minv: k_minv (pseudo-inverse, R11)
  }
  (void)mL; (void)mR;
}

// ------------------------------------------------------------------ vectors, projection, PCG
constexpr int VBS = 256;  // vector-kernel block size; grid fixed per context -> fixed reduction order

// sum of the constant-mode entries v[e*nm] (projection, R10)
__global__ void __launch_bounds__(VBS) k_mode0_sum(const double* __restrict__ v, int64_t n_el, int nm,
                                                   double* partial, unsigned* counter, double* total) {
  double s = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * VBS + threadIdx.x; e < n_el; e += (int64_t)gridDim.x * VBS) s += v[e * nm];
  grid_sum<VBS>(s, partial, counter, total);
}
// out = P in: copy, then subtract the mean of the mode-0 entries from them.
__global__ void k_project(const double* __restrict__ in, double* __restrict__ out, int64_t n, int nm,
                          int64_t n_el, const double* __restrict__ sum) {
  const double mean = *sum / (double)n_el;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (i % nm == 0) ? in[i] - mean : in[i];
}

// ---- PCG, vectors mode-major v[m*ne + e]; iteration i:
//   [stop_i] p_i = Minv r_i (+ beta_i p_{i-1}, beta_i = rz_i / rz_{i-1});  q = K p_i;
//   pq_i = <p_i, q>; [pq_i == 0 -> stop]; alpha = rz_i / pq_i; x += alpha p_i;
//   r -= alpha q; rz_{i+1} = <r, Minv r>; stop_{i+1} = (rz_{i+1} == 0).
// This is the oracle's recurrence (or_pcg) with the direction update moved to
// the top of the next iteration, so that it fuses into the K kernel.

// PCG control at the top of iteration i (first kernel of the iteration):
//   rz_i = sum of the previous kernel's <r, Minv r> partials (rzp, nrz),
//   stop_i = stop_{i-1} || pq_{i-1} == 0 || rz_i == 0   (stop_0 = rz_0 == 0),
//   beta_i = rz_i / rz_{i-1}; block 0 records rz_hist[i] and stop[i].
// Returns stop_i (uniform over the grid).
template <int BS>
__device__ __forceinline__ bool pcg_control(int i, const double* __restrict__ rzp, int nrz, double* rz_hist,
                                            const double* pq_hist, int* stop, double* beta) {
  // the history loads do not depend on the partial sum: issue them first
  const int st_prev = i > 0 ? stop[i - 1] : 0;
  const double pq_prev = i > 0 ? pq_hist[i - 1] : 1.0, rz_prev = i > 0 ? rz_hist[i - 1] : 1.0;
  const double rzi = sum_partials<BS>(rzp, nrz);
  const bool st = (i == 0) ? (rzi == 0.0) : (st_prev != 0 || pq_prev == 0.0 || rzi == 0.0);
  *beta = (i == 0 || st) ? 0.0 : rzi / rz_prev;
  if (blockIdx.x == 0 && threadIdx.x == 0) { rz_hist[i] = rzi; stop[i] = st ? 1 : 0; }
  return st;
}

// init: r = P b (element-major b -> mode-major r, constant-mode mean removed
// using bsum = sum_e b[e*nm]); x = 0; partials of rz_0 = <r, Minv r> -> rzp;
// z = Minv r stored when z != NULL (the TMA Poisson kernel reads it).
__global__ void __launch_bounds__(VBS) k_pcg_init(const double* __restrict__ b, const double* __restrict__ bsum,
                                                  double* x, double* r, const double* __restrict__ Minv, int64_t ne,
                                                  int nm, double* rzp, double* z, PLay L, int N) {
  const double mean = *bsum / (double)ne;
  const int64_t n = ne * nm;
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * VBS + threadIdx.x; i < n; i += (int64_t)gridDim.x * VBS) {
    const int64_t m = i / ne, e = i % ne;
    const int64_t j = L.at((int)m, e, N);
    const double bi = (m == 0) ? b[e * nm] - mean : b[e * nm + m];
    x[j] = 0.0; r[j] = bi;
    const double zi = Minv[j] * bi;
    if (z) z[j] = zi;
    s = fma(bi, zi, s);
  }
  store_partial<VBS>(s, rzp);
}

// k = 2 (n_m = 4): the same init / output through a shared-memory transpose.  A tile is
// 32 ey x 8 ex elements at one ez: element-major b rows (8 elements x 4 modes = 32
// consecutive words per ey) are read coalesced, the PCG vectors (y fastest, PLay) written
// coalesced along ey.  The per-thread loops above touch one 8-byte word per 32-byte sector.
constexpr int PT_Y = 32, PT_X = 8, PT_Q = PT_X * 4;
__device__ __forceinline__ void pt_tile(int tile, int N, int& ex0, int& ey0, int& ez) {
  const int nx = (N + PT_X - 1) / PT_X, ny = (N + PT_Y - 1) / PT_Y;
  ex0 = PT_X * (tile % nx); ey0 = PT_Y * ((tile / nx) % ny); ez = tile / (nx * ny);
}
// rz_0: one grid reduction (block partials in `partial`, summed in order by the last
// block) into rzp[0], rzp[1 .. nrz-1] = 0, so that the consumer's sum over nrz partials
// gives it unchanged; this lets the grid be as wide as the data, not red_blocks.
__global__ void __launch_bounds__(VBS) k_pcg_init_t(const double* __restrict__ b, const double* __restrict__ bsum,
                                                    double* x, double* r, const double* __restrict__ Minv, int64_t ne,
                                                    double* rzp, int nrz, double* partial, unsigned* counter,
                                                    double* z, PLay L, int N) {
  __shared__ double S[PT_Y][PT_Q + 1];
  const double mean = *bsum / (double)ne;
  const int nt = ((N + PT_X - 1) / PT_X) * ((N + PT_Y - 1) / PT_Y) * N;
  double s = 0.0;
  for (int tile = blockIdx.x; tile < nt; tile += gridDim.x) {
    int ex0, ey0, ez;
    pt_tile(tile, N, ex0, ey0, ez);
    for (int t = threadIdx.x; t < PT_Y * PT_Q; t += VBS) {
      const int yl = t / PT_Q, q = t % PT_Q, xl = q / 4, m = q % 4;
      const int ex = ex0 + xl, ey = ey0 + yl;
      double v = 0.0;
      if (ex < N && ey < N) {
        const int64_t e = ex + (int64_t)N * (ey + (int64_t)N * ez);
        v = b[e * 4 + m];
        if (m == 0) v -= mean;
      }
      S[yl][q] = v;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < PT_Y * PT_Q; t += VBS) {
      const int yl = t % PT_Y, q = t / PT_Y, xl = q / 4, m = q % 4;
      const int ex = ex0 + xl, ey = ey0 + yl;
      if (ex < N && ey < N) {
        const int64_t j = L.at(m, ex, ey, ez);
        const double bi = S[yl][q];
        x[j] = 0.0; r[j] = bi;
        const double zi = Minv[j] * bi;
        if (z) z[j] = zi;
        s = fma(bi, zi, s);
      }
    }
    __syncthreads();
  }
  if (grid_sum<VBS>(s, partial, counter, rzp))
    for (int i = 1; i < nrz; ++i) rzp[i] = 0.0;
}
__global__ void __launch_bounds__(VBS) k_pcg_out_t(const double* __restrict__ x, const double* __restrict__ xsum,
                                                   double* __restrict__ out, int64_t ne, PLay L, int N) {
  __shared__ double S[PT_Y][PT_Q + 1];
  const double mean = *xsum / (double)ne;
  const int nt = ((N + PT_X - 1) / PT_X) * ((N + PT_Y - 1) / PT_Y) * N;
  for (int tile = blockIdx.x; tile < nt; tile += gridDim.x) {
    int ex0, ey0, ez;
    pt_tile(tile, N, ex0, ey0, ez);
    for (int t = threadIdx.x; t < PT_Y * PT_Q; t += VBS) {
      const int yl = t % PT_Y, q = t / PT_Y, xl = q / 4, m = q % 4;
      const int ex = ex0 + xl, ey = ey0 + yl;
      S[yl][q] = (ex < N && ey < N) ? x[L.at(m, ex, ey, ez)] : 0.0;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < PT_Y * PT_Q; t += VBS) {
      const int yl = t / PT_Q, q = t % PT_Q, xl = q / 4, m = q % 4;
      const int ex = ex0 + xl, ey = ey0 + yl;
      if (ex < N && ey < N) {
        const int64_t e = ex + (int64_t)N * (ey + (int64_t)N * ez);
        const double v = S[yl][q];
        out[e * 4 + m] = (m == 0) ? v - mean : v;
      }
    }
    __syncthreads();
  }
}

// k = 2 Jacobi pseudo-inverse through the same tiled transpose as k_pcg_init_t
// (element-major diag K rows in, y-fastest PCG layout out): values as k_minv.
__global__ void __launch_bounds__(VBS) k_minv_t(const double* __restrict__ d, double* __restrict__ minv,
                                                const double* __restrict__ dmax, PLay L, int N) {
  __shared__ double S[PT_Y][PT_Q + 1];
  const double thr = 1e-13 * *dmax;
  const int nt = ((N + PT_X - 1) / PT_X) * ((N + PT_Y - 1) / PT_Y) * N;
  for (int tile = blockIdx.x; tile < nt; tile += gridDim.x) {
    int ex0, ey0, ez;
    pt_tile(tile, N, ex0, ey0, ez);
    for (int t = threadIdx.x; t < PT_Y * PT_Q; t += VBS) {
      const int yl = t / PT_Q, q = t % PT_Q, xl = q / 4, m = q % 4;
      const int ex = ex0 + xl, ey = ey0 + yl;
      S[yl][q] = (ex < N && ey < N) ? d[(ex + (int64_t)N * (ey + (int64_t)N * ez)) * 4 + m] : 0.0;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < PT_Y * PT_Q; t += VBS) {
      const int yl = t % PT_Y, q = t / PT_Y, xl = q / 4, m = q % 4;
      const int ex = ex0 + xl, ey = ey0 + yl;
      if (ex < N && ey < N) {
        const double v = S[yl][q];
        minv[L.at(m, ex, ey, ez)] = fabs(v) > thr ? 1.0 / v : 0.0;
      }
    }
    __syncthreads();
  }
}

// direction update (generic-k path; the k = 2 path fuses it into k_K2_fused).
// ctl: run pcg_control for iteration i (beta from the histories); otherwise
// mode 1 uses beta = rz_hist[i] / rz_hist[i-1] as recorded.
// mode 0: p = Minv r; 1: p = Minv r + beta pin  (pout may equal pin).
__global__ void __launch_bounds__(VBS) k_pupd(double* pout, const double* pin, const double* __restrict__ r,
                                              const double* __restrict__ Minv, int64_t n, int mode, int i, int ctl,
                                              const double* __restrict__ rzp, int nrz, double* rz_hist,
                                              const double* pq_hist, int* stop) {
  double beta = 0.0;
  if (ctl) {
    if (pcg_control<VBS>(i, rzp, nrz, rz_hist, pq_hist, stop, &beta)) return;
  } else if (mode == 1) {
    beta = rz_hist[i] / rz_hist[i - 1];
  }
  for (int64_t j = (int64_t)blockIdx.x * VBS + threadIdx.x; j < n; j += (int64_t)gridDim.x * VBS) {
    const double z = Minv[j] * r[j];
    pout[j] = mode == 1 ? fma(beta, pin[j], z) : z;
  }
}

// iteration i: pq_i = sum of the K kernel's <p_i, q> partials (pqp, npq);
// alpha = rz_i / pq_i; x += alpha p; r -= alpha q; partials of
// rz_{i+1} = <r, Minv r> -> rzp; z = Minv r stored when z != NULL.  Block 0
// records pq_hist[i].
// Streaming: the vectors are 16-byte aligned (cudaMalloc, n even), so each thread
// moves pairs (double2) and keeps U pairs of all five inputs in flight before any
// arithmetic; the first batch is issued before the pq reduction, which only the
// arithmetic needs.  The rz partial of a thread sums its entries in index order.
// Solution-update forms of k_pcg_upd (all bitwise equal to updating every iteration):
//   XU_SINGLE: x = fma(alpha_i, p_i, x)
//   XU_DEFER:  x untouched (even iterations of a loop; the next odd one applies it)
//   XU_PAIR:   x = fma(alpha_i, p_i, fma(alpha_{i-1}, p_{i-1}, x))  (odd iterations)
// p_{i-1} is still in the other direction buffer, so x is read and written every other
// iteration only.  k_pcg_xfin applies a deferred last update after the loop.
enum { XU_SINGLE = 0, XU_DEFER = 1, XU_PAIR = 2 };
template <int U, int XM>
__device__ __forceinline__ void pcg_upd_batch(int64_t j0, int64_t stride, int64_t n2, const double2* x,
                                              const double2* r, const double2* p, const double2* pp,
                                              const double2* q, const double2* M, double2 (&X)[U],
                                              double2 (&R)[U], double2 (&P)[U], double2 (&PP)[U], double2 (&Q)[U],
                                              double2 (&Mv)[U]) {
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t j = j0 + u * stride;
    if (j < n2) {
      if (XM != XU_DEFER) { X[u] = x[j]; P[u] = p[j]; }
      if (XM == XU_PAIR) PP[u] = pp[j];
      R[u] = r[j]; Q[u] = __ldcg(q + j); Mv[u] = M[j];
    }
  }
}
// iteration j made an update: not stopped and pq_j != 0 (pq_hist[j] is only valid then)
__device__ __forceinline__ double pcg_alpha(int j, const double* rz_hist, const double* pq_hist, const int* stop) {
  return (j >= 0 && stop[j] == 0 && pq_hist[j] != 0.0) ? rz_hist[j] / pq_hist[j] : 0.0;
}
// x = fma(alpha_j, p_j, x) if iteration j made an update (grid-stride)
__device__ __forceinline__ void pcg_x_single(double* x, const double* p, int64_t n, double a) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    x[k] = fma(a, p[k], x[k]);
}

// iteration i: pq_i = sum of the K kernel's <p_i, q> partials (pqp, npq);
// alpha = rz_i / pq_i; x update (XM above); r -= alpha q; partials of
// rz_{i+1} = <r, Minv r> -> rzp; z = Minv r stored when z != NULL.  Block 0
// records pq_hist[i].
// Streaming: the vectors are 16-byte aligned (cudaMalloc, n even), so each thread
// moves pairs (double2) and keeps U pairs of all inputs in flight before any
// arithmetic; the first batch is issued before the pq reduction, which only the
// arithmetic needs.  The rz partial of a thread sums its entries in index order.
template <int XM>
__global__ void __launch_bounds__(VBS) k_pcg_upd(double* x, double* r, const double* __restrict__ p,
                                                 const double* __restrict__ pprev, const double* __restrict__ q,
                                                 const double* __restrict__ Minv, int64_t n, int i,
                                                 const double* __restrict__ pqp, int npq, const double* rz_hist,
                                                 double* pq_hist, const int* stop, double* rzp, double* z) {
  constexpr int U = 2;
  if (stop[i]) {
    // a stopped odd iteration still owes the previous (even) iteration's deferred update
    if (XM == XU_PAIR) {
      const double ap = pcg_alpha(i - 1, rz_hist, pq_hist, stop);
      if (ap != 0.0) pcg_x_single(x, pprev, n, ap);
    }
    return;
  }
  const int64_t n2 = n / 2;  // n is even
  const int64_t stride = (int64_t)gridDim.x * VBS;
  double2* x2 = reinterpret_cast<double2*>(x);
  double2* r2 = reinterpret_cast<double2*>(r);
  double2* z2 = reinterpret_cast<double2*>(z);
  const double2* p2 = reinterpret_cast<const double2*>(p);
  const double2* pp2 = reinterpret_cast<const double2*>(pprev);
  const double2* q2 = reinterpret_cast<const double2*>(q);
  const double2* M2 = reinterpret_cast<const double2*>(Minv);
  double2 X[U], R[U], P[U], PP[U], Q[U], Mv[U];
  int64_t j0 = (int64_t)blockIdx.x * VBS + threadIdx.x;
  pcg_upd_batch<U, XM>(j0, stride, n2, x2, r2, p2, pp2, q2, M2, X, R, P, PP, Q, Mv);
  const double ap = XM == XU_PAIR ? pcg_alpha(i - 1, rz_hist, pq_hist, stop) : 0.0;
  const double pq = sum_partials<VBS>(pqp, npq);
  if (blockIdx.x == 0 && threadIdx.x == 0) pq_hist[i] = pq;
  if (pq == 0.0) {
    if (XM == XU_PAIR && ap != 0.0) pcg_x_single(x, pprev, n, ap);  // (no update of its own)
    return;
  }
  const double alpha = rz_hist[i] / pq;
  double s = 0.0;
  for (; j0 < n2; j0 += U * stride) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = j0 + u * stride;
      if (j < n2) {
        double2 ro, zo;
        if (XM == XU_SINGLE) {
          double2 xo;
          xo.x = fma(alpha, P[u].x, X[u].x); xo.y = fma(alpha, P[u].y, X[u].y);
          x2[j] = xo;
        } else if (XM == XU_PAIR) {
          double2 xo;
          xo.x = fma(alpha, P[u].x, fma(ap, PP[u].x, X[u].x));
          xo.y = fma(alpha, P[u].y, fma(ap, PP[u].y, X[u].y));
          x2[j] = xo;
        }
        ro.x = fma(-alpha, Q[u].x, R[u].x); ro.y = fma(-alpha, Q[u].y, R[u].y);
        zo.x = Mv[u].x * ro.x; zo.y = Mv[u].y * ro.y;
        r2[j] = ro;
        if (z) z2[j] = zo;
        s = fma(ro.x, zo.x, s);
        s = fma(ro.y, zo.y, s);
      }
    }
    pcg_upd_batch<U, XM>(j0 + U * stride, stride, n2, x2, r2, p2, pp2, q2, M2, X, R, P, PP, Q, Mv);
  }
  store_partial<VBS>(s, rzp);
}

// after a loop whose last iteration i deferred its update: x = fma(alpha_i, p_i, x)
__global__ void __launch_bounds__(VBS) k_pcg_xfin(double* x, const double* __restrict__ p, int64_t n, int i,
                                                  const double* rz_hist, const double* pq_hist, const int* stop) {
  const double a = pcg_alpha(i, rz_hist, pq_hist, stop);
  if (a != 0.0) pcg_x_single(x, p, n, a);
}

// out (element-major) = P x (mode-major), xsum = sum of the constant-mode entries.
__global__ void k_pcg_out(const double* __restrict__ x, const double* __restrict__ xsum, double* __restrict__ out,
                          int64_t ne, int nm, PLay L, int N) {
  const double mean = *xsum / (double)ne;
  const int64_t n = ne * nm;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i / nm, m = i % nm;
    const double v = x[L.at((int)m, e, N)];
    out[i] = (m == 0) ? v - mean : v;
  }
}

// layout conversion element-major <-> mode-major (debug one-step entry)
// element-major [e*nm + m] <-> PCG storage (PLay); to_soa: element-major -> PCG
// ---------------------------------------------------------------- FGMRES helpers (R19)
// *out = <a, b> (fixed-order grid reduction: block partials summed by the last block)
__global__ void __launch_bounds__(VBS) k_dot_dev(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                                                 double* partial, unsigned* counter, double* out) {
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * VBS + threadIdx.x; i < n; i += (int64_t)gridDim.x * VBS)
    s = fma(a[i], b[i], s);
  grid_sum<VBS>(s, partial, counter, out);
}
// w -= (*h) v  (the scalar stays on the device: modified Gram-Schmidt without host round trips)
__global__ void __launch_bounds__(VBS) k_axpy_dev(double* __restrict__ w, const double* __restrict__ v, int64_t n,
                                                  const double* __restrict__ h) {
  const double a = *h;
  for (int64_t i = (int64_t)blockIdx.x * VBS + threadIdx.x; i < n; i += (int64_t)gridDim.x * VBS) w[i] -= a * v[i];
}
// out = in / sqrt(*h2)
__global__ void __launch_bounds__(VBS) k_unit_dev(double* __restrict__ out, const double* __restrict__ in, int64_t n,
                                                  const double* __restrict__ h2) {
  const double nrm = sqrt(*h2);
  for (int64_t i = (int64_t)blockIdx.x * VBS + threadIdx.x; i < n; i += (int64_t)gridDim.x * VBS) out[i] = in[i] / nrm;
}
// FGMRES least-squares update on the device (R19), one thread: column j of the Hessenberg
// (h[0..j] Gram-Schmidt scalars, h[j+1] = <w, w>) gets the previous Givens rotations, a new
// rotation (cs[j], sn[j]) zeroes its subdiagonal, the rotated right-hand side g is updated,
// and R[i][j] (row stride m) is stored.  res[0] = |g[j+1]| (the residual estimate), res[1]
// = |h_{j+1,j}|.  The arithmetic is the host loop's, operation for operation (no contraction).
__global__ void k_givens(int j, int m, const double* __restrict__ h, double* __restrict__ R, double* __restrict__ cs,
                         double* __restrict__ sn, double* __restrict__ g, double* __restrict__ res) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double hn = sqrt(h[j + 1]);
  for (int i = 0; i <= j; ++i) R[(size_t)i * m + j] = h[i];
  for (int i = 0; i < j; ++i) {
    const double a = R[(size_t)i * m + j], b = R[(size_t)(i + 1) * m + j];
    R[(size_t)i * m + j] = __dadd_rn(__dmul_rn(cs[i], a), __dmul_rn(sn[i], b));
    R[(size_t)(i + 1) * m + j] = __dadd_rn(__dmul_rn(-sn[i], a), __dmul_rn(cs[i], b));
  }
  const double a = R[(size_t)j * m + j], den = sqrt(__dadd_rn(__dmul_rn(a, a), __dmul_rn(hn, hn)));
  cs[j] = den > 0.0 ? a / den : 1.0;
  sn[j] = den > 0.0 ? hn / den : 0.0;
  R[(size_t)j * m + j] = den;
  g[j + 1] = __dmul_rn(-sn[j], g[j]);
  g[j] = __dmul_rn(cs[j], g[j]);
  res[0] = fabs(g[j + 1]);
  res[1] = hn;
}
// back substitution R y = g on columns 0..jend (one thread), as the host loop did
__global__ void k_fgmres_y(int jend, int m, const double* __restrict__ R, const double* __restrict__ g,
                           double* __restrict__ y) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int i = jend; i >= 0; --i) {
    double t = g[i];
    for (int k = i + 1; k <= jend; ++k) t = __dsub_rn(t, __dmul_rn(R[(size_t)i * m + k], y[k]));
    y[i] = t / R[(size_t)i * m + i];
  }
}
// y += (*a) x  (device scalar)
__global__ void __launch_bounds__(VBS) k_axpy_devp(double* __restrict__ y, const double* __restrict__ x, int64_t n,
                                                   const double* __restrict__ a) {
  const double s = *a;
  for (int64_t i = (int64_t)blockIdx.x * VBS + threadIdx.x; i < n; i += (int64_t)gridDim.x * VBS) y[i] += s * x[i];
}
// y += a x  (host scalar)
__global__ void __launch_bounds__(VBS) k_axpy(double* __restrict__ y, const double* __restrict__ x, int64_t n, double a) {
  for (int64_t i = (int64_t)blockIdx.x * VBS + threadIdx.x; i < n; i += (int64_t)gridDim.x * VBS) y[i] += a * x[i];
}
// y = a x + b y
__global__ void __launch_bounds__(VBS) k_axpby(double* __restrict__ y, const double* __restrict__ x, int64_t n, double a,
                                               double b) {
  for (int64_t i = (int64_t)blockIdx.x * VBS + threadIdx.x; i < n; i += (int64_t)gridDim.x * VBS)
    y[i] = a * x[i] + b * y[i];
}

// ---------------------------------------------------------------- diag(A) (R18)
// Element part of diag(M A M): E[c][a][e] = sum_q mut_q (sum_j g_j^2 + g_c^2), g_j the
// reference derivative d/dxi_j phi_a at Gauss point q (mut = mu w_q h/2 carries the
// detJ (2/h)^2 factor, as in A).  g = prod_d (d == j ? D1 : I)[q_d][a_d] with I the
// GLL -> Gauss interpolation table and D1 = Dg I its derivative (exact: the Gauss
// interpolant of a degree-k polynomial is the polynomial).  mut layout: tile-blocked
// mutT[tile][q][le] when TX > 0 (k = 2, A's tiles), else mut[e][q].  One thread per element.
template <int K, int TX, int TY, int TZ>
__global__ void __launch_bounds__(128) k_diagA_elem(const double* __restrict__ mut, double* __restrict__ E, Geo G) {
  constexpr int n1 = K + 1, NQ = Ord<K>::NQ;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= G.n_el) return;
  int ex, ey, ez;
  elem_xyz(e, G.N, ex, ey, ez);
  int64_t mbase, mstride;
  if constexpr (TX > 0) {
    const int NTX = (G.N + TX - 1) / TX, NTY = (G.N + TY - 1) / TY;
    const int tile = ex / TX + NTX * (ey / TY + NTY * (ez / TZ));
    const int le = ex % TX + TX * (ey % TY + TY * (ez % TZ));
    constexpr int NE = TX > 0 ? TX * TY * TZ : 1;
    mbase = (int64_t)tile * NQ * NE + le; mstride = NE;
  } else {
    mbase = e * NQ; mstride = 1;
  }
  double D1[n1][n1];  // D1[i][a] = sum_k Dg[i][k] I[k][a]
#pragma unroll
  for (int i = 0; i < n1; ++i)
#pragma unroll
    for (int a = 0; a < n1; ++a) {
      double t = 0.0;
#pragma unroll
      for (int k = 0; k < n1; ++k) t = fma(TB(K).Dg[i][k], TB(K).I[k][a], t);
      D1[i][a] = t;
    }
#pragma unroll 1
  for (int a = 0; a < NQ; ++a) {
    const int ax = a % n1, ay = (a / n1) % n1, az = a / (n1 * n1);
    double t0 = 0.0, t1 = 0.0, t2 = 0.0;
#pragma unroll 1
    for (int q = 0; q < NQ; ++q) {
      const int qx = q % n1, qy = (q / n1) % n1, qz = q / (n1 * n1);
      const double Ix = TB(K).I[qx][ax], Iy = TB(K).I[qy][ay], Iz = TB(K).I[qz][az];
      const double gx = D1[qx][ax] * Iy * Iz, gy = Ix * D1[qy][ay] * Iz, gz = Ix * Iy * D1[qz][az];
      const double g2 = gx * gx + gy * gy + gz * gz;
      const double m = __ldg(mut + mbase + (int64_t)q * mstride);
      t0 = fma(m, g2 + gx * gx, t0);
      t1 = fma(m, g2 + gy * gy, t1);
      t2 = fma(m, g2 + gz * gz, t2);
    }
    E[eix<K>(0, a, e, G.n_el)] = t0;
    E[eix<K>(1, a, e, G.n_el)] = t1;
    E[eix<K>(2, a, e, G.n_el)] = t2;
  }
}
// Dinv = 1 / d where d > 0, else 0 (Dirichlet dofs, whose masked diagonal is 0)
__global__ void k_inv_pos(const double* __restrict__ d, double* __restrict__ dinv, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dinv[i] = d[i] > 0.0 ? 1.0 / d[i] : 0.0;
}
// out = M in (velocity SoA, Dirichlet dofs 0)
__global__ void k_mask_v(const double* __restrict__ in, double* __restrict__ out, Geo G) {
  const int64_t n = 3 * G.n_nodes;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = i % G.n_nodes;
    const int gx = (int)(g % G.nn1), gy = (int)((g / G.nn1) % G.nn1), gz = (int)(g / ((int64_t)G.nn1 * G.nn1));
    out[i] = node_bnd(gx, gy, gz, G.nn1) ? 0.0 : in[i];
  }
}
// Chebyshev step (as k_cheb) for any length, scalar: x += d; r -= q; d = c1 d + c2 (Minv r);
// first: d = c2 (Minv r) only
__global__ void __launch_bounds__(VBS) k_cheb_s(double* __restrict__ x, double* __restrict__ r, double* __restrict__ d,
                                                const double* __restrict__ q, const double* __restrict__ Minv,
                                                int64_t n, double c1, double c2, int first) {
  for (int64_t i = (int64_t)blockIdx.x * VBS + threadIdx.x; i < n; i += (int64_t)gridDim.x * VBS) {
    const double m = Minv[i];
    double rv = r[i];
    if (first) { d[i] = c2 * (m * rv); continue; }
    const double dv = d[i];
    x[i] += dv;
    rv -= q[i];
    r[i] = rv;
    d[i] = c1 * dv + c2 * (m * rv);
  }
}

// ---------------------------------------------------------------- Chebyshev-Jacobi
// One step of Saad's Alg. 12.1 after q = K d:  x += d; r -= q; d = c1 d + c2 (Minv r)
// with the host-computed scalars c1 = rho' rho, c2 = 2 rho' / delta.  first: the start
// d = c2 (Minv r) only (c2 = 1 / theta).  Pure streaming, no reduction.
__global__ void __launch_bounds__(VBS) k_cheb(double* __restrict__ x, double* __restrict__ r, double* __restrict__ d,
                                              const double* __restrict__ q, const double* __restrict__ Minv,
                                              int64_t n, double c1, double c2, int first) {
  const int64_t n2 = n / 2;  // n is even (PLay), 16-byte aligned vectors
  double2* x2 = reinterpret_cast<double2*>(x);
  double2* r2 = reinterpret_cast<double2*>(r);
  double2* d2 = reinterpret_cast<double2*>(d);
  const double2* q2 = reinterpret_cast<const double2*>(q);
  const double2* M2 = reinterpret_cast<const double2*>(Minv);
  for (int64_t j = (int64_t)blockIdx.x * VBS + threadIdx.x; j < n2; j += (int64_t)gridDim.x * VBS) {
    const double2 m = M2[j];
    double2 rv = r2[j];
    if (first) {
      d2[j] = make_double2(c2 * (m.x * rv.x), c2 * (m.y * rv.y));
      continue;
    }
    const double2 dv = d2[j], qv = __ldcg(q2 + j);
    double2 xv = x2[j];
    xv.x += dv.x; xv.y += dv.y;
    rv.x -= qv.x; rv.y -= qv.y;
    x2[j] = xv;
    r2[j] = rv;
    d2[j] = make_double2(c1 * dv.x + c2 * (m.x * rv.x), c1 * dv.y + c2 * (m.y * rv.y));
  }
}

// Power iteration (R16): partials of <w, w> with w = Minv o v (in place) when Minv != NULL,
// else of <v, v>.  Deferred reduction as the PCG kernels (k_pow_scale sums the partials).
__global__ void __launch_bounds__(VBS) k_pow_sumsq(double* __restrict__ v, const double* __restrict__ Minv,
                                                   int64_t n, double* part) {
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * VBS + threadIdx.x; i < n; i += (int64_t)gridDim.x * VBS) {
    double w = v[i];
    if (Minv) { w *= Minv[i]; v[i] = w; }
    s = fma(w, w, s);
  }
  store_partial<VBS>(s, part);
}
// out = in / ||in|| (||in|| = sqrt of the summed partials; 0 stays 0); block 0 stores ||in|| to *lam
__global__ void __launch_bounds__(VBS) k_pow_scale(const double* in, double* out, int64_t n,
                                                   const double* __restrict__ part, int npart, double* lam) {
  const double nrm = sqrt(sum_partials<VBS>(part, npart));
  if (blockIdx.x == 0 && threadIdx.x == 0) *lam = nrm;
  for (int64_t i = (int64_t)blockIdx.x * VBS + threadIdx.x; i < n; i += (int64_t)gridDim.x * VBS)
    out[i] = nrm > 0.0 ? in[i] / nrm : 0.0;
}

__global__ void k_transpose(const double* __restrict__ in, double* __restrict__ out, int64_t ne, int nm, int to_soa,
                            PLay L, int N) {
  const int64_t n = ne * nm;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = i / ne, e = i % ne;
    const int64_t j = L.at((int)m, e, N);
    if (to_soa) out[j] = in[e * nm + m];
    else out[e * nm + m] = in[j];
  }
}

}  // namespace wb
