// k2_tma.cuh -- the fused k = 2 Poisson operator (k2_fused.cuh) with TMA
// staging: persistent CTAs (one per SM) walk the element tiles; the halo box of
// p_old and z = Minv r (4-D tensor maps over the mode-major PCG vectors, hardware
// zero fill outside the mesh; z is stored by the PCG update kernel) and the X box (3-D tensor map over a copy of X
// with 16-byte-aligned rows) land in shared memory by cp.async.bulk.tensor,
// completion tracked by mbarriers.  Each buffer is refilled for the NEXT tile
// as soon as the current tile has consumed it (p, z after step 0, X after
// step 1, p after step 2), so the loads overlap the compute of steps 1 and 2.
// Same arithmetic as k_K2_fused (identical per-node / per-element order).
#pragma once
#include <cuda.h>
#include "k2_fused.cuh"
#include "mbar.cuh"

namespace wb {

// phase-timing probe (k_dbg bit 0x4000): thread 0 of every CTA adds its clock64 cycles
// per phase: [0] prologue/control, [1] wait p/r/Minv, [2] step 0 (+ barrier),
// [3] wait X, [4] step 1 (+ barrier), [5] step 2 (+ barrier), [6] tiles
__device__ unsigned long long g_kprof[8];
// launch timeline probe (WB_KPROF, k_dbg 0x4000, PCG iteration 5 only): per CTA the
// %globaltimer (ns) at entry, loop start, loop end and exit
__device__ unsigned long long g_ktl[512][4];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Layout constants of the TMA variant (tile TX x TY x TZ elements).
// The PCG vectors of these contexts are stored y fastest with a zero pad at each end
// of every y column (PLay, off = 1), so the halo box (HY, HZ, HX, 4 modes) starts at
// the even y index ey0 (fp64 TMA tile loads need a 16-byte-aligned innermost start:
// an odd start faults) and lands as [m][hx][hz][hy], the pencil layout; step 0 copies
// it into Ps with the padded qz stride (conflict-free pencil reads).
template <int TX, int TY, int TZ>
struct FKT {
  using F = FK2<TX, TY, TZ>;
  static constexpr int HX = TX + 2, HY = TY + 2, HZ = TZ + 2;
  static_assert(HY % 2 == 0 && TY % 2 == 0, "16-byte box rows, even y start");
  static constexpr int NB = HX * HY * HZ;  // raw box (HY, HZ, HX) per mode
  static constexpr unsigned PBYTES = 4u * NB * 8u;
  // Ps[m][qx][qz][qy]: a pencil's (qy, qz) row is the fastest index, so the lanes of a
  // pencil class (consecutive qy) read consecutive words
  // qz stride QS = 9 (mod 16) and >= HY: a class-(0,0) half-warp (9 qy per qz row)
  // then reads 16 distinct bank pairs
  static constexpr int QS = HY + ((25 - HY % 16) % 16);
  static constexpr int NHD = HX * HY * HZ;  // halo elements
  static constexpr int NHP = HX * HZ * QS;  // padded Ps stride per mode
  __host__ __device__ static constexpr int pidx(int qx, int qy, int qz) { return qy + QS * (qz + HZ * qx); }
  // T[c][col(nx)][row]: rows grouped by class (ny%2, nz%2), row = off[cls] + jy + CY jz;
  // column stride TC = 4 (mod 16) makes step 2 (4 x-elements x 4 y-elements per
  // half-warp) conflict-free, class-local rows make the pencil stores conflict-free
  static constexpr int R00 = (TY + 1) * (TZ + 1), R10 = TY * (TZ + 1), R01 = (TY + 1) * TZ, R11 = TY * TZ;
  static constexpr int NROW = R00 + R10 + R01 + R11;
  static constexpr int TC = NROW + ((20 - NROW % 16) % 16);
  static constexpr int TN = F::MX * TC;
  // X in pencil layout: per tile one contiguous block XT[nx][row] (row as above, no
  // padding), built at setup (k_x_tiles); a lane-consecutive pencil class reads
  // consecutive words.  Block length rounded to 16 bytes for the bulk copy.
  static constexpr int XTB = (F::MX * NROW + 1) & ~1;
  static constexpr unsigned XBYTES = (unsigned)XTB * 8u;
  // the thread that issues the per-tile TMA loads: lane 0 of the last warp (light
  // class-(1,1) pencils, no element in step 2), off the heavy warps' critical path
  static constexpr int TMA_T = F::NTH - 32;
  // row sums S[c][m1][lx][row] (x-contracted B per element of the row) in the T region
  __host__ __device__ static constexpr int sidx(int c, int m1, int lx) { return ((c * 2 + m1) * TX + lx) * TC; }
  static_assert(6 * TX <= 3 * F::MX, "S fits in the T region");
  // class (1,0) rows are jz-fastest (its pencils are assigned jz-fastest too): with the
  // Ps row stride QS = 9 (mod 16), 8-wide jy rows would put two lanes of a half-warp on
  // one bank pair; 9 jz values and the next jy's 7 hit 16 distinct ones
  __host__ __device__ static constexpr int row(int ny, int nz) {
    return ((ny & 1) && !(nz & 1)) ? R00 + (nz >> 1) + (TZ + 1) * (ny >> 1)
                                   : ((ny & 1) ? R00 + R10 + R01 : ((nz & 1) ? R00 + R10 : 0)) + (ny >> 1) +
                                         ((ny & 1) ? TY : TY + 1) * (nz >> 1);
  }
  // shared layout (bytes): raw p | raw r or z | raw Minv | Ps | X | T | barriers, each 1024-aligned
  static constexpr size_t al(size_t b) { return (b + 1023) & ~(size_t)1023; }
  static constexpr size_t OFF_P = 0, OFF_R = al(PBYTES), OFF_M = OFF_R + al(PBYTES), OFF_S = OFF_M + al(PBYTES),
                          OFF_X = OFF_S + al(4u * NHP * 8u), OFF_T = OFF_X + al(XBYTES),
                          OFF_B = OFF_T + al(3u * TN * 8u);
  static constexpr size_t SMEM = OFF_B + 64 + 1024;  // + slack for 1024-byte base alignment
};

// Step 0 copy, raw box [row][HY] -> Ps [row][QS] (row = (m, hx, hz)), in y-pairs:
// v = Minv r + beta p_old (mode 1), Minv r (mode 0) or p (mode 2).  Pair item t of a
// half-warp h = t / 16 takes pair column s = h % 5 of rows 16 (h / 5) + (t % 16): the
// 16-byte loads (pair 5 row + s) of a quarter-warp hit 8 distinct 16-byte slots and the
// two 8-byte stores (25 row + 2 s, + 1) of a half-warp 16 distinct bank pairs, since
// 5 and 9 = 25 mod 16 are odd.  (A row-major walk makes the stores 2-way conflicted.)
template <int TX, int TY, int TZ, bool ZB>
__device__ __forceinline__ void fkt_copy_pair_rs(int r, int sp, const double* __restrict__ Pb,
                                                 const double* __restrict__ Zb, const double* __restrict__ Mb,
                                                 double* __restrict__ Pd, int mode, double beta);
template <int TX, int TY, int TZ, bool ZB>
__device__ __forceinline__ void fkt_copy_pair(int t, const double* __restrict__ Pb, const double* __restrict__ Zb,
                                              const double* __restrict__ Mb, double* __restrict__ Pd, int mode,
                                              double beta) {
  using K = FKT<TX, TY, TZ>;
  static_assert(K::HY == 10 && K::QS % 16 == 9 && (4 * K::HX * K::HZ) % 16 == 0, "pair walk layout");
  const int h = t >> 4;
  fkt_copy_pair_rs<TX, TY, TZ, ZB>(16 * (h / 5) + (t & 15), h % 5, Pb, Zb, Mb, Pd, mode, beta);
}
// the same with the item's (row, pair column) given: the tile loop of k_K2_tma steps them
// incrementally instead of dividing the item index
template <int TX, int TY, int TZ, bool ZB>
__device__ __forceinline__ void fkt_copy_pair_rs(int r, int sp, const double* __restrict__ Pb,
                                                 const double* __restrict__ Zb, const double* __restrict__ Mb,
                                                 double* __restrict__ Pd, int mode, double beta) {
  using K = FKT<TX, TY, TZ>;
  const int j2 = 5 * r + sp;
  const double2 pp = reinterpret_cast<const double2*>(Pb)[j2];
  double2 v;
  if (mode == 2) v = pp;
  else {
    double2 z = reinterpret_cast<const double2*>(Zb)[j2];
    if (!ZB) {
      const double2 mm = reinterpret_cast<const double2*>(Mb)[j2];
      z.x = mm.x * z.x; z.y = mm.y * z.y;
    }
    v = z;
    if (mode == 1) { v.x = fma(beta, pp.x, z.x); v.y = fma(beta, pp.y, z.y); }
  }
  double* d = Pd + K::QS * r + 2 * sp;
  d[0] = v.x;
  d[1] = v.y;
}

// x-pencil as in fk2_pencil, with the staged layouts: Ps (padded qy-fastest rows), Xs (XT block)
template <int TX, int TY, int TZ, int RY, int RZ>
__device__ __forceinline__ void fkt_pencil(const double* __restrict__ Ps, double* __restrict__ T,
                                           const double* __restrict__ Xs, int jy, int jz, double sB) {
  using F = FK2<TX, TY, TZ>;
  using K = FKT<TX, TY, TZ>;
  const int ny = 2 * jy + RY, nz = 2 * jz + RZ;
  double acc[3][F::MX];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int nx = 0; nx < F::MX; ++nx) acc[c][nx] = 0.0;
  // Factorised B^T (product structure of the element matrix): per halo x-position qx,
  // first the (y, z) element combos of the row are folded into two x-mode weights
  // per component, W_c[m1] (4 FMA per combo and component), then the 1-D x
  // expansion adds W to the three nodes of element qx (6 FMA per node).
#pragma unroll
  for (int qx = 0; qx < K::HX; ++qx) {
    double W[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
    for (int iz = 0; iz < (RZ ? 1 : 2); ++iz) {
      const int qz = RZ ? jz + 1 : jz + iz;
      const int az = RZ ? 1 : (iz == 0 ? 2 : 0);
#pragma unroll
      for (int iy = 0; iy < (RY ? 1 : 2); ++iy) {
        const int qy = RY ? jy + 1 : jy + iy;
        const int ay = RY ? 1 : (iy == 0 ? 2 : 0);
        const int h = K::pidx(qx, qy, qz);
        const double p000 = Ps[h], p100 = Ps[K::NHP + h], p010 = Ps[2 * K::NHP + h], p001 = Ps[3 * K::NHP + h];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          if (w2_nz(c, ay, az, 0)) {
            W[c][0] = fma(c_W2[c][ay][az][0], p000, W[c][0]);
            W[c][1] = fma(c_W2[c][ay][az][0], p100, W[c][1]);
          }
          if (w2_nz(c, ay, az, 1)) W[c][0] = fma(c_W2[c][ay][az][1], p010, W[c][0]);
          if (w2_nz(c, ay, az, 2)) W[c][0] = fma(c_W2[c][ay][az][2], p001, W[c][0]);
        }
      }
    }
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      const int nx = 2 * qx - 2 + ax;
      if (nx < 0 || nx >= F::MX) continue;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        if (x2_nz(c, ax, 0)) acc[c][nx] = fma(c_X2[c][ax][0], W[c][0], acc[c][nx]);
        if (x2_nz(c, ax, 1)) acc[c][nx] = fma(c_X2[c][ax][1], W[c][1], acc[c][nx]);
      }
    }
  }
  // t = sB X^-1 (B^T p) at the row's nodes, then the x-contraction of B for the
  // row's elements: S_c[m1][lx] = sum_ax Mx_c[m1][ax] t_c(2 lx + ax)
  const double* Xr = Xs + K::row(ny, nz);
#pragma unroll
  for (int nx = 0; nx < F::MX; ++nx) {
    const double f = sB * Xr[nx * K::NROW];  // 0 outside the mesh; X = 0 on the boundary
#pragma unroll
    for (int c = 0; c < 3; ++c) acc[c][nx] *= f;
  }
  double* Sr = T + K::row(ny, nz);
#pragma unroll
  for (int lx = 0; lx < TX; ++lx)
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int m1 = 0; m1 < 2; ++m1) {
        double sv = 0.0;
#pragma unroll
        for (int ax = 0; ax < 3; ++ax)
          if (x2_nz(c, ax, m1)) sv = fma(c_X2[c][ax][m1], acc[c][2 * lx + ax], sv);
        Sr[K::sidx(c, m1, lx)] = sv;
      }
}

// Paired pencils (option "k2_pair"): the class-(0, RZ) pencil at (jy, jz) reads the element
// rows qy = jy, jy + 1; the class-(1, RZ) pencil at the same (jy, jz) reads qy = jy + 1 only,
// a subset.  One thread computes both from the same Ps loads (about 30 % fewer step-1 Ps reads
// per tile), with two accumulator rows.  hasB: jy < TY (the class-(1, RZ) pencil exists).
template <int TX, int TY, int TZ>
__device__ __forceinline__ void fkt_row_out(double (&acc)[3][FK2<TX, TY, TZ>::MX], double* __restrict__ T,
                                            const double* __restrict__ Xs, int ny, int nz, double sB) {
  using F = FK2<TX, TY, TZ>;
  using K = FKT<TX, TY, TZ>;
  const double* Xr = Xs + K::row(ny, nz);
#pragma unroll
  for (int nx = 0; nx < F::MX; ++nx) {
    const double f = sB * Xr[nx * K::NROW];
#pragma unroll
    for (int c = 0; c < 3; ++c) acc[c][nx] *= f;
  }
  double* Sr = T + K::row(ny, nz);
#pragma unroll
  for (int lx = 0; lx < TX; ++lx)
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int m1 = 0; m1 < 2; ++m1) {
        double sv = 0.0;
#pragma unroll
        for (int ax = 0; ax < 3; ++ax)
          if (x2_nz(c, ax, m1)) sv = fma(c_X2[c][ax][m1], acc[c][2 * lx + ax], sv);
        Sr[K::sidx(c, m1, lx)] = sv;
      }
}
template <int TX, int TY, int TZ, int RZ>
__device__ __forceinline__ void fkt_pencil2(const double* __restrict__ Ps, double* __restrict__ T,
                                            const double* __restrict__ Xs, int jy, int jz, double sB, bool hasB) {
  using F = FK2<TX, TY, TZ>;
  using K = FKT<TX, TY, TZ>;
  const int nz = 2 * jz + RZ;
  double accA[3][F::MX], accB[3][F::MX];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int nx = 0; nx < F::MX; ++nx) accA[c][nx] = accB[c][nx] = 0.0;
#pragma unroll
  for (int qx = 0; qx < K::HX; ++qx) {
    double WA[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}}, WB[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
    for (int iz = 0; iz < (RZ ? 1 : 2); ++iz) {
      const int qz = RZ ? jz + 1 : jz + iz;
      const int az = RZ ? 1 : (iz == 0 ? 2 : 0);
#pragma unroll
      for (int iy = 0; iy < 2; ++iy) {
        const int qy = jy + iy;
        const int ay = iy == 0 ? 2 : 0;
        const int h = K::pidx(qx, qy, qz);
        const double p000 = Ps[h], p100 = Ps[K::NHP + h], p010 = Ps[2 * K::NHP + h], p001 = Ps[3 * K::NHP + h];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          if (w2_nz(c, ay, az, 0)) {
            WA[c][0] = fma(c_W2[c][ay][az][0], p000, WA[c][0]);
            WA[c][1] = fma(c_W2[c][ay][az][0], p100, WA[c][1]);
          }
          if (w2_nz(c, ay, az, 1)) WA[c][0] = fma(c_W2[c][ay][az][1], p010, WA[c][0]);
          if (w2_nz(c, ay, az, 2)) WA[c][0] = fma(c_W2[c][ay][az][2], p001, WA[c][0]);
          if (iy == 1) {  // the class-(1, RZ) pencil: local y node 1 of element qy = jy + 1
            if (w2_nz(c, 1, az, 0)) {
              WB[c][0] = fma(c_W2[c][1][az][0], p000, WB[c][0]);
              WB[c][1] = fma(c_W2[c][1][az][0], p100, WB[c][1]);
            }
            if (w2_nz(c, 1, az, 1)) WB[c][0] = fma(c_W2[c][1][az][1], p010, WB[c][0]);
            if (w2_nz(c, 1, az, 2)) WB[c][0] = fma(c_W2[c][1][az][2], p001, WB[c][0]);
          }
        }
      }
    }
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      const int nx = 2 * qx - 2 + ax;
      if (nx < 0 || nx >= F::MX) continue;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        if (x2_nz(c, ax, 0)) {
          accA[c][nx] = fma(c_X2[c][ax][0], WA[c][0], accA[c][nx]);
          accB[c][nx] = fma(c_X2[c][ax][0], WB[c][0], accB[c][nx]);
        }
        if (x2_nz(c, ax, 1)) {
          accA[c][nx] = fma(c_X2[c][ax][1], WA[c][1], accA[c][nx]);
          accB[c][nx] = fma(c_X2[c][ax][1], WB[c][1], accB[c][nx]);
        }
      }
    }
  }
  fkt_row_out<TX, TY, TZ>(accA, T, Xs, 2 * jy, nz, sB);
  if (hasB) fkt_row_out<TX, TY, TZ>(accB, T, Xs, 2 * jy + 1, nz, sB);
}

// step 1 of the warp-specialised kernel: one pencil per consumer thread.  Not inlined, so
// the pencils get the registers to themselves (inlined into the tile loop, the loop state
// of step 2 is kept live across them and they spill under the 15-warp register cap).
template <int TX, int TY, int TZ>
__device__ __noinline__ void fkt_step1(const double* __restrict__ Pc, double* __restrict__ T,
                                       const double* __restrict__ Xs, double sB) {
  using F = FK2<TX, TY, TZ>;
  const int t = threadIdx.x;
  if (t < F::OFF1) {
    if (t < F::cls_n(0, 0)) fkt_pencil<TX, TY, TZ, 0, 0>(Pc, T, Xs, t % (TY + 1), t / (TY + 1), sB);
  } else if (t < F::OFF2) {
    const int i = t - F::OFF1;
    if (i < F::cls_n(1, 0)) fkt_pencil<TX, TY, TZ, 1, 0>(Pc, T, Xs, i / (TZ + 1), i % (TZ + 1), sB);
  } else if (t < F::OFF3) {
    const int i = t - F::OFF2;
    if (i < F::cls_n(0, 1)) fkt_pencil<TX, TY, TZ, 0, 1>(Pc, T, Xs, i % (TY + 1), i / (TY + 1), sB);
  } else {
    const int i = t - F::OFF3;
    if (i < F::cls_n(1, 1)) fkt_pencil<TX, TY, TZ, 1, 1>(Pc, T, Xs, i % TY, i / TY, sB);
  }
}

// step 2 of the warp-specialised kernel (q = sB Bt^T t per element, p_new, <p, q>),
// not inlined for the same reason; returns dot + this thread's terms
template <int TX, int TY, int TZ>
__device__ __noinline__ double fkt_step2(const double* __restrict__ Pc, const double* __restrict__ T,
                                         double* __restrict__ q, double* __restrict__ pnew, PLay L, int ex0, int ey0,
                                         int ez0, int N, double sB, double dot) {
  using F = FK2<TX, TY, TZ>;
  using K = FKT<TX, TY, TZ>;
  if (threadIdx.x >= F::NE) return dot;
  const int lx = threadIdx.x % TX, ly = (threadIdx.x / TX) % TY, lz = threadIdx.x / (TX * TY);
  const int ex = ex0 + lx, ey = ey0 + ly, ez = ez0 + lz;
  if (ex >= N || ey >= N || ez >= N) return dot;
  double qm[4] = {0.0, 0.0, 0.0, 0.0};
  const double* Sb = T + lx * K::TC;
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int az = 0; az < 3; ++az)
#pragma unroll
      for (int ay = 0; ay < 3; ++ay) {
        const double* Se = Sb + K::sidx(c, 0, 0) + K::row(2 * ly + ay, 2 * lz + az);
        const double s0 = Se[0];
        if (w2_nz(c, ay, az, 0)) {
          const double s1 = Se[K::sidx(0, 1, 0)];
          qm[0] = fma(c_W2[c][ay][az][0], s0, qm[0]);
          qm[1] = fma(c_W2[c][ay][az][0], s1, qm[1]);
        }
        if (w2_nz(c, ay, az, 1)) qm[2] = fma(c_W2[c][ay][az][1], s0, qm[2]);
        if (w2_nz(c, ay, az, 2)) qm[3] = fma(c_W2[c][ay][az][2], s0, qm[3]);
      }
  const int h = K::pidx(lx + 1, ly + 1, lz + 1);
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const double o = sB * qm[m];
    const double pv = Pc[m * K::NHP + h];
    const int64_t j = L.at(m, ex, ey, ez);
    q[j] = o;
    pnew[j] = pv;
    dot = fma(pv, o, dot);
  }
  return dot;
}

// Same contract as k_K2_fused (mode, ctl, partials), tensor maps instead of pointers for the
// loads: tm_pold / tm_r / tm_minv over [m][ez][ey][ex]; X from its tile-blocked pencil layout XT.
// ZB: the PCG update kernels store z = Minv r and the kernel loads a z box; else it
// loads r and Minv boxes and forms Minv r itself (same product either way).
template <int TX, int TY, int TZ, int MINB, bool ZB, bool PAIR = false>
__global__ void __launch_bounds__(FK2<TX, TY, TZ>::NTH, MINB)
    k_K2_tma(const __grid_constant__ CUtensorMap tm_pold, const __grid_constant__ CUtensorMap tm_z,
             const __grid_constant__ CUtensorMap tm_minv, const double* __restrict__ XT,
             double* __restrict__ pnew, double* __restrict__ q, Geo G, double sB, int mode, int it, int ctl,
             const double* __restrict__ rzp, int nrz, double* rz_hist, const double* pq_hist, int* stop,
             double* pqp, PLay L) {
  using F = FK2<TX, TY, TZ>;
  using K = FKT<TX, TY, TZ>;
#ifdef WB_KPROF
  const bool tl = (mode & 0x4000) && it == 5 && threadIdx.x == 0 && blockIdx.x < 512;
  if (tl) g_ktl[blockIdx.x][0] = gtimer();
#endif
  // offsets from the (1024-aligned) dynamic shared base itself, so that every access
  // below stays a shared-space access (LDS/STS), not a generic one
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sb = smraw;
  double* Pb = (double*)(sb + K::OFF_P);  // raw boxes [m][hx][hz][hy]
  double* Zb = (double*)(sb + K::OFF_R);  // z = Minv r (ZB), else r
  double* Mb = (double*)(sb + K::OFF_M);  // Minv (!ZB)
  constexpr unsigned RAWB = (ZB ? 2u : 3u) * K::PBYTES;
  double* Ps = (double*)(sb + K::OFF_S);  // p on the tile + halo, rows of F::PX
  double* Xs = (double*)(sb + K::OFF_X);
  double* T = (double*)(sb + K::OFF_T);
  uint64_t* bar = (uint64_t*)(sb + K::OFF_B);  // [0] r+Minv, [1] p_old, [2] X
  const int N = G.N;
  const int NTX = (N + TX - 1) / TX, NTY = (N + TY - 1) / TY, NTZ = (N + TZ - 1) / TZ;
  const int n_tiles = NTX * NTY * NTZ;
  auto coords = [&](int tile, int& ex0, int& ey0, int& ez0) {
    ex0 = TX * (tile % NTX); ey0 = TY * ((tile / NTX) % NTY); ez0 = TZ * (tile / (NTX * NTY));
  };
  // first tile's loads first: they do not depend on the control scalars, so the
  // reduction of the previous kernel's partials below overlaps them
  int tile = blockIdx.x;
  // mode 2 (q = K p_old as is): only the p box is loaded and p_new is not stored
  const bool pz = (mode & 0xff) != 2;
  const unsigned rawb = pz ? RAWB : K::PBYTES;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); mbar_init(&bar[2], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (tile < n_tiles) {
      int ex0, ey0, ez0;
      coords(tile, ex0, ey0, ez0);
      mbar_expect_tx(&bar[0], rawb);
      if (pz) tma_load_4d(Zb, &tm_z, ey0, ez0 - 1, ex0 - 1, 0, &bar[0]);  // y from ey0 - 1 + pad
      if (pz && !ZB) tma_load_4d(Mb, &tm_minv, ey0, ez0 - 1, ex0 - 1, 0, &bar[0]);
      tma_load_4d(Pb, &tm_pold, ey0, ez0 - 1, ex0 - 1, 0, &bar[0]);
      mbar_expect_tx(&bar[2], K::XBYTES);
      bulk_load(Xs, XT + (size_t)tile * K::XTB, K::XBYTES, &bar[2]);
    }
  }
  // timing probe bits (option k_dbg; results invalid): 0x100 skip step 1, 0x200 skip
  // step 2, 0x400 skip step 0's arithmetic and stores, 0x800 skip the q stores, 0x1000
  // skip the p_new stores, 0x2000 never stop
  const int dbg = mode & 0xff00;
  mode &= 0xff;
  double beta = 0.0;
  if (ctl) {
    if (pcg_control<F::NTH>(it, rzp, nrz, rz_hist, pq_hist, stop, &beta) && !(dbg & 0x2000)) {
      // stopped: drain the bulk copies in flight before the CTA exits
      if (threadIdx.x == 0 && tile < n_tiles) { mbar_wait(&bar[0], 0); mbar_wait(&bar[2], 0); }
      return;
    }
  } else if (mode == 1) {
    beta = rz_hist[it] / rz_hist[it - 1];
  }
  __syncthreads();  // barrier init visible to all threads (pcg_control ends with one too)
#ifdef WB_KPROF  // phase timers (tools/kphase.py builds with -DWB_KPROF)
  const bool prof = (dbg & 0x4000) && threadIdx.x == 0;
  unsigned long long pt[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // [7]: TMA issue after step 0
  long long tc = clock64();
  auto lap = [&](int k) {
    if (prof) { const long long n = clock64(); pt[k] += (unsigned long long)(n - tc); tc = n; }
  };
#else
  constexpr bool prof = false;
  unsigned long long pt[8];
  auto lap = [](int) {};
#endif
  lap(0);
#ifdef WB_KPROF
  if (tl) g_ktl[blockIdx.x][1] = gtimer();
#endif
  double dot = 0.0;
  // tile coordinates without divisions in the loop (the runtime div / mod chains ran on every
  // warp at the top of each tile with nothing to overlap them): the stride gridDim.x is
  // decomposed once, then each step adds it with carries
  const int cp_q = (threadIdx.x >> 4) / 5, cp_s = (threadIdx.x >> 4) % 5, cp_l = threadIdx.x & 15;  // step-0 item
  int sx, sy, sz, nx0, ny0, nz0;
  coords(gridDim.x, sx, sy, sz);  // = (TX tx, TY ty, TZ tz) of the stride
  coords(tile, nx0, ny0, nz0);
  const int LX = TX * NTX, LY = TY * NTY;
  for (int k = 0; tile < n_tiles; ++k, tile += gridDim.x) {
    const unsigned ph = k & 1;
    const int next = tile + gridDim.x;
    const int ex0 = nx0, ey0 = ny0, ez0 = nz0;
    nx0 += sx;
    if (nx0 >= LX) { nx0 -= LX; ny0 += TY; }
    ny0 += sy;
    if (ny0 >= LY) { ny0 -= LY; nz0 += TZ; }
    nz0 += sz;
    // 0. p = Minv r (+ beta p_old) from the raw boxes into Ps (the element step stores the
    // tile's own p_new)
    mbar_wait(&bar[0], ph);
    lap(1);
    // the raw box is [m][hx][hz][hy] = Ps's order with row length HY instead of QS:
    // a flat, lane-consecutive walk
    {
      // item t = threadIdx.x + i NTH: half-warp h = t / 16 takes pair column h % 5 of rows
      // 16 (h / 5) + (t % 16); h advances by NTH / 16 per pass
      constexpr int DH = F::NTH / 16, DQ = DH / 5, DS = DH % 5;
      static_assert(F::NTH % 16 == 0, "pass stride in whole half-warps");
      int rq = cp_q, sp = cp_s;
      for (int t = threadIdx.x; t < ((dbg & 0x400) ? 0 : 2 * K::NB); t += F::NTH) {
        fkt_copy_pair_rs<TX, TY, TZ, ZB>(16 * rq + cp_l, sp, Pb, Zb, Mb, Ps, mode, beta);
        sp += DS; rq += DQ;
        if (sp >= 5) { sp -= 5; ++rq; }
      }
    }
    __syncthreads();
    lap(2);
    if (threadIdx.x == K::TMA_T && next < n_tiles) {  // raw p, r, Minv buffers are free
      fence_proxy_async();
      mbar_expect_tx(&bar[0], rawb);
      if (pz) tma_load_4d(Zb, &tm_z, ny0, nz0 - 1, nx0 - 1, 0, &bar[0]);
      if (pz && !ZB) tma_load_4d(Mb, &tm_minv, ny0, nz0 - 1, nx0 - 1, 0, &bar[0]);
      tma_load_4d(Pb, &tm_pold, ny0, nz0 - 1, nx0 - 1, 0, &bar[0]);
    }
    lap(7);
    // 1. t at the tile nodes by x-pencils
    mbar_wait(&bar[2], ph);
    lap(3);
    if (PAIR && !(dbg & 0x100)) {
      // paired pencils: threads [0, (TY+1)(TZ+1)) the class-(0,0) + (1,0) pairs, then, from
      // the next warp boundary, the class-(0,1) + (1,1) pairs
      const int t = threadIdx.x;
      constexpr int P0 = (TY + 1) * (TZ + 1), O1 = (P0 + 31) / 32 * 32, P1 = (TY + 1) * TZ;
      if (t < P0) fkt_pencil2<TX, TY, TZ, 0>(Ps, T, Xs, t % (TY + 1), t / (TY + 1), sB, t % (TY + 1) < TY);
      else if (t >= O1 && t < O1 + P1) {
        const int i = t - O1;
        fkt_pencil2<TX, TY, TZ, 1>(Ps, T, Xs, i % (TY + 1), i / (TY + 1), sB, i % (TY + 1) < TY);
      }
    } else if (!(dbg & 0x100)) {
      const int t = threadIdx.x;
      if (t < F::OFF1) {
        if (t < F::cls_n(0, 0)) fkt_pencil<TX, TY, TZ, 0, 0>(Ps, T, Xs, t % (TY + 1), t / (TY + 1), sB);
      } else if (t < F::OFF2) {
        const int i = t - F::OFF1;
        if (i < F::cls_n(1, 0)) fkt_pencil<TX, TY, TZ, 1, 0>(Ps, T, Xs, i / (TZ + 1), i % (TZ + 1), sB);
      } else if (t < F::OFF3) {
        const int i = t - F::OFF2;
        if (i < F::cls_n(0, 1)) fkt_pencil<TX, TY, TZ, 0, 1>(Ps, T, Xs, i % (TY + 1), i / (TY + 1), sB);
      } else {
        const int i = t - F::OFF3;
        if (i < F::cls_n(1, 1)) fkt_pencil<TX, TY, TZ, 1, 1>(Ps, T, Xs, i % TY, i / TY, sB);
      }
    }
    __syncthreads();
    lap(4);
    if (threadIdx.x == K::TMA_T && next < n_tiles) {  // X buffer is free
      fence_proxy_async();
      mbar_expect_tx(&bar[2], K::XBYTES);
      bulk_load(Xs, XT + (size_t)next * K::XTB, K::XBYTES, &bar[2]);
    }
    // 2. q = sB Bt^T t per element, <p, q>
    if (threadIdx.x < F::NE && !(dbg & 0x200)) {
      const int lx = threadIdx.x % TX, ly = (threadIdx.x / TX) % TY, lz = threadIdx.x / (TX * TY);
      const int ex = ex0 + lx, ey = ey0 + ly, ez = ez0 + lz;
      if (ex < N && ey < N && ez < N) {
        // (y, z) contraction of the row sums: q_000 += W0 S[0], q_100 += W0 S[1],
        // q_010 += W1 S[0], q_001 += W2 S[0]  (W = c_W2[c][ay][az], exact zeros skipped)
        double qm[4] = {0.0, 0.0, 0.0, 0.0};
        const double* Sb = T + lx * K::TC;
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int az = 0; az < 3; ++az)
#pragma unroll
            for (int ay = 0; ay < 3; ++ay) {
              const double* Se = Sb + K::sidx(c, 0, 0) + K::row(2 * ly + ay, 2 * lz + az);
              const double s0 = Se[0];
              if (w2_nz(c, ay, az, 0)) {
                const double s1 = Se[K::sidx(0, 1, 0)];
                qm[0] = fma(c_W2[c][ay][az][0], s0, qm[0]);
                qm[1] = fma(c_W2[c][ay][az][0], s1, qm[1]);
              }
              if (w2_nz(c, ay, az, 1)) qm[2] = fma(c_W2[c][ay][az][1], s0, qm[2]);
              if (w2_nz(c, ay, az, 2)) qm[3] = fma(c_W2[c][ay][az][2], s0, qm[3]);
            }
        const int h = K::pidx(lx + 1, ly + 1, lz + 1);
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const double o = sB * qm[m];
          const double pv = Ps[m * K::NHP + h];
          const int64_t j = L.at(m, ex, ey, ez);
          if (!(dbg & 0x800)) q[j] = o;
          if (pz && !(dbg & 0x1000)) pnew[j] = pv;
          dot = fma(pv, o, dot);
        }
      }
    }
    __syncthreads();  // Ps, T are rewritten by the next tile
    lap(5);
    if (prof) ++pt[6];
  }
  if (prof)
    for (int k = 0; k < 8; ++k) atomicAdd(&g_kprof[k], pt[k]);
#ifdef WB_KPROF
  if (tl) g_ktl[blockIdx.x][2] = gtimer();
#endif
  store_partial<F::NTH>(dot, pqp);
#ifdef WB_KPROF
  if (tl) g_ktl[blockIdx.x][3] = gtimer();
#endif
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// barrier over a subset of the CTA's warps (ids 1, 2; 0 is __syncthreads)
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// Warp-specialised variant of k_K2_tma: the same three steps and arithmetic, but step 0
// (p = Minv r + beta p_old into Ps) runs in PW producer warps one tile ahead of the
// consumer warps, which run steps 1 and 2.  Ps is double-buffered without extra shared
// memory: buffer 1 sits in the padding of buffer 0's rows (offset HY in each QS-row, and
// QS >= 2 HY), so both keep the conflict-free pencil reads.  Handshake per Ps buffer:
// full[b] (producers arrive after writing), empty[b] (consumer thread 0 arrives after
// the tile's step 2).  The raw p / r / Minv boxes stay single-buffered: the producers
// issue the next tile's loads as soon as they have read them, which is a whole
// consumer tile before they are needed.  X stays with the consumers (loaded after step 1).
#ifndef WS_PW
#define WS_PW 4  // producer warps of k_K2_ws
#endif
template <int TX, int TY, int TZ>
struct FKW {
  using F = FK2<TX, TY, TZ>;
  using K = FKT<TX, TY, TZ>;
  static constexpr int PW = WS_PW, CNTH = F::NTH, PNTH = 32 * PW, NTH = CNTH + PNTH;
  static constexpr int OFFB = K::HY;  // second Ps buffer
  static_assert(K::QS >= 2 * K::HY, "both Ps buffers fit in one padded row");
  static constexpr size_t SMEM = K::SMEM;  // the 6 mbarriers fit in the 64-byte barrier slot
};

template <int TX, int TY, int TZ, bool ZB>
__global__ void __launch_bounds__(FKW<TX, TY, TZ>::NTH, 1)
    k_K2_ws(const __grid_constant__ CUtensorMap tm_pold, const __grid_constant__ CUtensorMap tm_z,
            const __grid_constant__ CUtensorMap tm_minv, const double* __restrict__ XT, double* __restrict__ pnew,
            double* __restrict__ q, Geo G, double sB, int mode, int it, int ctl, const double* __restrict__ rzp,
            int nrz, double* rz_hist, const double* pq_hist, int* stop, double* pqp, PLay L) {
  using F = FK2<TX, TY, TZ>;
  using K = FKT<TX, TY, TZ>;
  using W = FKW<TX, TY, TZ>;
  const int mode_in = mode;
#ifdef WB_KPROF
  const bool tl = (mode & 0x4000) && it == 5 && threadIdx.x == 0 && blockIdx.x < 512;
  if (tl) g_ktl[blockIdx.x][0] = gtimer();
#endif
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sb = smraw;
  double* Pb = (double*)(sb + K::OFF_P);
  double* Zb = (double*)(sb + K::OFF_R);
  double* Mb = (double*)(sb + K::OFF_M);
  constexpr unsigned RAWB = (ZB ? 2u : 3u) * K::PBYTES;
  double* Ps = (double*)(sb + K::OFF_S);
  double* Xs = (double*)(sb + K::OFF_X);
  double* T = (double*)(sb + K::OFF_T);
  uint64_t* bar = (uint64_t*)(sb + K::OFF_B);  // [0] raw boxes, [1] X, [2, 3] full, [4, 5] empty
  const int N = G.N;
  const int NTX = (N + TX - 1) / TX, NTY = (N + TY - 1) / TY, NTZ = (N + TZ - 1) / TZ;
  const int n_tiles = NTX * NTY * NTZ;
  auto coords = [&](int tile, int& ex0, int& ey0, int& ez0) {
    ex0 = TX * (tile % NTX); ey0 = TY * ((tile / NTX) % NTY); ez0 = TZ * (tile / (NTX * NTY));
  };
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1); mbar_init(&bar[1], 1);
    mbar_init(&bar[2], W::PNTH); mbar_init(&bar[3], W::PNTH);
    mbar_init(&bar[4], 1); mbar_init(&bar[5], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const int tile = blockIdx.x;
    if (tile < n_tiles) {
      int ex0, ey0, ez0;
      coords(tile, ex0, ey0, ez0);
      mbar_expect_tx(&bar[0], RAWB);
      tma_load_4d(Zb, &tm_z, ey0, ez0 - 1, ex0 - 1, 0, &bar[0]);
      if (!ZB) tma_load_4d(Mb, &tm_minv, ey0, ez0 - 1, ex0 - 1, 0, &bar[0]);
      tma_load_4d(Pb, &tm_pold, ey0, ez0 - 1, ex0 - 1, 0, &bar[0]);
      mbar_expect_tx(&bar[1], K::XBYTES);
      bulk_load(Xs, XT + (size_t)tile * K::XTB, K::XBYTES, &bar[1]);
    }
  }
  mode &= 0xff;
  double beta = 0.0;
  if (ctl) {
    if (pcg_control<W::NTH>(it, rzp, nrz, rz_hist, pq_hist, stop, &beta)) {
      if (threadIdx.x == 0 && (int)blockIdx.x < n_tiles) { mbar_wait(&bar[0], 0); mbar_wait(&bar[1], 0); }
      return;
    }
  } else if (mode == 1) {
    beta = rz_hist[it] / rz_hist[it - 1];
  }
  __syncthreads();
#ifdef WB_KPROF
  if (tl) g_ktl[blockIdx.x][1] = gtimer();
  // role probes (k_dbg 0x4000; tools/wsphase.py), cycles into g_kprof: consumer thread 0
  // [0] wait full, [1] wait X, [2] step 1 + barrier, [3] step 2 + barrier, [7] tiles;
  // producer thread 0 [4] wait empty, [5] wait raw boxes, [6] step 0 + barrier
  const bool prof = (mode_in & 0x4000) && (threadIdx.x == 0 || threadIdx.x == W::CNTH);
  unsigned long long pt_[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tc = clock64();
  auto lap = [&](int k) {
    if (prof) { const long long n = clock64(); pt_[k] += (unsigned long long)(n - tc); tc = n; }
  };
#else
  auto lap = [](int) {};
#endif
  double dot = 0.0;
  if (threadIdx.x >= W::CNTH) {
    // ---- producers: step 0 for tile k into Ps buffer k & 1
    const int pt = threadIdx.x - W::CNTH;
    int k = 0;
#pragma unroll 1
    for (int tile = blockIdx.x; tile < n_tiles; ++k, tile += gridDim.x) {
      const int b = k & 1;
      lap(6);
      if (k >= 2) mbar_wait(&bar[4 + b], ((k >> 1) - 1) & 1);
      lap(4);
      mbar_wait(&bar[0], k & 1);
      lap(5);
      double* Pd = Ps + b * W::OFFB;
#pragma unroll 4
      for (int t = pt; t < ((mode_in & 0x400) ? 0 : 2 * K::NB); t += W::PNTH)
        fkt_copy_pair<TX, TY, TZ, ZB>(t, Pb, Zb, Mb, Pd, mode, beta);
      named_bar(2, W::PNTH);  // raw boxes consumed
      const int next = tile + gridDim.x;
      if (pt == 0 && next < n_tiles) {
        int nx0, ny0, nz0;
        coords(next, nx0, ny0, nz0);
        fence_proxy_async();
        mbar_expect_tx(&bar[0], RAWB);
        tma_load_4d(Zb, &tm_z, ny0, nz0 - 1, nx0 - 1, 0, &bar[0]);
        if (!ZB) tma_load_4d(Mb, &tm_minv, ny0, nz0 - 1, nx0 - 1, 0, &bar[0]);
        tma_load_4d(Pb, &tm_pold, ny0, nz0 - 1, nx0 - 1, 0, &bar[0]);
      }
      mbar_arrive(&bar[2 + b]);
    }
  } else {
    // ---- consumers: steps 1 and 2 for tile k from Ps buffer k & 1
    int k = 0;
#pragma unroll 1
    for (int tile = blockIdx.x; tile < n_tiles; ++k, tile += gridDim.x) {
      const int b = k & 1;
      const double* Pc = Ps + b * W::OFFB;
      const int next = tile + gridDim.x;
      int ex0, ey0, ez0;
      coords(tile, ex0, ey0, ez0);
      lap(3);
      mbar_wait(&bar[2 + b], (k >> 1) & 1);
      lap(0);
      mbar_wait(&bar[1], k & 1);
      lap(1);
      fkt_step1<TX, TY, TZ>(Pc, T, Xs, sB);
      named_bar(1, W::CNTH);
      lap(2);
      if (threadIdx.x == K::TMA_T && next < n_tiles) {  // X buffer is free
        fence_proxy_async();
        mbar_expect_tx(&bar[1], K::XBYTES);
        bulk_load(Xs, XT + (size_t)next * K::XTB, K::XBYTES, &bar[1]);
      }
      dot = fkt_step2<TX, TY, TZ>(Pc, T, q, pnew, L, ex0, ey0, ez0, N, sB, dot);
      named_bar(1, W::CNTH);  // T and Ps buffer b are free
      if (threadIdx.x == 0) mbar_arrive(&bar[4 + b]);
#ifdef WB_KPROF
      if (prof) ++pt_[7];
#endif
    }
    lap(3);
  }
#ifdef WB_KPROF
  lap(6);
  if (prof)
    for (int j = 0; j < 8; ++j)
      if (pt_[j]) atomicAdd(&g_kprof[j], pt_[j]);
  if (tl) g_ktl[blockIdx.x][2] = gtimer();
#endif
  store_partial<W::NTH>(dot, pqp);  // producers add 0.0: same sums as k_K2_tma's 11 warps
#ifdef WB_KPROF
  if (tl) g_ktl[blockIdx.x][3] = gtimer();
#endif
}

// XT[tile][nx][row(ny, nz)] = X(2 ex0 + nx, 2 ey0 + ny, 2 ez0 + nz), 0 outside the mesh
// (the pencil layout of the TMA kernel's X block), both sides (L: C_w^-1, R: D_w^-1).
// One CTA per tile, one thread per node row (ny, nz): 2 x MX contiguous reads.
template <int TX, int TY, int TZ>
__global__ void __launch_bounds__(FK2<TX, TY, TZ>::MY * FK2<TX, TY, TZ>::MZ)
    k_x_tiles(const double* __restrict__ XL, const double* __restrict__ XR, double* __restrict__ XTL,
              double* __restrict__ XTR, int N) {
  using F = FK2<TX, TY, TZ>;
  using K = FKT<TX, TY, TZ>;
  const int nn1 = 2 * N + 1;
  const int NTX = (N + TX - 1) / TX, NTY = (N + TY - 1) / TY;
  const int tile = blockIdx.x;
  const int tx = tile % NTX, ty = (tile / NTX) % NTY, tz = tile / (NTX * NTY);
  const int ny = threadIdx.x % F::MY, nz = threadIdx.x / F::MY;
  const int gx0 = 2 * TX * tx, gy = 2 * TY * ty + ny, gz = 2 * TZ * tz + nz;
  const bool rowok = gy < nn1 && gz < nn1;
  const int64_t src = gx0 + (int64_t)nn1 * (gy + (int64_t)nn1 * gz);
  const int64_t dst = (int64_t)tile * K::XTB + K::row(ny, nz);
#pragma unroll
  for (int nx = 0; nx < F::MX; ++nx) {
    const bool ok = rowok && gx0 + nx < nn1;
    XTL[dst + nx * K::NROW] = ok ? XL[src + nx] : 0.0;
    XTR[dst + nx * K::NROW] = ok ? XR[src + nx] : 0.0;
  }
}

}  // namespace wb
