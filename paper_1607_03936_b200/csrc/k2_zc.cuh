// k2_zc.cuh -- B and B^T for k = 2 (rows a6, a7) by z-marching columns (option "bbt_zc"; the
// default on meshes with N >= 48: C5 B 34.9 -> 28.7 us, B^T 36.8 -> 33.7 us, L2 flushed; on C3
// the tile / box kernels stay faster, B 11 vs 23 us).
//
// The element matrix factorises into 1-D integrals, B_e[(m1,m2,m3),(c,a)] = sB prod_d
// M_cd[m_d][a_d] (M_cd = BD on the component's own axis, else BI; the k = 2 modes are
// (0,0,0), (1,0,0), (0,1,0), (0,0,1) in the R2 order).  A thread owns one column of the mesh
// and a chunk of CZ element layers along z and walks the node layers upwards, keeping
// the z-contraction in registers, so every velocity value is loaded (B) or stored (B^T) once
// per column with the warp's lanes on consecutive x:
//   B:   thread (ex, ey): per node layer gz, the 3 x 3 node rows of the element column are
//        contracted along x, then y (x-lanes read consecutive nodes), and added into the
//        element(s) containing the layer with the z weights; p_e is stored when complete.
//   B^T: thread (gx, gy): per element layer ez, the <= 4 elements around the column are
//        contracted along x and y into two numbers per component (m3 = 0 and 1); each node
//        of the column is then the z-combination of the two element layers around it.
// Every output is a fixed-order sum: bitwise reproducible.
#pragma once
#include "kernels.cuh"

namespace wb {

__device__ __forceinline__ double k2m(bool d, int m, int a) { return d ? TB(2).BD[m][a] : TB(2).BI[m][a]; }

// p[e se + m sm] = sB B (s o u), s = xs, else the Dirichlet mask (unless nomask)
template <int CZ>
__global__ void __launch_bounds__(128) k_B_zc2(const double* __restrict__ u, const double* __restrict__ xs,
                                               double* __restrict__ p, Geo G, double sB, int nomask, int64_t se,
                                               int64_t sm) {
  const int N = G.N, nn1 = G.nn1;
  const int nch = (N + CZ - 1) / CZ;
  const int64_t tid = (int64_t)blockIdx.x * 128 + threadIdx.x;
  if (tid >= (int64_t)N * N * nch) return;
  const int ex = (int)(tid % N), ey = (int)((tid / N) % N), cz = (int)(tid / ((int64_t)N * N));
  const int ez0 = cz * CZ, ez1 = min(N, ez0 + CZ);
  const int gx0 = 2 * ex, gy0 = 2 * ey;
  // element ez accumulates layers 2ez..2ez+2 in acc0 (ez even) or acc1 (ez odd)
  double acc0[4] = {0.0, 0.0, 0.0, 0.0}, acc1[4] = {0.0, 0.0, 0.0, 0.0};
  const int64_t nn2 = (int64_t)nn1 * nn1;
  // Dirichlet rows / columns of this element column (the z layers are checked per layer)
  bool bx[3], by[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    bx[a] = gx0 + a == 0 || gx0 + a == nn1 - 1;
    by[a] = gy0 + a == 0 || gy0 + a == nn1 - 1;
  }
  const int64_t col0 = (int64_t)gx0 + (int64_t)nn1 * gy0;
#pragma unroll 2
  for (int gz = 2 * ez0; gz <= 2 * ez1; ++gz) {
    // the layer's 3 x 3 node rows of this element column, all components
    const bool bz = gz == 0 || gz == nn1 - 1;
    double v[3][3][3];  // [c][ay][ax]
#pragma unroll
    for (int ay = 0; ay < 3; ++ay) {
      const int64_t row = col0 + (int64_t)ay * nn1 + gz * nn2;
#pragma unroll
      for (int ax = 0; ax < 3; ++ax) {
        double s = 1.0;
        if (xs) s = __ldg(xs + row + ax);
        else if (!nomask && (bx[ax] || by[ay] || bz)) s = 0.0;
#pragma unroll
        for (int c = 0; c < 3; ++c) v[c][ay][ax] = s * __ldg(u + (int64_t)c * G.n_nodes + row + ax);
      }
    }
    // x then y: Y[c][k], k = 0: (m1, m2) = (0, 0), 1: (1, 0), 2: (0, 1)
    double Y[3][3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      Y[c][0] = Y[c][1] = Y[c][2] = 0.0;
#pragma unroll
      for (int ay = 0; ay < 3; ++ay) {
        double X0 = 0.0, X1 = 0.0;
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
          X0 = fma(k2m(c == 0, 0, ax), v[c][ay][ax], X0);
          X1 = fma(k2m(c == 0, 1, ax), v[c][ay][ax], X1);
        }
        Y[c][0] = fma(k2m(c == 1, 0, ay), X0, Y[c][0]);
        Y[c][1] = fma(k2m(c == 1, 0, ay), X1, Y[c][1]);
        Y[c][2] = fma(k2m(c == 1, 1, ay), X0, Y[c][2]);
      }
    }
    // z: the layer is local node az = gz - 2 ez of element ez = gz / 2 (az 0, 1) and, if
    // gz is even, node 2 of element gz / 2 - 1
    const int ezu = gz >> 1;
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      const int ez = side == 0 ? ezu : ezu - 1;
      const int az = gz - 2 * ez;
      if (ez < ez0 || ez >= ez1 || az > 2) continue;
      auto add = [&](double (&A)[4]) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double w0 = k2m(c == 2, 0, az), w1 = k2m(c == 2, 1, az);
          A[0] = fma(w0, Y[c][0], A[0]);
          A[1] = fma(w0, Y[c][1], A[1]);
          A[2] = fma(w0, Y[c][2], A[2]);
          A[3] = fma(w1, Y[c][0], A[3]);
        }
        if (az == 2) {  // element ez complete
          const int64_t e = ex + (int64_t)N * (ey + (int64_t)N * ez);
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            p[e * se + m * sm] = sB * A[m];
            A[m] = 0.0;
          }
        }
      };
      if (ez & 1) add(acc1);
      else add(acc0);
    }
  }
}

// y = s o B^T p, s = xs, else the Dirichlet mask (unless nomask); p[e se + m sm]
template <int CZ>
__global__ void __launch_bounds__(128) k_BT_zc2(const double* __restrict__ p, const double* __restrict__ xs,
                                                double* __restrict__ y, Geo G, double sB, int nomask, int64_t se,
                                                int64_t sm) {
  const int N = G.N, nn1 = G.nn1;
  const int nch = (N + CZ - 1) / CZ;
  const int64_t tid = (int64_t)blockIdx.x * 128 + threadIdx.x;
  if (tid >= (int64_t)nn1 * nn1 * nch) return;
  const int gx = (int)(tid % nn1), gy = (int)((tid / nn1) % nn1), cz = (int)(tid / ((int64_t)nn1 * nn1));
  const int ez0 = cz * CZ, ez1 = min(N, ez0 + CZ);
  const int gz0 = 2 * ez0, gz1 = (ez1 == N) ? 2 * N : 2 * ez1 - 1;  // node layers of this chunk
  // the <= 2 x 2 elements around the column: (ex, ax) per axis, ax = local node index
  // slot 0: the lower element (local node 2) or, for an odd node, the element itself (node 1);
  // slot 1: the upper element (node 0), even nodes only
  const bool xodd = gx & 1, yodd = gy & 1;
  const int xe0 = xodd ? gx / 2 : gx / 2 - 1, xa0 = xodd ? 1 : 2, xe1 = gx / 2;
  const int ye0 = yodd ? gy / 2 : gy / 2 - 1, ya0 = yodd ? 1 : 2, ye1 = gy / 2;
  const bool xv0 = xe0 >= 0, xv1 = !xodd && xe1 < N, yv0 = ye0 >= 0, yv1 = !yodd && ye1 < N;
  // R[c][k] of element layer ez: the x-y contraction of its <= 4 elements around the column,
  // k = 0 the m3 = 0 modes, k = 1 the mode (0,0,1)
  auto layer = [&](int ez, double (&R)[3][2]) {
#pragma unroll
    for (int c = 0; c < 3; ++c) R[c][0] = R[c][1] = 0.0;
    if (ez < 0 || ez >= N) return;
#pragma unroll
    for (int iy = 0; iy < 2; ++iy) {
      if (!(iy == 0 ? yv0 : yv1)) continue;
#pragma unroll
      for (int ix = 0; ix < 2; ++ix) {
        if (!(ix == 0 ? xv0 : xv1)) continue;
        const int64_t e = (ix == 0 ? xe0 : xe1) + (int64_t)N * ((iy == 0 ? ye0 : ye1) + (int64_t)N * ez);
        const double p0 = __ldg(p + e * se), p1 = __ldg(p + e * se + sm), p2 = __ldg(p + e * se + 2 * sm),
                     p3 = __ldg(p + e * se + 3 * sm);
        const int ax = ix == 0 ? xa0 : 0, ay = iy == 0 ? ya0 : 0;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double x0 = k2m(c == 0, 0, ax), x1 = k2m(c == 0, 1, ax), y0 = k2m(c == 1, 0, ay),
                       y1 = k2m(c == 1, 1, ay);
          R[c][0] = fma(x0 * y0, p0, fma(x1 * y0, p1, fma(x0 * y1, p2, R[c][0])));
          R[c][1] = fma(x0 * y0, p3, R[c][1]);
        }
      }
    }
  };
  double Rlo[3][2], Rhi[3][2];  // element layers ez - 1 and ez around node layer 2 ez
  layer(ez0 - 1, Rlo);
  layer(ez0, Rhi);
  for (int gz = gz0; gz <= gz1; ++gz) {
    if (gz > gz0 && (gz & 1) == 0) {  // entering element layer gz / 2
#pragma unroll
      for (int c = 0; c < 3; ++c) { Rlo[c][0] = Rhi[c][0]; Rlo[c][1] = Rhi[c][1]; }
      layer(gz >> 1, Rhi);
    }
    const int64_t g = node_id(gx, gy, gz, nn1);
    double s = 1.0;
    if (xs) s = __ldg(xs + g);
    else if (!nomask && node_bnd(gx, gy, gz, nn1)) s = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double v;
      if (gz & 1) {  // interior node 1 of element gz / 2
        v = fma(k2m(c == 2, 0, 1), Rhi[c][0], k2m(c == 2, 1, 1) * Rhi[c][1]);
      } else {  // node 2 of the lower layer, then node 0 of the upper one
        v = fma(k2m(c == 2, 0, 2), Rlo[c][0], k2m(c == 2, 1, 2) * Rlo[c][1]);
        v = fma(k2m(c == 2, 0, 0), Rhi[c][0], fma(k2m(c == 2, 1, 0), Rhi[c][1], v));
      }
      y[(int64_t)c * G.n_nodes + g] = s * (sB * v);
    }
  }
}

}  // namespace wb
