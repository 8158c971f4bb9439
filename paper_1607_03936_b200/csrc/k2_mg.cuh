// k2_mg.cuh -- kernels of the geometric pressure multigrid for K_w (
// PAPER.md:2468-2546; reading R20), k = 2 (Q2 x P1disc):
//  * coarse weights by density injection: C_c[G] = C_f[iota(G)] * prod_d (G_d even ? 2 : 4)
//    -- the ratio M_c[G] / M_f[iota(G)] of the unweighted lumped masses (1-D vertex h/3,
//    mid-edge 2h/3 per unit weight, coarse h = 2 fine h), in closed form;
//  * transfers: the exact embedding of the coarse P1disc space in the fine one.  With the
//    orthonormal modes (1, L1(x), L1(y), L1(z)) on each reference element and the child
//    coordinate xi_c = (xi_f + s)/2, s = +-1 per axis, L1(xi_c) = L1(xi_f)/2 + (sqrt(3)/2)s L0:
//      fine f_0 = c_0 + (sqrt(3)/2)(s_x c_x + s_y c_y + s_z c_z),  f_d = c_d / 2;
//    restriction is the transpose (children summed in ascending s = sx + 2 sy + 4 sz);
//  * the splitmix64 start vector of the power iteration (same generator as the oracle).
#pragma once
#include "kernels.cuh"

namespace wb {

__device__ __forceinline__ double mg_sign(int s, int d) { return ((s >> d) & 1) ? 1.0 : -1.0; }

// coarse lumped masses of both sides from the fine ones (nodes of the coarse Q2 grid)
__global__ void k_mg_inject(const double* __restrict__ Cf, const double* __restrict__ Df, double* __restrict__ Cc,
                            double* __restrict__ Dc, int Nc) {
  const int nc = 2 * Nc + 1, nf = 4 * Nc + 1;
  const int64_t n = (int64_t)nc * nc * nc;
  for (int64_t G = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; G < n; G += (int64_t)gridDim.x * blockDim.x) {
    const int gx = (int)(G % nc), gy = (int)((G / nc) % nc), gz = (int)(G / ((int64_t)nc * nc));
    const int64_t f = (int64_t)(2 * gx) + (int64_t)nf * ((int64_t)(2 * gy) + (int64_t)nf * (2 * gz));
    const double r = ((gx & 1) ? 4.0 : 2.0) * ((gy & 1) ? 4.0 : 2.0) * ((gz & 1) ? 4.0 : 2.0);
    Cc[G] = Cf[f] * r;
    Dc[G] = Df[f] * r;
  }
}

// X = mask / C per side and the nonpositive interior counts (icount[0], icount[1])
__global__ void k_inv_lumped(const double* __restrict__ Cw, const double* __restrict__ Dw, double* __restrict__ Cinv,
                             double* __restrict__ Dinv, unsigned long long* icount, Geo G) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < G.n_nodes; g += (int64_t)gridDim.x * blockDim.x) {
    const int gx = (int)(g % G.nn1), gy = (int)((g / G.nn1) % G.nn1), gz = (int)(g / ((int64_t)G.nn1 * G.nn1));
    const bool bnd = node_bnd(gx, gy, gz, G.nn1);
    const double c = Cw[g], d = Dw[g];
    Cinv[g] = bnd ? 0.0 : 1.0 / c;
    Dinv[g] = bnd ? 0.0 : 1.0 / d;
    if (!bnd && !(c > 0.0)) atomicAdd(&icount[0], 1ull);  // (counts only: order-free)
    if (!bnd && !(d > 0.0)) atomicAdd(&icount[1], 1ull);
  }
}

__device__ __forceinline__ int64_t mg_child(int64_t ec, int Nc, int s) {
  const int cx = (int)(ec % Nc), cy = (int)((ec / Nc) % Nc), cz = (int)(ec / ((int64_t)Nc * Nc));
  const int Nf = 2 * Nc;
  return (int64_t)(2 * cx + (s & 1)) + (int64_t)Nf * ((int64_t)(2 * cy + ((s >> 1) & 1)) +
                                                      (int64_t)Nf * (2 * cz + ((s >> 2) & 1)));
}

// r_c = P^T r_f, element-major (4 modes per element)
__global__ void k_mg_restrict(const double* __restrict__ rf, double* __restrict__ rc, int Nc) {
  const double h3 = 0.86602540378443864676;  // sqrt(3) / 2
  const int64_t n = (int64_t)Nc * Nc * Nc;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const double* f = rf + 4 * mg_child(e, Nc, s);
      const double f0 = f[0];
      a0 += f0;
      a1 += h3 * mg_sign(s, 0) * f0 + 0.5 * f[1];
      a2 += h3 * mg_sign(s, 1) * f0 + 0.5 * f[2];
      a3 += h3 * mg_sign(s, 2) * f0 + 0.5 * f[3];
    }
    rc[4 * e] = a0; rc[4 * e + 1] = a1; rc[4 * e + 2] = a2; rc[4 * e + 3] = a3;
  }
}

// x_f += P x_c (one thread per fine element)
__global__ void k_mg_prolong_add(const double* __restrict__ xc, double* __restrict__ xf, int Nc) {
  const double h3 = 0.86602540378443864676;
  const int Nf = 2 * Nc;
  const int64_t n = (int64_t)Nf * Nf * Nf;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int fx = (int)(e % Nf), fy = (int)((e / Nf) % Nf), fz = (int)(e / ((int64_t)Nf * Nf));
    const int s = (fx & 1) | ((fy & 1) << 1) | ((fz & 1) << 2);
    const int64_t ec = (int64_t)(fx >> 1) + (int64_t)Nc * ((int64_t)(fy >> 1) + (int64_t)Nc * (fz >> 1));
    const double* c = xc + 4 * ec;
    double* f = xf + 4 * e;
    f[0] += c[0] + h3 * (mg_sign(s, 0) * c[1] + mg_sign(s, 1) * c[2] + mg_sign(s, 2) * c[3]);
    f[1] += 0.5 * c[1];
    f[2] += 0.5 * c[2];
    f[3] += 0.5 * c[3];
  }
}

// v_i = uniform [-1, 1) from the i-th splitmix64 output of state `seed` (Steele, Lea & Flood)
__global__ void k_splitmix(double* __restrict__ v, int64_t n, unsigned long long seed) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long z = seed + (unsigned long long)(i + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z = z ^ (z >> 31);
    v[i] = 2.0 * ((double)(z >> 11) * (1.0 / 9007199254740992.0)) - 1.0;
  }
}

// r = b - t
__global__ void k_mg_resid(double* __restrict__ r, const double* __restrict__ b, const double* __restrict__ t,
                           int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    r[i] = b[i] - t[i];
}

// element-major vector: subtract the mean of the mode-0 entries (R10 projection), mean
// from the fixed-order sum in *sum
__global__ void k_sub_mode0_mean(double* __restrict__ v, int64_t n_el, int nm, const double* __restrict__ sum) {
  const double mean = *sum / (double)n_el;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n_el; e += (int64_t)gridDim.x * blockDim.x)
    v[e * nm] -= mean;
}

// MG-PCG scalars on the device (O9 with M^-1 = V):  s[0] = rz, s[1] = pq, s[2] = rz', s[3] = stop
// alpha step: stop if rz == 0 or pq == 0; else x += a p, r -= a q, a = rz / pq
__global__ void k_mgcg_xr(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                          const double* __restrict__ q, int64_t n, double* s) {
  const double rz = s[0], pq = s[1];
  if (s[3] != 0.0 || rz == 0.0 || pq == 0.0) return;
  const double a = rz / pq;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = fma(a, p[i], x[i]);
    r[i] = fma(-a, q[i], r[i]);
  }
}
// beta step: p = z + (rz'/rz) p; then rz = rz' (the last block); stop flag latched
__global__ void k_mgcg_p(double* __restrict__ p, const double* __restrict__ z, int64_t n, double* s,
                         unsigned* counter) {
  const double rz = s[0], pq = s[1], rz1 = s[2];
  const bool stop = s[3] != 0.0 || rz == 0.0 || pq == 0.0;
  if (!stop) {
    const double b = rz1 / rz;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
      p[i] = fma(b, p[i], z[i]);
  }
  // every block has read s[0..3]; the last block to finish updates them
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned t = atomicAdd(counter, 1u);
    if (t == gridDim.x - 1) {
      if (stop) s[3] = 1.0;
      else s[0] = rz1;
      *counter = 0u;
    }
  }
}

}  // namespace wb

namespace wb {

// ---- velocity multigrid (R22): viscosity coarsening and Q2 nodal transfers (k = 2)
// mu_c at coarse Gauss point q of coarse element E: the mean, over the fine children of E
// whose closure contains the point, of each child's Gauss-weighted mean sum_q w_q mu_q / 8
// (coarse Gauss abscissae -sqrt(3/5), 0, +sqrt(3/5) lie in child 0, on the face, in child 1
// per axis).  Children in ascending (z, y, x) order.
__global__ void k_mu_coarsen(const double* __restrict__ muf, double* __restrict__ muc, int Nc) {
  const int Nf = 2 * Nc;
  const int64_t n = (int64_t)Nc * Nc * Nc * 27;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int q = (int)(i % 27);
    const int64_t E = i / 27;
    const int cx = (int)(E % Nc), cy = (int)((E / Nc) % Nc), cz = (int)(E / ((int64_t)Nc * Nc));
    const int qq[3] = {q % 3, (q / 3) % 3, q / 9};
    int lo[3], hi[3];
    for (int d = 0; d < 3; ++d) { lo[d] = qq[d] == 2 ? 1 : 0; hi[d] = qq[d] == 0 ? 0 : 1; }
    double acc = 0.0;
    int cnt = 0;
    for (int sz = lo[2]; sz <= hi[2]; ++sz)
      for (int sy = lo[1]; sy <= hi[1]; ++sy)
        for (int sx = lo[0]; sx <= hi[0]; ++sx) {
          const int64_t ef = (int64_t)(2 * cx + sx) + (int64_t)Nf * ((int64_t)(2 * cy + sy) + (int64_t)Nf * (2 * cz + sz));
          const double* m = muf + ef * 27;
          double s = 0.0;
          for (int k = 0; k < 27; ++k)
            s = fma(TB(2).w[k % 3] * TB(2).w[(k / 3) % 3] * TB(2).w[k / 9], m[k], s);
          acc += s / 8.0;
          ++cnt;
        }
    muc[i] = acc / (double)cnt;
  }
}

// 1-D weight of fine node i_f on coarse node I (Q2 nodal interpolation on the bisected
// mesh), d = i_f - 2 I: coarse vertex (I even) 1, 3/8, 0, -1/8 at |d| = 0..3; coarse
// mid-node (I odd) 1, 3/4 at |d| = 0, 1.
__device__ __forceinline__ double vmg_w(int I, int d) {
  const int a = d < 0 ? -d : d;
  if (I & 1) return a == 0 ? 1.0 : (a == 1 ? 0.75 : 0.0);
  return a == 0 ? 1.0 : (a == 1 ? 0.375 : (a == 3 ? -0.125 : 0.0));
}

// r_c = P^T (M r_f) on the coarse (2Nc+1)^3 grid, 3 SoA components, coarse boundary rows 0
__global__ void k_vmg_restrict(const double* __restrict__ rf, double* __restrict__ rc, int Nc) {
  const int nc = 2 * Nc + 1, nf = 4 * Nc + 1;
  const int64_t nnc = (int64_t)nc * nc * nc, nnf = (int64_t)nf * nf * nf;
  for (int64_t G = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; G < nnc; G += (int64_t)gridDim.x * blockDim.x) {
    const int I[3] = {(int)(G % nc), (int)((G / nc) % nc), (int)(G / ((int64_t)nc * nc))};
    if (node_bnd(I[0], I[1], I[2], nc)) { rc[G] = 0.0; rc[nnc + G] = 0.0; rc[2 * nnc + G] = 0.0; continue; }
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    for (int dz = -3; dz <= 3; ++dz) {
      const double wz = vmg_w(I[2], dz);
      const int fz = 2 * I[2] + dz;
      if (wz == 0.0 || fz < 0 || fz >= nf) continue;
      for (int dy = -3; dy <= 3; ++dy) {
        const double wy = vmg_w(I[1], dy);
        const int fy = 2 * I[1] + dy;
        if (wy == 0.0 || fy < 0 || fy >= nf) continue;
        for (int dx = -3; dx <= 3; ++dx) {
          const double wx = vmg_w(I[0], dx);
          const int fx = 2 * I[0] + dx;
          if (wx == 0.0 || fx < 0 || fx >= nf) continue;
          if (node_bnd(fx, fy, fz, nf)) continue;  // Dirichlet rows carry no residual (R6)
          const double w = wx * wy * wz;
          const int64_t f = (int64_t)fx + (int64_t)nf * ((int64_t)fy + (int64_t)nf * fz);
          a0 = fma(w, rf[f], a0);
          a1 = fma(w, rf[nnf + f], a1);
          a2 = fma(w, rf[2 * nnf + f], a2);
        }
      }
    }
    rc[G] = a0; rc[nnc + G] = a1; rc[2 * nnc + G] = a2;
  }
}

// x_f += P x_c at the fine interior nodes (fine boundary rows untouched: they stay 0)
__global__ void k_vmg_prolong_add(const double* __restrict__ xc, double* __restrict__ xf, int Nc) {
  const int nc = 2 * Nc + 1, nf = 4 * Nc + 1;
  const int64_t nnc = (int64_t)nc * nc * nc, nnf = (int64_t)nf * nf * nf;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < nnf; g += (int64_t)gridDim.x * blockDim.x) {
    const int f[3] = {(int)(g % nf), (int)((g / nf) % nf), (int)(g / ((int64_t)nf * nf))};
    if (node_bnd(f[0], f[1], f[2], nf)) continue;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    // coarse nodes with |f - 2 I| <= 3 per axis
    for (int Iz = (f[2] - 3 + 1) / 2; Iz <= (f[2] + 3) / 2; ++Iz) {
      if (Iz < 0 || Iz >= nc) continue;
      const double wz = vmg_w(Iz, f[2] - 2 * Iz);
      if (wz == 0.0) continue;
      for (int Iy = (f[1] - 3 + 1) / 2; Iy <= (f[1] + 3) / 2; ++Iy) {
        if (Iy < 0 || Iy >= nc) continue;
        const double wy = vmg_w(Iy, f[1] - 2 * Iy);
        if (wy == 0.0) continue;
        for (int Ix = (f[0] - 3 + 1) / 2; Ix <= (f[0] + 3) / 2; ++Ix) {
          if (Ix < 0 || Ix >= nc) continue;
          const double wx = vmg_w(Ix, f[0] - 2 * Ix);
          if (wx == 0.0) continue;
          const double w = wx * wy * wz;
          const int64_t G = (int64_t)Ix + (int64_t)nc * ((int64_t)Iy + (int64_t)nc * Iz);
          a0 = fma(w, xc[G], a0);
          a1 = fma(w, xc[nnc + G], a1);
          a2 = fma(w, xc[2 * nnc + G], a2);
        }
      }
    }
    xf[g] += a0; xf[nnf + g] += a1; xf[2 * nnf + g] += a2;
  }
}

}  // namespace wb

namespace wb {

// ---- the spectral (p) level for k = 4 (R20): Q4 x P3disc -> Q2 x P1disc
// on the same mesh.  Q2 node i (per axis) is Q4 node 2 i (the Q2 GLL points are Q4 GLL
// points); the unweighted lumped-mass ratio M_Q2 / M_Q4 there is 10/3 at a vertex (h/3 vs
// h/10; h/6 vs h/20 on the boundary) and 15/8 at a mid-node (2h/3 vs 16h/45) per axis.
__global__ void k_mg_inject_p(const double* __restrict__ Cf, const double* __restrict__ Df, double* __restrict__ Cc,
                              double* __restrict__ Dc, int N) {
  const int nc = 2 * N + 1, nf = 4 * N + 1;
  const int64_t n = (int64_t)nc * nc * nc;
  for (int64_t G = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; G < n; G += (int64_t)gridDim.x * blockDim.x) {
    const int gx = (int)(G % nc), gy = (int)((G / nc) % nc), gz = (int)(G / ((int64_t)nc * nc));
    const int64_t f = (int64_t)(2 * gx) + (int64_t)nf * ((int64_t)(2 * gy) + (int64_t)nf * (2 * gz));
    const double rx = (gx & 1) ? 15.0 / 8.0 : 10.0 / 3.0, ry = (gy & 1) ? 15.0 / 8.0 : 10.0 / 3.0,
                 rz = (gz & 1) ? 15.0 / 8.0 : 10.0 / 3.0;
    const double r = rx * ry * rz;
    Cc[G] = Cf[f] * r;
    Dc[G] = Df[f] * r;
  }
}
// P1disc modes are the first four P3disc modes (R2 ordering, orthonormal on the same element):
// restriction keeps them, prolongation adds into them
__global__ void k_mg_restrict_p(const double* __restrict__ rf, double* __restrict__ rc, int64_t n_el, int nmf) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < 4 * n_el; i += (int64_t)gridDim.x * blockDim.x)
    rc[i] = rf[(i / 4) * nmf + (i % 4)];
}
__global__ void k_mg_prolong_add_p(const double* __restrict__ xc, double* __restrict__ xf, int64_t n_el, int nmf) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < 4 * n_el; i += (int64_t)gridDim.x * blockDim.x)
    xf[(i / 4) * nmf + (i % 4)] += xc[i];
}

}  // namespace wb

namespace wb {

// ---- velocity spectral level for k = 4 (R22): Q4 -> Q2 on the same mesh
// mu at the 27 Q2 Gauss points from the 125 Q4 ones: per axis the 5-point samples grouped
// {0, 1}, {2}, {3, 4} (by position), Gauss-weighted mean of the tensor-product group
__global__ void k_mu_coarsen_p(const double* __restrict__ mu4, double* __restrict__ mu2, int64_t n_el) {
  const int64_t n = n_el * 27;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int q = (int)(i % 27);
    const int64_t e = i / 27;
    const int cq[3] = {q % 3, (q / 3) % 3, q / 9};
    int lo[3], hi[3];
    for (int d = 0; d < 3; ++d) { lo[d] = cq[d] == 0 ? 0 : (cq[d] == 1 ? 2 : 3); hi[d] = cq[d] == 0 ? 1 : (cq[d] == 1 ? 2 : 4); }
    const double* m = mu4 + e * 125;
    double num = 0.0, den = 0.0;
    for (int iz = lo[2]; iz <= hi[2]; ++iz)
      for (int iy = lo[1]; iy <= hi[1]; ++iy)
        for (int ix = lo[0]; ix <= hi[0]; ++ix) {
          const double w = TB(4).w[ix] * TB(4).w[iy] * TB(4).w[iz];
          num = fma(w, m[ix + 5 * (iy + 5 * iz)], num);
          den += w;
        }
    mu2[i] = num / den;
  }
}

// Q2 basis at the Q4 GLL abscissae -1, -s, 0, s, 1 (s = sqrt(3/7)): W[a2][a4]
__device__ __forceinline__ double vmgp_w(int a2, int a4) {
  const double s = 0.65465367070797714380, s2 = 3.0 / 7.0;  // sqrt(3/7)
  const double t = a4 == 0 ? -1.0 : (a4 == 1 ? -s : (a4 == 2 ? 0.0 : (a4 == 3 ? s : 1.0)));
  const double t2 = a4 == 1 || a4 == 3 ? s2 : t * t;
  if (a2 == 0) return 0.5 * (t2 - t);
  if (a2 == 1) return 1.0 - t2;
  return 0.5 * (t2 + t);
}
// per-axis coupling list of coarse (Q2) node I with fine (Q4) nodes j and weights (<= 7)
__device__ __forceinline__ int vmgp_list(int I, int N, int* j, double* w) {
  int n = 0;
  if (I & 1) {  // mid-node of element e: its interior Q4 nodes
    const int e = I >> 1;
    for (int a4 = 1; a4 <= 3; ++a4) { j[n] = 4 * e + a4; w[n] = vmgp_w(1, a4); ++n; }
  } else {
    const int e = I >> 1;
    if (e >= 1)
      for (int a4 = 1; a4 <= 3; ++a4) { j[n] = 4 * (e - 1) + a4; w[n] = vmgp_w(2, a4); ++n; }
    j[n] = 4 * e; w[n] = 1.0; ++n;
    if (e < N)
      for (int a4 = 1; a4 <= 3; ++a4) { j[n] = 4 * e + a4; w[n] = vmgp_w(0, a4); ++n; }
  }
  return n;
}
// r_c = P^T (M r_f) (Q4 grid -> Q2 grid, same mesh), coarse boundary rows 0
__global__ void k_vmg_restrict_p(const double* __restrict__ rf, double* __restrict__ rc, int N) {
  const int nc = 2 * N + 1, nf = 4 * N + 1;
  const int64_t nnc = (int64_t)nc * nc * nc, nnf = (int64_t)nf * nf * nf;
  for (int64_t G = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; G < nnc; G += (int64_t)gridDim.x * blockDim.x) {
    const int I[3] = {(int)(G % nc), (int)((G / nc) % nc), (int)(G / ((int64_t)nc * nc))};
    if (node_bnd(I[0], I[1], I[2], nc)) { rc[G] = 0.0; rc[nnc + G] = 0.0; rc[2 * nnc + G] = 0.0; continue; }
    int jx[7], jy[7], jz[7];
    double wx[7], wy[7], wz[7];
    const int nx = vmgp_list(I[0], N, jx, wx), ny = vmgp_list(I[1], N, jy, wy), nz = vmgp_list(I[2], N, jz, wz);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    for (int kz = 0; kz < nz; ++kz)
      for (int ky = 0; ky < ny; ++ky)
        for (int kx = 0; kx < nx; ++kx) {
          if (node_bnd(jx[kx], jy[ky], jz[kz], nf)) continue;
          const double w = wx[kx] * wy[ky] * wz[kz];
          const int64_t f = (int64_t)jx[kx] + (int64_t)nf * ((int64_t)jy[ky] + (int64_t)nf * jz[kz]);
          a0 = fma(w, rf[f], a0);
          a1 = fma(w, rf[nnf + f], a1);
          a2 = fma(w, rf[2 * nnf + f], a2);
        }
    rc[G] = a0; rc[nnc + G] = a1; rc[2 * nnc + G] = a2;
  }
}
// x_f += P x_c at the interior Q4 nodes
__global__ void k_vmg_prolong_add_p(const double* __restrict__ xc, double* __restrict__ xf, int N) {
  const int nc = 2 * N + 1, nf = 4 * N + 1;
  const int64_t nnc = (int64_t)nc * nc * nc, nnf = (int64_t)nf * nf * nf;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < nnf; g += (int64_t)gridDim.x * blockDim.x) {
    const int f[3] = {(int)(g % nf), (int)((g / nf) % nf), (int)(g / ((int64_t)nf * nf))};
    if (node_bnd(f[0], f[1], f[2], nf)) continue;
    int I[3][3], n[3];
    double w[3][3];
    for (int d = 0; d < 3; ++d) {
      const int j = f[d];
      if ((j & 3) == 0) { I[d][0] = j >> 1; w[d][0] = 1.0; n[d] = 1; }
      else {
        const int e = j >> 2, a4 = j & 3;
        n[d] = 0;
        for (int a2 = 0; a2 < 3; ++a2) {
          const double ww = vmgp_w(a2, a4);
          if (ww != 0.0) { I[d][n[d]] = 2 * e + a2; w[d][n[d]] = ww; ++n[d]; }
        }
      }
    }
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    for (int kz = 0; kz < n[2]; ++kz)
      for (int ky = 0; ky < n[1]; ++ky)
        for (int kx = 0; kx < n[0]; ++kx) {
          const double ww = w[0][kx] * w[1][ky] * w[2][kz];
          const int64_t G = (int64_t)I[0][kx] + (int64_t)nc * ((int64_t)I[1][ky] + (int64_t)nc * I[2][kz]);
          a0 = fma(ww, xc[G], a0);
          a1 = fma(ww, xc[nnc + G], a1);
          a2 = fma(ww, xc[2 * nnc + G], a2);
        }
    xf[g] += a0; xf[nnf + g] += a1; xf[2 * nnf + g] += a2;
  }
}

}  // namespace wb
