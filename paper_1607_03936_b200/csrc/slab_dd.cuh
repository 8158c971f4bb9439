// slab_dd.cuh -- kernels of the z-slab domain decomposition (the
// element-partition decomposition of PAPER.md:2480-2487; reading R24, wbfbt.h "z-slab").
//
// A slab context is a cube context whose z-lo / z-hi faces may be shared with a neighbouring
// rank (Geo::zopen).  The operators run the cube kernels WITHOUT their built-in Dirichlet mask
// (nomask, or a nodal scaling xs), the shared planes' partial sums are exchanged and added
// (k_dd_unpack_add), and the GLOBAL mask gm is applied here.  Both owners of a shared plane compute
// own + received: the two-term sum commutes, so their copies agree bit for bit.
#pragma once
#include "kernels.cuh"

namespace wb {

// gm[g] = 0 on the global Dirichlet boundary, else 1 (shared planes are interior off their rim)
__global__ void k_dd_mask(double* __restrict__ gm, Geo G) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= G.n_nodes) return;
  const int nn1 = G.nn1;
  const int gx = (int)(g % nn1), gy = (int)((g / nn1) % nn1), gz = (int)(g / ((int64_t)nn1 * nn1));
  const bool b = gx == 0 || gy == 0 || gx == nn1 - 1 || gy == nn1 - 1 || (gz == 0 && !(G.zopen & 1)) ||
                 (gz == nn1 - 1 && !(G.zopen & 2));
  gm[g] = b ? 0.0 : 1.0;
}

// ABI mask (1 = boundary) for the 3 components from gm
__global__ void k_dd_bmask(uint8_t* __restrict__ mask, const double* __restrict__ gm, int64_t n_nodes) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_nodes) return;
  const uint8_t b = gm[g] == 0.0 ? 1 : 0;
  mask[g] = b; mask[n_nodes + g] = b; mask[2 * n_nodes + g] = b;
}

// The shared planes of up to 3 nodal fields (n_nodes each; plane z = 0 is the first np entries,
// plane z = kN the last np) in one launch: pack into the send buffers, or add the received
// partials.  zopen bit 0 / 1 selects the lo / hi plane.
struct DDFields {
  double* f[3];
  int nf;
};
__global__ void k_dd_pack(DDFields F, double* __restrict__ send_lo, double* __restrict__ send_hi, int64_t np,
                          int64_t n_nodes, int zopen) {
  const int64_t n = np * F.nf;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(i / np);
    const int64_t j = i - k * np;
    if (zopen & 1) send_lo[i] = F.f[k][j];
    if (zopen & 2) send_hi[i] = F.f[k][n_nodes - np + j];
  }
}
__global__ void k_dd_unpack_add(DDFields F, const double* __restrict__ recv_lo, const double* __restrict__ recv_hi,
                                int64_t np, int64_t n_nodes, int zopen) {
  const int64_t n = np * F.nf;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(i / np);
    const int64_t j = i - k * np;
    if (zopen & 1) F.f[k][j] += recv_lo[i];
    if (zopen & 2) F.f[k][n_nodes - np + j] += recv_hi[i];
  }
}

// Cinv = gm / C_w, Dinv = gm / D_w from the plane-summed lumped masses (row a3 with the global
// mask); nonpositive unmasked entries counted (shared-plane nodes by both owners)
__global__ void k_dd_inv(const double* __restrict__ Cw, const double* __restrict__ Dw, const double* __restrict__ gm,
                         double* __restrict__ Cinv, double* __restrict__ Dinv, unsigned long long* nonpos,
                         int64_t n) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n; g += (int64_t)gridDim.x * blockDim.x) {
    const bool b = gm[g] == 0.0;
    const double cl = Cw[g], cr = Dw[g];
    Cinv[g] = b ? 0.0 : 1.0 / cl;
    Dinv[g] = b ? 0.0 : 1.0 / cr;
    if (!b && cl <= 0.0) atomicAdd(nonpos + 0, 1ull);  // (counts only: order-free)
    if (!b && cr <= 0.0) atomicAdd(nonpos + 1, 1ull);
  }
}

// y[(c, g)] = x[(c, g)] w[g]: a nodal scalar on the 3 SoA components (y may equal x)
__global__ void k_dd_scale3(double* y, const double* x, const double* __restrict__ w, int64_t n_nodes) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n_nodes; g += (int64_t)gridDim.x * blockDim.x) {
    const double s = w[g];
    y[g] = x[g] * s;
    y[n_nodes + g] = x[n_nodes + g] * s;
    y[2 * n_nodes + g] = x[2 * n_nodes + g] * s;
  }
}

// R10 projection on the local part of an element-major vector: subtract the GLOBAL mean of the
// mode-0 entries (*sum = their all-reduced sum, n_glob = the global element count)
__global__ void k_dd_sub_mean(double* __restrict__ v, int64_t n_el, int nm, const double* __restrict__ sum,
                              double n_glob) {
  const double mean = *sum / n_glob;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n_el; e += (int64_t)gridDim.x * blockDim.x)
    v[e * nm] -= mean;
}

}  // namespace wb
