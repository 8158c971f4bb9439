// wbfbt.cu -- host side of libwbfbt.so: the C ABI of include/wbfbt.h.
//
// The context owns all workspace; every call enqueues kernels on the context
// stream.  See DESIGN.md for the data layout and the kernel list.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>

#include "../../include/wbfbt.h"
#include "kernels.cuh"

using namespace wb;

#define WB_VERSION "wbfbt-b200 0.1 (sm_100a, fp64)"

struct wb_ctx {
  int N = 0, k = 0, n1 = 0, nq = 0, nm = 0;
  unsigned flags = 0;
  cudaStream_t stream = nullptr;
  Geo G{};
  int64_t n_el = 0, n_nodes = 0, n_v = 0, n_p = 0;
  double h = 0, detJ = 0, sB = 0;
  // setup results
  double *mut = nullptr, *Cw = nullptr, *Dw = nullptr, *Cinv = nullptr, *Dinv = nullptr;
  double *dKl = nullptr, *dKr = nullptr, *MinvL = nullptr, *MinvR = nullptr;
  bool have_visc = false;
  long long n_nonpos[2] = {0, 0};
  // work vectors
  double* E = nullptr;                 // element-local velocity values, 3*nq*n_el
  double *tv = nullptr, *tw = nullptr;  // n_v
  double *pr = nullptr, *pp = nullptr, *pq = nullptr;  // PCG r, p, q (n_p)
  double *s0 = nullptr, *s1 = nullptr, *s2 = nullptr;  // n_p scratch
  // scalars
  double* partial = nullptr;  // reduction partials
  unsigned* counter = nullptr;
  double* scal = nullptr;  // [0..7] misc totals, then rz_hist, pq_hist, rzn_hist
  int* stop = nullptr;
  int it_cap = 0;
  unsigned long long* icount = nullptr;  // [0] bad mu, [1] nonpos Cw, [2] nonpos Dw
  int red_blocks = 0, max_partials = 0;
  double* stage = nullptr;  // wb_hotpath_host staging (lazily allocated)
  long long launches = 0;
  char err[512] = {0};
};

namespace {

bool g_tabs_ready = false;

wb_status set_err(wb_ctx* c, wb_status s, const char* fmt, ...) {
  if (c) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(c->err, sizeof(c->err), fmt, ap);
    va_end(ap);
  }
  return s;
}

#define CUDA_TRY(c, expr)                                                                        \
  do {                                                                                           \
    cudaError_t e_ = (expr);                                                                     \
    if (e_ != cudaSuccess)                                                                       \
      return set_err((c), WB_ECUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)

#define LAUNCH_CHECK(c)                                                                          \
  do {                                                                                           \
    (c)->launches++;                                                                             \
    cudaError_t e_ = cudaGetLastError();                                                         \
    if (e_ != cudaSuccess)                                                                       \
      return set_err((c), WB_ECUDA, "launch: %s (%s:%d)", cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)

inline unsigned nblk(int64_t n, int bs) { return (unsigned)((n + bs - 1) / bs); }

bool overlaps(const void* a, size_t na, const void* b, size_t nb) {
  const char* x = (const char*)a;
  const char* y = (const char*)b;
  return x < y + nb && y < x + na;
}

// scalar slots
enum { S_SUM = 0, S_PQ1 = 1, S_NSCAL = 8 };
inline double* rz_hist(wb_ctx* c) { return c->scal + S_NSCAL; }
inline double* pq_hist(wb_ctx* c) { return c->scal + S_NSCAL + (c->it_cap + 1); }
inline double* rzn_hist(wb_ctx* c) { return c->scal + S_NSCAL + 2 * (c->it_cap + 1); }

wb_status ensure_iters(wb_ctx* c, int iters) {
  if (iters <= c->it_cap) return WB_OK;
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (c->scal) cudaFree(c->scal);
  if (c->stop) cudaFree(c->stop);
  c->scal = nullptr; c->stop = nullptr;
  int cap = iters < 128 ? 128 : iters;
  if (cudaMalloc(&c->scal, sizeof(double) * (S_NSCAL + 3 * (cap + 1))) != cudaSuccess ||
      cudaMalloc(&c->stop, sizeof(int) * (cap + 1)) != cudaSuccess) {
    c->it_cap = 0;
    return set_err(c, WB_ENOMEM, "scalar workspace allocation failed");
  }
  CUDA_TRY(c, cudaMemsetAsync(c->scal, 0, sizeof(double) * (S_NSCAL + 3 * (cap + 1)), c->stream));
  CUDA_TRY(c, cudaMemsetAsync(c->stop, 0, sizeof(int) * (cap + 1), c->stream));
  c->it_cap = cap;
  return WB_OK;
}

// ---------------------------------------------------------------- kernel dispatch helpers
template <int K>
wb_status launch_A_t(wb_ctx* c, const double* u, double* out_E, int nomask) {
  if constexpr (K == 2) {
    constexpr int NE = 64;
    k_A_reg<2, NE><<<nblk(c->n_el, NE), 3 * NE, 0, c->stream>>>(c->mut, u, out_E, c->G, nomask);
  } else {
    constexpr int NE = (K == 3) ? 8 : 5;
    const size_t smem = (size_t)NE * 12 * Ord<K>::NQ * sizeof(double);
    static bool attr = false;
    if (!attr) {
      CUDA_TRY(c, cudaFuncSetAttribute(k_A_slice<K, NE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr = true;
    }
    k_A_slice<K, NE><<<nblk(c->n_el, NE), NE * (K + 1) * (K + 1), smem, c->stream>>>(c->mut, u, out_E, c->G, nomask);
  }
  LAUNCH_CHECK(c);
  return WB_OK;
}

template <int K>
wb_status launch_gather_t(wb_ctx* c, const double* s, double* y, int nomask) {
  k_gather<K><<<nblk(c->n_nodes, 256), 256, 0, c->stream>>>(c->E, s, y, c->G, nomask);
  LAUNCH_CHECK(c);
  return WB_OK;
}

template <int K>
wb_status launch_BT_t(wb_ctx* c, const double* p, const int* stop) {
  k_BT_elem<K><<<nblk(c->n_el, 128), 128, 0, c->stream>>>(p, c->E, c->G, c->sB, stop);
  LAUNCH_CHECK(c);
  return WB_OK;
}

template <int K>
wb_status launch_B_t(wb_ctx* c, const double* u, const double* xs, double* p, int nomask, const int* stop,
                     const double* dv, double* total) {
  constexpr int BS = 128;
  k_B<K, BS><<<nblk(c->n_el, BS), BS, 0, c->stream>>>(u, xs, p, c->G, c->sB, nomask, stop, dv,
                                                       dv ? c->partial : nullptr, c->counter, total);
  LAUNCH_CHECK(c);
  return WB_OK;
}

#define DISPATCH_K(c, fn, ...)                                   \
  ((c)->k == 2 ? fn<2>(c, __VA_ARGS__)                           \
               : ((c)->k == 3 ? fn<3>(c, __VA_ARGS__) : fn<4>(c, __VA_ARGS__)))

wb_status run_A(wb_ctx* c, const double* u, double* y, int nomask) {
  wb_status s = DISPATCH_K(c, launch_A_t, u, c->E, nomask);
  if (s) return s;
  return DISPATCH_K(c, launch_gather_t, (const double*)nullptr, y, nomask);
}
wb_status run_BT(wb_ctx* c, const double* p, const double* xs, double* y, int nomask, const int* stop) {
  wb_status s = DISPATCH_K(c, launch_BT_t, p, stop);
  if (s) return s;
  if (stop) {
    // the gather of a stopped PCG iteration is harmless (its result is unused)
  }
  return DISPATCH_K(c, launch_gather_t, xs, y, nomask);
}
wb_status run_B(wb_ctx* c, const double* u, const double* xs, double* p, int nomask, const int* stop,
                const double* dv, double* total) {
  return DISPATCH_K(c, launch_B_t, u, xs, p, nomask, stop, dv, total);
}

// q = K_side p  (+ <p, q> into *total when dot)
wb_status run_K(wb_ctx* c, int side, const double* p, double* q, const int* stop, bool dot, double* total) {
  wb_status s = run_BT(c, p, nullptr, c->tv, 0, stop);
  if (s) return s;
  const double* X = side == 0 ? c->Cinv : c->Dinv;
  return run_B(c, c->tv, X, q, 0, stop, dot ? p : nullptr, total);
}

// out = P in (out may equal in)
wb_status run_project(wb_ctx* c, const double* in, double* out) {
  k_mode0_sum<<<c->red_blocks, VBS, 0, c->stream>>>(in, c->n_el, c->nm, c->partial, c->counter, c->scal + S_SUM);
  LAUNCH_CHECK(c);
  k_project<<<c->red_blocks, VBS, 0, c->stream>>>(in, out, c->n_p, c->nm, c->n_el, c->scal + S_SUM);
  LAUNCH_CHECK(c);
  return WB_OK;
}

// x = PCG(K_side, b), exactly `iters` iterations (break rules of DESIGN.md Sec. 4)
wb_status run_pcg(wb_ctx* c, int side, const double* b, double* x, int iters) {
  wb_status s = ensure_iters(c, iters);
  if (s) return s;
  const double* Minv = side == 0 ? c->MinvL : c->MinvR;
  k_pcg_init<<<c->red_blocks, VBS, 0, c->stream>>>(b, x, c->pr, c->pp, Minv, c->n_p, c->partial, c->counter,
                                                   rz_hist(c), c->stop);
  LAUNCH_CHECK(c);
  for (int it = 0; it < iters; ++it) {
    const int* st = c->stop + it;
    s = run_K(c, side, c->pp, c->pq, st, true, pq_hist(c) + it);
    if (s) return s;
    k_pcg_upd1<<<c->red_blocks, VBS, 0, c->stream>>>(x, c->pr, c->pp, c->pq, Minv, c->n_p, pq_hist(c) + it,
                                                     rz_hist(c) + it, rzn_hist(c) + it, st, c->partial, c->counter);
    LAUNCH_CHECK(c);
    k_pcg_upd2<<<c->red_blocks, VBS, 0, c->stream>>>(c->pr, c->pp, Minv, c->n_p, pq_hist(c) + it, rz_hist(c) + it,
                                                     rzn_hist(c) + it, rz_hist(c) + it + 1, st, c->stop + it + 1);
    LAUNCH_CHECK(c);
  }
  return WB_OK;
}

wb_status run_poisson(wb_ctx* c, int side, const double* b, double* x, int iters) {
  wb_status s = run_project(c, b, c->s0);
  if (s) return s;
  s = run_pcg(c, side, c->s0, c->s1, iters);
  if (s) return s;
  return run_project(c, c->s1, x);
}

wb_status run_wbfbt(wb_ctx* c, const double* r, double* z, int iters) {
  // y = P PCG(K_r, P r)
  wb_status s = run_poisson(c, 1, r, c->s2, iters);
  if (s) return s;
  // v = Dinv o (B^T y)
  s = run_BT(c, c->s2, c->Dinv, c->tw, 0, nullptr);
  if (s) return s;
  // w = A v
  s = run_A(c, c->tw, c->tv, 0);
  if (s) return s;
  // s = P B (Cinv o w)
  s = run_B(c, c->tv, c->Cinv, c->s2, 0, nullptr, nullptr, nullptr);
  if (s) return s;
  // z = P PCG(K_l, s)   (run_poisson projects its input first)
  return run_poisson(c, 0, c->s2, z, iters);
}

wb_status check_ctx(wb_ctx* c, bool need_visc) {
  if (!c) return WB_EINVAL;
  if (need_visc && !c->have_visc) return set_err(c, WB_ESTATE, "wb_set_viscosity has not been called");
  return WB_OK;
}

void free_all(wb_ctx* c) {
  double** bufs[] = {&c->mut, &c->Cw, &c->Dw, &c->Cinv, &c->Dinv, &c->dKl, &c->dKr, &c->MinvL, &c->MinvR,
                     &c->E, &c->tv, &c->tw, &c->pr, &c->pp, &c->pq, &c->s0, &c->s1, &c->s2, &c->partial, &c->scal,
                     &c->stage};
  for (double** b : bufs)
    if (*b) { cudaFree(*b); *b = nullptr; }
  if (c->counter) cudaFree(c->counter);
  if (c->stop) cudaFree(c->stop);
  if (c->icount) cudaFree(c->icount);
  c->counter = nullptr; c->stop = nullptr; c->icount = nullptr;
}

}  // namespace

// ================================================================ C ABI
extern "C" {

const char* wb_version(void) { return WB_VERSION; }

wb_status wb_create(wb_ctx** out, int N, int k, unsigned flags, void* stream) {
  if (!out) return WB_EINVAL;
  *out = nullptr;
  if (N < 1 || N > 4096 || k < 2 || k > 4) return WB_EINVAL;
  wb_ctx* c = new (std::nothrow) wb_ctx();
  if (!c) return WB_ENOMEM;
  c->N = N; c->k = k; c->n1 = k + 1; c->nq = c->n1 * c->n1 * c->n1; c->nm = k * (k + 1) * (k + 2) / 6;
  c->flags = flags;
  c->stream = (cudaStream_t)stream;
  c->n_el = (int64_t)N * N * N;
  const int64_t nn1 = (int64_t)k * N + 1;
  c->n_nodes = nn1 * nn1 * nn1;
  c->n_v = 3 * c->n_nodes;
  c->n_p = (int64_t)c->nm * c->n_el;
  c->G = Geo{N, k, (int)nn1, c->n_el, c->n_nodes, c->n_p};
  c->h = 1.0 / N;
  c->detJ = (c->h / 2) * (c->h / 2) * (c->h / 2);
  c->sB = -(2.0 / c->h) * c->detJ;
  if (!g_tabs_ready) {
    Tab t[3] = {make_tab(2), make_tab(3), make_tab(4)};
    cudaError_t e = cudaMemcpyToSymbol(c_tab, t, sizeof(t));
    if (e != cudaSuccess) {
      delete c;
      return WB_ECUDA;
    }
    g_tabs_ready = true;
  }
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  c->red_blocks = 2 * nsm;
  c->max_partials = (int)std::max<int64_t>(c->red_blocks, (c->n_el + 127) / 128 + 1);
  bool ok = true;
  auto alloc = [&](double** p, int64_t n) {
    if (ok && cudaMalloc(p, sizeof(double) * (size_t)(n > 0 ? n : 1)) != cudaSuccess) ok = false;
  };
  alloc(&c->mut, c->n_el * c->nq);
  alloc(&c->Cw, c->n_nodes); alloc(&c->Dw, c->n_nodes); alloc(&c->Cinv, c->n_nodes); alloc(&c->Dinv, c->n_nodes);
  alloc(&c->dKl, c->n_p); alloc(&c->dKr, c->n_p); alloc(&c->MinvL, c->n_p); alloc(&c->MinvR, c->n_p);
  alloc(&c->E, 3 * c->nq * c->n_el);
  alloc(&c->tv, c->n_v); alloc(&c->tw, c->n_v);
  alloc(&c->pr, c->n_p); alloc(&c->pp, c->n_p); alloc(&c->pq, c->n_p);
  alloc(&c->s0, c->n_p); alloc(&c->s1, c->n_p); alloc(&c->s2, c->n_p);
  alloc(&c->partial, c->max_partials);
  if (ok && cudaMalloc(&c->counter, sizeof(unsigned) * 4) != cudaSuccess) ok = false;
  if (ok && cudaMalloc(&c->icount, sizeof(unsigned long long) * 4) != cudaSuccess) ok = false;
  if (!ok) {
    free_all(c);
    delete c;
    cudaGetLastError();
    return WB_ENOMEM;
  }
  if (cudaMemsetAsync(c->counter, 0, sizeof(unsigned) * 4, c->stream) != cudaSuccess ||
      ensure_iters(c, 128) != WB_OK || cudaStreamSynchronize(c->stream) != cudaSuccess) {
    free_all(c);
    delete c;
    return WB_ECUDA;
  }
  *out = c;
  return WB_OK;
}

void wb_destroy(wb_ctx* c) {
  if (!c) return;
  cudaStreamSynchronize(c->stream);
  free_all(c);
  delete c;
}

wb_status wb_set_stream(wb_ctx* c, void* stream) {
  if (!c) return WB_EINVAL;
  c->stream = (cudaStream_t)stream;
  return WB_OK;
}

const char* wb_last_error(const wb_ctx* c) { return c ? c->err : "null context"; }

wb_status wb_sizes(const wb_ctx* c, int64_t* n_el, int64_t* n_nodes, int64_t* n_v, int64_t* n_p, int64_t* n_q) {
  if (!c) return WB_EINVAL;
  if (n_el) *n_el = c->n_el;
  if (n_nodes) *n_nodes = c->n_nodes;
  if (n_v) *n_v = c->n_v;
  if (n_p) *n_p = c->n_p;
  if (n_q) *n_q = c->nq;
  return WB_OK;
}

wb_status wb_get_dofmap(wb_ctx* c, int64_t* map) {
  if (!c || !map) return WB_EINVAL;
  const int64_t n = c->n_el * c->nq;
  switch (c->k) {
    case 2: k_dofmap<2><<<nblk(n, 256), 256, 0, c->stream>>>(map, c->G); break;
    case 3: k_dofmap<3><<<nblk(n, 256), 256, 0, c->stream>>>(map, c->G); break;
    default: k_dofmap<4><<<nblk(n, 256), 256, 0, c->stream>>>(map, c->G); break;
  }
  LAUNCH_CHECK(c);
  return WB_OK;
}

wb_status wb_get_boundary_mask(wb_ctx* c, uint8_t* mask) {
  if (!c || !mask) return WB_EINVAL;
  k_bmask<<<nblk(c->n_nodes, 256), 256, 0, c->stream>>>(mask, c->G);
  LAUNCH_CHECK(c);
  return WB_OK;
}

}  // extern "C"

template <int K>
static wb_status setup_t(wb_ctx* c, const double* mu, double a_l, double a_r) {
  const int64_t nmu = c->n_el * c->nq;
  CUDA_TRY(c, cudaMemsetAsync(c->icount, 0, sizeof(unsigned long long) * 4, c->stream));
  k_prescale<K><<<nblk(nmu, 256), 256, 0, c->stream>>>(mu, c->mut, nmu, c->h / 2, c->icount);
  LAUNCH_CHECK(c);
  unsigned long long bad = 0;
  CUDA_TRY(c, cudaMemcpyAsync(&bad, c->icount, sizeof(bad), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (bad) {
    c->have_visc = false;
    return set_err(c, WB_ENONPOS_MU, "%llu viscosity samples are <= 0 or non-finite", bad);
  }
  // lumped masses: element part into E (1 component), node gather
  k_lump_elem<K><<<nblk(c->n_el, 128), 128, 0, c->stream>>>(mu, c->E, c->G, c->detJ);
  LAUNCH_CHECK(c);
  k_lump_node<K><<<nblk(c->n_nodes, 256), 256, 0, c->stream>>>(c->E, a_l, a_r, c->Cw, c->Dw, c->Cinv, c->Dinv,
                                                               c->icount + 1, c->G);
  LAUNCH_CHECK(c);
  k_jacobi<K><<<nblk(c->n_el, 128), 128, 0, c->stream>>>(c->Cinv, c->Dinv, c->dKl, c->dKr, c->MinvL, c->MinvR,
                                                         c->G, c->sB);
  LAUNCH_CHECK(c);
  unsigned long long np[2] = {0, 0};
  CUDA_TRY(c, cudaMemcpyAsync(np, c->icount + 1, sizeof(np), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  c->n_nonpos[0] = (long long)np[0];
  c->n_nonpos[1] = (long long)np[1];
  c->have_visc = true;
  if ((c->flags & WB_STRICT_LUMP) && (np[0] || np[1]))
    return set_err(c, WB_ENONPOS_LUMP, "nonpositive lumped entries: C_w %llu, D_w %llu", np[0], np[1]);
  return WB_OK;
}

extern "C" {

wb_status wb_set_viscosity(wb_ctx* c, const double* mu_q, double a_l, double a_r) {
  if (!c || !mu_q) return WB_EINVAL;
  if (!(a_l >= 1.0) || !(a_r >= 1.0) || !std::isfinite(a_l) || !std::isfinite(a_r))
    return set_err(c, WB_EINVAL, "a_l, a_r must be finite and >= 1");
  switch (c->k) {
    case 2: return setup_t<2>(c, mu_q, a_l, a_r);
    case 3: return setup_t<3>(c, mu_q, a_l, a_r);
    default: return setup_t<4>(c, mu_q, a_l, a_r);
  }
}

wb_status wb_apply_A(wb_ctx* c, const double* u, double* y) {
  wb_status s = check_ctx(c, true);
  if (s) return s;
  if (!u || !y) return set_err(c, WB_EINVAL, "null pointer");
  if (overlaps(u, 8 * c->n_v, y, 8 * c->n_v)) return set_err(c, WB_EALIAS, "u and y overlap");
  return run_A(c, u, y, (c->flags & WB_DEBUG_NOMASK) ? 1 : 0);
}

wb_status wb_apply_B(wb_ctx* c, const double* u, double* p) {
  wb_status s = check_ctx(c, false);
  if (s) return s;
  if (!u || !p) return set_err(c, WB_EINVAL, "null pointer");
  if (overlaps(u, 8 * c->n_v, p, 8 * c->n_p)) return set_err(c, WB_EALIAS, "u and p overlap");
  return run_B(c, u, nullptr, p, (c->flags & WB_DEBUG_NOMASK) ? 1 : 0, nullptr, nullptr, nullptr);
}

wb_status wb_apply_BT(wb_ctx* c, const double* p, double* y) {
  wb_status s = check_ctx(c, false);
  if (s) return s;
  if (!p || !y) return set_err(c, WB_EINVAL, "null pointer");
  if (overlaps(p, 8 * c->n_p, y, 8 * c->n_v)) return set_err(c, WB_EALIAS, "p and y overlap");
  return run_BT(c, p, nullptr, y, (c->flags & WB_DEBUG_NOMASK) ? 1 : 0, nullptr);
}

wb_status wb_apply_K(wb_ctx* c, int side, const double* p, double* q) {
  wb_status s = check_ctx(c, true);
  if (s) return s;
  if (!p || !q || (side != 0 && side != 1)) return set_err(c, WB_EINVAL, "bad argument");
  if (overlaps(p, 8 * c->n_p, q, 8 * c->n_p)) return set_err(c, WB_EALIAS, "p and q overlap");
  return run_K(c, side, p, q, nullptr, false, nullptr);
}

wb_status wb_poisson_pcg(wb_ctx* c, int side, const double* b, double* x, int iters) {
  wb_status s = check_ctx(c, true);
  if (s) return s;
  if (!b || !x || (side != 0 && side != 1) || iters < 0) return set_err(c, WB_EINVAL, "bad argument");
  if (overlaps(b, 8 * c->n_p, x, 8 * c->n_p)) return set_err(c, WB_EALIAS, "b and x overlap");
  return run_poisson(c, side, b, x, iters);
}

wb_status wb_apply_wbfbt(wb_ctx* c, const double* r, double* z, int iters) {
  wb_status s = check_ctx(c, true);
  if (s) return s;
  if (!r || !z || iters < 0) return set_err(c, WB_EINVAL, "bad argument");
  if (overlaps(r, 8 * c->n_p, z, 8 * c->n_p)) return set_err(c, WB_EALIAS, "r and z overlap");
  return run_wbfbt(c, r, z, iters);
}

wb_status wb_hotpath(wb_ctx* c, const double* mu_q, double a_l, double a_r, const double* u, const double* p,
                     int iters, double* yA, double* pB, double* yBT, double* z) {
  wb_status s = wb_set_viscosity(c, mu_q, a_l, a_r);
  if (s) return s;
  if ((s = wb_apply_A(c, u, yA))) return s;
  if ((s = wb_apply_B(c, u, pB))) return s;
  if ((s = wb_apply_BT(c, p, yBT))) return s;
  if ((s = wb_apply_wbfbt(c, p, z, iters))) return s;
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return WB_OK;
}

wb_status wb_hotpath_host(wb_ctx* c, const double* mu_q, double a_l, double a_r, const double* u, const double* p,
                          int iters, double* yA, double* pB, double* yBT, double* z) {
  if (!c || !mu_q || !u || !p || !yA || !pB || !yBT || !z) return WB_EINVAL;
  const int64_t nmu = c->n_el * c->nq;
  if (!c->stage) {
    if (cudaMalloc(&c->stage, sizeof(double) * (size_t)(nmu + 3 * c->n_v + 3 * c->n_p)) != cudaSuccess) {
      c->stage = nullptr;
      cudaGetLastError();
      return set_err(c, WB_ENOMEM, "staging allocation failed");
    }
  }
  double* dmu = c->stage;
  double* du = dmu + nmu;
  double* dyA = du + c->n_v;
  double* dyBT = dyA + c->n_v;
  double* dp = dyBT + c->n_v;
  double* dpB = dp + c->n_p;
  double* dz = dpB + c->n_p;
  const size_t bmu = sizeof(double) * nmu, bv = sizeof(double) * c->n_v, bp = sizeof(double) * c->n_p;
  CUDA_TRY(c, cudaMemcpyAsync(dmu, mu_q, bmu, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(du, u, bv, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(dp, p, bp, cudaMemcpyHostToDevice, c->stream));
  wb_status s = wb_hotpath(c, dmu, a_l, a_r, du, dp, iters, dyA, dpB, dyBT, dz);
  if (s) return s;
  CUDA_TRY(c, cudaMemcpyAsync(yA, dyA, bv, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(pB, dpB, bp, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(yBT, dyBT, bv, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(z, dz, bp, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return WB_OK;
}

wb_status wb_debug_pcg_step(wb_ctx* c, int side, double* x, double* r, double* p, double* rz) {
  wb_status s = check_ctx(c, true);
  if (s) return s;
  if (!x || !r || !p || !rz || (side != 0 && side != 1)) return set_err(c, WB_EINVAL, "bad argument");
  if ((s = ensure_iters(c, 1))) return s;
  const double* Minv = side == 0 ? c->MinvL : c->MinvR;
  CUDA_TRY(c, cudaMemcpyAsync(rz_hist(c), rz, sizeof(double), cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemsetAsync(c->stop, 0, sizeof(int), c->stream));
  if ((s = run_K(c, side, p, c->pq, c->stop, true, pq_hist(c)))) return s;
  k_pcg_upd1<<<c->red_blocks, VBS, 0, c->stream>>>(x, r, p, c->pq, Minv, c->n_p, pq_hist(c), rz_hist(c),
                                                   rzn_hist(c), c->stop, c->partial, c->counter);
  LAUNCH_CHECK(c);
  k_pcg_upd2<<<c->red_blocks, VBS, 0, c->stream>>>(r, p, Minv, c->n_p, pq_hist(c), rz_hist(c), rzn_hist(c),
                                                   rz_hist(c) + 1, c->stop, c->stop + 1);
  LAUNCH_CHECK(c);
  CUDA_TRY(c, cudaMemcpyAsync(rz, rz_hist(c) + 1, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return WB_OK;
}

wb_status wb_get_lumped(wb_ctx* c, double* Cw, double* Dw, double* Cinv, double* Dinv) {
  wb_status s = check_ctx(c, true);
  if (s) return s;
  const size_t b = sizeof(double) * c->n_nodes;
  if (Cw) CUDA_TRY(c, cudaMemcpyAsync(Cw, c->Cw, b, cudaMemcpyDeviceToDevice, c->stream));
  if (Dw) CUDA_TRY(c, cudaMemcpyAsync(Dw, c->Dw, b, cudaMemcpyDeviceToDevice, c->stream));
  if (Cinv) CUDA_TRY(c, cudaMemcpyAsync(Cinv, c->Cinv, b, cudaMemcpyDeviceToDevice, c->stream));
  if (Dinv) CUDA_TRY(c, cudaMemcpyAsync(Dinv, c->Dinv, b, cudaMemcpyDeviceToDevice, c->stream));
  return WB_OK;
}

wb_status wb_get_jacobi(wb_ctx* c, double* dKl, double* dKr) {
  wb_status s = check_ctx(c, true);
  if (s) return s;
  const size_t b = sizeof(double) * c->n_p;
  if (dKl) CUDA_TRY(c, cudaMemcpyAsync(dKl, c->dKl, b, cudaMemcpyDeviceToDevice, c->stream));
  if (dKr) CUDA_TRY(c, cudaMemcpyAsync(dKr, c->dKr, b, cudaMemcpyDeviceToDevice, c->stream));
  return WB_OK;
}

wb_status wb_query(wb_ctx* c, const char* key, double* value) {
  if (!c || !key || !value) return WB_EINVAL;
  if (!strcmp(key, "n_nonpos_Cw")) *value = (double)c->n_nonpos[0];
  else if (!strcmp(key, "n_nonpos_Dw")) *value = (double)c->n_nonpos[1];
  else if (!strcmp(key, "n_el")) *value = (double)c->n_el;
  else if (!strcmp(key, "n_p")) *value = (double)c->n_p;
  else if (!strcmp(key, "n_v")) *value = (double)c->n_v;
  else if (!strcmp(key, "kernel_launches")) *value = (double)c->launches;
  else if (!strcmp(key, "last_pcg_stop_iter")) {
    int st[1024];
    int n = c->it_cap + 1 < 1024 ? c->it_cap + 1 : 1024;
    CUDA_TRY(c, cudaMemcpyAsync(st, c->stop, sizeof(int) * n, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    int first = -1;
    for (int i = 0; i < n; ++i)
      if (st[i]) { first = i; break; }
    *value = first;
  } else
    return set_err(c, WB_EINVAL, "unknown query key '%s'", key);
  return WB_OK;
}

wb_status wb_sync(wb_ctx* c) {
  if (!c) return WB_EINVAL;
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  CUDA_TRY(c, cudaGetLastError());
  return WB_OK;
}

}  // extern "C"
