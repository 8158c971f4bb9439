// wbfbt.cu -- host side of libwbfbt.so: the C ABI of include/wbfbt.h.
//
// The context owns all workspace; every call enqueues kernels on the context
// stream.  See DESIGN.md for the data layout and the kernel list.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <new>

#include "../../include/wbfbt.h"
#include "kernels_k2.cuh"
#include "slab_dd.cuh"

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
  int last_pcg_iters = -1;  // iteration count of the last PCG solve (its histories are on the device)
  bool nonpos_pending = false;  // icount[1..2] not yet copied to n_nonpos
  // work vectors
  double* E = nullptr;                 // element-local velocity values, 3*nq*n_el
  double *tv = nullptr, *tw = nullptr;  // n_v
  // PCG vectors, mode-major v[m*n_el + e]: x, r, p (double buffer), q
  double *px = nullptr, *pr = nullptr, *pp = nullptr, *pp1 = nullptr, *pq = nullptr;
  double* pz = nullptr;  // z = Minv r, stored by the PCG init/update kernels for the TMA Poisson kernel
  PLay pl = {};        // storage of the PCG vectors (kernels.cuh)
  bool ylay = false;   // y-fastest padded PCG storage: contexts of the TMA Poisson kernel
  // CUDA graphs of the PCG iteration loop, keyed by (side, iters)
  // a captured loop: kind 0 = PCG iterations, 1 = Chebyshev iterations (interval lo, hi)
  struct GraphEntry {
    int kind = 0, side = 0, iters = 0;
    double lo = 0.0, hi = 0.0;
    long long n_launch = 0;
    cudaGraphExec_t exec = nullptr;
  };
  static constexpr int MAX_GRAPHS = 16;
  bool in_capture = false;  // a caller is capturing a graph on this context's stream: launch directly
  GraphEntry graphs[MAX_GRAPHS];
  int n_graphs = 0;
  cudaStream_t cap_stream = nullptr;
  double *s0 = nullptr, *s1 = nullptr, *s2 = nullptr;  // n_p scratch
  // scalars
  double* partial = nullptr;  // reduction partials
  double *pqp = nullptr, *rzp = nullptr;  // PCG deferred-reduction partials (<p,Kp> per K block, <r,Mr> per vector block)
  unsigned* counter = nullptr;
  double* scal = nullptr;  // [0..7] misc totals, then rz_hist, pq_hist, rzn_hist
  int* stop = nullptr;
  int it_cap = 0;
  unsigned long long* icount = nullptr;  // [0] bad mu, [1] nonpos Cw, [2] nonpos Dw
  int red_blocks = 0, max_partials = 0, nsm = 148;
  double* stage = nullptr;  // wb_hotpath_host staging (lazily allocated)
  cudaStream_t copy_stream = nullptr;  // wb_hotpath_host: copies overlapped with compute
  cudaEvent_t ev_in = nullptr, ev_ab = nullptr, ev_bt = nullptr, ev_done = nullptr, ev_p = nullptr;
  // k = 2 tile-assembled A (4x4x4 tiles): upper-shell and lower-face node partials
  // (L2-resident), summed by the skeleton kernel; mut is tile-blocked for k = 2
  double* Fu = nullptr;
  double* mueff = nullptr;  // n_el * n_q: the viscosity-gradient weights' mu_eff (option "weights" 1, R17)
  // diag(A) and the velocity smoother (R18), allocated on first use: k = 2 element buffer
  // (3 components), mask / diag(A), a third n_v scratch vector
  double *E3 = nullptr, *dAinv = nullptr, *tq = nullptr;
  bool dA_valid = false;
  // FGMRES Stokes solve (R19): Krylov bases V (m+1 vectors) and Z (m), work vectors, an
  // n_v scratch, device scalars; sized for the largest restart length used so far
  double *gV = nullptr, *gZ = nullptr, *gw = nullptr, *gb = nullptr, *gx = nullptr, *gsa = nullptr,
         *gh = nullptr;
  double* gls = nullptr;  // FGMRES least-squares state on the device: R (m x m), cs, sn, g, y, residual
  double* gres_h = nullptr;  // pinned host copy of the residual estimate (2 doubles)
  int g_m = 0;
  // wBFBT inner Poisson solves: 0 = Jacobi-PCG (a9), 1 = Chebyshev-Jacobi on [cheb_lo, cheb_hi]
  // per side (0 = l, 1 = r), set by wb_set_inner_cheb
  int inner = 0;
  double cheb_lo[2] = {0.0, 0.0}, cheb_hi[2] = {0.0, 0.0};
  int weights = 0;
  int n_tiles = 0;
  int use_graph = 1;
  int k_var = 1;  // k = 2 fused K variant: 0 = 2 CTAs/SM (register-capped), 1 = 1 CTA/SM (faster: L1 left free)
  // TMA variant of the fused K kernel (k = 2, even N, large meshes): tensor maps over the
  // mode-major PCG vectors and over row-padded copies of C_w^-1 / D_w^-1
  bool tma_ok = false;
  int use_tma = 1;
  int k_ws = 0;  // 1: the TMA Poisson operator runs warp-specialised (k_K2_ws)
  int k2_pair = 0;  // 1: the TMA Poisson kernel computes the class-(1, *) pencils with their class-(0, *) partners
  double *XpL = nullptr, *XpR = nullptr;  // C_w^-1, D_w^-1 in the TMA kernel's X-block layout (k_x_tiles)
  // k = 2, even N: MinvL | XpL | x r p p' q z | MinvR | XpR carved from one slab (each
  // side's PCG working set contiguous; a persisting L2 access-policy window over it was
  // measured and gave no gain)
  double* slab = nullptr;
  CUtensorMap tm_pp, tm_pp1, tm_pz, tm_pr, tm_mL, tm_mR;
  // node-owner z-march Poisson kernel (k2_zm.cuh): tensor maps with its per-layer box,
  // X prescaled on the padded nodal grid, option "k_zm" (default on), z-chunk length
  bool zm_ok = false, xz_valid = false;
  int use_zm = 0, zm_zc = 4, zm_var = 0;
  double *XzL = nullptr, *XzR = nullptr;
  static constexpr int ZM_NV = 5;  // kernel variants (tile shape, CTAs per SM): zm_variants below
  CUtensorMap tz[ZM_NV][3];        // per variant: maps of pp, pp1, pz
  // k = 3, 4 standalone B^T / B: 1 = B^T by the tile kernel (k4_fused.cuh), 2 = B^T and B by the tile
  // kernels, 0 = the element kernels (+ gather).  Measured at C4: B^T 33 vs 43 us, B 54 vs 23 us.
  // k = 2 B / B^T: 0 = tile / box kernels, 2 / 4 / 8 = z-marching column kernels (k2_zc.cuh) with CZ
  // element layers per chunk, -1 = auto (4 on meshes with N >= 48, else 0)
  int bbt_zc = -1;
  int k4bt = 1;
  int k4f = 1, k4_var = 1;  // k = 3, 4: fused Poisson kernel (k4_fused.cuh) on, its tile variant
  // k = 4, even N: TMA tensor maps of the fused kernel's tile variant 1 (z, p boxes; X with
  // padded rows X4L / X4R)
  bool tma4_ok = false;
  double *X4L = nullptr, *X4R = nullptr;
  struct K4Maps { CUtensorMap pp, pp1, pz, xL, xR; };
  K4Maps tm4[4];  // per TMA tile shape: 4 x 4 x 2 (k4_var 1, 6, 8), 4 x 2 x 2 (5), 4 x 4 x 3 (7), 4 x 3 x 2 (9)
  int kz = 0;  // TMA Poisson kernel: 1 = z = Minv r stored by the PCG update and loaded as one box; 0 = r + Minv boxes (default: faster with the y-fastest storage)
  int k_dbg = 0;  // timing probe bits for the fused K kernel (results invalid when nonzero)
  // profiling: CUDA-event pairs around every Poisson-operator launch (direct launches)
  int profile = 0;
  static constexpr int PROF_MAX = 4096;
  cudaEvent_t prof_ev[2 * PROF_MAX] = {};
  int prof_n = 0;
  bool prof_cap = false;  // profiling inside a stream capture: event-record graph nodes
  std::vector<cudaGraphExec_t> prof_execs;  // the profiled loops' graphs
  long long launches = 0;
  struct DD* dd = nullptr;  // z-slab domain decomposition state (slab contexts only; wb_slab_create)
  struct MGH* mg = nullptr;  // pressure multigrid hierarchy (R20), built by wb_setup_mg
  // Schur-complement variant of the Stokes preconditioner: 0 = wBFBT,
  // 1 = diag(A)-BFBT, 2 = M_p(1/mu)^-1 element blocks (R21, built in
  // wb_set_viscosity when selected)
  int schur = 0;
  bool dab_valid = false, mp_valid = false;
  double *dKd = nullptr, *mKd = nullptr, *dv = nullptr;                       // diag(A)-BFBT Poisson
  double *gp_r = nullptr, *gp_z = nullptr, *gp_p = nullptr, *gp_q = nullptr, *gp_x = nullptr,
         *gp_y = nullptr, *gp_s = nullptr;                                    // its PCG (element-major)
  double* mpinv = nullptr;                                                   // n_el x n_m^2
  char err[512] = {0};
};

// Pressure multigrid (R20): level l = 0 is the context itself, l >= 1 are internal
// k = 2 contexts on the N / 2^l meshes; per level element-major work vectors.
struct MGH {
  int nl = 0, nu = 3;
  int Ns[16] = {}, Ks[16] = {};  // level mesh and order (k = 4: a spectral level to k = 2 first)
  wb_ctx* lev[16] = {};
  double lam[2][16] = {};
  double *b[16] = {}, *x[16] = {}, *r[16] = {}, *t[16] = {};
  double *rk = nullptr, *zk = nullptr, *pk = nullptr, *qk = nullptr, *xk = nullptr;  // MG-PCG on level 0
  double* s = nullptr;  // device scalars: rz, pq, rz', stop
  int inner_iters = 0;  // wBFBT inner solves by MG-PCG with this many iterations (0: off)
  // velocity multigrid (R22), built when wb_setup_mg gets mu: coarsened viscosities (levels
  // >= 1, owned), SoA n_v work vectors per level, Chebyshev scales of A_l
  bool vel = false;
  double* mu[16] = {};
  double *vb[16] = {}, *vx[16] = {}, *vr[16] = {}, *vt[16] = {};
  double vlam[16] = {};
  double *vin = nullptr, *vout = nullptr;  // fixed in/out of the captured velocity cycles
  int vcycles = 0;  // Stokes At^-1 by this many V-cycles (0: the Chebyshev smoother, R18)
};
// z-slab domain decomposition: this rank's place in the z-stack, the
// caller's communicator, the global Dirichlet mask and the element-major PCG vectors
struct DD {
  int rank = 0, nranks = 1;
  bool have_comm = false;
  wb_slab_comm comm{};
  double* own_scal = nullptr;  // nranks = 1 without a communicator: local scalar slots
  double* gm = nullptr;        // n_nodes: 0 on the global boundary, else 1
  double* vs = nullptr;        // n_v scratch (masked input of A, nodal B^T p of K_w)
  double *r = nullptr, *z = nullptr, *p = nullptr, *q = nullptr, *x = nullptr, *y = nullptr;  // n_p
  double* mK[2] = {nullptr, nullptr};  // pinv(diag K_side), element-major
  double* scal() const { return have_comm ? comm.scal : own_scal; }
};
void mg_free(wb_ctx* c);
wb_status run_mgcg(wb_ctx* c, int side, const double* b, double* x, int iters);
wb_status run_vmg(wb_ctx* c, const double* b, double* x);

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
// grid of a pure streaming kernel (no reduction partials): one item per thread, up to 16
// waves of 148 SMs (the grid-stride loop covers the rest) -- enough loads in flight to
// approach HBM bandwidth; the reduction grid (red_blocks) leaves the SMs latency-bound here
inline unsigned stream_blocks(int64_t items) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(nblk(items, VBS), 148 * 16));
}

bool overlaps(const void* a, size_t na, const void* b, size_t nb) {
  const char* x = (const char*)a;
  const char* y = (const char*)b;
  return x < y + nb && y < x + na;
}

// scalar slots
// S_SUM..S_SUM+1: constant-mode sums; S_DMAX, S_DMAX+1: max|diag K_l|, max|diag K_r|; S_SCR: scratch dot
enum { S_SUM = 0, S_DMAX = 2, S_SCR = 4, S_NSCAL = 8 };
// rz_hist[i] = rz_i (i = 0..it_cap+1), pq_hist[i] = <p_i, K p_i>, stop[i]: iteration i is skipped
inline double* rz_hist(wb_ctx* c) { return c->scal + S_NSCAL; }
inline double* pq_hist(wb_ctx* c) { return c->scal + S_NSCAL + (c->it_cap + 2); }

void clear_graphs(wb_ctx* c);

wb_status ensure_iters(wb_ctx* c, int iters) {
  if (iters + 2 <= c->it_cap) return WB_OK;
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  clear_graphs(c);
  if (c->scal) cudaFree(c->scal);
  if (c->stop) cudaFree(c->stop);
  c->scal = nullptr; c->stop = nullptr;
  int cap = iters + 2 < 128 ? 128 : iters + 2;
  if (cudaMalloc(&c->scal, sizeof(double) * (S_NSCAL + 2 * (cap + 2))) != cudaSuccess ||
      cudaMalloc(&c->stop, sizeof(int) * (cap + 2)) != cudaSuccess) {
    c->it_cap = 0;
    return set_err(c, WB_ENOMEM, "scalar workspace allocation failed");
  }
  CUDA_TRY(c, cudaMemsetAsync(c->scal, 0, sizeof(double) * (S_NSCAL + 2 * (cap + 2)), c->stream));
  CUDA_TRY(c, cudaMemsetAsync(c->stop, 0, sizeof(int) * (cap + 2), c->stream));
  c->it_cap = cap;
  return WB_OK;
}

// elements per block of the k = 4 A slice kernel (9 NQ doubles of shared memory each)
#ifndef A4_NE
#define A4_NE 4
#endif
// ---------------------------------------------------------------- kernel dispatch helpers
template <int K>
wb_status launch_A_t(wb_ctx* c, const double* u, double* out_E, int nomask) {
  if constexpr (K == 2) {  // k = 2 goes through the tile kernels (run_A)
    return set_err(c, WB_ESTATE, "internal: element-local A path is not used for k = 2");
  } else {
    constexpr int NE = (K == 3) ? 8 : A4_NE;
    const size_t smem = (size_t)NE * 9 * Ord<K>::NQ * sizeof(double);  // attribute set in configure_kernels
    k_A_slice<K, NE><<<nblk(c->n_el, NE), NE * (K + 1) * (K + 1), smem, c->stream>>>(c->mut, u, out_E, c->G, nomask);
    LAUNCH_CHECK(c);
    return WB_OK;
  }
}

template <int K>
wb_status launch_gather_t(wb_ctx* c, const double* s, double* y, int nomask) {
  k_gather<K><<<nblk(c->n_nodes, 256), 256, 0, c->stream>>>(c->E, s, y, c->G, nomask);
  LAUNCH_CHECK(c);
  return WB_OK;
}

#ifndef RED_MULT
#define RED_MULT 2  // blocks per SM of the PCG vector kernels (their rz partials: red_blocks)
#endif
#ifndef BSPLIT_EPB
#define BSPLIT_EPB 16  // elements per block of the generic split B kernel (k = 3, 4; >= 8, see pqp)
#endif
template <int K>
wb_status launch_BT_t(wb_ctx* c, const double* p, const int* stop, int64_t se, int64_t sm) {
  if constexpr (K == 2)
    k_BT_elem<K><<<nblk(c->n_el, 128), 128, 0, c->stream>>>(p, c->E, c->G, c->sB, stop, se, sm);
  else
    k_BT_split<K><<<nblk(c->n_el * 3 * (K + 1), 256), 256, 0, c->stream>>>(p, c->E, c->G, c->sB, stop, se, sm);
  LAUNCH_CHECK(c);
  return WB_OK;
}

template <int K>
wb_status launch_B_t(wb_ctx* c, const double* u, const double* xs, double* p, int nomask, const int* stop,
                     const double* dv, double* total, int64_t se, int64_t sm) {
  constexpr int BS = 128;
  // dv: fused <p_out, dv> block partials into `total` (deferred reduction, PCG only)
  if constexpr (K == 2) {
    k_B<K, BS><<<nblk(c->n_el, BS), BS, 0, c->stream>>>(u, xs, p, c->G, c->sB, nomask, stop, dv,
                                                         dv ? total : nullptr, c->counter, nullptr, se, sm);
  } else {
    constexpr int EPB = BSPLIT_EPB;
    k_B_split<K, EPB><<<nblk(c->n_el, EPB), BSplit<K, EPB>::NT, 0, c->stream>>>(u, xs, p, c->G, c->sB, nomask, stop,
                                                                                dv, dv ? total : nullptr, se, sm);
  }
  LAUNCH_CHECK(c);
  return WB_OK;
}
// number of dot partials launch_B_t leaves (one per block)
inline int b_blocks(const wb_ctx* c) { return (int)nblk(c->n_el, c->k == 2 ? 128 : BSPLIT_EPB); }

// fused k = 2 Poisson operator (+ PCG direction update), see k2_fused.cuh
struct PcgArgs {  // PCG iteration context for the first kernel of an iteration
  int it = 0, ctl = 0;
};

template <int TX, int TY, int TZ, int MINB>
wb_status launch_k2f_t(wb_ctx* c, const double* pold, double* pnew, const double* r, const double* Minv,
                       const double* X, double* q, int mode, PcgArgs a, int* npq) {
  const int N = c->N;
  const int nt = ((N + TX - 1) / TX) * ((N + TY - 1) / TY) * ((N + TZ - 1) / TZ);
  // persistent CTAs: as many as are resident at once (fixed per context -> fixed reduction order)
  int occ = 0;
  CUDA_TRY(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_K2_fused<TX, TY, TZ, MINB>, FK2<TX, TY, TZ>::NTH,
                                                            FK2<TX, TY, TZ>::SMEM));
  const int grid = std::max(1, std::min(nt, occ * c->nsm));
  k_K2_fused<TX, TY, TZ, MINB><<<grid, FK2<TX, TY, TZ>::NTH, FK2<TX, TY, TZ>::SMEM, c->stream>>>(
      pold, pnew, r, Minv, X, q, c->G, c->sB, mode | c->k_dbg, a.it, a.ctl, c->rzp, c->red_blocks, rz_hist(c), pq_hist(c),
      c->stop, c->pqp);
  LAUNCH_CHECK(c);
  *npq = grid;
  return WB_OK;
}
// fused k = 3, 4 Poisson operator (+ PCG direction update), one CTA per element tile
template <int K, int TX, int TY, int TZ, int MINB, bool TMA = false, bool XG = false>
wb_status launch_k4f_t(wb_ctx* c, const double* pold, double* pnew, const double* X, double* q, int mode, PcgArgs a,
                       int* npq, const CUtensorMap* tp = nullptr, const CUtensorMap* tz = nullptr,
                       const CUtensorMap* tx = nullptr) {
  using F = FK4<K, TX, TY, TZ, TMA, XG>;
  const int N = c->N;
  const int nt = ((N + TX - 1) / TX) * ((N + TY - 1) / TY) * ((N + TZ - 1) / TZ);
  static const CUtensorMap none{};
  k_K4_fused<K, TX, TY, TZ, MINB, TMA, XG><<<nt, F::NTH, F::SMEM, c->stream>>>(
      pold, pnew, c->pz, X, q, c->G, c->sB, mode, a.it, a.ctl, c->rzp, c->red_blocks, rz_hist(c), pq_hist(c),
      c->stop, c->pqp, tp ? *tp : none, tz ? *tz : none, tx ? *tx : none);
  LAUNCH_CHECK(c);
  *npq = nt;
  return WB_OK;
}
#define K4_VARIANTS(X_)                                                                                         \
  X_(4, 3, 3, 3, 1, false) X_(4, 4, 4, 2, 2, false) X_(4, 4, 4, 2, 2, true) X_(4, 2, 2, 2, 2, false)             \
  X_(4, 4, 4, 4, 1, false) X_(3, 3, 3, 3, 2, false) X_(3, 4, 4, 4, 2, false) X_(4, 4, 2, 2, 3, false)           \
  X_(4, 4, 2, 2, 3, true) X_(4, 4, 3, 2, 2, true) X_(4, 4, 3, 2, 2, false)
constexpr int K4_NV = 10;  // variants per order: k4_var indexes them (k = 3 has 2)
wb_status run_k4f(wb_ctx* c, const double* pold, double* pnew, const double* X, double* q, int mode, PcgArgs a,
                  int* npq) {
  if (c->k == 4) {
    switch (c->k4_var) {
      case 1:    // 4 x 4 x 2 tiles, TMA staging where the maps exist (else the same kernel with loads)
      case 5: {  // 4 x 2 x 2 tiles, TMA, three CTAs per SM
        const wb_ctx::K4Maps& m = c->tm4[c->k4_var == 1 ? 0 : 1];
        const CUtensorMap* tp = pold == c->pp ? &m.pp : (pold == c->pp1 ? &m.pp1 : nullptr);
        const CUtensorMap* tx = X == c->Cinv ? &m.xL : (X == c->Dinv ? &m.xR : nullptr);
        if (c->k4_var == 5) {
          if (c->tma4_ok && tp && tx)
            return launch_k4f_t<4, 4, 2, 2, 3, true>(c, pold, pnew, X, q, mode, a, npq, tp, &m.pz, tx);
          return launch_k4f_t<4, 4, 2, 2, 3>(c, pold, pnew, X, q, mode, a, npq);
        }
        if (c->tma4_ok && tp && tx)
          return launch_k4f_t<4, 4, 4, 2, 2, true>(c, pold, pnew, X, q, mode, a, npq, tp, &m.pz, tx);
        return launch_k4f_t<4, 4, 4, 2, 2>(c, pold, pnew, X, q, mode, a, npq);
      }
      case 6: {  // 4 x 4 x 2 tiles, the three components concurrently (k_K4_3c), TMA only
        const wb_ctx::K4Maps& m = c->tm4[0];
        const CUtensorMap* tp = pold == c->pp ? &m.pp : (pold == c->pp1 ? &m.pp1 : nullptr);
        const CUtensorMap* tx = X == c->Cinv ? &m.xL : (X == c->Dinv ? &m.xR : nullptr);
        if (!(c->tma4_ok && tp && tx)) return launch_k4f_t<4, 4, 4, 2, 2>(c, pold, pnew, X, q, mode, a, npq);
        using H = FK43<4, 4, 4, 2>;
        const int N = c->N, nt = ((N + 3) / 4) * ((N + 3) / 4) * ((N + 1) / 2);
        k_K4_3c<4, 4, 4, 2><<<nt, H::NTH, H::SMEM, c->stream>>>(pnew, q, c->G, c->sB, mode, a.it, a.ctl, c->rzp,
                                                                c->red_blocks, rz_hist(c), pq_hist(c), c->stop,
                                                                c->pqp, *tp, m.pz, *tx);
        LAUNCH_CHECK(c);
        *npq = nt;
        return WB_OK;
      }
      case 7:    // X from the padded global copy (no Xs): 4 x 4 x 3 tiles (one wave at C4), 4 x 4 x 2
      case 8: {
        const wb_ctx::K4Maps& m = c->tm4[c->k4_var == 7 ? 2 : 0];
        const CUtensorMap* tp = pold == c->pp ? &m.pp : (pold == c->pp1 ? &m.pp1 : nullptr);
        const double* xg = X == c->Cinv ? c->X4L : (X == c->Dinv ? c->X4R : nullptr);
        if (!(c->tma4_ok && tp && xg)) return launch_k4f_t<4, 4, 4, 2, 2>(c, pold, pnew, X, q, mode, a, npq);
        if (c->k4_var == 7)
          return launch_k4f_t<4, 4, 4, 3, 2, true, true>(c, pold, pnew, xg, q, mode, a, npq, tp, &m.pz, &m.xL);
        return launch_k4f_t<4, 4, 4, 2, 2, true, true>(c, pold, pnew, xg, q, mode, a, npq, tp, &m.pz, &m.xL);
      }
      case 9: {  // 4 x 3 x 2 tiles (576 at C4: 1.95 waves of two CTAs per SM), TMA
        const wb_ctx::K4Maps& m = c->tm4[3];
        const CUtensorMap* tp = pold == c->pp ? &m.pp : (pold == c->pp1 ? &m.pp1 : nullptr);
        const CUtensorMap* tx = X == c->Cinv ? &m.xL : (X == c->Dinv ? &m.xR : nullptr);
        if (c->tma4_ok && tp && tx)
          return launch_k4f_t<4, 4, 3, 2, 2, true>(c, pold, pnew, X, q, mode, a, npq, tp, &m.pz, tx);
        return launch_k4f_t<4, 4, 3, 2, 2>(c, pold, pnew, X, q, mode, a, npq);
      }
      case 2: return launch_k4f_t<4, 2, 2, 2, 2>(c, pold, pnew, X, q, mode, a, npq);
      case 3: return launch_k4f_t<4, 4, 4, 4, 1>(c, pold, pnew, X, q, mode, a, npq);
      case 4: return launch_k4f_t<4, 4, 4, 2, 2>(c, pold, pnew, X, q, mode, a, npq);
      default: return launch_k4f_t<4, 3, 3, 3, 1>(c, pold, pnew, X, q, mode, a, npq);
    }
  }
  if (c->k4_var == 1) return launch_k4f_t<3, 4, 4, 4, 2>(c, pold, pnew, X, q, mode, a, npq);
  return launch_k4f_t<3, 3, 3, 3, 2>(c, pold, pnew, X, q, mode, a, npq);
}

// element tile of the k = 2 A kernels and its CTAs per SM
#ifndef A_TX
#define A_TX 4
#endif
#ifndef A_TY
#define A_TY 4
#endif
#ifndef A_TZ
#define A_TZ 2
#endif
#ifndef A_MINB
#define A_MINB 4
#endif
// element tile of the TMA Poisson kernel and its CTAs per SM
#ifndef TMA_TX
#define TMA_TX 4
#define TMA_TY 8
#define TMA_TZ 8
#define TMA_MINB 1
#endif
// length (doubles) of one side's X in the TMA kernel's tile-blocked pencil layout
int64_t xt_len(int N) {
  const int64_t nt = (int64_t)((N + TMA_TX - 1) / TMA_TX) * ((N + TMA_TY - 1) / TMA_TY) * ((N + TMA_TZ - 1) / TMA_TZ);
  return nt * FKT<TMA_TX, TMA_TY, TMA_TZ>::XTB;
}
const CUtensorMap* tmap_of(wb_ctx* c, const double* p) {
  if (p == c->pp) return &c->tm_pp;
  if (p == c->pp1) return &c->tm_pp1;
  if (p == c->pz) return &c->tm_pz;
  if (p == c->pr) return &c->tm_pr;
  if (p == c->MinvL) return &c->tm_mL;
  if (p == c->MinvR) return &c->tm_mR;
  return nullptr;
}

// the k = 2 Poisson operator runs as the TMA kernel (k_K2_tma); the PCG init/update
// kernels then also store z = Minv r, which it reads instead of r and Minv
// smallest mesh (elements) that gets the TMA Poisson kernel's y-fastest storage (even N only).
// Every even mesh by default: measured against the pointer kernel (4 x 4 x 4 tiles) on the
// small configs, wBFBT applies/s C1 2056 -> 2353, C2 797 -> 1012, C3 598 -> 876 (round 1 kept
// the pointer kernel below two 256-element tiles per SM).  WB_TMA_MIN_EL overrides it at
// wb_create (measurement only).
int64_t tma_min_el() {
  static int64_t v = -1;
  if (v < 0) {
    const char* e = getenv("WB_TMA_MIN_EL");
    v = e ? atoll(e) : 0;
  }
  return v;
}
bool tma_active(const wb_ctx* c) { return c->k == 2 && c->tma_ok && c->use_tma && c->ylay; }
// the node-owner z-march kernel (k2_zm.cuh) replaces it where set up; it always reads z
bool zm_active(const wb_ctx* c) { return tma_active(c) && c->zm_ok && c->use_zm; }
// X = sB^2 C_w^-1, sB^2 D_w^-1 on the padded nodal grid of the z-march kernel: built eagerly
// (setup with the option on, or when the option is switched on), never inside a captured loop
wb_status build_xz(wb_ctx* c) {
  const double s2 = c->sB * c->sB;
  k_xz_build<<<4 * c->nsm, 256, 0, c->stream>>>(c->Cinv, c->XzL, c->N, s2);
  k_xz_build<<<4 * c->nsm, 256, 0, c->stream>>>(c->Dinv, c->XzR, c->N, s2);
  if (cudaGetLastError() != cudaSuccess) return WB_ECUDA;
  c->xz_valid = true;
  return WB_OK;
}
// k = 3, 4: the fused Poisson kernel (k4_fused.cuh); it reads z = Minv r from the PCG kernels
bool k4f_active(const wb_ctx* c) { return c->k >= 3 && c->k4f; }
double* z_out(const wb_ctx* c) {
  return (tma_active(c) && (c->kz || zm_active(c))) || k4f_active(c) ? c->pz : nullptr;
}
const CUtensorMap* zmap_of(wb_ctx* c, const double* p) {
  if (p == c->pp) return &c->tz[c->zm_var][0];
  if (p == c->pp1) return &c->tz[c->zm_var][1];
  if (p == c->pz) return &c->tz[c->zm_var][2];
  return nullptr;
}
// z-march kernel variants: (TY, TX, CTAs per SM)
struct ZmVar { int ty, tx, minb; };
constexpr ZmVar zm_variants[wb_ctx::ZM_NV] = {{16, 8, 2}, {16, 8, 3}, {8, 8, 4}, {8, 8, 5}, {32, 4, 2}};
template <int TY, int TX, int MINB>
void launch_zm_t(wb_ctx* c, const CUtensorMap* tp, const CUtensorMap* tz, const double* xz, double* pnew, double* q,
                 int mode, PcgArgs a, int* npq) {
  using K = ZMK<TY, TX>;
  const int N = c->N, zc = c->zm_zc;
  const int grid = ((N + TY - 1) / TY) * ((N + TX - 1) / TX) * ((N + zc - 1) / zc);
  k_K2_zm<TY, TX, MINB><<<grid, K::NTH, K::SMEM, c->stream>>>(*tp, *tz, xz, pnew, q, N, zc, mode | c->k_dbg, a.it,
                                                               a.ctl, c->rzp, c->red_blocks, rz_hist(c), pq_hist(c),
                                                               c->stop, c->pqp, c->pl);
  *npq = grid;
}
template <int TY, int TX, int MINB>
bool attr_zm_t() {
  return cudaFuncSetAttribute(k_K2_zm<TY, TX, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)ZMK<TY, TX>::SMEM) == cudaSuccess;
}

wb_status run_k2f(wb_ctx* c, const double* pold, double* pnew, const double* r, const double* Minv, const double* X,
                  double* q, int mode, PcgArgs a, int* npq) {
  if (zm_active(c)) {
    const CUtensorMap *tp = zmap_of(c, pold), *tz = zmap_of(c, c->pz);
    const double* xz = X == c->Cinv ? c->XzL : (X == c->Dinv ? c->XzR : nullptr);
    if (tp && tz && xz && c->xz_valid && (mode == 2 || r == c->pr)) {
      switch (c->zm_var) {
        case 0: launch_zm_t<16, 8, 2>(c, tp, tz, xz, pnew, q, mode, a, npq); break;
        case 1: launch_zm_t<16, 8, 3>(c, tp, tz, xz, pnew, q, mode, a, npq); break;
        case 2: launch_zm_t<8, 8, 4>(c, tp, tz, xz, pnew, q, mode, a, npq); break;
        case 3: launch_zm_t<8, 8, 5>(c, tp, tz, xz, pnew, q, mode, a, npq); break;
        default: launch_zm_t<32, 4, 2>(c, tp, tz, xz, pnew, q, mode, a, npq); break;
      }
      LAUNCH_CHECK(c);
      return WB_OK;
    }
  }
  if (tma_active(c)) {
    using KT = FKT<TMA_TX, TMA_TY, TMA_TZ>;
    const CUtensorMap *tp = tmap_of(c, pold), *tz = tmap_of(c, c->kz ? c->pz : c->pr), *tm = tmap_of(c, Minv);
    const double* xt = X == c->Cinv ? c->XpL : (X == c->Dinv ? c->XpR : nullptr);  // X in pencil layout
    if (tp && tz && tm && xt && (mode == 2 || r == c->pr)) {
      const int N = c->N;
      const int nt = ((N + TMA_TX - 1) / TMA_TX) * ((N + TMA_TY - 1) / TMA_TY) * ((N + TMA_TZ - 1) / TMA_TZ);
      const int grid = std::max(1, std::min(nt, TMA_MINB * c->nsm));  // persistent, all resident
      using KW = FKW<TMA_TX, TMA_TY, TMA_TZ>;
      auto kern = c->k_ws ? (c->kz ? k_K2_ws<TMA_TX, TMA_TY, TMA_TZ, true> : k_K2_ws<TMA_TX, TMA_TY, TMA_TZ, false>)
                  : c->k2_pair ? (c->kz ? k_K2_tma<TMA_TX, TMA_TY, TMA_TZ, TMA_MINB, true, true>
                                        : k_K2_tma<TMA_TX, TMA_TY, TMA_TZ, TMA_MINB, false, true>)
                               : (c->kz ? k_K2_tma<TMA_TX, TMA_TY, TMA_TZ, TMA_MINB, true>
                                        : k_K2_tma<TMA_TX, TMA_TY, TMA_TZ, TMA_MINB, false>);
      const int nth = c->k_ws ? KW::NTH : FK2<TMA_TX, TMA_TY, TMA_TZ>::NTH;
      const size_t smem = c->k_ws ? KW::SMEM : KT::SMEM;
      kern<<<grid, nth, smem, c->stream>>>(
          *tp, *tz, *tm, xt, pnew, q, c->G, c->sB, mode | c->k_dbg, a.it, a.ctl, c->rzp, c->red_blocks, rz_hist(c),
          pq_hist(c), c->stop, c->pqp, c->pl);
      LAUNCH_CHECK(c);
      *npq = grid;
      return WB_OK;
    }
  }
  if (c->n_el >= 148 * 256 * 2)
    return c->k_var == 1 ? launch_k2f_t<4, 8, 8, 1>(c, pold, pnew, r, Minv, X, q, mode, a, npq)
                         : launch_k2f_t<4, 8, 8, 2>(c, pold, pnew, r, Minv, X, q, mode, a, npq);
  return launch_k2f_t<4, 4, 4, 6>(c, pold, pnew, r, Minv, X, q, mode, a, npq);
}

// ---- TMA tensor maps (driver entry point through the runtime; no libcuda link)
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
bool get_encode() {
  if (g_encode) return true;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !fn) {
    cudaGetLastError();
    return false;
  }
  g_encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  return true;
}
// mode-major PCG vector [m][ez][ey][ex]: 4-D map, box = one tile + halo, all modes
// PCG vector in the y-fastest padded storage (PLay, off = 1): 4-D map (y incl. pads, z, x,
// mode), box = the tile's halo (HY, HZ, HX) for all modes
bool make_tm_vec(CUtensorMap* tm, const double* base, int N, int nm) {
  using KT = FKT<TMA_TX, TMA_TY, TMA_TZ>;
  const cuuint64_t ny = (cuuint64_t)N + 2;
  const cuuint64_t dims[4] = {ny, (cuuint64_t)N, (cuuint64_t)N, (cuuint64_t)nm};
  const cuuint64_t strides[3] = {ny * 8, ny * N * 8, ny * N * N * 8};
  const cuuint32_t box[4] = {(cuuint32_t)KT::HY, (cuuint32_t)KT::HZ, (cuuint32_t)KT::HX, (cuuint32_t)nm};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  return g_encode(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void*)base, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// the same storage, box = one layer of the z-march kernel's column tile + halo, all modes
bool make_tm_zm(CUtensorMap* tm, const double* base, int N, int nm, int ty, int tx) {
  const cuuint64_t ny = (cuuint64_t)N + 2;
  const cuuint64_t dims[4] = {ny, (cuuint64_t)N, (cuuint64_t)N, (cuuint64_t)nm};
  const cuuint64_t strides[3] = {ny * 8, ny * N * 8, ny * N * N * 8};
  const cuuint32_t box[4] = {(cuuint32_t)(ty + 2), 1u, (cuuint32_t)(tx + 2), (cuuint32_t)nm};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  return g_encode(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void*)base, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
bool setup_zm(wb_ctx* c) {
  if (!c->ylay || c->nm != 4) return false;
  const int64_t R = 2 * (int64_t)c->N + 2;
  const size_t bx = sizeof(double) * (size_t)(R * R * R);
  if (cudaMalloc(&c->XzL, bx) != cudaSuccess || cudaMalloc(&c->XzR, bx) != cudaSuccess || !attr_zm_t<16, 8, 2>() ||
      !attr_zm_t<16, 8, 3>() || !attr_zm_t<8, 8, 4>() || !attr_zm_t<8, 8, 5>() || !attr_zm_t<32, 4, 2>()) {
    cudaGetLastError();
    return false;
  }
  for (int v = 0; v < wb_ctx::ZM_NV; ++v) {
    const int ty = zm_variants[v].ty, tx = zm_variants[v].tx;
    if (!make_tm_zm(&c->tz[v][0], c->pp, c->N, c->nm, ty, tx) || !make_tm_zm(&c->tz[v][1], c->pp1, c->N, c->nm, ty, tx) ||
        !make_tm_zm(&c->tz[v][2], c->pz, c->N, c->nm, ty, tx))
      return false;
  }
  return true;
}
bool setup_tma(wb_ctx* c) {
  if (!c->ylay) return false;
  const size_t bx = sizeof(double) * (size_t)xt_len(c->N);
  if (!c->slab && (cudaMalloc(&c->XpL, bx) != cudaSuccess || cudaMalloc(&c->XpR, bx) != cudaSuccess)) {
    cudaGetLastError();
    return false;
  }
  if (cudaFuncSetAttribute(k_K2_tma<TMA_TX, TMA_TY, TMA_TZ, TMA_MINB, true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FKT<TMA_TX, TMA_TY, TMA_TZ>::SMEM) != cudaSuccess ||
      cudaFuncSetAttribute(k_K2_tma<TMA_TX, TMA_TY, TMA_TZ, TMA_MINB, false>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FKT<TMA_TX, TMA_TY, TMA_TZ>::SMEM) != cudaSuccess ||
      cudaFuncSetAttribute(k_K2_tma<TMA_TX, TMA_TY, TMA_TZ, TMA_MINB, true, true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FKT<TMA_TX, TMA_TY, TMA_TZ>::SMEM) != cudaSuccess ||
      cudaFuncSetAttribute(k_K2_tma<TMA_TX, TMA_TY, TMA_TZ, TMA_MINB, false, true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FKT<TMA_TX, TMA_TY, TMA_TZ>::SMEM) != cudaSuccess ||
      cudaFuncSetAttribute(k_K2_ws<TMA_TX, TMA_TY, TMA_TZ, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)FKW<TMA_TX, TMA_TY, TMA_TZ>::SMEM) != cudaSuccess ||
      cudaFuncSetAttribute(k_K2_ws<TMA_TX, TMA_TY, TMA_TZ, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)FKW<TMA_TX, TMA_TY, TMA_TZ>::SMEM) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return make_tm_vec(&c->tm_pp, c->pp, c->N, c->nm) && make_tm_vec(&c->tm_pp1, c->pp1, c->N, c->nm) &&
         make_tm_vec(&c->tm_pz, c->pz, c->N, c->nm) && make_tm_vec(&c->tm_pr, c->pr, c->N, c->nm) &&
         make_tm_vec(&c->tm_mL, c->MinvL, c->N, c->nm) && make_tm_vec(&c->tm_mR, c->MinvR, c->N, c->nm);
}

// k = 4 fused Poisson kernel, TMA tile variants: 4-D maps of the mode-major PCG vectors
// [m][ez][ey][ex] (row stride N: N even), box = x from ex0 - 2, 8 wide, the tile's y / z
// halo, all modes; 3-D maps of X with rows padded to nn1 + 1, box = the tile's nodes
template <class F>
bool make_tm4_vec(CUtensorMap* tm, const double* base, int N) {
  const cuuint64_t n = (cuuint64_t)N;
  const cuuint64_t dims[4] = {n, n, n, (cuuint64_t)F::NM};
  const cuuint64_t strides[3] = {n * 8, n * n * 8, n * n * n * 8};
  const cuuint32_t box[4] = {(cuuint32_t)F::BX, (cuuint32_t)F::EY, (cuuint32_t)F::EZ, (cuuint32_t)F::NM};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  return g_encode(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void*)base, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
template <class F>
bool make_tm4_x(CUtensorMap* tm, const double* base, int nn1) {
  const cuuint64_t r = (cuuint64_t)nn1 + 1, n = (cuuint64_t)nn1;
  const cuuint64_t dims[3] = {r, n, n};
  const cuuint64_t strides[2] = {r * 8, r * n * 8};
  const cuuint32_t box[3] = {(cuuint32_t)F::XR, (cuuint32_t)F::NY, (cuuint32_t)F::NZ};
  const cuuint32_t es[3] = {1, 1, 1};
  return g_encode(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)base, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
template <class F>
bool make_tm4(wb_ctx* c, wb_ctx::K4Maps& m) {
  return make_tm4_vec<F>(&m.pp, c->pp, c->N) && make_tm4_vec<F>(&m.pp1, c->pp1, c->N) &&
         make_tm4_vec<F>(&m.pz, c->pz, c->N) && make_tm4_x<F>(&m.xL, c->X4L, c->G.nn1) &&
         make_tm4_x<F>(&m.xR, c->X4R, c->G.nn1);
}
bool setup_tma4(wb_ctx* c) {
  if (c->k != 4 || (c->N & 1) || c->pl.off != 0 || c->pl.sm != c->n_el || !get_encode()) return false;
  const size_t bx = sizeof(double) * (size_t)(c->G.nn1 + 1) * c->G.nn1 * c->G.nn1;
  if (cudaMalloc(&c->X4L, bx) != cudaSuccess || cudaMalloc(&c->X4R, bx) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return make_tm4<FK4<4, 4, 4, 2, true>>(c, c->tm4[0]) && make_tm4<FK4<4, 4, 2, 2, true>>(c, c->tm4[1]) &&
         make_tm4<FK4<4, 4, 4, 3, true>>(c, c->tm4[2]) && make_tm4<FK4<4, 4, 3, 2, true>>(c, c->tm4[3]);
}

wb_status configure_kernels(wb_ctx* c) {
  CUDA_TRY(c, cudaFuncSetAttribute(k_A_tile<A_TX, A_TY, A_TZ, A_MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)Tile2<A_TX, A_TY, A_TZ>::SMEM));
  CUDA_TRY(c, cudaFuncSetAttribute(k_K2_fused<4, 8, 8, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)FK2<4, 8, 8>::SMEM));
  CUDA_TRY(c, cudaFuncSetAttribute(k_K2_fused<4, 8, 8, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)FK2<4, 8, 8>::SMEM));
  CUDA_TRY(c, cudaFuncSetAttribute(k_K2_fused<4, 4, 4, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)FK2<4, 4, 4>::SMEM));
#define K4_ATTR(K_, TX_, TY_, TZ_, MB_, T_)                                                  \
  CUDA_TRY(c, cudaFuncSetAttribute(k_K4_fused<K_, TX_, TY_, TZ_, MB_, T_>,                       \
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FK4<K_, TX_, TY_, TZ_, T_>::SMEM));
  K4_VARIANTS(K4_ATTR)
#undef K4_ATTR
  CUDA_TRY(c, cudaFuncSetAttribute(k_K4_fused<4, 4, 4, 3, 2, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)FK4<4, 4, 4, 3, true, true>::SMEM));
  CUDA_TRY(c, cudaFuncSetAttribute(k_K4_fused<4, 4, 4, 2, 2, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)FK4<4, 4, 4, 2, true, true>::SMEM));
  CUDA_TRY(c, cudaFuncSetAttribute(k_BT4_tile<4, 4, 4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)FB4<4, 4, 4, 2>::SMEM_BT));
  CUDA_TRY(c, cudaFuncSetAttribute(k_BT4_tile<3, 4, 4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)FB4<3, 4, 4, 4>::SMEM_BT));
  CUDA_TRY(c, cudaFuncSetAttribute(k_K4_3c<4, 4, 4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)FK43<4, 4, 4, 2>::SMEM));
  CUDA_TRY(c, cudaFuncSetAttribute(k_A_slice<3, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(8 * 9 * Ord<3>::NQ * sizeof(double))));
  CUDA_TRY(c, cudaFuncSetAttribute(k_A_slice<4, A4_NE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(A4_NE * 9 * Ord<4>::NQ * sizeof(double))));
  return WB_OK;
}

#define DISPATCH_K(c, fn, ...)                                   \
  ((c)->k == 2 ? fn<2>(c, __VA_ARGS__)                           \
               : ((c)->k == 3 ? fn<3>(c, __VA_ARGS__) : fn<4>(c, __VA_ARGS__)))

wb_status run_A(wb_ctx* c, const double* u, double* y, int nomask) {
  if (c->k == 2) {
    const dim3 tg((c->N + A_TX - 1) / A_TX, (c->N + A_TY - 1) / A_TY, (c->N + A_TZ - 1) / A_TZ);  // = n_tiles
    k_A_tile<A_TX, A_TY, A_TZ, A_MINB><<<tg, 3 * A_TX * A_TY * A_TZ, Tile2<A_TX, A_TY, A_TZ>::SMEM,
                                         c->stream>>>(c->mut, u, y, c->Fu, c->G, nomask);
    LAUNCH_CHECK(c);
    k_A_skel<A_TX, A_TY, A_TZ><<<nblk(a2_skel_count<A_TX, A_TY, A_TZ>(c->N), 256), 256, 0, c->stream>>>(
        c->Fu, y, c->G, nomask);
    LAUNCH_CHECK(c);
    return WB_OK;
  }
  wb_status s = DISPATCH_K(c, launch_A_t, u, c->E, nomask);
  if (s) return s;
  return DISPATCH_K(c, launch_gather_t, (const double*)nullptr, y, nomask);
}
// chunk length of the k = 2 z-march B / B^T kernels, 0 = the tile / box kernels
int zc_of(const wb_ctx* c) { return c->bbt_zc >= 0 ? c->bbt_zc : (c->N >= 48 ? 4 : 0); }
// y = M B^T p (X o ... if xs), p[e*se + m*sm]
template <int K, int TX, int TY, int TZ>
void launch_bt4(wb_ctx* c, const double* p, const double* xs, double* y, int nomask, int64_t se, int64_t sm) {
  const int N = c->N, nt = ((N + TX - 1) / TX) * ((N + TY - 1) / TY) * ((N + TZ - 1) / TZ);
  k_BT4_tile<K, TX, TY, TZ><<<nt, FK4<K, TX, TY, TZ>::NTH, FB4<K, TX, TY, TZ>::SMEM_BT, c->stream>>>(
      p, xs, y, c->G, c->sB, nomask, se, sm);
}
template <int K, int TX, int TY, int TZ>
void launch_b4(wb_ctx* c, const double* u, const double* xs, double* p, int nomask, int64_t se, int64_t sm) {
  const int N = c->N, nt = ((N + TX - 1) / TX) * ((N + TY - 1) / TY) * ((N + TZ - 1) / TZ);
  k_B4_tile<K, TX, TY, TZ><<<nt, FB4<K, TX, TY, TZ>::NTH_B, FB4<K, TX, TY, TZ>::SMEM_B, c->stream>>>(
      u, xs, p, c->G, c->sB, nomask, se, sm);
}
wb_status run_BT(wb_ctx* c, const double* p, const double* xs, double* y, int nomask, const int* stop,
                 int64_t se, int64_t sm) {
  if (c->k >= 3 && c->k4bt && !stop) {  // tile kernels (k4_fused.cuh)
    if (c->k == 4) launch_bt4<4, 4, 4, 2>(c, p, xs, y, nomask, se, sm);
    else launch_bt4<3, 4, 4, 4>(c, p, xs, y, nomask, se, sm);
    LAUNCH_CHECK(c);
    return WB_OK;
  }
  if (c->k == 2 && !stop && zc_of(c)) {  // z-marching columns (k2_zc.cuh)
    const int64_t nc = (int64_t)c->G.nn1 * c->G.nn1;
    const int cz = zc_of(c);
    const int64_t nt = nc * ((c->N + cz - 1) / cz);
    const unsigned nb = (unsigned)((nt + 127) / 128);
    if (cz == 2) k_BT_zc2<2><<<nb, 128, 0, c->stream>>>(p, xs, y, c->G, c->sB, nomask, se, sm);
    else if (cz == 4) k_BT_zc2<4><<<nb, 128, 0, c->stream>>>(p, xs, y, c->G, c->sB, nomask, se, sm);
    else k_BT_zc2<8><<<nb, 128, 0, c->stream>>>(p, xs, y, c->G, c->sB, nomask, se, sm);
    LAUNCH_CHECK(c);
    return WB_OK;
  }
  if (c->k == 2) {
    if (stop) {  // (generic-k PCG only; kept for completeness)
      dim3 grid(nblk(c->N + 1, 64), nblk(c->G.nn1, 4), 2 * c->G.nn1);
      k_BT_node2<<<grid, dim3(64, 4), 0, c->stream>>>(p, xs, y, c->G, c->sB, nomask, stop, se, sm);
    } else {
      const int nb = (c->G.nn1 + 7) / 8;
      k_BT_box2<8><<<nb * nb * nb, 256, 0, c->stream>>>(p, xs, y, c->G, c->sB, nomask, se, sm);
    }
    LAUNCH_CHECK(c);
    return WB_OK;
  }
  wb_status s = DISPATCH_K(c, launch_BT_t, p, stop, se, sm);
  if (s) return s;
  return DISPATCH_K(c, launch_gather_t, xs, y, nomask);
}
wb_status run_B(wb_ctx* c, const double* u, const double* xs, double* p, int nomask, const int* stop,
                const double* dv, double* total, int64_t se, int64_t sm) {
  if (c->k >= 3 && c->k4bt == 2 && !stop && !dv) {  // tile kernel (k4_fused.cuh)
    if (c->k == 4) launch_b4<4, 4, 4, 2>(c, u, xs, p, nomask, se, sm);
    else launch_b4<3, 4, 4, 4>(c, u, xs, p, nomask, se, sm);
    LAUNCH_CHECK(c);
    return WB_OK;
  }
  if (c->k == 2 && !stop && !dv && zc_of(c)) {  // z-marching columns (k2_zc.cuh)
    const int cz = zc_of(c);
    const int64_t nt = (int64_t)c->N * c->N * ((c->N + cz - 1) / cz);
    const unsigned nb = (unsigned)((nt + 127) / 128);
    if (cz == 2) k_B_zc2<2><<<nb, 128, 0, c->stream>>>(u, xs, p, c->G, c->sB, nomask, se, sm);
    else if (cz == 4) k_B_zc2<4><<<nb, 128, 0, c->stream>>>(u, xs, p, c->G, c->sB, nomask, se, sm);
    else k_B_zc2<8><<<nb, 128, 0, c->stream>>>(u, xs, p, c->G, c->sB, nomask, se, sm);
    LAUNCH_CHECK(c);
    return WB_OK;
  }
  if (c->k == 2 && !stop && !dv) {
    const int nt = ((c->N + 3) / 4) * ((c->N + 3) / 4) * ((c->N + 3) / 4);
    k_B_tile2<4, 4, 4><<<nt, BTile2<4, 4, 4>::NTH, BTile2<4, 4, 4>::SMEM, c->stream>>>(u, xs, p, c->G, c->sB, nomask,
                                                                                       se, sm);
    LAUNCH_CHECK(c);
    return WB_OK;
  }
  return DISPATCH_K(c, launch_B_t, u, xs, p, nomask, stop, dv, total, se, sm);
}

// Mode-major K_side p_cur -> q (pq_out = <p_cur, q>), p_cur produced from
// (pold, r) by the direction-update `mode` (0: Minv r, 1: Minv r + beta pold,
// 2: pold as is).  Returns the buffer that holds p_cur.
// Mode-major q = K_side p_cur, with the <p_cur, q> block partials in pqp
// (*npq of them), p_cur produced from (pold, r) by the direction-update `mode`
// (0: Minv r, 1: Minv r + beta pold, 2: pold as is).  a.ctl: this is the first
// kernel of PCG iteration a.it (runs pcg_control: stop test, beta).
// Returns the buffer that holds p_cur.
wb_status run_K_pcg(wb_ctx* c, int side, int mode, const double* pold, double* pnew, const double* r, double* q,
                    PcgArgs a, const double** pcur, int* npq) {
  const double* Minv = side == 0 ? c->MinvL : c->MinvR;
  const double* X = side == 0 ? c->Cinv : c->Dinv;
  if (c->k == 2) {
    *pcur = mode == 2 ? pold : pnew;  // (mode 2 leaves p as is; the TMA kernel then skips the copy)
    return run_k2f(c, pold, pnew, r, Minv, X, q, mode, a, npq);
  }
  if (k4f_active(c) && (mode == 2 || r == c->pr)) {  // k = 3, 4: the fused tile kernel (k4_fused.cuh)
    *pcur = mode == 2 ? pold : pnew;
    return run_k4f(c, pold, pnew, X, q, mode, a, npq);
  }
  // generic k: direction update pold -> pnew (+ control), then B^T (element + gather) and B (+ dot)
  const double* p = pold;
  const int* stop = a.ctl ? c->stop + a.it : nullptr;
  if (mode != 2) {
    k_pupd<<<c->red_blocks, VBS, 0, c->stream>>>(pnew, pold, r, Minv, c->pl.n, mode, a.it, a.ctl, c->rzp,
                                                 c->red_blocks, rz_hist(c), pq_hist(c), c->stop);
    LAUNCH_CHECK(c);
    p = pnew;
  }
  *pcur = p;
  wb_status s = run_BT(c, p, nullptr, c->tv, 0, stop, 1, c->n_el);
  if (s) return s;
  *npq = b_blocks(c);
  return run_B(c, c->tv, X, q, 0, stop, p, c->pqp, 1, c->n_el);
}

// the PCG iterations proper (no init / output), on c->stream
wb_status pcg_loop_direct(wb_ctx* c, int side, int iters) {
  const double* Minv = side == 0 ? c->MinvL : c->MinvR;
  double* PB[2] = {c->pp, c->pp1};
  const double* pprev = nullptr;  // p_{it-1}: K reads it, writes p_it into the other buffer
  for (int it = 0; it < iters; ++it) {
    const double* pcur = nullptr;
    const bool prof = c->profile && c->prof_n < wb_ctx::PROF_MAX;
    if (prof) {
      cudaEvent_t* ev = c->prof_ev + 2 * c->prof_n;
      if (!ev[0]) { cudaEventCreate(&ev[0]); cudaEventCreate(&ev[1]); }
      CUDA_TRY(c, cudaEventRecordWithFlags(ev[0], c->stream, c->prof_cap ? cudaEventRecordExternal : 0));
    }
    PcgArgs a;
    a.it = it; a.ctl = 1;
    int npq = 0;
    wb_status s = run_K_pcg(c, side, it == 0 ? 0 : 1, PB[(it + 1) & 1], PB[it & 1], c->pr, c->pq, a, &pcur, &npq);
    if (s) return s;
    if (prof)
      CUDA_TRY(c, cudaEventRecordWithFlags(c->prof_ev[2 * c->prof_n++ + 1], c->stream,
                                           c->prof_cap ? cudaEventRecordExternal : 0));
    // x updates in pairs (odd iterations), bitwise equal to every iteration (kernels.cuh)
    if (it & 1)
      k_pcg_upd<XU_PAIR><<<c->red_blocks, VBS, 0, c->stream>>>(c->px, c->pr, pcur, pprev, c->pq, Minv, c->pl.n, it,
                                                               c->pqp, npq, rz_hist(c), pq_hist(c), c->stop,
                                                               c->rzp, z_out(c));
    else
      k_pcg_upd<XU_DEFER><<<c->red_blocks, VBS, 0, c->stream>>>(c->px, c->pr, pcur, pprev, c->pq, Minv, c->pl.n,
                                                                it, c->pqp, npq, rz_hist(c), pq_hist(c), c->stop,
                                                                c->rzp, z_out(c));
    LAUNCH_CHECK(c);
    pprev = pcur;
  }
  if (iters > 0 && !((iters - 1) & 1)) {  // the last iteration was even: its update is pending
    k_pcg_xfin<<<c->red_blocks, VBS, 0, c->stream>>>(c->px, pprev, c->pl.n, iters - 1, rz_hist(c),
                                                     pq_hist(c), c->stop);
    LAUNCH_CHECK(c);
  }
  return WB_OK;
}

void clear_graphs(wb_ctx* c) {
  for (int i = 0; i < c->n_graphs; ++i)
    if (c->graphs[i].exec) cudaGraphExecDestroy(c->graphs[i].exec);
  c->n_graphs = 0;
  if (!c->prof_execs.empty()) {
    cudaStreamSynchronize(c->stream);
    for (cudaGraphExec_t e : c->prof_execs) cudaGraphExecDestroy(e);
    c->prof_execs.clear();
  }
}

// replay of an iteration loop as one CUDA graph (captured on a private stream), keyed
// by (kind, side, iters, lo, hi); `direct` issues the loop's launches on c->stream
template <class F>
wb_status graph_loop(wb_ctx* c, int kind, int side, int iters, double lo, double hi, F direct) {
  if (c->profile && c->use_graph && iters > 0 && c->cap_stream) {
    // profiled replay: the loop is captured afresh with an event-record NODE around every
    // Poisson-operator launch, so the kernels run with graph launch gaps (as in the
    // unprofiled step) and the event pairs time the kernels, not host launch latency
    cudaStream_t saved = c->stream;
    const long long l0 = c->launches;
    CUDA_TRY(c, cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal));
    c->stream = c->cap_stream;
    c->prof_cap = true;
    wb_status s = direct();
    c->prof_cap = false;
    c->stream = saved;
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(c->cap_stream, &graph);
    if (s) { if (graph) cudaGraphDestroy(graph); return s; }
    if (e != cudaSuccess) return set_err(c, WB_ECUDA, "graph capture: %s", cudaGetErrorString(e));
    cudaGraphExec_t ex = nullptr;
    e = cudaGraphInstantiate(&ex, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return set_err(c, WB_ECUDA, "graph instantiate: %s", cudaGetErrorString(e));
    c->prof_execs.push_back(ex);  // destroyed by clear_graphs (after a sync)
    e = cudaGraphLaunch(ex, c->stream);
    if (e != cudaSuccess) return set_err(c, WB_ECUDA, "graph launch: %s", cudaGetErrorString(e));
    (void)l0;
    return WB_OK;
  }
  if (c->in_capture || !c->use_graph || c->profile || iters == 0 || !c->cap_stream) return direct();
  wb_ctx::GraphEntry* g = nullptr;
  for (int i = 0; i < c->n_graphs; ++i) {
    const wb_ctx::GraphEntry& e = c->graphs[i];
    if (e.kind == kind && e.side == side && e.iters == iters && e.lo == lo && e.hi == hi) g = &c->graphs[i];
  }
  if (!g) {
    if (c->n_graphs == wb_ctx::MAX_GRAPHS) clear_graphs(c);
    g = &c->graphs[c->n_graphs];
    cudaStream_t saved = c->stream;
    const long long l0 = c->launches;
    CUDA_TRY(c, cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal));
    c->stream = c->cap_stream;
    c->in_capture = true;
    wb_status s = direct();
    c->in_capture = false;
    c->stream = saved;
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(c->cap_stream, &graph);
    if (s) { if (graph) cudaGraphDestroy(graph); return s; }
    if (e != cudaSuccess) return set_err(c, WB_ECUDA, "graph capture: %s", cudaGetErrorString(e));
    e = cudaGraphInstantiate(&g->exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return set_err(c, WB_ECUDA, "graph instantiate: %s", cudaGetErrorString(e));
    g->kind = kind; g->side = side; g->iters = iters; g->lo = lo; g->hi = hi;
    g->n_launch = c->launches - l0;
    c->launches = l0;
    ++c->n_graphs;
  }
  CUDA_TRY(c, cudaGraphLaunch(g->exec, c->stream));
  c->launches += g->n_launch;
  return WB_OK;
}

wb_status pcg_loop(wb_ctx* c, int side, int iters) {
  return graph_loop(c, 0, side, iters, 0.0, 0.0, [&] { return pcg_loop_direct(c, side, iters); });
}

// x = P PCG(K_side, P b), exactly `iters` iterations (b, x element-major)
// PCG input / output (R10 projection and the PLay transposes): tiled for k = 2
wb_status launch_pcg_init(wb_ctx* c, const double* b, const double* Minv, double* z) {
  if (c->nm == 4)
    k_pcg_init_t<<<std::min<unsigned>(stream_blocks(c->n_p / 4), (unsigned)c->max_partials), VBS, 0, c->stream>>>(
        b, c->scal + S_SUM, c->px, c->pr, Minv, c->n_el, c->rzp, c->red_blocks, c->partial, c->counter, z, c->pl, c->N);
  else
    k_pcg_init<<<c->red_blocks, VBS, 0, c->stream>>>(b, c->scal + S_SUM, c->px, c->pr, Minv, c->n_el, c->nm, c->rzp, z,
                                                     c->pl, c->N);
  LAUNCH_CHECK(c);
  return WB_OK;
}
wb_status launch_pcg_out(wb_ctx* c, double* x) {
  if (c->nm == 4)
    k_pcg_out_t<<<stream_blocks(c->n_p / 4), VBS, 0, c->stream>>>(c->px, c->scal + S_SUM + 1, x, c->n_el, c->pl, c->N);
  else
    k_pcg_out<<<stream_blocks(c->n_p), VBS, 0, c->stream>>>(c->px, c->scal + S_SUM + 1, x, c->n_el, c->nm, c->pl, c->N);
  LAUNCH_CHECK(c);
  return WB_OK;
}
#define LAUNCH_OR_RET(call) \
  do {                      \
    wb_status st_ = (call); \
    if (st_) return st_;    \
  } while (0)

wb_status run_poisson(wb_ctx* c, int side, const double* b, double* x, int iters) {
  wb_status s = ensure_iters(c, iters);
  if (s) return s;
  c->last_pcg_iters = iters;
  const double* Minv = side == 0 ? c->MinvL : c->MinvR;
  k_mode0_sum<<<c->red_blocks, VBS, 0, c->stream>>>(b, c->n_el, c->nm, c->partial, c->counter, c->scal + S_SUM);
  LAUNCH_CHECK(c);
  LAUNCH_OR_RET(launch_pcg_init(c, b, Minv, z_out(c)));
  if ((s = pcg_loop(c, side, iters))) return s;
  k_mode0_sum<<<c->red_blocks, VBS, 0, c->stream>>>(c->px, c->pl.sm, 1, c->partial, c->counter, c->scal + S_SUM + 1);
  LAUNCH_CHECK(c);
  LAUNCH_OR_RET(launch_pcg_out(c, x));
  return WB_OK;
}


// the Chebyshev iterations proper (Saad Alg. 12.1 steps after the start d), on c->stream
wb_status cheb_loop_direct(wb_ctx* c, int side, int iters, double lmin, double lmax) {
  const double* Minv = side == 0 ? c->MinvL : c->MinvR;
  const double theta = 0.5 * (lmax + lmin), delta = 0.5 * (lmax - lmin), sigma1 = theta / delta;
  double rho = 1.0 / sigma1;
  for (int it = 0; it < iters; ++it) {
    const double* pcur = nullptr;
    int npq = 0;
    wb_status s = run_K_pcg(c, side, 2, c->pp, c->pp1, nullptr, c->pq, PcgArgs{}, &pcur, &npq);
    if (s) return s;
    const double rho1 = 1.0 / (2.0 * sigma1 - rho);
    k_cheb<<<stream_blocks(c->pl.n / 2), VBS, 0, c->stream>>>(c->px, c->pr, c->pp, c->pq, Minv, c->pl.n, rho1 * rho,
                                                 2.0 * rho1 / delta, 0);
    LAUNCH_CHECK(c);
    rho = rho1;
  }
  return WB_OK;
}

// x = P Cheb(K_side, P b) (R16): Saad Alg. 12.1 on Minv K, exactly iters steps.  The
// direction d lives in c->pp (a TMA-mapped PCG buffer), K d goes through the Poisson
// kernel in mode 2 ("p as is"; its p_new copy lands in c->pp1, unused); the scalars
// are data-independent and computed here in the oracle's order.
wb_status run_cheb(wb_ctx* c, int side, const double* b, double* x, int iters, double lmin, double lmax) {
  const double* Minv = side == 0 ? c->MinvL : c->MinvR;
  const int64_t n = c->pl.n;
  k_mode0_sum<<<c->red_blocks, VBS, 0, c->stream>>>(b, c->n_el, c->nm, c->partial, c->counter, c->scal + S_SUM);
  LAUNCH_CHECK(c);
  LAUNCH_OR_RET(launch_pcg_init(c, b, Minv, nullptr));
  const double theta = 0.5 * (lmax + lmin);
  k_cheb<<<stream_blocks(n / 2), VBS, 0, c->stream>>>(c->px, c->pr, c->pp, nullptr, Minv, n, 0.0, 1.0 / theta, 1);
  LAUNCH_CHECK(c);
  wb_status s = graph_loop(c, 1, side, iters, lmin, lmax, [&] { return cheb_loop_direct(c, side, iters, lmin, lmax); });
  if (s) return s;
  k_mode0_sum<<<c->red_blocks, VBS, 0, c->stream>>>(c->px, c->pl.sm, 1, c->partial, c->counter, c->scal + S_SUM + 1);
  LAUNCH_CHECK(c);
  LAUNCH_OR_RET(launch_pcg_out(c, x));
  return WB_OK;
}

// *lam = power-iteration estimate of the largest |eigenvalue| of Minv K_side (R16):
// v = v0 / ||v0||; iters x { w = Minv (K v); lam = ||w||; v = w / lam }.  v in c->pp.
wb_status run_eigmax(wb_ctx* c, int side, const double* v0, int iters, double* lam) {
  const double* Minv = side == 0 ? c->MinvL : c->MinvR;
  const int64_t n = c->pl.n;
  const int nb = c->red_blocks;
  double* dlam = c->scal + S_SCR;
  CUDA_TRY(c, cudaMemsetAsync(c->pp, 0, sizeof(double) * n, c->stream));  // pads stay 0
  k_transpose<<<stream_blocks(c->n_p), VBS, 0, c->stream>>>(v0, c->pp, c->n_el, c->nm, 1, c->pl, c->N);
  LAUNCH_CHECK(c);
  k_pow_sumsq<<<nb, VBS, 0, c->stream>>>(c->pp, nullptr, n, c->rzp);
  LAUNCH_CHECK(c);
  k_pow_scale<<<stream_blocks(n), VBS, 0, c->stream>>>(c->pp, c->pp, n, c->rzp, nb, dlam);
  LAUNCH_CHECK(c);
  CUDA_TRY(c, cudaMemsetAsync(dlam, 0, sizeof(double), c->stream));  // lam = 0 for iters = 0 (as the oracle)
  for (int it = 0; it < iters; ++it) {
    const double* pcur = nullptr;
    int npq = 0;
    wb_status s = run_K_pcg(c, side, 2, c->pp, c->pp1, nullptr, c->pq, PcgArgs{}, &pcur, &npq);
    if (s) return s;
    k_pow_sumsq<<<nb, VBS, 0, c->stream>>>(c->pq, Minv, n, c->rzp);
    LAUNCH_CHECK(c);
    k_pow_scale<<<stream_blocks(n), VBS, 0, c->stream>>>(c->pq, c->pp, n, c->rzp, nb, dlam);
    LAUNCH_CHECK(c);
  }
  CUDA_TRY(c, cudaMemcpyAsync(lam, dlam, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return WB_OK;
}

// ---- diag(A) and the Chebyshev-Jacobi smoother on A (R18)
bool lazy_alloc(double** p, int64_t n) {
  if (*p) return true;
  if (cudaMalloc(p, sizeof(double) * (size_t)n) != cudaSuccess) { cudaGetLastError(); *p = nullptr; return false; }
  return true;
}
// out (n_v) = diag(M A M): element diagonals, then the fixed-order node gather (masked)
wb_status run_diagA(wb_ctx* c, double* out) {
  double* E = c->E;
  if (c->k == 2) {
    if (!lazy_alloc(&c->E3, 3 * c->nq * c->n_el)) return set_err(c, WB_ENOMEM, "diag(A) buffer allocation failed");
    E = c->E3;
  }
  const unsigned nb = (unsigned)nblk(c->n_el, 128);
  switch (c->k) {
    case 2: k_diagA_elem<2, A_TX, A_TY, A_TZ><<<nb, 128, 0, c->stream>>>(c->mut, E, c->G); break;
    case 3: k_diagA_elem<3, 0, 0, 0><<<nb, 128, 0, c->stream>>>(c->mut, E, c->G); break;
    default: k_diagA_elem<4, 0, 0, 0><<<nb, 128, 0, c->stream>>>(c->mut, E, c->G); break;
  }
  LAUNCH_CHECK(c);
  switch (c->k) {
    case 2: k_gather<2><<<nblk(c->n_nodes, 256), 256, 0, c->stream>>>(E, nullptr, out, c->G, 0); break;
    case 3: k_gather<3><<<nblk(c->n_nodes, 256), 256, 0, c->stream>>>(E, nullptr, out, c->G, 0); break;
    default: k_gather<4><<<nblk(c->n_nodes, 256), 256, 0, c->stream>>>(E, nullptr, out, c->G, 0); break;
  }
  LAUNCH_CHECK(c);
  return WB_OK;
}
wb_status ensure_dAinv(wb_ctx* c) {
  if (c->dA_valid) return WB_OK;
  if (!lazy_alloc(&c->dAinv, c->n_v) || !lazy_alloc(&c->tq, c->n_v))
    return set_err(c, WB_ENOMEM, "smoother buffer allocation failed");
  wb_status s = run_diagA(c, c->dAinv);
  if (s) return s;
  k_inv_pos<<<stream_blocks(c->n_v), VBS, 0, c->stream>>>(c->dAinv, c->dAinv, c->n_v);
  LAUNCH_CHECK(c);
  c->dA_valid = true;
  return WB_OK;
}
// x = Cheb(M A M, M b) with the Jacobi inverse mask / diag(A), as or_velocity_cheb
wb_status run_vcheb(wb_ctx* c, const double* b, double* x, int iters, double lmin, double lmax) {
  wb_status s = ensure_dAinv(c);
  if (s) return s;
  const int64_t n = c->n_v;
  double *r = c->tv, *d = c->tw, *q = c->tq;
  CUDA_TRY(c, cudaMemsetAsync(x, 0, sizeof(double) * n, c->stream));
  k_mask_v<<<stream_blocks(c->n_v), VBS, 0, c->stream>>>(b, r, c->G);
  LAUNCH_CHECK(c);
  const double theta = 0.5 * (lmax + lmin), delta = 0.5 * (lmax - lmin), sigma1 = theta / delta;
  double rho = 1.0 / sigma1;
  k_cheb_s<<<stream_blocks(n), VBS, 0, c->stream>>>(x, r, d, nullptr, c->dAinv, n, 0.0, 1.0 / theta, 1);
  LAUNCH_CHECK(c);
  for (int it = 0; it < iters; ++it) {
    if ((s = run_A(c, d, q, 0))) return s;
    const double rho1 = 1.0 / (2.0 * sigma1 - rho);
    k_cheb_s<<<stream_blocks(n), VBS, 0, c->stream>>>(x, r, d, q, c->dAinv, n, rho1 * rho, 2.0 * rho1 / delta, 0);
    LAUNCH_CHECK(c);
    rho = rho1;
  }
  return WB_OK;
}
// power-iteration estimate of the largest |eigenvalue| of (mask / diag A) M A M
wb_status run_veigmax(wb_ctx* c, const double* v0, int iters, double* lam) {
  wb_status s = ensure_dAinv(c);
  if (s) return s;
  const int64_t n = c->n_v;
  const int nb = c->red_blocks;
  double *v = c->tw, *q = c->tq, *dlam = c->scal + S_SCR;
  k_pow_sumsq<<<nb, VBS, 0, c->stream>>>(const_cast<double*>(v0), nullptr, n, c->rzp);  // (no write: Minv = NULL)
  LAUNCH_CHECK(c);
  k_pow_scale<<<stream_blocks(n), VBS, 0, c->stream>>>(v0, v, n, c->rzp, nb, dlam);
  LAUNCH_CHECK(c);
  CUDA_TRY(c, cudaMemsetAsync(dlam, 0, sizeof(double), c->stream));
  for (int it = 0; it < iters; ++it) {
    if ((s = run_A(c, v, q, 0))) return s;
    k_pow_sumsq<<<nb, VBS, 0, c->stream>>>(q, c->dAinv, n, c->rzp);
    LAUNCH_CHECK(c);
    k_pow_scale<<<stream_blocks(n), VBS, 0, c->stream>>>(q, v, n, c->rzp, nb, dlam);
    LAUNCH_CHECK(c);
  }
  CUDA_TRY(c, cudaMemcpyAsync(lam, dlam, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return WB_OK;
}

// q = K_side p, element-major in and out (through the PCG kernels, mode "p as is")
wb_status run_K(wb_ctx* c, int side, const double* p, double* q) {
  k_transpose<<<stream_blocks(c->n_p), VBS, 0, c->stream>>>(p, c->pp, c->n_el, c->nm, 1, c->pl, c->N);
  LAUNCH_CHECK(c);
  const double* pcur = nullptr;
  int npq = 0;
  wb_status s = run_K_pcg(c, side, 2, c->pp, c->pp1, nullptr, c->pq, PcgArgs{}, &pcur, &npq);
  if (s) return s;
  k_transpose<<<stream_blocks(c->n_p), VBS, 0, c->stream>>>(c->pq, q, c->n_el, c->nm, 0, c->pl, c->N);
  LAUNCH_CHECK(c);
  return WB_OK;
}

// wBFBT's inner Poisson solve: PCG, or Chebyshev-Jacobi when wb_set_inner_cheb chose it
wb_status run_inner(wb_ctx* c, int side, const double* b, double* x, int iters) {
  if (c->mg && c->mg->inner_iters > 0) return run_mgcg(c, side, b, x, c->mg->inner_iters);
  if (c->inner) return run_cheb(c, side, b, x, iters, c->cheb_lo[side], c->cheb_hi[side]);
  return run_poisson(c, side, b, x, iters);
}

wb_status run_wbfbt(wb_ctx* c, const double* r, double* z, int iters) {
  // y = P PCG(K_r, P r)
  wb_status s = run_inner(c, 1, r, c->s2, iters);
  if (s) return s;
  // v = Dinv o (B^T y)
  s = run_BT(c, c->s2, c->Dinv, c->tw, 0, nullptr, c->nm, 1);
  if (s) return s;
  // w = A v
  s = run_A(c, c->tw, c->tv, 0);
  if (s) return s;
  // s = P B (Cinv o w)
  s = run_B(c, c->tv, c->Cinv, c->s2, 0, nullptr, nullptr, nullptr, c->nm, 1);
  if (s) return s;
  // z = P PCG(K_l, s)   (run_poisson projects its input first)
  return run_inner(c, 0, c->s2, z, iters);
}

wb_status dev_dot(wb_ctx* c, const double* a, const double* b, int64_t n, double* out_dev) {
  k_dot_dev<<<c->red_blocks, VBS, 0, c->stream>>>(a, b, n, c->partial, c->counter, out_dev);
  LAUNCH_CHECK(c);
  return WB_OK;
}
// ---- diag(A)-BFBT: C = D = diag(A), a per-DOF weight
// X = mask / diag(A); its Poisson operator K_d = B X B^T runs through the generic B^T / B
// kernels (element-major vectors) and its inverse is the O9 Jacobi-PCG with device scalars.
wb_status ensure_dab(wb_ctx* c) {
  if (c->dab_valid) return WB_OK;
  wb_status s = ensure_dAinv(c);
  if (s) return s;
  for (double** b : {&c->dKd, &c->mKd, &c->gp_r, &c->gp_z, &c->gp_p, &c->gp_q, &c->gp_x, &c->gp_y})
    if (!lazy_alloc(b, c->n_p)) return set_err(c, WB_ENOMEM, "diag(A)-BFBT allocation failed");
  if (!lazy_alloc(&c->dv, c->n_v) || !lazy_alloc(&c->gp_s, 4)) return set_err(c, WB_ENOMEM, "allocation failed");
  const unsigned nb = nblk(c->n_el, 128);
  switch (c->k) {
    case 2: k_jacobi_dof<2><<<nb, 128, 0, c->stream>>>(c->dAinv, c->dKd, c->G, c->sB); break;
    case 3: k_jacobi_dof<3><<<nb, 128, 0, c->stream>>>(c->dAinv, c->dKd, c->G, c->sB); break;
    default: k_jacobi_dof<4><<<nb, 128, 0, c->stream>>>(c->dAinv, c->dKd, c->G, c->sB); break;
  }
  LAUNCH_CHECK(c);
  double* dmax = c->scal + S_SCR + 2;
  k_absmax<VBS><<<c->red_blocks, VBS, 0, c->stream>>>(c->dKd, c->n_p, c->partial, c->counter, dmax);
  LAUNCH_CHECK(c);
  k_pinv_diag<<<stream_blocks(c->n_p), VBS, 0, c->stream>>>(c->dKd, c->mKd, c->n_p, dmax);
  LAUNCH_CHECK(c);
  c->dab_valid = true;
  return WB_OK;
}
// q = B (X o B^T p), element-major, X = mask / diag(A) per DOF
wb_status run_Kd(wb_ctx* c, const double* p, double* q) {
  wb_status s = run_BT(c, p, nullptr, c->dv, 0, nullptr, c->nm, 1);
  if (s) return s;
  k_mul<<<stream_blocks(c->n_v), VBS, 0, c->stream>>>(c->dv, c->dv, c->dAinv, c->n_v);
  LAUNCH_CHECK(c);
  return run_B(c, c->dv, nullptr, q, 0, nullptr, nullptr, nullptr, c->nm, 1);
}
static wb_status em_project(wb_ctx* c, double* v) {  // R10 on an element-major vector
  k_mode0_sum<<<c->red_blocks, VBS, 0, c->stream>>>(v, c->n_el, c->nm, c->partial, c->counter, c->scal + S_SCR + 3);
  LAUNCH_CHECK(c);
  k_sub_mode0_mean<<<stream_blocks(c->n_el), VBS, 0, c->stream>>>(v, c->n_el, c->nm, c->scal + S_SCR + 3);
  LAUNCH_CHECK(c);
  return WB_OK;
}
// x = P PCG(K_d, P b), O9 with Minv = pinv(diag K_d), exactly iters iterations
wb_status run_dpcg(wb_ctx* c, const double* b, double* x, int iters) {
  const int64_t n = c->n_p;
  const unsigned nb = stream_blocks(n);
  CUDA_TRY(c, cudaMemcpyAsync(c->gp_r, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
  wb_status s = em_project(c, c->gp_r);
  if (s) return s;
  CUDA_TRY(c, cudaMemsetAsync(c->gp_x, 0, sizeof(double) * n, c->stream));
  CUDA_TRY(c, cudaMemsetAsync(c->gp_s, 0, sizeof(double) * 4, c->stream));
  k_mul<<<nb, VBS, 0, c->stream>>>(c->gp_z, c->gp_r, c->mKd, n);
  LAUNCH_CHECK(c);
  CUDA_TRY(c, cudaMemcpyAsync(c->gp_p, c->gp_z, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
  if ((s = dev_dot(c, c->gp_r, c->gp_z, n, c->gp_s))) return s;
  for (int it = 0; it < iters; ++it) {
    if ((s = run_Kd(c, c->gp_p, c->gp_q))) return s;
    if ((s = dev_dot(c, c->gp_p, c->gp_q, n, c->gp_s + 1))) return s;
    k_mgcg_xr<<<nb, VBS, 0, c->stream>>>(c->gp_x, c->gp_r, c->gp_p, c->gp_q, n, c->gp_s);
    LAUNCH_CHECK(c);
    k_mul<<<nb, VBS, 0, c->stream>>>(c->gp_z, c->gp_r, c->mKd, n);
    LAUNCH_CHECK(c);
    if ((s = dev_dot(c, c->gp_r, c->gp_z, n, c->gp_s + 2))) return s;
    k_mgcg_p<<<nb, VBS, 0, c->stream>>>(c->gp_p, c->gp_z, n, c->gp_s, c->counter + 3);
    LAUNCH_CHECK(c);
  }
  CUDA_TRY(c, cudaMemcpyAsync(x, c->gp_x, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
  return em_project(c, x);
}
// z = (B X B^T)^-1 (B X A X B^T) (B X B^T)^-1 r, X = mask / diag(A), O10 order
wb_status run_dabfbt(wb_ctx* c, const double* r, double* z, int iters) {
  wb_status s = ensure_dab(c);
  if (s) return s;
  if ((s = run_dpcg(c, r, c->gp_y, iters))) return s;
  if ((s = run_BT(c, c->gp_y, nullptr, c->tw, 0, nullptr, c->nm, 1))) return s;
  k_mul<<<stream_blocks(c->n_v), VBS, 0, c->stream>>>(c->tw, c->tw, c->dAinv, c->n_v);
  LAUNCH_CHECK(c);
  if ((s = run_A(c, c->tw, c->tv, 0))) return s;
  k_mul<<<stream_blocks(c->n_v), VBS, 0, c->stream>>>(c->tv, c->tv, c->dAinv, c->n_v);
  LAUNCH_CHECK(c);
  if ((s = run_B(c, c->tv, nullptr, c->gp_y, 0, nullptr, nullptr, nullptr, c->nm, 1))) return s;
  return run_dpcg(c, c->gp_y, z, iters);  // (run_dpcg projects its input)
}
// z = scale M_p(1/mu)^-1 r, element blocks (R21)
wb_status run_mpinv(wb_ctx* c, const double* r, double* z, double scale) {
  if (!c->mp_valid) return set_err(c, WB_ESTATE, "M_p(1/mu) blocks not built: wb_set_schur(ctx, 2) before wb_set_viscosity");
  const unsigned nb = nblk(c->n_el, 128);
  switch (c->nm) {
    case 4: k_mp_apply<4><<<nb, 128, 0, c->stream>>>(c->mpinv, r, z, c->n_el, scale); break;
    case 10: k_mp_apply<10><<<nb, 128, 0, c->stream>>>(c->mpinv, r, z, c->n_el, scale); break;
    default: k_mp_apply<20><<<nb, 128, 0, c->stream>>>(c->mpinv, r, z, c->n_el, scale); break;
  }
  LAUNCH_CHECK(c);
  return WB_OK;
}

// ---- Stokes solve (R19): flexible GMRES on [A B^T; B 0] with P^-1 (a; b) =
// (At^-1 (a - B^T y); y), y = -wBFBT(b), At^-1 = the smoother on A.  Vectors are [u | p],
// p element-major.  The Gram-Schmidt scalars stay on the device (k_dot_dev / k_axpy_dev);
// the Givens rotations, the Hessenberg (as R) and the back substitution stay on the device;
// the host reads the 16-byte residual estimate once per iteration for the stop test.
struct StokesPar { int pcg, sm; double lo, hi; };
wb_status stokes_K(wb_ctx* c, const double* x, double* y) {
  wb_status s;
  if ((s = run_A(c, x, y, 0))) return s;
  if ((s = run_BT(c, x + c->n_v, nullptr, c->gsa, 0, nullptr, c->nm, 1))) return s;
  k_axpy<<<stream_blocks(c->n_v), VBS, 0, c->stream>>>(y, c->gsa, c->n_v, 1.0);
  LAUNCH_CHECK(c);
  return run_B(c, x, nullptr, y + c->n_v, 0, nullptr, nullptr, nullptr, c->nm, 1);
}
wb_status stokes_P(wb_ctx* c, const double* v, double* z, const StokesPar& P) {
  wb_status s;
  double* y = z + c->n_v;
  // y = -S~^-1 b: wBFBT (default), diag(A)-BFBT or M_p(1/mu)^-1
  if (c->schur == 2) {
    if ((s = run_mpinv(c, v + c->n_v, y, -1.0))) return s;
  } else {
    if ((s = c->schur == 1 ? run_dabfbt(c, v + c->n_v, y, P.pcg) : run_wbfbt(c, v + c->n_v, y, P.pcg))) return s;
    k_axpby<<<stream_blocks(c->n_p), VBS, 0, c->stream>>>(y, y, c->n_p, 0.0, -1.0);
    LAUNCH_CHECK(c);
  }
  if ((s = run_BT(c, y, nullptr, c->gsa, 0, nullptr, c->nm, 1))) return s;
  k_axpby<<<stream_blocks(c->n_v), VBS, 0, c->stream>>>(c->gsa, v, c->n_v, 1.0, -1.0);  // a - B^T y
  LAUNCH_CHECK(c);
  if (c->mg && c->mg->vel && c->mg->vcycles > 0) return run_vmg(c, c->gsa, z);  // At^-1: velocity V-cycles (R22)
  return run_vcheb(c, c->gsa, z, P.sm, P.lo, P.hi);
}
wb_status host_scalar(wb_ctx* c, const double* dev, double* h) {
  CUDA_TRY(c, cudaMemcpyAsync(h, dev, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return WB_OK;
}
wb_status run_stokes(wb_ctx* c, const double* f, const double* g, double* u, double* p, int m, int max_iters,
                     double rtol, const StokesPar& P, int* iters_out, double* relres_out) {
  const int64_t n = c->n_v + c->n_p;
  if (m > c->g_m) {  // the basis and the Hessenberg column grow with the restart length
    cudaStreamSynchronize(c->stream);
    for (double** b : {&c->gV, &c->gZ, &c->gh, &c->gls}) { if (*b) cudaFree(*b); *b = nullptr; }
    if (!lazy_alloc(&c->gV, n * (m + 1)) || !lazy_alloc(&c->gZ, n * m) || !lazy_alloc(&c->gh, (int64_t)m + 2) ||
        !lazy_alloc(&c->gls, (int64_t)m * m + 4 * (int64_t)m + 4)) {
      c->g_m = 0;
      return set_err(c, WB_ENOMEM, "FGMRES basis allocation failed (restart %d)", m);
    }
    c->g_m = m;
  }
  if (!lazy_alloc(&c->gw, n) || !lazy_alloc(&c->gb, n) || !lazy_alloc(&c->gx, n) || !lazy_alloc(&c->gsa, c->n_v) ||
      !lazy_alloc(&c->gh, (int64_t)m + 2))
    return set_err(c, WB_ENOMEM, "FGMRES work allocation failed");
  if (c->g_m < m) return set_err(c, WB_ENOMEM, "FGMRES basis too small");
  if (!c->gres_h && cudaMallocHost(&c->gres_h, 2 * sizeof(double)) != cudaSuccess) {
    cudaGetLastError();
    c->gres_h = nullptr;
    return set_err(c, WB_ENOMEM, "FGMRES pinned scalar allocation failed");
  }
  // device least-squares state (the Hessenberg never leaves the device; the host reads the
  // 16-byte residual estimate once per iteration for the stop test)
  const int gm = c->g_m;
  double *dR = c->gls, *dcs = dR + (int64_t)gm * gm, *dsn = dcs + gm, *dg = dsn + gm, *dy = dg + gm + 1,
         *dres = dy + gm;
  wb_status s;
  k_mask_v<<<stream_blocks(c->n_v), VBS, 0, c->stream>>>(f, c->gb, c->G);  // b = (M f; g)
  LAUNCH_CHECK(c);
  CUDA_TRY(c, cudaMemcpyAsync(c->gb + c->n_v, g, sizeof(double) * c->n_p, cudaMemcpyDeviceToDevice, c->stream));
  CUDA_TRY(c, cudaMemsetAsync(c->gx, 0, sizeof(double) * n, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(c->gw, c->gb, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
  double bn2 = 0.0;
  if ((s = dev_dot(c, c->gb, c->gb, n, c->gh)) || (s = host_scalar(c, c->gh, &bn2))) return s;
  const double bnorm = std::sqrt(bn2);
  double beta = bnorm;
  int total = 0;
  while (beta > rtol * bnorm && total < max_iters) {
    // V_0 = w / beta, beta^2 = <w, w> still in gh[0] from the dot that gave beta
    k_unit_dev<<<stream_blocks(c->n_v), VBS, 0, c->stream>>>(c->gV, c->gw, n, c->gh);
    LAUNCH_CHECK(c);
    CUDA_TRY(c, cudaMemsetAsync(dg, 0, sizeof(double) * (gm + 1), c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(dg, &beta, sizeof(double), cudaMemcpyHostToDevice, c->stream));
    int jend = -1;
    for (int j = 0; j < m && total < max_iters; ++j) {
      double* Vj = c->gV + (int64_t)j * n;
      double* Zj = c->gZ + (int64_t)j * n;
      if ((s = stokes_P(c, Vj, Zj, P)) || (s = stokes_K(c, Zj, c->gw))) return s;
      for (int i = 0; i <= j; ++i) {  // modified Gram-Schmidt, scalars on the device
        if ((s = dev_dot(c, c->gw, c->gV + (int64_t)i * n, n, c->gh + i))) return s;
        k_axpy_dev<<<stream_blocks(c->n_v), VBS, 0, c->stream>>>(c->gw, c->gV + (int64_t)i * n, n, c->gh + i);
        LAUNCH_CHECK(c);
      }
      if ((s = dev_dot(c, c->gw, c->gw, n, c->gh + j + 1))) return s;
      k_givens<<<1, 1, 0, c->stream>>>(j, gm, c->gh, dR, dcs, dsn, dg, dres);
      LAUNCH_CHECK(c);
      CUDA_TRY(c, cudaMemcpyAsync(c->gres_h, dres, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
      CUDA_TRY(c, cudaStreamSynchronize(c->stream));
      const double gres = c->gres_h[0], hn = c->gres_h[1];
      ++total;
      jend = j;
      if (hn > 0.0) {
        k_unit_dev<<<stream_blocks(c->n_v), VBS, 0, c->stream>>>(c->gV + (int64_t)(j + 1) * n, c->gw, n, c->gh + j + 1);
        LAUNCH_CHECK(c);
      }
      if (gres <= rtol * bnorm || hn == 0.0) break;
    }
    if (jend >= 0) {
      k_fgmres_y<<<1, 1, 0, c->stream>>>(jend, gm, dR, dg, dy);
      LAUNCH_CHECK(c);
    }
    for (int i = 0; i <= jend; ++i) {
      k_axpy_devp<<<stream_blocks(c->n_v), VBS, 0, c->stream>>>(c->gx, c->gZ + (int64_t)i * n, n, dy + i);
      LAUNCH_CHECK(c);
    }
    if ((s = stokes_K(c, c->gx, c->gw))) return s;  // true residual
    k_axpby<<<stream_blocks(c->n_v), VBS, 0, c->stream>>>(c->gw, c->gb, n, 1.0, -1.0);
    LAUNCH_CHECK(c);
    if ((s = dev_dot(c, c->gw, c->gw, n, c->gh)) || (s = host_scalar(c, c->gh, &bn2))) return s;
    beta = std::sqrt(bn2);
    if (jend < 0) break;
  }
  CUDA_TRY(c, cudaMemcpyAsync(u, c->gx, sizeof(double) * c->n_v, cudaMemcpyDeviceToDevice, c->stream));
  // p = P x_p (R10)
  k_mode0_sum<<<c->red_blocks, VBS, 0, c->stream>>>(c->gx + c->n_v, c->n_el, c->nm, c->partial, c->counter,
                                                    c->scal + S_SUM);
  LAUNCH_CHECK(c);
  k_project<<<c->red_blocks, VBS, 0, c->stream>>>(c->gx + c->n_v, p, c->n_p, c->nm, c->n_el, c->scal + S_SUM);
  LAUNCH_CHECK(c);
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (iters_out) *iters_out = total;
  if (relres_out) *relres_out = bnorm > 0.0 ? beta / bnorm : 0.0;
  return WB_OK;
}

// ================================================================ z-slab domain decomposition
// (R24).  The global operators from the cube
// kernels: unmasked local applies, one sum of the shared planes' partials, the global mask.
enum { DS_RZ = 0, DS_PQ = 1, DS_RZ1 = 2, DS_STOP = 3, DS_MEAN = 4, DS_MAX = 5 };

wb_status dd_allreduce(wb_ctx* c, int offset, int n, int op) {
  DD* d = c->dd;
  if (d->nranks == 1) return WB_OK;
  if (d->comm.allreduce(d->comm.user, offset, n, op) != 0)
    return set_err(c, WB_ECUDA, "slab communicator: allreduce failed");
  return WB_OK;
}
// sum the shared z planes of nf nodal fields (n_nodes each) with the neighbours' partials
wb_status dd_plane_sum(wb_ctx* c, double* const* f, int nf) {
  DD* d = c->dd;
  if (d->nranks == 1) return WB_OK;
  if (nf > 3) return set_err(c, WB_EINVAL, "at most 3 fields per plane sum");
  const int64_t np = (int64_t)c->G.nn1 * c->G.nn1, n = np * nf;
  if (n > d->comm.cap) return set_err(c, WB_EINVAL, "slab exchange buffers too small");
  const int zo = c->G.zopen;
  DDFields F{};
  F.nf = nf;
  for (int i = 0; i < nf; ++i) F.f[i] = f[i];
  k_dd_pack<<<stream_blocks(n), VBS, 0, c->stream>>>(F, d->comm.send_lo, d->comm.send_hi, np, c->n_nodes, zo);
  LAUNCH_CHECK(c);
  if (d->comm.exchange(d->comm.user, n) != 0) return set_err(c, WB_ECUDA, "slab communicator: exchange failed");
  k_dd_unpack_add<<<stream_blocks(n), VBS, 0, c->stream>>>(F, d->comm.recv_lo, d->comm.recv_hi, np, c->n_nodes, zo);
  LAUNCH_CHECK(c);
  return WB_OK;
}
wb_status dd_plane_sum3(wb_ctx* c, double* v) {
  double* f[3] = {v, v + c->n_nodes, v + 2 * c->n_nodes};
  return dd_plane_sum(c, f, 3);
}
// row a3 on a slab: plane-sum C_w, D_w, then the inverses under the global mask
wb_status dd_finish_lump(wb_ctx* c) {
  double* f[2] = {c->Cw, c->Dw};
  wb_status s = dd_plane_sum(c, f, 2);
  if (s) return s;
  CUDA_TRY(c, cudaMemsetAsync(c->icount + 1, 0, sizeof(unsigned long long) * 2, c->stream));
  k_dd_inv<<<stream_blocks(c->n_nodes), VBS, 0, c->stream>>>(c->Cw, c->Dw, c->dd->gm, c->Cinv, c->Dinv,
                                                              c->icount + 1, c->n_nodes);
  LAUNCH_CHECK(c);
  return WB_OK;
}
// max|diag K_side| over all ranks (the R11 threshold is global), then this rank's element-major Minv
wb_status dd_after_dmax(wb_ctx* c, int side, const double* diag, double* dmax) {
  DD* d = c->dd;
  double* sc = d->scal();
  CUDA_TRY(c, cudaMemcpyAsync(sc + DS_MAX, dmax, sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  wb_status s = dd_allreduce(c, DS_MAX, 1, 1);
  if (s) return s;
  CUDA_TRY(c, cudaMemcpyAsync(dmax, sc + DS_MAX, sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  k_pinv_diag<<<stream_blocks(c->n_p), VBS, 0, c->stream>>>(diag, d->mK[side], c->n_p, dmax);
  LAUNCH_CHECK(c);
  return WB_OK;
}
// y = M A M u (global): mask the input, unmasked cube apply, plane sum, mask
wb_status dd_A(wb_ctx* c, const double* u, double* y, bool u_masked) {
  DD* d = c->dd;
  const double* in = u;
  if (!u_masked) {
    k_dd_scale3<<<stream_blocks(c->n_nodes), VBS, 0, c->stream>>>(d->vs, u, d->gm, c->n_nodes);
    LAUNCH_CHECK(c);
    in = d->vs;
  }
  wb_status s = run_A(c, in, y, 1);
  if (s) return s;
  if ((s = dd_plane_sum3(c, y))) return s;
  k_dd_scale3<<<stream_blocks(c->n_nodes), VBS, 0, c->stream>>>(y, y, d->gm, c->n_nodes);
  LAUNCH_CHECK(c);
  return WB_OK;
}
// p = B (xs o u), xs a nodal scaling that carries the global mask (default: the mask itself)
wb_status dd_B(wb_ctx* c, const double* u, const double* xs, double* p) {
  return run_B(c, u, xs ? xs : c->dd->gm, p, 0, nullptr, nullptr, nullptr, c->nm, 1);
}
// y = xs o (B^T p) (global), xs as above
wb_status dd_BT(wb_ctx* c, const double* p, const double* xs, double* y) {
  wb_status s = run_BT(c, p, nullptr, y, 1, nullptr, c->nm, 1);
  if (s) return s;
  if ((s = dd_plane_sum3(c, y))) return s;
  k_dd_scale3<<<stream_blocks(c->n_nodes), VBS, 0, c->stream>>>(y, y, xs ? xs : c->dd->gm, c->n_nodes);
  LAUNCH_CHECK(c);
  return WB_OK;
}
// q = B (X o B^T p) (global, O6), X = C_w^-1 or D_w^-1 with the global mask
wb_status dd_K(wb_ctx* c, int side, const double* p, double* q) {
  DD* d = c->dd;
  wb_status s = run_BT(c, p, nullptr, d->vs, 1, nullptr, c->nm, 1);
  if (s) return s;
  if ((s = dd_plane_sum3(c, d->vs))) return s;
  return run_B(c, d->vs, side == 0 ? c->Cinv : c->Dinv, q, 0, nullptr, nullptr, nullptr, c->nm, 1);
}
// global <a, b> into scalar slot `slot`: this rank's fixed-order sum, then one all-reduce
wb_status dd_dot(wb_ctx* c, const double* a, const double* b, int slot) {
  wb_status s = dev_dot(c, a, b, c->n_p, c->dd->scal() + slot);
  if (s) return s;
  return dd_allreduce(c, slot, 1, 0);
}
// R10 on the local part of an element-major vector (global mean)
wb_status dd_project(wb_ctx* c, double* v) {
  DD* d = c->dd;
  k_mode0_sum<<<c->red_blocks, VBS, 0, c->stream>>>(v, c->n_el, c->nm, c->partial, c->counter, d->scal() + DS_MEAN);
  LAUNCH_CHECK(c);
  wb_status s = dd_allreduce(c, DS_MEAN, 1, 0);
  if (s) return s;
  k_dd_sub_mean<<<stream_blocks(c->n_el), VBS, 0, c->stream>>>(v, c->n_el, c->nm, d->scal() + DS_MEAN,
                                                               (double)c->n_el * d->nranks);
  LAUNCH_CHECK(c);
  return WB_OK;
}
// x = P PCG(K_side, P b), the O9 recurrence with the scalars on the device, exactly iters iterations
wb_status dd_pcg(wb_ctx* c, int side, const double* b, double* x, int iters) {
  DD* d = c->dd;
  const int64_t n = c->n_p;
  const unsigned nb = stream_blocks(n);
  double* sc = d->scal();
  CUDA_TRY(c, cudaMemcpyAsync(d->r, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
  wb_status s = dd_project(c, d->r);
  if (s) return s;
  CUDA_TRY(c, cudaMemsetAsync(d->x, 0, sizeof(double) * n, c->stream));
  CUDA_TRY(c, cudaMemsetAsync(sc, 0, sizeof(double) * 4, c->stream));
  k_mul<<<nb, VBS, 0, c->stream>>>(d->z, d->r, d->mK[side], n);
  LAUNCH_CHECK(c);
  CUDA_TRY(c, cudaMemcpyAsync(d->p, d->z, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
  if ((s = dd_dot(c, d->r, d->z, DS_RZ))) return s;
  for (int it = 0; it < iters; ++it) {
    if ((s = dd_K(c, side, d->p, d->q))) return s;
    if ((s = dd_dot(c, d->p, d->q, DS_PQ))) return s;
    k_mgcg_xr<<<nb, VBS, 0, c->stream>>>(d->x, d->r, d->p, d->q, n, sc);
    LAUNCH_CHECK(c);
    k_mul<<<nb, VBS, 0, c->stream>>>(d->z, d->r, d->mK[side], n);
    LAUNCH_CHECK(c);
    if ((s = dd_dot(c, d->r, d->z, DS_RZ1))) return s;
    k_mgcg_p<<<nb, VBS, 0, c->stream>>>(d->p, d->z, n, sc, c->counter + 3);
    LAUNCH_CHECK(c);
  }
  CUDA_TRY(c, cudaMemcpyAsync(x, d->x, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
  return dd_project(c, x);
}
// O10 on the slab: z = P PCG(K_l) P B C_w^-1 A D_w^-1 B^T P PCG(K_r) P r
wb_status dd_wbfbt(wb_ctx* c, const double* r, double* z, int iters) {
  DD* d = c->dd;
  wb_status s = dd_pcg(c, 1, r, d->y, iters);
  if (s) return s;
  if ((s = dd_BT(c, d->y, c->Dinv, c->tw))) return s;
  if ((s = dd_A(c, c->tw, c->tv, true))) return s;
  if ((s = dd_B(c, c->tv, c->Cinv, d->y))) return s;
  return dd_pcg(c, 0, d->y, z, iters);
}
void dd_free(wb_ctx* c) {
  DD* d = c->dd;
  if (!d) return;
  for (double** b : {&d->own_scal, &d->gm, &d->vs, &d->r, &d->z, &d->p, &d->q, &d->x, &d->y, &d->mK[0], &d->mK[1]})
    if (*b) cudaFree(*b);
  delete d;
  c->dd = nullptr;
}

wb_status check_ctx(wb_ctx* c, bool need_visc, bool dd_ok = false) {
  if (!c) return WB_EINVAL;
  if (c->dd && !dd_ok) return set_err(c, WB_ESTATE, "this call is not available on a slab context (wbfbt.h, z-slab)");
  if (c->dd && c->dd->nranks > 1 && !c->dd->have_comm)
    return set_err(c, WB_ESTATE, "slab context without a communicator: wb_slab_set_comm first");
  if (need_visc && !c->have_visc) return set_err(c, WB_ESTATE, "wb_set_viscosity has not been called");
  return WB_OK;
}

void free_all(wb_ctx* c) {
  mg_free(c);
  dd_free(c);
  double** bufs[] = {&c->dKd, &c->mKd, &c->dv, &c->gp_r, &c->gp_z, &c->gp_p, &c->gp_q, &c->gp_x, &c->gp_y,
                     &c->gp_s, &c->mpinv, &c->mut, &c->Cw, &c->Dw, &c->Cinv, &c->Dinv, &c->dKl, &c->dKr, &c->MinvL, &c->MinvR,
                     &c->E, &c->tv, &c->tw, &c->px, &c->pr, &c->pp, &c->pp1, &c->pq, &c->pz, &c->s0, &c->s1, &c->s2,
                     &c->partial, &c->pqp, &c->rzp, &c->scal, &c->stage, &c->Fu, &c->mueff,
                     &c->E3, &c->dAinv, &c->tq, &c->gV, &c->gZ, &c->gw, &c->gb, &c->gx, &c->gsa, &c->gh, &c->gls};
  clear_graphs(c);
  if (c->gres_h) { cudaFreeHost(c->gres_h); c->gres_h = nullptr; }
  if (c->cap_stream) { cudaStreamDestroy(c->cap_stream); c->cap_stream = nullptr; }
  if (c->copy_stream) { cudaStreamDestroy(c->copy_stream); c->copy_stream = nullptr; }
  for (cudaEvent_t* e : {&c->ev_in, &c->ev_ab, &c->ev_bt, &c->ev_done, &c->ev_p})
    if (*e) { cudaEventDestroy(*e); *e = nullptr; }
  for (int i = 0; i < 2 * wb_ctx::PROF_MAX; ++i)
    if (c->prof_ev[i]) { cudaEventDestroy(c->prof_ev[i]); c->prof_ev[i] = nullptr; }
  if (c->slab) {  // carved arrays: one free, before the per-buffer frees below
    c->MinvL = c->MinvR = c->XpL = c->XpR = c->px = c->pr = c->pp = c->pp1 = c->pq = c->pz = nullptr;
    cudaFree(c->slab);
    c->slab = nullptr;
  }
  for (double** b : bufs)
    if (*b) { cudaFree(*b); *b = nullptr; }
  if (c->counter) cudaFree(c->counter);
  if (c->stop) cudaFree(c->stop);
  if (c->icount) cudaFree(c->icount);
  if (c->XzL) cudaFree(c->XzL);
  if (c->XzR) cudaFree(c->XzR);
  c->XzL = c->XzR = nullptr;
  if (c->XpL) cudaFree(c->XpL);
  if (c->XpR) cudaFree(c->XpR);
  c->XpL = c->XpR = nullptr;
  if (c->X4L) cudaFree(c->X4L);
  if (c->X4R) cudaFree(c->X4R);
  c->X4L = c->X4R = nullptr;
  c->counter = nullptr; c->stop = nullptr; c->icount = nullptr;
  cudaGetLastError();  // teardown must not leave an error for the next context's launch checks
}

}  // namespace

// ================================================================ C ABI
extern "C" {

const char* wb_version(void) { return WB_VERSION; }

wb_status wb_create(wb_ctx** out, int N, int k, unsigned flags, void* stream) {
  if (!out) return WB_EINVAL;
  *out = nullptr;
  if (N < 1 || N > 4096 || k < 2 || k > 4) return WB_EINVAL;
  if (flags & ~(WB_STRICT_LUMP | WB_DEBUG_NOMASK | WB_DEBUG_SCALARS)) return WB_EINVAL;
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
    // k = 2 dense gradient table (without sB): prod_d (d == c ? BD : BI)[m_d][a_d]
    double bt2[3][27][4];
    const int md[4][3] = {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}};  // mode order of wbfbt.h
    for (int cc = 0; cc < 3; ++cc)
      for (int a = 0; a < 27; ++a)
        for (int m = 0; m < 4; ++m) {
          const int ad[3] = {a % 3, (a / 3) % 3, a / 9};
          long double v = 1.0L;
          for (int d = 0; d < 3; ++d) v *= (d == cc ? t[0].BD[md[m][d]][ad[d]] : t[0].BI[md[m][d]][ad[d]]);
          bt2[cc][a][m] = (double)v;
        }
    // factorised tables (k = 2): c_W2[c][ay][az][k], c_X2[c][ax][m1]
    double w2[3][3][3][3], x2[3][3][2];
    for (int cc = 0; cc < 3; ++cc) {
      auto M = [&](int d, int m, int a) { return (long double)(d == cc ? t[0].BD[m][a] : t[0].BI[m][a]); };
      for (int ay = 0; ay < 3; ++ay)
        for (int az = 0; az < 3; ++az) {
          w2[cc][ay][az][0] = (double)(M(1, 0, ay) * M(2, 0, az));
          w2[cc][ay][az][1] = (double)(M(1, 1, ay) * M(2, 0, az));
          w2[cc][ay][az][2] = (double)(M(1, 0, ay) * M(2, 1, az));
        }
      for (int ax = 0; ax < 3; ++ax)
        for (int m1 = 0; m1 < 2; ++m1) x2[cc][ax][m1] = (double)M(0, m1, ax);
    }
    if (cudaMemcpyToSymbol(c_W2, w2, sizeof(w2)) != cudaSuccess ||
        cudaMemcpyToSymbol(c_X2, x2, sizeof(x2)) != cudaSuccess) {
      delete c;
      return WB_ECUDA;
    }
    double j2[27][4];  // Jacobi weights: sum_c bt2[c][a][m]^2
    for (int a = 0; a < 27; ++a)
      for (int m = 0; m < 4; ++m) {
        long double v = 0.0L;
        for (int cc = 0; cc < 3; ++cc) v += (long double)bt2[cc][a][m] * (long double)bt2[cc][a][m];
        j2[a][m] = (double)v;
      }
    if (cudaMemcpyToSymbol(c_Bt2, bt2, sizeof(bt2)) != cudaSuccess ||
        cudaMemcpyToSymbol(c_J2, j2, sizeof(j2)) != cudaSuccess) {
      delete c;
      return WB_ECUDA;
    }
    g_tabs_ready = true;
  }
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  c->red_blocks = RED_MULT * nsm;
  c->nsm = nsm;
  c->max_partials = (int)std::max<int64_t>(c->red_blocks, (c->n_el + 127) / 128 + 1);
  bool ok = true;
  auto alloc = [&](double** p, int64_t n) {
    if (ok && cudaMalloc(p, sizeof(double) * (size_t)(n > 0 ? n : 1)) != cudaSuccess) ok = false;
  };
  alloc(&c->Cw, c->n_nodes); alloc(&c->Dw, c->n_nodes); alloc(&c->Cinv, c->n_nodes); alloc(&c->Dinv, c->n_nodes);
  // PCG vector storage: y fastest with zero pads for the TMA Poisson kernel (k = 2, even N,
  // large meshes, tensor-map encoder available), else mode-major m n_el + e
  c->ylay = k == 2 && !(N & 1) && c->n_el >= tma_min_el() && get_encode();
  if (c->ylay) {
    const int64_t sz = N + 2, sx = (int64_t)N * sz, sm = (int64_t)N * sx;
    c->pl = PLay{sm, sx, 1, sz, c->nm * sm, 1};
  } else {
    c->pl = PLay{c->n_el, 1, N, (int64_t)N * N, c->n_p, 0};
  }
  if (k == 2 && !(N & 1)) {
    auto up = [](int64_t n) { return (n + 31) & ~(int64_t)31; };  // 256-byte sub-arrays
    const int64_t np = up(c->pl.n), nx = up(xt_len(N));
    if (ok && cudaMalloc(&c->slab, sizeof(double) * (size_t)(8 * np + 2 * nx)) != cudaSuccess) ok = false;
    if (ok) {
      double* q = c->slab;
      c->MinvL = q; q += np; c->XpL = q; q += nx;
      c->px = q; q += np; c->pr = q; q += np; c->pp = q; q += np; c->pp1 = q; q += np; c->pq = q; q += np;
      c->pz = q; q += np;
      c->MinvR = q; q += np; c->XpR = q;
      // zero: the pads of the y-fastest storage stay 0 for good
      if (cudaMemsetAsync(c->slab, 0, sizeof(double) * (size_t)(8 * np + 2 * nx), c->stream) != cudaSuccess) ok = false;
    }
  }
  alloc(&c->dKl, c->n_p); alloc(&c->dKr, c->n_p);
  if (!c->slab) { alloc(&c->MinvL, c->n_p); alloc(&c->MinvR, c->n_p); }
  alloc(&c->E, (k == 2 ? 1 : 3) * c->nq * c->n_el);  // k = 2: setup only (lumped element values)
  alloc(&c->tv, c->n_v); alloc(&c->tw, c->n_v);
  if (!c->slab) {
    alloc(&c->px, c->n_p); alloc(&c->pr, c->n_p); alloc(&c->pp, c->n_p); alloc(&c->pp1, c->n_p);
    alloc(&c->pq, c->n_p); alloc(&c->pz, c->n_p);
  }
  alloc(&c->s0, c->n_p); alloc(&c->s1, c->n_p); alloc(&c->s2, c->n_p);
  alloc(&c->partial, c->max_partials);
  alloc(&c->pqp, c->n_el / 8 + 1024);  // >= blocks of any K-apply grid (tiles >= 64 elements, k_B_split >= 8)
  alloc(&c->rzp, c->red_blocks);
  if (k == 2) {
    // A tiles of A_TX x A_TY x A_TZ elements; mut tile-blocked and zero for elements
    // outside the mesh (ragged tiles)
    const int64_t nt = (int64_t)((N + A_TX - 1) / A_TX) * ((N + A_TY - 1) / A_TY) * ((N + A_TZ - 1) / A_TZ);
    constexpr int64_t ne_t = A_TX * A_TY * A_TZ;
    c->n_tiles = (int)nt;
    alloc(&c->mut, nt * 27 * ne_t);
    if (ok && cudaMemsetAsync(c->mut, 0, sizeof(double) * (size_t)(nt * 27 * ne_t), c->stream) != cudaSuccess) ok = false;
    alloc(&c->Fu, nt * 3 * Tile2<A_TX, A_TY, A_TZ>::SHELL);
  } else {
    alloc(&c->mut, c->n_el * c->nq);
  }
  if (ok && cudaMalloc(&c->counter, sizeof(unsigned) * 4) != cudaSuccess) ok = false;
  if (ok && cudaMalloc(&c->icount, sizeof(unsigned long long) * 4) != cudaSuccess) ok = false;
  if (!ok) {
    free_all(c);
    delete c;
    cudaGetLastError();
    return WB_ENOMEM;
  }
  if (cudaMemsetAsync(c->counter, 0, sizeof(unsigned) * 4, c->stream) != cudaSuccess ||
      ensure_iters(c, 126) != WB_OK || configure_kernels(c) != WB_OK ||
      cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamSynchronize(c->stream) != cudaSuccess) {
    free_all(c);
    delete c;
    return WB_ECUDA;
  }
  c->tma_ok = setup_tma(c);  // the pointer kernel serves contexts without the y-fastest storage
  c->tma4_ok = setup_tma4(c);  // k = 4, even N: the fused kernel's TMA variant (else its LDG form)
  c->zm_ok = false;  // the opt-in z-march kernel's buffers and maps: set up when option k_zm is first set
  if (c->ylay && !c->tma_ok) {
    free_all(c);
    delete c;
    return WB_ECUDA;
  }
  *out = c;
  return WB_OK;
}

wb_status wb_slab_create(wb_ctx** out, int N, int k, int rank, int nranks, unsigned flags, void* stream) {
  if (!out) return WB_EINVAL;
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks || (flags & WB_DEBUG_NOMASK)) return WB_EINVAL;
  wb_ctx* c = nullptr;
  wb_status s = wb_create(&c, N, k, flags, stream);
  if (s) return s;
  DD* d = new (std::nothrow) DD();
  if (!d) { wb_destroy(c); return WB_ENOMEM; }
  c->dd = d;
  d->rank = rank; d->nranks = nranks;
  c->G.zopen = (rank > 0 ? 1 : 0) | (rank < nranks - 1 ? 2 : 0);
  bool ok = lazy_alloc(&d->gm, c->n_nodes) && lazy_alloc(&d->vs, c->n_v) && lazy_alloc(&d->own_scal, 8);
  for (double** b : {&d->r, &d->z, &d->p, &d->q, &d->x, &d->y, &d->mK[0], &d->mK[1]}) ok = ok && lazy_alloc(b, c->n_p);
  if (!ok) { wb_destroy(c); return WB_ENOMEM; }
  k_dd_mask<<<nblk(c->n_nodes, 256), 256, 0, c->stream>>>(d->gm, c->G);
  if (cudaGetLastError() != cudaSuccess || cudaMemsetAsync(d->own_scal, 0, sizeof(double) * 8, c->stream) != cudaSuccess ||
      cudaStreamSynchronize(c->stream) != cudaSuccess) {
    wb_destroy(c);
    return WB_ECUDA;
  }
  *out = c;
  return WB_OK;
}

wb_status wb_slab_set_comm(wb_ctx* c, const wb_slab_comm* comm) {
  if (!c || !comm) return WB_EINVAL;
  if (!c->dd) return set_err(c, WB_ESTATE, "not a slab context (wb_slab_create)");
  const int64_t np = (int64_t)c->G.nn1 * c->G.nn1;
  if (!comm->exchange || !comm->allreduce || !comm->send_lo || !comm->recv_lo || !comm->send_hi || !comm->recv_hi ||
      !comm->scal || comm->cap < 3 * np)
    return set_err(c, WB_EINVAL, "slab communicator: null callback / buffer, or cap < 3 (kN+1)^2");
  c->dd->comm = *comm;
  c->dd->have_comm = true;
  c->have_visc = false;  // the lumped masses depend on the neighbours: wb_set_viscosity again
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
  if (c->dd) {
    k_dd_bmask<<<nblk(c->n_nodes, 256), 256, 0, c->stream>>>(mask, c->dd->gm, c->n_nodes);
    LAUNCH_CHECK(c);
    return WB_OK;
  }
  k_bmask<<<nblk(c->n_nodes, 256), 256, 0, c->stream>>>(mask, c->G);
  LAUNCH_CHECK(c);
  return WB_OK;
}

}  // extern "C"

// copy the nonpositive-lumped-entry counts of the last setup (synchronises the stream)
static wb_status read_nonpos(wb_ctx* c) {
  if (!c->nonpos_pending) return WB_OK;
  unsigned long long np[2] = {0, 0};
  CUDA_TRY(c, cudaMemcpyAsync(np, c->icount + 1, sizeof(np), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  c->n_nonpos[0] = (long long)np[0];
  c->n_nonpos[1] = (long long)np[1];
  c->nonpos_pending = false;
  return WB_OK;
}

template <int K>
static wb_status finish_lumped(wb_ctx* c);
template <int K>
static wb_status setup_t(wb_ctx* c, const double* mu, double a_l, double a_r) {
  mg_free(c);  // a multigrid hierarchy belongs to the previous viscosity
  c->dab_valid = false;
  c->mp_valid = false;
  const int64_t nmu = c->n_el * c->nq;
  CUDA_TRY(c, cudaMemsetAsync(c->icount, 0, sizeof(unsigned long long) * 4, c->stream));
  c->dA_valid = false;
  const double* wsrc = nullptr;  // lumping weight source: mu (eq:wbfbt) or mu_eff (R17)
  if (c->weights == 1) {
    if (!c->mueff && cudaMalloc(&c->mueff, sizeof(double) * nmu) != cudaSuccess) {
      cudaGetLastError();
      c->mueff = nullptr;
      return set_err(c, WB_ENOMEM, "gradient-weight buffer allocation failed");
    }
    k_grad_weights<K><<<nblk(nmu, 256), 256, 0, c->stream>>>(mu, c->mueff, nmu, 2.0 / c->h);
    LAUNCH_CHECK(c);
    wsrc = c->mueff;
  }
  if constexpr (K == 2)  // mut and the element lumping values in one pass over mu
    k_setup_mu2<A_TX, A_TY, A_TZ><<<nblk(c->n_el, 128), 128, 0, c->stream>>>(mu, c->mut, c->E, c->N, c->h / 2,
                                                                            c->detJ, c->icount, wsrc);
  else
    k_prescale<K><<<nblk(nmu, 256), 256, 0, c->stream>>>(mu, c->mut, nmu, c->h / 2, c->icount);
  LAUNCH_CHECK(c);
  unsigned long long bad = 0;
  CUDA_TRY(c, cudaMemcpyAsync(&bad, c->icount, sizeof(bad), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (bad) {
    c->have_visc = false;
    return set_err(c, WB_ENONPOS_MU, "%llu viscosity samples are <= 0 or non-finite", bad);
  }
  if (c->schur == 2) {  // M_p(1/mu)^-1 element blocks (R21)
    if (!lazy_alloc(&c->mpinv, c->n_el * c->nm * c->nm)) return set_err(c, WB_ENOMEM, "M_p allocation failed");
    k_mp_setup<K><<<nblk(c->n_el, 64), 64, 0, c->stream>>>(mu, c->mpinv, c->n_el, c->detJ);
    LAUNCH_CHECK(c);
    c->mp_valid = true;
  }
  // lumped masses: element part into E (1 component; k = 2: by k_setup_mu2), node gather
  if constexpr (K == 2) {
    dim3 grid(nblk(c->N + 1, 64), nblk(c->G.nn1, 4), 2 * c->G.nn1);
    k_lump_node2<<<grid, dim3(64, 4), 0, c->stream>>>(c->E, a_l, a_r, c->Cw, c->Dw, c->Cinv, c->Dinv,
                                                     c->icount + 1, c->G);
  } else {
    k_lump_elem<K><<<nblk(c->n_el, 128), 128, 0, c->stream>>>(wsrc ? wsrc : mu, c->E, c->G, c->detJ);
    LAUNCH_CHECK(c);
    k_lump_node<K><<<nblk(c->n_nodes, 256), 256, 0, c->stream>>>(c->E, a_l, a_r, c->Cw, c->Dw, c->Cinv, c->Dinv,
                                                                 c->icount + 1, c->G);
  }
  LAUNCH_CHECK(c);
  if (c->dd) {  // slab: C_w, D_w summed over the shared planes, inverses under the global mask
    wb_status sd = dd_finish_lump(c);
    if (sd) return sd;
  }
  return finish_lumped<K>(c);
}

// everything downstream of C_w, D_w, C_w^-1, D_w^-1 (and the nonpositive counts in
// icount[1..2]): the Poisson kernels' X layouts, Jacobi diagonals, Minv
template <int K>
static wb_status finish_lumped(wb_ctx* c) {
  if (c->tma_ok) {  // X = C_w^-1, D_w^-1 in the tile-blocked pencil layout of the TMA kernel
    using F = FK2<TMA_TX, TMA_TY, TMA_TZ>;
    const int nt = ((c->N + TMA_TX - 1) / TMA_TX) * ((c->N + TMA_TY - 1) / TMA_TY) * ((c->N + TMA_TZ - 1) / TMA_TZ);
    k_x_tiles<TMA_TX, TMA_TY, TMA_TZ><<<nt, F::MY * F::MZ, 0, c->stream>>>(c->Cinv, c->Dinv, c->XpL, c->XpR, c->N);
    LAUNCH_CHECK(c);
  }
  if (c->tma4_ok) {  // X with padded rows for the k = 4 fused kernel's TMA variant
    k_xpad4<<<stream_blocks(c->n_nodes), VBS, 0, c->stream>>>(c->Cinv, c->Dinv, c->X4L, c->X4R, c->G.nn1);
    LAUNCH_CHECK(c);
  }
  c->xz_valid = false;  // the z-march kernel's X copy (opt-in)
  if (c->zm_ok && c->use_zm) {
    wb_status sx = build_xz(c);
    if (sx) return set_err(c, sx, "z-march X build failed");
  }
  if constexpr (K == 2)
    k_jacobi2<<<nblk(c->n_el, 128), 128, 0, c->stream>>>(c->Cinv, c->Dinv, c->dKl, c->dKr, c->G, c->sB * c->sB);
  else
    k_jacobi<K><<<nblk(c->n_el, 128), 128, 0, c->stream>>>(c->Cinv, c->Dinv, c->dKl, c->dKr, c->MinvL, c->MinvR,
                                                           c->G, c->sB);
  LAUNCH_CHECK(c);
  for (int side = 0; side < 2; ++side) {
    const double* d = side == 0 ? c->dKl : c->dKr;
    double* dmax = c->scal + S_DMAX + side;
    k_absmax<VBS><<<c->red_blocks, VBS, 0, c->stream>>>(d, c->n_p, c->partial, c->counter, dmax);
    LAUNCH_CHECK(c);
    if (c->dd) {
      wb_status sd = dd_after_dmax(c, side, d, dmax);
      if (sd) return sd;
    }
    if (c->nm == 4)
      k_minv_t<<<stream_blocks(c->n_p / 4), VBS, 0, c->stream>>>(d, side == 0 ? c->MinvL : c->MinvR, dmax, c->pl,
                                                                 c->N);
    else
      k_minv<<<c->red_blocks, VBS, 0, c->stream>>>(d, side == 0 ? c->MinvL : c->MinvR, c->n_el, c->nm, dmax, c->pl,
                                                   c->N);
    LAUNCH_CHECK(c);
  }
  c->have_visc = true;
  c->nonpos_pending = true;  // counts read lazily (wb_query), or now in strict mode
  if (c->flags & WB_STRICT_LUMP) {
    wb_status s = read_nonpos(c);
    if (s) return s;
    if (c->n_nonpos[0] || c->n_nonpos[1])
      return set_err(c, WB_ENONPOS_LUMP, "nonpositive lumped entries: C_w %lld, D_w %lld", c->n_nonpos[0],
                     c->n_nonpos[1]);
  }
  return WB_OK;
}

// ================================================================ pressure multigrid (R20)
void mg_free(wb_ctx* c) {
  MGH* M = c->mg;
  if (!M) return;
  cudaStreamSynchronize(c->stream);
  for (int l = 0; l < M->nl; ++l) {
    for (double** b : {&M->b[l], &M->x[l], &M->r[l], &M->t[l]})
      if (*b) cudaFree(*b);
    if (l > 0 && M->lev[l]) wb_destroy(M->lev[l]);
  }
  for (int l = 0; l < M->nl; ++l)
    for (double** b : {&M->mu[l], &M->vb[l], &M->vx[l], &M->vr[l], &M->vt[l]})
      if (*b) cudaFree(*b);
  for (double** b : {&M->rk, &M->zk, &M->pk, &M->qk, &M->xk, &M->s, &M->vin, &M->vout})
    if (*b) cudaFree(*b);
  clear_graphs(c);  // graphs that captured the hierarchy's buffers
  delete M;
  c->mg = nullptr;
  cudaGetLastError();
}

static wb_status mg_project(wb_ctx* c, double* v) {  // R10 on an element-major vector of c
  k_mode0_sum<<<c->red_blocks, VBS, 0, c->stream>>>(v, c->n_el, c->nm, c->partial, c->counter, c->scal + S_SCR + 1);
  LAUNCH_CHECK(c);
  k_sub_mode0_mean<<<stream_blocks(c->n_el), VBS, 0, c->stream>>>(v, c->n_el, c->nm, c->scal + S_SCR + 1);
  LAUNCH_CHECK(c);
  return WB_OK;
}

// x = V_l(b): x = S(b); x += P V_{l+1}(P^T (b - K x)); x += S(b - K x)  (element-major)
static wb_status mg_vcycle(wb_ctx* c, int side, int l, const double* b, double* x) {
  MGH& M = *c->mg;
  wb_ctx* L = M.lev[l];
  L->stream = c->stream;
  if (l > 0) L->in_capture = c->in_capture;
  const int64_t n = L->n_p;
  if (l == M.nl - 1) return run_poisson(L, side, b, x, (int)std::min<int64_t>(n, 256));
  const double lam = M.lam[side][l];
  wb_status s = run_cheb(L, side, b, x, M.nu, 0.1 * lam, 1.1 * lam);
  if (s) return s;
  if ((s = run_K(L, side, x, M.t[l]))) return s;
  k_mg_resid<<<stream_blocks(n), VBS, 0, c->stream>>>(M.r[l], b, M.t[l], n);
  LAUNCH_CHECK(c);
  const int Nc = M.Ns[l + 1];
  const bool pl = Nc == M.Ns[l];  // spectral level (same mesh, lower order)
  if (pl)
    k_mg_restrict_p<<<stream_blocks(4 * L->n_el), VBS, 0, c->stream>>>(M.r[l], M.b[l + 1], L->n_el, L->nm);
  else
    k_mg_restrict<<<stream_blocks((int64_t)Nc * Nc * Nc), VBS, 0, c->stream>>>(M.r[l], M.b[l + 1], Nc);
  LAUNCH_CHECK(c);
  if ((s = mg_vcycle(c, side, l + 1, M.b[l + 1], M.x[l + 1]))) return s;
  if (pl)
    k_mg_prolong_add_p<<<stream_blocks(4 * L->n_el), VBS, 0, c->stream>>>(M.x[l + 1], x, L->n_el, L->nm);
  else
    k_mg_prolong_add<<<stream_blocks(L->n_el), VBS, 0, c->stream>>>(M.x[l + 1], x, Nc);
  LAUNCH_CHECK(c);
  if ((s = run_K(L, side, x, M.t[l]))) return s;
  k_mg_resid<<<stream_blocks(n), VBS, 0, c->stream>>>(M.r[l], b, M.t[l], n);
  LAUNCH_CHECK(c);
  if ((s = run_cheb(L, side, M.r[l], M.t[l], M.nu, 0.1 * lam, 1.1 * lam))) return s;
  k_axpy<<<stream_blocks(n), VBS, 0, c->stream>>>(x, M.t[l], n, 1.0);
  LAUNCH_CHECK(c);
  return WB_OK;
}

// x = P MGPCG(K_side, P b): the O9 recurrence with M^-1 = one V-cycle, exactly iters
// iterations, scalars on the device
wb_status run_mgcg(wb_ctx* c, int side, const double* b, double* x, int iters) {
  MGH& M = *c->mg;
  const int64_t n = c->n_p;
  const unsigned nb = stream_blocks(n);
  CUDA_TRY(c, cudaMemcpyAsync(M.rk, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
  wb_status s = mg_project(c, M.rk);
  if (s) return s;
  CUDA_TRY(c, cudaMemsetAsync(M.xk, 0, sizeof(double) * n, c->stream));
  CUDA_TRY(c, cudaMemsetAsync(M.s, 0, sizeof(double) * 4, c->stream));
  // the V-cycle on the fixed buffers rk -> zk is replayed as one CUDA graph (kind 10 + side)
  auto vc = [&] { return graph_loop(c, 10 + side, side, 1, 0.0, 0.0, [&] { return mg_vcycle(c, side, 0, M.rk, M.zk); }); };
  if ((s = vc())) return s;
  CUDA_TRY(c, cudaMemcpyAsync(M.pk, M.zk, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
  if ((s = dev_dot(c, M.rk, M.zk, n, M.s))) return s;
  for (int it = 0; it < iters; ++it) {
    if ((s = run_K(c, side, M.pk, M.qk))) return s;
    if ((s = dev_dot(c, M.pk, M.qk, n, M.s + 1))) return s;
    k_mgcg_xr<<<nb, VBS, 0, c->stream>>>(M.xk, M.rk, M.pk, M.qk, n, M.s);
    LAUNCH_CHECK(c);
    if ((s = vc())) return s;
    if ((s = dev_dot(c, M.rk, M.zk, n, M.s + 2))) return s;
    k_mgcg_p<<<nb, VBS, 0, c->stream>>>(M.pk, M.zk, n, M.s, c->counter + 3);
    LAUNCH_CHECK(c);
  }
  CUDA_TRY(c, cudaMemcpyAsync(x, M.xk, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
  return mg_project(c, x);
}

// x = V_l(b) for M A M (velocity, SoA n_v, R22): x = S(b); x += P V_{l+1}(P^T (b - A x));
// x += S(b - A x); S = nu Chebyshev-Jacobi steps on [0.1, 1.1] lambda_l; coarsest level: 30 steps
static wb_status vmg_vcycle(wb_ctx* c, int l, const double* b, double* x) {
  MGH& M = *c->mg;
  wb_ctx* L = M.lev[l];
  L->stream = c->stream;
  if (l > 0) L->in_capture = c->in_capture;
  const int64_t n = L->n_v;
  const double lam = M.vlam[l];
  if (l == M.nl - 1) return run_vcheb(L, b, x, 30, 0.1 * lam, 1.1 * lam);
  wb_status s = run_vcheb(L, b, x, M.nu, 0.1 * lam, 1.1 * lam);
  if (s) return s;
  if ((s = run_A(L, x, M.vt[l], 0))) return s;
  k_mg_resid<<<stream_blocks(n), VBS, 0, c->stream>>>(M.vr[l], b, M.vt[l], n);
  LAUNCH_CHECK(c);
  const int Nc = M.Ns[l + 1];
  const bool pl = Nc == M.Ns[l];  // spectral level (Q4 -> Q2 on the same mesh)
  if (pl)
    k_vmg_restrict_p<<<stream_blocks(M.lev[l + 1]->n_nodes), VBS, 0, c->stream>>>(M.vr[l], M.vb[l + 1], Nc);
  else
    k_vmg_restrict<<<stream_blocks(M.lev[l + 1]->n_nodes), VBS, 0, c->stream>>>(M.vr[l], M.vb[l + 1], Nc);
  LAUNCH_CHECK(c);
  if ((s = vmg_vcycle(c, l + 1, M.vb[l + 1], M.vx[l + 1]))) return s;
  if (pl)
    k_vmg_prolong_add_p<<<stream_blocks(L->n_nodes), VBS, 0, c->stream>>>(M.vx[l + 1], x, Nc);
  else
    k_vmg_prolong_add<<<stream_blocks(L->n_nodes), VBS, 0, c->stream>>>(M.vx[l + 1], x, Nc);
  LAUNCH_CHECK(c);
  if ((s = run_A(L, x, M.vt[l], 0))) return s;
  k_mg_resid<<<stream_blocks(n), VBS, 0, c->stream>>>(M.vr[l], b, M.vt[l], n);
  LAUNCH_CHECK(c);
  if ((s = run_vcheb(L, M.vr[l], M.vt[l], M.nu, 0.1 * lam, 1.1 * lam))) return s;
  k_axpy<<<stream_blocks(n), VBS, 0, c->stream>>>(x, M.vt[l], n, 1.0);
  LAUNCH_CHECK(c);
  return WB_OK;
}
// x = M.vcycles stationary V-cycles on A x = b from x0 = 0 (level 0 vectors reused)
wb_status run_vmg(wb_ctx* c, const double* b, double* x) {
  MGH& M = *c->mg;
  const int64_t n = c->n_v;
  CUDA_TRY(c, cudaMemcpyAsync(M.vin, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
  // the cycles on the fixed buffers vin -> vout, replayed as one CUDA graph (kind 12)
  wb_status s = graph_loop(c, 12, 0, M.vcycles, 0.0, 0.0, [&] {
    wb_status st = vmg_vcycle(c, 0, M.vin, M.vout);
    for (int k = 1; k < M.vcycles && !st; ++k) {
      if ((st = run_A(c, M.vout, M.vb[0], 0))) return st;
      k_mg_resid<<<stream_blocks(n), VBS, 0, c->stream>>>(M.vb[0], M.vin, M.vb[0], n);
      LAUNCH_CHECK(c);
      if ((st = vmg_vcycle(c, 0, M.vb[0], M.vx[0]))) return st;
      k_axpy<<<stream_blocks(n), VBS, 0, c->stream>>>(M.vout, M.vx[0], n, 1.0);
      LAUNCH_CHECK(c);
    }
    return st;
  });
  if (s) return s;
  CUDA_TRY(c, cudaMemcpyAsync(x, M.vout, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
  return WB_OK;
}

template <int K>
static wb_status setup_t(wb_ctx* c, const double* mu, double a_l, double a_r);

static wb_status mg_setup_body(wb_ctx* c, int nu, const double* mu0) {
  mg_free(c);
  MGH* M = new (std::nothrow) MGH();
  if (!M) return set_err(c, WB_ENOMEM, "multigrid allocation failed");
  c->mg = M;
  M->nu = nu;
  int N = c->N;
  M->Ns[M->nl] = N; M->Ks[M->nl++] = c->k;
  if (c->k == 4) { M->Ns[M->nl] = N; M->Ks[M->nl++] = 2; }  // spectral level first
  while (N % 2 == 0 && N > 1 && M->nl < 16) { N /= 2; M->Ns[M->nl] = N; M->Ks[M->nl++] = 2; }
  M->lev[0] = c;
  auto fail = [&](wb_status st, const char* what) {
    mg_free(c);
    return set_err(c, st, "multigrid setup: %s", what);
  };
  for (int l = 1; l < M->nl; ++l) {
    wb_ctx* L = nullptr;
    wb_status st = wb_create(&L, M->Ns[l], M->Ks[l], 0, (void*)c->stream);
    if (st) return fail(st, "level context");
    M->lev[l] = L;
    wb_ctx* F = M->lev[l - 1];
    if (mu0) {  // velocity hierarchy: coarsened viscosity, the level's A (and, overwritten below, its lumping)
      if (!lazy_alloc(&M->mu[l], L->n_el * 27)) return fail(WB_ENOMEM, "coarse viscosity");
      const double* muf = l == 1 ? mu0 : M->mu[l - 1];
      if (M->Ns[l] == M->Ns[l - 1])  // spectral level: 125 -> 27 Gauss points per element
        k_mu_coarsen_p<<<stream_blocks(L->n_el * 27), VBS, 0, c->stream>>>(muf, M->mu[l], L->n_el);
      else
        k_mu_coarsen<<<stream_blocks(L->n_el * 27), VBS, 0, c->stream>>>(muf, M->mu[l], M->Ns[l]);
      LAUNCH_CHECK(c);
      if ((st = setup_t<2>(L, M->mu[l], 1.0, 1.0))) return fail(st, wb_last_error(L));
    }
    CUDA_TRY(c, cudaMemsetAsync(L->icount, 0, sizeof(unsigned long long) * 4, c->stream));
    if (M->Ns[l] == M->Ns[l - 1])
      k_mg_inject_p<<<stream_blocks(L->n_nodes), VBS, 0, c->stream>>>(F->Cw, F->Dw, L->Cw, L->Dw, M->Ns[l]);
    else
      k_mg_inject<<<stream_blocks(L->n_nodes), VBS, 0, c->stream>>>(F->Cw, F->Dw, L->Cw, L->Dw, M->Ns[l]);
    LAUNCH_CHECK(c);
    k_inv_lumped<<<stream_blocks(L->n_nodes), VBS, 0, c->stream>>>(L->Cw, L->Dw, L->Cinv, L->Dinv, L->icount + 1,
                                                                   L->G);
    LAUNCH_CHECK(c);
    if ((st = finish_lumped<2>(L))) return fail(st, wb_last_error(L));
  }
  auto dalloc = [](double** p, int64_t n) {
    return cudaMalloc(p, sizeof(double) * (size_t)std::max<int64_t>(n, 1)) == cudaSuccess;
  };
  for (int l = 0; l < M->nl; ++l) {
    const int64_t n = M->lev[l]->n_p;
    if (!dalloc(&M->b[l], n) || !dalloc(&M->x[l], n) || !dalloc(&M->r[l], n) || !dalloc(&M->t[l], n))
      return fail(WB_ENOMEM, "level vectors");
  }
  const int64_t n0 = c->n_p;
  if (!dalloc(&M->rk, n0) || !dalloc(&M->zk, n0) || !dalloc(&M->pk, n0) || !dalloc(&M->qk, n0) ||
      !dalloc(&M->xk, n0) || !dalloc(&M->s, 4))
    return fail(WB_ENOMEM, "MG-PCG vectors");
  if (mu0) {
    M->vel = true;
    if (!dalloc(&M->vin, c->n_v) || !dalloc(&M->vout, c->n_v)) return fail(WB_ENOMEM, "velocity cycle vectors");
    for (int l = 0; l < M->nl; ++l) {
      wb_ctx* L = M->lev[l];
      const int64_t nv = L->n_v;
      if (!dalloc(&M->vb[l], nv) || !dalloc(&M->vx[l], nv) || !dalloc(&M->vr[l], nv) || !dalloc(&M->vt[l], nv))
        return fail(WB_ENOMEM, "velocity level vectors");
      k_splitmix<<<stream_blocks(nv), VBS, 0, c->stream>>>(M->vb[l], nv, 0x5EEDull);
      LAUNCH_CHECK(c);
      wb_status st = run_veigmax(L, M->vb[l], 20, &M->vlam[l]);
      if (st) return fail(st, "velocity eigenvalue estimate");
    }
  }
  {  // the coarsest solve's PCG histories, allocated now: the V-cycle is replayed as a captured graph
    wb_ctx* Lc = M->lev[M->nl - 1];
    wb_status st = ensure_iters(Lc, (int)std::min<int64_t>(Lc->n_p, 256));
    if (st) return fail(st, "coarse PCG histories");
  }
  // Chebyshev intervals: power iteration (20 steps) from the splitmix64 start vector
  for (int l = 0; l < M->nl - 1; ++l) {
    wb_ctx* L = M->lev[l];
    k_splitmix<<<stream_blocks(L->n_p), VBS, 0, c->stream>>>(M->b[l], L->n_p, 0x5EEDull);
    LAUNCH_CHECK(c);
    for (int side = 0; side < 2; ++side) {
      wb_status st = run_eigmax(L, side, M->b[l], 20, &M->lam[side][l]);
      if (st) return fail(st, "eigenvalue estimate");
    }
  }
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return WB_OK;
}
static wb_status mg_setup(wb_ctx* c, int nu, const double* mu0) {
  const wb_status s = mg_setup_body(c, nu, mu0);
  if (s && c->mg) {
    char msg[sizeof(c->err)];
    std::memcpy(msg, c->err, sizeof(msg));
    mg_free(c);  // never leave a partial hierarchy behind
    std::memcpy(c->err, msg, sizeof(msg));
  }
  return s;
}

extern "C" {

wb_status wb_set_viscosity(wb_ctx* c, const double* mu_q, double a_l, double a_r) {
  if (!c || !mu_q) return WB_EINVAL;
  if (c->dd && c->dd->nranks > 1 && !c->dd->have_comm)
    return set_err(c, WB_ESTATE, "slab context without a communicator: wb_slab_set_comm first");
  if (!(a_l >= 1.0) || !(a_r >= 1.0) || !std::isfinite(a_l) || !std::isfinite(a_r))
    return set_err(c, WB_EINVAL, "a_l, a_r must be finite and >= 1");
  switch (c->k) {
    case 2: return setup_t<2>(c, mu_q, a_l, a_r);
    case 3: return setup_t<3>(c, mu_q, a_l, a_r);
    default: return setup_t<4>(c, mu_q, a_l, a_r);
  }
}

wb_status wb_apply_A(wb_ctx* c, const double* u, double* y) {
  wb_status s = check_ctx(c, true, true);
  if (s) return s;
  if (!u || !y) return set_err(c, WB_EINVAL, "null pointer");
  if (overlaps(u, 8 * c->n_v, y, 8 * c->n_v)) return set_err(c, WB_EALIAS, "u and y overlap");
  if (c->dd) return dd_A(c, u, y, false);
  return run_A(c, u, y, (c->flags & WB_DEBUG_NOMASK) ? 1 : 0);
}

wb_status wb_apply_B(wb_ctx* c, const double* u, double* p) {
  wb_status s = check_ctx(c, false, true);
  if (s) return s;
  if (!u || !p) return set_err(c, WB_EINVAL, "null pointer");
  if (overlaps(u, 8 * c->n_v, p, 8 * c->n_p)) return set_err(c, WB_EALIAS, "u and p overlap");
  if (c->dd) return dd_B(c, u, nullptr, p);
  return run_B(c, u, nullptr, p, (c->flags & WB_DEBUG_NOMASK) ? 1 : 0, nullptr, nullptr, nullptr, c->nm, 1);
}

wb_status wb_apply_BT(wb_ctx* c, const double* p, double* y) {
  wb_status s = check_ctx(c, false, true);
  if (s) return s;
  if (!p || !y) return set_err(c, WB_EINVAL, "null pointer");
  if (overlaps(p, 8 * c->n_p, y, 8 * c->n_v)) return set_err(c, WB_EALIAS, "p and y overlap");
  if (c->dd) return dd_BT(c, p, nullptr, y);
  return run_BT(c, p, nullptr, y, (c->flags & WB_DEBUG_NOMASK) ? 1 : 0, nullptr, c->nm, 1);
}

wb_status wb_apply_K(wb_ctx* c, int side, const double* p, double* q) {
  wb_status s = check_ctx(c, true, true);
  if (s) return s;
  if (!p || !q || (side != 0 && side != 1)) return set_err(c, WB_EINVAL, "bad argument");
  if (overlaps(p, 8 * c->n_p, q, 8 * c->n_p)) return set_err(c, WB_EALIAS, "p and q overlap");
  if (c->dd) return dd_K(c, side, p, q);
  return run_K(c, side, p, q);
}

wb_status wb_poisson_pcg(wb_ctx* c, int side, const double* b, double* x, int iters) {
  wb_status s = check_ctx(c, true, true);
  if (s) return s;
  if (!b || !x || (side != 0 && side != 1) || iters < 0) return set_err(c, WB_EINVAL, "bad argument");
  if (overlaps(b, 8 * c->n_p, x, 8 * c->n_p)) return set_err(c, WB_EALIAS, "b and x overlap");
  if (c->dd) return dd_pcg(c, side, b, x, iters);
  return run_poisson(c, side, b, x, iters);
}

wb_status wb_poisson_cheb(wb_ctx* c, int side, const double* b, double* x, int iters, double lmin, double lmax) {
  wb_status s = check_ctx(c, true);
  if (s) return s;
  if (!b || !x || (side != 0 && side != 1) || iters < 0) return set_err(c, WB_EINVAL, "bad argument");
  if (!(lmin > 0.0) || !(lmax > lmin) || !std::isfinite(lmax))
    return set_err(c, WB_EINVAL, "the interval must satisfy 0 < lmin < lmax < inf");
  if (overlaps(b, 8 * c->n_p, x, 8 * c->n_p)) return set_err(c, WB_EALIAS, "b and x overlap");
  return run_cheb(c, side, b, x, iters, lmin, lmax);
}

wb_status wb_poisson_eigmax(wb_ctx* c, int side, const double* v0, int iters, double* lmax) {
  wb_status s = check_ctx(c, true);
  if (s) return s;
  if (!v0 || !lmax || (side != 0 && side != 1) || iters < 0) return set_err(c, WB_EINVAL, "bad argument");
  return run_eigmax(c, side, v0, iters, lmax);
}

wb_status wb_get_diagA(wb_ctx* c, double* dA) {
  wb_status s = check_ctx(c, true);
  if (s) return s;
  if (!dA) return set_err(c, WB_EINVAL, "bad argument");
  return run_diagA(c, dA);
}

wb_status wb_velocity_cheb(wb_ctx* c, const double* b, double* x, int iters, double lmin, double lmax) {
  wb_status s = check_ctx(c, true);
  if (s) return s;
  if (!b || !x || iters < 0) return set_err(c, WB_EINVAL, "bad argument");
  if (!(lmin > 0.0) || !(lmax > lmin) || !std::isfinite(lmax))
    return set_err(c, WB_EINVAL, "the interval must satisfy 0 < lmin < lmax < inf");
  if (overlaps(b, 8 * c->n_v, x, 8 * c->n_v)) return set_err(c, WB_EALIAS, "b and x overlap");
  return run_vcheb(c, b, x, iters, lmin, lmax);
}

wb_status wb_velocity_eigmax(wb_ctx* c, const double* v0, int iters, double* lmax) {
  wb_status s = check_ctx(c, true);
  if (s) return s;
  if (!v0 || !lmax || iters < 0) return set_err(c, WB_EINVAL, "bad argument");
  return run_veigmax(c, v0, iters, lmax);
}

wb_status wb_stokes_fgmres(wb_ctx* c, const double* f, const double* g, double* u, double* p, int restart,
                           int max_iters, double rtol, int pcg_iters, int smooth_iters, double lmin, double lmax,
                           int* iters, double* relres) {
  wb_status s = check_ctx(c, true);
  if (s) return s;
  if (!f || !g || !u || !p || restart < 1 || max_iters < 0 || !(rtol >= 0.0) || pcg_iters < 0 || smooth_iters < 0)
    return set_err(c, WB_EINVAL, "bad argument");
  if (!(lmin > 0.0) || !(lmax > lmin) || !std::isfinite(lmax))
    return set_err(c, WB_EINVAL, "the smoother interval must satisfy 0 < lmin < lmax < inf");
  if (overlaps(u, 8 * c->n_v, f, 8 * c->n_v) || overlaps(p, 8 * c->n_p, g, 8 * c->n_p) ||
      overlaps(u, 8 * c->n_v, p, 8 * c->n_p))
    return set_err(c, WB_EALIAS, "outputs overlap inputs or each other");
  return run_stokes(c, f, g, u, p, restart, max_iters, rtol, StokesPar{pcg_iters, smooth_iters, lmin, lmax}, iters,
                    relres);
}

wb_status wb_set_inner_cheb(wb_ctx* c, double lmin_l, double lmax_l, double lmin_r, double lmax_r) {
  if (!c) return WB_EINVAL;
  if (c->dd) return check_ctx(c, false);
  if (lmin_l == 0.0 && lmax_l == 0.0 && lmin_r == 0.0 && lmax_r == 0.0) {
    c->inner = 0;
    return WB_OK;
  }
  const double lo[2] = {lmin_l, lmin_r}, hi[2] = {lmax_l, lmax_r};
  for (int i = 0; i < 2; ++i)
    if (!(lo[i] > 0.0) || !(hi[i] > lo[i]) || !std::isfinite(hi[i]))
      return set_err(c, WB_EINVAL, "each interval must satisfy 0 < lmin < lmax < inf (or all four 0)");
  for (int i = 0; i < 2; ++i) { c->cheb_lo[i] = lo[i]; c->cheb_hi[i] = hi[i]; }
  c->inner = 1;
  return WB_OK;
}

wb_status wb_set_schur(wb_ctx* c, int kind) {
  if (!c) return WB_EINVAL;
  if (c->dd) return check_ctx(c, false);
  if (kind < 0 || kind > 2) return set_err(c, WB_EINVAL, "kind must be 0 (wBFBT), 1 (diag(A)-BFBT) or 2 (M_p)");
  c->schur = kind;
  return WB_OK;
}

wb_status wb_apply_dabfbt(wb_ctx* c, const double* r, double* z, int iters) {
  wb_status s = check_ctx(c, true);
  if (s) return s;
  if (!r || !z || iters < 0) return set_err(c, WB_EINVAL, "bad argument");
  const size_t bp = sizeof(double) * c->n_p;
  if (overlaps(r, bp, z, bp)) return set_err(c, WB_EALIAS, "r and z overlap");
  return run_dabfbt(c, r, z, iters);
}

wb_status wb_apply_mpinv(wb_ctx* c, const double* r, double* z) {
  wb_status s = check_ctx(c, true);
  if (s) return s;
  if (!r || !z) return set_err(c, WB_EINVAL, "bad argument");
  const size_t bp = sizeof(double) * c->n_p;
  if (overlaps(r, bp, z, bp)) return set_err(c, WB_EALIAS, "r and z overlap");
  return run_mpinv(c, r, z, 1.0);
}

wb_status wb_load_vector(wb_ctx* c, const double* fq, double* F) {
  if (!c || !fq || !F) return c ? set_err(c, WB_EINVAL, "null pointer") : WB_EINVAL;
  if (c->dd) return check_ctx(c, false);
  if (overlaps(fq, sizeof(double) * 3 * c->n_el * c->nq, F, sizeof(double) * c->n_v))
    return set_err(c, WB_EALIAS, "fq and F overlap");
  const unsigned nb = nblk(c->n_nodes, 128);
  switch (c->k) {
    case 2: k_load_node<2><<<nb, 128, 0, c->stream>>>(fq, F, c->G, c->detJ); break;
    case 3: k_load_node<3><<<nb, 128, 0, c->stream>>>(fq, F, c->G, c->detJ); break;
    default: k_load_node<4><<<nb, 128, 0, c->stream>>>(fq, F, c->G, c->detJ); break;
  }
  LAUNCH_CHECK(c);
  return WB_OK;
}

wb_status wb_setup_mg(wb_ctx* c, int nu, const double* mu_q) {
  wb_status s = check_ctx(c, true);
  if (s) return s;
  if (c->k != 2 && c->k != 4) return set_err(c, WB_EINVAL, "the multigrid is built for k = 2 and 4 (R20)");
  if (nu < 1 || nu > 16) return set_err(c, WB_EINVAL, "nu must be in [1, 16]");
  return mg_setup(c, nu, mu_q);
}

wb_status wb_velocity_vcycle(wb_ctx* c, const double* b, double* x) {
  wb_status s = check_ctx(c, true);
  if (s) return s;
  if (!c->mg || !c->mg->vel) return set_err(c, WB_ESTATE, "no velocity multigrid (wb_setup_mg with mu)");
  if (!b || !x) return set_err(c, WB_EINVAL, "bad argument");
  const size_t bv = sizeof(double) * c->n_v;
  if (overlaps(b, bv, x, bv)) return set_err(c, WB_EALIAS, "b and x overlap");
  return vmg_vcycle(c, 0, b, x);
}

wb_status wb_set_velocity_mg(wb_ctx* c, int cycles) {
  if (!c) return WB_EINVAL;
  if (c->dd) return check_ctx(c, false);
  if (cycles < 0) return set_err(c, WB_EINVAL, "cycles must be >= 0");
  if (cycles > 0 && !(c->mg && c->mg->vel)) return set_err(c, WB_ESTATE, "no velocity multigrid (wb_setup_mg with mu)");
  if (c->mg) c->mg->vcycles = cycles;
  return WB_OK;
}

wb_status wb_mg_vcycle(wb_ctx* c, int side, const double* b, double* x) {
  wb_status s = check_ctx(c, true);
  if (s) return s;
  if (!c->mg) return set_err(c, WB_ESTATE, "no multigrid hierarchy (wb_setup_mg)");
  if (!b || !x || (side != 0 && side != 1)) return set_err(c, WB_EINVAL, "bad argument");
  const size_t bp = sizeof(double) * c->n_p;
  if (overlaps(b, bp, x, bp)) return set_err(c, WB_EALIAS, "b and x overlap");
  return mg_vcycle(c, side, 0, b, x);
}

wb_status wb_poisson_mgcg(wb_ctx* c, int side, const double* b, double* x, int iters) {
  wb_status s = check_ctx(c, true);
  if (s) return s;
  if (!c->mg) return set_err(c, WB_ESTATE, "no multigrid hierarchy (wb_setup_mg)");
  if (!b || !x || (side != 0 && side != 1) || iters < 0) return set_err(c, WB_EINVAL, "bad argument");
  const size_t bp = sizeof(double) * c->n_p;
  if (overlaps(b, bp, x, bp)) return set_err(c, WB_EALIAS, "b and x overlap");
  return run_mgcg(c, side, b, x, iters);
}

wb_status wb_set_inner_mg(wb_ctx* c, int iters) {
  if (!c) return WB_EINVAL;
  if (c->dd) return check_ctx(c, false);
  if (iters < 0) return set_err(c, WB_EINVAL, "iters must be >= 0");
  if (iters > 0 && !c->mg) return set_err(c, WB_ESTATE, "no multigrid hierarchy (wb_setup_mg)");
  if (c->mg) c->mg->inner_iters = iters;
  return WB_OK;
}

wb_status wb_mg_get_lumped(wb_ctx* c, int level, double* Cw, double* Dw) {
  if (!c) return WB_EINVAL;
  if (c->dd) return check_ctx(c, false);
  if (!c->mg) return set_err(c, WB_ESTATE, "no multigrid hierarchy (wb_setup_mg)");
  if (level < 0 || level >= c->mg->nl) return set_err(c, WB_EINVAL, "bad level");
  wb_ctx* L = c->mg->lev[level];
  const size_t bn = sizeof(double) * L->n_nodes;
  if (Cw) CUDA_TRY(c, cudaMemcpyAsync(Cw, L->Cw, bn, cudaMemcpyDeviceToDevice, c->stream));
  if (Dw) CUDA_TRY(c, cudaMemcpyAsync(Dw, L->Dw, bn, cudaMemcpyDeviceToDevice, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return WB_OK;
}

wb_status wb_apply_wbfbt(wb_ctx* c, const double* r, double* z, int iters) {
  wb_status s = check_ctx(c, true, true);
  if (s) return s;
  if (!r || !z || iters < 0) return set_err(c, WB_EINVAL, "bad argument");
  if (overlaps(r, 8 * c->n_p, z, 8 * c->n_p)) return set_err(c, WB_EALIAS, "r and z overlap");
  if (c->dd) return dd_wbfbt(c, r, z, iters);
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

static wb_status hotpath_host_body(wb_ctx* c, double* dmu, double a_l, double a_r, double* du, double* dp, int iters,
                                   double* dyA, double* dpB, double* dyBT, double* dz, double* yA, double* pB,
                                   double* yBT, double* z, size_t bv, size_t bp);

wb_status wb_hotpath_host(wb_ctx* c, const double* mu_q, double a_l, double a_r, const double* u, const double* p,
                          int iters, double* yA, double* pB, double* yBT, double* z) {
  if (!c || !mu_q || !u || !p || !yA || !pB || !yBT || !z) return WB_EINVAL;
  if (c->dd) return check_ctx(c, false);
  // validate everything that can be checked on the host before any copy is issued
  if (iters < 0) return set_err(c, WB_EINVAL, "iters must be >= 0");
  if (!(a_l >= 1.0) || !(a_r >= 1.0) || !std::isfinite(a_l) || !std::isfinite(a_r))
    return set_err(c, WB_EINVAL, "a_l, a_r must be finite and >= 1");
  // sub-buffers rounded to 32 doubles (256-byte aligned)
  auto rnd = [](int64_t n) { return (n + 31) & ~(int64_t)31; };
  const int64_t nmu = c->n_el * c->nq, rmu = rnd(nmu), rv = rnd(c->n_v), rp = rnd(c->n_p);
  if (!c->stage) {
    if (cudaMalloc(&c->stage, sizeof(double) * (size_t)(rmu + 3 * rv + 3 * rp)) != cudaSuccess) {
      c->stage = nullptr;
      cudaGetLastError();
      return set_err(c, WB_ENOMEM, "staging allocation failed");
    }
  }
  double* dmu = c->stage;
  double* du = dmu + rmu;
  double* dyA = du + rv;
  double* dyBT = dyA + rv;
  double* dp = dyBT + rv;
  double* dpB = dp + rp;
  double* dz = dpB + rp;
  const size_t bmu = sizeof(double) * nmu, bv = sizeof(double) * c->n_v, bp = sizeof(double) * c->n_p;
  // Copies overlap compute (pinned host memory makes them asynchronous).  Order of work:
  // mu in (critical) -> setup -> wBFBT's right Poisson solve (needs only p, which
  // arrives first on the copy stream) while u arrives -> the standalone A, B, B^T ->
  // the middle of wBFBT -> its left Poisson solve, while yA, pB and yBT travel back;
  // then z out.  The wBFBT kernel sequence is exactly run_wbfbt's.
  if (!c->copy_stream) {
    if (cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking) != cudaSuccess) {
      c->copy_stream = nullptr;
      cudaGetLastError();
      return set_err(c, WB_ECUDA, "copy stream creation failed");
    }
    for (cudaEvent_t* e : {&c->ev_in, &c->ev_ab, &c->ev_bt, &c->ev_done, &c->ev_p})
      CUDA_TRY(c, cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  }
  cudaStream_t cs = c->copy_stream;
  CUDA_TRY(c, cudaEventRecord(c->ev_done, c->stream));  // previous work on the context stream
  CUDA_TRY(c, cudaStreamWaitEvent(cs, c->ev_done, 0));
  CUDA_TRY(c, cudaMemcpyAsync(dmu, mu_q, bmu, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(dp, p, bp, cudaMemcpyHostToDevice, cs));
  CUDA_TRY(c, cudaEventRecord(c->ev_p, cs));
  CUDA_TRY(c, cudaMemcpyAsync(du, u, bv, cudaMemcpyHostToDevice, cs));
  CUDA_TRY(c, cudaEventRecord(c->ev_in, cs));
  // From here on the copy stream may still be reading the caller's host buffers: every
  // return path drains it first, so the caller may free or reuse them on return.
  wb_status s = hotpath_host_body(c, dmu, a_l, a_r, du, dp, iters, dyA, dpB, dyBT, dz, yA, pB, yBT, z, bv, bp);
  cudaStreamSynchronize(cs);
  if (s) return s;
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return WB_OK;
}

static wb_status hotpath_host_body(wb_ctx* c, double* dmu, double a_l, double a_r, double* du, double* dp, int iters,
                                   double* dyA, double* dpB, double* dyBT, double* dz, double* yA, double* pB,
                                   double* yBT, double* z, size_t bv, size_t bp) {
  cudaStream_t cs = c->copy_stream;
  wb_status s = wb_set_viscosity(c, dmu, a_l, a_r);  // synchronous (status)
  if (s) return s;
  const int nomask = (c->flags & WB_DEBUG_NOMASK) ? 1 : 0;
  // wBFBT, right solve: y = P PCG(K_r, P p)
  CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->ev_p, 0));
  if ((s = run_inner(c, 1, dp, c->s2, iters))) return s;
  // standalone applies
  CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->ev_in, 0));
  if ((s = run_A(c, du, dyA, nomask))) return s;
  if ((s = run_B(c, du, nullptr, dpB, nomask, nullptr, nullptr, nullptr, c->nm, 1))) return s;
  CUDA_TRY(c, cudaEventRecord(c->ev_ab, c->stream));
  if ((s = run_BT(c, dp, nullptr, dyBT, nomask, nullptr, c->nm, 1))) return s;
  CUDA_TRY(c, cudaEventRecord(c->ev_bt, c->stream));
  CUDA_TRY(c, cudaStreamWaitEvent(cs, c->ev_ab, 0));
  CUDA_TRY(c, cudaMemcpyAsync(yA, dyA, bv, cudaMemcpyDeviceToHost, cs));
  CUDA_TRY(c, cudaMemcpyAsync(pB, dpB, bp, cudaMemcpyDeviceToHost, cs));
  CUDA_TRY(c, cudaStreamWaitEvent(cs, c->ev_bt, 0));
  CUDA_TRY(c, cudaMemcpyAsync(yBT, dyBT, bv, cudaMemcpyDeviceToHost, cs));
  // wBFBT, middle and left solve (as run_wbfbt)
  if ((s = run_BT(c, c->s2, c->Dinv, c->tw, 0, nullptr, c->nm, 1))) return s;
  if ((s = run_A(c, c->tw, c->tv, 0))) return s;
  if ((s = run_B(c, c->tv, c->Cinv, c->s2, 0, nullptr, nullptr, nullptr, c->nm, 1))) return s;
  if ((s = run_inner(c, 0, c->s2, dz, iters))) return s;
  CUDA_TRY(c, cudaMemcpyAsync(z, dz, bp, cudaMemcpyDeviceToHost, c->stream));
  return WB_OK;
}

wb_status wb_debug_pcg_step(wb_ctx* c, int side, double* x, double* r, double* p, double* rz) {
  wb_status s = check_ctx(c, true);
  if (s) return s;
  if (!x || !r || !p || !rz || (side != 0 && side != 1)) return set_err(c, WB_EINVAL, "bad argument");
  if ((s = ensure_iters(c, 2))) return s;
  const double* Minv = side == 0 ? c->MinvL : c->MinvR;
  // state in (element-major -> mode-major), rz as rz_1, iteration index 1
  for (int i = 0; i < 3; ++i) {
    k_transpose<<<stream_blocks(c->n_p), VBS, 0, c->stream>>>(i == 0 ? x : (i == 1 ? r : p), i == 0 ? c->px : (i == 1 ? c->pr : c->pp),
                                                      c->n_el, c->nm, 1, c->pl, c->N);
    LAUNCH_CHECK(c);
  }
  CUDA_TRY(c, cudaMemcpyAsync(rz_hist(c) + 1, rz, sizeof(double), cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemsetAsync(c->stop, 0, 3 * sizeof(int), c->stream));
  const double* pcur = nullptr;
  int npq = 0;
  PcgArgs a;
  a.it = 1; a.ctl = 0;  // rz_1 and stop_1 given
  if ((s = run_K_pcg(c, side, 2, c->pp, c->pp1, c->pr, c->pq, a, &pcur, &npq))) return s;
  k_pcg_upd<XU_SINGLE><<<c->red_blocks, VBS, 0, c->stream>>>(c->px, c->pr, pcur, nullptr, c->pq, Minv, c->pl.n, 1,
                                                             c->pqp, npq,
                                                  rz_hist(c), pq_hist(c), c->stop, c->rzp, nullptr);
  LAUNCH_CHECK(c);
  // p = Minv r + (rz_2 / rz_1) p with the control of iteration 2 (records rz_2)
  double* pc = const_cast<double*>(pcur);
  k_pupd<<<c->red_blocks, VBS, 0, c->stream>>>(pc, pc, c->pr, Minv, c->pl.n, 1, 2, 1, c->rzp, c->red_blocks,
                                               rz_hist(c), pq_hist(c), c->stop);
  LAUNCH_CHECK(c);
  for (int i = 0; i < 3; ++i) {
    k_transpose<<<stream_blocks(c->n_p), VBS, 0, c->stream>>>(i == 0 ? c->px : (i == 1 ? c->pr : pc), i == 0 ? x : (i == 1 ? r : p),
                                                      c->n_el, c->nm, 0, c->pl, c->N);
    LAUNCH_CHECK(c);
  }
  CUDA_TRY(c, cudaMemcpyAsync(rz, rz_hist(c) + 2, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return WB_OK;
}

wb_status wb_get_lumped(wb_ctx* c, double* Cw, double* Dw, double* Cinv, double* Dinv) {
  wb_status s = check_ctx(c, true, true);
  if (s) return s;
  const size_t b = sizeof(double) * c->n_nodes;
  if (Cw) CUDA_TRY(c, cudaMemcpyAsync(Cw, c->Cw, b, cudaMemcpyDeviceToDevice, c->stream));
  if (Dw) CUDA_TRY(c, cudaMemcpyAsync(Dw, c->Dw, b, cudaMemcpyDeviceToDevice, c->stream));
  if (Cinv) CUDA_TRY(c, cudaMemcpyAsync(Cinv, c->Cinv, b, cudaMemcpyDeviceToDevice, c->stream));
  if (Dinv) CUDA_TRY(c, cudaMemcpyAsync(Dinv, c->Dinv, b, cudaMemcpyDeviceToDevice, c->stream));
  return WB_OK;
}

wb_status wb_get_jacobi(wb_ctx* c, double* dKl, double* dKr) {
  wb_status s = check_ctx(c, true, true);
  if (s) return s;
  const size_t b = sizeof(double) * c->n_p;
  if (dKl) CUDA_TRY(c, cudaMemcpyAsync(dKl, c->dKl, b, cudaMemcpyDeviceToDevice, c->stream));
  if (dKr) CUDA_TRY(c, cudaMemcpyAsync(dKr, c->dKr, b, cudaMemcpyDeviceToDevice, c->stream));
  return WB_OK;
}

wb_status wb_query(wb_ctx* c, const char* key, double* value) {
  if (!c || !key || !value) return WB_EINVAL;
  if (!strcmp(key, "n_nonpos_Cw") || !strcmp(key, "n_nonpos_Dw")) {
    wb_status s = read_nonpos(c);
    if (s) return s;
    *value = (double)c->n_nonpos[key[9] == 'C' ? 0 : 1];  // "n_nonpos_Cw"[9] == 'C'
  }
  else if (!strcmp(key, "n_el")) *value = (double)c->n_el;
  else if (!strcmp(key, "n_p")) *value = (double)c->n_p;
  else if (!strcmp(key, "n_v")) *value = (double)c->n_v;
  else if (!strcmp(key, "kernel_launches")) *value = (double)c->launches;
  else if (!strcmp(key, "prof_k_count")) *value = (double)c->prof_n;
  else if (!strcmp(key, "occ_k2")) {  // resident CTAs per SM of the large-mesh fused K kernel
    int nb = 0;
    CUDA_TRY(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_K2_fused<4, 8, 8, 2>, FK2<4, 8, 8>::NTH,
                                                              FK2<4, 8, 8>::SMEM));
    *value = nb;
#ifdef WB_KPROF
  } else if (!strncmp(key, "aprof", 5) && key[5] >= '0' && key[5] <= '7' && !key[6]) {
    // phase-timing probe of the A tile kernel; reading "aprof7" clears the counters
    unsigned long long h[8];
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    CUDA_TRY(c, cudaMemcpyFromSymbol(h, g_aprof, sizeof(h)));
    *value = (double)h[key[5] - '0'];
    if (key[5] == '7') {
      memset(h, 0, sizeof(h));
      CUDA_TRY(c, cudaMemcpyToSymbol(g_aprof, h, sizeof(h)));
    }
#endif
#ifdef WB_KPROF
  } else if (!strncmp(key, "ktl", 3) && key[3] >= '0' && key[3] <= '5' && !key[4]) {
    // launch timeline of PCG iteration 5 (ns): 0 span (last exit - first entry), 1 entry
    // spread, 2 mean entry -> loop start, 3 mean loop, 4 mean loop end -> exit, 5 exit spread
    unsigned long long h[512][4];
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    CUDA_TRY(c, cudaMemcpyFromSymbol(h, g_ktl, sizeof(h)));
    const int n = std::min(c->nsm, 512);
    unsigned long long e0 = ~0ull, e1 = 0, x0 = ~0ull, x1 = 0;
    double pro = 0, loop = 0, epi = 0;
    for (int i = 0; i < n; ++i) {
      e0 = std::min(e0, h[i][0]); e1 = std::max(e1, h[i][0]);
      x0 = std::min(x0, h[i][3]); x1 = std::max(x1, h[i][3]);
      pro += (double)(h[i][1] - h[i][0]); loop += (double)(h[i][2] - h[i][1]); epi += (double)(h[i][3] - h[i][2]);
    }
    const double v[6] = {(double)(x1 - e0), (double)(e1 - e0), pro / n, loop / n, epi / n, (double)(x1 - x0)};
    *value = v[key[3] - '0'];
#endif
  } else if (!strncmp(key, "kprof", 5) && key[5] >= '0' && key[5] <= '7' && !key[6]) {
    // phase-timing probe of the TMA Poisson kernel (k_dbg 0x4000): accumulated cycles;
    // reading "kprof7" (the last) clears the counters
    unsigned long long h[8];
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    CUDA_TRY(c, cudaMemcpyFromSymbol(h, g_kprof, sizeof(h)));
    *value = (double)h[key[5] - '0'];
    if (key[5] == '7') {
      memset(h, 0, sizeof(h));
      CUDA_TRY(c, cudaMemcpyToSymbol(g_kprof, h, sizeof(h)));
    }
  } else if (!strcmp(key, "kz")) {  // 1: the PCG update stores z = Minv r and the TMA kernel loads it
    *value = (tma_active(c) && c->kz) ? 1.0 : 0.0;
  } else if (!strcmp(key, "k_tma")) {  // 1: the Poisson operator runs as the TMA kernel (k_K2_tma)
    *value = tma_active(c) ? 1.0 : 0.0;
  } else if (!strcmp(key, "weights")) {
    *value = c->weights;
  } else if (!strcmp(key, "inner")) {  // 1: wBFBT's inner solves are Chebyshev-Jacobi (wb_set_inner_cheb)
    *value = c->inner;
  } else if (!strcmp(key, "mg_levels")) {  // levels of the pressure multigrid (0: none built)
    *value = c->mg ? c->mg->nl : 0;
  } else if (!strncmp(key, "mg_vlambda_", 11)) {  // Chebyshev scale of the level-l velocity smoother
    const int l = atoi(key + 11);
    if (!c->mg || !c->mg->vel || l < 0 || l >= c->mg->nl) return set_err(c, WB_EINVAL, "bad key '%s'", key);
    *value = c->mg->vlam[l];
  } else if (!strncmp(key, "mg_N_", 5) || !strncmp(key, "mg_k_", 5) || !strncmp(key, "mg_lambda_", 10) ||
             !strncmp(key, "mg_nonpos_", 10)) {
    // mg_N_<l>; mg_lambda_<side>_<l> (Chebyshev interval scale); mg_nonpos_<side>_<l>
    if (!c->mg) return set_err(c, WB_ESTATE, "no multigrid hierarchy (wb_setup_mg)");
    int side = 0, l = -1;
    if (key[3] == 'N' || key[3] == 'k') l = atoi(key + 5);
    else if (sscanf(key + (key[3] == 'l' ? 10 : 10), "%d_%d", &side, &l) != 2) l = -1;
    if (l < 0 || l >= c->mg->nl || side < 0 || side > 1) return set_err(c, WB_EINVAL, "bad multigrid key '%s'", key);
    if (key[3] == 'N') *value = c->mg->Ns[l];
    else if (key[3] == 'k') *value = c->mg->Ks[l];
    else if (key[3] == 'l') *value = c->mg->lam[side][l];
    else {
      wb_status st = read_nonpos(c->mg->lev[l]);
      if (st) return st;
      *value = (double)c->mg->lev[l]->n_nonpos[side];
    }
  } else if (!strcmp(key, "k_zm")) {  // 1: the Poisson operator runs as the node-owner z-march kernel
    *value = zm_active(c) ? 1.0 : 0.0;
  } else if (!strcmp(key, "zm_zc")) {
    *value = (double)c->zm_zc;
  } else if (!strcmp(key, "k_ws")) {  // 1: ... as the warp-specialised TMA kernel (k_K2_ws)
    *value = (tma_active(c) && c->k_ws) ? 1.0 : 0.0;
  } else if (!strcmp(key, "occ_a2")) {
    int nb = 0;
    CUDA_TRY(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_A_tile<A_TX, A_TY, A_TZ, A_MINB>, 3 * A_TX * A_TY * A_TZ, Tile2<A_TX, A_TY, A_TZ>::SMEM));
    *value = nb;
  }
  else if (!strcmp(key, "prof_k_ms")) {
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    double t = 0.0;
    for (int i = 0; i < c->prof_n; ++i) {
      float ms = 0.f;
      CUDA_TRY(c, cudaEventElapsedTime(&ms, c->prof_ev[2 * i], c->prof_ev[2 * i + 1]));
      t += ms;
    }
    *value = t;
  }
  else if (!strcmp(key, "pcg_iters") || !strncmp(key, "alpha_", 6) || !strncmp(key, "beta_", 5) ||
           !strcmp(key, "last_alpha_beta") || !strcmp(key, "last_beta")) {
    // PCG scalars of the last solve (WB_DEBUG_SCALARS), from the device histories:
    // alpha_i = rz_i / pq_i, beta_i = rz_{i+1} / rz_i; 0 for iterations not run (O9)
    if (!(c->flags & WB_DEBUG_SCALARS)) return set_err(c, WB_ESTATE, "create the context with WB_DEBUG_SCALARS");
    const int n = c->last_pcg_iters;
    if (n < 0) return set_err(c, WB_ESTATE, "no PCG solve yet");
    if (!strcmp(key, "pcg_iters")) { *value = n; return WB_OK; }
    int i;
    if (!strcmp(key, "last_alpha_beta")) i = n - 1;          // alpha of the last iteration
    else if (!strcmp(key, "last_beta")) i = n - 1;
    else {
      char* end = nullptr;
      const char* num = key + (key[0] == 'a' ? 6 : 5);
      i = (int)strtol(num, &end, 10);
      if (end == num || *end) return set_err(c, WB_EINVAL, "bad iteration index in '%s'", key);
    }
    if (i < 0 || i >= n) return set_err(c, WB_EINVAL, "iteration %d outside the last solve (%d)", i, n);
    double rz[2], pq = 0.0;
    int st = 0;
    CUDA_TRY(c, cudaMemcpyAsync(rz, rz_hist(c) + i, sizeof(double) * (i + 1 < n ? 2 : 1), cudaMemcpyDeviceToHost,
                                c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(&pq, pq_hist(c) + i, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(&st, c->stop + i, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    if (i + 1 == n) {  // rz_n: the last update's partials, summed here in index order
      std::vector<double> part(c->red_blocks);
      CUDA_TRY(c, cudaMemcpyAsync(part.data(), c->rzp, sizeof(double) * c->red_blocks, cudaMemcpyDeviceToHost,
                                  c->stream));
      CUDA_TRY(c, cudaStreamSynchronize(c->stream));
      rz[1] = 0.0;
      for (double v : part) rz[1] += v;
    }
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    const bool ran = !st && pq != 0.0;
    const bool is_alpha = key[0] == 'a' || !strcmp(key, "last_alpha_beta");
    *value = !ran ? 0.0 : (is_alpha ? rz[0] / pq : rz[1] / rz[0]);
  }
  else if (!strcmp(key, "pcg_nonfinite")) {
    // failure detection: the number of non-finite control scalars (rz_i, pq_i) of
    // the last PCG solve, from the device histories (0 for a healthy solve); available in every
    // context, read on demand (one small copy, synchronises)
    const int n = c->last_pcg_iters;
    if (n < 0) return set_err(c, WB_ESTATE, "no PCG solve yet");
    std::vector<double> rz(n + 1, 0.0), pq(n + 1, 0.0);
    std::vector<int> st(n + 1, 0);
    if (n > 0) {
      CUDA_TRY(c, cudaMemcpyAsync(rz.data(), rz_hist(c), sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
      CUDA_TRY(c, cudaMemcpyAsync(pq.data(), pq_hist(c), sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
      CUDA_TRY(c, cudaMemcpyAsync(st.data(), c->stop, sizeof(int) * n, cudaMemcpyDeviceToHost, c->stream));
    }
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    int bad = 0;
    for (int i = 0; i < n; ++i) {
      if (!std::isfinite(rz[i])) ++bad;
      if (!st[i] && !std::isfinite(pq[i])) ++bad;
    }
    *value = bad;
  }
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

wb_status wb_set_option(wb_ctx* c, const char* key, double value) {
  if (!c || !key) return WB_EINVAL;
  if (!strcmp(key, "graph")) {
    if (value != 0.0 && value != 1.0) return set_err(c, WB_EINVAL, "graph must be 0 or 1");
    c->use_graph = (int)value;
  } else if (!strcmp(key, "k_variant")) {
    if (value != 0.0 && value != 1.0) return set_err(c, WB_EINVAL, "k_variant must be 0 or 1");
    c->k_var = (int)value;
    clear_graphs(c);
  } else if (!strcmp(key, "kz")) {
    if (value != 0.0 && value != 1.0) return set_err(c, WB_EINVAL, "kz must be 0 or 1");
    c->kz = (int)value;
    clear_graphs(c);
  } else if (!strcmp(key, "weights")) {  // wBFBT weights of the next wb_set_viscosity (R17)
    if (value != 0.0 && value != 1.0) return set_err(c, WB_EINVAL, "weights must be 0 or 1");
    c->weights = (int)value;
  } else if (!strcmp(key, "k4f")) {  // k = 3, 4: 1 = fused tile Poisson kernel, 0 = B^T / gather / B kernels
    if (value != 0.0 && value != 1.0) return set_err(c, WB_EINVAL, "k4f must be 0 or 1");
    c->k4f = (int)value;
    clear_graphs(c);
  } else if (!strcmp(key, "bbt_zc")) {  // k = 2 B / B^T: 0 = tile / box kernels, 2, 4, 8 = z-march, CZ layers
    if (value != -1.0 && value != 0.0 && value != 2.0 && value != 4.0 && value != 8.0)
      return set_err(c, WB_EINVAL, "bbt_zc must be -1 (auto), 0, 2, 4 or 8");
    c->bbt_zc = (int)value;
  } else if (!strcmp(key, "k4bt")) {  // k = 3, 4: 1 = B^T tile kernel, 2 = B^T and B tile kernels, 0 = neither
    if (value != 0.0 && value != 1.0 && value != 2.0) return set_err(c, WB_EINVAL, "k4bt must be 0, 1 or 2");
    c->k4bt = (int)value;
  } else if (!strcmp(key, "k4_var")) {  // tile variant of the fused k = 3, 4 Poisson kernel
    if (!(value >= 0.0 && value < K4_NV) || value != (double)(int)value)
      return set_err(c, WB_EINVAL, "k4_var must be an integer in [0, %d)", K4_NV);
    c->k4_var = (int)value;
    clear_graphs(c);
  } else if (!strcmp(key, "k2_pair")) {  // TMA Poisson kernel: paired class-(0,*) / (1,*) pencils
    if (value != 0.0 && value != 1.0) return set_err(c, WB_EINVAL, "k2_pair must be 0 or 1");
    c->k2_pair = (int)value;
    clear_graphs(c);
  } else if (!strcmp(key, "k_ws")) {
    if (value != 0.0 && value != 1.0) return set_err(c, WB_EINVAL, "k_ws must be 0 or 1");
    c->k_ws = (int)value;
    clear_graphs(c);
  } else if (!strcmp(key, "k_zm")) {  // 1: the node-owner z-march Poisson kernel where set up
    if (value != 0.0 && value != 1.0) return set_err(c, WB_EINVAL, "k_zm must be 0 or 1");
    c->use_zm = (int)value;
    clear_graphs(c);
    if (c->use_zm && c->tma_ok && !c->zm_ok && !(c->zm_ok = setup_zm(c)))
      return set_err(c, WB_ECUDA, "z-march kernel setup failed");
    if (c->use_zm && c->zm_ok && c->have_visc && !c->xz_valid && build_xz(c)) return set_err(c, WB_ECUDA, "X build");
  } else if (!strcmp(key, "zm_var")) {  // z-march kernel variant (tile shape, CTAs per SM)
    if (!(value >= 0.0 && value < wb_ctx::ZM_NV) || value != (double)(int)value)
      return set_err(c, WB_EINVAL, "zm_var must be an integer in [0, %d)", wb_ctx::ZM_NV);
    c->zm_var = (int)value;
    clear_graphs(c);
  } else if (!strcmp(key, "zm_zc")) {  // element layers per CTA of the z-march kernel
    if (!(value >= 1.0 && value <= 64.0) || value != (double)(int)value)
      return set_err(c, WB_EINVAL, "zm_zc must be an integer in [1, 64]");
    c->zm_zc = (int)value;
    clear_graphs(c);
  } else if (!strcmp(key, "tma")) {
    if (value != 0.0 && value != 1.0) return set_err(c, WB_EINVAL, "tma must be 0 or 1");
    if (c->ylay && value == 0.0)
      return set_err(c, WB_EINVAL, "this context's PCG storage is the TMA kernel's (y fastest): tma must stay 1");
    c->use_tma = (int)value;
    clear_graphs(c);
  } else if (!strcmp(key, "k_dbg")) {  // timing probe only: 0x100 / 0x200 / 0x400 skip phases
    c->k_dbg = ((int)value) & 0xff00;
    clear_graphs(c);
  } else if (!strcmp(key, "profile")) {
    if (value != 0.0 && value != 1.0) return set_err(c, WB_EINVAL, "profile must be 0 or 1");
    c->profile = (int)value;
    c->prof_n = 0;  // (re)start the record
    clear_graphs(c);
  } else
    return set_err(c, WB_EINVAL, "unknown option '%s'", key);
  return WB_OK;
}

wb_status wb_sync(wb_ctx* c) {
  if (!c) return WB_EINVAL;
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  CUDA_TRY(c, cudaGetLastError());
  return WB_OK;
}

}  // extern "C"
