/*
 * wbfbt.h -- C ABI of libwbfbt.so, the B200 (sm_100a) FP64 hot path of the
 * weighted-BFBT Stokes preconditioner of Rudi, Stadler & Ghattas,
 * "Weighted BFBT Preconditioner for Stokes Flow Problems with Highly
 * Heterogeneous Viscosity" (arXiv 1607.03936).  Citations are PAPER.md line
 * numbers of /root/reference/PAPER.md plus the section / equation label.
 *
 * Problem (eq:stokes, eq:discrete-stokes):
 * homogeneous-Dirichlet Stokes on the unit cube, uniform N^3 hexahedral mesh,
 * continuous nodal Q_k velocity (GLL nodes) x discontinuous modal P_{k-1}
 * pressure (orthonormal Legendre, total degree), viscosity mu given at the
 * (k+1)^3 Gauss-Legendre points of every element.
 *
 * Layouts (all FP64 arrays are contiguous, caller-owned DEVICE pointers unless
 * a function name ends in _host):
 *   element  e = ex + N*(ey + N*ez)
 *   node     g = gx + (kN+1)*(gy + (kN+1)*gz),   n_nodes = (kN+1)^3
 *   velocity u[c*n_nodes + g], c in {0,1,2}       n_v = 3*n_nodes  (SoA)
 *   pressure p[e*n_m + m], n_m = C(k+2,3), modes ordered
 *            for d in 0..k-1: for m3 in 0..d: for m2 in 0..d-m3: m1 = d-m2-m3
 *            (mode (m1,m2,m3) = Lhat_m1(xi1) Lhat_m2(xi2) Lhat_m3(xi3))
 *   mu_q     mu_q[e*n_q + q], q = qx + (k+1)*(qy + (k+1)*qz), n_q = (k+1)^3
 *
 * Dirichlet elimination (R6): boundary entries of every velocity
 * INPUT are ignored; boundary entries of every velocity OUTPUT are written as
 * exactly 0.0.  The Poisson solves and wBFBT project inputs and outputs off the
 * constant pressure (Neumann null space).
 *
 * Errors: every call returns a wb_status (0 = WB_OK, < 0 error); the message of
 * the last error is wb_last_error(ctx).  Applies are asynchronous on the
 * context's stream: device faults surface at wb_sync() or a later call.
 * Setup calls (wb_create, wb_set_viscosity) synchronise the stream.
 *
 * Concurrency: one context = one stream + its own workspace.  Calls on one
 * context must be externally serialised; use one context per stream to run
 * concurrently.  Aliasing: an output may not overlap any input (WB_EALIAS).
 *
 * Determinism: no floating-point atomics anywhere; every reduction has a fixed
 * order, so results are bitwise reproducible run to run on the same GPU.
 */
#ifndef WBFBT_H
#define WBFBT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct wb_ctx wb_ctx; /* opaque, library-owned */
typedef int wb_status;

#define WB_OK 0
#define WB_EINVAL (-1)       /* bad N / k / iters / null pointer / side          */
#define WB_ENONPOS_MU (-2)   /* some mu_q <= 0 or non-finite                     */
#define WB_ENONPOS_LUMP (-3) /* nonpositive C_w / D_w entry under WB_STRICT_LUMP */
#define WB_ECUDA (-4)        /* CUDA runtime error (message in wb_last_error)    */
#define WB_ENOMEM (-5)       /* device allocation failed                         */
#define WB_EALIAS (-6)       /* an output overlaps an input                      */
#define WB_ESTATE (-7)       /* operator needs wb_set_viscosity first            */

/* flags for wb_create */
#define WB_STRICT_LUMP 1u  /* nonpositive interior C_w/D_w entry -> WB_ENONPOS_LUMP */
#define WB_DEBUG_NOMASK 2u /* tests only: A, B, B^T skip the Dirichlet mask        */
#define WB_DEBUG_SCALARS 4u /* wb_query may read the last PCG solve's alpha / beta */

/* Library version string. */
const char* wb_version(void);

/* Create a context for the N^3 mesh with Q_k x P_{k-1}^disc, k in {2,3,4},
 * N >= 1.  `stream` is a cudaStream_t (NULL = legacy default stream); all
 * work of the context is enqueued on it.  Allocates the workspace on the
 * current CUDA device.  Synchronous. */
wb_status wb_create(wb_ctx** out, int N, int k, unsigned flags, void* stream);
void wb_destroy(wb_ctx* ctx);
/* Re-target the context to another stream (e.g. torch's current stream). */
wb_status wb_set_stream(wb_ctx* ctx, void* stream);
const char* wb_last_error(const wb_ctx* ctx);

/* Structured counts (Table 3 counts boundary dofs):
 * n_el = N^3, n_nodes = (kN+1)^3, n_v = 3 n_nodes, n_p = C(k+2,3) N^3,
 * n_q = (k+1)^3.  Any output pointer may be NULL. */
wb_status wb_sizes(const wb_ctx* ctx, int64_t* n_el, int64_t* n_nodes, int64_t* n_v,
                   int64_t* n_p, int64_t* n_q);

/* Row a1 -- dof map and boundary mask.
 * map[e*n_q + a] = global node of local node a = ax + (k+1)(ay + (k+1)az) of
 * element e (device int64, n_el*n_q).  mask[c*n_nodes + g] = 1 iff velocity
 * dof (c,g) is a Dirichlet (boundary) dof (device uint8, n_v). */
wb_status wb_get_dofmap(wb_ctx* ctx, int64_t* map);
wb_status wb_get_boundary_mask(wb_ctx* ctx, uint8_t* mask);

/* Rows a3, a4 -- setup from mu at quadrature points (device, n_el*n_q).
 *   C_w = lumped M_u(w_l), D_w = lumped M_u(w_r), w_l = a_l(e) sqrt(mu),
 *   w_r = a_r(e) sqrt(mu)  (eq:lumping PAPER.md:310-323, eq:wbfbt
 *   PAPER.md:436-454, eq:bdramp PAPER.md:2219-2251: a_l(e) = a_l on elements
 *   touching the boundary, 1 elsewhere; a_l, a_r >= 1).
 *   Jacobi diagonals of K_l = B C_w^-1 B^T and K_r = B D_w^-1 B^T.
 * Also stores mu * w_q * detJ * (2/h)^2 for A.  Fails with WB_ENONPOS_MU if any
 * mu_q <= 0 or non-finite.  Nonpositive interior lumped entries are counted
 * (wb_query "n_nonpos_Cw"/"n_nonpos_Dw") and are an error only with
 * WB_STRICT_LUMP.  mu_q may be freed once the call returns.  Synchronous. */
wb_status wb_set_viscosity(wb_ctx* ctx, const double* mu_q, double a_l, double a_r);

/* Row a5 -- y = M A(mu) M u, A = weak form of -div[mu(grad u + grad u^T)]
 * (eq:stokes PAPER.md:148-151; A_mu PAPER.md:986-990), Gauss (k+1)^3
 * quadrature, sum-factorised.  u, y: n_v. */
wb_status wb_apply_A(wb_ctx* ctx, const double* u, double* y);
/* Row a6 -- p = B M u, B u := -div u. u: n_v, p: n_p. */
wb_status wb_apply_B(wb_ctx* ctx, const double* u, double* p);
/* Row a7 -- y = M B^T p (gradient).  p: n_p, y: n_v. */
wb_status wb_apply_BT(wb_ctx* ctx, const double* p, double* y);
/* Row a8 -- q = K p, K = B X^-1 B^T with X = C_w (side 0, "l") or D_w (side 1,
 * "r").  No projection.  p, q: n_p. */
wb_status wb_apply_K(wb_ctx* ctx, int side, const double* p, double* q);
/* Row a9 -- x = P PCG(K_side, P b) with exactly `iters` Jacobi-PCG iterations
 * (x0 = 0, M = diag K, no tolerance; stands in for the paper's HMG V-cycle,
 * PAPER.md:2503-2529; recurrence in DESIGN.md Sec. 4).  b, x: n_p. */
wb_status wb_poisson_pcg(wb_ctx* ctx, int side, const double* b, double* x, int iters);
/* x = P Cheb(K_side, P b): Chebyshev-accelerated point-Jacobi, the
 * paper's smoother as a fixed-iteration inner solve.  Saad (2003)
 * Alg. 12.1 on Minv K_side (Minv = the Jacobi pseudo-inverse of wb_poisson_pcg), x0 = 0,
 * exactly `iters` steps, [lmin, lmax] the caller's interval of the spectrum of
 * Minv K_side (reading R16).  b, x: device, element-major n_p; b is not
 * modified.  WB_EINVAL for side not 0/1, iters < 0, null pointers or unless
 * 0 < lmin < lmax < inf; WB_EALIAS if b and x overlap; WB_ESTATE before
 * wb_set_viscosity.  Asynchronous on the context stream. */
wb_status wb_poisson_cheb(wb_ctx* ctx, int side, const double* b, double* x, int iters, double lmin, double lmax);
/* *lmax = power-iteration estimate of the largest |eigenvalue| of Minv K_side (R16):
 * v = v0/||v0||, then `iters` times w = Minv (K_side v), lambda = ||w||, v = w/lambda;
 * *lmax = the last lambda (0 if iters = 0 or an iterate vanishes).  v0: device,
 * element-major n_p, not modified (the start vector is an input, so runs are
 * reproducible).  lmax: host.  Synchronises the context stream.  WB_EINVAL for
 * side not 0/1, iters < 0 or null pointers; WB_ESTATE before wb_set_viscosity. */
wb_status wb_poisson_eigmax(wb_ctx* ctx, int side, const double* v0, int iters, double* lmax);
/* SURVEY 8(f) #2 "as the inner Poisson solve": from now on wBFBT (wb_apply_wbfbt,
 * wb_hotpath[_host], wb_stokes_fgmres) solves its two Poisson problems with
 * wb_poisson_cheb on [lmin_l, lmax_l] (K_l, side 0) and [lmin_r, lmax_r] (K_r, side 1),
 * `iters` steps each, instead of PCG; wBFBT is then a fixed linear map (R16).  All four 0:
 * back to PCG (the default).  WB_EINVAL unless each 0 < lmin < lmax < inf.  wb_query
 * "inner" reads the choice. */
wb_status wb_set_inner_cheb(wb_ctx* ctx, double lmin_l, double lmax_l, double lmin_r, double lmax_r);

/* ---- Schur-complement variants beside wBFBT, on the same kernels.
 * wb_set_schur selects the S~^-1 of the Stokes preconditioner (wb_stokes_fgmres):
 * 0 = wBFBT (default, eq:wbfbt); 1 = diag(A)-BFBT (C = D = diag(A));
 * 2 = M_p(1/mu)^-1, applied exactly per element (reading R21: the
 * eq:lumping diagonal degenerates in the orthonormal modal basis R2).  Kind 2 builds its
 * element blocks in wb_set_viscosity, so select it before that call.  WB_EINVAL otherwise. */
wb_status wb_set_schur(wb_ctx* ctx, int kind);
/* z = (B X B^T)^-1 (B X A X B^T) (B X B^T)^-1 r with X = mask / diag(A) (per DOF), both
 * Poisson inverses by Jacobi-PCG (O9, `iters` iterations, pseudo-inverse diagonal R11), input
 * and output projected (R10).  r, z: device, element-major n_p.  Asynchronous.  WB_ESTATE
 * before wb_set_viscosity; WB_EINVAL; WB_EALIAS. */
wb_status wb_apply_dabfbt(wb_ctx* ctx, const double* r, double* z, int iters);
/* z = M_p(1/mu)^-1 r, M_p[i][j] = int q_i q_j / mu per element (Gauss quadrature of R3; the
 * blocks are inverted by Cholesky in wb_set_viscosity).  WB_ESTATE unless kind 2 was selected
 * before wb_set_viscosity. */
wb_status wb_apply_mpinv(wb_ctx* ctx, const double* r, double* z);

/* Load vector of a body force (the multi-sinker forcing
 * f = (0, 0, beta (chi_n - 1)), beta = 10, the right-hand side of
 * eq:discrete-stokes): F[(c, g)] = sum_e sum_q w_q detJ f_c(x_q) phi_a(xi_q), Dirichlet rows
 * 0 (R6).  fq: device, 3 x n_el x n_q, component-major, per element its Gauss points
 * (q x fastest, the layout of mu_q); F: device, n_v (SoA).  Asynchronous; does not need
 * wb_set_viscosity.  WB_EINVAL (null), WB_EALIAS. */
wb_status wb_load_vector(wb_ctx* ctx, const double* fq, double* F);

/* ---- Geometric pressure multigrid for K_w (second half; PAPER.md:2468-2546,
 * Sec. "Parallel hybrid spectral-geometric-algebraic multigrid (HMG) for wBFBT"; reading R20
 * of DESIGN.md).  k = 2: levels N, N/2, ... while N is even and > 1 (uniform element
 * bisection); k = 4: first the spectral level Q4 x P3disc -> Q2 x P1disc on
 * the same mesh (P1disc modes are the first four P3disc modes, the Q2 GLL
 * nodes are Q4 GLL nodes), then the k = 2 levels; on every level the operator is re-discretised
 * as K_l = B_l X_l B_l^T with X_l = mask / C_l, the coarse lumped masses
 * C_l[G] = C_{l-1}[iota(G)] M_l[G] / M_{l-1}[iota(G)] (the weight density injected at the
 * coincident node; M = unweighted lumped mass); transfers are the exact P1disc embedding and
 * its transpose; smoother: nu steps of Chebyshev-accelerated Jacobi on
 * [0.1, 1.1] x a 20-step power-iteration estimate (splitmix64 start vector); coarsest level:
 * Jacobi-PCG with min(n_p, 256) iterations. */
/* Builds the hierarchy of both sides from the current C_w, D_w (after wb_set_viscosity; a
 * later wb_set_viscosity discards it).  nu in [1, 16] (the paper: 3).  mu_q (device, the
 * n_el x n_q viscosity given to wb_set_viscosity, or NULL): when given, the velocity
 * hierarchy of A is built too (R22: mu coarsened level by level; A
 * re-discretised; Q2 nodal interpolation and its transpose as transfers; the same smoother
 * on A, R18).  Allocates one internal context per coarse level and synchronises the stream.
 * For k = 4 the velocity hierarchy starts with the spectral level too (Q2-in-Q4 nodal transfers,
 * mu grouped onto the Q2 Gauss points).  WB_EINVAL for k not 2 or 4 or nu out of range,
 * WB_ESTATE before wb_set_viscosity, WB_ENOMEM.  Queries "mg_N_<l>", "mg_k_<l>" give each
 * level's mesh and order. */
wb_status wb_setup_mg(wb_ctx* ctx, int nu, const double* mu_q);
/* x = V(b), one velocity V-cycle on M A M (b, x: device SoA n_v; boundary entries of b are
 * ignored, of x written 0).  WB_ESTATE without a velocity hierarchy. */
wb_status wb_velocity_vcycle(wb_ctx* ctx, const double* b, double* x);
/* From now on the Stokes preconditioner's At^-1 (eq:precond-stokes) is `cycles` stationary
 * velocity V-cycles from x0 = 0 (the paper's choice: an HMG V-cycle)
 * instead of the Chebyshev smoother; 0: back to the smoother.  WB_ESTATE without a
 * velocity hierarchy. */
wb_status wb_set_velocity_mg(wb_ctx* ctx, int cycles);
/* x = V(b), one V-cycle on K_side (side 0 = l, 1 = r).  b, x: device, element-major n_p,
 * caller-owned; b should be projected (R10).  Asynchronous.  WB_ESTATE without a hierarchy,
 * WB_EINVAL, WB_EALIAS. */
wb_status wb_mg_vcycle(wb_ctx* ctx, int side, const double* b, double* x);
/* x = P MGPCG(K_side, P b): the O9 recurrence with M^-1 = one V-cycle, exactly `iters`
 * iterations (scalars on the device), input and output projected (R10).  Errors as
 * wb_mg_vcycle; iters >= 0. */
wb_status wb_poisson_mgcg(wb_ctx* ctx, int side, const double* b, double* x, int iters);
/* From now on wBFBT solves its two Poisson problems by wb_poisson_mgcg with `iters`
 * iterations (its own `iters` argument is then unused); 0: back to the previous inner solve.
 * WB_ESTATE without a hierarchy (iters > 0). */
wb_status wb_set_inner_mg(wb_ctx* ctx, int iters);
/* The level-`level` lumped masses C_l, D_l (device, n_nodes of that level's (2 N_l + 1)^3
 * grid; either may be NULL).  Synchronises.  WB_EINVAL for a bad level. */
wb_status wb_mg_get_lumped(wb_ctx* ctx, int level, double* Cw, double* Dw);
/* diag(M A M) (reading R18): dA[c * n_nodes + g] = sum over the elements holding node g of
 * the element matrix diagonal, sum_q mu w_q detJ (2/h)^2 (|grad_xi phi_a|^2 + (d_xi_c phi_a)^2);
 * Dirichlet dofs 0.  dA: device, n_v (SoA).  WB_EINVAL for a null pointer; WB_ESTATE
 * before wb_set_viscosity; WB_ENOMEM if the k = 2 element buffer cannot be allocated.
 * Asynchronous on the context stream. */
wb_status wb_get_diagA(wb_ctx* ctx, double* dA);
/* x = Cheb(M A M, M b): the Chebyshev-accelerated point-Jacobi smoother on the viscous
 * block (the paper's smoother; an approximate A^-1 for SURVEY 8(f) #1),
 * Saad Alg. 12.1 as wb_poisson_cheb with the Jacobi inverse mask / diag(A), x0 = 0,
 * exactly `iters` steps on [lmin, lmax] (R16, R18).  b, x: device, n_v; b is not modified.
 * Errors as wb_poisson_cheb.  Asynchronous on the context stream. */
wb_status wb_velocity_cheb(wb_ctx* ctx, const double* b, double* x, int iters, double lmin, double lmax);
/* *lmax = power-iteration estimate of the largest |eigenvalue| of (mask / diag A) M A M from
 * the device start vector v0 (n_v, not modified), as wb_poisson_eigmax.  Synchronises. */
wb_status wb_velocity_eigmax(wb_ctx* ctx, const double* v0, int iters, double* lmax);
/* the Stokes solve [A B^T; B 0] (u; p) = (f; g) (eq:discrete-stokes,
 * PAPER.md:187-204; A, B^T masked, B on masked u) by flexible GMRES with the right
 * preconditioner of eq:precond-stokes: P^-1 (a; b) = (At^-1 (a - B^T y); y),
 * y = -wBFBT(b) with `pcg_iters` PCG iterations per inner Poisson solve, At^-1 =
 * wb_velocity_cheb with `smooth_iters` steps on [lmin, lmax] (reading R19).  Restarted every
 * `restart` iterations, x0 = 0, stops when the residual estimate is <= rtol ||(M f; g)|| or
 * after max_iters iterations; p is projected off the constants (R10).  f, u: device n_v;
 * g, p: device n_p (element-major).  *iters (host, may be NULL): iterations run; *relres (host,
 * may be NULL): ||b - K x|| / ||b|| of the returned solution.  Memory: (2 restart + 4)(n_v + n_p)
 * doubles, kept for later calls.  WB_EINVAL for bad arguments or interval, WB_EALIAS for
 * overlapping outputs, WB_ESTATE before wb_set_viscosity, WB_ENOMEM.  Synchronises. */
wb_status wb_stokes_fgmres(wb_ctx* ctx, const double* f, const double* g, double* u, double* p, int restart,
                           int max_iters, double rtol, int pcg_iters, int smooth_iters, double lmin, double lmax,
                           int* iters, double* relres);
/* Row a10 -- z = S~^-1_wBFBT r (eq:wbfbt PAPER.md:436-454), applied right to
 * left:  y = P PCG(K_r, P r); v = D_w^-1 B^T y; v = A v; v = C_w^-1 v;
 * s = P B v; z = P PCG(K_l, s).  r, z: n_p. */
wb_status wb_apply_wbfbt(wb_ctx* ctx, const double* r, double* z, int iters);

/* One full hot-path step (rows a3-a10 once): set_viscosity(mu_q, a_l, a_r),
 * yA = A u, pB = B u, yBT = B^T p, z = wBFBT(p).  Device pointers.
 * Synchronous (setup reports status). */
wb_status wb_hotpath(wb_ctx* ctx, const double* mu_q, double a_l, double a_r, const double* u,
                     const double* p, int iters, double* yA, double* pB, double* yBT, double* z);
/* The same step with HOST buffers (pinned host memory gives asynchronous
 * copies): mu_q is copied on the context stream, p and u on a library-owned copy
 * stream that overlaps the setup and wBFBT's right Poisson solve; the standalone
 * A, B, B^T run between the two wBFBT solves and yA, pB, yBT travel back during
 * the left one; z last.  Same results as wb_hotpath.  The staging buffers
 * (n_el n_q + 3 n_v + 3 n_p doubles) are allocated on first use.  Synchronous. */
wb_status wb_hotpath_host(wb_ctx* ctx, const double* mu_q, double a_l, double a_r,
                          const double* u, const double* p, int iters, double* yA, double* pB,
                          double* yBT, double* z);

/* ---- z-slab domain decomposition (the element-partition domain
 * decomposition of PAPER.md:2480-2487; reading R24).  One context per rank (one process per
 * GPU).  Rank r of R owns the r-th of R cubes of N^3 elements stacked along z: the global mesh
 * has N x N x (R N) elements of side h = 1/N on [0,1]^2 x [0,R] (global element
 * e = ex + N (ey + N (r N + ez))), and neighbouring ranks share (replicate) the node plane
 * between them.  Every vector argument of the calls below is the rank's LOCAL part in the cube
 * layouts of this header: velocity vectors carry both shared planes, and a velocity OUTPUT
 * holds the full (summed) value on them, identical bit for bit on both owners; pressure vectors
 * are element-local and never shared.  The Dirichlet boundary is the GLOBAL box boundary: the
 * shared planes are interior except on their x / y rim, and the boundary amplification a_l, a_r
 * (eq:bdramp) applies to elements on the global boundary only.
 *
 * On a slab context the calls wb_set_viscosity, wb_apply_A, wb_apply_B, wb_apply_BT,
 * wb_apply_K, wb_poisson_pcg, wb_apply_wbfbt, wb_hotpath (device pointers), wb_get_lumped,
 * wb_get_jacobi, wb_get_boundary_mask (the global mask), wb_sizes (local sizes), wb_sync and
 * wb_query compute the GLOBAL operators; the setup, apply and solve calls must be entered by all
 * R ranks together (they are collective; a rank that fails alone, e.g. WB_ENONPOS_MU, leaves its
 * neighbours waiting in the exchange, so validate inputs collectively).  "n_nonpos_Cw" /
 * "n_nonpos_Dw" count this rank's nodes, shared-plane nodes on both of their owners.  Per
 * operator apply there is one exchange: the partial nodal sums on the shared planes
 * (3 (kN+1)^2 doubles per plane; C_w, D_w once per wb_set_viscosity), and every inner product,
 * the projection mean and max|diag K| is one all-reduce of 1 double.  K_w runs unfused
 * (B^T, plane sum, B) and the PCG is the O9 recurrence with device scalars; the single-GPU
 * fused kernels and CUDA graphs are not used.  Every other call returns WB_ESTATE.
 *
 * Communication is the caller's (torch.distributed over NCCL in the Python binding): the two
 * callbacks act on buffers the caller owns and registers here.
 *   send_lo, recv_lo, send_hi, recv_hi: device, `cap` doubles each, cap >= 3 (kN+1)^2;
 *   scal: device, >= 8 doubles.
 *   exchange(user, n): send send_lo[0..n) to rank-1 and send_hi[0..n) to rank+1; receive
 *     rank-1's send_hi into recv_lo and rank+1's send_lo into recv_hi (rank 0 has no lower,
 *     rank R-1 no upper neighbour: skip those).  The library has enqueued the packing on the
 *     context's stream before the call and enqueues the unpacking after it, so the transfer
 *     must be ordered on that stream (NCCL on the same stream) or be complete on return after
 *     synchronising it.
 *   allreduce(user, offset, n, op): reduce scal[offset..offset+n) over all ranks in place, the
 *     same bits on every rank; op 0 = sum, 1 = max.  Same stream rule.
 *   Both return 0 on success; anything else aborts the call with WB_ECUDA.
 * wb_slab_create: rank in [0, nranks), nranks >= 1 (nranks = 1 is the plain cube through the
 * slab code path), other arguments as wb_create; WB_DEBUG_NOMASK is refused.  Errors as
 * wb_create. */
typedef struct wb_slab_comm {
  void* user;
  int (*exchange)(void* user, int64_t n);
  int (*allreduce)(void* user, int offset, int n, int op);
  double *send_lo, *recv_lo, *send_hi, *recv_hi;
  int64_t cap;
  double* scal;
} wb_slab_comm;
wb_status wb_slab_create(wb_ctx** out, int N, int k, int rank, int nranks, unsigned flags, void* stream);
/* Registers the communicator (copied).  WB_EINVAL for a null callback / buffer or cap too small,
 * WB_ESTATE on a context that is not a slab context. */
wb_status wb_slab_set_comm(wb_ctx* ctx, const wb_slab_comm* comm);

/* One PCG iteration (DESIGN.md Sec. 4 recurrence) from a supplied state, in
 * place: x, r, p device n_p; *rz host in/out.  Test entry for one-step
 * parity. */
wb_status wb_debug_pcg_step(wb_ctx* ctx, int side, double* x, double* r, double* p, double* rz);

/* Copies of the setup results (device pointers; any may be NULL):
 * Cw, Dw, Cinv, Dinv: n_nodes; diagKl, diagKr: n_p. */
wb_status wb_get_lumped(wb_ctx* ctx, double* Cw, double* Dw, double* Cinv, double* Dinv);
wb_status wb_get_jacobi(wb_ctx* ctx, double* diagKl, double* diagKr);

/* Scalar queries: "n_nonpos_Cw", "n_nonpos_Dw", "n_el", "n_p", "n_v",
 * "kernel_launches" (launches since create), "last_pcg_stop_iter",
 * with WB_DEBUG_SCALARS: "pcg_iters" (iterations of the last PCG solve, n),
 * "alpha_<i>" = rz_i / pq_i and "beta_<i>" = rz_{i+1} / rz_i of its iteration i
 * (0 <= i < n; 0 for iterations not run, as the oracle's O9 records them),
 * "last_alpha_beta" = alpha_{n-1}, "last_beta" = beta_{n-1} (WB_ESTATE without the
 * flag or before a solve, WB_EINVAL for i outside [0, n)), "kz" (1 if the PCG
 * update stores z = Minv r for the TMA Poisson kernel), "k_tma" (1 if
 * the k = 2 Poisson operator runs as the TMA kernel for this mesh), "k_ws" (1 if
 * it runs as the warp-specialised TMA kernel), "weights" (the option below),
 * "pcg_nonfinite" (failure detection: the number of non-finite rz_i / pq_i control scalars of
 * the last PCG solve, 0 when healthy; WB_ESTATE before a solve), "k_zm" / "zm_zc" (the opt-in
 * z-march Poisson kernel), "mg_levels", "mg_N_<l>", "mg_lambda_<side>_<l>",
 * "mg_nonpos_<side>_<l>", "mg_vlambda_<l>", "mg_k_<l>" (the multigrid hierarchy of wb_setup_mg),
 * "inner" (wBFBT's inner solve: 0 PCG, 1 Chebyshev), "prof_k_ms" / "prof_k_count" (option
 * "profile"), "occ_k2" / "occ_a2" (resident CTAs per SM of the k = 2 Poisson / A kernels), and, in
 * builds with -DWB_KPROF only, the phase-timer probes "kprof_<i>", "aprof_<i>", "ktl_<cta>_<i>". */
wb_status wb_query(wb_ctx* ctx, const char* key, double* value);
/* Method option (changes the results): "weights", the wBFBT weights the next
 * wb_set_viscosity lumps: 0 = w_l = w_r = sqrt(mu), eq:wbfbt, the default; 1 = the
 * viscosity-gradient weights (mu^2 + |grad mu|^2)^(1/4) of rmk:wbfbt-visc-grad,
 * PAPER.md:2132-2150, with grad mu that of each element's Gauss-point interpolant
 * (reading R17); A keeps mu.
 * Tuning knobs (results are identical up to rounding for every setting):
 * "kz" (k = 2 TMA Poisson kernel: 1 = the PCG update stores z = Minv r and the
 * kernel loads it as one box; 0 = it loads r and Minv, the default),
 * "k2_pair" (k = 2 TMA Poisson kernel: 1 = each class-(0, *) pencil thread also computes the
 * class-(1, *) pencil of the same (y, z) from its loads), "k_ws" (k = 2 TMA Poisson kernel: 1 = warp-specialised, producer warps build
 * the next tile's direction box while the consumer warps apply B^T X^-1 B),
 * "k4f" (k = 3, 4: 1 = the fused tile Poisson kernel of k4_fused.cuh, K_w = B X B^T by
 * assembled 1-D contractions with the PCG direction update folded in, default; 0 = the
 * B^T element kernel + node gather + B kernel), "k4_var" (its tile variant, 0..8; 1 =
 * 4 x 4 x 2 tiles with TMA staging, the default; DESIGN.md Sec. 7 lists the others),
 * "k4bt" (k = 3, 4 standalone B^T / B: 1 = B^T by the tile kernel, default; 2 = B too;
 * 0 = the element kernels), "bbt_zc" (k = 2 standalone B / B^T: -1 = auto, the z-marching column
 * kernels with 4 element layers per chunk on meshes with N >= 48, else the tile / box kernels,
 * default; 0 = always the tile / box kernels; 2, 4, 8 = the column kernels with that chunk), "k_zm" / "zm_var" / "zm_zc" (k = 2: the opt-in z-march Poisson
 * kernel, its variant and z-chunk length), "tma" (k = 2: 1 = the TMA Poisson kernel where the
 * context's storage allows it, default), "k_variant" (k = 2 pointer Poisson kernel: 1 or 2 CTAs
 * per SM), "k_dbg" (timing probe bits that skip kernel phases: results invalid, tools only),
 * "graph" (1 = replay the PCG iteration loop as a CUDA graph, default; 0 =
 * plain launches), "profile" (1 = plain launches with a CUDA-event pair around
 * every Poisson-operator launch; wb_query "prof_k_ms" / "prof_k_count" read
 * the total time / count since the option was set).  WB_EINVAL for an
 * unknown key or value. */
wb_status wb_set_option(wb_ctx* ctx, const char* key, double value);
/* Synchronise the context stream; surfaces asynchronous CUDA errors. */
wb_status wb_sync(wb_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* WBFBT_H */
