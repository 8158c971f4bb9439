/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the wBFBT hot path
 * of Rudi, Stadler & Ghattas, "Weighted BFBT preconditioner for Stokes flow
 * problems with highly heterogeneous viscosity" (arXiv 1607.03936).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_1607_03936_b200/) never links or calls it, and the
 * two share no code, headers or tables: this file derives its 1-D tables by
 * Newton iteration in long double; the CUDA path uses closed-form constants.
 *
 * Everything is IEEE binary64 (the paper fixes no precision), compiled with
 * -O2 -fno-fast-math -ffp-contract=off.  OpenMP (if enabled) only computes
 * element-local quantities into a buffer; every global sum (scatter-add,
 * dot product) runs serially in a fixed order, so results are bit-identical
 * for any thread count.
 *
 * Citations: PAPER.md line numbers (+ section / equation label).
 *   eq:stokes          PAPER.md:145-162   -div[mu(grad u + grad u^T)] + grad p = f, -div u = 0, u=0 on boundary
 *   eq:discrete-stokes PAPER.md:187-204   [A B^T; B 0]
 *   Q_k x P_{k-1}^disc PAPER.md:205-209   continuous nodal velocity, discontinuous modal pressure
 *   B u := -div u
 *   eq:lumping         PAPER.md:310-323   lumping with the coefficient vector of the constant 1
 *   eq:wbfbt           PAPER.md:438-454   C_w = M~_u(w_l), D_w = M~_u(w_r), w = sqrt(mu)
 *   eq:bdramp          PAPER.md:2219-2251 boundary amplification a_l, a_r on elements touching the boundary
 *   K_w (Neumann)
 *   mu at quad points
 *   element partition  PAPER.md:2480-2487 the box mesh N x N x Nz (or_create_box) is the global
 *                      mesh of the z-slab decomposition (R24); pinned in tests/test_oracle_box.py
 * Readings of silences (R1..R24) are listed in DESIGN.md Sec. 3; the ones used
 * here are cited inline.
 *
 * Parity pins: every function below is pinned by tests/test_oracle_*.py
 * against closed forms, paper tables, invariants or brute force -- except the
 * fixed-iteration PCG / wBFBT VALUES, whose only pins are the converged
 * limit, scale invariance and one-step agreement: "parity unpinned" beyond
 * those.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_MAXN1 9 /* up to k = 8 */

typedef struct {
  int N, Nz, k, n1, nq, nm;      /* N x N x Nz elements of side h = 1/N (Nz = N: the unit cube) */
  int64_t n_el, n_nodes, n_v, n_p;
  double h, detJ;                  /* h = 1/N, detJ = (h/2)^3 */
  double xn[OR_MAXN1];             /* GLL nodes (R1) */
  double xg[OR_MAXN1], wg[OR_MAXN1]; /* Gauss-Legendre points / weights (R3) */
  double phi[OR_MAXN1][OR_MAXN1];  /* phi[a][i]  = phi_a(xg_i)   */
  double dphi[OR_MAXN1][OR_MAXN1]; /* dphi[a][i] = phi_a'(xg_i)  */
  double leg[OR_MAXN1][OR_MAXN1];  /* leg[m][i]  = Lhat_m(xg_i)  */
  int mode[200][3];                /* pressure mode exponents (R2) */
  /* tabulated 3-D quantities on the reference element */
  double* gphi;  /* [a][q][j] = d/dxi_j phi_a(xi_q)  (reference gradient) */
  double* vphi;  /* [a][q]    = phi_a(xi_q) */
  double* wq;    /* [q]       = w_qx w_qy w_qz */
  double* Be;    /* [m][c*nq + a] element divergence matrix (constant on the uniform mesh) */
  double* work;  /* element-local scratch for chunked parallel loops */
  int64_t chunk;
} or_ctx;

/* ---------------------------------------------------------------- 1-D tables
 * Legendre P_n and P_n' by the three-term recurrence, long double.           */
static void legendre(int n, long double x, long double* P, long double* dP) {
  long double p0 = 1.0L, p1 = x;
  if (n == 0) { *P = 1.0L; *dP = 0.0L; return; }
  for (int j = 2; j <= n; ++j) {
    long double p2 = ((2.0L * j - 1.0L) * x * p1 - (j - 1.0L) * p0) / j;
    p0 = p1; p1 = p2;
  }
  *P = p1;
  /* P_n' = n (x P_n - P_{n-1}) / (x^2 - 1), valid off +-1 */
  *dP = n * (x * p1 - p0) / (x * x - 1.0L);
}

static void sort_ld(long double* v, int n) {
  for (int i = 1; i < n; ++i)
    for (int j = i; j > 0 && v[j] < v[j - 1]; --j) { long double t = v[j]; v[j] = v[j - 1]; v[j - 1] = t; }
}

/* Gauss-Legendre: roots of P_n, weights 2 / ((1-x^2) P_n'(x)^2). */
static void gauss_legendre(int n, double* x, double* w) {
  long double r[OR_MAXN1], wl[OR_MAXN1];
  for (int i = 0; i < n; ++i) {
    long double z = cosl(3.14159265358979323846264338327950288L * (i + 0.75L) / (n + 0.5L));
    for (int it = 0; it < 100; ++it) {
      long double P, dP; legendre(n, z, &P, &dP);
      long double dz = P / dP; z -= dz;
      if (fabsl(dz) < 1e-30L) break;
    }
    r[i] = z;
  }
  sort_ld(r, n);
  for (int i = 0; i < n; ++i) {
    long double P, dP; legendre(n, r[i], &P, &dP);
    wl[i] = 2.0L / ((1.0L - r[i] * r[i]) * dP * dP);
    x[i] = (double)r[i]; w[i] = (double)wl[i];
  }
}

/* GLL nodes of degree k: -1, roots of P_k', +1.  Newton on P_k' with
 * P_k'' = (2x P_k' - k(k+1) P_k) / (1 - x^2) (Legendre ODE).                 */
static void gll_nodes(int k, double* x) {
  long double r[OR_MAXN1];
  r[0] = -1.0L; r[k] = 1.0L;
  for (int i = 1; i < k; ++i) {
    long double z = -cosl(3.14159265358979323846264338327950288L * i / k);
    for (int it = 0; it < 100; ++it) {
      long double P, dP; legendre(k, z, &P, &dP);
      long double d2P = (2.0L * z * dP - k * (k + 1.0L) * P) / (1.0L - z * z);
      long double dz = dP / d2P; z -= dz;
      if (fabsl(dz) < 1e-30L) break;
    }
    r[i] = z;
  }
  sort_ld(r, k + 1);
  for (int i = 0; i <= k; ++i) x[i] = (double)r[i];
}

/* Lagrange basis on nodes xn (product formula), value and derivative at t. */
static long double lagrange(const double* xn, int n1, int a, long double t) {
  long double v = 1.0L;
  for (int b = 0; b < n1; ++b) if (b != a) v *= (t - xn[b]) / ((long double)xn[a] - xn[b]);
  return v;
}
static long double dlagrange(const double* xn, int n1, int a, long double t) {
  long double s = 0.0L;
  for (int j = 0; j < n1; ++j) {
    if (j == a) continue;
    long double v = 1.0L / ((long double)xn[a] - xn[j]);
    for (int b = 0; b < n1; ++b) if (b != a && b != j) v *= (t - xn[b]) / ((long double)xn[a] - xn[b]);
    s += v;
  }
  return s;
}

/* ---------------------------------------------------------------- context */
static int or_nmodes(int k) { return k * (k + 1) * (k + 2) / 6; } /* C(k+2,3) = dim P_{k-1} in 3-D */

/* Box mesh: N x N x Nz cubic elements of side h = 1/N on [0,1]^2 x [0, Nz/N].  Nz = N is the
 * paper's unit cube; Nz != N is the union of z-stacked cubes that the
 * element-partition domain decomposition of PAPER.md:2480-2487 distributes (SURVEY 8(e),
 * DESIGN.md reading R24).  Every formula below is per element and does not see Nz. */
or_ctx* or_create_box(int N, int Nz, int k) {
  if (N < 1 || Nz < 1 || k < 1 || k + 1 > OR_MAXN1) return NULL;
  or_ctx* c = (or_ctx*)calloc(1, sizeof(or_ctx));
  c->N = N; c->Nz = Nz; c->k = k; c->n1 = k + 1; c->nq = c->n1 * c->n1 * c->n1; c->nm = or_nmodes(k);
  c->n_el = (int64_t)N * N * Nz;
  int64_t nn1 = (int64_t)k * N + 1;
  c->n_nodes = nn1 * nn1 * ((int64_t)k * Nz + 1); c->n_v = 3 * c->n_nodes; c->n_p = c->nm * c->n_el;
  c->h = 1.0 / N;
  c->detJ = (c->h / 2) * (c->h / 2) * (c->h / 2);
  gll_nodes(k, c->xn);
  gauss_legendre(c->n1, c->xg, c->wg);
  for (int a = 0; a < c->n1; ++a)
    for (int i = 0; i < c->n1; ++i) {
      c->phi[a][i] = (double)lagrange(c->xn, c->n1, a, c->xg[i]);
      c->dphi[a][i] = (double)dlagrange(c->xn, c->n1, a, c->xg[i]);
    }
  /* orthonormal Legendre Lhat_m = sqrt((2m+1)/2) P_m (R2) */
  for (int m = 0; m < c->n1; ++m)
    for (int i = 0; i < c->n1; ++i) {
      long double P, dP;
      if (m == 0) P = 1.0L; else legendre(m, c->xg[i], &P, &dP);
      c->leg[m][i] = (double)(sqrtl((2.0L * m + 1.0L) / 2.0L) * P);
    }
  /* mode order (R2): for d in 0..k-1, for cz in 0..d, for cy in 0..d-cz: cx = d-cy-cz */
  int m = 0;
  for (int d = 0; d <= k - 1; ++d)
    for (int cz = 0; cz <= d; ++cz)
      for (int cy = 0; cy <= d - cz; ++cy) { c->mode[m][0] = d - cy - cz; c->mode[m][1] = cy; c->mode[m][2] = cz; ++m; }
  const int n1 = c->n1, nq = c->nq;
  c->gphi = (double*)malloc(sizeof(double) * nq * nq * 3);
  c->vphi = (double*)malloc(sizeof(double) * nq * nq);
  c->wq = (double*)malloc(sizeof(double) * nq);
  for (int a = 0; a < nq; ++a) {
    int ax = a % n1, ay = (a / n1) % n1, az = a / (n1 * n1);
    for (int q = 0; q < nq; ++q) {
      int qx = q % n1, qy = (q / n1) % n1, qz = q / (n1 * n1);
      double px = c->phi[ax][qx], py = c->phi[ay][qy], pz = c->phi[az][qz];
      c->vphi[a * nq + q] = px * py * pz;
      c->gphi[(a * nq + q) * 3 + 0] = c->dphi[ax][qx] * py * pz;
      c->gphi[(a * nq + q) * 3 + 1] = px * c->dphi[ay][qy] * pz;
      c->gphi[(a * nq + q) * 3 + 2] = px * py * c->dphi[az][qz];
    }
  }
  for (int q = 0; q < nq; ++q) {
    int qx = q % n1, qy = (q / n1) % n1, qz = q / (n1 * n1);
    c->wq[q] = c->wg[qx] * c->wg[qy] * c->wg[qz];
  }
  /* B_e[m][(c,a)] = - sum_q q_m(xi_q) d_c phi_a(xi_q) w_q detJ, d_c = (2/h) d/dxi_c
   * (B u := -div u; B_ij = -int q_i div phi_j). */
  c->Be = (double*)malloc(sizeof(double) * c->nm * 3 * nq);
  for (int mm = 0; mm < c->nm; ++mm)
    for (int cc = 0; cc < 3; ++cc)
      for (int a = 0; a < nq; ++a) {
        double s = 0.0;
        for (int q = 0; q < nq; ++q) {
          int qx = q % n1, qy = (q / n1) % n1, qz = q / (n1 * n1);
          double qm = c->leg[c->mode[mm][0]][qx] * c->leg[c->mode[mm][1]][qy] * c->leg[c->mode[mm][2]][qz];
          s += qm * ((2.0 / c->h) * c->gphi[(a * nq + q) * 3 + cc]) * c->wq[q] * c->detJ;
        }
        c->Be[(int64_t)mm * 3 * nq + cc * nq + a] = -s;
      }
  c->chunk = 2048;
  c->work = (double*)malloc(sizeof(double) * c->chunk * 3 * nq);
  return c;
}

or_ctx* or_create(int N, int k) { return or_create_box(N, N, k); }

void or_destroy(or_ctx* c) {
  if (!c) return;
  free(c->gphi); free(c->vphi); free(c->wq); free(c->Be); free(c->work); free(c);
}

/* Structured sizes without building tables (n_el, n_nodes, n_v, n_p, n_q, n_m). */
void or_sizes_only(int N, int k, int64_t* out) {
  int64_t nn1 = (int64_t)k * N + 1, n1 = k + 1;
  out[0] = (int64_t)N * N * N; out[1] = nn1 * nn1 * nn1; out[2] = 3 * out[1];
  out[3] = (int64_t)or_nmodes(k) * out[0]; out[4] = n1 * n1 * n1; out[5] = or_nmodes(k);
}

/* Exports for tests (tables and sizes). */
void or_sizes(const or_ctx* c, int64_t* out) {
  out[0] = c->n_el; out[1] = c->n_nodes; out[2] = c->n_v; out[3] = c->n_p; out[4] = c->nq; out[5] = c->nm;
}
void or_tables(const or_ctx* c, double* xn, double* xg, double* wg, double* phi, double* dphi, double* leg, int* modes) {
  for (int i = 0; i < c->n1; ++i) { xn[i] = c->xn[i]; xg[i] = c->xg[i]; wg[i] = c->wg[i]; }
  for (int a = 0; a < c->n1; ++a) for (int i = 0; i < c->n1; ++i) {
    phi[a * c->n1 + i] = c->phi[a][i]; dphi[a * c->n1 + i] = c->dphi[a][i]; leg[a * c->n1 + i] = c->leg[a][i];
  }
  for (int m = 0; m < c->nm; ++m) for (int d = 0; d < 3; ++d) modes[m * 3 + d] = c->mode[m][d];
}
void or_element_B(const or_ctx* c, double* Be) { memcpy(Be, c->Be, sizeof(double) * c->nm * 3 * c->nq); }

/* ---------------------------------------------------------------- structure
 * a1: e = ex + N(ey + N ez); local a = ax + n1(ay + n1 az);
 * g = (k ex + ax) + (kN+1)[(k ey + ay) + (kN+1)(k ez + az)];
 * velocity dof (c, g) -> c*n_nodes + g (SoA); pressure (e, m) -> e*n_m + m.   */
static int64_t or_node(const or_ctx* c, int64_t e, int a) {
  int64_t N = c->N, k = c->k, n1 = c->n1, nn1 = k * N + 1;
  int64_t ex = e % N, ey = (e / N) % N, ez = e / (N * N);
  int64_t ax = a % n1, ay = (a / n1) % n1, az = a / (n1 * n1);
  return (k * ex + ax) + nn1 * ((k * ey + ay) + nn1 * (k * ez + az));
}
/* boundary node iff any grid index is 0 or kN (u = 0 on the boundary) */
static int or_node_is_boundary(const or_ctx* c, int64_t g) {
  int64_t nn1 = (int64_t)c->k * c->N + 1;
  int64_t gx = g % nn1, gy = (g / nn1) % nn1, gz = g / (nn1 * nn1);
  return gx == 0 || gy == 0 || gz == 0 || gx == nn1 - 1 || gy == nn1 - 1 || gz == (int64_t)c->k * c->Nz;
}
/* element touches the boundary iff any index is 0 or N-1 (eq:bdramp set D) */
static int or_elem_on_boundary(const or_ctx* c, int64_t e) {
  int64_t N = c->N, ex = e % N, ey = (e / N) % N, ez = e / (N * N);
  return ex == 0 || ey == 0 || ez == 0 || ex == N - 1 || ey == N - 1 || ez == c->Nz - 1;
}

void or_boundary_elements(const or_ctx* c, uint8_t* flag) {
  for (int64_t e = 0; e < c->n_el; ++e) flag[e] = (uint8_t)or_elem_on_boundary(c, e);
}
void or_dofmap(const or_ctx* c, int64_t* map) {
  for (int64_t e = 0; e < c->n_el; ++e)
    for (int a = 0; a < c->nq; ++a) map[e * c->nq + a] = or_node(c, e, a);
}
void or_boundary_mask(const or_ctx* c, uint8_t* mask) { /* 1 = boundary (eliminated) dof */
  for (int cc = 0; cc < 3; ++cc)
    for (int64_t g = 0; g < c->n_nodes; ++g) mask[cc * c->n_nodes + g] = (uint8_t)or_node_is_boundary(c, g);
}

/* Gather element-local velocity (c, a), Dirichlet entries zeroed unless nomask. */
/* Summation-order switch for the self-discrepancy delta_self (SURVEY.md 8(c) 12(ii):
 * "the oracle vs itself with reversed element and dot order").  0 (default): element
 * scatter-adds and dot products in ascending order; 1: both descending; 2: dot products as
 * (sum of even-indexed terms) + (sum of odd-indexed terms), scatters ascending.  Same arithmetic,
 * another rounding order -- it measures how far the fixed-iteration CG amplifies
 * summation-order rounding alone. */
static int g_rev = 0;
void or_set_order(int rev) { g_rev = (rev == 1 || rev == 2) ? rev : 0; }

static void gather_u(const or_ctx* c, int64_t e, const double* u, double* ue, int nomask) {
  for (int cc = 0; cc < 3; ++cc)
    for (int a = 0; a < c->nq; ++a) {
      int64_t g = or_node(c, e, a);
      ue[cc * c->nq + a] = (!nomask && or_node_is_boundary(c, g)) ? 0.0 : u[cc * c->n_nodes + g];
    }
}
/* Scatter-add element vectors chunk [e0, e1) in element order (serial => fixed order). */
static void scatter_chunk(const or_ctx* c, int64_t e0, int64_t e1, const double* ye, double* y) {
  for (int64_t i = e0; i < e1; ++i) {
    const int64_t e = g_rev ? e1 - 1 - (i - e0) : i;
    for (int cc = 0; cc < 3; ++cc)
      for (int a = 0; a < c->nq; ++a)
        y[cc * c->n_nodes + or_node(c, e, a)] += ye[(e - e0) * 3 * c->nq + cc * c->nq + a];
  }
}
static void mask_velocity(const or_ctx* c, double* y) {
  for (int cc = 0; cc < 3; ++cc)
    for (int64_t g = 0; g < c->n_nodes; ++g) if (or_node_is_boundary(c, g)) y[cc * c->n_nodes + g] = 0.0;
}

/* ---------------------------------------------------------------- A(mu)
 * Element viscous-stress action by dense Gauss quadrature (R3, R4):
 *   (A_e u_e)_{c,a} = sum_q mu_q w_q detJ sum_j d_j phi_a(x_q) (d_j u_c + d_c u_j)(x_q)
 * i.e. int 2 mu eps(u):eps(phi_a e_c), the weak form of -div[mu(grad u + grad u^T)]
 * (eq:stokes; A_mu = -div(2 mu grad_s u)),
 * d_j = (2/h) d/dxi_j on the uniform mesh.                                    */
static void element_A_apply(const or_ctx* c, const double* mue, const double* ue, double* ye) {
  const int nq = c->nq; const double s = 2.0 / c->h;
  for (int i = 0; i < 3 * nq; ++i) ye[i] = 0.0;
  for (int q = 0; q < nq; ++q) {
    double G[3][3]; /* G[cc][j] = d_j u_cc at x_q */
    for (int cc = 0; cc < 3; ++cc) for (int j = 0; j < 3; ++j) {
      double t = 0.0;
      for (int a = 0; a < nq; ++a) t += ue[cc * nq + a] * (s * c->gphi[(a * nq + q) * 3 + j]);
      G[cc][j] = t;
    }
    double wmu = mue[q] * c->wq[q] * c->detJ;
    for (int cc = 0; cc < 3; ++cc)
      for (int a = 0; a < nq; ++a) {
        double t = 0.0;
        for (int j = 0; j < 3; ++j) t += (s * c->gphi[(a * nq + q) * 3 + j]) * (G[cc][j] + G[j][cc]);
        ye[cc * nq + a] += wmu * t;
      }
  }
}

/* Explicit element matrix (tests / dense assembly):
 * A_e[(c,a),(d,b)] = sum_q mu_q w_q detJ [delta_cd grad phi_a . grad phi_b + d_d phi_a d_c phi_b] */
void or_element_A_matrix(const or_ctx* c, const double* mue, double* Ae) {
  const int nq = c->nq, n = 3 * nq; const double s = 2.0 / c->h;
  for (int64_t i = 0; i < (int64_t)n * n; ++i) Ae[i] = 0.0;
  for (int q = 0; q < nq; ++q) {
    double wmu = mue[q] * c->wq[q] * c->detJ;
    for (int cc = 0; cc < 3; ++cc) for (int a = 0; a < nq; ++a)
      for (int d = 0; d < 3; ++d) for (int b = 0; b < nq; ++b) {
        double v = 0.0;
        if (cc == d) for (int j = 0; j < 3; ++j) v += (s * c->gphi[(a * nq + q) * 3 + j]) * (s * c->gphi[(b * nq + q) * 3 + j]);
        v += (s * c->gphi[(a * nq + q) * 3 + d]) * (s * c->gphi[(b * nq + q) * 3 + cc]);
        Ae[(int64_t)(cc * nq + a) * n + d * nq + b] += wmu * v;
      }
  }
}

/* y = M A(mu) M u  (nomask != 0: no Dirichlet elimination -- test pins only) */
void or_apply_A(or_ctx* c, const double* mu_q, const double* u, double* y, int nomask) {
  const int nq = c->nq;
  memset(y, 0, sizeof(double) * c->n_v);
  for (int64_t e0 = 0; e0 < c->n_el; e0 += c->chunk) {
    int64_t e1 = e0 + c->chunk < c->n_el ? e0 + c->chunk : c->n_el;
#pragma omp parallel for schedule(static)
    for (int64_t e = e0; e < e1; ++e) {
      double ue[3 * 729];
      gather_u(c, e, u, ue, nomask);
      element_A_apply(c, mu_q + e * nq, ue, c->work + (e - e0) * 3 * nq);
    }
    scatter_chunk(c, e0, e1, c->work, y);
  }
  if (!nomask) mask_velocity(c, y);
}

/* A at sampled velocity dofs only: y_s = (M A M u)[dofs[s]] (full-size sampled parity). */
void or_apply_A_sampled(or_ctx* c, const double* mu_q, const double* u, const int64_t* dofs, int64_t ns, double* ys) {
  const int nq = c->nq, n1 = c->n1; const int64_t N = c->N, k = c->k, nn1 = k * N + 1;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t s = 0; s < ns; ++s) {
    int64_t dof = dofs[s]; int cc = (int)(dof / c->n_nodes); int64_t g = dof % c->n_nodes;
    double acc = 0.0;
    if (!or_node_is_boundary(c, g)) {
      int64_t gx = g % nn1, gy = (g / nn1) % nn1, gz = g / (nn1 * nn1);
      /* elements containing node g, in increasing element index */
      for (int64_t ez = 0; ez < c->Nz; ++ez) { int64_t az = gz - k * ez; if (az < 0 || az > k) continue;
        for (int64_t ey = 0; ey < N; ++ey) { int64_t ay = gy - k * ey; if (ay < 0 || ay > k) continue;
          for (int64_t ex = 0; ex < N; ++ex) { int64_t ax = gx - k * ex; if (ax < 0 || ax > k) continue;
            int64_t e = ex + N * (ey + N * ez);
            double ue[3 * 729], ye[3 * 729];
            gather_u(c, e, u, ue, 0);
            element_A_apply(c, mu_q + e * nq, ue, ye);
            acc += ye[cc * nq + (int)(ax + n1 * (ay + n1 * az))];
          } } }
    }
    ys[s] = acc;
  }
}

/* ---------------------------------------------------------------- B, B^T
 * p_e = B_e (M u)_e  (divergence, B u := -div u)                */
void or_apply_B(or_ctx* c, const double* u, double* p, int nomask) {
  const int nq = c->nq, nm = c->nm;
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < c->n_el; ++e) {
    double ue[3 * 729];
    gather_u(c, e, u, ue, nomask);
    for (int m = 0; m < nm; ++m) {
      double s = 0.0;
      for (int i = 0; i < 3 * nq; ++i) s += c->Be[(int64_t)m * 3 * nq + i] * ue[i];
      p[e * nm + m] = s;
    }
  }
}

/* y = M B^T p  (gradient) */
void or_apply_BT(or_ctx* c, const double* p, double* y, int nomask) {
  const int nq = c->nq, nm = c->nm;
  memset(y, 0, sizeof(double) * c->n_v);
  const int64_t nch = (c->n_el + c->chunk - 1) / c->chunk;
  for (int64_t ic = 0; ic < nch; ++ic) {
    const int64_t e0 = (g_rev ? nch - 1 - ic : ic) * c->chunk;
    int64_t e1 = e0 + c->chunk < c->n_el ? e0 + c->chunk : c->n_el;
#pragma omp parallel for schedule(static)
    for (int64_t e = e0; e < e1; ++e) {
      double* ye = c->work + (e - e0) * 3 * nq;
      for (int i = 0; i < 3 * nq; ++i) {
        double s = 0.0;
        for (int m = 0; m < nm; ++m) s += c->Be[(int64_t)m * 3 * nq + i] * p[e * nm + m];
        ye[i] = s;
      }
    }
    scatter_chunk(c, e0, e1, c->work, y);
  }
  if (!nomask) mask_velocity(c, y);
}

/* ---------------------------------------------------------------- C_w, D_w
 * Lumped weighted velocity mass (eq:lumping generalised as in eq:wbfbt,
 * PAPER.md:310-323, 446-454; R7: w = sqrt(mu); eq:bdramp PAPER.md:2232-2245):
 *   l_e[a](w) = sum_q w_{e,q} phi_a(xi_q) w_q detJ,   C[g] = sum_{e ni g} l_e[a](w_l)
 * (row sums: the coefficient vector of the constant 1 is all-ones, R8).
 * Cinv = M/C, Dinv = M/D on nodes; entries <= 0 at interior nodes are counted
 * and reported, not altered (R9).                                             */
void or_lumped(or_ctx* c, const double* mu_q, double a_l, double a_r,
               double* Cw, double* Dw, double* Cinv, double* Dinv, int64_t* nonpos) {
  const int nq = c->nq;
  memset(Cw, 0, sizeof(double) * c->n_nodes);
  memset(Dw, 0, sizeof(double) * c->n_nodes);
  double* le = (double*)malloc(sizeof(double) * nq);
  for (int64_t e = 0; e < c->n_el; ++e) {
    int onb = or_elem_on_boundary(c, e);
    double al = onb ? a_l : 1.0, ar = onb ? a_r : 1.0;
    for (int a = 0; a < nq; ++a) {
      double sl = 0.0, sr = 0.0;
      for (int q = 0; q < nq; ++q) {
        double sq = sqrt(mu_q[e * nq + q]);
        sl += (al * sq) * c->vphi[a * nq + q] * c->wq[q] * c->detJ;
        sr += (ar * sq) * c->vphi[a * nq + q] * c->wq[q] * c->detJ;
      }
      int64_t g = or_node(c, e, a);
      Cw[g] += sl; Dw[g] += sr;
    }
  }
  free(le);
  nonpos[0] = nonpos[1] = 0;
  for (int64_t g = 0; g < c->n_nodes; ++g) {
    int b = or_node_is_boundary(c, g);
    if (!b && Cw[g] <= 0.0) nonpos[0]++;
    if (!b && Dw[g] <= 0.0) nonpos[1]++;
    Cinv[g] = b ? 0.0 : 1.0 / Cw[g];
    Dinv[g] = b ? 0.0 : 1.0 / Dw[g];
  }
}

/* Viscosity-gradient wBFBT weights (rmk:wbfbt-visc-grad):
 *   w_l = w_r = (mu^2 + |grad mu|^2)^{1/4}.
 * mu is given only at the Gauss points, so grad mu is the gradient of the element's
 * tensor-product Lagrange interpolant through its (k+1)^3 Gauss-point samples,
 * d/dx_d = (2/h) d/dxi_d (reading R17).  Returned as mu_eff = sqrt(mu^2 + |grad mu|^2)
 * = w^2, so that or_lumped(mu_eff) lumps with its weight sqrt(mu_eff) = w.        */
void or_grad_weights(const or_ctx* c, const double* mu_q, double* mu_eff) {
  const int n1 = c->n1, nq = c->nq;
  double D[OR_MAXN1][OR_MAXN1]; /* D[i][j] = l_j'(xg_i), Lagrange basis on the Gauss points */
  for (int i = 0; i < n1; ++i)
    for (int j = 0; j < n1; ++j) D[i][j] = (double)dlagrange(c->xg, n1, j, c->xg[i]);
  const double s = 2.0 / c->h;
  for (int64_t e = 0; e < c->n_el; ++e) {
    const double* m = mu_q + e * nq;
    for (int qz = 0; qz < n1; ++qz)
      for (int qy = 0; qy < n1; ++qy)
        for (int qx = 0; qx < n1; ++qx) {
          double gx = 0.0, gy = 0.0, gz = 0.0;
          for (int j = 0; j < n1; ++j) {
            gx += D[qx][j] * m[j + n1 * (qy + n1 * qz)];
            gy += D[qy][j] * m[qx + n1 * (j + n1 * qz)];
            gz += D[qz][j] * m[qx + n1 * (qy + n1 * j)];
          }
          gx *= s; gy *= s; gz *= s;
          const double mu = m[qx + n1 * (qy + n1 * qz)];
          mu_eff[e * nq + qx + n1 * (qy + n1 * qz)] = sqrt(mu * mu + (gx * gx + gy * gy + gz * gz));
        }
  }
}

/* ---------------------------------------------------------------- K_w, diag
 * K p = B (Xinv o (B^T p)), Xinv a nodal diagonal acting on all 3 components
 * (PAPER.md:2453-2461).                                                       */
void or_apply_K(or_ctx* c, const double* Xinv, const double* p, double* q, double* tmp_v /* n_v */) {
  or_apply_BT(c, p, tmp_v, 0);
  for (int cc = 0; cc < 3; ++cc)
    for (int64_t g = 0; g < c->n_nodes; ++g) tmp_v[cc * c->n_nodes + g] *= Xinv[g];
  or_apply_B(c, tmp_v, q, 0);
}

/* diag(K)_{e,m} = sum_{c,a} B_e[m,(c,a)]^2 Xinv[g(e,a)] */
void or_jacobi_diag(or_ctx* c, const double* Xinv, double* diag) {
  const int nq = c->nq, nm = c->nm;
  for (int64_t e = 0; e < c->n_el; ++e)
    for (int m = 0; m < nm; ++m) {
      double s = 0.0;
      for (int cc = 0; cc < 3; ++cc)
        for (int a = 0; a < nq; ++a) {
          double b = c->Be[(int64_t)m * 3 * nq + cc * nq + a];
          s += b * b * Xinv[or_node(c, e, a)];
        }
      diag[e * nm + m] = s;
    }
}

/* ---------------------------------------------------------------- projection
 * P v = v - (z0.v / z0.z0) z0, z0 = coefficients of the constant pressure:
 * 1 = 2^{3/2} Lhat_0^3, so z0 = 2^{3/2} on mode 0 of every element (R10;
 * Neumann null space).                         */
static double dot(const double* a, const double* b, int64_t n) {
  double s = 0.0;
  if (g_rev == 1)
    for (int64_t i = n - 1; i >= 0; --i) s += a[i] * b[i];
  else if (g_rev == 2) { /* even-indexed terms, then odd-indexed terms */
    double s1 = 0.0;
    for (int64_t i = 0; i < n; i += 2) s += a[i] * b[i];
    for (int64_t i = 1; i < n; i += 2) s1 += a[i] * b[i];
    s += s1;
  } else
    for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}
void or_project(const or_ctx* c, double* v) {
  const double z = 2.0 * sqrt(2.0);
  double zv = 0.0, zz = 0.0;
  for (int64_t e = 0; e < c->n_el; ++e) { zv += z * v[e * c->nm]; zz += z * z; }
  double f = zv / zz;
  for (int64_t e = 0; e < c->n_el; ++e) v[e * c->nm] -= f * z;
}

/* ---------------------------------------------------------------- PCG
 * Fixed-iteration Jacobi-PCG standing in for the paper's HMG V-cycle
 * (north_star (5), reading R11):
 *   x=0; r=b; z=Minv r; p=z; rz=<r,z>
 *   repeat iters: if rz==0 break; q=Kp; pq=<p,q>; if pq==0 break;
 *     a=rz/pq; x+=a p; r-=a q; z=Minv r; rz'=<r,z>; b=rz'/rz; p=z+b p; rz=rz'  */
typedef struct { double* r; double* z; double* p; double* q; double* tv; } or_pcg_ws;

static void pcg_step(or_ctx* c, const double* Xinv, const double* Minv, double* x, double* r, double* p,
                     double* rz, double* z, double* q, double* tv, double* ab) {
  const int64_t n = c->n_p;
  or_apply_K(c, Xinv, p, q, tv);
  double pq = dot(p, q, n);
  if (pq == 0.0) { if (ab) { ab[0] = 0; ab[1] = 0; } return; }
  double alpha = *rz / pq;
  for (int64_t i = 0; i < n; ++i) x[i] += alpha * p[i];
  for (int64_t i = 0; i < n; ++i) r[i] -= alpha * q[i];
  for (int64_t i = 0; i < n; ++i) z[i] = Minv[i] * r[i];
  double rz2 = dot(r, z, n);
  double beta = rz2 / *rz;
  for (int64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
  *rz = rz2;
  if (ab) { ab[0] = alpha; ab[1] = beta; }
}

/* Minv = pseudo-inverse of diag(K) (R11): 1/d_i, except 0 where |d_i| <= 1e-13 max|d|
 * (a row of K that vanishes up to rounding, e.g. the constant mode when N = 1). */
static void jacobi_minv(const double* diagK, double* Minv, int64_t n) {
  double dmax = 0.0;
  for (int64_t i = 0; i < n; ++i) dmax = fabs(diagK[i]) > dmax ? fabs(diagK[i]) : dmax;
  for (int64_t i = 0; i < n; ++i) Minv[i] = fabs(diagK[i]) > 1e-13 * dmax ? 1.0 / diagK[i] : 0.0;
}

/* x = PCG(K_side, b) with K_side = B Xinv B^T, Minv = 1/diag(K_side) (R11).  When
 * alpha / beta are non-NULL (length iters) they receive the scalars of O9 in iteration
 * order: alpha_i = rz_i / pq_i and beta_i = rz_{i+1} / rz_i; iterations not run (a
 * break of O9) are recorded as 0.  Returns the number of iterations run. */
int or_pcg_rec(or_ctx* c, const double* Xinv, const double* diagK, const double* b, double* x, int iters,
               double* alpha, double* beta);
void or_pcg(or_ctx* c, const double* Xinv, const double* diagK, const double* b, double* x, int iters) {
  (void)or_pcg_rec(c, Xinv, diagK, b, x, iters, NULL, NULL);
}
int or_pcg_rec(or_ctx* c, const double* Xinv, const double* diagK, const double* b, double* x, int iters,
               double* alpha, double* beta) {
  const int64_t n = c->n_p;
  double* r = (double*)malloc(sizeof(double) * n); double* z = (double*)malloc(sizeof(double) * n);
  double* p = (double*)malloc(sizeof(double) * n); double* q = (double*)malloc(sizeof(double) * n);
  double* Minv = (double*)malloc(sizeof(double) * n); double* tv = (double*)malloc(sizeof(double) * c->n_v);
  jacobi_minv(diagK, Minv, n);
  for (int64_t i = 0; i < n; ++i) { x[i] = 0.0; r[i] = b[i]; z[i] = Minv[i] * r[i]; p[i] = z[i]; }
  double rz = dot(r, z, n);
  int run = 0;
  for (int it = 0; it < iters; ++it) {
    if (alpha) alpha[it] = 0.0;
    if (beta) beta[it] = 0.0;
  }
  for (int it = 0; it < iters; ++it) {
    if (rz == 0.0) break;
    double ab[2];
    pcg_step(c, Xinv, Minv, x, r, p, &rz, z, q, tv, ab);
    if (ab[0] == 0.0 && ab[1] == 0.0) break; /* pq == 0 */
    if (alpha) alpha[it] = ab[0];
    if (beta) beta[it] = ab[1];
    run = it + 1;
  }
  free(r); free(z); free(p); free(q); free(Minv); free(tv);
  return run;
}

/* One PCG iteration from a supplied state (x, r, p, rz) -- one-step parity. */
void or_pcg_step(or_ctx* c, const double* Xinv, const double* diagK, double* x, double* r, double* p, double* rz) {
  const int64_t n = c->n_p;
  double* z = (double*)malloc(sizeof(double) * n); double* q = (double*)malloc(sizeof(double) * n);
  double* Minv = (double*)malloc(sizeof(double) * n); double* tv = (double*)malloc(sizeof(double) * c->n_v);
  jacobi_minv(diagK, Minv, n);
  pcg_step(c, Xinv, Minv, x, r, p, rz, z, q, tv, NULL);
  free(z); free(q); free(Minv); free(tv);
}

/* Projected Poisson solve: x = P PCG(K_side, P b) (R10). */
void or_poisson(or_ctx* c, const double* Xinv, const double* diagK, const double* b, double* x, int iters) {
  double* bb = (double*)malloc(sizeof(double) * c->n_p);
  memcpy(bb, b, sizeof(double) * c->n_p);
  or_project(c, bb);
  or_pcg(c, Xinv, diagK, bb, x, iters);
  or_project(c, x);
  free(bb);
}

/* ---------------------------------------------------------------- Chebyshev
 * Chebyshev-accelerated point-Jacobi (the paper's smoother, PAPER.md:2531-2546;
 * SURVEY.md 8(f) #2) as a fixed-iteration inner solve.  The paper gives no
 * recurrence or spectrum bounds (reading R16): Saad, "Iterative Methods
 * for Sparse Linear Systems" (2003), Alg. 12.1 (Chebyshev acceleration) on
 * M^-1 K with the Jacobi pseudo-inverse Minv of R11 as M^-1 and the caller's
 * interval [lmin, lmax] of the spectrum of M^-1 K, from x0 = 0:
 *   theta = (lmax + lmin)/2; delta = (lmax - lmin)/2; sigma1 = theta/delta; rho = 1/sigma1
 *   r = b; d = (1/theta) Minv r
 *   repeat iters: x += d; r -= K d; rho' = 1/(2 sigma1 - rho);
 *                 d = rho' rho d + (2 rho'/delta) Minv r; rho = rho'
 * The recurrence is written once (cheb_run) over an operator callback; the dense
 * form (or_cheb_dense) is what tests/test_oracle_cheb.py pins against the closed
 * form e_k = T_k((theta - lambda)/delta) / T_k(sigma1) e_0 of the error on a
 * diagonal system.                                                            */
typedef void (*or_op)(void* ctx, const double* in, double* out);
static void cheb_run(or_op K, void* kctx, int64_t n, const double* Minv, const double* b, double* x, int iters,
                     double lmin, double lmax) {
  double* r = (double*)malloc(sizeof(double) * n);
  double* d = (double*)malloc(sizeof(double) * n);
  double* q = (double*)malloc(sizeof(double) * n);
  const double theta = 0.5 * (lmax + lmin), delta = 0.5 * (lmax - lmin);
  const double sigma1 = theta / delta;
  double rho = 1.0 / sigma1;
  for (int64_t i = 0; i < n; ++i) { x[i] = 0.0; r[i] = b[i]; d[i] = (1.0 / theta) * (Minv[i] * r[i]); }
  for (int it = 0; it < iters; ++it) {
    for (int64_t i = 0; i < n; ++i) x[i] += d[i];
    K(kctx, d, q);
    for (int64_t i = 0; i < n; ++i) r[i] -= q[i];
    const double rho1 = 1.0 / (2.0 * sigma1 - rho);
    const double c1 = rho1 * rho, c2 = 2.0 * rho1 / delta;
    for (int64_t i = 0; i < n; ++i) d[i] = c1 * d[i] + c2 * (Minv[i] * r[i]);
    rho = rho1;
  }
  free(r); free(d); free(q);
}

typedef struct { int64_t n; const double* A; } or_dense;
static void dense_op(void* ctx, const double* in, double* out) {
  const or_dense* D = (const or_dense*)ctx;
  for (int64_t i = 0; i < D->n; ++i) {
    double s = 0.0;
    for (int64_t j = 0; j < D->n; ++j) s += D->A[i * D->n + j] * in[j];
    out[i] = s;
  }
}
/* the recurrence on a dense n x n matrix A (row-major) with Jacobi inverse Minv */
void or_cheb_dense(int64_t n, const double* A, const double* Minv, const double* b, double* x, int iters,
                   double lmin, double lmax) {
  or_dense D = {n, A};
  cheb_run(dense_op, &D, n, Minv, b, x, iters, lmin, lmax);
}

typedef struct { or_ctx* c; const double* Xinv; double* tv; } or_kop;
static void k_op(void* ctx, const double* in, double* out) {
  or_kop* k = (or_kop*)ctx;
  or_apply_K(k->c, k->Xinv, in, out, k->tv);
}
/* Projected Chebyshev solve: x = P Cheb(K_side, P b) (R10, R16). */
void or_poisson_cheb(or_ctx* c, const double* Xinv, const double* diagK, const double* b, double* x, int iters,
                     double lmin, double lmax) {
  const int64_t n = c->n_p;
  double* bb = (double*)malloc(sizeof(double) * n);
  double* Minv = (double*)malloc(sizeof(double) * n);
  or_kop k = {c, Xinv, (double*)malloc(sizeof(double) * c->n_v)};
  memcpy(bb, b, sizeof(double) * n);
  or_project(c, bb);
  jacobi_minv(diagK, Minv, n);
  cheb_run(k_op, &k, n, Minv, bb, x, iters, lmin, lmax);
  or_project(c, x);
  free(bb); free(Minv); free(k.tv);
}

/* Power-iteration estimate of the largest-magnitude eigenvalue of Minv K (the
 * input the caller turns into a Chebyshev interval, R16):
 *   v = v0 / ||v0||; repeat iters: w = Minv (K v); lambda = ||w||; v = w / lambda
 * Returns lambda of the last step (0 if an iterate vanishes). */
static double power_run(or_op K, void* kctx, int64_t n, const double* Minv, const double* v0, int iters) {
  double* v = (double*)malloc(sizeof(double) * n);
  double* w = (double*)malloc(sizeof(double) * n);
  double nv = sqrt(dot(v0, v0, n)), lam = 0.0;
  for (int64_t i = 0; i < n; ++i) v[i] = nv > 0.0 ? v0[i] / nv : 0.0;
  for (int it = 0; it < iters && nv > 0.0; ++it) {
    K(kctx, v, w);
    for (int64_t i = 0; i < n; ++i) w[i] = Minv[i] * w[i];
    lam = sqrt(dot(w, w, n));
    if (lam == 0.0) break;
    for (int64_t i = 0; i < n; ++i) v[i] = w[i] / lam;
  }
  free(v); free(w);
  return lam;
}
double or_eigmax_dense(int64_t n, const double* A, const double* Minv, const double* v0, int iters) {
  or_dense D = {n, A};
  return power_run(dense_op, &D, n, Minv, v0, iters);
}
double or_poisson_eigmax(or_ctx* c, const double* Xinv, const double* diagK, const double* v0, int iters) {
  const int64_t n = c->n_p;
  double* Minv = (double*)malloc(sizeof(double) * n);
  or_kop k = {c, Xinv, (double*)malloc(sizeof(double) * c->n_v)};
  jacobi_minv(diagK, Minv, n);
  const double lam = power_run(k_op, &k, n, Minv, v0, iters);
  free(Minv); free(k.tv);
  return lam;
}

/* ---------------------------------------------------------------- diag(A), Chebyshev on A
 * diag(M A M)_{(c,g)} = sum_{e ni g} A_e[(c,a),(c,a)] (elements ascending), with
 *   A_e[(c,a),(c,a)] = sum_q mu_q w_q detJ s^2 [ sum_j gphi(a,q,j)^2 + gphi(a,q,c)^2 ],
 * the cc == d, b == a entries of or_element_A_matrix (s = 2/h); Dirichlet dofs 0 (the
 * masked operator's diagonal).  Building block of the Jacobi/Chebyshev smoother on A
 * that the paper's HMG uses for the viscous block (SURVEY 8(f) #1's
 * approximate A^-1; reading R18).                                                     */
void or_diag_A(or_ctx* c, const double* mu_q, double* diag) {
  const int nq = c->nq; const double s = 2.0 / c->h;
  memset(diag, 0, sizeof(double) * c->n_v);
  for (int64_t e = 0; e < c->n_el; ++e)
    for (int cc = 0; cc < 3; ++cc)
      for (int a = 0; a < nq; ++a) {
        double t = 0.0;
        for (int q = 0; q < nq; ++q) {
          double g2 = 0.0;
          for (int j = 0; j < 3; ++j) { const double g = s * c->gphi[(a * nq + q) * 3 + j]; g2 += g * g; }
          const double gc = s * c->gphi[(a * nq + q) * 3 + cc];
          t += mu_q[e * nq + q] * c->wq[q] * c->detJ * (g2 + gc * gc);
        }
        diag[cc * c->n_nodes + or_node(c, e, a)] += t;
      }
  mask_velocity(c, diag);
}

typedef struct { or_ctx* c; const double* mu_q; } or_aop;
static void a_op(void* ctx, const double* in, double* out) {
  or_aop* a = (or_aop*)ctx;
  or_apply_A(a->c, a->mu_q, in, out, 0);
}
static void masked_jacobi(const or_ctx* c, const double* diag, double* Minv) {
  for (int64_t i = 0; i < c->n_v; ++i) Minv[i] = diag[i] > 0.0 ? 1.0 / diag[i] : 0.0;
}
/* x = Cheb(M A M, M b) (Saad Alg. 12.1 as or_poisson_cheb, R16) with the Jacobi inverse
 * mask / diag(A) (R18): the Chebyshev-accelerated point-Jacobi smoother on A, x0 = 0. */
void or_velocity_cheb(or_ctx* c, const double* mu_q, const double* b, double* x, int iters, double lmin,
                      double lmax) {
  const int64_t n = c->n_v;
  double* bb = (double*)malloc(sizeof(double) * n);
  double* d = (double*)malloc(sizeof(double) * n);
  memcpy(bb, b, sizeof(double) * n);
  mask_velocity(c, bb);
  or_diag_A(c, mu_q, d);
  masked_jacobi(c, d, d);
  or_aop a = {c, mu_q};
  cheb_run(a_op, &a, n, d, bb, x, iters, lmin, lmax);
  free(bb); free(d);
}
/* power-iteration estimate of the largest |eigenvalue| of (mask/diag A) M A M (R18) */
double or_velocity_eigmax(or_ctx* c, const double* mu_q, const double* v0, int iters) {
  double* d = (double*)malloc(sizeof(double) * c->n_v);
  or_diag_A(c, mu_q, d);
  masked_jacobi(c, d, d);
  or_aop a = {c, mu_q};
  const double lam = power_run(a_op, &a, c->n_v, d, v0, iters);
  free(d);
  return lam;
}

/* ---------------------------------------------------------------- wBFBT
 * z = S~^{-1}_wBFBT r  (eq:wbfbt), applied right to left:
 *   y = P PCG(K_r, P r); v = Dinv o (B^T y); v = A v; v = Cinv o v; s = P(B v);
 *   z = P PCG(K_l, s)
 * with K_l = B Cinv B^T, K_r = B Dinv B^T.              */
void or_wbfbt(or_ctx* c, const double* mu_q, const double* Cinv, const double* Dinv,
              const double* diagKl, const double* diagKr, const double* r, double* z, int iters) {
  const int64_t np = c->n_p, nv = c->n_v, nn = c->n_nodes;
  double* y = (double*)malloc(sizeof(double) * np);
  double* s = (double*)malloc(sizeof(double) * np);
  double* v = (double*)malloc(sizeof(double) * nv);
  double* w = (double*)malloc(sizeof(double) * nv);
  double* rr = (double*)malloc(sizeof(double) * np);
  memcpy(rr, r, sizeof(double) * np);
  or_project(c, rr);
  or_pcg(c, Dinv, diagKr, rr, y, iters);
  or_project(c, y);
  free(rr);
  or_apply_BT(c, y, v, 0);
  for (int cc = 0; cc < 3; ++cc) for (int64_t g = 0; g < nn; ++g) v[cc * nn + g] *= Dinv[g];
  or_apply_A(c, mu_q, v, w, 0);
  for (int cc = 0; cc < 3; ++cc) for (int64_t g = 0; g < nn; ++g) w[cc * nn + g] *= Cinv[g];
  or_apply_B(c, w, s, 0);
  or_project(c, s);
  or_pcg(c, Cinv, diagKl, s, z, iters);
  or_project(c, z);
  free(y); free(s); free(v); free(w);
}

/* ---------------------------------------------------------------- Stokes solve
 * SURVEY 8(f) #1, reading R19.  [A B^T; B 0] [u; p] = [f; g] with A = M A M, B^T = M B^T
 * and B acting on M u, right-preconditioned by eq:precond-stokes:
 *   P = [At B^T; 0 St],  P^{-1} (a; b) = (At^{-1} (a - B^T y); y),  y = St^{-1} b,
 * St^{-1} = -(wBFBT) (the paper's S := B A^{-1} B^T is positive, so St ~ -S and the
 * exact choices converge in two iterations), At^{-1} = the Chebyshev-Jacobi smoother on
 * A (R18).  Flexible GMRES (Saad 1993: restarted, modified Gram-Schmidt Arnoldi, Givens
 * rotations, x = x0 + Z y) because the fixed-iteration PCG inside wBFBT is not a linear
 * map; with a fixed linear preconditioner it is GMRES.  x0 = 0; stops when the Givens
 * residual estimate is <= rtol ||b|| or after max_iters iterations; the final pressure
 * is projected (R10).  The core runs over operator / preconditioner callbacks, and the
 * dense form or_fgmres_dense is what tests/test_oracle_stokes.py pins.                */
void or_wbfbt_cheb(or_ctx* c, const double* mu_q, const double* Cinv, const double* Dinv, const double* diagKl,
                   const double* diagKr, const double* r, double* z, int iters, double lmin_l, double lmax_l,
                   double lmin_r, double lmax_r);
typedef void (*or_vop)(void* ctx, const double* in, double* out);
static int fgmres_run(or_vop K, or_vop Pinv, void* ctx, int64_t n, const double* b, double* x, int m, int max_iters,
                      double rtol, double* relres) {
  double* V = (double*)malloc(sizeof(double) * n * (m + 1));
  double* Z = (double*)malloc(sizeof(double) * n * m);
  double* w = (double*)malloc(sizeof(double) * n);
  double* H = (double*)calloc((size_t)(m + 1) * m, sizeof(double)); /* H[i*m + j] */
  double* cs = (double*)malloc(sizeof(double) * m);
  double* sn = (double*)malloc(sizeof(double) * m);
  double* g = (double*)malloc(sizeof(double) * (m + 1));
  double* y = (double*)malloc(sizeof(double) * m);
  for (int64_t i = 0; i < n; ++i) { x[i] = 0.0; w[i] = b[i]; }
  const double bnorm = sqrt(dot(b, b, n));
  double beta = bnorm;
  int total = 0;
  while (beta > rtol * bnorm && total < max_iters) {
    for (int64_t i = 0; i < n; ++i) V[i] = w[i] / beta;
    for (int i = 0; i <= m; ++i) g[i] = 0.0;
    g[0] = beta;
    int jend = -1;
    for (int j = 0; j < m && total < max_iters; ++j) {
      Pinv(ctx, V + (int64_t)j * n, Z + (int64_t)j * n);
      K(ctx, Z + (int64_t)j * n, w);
      for (int i = 0; i <= j; ++i) {
        const double hij = dot(w, V + (int64_t)i * n, n);
        H[i * m + j] = hij;
        for (int64_t t = 0; t < n; ++t) w[t] -= hij * V[(int64_t)i * n + t];
      }
      const double hn = sqrt(dot(w, w, n));
      for (int i = 0; i < j; ++i) { /* previous rotations on column j */
        const double a = H[i * m + j], bb = H[(i + 1) * m + j];
        H[i * m + j] = cs[i] * a + sn[i] * bb;
        H[(i + 1) * m + j] = -sn[i] * a + cs[i] * bb;
      }
      const double a = H[j * m + j], den = sqrt(a * a + hn * hn);
      cs[j] = den > 0.0 ? a / den : 1.0;
      sn[j] = den > 0.0 ? hn / den : 0.0;
      H[j * m + j] = den;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      ++total;
      jend = j;
      if (hn > 0.0) for (int64_t t = 0; t < n; ++t) V[(int64_t)(j + 1) * n + t] = w[t] / hn;
      if (fabs(g[j + 1]) <= rtol * bnorm || hn == 0.0) break;
    }
    for (int i = jend; i >= 0; --i) { /* back substitution */
      double t = g[i];
      for (int k = i + 1; k <= jend; ++k) t -= H[i * m + k] * y[k];
      y[i] = t / H[i * m + i];
    }
    for (int i = 0; i <= jend; ++i)
      for (int64_t t = 0; t < n; ++t) x[t] += y[i] * Z[(int64_t)i * n + t];
    K(ctx, x, w); /* true residual for the restart / the stop test */
    for (int64_t t = 0; t < n; ++t) w[t] = b[t] - w[t];
    beta = sqrt(dot(w, w, n));
    if (jend < 0) break;
  }
  if (relres) *relres = bnorm > 0.0 ? beta / bnorm : 0.0;
  free(V); free(Z); free(w); free(H); free(cs); free(sn); free(g); free(y);
  return total;
}

typedef struct { int64_t n; const double *A, *P; } or_dense2;
static void dense2_K(void* c, const double* in, double* out) {
  const or_dense2* D = (const or_dense2*)c;
  for (int64_t i = 0; i < D->n; ++i) { double s = 0.0; for (int64_t j = 0; j < D->n; ++j) s += D->A[i * D->n + j] * in[j]; out[i] = s; }
}
static void dense2_P(void* c, const double* in, double* out) {
  const or_dense2* D = (const or_dense2*)c;
  for (int64_t i = 0; i < D->n; ++i) { double s = 0.0; for (int64_t j = 0; j < D->n; ++j) s += D->P[i * D->n + j] * in[j]; out[i] = s; }
}
/* the FGMRES core on a dense system A x = b with the dense right preconditioner P ~ A^-1 */
int or_fgmres_dense(int64_t n, const double* A, const double* P, const double* b, double* x, int m, int max_iters,
                    double rtol, double* relres) {
  or_dense2 D = {n, A, P};
  return fgmres_run(dense2_K, dense2_P, &D, n, b, x, m, max_iters, rtol, relres);
}

typedef struct {
  or_ctx* c; const double *mu, *Cinv, *Dinv, *dKl, *dKr;
  int pcg, sm; double lo, hi; double *tv, *tp;
  double ilo_l, ihi_l, ilo_r, ihi_r; /* > 0: wBFBT's inner solves are Chebyshev (R16) */
} or_stokes;
static void stokes_K(void* ctx, const double* in, double* out) { /* [A B^T; B 0] (u; p) */
  or_stokes* S = (or_stokes*)ctx;
  or_ctx* c = S->c;
  or_apply_A(c, S->mu, in, out, 0);
  or_apply_BT(c, in + c->n_v, S->tv, 0);
  for (int64_t i = 0; i < c->n_v; ++i) out[i] += S->tv[i];
  or_apply_B(c, in, out + c->n_v, 0);
}
static void stokes_P(void* ctx, const double* in, double* out) { /* P^{-1} (a; b) */
  or_stokes* S = (or_stokes*)ctx;
  or_ctx* c = S->c;
  double* y = out + c->n_v;
  if (S->ilo_l > 0.0)
    or_wbfbt_cheb(c, S->mu, S->Cinv, S->Dinv, S->dKl, S->dKr, in + c->n_v, y, S->pcg, S->ilo_l, S->ihi_l, S->ilo_r,
                  S->ihi_r);
  else
    or_wbfbt(c, S->mu, S->Cinv, S->Dinv, S->dKl, S->dKr, in + c->n_v, y, S->pcg);
  for (int64_t i = 0; i < c->n_p; ++i) y[i] = -y[i];
  or_apply_BT(c, y, S->tv, 0);
  for (int64_t i = 0; i < c->n_v; ++i) S->tv[i] = in[i] - S->tv[i];
  or_velocity_cheb(c, S->mu, S->tv, out, S->sm, S->lo, S->hi);
}
/* inner (may be NULL): {lmin_l, lmax_l, lmin_r, lmax_r} -> wBFBT with Chebyshev inner solves */
int or_stokes_fgmres(or_ctx* c, const double* mu_q, const double* Cinv, const double* Dinv, const double* diagKl,
                     const double* diagKr, const double* f, const double* g, double* u, double* p, int m,
                     int max_iters, double rtol, int pcg_iters, int smooth_iters, double lmin, double lmax,
                     double* relres, const double* inner) {
  const int64_t n = c->n_v + c->n_p;
  double* b = (double*)malloc(sizeof(double) * n);
  double* x = (double*)malloc(sizeof(double) * n);
  or_stokes S = {c, mu_q, Cinv, Dinv, diagKl, diagKr, pcg_iters, smooth_iters, lmin, lmax,
                 (double*)malloc(sizeof(double) * c->n_v), NULL,
                 inner ? inner[0] : 0.0, inner ? inner[1] : 0.0, inner ? inner[2] : 0.0, inner ? inner[3] : 0.0};
  memcpy(b, f, sizeof(double) * c->n_v);
  mask_velocity(c, b);
  memcpy(b + c->n_v, g, sizeof(double) * c->n_p);
  const int it = fgmres_run(stokes_K, stokes_P, &S, n, b, x, m, max_iters, rtol, relres);
  memcpy(u, x, sizeof(double) * c->n_v);
  memcpy(p, x + c->n_v, sizeof(double) * c->n_p);
  or_project(c, p);
  free(b); free(x); free(S.tv);
  return it;
}

/* wBFBT with Chebyshev-accelerated Jacobi as the inner Poisson solves (SURVEY 8(f) #2 "as
 * the inner Poisson solve", R16): or_wbfbt with y = P Cheb(K_r, P r) on [lmin_r, lmax_r] and
 * z = P Cheb(K_l, s) on [lmin_l, lmax_l].  A fixed linear map of r (unlike the PCG form). */
void or_wbfbt_cheb(or_ctx* c, const double* mu_q, const double* Cinv, const double* Dinv, const double* diagKl,
                   const double* diagKr, const double* r, double* z, int iters, double lmin_l, double lmax_l,
                   double lmin_r, double lmax_r) {
  const int64_t np = c->n_p, nv = c->n_v, nn = c->n_nodes;
  double* y = (double*)malloc(sizeof(double) * np);
  double* s = (double*)malloc(sizeof(double) * np);
  double* v = (double*)malloc(sizeof(double) * nv);
  double* w = (double*)malloc(sizeof(double) * nv);
  or_poisson_cheb(c, Dinv, diagKr, r, y, iters, lmin_r, lmax_r);
  or_apply_BT(c, y, v, 0);
  for (int cc = 0; cc < 3; ++cc) for (int64_t g = 0; g < nn; ++g) v[cc * nn + g] *= Dinv[g];
  or_apply_A(c, mu_q, v, w, 0);
  for (int cc = 0; cc < 3; ++cc) for (int64_t g = 0; g < nn; ++g) w[cc * nn + g] *= Cinv[g];
  or_apply_B(c, w, s, 0);
  or_poisson_cheb(c, Cinv, diagKl, s, z, iters, lmin_l, lmax_l);
  free(y); free(s); free(v); free(w);
}

/* Relative residual ||b - K x|| / ||b|| of a Poisson solve (quality check). */
double or_poisson_relres(or_ctx* c, const double* Xinv, const double* b, const double* x) {
  double* q = (double*)malloc(sizeof(double) * c->n_p);
  double* tv = (double*)malloc(sizeof(double) * c->n_v);
  or_apply_K(c, Xinv, x, q, tv);
  double nr = 0.0, nb = 0.0;
  for (int64_t i = 0; i < c->n_p; ++i) { double d = b[i] - q[i]; nr += d * d; nb += b[i] * b[i]; }
  free(q); free(tv);
  return sqrt(nr) / sqrt(nb);
}

int or_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
