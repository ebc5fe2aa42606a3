/*
 * oracle/adi_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow fp64 CPU implementation of the ADI
 * isogeometric Maxwell time step of arXiv 2103.06998 ("PAPER.md" below,
 * cited as P:<line>).  It exists to define "correct" for the CUDA path in
 * paper_2103_06998_b200/ and is pinned by tests/ against values the paper
 * prints, closed forms, and an independent dense brute-force assembly
 * (tests/dense_ref.py).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares NO code with the
 * CUDA path (no headers, helpers, tables or generators).
 *
 * Readings of silent / garbled passages follow SURVEY.md §0 (D1..D16) and
 * are listed in DESIGN.md.  Every Kronecker product is evaluated literally:
 *   [(X (x) Y (x) Z) u]_{rst} = sum_{l,m,o} X_{rl} Y_{sm} Z_{to} u_{lmo}
 * with X acting on x (first index), restricted to the band |r-l|<=p
 * (the entries outside the band are exact zeros, P:429-440 / P:830).
 *
 * Layout (D14): coefficient (i,j,k) -> i + N*(j + N*k), x fastest.
 * Element (a,b,c) -> a + n*(b + n*c).
 * Components: 0..2 = E1,E2,E3 ; 3..5 = H1,H2,H3.
 *
 * Threads: single-threaded unless orc_set_threads(P, t > 1) is called (only
 * tools/make_golden.py does, for the long c4 run).  Then the loops over
 * independent outputs -- the output points of kron3 and the fibers of a
 * sweep -- are split over t OpenMP threads; every output is still computed by
 * exactly the same sequence of operations, so results are bit-identical to the
 * single-threaded run (tests/test_oracle_pins.py::test_threads_bit_identical).
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_ERR_ARG 1
#define ORC_ERR_STATE 2
#define ORC_ERR_SINGULAR 3

static char g_err[512];
static void set_err(const char* m) { snprintf(g_err, sizeof g_err, "%s", m); }
const char* orc_last_error(void) { return g_err; }

typedef struct {
  int n, p, N, bc; /* bc: 0 = PEC by elimination (D1), 1 = natural */
  double tau;
  double* t;  /* knots, n + 2p + 1 */
  double *M, *S, *A; /* dense N x N, [row*N + col], row = test fn, col = trial fn */
  double *epsh, *muh; /* per-test-function material (D5/D6), N^3 */
  double *a, *b, *c;  /* a = tau/(2 eps^), b = tau/(2 mu^), c = tau^2/(4 eps^ mu^) (D13) */
  double* F[6];
  double* load[3];
  double* signal;
  int64_t nsig;
  int64_t step_index;
  int have_fields;
  int order_variant; /* 0 = stiffened axis first (D7), 1 = paper-literal x->y->z (V1) */
  int rhs_variant;   /* 0 = material of the test function on the RHS rows (D5); 2 = element-wise
                        material inside the RHS quadrature (V2) */
  double *eps_el, *mu_el; /* element-wise material of the last orc_set_materials (NULL after _tf) */
  double max_growth; /* max growth factor seen in banded LU (pin P9) */
  int threads;       /* OpenMP threads for the independent-output loops (<= 1: single thread) */
} orc_patch;

static int nthreads(const orc_patch* P) { return P->threads > 1 ? P->threads : 1; }

#define IDX(N, i, j, k) ((int64_t)(i) + (int64_t)(N) * ((int64_t)(j) + (int64_t)(N) * (int64_t)(k)))

/* ------------------------------------------------------------------------- */
/* 1D B-spline space (DS-1)                 */
/* ------------------------------------------------------------------------- */

/* Open uniform knot vector on [0,1]: p+1 zeros, interior knots e/n, p+1 ones. */
static void make_knots(int n, int p, double* t) {
  int m = n + 2 * p + 1;
  for (int i = 0; i < m; i++) {
    if (i <= p) t[i] = 0.0;
    else if (i >= n + p) t[i] = 1.0;
    else t[i] = (double)(i - p) / (double)n;
  }
}

/* Cox-de Boor recursion (values of all N basis functions of degree p at x),
 * plus first derivatives B'_{i,p} = p/(t_{i+p}-t_i) B_{i,p-1}
 *                                  - p/(t_{i+p+1}-t_{i+1}) B_{i+1,p-1}.
 * 0/0 := 0.  Degree-0 functions are indicator functions of [t_i, t_{i+1}),
 * except that the last non-empty interval is closed so that x = 1 is covered. */
static void basis_all(const double* t, int n, int p, double x, double* val, double* der) {
  int m = n + 2 * p + 1; /* number of knots */
  int N = n + p;
  double* B = (double*)calloc((size_t)m * (p + 1), sizeof(double)); /* B[k*m + i] */
  int last = -1;
  for (int i = 0; i + 1 < m; i++)
    if (t[i] < t[i + 1]) last = i;
  for (int i = 0; i + 1 < m; i++) {
    int inside = (t[i] <= x && x < t[i + 1]) || (i == last && x == t[i + 1]);
    B[0 * m + i] = (t[i] < t[i + 1] && inside) ? 1.0 : 0.0;
  }
  for (int k = 1; k <= p; k++) {
    for (int i = 0; i + k + 1 < m; i++) {
      double v = 0.0;
      double d1 = t[i + k] - t[i];
      double d2 = t[i + k + 1] - t[i + 1];
      if (d1 > 0) v += (x - t[i]) / d1 * B[(k - 1) * m + i];
      if (d2 > 0) v += (t[i + k + 1] - x) / d2 * B[(k - 1) * m + i + 1];
      B[k * m + i] = v;
    }
  }
  for (int i = 0; i < N; i++) {
    val[i] = B[p * m + i];
    double d = 0.0;
    if (p >= 1) {
      double d1 = t[i + p] - t[i];
      double d2 = t[i + p + 1] - t[i + 1];
      if (d1 > 0) d += (double)p / d1 * B[(p - 1) * m + i];
      if (d2 > 0) d -= (double)p / d2 * B[(p - 1) * m + i + 1];
    }
    der[i] = d;
  }
  free(B);
}

/* Gauss-Legendre nodes/weights on [-1,1] (Newton iteration on P_q). */
static void legendre(int q, double z, double* pq, double* dpq) {
  double p0 = 1.0, p1 = 0.0;
  for (int j = 1; j <= q; j++) {
    double p2 = p1;
    p1 = p0;
    p0 = ((2.0 * j - 1.0) * z * p1 - (j - 1.0) * p2) / j;
  }
  *pq = p0;
  *dpq = q * (z * p0 - p1) / (z * z - 1.0);
}

static void gauss_legendre(int q, double* x, double* w) {
  for (int i = 0; i < q; i++) {
    double z = cos(M_PI * (i + 0.75) / (q + 0.5)), pq, dp;
    for (int it = 0; it < 100; it++) {
      legendre(q, z, &pq, &dp);
      double dz = pq / dp;
      z -= dz;
      if (fabs(dz) < 1e-16) break;
    }
    legendre(q, z, &pq, &dp);
    x[i] = -z;
    w[i] = 2.0 / ((1.0 - z * z) * dp * dp);
  }
}

/* 1D Galerkin matrices (P:261 + D4, D11: Gauss q = p+1 per element, exact):
 *   M[l][i] = int B_l B_i,  S[l][i] = int B_l' B_i',  A[l][i] = int B_l B_i'
 * (derivative on the trial function i); B = A^T is never stored. */
static void assemble_1d(const double* t, int n, int p, double* M, double* S, double* A) {
  int N = n + p, q = p + 1;
  double gx[16], gw[16];
  gauss_legendre(q, gx, gw);
  double* v = (double*)malloc(sizeof(double) * N);
  double* d = (double*)malloc(sizeof(double) * N);
  memset(M, 0, sizeof(double) * N * N);
  memset(S, 0, sizeof(double) * N * N);
  memset(A, 0, sizeof(double) * N * N);
  for (int e = 0; e < n; e++) {
    double x0 = t[p + e], x1 = t[p + e + 1], h = x1 - x0;
    for (int g = 0; g < q; g++) {
      double x = x0 + 0.5 * h * (gx[g] + 1.0), w = 0.5 * h * gw[g];
      basis_all(t, n, p, x, v, d);
      for (int l = 0; l < N; l++)
        for (int i = 0; i < N; i++) {
          M[l * N + i] += v[l] * v[i] * w;
          S[l * N + i] += d[l] * d[i] * w;
          A[l * N + i] += v[l] * d[i] * w;
        }
    }
  }
  free(v);
  free(d);
}

/* ------------------------------------------------------------------------- */
/* Patch lifetime                                                             */
/* ------------------------------------------------------------------------- */

void orc_destroy(orc_patch* P) {
  if (!P) return;
  free(P->t); free(P->M); free(P->S); free(P->A);
  free(P->epsh); free(P->muh); free(P->a); free(P->b); free(P->c);
  for (int i = 0; i < 6; i++) free(P->F[i]);
  for (int i = 0; i < 3; i++) free(P->load[i]);
  free(P->signal);
  free(P->eps_el); free(P->mu_el);
  free(P);
}

static void derive_abc(orc_patch* P) {
  /* a = tau/(2 eps^), b = tau/(2 mu^), c = tau^2/(4 eps^ mu^): P:233-245 with the
   * material of the test function (D5), tau^ = tau (D13). */
  int64_t U = (int64_t)P->N * P->N * P->N;
  for (int64_t I = 0; I < U; I++) {
    P->a[I] = P->tau / (2.0 * P->epsh[I]);
    P->b[I] = P->tau / (2.0 * P->muh[I]);
    P->c[I] = P->tau * P->tau / (4.0 * P->epsh[I] * P->muh[I]);
  }
}

orc_patch* orc_create(int n, int p, double tau, int bc) {
  if (n < 1 || p < 1 || p > 5 || !(tau > 0) || !isfinite(tau) || (bc != 0 && bc != 1)) {
    set_err("orc_create: invalid argument (need n>=1, 1<=p<=5, finite tau>0, bc in {0,1})");
    return NULL;
  }
  orc_patch* P = (orc_patch*)calloc(1, sizeof(orc_patch));
  P->n = n; P->p = p; P->N = n + p; P->tau = tau; P->bc = bc;
  int N = P->N;
  int64_t U = (int64_t)N * N * N;
  P->t = (double*)malloc(sizeof(double) * (n + 2 * p + 1));
  make_knots(n, p, P->t);
  P->M = (double*)malloc(sizeof(double) * N * N);
  P->S = (double*)malloc(sizeof(double) * N * N);
  P->A = (double*)malloc(sizeof(double) * N * N);
  assemble_1d(P->t, n, p, P->M, P->S, P->A);
  P->epsh = (double*)malloc(sizeof(double) * U);
  P->muh = (double*)malloc(sizeof(double) * U);
  P->a = (double*)malloc(sizeof(double) * U);
  P->b = (double*)malloc(sizeof(double) * U);
  P->c = (double*)malloc(sizeof(double) * U);
  for (int64_t I = 0; I < U; I++) { P->epsh[I] = 1.0; P->muh[I] = 1.0; }
  derive_abc(P);
  for (int i = 0; i < 6; i++) P->F[i] = (double*)calloc(U, sizeof(double));
  return P;
}

int orc_dims(orc_patch* P, int* N) { *N = P->N; return ORC_OK; }
void orc_set_order_variant(orc_patch* P, int v) { P->order_variant = v; }
void orc_set_threads(orc_patch* P, int t) { P->threads = t; }
double orc_max_growth(orc_patch* P) { return P->max_growth; }
int64_t orc_step_index(orc_patch* P) { return P->step_index; }

void orc_knots(orc_patch* P, double* out) { memcpy(out, P->t, sizeof(double) * (P->n + 2 * P->p + 1)); }
void orc_matrices(orc_patch* P, double* M, double* S, double* A) {
  int N = P->N;
  if (M) memcpy(M, P->M, sizeof(double) * N * N);
  if (S) memcpy(S, P->S, sizeof(double) * N * N);
  if (A) memcpy(A, P->A, sizeof(double) * N * N);
}
/* Basis values/derivatives at x (all N functions) -- exposed for pins P1c. */
void orc_basis(orc_patch* P, double x, double* val, double* der) { basis_all(P->t, P->n, P->p, x, val, der); }

int orc_set_tau(orc_patch* P, double tau) {
  if (!(tau > 0) || !isfinite(tau)) { set_err("orc_set_tau: tau must be finite and > 0"); return ORC_ERR_ARG; }
  P->tau = tau;
  derive_abc(P);
  return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* Materials (ALG-12; D5, D6)                                       */
/* ------------------------------------------------------------------------- */

/* w[r*n + a] = int_{element a} B_r / int_0^1 B_r  (D6), by Gauss q=p+1 (exact). */
static void material_weights(orc_patch* P, double* w) {
  int n = P->n, p = P->p, N = P->N, q = p + 1;
  double gx[16], gw[16];
  gauss_legendre(q, gx, gw);
  double* v = (double*)malloc(sizeof(double) * N);
  double* d = (double*)malloc(sizeof(double) * N);
  memset(w, 0, sizeof(double) * N * n);
  for (int e = 0; e < n; e++) {
    double x0 = P->t[p + e], x1 = P->t[p + e + 1], h = x1 - x0;
    for (int g = 0; g < q; g++) {
      double x = x0 + 0.5 * h * (gx[g] + 1.0), ww = 0.5 * h * gw[g];
      basis_all(P->t, n, p, x, v, d);
      for (int r = 0; r < N; r++) w[r * n + e] += v[r] * ww;
    }
  }
  for (int r = 0; r < N; r++) {
    double s = 0.0;
    for (int e = 0; e < n; e++) s += w[r * n + e];
    for (int e = 0; e < n; e++) w[r * n + e] /= s;
  }
  free(v);
  free(d);
}

void orc_material_weights(orc_patch* P, double* w) { material_weights(P, w); }

/* eps^_{rst} = sum_{abc} w_{ra} w_{sb} w_{tc} eps_{abc}  (D6); same for mu. */
int orc_set_materials(orc_patch* P, const double* eps_e, const double* mu_e) {
  int n = P->n, N = P->N, p = P->p;
  int64_t ne = (int64_t)n * n * n, U = (int64_t)N * N * N;
  if (!eps_e) { set_err("orc_set_materials: eps is NULL"); return ORC_ERR_ARG; }
  for (int64_t e = 0; e < ne; e++) {
    if (!(eps_e[e] > 0) || !isfinite(eps_e[e])) { snprintf(g_err, sizeof g_err, "orc_set_materials: eps[%lld] not finite > 0", (long long)e); return ORC_ERR_ARG; }
    if (mu_e && (!(mu_e[e] > 0) || !isfinite(mu_e[e]))) { snprintf(g_err, sizeof g_err, "orc_set_materials: mu[%lld] not finite > 0", (long long)e); return ORC_ERR_ARG; }
  }
  double* w = (double*)malloc(sizeof(double) * N * n);
  material_weights(P, w);
  for (int t = 0; t < N; t++)
    for (int s = 0; s < N; s++)
      for (int r = 0; r < N; r++) {
        double se = 0.0, sm = 0.0;
        for (int c = (t - p > 0 ? t - p : 0); c <= t && c < n; c++)
          for (int b = (s - p > 0 ? s - p : 0); b <= s && b < n; b++)
            for (int a = (r - p > 0 ? r - p : 0); a <= r && a < n; a++) {
              double ww = w[r * n + a] * w[s * n + b] * w[t * n + c];
              int64_t e = a + (int64_t)n * (b + (int64_t)n * c);
              se += ww * eps_e[e];
              sm += ww * (mu_e ? mu_e[e] : 1.0);
            }
        P->epsh[IDX(N, r, s, t)] = se;
        P->muh[IDX(N, r, s, t)] = sm;
      }
  free(w);
  (void)U;
  derive_abc(P);
  free(P->eps_el); free(P->mu_el);
  P->eps_el = (double*)malloc(sizeof(double) * ne);
  P->mu_el = (double*)malloc(sizeof(double) * ne);
  for (int64_t e = 0; e < ne; e++) { P->eps_el[e] = eps_e[e]; P->mu_el[e] = mu_e ? mu_e[e] : 1.0; }
  return ORC_OK;
}

int orc_set_materials_tf(orc_patch* P, const double* eps_tf, const double* mu_tf) {
  free(P->eps_el); free(P->mu_el);
  P->eps_el = P->mu_el = NULL; /* per-test-function input: no element-wise material (V2 unavailable) */
  int64_t U = (int64_t)P->N * P->N * P->N;
  if (!eps_tf) { set_err("orc_set_materials_tf: eps is NULL"); return ORC_ERR_ARG; }
  for (int64_t I = 0; I < U; I++) {
    if (!(eps_tf[I] > 0) || !isfinite(eps_tf[I])) { snprintf(g_err, sizeof g_err, "orc_set_materials_tf: eps[%lld] not finite > 0", (long long)I); return ORC_ERR_ARG; }
    if (mu_tf && (!(mu_tf[I] > 0) || !isfinite(mu_tf[I]))) { snprintf(g_err, sizeof g_err, "orc_set_materials_tf: mu[%lld] not finite > 0", (long long)I); return ORC_ERR_ARG; }
  }
  for (int64_t I = 0; I < U; I++) { P->epsh[I] = eps_tf[I]; P->muh[I] = mu_tf ? mu_tf[I] : 1.0; }
  derive_abc(P);
  return ORC_OK;
}

void orc_get_materials_tf(orc_patch* P, double* eps_tf, double* mu_tf) {
  int64_t U = (int64_t)P->N * P->N * P->N;
  if (eps_tf) memcpy(eps_tf, P->epsh, sizeof(double) * U);
  if (mu_tf) memcpy(mu_tf, P->muh, sizeof(double) * U);
}

/* ------------------------------------------------------------------------- */
/* PEC active sets (D1): E_d uses [0,N) along axis d, [1,N-1) along the other   */
/* two axes; H uses [0,N) everywhere.                                          */
/* ------------------------------------------------------------------------- */

static void active_range(const orc_patch* P, int comp, int axis, int* lo, int* hi) {
  *lo = 0; *hi = P->N;
  if (P->bc == 0 && comp < 3 && axis != comp) { *lo = 1; *hi = P->N - 1; }
}

static int is_active(const orc_patch* P, int comp, int i, int j, int k) {
  int lo, hi, ijk[3] = {i, j, k};
  for (int ax = 0; ax < 3; ax++) {
    active_range(P, comp, ax, &lo, &hi);
    if (ijk[ax] < lo || ijk[ax] >= hi) return 0;
  }
  return 1;
}

static void zero_inactive(const orc_patch* P, int comp, double* u) {
  int N = P->N;
  for (int k = 0; k < N; k++)
    for (int j = 0; j < N; j++)
      for (int i = 0; i < N; i++)
        if (!is_active(P, comp, i, j, k)) u[IDX(N, i, j, k)] = 0.0;
}

int orc_set_fields(orc_patch* P, const double* const* f) {
  int64_t U = (int64_t)P->N * P->N * P->N;
  for (int c = 0; c < 6; c++) {
    if (!f[c]) { set_err("orc_set_fields: NULL field pointer"); return ORC_ERR_ARG; }
  }
  for (int c = 0; c < 6; c++) {
    memcpy(P->F[c], f[c], sizeof(double) * U);
    if (c < 3) zero_inactive(P, c, P->F[c]);
  }
  P->have_fields = 1;
  return ORC_OK;
}

int orc_get_fields(orc_patch* P, double* const* f) {
  int64_t U = (int64_t)P->N * P->N * P->N;
  for (int c = 0; c < 6; c++)
    if (f[c]) memcpy(f[c], P->F[c], sizeof(double) * U);
  return ORC_OK;
}

/* Sources (D9): RHS_E -= a (.) s((n+1/2) tau) J_load in both substeps. */
int orc_set_source(orc_patch* P, const double* const* load, const double* signal, int64_t nsig) {
  int64_t U = (int64_t)P->N * P->N * P->N;
  for (int d = 0; d < 3; d++) {
    free(P->load[d]);
    P->load[d] = NULL;
    if (load && load[d]) {
      P->load[d] = (double*)malloc(sizeof(double) * U);
      memcpy(P->load[d], load[d], sizeof(double) * U);
    }
  }
  free(P->signal);
  P->signal = NULL;
  P->nsig = 0;
  if (signal && nsig > 0) {
    P->signal = (double*)malloc(sizeof(double) * nsig);
    memcpy(P->signal, signal, sizeof(double) * nsig);
    P->nsig = nsig;
  }
  return ORC_OK;
}

/* Load vector of a point source delta(x - x_s): J_rst = B_r(x_s) B_s(y_s) B_t(z_s). */
void orc_point_load(orc_patch* P, double xs, double ys, double zs, double* out) {
  int N = P->N;
  double *vx = malloc(sizeof(double) * N), *vy = malloc(sizeof(double) * N), *vz = malloc(sizeof(double) * N);
  double* d = malloc(sizeof(double) * N);
  basis_all(P->t, P->n, P->p, xs, vx, d);
  basis_all(P->t, P->n, P->p, ys, vy, d);
  basis_all(P->t, P->n, P->p, zs, vz, d);
  for (int k = 0; k < N; k++)
    for (int j = 0; j < N; j++)
      for (int i = 0; i < N; i++) out[IDX(N, i, j, k)] = vx[i] * vy[j] * vz[k];
  free(vx); free(vy); free(vz); free(d);
}

/* ------------------------------------------------------------------------- */
/* Kronecker apply (K-3): out = (X (x) Y (x) Z) u, literal triple sum.         */
/* X acts on x (index i / r), Y on y, Z on z.  Transposed operands (B = A^T)    */
/* are requested with the *T flags: entry (r,l) of B is A[l][r].               */
/* ------------------------------------------------------------------------- */

static double ent(const double* X, int tr, int N, int r, int l) { return tr ? X[l * N + r] : X[r * N + l]; }

static void kron3(const orc_patch* P, const double* X, int xT, const double* Y, int yT, const double* Z, int zT,
                  const double* u, double* out) {
  int N = P->N, p = P->p;
#pragma omp parallel for num_threads(nthreads(P)) schedule(static)
  for (int t = 0; t < N; t++)
    for (int s = 0; s < N; s++)
      for (int r = 0; r < N; r++) {
        double acc = 0.0;
        for (int o = (t - p > 0 ? t - p : 0); o <= t + p && o < N; o++)
          for (int m = (s - p > 0 ? s - p : 0); m <= s + p && m < N; m++) {
            double yz = ent(Y, yT, N, s, m) * ent(Z, zT, N, t, o);
            const double* um = u + IDX(N, 0, m, o);
            for (int l = (r - p > 0 ? r - p : 0); l <= r + p && l < N; l++)
              acc += yz * ent(X, xT, N, r, l) * um[l];
          }
        out[IDX(N, r, s, t)] = acc;
      }
}

/* ------------------------------------------------------------------------- */
/* Banded LU with partial pivoting (D12) for one fiber system.          */
/* Solves  sum_j Amat(i,j) x_j = f_i  for i,j in [0,m), |i-j| <= p.            */
/* Row storage W[i][j-i+p], j-i in [-p, 2p] (fill-in from pivoting).           */
/* ------------------------------------------------------------------------- */

static int band_solve_pp(int m, int p, double* W /* m*(3p+1) */, double* f, double* x, double* growth) {
  int w = 3 * p + 1;
#define AW(i, j) W[(int64_t)(i) * w + ((j) - (i) + p)]
  double amax = 0.0;
  for (int i = 0; i < m; i++)
    for (int j = (i - p > 0 ? i - p : 0); j <= i + p && j < m; j++)
      if (fabs(AW(i, j)) > amax) amax = fabs(AW(i, j));
  for (int k = 0; k < m; k++) {
    int piv = k;
    double best = fabs(AW(k, k));
    for (int i = k + 1; i <= k + p && i < m; i++)
      if (fabs(AW(i, k)) > best) { best = fabs(AW(i, k)); piv = i; }
    if (piv != k) {
      for (int j = k; j <= k + 2 * p && j < m; j++) {
        double tk = (j - k <= 2 * p) ? AW(k, j) : 0.0;
        double tp = (j - piv >= -p && j - piv <= 2 * p) ? AW(piv, j) : 0.0;
        AW(k, j) = tp;
        if (j - piv >= -p && j - piv <= 2 * p) AW(piv, j) = tk;
      }
      double tf = f[k]; f[k] = f[piv]; f[piv] = tf;
    }
    double rowmax = 0.0;
    for (int j = k; j <= k + 2 * p && j < m; j++) if (fabs(AW(k, j)) > rowmax) rowmax = fabs(AW(k, j));
    if (!(fabs(AW(k, k)) >= 1e-14 * rowmax) || rowmax == 0.0) return k + 1;
    for (int i = k + 1; i <= k + p && i < m; i++) {
      double l = AW(i, k) / AW(k, k);
      AW(i, k) = 0.0;
      for (int j = k + 1; j <= k + 2 * p && j < m; j++) AW(i, j) -= l * AW(k, j);
      f[i] -= l * f[k];
    }
  }
  double umax = 0.0;
  for (int k = m - 1; k >= 0; k--) {
    double s = f[k];
    for (int j = k + 1; j <= k + 2 * p && j < m; j++) s -= AW(k, j) * x[j];
    x[k] = s / AW(k, k);
    for (int j = k; j <= k + 2 * p && j < m; j++) if (fabs(AW(k, j)) > umax) umax = fabs(AW(k, j));
  }
  if (growth && amax > 0) *growth = umax / amax;
#undef AW
  return 0;
}

/* One directional sweep (ALG-11/12, K-1/K-2): along `axis`, for every fiber
 * whose other two indices lie in the component's active ranges, solve
 *   sum_j (M[k][j] + c_row(k) S[k][j]) x_j = f_k   on k,j in [lo,hi)
 * where c_row(k) is the per-test-function coefficient of the row's test
 * function rst or 0 for a mass sweep (c == NULL).
 * Rows outside [lo,hi) (PEC-eliminated) are set to 0. In-place on u. */
static int sweep(orc_patch* P, int comp, int axis, const double* c, double* u) {
  int N = P->N, p = P->p;
  int lo, hi;
  active_range(P, comp, axis, &lo, &hi);
  int m = hi - lo;
  int ax1 = (axis + 1) % 3, ax2 = (axis + 2) % 3;
  int lo1, hi1, lo2, hi2;
  active_range(P, comp, ax1, &lo1, &hi1);
  active_range(P, comp, ax2, &lo2, &hi2);
  int64_t nf1 = hi1 - lo1, nfib = nf1 * (hi2 - lo2);
  int64_t bad_fiber = nfib; /* first singular fiber in (q2, q1) loop order */
  int bad_row = 0;
  double gmax = P->max_growth;
#pragma omp parallel num_threads(nthreads(P))
  {
    double* W = (double*)malloc(sizeof(double) * m * (3 * p + 1));
    double* f = (double*)malloc(sizeof(double) * m);
    double* x = (double*)malloc(sizeof(double) * m);
    double gloc = 0.0;
#pragma omp for schedule(static)
    for (int64_t q = 0; q < nfib; q++) {
      int ijk[3];
      ijk[ax1] = lo1 + (int)(q % nf1);
      ijk[ax2] = lo2 + (int)(q / nf1);
      memset(W, 0, sizeof(double) * m * (3 * p + 1));
      for (int k = lo; k < hi; k++) {
        ijk[axis] = k;
        int64_t I = IDX(N, ijk[0], ijk[1], ijk[2]);
        double ck = c ? c[I] : 0.0;
        f[k - lo] = u[I];
        for (int j = (k - p > lo ? k - p : lo); j <= k + p && j < hi; j++)
          W[(int64_t)(k - lo) * (3 * p + 1) + (j - k + p)] = P->M[k * N + j] + ck * P->S[k * N + j];
      }
      double g = 0.0;
      int bad = band_solve_pp(m, p, W, f, x, &g);
      if (bad) {
#pragma omp critical(orc_sweep_bad)
        if (q < bad_fiber) { bad_fiber = q; bad_row = lo + bad - 1; }
        continue;
      }
      if (g > gloc) gloc = g;
      for (int k = lo; k < hi; k++) {
        ijk[axis] = k;
        u[IDX(N, ijk[0], ijk[1], ijk[2])] = x[k - lo];
      }
    }
#pragma omp critical(orc_sweep_growth)
    if (gloc > gmax) gmax = gloc;
    free(W); free(f); free(x);
  }
  P->max_growth = gmax;
  if (bad_fiber < nfib) {
    snprintf(g_err, sizeof g_err, "sweep: singular pivot (comp %d, axis %d, fiber (%d,%d), row %d)", comp, axis,
             lo1 + (int)(bad_fiber % nf1), lo2 + (int)(bad_fiber / nf1), bad_row);
    return ORC_ERR_SINGULAR;
  }
  zero_inactive(P, comp, u); /* rows outside the active set stay 0 */
  return ORC_OK;
}

/* Stiffened axis of E component d (0-based) in substep s (1 or 2):
 * K1: E1->y, E2->z, E3->x ;  K2: E1->z, E2->x, E3->y. */
static int stiff_axis(int s, int d) {
  static const int k1[3] = {1, 2, 0}, k2[3] = {2, 0, 1};
  return s == 1 ? k1[d] : k2[d];
}

/* E solve for one component (ALG-11/12/13): stiffened axis first with the
 * per-row coefficient c (D7), then the two mass sweeps in
 * ascending axis order.  order_variant 1 = paper-literal x->y->z (V1). */
static int solve_E(orc_patch* P, int s, int d, double* u) {
  int sa = stiff_axis(s, d);
  int st;
  if (P->order_variant == 1) {
    for (int ax = 0; ax < 3; ax++)
      if ((st = sweep(P, d, ax, ax == sa ? P->c : NULL, u))) return st;
    return ORC_OK;
  }
  if ((st = sweep(P, d, sa, P->c, u))) return st;
  for (int ax = 0; ax < 3; ax++)
    if (ax != sa && (st = sweep(P, d, ax, NULL, u))) return st;
  return ORC_OK;
}

/* H solve: (M (x) M (x) M)^{-1}, three mass sweeps. */
static int solve_H(orc_patch* P, int d, double* u) {
  int st;
  for (int ax = 0; ax < 3; ax++)
    if ((st = sweep(P, 3 + d, ax, NULL, u))) return st;
  return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* Right-hand sides.                               */
/* ------------------------------------------------------------------------- */

static double source_value(const orc_patch* P) {
  if (P->signal && P->step_index < P->nsig) return P->signal[P->step_index];
  return 0.0;
}

/* RHS of the E systems.
 * Substep 1 (discrete1; expanded in dupa1ab P:373-386):
 *   R1 = M^3 E1 + a.[-(M(x)M(x)A) H2 + (M(x)A(x)M) H3] + c.(A(x)B(x)M) E2
 *   R2 = M^3 E2 + a.[ (M(x)M(x)A) H1 - (A(x)M(x)M) H3] + c.(M(x)A(x)B) E3
 *   R3 = M^3 E3 + a.[-(M(x)A(x)M) H1 + (A(x)M(x)M) H2] + c.(B(x)M(x)A) E1
 * Substep 2 (discrete3; R2 blocks P:253, weak3 P:211-219):
 *   R1 = M^3 E1 + a.[...same C-term...] + c.(A(x)M(x)B) E3
 *   R2 = M^3 E2 + a.[...]               + c.(B(x)A(x)M) E1
 *   R3 = M^3 E3 + a.[...]               + c.(M(x)B(x)A) E2
 * minus a.s.J (D9); rows of PEC-eliminated test functions are zeroed (D1). */
/* ---- NEXT-2 variant V2: element-wise material inside the RHS quadrature ---------------------
 * Literal reading of "element-wise eps, mu" / "RHS-hat with material data": every
 * material-carrying RHS term is the Galerkin integral with the element's coefficient inside,
 *   [sum_e w_e (X^{e_x} (x) Y^{e_y} (x) Z^{e_z}) u]_{rst},
 * X^{a} the element-a part of the 1D matrix X (Gauss q = p+1 on element a: M^a_{il} = int_a B_i B_l,
 * A^a_{il} = int_a B_i B_l', B^a = (A^a)^T), summed element by element (no Kronecker factoring). */
static void element_matrices(const orc_patch* P, double* Me, double* Ae) {
  int n = P->n, p = P->p, N = P->N, q = p + 1, w1 = p + 1;
  double gx[16], gw[16];
  gauss_legendre(q, gx, gw);
  double* v = (double*)malloc(sizeof(double) * N);
  double* d = (double*)malloc(sizeof(double) * N);
  memset(Me, 0, sizeof(double) * n * w1 * w1);
  memset(Ae, 0, sizeof(double) * n * w1 * w1);
  for (int e = 0; e < n; e++) {
    double x0 = P->t[p + e], x1 = P->t[p + e + 1], h = x1 - x0;
    for (int g = 0; g < q; g++) {
      double x = x0 + 0.5 * h * (gx[g] + 1.0), w = 0.5 * h * gw[g];
      basis_all(P->t, n, p, x, v, d);
      for (int i = 0; i <= p; i++)
        for (int l = 0; l <= p; l++) {
          Me[(e * w1 + i) * w1 + l] += v[e + i] * v[e + l] * w;
          Ae[(e * w1 + i) * w1 + l] += v[e + i] * d[e + l] * w;
        }
    }
  }
  free(v);
  free(d);
}

/* op: 0 = M, 1 = A, 2 = B; entry (test i, trial l) of element e's local matrix */
static double eloc(const double* Me, const double* Ae, int p, int op, int e, int i, int l) {
  int w1 = p + 1;
  if (op == 0) return Me[(e * w1 + i) * w1 + l];
  if (op == 1) return Ae[(e * w1 + i) * w1 + l];
  return Ae[(e * w1 + l) * w1 + i];
}

static void kron3_w(const orc_patch* P, const double* Me, const double* Ae, int ox, int oy, int oz,
                    const double* w_el, const double* u, double* out) {
  int n = P->n, p = P->p, N = P->N;
  memset(out, 0, sizeof(double) * (int64_t)N * N * N);
  for (int c = 0; c < n; c++)
    for (int b = 0; b < n; b++)
      for (int a = 0; a < n; a++) {
        double we = w_el[a + (int64_t)n * (b + (int64_t)n * c)];
        for (int k = 0; k <= p; k++)
          for (int j = 0; j <= p; j++)
            for (int i = 0; i <= p; i++) {
              double acc = 0.0;
              for (int o = 0; o <= p; o++)
                for (int m = 0; m <= p; m++)
                  for (int l = 0; l <= p; l++)
                    acc += eloc(Me, Ae, p, ox, a, i, l) * eloc(Me, Ae, p, oy, b, j, m) *
                           eloc(Me, Ae, p, oz, c, k, o) * u[IDX(N, a + l, b + m, c + o)];
              out[IDX(N, a + i, b + j, c + k)] += we * acc;
            }
      }
}

void orc_set_rhs_variant(orc_patch* P, int v) { P->rhs_variant = v; }

/* V2 right-hand sides of the E systems: the D5 terms of rhs_E below with a = tau/(2 eps_e) and
 * c = tau^2/(4 eps_e mu_e) of each element inside the integrals; M^3 E carries no material; the
 * source keeps the row factor of D9. */
static void rhs_E_v2(orc_patch* P, int s, double* const* R) {
  int n = P->n, p = P->p;
  int64_t U = (int64_t)P->N * P->N * P->N, ne = (int64_t)n * n * n;
  double* Me = (double*)malloc(sizeof(double) * n * (p + 1) * (p + 1));
  double* Ae = (double*)malloc(sizeof(double) * n * (p + 1) * (p + 1));
  element_matrices(P, Me, Ae);
  double* ae = (double*)malloc(sizeof(double) * ne);
  double* ce = (double*)malloc(sizeof(double) * ne);
  for (int64_t e = 0; e < ne; e++) {
    ae[e] = P->tau / (2.0 * P->eps_el[e]);
    ce[e] = P->tau * P->tau / (4.0 * P->eps_el[e] * P->mu_el[e]);
  }
  double* t1 = (double*)malloc(sizeof(double) * U);
  double* t2 = (double*)malloc(sizeof(double) * U);
  double* t3 = (double*)malloc(sizeof(double) * U);
  double* t4 = (double*)malloc(sizeof(double) * U);
  double** E = P->F;
  double** H = P->F + 3;
  double sv = source_value(P);
  for (int d = 0; d < 3; d++) {
    kron3(P, P->M, 0, P->M, 0, P->M, 0, E[d], t1);
    if (d == 0) {
      kron3_w(P, Me, Ae, 0, 0, 1, ae, H[1], t2);
      kron3_w(P, Me, Ae, 0, 1, 0, ae, H[2], t3);
      for (int64_t I = 0; I < U; I++) t2[I] = -t2[I] + t3[I];
      if (s == 1) kron3_w(P, Me, Ae, 1, 2, 0, ce, E[1], t4);
      else        kron3_w(P, Me, Ae, 1, 0, 2, ce, E[2], t4);
    } else if (d == 1) {
      kron3_w(P, Me, Ae, 0, 0, 1, ae, H[0], t2);
      kron3_w(P, Me, Ae, 1, 0, 0, ae, H[2], t3);
      for (int64_t I = 0; I < U; I++) t2[I] = t2[I] - t3[I];
      if (s == 1) kron3_w(P, Me, Ae, 0, 1, 2, ce, E[2], t4);
      else        kron3_w(P, Me, Ae, 2, 1, 0, ce, E[0], t4);
    } else {
      kron3_w(P, Me, Ae, 0, 1, 0, ae, H[0], t2);
      kron3_w(P, Me, Ae, 1, 0, 0, ae, H[1], t3);
      for (int64_t I = 0; I < U; I++) t2[I] = -t2[I] + t3[I];
      if (s == 1) kron3_w(P, Me, Ae, 2, 0, 1, ce, E[0], t4);
      else        kron3_w(P, Me, Ae, 0, 2, 1, ce, E[1], t4);
    }
    for (int64_t I = 0; I < U; I++) {
      double v = t1[I] + t2[I] + t4[I];
      if (P->load[d]) v -= P->a[I] * sv * P->load[d][I];
      R[d][I] = v;
    }
    zero_inactive(P, d, R[d]);
  }
  free(t1); free(t2); free(t3); free(t4); free(Me); free(Ae); free(ae); free(ce);
}

static void rhs_E(orc_patch* P, int s, double* const* R) {
  int64_t U = (int64_t)P->N * P->N * P->N;
  const double *M = P->M, *A = P->A;
  double* t1 = (double*)malloc(sizeof(double) * U);
  double* t2 = (double*)malloc(sizeof(double) * U);
  double* t3 = (double*)malloc(sizeof(double) * U);
  double* t4 = (double*)malloc(sizeof(double) * U);
  double** E = P->F;
  double** H = P->F + 3;
  double sv = source_value(P);
  for (int d = 0; d < 3; d++) {
    kron3(P, M, 0, M, 0, M, 0, E[d], t1); /* M^3 E_d */
    if (d == 0) {
      kron3(P, M, 0, M, 0, A, 0, H[1], t2); /* (M M A) H2 */
      kron3(P, M, 0, A, 0, M, 0, H[2], t3); /* (M A M) H3 */
      for (int64_t I = 0; I < U; I++) t2[I] = -t2[I] + t3[I];
      if (s == 1) kron3(P, A, 0, A, 1, M, 0, E[1], t4); /* (A B M) E2 */
      else        kron3(P, A, 0, M, 0, A, 1, E[2], t4); /* (A M B) E3 */
    } else if (d == 1) {
      kron3(P, M, 0, M, 0, A, 0, H[0], t2); /* (M M A) H1 */
      kron3(P, A, 0, M, 0, M, 0, H[2], t3); /* (A M M) H3 */
      for (int64_t I = 0; I < U; I++) t2[I] = t2[I] - t3[I];
      if (s == 1) kron3(P, M, 0, A, 0, A, 1, E[2], t4); /* (M A B) E3 */
      else        kron3(P, A, 1, A, 0, M, 0, E[0], t4); /* (B A M) E1 */
    } else {
      kron3(P, M, 0, A, 0, M, 0, H[0], t2); /* (M A M) H1 */
      kron3(P, A, 0, M, 0, M, 0, H[1], t3); /* (A M M) H2 */
      for (int64_t I = 0; I < U; I++) t2[I] = -t2[I] + t3[I];
      if (s == 1) kron3(P, A, 1, M, 0, A, 0, E[0], t4); /* (B M A) E1 */
      else        kron3(P, M, 0, A, 1, A, 0, E[1], t4); /* (M B A) E2 */
    }
    for (int64_t I = 0; I < U; I++) {
      double v = t1[I] + P->a[I] * t2[I] + P->c[I] * t4[I];
      if (P->load[d]) v -= P->a[I] * sv * P->load[d][I];
      R[d][I] = v;
    }
    zero_inactive(P, d, R[d]);
  }
  free(t1); free(t2); free(t3); free(t4);
}

/* RHS of the H systems, with Eo = E at the start of the substep and
 * En = the freshly solved E.
 * Substep 1 (discrete2; C1, C2 blocks P:254-255 with D3):
 *   G1 = M^3 H1 - b.(M(x)A(x)M) Eo3 + b.(M(x)M(x)A) En2
 *   G2 = M^3 H2 - b.(M(x)M(x)A) Eo1 + b.(A(x)M(x)M) En3
 *   G3 = M^3 H3 - b.(A(x)M(x)M) Eo2 + b.(M(x)A(x)M) En1
 * Substep 2 (discrete4, P:244 with the sign of P:120/P:226, D2):
 *   G1 = M^3 H1 + b.(M(x)M(x)A) Eo2 - b.(M(x)A(x)M) En3
 *   G2 = M^3 H2 + b.(A(x)M(x)M) Eo3 - b.(M(x)M(x)A) En1
 *   G3 = M^3 H3 + b.(M(x)A(x)M) Eo1 - b.(A(x)M(x)M) En2                       */
static void rhs_H(orc_patch* P, int s, double* const* Eo, double* const* En, double* const* G) {
  int64_t U = (int64_t)P->N * P->N * P->N;
  const double *M = P->M, *A = P->A;
  double* t1 = (double*)malloc(sizeof(double) * U);
  double* t2 = (double*)malloc(sizeof(double) * U);
  double* t3 = (double*)malloc(sizeof(double) * U);
  double** H = P->F + 3;
  for (int d = 0; d < 3; d++) {
    kron3(P, M, 0, M, 0, M, 0, H[d], t1);
    double sg2, sg3;
    if (s == 1) {
      sg2 = -1.0; sg3 = +1.0;
      if (d == 0) { kron3(P, M, 0, A, 0, M, 0, Eo[2], t2); kron3(P, M, 0, M, 0, A, 0, En[1], t3); }
      else if (d == 1) { kron3(P, M, 0, M, 0, A, 0, Eo[0], t2); kron3(P, A, 0, M, 0, M, 0, En[2], t3); }
      else { kron3(P, A, 0, M, 0, M, 0, Eo[1], t2); kron3(P, M, 0, A, 0, M, 0, En[0], t3); }
    } else {
      sg2 = +1.0; sg3 = -1.0;
      if (d == 0) { kron3(P, M, 0, M, 0, A, 0, Eo[1], t2); kron3(P, M, 0, A, 0, M, 0, En[2], t3); }
      else if (d == 1) { kron3(P, A, 0, M, 0, M, 0, Eo[2], t2); kron3(P, M, 0, M, 0, A, 0, En[0], t3); }
      else { kron3(P, M, 0, A, 0, M, 0, Eo[0], t2); kron3(P, A, 0, M, 0, M, 0, En[1], t3); }
    }
    for (int64_t I = 0; I < U; I++) G[d][I] = t1[I] + P->b[I] * (sg2 * t2[I] + sg3 * t3[I]);
  }
  free(t1); free(t2); free(t3);
}

/* One substep (ALG-2/ALG-7): RHS_E -> E solve -> RHS_H -> H solve. */
static int substep(orc_patch* P, int s) {
  int64_t U = (int64_t)P->N * P->N * P->N;
  double *R[3], *Eo[3], *G[3];
  int st = ORC_OK;
  for (int d = 0; d < 3; d++) {
    R[d] = (double*)malloc(sizeof(double) * U);
    Eo[d] = (double*)malloc(sizeof(double) * U);
    G[d] = (double*)malloc(sizeof(double) * U);
    memcpy(Eo[d], P->F[d], sizeof(double) * U);
  }
  if (P->rhs_variant == 2) rhs_E_v2(P, s, R);
  else rhs_E(P, s, R);
  for (int d = 0; d < 3 && st == ORC_OK; d++) st = solve_E(P, s, d, R[d]);
  if (st == ORC_OK) {
    rhs_H(P, s, Eo, R, G);
    for (int d = 0; d < 3 && st == ORC_OK; d++) st = solve_H(P, d, G[d]);
  }
  if (st == ORC_OK)
    for (int d = 0; d < 3; d++) {
      memcpy(P->F[d], R[d], sizeof(double) * U);
      memcpy(P->F[3 + d], G[d], sizeof(double) * U);
    }
  for (int d = 0; d < 3; d++) { free(R[d]); free(Eo[d]); free(G[d]); }
  return st;
}

int orc_step(orc_patch* P, int64_t k) {
  if (!P->have_fields) { set_err("orc_step: fields not set"); return ORC_ERR_STATE; }
  if (P->rhs_variant == 2 && !P->eps_el) { set_err("orc_step: V2 needs element-wise materials (orc_set_materials)"); return ORC_ERR_STATE; }
  if (k < 0) { set_err("orc_step: k < 0"); return ORC_ERR_ARG; }
  for (int64_t i = 0; i < k; i++) {
    int st;
    if ((st = substep(P, 1))) return st;
    if ((st = substep(P, 2))) return st;
    P->step_index++;
  }
  return ORC_OK;
}

/* ---- debug entry points (per-stage parity / pins) ----------------------- */

/* RHS of the E systems of substep s from the current fields (3 outputs). */
int orc_debug_rhs_e(orc_patch* P, int s, double* const* R) {
  if (P->rhs_variant == 2) {
    if (!P->eps_el) { set_err("orc_debug_rhs_e: V2 needs element-wise materials"); return ORC_ERR_STATE; }
    rhs_E_v2(P, s, R);
  } else {
    rhs_E(P, s, R);
  }
  return ORC_OK;
}

/* RHS of the H systems of substep s, given Eo (start of substep) and En. */
int orc_debug_rhs_h(orc_patch* P, int s, double* const* Eo, double* const* En, double* const* G) {
  rhs_H(P, s, Eo, En, G);
  return ORC_OK;
}

/* E-component solve (in place): stiffened-first three sweeps. */
int orc_debug_solve_e(orc_patch* P, int s, int d, double* u) { return solve_E(P, s, d, u); }

/* Single sweep: comp in 0..5 selects the active set; modified != 0 uses the
 * patch's c = tau^2/(4 eps^ mu^) per row. In place. */
int orc_debug_sweep(orc_patch* P, int comp, int axis, int modified, double* u) {
  return sweep(P, comp, axis, modified ? P->c : NULL, u);
}

/* Single sweep with caller-provided per-row coefficient (N^3). */
int orc_debug_sweep_c(orc_patch* P, int comp, int axis, const double* c, double* u) { return sweep(P, comp, axis, c, u); }

/* Kronecker apply with 1D operators chosen by code: 0=M, 1=A, 2=B(=A^T), 3=S. */
void orc_debug_kron(orc_patch* P, int ox, int oy, int oz, const double* u, double* out) {
  const double* mats[4] = {P->M, P->A, P->A, P->S};
  int trs[4] = {0, 0, 1, 0};
  kron3(P, mats[ox], trs[ox], mats[oy], trs[oy], mats[oz], trs[oz], u, out);
}

/* ------------------------------------------------------------------------- */
/* Manufactured solution (ALG-14, with D8) and error norms         */
/* (ALG-15).                                                        */
/* ------------------------------------------------------------------------- */

/* u_A = g u^1_{1,1} + 2g u^2_{1,1} + 3g u^3_{1,1}, g = 2/sqrt(14),
 * omega = sqrt(2) pi.  u^2's H components carry the sign fix D8.
 * out[0..2] = E, out[3..5] = H, curl[0..2] = curl E, curl[3..5] = curl H. */
void orc_exact_uA(double x, double y, double z, double t, double* out, double* curl) {
  const double g = 2.0 / sqrt(14.0), pi = M_PI, r = 1.0 / sqrt(2.0), w = sqrt(2.0) * M_PI;
  double sx = sin(pi * x), cx = cos(pi * x), sy = sin(pi * y), cy = cos(pi * y), sz = sin(pi * z), cz = cos(pi * z);
  double ct = cos(w * t), st = sin(w * t);
  /* u1: E1 = sy sz ct, H2 = -r sy cz st, H3 = r cy sz st */
  /* u2 (D8): E2 = sx sz ct, H1 = +r sx cz st, H3 = -r cx sz st */
  /* u3: E3 = sx sy ct, H1 = -r sx cy st, H2 = r cx sy st */
  double c1 = g, c2 = 2 * g, c3 = 3 * g;
  double E1 = c1 * sy * sz * ct, E2 = c2 * sx * sz * ct, E3 = c3 * sx * sy * ct;
  double H1 = c2 * r * sx * cz * st - c3 * r * sx * cy * st;
  double H2 = -c1 * r * sy * cz * st + c3 * r * cx * sy * st;
  double H3 = c1 * r * cy * sz * st - c2 * r * cx * sz * st;
  if (out) { out[0] = E1; out[1] = E2; out[2] = E3; out[3] = H1; out[4] = H2; out[5] = H3; }
  if (curl) {
    /* derivatives, by hand */
    double dE1dy = c1 * pi * cy * sz * ct, dE1dz = c1 * pi * sy * cz * ct;
    double dE2dx = c2 * pi * cx * sz * ct, dE2dz = c2 * pi * sx * cz * ct;
    double dE3dx = c3 * pi * cx * sy * ct, dE3dy = c3 * pi * sx * cy * ct;
    double dH1dy = c3 * r * pi * sx * sy * st;                      /* d/dy of -c3 r sx cy st */
    double dH1dz = -c2 * r * pi * sx * sz * st;                     /* d/dz of  c2 r sx cz st */
    double dH2dx = -c3 * r * pi * sx * sy * st;                     /* d/dx of  c3 r cx sy st */
    double dH2dz = c1 * r * pi * sy * sz * st;                      /* d/dz of -c1 r sy cz st */
    double dH3dx = c2 * r * pi * sx * sz * st;                      /* d/dx of -c2 r cx sz st */
    double dH3dy = -c1 * r * pi * sy * sz * st;                     /* d/dy of  c1 r cy sz st */
    curl[0] = dE3dy - dE2dz; curl[1] = dE1dz - dE3dx; curl[2] = dE2dx - dE1dy;
    curl[3] = dH3dy - dH2dz; curl[4] = dH1dz - dH3dx; curl[5] = dH2dx - dH1dy;
  }
}

/* 1D tables of the p+1 basis functions that are non-zero on element e
 * (indices e..e+p) and their derivatives, at the q Gauss points of e.
 * tab[((e*q + g)*(p+1) + j)*2 + {0: value, 1: derivative}] for B_{e+j}. */
static double* basis_table(orc_patch* P, int q, const double* gx) {
  int n = P->n, p = P->p, N = P->N;
  double* tab = (double*)malloc(sizeof(double) * n * q * (p + 1) * 2);
  double *v = malloc(sizeof(double) * N), *d = malloc(sizeof(double) * N);
  for (int e = 0; e < n; e++)
    for (int g = 0; g < q; g++) {
      double x0 = P->t[p + e], h = P->t[p + e + 1] - x0;
      basis_all(P->t, n, p, x0 + 0.5 * h * (gx[g] + 1.0), v, d);
      for (int j = 0; j <= p; j++) {
        tab[((e * q + g) * (p + 1) + j) * 2 + 0] = v[e + j];
        tab[((e * q + g) * (p + 1) + j) * 2 + 1] = d[e + j];
      }
    }
  free(v); free(d);
  return tab;
}

/* Errors of the current fields against u_A(., t):
 * out[0] = ||E_h - E||_L2, out[1] = ||H_h - H||_L2,
 * out[2] = ||E_h - E||_Hcurl, out[3] = ||H_h - H||_Hcurl
 * (H(curl) = sqrt(L2^2 + ||curl(.)||^2), exact curl).  Gauss q = p+3 (D11).
 * Only the (p+1)^3 basis functions non-zero on an element are summed. */
void orc_errors_uA(orc_patch* P, double t, double* out) {
  int n = P->n, p = P->p, q = p + 3, N = P->N, pp = p + 1;
  double gx[16], gw[16];
  gauss_legendre(q, gx, gw);
  double* tab = basis_table(P, q, gx);
  double eE = 0, eH = 0, cE = 0, cH = 0;
  for (int ec = 0; ec < n; ec++)
    for (int eb = 0; eb < n; eb++)
      for (int ea = 0; ea < n; ea++) {
        double hx = P->t[p + ea + 1] - P->t[p + ea], hy = P->t[p + eb + 1] - P->t[p + eb], hz = P->t[p + ec + 1] - P->t[p + ec];
        for (int gk = 0; gk < q; gk++)
          for (int gj = 0; gj < q; gj++)
            for (int gi = 0; gi < q; gi++) {
              double x = P->t[p + ea] + 0.5 * hx * (gx[gi] + 1), y = P->t[p + eb] + 0.5 * hy * (gx[gj] + 1), z = P->t[p + ec] + 0.5 * hz * (gx[gk] + 1);
              double w = gw[gi] * gw[gj] * gw[gk] * (0.5 * hx) * (0.5 * hy) * (0.5 * hz);
              const double* tx = tab + (ea * q + gi) * pp * 2;
              const double* ty = tab + (eb * q + gj) * pp * 2;
              const double* tz = tab + (ec * q + gk) * pp * 2;
              double g[6][4];
              memset(g, 0, sizeof g);
              for (int c = 0; c < 6; c++)
                for (int kk = 0; kk <= p; kk++)
                  for (int jj = 0; jj <= p; jj++)
                    for (int ii = 0; ii <= p; ii++) {
                      double u = P->F[c][IDX(N, ea + ii, eb + jj, ec + kk)];
                      g[c][0] += u * tx[2 * ii] * ty[2 * jj] * tz[2 * kk];
                      g[c][1] += u * tx[2 * ii + 1] * ty[2 * jj] * tz[2 * kk];
                      g[c][2] += u * tx[2 * ii] * ty[2 * jj + 1] * tz[2 * kk];
                      g[c][3] += u * tx[2 * ii] * ty[2 * jj] * tz[2 * kk + 1];
                    }
              double cu[6];
              cu[0] = g[2][2] - g[1][3]; cu[1] = g[0][3] - g[2][1]; cu[2] = g[1][1] - g[0][2];
              cu[3] = g[5][2] - g[4][3]; cu[4] = g[3][3] - g[5][1]; cu[5] = g[4][1] - g[3][2];
              double ex[6], ecu[6];
              orc_exact_uA(x, y, z, t, ex, ecu);
              for (int c = 0; c < 3; c++) {
                eE += w * (g[c][0] - ex[c]) * (g[c][0] - ex[c]);
                eH += w * (g[3 + c][0] - ex[3 + c]) * (g[3 + c][0] - ex[3 + c]);
                cE += w * (cu[c] - ecu[c]) * (cu[c] - ecu[c]);
                cH += w * (cu[3 + c] - ecu[3 + c]) * (cu[3 + c] - ecu[3 + c]);
              }
            }
      }
  free(tab);
  out[0] = sqrt(eE); out[1] = sqrt(eH); out[2] = sqrt(eE + cE); out[3] = sqrt(eH + cH);
}

/* L2 projection of u_A(., t) onto the discrete spaces (D10): load vectors by
 * Gauss q = p+3 over each element, restricted to active test functions, then
 * the Kronecker mass solve (three mass sweeps) on the active sub-block.
 * Writes the projected fields into the patch (and marks fields as set). */
int orc_project_uA(orc_patch* P, double t) {
  int n = P->n, p = P->p, N = P->N, q = p + 3, pp = p + 1;
  int64_t U = (int64_t)N * N * N;
  double gx[16], gw[16];
  gauss_legendre(q, gx, gw);
  double* tab = basis_table(P, q, gx);
  double* L[6];
  for (int c = 0; c < 6; c++) L[c] = (double*)calloc(U, sizeof(double));
  for (int ec = 0; ec < n; ec++)
    for (int eb = 0; eb < n; eb++)
      for (int ea = 0; ea < n; ea++) {
        double hx = P->t[p + ea + 1] - P->t[p + ea], hy = P->t[p + eb + 1] - P->t[p + eb], hz = P->t[p + ec + 1] - P->t[p + ec];
        for (int gk = 0; gk < q; gk++)
          for (int gj = 0; gj < q; gj++)
            for (int gi = 0; gi < q; gi++) {
              double x = P->t[p + ea] + 0.5 * hx * (gx[gi] + 1), y = P->t[p + eb] + 0.5 * hy * (gx[gj] + 1), z = P->t[p + ec] + 0.5 * hz * (gx[gk] + 1);
              double w = gw[gi] * gw[gj] * gw[gk] * (0.5 * hx) * (0.5 * hy) * (0.5 * hz);
              const double* tx = tab + (ea * q + gi) * pp * 2;
              const double* ty = tab + (eb * q + gj) * pp * 2;
              const double* tz = tab + (ec * q + gk) * pp * 2;
              double ex[6];
              orc_exact_uA(x, y, z, t, ex, NULL);
              for (int kk = 0; kk <= p; kk++)
                for (int jj = 0; jj <= p; jj++)
                  for (int ii = 0; ii <= p; ii++) {
                    double B = tx[2 * ii] * ty[2 * jj] * tz[2 * kk] * w;
                    for (int c = 0; c < 6; c++) L[c][IDX(N, ea + ii, eb + jj, ec + kk)] += ex[c] * B;
                  }
            }
      }
  free(tab);
  int st = ORC_OK;
  for (int c = 0; c < 6 && st == ORC_OK; c++) {
    if (c < 3) zero_inactive(P, c, L[c]);
    for (int ax = 0; ax < 3 && st == ORC_OK; ax++) st = sweep(P, c, ax, NULL, L[c]);
  }
  if (st == ORC_OK) {
    for (int c = 0; c < 6; c++) memcpy(P->F[c], L[c], sizeof(double) * U);
    P->have_fields = 1;
  }
  for (int c = 0; c < 6; c++) free(L[c]);
  return st;
}

/* ------------------------------------------------------------------------- */
/* NEXT-4: the test-function-weighted L2 projection of the Appendix            */
/* (P:680-830), written in 3D.  The system (with the coefficient    */
/* carrying the index of the test function) is                      */
/*   sum_J eps_I (M (x) M (x) M)_{IJ} u_J = f_I .                               */
/* Step by step as the Appendix splits it:                                     */
/*  (split1) for every (j,k), the x-block A_{jk} = the x mass       */
/*    matrix with row i multiplied by eps_{ijk}, solved for        */
/*    G_{.jk}:  A_{jk} G_{.jk} = F_{.jk};                                      */
/*  (split2) the remaining Kronecker mass systems: M along y, then  */
/*    M along z (the 2D example has one; 3D has two).                          */
/* Banded LU with partial pivoting per fiber; full index range (no PEC).       */
/* ------------------------------------------------------------------------- */
int orc_project_weighted(orc_patch* P, const double* f, const double* eps, double* u) {
  int N = P->N, p = P->p;
  for (int64_t I = 0; I < (int64_t)N * N * N; I++)
    if (!(eps[I] > 0.0) || !isfinite(eps[I])) { set_err("project_weighted: eps must be finite and > 0"); return ORC_ERR_ARG; }
  memcpy(u, f, sizeof(double) * (size_t)N * N * N);
  double* W = (double*)malloc(sizeof(double) * N * (3 * p + 1));
  double* g = (double*)malloc(sizeof(double) * N);
  double* x = (double*)malloc(sizeof(double) * N);
  int status = ORC_OK;
  /* (split1) x-blocks with eps-scaled rows */
  for (int k = 0; k < N && status == ORC_OK; k++)
    for (int j = 0; j < N && status == ORC_OK; j++) {
      memset(W, 0, sizeof(double) * N * (3 * p + 1));
      for (int i = 0; i < N; i++) {
        double e = eps[IDX(N, i, j, k)];
        g[i] = u[IDX(N, i, j, k)];
        for (int l = (i - p > 0 ? i - p : 0); l <= i + p && l < N; l++)
          W[(int64_t)i * (3 * p + 1) + (l - i + p)] = e * P->M[i * N + l];
      }
      if (band_solve_pp(N, p, W, g, x, NULL)) { set_err("project_weighted: singular x-block"); status = ORC_ERR_SINGULAR; break; }
      for (int i = 0; i < N; i++) u[IDX(N, i, j, k)] = x[i];
    }
  free(W); free(g); free(x);
  if (status != ORC_OK) return status;
  /* (split2) the mass systems along y and z (component 3 = H1: full range under either BC) */
  if ((status = sweep(P, 3, 1, NULL, u)) != ORC_OK) return status;
  return sweep(P, 3, 2, NULL, u);
}
