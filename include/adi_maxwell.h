/*
 * adi_maxwell.h -- C ABI of libadimaxwell.so, the B200 (sm_100a) hot path of
 * the alternating-direction-implicit isogeometric Maxwell solver of
 * arXiv 2103.06998 (Paszynski, Los, Munoz-Matute).  PAPER.md line numbers are
 * cited as P:<line>; readings of silent/garbled passages as D1..D16
 * (restated in DESIGN.md).
 *
 * What one call of adi_step(k) computes, per time step n -> n+1 (two
 * substeps, P:95-121 scheme1a-scheme1d; discrete form P:233-258
 * discrete1-discrete4):
 *   substep 1: R = M E^n + (tau/2eps) C H^n + (tau^2/4eps mu) R1 E^n      (discrete1)
 *              (M + tau^2/(4 eps mu) K1) E^{n+1/2} = R                    -> 3 sweeps per component
 *              M H^{n+1/2} = M H^n - (tau/2mu) C1 E^n + (tau/2mu) C2 E^{n+1/2}   (discrete2)
 *   substep 2: same with K2, R2 and (discrete4, sign per D2)
 * with per-test-function material (D5): row rst of every system
 * uses a = tau/(2 eps^_rst), b = tau/(2 mu^_rst), c = tau^2/(4 eps^ mu^)_rst,
 * and the stiffened (row-modified) sweep is solved first (D7).
 * PEC by elimination (D1): E_d drops the first and last B-spline along every
 * axis a != d; those coefficients are held at 0.
 *
 * Layout (D14): every field is N^3 doubles, N = n + p, coefficient (i,j,k)
 * at i + N*(j + N*k) (x fastest).  Element (a,b,c) at a + n*(b + n*c).
 * Components: f[0..2] = E1,E2,E3 ; f[3..5] = H1,H2,H3.
 *
 * Pointers: every `const double*` / `double*` argument may be a host pointer
 * or a CUDA device pointer of the patch's device (classified with
 * cudaPointerGetAttributes); copies run on the patch stream.  The caller owns
 * all pointers; the library copies on set_* and never keeps caller pointers
 * beyond the call.  The patch owns its device buffers (cudaMalloc).
 *
 * Errors: every call returns adi_status; no C++ exception crosses the ABI.
 * ADI_ERR_CUDA / ADI_ERR_NCCL poison the patch: every later call except
 * adi_destroy returns the same code.  A failed set_* leaves the previous
 * state intact.  adi_last_error() returns a thread-local message valid until
 * the next call on the same thread.
 *
 * Threading: a patch is not thread-safe; separate patches are independent.
 */
#ifndef ADI_MAXWELL_H
#define ADI_MAXWELL_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct adi_patch_s* adi_patch; /* opaque; owns device state */

typedef enum {
  ADI_OK = 0,
  ADI_ERR_ARG = 1,      /* invalid argument (message names the first offending index) */
  ADI_ERR_STATE = 2,    /* e.g. adi_step before adi_set_fields */
  ADI_ERR_SINGULAR = 3, /* a pivot |u_kk| < 1e-14 max|row| in a factorisation */
  ADI_ERR_CUDA = 4,     /* CUDA runtime error: patch poisoned */
  ADI_ERR_NCCL = 5,     /* NCCL / exchange failure in distributed mode: patch poisoned */
  ADI_ERR_OOM = 6       /* device allocation failed */
} adi_status;

typedef enum { ADI_BC_PEC = 0, ADI_BC_NATURAL = 1 } adi_bc;

typedef struct {
  int32_t n;       /* elements per axis, >= 1 (uniform knots on [0,1], open, C^{p-1}) */
  int32_t p;       /* B-spline degree, 1..5 */
  double tau;      /* time step, finite, > 0 */
  int32_t bc;      /* adi_bc; ADI_BC_PEC (D1) is the paper's Eq. (1) E x n = 0 */
  int32_t device;  /* CUDA device ordinal */
  int32_t rank;    /* this process's rank (0 for a single GPU) */
  int32_t nranks;  /* 1: whole patch on this device; > 1: one z-slab per rank (see below) */
  void* stream;    /* cudaStream_t to run on; NULL = a library-owned non-blocking stream */
  /* Distributed mode (nranks > 1).  Exactly one transport, or neither:
   *   nccl_id:  the 128-byte ncclUniqueId from adi_nccl_unique_id() on rank 0, broadcast to every
   *             rank (e.g. torch.distributed.broadcast_object_list); the patch creates and owns an
   *             NCCL communicator of nranks ranks, one process (or thread) and one GPU per rank.
   *             NCCL is loaded at run time (dlopen "libnccl.so.2"); failures are ADI_ERR_NCCL.
   *   loopback: a group from adi_loopback_create(nranks) shared by nranks patches of ONE process,
   *             each driven by its own host thread (tests / single-device runs): exchanges are
   *             device copies between the patches' buffers ordered by a host barrier (no kernel ever
   *             waits on another rank's kernel).
   *   neither:  "box mode": the patch holds only the 1D operators and the adi_box_* entry points
   *             (the caller owns the slabs and the schedule, e.g. paper_2103_06998_b200.dist). */
  const void* nccl_id;
  void* loopback;
} adi_config;

/* Create a patch: assembles the 1D Galerkin matrices M, S, A (B = A^T) by
 * Gauss quadrature q = p+1 (D4, D11), factors the constant mass sweeps,
 * allocates the field, scratch and material arrays (whole patch: N^3 each; distributed:
 * the rank's z-slab with p halo planes per side, and y-slab work buffers), sets eps = mu = 1.
 * Distributed mode is collective: every rank must call adi_create (and later every set_* and
 * adi_step) with the same arguments except rank.
 * ADI_ERR_ARG: n < 1, p outside 1..5, tau <= 0 / non-finite, bc invalid, rank outside
 * [0, nranks), nranks > N, both nccl_id and loopback given.  ADI_ERR_OOM: device allocation
 * failed.  ADI_ERR_NCCL: communicator creation failed.  *out = NULL on error. */
adi_status adi_create(const adi_config* cfg, adi_patch* out);

/* Rank 0 of a distributed run: writes a fresh ncclUniqueId (128 bytes) to id_out, to be
 * broadcast to all ranks and passed as adi_config.nccl_id.  ADI_ERR_NCCL if NCCL is unavailable. */
adi_status adi_nccl_unique_id(void* id_out);

/* In-process exchange group for nranks patches driven by nranks host threads (loopback
 * transport).  The group must outlive its patches.  ADI_ERR_ARG for nranks < 1. */
adi_status adi_loopback_create(int32_t nranks, void** group_out);
void adi_loopback_destroy(void* group);

/* Free all device state. NULL-safe. */
void adi_destroy(adi_patch patch);

/* N = n + p and the z-slab [k0, k1) held by this patch (the whole grid: 0, N). */
adi_status adi_layout(adi_patch patch, int64_t* N, int64_t* k0, int64_t* k1);

/* Change tau; rebuilds the row factors a, b, c (P:545 with tau^ = tau, D13). */
adi_status adi_set_tau(adi_patch patch, double tau);

/* Element-wise materials eps_elem, mu_elem (n^3 each; mu NULL => 1).  Mapped to
 * test functions by the B-spline-weighted average (D6):
 *   eps^_rst = sum_abc w_ra w_sb w_tc eps_abc,  w_ra = int_{elem a} B_r / int B_r.
 * ADI_ERR_ARG if any value is <= 0 or non-finite (eps, mu >= delta > 0). */
adi_status adi_set_materials(adi_patch patch, const double* eps_elem, const double* mu_elem);

/* Per-test-function materials given directly (N^3 each; mu NULL => 1).
 * Distributed mode: material and source arrays are GLOBAL (the whole patch, given on every
 * rank); each rank keeps its slabs of them. */
adi_status adi_set_materials_tf(adi_patch patch, const double* eps_tf, const double* mu_tf);

/* Set the six coefficient fields: whole patch N^3 each; distributed: the rank's local z-slab,
 * N x N x (k1 - k0) from adi_layout (x fastest, planes k0..k1-1 of the global grid).
 * PEC-eliminated E entries are forced to 0 (D1).  Resets nothing else (step index is kept). */
adi_status adi_set_fields(adi_patch patch, const double* const f[6]);

/* Read the six fields into caller buffers (same extents as adi_set_fields; NULL entries
 * skipped).  Synchronises the patch stream. */
adi_status adi_get_fields(adi_patch patch, double* const f[6]);

/* Sources (D9): in both substeps of step m, R_d -= a (.) signal[m] * load[d],
 * load[d] an N^3 load vector (int j_d B_rst) or NULL; signal[m] = s((m+1/2) tau),
 * 0 past nsig.  load == NULL or nsig == 0 removes the source. */
adi_status adi_set_source(adi_patch patch, const double* const load[3], const double* signal, int64_t nsig);

/* Point dipole j = e_comp delta(x - x_s) s(t): the library evaluates
 * load_rst = B_r(xs) B_s(ys) B_t(zs) itself.  comp in 0..2, x_s in [0,1]^3. */
adi_status adi_set_point_source(adi_patch patch, int32_t comp, double xs, double ys, double zs,
                                const double* signal, int64_t nsig);

/* Advance k >= 0 full time steps.  Asynchronous on the patch stream (the first
 * call for a given patch state captures the step into a CUDA graph; distributed NCCL patches
 * capture the NCCL exchanges into the same graph, loopback patches run eagerly).
 * Distributed mode (collective): per substep a p-plane halo exchange of the six fields before
 * the RHS stencils, x / y sweeps on the z-slab, and every z sweep on y-slabs between batched
 * all-to-all transposes (one exchange per stage for all components); SURVEY §8(e).
 * ADI_ERR_STATE before adi_set_fields. */
adi_status adi_step(adi_patch patch, int64_t k);

/* Order of the three sweeps of each E solve (variant V1):
 * 0 (default): the row-modified (stiffened) axis first, then the two mass sweeps in
 *   ascending order (D7) -- equal to the row-modified global system for any material;
 * 1: the paper's main-text order x -> y -> z, the modified matrix at the
 *   stiffened axis -- exact only when c does not vary along the axes swept before it.
 * ADI_ERR_ARG for other values. */
adi_status adi_set_sweep_order(adi_patch patch, int32_t order);

/* NEXT-2 variant V2: where the material enters the E right-hand sides.
 *   0 (default, D5): every RHS row is scaled by its test function's a = tau/(2 eps^), c =
 *      tau^2/(4 eps^ mu^) (P:545-549 read as "material data of the test B-spline");
 *   2: "element-wise eps, mu" read literally -- the curl and mixed-derivative integrals of the E
 *      right-hand sides carry each element's a_e, c_e INSIDE the Gauss quadrature (q = p + 1 per
 *      element, sum-factorised interpolation / projection); the LHS (row-modified sweeps), the H
 *      updates and the source keep the row factors.  Needs element materials (adi_set_materials;
 *      after adi_set_materials_tf adi_step returns ADI_ERR_STATE) and allocates two (n (p+1))^3
 *      work arrays (ADI_ERR_OOM if they do not fit).  Whole patches only (ADI_ERR_STATE otherwise).
 * ADI_ERR_ARG for other values. */
adi_status adi_set_rhs_variant(adi_patch patch, int32_t variant);

/* NEXT-1 (the linear cost of banded direction solves): how a
 * distributed patch solves its CONSTANT sweeps along the partitioned axis z (the mass sweeps of
 * the E solves, a2/a6, and the M^{-1} of the uniform-mu derivative projections, a3/a4, a7/a8):
 *   1 (default): partitioned (SPIKE) solve in place on the z-slabs -- each rank solves its
 *      diagonal block of the banded matrix, the ranks all-gather 2p interface values per fiber
 *      (instead of the fiber), and every rank finishes with the precomputed rows of the
 *      2pR x 2pR interface system (adi_zsolve_tables); the row-modified z sweep (a per-fiber
 *      matrix M + diag(c) S) all-gathers 2p + 4p^2 spike tips per fiber and eliminates the
 *      block-tridiagonal interface system per fiber: no transposes at all;
 *   0: every z sweep between all-to-all transposes (the per-fiber arithmetic of a whole patch:
 *      bit-identical for any number of ranks).
 * *active (may be NULL) = 1 if mode 1 is in effect: a distributed patch whose every rank holds
 * >= 2p active rows of both PEC ranges.  ADI_ERR_ARG for other modes. */
adi_status adi_set_zsolve(adi_patch patch, int32_t mode, int32_t* active);

/* Host-only (no device): the tables of the partitioned z-solve for rank `rank` of `nranks`
 * (rows of the axis split as adi_layout splits z) of the 1D mass matrix of (n, p) restricted to
 * the active rows [lo, hi) (D1: [0, N) or [1, N-1)).  Outputs (caller-allocated, N = n + p):
 *   *g0, *m: first active row of the rank and its number of active rows;
 *   fac: m x (2p+1) banded LU (no pivoting) of the diagonal block A_r: per row l_{k,k-1-q}
 *        (q < p), 1 / u_kk, u_{k,k+1+q};
 *   tw:  2p x m, rows 0..p-1 and m-p..m-1 of A_r^{-1} (the tips of y = A_r^{-1} f);
 *   cb:  2 p x p: the coupling C_r (rows g0.., columns g0-p..) then B_r (rows g0+m-p.., columns g0+m..);
 *   q:   2p x 2p nranks: rows of K^{-1} (K: the interface system over the tips [t_s, b_s]_s) giving
 *        t_{r+1} (rows 0..p-1) and b_{r-1} (rows p..2p-1), zero where the neighbour is absent.
 * ADI_ERR_ARG: bad sizes, a rank with fewer than 2p active rows, or a singular block. */
adi_status adi_zsolve_tables(int32_t n, int32_t p, int32_t nranks, int32_t rank, int32_t lo, int32_t hi, int32_t* g0,
                             int32_t* m, double* fac, double* tw, double* cb, double* q);

/* On-device diagnostic: out[c] = f_c^T (M (x) M (x) M) f_c for the six
 * fields and out[6] = 1/2 sum_c out[c], the discrete M-norm energy 1/2 (e^T M e + h^T M h)
 * (conserved by the curl part of the scheme).  Synchronises.  Whole patches only. */
adi_status adi_energy(adi_patch patch, double out[7]);

/* On-device diagnostic: errors of the current fields against the
 * manufactured solution u_A(., t) (sign reading D8; valid for eps = mu = 1):
 * out[0] = ||E_h - E||_L2, out[1] = ||H_h - H||_L2, out[2] = ||E_h - E||_H(curl),
 * out[3] = ||H_h - H||_H(curl) (H(curl)^2 = L2^2 + ||curl||^2, exact curl), by Gauss
 * quadrature with q = p + 3 points per axis and element (D11).  Synchronises.  ADI_ERR_ARG
 * for out == NULL; ADI_ERR_STATE for a box-mode patch.  Whole patches only. */
adi_status adi_errors_uA(adi_patch patch, double t, double out[4]);

/* On-device diagnostic: out[0] = ||div E_h||_L2, out[1] = ||div H_h||_L2
 * of the current fields, Gauss q = p + 3 per axis and element.  Synchronises.  ADI_ERR_ARG for
 * out == NULL; ADI_ERR_STATE for a box-mode patch.  Whole patches only. */
adi_status adi_divergence(adi_patch patch, double out[2]);

/* Second workload: the test-function-weighted L2 projection of the
 * Appendix, in 3D: solve K u = f with K = diag(eps^) (M (x) M (x) M), i.e. row i
 * of the Kronecker mass matrix scaled by eps^_i (the coefficient carries the index of the test
 * function).  The Appendix's block splitting (eqs. split1, split2) gives
 * u = (M^-1 (x) M^-1 (x) M^-1)(f / eps^): one division pass and three mass sweeps, O(N^3).
 * f, eps_tf, u: DEVICE pointers to N^3 doubles (x fastest), owned by the caller; u may equal f.
 * Full index range along every axis (no PEC elimination).  Runs on the patch's stream
 * (asynchronous except for the eps check, which synchronises).  ADI_ERR_ARG for NULL pointers
 * or an eps^ entry that is not finite and > 0 (u untouched); ADI_ERR_STATE for a box-mode
 * patch.  Whole patches only. */
adi_status adi_project_weighted(adi_patch patch, const double* f, const double* eps_tf, double* u);

/* Block until all work queued on the patch stream has finished. */
adi_status adi_synchronize(adi_patch patch);

/* Number of full steps taken since creation. */
int64_t adi_step_index(adi_patch patch);

/* Number of kernel launches one adi_step(1) issues (known after the first adi_step). */
int64_t adi_launches_per_step(adi_patch patch);

/* The cudaStream_t the patch runs on. */
void* adi_stream(adi_patch patch);

/* Thread-local message describing the last error (or ""). */
const char* adi_last_error(void);

/* ---- per-kernel timing (bench instrumentation) -------------------------- */
/* Kernel classes used by the timing report. */
enum { ADI_K_RHS_E = 0, ADI_K_RHS_H = 1, ADI_K_SWEEP_MASS = 2, ADI_K_SWEEP_MOD = 3, ADI_K_OTHER = 4,
       ADI_K_SWEEP_DER = 5, ADI_K_NCLASS = 6 };

/* enable != 0: subsequent adi_step calls launch kernels directly (no graph),
 * bracketing each launch with CUDA events on the patch stream; accumulated
 * per-class device time can then be read with adi_timing_report (which
 * synchronises).  enable == 0 resets and disables. */
adi_status adi_set_timing(adi_patch patch, int32_t enable);
adi_status adi_timing_report(adi_patch patch, double ms[ADI_K_NCLASS], int64_t launches[ADI_K_NCLASS]);

/* ---- test-only entry points (per-stage parity) --------------------------- */
/* Host copies of the dense 1D matrices (N x N each, row = test function). */
adi_status adi_debug_matrices(adi_patch patch, double* M, double* S, double* A);
/* Per-test-function eps^, mu^ currently in use (N^3 each). */
adi_status adi_debug_materials_tf(adi_patch patch, double* eps_tf, double* mu_tf);
/* One sweep along `axis` for component comp (0..5 selects the PEC active set);
 * modified != 0 uses M + diag(c) S with the patch's per-row c, else M. */
adi_status adi_debug_sweep(adi_patch patch, int32_t comp, int32_t axis, int32_t modified, const double* rhs, double* out);
/* RHS of the E systems of substep s (1|2) from the current fields. */
adi_status adi_debug_rhs_e(adi_patch patch, int32_t s, double* const R[3]);
/* RHS of the H systems of substep s given Eo (start of substep) and En. */
adi_status adi_debug_rhs_h(adi_patch patch, int32_t s, const double* const Eo[3], const double* const En[3], double* const G[3]);
/* E-component solve of substep s: stiffened sweep first, then the two mass sweeps. */
adi_status adi_debug_solve_e(adi_patch patch, int32_t s, int32_t d, const double* rhs, double* out);

/* ---- box-level entry points (slab-decomposed multi-GPU path) -------------
 * SURVEY §8(e).  A patch created with nranks > 1 is a "box-mode" patch: it holds
 * only the 1D operators (band tables, mass factors, interior constants) and the
 * sweep checkpoints; the caller (paper_2103_06998_b200.dist) owns the slab buffers
 * and drives the schedule -- halo exchange and all-to-all transposes between
 * these calls go over NCCL via torch.distributed.  adi_layout gives the rank's
 * z-slab [r N / R, (r+1) N / R).  All pointers are device pointers of the
 * patch's device, arrays are x fastest; calls are asynchronous on the patch
 * stream unless stated.  The single-patch calls (set_*, step, get_fields)
 * return ADI_ERR_STATE on a box-mode patch. */
typedef struct {
  const double* in;   /* right-hand side (mass / modified) or u (derivative projection) */
  double* out;        /* solution; may alias in (or base) */
  const double* c;    /* modified: per-test-function c = tau^2/(4 eps^ mu^), same layout as in */
  const double* iu;   /* modified: pivot cache from adi_box_factor for the same (comp, axis, layout) */
  const double* base; /* derivative projection: out = base + coef * M^{-1} (A in) along axis */
  double coef;
  int64_t dims[3];    /* box extents; dims[axis] must equal N (fibers span the patch) */
  int32_t axis;       /* 0 = x, 1 = y, 2 = z */
  int32_t comp;       /* 0..5 (E1..H3): PEC row range along axis (D1) */
} adi_sweep_job;

/* 1..3 independent sweeps of one kind in one launch.  mode 0: M x = f; 1: (M + diag(c) S) x = f
 * (no pivoting, D12); 2: derivative projection (uniform-mu H update, SURVEY §8(a) note). */
adi_status adi_box_sweep(adi_patch patch, int32_t mode, int32_t njobs, const adi_sweep_job* jobs);
/* Pivot cache 1/u_kk of the row-modified matrices of component comp along axis for a box
 * layout (dims[axis] = N).  Synchronises; ADI_ERR_SINGULAR on a tiny pivot (D12 gate). */
adi_status adi_box_factor(adi_patch patch, int32_t comp, int32_t axis, const int64_t dims[3], const double* c, double* iu);
/* RHS of the E (kind 0, a1/a5) or H (kind 1, a3/a7) system of component d (0..2) in
 * substep s (1|2) for output planes [kg0, kg0 + nzout) of the patch.  in[t]: the term
 * inputs (order of the kernel programs: E: E_d, H_{d+2}, H_{d+1}, E_sigma; H: H_d, Eo, En),
 * each N x N x nzin, plane zoff + k holding global plane kg0 + k (halo planes around it,
 * zeros outside the patch); a, b, c, load: out layout; sval: source amplitude s((m+1/2)tau) (D9). */
adi_status adi_box_rhs(adi_patch patch, int32_t kind, int32_t s, int32_t d, const double* const in[4], int64_t nzin,
                       int64_t zoff, int64_t kg0, int64_t nzout, const double* a, const double* b, const double* c,
                       const double* load, double sval, double* out);
/* dst[doff + x] = src[soff + x] for x in the box ext (3D strided copy). */
adi_status adi_box_copy(adi_patch patch, double* dst, const int64_t ddims[3], const int64_t doff[3], const double* src,
                        const int64_t sdims[3], const int64_t soff[3], const int64_t ext[3]);
/* Row factors a = tau/(2 eps^), b = tau/(2 mu^), c = tau^2/(4 eps^ mu^) of count entries. */
adi_status adi_box_abc(adi_patch patch, const double* eps_tf, const double* mu_tf, int64_t count, double* a, double* b,
                       double* c);
/* Zero the PEC-eliminated entries (D1) of component comp held in a box at global offset off. */
adi_status adi_box_pec(adi_patch patch, int32_t comp, double* u, const int64_t dims[3], const int64_t off[3]);
/* Element-wise eps, mu (global n^3, host or device; mu NULL => 1) -> per-test-function
 * eps^, mu^ (global N^3 device arrays, D6).  Synchronises. */
adi_status adi_box_materials_tf(adi_patch patch, const double* eps_elem, const double* mu_elem, double* eps_tf,
                                double* mu_tf);

#ifdef __cplusplus
}
#endif
#endif /* ADI_MAXWELL_H */
