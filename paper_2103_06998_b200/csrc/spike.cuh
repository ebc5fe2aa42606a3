// spike.cuh -- NEXT-1: the constant banded solves along the PARTITIONED axis z of the
// slab decomposition, solved where the data lives instead of behind two all-to-all transposes.
//
// The paper keeps the cost of every direction solve linear through the banded structure of the 1D
// matrices.  Rank r owns the z-rows [g0, g0 + m) of every z-fiber (after the PEC
// restriction, D1).  For a constant matrix X (the mass matrix M: the mass sweeps of the E solves,
// and the M^{-1} of the uniform-mu derivative projections) the global system splits as
//     A_r x_r = w_r - [C_r b_{r-1}; 0] - [0; B_r t_{r+1}]
// with A_r the diagonal block of the rank, C_r / B_r the p x p couplings to the last p rows b_{r-1}
// of rank r-1 and the first p rows t_{r+1} of rank r+1.  With y_r = A_r^{-1} w_r the interface
// values solve a 2pR x 2pR system K xi = [y_s^top, y_s^bot]_s whose matrix depends only on X and the
// partition (SPIKE; the host precomputes K^{-1}'s rows Q_r for the values rank r needs).  Per fiber:
//   spike_tips_kernel:  the 2p tips of y_r = rows {0..p-1, m-p..m-1} of A_r^{-1} applied to w_r
//                       (tip weights tw, one streaming read of the fiber segment);
//   (all-gather of the tips: 2p values per fiber and rank instead of the fiber itself)
//   spike_solve_kernel: (t_{r+1}, b_{r-1}) = Q_r tips, the corrected right-hand side, and the banded
//                       LU solve of A_r (factors fac, no pivoting: M is SPD) -- forward elimination
//                       into gbuf, back substitution into out.
// Mass sweep: w = f.  Derivative projection (uniform mu, SURVEY §8(a) note): w = A u along z from the
// halo'd input (p planes per side), out = base + coef x.
// One thread per z-fiber; the 32 lanes of a warp take 32 consecutive x (256-byte rows, coalesced).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace adi {

struct SpikeTabDev {
  const double* fac;  // m x W: l_{k,k-1-q} (q < P), 1/u_kk, u_{k,k+1+q}
  const double* tw;   // 2P x m tip weights
  const double* cb;   // C_r (P x P) then B_r (P x P)
  const double* q;    // 2P x 2PR
  int g0l, m;         // first active plane (rank-local), active planes
};

struct SpikeJob {
  const double* in;    // mass: f; derivative projection: u (halo'd, planes -P .. nz+P-1 readable)
  const double* base;  // derivative projection
  double* out;
  double* gbuf;        // forward-elimination values (may be out; never base)
  double coef;
  int der, v;
};

struct SpikeBatch {
  int64_t NN;           // fibers per job (N * N)
  int nz, njobs, R, N, k0;
  SpikeJob job[3];
  SpikeTabDev tab[2];
  const double* Ab;     // band rows of A (global row g: Ab + g W)
  double* tips;         // [job][2P][NN]
  const double* gath;   // [R][job][2P][NN]
};

template <int P>
__global__ void __launch_bounds__(256) spike_tips_kernel(const __grid_constant__ SpikeBatch B) {
  constexpr int W = 2 * P + 1;
  const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= B.NN) return;
  const SpikeJob& J = B.job[blockIdx.y];
  const SpikeTabDev& T = B.tab[J.v];
  const int64_t NN = B.NN;
  double acc[2 * P];
#pragma unroll
  for (int i = 0; i < 2 * P; i++) acc[i] = 0.0;
  const double* in = J.in + f;
  if (!J.der) {
    for (int k = 0; k < T.m; k++) {
      const double w = in[(int64_t)(T.g0l + k) * NN];
#pragma unroll
      for (int i = 0; i < 2 * P; i++) acc[i] = fma(__ldg(T.tw + (int64_t)i * T.m + k), w, acc[i]);
    }
  } else {
    double u[W];  // window of planes g0l + k - P .. g0l + k + P
#pragma unroll
    for (int q = 0; q < W - 1; q++) u[q] = in[(int64_t)(T.g0l - P + q) * NN];
    for (int k = 0; k < T.m; k++) {
      u[W - 1] = in[(int64_t)(T.g0l + k + P) * NN];
      const double* a = B.Ab + (int64_t)(B.k0 + T.g0l + k) * W;
      double w = 0.0;
#pragma unroll
      for (int q = 0; q < W; q++) w = fma(__ldg(a + q), u[q], w);
#pragma unroll
      for (int i = 0; i < 2 * P; i++) acc[i] = fma(__ldg(T.tw + (int64_t)i * T.m + k), w, acc[i]);
#pragma unroll
      for (int q = 0; q < W - 1; q++) u[q] = u[q + 1];
    }
  }
#pragma unroll
  for (int i = 0; i < 2 * P; i++) B.tips[((int64_t)blockIdx.y * 2 * P + i) * NN + f] = acc[i];
}

template <int P>
__global__ void __launch_bounds__(256) spike_solve_kernel(const __grid_constant__ SpikeBatch B) {
  constexpr int W = 2 * P + 1;
  const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= B.NN) return;
  const SpikeJob& J = B.job[blockIdx.y];
  const SpikeTabDev& T = B.tab[J.v];
  const int64_t NN = B.NN;
  const int m = T.m;
  // interface values: tn = t_{r+1} (rows 0..P-1 of Q), bp = b_{r-1} (rows P..2P-1)
  double tb[2 * P];
#pragma unroll
  for (int i = 0; i < 2 * P; i++) tb[i] = 0.0;
  const int nK = 2 * P * B.R;
  for (int c = 0; c < nK; c++) {
    const int s = c / (2 * P), i = c - s * 2 * P;
    const double y = B.gath[(((int64_t)s * B.njobs + blockIdx.y) * 2 * P + i) * NN + f];
#pragma unroll
    for (int j = 0; j < 2 * P; j++) tb[j] = fma(__ldg(T.q + (int64_t)j * nK + c), y, tb[j]);
  }
  const double* in = J.in + f;
  double* gb = J.gbuf + f;
  double* out = J.out + f;
  // forward elimination of the corrected right-hand side
  double g[P + 1];  // g[0] = newest
#pragma unroll
  for (int q = 0; q <= P; q++) g[q] = 0.0;
  double u[W];
  if (J.der) {
#pragma unroll
    for (int q = 0; q < W - 1; q++) u[q] = in[(int64_t)(T.g0l - P + q) * NN];
  }
  for (int k = 0; k < m; k++) {
    const int64_t pl = (int64_t)(T.g0l + k) * NN;
    double w;
    if (!J.der) {
      w = in[pl];
    } else {
      u[W - 1] = in[(int64_t)(T.g0l + k + P) * NN];
      const double* a = B.Ab + (int64_t)(B.k0 + T.g0l + k) * W;
      w = 0.0;
#pragma unroll
      for (int q = 0; q < W; q++) w = fma(__ldg(a + q), u[q], w);
#pragma unroll
      for (int q = 0; q < W - 1; q++) u[q] = u[q + 1];
    }
    if (k < P) {
#pragma unroll
      for (int j = 0; j < P; j++) w = fma(-__ldg(T.cb + k * P + j), tb[P + j], w);
    }
    if (k >= m - P) {
#pragma unroll
      for (int j = 0; j < P; j++) w = fma(-__ldg(T.cb + P * P + (k - (m - P)) * P + j), tb[j], w);
    }
    const double* fr = T.fac + (int64_t)k * W;
#pragma unroll
    for (int q = P; q > 0; q--) g[q] = g[q - 1];
    double s = w;
#pragma unroll
    for (int q = 0; q < P; q++) s = fma(-__ldg(fr + q), g[q + 1], s);
    g[0] = s;
    gb[pl] = s;
  }
  // back substitution
  double x[P + 1];
#pragma unroll
  for (int q = 0; q <= P; q++) x[q] = 0.0;
  for (int k = m - 1; k >= 0; k--) {
    const int64_t pl = (int64_t)(T.g0l + k) * NN;
    const double* fr = T.fac + (int64_t)k * W;
#pragma unroll
    for (int q = P; q > 0; q--) x[q] = x[q - 1];
    double s = gb[pl];
#pragma unroll
    for (int q = 0; q < P; q++) s = fma(-__ldg(fr + P + 1 + q), x[q + 1], s);
    x[0] = s * __ldg(fr + P);
    out[pl] = J.der ? fma(J.coef, x[0], J.base[f + pl]) : x[0];
  }
  // rows of the slab outside the active range (PEC, D1): stored zeros
  for (int k = 0; k < B.nz; k++)
    if (k < T.g0l || k >= T.g0l + m) out[(int64_t)k * NN] = 0.0;
}

// ---------------------------------------------------------------------------------------------
// The row-modified sweep along z (M + diag(c) S of the z-stiffened E component) with a
// per-fiber matrix: no host tables.  Per fiber, rank r:
//   spike_mod_tips_kernel: the block A_r = (M + diag(c) S)[g0:g0+m] is LU-factorised on the fly
//     (no pivoting, D12) twice -- top -> bottom (giving the bottom p rows of A_r^{-1} X) and
//     bottom -> top (the top p rows) -- for the columns X = [w, W-spike RHS [C_r; 0], V-spike RHS
//     [0; B_r]]: tips yt, yb (p), Wt, Wb, Vt, Vb (p x p), 2p + 4p^2 values per fiber;
//   all-gather of the tips;
//   spike_mod_solve_kernel: the interface system over z_s = (b_s, t_{s+1}), s = 0..R-2,
//     [I Vb_s; Wt_{s+1} I] z_s + [Wb_s b_{s-1}; 0] + [0; Vt_{s+1} t_{s+2}] = [yb_s; yt_{s+1}],
//     block tridiagonal, eliminated from both ends towards the rank's two interfaces (2p x 2p
//     blocks, O(R) per fiber), then the corrected segment solve (LU on the fly, forward values in
//     out, U rows in scratch, back substitution).
// ---------------------------------------------------------------------------------------------
struct SpikeModArgs {
  int64_t NN;
  int nz, R, r, N, k0, g0l, m;
  const double* f;       // rhs = solution (in place), z-slab inner planes
  const double* c;       // c per row, same layout
  double* out;
  double* scratch;       // (P + 1) * nz * NN: U rows and inverse pivots of the solve pass
  const double* Mb;      // band rows of M (global row g: Mb + g W)
  const double* Sb;      // band rows of S
  double* tips;          // [2P + 4P^2][NN]
  const double* gath;    // [R][2P + 4P^2][NN]
};

// small dense solve A x = b (n <= NMAX, partial pivoting), in place; k right-hand sides in B (n x k)
template <int NMAX>
__device__ void spk_solve(double (&A)[NMAX][NMAX], double* B, int n, int k) {
  for (int c = 0; c < n; c++) {
    int piv = c;
    double best = fabs(A[c][c]);
    for (int i = c + 1; i < n; i++)
      if (fabs(A[i][c]) > best) best = fabs(A[i][c]), piv = i;
    if (piv != c) {
      for (int j = 0; j < n; j++) { const double t = A[c][j]; A[c][j] = A[piv][j]; A[piv][j] = t; }
      for (int j = 0; j < k; j++) { const double t = B[c * k + j]; B[c * k + j] = B[piv * k + j]; B[piv * k + j] = t; }
    }
    const double inv = 1.0 / A[c][c];
    for (int i = c + 1; i < n; i++) {
      const double l = A[i][c] * inv;
      if (l == 0.0) continue;
      for (int j = c; j < n; j++) A[i][j] = fma(-l, A[c][j], A[i][j]);
      for (int j = 0; j < k; j++) B[i * k + j] = fma(-l, B[c * k + j], B[i * k + j]);
    }
  }
  for (int c = n - 1; c >= 0; c--) {
    const double inv = 1.0 / A[c][c];
    for (int j = 0; j < k; j++) {
      double s = B[c * k + j];
      for (int t = c + 1; t < n; t++) s = fma(-A[c][t], B[t * k + j], s);
      B[c * k + j] = s * inv;
    }
  }
}

// entry (global row g, column g + q) of M + c_g S restricted to the block rows [g0, g0 + m)
template <int P>
__device__ __forceinline__ double spk_a(const SpikeModArgs& A, int g, int q, double cg) {
  constexpr int W = 2 * P + 1;
  return fma(cg, __ldg(A.Sb + (int64_t)g * W + P + q), __ldg(A.Mb + (int64_t)g * W + P + q));
}

// One elimination pass over the block for NC columns: rev = false top -> bottom, true bottom ->
// top (pass row i <-> block row k = rev ? m-1-i : i; band offsets negate).  rhs(k, col) gives the
// right-hand side of block row k; out[i][col] = the last P solution rows of the pass, i = 0 the
// last row of the pass (block row m-1, resp. 0).
template <int P, int NC, class RHS>
__device__ void spk_pass(const SpikeModArgs& A, const double* cf, bool rev, RHS rhs, double (&out)[P][NC]) {
  const int m = A.m;
  double uw[P][P + 1];  // uw[j]: U row of pass row i-1-j (entries t = 0..P: columns i-1-j+t), uw[j][0] = 1/u
  double gw[P][NC];
#pragma unroll
  for (int j = 0; j < P; j++) {
#pragma unroll
    for (int t = 0; t <= P; t++) uw[j][t] = 0.0;
#pragma unroll
    for (int cc = 0; cc < NC; cc++) gw[j][cc] = 0.0;
  }
  for (int i = 0; i < m; i++) {
    const int k = rev ? m - 1 - i : i;
    const int g = A.k0 + A.g0l + k;
    const double cg = cf[(int64_t)(A.g0l + k) * A.NN];
    double rr[2 * P + 1];  // pass-row entries, offset q in -P..P (pass columns i+q)
#pragma unroll
    for (int q = -P; q <= P; q++) {
      const int ip = i + q;
      rr[q + P] = (ip >= 0 && ip < m) ? spk_a<P>(A, g, rev ? -q : q, cg) : 0.0;
    }
    double rv[NC];
#pragma unroll
    for (int cc = 0; cc < NC; cc++) rv[cc] = rhs(k, cc);
#pragma unroll
    for (int j = P; j >= 1; j--) {  // eliminate with pass row i-j (farthest first)
      if (i - j < 0) continue;
      const double l = rr[P - j] * uw[j - 1][0];
#pragma unroll
      for (int t = 1; t <= P; t++)
        if (-j + t <= P) rr[P - j + t] = fma(-l, uw[j - 1][t], rr[P - j + t]);
#pragma unroll
      for (int cc = 0; cc < NC; cc++) rv[cc] = fma(-l, gw[j - 1][cc], rv[cc]);
    }
#pragma unroll
    for (int j = P - 1; j > 0; j--) {
#pragma unroll
      for (int t = 0; t <= P; t++) uw[j][t] = uw[j - 1][t];
#pragma unroll
      for (int cc = 0; cc < NC; cc++) gw[j][cc] = gw[j - 1][cc];
    }
    uw[0][0] = 1.0 / rr[P];
#pragma unroll
    for (int t = 1; t <= P; t++) uw[0][t] = rr[P + t];
#pragma unroll
    for (int cc = 0; cc < NC; cc++) gw[0][cc] = rv[cc];
  }
  // back substitution over the last P pass rows (uw[j], gw[j]: pass row m-1-j)
#pragma unroll
  for (int j = 0; j < P; j++) {
#pragma unroll
    for (int cc = 0; cc < NC; cc++) {
      double s = gw[j][cc];
#pragma unroll
      for (int t = 1; t <= P; t++)
        if (j - t >= 0) s = fma(-uw[j][t], out[j - t][cc], s);
      out[j][cc] = s * uw[j][0];
    }
  }
}

template <int P>
__device__ __forceinline__ void spk_couplings(const SpikeModArgs& A, const double* cf, double (&C)[P][P], double (&Bm)[P][P]) {
  const int g0 = A.k0 + A.g0l, g1 = g0 + A.m;
#pragma unroll
  for (int i = 0; i < P; i++) {
    const double c0 = cf[(int64_t)(A.g0l + i) * A.NN], c1 = cf[(int64_t)(A.g0l + A.m - P + i) * A.NN];
#pragma unroll
    for (int j = 0; j < P; j++) {
      const int qc = j - i - P, qb = j - i + P;  // band offsets of the coupling entries (|q| <= P inside the band)
      C[i][j] = (A.r > 0 && qc >= -P) ? spk_a<P>(A, g0 + i, qc, c0) : 0.0;
      Bm[i][j] = (A.r < A.R - 1 && qb <= P) ? spk_a<P>(A, g1 - P + i, qb, c1) : 0.0;
    }
  }
}

template <int P>
__global__ void __launch_bounds__(128) spike_mod_tips_kernel(const __grid_constant__ SpikeModArgs A) {
  constexpr int NC = 1 + 2 * P, NT = 2 * P + 4 * P * P;
  const int64_t fb = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (fb >= A.NN) return;
  const double* f = A.f + fb;
  const double* cf = A.c + fb;
  double C[P][P], Bm[P][P];
  spk_couplings<P>(A, cf, C, Bm);
  const int m = A.m;
  auto rhs = [&](int k, int cc) -> double {
    if (cc == 0) return f[(int64_t)(A.g0l + k) * A.NN];
    if (cc <= P) return k < P ? C[k][cc - 1] : 0.0;
    return k >= m - P ? Bm[k - (m - P)][cc - 1 - P] : 0.0;
  };
  double bot[P][NC], top[P][NC];
  spk_pass<P, NC>(A, cf, false, rhs, bot);  // bot[j]: block row m-1-j
  spk_pass<P, NC>(A, cf, true, rhs, top);   // top[j]: block row j
  // layout: yt[P], yb[P], Wt[P][P], Wb[P][P], Vt[P][P], Vb[P][P] (row i = block row i resp. m-P+i)
  double* o = A.tips + fb;
  const int64_t NN = A.NN;
#pragma unroll
  for (int i = 0; i < P; i++) {
    o[(int64_t)i * NN] = top[i][0];
    o[(int64_t)(P + i) * NN] = bot[P - 1 - i][0];
#pragma unroll
    for (int j = 0; j < P; j++) {
      o[(int64_t)(2 * P + i * P + j) * NN] = top[i][1 + j];
      o[(int64_t)(2 * P + P * P + i * P + j) * NN] = bot[P - 1 - i][1 + j];
      o[(int64_t)(2 * P + 2 * P * P + i * P + j) * NN] = top[i][1 + P + j];
      o[(int64_t)(2 * P + 3 * P * P + i * P + j) * NN] = bot[P - 1 - i][1 + P + j];
    }
  }
  (void)NT;
}

template <int P>
__global__ void __launch_bounds__(128) spike_mod_solve_kernel(const __grid_constant__ SpikeModArgs A) {
  constexpr int NT = 2 * P + 4 * P * P, B2 = 2 * P;
  const int64_t fb = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (fb >= A.NN) return;
  const int64_t NN = A.NN;
  const int R = A.R, r = A.r;
  // tip t of rank s
  auto tip = [&](int s, int t) { return A.gath[((int64_t)s * NT + t) * NN + fb]; };
  auto yt = [&](int s, int i) { return tip(s, i); };
  auto yb = [&](int s, int i) { return tip(s, P + i); };
  auto Wt = [&](int s, int i, int j) { return tip(s, 2 * P + i * P + j); };
  auto Wb = [&](int s, int i, int j) { return tip(s, 2 * P + P * P + i * P + j); };
  auto Vt = [&](int s, int i, int j) { return tip(s, 2 * P + 2 * P * P + i * P + j); };
  auto Vb = [&](int s, int i, int j) { return tip(s, 2 * P + 3 * P * P + i * P + j); };
  // D_s z_s + L_s z_{s-1} + U_s z_{s+1} = r_s, z_s = (b_s, t_{s+1})
  auto Dmat = [&](int s, double (&D)[B2][B2]) {
    for (int i = 0; i < B2; i++)
      for (int j = 0; j < B2; j++) D[i][j] = i == j ? 1.0 : 0.0;
    for (int i = 0; i < P; i++)
      for (int j = 0; j < P; j++) D[i][P + j] = Vb(s, i, j), D[P + i][j] = Wt(s + 1, i, j);
  };
  auto rvec = [&](int s, double* v) {
    for (int i = 0; i < P; i++) v[i] = yb(s, i), v[P + i] = yt(s + 1, i);
  };
  double tn[P], bp[P];
  for (int i = 0; i < P; i++) tn[i] = bp[i] = 0.0;
  if (R > 1) {
    // top-down to interface r-1: Dt z_{r-1} + U_{r-1} z_r = rt
    double Dt[B2][B2], rt[B2];
    if (r >= 1) {
      Dmat(0, Dt);
      rvec(0, rt);
      for (int s = 1; s <= r - 1; s++) {
        // X = Dt^{-1} [U_{s-1} | rt]: U_{s-1} nonzero in rows P.., columns P.. (Vt_s)
        double Dc[B2][B2], X[B2 * (B2 + 1)];
        for (int i = 0; i < B2; i++)
          for (int j = 0; j < B2; j++) Dc[i][j] = Dt[i][j];
        for (int i = 0; i < B2; i++) {
          for (int j = 0; j < B2; j++) X[i * (B2 + 1) + j] = (i >= P && j >= P) ? Vt(s, i - P, j - P) : 0.0;
          X[i * (B2 + 1) + B2] = rt[i];
        }
        spk_solve<B2>(Dc, X, B2, B2 + 1);
        // L_s picks b_{s-1} = first P entries, into the first P rows with Wb_s
        Dmat(s, Dt);
        rvec(s, rt);
        for (int i = 0; i < P; i++)
          for (int q = 0; q < P; q++) {
            const double w = Wb(s, i, q);
            for (int j = 0; j < B2; j++) Dt[i][j] = fma(-w, X[q * (B2 + 1) + j], Dt[i][j]);
            rt[i] = fma(-w, X[q * (B2 + 1) + B2], rt[i]);
          }
      }
    }
    // bottom-up to interface r: Dh z_r + L_r z_{r-1} = rh
    double Dh[B2][B2], rh[B2];
    if (r <= R - 2) {
      Dmat(R - 2, Dh);
      rvec(R - 2, rh);
      for (int s = R - 3; s >= r; s--) {
        // X = Dh^{-1} [L_{s+1} | rh]: L_{s+1} nonzero in rows 0..P-1, columns 0..P-1 (Wb_{s+1})
        double Dc[B2][B2], X[B2 * (B2 + 1)];
        for (int i = 0; i < B2; i++)
          for (int j = 0; j < B2; j++) Dc[i][j] = Dh[i][j];
        for (int i = 0; i < B2; i++) {
          for (int j = 0; j < B2; j++) X[i * (B2 + 1) + j] = (i < P && j < P) ? Wb(s + 1, i, j) : 0.0;
          X[i * (B2 + 1) + B2] = rh[i];
        }
        spk_solve<B2>(Dc, X, B2, B2 + 1);
        // U_s picks t_{s+2} = entries P.. of z_{s+1}, into rows P.. with Vt_{s+1}
        Dmat(s, Dh);
        rvec(s, rh);
        for (int i = 0; i < P; i++)
          for (int q = 0; q < P; q++) {
            const double v = Vt(s + 1, i, q);
            for (int j = 0; j < B2; j++) Dh[P + i][j] = fma(-v, X[(P + q) * (B2 + 1) + j], Dh[P + i][j]);
            rh[P + i] = fma(-v, X[(P + q) * (B2 + 1) + B2], rh[P + i]);
          }
      }
    }
    if (r == 0) {
      double x[B2];
      for (int i = 0; i < B2; i++) x[i] = rh[i];
      spk_solve<B2>(Dh, x, B2, 1);
      for (int i = 0; i < P; i++) tn[i] = x[P + i];
    } else if (r == R - 1) {
      double x[B2];
      for (int i = 0; i < B2; i++) x[i] = rt[i];
      spk_solve<B2>(Dt, x, B2, 1);
      for (int i = 0; i < P; i++) bp[i] = x[i];
    } else {
      // [[Dt, U_{r-1}], [L_r, Dh]] [z_{r-1}; z_r] = [rt; rh]
      constexpr int B4 = 4 * P;
      double K[B4][B4], x[B4];
      for (int i = 0; i < B4; i++)
        for (int j = 0; j < B4; j++) K[i][j] = 0.0;
      for (int i = 0; i < B2; i++)
        for (int j = 0; j < B2; j++) K[i][j] = Dt[i][j], K[B2 + i][B2 + j] = Dh[i][j];
      for (int i = 0; i < P; i++)
        for (int j = 0; j < P; j++) {
          K[P + i][B2 + P + j] = Vt(r, i, j);  // U_{r-1}: t_{r+1} into the rows of t_r
          K[B2 + i][j] = Wb(r, i, j);          // L_r: b_{r-1} into the rows of b_r
        }
      for (int i = 0; i < B2; i++) x[i] = rt[i], x[B2 + i] = rh[i];
      spk_solve<B4>(K, x, B4, 1);
      for (int i = 0; i < P; i++) bp[i] = x[i], tn[i] = x[B2 + P + i];
    }
  }
  // corrected segment solve: A_r x = f - [C b_{r-1}; 0] - [0; B t_{r+1}]
  constexpr int W = 2 * P + 1;
  const double* cf = A.c + fb;
  double C[P][P], Bm[P][P];
  spk_couplings<P>(A, cf, C, Bm);
  const int m = A.m;
  double* out = A.out + fb;
  double* sc = A.scratch + fb;
  const int64_t UL = (int64_t)A.nz * NN;
  double uw[P][P + 1], gwin[P];
  for (int j = 0; j < P; j++) {
    for (int t = 0; t <= P; t++) uw[j][t] = 0.0;
    gwin[j] = 0.0;
  }
  for (int k = 0; k < m; k++) {
    const int g = A.k0 + A.g0l + k;
    const int64_t pl = (int64_t)(A.g0l + k) * NN;
    const double cg = cf[pl];
    double rr[W];
#pragma unroll
    for (int q = -P; q <= P; q++) rr[q + P] = (k + q >= 0 && k + q < m) ? spk_a<P>(A, g, q, cg) : 0.0;
    double rv = A.f[fb + pl];
    if (k < P) {
#pragma unroll
      for (int j = 0; j < P; j++) rv = fma(-C[k][j], bp[j], rv);
    }
    if (k >= m - P) {
#pragma unroll
      for (int j = 0; j < P; j++) rv = fma(-Bm[k - (m - P)][j], tn[j], rv);
    }
#pragma unroll
    for (int j = P; j >= 1; j--) {
      if (k - j < 0) continue;
      const double l = rr[P - j] * uw[j - 1][0];
#pragma unroll
      for (int t = 1; t <= P; t++)
        if (-j + t <= P) rr[P - j + t] = fma(-l, uw[j - 1][t], rr[P - j + t]);
      rv = fma(-l, gwin[j - 1], rv);
    }
#pragma unroll
    for (int j = P - 1; j > 0; j--) {
#pragma unroll
      for (int t = 0; t <= P; t++) uw[j][t] = uw[j - 1][t];
      gwin[j] = gwin[j - 1];
    }
    uw[0][0] = 1.0 / rr[P];
#pragma unroll
    for (int t = 1; t <= P; t++) uw[0][t] = rr[P + t];
    gwin[0] = rv;
    out[pl] = rv;
#pragma unroll
    for (int t = 0; t <= P; t++) sc[(int64_t)t * UL + pl] = uw[0][t];
  }
  double xw[P];
  for (int j = 0; j < P; j++) xw[j] = 0.0;
  for (int k = m - 1; k >= 0; k--) {
    const int64_t pl = (int64_t)(A.g0l + k) * NN;
    double s = out[pl];
#pragma unroll
    for (int t = 1; t <= P; t++)
      if (k + t < m) s = fma(-sc[(int64_t)t * UL + pl], xw[t - 1], s);
    const double x = s * sc[pl];
#pragma unroll
    for (int j = P - 1; j > 0; j--) xw[j] = xw[j - 1];
    xw[0] = x;
    out[pl] = x;
  }
  for (int k = 0; k < A.nz; k++)
    if (k < A.g0l || k >= A.g0l + m) out[(int64_t)k * NN] = 0.0;
}

}  // namespace adi
