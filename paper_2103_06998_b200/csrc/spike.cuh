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

}  // namespace adi
