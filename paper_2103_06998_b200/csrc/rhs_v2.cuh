// rhs_v2.cuh -- NEXT-2 variant V2: the E right-hand sides with the element-wise
// material INSIDE the quadrature of their curl and mixed-derivative integrals (P:548-549 read as
// "element-wise eps, mu"; the paper-literal default D5 scales whole rows by the test function's
// material instead).  Each such term
//     [sum_e w_e (X^{e_x} (x) Y^{e_y} (x) Z^{e_z}) u]_{rst}
// is evaluated by quadrature with sum factorisation:
//   interpolate u (or its derivative along the trial-derivative axes) to the Gauss points of every
//   element, axis by axis (N -> n q per axis, q = p + 1 points per element; D11);
//   multiply by the element coefficient w_e (a_e = tau/(2 eps_e) or c_e = tau^2/(4 eps_e mu_e));
//   integrate against the test functions (or their derivatives), axis by axis (n q -> N), with
//   the Gauss weights h w_g folded into the projection tables.
// Every pass is one banded 1D operator along one axis of a 3D array (x fastest):
//   out[.., i, ..] = scale * sum_{t < w} tab[i w + t] in[.., start[i] + t, ..]  (+ out if accumulate)
// One thread per output entry; the passes are HBM-bound streams (a comparison variant, not the
// hot path: its cost is reported in DESIGN.md).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace adi {

__global__ void v2_pass_kernel(const double* __restrict__ in, int64_t d0, int64_t d1, int64_t d2, int ax,
                               double* __restrict__ out, int64_t nout, const double* __restrict__ tab,
                               const int* __restrict__ start, int w, double scale, int accumulate) {
  // output dims: d with d[ax] replaced by nout
  const int64_t o0 = ax == 0 ? nout : d0, o1 = ax == 1 ? nout : d1, o2 = ax == 2 ? nout : d2;
  const int64_t total = o0 * o1 * o2;
  const int64_t sin = ax == 0 ? 1 : ax == 1 ? d0 : d0 * d1;  // input stride along ax
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = e % o0, yz = e / o0, y = yz % o1, z = yz / o1;
    const int64_t i = ax == 0 ? x : ax == 1 ? y : z;
    const int64_t base = (ax == 0 ? 0 : x) + d0 * ((ax == 1 ? 0 : y) + d1 * (ax == 2 ? 0 : z));
    const double* row = tab + i * w;
    const double* src = in + base + (int64_t)start[i] * sin;
    double acc = 0.0;
    for (int t = 0; t < w; t++) acc = fma(row[t], src[(int64_t)t * sin], acc);
    out[e] = accumulate ? fma(scale, acc, out[e]) : scale * acc;
  }
}

// T[qx, qy, qz] *= w_e of the element holding the Gauss point: kind 0: a_e = tau / (2 eps_e),
// kind 1: c_e = tau^2 / (4 eps_e mu_e) (P:545 with the element's material)
__global__ void v2_weight_kernel(double* __restrict__ T, int n, int q, const double* __restrict__ eps,
                                 const double* __restrict__ mu, double tau, int kind) {
  const int64_t nq = (int64_t)n * q, total = nq * nq * nq;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = e % nq, yz = e / nq, y = yz % nq, z = yz / nq;
    const int64_t el = x / q + n * (y / q + (int64_t)n * (z / q));
    T[e] *= kind == 0 ? tau / (2.0 * eps[el]) : tau * tau / (4.0 * eps[el] * mu[el]);
  }
}

// R -= a s J (D9, the row factor of the source term), s = signal[*step] when step < nsig
__global__ void v2_source_kernel(double* __restrict__ R, const double* __restrict__ a, const double* __restrict__ J,
                                 const double* __restrict__ signal, const int64_t* __restrict__ step, int64_t nsig,
                                 int64_t U) {
  const int64_t s = *step;
  if (s >= nsig) return;
  const double sv = signal[s];
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < U; e += (int64_t)gridDim.x * blockDim.x)
    R[e] -= a[e] * sv * J[e];
}

}  // namespace adi
