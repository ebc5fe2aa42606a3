// setup_kernels.cuh -- amortised setup kernels (a0) of libadimaxwell.so:
// material map (D6), row factors a, b, c, input validation, PEC
// zeroing (D1).  Included by the host translation unit only.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace adi {

// ---------------------------------------------------------------------------
// Setup kernels (a0, amortised)
// ---------------------------------------------------------------------------

// One separable pass of the material map (D6): out[.., r, ..] = sum_e w[r*n + e] in[.., e, ..]
// along `axis` of an (nx, ny, nz) array; output extent along the axis is N.
__global__ void material_pass_kernel(const double* __restrict__ in, double* __restrict__ out, const double* __restrict__ w,
                                     int n, int N, int p, int axis, int nx, int ny, int nz) {
  // output dims
  int ox = axis == 0 ? N : nx, oy = axis == 1 ? N : ny, oz = axis == 2 ? N : nz;
  int64_t total = (int64_t)ox * oy * oz;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total; id += (int64_t)gridDim.x * blockDim.x) {
    int x = (int)(id % ox);
    int y = (int)((id / ox) % oy);
    int z = (int)(id / ((int64_t)ox * oy));
    int r = axis == 0 ? x : axis == 1 ? y : z;
    double s = 0.0;
    int e0 = r - p < 0 ? 0 : r - p;
    int e1 = r < n - 1 ? r : n - 1;
    for (int e = e0; e <= e1; e++) {
      int xi = axis == 0 ? e : x, yi = axis == 1 ? e : y, zi = axis == 2 ? e : z;
      s += w[r * n + e] * in[xi + (int64_t)nx * (yi + (int64_t)ny * zi)];
    }
    out[id] = s;
  }
}

// a = tau/(2 eps), b = tau/(2 mu), c = tau^2/(4 eps mu)  (D13)
__global__ void abc_kernel(const double* __restrict__ eps, const double* __restrict__ mu, double tau, int64_t U,
                           double* __restrict__ a, double* __restrict__ b, double* __restrict__ c) {
  for (int64_t I = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; I < U; I += (int64_t)gridDim.x * blockDim.x) {
    const double e = eps[I], m = mu ? mu[I] : 1.0;
    a[I] = tau / (2.0 * e);
    b[I] = tau / (2.0 * m);
    c[I] = tau * tau / (4.0 * e * m);
  }
}

// validity check of positive finite values; writes the first offending index
__global__ void check_positive_kernel(const double* __restrict__ x, int64_t n, unsigned long long* bad) {
  for (int64_t I = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; I < n; I += (int64_t)gridDim.x * blockDim.x) {
    const double v = x[I];
    if (!(v > 0.0) || !isfinite(v)) atomicMin(bad, (unsigned long long)I);
  }
}

// zero the PEC-eliminated entries of an E component (D1)
__global__ void pec_zero_kernel(double* __restrict__ u, int N, int lo0, int hi0, int lo1, int hi1, int lo2, int hi2) {
  const int64_t U = (int64_t)N * N * N;
  for (int64_t I = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; I < U; I += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(I % N), j = (int)((I / N) % N), k = (int)(I / ((int64_t)N * N));
    if (i < lo0 || i >= hi0 || j < lo1 || j >= hi1 || k < lo2 || k >= hi2) u[I] = 0.0;
  }
}

__global__ void increment_kernel(int64_t* counter) { *counter += 1; }

// u = f / eps (first step of the eps-weighted projection, Appendix eq. split1); u may alias f
__global__ void div_kernel(double* u, const double* f, const double* __restrict__ eps, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    u[i] = f[i] / eps[i];
}

// Manufactured solution u_A = g u^1_{1,1} + 2g u^2_{1,1} + 3g u^3_{1,1}, g = 2/sqrt(14)
// (u^2 with the sign reading D8), and its curl (derived by hand):
//   E = C (a1 sy sz, a2 sx sz, a3 sx sy),               C = cos(sqrt2 pi t), a_d = d g
//   H = r S (sx (a2 cz - a3 cy), sy (a3 cx - a1 cz), sz (a1 cy - a2 cx)),  S = sin(sqrt2 pi t), r = 1/sqrt2
//   curl E = pi C (sx (a3 cy - a2 cz), sy (a1 cz - a3 cx), sz (a2 cx - a1 cy))
//   curl H = -2 pi r S (a1 sy sz, a2 sx sz, a3 sx sy)
__device__ __forceinline__ void uA_field(double x, double y, double z, double t, double* f, double* cf) {
  const double g = 2.0 / sqrt(14.0), a1 = g, a2 = 2.0 * g, a3 = 3.0 * g;
  const double pi = 3.14159265358979323846, r = 0.70710678118654752440, om = 1.41421356237309504880 * pi;
  double sx, cx, sy, cy, sz, cz, S, C;
  sincos(pi * x, &sx, &cx);
  sincos(pi * y, &sy, &cy);
  sincos(pi * z, &sz, &cz);
  sincos(om * t, &S, &C);
  f[0] = C * a1 * sy * sz;
  f[1] = C * a2 * sx * sz;
  f[2] = C * a3 * sx * sy;
  f[3] = r * S * sx * (a2 * cz - a3 * cy);
  f[4] = r * S * sy * (a3 * cx - a1 * cz);
  f[5] = r * S * sz * (a1 * cy - a2 * cx);
  cf[0] = pi * C * sx * (a3 * cy - a2 * cz);
  cf[1] = pi * C * sy * (a1 * cz - a3 * cx);
  cf[2] = pi * C * sz * (a2 * cx - a1 * cy);
  cf[3] = -2.0 * pi * r * S * a1 * sy * sz;
  cf[4] = -2.0 * pi * r * S * a2 * sx * sz;
  cf[5] = -2.0 * pi * r * S * a3 * sx * sy;
}

// Squared L2 errors of the discrete fields and of their curls against u_A(., t), by
// Gauss quadrature with q points per axis on every element; one thread per (element,
// Gauss point).  bv/bd[(e*q + g)*(p+1) + j]: B_{e+j} and B'_{e+j} at Gauss point g of
// element e; x0/xg/wg: element starts (uniform h), points and weights on [0, h].
// acc[0..3] += (E L2^2, H L2^2, curl E L2^2, curl H L2^2).
__global__ void errors_uA_kernel(const double* const* __restrict__ F, int n, int p, int q,
                                 const double* __restrict__ bv, const double* __restrict__ bd,
                                 const double* __restrict__ xg, const double* __restrict__ wg, double h, double t,
                                 double* acc) {
  const int N = n + p, pp = p + 1;
  const int64_t total = (int64_t)n * n * n * q * q * q;
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total; id += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = id;
    const int gi = (int)(r % q); r /= q;
    const int gj = (int)(r % q); r /= q;
    const int gk = (int)(r % q); r /= q;
    const int ea = (int)(r % n); r /= n;
    const int eb = (int)(r % n); r /= n;
    const int ec = (int)r;
    const double* vx = bv + ((int64_t)ea * q + gi) * pp;
    const double* vy = bv + ((int64_t)eb * q + gj) * pp;
    const double* vz = bv + ((int64_t)ec * q + gk) * pp;
    const double* dx = bd + ((int64_t)ea * q + gi) * pp;
    const double* dy = bd + ((int64_t)eb * q + gj) * pp;
    const double* dz = bd + ((int64_t)ec * q + gk) * pp;
    double val[6], gx[6], gy[6], gz[6];  // value and gradient of each discrete field
    for (int c = 0; c < 6; c++) {
      double v = 0.0, ax = 0.0, ay = 0.0, az = 0.0;
      for (int kk = 0; kk < pp; kk++)
        for (int jj = 0; jj < pp; jj++) {
          const double* row = F[c] + (ea + (int64_t)N * ((eb + jj) + (int64_t)N * (ec + kk)));
          const double yz = vy[jj] * vz[kk], dyz = dy[jj] * vz[kk], ydz = vy[jj] * dz[kk];
          for (int ii = 0; ii < pp; ii++) {
            const double u = row[ii];
            v += u * vx[ii] * yz;
            ax += u * dx[ii] * yz;
            ay += u * vx[ii] * dyz;
            az += u * vx[ii] * ydz;
          }
        }
      val[c] = v, gx[c] = ax, gy[c] = ay, gz[c] = az;
    }
    const double cu[6] = {gy[2] - gz[1], gz[0] - gx[2], gx[1] - gy[0], gy[5] - gz[4], gz[3] - gx[5], gx[4] - gy[3]};
    double ex[6], ecu[6];
    uA_field(ea * h + xg[gi], eb * h + xg[gj], ec * h + xg[gk], t, ex, ecu);
    const double w = wg[gi] * wg[gj] * wg[gk];
    for (int c = 0; c < 3; c++) {
      const double e0 = val[c] - ex[c], e1 = val[3 + c] - ex[3 + c], c0 = cu[c] - ecu[c], c1 = cu[3 + c] - ecu[3 + c];
      s[0] += w * e0 * e0;
      s[1] += w * e1 * e1;
      s[2] += w * c0 * c0;
      s[3] += w * c1 * c1;
    }
  }
  __shared__ double red[4][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int k = 0; k < 4; k++) {
    double v = s[k];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[k][wid] = v;
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    double v = 0.0;
    for (int w2 = 0; w2 < (int)(blockDim.x >> 5); w2++) v += red[threadIdx.x][w2];
    atomicAdd(acc + threadIdx.x, v);
  }
}

// ||div E||^2 and ||div H||^2 of the discrete fields by Gauss quadrature (same tables and
// thread mapping as errors_uA_kernel); acc[0..1] += (div E L2^2, div H L2^2).
__global__ void divergence_kernel(const double* const* __restrict__ F, int n, int p, int q,
                                  const double* __restrict__ bv, const double* __restrict__ bd,
                                  const double* __restrict__ wg, double* acc) {
  const int N = n + p, pp = p + 1;
  const int64_t total = (int64_t)n * n * n * q * q * q;
  double s[2] = {0.0, 0.0};
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total; id += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = id;
    const int gi = (int)(r % q); r /= q;
    const int gj = (int)(r % q); r /= q;
    const int gk = (int)(r % q); r /= q;
    const int ea = (int)(r % n); r /= n;
    const int eb = (int)(r % n); r /= n;
    const int ec = (int)r;
    const int64_t ox = ((int64_t)ea * q + gi) * pp, oy = ((int64_t)eb * q + gj) * pp, oz = ((int64_t)ec * q + gk) * pp;
    double dv[2] = {0.0, 0.0};
    for (int f = 0; f < 2; f++)        // E, H
      for (int d = 0; d < 3; d++) {    // d/dx_d of component d
        const double* X = d == 0 ? bd + ox : bv + ox;
        const double* Y = d == 1 ? bd + oy : bv + oy;
        const double* Z = d == 2 ? bd + oz : bv + oz;
        const double* u = F[3 * f + d];
        double a = 0.0;
        for (int kk = 0; kk < pp; kk++)
          for (int jj = 0; jj < pp; jj++) {
            const double* row = u + (ea + (int64_t)N * ((eb + jj) + (int64_t)N * (ec + kk)));
            const double yz = Y[jj] * Z[kk];
            for (int ii = 0; ii < pp; ii++) a += row[ii] * X[ii] * yz;
          }
        dv[f] += a;
      }
    const double w = wg[gi] * wg[gj] * wg[gk];
    s[0] += w * dv[0] * dv[0];
    s[1] += w * dv[1] * dv[1];
  }
  __shared__ double red[2][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int k = 0; k < 2; k++) {
    double v = s[k];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[k][wid] = v;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    double v = 0.0;
    for (int w2 = 0; w2 < (int)(blockDim.x >> 5); w2++) v += red[threadIdx.x][w2];
    atomicAdd(acc + threadIdx.x, v);
  }
}

__global__ void fill_kernel(double* __restrict__ x, int64_t n, double v) {
  for (int64_t I = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; I < n; I += (int64_t)gridDim.x * blockDim.x) x[I] = v;
}

// min and max of a positive array (IEEE order of positive doubles = order of their bit patterns)
__global__ void minmax_pos_kernel(const double* __restrict__ x, int64_t n, unsigned long long* mm) {
  unsigned long long lo = ~0ull, hi = 0ull;
  for (int64_t I = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; I < n; I += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long v = (unsigned long long)__double_as_longlong(x[I]);
    lo = v < lo ? v : lo;
    hi = v > hi ? v : hi;
  }
  atomicMin(&mm[0], lo);
  atomicMax(&mm[1], hi);
}

// dst box <- src box (3D strided copy; x fastest in both arrays)
__global__ void copy_box_kernel(double* __restrict__ dst, int64_t dx, int64_t dy, int64_t ox, int64_t oy, int64_t oz,
                                const double* __restrict__ src, int64_t sx, int64_t sy, int64_t px, int64_t py, int64_t pz,
                                int64_t ex, int64_t ey, int64_t ez) {
  const int64_t total = ex * ey * ez;
  for (int64_t I = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; I < total; I += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = I % ex, y = (I / ex) % ey, z = I / (ex * ey);
    dst[(ox + x) + dx * ((oy + y) + dy * (oz + z))] = src[(px + x) + sx * ((py + y) + sy * (pz + z))];
  }
}

// zero the PEC-eliminated entries (D1) of an E component held in a box at global offset (ox, oy, oz)
__global__ void pec_box_kernel(double* __restrict__ u, int64_t nx, int64_t ny, int64_t nz, int64_t ox, int64_t oy, int64_t oz,
                               int lo0, int hi0, int lo1, int hi1, int lo2, int hi2) {
  const int64_t total = nx * ny * nz;
  for (int64_t I = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; I < total; I += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = ox + I % nx, j = oy + (I / nx) % ny, k = oz + I / (nx * ny);
    if (i < lo0 || i >= hi0 || j < lo1 || j >= hi1 || k < lo2 || k >= hi2) u[I] = 0.0;
  }
}

// sum over the patch of u (.) ((M (x) M (x) M) u) (the M-norm squared; diagnostic, not on the
// step path): direct (2p+1)^3 stencil from the band table of M, block reduction, one atomic per block
__global__ void mnorm_kernel(const double* __restrict__ u, const double* __restrict__ tabM, int N, int p,
                             double* __restrict__ acc) {
  const int W = 2 * p + 1;
  const int64_t U = (int64_t)N * N * N;
  double s = 0.0;
  for (int64_t I = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; I < U; I += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(I % N), j = (int)((I / N) % N), k = (int)(I / ((int64_t)N * N));
    double v = 0.0;
    for (int c = 0; c < W; c++) {
      const int o = k - p + c;
      if (o < 0 || o >= N) continue;
      const double mz = tabM[(int64_t)k * W + c];
      for (int b = 0; b < W; b++) {
        const int m = j - p + b;
        if (m < 0 || m >= N) continue;
        const double myz = mz * tabM[(int64_t)j * W + b];
        const double* row = u + (int64_t)N * (m + (int64_t)N * o);
        for (int a = 0; a < W; a++) {
          const int l = i - p + a;
          if (l < 0 || l >= N) continue;
          v = fma(myz * tabM[(int64_t)i * W + a], row[l], v);
        }
      }
    }
    s = fma(u[I], v, s);
  }
  __shared__ double red[256];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) atomicAdd(acc, red[0]);
}

}  // namespace adi
