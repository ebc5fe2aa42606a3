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
