// kernels.cuh -- sm_100a fp64 kernels of the ADI-IGA Maxwell step
// (arXiv 2103.06998).  Product code: shares nothing with oracle/.
//
// Two kernel families carry the whole step:
//   * rhs_kernel   : right-hand sides as sums of row-scaled Kronecker products
//                    (X (x) Y (x) Z) u, sum-factorised:
//                    x-pass and y-pass on a shared-memory xy tile, z-pass on a
//                    register window while the block streams along z.
//   * sweep_kernel : batched banded LU along one axis for every fiber
//                    (P:468-527), constant mass matrix (precomputed factors) or
//                    row-modified M + diag(c) S (factored on the fly
//                    per fiber, no pivoting -- D12), one fiber per lane.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace adi {

// 1D operator codes of the band tables: tab[(op*N + row)*(2P+1) + q] holds the
// entry in column row-P+q (0 outside [0,N)).
enum Op { OP_M = 0, OP_A = 1, OP_B = 2, OP_S = 3, NUM_OPS = 4 };
enum Scale { SC_ONE = 0, SC_A = 1, SC_C = 2, SC_B = 3 };

constexpr int RHS_TX = 32;
constexpr int RHS_TY = 8;
constexpr int RHS_MAXT = 4;

struct RhsTerm {
  const double* u;  // input field (N^3)
  int op[3];        // x, y, z operator codes
  int scale;        // Scale
  double sign;      // +1 / -1
};

struct RhsArgs {
  int N;
  int kchunk;            // z-planes per block
  const double* tab;     // band tables, 4 ops
  RhsTerm term[RHS_MAXT];
  const double* a;       // tau/(2 eps^)
  const double* b;       // tau/(2 mu^)
  const double* c;       // tau^2/(4 eps^ mu^)
  const double* load;    // source load vector for this component, or nullptr (D9)
  const double* signal;  // device signal array (nsig) or nullptr
  const int64_t* step;   // device step counter
  int64_t nsig;
  int lo[3], hi[3];      // active ranges of the output component (PEC, D1)
  double* out;
};

// out[I] = sum_t sign_t * scale_t[I] * ((X_t (x) Y_t (x) Z_t) u_t)[I]  (- a s J),
// zero outside the active set.
template <int P, int NT>
__global__ void __launch_bounds__(RHS_TX * RHS_TY)
rhs_kernel(const RhsArgs args) {
  constexpr int W = 2 * P + 1;
  constexpr int HX = RHS_TX + 2 * P;
  constexpr int HY = RHS_TY + 2 * P;
  __shared__ double s_in[NT][HY][HX];
  __shared__ double s_x[NT][HY][RHS_TX];

  const int N = args.N;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = ty * RHS_TX + tx;
  const int i0 = blockIdx.x * RHS_TX, j0 = blockIdx.y * RHS_TY;
  const int k0 = blockIdx.z * args.kchunk;
  const int k1 = min(N, k0 + args.kchunk);
  const int i = i0 + tx, j = j0 + ty;
  const int64_t NN = (int64_t)N * N;

  double cx[NT][W], cy[NT][W], w[NT][W];
#pragma unroll
  for (int t = 0; t < NT; t++) {
#pragma unroll
    for (int q = 0; q < W; q++) {
      cx[t][q] = (i < N) ? args.tab[((int64_t)args.term[t].op[0] * N + i) * W + q] : 0.0;
      cy[t][q] = (j < N) ? args.tab[((int64_t)args.term[t].op[1] * N + j) * W + q] : 0.0;
      w[t][q] = 0.0;
    }
  }
  double sval = 0.0;
  if (args.load != nullptr && args.signal != nullptr) {
    const int64_t s = *args.step;
    if (s < args.nsig) sval = args.signal[s];
  }

  for (int kin = k0 - P; kin < k1 + P; kin++) {
    __syncthreads();
    const bool kok = (kin >= 0 && kin < N);
#pragma unroll
    for (int t = 0; t < NT; t++) {
      const double* __restrict__ u = args.term[t].u;
      for (int idx = tid; idx < HY * HX; idx += RHS_TX * RHS_TY) {
        const int yy = idx / HX, xx = idx - yy * HX;
        const int gi = i0 - P + xx, gj = j0 - P + yy;
        double v = 0.0;
        if (kok && gi >= 0 && gi < N && gj >= 0 && gj < N) v = __ldg(u + gi + (int64_t)N * gj + NN * kin);
        s_in[t][yy][xx] = v;
      }
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < NT; t++) {
      for (int yy = ty; yy < HY; yy += RHS_TY) {
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < W; q++) acc = fma(cx[t][q], s_in[t][yy][tx + q], acc);
        s_x[t][yy][tx] = acc;
      }
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < NT; t++) {
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < W; q++) acc = fma(cy[t][q], s_x[t][ty + q][tx], acc);
#pragma unroll
      for (int q = 0; q < W - 1; q++) w[t][q] = w[t][q + 1];
      w[t][W - 1] = acc;
    }
    const int k = kin - P;
    if (k >= k0 && k < k1 && i < N && j < N) {
      const int64_t I = i + (int64_t)N * j + NN * k;
      const bool active = i >= args.lo[0] && i < args.hi[0] && j >= args.lo[1] && j < args.hi[1] &&
                          k >= args.lo[2] && k < args.hi[2];
      double val = 0.0;
      if (active) {
#pragma unroll
        for (int t = 0; t < NT; t++) {
          const double* zc = args.tab + ((int64_t)args.term[t].op[2] * N + k) * W;
          double z = 0.0;
#pragma unroll
          for (int q = 0; q < W; q++) z = fma(__ldg(zc + q), w[t][q], z);
          double sc = 1.0;
          const int kind = args.term[t].scale;
          if (kind == SC_A) sc = args.a[I];
          else if (kind == SC_C) sc = args.c[I];
          else if (kind == SC_B) sc = args.b[I];
          val = fma(args.term[t].sign * sc, z, val);
        }
        if (sval != 0.0) val -= args.a[I] * sval * args.load[I];
      }
      args.out[I] = val;
    }
  }
}

// ---------------------------------------------------------------------------
// Sweeps
// ---------------------------------------------------------------------------
struct SweepArgs {
  int N;
  int axis;          // 0 = x, 1 = y, 2 = z
  int lo, hi;        // active rows along the axis
  int ntiles;        // 32-fiber tiles
  int64_t nfpad;     // ntiles * 32 (scratch plane pitch)
  const double* in;  // rhs
  double* out;       // solution (may equal in)
  double* scr;       // scratch: (P+2) planes of N * nfpad doubles
  // mass sweep: factor table fac[kk*(2P+1) + {0..P-1: l_{kk,kk-1-q}, P: 1/u_kk, P+1..2P: u_{kk,kk+1+q}}]
  const double* fac;
  // modified sweep: band tables of M and S restricted to [lo,hi) (row-major, 2P+1 per row, N rows)
  const double* Mb;
  const double* Sb;
  const double* c;   // per-test-function c (N^3)
};

// fiber geometry for lane `lane` of tile `tile`: returns base offset and the
// element stride along the axis; `valid` false for padding lanes.
__device__ __forceinline__ void fiber_geom(const SweepArgs& A, int tile, int lane, int64_t& base, int64_t& stride,
                                           bool& valid) {
  const int N = A.N;
  const int64_t NN = (int64_t)N * N;
  if (A.axis == 2) {
    const int64_t f = (int64_t)tile * 32 + lane;
    valid = f < NN;
    base = f;
    stride = NN;
  } else if (A.axis == 1) {
    const int tpk = (N + 31) / 32;
    const int k = tile / tpk;
    const int i = (tile - k * tpk) * 32 + lane;
    valid = i < N;
    base = i + NN * k;
    stride = N;
  } else {
    const int64_t f = (int64_t)tile * 32 + lane;
    valid = f < NN;
    base = (int64_t)N * f;
    stride = 1;
  }
}

// Load rows [c0, c0+CH) of the warp's 32 fibers into v[] (lane = fiber).
// x-axis fibers are contiguous, so they go through a per-warp smem transpose.
template <int CH>
__device__ __forceinline__ void load_rows(const SweepArgs& A, const double* __restrict__ src, int tile, int lane,
                                          int64_t base, int64_t stride, bool valid, int c0, double (*T)[33],
                                          double* v) {
  if (A.axis != 0) {
#pragma unroll
    for (int r = 0; r < CH; r++) {
      const int row = c0 + r;
      v[r] = (valid && row < A.hi) ? __ldg(src + base + (int64_t)row * stride) : 0.0;
    }
  } else {
    const int64_t NN = (int64_t)A.N * A.N;
    const int64_t f0 = (int64_t)tile * 32;
    const int row = c0 + lane;
#pragma unroll 4
    for (int r = 0; r < 32; r++) {
      double x = 0.0;
      if (lane < CH && f0 + r < NN && row < A.hi) x = __ldg(src + (int64_t)A.N * (f0 + r) + row);
      T[r][lane] = x;
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < CH; r++) v[r] = T[lane][r];
    __syncwarp();
  }
}

template <int CH>
__device__ __forceinline__ void store_rows(const SweepArgs& A, double* __restrict__ dst, int tile, int lane,
                                           int64_t base, int64_t stride, bool valid, int c0, double (*T)[33],
                                           const double* v) {
  if (A.axis != 0) {
#pragma unroll
    for (int r = 0; r < CH; r++) {
      const int row = c0 + r;
      if (valid && row < A.hi) dst[base + (int64_t)row * stride] = v[r];
    }
  } else {
    const int64_t NN = (int64_t)A.N * A.N;
    const int64_t f0 = (int64_t)tile * 32;
#pragma unroll
    for (int r = 0; r < CH; r++) T[lane][r] = v[r];
    __syncwarp();
    const int row = c0 + lane;
#pragma unroll 4
    for (int r = 0; r < 32; r++) {
      if (lane < CH && f0 + r < NN && row < A.hi) dst[(int64_t)A.N * (f0 + r) + row] = T[r][lane];
    }
    __syncwarp();
  }
}

// scratch plane `pl`, row `row`: lane-contiguous (always coalesced)
__device__ __forceinline__ int64_t scr_idx(const SweepArgs& A, int pl, int row, int tile, int lane) {
  return ((int64_t)pl * A.N + row) * A.nfpad + (int64_t)tile * 32 + lane;
}

constexpr int SWEEP_WARPS = 4;

// Constant-matrix (mass) sweep: forward elimination with the precomputed
// unit-lower factor, then back substitution; the forward intermediate goes
// through scratch plane 0.
template <int P, int CH>
__global__ void __launch_bounds__(32 * SWEEP_WARPS)
sweep_mass_kernel(const SweepArgs A) {
  constexpr int W = 2 * P + 1;
  extern __shared__ double smem[];
  double* fac = smem;                                                  // N * W
  double(*T)[33] = reinterpret_cast<double(*)[33]>(smem + A.N * W) + (threadIdx.x >> 5) * 32;
  for (int x = threadIdx.x; x < A.N * W; x += blockDim.x) fac[x] = A.fac[x];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warp = blockIdx.x * SWEEP_WARPS + (threadIdx.x >> 5);
  const int nwarps = gridDim.x * SWEEP_WARPS;
  const int lo = A.lo, hi = A.hi;
  const int last = lo + ((hi - lo - 1) / CH) * CH;
  for (int tile = warp; tile < A.ntiles; tile += nwarps) {
    int64_t base, stride;
    bool valid;
    fiber_geom(A, tile, lane, base, stride, valid);
    double yw[P];
#pragma unroll
    for (int q = 0; q < P; q++) yw[q] = 0.0;
    for (int c0 = lo; c0 < hi; c0 += CH) {
      double v[CH];
      load_rows<CH>(A, A.in, tile, lane, base, stride, valid, c0, T, v);
#pragma unroll
      for (int r = 0; r < CH; r++) {
        const int row = c0 + r;
        if (row < hi) {
          const double* fr = fac + (row - lo) * W;
          double y = v[r];
#pragma unroll
          for (int q = 0; q < P; q++) y = fma(-fr[q], yw[q], y);
#pragma unroll
          for (int q = P - 1; q > 0; q--) yw[q] = yw[q - 1];
          yw[0] = y;
          A.scr[scr_idx(A, 0, row, tile, lane)] = y;
        }
      }
    }
    double xw[P];
#pragma unroll
    for (int q = 0; q < P; q++) xw[q] = 0.0;
    for (int c0 = last; c0 >= lo; c0 -= CH) {
      double v[CH];
#pragma unroll
      for (int r = 0; r < CH; r++) {
        const int row = c0 + r;
        v[r] = row < hi ? A.scr[scr_idx(A, 0, row, tile, lane)] : 0.0;
      }
#pragma unroll
      for (int r = CH - 1; r >= 0; r--) {
        const int row = c0 + r;
        if (row < hi) {
          const double* fr = fac + (row - lo) * W;
          double x = v[r];
#pragma unroll
          for (int q = 0; q < P; q++) x = fma(-fr[P + 1 + q], xw[q], x);
          x *= fr[P];
#pragma unroll
          for (int q = P - 1; q > 0; q--) xw[q] = xw[q - 1];
          xw[0] = x;
          v[r] = x;
        }
      }
      store_rows<CH>(A, A.out, tile, lane, base, stride, valid, c0, T, v);
    }
  }
}

// Row-modified sweep: row k of fiber solves
//   sum_j (M_kj + c_k S_kj) x_j = f_k,   c_k = c of the row's test function,
// banded LU without pivoting computed on the fly (Doolittle), intermediates
// (y_k, 1/u_kk, u_{k,k+1..k+P}) through scratch planes 0..P+1.
template <int P, int CH>
__global__ void __launch_bounds__(32 * SWEEP_WARPS)
sweep_mod_kernel(const SweepArgs A) {
  constexpr int W = 2 * P + 1;
  extern __shared__ double smem[];
  double* Mb = smem;           // N * W
  double* Sb = smem + A.N * W; // N * W
  double(*T)[33] = reinterpret_cast<double(*)[33]>(smem + 2 * A.N * W) + (threadIdx.x >> 5) * 32;
  for (int x = threadIdx.x; x < A.N * W; x += blockDim.x) {
    Mb[x] = A.Mb[x];
    Sb[x] = A.Sb[x];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warp = blockIdx.x * SWEEP_WARPS + (threadIdx.x >> 5);
  const int nwarps = gridDim.x * SWEEP_WARPS;
  const int lo = A.lo, hi = A.hi;
  const int last = lo + ((hi - lo - 1) / CH) * CH;
  for (int tile = warp; tile < A.ntiles; tile += nwarps) {
    int64_t base, stride;
    bool valid;
    fiber_geom(A, tile, lane, base, stride, valid);
    // window of the previous P rows: uw[m-1][q] = u_{k-m, k-m+q}, iw[m-1] = 1/u_{k-m,k-m}, yw[m-1] = y_{k-m}
    double uw[P][P + 1], iw[P], yw[P];
#pragma unroll
    for (int m = 0; m < P; m++) {
      iw[m] = 0.0;
      yw[m] = 0.0;
#pragma unroll
      for (int q = 0; q <= P; q++) uw[m][q] = 0.0;
    }
    for (int c0 = lo; c0 < hi; c0 += CH) {
      double f[CH], cc[CH];
      load_rows<CH>(A, A.in, tile, lane, base, stride, valid, c0, T, f);
      load_rows<CH>(A, A.c, tile, lane, base, stride, valid, c0, T, cc);
#pragma unroll
      for (int r = 0; r < CH; r++) {
        const int row = c0 + r;
        if (row < hi) {
          const double* mr = Mb + row * W;
          const double* sr = Sb + row * W;
          double a[W];
#pragma unroll
          for (int q = 0; q < W; q++) a[q] = fma(cc[r], sr[q], mr[q]);  // a[q] = A_{k, k-P+q}
          // multipliers l_{k,k-m}, m = P..1
          double l[P + 1];
#pragma unroll
          for (int m = P; m >= 1; m--) {
            double s = a[P - m];
#pragma unroll
            for (int mp = P; mp > m; mp--) s = fma(-l[mp], uw[mp - 1][mp - m], s);
            l[m] = s * iw[m - 1];
          }
          // U row
          double u[P + 1];
#pragma unroll
          for (int q = 0; q <= P; q++) {
            double s = a[P + q];
#pragma unroll
            for (int m = 1; m <= P; m++)
              if (m + q <= P) s = fma(-l[m], uw[m - 1][m + q], s);
            u[q] = s;
          }
          const double iu = valid ? __drcp_rn(u[0]) : 0.0;
          double y = f[r];
#pragma unroll
          for (int m = 1; m <= P; m++) y = fma(-l[m], yw[m - 1], y);
          // shift windows
#pragma unroll
          for (int m = P - 1; m > 0; m--) {
            iw[m] = iw[m - 1];
            yw[m] = yw[m - 1];
#pragma unroll
            for (int q = 0; q <= P; q++) uw[m][q] = uw[m - 1][q];
          }
          iw[0] = iu;
          yw[0] = y;
#pragma unroll
          for (int q = 0; q <= P; q++) uw[0][q] = u[q];
          A.scr[scr_idx(A, 0, row, tile, lane)] = y;
          A.scr[scr_idx(A, 1, row, tile, lane)] = iu;
#pragma unroll
          for (int q = 1; q <= P; q++) A.scr[scr_idx(A, 1 + q, row, tile, lane)] = u[q];
        }
      }
    }
    double xw[P];
#pragma unroll
    for (int q = 0; q < P; q++) xw[q] = 0.0;
    for (int c0 = last; c0 >= lo; c0 -= CH) {
      double v[CH];
#pragma unroll
      for (int r = CH - 1; r >= 0; r--) {
        const int row = c0 + r;
        if (row < hi) {
          double x = A.scr[scr_idx(A, 0, row, tile, lane)];
#pragma unroll
          for (int q = 0; q < P; q++) x = fma(-A.scr[scr_idx(A, 2 + q, row, tile, lane)], xw[q], x);
          x *= A.scr[scr_idx(A, 1, row, tile, lane)];
#pragma unroll
          for (int q = P - 1; q > 0; q--) xw[q] = xw[q - 1];
          xw[0] = x;
          v[r] = x;
        } else {
          v[r] = 0.0;
        }
      }
      store_rows<CH>(A, A.out, tile, lane, base, stride, valid, c0, T, v);
    }
  }
}

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

__global__ void fill_kernel(double* __restrict__ x, int64_t n, double v) {
  for (int64_t I = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; I < n; I += (int64_t)gridDim.x * blockDim.x) x[I] = v;
}

// Pivot scan of the row-modified factorisations (D12 gate): for every fiber of
// the given sweep, run the no-pivot LU and record min |u_kk| / max|row|.
template <int P>
__global__ void pivot_scan_kernel(const SweepArgs A, unsigned long long* bad_fiber, double tol) {
  constexpr int W = 2 * P + 1;
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int tile = warp; tile < A.ntiles; tile += nwarps) {
    int64_t base, stride;
    bool valid;
    fiber_geom(A, tile, lane, base, stride, valid);
    if (!valid) continue;
    double uw[P][P + 1], iw[P];
    for (int m = 0; m < P; m++) {
      iw[m] = 0.0;
      for (int q = 0; q <= P; q++) uw[m][q] = 0.0;
    }
    for (int row = A.lo; row < A.hi; row++) {
      const double cr = A.c[base + (int64_t)row * stride];
      double a[W], amax = 0.0;
      for (int q = 0; q < W; q++) {
        a[q] = fma(cr, A.Sb[row * W + q], A.Mb[row * W + q]);
        amax = fmax(amax, fabs(a[q]));
      }
      double l[P + 1];
      for (int m = P; m >= 1; m--) {
        double s = a[P - m];
        for (int mp = P; mp > m; mp--) s = fma(-l[mp], uw[mp - 1][mp - m], s);
        l[m] = s * iw[m - 1];
      }
      double u[P + 1];
      for (int q = 0; q <= P; q++) {
        double s = a[P + q];
        for (int m = 1; m <= P; m++)
          if (m + q <= P) s = fma(-l[m], uw[m - 1][m + q], s);
        u[q] = s;
      }
      if (!(fabs(u[0]) >= tol * amax)) {
        atomicMin(bad_fiber, (unsigned long long)((int64_t)tile * 32 + lane));
        break;
      }
      for (int m = P - 1; m > 0; m--) {
        iw[m] = iw[m - 1];
        for (int q = 0; q <= P; q++) uw[m][q] = uw[m - 1][q];
      }
      iw[0] = 1.0 / u[0];
      for (int q = 0; q <= P; q++) uw[0][q] = u[q];
    }
  }
}

}  // namespace adi
