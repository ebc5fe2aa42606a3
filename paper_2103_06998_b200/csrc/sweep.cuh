// sweep.cuh -- batched banded sweeps along one axis for every fiber
// (P:468-527 systems A, B, C; row-modified form P:529-594 / Appendix).
//
// One lane solves one fiber; a warp owns a tile of 32 fibers; a launch carries
// up to three independent jobs (e.g. the three field components, each with its
// own axis and PEC row range, D1).  Per tile:
//   pass 1  streams the fiber rows forward through a per-warp cp.async ring in
//           shared memory (RS chunks of CH rows in flight), runs the forward
//           elimination and stores only the recurrence state at every chunk
//           start (a per-warp checkpoint slot in global memory, L2-resident);
//   pass 2  walks the chunks backwards: the ring re-loads a chunk (an L2 hit
//           for recently streamed fibers), the forward elimination of that
//           chunk is recomputed from its checkpoint and the back substitution
//           writes the solution.
// HBM traffic is the algorithmic minimum: read f (and c, pivots), write x.
//
// Modes: SW_MASS solves M x = f; SW_MOD solves (M + diag(c) S) x = f; SW_DER
// is the derivative projection of the uniform-mu H update (SURVEY §8(a)
// note: M^{-1}(M (x) A (x) M) = I (x) M^{-1}A (x) I along the axis):
//   out = base + coef * M^{-1} (A u)       (A applied on the fly, window +-P)
// Constant (mass) matrix: precomputed LU factors; rows [hk, tk) equal the
// interior factor row to 2 ulp and come from the kernel parameters.
// Row-modified matrix M + diag(c) S (c = tau^2/(4 eps^ mu^) of the row's test
// function): the pivots 1/u_kk are cached per fiber at set_materials/set_tau
// (factor_kernel); the multipliers and the U row are recomputed from c in
// registers, so the recurrence carries no division.  No pivoting (D12; the
// factor kernel rejects tiny pivots).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include <type_traits>

namespace adi {

constexpr int SW_MAXJOBS = 3;
constexpr int SW_WARPS = 4;  // warps per block
enum SweepMode { SW_MASS = 0, SW_MOD = 1, SW_DER = 2 };
// chunk rows (CH) and ring depth (RS) per mode
#ifndef ADI_SW_TUNE  // (tuning builds override these with -D)
#define ADI_SW_CH_MASS 16
#define ADI_SW_RS_MASS 4
#define ADI_SW_CH_MOD 8
#define ADI_SW_RS_MOD 3
#define ADI_SW_CH_DER 8
#define ADI_SW_RS_DER 4
#endif
// Row-modified sweep: recompute the pivots 1/u_kk in the recurrence (1) instead of
// streaming the cached pivot array (0).  The cache is still built (and gated, D12) at
// set_materials; the recomputation is the same arithmetic, so results are bit-identical.
#ifndef ADI_SW_MOD_RECIP
#define ADI_SW_MOD_RECIP 1
#endif
// Mass sweep: pass 1 stores the forward-eliminated y in `out` and pass 2 only
// back-substitutes from it (1), instead of re-reading f and recomputing (0).
#ifndef ADI_SW_MASS_Y
#define ADI_SW_MASS_Y 0
#endif
#ifndef ADI_SW_MINB_MASS  // resident blocks the mass kernel's register budget is sized for
#define ADI_SW_MINB_MASS 2
#endif
#ifndef ADI_SW_MINB_MOD
#define ADI_SW_MINB_MOD 1
#endif
constexpr int SW_CH_MASS = ADI_SW_CH_MASS, SW_RS_MASS = ADI_SW_RS_MASS;
constexpr int SW_CH_MOD = ADI_SW_CH_MOD, SW_RS_MOD = ADI_SW_RS_MOD;
constexpr int SW_CH_DER = ADI_SW_CH_DER, SW_RS_DER = ADI_SW_RS_DER;
__host__ __device__ constexpr int sw_ch(int mode) { return mode == SW_MOD ? SW_CH_MOD : mode == SW_DER ? SW_CH_DER : SW_CH_MASS; }
__host__ __device__ constexpr int sw_rs(int mode) { return mode == SW_MOD ? SW_RS_MOD : mode == SW_DER ? SW_RS_DER : SW_RS_MASS; }
constexpr bool SW_MOD_RECIP = ADI_SW_MOD_RECIP != 0;
__host__ __device__ constexpr int sw_na(int mode) { return mode == SW_MOD ? (SW_MOD_RECIP ? 2 : 3) : mode == SW_DER ? 2 : 1; }
// checkpoint words per chunk: y window (P); MOD adds the U entries u_{k-m,k-m+j}, j < P
// (P(P-1); u_{k-m,k-m+P} = M + c S entries are re-read from c, the pivots 1/u_{k-m,k-m}
// from the pivot cache or, with SW_MOD_RECIP, kept in the checkpoint: P more words);
// DER: y only (the u window is re-read from u)
__host__ __device__ constexpr int sw_state_words(int mode, int P) {
  return mode == SW_MOD ? P * P + (SW_MOD_RECIP ? P : 0) : P;
}
// (the twisted kernel keeps the u window in its checkpoints)
__host__ __device__ constexpr int sw_state_words_tw(int mode, int P) { return mode == SW_DER ? 2 * P : P; }
template <int MODE>
constexpr size_t sw_smem_bytes() {
  return sizeof(double) * (size_t)SW_WARPS * sw_rs(MODE) * sw_na(MODE) * sw_ch(MODE) * 33;
}

struct SweepJob {
  const double* in;   // right-hand side (MASS/MOD) or u (DER), N^3
  double* out;        // solution (may equal in / base)
  const double* c;    // per-test-function c (MOD)
  const double* iu;   // cached pivots 1/u_kk of this family (MOD)
  const double* base; // DER: out = base + coef * M^{-1} A u
  double* out2;       // DER, TMA-staged kernel only (or nullptr): out2 = out + coef * M^{-1} A u
  double coef;
  int axis;           // 0 = x, 1 = y, 2 = z
  int lo, hi;         // active rows along the axis (PEC, D1)
  int var;            // band-table variant: 0 = [0,N), 1 = [1,N-1)
  int dims[3];        // box extents (x fastest); dims[axis] = N (fibers span the patch)
  int tile0;          // first tile of this job in the launch
};

struct SweepBatch {
  SweepJob job[SW_MAXJOBS];
  int njobs;
  int N;               // fiber length (global extent along the sweep axis)
  int ntiles;          // 32-fiber tiles of all jobs
  int nck;             // checkpoint slots per warp (chunks per fiber)
  double* ckpt;        // per-warp checkpoint slots
  // constant (mass) factors per variant: rows = absolute row index, W entries:
  //   [0..P-1] l_{k,k-1-q}, [P] 1/u_kk, [P+1..2P] u_{k,k+1+q}
  const double* fac[2];
  int hk[2], tk[2];    // rows in [hk, tk) equal kfac to 2 ulp
  double kfac[2][11];
  // row-modified: band rows of M and S restricted to the variant's range
  const double* Mb[2];
  const double* Sb[2];
  double kM[11], kS[11];  // interior Toeplitz rows (rows in [2P, N-2P))
  // derivative projection: band rows of A (full range) and its interior row
  const double* Ab;
  double kA[11];
  // twisted (two-segment SPIKE) constant-matrix sweeps, per variant: split row m1,
  // spike columns sp[row * P + j] (V1 above m1, W2 from m1 on) and the interface
  // matrices Vb, Wt and K = (I - Vb Wt)^{-1} (P x P, row-major) -- sweep_tw.cuh
  const double* sp[2];
  int m1[2];
  int spl[2], sph[2];  // spike entries outside patch rows [spl, sph) are below 1e-20 of the largest (dropped)
  double vb[2][25], wt[2][25], kk[2][25];
};

__device__ __forceinline__ void sw_cp_async8(double* smem_dst, const double* gsrc) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void sw_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void sw_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

template <int P, int MODE>
__global__ void __launch_bounds__(32 * SW_WARPS, MODE == SW_MASS ? ADI_SW_MINB_MASS : MODE == SW_MOD ? ADI_SW_MINB_MOD : 1) sweep_kernel(const __grid_constant__ SweepBatch B) {
  constexpr bool MOD = MODE == SW_MOD, DER = MODE == SW_DER;
  constexpr int CH = sw_ch(MODE), RS = sw_rs(MODE), NA = sw_na(MODE);
  constexpr int W = 2 * P + 1;
  constexpr int SLOT = NA * CH * 33;
  constexpr int SWD = sw_state_words(MODE, P);
  constexpr int UW = MOD && P > 1 ? P - 1 : 1;  // stash width of U entries per row (pass 2)
  constexpr bool RECIP = MOD && SW_MOD_RECIP;     // pivots recomputed, not streamed
  constexpr bool YST = MODE == SW_MASS && ADI_SW_MASS_Y;  // y stored by pass 1 (no recompute)
  static_assert(!DER || (RS >= 3 && CH >= P), "derivative mode needs the next chunk resident");
  extern __shared__ double sw_smem[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* ring = sw_smem + (size_t)wib * RS * SLOT;
  const int gw = blockIdx.x * SW_WARPS + wib;
  const int nw = gridDim.x * SW_WARPS;
  const int N = B.N;
  double* ck = B.ckpt + (size_t)gw * B.nck * SWD * 32 + lane;
  const int total = B.ntiles;

  for (int t = gw; t < total; t += nw) {
    const int jb = (B.njobs > 1 && t >= B.job[1].tile0) + (B.njobs > 2 && t >= B.job[2].tile0);
    const double* src[3];
    double* out;
    double coef;
    int axis, lo, hi, var, nx, ny, tile;
    int64_t NN;  // fibers of the job
    {
      const SweepJob& J = jb == 0 ? B.job[0] : jb == 1 ? B.job[1] : B.job[2];
      tile = t - J.tile0;
      nx = J.dims[0];
      ny = J.dims[1];
      NN = J.axis == 0 ? (int64_t)J.dims[1] * J.dims[2] : J.axis == 1 ? (int64_t)J.dims[0] * J.dims[2]
                                                                       : (int64_t)J.dims[0] * J.dims[1];
      src[0] = J.in;
      src[1] = DER ? J.base : J.c;
      src[2] = RECIP ? nullptr : J.iu;
      out = J.out;
      coef = J.coef;
      axis = J.axis;
      lo = J.lo;
      hi = J.hi;
      var = J.var;
    }
    const int64_t f0 = (int64_t)tile * 32;
    const int64_t f = f0 + lane;
    const bool fval = f < NN;
    const int64_t fc = fval ? f : NN - 1;  // invalid lanes load (and never store) a valid fiber
    int64_t base, stride;
    if (axis == 2) {
      base = fc;
      stride = (int64_t)nx * ny;
    } else if (axis == 1) {
      base = (fc % nx) + (int64_t)nx * ny * (fc / nx);
      stride = nx;
    } else {
      base = (int64_t)nx * fc;
      stride = 1;
    }
    const int nc = (hi - lo + CH - 1) / CH;
    // x axis: lane loads row (lane % CH) of fiber m*(32/CH) + lane/CH, m = 0..CH-1
    constexpr int FPI = 32 / CH;
    const int xr = lane % CH, xf = lane / CH;

    // chunk c of the tile -> ring slot c % RS (layout [array][row][33], lane = fiber).
    // Rows past hi are not loaded (the compute skips them).  na: arrays to load
    // (DER loads `base` only in pass 2).
    auto issue = [&](int c, int na) {
      double* sl = ring + (c % RS) * SLOT;
      const int r0 = lo + c * CH;
      const int nr = min(CH, hi - r0);
      if (axis != 0) {
        const int64_t o = base + (int64_t)r0 * stride;
        const double* p0 = src[0] + o;
        const double* p1 = NA > 1 ? src[1] + o : nullptr;
        const double* p2 = NA > 2 ? src[2] + o : nullptr;
#pragma unroll
        for (int r = 0; r < CH; r++) {
          if (r < nr) {
            sw_cp_async8(sl + r * 33 + lane, p0);
            if (NA > 1 && (!DER || na > 1)) sw_cp_async8(sl + (CH + r) * 33 + lane, p1);
            if (NA > 2) sw_cp_async8(sl + (2 * CH + r) * 33 + lane, p2);
          }
          p0 += stride;
          if (NA > 1) p1 += stride;
          if (NA > 2) p2 += stride;
        }
      } else {
        const int row = min(r0 + xr, hi - 1);
        const int64_t o0 = (int64_t)nx * f0 + row;
        const int64_t fmax = NN - 1 - f0;  // last valid fiber offset in the tile
#pragma unroll
        for (int m = 0; m < CH; m++) {
          const int ff = m * FPI + xf;
          const int64_t off = ff <= fmax ? o0 + (int64_t)nx * ff : o0;
          double* d = sl + xr * 33 + ff;
          sw_cp_async8(d, src[0] + off);
          if (NA > 1 && (!DER || na > 1)) sw_cp_async8(d + CH * 33, src[1] + off);
          if (NA > 2) sw_cp_async8(d + 2 * CH * 33, src[2] + off);
        }
      }
      sw_commit();
    };

    // per-tile constants in registers (var is runtime: no dynamic parameter indexing per row)
    const double* fac = var ? B.fac[1] : B.fac[0];
    const double* Mb = var ? B.Mb[1] : B.Mb[0];
    const double* Sb = var ? B.Sb[1] : B.Sb[0];
    const int hk = var ? B.hk[1] : B.hk[0];
    const int tk = var ? B.tk[1] : B.tk[0];
    double kf[MOD ? 1 : W];
    if (!MOD) {
#pragma unroll
      for (int q = 0; q < W; q++) kf[q] = var ? B.kfac[1][q] : B.kfac[0][q];
    }

    // recurrence state: yw[m-1] = y_{k-m}; (MOD) uw[m-1][j-1] = u_{k-m,k-m+j}, iw[m-1] = 1/u_{k-m,k-m};
    // (DER) dv[0..2P-1] = u_{k-P..k+P-1} before row k is eliminated
    double yw[P];
    double uw[MOD ? P : 1][P];
    double iw[MOD ? P : 1];
    double dv[DER ? W : 1];
#pragma unroll
    for (int m = 0; m < P; m++) yw[m] = 0.0;
    if (MOD) {
#pragma unroll
      for (int m = 0; m < P; m++) {
        iw[m] = 0.0;
#pragma unroll
        for (int j = 0; j < P; j++) uw[m][j] = 0.0;
      }
    }
    if (DER) {
#pragma unroll
      for (int q = 0; q < W; q++) dv[q] = 0.0;
    }

    // entry q of row k of the modified matrix: M_{k,k-P+q} + c_k S_{k,k-P+q};
    // FAST: the row is Toeplitz (k in [2P, N-2P)), entries from the parameter bank
    auto mod_entry = [&](auto fast, int row, double cc, int q) -> double {
      if constexpr (decltype(fast)::value) {
        return fma(cc, B.kS[q], B.kM[q]);
      } else {
        const bool in = row >= 2 * P && row < N - 2 * P;
        const double mq = in ? B.kM[q] : __ldg(Mb + (size_t)row * W + q);
        const double sq = in ? B.kS[q] : __ldg(Sb + (size_t)row * W + q);
        return fma(cc, sq, mq);
      }
    };
    // factor entry q of row k of the mass LU; FAST: k in [hk, tk)
    auto fac_entry = [&](auto fast, int row, int q) -> double {
      if constexpr (decltype(fast)::value) {
        return kf[q];
      } else {
        const bool in = row >= hk && row < tk;
        return in ? kf[q] : __ldg(fac + (size_t)row * W + q);
      }
    };
    // (DER) f_k = sum_q A_{k,k-P+q} u_{k-P+q} from the window dv
    auto der_rhs = [&](auto fast, int row) -> double {
      double fv = 0.0;
#pragma unroll
      for (int q = 0; q < W; q++) {
        double aq;
        if constexpr (decltype(fast)::value) {
          aq = B.kA[q];
        } else {
          const bool in = row >= 2 * P && row < N - 2 * P;
          aq = in ? B.kA[q] : __ldg(B.Ab + (size_t)row * W + q);
        }
        fv = fma(aq, dv[q], fv);
      }
      return fv;
    };
    // one forward elimination step (row k): returns y_k, and (MOD) u_{k,k+q}, q = 1..P in un[]
    auto fwd = [&](auto fast, int row, double fv, double cc, double ivk, double* un, double& ivo) -> double {
      double y = fv;
      if (MOD) {
        double a[W];
#pragma unroll
        for (int q = 0; q < W; q++) a[q] = mod_entry(fast, row, cc, q);
        double l[P + 1];
#pragma unroll
        for (int m = P; m >= 1; m--) {
          double s = a[P - m];
#pragma unroll
          for (int mp = P; mp > m; mp--) s = fma(-l[mp], uw[mp - 1][mp - m - 1], s);
          l[m] = s * iw[m - 1];
        }
        if (RECIP) {  // u_kk exactly as factor_kernel forms it
          double u0 = a[P];
#pragma unroll
          for (int m = 1; m <= P; m++) u0 = fma(-l[m], uw[m - 1][m - 1], u0);
          ivk = 1.0 / u0;
        }
        ivo = ivk;
#pragma unroll
        for (int q = 1; q <= P; q++) {
          double s = a[P + q];
#pragma unroll
          for (int m = 1; m + q <= P; m++) s = fma(-l[m], uw[m - 1][m + q - 1], s);
          un[q - 1] = s;
        }
#pragma unroll
        for (int m = P; m >= 1; m--) y = fma(-l[m], yw[m - 1], y);
#pragma unroll
        for (int m = P - 1; m > 0; m--) {
          iw[m] = iw[m - 1];
#pragma unroll
          for (int j = 0; j < P; j++) uw[m][j] = uw[m - 1][j];
        }
        iw[0] = ivk;
#pragma unroll
        for (int j = 0; j < P; j++) uw[0][j] = un[j];
      } else {
#pragma unroll
        for (int q = P - 1; q >= 0; q--) y = fma(-fac_entry(fast, row, q), yw[q], y);
      }
#pragma unroll
      for (int m = P - 1; m > 0; m--) yw[m] = yw[m - 1];
      yw[0] = y;
      return y;
    };
    auto save_state = [&](int c) {
      double* p = ck + (size_t)c * SWD * 32;
#pragma unroll
      for (int m = 0; m < P; m++) p[m * 32] = yw[m];
      if (MOD) {
#pragma unroll
        for (int m = 0; m < P; m++)
#pragma unroll
          for (int j = 0; j < P - 1; j++) p[(P + m * (P - 1) + j) * 32] = uw[m][j];
      }
      if (RECIP) {
#pragma unroll
        for (int m = 0; m < P; m++) p[(P * P + m) * 32] = iw[m];
      }
    };
    // pv[m-1], pc[m-1]: pivot 1/u and c of patch row r0 - m (MOD; loaded ahead of time)
    auto set_state = [&](const double* p, const double* pv, const double* pc, int r0) {
#pragma unroll
      for (int m = 0; m < P; m++) yw[m] = p[m];
      if (MOD) {
#pragma unroll
        for (int m = 0; m < P; m++) {
#pragma unroll
          for (int j = 0; j < P - 1; j++) uw[m][j] = p[P + m * (P - 1) + j];
          const int row = r0 - 1 - m;
          iw[m] = row >= lo ? (RECIP ? p[P * P + m] : pv[m]) : 0.0;
          uw[m][P - 1] = row >= lo ? mod_entry(std::false_type{}, row, pc[m], 2 * P) : 0.0;
        }
      }
      if (DER) {  // dv[q] = u_{r0-P+q}: pv[m] holds u at row r0-1-m
#pragma unroll
        for (int q = 0; q < P; q++) dv[q] = (r0 - P + q >= lo) ? pv[P - 1 - q] : 0.0;
      }
    };
    // chunk rows all in [lo,hi) and in the Toeplitz / converged range?
    auto chunk_fast = [&](int r0) {
      return r0 + CH <= hi && (MOD || DER ? (r0 >= 2 * P && r0 + CH <= N - 2 * P) : true) &&
             (MOD ? true : (r0 >= hk && r0 + CH <= tk));
    };
    // (DER) u at row r0+r of chunk slot sl, rows past the chunk from `nx` (next chunk) or `hd` (saved head)
    auto der_u = [&](const double* sl, const double* nx, const double* hd, int r0, int r) -> double {
      if (r0 + r >= hi) return 0.0;
      if (r < CH) return sl[r * 33 + lane];
      return nx ? nx[(r - CH) * 33 + lane] : hd[r - CH];
    };
    // forward elimination of one chunk (pass 1 or the pass-2 recompute); y[] gets y_k,
    // us[] (MOD) u_{k,k+q}, q = 1..P-1.  DER: dv holds u_{r0-P..r0+P-1} on entry
    // (and u_{r0+CH-P..r0+CH+P-1} on exit).
    double xw[P];
    auto fwd_chunk = [&](auto fast, const double* sl, const double* nx, const double* hd, int r0, double* y,
                         double* us, double* ivs) {
#pragma unroll
      for (int r = 0; r < CH; r++) {
        const int row = r0 + r;
        if (decltype(fast)::value || row < hi) {
          double un[P];
          double fv;
          if (DER) {
            // dv[0..2P-1] = u_{row-P..row+P-1} on entry: append u_{row+P}, apply A, slide
            dv[W - 1] = der_u(sl, nx, hd, r0, r + P);
            fv = der_rhs(fast, row);
#pragma unroll
            for (int q = 0; q < W - 1; q++) dv[q] = dv[q + 1];
          } else {
            fv = sl[r * 33 + lane];
          }
          double ivo;
          const double yy = fwd(fast, row, fv, MOD ? sl[(CH + r) * 33 + lane] : 0.0,
                                MOD && !RECIP ? sl[(2 * CH + r) * 33 + lane] : 0.0, un, ivo);
          if (y) y[r] = yy;
          if (RECIP && ivs) ivs[r] = ivo;
          if (MOD && us) {
#pragma unroll
            for (int q = 0; q < P - 1; q++) us[r * UW + q] = un[q];
          }
        }
      }
    };
    // back substitution of one chunk (y[] -> x[] in place)
    auto bwd_chunk = [&](auto fast, const double* sl, int r0, double* y, double* us, const double* ivs) {
#pragma unroll
      for (int r = CH - 1; r >= 0; r--) {
        const int row = r0 + r;
        if (decltype(fast)::value || row < hi) {
          double x = y[r];
          if (MOD) {
            const double cc = sl[(CH + r) * 33 + lane];
            x = fma(-mod_entry(fast, row, cc, 2 * P), xw[P - 1], x);
#pragma unroll
            for (int q = P - 1; q >= 1; q--) x = fma(-us[r * UW + q - 1], xw[q - 1], x);
            x *= RECIP ? ivs[r] : sl[(2 * CH + r) * 33 + lane];
          } else {
#pragma unroll
            for (int q = P - 1; q >= 0; q--) x = fma(-fac_entry(fast, row, P + 1 + q), xw[q], x);
            x *= fac_entry(fast, row, P);
          }
#pragma unroll
          for (int q = P - 1; q > 0; q--) xw[q] = xw[q - 1];
          xw[0] = x;
          y[r] = x;
        }
      }
    };
    // DER: load u_{r0..r0+P-1} (the first P rows of the chunk) into dv[P..2P-1]
    auto der_prime = [&](const double* sl, int r0) {
#pragma unroll
      for (int q = 0; q < P; q++) dv[P + q] = (r0 + q < hi) ? sl[q * 33 + lane] : 0.0;
    };
    // Fast chunks of the constant-matrix modes (every row interior and converged):
    // static row arrays instead of shifting windows (no register moves per row).
    // yv[P + r] = y_{r0+r}; yv[0..P-1] = y_{r0-P..r0-1} from the recurrence state.
    auto fwd_fast_cm = [&](const double* sl, const double* nx, const double* hd, double* yv) {
#pragma unroll
      for (int q = 0; q < P; q++) yv[q] = yw[P - 1 - q];
      double uv[DER ? CH + 2 * P : 1];  // (DER) u_{r0-P+j}
      if (DER) {
#pragma unroll
        for (int q = 0; q < P; q++) uv[q] = dv[q];
#pragma unroll
        for (int r = 0; r < CH; r++) uv[P + r] = sl[r * 33 + lane];
#pragma unroll
        for (int q = 0; q < P; q++) uv[P + CH + q] = nx ? nx[q * 33 + lane] : hd[q];
      }
#pragma unroll
      for (int r = 0; r < CH; r++) {
        double y;
        if (DER) {
          y = 0.0;
#pragma unroll
          for (int q = 0; q < W; q++) y = fma(B.kA[q], uv[r + q], y);
        } else {
          y = sl[r * 33 + lane];
        }
#pragma unroll
        for (int q = P - 1; q >= 0; q--) y = fma(-kf[q], yv[P + r - 1 - q], y);
        yv[P + r] = y;
      }
#pragma unroll
      for (int q = 0; q < P; q++) yw[q] = yv[P + CH - 1 - q];
      if (DER) {
#pragma unroll
        for (int q = 0; q < P; q++) dv[q] = uv[CH + q];
      }
    };
    auto bwd_fast_cm = [&](const double* yv, double* y) {
      double xv[CH + P];  // xv[r] = x_{r0+r}; xv[CH+q] = x_{r0+CH+q}
#pragma unroll
      for (int q = 0; q < P; q++) xv[CH + q] = xw[q];
#pragma unroll
      for (int r = CH - 1; r >= 0; r--) {
        double x = yv[P + r];
#pragma unroll
        for (int q = P - 1; q >= 0; q--) x = fma(-kf[P + 1 + q], xv[r + 1 + q], x);
        xv[r] = x * kf[P];
      }
#pragma unroll
      for (int q = 0; q < P; q++) xw[q] = xv[q];
#pragma unroll
      for (int r = 0; r < CH; r++) y[r] = xv[r];
    };

    // store rows [r0, r0+CH) of the tile from y[] (x axis: transposed through slot sl)
    auto store_chunk = [&](double* sl, int r0, const double* y) {
      if (axis != 0) {
        double* po = out + base + (int64_t)r0 * stride;
#pragma unroll
        for (int r = 0; r < CH; r++) {
          if (fval && r0 + r < hi) *po = y[r];
          po += stride;
        }
        if (YST) {
#pragma unroll
          for (int r = 0; r < CH; r++) sl[r * 33 + lane] = y[r];
        }
      } else {
        __syncwarp();
#pragma unroll
        for (int r = 0; r < CH; r++) sl[r * 33 + lane] = y[r];
        __syncwarp();
        const int row = r0 + xr;
        double* po = out + (int64_t)nx * f0 + row;
#pragma unroll
        for (int m = 0; m < CH; m++) {
          const int ff = m * FPI + xf;
          if (f0 + ff < NN && row < hi) po[(int64_t)nx * ff] = sl[xr * 33 + ff];
        }
      }
    };

    // ---------------- pass 1: forward elimination, checkpoints ----------------
    // DER needs chunk c+1 resident while eliminating chunk c (window u_{k+P}).
    constexpr int AHEAD = DER ? 1 : 0;
#pragma unroll
    for (int c = 0; c < RS - 1; c++) {
      if (c < nc) issue(c, 1);
      else sw_commit();
    }
    for (int c = 0; c < nc; c++) {
      sw_wait<RS - 2 - AHEAD>();
      __syncwarp();
      const double* sl = ring + (c % RS) * SLOT;
      const double* nx = (DER && c + 1 < nc) ? ring + ((c + 1) % RS) * SLOT : nullptr;
      const int r0 = lo + c * CH;
      if (DER) der_prime(sl, r0);
      if (YST) {
        double y[CH];
        if (chunk_fast(r0)) {
          double yv[P + CH];
          fwd_fast_cm(sl, nx, nullptr, yv);
#pragma unroll
          for (int r = 0; r < CH; r++) y[r] = yv[P + r];
        } else {
#pragma unroll
          for (int r = 0; r < CH; r++) y[r] = 0.0;
          fwd_chunk(std::false_type{}, sl, nx, nullptr, r0, y, nullptr, nullptr);
        }
        __syncwarp();
        store_chunk(const_cast<double*>(sl), r0, y);
      } else {
      save_state(c);
      if (!MOD && chunk_fast(r0)) {
        double yv[P + CH];
        fwd_fast_cm(sl, nx, nullptr, yv);
      } else if (chunk_fast(r0)) {
        fwd_chunk(std::true_type{}, sl, nx, nullptr, r0, nullptr, nullptr, nullptr);
      } else {
        fwd_chunk(std::false_type{}, sl, nx, nullptr, r0, nullptr, nullptr, nullptr);
      }
      }
      __syncwarp();
      if (c + RS - 1 < nc) issue(c + RS - 1, 1);
      else sw_commit();
    }
    sw_wait<0>();
    __syncwarp();
    // ---------------- pass 2: recompute per chunk, back substitution ----------
    // DER re-loads every chunk (u and base); MASS/MOD keep the last RS chunks of pass 1.
    constexpr int KEEP = DER ? 0 : RS;
#pragma unroll
    for (int q = 0; q < P; q++) xw[q] = 0.0;
    double hd[DER ? P : 1];  // (DER) u of the first P rows of chunk c+1
    double nxt[SWD];         // checkpoint of the next chunk to process, loaded one iteration ahead
    double pv[MOD || DER ? P : 1], pc[MOD ? P : 1];  // pivots and c (MOD) / u (DER) of the P rows before that chunk
    auto load_prev = [&](int c) {
#pragma unroll
      for (int q = 0; q < SWD; q++) nxt[q] = ck[((size_t)c * SWD + q) * 32];
      if (MOD || DER) {
        const int r0 = lo + c * CH;
#pragma unroll
        for (int m = 0; m < P; m++) {
          const int row = max(r0 - 1 - m, lo);
          if (MOD) {
            if (!RECIP) pv[m] = __ldg(src[2] + base + (int64_t)row * stride);
            pc[m] = __ldg(src[1] + base + (int64_t)row * stride);
          } else {
            pv[m] = __ldg(src[0] + base + (int64_t)row * stride);
          }
        }
      }
    };
    if (YST) src[0] = out;  // pass 2 streams y back from out
    else load_prev(nc - 1);
    if (DER) {
#pragma unroll
      for (int c = 0; c < RS - 1; c++) {
        if (nc - 1 - c >= 0) issue(nc - 1 - c, 2);
        else sw_commit();
      }
#pragma unroll
      for (int q = 0; q < P; q++) hd[q] = 0.0;
    }
    for (int c = nc - 1; c >= 0; c--) {
      if (c < nc - KEEP) sw_wait<RS - 2>();  // issued RS-1 iterations ago
      __syncwarp();
      double* sl = ring + (c % RS) * SLOT;
      const int r0 = lo + c * CH;
      if (!YST) {
        set_state(nxt, pv, pc, r0);
        if (c > 0) load_prev(c - 1);
      }
      if (DER) der_prime(sl, r0);
      double y[CH];
      double us[CH * UW];  // u_{k,k+q}, q = 1..P-1 (u_{k,k+P} = a[2P] is recomputed)
      double ivs[RECIP ? CH : 1];  // recomputed pivots 1/u_kk of the chunk
      if (YST && chunk_fast(r0)) {
        double yv[P + CH];
#pragma unroll
        for (int r = 0; r < CH; r++) yv[P + r] = sl[r * 33 + lane];
        bwd_fast_cm(yv, y);
      } else if (YST) {
#pragma unroll
        for (int r = 0; r < CH; r++) y[r] = sl[r * 33 + lane];
        bwd_chunk(std::false_type{}, sl, r0, y, us, ivs);
      } else if (!MOD && chunk_fast(r0)) {
        double yv[P + CH];
        fwd_fast_cm(sl, nullptr, hd, yv);
        bwd_fast_cm(yv, y);
      } else if (chunk_fast(r0)) {
        fwd_chunk(std::true_type{}, sl, nullptr, hd, r0, y, us, ivs);
        bwd_chunk(std::true_type{}, sl, r0, y, us, ivs);
      } else {
#pragma unroll
        for (int r = 0; r < CH; r++) y[r] = 0.0;
        fwd_chunk(std::false_type{}, sl, nullptr, hd, r0, y, us, ivs);
        bwd_chunk(std::false_type{}, sl, r0, y, us, ivs);
      }
      if (DER) {
#pragma unroll
        for (int q = 0; q < P; q++) hd[q] = (r0 + q < hi) ? sl[q * 33 + lane] : 0.0;
#pragma unroll
        for (int r = 0; r < CH; r++) y[r] = fma(coef, y[r], sl[(CH + r) * 33 + lane]);
      }
      // store the chunk
      if (YST) __syncwarp();
      store_chunk(sl, r0, y);
      __syncwarp();
      // refill: MASS/MOD slot (c+1)%RS (chunk c+1 done) <- chunk c+1-RS; DER slot c%RS <- chunk c-(RS-1)
      if (DER) {
        if (c - (RS - 1) >= 0) issue(c - (RS - 1), 2);
        else sw_commit();
      } else {
        if (c < nc - 1 && c + 1 - RS >= 0) issue(c + 1 - RS, 1);
        else sw_commit();
      }
    }
    sw_wait<0>();
    __syncwarp();
  }
}

// Pivot cache of one row-modified family (set_materials / set_tau, amortised):
// for every fiber along `axis`, the no-pivot banded LU of M + diag(c) S on
// [lo, hi) in the same arithmetic as sweep_kernel<MOD>; writes 1/u_kk and
// records the first fiber with |u_kk| < tol * max|row| (D12 gate).
template <int P>
__global__ void factor_kernel(const SweepBatch B, double* __restrict__ iu_out, unsigned long long* bad, double tol) {
  constexpr int W = 2 * P + 1;
  const SweepJob& J = B.job[0];
  const int N = B.N;
  const int nx = J.dims[0], ny = J.dims[1];
  const int64_t NN = J.axis == 0 ? (int64_t)J.dims[1] * J.dims[2] : J.axis == 1 ? (int64_t)nx * J.dims[2] : (int64_t)nx * ny;
  const int var = J.var;
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < NN; f += (int64_t)gridDim.x * blockDim.x) {
    int64_t base, stride;
    if (J.axis == 2) {
      base = f;
      stride = (int64_t)nx * ny;
    } else if (J.axis == 1) {
      base = (f % nx) + (int64_t)nx * ny * (f / nx);
      stride = nx;
    } else {
      base = (int64_t)nx * f;
      stride = 1;
    }
    double uw[P][P], iw[P];
    for (int m = 0; m < P; m++) {
      iw[m] = 0.0;
      for (int j = 0; j < P; j++) uw[m][j] = 0.0;
    }
    bool failed = false;
    for (int row = J.lo; row < J.hi; row++) {
      const double cc = J.c[base + (int64_t)row * stride];
      const bool in = row >= 2 * P && row < N - 2 * P;
      double a[W], amax = 0.0;
      for (int q = 0; q < W; q++) {
        const double mq = in ? B.kM[q] : B.Mb[var][(size_t)row * W + q];
        const double sq = in ? B.kS[q] : B.Sb[var][(size_t)row * W + q];
        a[q] = fma(cc, sq, mq);
        amax = fmax(amax, fabs(a[q]));
      }
      double l[P + 1];
      for (int m = P; m >= 1; m--) {
        double s = a[P - m];
        for (int mp = P; mp > m; mp--) s = fma(-l[mp], uw[mp - 1][mp - m - 1], s);
        l[m] = s * iw[m - 1];
      }
      double u0 = a[P];
      for (int m = 1; m <= P; m++) u0 = fma(-l[m], uw[m - 1][m - 1], u0);
      double un[P];
      for (int q = 1; q <= P; q++) {
        double s = a[P + q];
        for (int m = 1; m + q <= P; m++) s = fma(-l[m], uw[m - 1][m + q - 1], s);
        un[q - 1] = s;
      }
      if (!(fabs(u0) >= tol * amax)) failed = true;
      const double ivk = failed ? 0.0 : 1.0 / u0;
      iu_out[base + (int64_t)row * stride] = ivk;
      for (int m = P - 1; m > 0; m--) {
        iw[m] = iw[m - 1];
        for (int j = 0; j < P; j++) uw[m][j] = uw[m - 1][j];
      }
      iw[0] = ivk;
      for (int j = 0; j < P; j++) uw[0][j] = un[j];
    }
    if (failed) atomicMin(bad, (unsigned long long)f);
  }
}

}  // namespace adi
