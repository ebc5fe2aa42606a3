// sweep_tma.cuh -- the batched banded sweeps of sweep.cuh (mass, row-modified,
// derivative projection; Appendix) with
// Blackwell bulk data movement.
//
// Same algorithm as sweep_kernel (lane = fiber, warp = 32 fibers, pass 1 =
// forward elimination with per-chunk checkpoints, pass 2 = per-chunk recompute
// + back substitution), but every chunk of 32 fibers x 16 rows moves as ONE
// TMA box (cp.async.bulk.tensor, 4 KB per array) into a per-warp ring of
// mbarrier-tracked slots, and every solved chunk leaves through shared memory
// as ONE TMA store -- instead of 16 per-lane 8-byte cp.async plus 16 scalar
// stores.  The legacy kernel was bound by load/store instruction issue; this
// one issues ~1 bulk copy per 4 KB.
//
// Layout of a slot array (32 fibers x 16 rows, fp64):
//   y / z sweeps: box {32 x-fibers, 16 rows} -> [row][fiber], lane reads row r at
//                 r*32 + lane (conflict-free);
//   x sweeps:     box {16 rows (x), 32 fibers (y)} with the 128-byte swizzle ->
//                 fiber f's 128-byte row holds 16-byte chunk j at (j ^ (f & 7)).
// L2 policy: pass-1 loads evict_last (they are re-read by pass 2), pass-2 loads
// and the stores evict_first, so the re-read window stays resident.
// Fewer warps per SM than the legacy kernel: the pass-2 re-read working set
// (fibers in flight x fiber bytes) must stay well inside the 126 MB L2.
//
// The row-modified mode streams the cached pivots 1/u_kk of the family
// (factor_kernel, the north star's "factorisations cached across steps"):
// with them the forward recurrence has no division on its dependency chain.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "rhs.cuh"
#include "sweep.cuh"

namespace adi {

using st_med = std::integral_constant<int, 2>;  // chunk tag: every row active, per-row tables
constexpr int ST_CH = 16;              // rows per chunk (x sweeps: one 128-byte swizzle row per fiber)
constexpr int ST_ARR = 32 * ST_CH;     // doubles per array per slot (4 KB)
#ifndef ADI_ST_WARPS_MASS
#define ADI_ST_WARPS_MASS 4
#endif
#ifndef ADI_ST_WARPS_MOD
#define ADI_ST_WARPS_MOD 4
#endif
#ifndef ADI_ST_WARPS_DER
#define ADI_ST_WARPS_DER 8
#endif
#ifndef ADI_ST_RS_MASS
#define ADI_ST_RS_MASS 10
#endif
#ifndef ADI_ST_RS_MOD
#define ADI_ST_RS_MOD 4
#endif
#ifndef ADI_ST_RS_DER
#define ADI_ST_RS_DER 3
#endif
__host__ __device__ constexpr int st_warps(int mode) {
  return mode == SW_MOD ? ADI_ST_WARPS_MOD : mode == SW_DER ? ADI_ST_WARPS_DER : ADI_ST_WARPS_MASS;
}
__host__ __device__ constexpr int st_rs(int mode) {
  return mode == SW_MOD ? ADI_ST_RS_MOD : mode == SW_DER ? ADI_ST_RS_DER : ADI_ST_RS_MASS;
}
// arrays per slot: MASS f; MOD f, c, pivots; DER u, base (base only in pass 2)
__host__ __device__ constexpr int st_na(int mode) { return mode == SW_MOD ? 3 : mode == SW_DER ? 2 : 1; }
// checkpoint words per chunk: y window (P); MOD adds u_{k-m,k-m+j}, j < P (the pivots come from the cache)
__host__ __device__ constexpr int st_state_words(int mode, int P) { return mode == SW_MOD ? P * P : P; }
template <int MODE>
constexpr size_t st_smem_bytes() {
  return sizeof(double) * (size_t)st_warps(MODE) * st_rs(MODE) * st_na(MODE) * ST_ARR +
         sizeof(uint64_t) * (size_t)st_warps(MODE) * st_rs(MODE) + 1024;  // + alignment slack
}

// tensor maps of a launch: per job the input, the aux array (c | base), the pivot cache, the output
struct SweepTmaMaps {
  CUtensorMap m[SW_MAXJOBS][4];
};

// fraction of the pass-1 lines that get evict_last priority, per mode: where the in-flight window of
// all resident warps exceeds L2 (derivative projection at 8 warps per SM: 156 MB), protecting every
// line protects none; a fraction that fits stays resident for the pass-2 re-read
#ifndef ADI_ST_KEEP_DER
#define ADI_ST_KEEP_DER 0.15  // measured at c5: 1.0 3.49 ms, 0.7 3.46, 0.5 3.44, 0.3 3.42, 0.15 3.39 per launch
#endif
#ifndef ADI_ST_KEEP_MASS
#define ADI_ST_KEEP_MASS 1.0
#endif
#define ADI_ST_STR2(x) #x
#define ADI_ST_STR(x) ADI_ST_STR2(x)
template <int MODE>
__device__ __forceinline__ uint64_t st_policy_last() {
  uint64_t p;
  if (MODE == SW_DER)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, " ADI_ST_STR(ADI_ST_KEEP_DER) ";\n" : "=l"(p));
  else if (MODE == SW_MASS)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, " ADI_ST_STR(ADI_ST_KEEP_MASS) ";\n" : "=l"(p));
  else
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t st_policy_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st_load(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar,
                                        uint64_t pol) {
#ifdef ADI_ST_NOHINT
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
  return;
#endif
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void st_store(const CUtensorMap* map, int x, int y, int z, const void* src, uint64_t pol) {
#ifdef ADI_ST_NOHINT
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(z), "r"(smem_u32(src))
               : "memory");
  return;
#endif
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2, %3}], [%4], %5;\n" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(x), "r"(y), "r"(z), "r"(smem_u32(src)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void st_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void st_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void st_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void st_fence_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// One tile (32 fibers of one job) of sweep_tma_kernel; XAX: x sweep (swizzled boxes), else y / z.
template <int P, int MODE, bool XAX>
__device__ __forceinline__ void st_tile(const SweepBatch& B, const SweepTmaMaps& MP, const int t, const int jb,
                                        double* ring, uint64_t* bar, unsigned& phase, const uint64_t pol_keep,
                                        const uint64_t pol_drop, double* ck, const int lane) {
  constexpr bool MOD = MODE == SW_MOD, DER = MODE == SW_DER;
  constexpr int CH = ST_CH, RS = st_rs(MODE), NA = st_na(MODE);
  constexpr int W = 2 * P + 1;
  constexpr int SLOT = NA * ST_ARR;
  constexpr int SWD = st_state_words(MODE, P);
  constexpr int UW = MOD && P > 1 ? P - 1 : 1;
  const int N = B.N;
  const SweepJob& J = B.job[jb];
  const int tile = t - J.tile0;
  const int axis = J.axis, lo = J.lo, hi = J.hi, var = J.var;
  const int nx = J.dims[0], ny = J.dims[1];
  const double coef = J.coef;
  // fibers: (x, y) for z sweeps, (x, z) for y sweeps, (y, z) for x sweeps; 32 consecutive
  // along the first of them per tile (TMA zero-fills / clips the ragged tail)
  const int nf = axis == 0 ? ny : nx;
  const int ntf = (nf + 31) >> 5;
  const int tf = tile % ntf, ts = tile / ntf;
  const int f0 = tf * 32;
  constexpr bool xax = XAX;
  const CUtensorMap* m_in = &MP.m[jb][0];
  const CUtensorMap* m_aux = &MP.m[jb][1];
  const CUtensorMap* m_iu = &MP.m[jb][2];
  const CUtensorMap* m_out = &MP.m[jb][3];
  // chunks are aligned to the patch rows (chunk c = rows [16c, 16c + 16)), so every box starts at a
  // 128-byte boundary of an x-fiber; rows outside [lo, hi) (PEC, D1) are skipped and stored back as loaded
  const int nc = (hi + CH - 1) / CH;
  // global coordinates (x, y, z) of the box of chunk c
  auto coords = [&](int c, int& x, int& y, int& z) {
    const int r0 = c * CH;
    if (axis == 2) x = f0, y = ts, z = r0;
    else if (axis == 1) x = f0, y = r0, z = ts;
    else x = r0, y = f0, z = ts;
  };
  // element (lane's fiber, row r) of one slot array
  auto at = [&](const double* a, int r) -> const double& {
    return xax ? a[lane * 16 + ((((r >> 1) ^ (lane & 7)) << 1) | (r & 1))] : a[r * 32 + lane];
  };
  auto atw = [&](double* a, int r) -> double& {
    return xax ? a[lane * 16 + ((((r >> 1) ^ (lane & 7)) << 1) | (r & 1))] : a[r * 32 + lane];
  };
  // lane 0: load chunk c (na arrays) into slot s (= c % RS, tracked incrementally by the callers:
  // the per-chunk modulo and the per-row range predicates were half of the issue slots at c5)
  auto issue = [&](int c, int s, int na, uint64_t pol) {
    if (lane == 0) {
      double* sl = ring + s * SLOT;
      int x, y, z;
      coords(c, x, y, z);
      mbar_expect_tx(&bar[s], (unsigned)(na * ST_ARR * sizeof(double)));
      st_load(sl, m_in, x, y, z, &bar[s], pol);
      if (na > 1) st_load(sl + ST_ARR, m_aux, x, y, z, &bar[s], pol);
      if (na > 2) st_load(sl + 2 * ST_ARR, m_iu, x, y, z, &bar[s], pol);
    }
  };
  auto wait_slot = [&](int s) {
    mbar_wait(&bar[s], (phase >> s) & 1u);
    phase ^= 1u << s;
  };
  auto next_slot = [](int s) { return s + 1 == RS ? 0 : s + 1; };
  auto prev_slot = [](int s) { return s == 0 ? RS - 1 : s - 1; };

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
#ifdef ADI_ST_PRESCALE
  double ks[P];  // U entries scaled by the inverse pivot: back substitution with one FMA on the chain
#pragma unroll
  for (int q = 0; q < P; q++) ks[q] = MOD ? 0.0 : kf[P + 1 + q] * kf[P];
#endif
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
  // fast tag: true_type = interior chunk (constants), st_med = every row active but table factors /
  // boundary stencils (unpredicated table reads: the host stores the reference row in rows [hk, tk),
  // so the read equals the select of the general path bit for bit), false_type = general
  auto fac_entry = [&](auto fast, int row, int q) -> double {
    if constexpr (decltype(fast)::value == 1) {
      return kf[q];
    } else if constexpr (decltype(fast)::value == 2) {
      return __ldg(fac + (size_t)row * W + q);
    } else {
      const bool in = row >= hk && row < tk;
      return in ? kf[q] : __ldg(fac + (size_t)row * W + q);
    }
  };
  auto der_rhs = [&](auto fast, int row) -> double {
    double fv = 0.0;
#pragma unroll
    for (int q = 0; q < W; q++) {
      double aq;
      if constexpr (decltype(fast)::value == 1) {
        aq = B.kA[q];
      } else {  // (general and medium chunks: the A table is shared with the RHS kernels, keep the select)
        const bool in = row >= 2 * P && row < N - 2 * P;
        aq = in ? B.kA[q] : __ldg(B.Ab + (size_t)row * W + q);
      }
      fv = fma(aq, dv[q], fv);
    }
    return fv;
  };
  // one forward elimination step of row k; (MOD) ivk = cached 1/u_kk, un[] = u_{k,k+q}
  auto fwd = [&](auto fast, int row, double fv, double cc, double ivk, double* un) -> double {
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
  };
  // pv[m-1], pc[m-1]: pivot 1/u and c (MOD) / u (DER) of patch row r0 - m
  auto set_state = [&](const double* p, const double* pv, const double* pc, int r0) {
#pragma unroll
    for (int m = 0; m < P; m++) yw[m] = p[m];
    if (MOD) {
#pragma unroll
      for (int m = 0; m < P; m++) {
#pragma unroll
        for (int j = 0; j < P - 1; j++) uw[m][j] = p[P + m * (P - 1) + j];
        const int row = r0 - 1 - m;
        iw[m] = row >= lo ? pv[m] : 0.0;
        uw[m][P - 1] = row >= lo ? mod_entry(std::false_type{}, row, pc[m], 2 * P) : 0.0;
      }
    }
    if (DER) {
#pragma unroll
      for (int q = 0; q < P; q++) dv[q] = (r0 - P + q >= lo) ? pv[P - 1 - q] : 0.0;
    }
  };
  // chunks [cf0, cf1) are "fast": every row active, interior stencils / converged factors
  int cf0, cf1;
  {
    int a = lo, b = hi;
    if (MOD || DER) a = max(a, 2 * P), b = min(b, N - 2 * P);
    if (!MOD) a = max(a, hk), b = min(b, tk);
    cf0 = (a + CH - 1) / CH;
    cf1 = b / CH;
  }
  auto chunk_fast = [&](int c) { return c >= cf0 && c < cf1; };
  // (MASS / DER) chunks [cm0, cm1) have every row active: outside [cf0, cf1) they take the medium path
  const int cm0 = (lo + CH - 1) / CH, cm1 = hi / CH;
#ifndef ADI_ST_MED_DER
#define ADI_ST_MED_DER 0  // the derivative projection is traffic bound: the medium path only costs it registers
#endif
  auto chunk_med = [&](int c) { return (MODE == SW_MASS || (DER && ADI_ST_MED_DER)) && c >= cm0 && c < cm1; };
  // (DER) u at row r0+r of chunk slot sl; rows past the chunk from nx (next chunk) or hd (saved head)
  auto der_u = [&](const double* sl, const double* nxs, const double* hd, int r0, int r) -> double {
    if (r0 + r >= hi || r0 + r < lo) return 0.0;
    if (r < CH) return at(sl, r);
    return nxs ? at(nxs, r - CH) : hd[r - CH];
  };
  auto fwd_chunk = [&](auto fast, const double* sl, const double* nxs, const double* hd, int r0, double* y,
                       double* us, double* ivs) {
#pragma unroll
    for (int r = 0; r < CH; r++) {
      const int row = r0 + r;
      if (decltype(fast)::value || (row >= lo && row < hi)) {
        double un[P];
        double fv;
        if (DER) {
          dv[W - 1] = der_u(sl, nxs, hd, r0, r + P);
          fv = der_rhs(fast, row);
#pragma unroll
          for (int q = 0; q < W - 1; q++) dv[q] = dv[q + 1];
        } else {
          fv = at(sl, r);
        }
        const double ivk = MOD ? at(sl + 2 * ST_ARR, r) : 0.0;
        const double yy = fwd(fast, row, fv, MOD ? at(sl + ST_ARR, r) : 0.0, ivk, un);
        if (y) y[r] = yy;
        if (MOD && ivs) ivs[r] = ivk;
        if (MOD && us) {
#pragma unroll
          for (int q = 0; q < P - 1; q++) us[r * UW + q] = un[q];
        }
      }
    }
  };
  double xw[P];
  auto bwd_chunk = [&](auto fast, const double* sl, int r0, double* y, double* us, const double* ivs) {
#pragma unroll
    for (int r = CH - 1; r >= 0; r--) {
      const int row = r0 + r;
      if (decltype(fast)::value || (row >= lo && row < hi)) {
        double x = y[r];
        if (MOD) {
          const double cc = at(sl + ST_ARR, r);
          x = fma(-mod_entry(fast, row, cc, 2 * P), xw[P - 1], x);
#pragma unroll
          for (int q = P - 1; q >= 1; q--) x = fma(-us[r * UW + q - 1], xw[q - 1], x);
          x *= ivs[r];
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
  auto der_prime = [&](const double* sl, int r0) {
#pragma unroll
    for (int q = 0; q < P; q++) dv[P + q] = (r0 + q < hi && r0 + q >= lo) ? at(sl, q) : 0.0;
  };
  auto fwd_fast_cm = [&](const double* sl, const double* nxs, const double* hd, double* yv) {
#pragma unroll
    for (int q = 0; q < P; q++) yv[q] = yw[P - 1 - q];
    double uv[DER ? CH + 2 * P : 1];
    if (DER) {
#pragma unroll
      for (int q = 0; q < P; q++) uv[q] = dv[q];
#pragma unroll
      for (int r = 0; r < CH; r++) uv[P + r] = at(sl, r);
#pragma unroll
      for (int q = 0; q < P; q++) uv[P + CH + q] = nxs ? at(nxs, q) : hd[q];
    }
#pragma unroll
    for (int r = 0; r < CH; r++) {
      double y;
      if (DER) {
        y = 0.0;
#pragma unroll
        for (int q = 0; q < W; q++) y = fma(B.kA[q], uv[r + q], y);
      } else {
        y = at(sl, r);
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
    double xv[CH + P];
#pragma unroll
    for (int q = 0; q < P; q++) xv[CH + q] = xw[q];
#pragma unroll
    for (int r = CH - 1; r >= 0; r--) {
#ifdef ADI_ST_PRESCALE
      double x = yv[P + r] * kf[P];
#pragma unroll
      for (int q = P - 1; q >= 0; q--) x = fma(-ks[q], xv[r + 1 + q], x);
      xv[r] = x;
#else
      double x = yv[P + r];
#pragma unroll
      for (int q = P - 1; q >= 0; q--) x = fma(-kf[P + 1 + q], xv[r + 1 + q], x);
      xv[r] = x * kf[P];
#endif
    }
#pragma unroll
    for (int q = 0; q < P; q++) xw[q] = xv[q];
#pragma unroll
    for (int r = 0; r < CH; r++) y[r] = xv[r];
  };

  // ---------------- pass 1: forward elimination, checkpoints ----------------
  constexpr int AHEAD = DER ? 1 : 0;
  const int pre = min(RS, nc);
  constexpr int NA1 = DER ? 1 : NA;  // arrays loaded in pass 1 (DER: u only; base in pass 2)
  for (int c = 0; c < pre; c++) issue(c, c, NA1, pol_keep);
  // chunk c is waited for in order; DER also needs chunk c + 1 (AHEAD) before eliminating chunk c
  for (int c = 0, sc = 0; c < nc; c++, sc = next_slot(sc)) {
    const int sn = next_slot(sc);
    if (AHEAD) {
      if (c == 0) wait_slot(sc);
      if (c + 1 < nc) wait_slot(sn);
    } else {
      wait_slot(sc);
    }
    const double* sl = ring + sc * SLOT;
    const double* nxs = (DER && c + 1 < nc) ? ring + sn * SLOT : nullptr;
    const int r0 = c * CH;
    const bool fastc = chunk_fast(c);
    if (DER) der_prime(sl, r0);
    save_state(c);
    if (!MOD && fastc) {
      double yv[P + CH];
      fwd_fast_cm(sl, nxs, nullptr, yv);
    } else if (fastc) {
      fwd_chunk(std::true_type{}, sl, nxs, nullptr, r0, nullptr, nullptr, nullptr);
    } else if (chunk_med(c)) {
      fwd_chunk(st_med{}, sl, nxs, nullptr, r0, nullptr, nullptr, nullptr);
    } else {
      fwd_chunk(std::false_type{}, sl, nxs, nullptr, r0, nullptr, nullptr, nullptr);
    }
    __syncwarp();
    if (c + RS < nc) issue(c + RS, sc, NA1, pol_keep);
  }
  // ---------------- pass 2: recompute per chunk, back substitution ----------
  // MASS/MOD keep the last min(RS, nc) chunks of pass 1; DER reloads every chunk (u and base).
  const int keep_from = DER ? nc : nc - pre;  // chunks >= keep_from are still resident
  if (DER) {
    for (int c = nc - 1; c >= max(0, nc - (RS - 1)); c--) issue(c, c % RS, NA, pol_drop);
  }
#pragma unroll
  for (int q = 0; q < P; q++) xw[q] = 0.0;
  double hd[DER ? P : 1];
#pragma unroll
  for (int q = 0; q < (DER ? P : 1); q++) hd[q] = 0.0;
  double nxt[SWD];
  double pv[MOD || DER ? P : 1], pc[MOD ? P : 1];
  const double* gsrc0 = J.in;
  const double* gsrc1 = MOD ? J.c : nullptr;
  const double* gsrc2 = MOD ? J.iu : nullptr;
  // global offset of (lane's fiber, row): for the checkpoint-neighbour rows read with __ldg
  const int fib = f0 + lane;
  const bool fval = fib < nf;
  int64_t gbase, gstride;
  {
    const int fc = fval ? fib : nf - 1;
    if (axis == 2) gbase = fc + (int64_t)nx * ts, gstride = (int64_t)nx * ny;
    else if (axis == 1) gbase = fc + (int64_t)nx * ny * ts, gstride = nx;
    else gbase = (int64_t)nx * (fc + (int64_t)ny * ts), gstride = 1;
  }
  auto load_prev = [&](int c) {
#pragma unroll
    for (int q = 0; q < SWD; q++) nxt[q] = ck[((size_t)c * SWD + q) * 32];
    if (MOD || DER) {
      const int r0 = c * CH;
#pragma unroll
      for (int m = 0; m < P; m++) {
        const int row = max(r0 - 1 - m, lo);
        if (MOD) {
          pv[m] = __ldg(gsrc2 + gbase + (int64_t)row * gstride);
          pc[m] = __ldg(gsrc1 + gbase + (int64_t)row * gstride);
        } else {
          pv[m] = __ldg(gsrc0 + gbase + (int64_t)row * gstride);
        }
      }
    }
  };
  load_prev(nc - 1);
  for (int c = nc - 1, sc = (nc - 1) % RS; c >= 0; c--, sc = prev_slot(sc)) {
    if (c < keep_from) wait_slot(sc);
    double* sl = ring + sc * SLOT;
    const int r0 = c * CH;
    const bool fastc = chunk_fast(c), medc = !fastc && chunk_med(c);
    set_state(nxt, pv, pc, r0);
    if (c > 0) load_prev(c - 1);
    if (DER) der_prime(sl, r0);
    double y[CH];
    double us[CH * UW];
    double ivs[MOD ? CH : 1];
    if (!MOD && fastc) {
      double yv[P + CH];
      fwd_fast_cm(sl, nullptr, hd, yv);
      bwd_fast_cm(yv, y);
    } else if (fastc) {
      fwd_chunk(std::true_type{}, sl, nullptr, hd, r0, y, us, ivs);
      bwd_chunk(std::true_type{}, sl, r0, y, us, ivs);
    } else if (medc) {
      fwd_chunk(st_med{}, sl, nullptr, hd, r0, y, us, ivs);
      bwd_chunk(st_med{}, sl, r0, y, us, ivs);
    } else {
#pragma unroll
      for (int r = 0; r < CH; r++) y[r] = 0.0;
      fwd_chunk(std::false_type{}, sl, nullptr, hd, r0, y, us, ivs);
      bwd_chunk(std::false_type{}, sl, r0, y, us, ivs);
    }
    double* dst = sl;  // the solution overwrites the chunk's input rows (DER: its base rows)
    double y2[DER ? CH : 1];
    if (DER) {
#pragma unroll
      for (int q = 0; q < P; q++) hd[q] = (r0 + q < hi && r0 + q >= lo) ? at(sl, q) : 0.0;
      dst = sl + ST_ARR;
      // out = base + coef x; with out2: also out2 = out + coef x (the next substep's first
      // projection of the same derivative, SURVEY §8(a) note; same operations as two launches)
#pragma unroll
      for (int r = 0; r < CH; r++) {
        const double x = y[r];
        y[r] = fma(coef, x, at(sl + ST_ARR, r));
        y2[r] = fma(coef, x, y[r]);
      }
    }
    __syncwarp();  // every lane has read the slot
    if (fastc || medc) {  // every row active: plain stores at constant offsets
#pragma unroll
      for (int r = 0; r < CH; r++) atw(dst, r) = y[r];
      if (DER && J.out2) {
#pragma unroll
        for (int r = 0; r < CH; r++) atw(sl, r) = y2[r];
      }
    } else {
#pragma unroll
      for (int r = 0; r < CH; r++)
        if (r0 + r >= lo && r0 + r < hi) {
          atw(dst, r) = y[r];  // rows outside [lo, hi) keep their loaded value
          if (DER && J.out2) atw(sl, r) = y2[r];  // the chunk's u rows are consumed (hd saved)
        }
    }
    st_fence_async();  // every lane's shared writes -> visible to the async (TMA) proxy
    __syncwarp();
    if (lane == 0) {
      int x, yy, z;
      coords(c, x, yy, z);
      st_store(m_out, x, yy, z, dst, pol_drop);
      if (DER && J.out2) st_store(m_iu, x, yy, z, sl, pol_drop);
      st_commit();
      // refill the slot of chunk c+1 (stored one iteration ago) with chunk c+1-RS
      const int nxt_c = c + 1 - RS;
      if (nxt_c >= 0 && nxt_c < keep_from) {
        st_wait_read<1>();
        issue(nxt_c, next_slot(sc), NA, pol_drop);
      }
    }
    __syncwarp();
  }
  if (lane == 0) st_wait_read<0>();
  __syncwarp();
}

template <int P, int MODE>
__global__ void __launch_bounds__(32 * st_warps(MODE), 1)
sweep_tma_kernel(const __grid_constant__ SweepBatch B, const __grid_constant__ SweepTmaMaps MP) {
  constexpr int RS = st_rs(MODE), NA = st_na(MODE), WARPS = st_warps(MODE);
  constexpr int SLOT = NA * ST_ARR;
  constexpr int SWD = st_state_words(MODE, P);
  static_assert(RS >= 3, "ring too shallow");
  static_assert(ST_CH >= P, "derivative mode reads P rows of the next chunk");
  extern __shared__ __align__(1024) unsigned char st_raw[];
  // 1024-byte aligned base (the 128-byte swizzle atom); integer offset keeps the shared address space
  double* st_smem = reinterpret_cast<double*>(st_raw + ((1024u - (smem_u32(st_raw) & 1023u)) & 1023u));
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* ring = st_smem + (size_t)wib * RS * SLOT;
  uint64_t* bar = reinterpret_cast<uint64_t*>(st_smem + (size_t)WARPS * RS * SLOT) + wib * RS;
  if (lane == 0) {
    for (int s = 0; s < RS; s++) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();
  unsigned phase = 0;  // bit s: parity of the next completion of slot s
  const uint64_t pol_keep = st_policy_last<MODE>(), pol_drop = st_policy_first();
  const int gw = blockIdx.x * WARPS + wib;
  const int nw = gridDim.x * WARPS;
  double* ck = B.ckpt + (size_t)gw * B.nck * SWD * 32 + lane;
  const int total = B.ntiles;

  for (int t = gw; t < total; t += nw) {
    const int jb = (B.njobs > 1 && t >= B.job[1].tile0) + (B.njobs > 2 && t >= B.job[2].tile0);
    if (B.job[jb].axis == 0) st_tile<P, MODE, true>(B, MP, t, jb, ring, bar, phase, pol_keep, pol_drop, ck, lane);
    else st_tile<P, MODE, false>(B, MP, t, jb, ring, bar, phase, pol_keep, pol_drop, ck, lane);
  }
  if (lane == 0) st_wait_all();
}

}  // namespace adi
