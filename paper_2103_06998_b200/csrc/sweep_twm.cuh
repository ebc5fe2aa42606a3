// sweep_twm.cuh -- "twisted" row-modified sweep: the stiffened-axis solves of
// a2/a6, (M + diag(c) S) x = f per fiber (Appendix), the
// same system as sweep_kernel<SW_MOD>, split into two segments per fiber.
//
// Every fiber's active rows [lo, hi) are split at m1 = lo + ceil(L/2).  A warp
// owns 16 fibers; lanes 0-15 eliminate the top segment [lo, m1) top-down
// (the first m1 - lo rows of the no-pivot banded LU of the whole fiber, D12),
// lanes 16-31 the bottom segment [m1, hi) bottom-up: in the reversed frame
// (frame row r = patch row hi-1-r) the matrix J A J is again banded, its row r
// being row hi-1-r of A read backwards (entry q <-> 2P-q of the band tables),
// so the bottom lane runs the same recurrence on the mirrored stencil.  Both
// recurrences recompute the multipliers, the U rows and the pivots from c in
// registers (no pivot stream), exactly as sweep_kernel<SW_MOD> with
// ADI_SW_MOD_RECIP.
//
// After pass 1 each lane holds its segment's last P eliminated rows
//   x_k + sum_{j=1..P} (u_{k,k+j}/u_kk) x_{k+j} = y_k/u_kk        (own frame)
// which reach P rows into the other segment.  The two lanes of a fiber swap
// them (__shfl_xor 16) and both solve the same 2P x 2P system over the unknowns
// at patch rows [m1-P, m1+P) (Gaussian elimination in a fixed order: it is the
// continuation of the top-down LU through the bottom rows' reversed
// elimination, the twisted factorisation of the banded matrix).  Pass 2 then
// back-substitutes each segment from the other segment's P interface values,
// outward from the split (bottom lanes in the reversed frame).
//
// Why: with one lane per fiber, the pass-2 re-read of a row happens a whole
// fiber after its pass-1 load and the per-warp in-flight window is the whole
// fiber (f and c) -- at c5 the window of all resident warps overflows L2 and
// the re-reads go to DRAM (2.05x compulsory traffic, profiles/ncu_c5_r2.md).
// Two half-length segments per fiber halve that window at the same number of
// rows in flight.
#pragma once
#include "sweep.cuh"

// L2 priorities (ADI_TWM_HINT=1): checkpoints evict_last (rewritten every tile by the same warp:
// resident lines never reach DRAM), pass-2 loads and the solution stores evict_first (last use).
#ifndef ADI_TWM_HINT
#define ADI_TWM_HINT 0
#endif

namespace adi {

__device__ __forceinline__ uint64_t twm_policy(bool last) {
  uint64_t p;
  if (last) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  else asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ void twm_cp8(double* smem_dst, const double* gsrc, uint64_t pol) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;\n" ::"r"(d), "l"(gsrc), "l"(pol) : "memory");
}
__device__ __forceinline__ void twm_st(double* p, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;\n" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ double twm_ld(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;\n" : "=d"(v) : "l"(p), "l"(pol) : "memory");
  return v;
}

template <int P>
__global__ void __launch_bounds__(32 * SW_WARPS, ADI_SW_MINB_MOD) sweep_twm_kernel(const __grid_constant__ SweepBatch B) {
  static_assert(SW_MOD_RECIP, "the twisted row-modified sweep recomputes its pivots");
  constexpr int CH = sw_ch(SW_MOD), RS = sw_rs(SW_MOD), NA = 2;
  constexpr int W = 2 * P + 1;
  constexpr int SLOT = NA * CH * 33;
  constexpr int SWD = sw_state_words(SW_MOD, P);  // y (P), u_{k-m,k-m+j} j < P (P(P-1)), 1/u (P)
  constexpr int UW = P > 1 ? P - 1 : 1;
  constexpr int FPI = 32 / CH;
  static_assert(NA == sw_na(SW_MOD), "ring slot layout shared with sweep_kernel<SW_MOD>");
  extern __shared__ double sw_smem[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int fr = lane >> 4;  // 0: top segment, forward; 1: bottom segment, reversed frame
  double* ring = sw_smem + (size_t)wib * RS * SLOT;
  const int gw = blockIdx.x * SW_WARPS + wib;
  const int nw = gridDim.x * SW_WARPS;
  const int N = B.N;
  double* ck = B.ckpt + (size_t)gw * B.nck * SWD * 32 + lane;
  const int total = B.ntiles;
  const uint64_t pol_keep = twm_policy(true), pol_drop = twm_policy(false);
  // 8-byte copy into the ring: pass 1 plain, pass 2 (last use) evict_first
  auto cp8 = [&](double* d, const double* g, bool last_use) {
    if (ADI_TWM_HINT && last_use) twm_cp8(d, g, pol_drop);
    else sw_cp_async8(d, g);
  };
  auto ck_st = [&](double* p, double v) {
    if (ADI_TWM_HINT) twm_st(p, v, pol_keep);
    else *p = v;
  };
  auto ck_ld = [&](const double* p) -> double { return ADI_TWM_HINT ? twm_ld(p, pol_keep) : *p; };

  for (int t = gw; t < total; t += nw) {
    const int jb = (B.njobs > 1 && t >= B.job[1].tile0) + (B.njobs > 2 && t >= B.job[2].tile0);
    const double* src[2];
    double* out;
    int axis, lo, hi, var, nx, ny, tile;
    int64_t NN;
    {
      const SweepJob& J = jb == 0 ? B.job[0] : jb == 1 ? B.job[1] : B.job[2];
      tile = t - J.tile0;
      nx = J.dims[0];
      ny = J.dims[1];
      NN = J.axis == 0 ? (int64_t)J.dims[1] * J.dims[2] : J.axis == 1 ? (int64_t)J.dims[0] * J.dims[2]
                                                                       : (int64_t)J.dims[0] * J.dims[1];
      src[0] = J.in;
      src[1] = J.c;
      out = J.out;
      axis = J.axis;
      lo = J.lo;
      hi = J.hi;
      var = J.var;
    }
    const int L = hi - lo;
    const int m1 = lo + (L + 1) / 2;
    const int lenF = m1 - lo, lenR = hi - m1;  // segment lengths (lenF >= lenR >= P: host check)
    const int seg = fr ? lenR : lenF;
    const int nce = (lenF + CH - 1) / CH;
    const int64_t f0 = (int64_t)tile * 16;
    const int64_t f = f0 + (lane & 15);
    const bool fval = f < NN;
    const int64_t fc = fval ? f : NN - 1;
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
    // frame row r <-> patch row: top lo + r, bottom hi - 1 - r
    const int64_t rstep = fr ? -stride : stride;
    const int64_t off0 = base + (int64_t)(fr ? hi - 1 : lo) * stride;
    const int xr = lane % CH, xc = lane / CH;

    // chunk c of both frames -> ring slot c % RS (layout [array][row][33], column = lane)
    auto issue = [&](int c, bool p2) {
      double* sl = ring + (c % RS) * SLOT;
      const int r0 = c * CH;
      if (axis != 0) {
        const int nr = min(CH, seg - r0);
        const double* p0 = src[0] + off0 + (int64_t)r0 * rstep;
        const double* p1 = src[1] + off0 + (int64_t)r0 * rstep;
#pragma unroll
        for (int r = 0; r < CH; r++) {
          if (r < nr) {
            cp8(sl + r * 33 + lane, p0, p2);
            cp8(sl + (CH + r) * 33 + lane, p1, p2);
          }
          p0 += rstep;
          p1 += rstep;
        }
      } else {
        // column cc = (frame, fiber) of the slot; lane loads frame row r0 + xr of columns m*FPI + xc
#pragma unroll
        for (int m = 0; m < CH; m++) {
          const int cc = m * FPI + xc;
          const int cfr = cc >> 4;
          const int64_t fib = min(f0 + (cc & 15), NN - 1);
          const int rr = min(r0 + xr, (cfr ? lenR : lenF) - 1);
          const int64_t off = (int64_t)nx * fib + (cfr ? hi - 1 - rr : lo + rr);
          double* d = sl + xr * 33 + cc;
          cp8(d, src[0] + off, p2);
          cp8(d + CH * 33, src[1] + off, p2);
        }
      }
      sw_commit();
    };

    // the lane's stencil: entry q of frame row r is entry q (top) / 2P-q (bottom) of patch row g
    const double* Mb = var ? B.Mb[1] : B.Mb[0];
    const double* Sb = var ? B.Sb[1] : B.Sb[0];
    double km[W], ks[W];
#pragma unroll
    for (int q = 0; q < W; q++) {
      km[q] = fr ? B.kM[2 * P - q] : B.kM[q];
      ks[q] = fr ? B.kS[2 * P - q] : B.kS[q];
    }
    auto mod_entry = [&](auto fast, int r, double cc, int q) -> double {
      if constexpr (decltype(fast)::value) {
        return fma(cc, ks[q], km[q]);
      } else {
        const int g = fr ? hi - 1 - r : lo + r;
        const int qq = fr ? 2 * P - q : q;
        const bool in = g >= 2 * P && g < N - 2 * P;
        const double mq = in ? km[q] : __ldg(Mb + (size_t)g * W + qq);
        const double sq = in ? ks[q] : __ldg(Sb + (size_t)g * W + qq);
        return fma(cc, sq, mq);
      }
    };

    // recurrence state: yw[m-1] = y_{k-m}; uw[m-1][j-1] = u_{k-m,k-m+j}; iw[m-1] = 1/u_{k-m,k-m}
    double yw[P], uw[P][P], iw[P];
#pragma unroll
    for (int m = 0; m < P; m++) {
      yw[m] = 0.0;
      iw[m] = 0.0;
#pragma unroll
      for (int j = 0; j < P; j++) uw[m][j] = 0.0;
    }
    // one forward elimination step of frame row r: y_r, u_{r,r+q} (q = 1..P) in un[], 1/u_rr in ivo
    auto fwd = [&](auto fast, int r, double fv, double cc, double* un, double& ivo) -> double {
      double a[W];
#pragma unroll
      for (int q = 0; q < W; q++) a[q] = mod_entry(fast, r, cc, q);
      double l[P + 1];
#pragma unroll
      for (int m = P; m >= 1; m--) {
        double s = a[P - m];
#pragma unroll
        for (int mp = P; mp > m; mp--) s = fma(-l[mp], uw[mp - 1][mp - m - 1], s);
        l[m] = s * iw[m - 1];
      }
      double u0 = a[P];
#pragma unroll
      for (int m = 1; m <= P; m++) u0 = fma(-l[m], uw[m - 1][m - 1], u0);
      const double ivk = 1.0 / u0;
      ivo = ivk;
#pragma unroll
      for (int q = 1; q <= P; q++) {
        double s = a[P + q];
#pragma unroll
        for (int m = 1; m + q <= P; m++) s = fma(-l[m], uw[m - 1][m + q - 1], s);
        un[q - 1] = s;
      }
      double y = fv;
#pragma unroll
      for (int m = P; m >= 1; m--) y = fma(-l[m], yw[m - 1], y);
#pragma unroll
      for (int m = P - 1; m > 0; m--) {
        iw[m] = iw[m - 1];
        yw[m] = yw[m - 1];
#pragma unroll
        for (int j = 0; j < P; j++) uw[m][j] = uw[m - 1][j];
      }
      iw[0] = ivk;
      yw[0] = y;
#pragma unroll
      for (int j = 0; j < P; j++) uw[0][j] = un[j];
      return y;
    };
    auto save_state = [&](int c) {
      double* p = ck + (size_t)c * SWD * 32;
#pragma unroll
      for (int m = 0; m < P; m++) ck_st(p + m * 32, yw[m]);
#pragma unroll
      for (int m = 0; m < P; m++)
#pragma unroll
        for (int j = 0; j < P - 1; j++) ck_st(p + (P + m * (P - 1) + j) * 32, uw[m][j]);
#pragma unroll
      for (int m = 0; m < P; m++) ck_st(p + (P * P + m) * 32, iw[m]);
    };
    // pc[m-1]: c of frame row r0 - m
    auto set_state = [&](const double* p, const double* pc, int r0) {
#pragma unroll
      for (int m = 0; m < P; m++) {
        yw[m] = p[m];
#pragma unroll
        for (int j = 0; j < P - 1; j++) uw[m][j] = p[P + m * (P - 1) + j];
        const int r = r0 - 1 - m;
        iw[m] = r >= 0 ? p[P * P + m] : 0.0;
        uw[m][P - 1] = r >= 0 ? mod_entry(std::false_type{}, r, pc[m], 2 * P) : 0.0;
      }
    };
    // chunk inside both segments and Toeplitz (interior) in both frames?  (warp-uniform)
    auto chunk_fast = [&](int r0) {
      return r0 + CH <= lenR && lo + r0 >= 2 * P && lo + r0 + CH <= N - 2 * P && hi - r0 - CH >= 2 * P &&
             hi - 1 - r0 < N - 2 * P;
    };
    auto fwd_chunk = [&](auto fast, const double* sl, int r0, double* y, double* us, double* ivs) {
#pragma unroll
      for (int r = 0; r < CH; r++) {
        if (decltype(fast)::value || r0 + r < seg) {
          double un[P];
          double ivo;
          const double yy = fwd(fast, r0 + r, sl[r * 33 + lane], sl[(CH + r) * 33 + lane], un, ivo);
          if (y) y[r] = yy;
          if (ivs) ivs[r] = ivo;
          if (us) {
#pragma unroll
            for (int q = 0; q < P - 1; q++) us[r * UW + q] = un[q];
          }
        }
      }
    };
    double xw[P];  // x of the P frame rows after the row being back-substituted
    auto bwd_chunk = [&](auto fast, const double* sl, int r0, double* y, const double* us, const double* ivs) {
#pragma unroll
      for (int r = CH - 1; r >= 0; r--) {
        if (decltype(fast)::value || r0 + r < seg) {
          double x = y[r];
          const double cc = sl[(CH + r) * 33 + lane];
          x = fma(-mod_entry(fast, r0 + r, cc, 2 * P), xw[P - 1], x);
#pragma unroll
          for (int q = P - 1; q >= 1; q--) x = fma(-us[r * UW + q - 1], xw[q - 1], x);
          x *= ivs[r];
#pragma unroll
          for (int q = P - 1; q > 0; q--) xw[q] = xw[q - 1];
          xw[0] = x;
          y[r] = x;
        }
      }
    };

    // ---------------- pass 1: forward elimination of both segments, checkpoints ----------------
#pragma unroll
    for (int c = 0; c < RS - 1; c++) {
      if (c < nce) issue(c, false);
      else sw_commit();
    }
    for (int c = 0; c < nce; c++) {
      sw_wait<RS - 2>();
      __syncwarp();
      const double* sl = ring + (c % RS) * SLOT;
      const int r0 = c * CH;
      save_state(c);
      if (chunk_fast(r0)) fwd_chunk(std::true_type{}, sl, r0, nullptr, nullptr, nullptr);
      else fwd_chunk(std::false_type{}, sl, r0, nullptr, nullptr, nullptr);
      __syncwarp();
      if (c + RS - 1 < nce) issue(c + RS - 1, false);
      else sw_commit();
    }
    sw_wait<0>();
    __syncwarp();

    // ---------------- interface: 2P x 2P system over patch rows [m1-P, m1+P) ----------------
    // own last P rows, normalised: x_k + sum_j e[m][j] x_{k+j} = h[m]  (k = seg - 1 - m, own frame)
    double z[2 * P];
    {
      double eT[P][P], hT[P], eB[P][P], hB[P];
#pragma unroll
      for (int m = 0; m < P; m++) {
        const double hm = yw[m] * iw[m];
        const double ho = __shfl_xor_sync(0xffffffffu, hm, 16);
        hT[m] = fr ? ho : hm;
        hB[m] = fr ? hm : ho;
#pragma unroll
        for (int j = 0; j < P; j++) {
          const double em = uw[m][j] * iw[m];
          const double eo = __shfl_xor_sync(0xffffffffu, em, 16);
          eT[m][j] = fr ? eo : em;
          eB[m][j] = fr ? em : eo;
        }
      }
      // unknown a <-> patch row m1 - P + a.  Top row for k = m1-1-m (a = P-1-m): columns a+1+j.
      // Bottom row for patch row m1+m (a = P+m): columns a-1-j.
      double Z[2 * P][2 * P];
#pragma unroll
      for (int i = 0; i < 2 * P; i++)
#pragma unroll
        for (int j = 0; j < 2 * P; j++) Z[i][j] = i == j ? 1.0 : 0.0;
#pragma unroll
      for (int m = 0; m < P; m++) {
        const int a = P - 1 - m;
#pragma unroll
        for (int j = 0; j < P; j++)
          if (a + 1 + j < 2 * P) Z[a][a + 1 + j] = eT[m][j];
        z[a] = hT[m];
        const int b = P + m;
#pragma unroll
        for (int j = 0; j < P; j++)
          if (b - 1 - j >= 0) Z[b][b - 1 - j] = eB[m][j];
        z[b] = hB[m];
      }
      // Gaussian elimination in natural order (no pivoting; the top rows are the LU's own
      // rows, so this continues the top-down elimination through the bottom rows)
#pragma unroll
      for (int k = 0; k < 2 * P; k++) {
        const double ip = 1.0 / Z[k][k];
#pragma unroll
        for (int i = k + 1; i < 2 * P; i++) {
          const double l = Z[i][k] * ip;
#pragma unroll
          for (int j = k + 1; j < 2 * P; j++) Z[i][j] = fma(-l, Z[k][j], Z[i][j]);
          z[i] = fma(-l, z[k], z[i]);
        }
      }
#pragma unroll
      for (int k = 2 * P - 1; k >= 0; k--) {
        double s = z[k];
#pragma unroll
        for (int j = k + 1; j < 2 * P; j++) s = fma(-Z[k][j], z[j], s);
        z[k] = s / Z[k][k];
      }
    }
    // the other segment's P interface values, nearest first: top x_{m1+q}, bottom x_{m1-1-q}
#pragma unroll
    for (int q = 0; q < P; q++) xw[q] = fr ? z[P - 1 - q] : z[P + q];

    // ---------------- pass 2: recompute per chunk, back substitution outward ----------------
    constexpr int KEEP = RS;  // the last RS chunks of pass 1 are still in the ring
    double nxt[SWD], pc[P];
    auto load_prev = [&](int c) {
#pragma unroll
      for (int q = 0; q < SWD; q++) nxt[q] = ck_ld(ck + ((size_t)c * SWD + q) * 32);
      const int r0 = c * CH;
#pragma unroll
      for (int m = 0; m < P; m++) {
        const int r = max(r0 - 1 - m, 0);
        pc[m] = __ldg(src[1] + off0 + (int64_t)r * rstep);
      }
    };
    load_prev(nce - 1);
    for (int c = nce - 1; c >= 0; c--) {
      if (c < nce - KEEP) sw_wait<RS - 2>();
      __syncwarp();
      double* sl = ring + (c % RS) * SLOT;
      const int r0 = c * CH;
      set_state(nxt, pc, r0);
      if (c > 0) load_prev(c - 1);
      double y[CH];
      double us[CH * UW];
      double ivs[CH];
      if (chunk_fast(r0)) {
        fwd_chunk(std::true_type{}, sl, r0, y, us, ivs);
        bwd_chunk(std::true_type{}, sl, r0, y, us, ivs);
      } else {
#pragma unroll
        for (int r = 0; r < CH; r++) y[r] = 0.0, ivs[r] = 0.0;
        fwd_chunk(std::false_type{}, sl, r0, y, us, ivs);
        bwd_chunk(std::false_type{}, sl, r0, y, us, ivs);
      }
      // store the chunk
      if (axis != 0) {
        double* po = out + off0 + (int64_t)r0 * rstep;
#pragma unroll
        for (int r = 0; r < CH; r++) {
          if (fval && r0 + r < seg) {
            if (ADI_TWM_HINT) twm_st(po, y[r], pol_drop);
            else *po = y[r];
          }
          po += rstep;
        }
      } else {
        __syncwarp();
#pragma unroll
        for (int r = 0; r < CH; r++) sl[r * 33 + lane] = y[r];
        __syncwarp();
#pragma unroll
        for (int m = 0; m < CH; m++) {
          const int cc = m * FPI + xc;
          const int cfr = cc >> 4;
          const int64_t fib = f0 + (cc & 15);
          const int rr = r0 + xr;
          if (fib < NN && rr < (cfr ? lenR : lenF)) out[(int64_t)nx * fib + (cfr ? hi - 1 - rr : lo + rr)] = sl[xr * 33 + cc];
        }
      }
      __syncwarp();
      if (c < nce - 1 && c + 1 - RS >= 0) issue(c + 1 - RS, true);
      else sw_commit();
    }
    sw_wait<0>();
    __syncwarp();
  }
}

}  // namespace adi
