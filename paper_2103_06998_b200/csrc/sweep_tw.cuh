// sweep_tw.cuh -- "twisted" (two-segment SPIKE) constant-matrix sweeps: the
// mass solves of a2/a6 (and a4/a8 on the general-mu path) and the derivative
// projection of the uniform-mu H update, same operations as sweep_kernel
// SW_MASS / SW_DER.
//
// Every fiber's active rows [lo, hi) are split at m1 = lo + ceil(L/2).  A warp
// owns 16 fibers; lanes 0-15 solve the top segment [lo, m1) top-down, lanes
// 16-31 the bottom segment [m1, hi) bottom-up, both with the same two-pass
// (checkpointed recompute) code: the active mass matrix is persymmetric
// (flip(M) = M: the B-spline basis is symmetric under x -> 1-x; enforced exactly
// at adi_create), so the bottom segment read in reverse order is the leading
// block of M and uses the same LU factor table.  After pass 1 each lane has the
// last p values of its segment solution y; the two lanes of a fiber exchange
// them (__shfl_xor 16) and solve the 2p x 2p interface system of the SPIKE
// decomposition (constant matrices, host-computed):
//   eta = K (y1b - Vb y2t),  xi = y2t - Wt eta,    K = (I - Vb Wt)^{-1}
// (eta: last p unknowns of the top segment, xi: first p of the bottom one).
// Pass 2 back-substitutes and corrects with the spike columns
//   top: x = y1 - V1 xi,  bottom: x = y2 - W2 eta   (V1 = A1^{-1} B, W2 = A2^{-1} C).
// Compared with one lane per fiber, each row is re-read from L2 after half the
// time and a fiber finishes in half the time: the in-flight working set is a
// quarter for the same bandwidth, which keeps the pass-2 re-reads in L2.
#pragma once
#include "sweep.cuh"

namespace adi {

template <int P, int MODE>
__global__ void __launch_bounds__(32 * SW_WARPS, MODE == SW_MASS ? ADI_SW_MINB_MASS : 1)
sweep_tw_kernel(const __grid_constant__ SweepBatch B) {
  constexpr bool DER = MODE == SW_DER;
  static_assert(MODE == SW_MASS || MODE == SW_DER, "twisted sweeps: constant matrices only");
  constexpr int CH = sw_ch(MODE), RS = sw_rs(MODE), NA = sw_na(MODE);
  constexpr int W = 2 * P + 1;
  constexpr int SLOT = NA * CH * 33;
  constexpr int SWD = sw_state_words_tw(MODE, P);
  static_assert(!DER || (RS >= 3 && CH >= P), "derivative mode needs the next chunk resident");
  constexpr int FPI = 32 / CH;
  extern __shared__ double sw_smem[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int fr = lane >> 4;  // 0: top segment, forward; 1: bottom segment, reversed
  double* ring = sw_smem + (size_t)wib * RS * SLOT;
  const int gw = blockIdx.x * SW_WARPS + wib;
  const int nw = gridDim.x * SW_WARPS;
  const int N = B.N;
  double* ck = B.ckpt + (size_t)gw * B.nck * SWD * 32 + lane;
  const int total = B.ntiles;

  for (int t = gw; t < total; t += nw) {
    const int jb = (B.njobs > 1 && t >= B.job[1].tile0) + (B.njobs > 2 && t >= B.job[2].tile0);
    const double* src[2];
    double* out;
    double coef;
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
      src[1] = J.base;
      out = J.out;
      coef = J.coef;
      axis = J.axis;
      lo = J.lo;
      hi = J.hi;
      var = J.var;
    }
    const int m1 = var ? B.m1[1] : B.m1[0];
    const int lenF = m1 - lo, lenR = hi - m1;                 // segment lengths (lenF >= lenR)
    const int seg = fr ? lenR : lenF;                          // this lane's segment length
    const int L = hi - lo;
    const int ldF = DER ? min(lenF + P, L) : lenF;             // frame rows loaded (DER: window over the split)
    const int ldR = DER ? min(lenR + P, L) : lenR;
    const int ld = fr ? ldR : ldF;
    const int nce = (lenF + CH - 1) / CH;                      // chunks eliminated
    const int ncl = (max(ldF, ldR) + CH - 1) / CH;             // chunks loaded
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

    auto issue = [&](int c, int na) {
      double* sl = ring + (c % RS) * SLOT;
      const int r0 = c * CH;
      if (axis != 0) {
        const int nr = min(CH, ld - r0);
        const double* p0 = src[0] + off0 + (int64_t)r0 * rstep;
        const double* p1 = NA > 1 ? src[1] + off0 + (int64_t)r0 * rstep : nullptr;
#pragma unroll
        for (int r = 0; r < CH; r++) {
          if (r < nr) {
            sw_cp_async8(sl + r * 33 + lane, p0);
            if (NA > 1 && na > 1) sw_cp_async8(sl + (CH + r) * 33 + lane, p1);
          }
          p0 += rstep;
          if (NA > 1) p1 += rstep;
        }
      } else {
        // column cc = (frame, fiber) of the slot; lane loads frame row r0 + xr of columns m*FPI + xc
#pragma unroll
        for (int m = 0; m < CH; m++) {
          const int cc = m * FPI + xc;
          const int cfr = cc >> 4;
          const int64_t fib = min(f0 + (cc & 15), NN - 1);
          const int rr = min(r0 + xr, (cfr ? ldR : ldF) - 1);
          const int64_t off = (int64_t)nx * fib + (cfr ? hi - 1 - rr : lo + rr);
          double* d = sl + xr * 33 + cc;
          sw_cp_async8(d, src[0] + off);
          if (NA > 1 && na > 1) sw_cp_async8(d + CH * 33, src[1] + off);
        }
      }
      sw_commit();
    };

    const double* fac = var ? B.fac[1] : B.fac[0];
    const double* sp = var ? B.sp[1] : B.sp[0];
    const int spl = var ? B.spl[1] : B.spl[0], sph = var ? B.sph[1] : B.sph[0];
    const int hk = var ? B.hk[1] : B.hk[0];
    const int tk = var ? B.tk[1] : B.tk[0];
    double kf[W];
#pragma unroll
    for (int q = 0; q < W; q++) kf[q] = var ? B.kfac[1][q] : B.kfac[0][q];
    const double dsign = fr ? -1.0 : 1.0;  // A is anti-persymmetric: reversed frame sees -A

    double yw[P];
    double dv[DER ? W : 1];
#pragma unroll
    for (int m = 0; m < P; m++) yw[m] = 0.0;
    if (DER) {
#pragma unroll
      for (int q = 0; q < W; q++) dv[q] = 0.0;
    }
    // factor entry q of frame row r (table row lo + r)
    auto fac_entry = [&](auto fast, int r, int q) -> double {
      if constexpr (decltype(fast)::value) {
        return kf[q];
      } else {
        const int row = lo + r;
        const bool in = row >= hk && row < tk;
        return in ? kf[q] : __ldg(fac + (size_t)row * W + q);
      }
    };
    auto der_rhs = [&](auto fast, int r) -> double {
      double fv = 0.0;
#pragma unroll
      for (int q = 0; q < W; q++) {
        double aq;
        if constexpr (decltype(fast)::value) {
          aq = B.kA[q];
        } else {
          const int row = lo + r;
          const bool in = row >= 2 * P && row < N - 2 * P;
          aq = in ? B.kA[q] : __ldg(B.Ab + (size_t)row * W + q);
        }
        fv = fma(aq, dv[q], fv);
      }
      return dsign * fv;
    };
    auto fwd = [&](auto fast, int r, double fv) -> double {
      double y = fv;
#pragma unroll
      for (int q = P - 1; q >= 0; q--) y = fma(-fac_entry(fast, r, q), yw[q], y);
#pragma unroll
      for (int m = P - 1; m > 0; m--) yw[m] = yw[m - 1];
      yw[0] = y;
      return y;
    };
    auto save_state = [&](int c) {
      double* p = ck + (size_t)c * SWD * 32;
#pragma unroll
      for (int m = 0; m < P; m++) p[m * 32] = yw[m];
      if (DER) {
#pragma unroll
        for (int q = 0; q < P; q++) p[(P + q) * 32] = dv[q];
      }
    };
    auto set_state = [&](const double* p) {
#pragma unroll
      for (int m = 0; m < P; m++) yw[m] = p[m];
      if (DER) {
#pragma unroll
        for (int q = 0; q < P; q++) dv[q] = p[P + q];
      }
    };
    // chunk uniformly inside both segments and the converged / Toeplitz rows?
    auto chunk_fast = [&](int r0) {
      return r0 + CH <= lenR && lo + r0 >= hk && lo + r0 + CH <= tk &&
             (!DER || (lo + r0 >= 2 * P && lo + r0 + CH <= N - 2 * P));
    };
    auto der_u = [&](const double* sl, const double* nx_, const double* hd, int r0, int r) -> double {
      if (r0 + r >= ld) return 0.0;
      if (r < CH) return sl[r * 33 + lane];
      return nx_ ? nx_[(r - CH) * 33 + lane] : hd[r - CH];
    };
    auto fwd_chunk = [&](auto fast, const double* sl, const double* nx_, const double* hd, int r0, double* y) {
#pragma unroll
      for (int r = 0; r < CH; r++) {
        if (decltype(fast)::value || r0 + r < seg) {
          double fv;
          if (DER) {
            dv[W - 1] = der_u(sl, nx_, hd, r0, r + P);
            fv = der_rhs(fast, r0 + r);
#pragma unroll
            for (int q = 0; q < W - 1; q++) dv[q] = dv[q + 1];
          } else {
            fv = sl[r * 33 + lane];
          }
          const double yy = fwd(fast, r0 + r, fv);
          if (y) y[r] = yy;
        }
      }
    };
    double xw[P];
    auto bwd_chunk = [&](auto fast, int r0, double* y) {
#pragma unroll
      for (int r = CH - 1; r >= 0; r--) {
        if (decltype(fast)::value || r0 + r < seg) {
          double x = y[r];
#pragma unroll
          for (int q = P - 1; q >= 0; q--) x = fma(-fac_entry(fast, r0 + r, P + 1 + q), xw[q], x);
          x *= fac_entry(fast, r0 + r, P);
#pragma unroll
          for (int q = P - 1; q > 0; q--) xw[q] = xw[q - 1];
          xw[0] = x;
          y[r] = x;
        }
      }
    };
    auto der_prime = [&](const double* sl, int r0) {
#pragma unroll
      for (int q = 0; q < P; q++) dv[P + q] = (r0 + q < ld) ? sl[q * 33 + lane] : 0.0;
    };

    // ---------------- pass 1: forward elimination of both segments ----------------
    constexpr int AHEAD = DER ? 1 : 0;
#pragma unroll
    for (int c = 0; c < RS - 1; c++) {
      if (c < ncl) issue(c, 1);
      else sw_commit();
    }
    for (int c = 0; c < ncl; c++) {
      sw_wait<RS - 2 - AHEAD>();
      __syncwarp();
      const double* sl = ring + (c % RS) * SLOT;
      const double* nx_ = (DER && c + 1 < ncl) ? ring + ((c + 1) % RS) * SLOT : nullptr;
      const int r0 = c * CH;
      if (c < nce) {
        if (DER) der_prime(sl, r0);
        save_state(c);
        if (chunk_fast(r0)) fwd_chunk(std::true_type{}, sl, nx_, nullptr, r0, nullptr);
        else fwd_chunk(std::false_type{}, sl, nx_, nullptr, r0, nullptr);
      }
      __syncwarp();
      if (c + RS - 1 < ncl) issue(c + RS - 1, 1);
      else sw_commit();
    }
    sw_wait<0>();
    __syncwarp();
    double hd[DER ? P : 1];  // (DER) u of the first P frame rows after the chunk being processed
    if (DER) {
      const double* sl = ring + (nce % RS) * SLOT;  // chunk nce (window rows across the split), if loaded
#pragma unroll
      for (int q = 0; q < P; q++) hd[q] = (nce < ncl && nce * CH + q < ld) ? sl[q * 33 + lane] : 0.0;
    }
    // ---------------- interface: last p values of each segment, 2p x 2p solve ----------
    double iface[P];
    {
      double yl[P];  // y at frame rows seg-1-t
#pragma unroll
      for (int q = 0; q < P; q++) xw[q] = 0.0;
#pragma unroll
      for (int tq = 0; tq < P; tq++) {
        const int r = seg - 1 - tq;
        double x = yw[tq];
#pragma unroll
        for (int q = P - 1; q >= 0; q--) x = fma(-fac_entry(std::false_type{}, r, P + 1 + q), xw[q], x);
        x *= fac_entry(std::false_type{}, r, P);
#pragma unroll
        for (int q = P - 1; q > 0; q--) xw[q] = xw[q - 1];
        xw[0] = x;
        yl[tq] = x;
      }
      double y1b[P], y2t[P];
#pragma unroll
      for (int q = 0; q < P; q++) {
        // top lane holds y1b[q] = yl[P-1-q] (patch row m1-P+q), bottom lane y2t[q] = yl[q] (patch row m1+q)
        const double mine = fr ? yl[q] : yl[P - 1 - q];
        const double other = __shfl_xor_sync(0xffffffffu, mine, 16);
        y1b[q] = fr ? other : mine;
        y2t[q] = fr ? mine : other;
      }
      double eta[P], xi[P];
#pragma unroll
      for (int a = 0; a < P; a++) {
        double s = y1b[a];
#pragma unroll
        for (int b = 0; b < P; b++) s = fma(-(var ? B.vb[1][a * P + b] : B.vb[0][a * P + b]), y2t[b], s);
        xi[a] = s;  // temporary: y1b - Vb y2t
      }
#pragma unroll
      for (int a = 0; a < P; a++) {
        double s = 0.0;
#pragma unroll
        for (int b = 0; b < P; b++) s = fma(var ? B.kk[1][a * P + b] : B.kk[0][a * P + b], xi[b], s);
        eta[a] = s;
      }
#pragma unroll
      for (int a = 0; a < P; a++) {
        double s = y2t[a];
#pragma unroll
        for (int b = 0; b < P; b++) s = fma(-(var ? B.wt[1][a * P + b] : B.wt[0][a * P + b]), eta[b], s);
        xi[a] = s;
      }
#pragma unroll
      for (int q = 0; q < P; q++) iface[q] = fr ? eta[q] : xi[q];
    }
    // ---------------- pass 2: recompute per chunk, back substitution, spike correction ----
    constexpr int KEEP = DER ? 0 : RS;
#pragma unroll
    for (int q = 0; q < P; q++) xw[q] = 0.0;
    double nxt[SWD];
#pragma unroll
    for (int q = 0; q < SWD; q++) nxt[q] = ck[((size_t)(nce - 1) * SWD + q) * 32];
    if (DER) {
#pragma unroll
      for (int c = 0; c < RS - 1; c++) {
        if (nce - 1 - c >= 0) issue(nce - 1 - c, 2);
        else sw_commit();
      }
    }
    for (int c = nce - 1; c >= 0; c--) {
      if (!DER && c < ncl - KEEP) sw_wait<RS - 2>();
      if (DER) sw_wait<RS - 2>();
      __syncwarp();
      double* sl = ring + (c % RS) * SLOT;
      const int r0 = c * CH;
      set_state(nxt);
      if (c > 0) {
#pragma unroll
        for (int q = 0; q < SWD; q++) nxt[q] = ck[((size_t)(c - 1) * SWD + q) * 32];
      }
      if (DER) der_prime(sl, r0);
      double y[CH];
      const bool fast = chunk_fast(r0);
      if (fast) {
        fwd_chunk(std::true_type{}, sl, nullptr, hd, r0, y);
        bwd_chunk(std::true_type{}, r0, y);
      } else {
#pragma unroll
        for (int r = 0; r < CH; r++) y[r] = 0.0;
        fwd_chunk(std::false_type{}, sl, nullptr, hd, r0, y);
        bwd_chunk(std::false_type{}, r0, y);
      }
      // spike correction: top x = y1 - V1 xi, bottom x = y2 - W2 eta (table by patch row).
      // The spikes decay geometrically away from the split; rows whose entries are all
      // below 1e-20 of the largest (outside [spl, sph)) skip the correction -- a change
      // four orders of magnitude below the rounding of the solve.
      const int pF = lo + r0, pR = hi - 1 - r0;  // patch row of frame row r0 in each frame
      const bool near = (pF + CH > spl && pF < sph) || (pR >= spl && pR - CH < sph - 1);
      if (near) {
#pragma unroll
        for (int r = 0; r < CH; r++) {
          if (r0 + r < seg) {
            const int prow = fr ? hi - 1 - (r0 + r) : lo + r0 + r;
            const double* s = sp + (size_t)prow * P;
            double x = y[r];
#pragma unroll
            for (int q = 0; q < P; q++) x = fma(-__ldg(s + q), iface[q], x);
            y[r] = x;
          }
        }
      }
      if (DER) {
#pragma unroll
        for (int r = 0; r < CH; r++) y[r] = fma(coef, y[r], sl[(CH + r) * 33 + lane]);
      }
      if (DER) {
#pragma unroll
        for (int q = 0; q < P; q++) hd[q] = (r0 + q < ld) ? sl[q * 33 + lane] : 0.0;
      }
      // store the chunk
      if (axis != 0) {
        double* po = out + off0 + (int64_t)r0 * rstep;
#pragma unroll
        for (int r = 0; r < CH; r++) {
          if (fval && r0 + r < seg) *po = y[r];
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
          if (fib < NN && rr < (cfr ? lenR : lenF))
            out[(int64_t)nx * fib + (cfr ? hi - 1 - rr : lo + rr)] = sl[xr * 33 + cc];
        }
      }
      __syncwarp();
      if (DER) {
        if (c - (RS - 1) >= 0) issue(c - (RS - 1), 2);
        else sw_commit();
      } else {
        if (c < nce - 1 && c + 1 - RS >= 0) issue(c + 1 - RS, 1);
        else sw_commit();
      }
    }
    sw_wait<0>();
    __syncwarp();
  }
}

}  // namespace adi
