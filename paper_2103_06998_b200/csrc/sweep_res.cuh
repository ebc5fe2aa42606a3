// sweep_res.cuh -- fiber-resident two-segment (SPIKE) sweeps for the constant matrices:
// the mass solves of a2/a6 (and a4/a8 on the general-mu path) and the derivative projection
// of the uniform-mu H update (SURVEY §8(a) note), i.e. the SW_MASS / SW_DER modes of
// sweep.cuh, with the split, factors and interface algebra of sweep_tw.cuh.
//
// A warp owns a tile of 16 whole fibers.  The tile's N rows x 16 fibers stay in shared
// memory for the whole solve: TMA boxes bring the rows in (one mbarrier per 64-row slot),
// lanes 0-15 eliminate the top segment [lo, m1) top-down and lanes 16-31 the bottom segment
// [m1, hi) bottom-up (the active mass matrix is persymmetric, so the reversed bottom block
// uses the same LU table), writing y over f in place; after the 2p x 2p interface solve the
// back substitution writes x over y in place, and TMA stores send the tile back.  Every
// fiber row crosses HBM exactly once in each direction (plus, for the derivative projection,
// one read of `base`): no checkpoints, no recomputation, no second read of f.
//
// Shared layout of a tile (rows padded to 64-row slots):
//   y / z sweeps: [row][16 fibers]   (box {16 fibers, 64 rows}, fiber f of row r at r*16 + f)
//   x sweeps:     16-row boxes {16 rows, 16 fibers} with the 128-byte swizzle:
//                 (f, r) at (r/16)*256 + f*16 + ((((r%16)/2) ^ (f%8))*2) + r%2
// Derivative projection: out = base + coef * M^-1 (A u); u -> y -> x in place, then `base`
// streams through a 3-slot ring and out is formed element-parallel and stored from there.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "sweep_tma.cuh"

namespace adi {

constexpr int SR_SLOT = 64;                   // rows per slot / barrier
constexpr int SR_SLOTD = SR_SLOT * 16;        // doubles per slot (8 KB)
constexpr int SR_BRING = 3;                   // base ring slots (derivative projection)
constexpr int SR_MAXW = 8;                    // warps per block (cap)

__host__ __device__ inline int sr_nslot(int N) { return (N + SR_SLOT - 1) / SR_SLOT; }
// shared bytes per warp: tile + (DER) base ring + barriers
__host__ __device__ inline size_t sr_warp_bytes(int N, int mode) {
  const int ns = sr_nslot(N);
  return sizeof(double) * (size_t)(ns + (mode == SW_DER ? SR_BRING : 0)) * SR_SLOTD +
         sizeof(uint64_t) * (size_t)(ns + SR_BRING);
}

// tensor maps of a launch: per job the input (f | u), base (DER), output
struct SweepResMaps {
  CUtensorMap m[SW_MAXJOBS][3];
};

template <bool XAX>
__device__ __forceinline__ int sr_addr(int f, int r) {
  if constexpr (XAX) return ((r >> 4) << 8) + (f << 4) + (((((r & 15) >> 1) ^ (f & 7))) << 1) + (r & 1);
  else return (r << 4) + f;
}

// One tile (16 fibers of one job).  Lanes 0-15: top segment, lanes 16-31: bottom segment.
template <int P, int MODE, bool XAX>
__device__ __forceinline__ void sr_tile(const SweepBatch& B, const SweepResMaps& MP, const int t, const int jb,
                                        double* tileb, double* bring, uint64_t* bar, const unsigned par,
                                        unsigned& bphase, const uint64_t pol_in, const uint64_t pol_out,
                                        const int lane) {
  constexpr bool DER = MODE == SW_DER;
  constexpr int W = 2 * P + 1;
  constexpr int CH = 16;
  const SweepJob& J = B.job[jb];
  const int N = B.N;
  const int axis = J.axis, lo = J.lo, hi = J.hi, var = J.var;
  const int nx = J.dims[0], ny = J.dims[1];
  const int nf = axis == 0 ? ny : nx;
  const int ntf = (nf + 15) >> 4;
  const int tile = t - J.tile0;
  const int tf = tile % ntf, ts = tile / ntf;
  const int f0 = tf * 16;
  const int fr = lane >> 4, fib = lane & 15;
  const int ns = sr_nslot(N);
  const CUtensorMap* m_in = &MP.m[jb][0];
  const CUtensorMap* m_base = &MP.m[jb][1];
  const CUtensorMap* m_out = &MP.m[jb][2];
  uint64_t* bbar = bar + ns;  // base ring barriers (DER)

  // box coordinates of slot s (row 64 s): x sweeps issue 4 boxes of 16 rows
  auto box_xyz = [&](int row, int& x, int& y, int& z) {
    if (axis == 2) x = f0, y = ts, z = row;
    else if (axis == 1) x = f0, y = row, z = ts;
    else x = row, y = f0, z = ts;
  };
  auto load_slot = [&](const CUtensorMap* map, double* dst, uint64_t* b, int s) {
    mbar_expect_tx(b, (unsigned)(SR_SLOTD * sizeof(double)));
    int x, y, z;
    if (XAX) {
#pragma unroll
      for (int k = 0; k < 4; k++) {
        box_xyz(s * SR_SLOT + 16 * k, x, y, z);
        st_load(dst + k * 256, map, x, y, z, b, pol_in);
      }
    } else {
      box_xyz(s * SR_SLOT, x, y, z);
      st_load(dst, map, x, y, z, b, pol_in);
    }
  };
  auto store_slot = [&](const CUtensorMap* map, const double* src, int s) {
    int x, y, z;
    if (XAX) {
#pragma unroll
      for (int k = 0; k < 4; k++) {
        box_xyz(s * SR_SLOT + 16 * k, x, y, z);
        st_store(map, x, y, z, src + k * 256, pol_out);
      }
    } else {
      box_xyz(s * SR_SLOT, x, y, z);
      st_store(map, x, y, z, src, pol_out);
    }
  };

  // ---- loads: every slot of the tile, both ends first (the two segments start there) ----
  if (lane == 0) {
    for (int k = 0; k < ns; k++) {
      const int s = (k & 1) ? ns - 1 - (k >> 1) : (k >> 1);
      load_slot(m_in, tileb + (size_t)s * SR_SLOTD, &bar[s], s);
    }
  }

  const int m1 = var ? B.m1[1] : B.m1[0];
  const int lenF = m1 - lo, lenR = hi - m1;
  const int seg = fr ? lenR : lenF;
  const double* fac = var ? B.fac[1] : B.fac[0];
  const double* sp = var ? B.sp[1] : B.sp[0];
  const int spl = var ? B.spl[1] : B.spl[0], sph = var ? B.sph[1] : B.sph[0];
  const int hk = var ? B.hk[1] : B.hk[0];
  const int tk = var ? B.tk[1] : B.tk[0];
  double kf[W];
#pragma unroll
  for (int q = 0; q < W; q++) kf[q] = var ? B.kfac[1][q] : B.kfac[0][q];
  const double dsign = fr ? -1.0 : 1.0;  // A is anti-persymmetric: the reversed frame sees -A
  // frame row r <-> patch row prow(r); shared address of (fib, prow(r))
  auto prow = [&](int r) { return fr ? hi - 1 - r : lo + r; };
  auto at = [&](int r) -> double& { return tileb[sr_addr<XAX>(fib, prow(r))]; };
  // slots are waited in frame order: top lane upwards from slot 0, bottom lane downwards
  int sw_next = 0;  // slots [0, sw_next) of this lane's frame order complete
  auto need_row = [&](int r) {  // make frame row r (and the DER window) resident
    const int pr = prow(min(r, (DER ? hi - lo : seg) - 1));
    const int k = fr ? ns - 1 - pr / SR_SLOT : pr / SR_SLOT;  // frame-order index of its slot
    while (sw_next <= k) {
      const int s = fr ? ns - 1 - sw_next : sw_next;
      mbar_wait(&bar[s], par);
      sw_next++;
    }
  };
  auto fac_entry = [&](auto fast, int r, int q) -> double {
    if constexpr (decltype(fast)::value) {
      return kf[q];
    } else {
      const int row = lo + r;
      return (row >= hk && row < tk) ? kf[q] : __ldg(fac + (size_t)row * W + q);
    }
  };
  auto a_entry = [&](auto fast, int r, int q) -> double {
    if constexpr (decltype(fast)::value) {
      return B.kA[q];
    } else {
      const int row = lo + r;
      return (row >= 2 * P && row < N - 2 * P) ? B.kA[q] : __ldg(B.Ab + (size_t)row * W + q);
    }
  };
  auto chunk_fast = [&](int r0) {
    return r0 + CH <= lenR && lo + r0 >= hk && lo + r0 + CH <= tk &&
           (!DER || (lo + r0 >= 2 * P && lo + r0 + CH <= N - 2 * P));
  };

  // (DER) u across the split: the other segment overwrites it with y during the sweep
  double ux[DER ? P : 1];
  if (DER) {
    need_row(seg - 1 + P);
#pragma unroll
    for (int q = 0; q < P; q++) {
      const int r = seg + q;  // frame rows past the segment
      ux[q] = (r < hi - lo) ? at(r) : 0.0;
    }
    __syncwarp();
  }

  // ---------------- forward elimination (y over f / u in place) ----------------
  double yw[P];
#pragma unroll
  for (int m = 0; m < P; m++) yw[m] = 0.0;
  double dv[DER ? W : 1];  // (DER) u at frame rows r-P .. r+P
  if (DER) {
#pragma unroll
    for (int q = 0; q < P; q++) dv[q] = 0.0;
#pragma unroll
    for (int q = 0; q < P; q++) dv[P + q] = (q < seg) ? at(q) : ux[q - seg];
  }
  auto urow = [&](int r) -> double {  // (DER) u at frame row r >= current row
    if (r < seg) return at(r);
    const int k = r - seg;
    return (k < P && r < hi - lo) ? ux[k] : 0.0;
  };
  // one chunk of CH frame rows: all loads first, then the recurrence in registers, then the
  // stores (the shared loads never wait behind the chunk's own stores)
  auto fwd_chunk = [&](auto fast, int r0) {
    constexpr int NV = DER ? CH + P : CH;
    double v[NV];
#pragma unroll
    for (int r = 0; r < NV; r++) {
      const int rr = r0 + r;
      if (DER) v[r] = urow(rr);
      else v[r] = (decltype(fast)::value || rr < seg) ? at(rr) : 0.0;
    }
#pragma unroll
    for (int r = 0; r < CH; r++) {
      const int rr = r0 + r;
      if (decltype(fast)::value || rr < seg) {
        double f;
        if (DER) {
          dv[W - 1] = v[r + P];
          double s = 0.0;
#pragma unroll
          for (int q = 0; q < W; q++) s = fma(a_entry(fast, rr, q), dv[q], s);
          f = dsign * s;
#pragma unroll
          for (int q = 0; q < W - 1; q++) dv[q] = dv[q + 1];
        } else {
          f = v[r];
        }
        double y = f;
#pragma unroll
        for (int q = P - 1; q >= 0; q--) y = fma(-fac_entry(fast, rr, q), yw[q], y);
#pragma unroll
        for (int m = P - 1; m > 0; m--) yw[m] = yw[m - 1];
        yw[0] = y;
        v[r] = y;
      }
    }
#pragma unroll
    for (int r = 0; r < CH; r++) {
      const int rr = r0 + r;
      if (decltype(fast)::value || rr < seg) at(rr) = v[r];
    }
  };
  const int nce = (lenF + CH - 1) / CH;
  for (int c = 0; c < nce; c++) {
    const int r0 = c * CH;
    need_row(r0 + CH - 1 + (DER ? P : 0));
    if (chunk_fast(r0)) fwd_chunk(std::true_type{}, r0);
    else fwd_chunk(std::false_type{}, r0);
  }
  __syncwarp();

  // ---------------- interface: last p values of each segment, 2p x 2p solve ----------------
  double iface[P];
  {
    double xw[P], yl[P];
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
      xi[a] = s;
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

  // (DER) base ring: start streaming base while the back substitution runs
  if (DER && lane == 0) {
    for (int s = 0; s < min(SR_BRING, ns); s++) {
      // the ring slot's previous store must have read it (two tiles ago at the latest)
      load_slot(m_base, bring + (size_t)(s % SR_BRING) * SR_SLOTD, &bbar[s % SR_BRING], s);
    }
  }

  // ---------------- back substitution (x over y), spike correction ----------------
  double xw[P];
#pragma unroll
  for (int q = 0; q < P; q++) xw[q] = 0.0;
  auto bwd_chunk = [&](auto fast, int r0) {
    double xs[CH];
#pragma unroll
    for (int r = 0; r < CH; r++) {
      const int rr = r0 + r;
      xs[r] = (decltype(fast)::value || rr < seg) ? at(rr) : 0.0;
    }
#pragma unroll
    for (int r = CH - 1; r >= 0; r--) {
      const int rr = r0 + r;
      if (decltype(fast)::value || rr < seg) {
        double x = xs[r];
#pragma unroll
        for (int q = P - 1; q >= 0; q--) x = fma(-fac_entry(fast, rr, P + 1 + q), xw[q], x);
        x *= fac_entry(fast, rr, P);
#pragma unroll
        for (int q = P - 1; q > 0; q--) xw[q] = xw[q - 1];
        xw[0] = x;
        xs[r] = x;
      }
    }
    // spike correction (top x = y1 - V1 xi, bottom x = y2 - W2 eta); the spikes decay away
    // from the split and are dropped outside patch rows [spl, sph) (below 1e-20 of the largest)
    const int pF = lo + r0, pR = hi - 1 - r0;
    const bool near = (pF + CH > spl && pF < sph) || (pR >= spl && pR - CH < sph - 1);
    if (near) {
#pragma unroll
      for (int r = 0; r < CH; r++) {
        const int rr = r0 + r;
        if (rr < seg) {
          const double* sq = sp + (size_t)prow(rr) * P;
#pragma unroll
          for (int q = 0; q < P; q++) xs[r] = fma(-__ldg(sq + q), iface[q], xs[r]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < CH; r++) {
      const int rr = r0 + r;
      if (decltype(fast)::value || rr < seg) at(rr) = xs[r];
    }
  };
  for (int c = nce - 1; c >= 0; c--) {
    const int r0 = c * CH;
    if (chunk_fast(r0)) bwd_chunk(std::true_type{}, r0);
    else bwd_chunk(std::false_type{}, r0);
  }
  st_fence_async();  // every lane's shared writes -> visible to the async (TMA) proxy
  __syncwarp();

  if (!DER) {
    if (lane == 0) {
      for (int s = 0; s < ns; s++) store_slot(m_out, tileb + (size_t)s * SR_SLOTD, s);
      st_commit();
    }
  } else {
    // out = base + coef * x, element-parallel per slot through the base ring
    const double coef = J.coef;
    for (int s = 0; s < ns; s++) {
      const int b = s % SR_BRING;
      double* bs = bring + (size_t)b * SR_SLOTD;
      mbar_wait(&bbar[b], (bphase >> b) & 1u);
      bphase ^= 1u << b;
      const double* xs = tileb + (size_t)s * SR_SLOTD;
#pragma unroll 4
      for (int e = lane; e < SR_SLOTD; e += 32) bs[e] = fma(coef, xs[e], bs[e]);
      st_fence_async();
      __syncwarp();
      if (lane == 0) {
        store_slot(m_out, bs, s);
        st_commit();
        if (s + SR_BRING < ns) {
          st_wait_read<0>();  // this ring slot's store has read it
          load_slot(m_base, bs, &bbar[b], s + SR_BRING);
        }
      }
      __syncwarp();
    }
  }
  // the tile buffer (and ring) is reused by the next tile: wait until the stores have read it
  if (lane == 0) st_wait_read<0>();
  __syncwarp();
}

template <int P, int MODE>
__global__ void __launch_bounds__(32 * SR_MAXW, 1)
sweep_res_kernel(const __grid_constant__ SweepBatch B, const __grid_constant__ SweepResMaps MP) {
  extern __shared__ __align__(1024) unsigned char sr_raw[];
  double* base = reinterpret_cast<double*>(sr_raw + ((1024u - (smem_u32(sr_raw) & 1023u)) & 1023u));
  const int warps = blockDim.x >> 5;
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int N = B.N;
  const int ns = sr_nslot(N);
  const size_t per = (size_t)(ns + (MODE == SW_DER ? SR_BRING : 0)) * SR_SLOTD;
  double* tileb = base + (size_t)wib * per;
  double* bring = tileb + (size_t)ns * SR_SLOTD;
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + (size_t)warps * per) + (size_t)wib * (ns + SR_BRING);
  if (lane == 0) {
    for (int s = 0; s < ns + SR_BRING; s++) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();
  const uint64_t pol_in = st_policy_first(), pol_out = st_policy_first();
  const int gw = blockIdx.x * warps + wib;
  const int nw = gridDim.x * warps;
  unsigned par = 0, bphase = 0;
  for (int t = gw; t < B.ntiles; t += nw) {
    const int jb = (B.njobs > 1 && t >= B.job[1].tile0) + (B.njobs > 2 && t >= B.job[2].tile0);
    if (B.job[jb].axis == 0) sr_tile<P, MODE, true>(B, MP, t, jb, tileb, bring, bar, par, bphase, pol_in, pol_out, lane);
    else sr_tile<P, MODE, false>(B, MP, t, jb, tileb, bring, bar, par, bphase, pol_in, pol_out, lane);
    par ^= 1u;
  }
  if (lane == 0) st_wait_all();
}

}  // namespace adi
