// rhs.cuh -- right-hand sides of the E and H systems
// as sums of row-scaled Kronecker products (X (x) Y (x) Z) u (P:233-258,
// expanded per component in dupa1ab P:373-386), sum-factorised.
//
// One block owns a 32 x 16 (x, y) tile and streams a z-chunk of planes.  The
// input planes of every term arrive with a P-wide x/y halo in a 3-deep
// shared-memory ring (TMA cp.async.bulk.tensor + mbarrier when N is even so
// that the 8-byte row pitch is 16-byte aligned; cp.async otherwise).  Per
// plane: the x-pass (two outputs per thread, 128-bit shared loads) writes a
// double-buffered x-filtered plane; the y-pass (two rows per thread) feeds a
// (2P+1)-plane register window per term; the z-pass runs on that window.
// Interior rows use the Toeplitz stencils from the parameter bank; the 2P
// boundary rows at each end of an axis read the band tables.  Row scaling by
// a, b, c and the PEC restriction (D1) are applied at the output.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include <type_traits>

namespace adi {

// 1D operator codes of the band tables: tab[(op*N + row)*(2P+1) + q] holds the
// entry in column row-P+q (0 outside [0,N)).
enum Op { OP_M = 0, OP_A = 1, OP_B = 2, OP_S = 3, NUM_OPS = 4 };
enum Scale { SC_ONE = 0, SC_A = 1, SC_C = 2, SC_B = 3 };

// The right-hand sides as compile-time "programs" of row-scaled Kronecker terms.
// KIND 0 = E system of component D in substep S (a1/a5):
//   R_D = M^3 E_D + a [ d_{D+1} H_{D+2} - d_{D+2} H_{D+1} ] + c (A on D, B on sigma) E_sigma,
//   sigma = stiffened axis ((D+1)%3 in substep 1, (D+2)%3 in substep 2; K1/K2 of P:250-251);
//   (discrete1/discrete3 P:235/241; expanded in dupa1ab P:373-386).
// KIND 1 = H system of component D (a3/a7):
//   S=1: G_D = M^3 H_D - b d_{D+1} Eo_{D+2} + b d_{D+2} En_{D+1}   (discrete2 P:238, C1/C2 P:254-255 + D3)
//   S=2: G_D = M^3 H_D + b d_{D+2} Eo_{D+1} - b d_{D+1} En_{D+2}   (discrete4 P:244 with the sign D2)
// "d_a" is the advection matrix A (derivative on the trial function, D4) on axis a.
template <int KIND, int S, int D>
struct RhsProg {
  static constexpr int NT = KIND == 0 ? 4 : 3;
  static constexpr int SIG = S == 1 ? (D + 1) % 3 : (D + 2) % 3;
  __host__ __device__ static constexpr int op(int t, int ax) {
    return t == 0 ? OP_M
         : KIND == 0 ? (t == 1 ? (ax == (D + 1) % 3 ? OP_A : OP_M)
                      : t == 2 ? (ax == (D + 2) % 3 ? OP_A : OP_M)
                               : (ax == D ? OP_A : ax == SIG ? OP_B : OP_M))
         : S == 1 ? (t == 1 ? (ax == (D + 1) % 3 ? OP_A : OP_M) : (ax == (D + 2) % 3 ? OP_A : OP_M))
                  : (t == 1 ? (ax == (D + 2) % 3 ? OP_A : OP_M) : (ax == (D + 1) % 3 ? OP_A : OP_M));
  }
  __host__ __device__ static constexpr int scale(int t) {
    return t == 0 ? SC_ONE : KIND == 0 ? (t == 3 ? SC_C : SC_A) : SC_B;
  }
  __host__ __device__ static constexpr double sign(int t) {
    return t == 0 ? 1.0
         : KIND == 0 ? (t == 2 ? -1.0 : 1.0)
         : S == 1 ? (t == 1 ? -1.0 : 1.0) : (t == 1 ? 1.0 : -1.0);
  }
};

constexpr int RX_TX = 32;
constexpr int RX_TY = 16;
constexpr int RX_THREADS = 256;  // 32 x 8, two output rows each
constexpr int RX_MAXT = 4;
#ifndef ADI_RX_RING
#define ADI_RX_RING 2
#endif
constexpr int RX_RING = ADI_RX_RING;  // TMA ring slots (input planes in flight)
#ifndef ADI_RX_KCMAX
#define ADI_RX_KCMAX 128
#endif
constexpr int RX_KCMAX = ADI_RX_KCMAX;  // max z-chunk (rows of the per-block z-coefficient table)

struct RhsArgs {
  int N;                      // global extent (x, y: the arrays' extents; z: of the patch)
  int kchunk;                 // z-planes per block
  int nzin, zoff;             // input arrays hold nzin planes; output plane k <-> input plane k + zoff
  int kg0, nzout;             // output arrays hold global planes [kg0, kg0 + nzout)
  int use_sdirect;            // source amplitude given directly (sdirect) instead of signal[*step]
  double sdirect;
  int ntx, nty, fx, fy;       // tiles per axis; interior tiles are [1, fx] x [1, fy] (the FAST launch)
  const double* tab;          // band tables, 4 ops
  const double* u[RX_MAXT];   // term inputs
  const double* a;            // tau/(2 eps^)
  const double* b;            // tau/(2 mu^)
  const double* c;            // tau^2/(4 eps^ mu^)
  const double* load;         // source load vector of this component, or nullptr (D9)
  const double* signal;       // device signal array (nsig) or nullptr
  const int64_t* step;        // device step counter
  int64_t nsig;
  int lo[3], hi[3];           // active ranges of the output component (PEC, D1)
  double kint[3][11];         // interior (Toeplitz) rows of M, A, B (rows 2P..N-2P-1)
  double* out;
};

struct RhsMaps {
  CUtensorMap m[RX_MAXT];
};

template <int P>
struct RxGeom {
  static constexpr int W = 2 * P + 1;
  static constexpr int HX = RX_TX + 2 * P;
  static constexpr int HY = RX_TY + 2 * P;
  static constexpr int PLANE = HX * HY;
  static constexpr int PLANEP = (PLANE + 15) / 16 * 16;  // 128-byte aligned slices
};

template <int P, int NT>
__host__ __device__ constexpr size_t rhs_smem_bytes() {
  using G = RxGeom<P>;
  return sizeof(double) * ((size_t)RX_RING * NT * G::PLANEP + (size_t)NT * G::HY * RX_TX +
                           (size_t)3 * (RX_KCMAX + RX_TX + RX_TY) * (2 * P + 1)) +
         RX_RING * sizeof(uint64_t);
}

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void rx_cp_async8(double* smem_dst, const double* gsrc, bool valid) {
  const unsigned d = smem_u32(smem_dst);
  const int sz = valid ? 8 : 0;  // src-size 0 => zero fill
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(gsrc), "r"(sz) : "memory");
}
__device__ __forceinline__ void rx_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void rx_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }


// out[I] = sum_t sign_t * scale_t[I] * ((X_t (x) Y_t (x) Z_t) u_t)[I]  (- a s J),
// zero outside the active set.
// One (x,y) tile, z-chunk blockIdx.z.  FAST: the tile is interior in x and y (every
// output row Toeplitz): x/y coefficients come from the parameter bank; the general
// variant (rim tiles) reads them from per-block shared tables (rows of the band
// tables).  z coefficients always come from a per-block shared table (uniform
// broadcast reads).  bid: the tile's index among the interior / rim tiles.
template <int P, int KIND, int S, int D, bool TMA, bool FAST>
__device__ __forceinline__ void rhs_tile(const RhsMaps& maps, const RhsArgs& args, const int bid) {
  using Prog = RhsProg<KIND, S, D>;
  using G = RxGeom<P>;
  constexpr int NT = Prog::NT;
  constexpr int W = G::W, HX = G::HX, HY = G::HY, PLANE = G::PLANE, PLANEP = G::PLANEP;
  extern __shared__ __align__(1024) double rx_smem[];
  double* ring = rx_smem;                                           // [RING][NT][PLANEP]
  double* sx = rx_smem + RX_RING * NT * PLANEP;                     // [NT][HY][TX]
  double* czs = sx + NT * HY * RX_TX;                               // [3][KCMAX][W]
  double* cxs = czs + 3 * RX_KCMAX * W;                             // [3][TX][W]
  double* cys = cxs + 3 * RX_TX * W;                                // [3][TY][W]
  uint64_t* bar = reinterpret_cast<uint64_t*>(cys + 3 * RX_TY * W);  // [RING]

  const int N = args.N;
  const int tid = threadIdx.x;
  const int tx = tid & 31, ty = tid >> 5;  // y-pass / output: column tx, rows 2ty, 2ty+1
  // FAST: grid (fx, fy) over the interior tiles; general: the rim tiles, enumerated as
  // full rows {0} u [fy+1, nty) followed by the side tiles {0} u [fx+1, ntx) of rows [1, fy]
  int bx, by;
  if (FAST) {
    by = bid / args.fx;
    bx = bid - by * args.fx + 1;
    by += 1;
  } else {
    const int e = bid, nfull = (args.nty - args.fy) * args.ntx;
    if (e < nfull) {
      const int ri = e / args.ntx;
      bx = e - ri * args.ntx;
      by = ri == 0 ? 0 : args.fy + ri;
    } else {
      const int nside = args.ntx - args.fx, e2 = e - nfull, ri = e2 / nside, k = e2 - ri * nside;
      by = 1 + ri;
      bx = k == 0 ? 0 : args.fx + k;
    }
  }
  const int i0 = bx * RX_TX, j0 = by * RX_TY;
  // (general tiles) x / y rows of the tile all Toeplitz? then that pass uses the parameter-bank stencils
  const bool xint = FAST || (i0 >= 2 * P && i0 + RX_TX <= N - 2 * P);
  const bool yint = FAST || (j0 >= 2 * P && j0 + RX_TY <= N - 2 * P);
  // output planes (local) [k0, k1); input planes (local) kin = k + zoff + q - P
  const int k0 = blockIdx.z * args.kchunk;
  const int k1 = min(args.nzout, k0 + args.kchunk);
  const int zoff = args.zoff, kg0 = args.kg0;
  const int i = i0 + tx;
  const int jA = j0 + 2 * ty;
  const int64_t NN = (int64_t)N * N;
  const int kbeg = k0 + zoff - P, kend = k1 + zoff + P;  // input planes [kbeg, kend)

  // per-block coefficient tables: rows of the band tables (0 outside [0,N))
  for (int e = tid; e < 3 * (k1 - k0) * W; e += RX_THREADS) {
    const int o = e / ((k1 - k0) * W), r = e - o * (k1 - k0) * W;
    czs[o * RX_KCMAX * W + r] = args.tab[((int64_t)o * N + kg0 + k0) * W + r];
  }
  if (!FAST) {
    for (int e = tid; e < 3 * RX_TX * W; e += RX_THREADS) {
      const int o = e / (RX_TX * W), r = e - o * RX_TX * W, row = i0 + r / W;
      cxs[e] = row < N ? args.tab[((int64_t)o * N + i0) * W + r] : 0.0;
    }
    for (int e = tid; e < 3 * RX_TY * W; e += RX_THREADS) {
      const int o = e / (RX_TY * W), r = e - o * RX_TY * W, row = j0 + r / W;
      cys[e] = row < N ? args.tab[((int64_t)o * N + j0) * W + r] : 0.0;
    }
  }
  if (TMA && tid == 0) {
    for (int s = 0; s < RX_RING; s++) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  __syncthreads();
  // producer of input plane kin into its ring slot
  auto produce = [&](int kin) {
    const int st = (kin - kbeg) % RX_RING;
    double* slot = ring + st * NT * PLANEP;
    if (TMA) {
      if (tid == 0) {
        if (kin < kend) {
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          mbar_expect_tx(&bar[st], (unsigned)(NT * PLANE * sizeof(double)));
#pragma unroll
          for (int t = 0; t < NT; t++) tma_load_3d(slot + t * PLANEP, &maps.m[t], i0 - P, j0 - P, kin, &bar[st]);
        }
      }
    } else {
      if (kin < kend) {
        const bool kok = kin >= 0 && kin < args.nzin;
        const int64_t pb = kok ? NN * kin : 0;
        for (int e = tid; e < PLANE; e += RX_THREADS) {
          const int yy = e / HX, xx = e - yy * HX;
          const int gi = i0 - P + xx, gj = j0 - P + yy;
          const bool ok = kok && gi >= 0 && gi < N && gj >= 0 && gj < N;
          const int64_t off = ok ? pb + gi + (int64_t)N * gj : 0;
#pragma unroll
          for (int t = 0; t < NT; t++) rx_cp_async8(slot + t * PLANEP + e, args.u[t] + off, ok);
        }
      }
      rx_commit();  // (empty groups keep the wait arithmetic uniform)
    }
  };
  for (int q = 0; q < RX_RING; q++) produce(kbeg + q);

  double w[NT][2][W];
#pragma unroll
  for (int t = 0; t < NT; t++)
#pragma unroll
    for (int r = 0; r < 2; r++)
#pragma unroll
      for (int q = 0; q < W; q++) w[t][r][q] = 0.0;
  double sval = 0.0;
  if (KIND == 0 && args.load != nullptr) {
    if (args.use_sdirect) {
      sval = args.sdirect;
    } else if (args.signal != nullptr) {
      const int64_t s = *args.step;
      if (s < args.nsig) sval = args.signal[s];
    }
  }
  const bool act_ij = i < N && i >= args.lo[0] && i < args.hi[0];
  const int u = tid & 15;  // x-pass: outputs 2u, 2u+1 of rows (tid >> 4) + 16 m
  const int xrow0 = tid >> 4;

  for (int g0 = kbeg; g0 < kend; g0 += W) {
#pragma unroll
    for (int ph = 0; ph < W; ph++) {
      const int kin = g0 + ph;
      if (kin < kend) {
        const int it = kin - kbeg;
        const int st = it % RX_RING;
        const double* slot = ring + st * NT * PLANEP;
        double* sxb = sx;
        // prefetch the row scales of the output plane k = kin - P
        const int k = kin - P - zoff;  // output plane (local)
        const bool kout = k >= k0 && i < N;
        double sc[2][3];
#pragma unroll
        for (int r = 0; r < 2; r++) {
          const int j = jA + r;
          const bool ok = kout && j < N;
          const int64_t I = ok ? i + (int64_t)N * j + NN * k : 0;
          if (KIND == 0) {
            sc[r][0] = ok ? args.a[I] : 0.0;
            sc[r][1] = ok ? args.c[I] : 0.0;
            sc[r][2] = (ok && sval != 0.0) ? args.load[I] : 0.0;
          } else {
            sc[r][0] = ok ? args.b[I] : 0.0;
            sc[r][1] = sc[r][2] = 0.0;
          }
        }
        if (TMA) {
          mbar_wait(&bar[st], (unsigned)((it / RX_RING) & 1));
        } else {
          rx_wait<RX_RING - 1>();
          __syncthreads();
        }
        // ---- x-pass: rows yy of every term, two outputs (2u, 2u+1) per task
        auto xpass = [&](auto kx) {
#pragma unroll
          for (int t = 0; t < NT; t++) {
            const int xop = Prog::op(t, 0);
            // rows 0..15: one per thread; the 2P halo rows 16..HY-1 (32P tasks) go to a
            // different group of threads for every term, so the warps stay balanced at the barrier
            static_assert(HY - 16 <= 16, "x-pass task map assumes at most 16 extra rows");
#pragma unroll
            for (int m = 0; m < 2; m++) {
              const int ex = (tid - 64 * t + 4 * RX_THREADS) % RX_THREADS;  // extra-task index of this thread
              const int yy = m == 0 ? xrow0 : 16 + (ex >> 4);
              if (m == 0 || ex < (HY - 16) * 16) {
                const double2* rp = reinterpret_cast<const double2*>(slot + t * PLANEP + yy * HX + 2 * u);
                double v[2 * P + 2];
#pragma unroll
                for (int q = 0; q <= P; q++) {
                  const double2 d2 = rp[q];
                  v[2 * q] = d2.x;
                  v[2 * q + 1] = d2.y;
                }
                double o0 = 0.0, o1 = 0.0;
#pragma unroll
                for (int q = 0; q < W; q++) {
                  const double c0 = decltype(kx)::value ? args.kint[xop][q] : cxs[(xop * RX_TX + 2 * u) * W + q];
                  const double c1 = decltype(kx)::value ? args.kint[xop][q] : cxs[(xop * RX_TX + 2 * u + 1) * W + q];
                  o0 = fma(c0, v[q], o0);
                  o1 = fma(c1, v[q + 1], o1);
                }
                *reinterpret_cast<double2*>(sxb + (t * HY + yy) * RX_TX + 2 * u) = make_double2(o0, o1);
              }
            }
          }
        };
        if (FAST || xint) xpass(std::true_type{});
        else xpass(std::false_type{});
        __syncthreads();  // x-pass(kin) visible; ring slot st free
        produce(kin + RX_RING);
        // ---- y-pass: rows 2ty, 2ty+1 of column tx -> z-window slot ph
#pragma unroll
        for (int t = 0; t < NT; t++) {
          const int yop = Prog::op(t, 1);
          double col[W + 1];
#pragma unroll
          for (int q = 0; q <= W; q++) col[q] = sxb[(t * HY + 2 * ty + q) * RX_TX + tx];
          double vA = 0.0, vB = 0.0;
          if (FAST || yint) {
#pragma unroll
            for (int q = 0; q < W; q++) {
              vA = fma(args.kint[yop][q], col[q], vA);
              vB = fma(args.kint[yop][q], col[q + 1], vB);
            }
          } else {
#pragma unroll
            for (int q = 0; q < W; q++) {  // (warp-uniform rows: broadcast reads)
              vA = fma(cys[(yop * RX_TY + 2 * ty) * W + q], col[q], vA);
              vB = fma(cys[(yop * RX_TY + 2 * ty + 1) * W + q], col[q + 1], vB);
            }
          }
          w[t][0][ph] = vA;
          w[t][1][ph] = vB;
        }
        __syncthreads();  // sx consumed: the next plane's x-pass may overwrite it
        // ---- z-pass + row scaling for the output plane k = kin - P
        if (kout) {
          const bool ak = act_ij && kg0 + k >= args.lo[2] && kg0 + k < args.hi[2];
          const double* zrow = czs + (k - k0) * W;
#pragma unroll
          for (int r = 0; r < 2; r++) {
            const int j = jA + r;
            if (j < N) {
              double zs[3] = {0.0, 0.0, 0.0};  // scale groups: one, a|b, c
#pragma unroll
              for (int t = 0; t < NT; t++) {
                const int zop = Prog::op(t, 2);
                double z = 0.0;
#pragma unroll
                for (int q = 0; q < W; q++) z = fma(zrow[zop * RX_KCMAX * W + q], w[t][r][(ph + 1 + q) % W], z);
                const int grp = Prog::scale(t) == SC_ONE ? 0 : Prog::scale(t) == SC_C ? 2 : 1;
                zs[grp] = fma(Prog::sign(t), z, zs[grp]);
              }
              double val = 0.0;
              if (ak && j >= args.lo[1] && j < args.hi[1]) {
                if (KIND == 0) {
                  val = zs[0] + sc[r][0] * zs[1] + sc[r][1] * zs[2];
                  if (sval != 0.0) val -= sc[r][0] * sval * sc[r][2];
                } else {
                  val = zs[0] + sc[r][0] * zs[1];
                }
              }
              args.out[i + (int64_t)N * j + NN * k] = val;
            }
          }
        }
      }
    }
  }
  if (!TMA) rx_wait<0>();
}

// One launch covers every tile: in each z-chunk the rim tiles come first (they
// are slower: shared-table stencils, ragged tails), then the interior tiles, so
// the rim overlaps the interior work instead of forming a launch of its own.
template <int P, int KIND, int S, int D, bool TMA>
__global__ void __launch_bounds__(RX_THREADS, 2)
rhs_kernel(const __grid_constant__ RhsMaps maps, const __grid_constant__ RhsArgs args) {
  const int nrim = args.ntx * args.nty - args.fx * args.fy;
  const int b = blockIdx.x;
  if (b < nrim) rhs_tile<P, KIND, S, D, TMA, false>(maps, args, b);
  else rhs_tile<P, KIND, S, D, TMA, true>(maps, args, b - nrim);
}

}  // namespace adi
