// rhs3.cuh -- the three right-hand sides of the E systems of one substep (SURVEY §8(a) a1 / a5,
// discrete1 / discrete3 P:235 / P:241, expanded per component in dupa1ab P:373-386) in ONE
// pass over the six fields:
//   R_D = M^3 E_D + a [ (A on D+1) H_{D+2} - (A on D+2) H_{D+1} ] + c (A on D, B on sigma) E_sigma
//         (- a s J_D, D9),   sigma = D+1 (substep 1) / D+2 (substep 2)   (K1 / K2)
// with the row factors a = tau/(2 eps^), c = tau^2/(4 eps^ mu^) of the output row (D5)
// and the PEC rows zeroed (D1).
//
// One block owns a 32 x 16 (x, y) tile and streams a z-chunk.  Every input plane of the six
// fields arrives once, with a P-wide x/y halo, by TMA into a 3-slot ring (one read of each
// field from HBM per substep instead of the 4 fields per component of rhs_kernel).  Per plane:
//   x-pass: each field's halo'd rows are read ONCE and every x-operator of that field
//           (1 or 2 of M, A, B; 10 distinct (field, operator) pairs) is applied from registers;
//   y-pass: two output rows per thread from each x-filtered column (12 products);
//   z-pass: scatter-accumulate into per-(component, scale group) accumulators of the 2P+1
//           output planes the input plane touches (9 groups: scale 1, a, c per component);
//           the output plane k = kin - P is then complete: R = acc_1 + a acc_a + c acc_c.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include <type_traits>

#include "rhs.cuh"

namespace adi {

// product t = 4 D + k of substep S (D = output component):
//   k = 0: E_D, M M M, scale 1;  k = 1: +H_{D+2}, A on axis D+1, scale a;
//   k = 2: -H_{D+1}, A on axis D+2, scale a;  k = 3: E_sigma, A on axis D, B on sigma, scale c.
// compile-time loop: f(integral_constant<int, B>), ..., f(integral_constant<int, E-1>)
template <int B, int E, class F>
__device__ __forceinline__ void rx3_static_for(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    rx3_static_for<B + 1, E>(f);
  }
}

template <int S>
struct Rhs3Prog {
  static constexpr int NP = 12;
  __host__ __device__ static constexpr int comp(int t) { return t / 4; }
  __host__ __device__ static constexpr int sigma(int D) { return S == 1 ? (D + 1) % 3 : (D + 2) % 3; }
  __host__ __device__ static constexpr int field(int t) {
    return t % 4 == 0 ? t / 4 : t % 4 == 1 ? 3 + (t / 4 + 2) % 3 : t % 4 == 2 ? 3 + (t / 4 + 1) % 3 : sigma(t / 4);
  }
  __host__ __device__ static constexpr int op(int t, int ax) {
    return t % 4 == 0 ? OP_M
         : t % 4 == 1 ? (ax == (t / 4 + 1) % 3 ? OP_A : OP_M)
         : t % 4 == 2 ? (ax == (t / 4 + 2) % 3 ? OP_A : OP_M)
                      : (ax == t / 4 ? OP_A : ax == sigma(t / 4) ? OP_B : OP_M);
  }
  __host__ __device__ static constexpr int group(int t) { return t % 4 == 0 ? 0 : t % 4 == 3 ? 2 : 1; }
  __host__ __device__ static constexpr double sign(int t) { return t % 4 == 2 ? -1.0 : 1.0; }
  __host__ __device__ static constexpr int gi(int t) { return comp(t) * 3 + group(t); }
  // distinct (field, x-operator) pairs, numbered by first appearance (loops only, no recursion:
  // every call site has constant arguments after unrolling and folds at compile time)
  __host__ __device__ static constexpr int xkey(int t) { return field(t) * 4 + op(t, 0); }
  __host__ __device__ static constexpr int first(int t) {
    for (int u = 0; u < t; u++)
      if (xkey(u) == xkey(t)) return u;
    return t;
  }
  __host__ __device__ static constexpr int xslot(int t) {
    const int f = first(t);
    int n = 0;
    for (int u = 0; u < f; u++)
      if (first(u) == u) n++;
    return n;
  }
  __host__ __device__ static constexpr int nx() {
    int n = 0;
    for (int u = 0; u < NP; u++)
      if (first(u) == u) n++;
    return n;
  }
  // x-slot -> its field / operator (the first product using it)
  __host__ __device__ static constexpr int xs_prod(int xs) {
    for (int t = 0; t < NP; t++)
      if (xslot(t) == xs) return t;
    return 0;
  }
  __host__ __device__ static constexpr int xs_field(int xs) { return field(xs_prod(xs)); }
  __host__ __device__ static constexpr int xs_op(int xs) { return op(xs_prod(xs), 0); }
};

struct Rhs3Args {
  int N, kchunk, nzin, zoff, kg0, nzout;
  int use_sdirect;
  double sdirect;
  int ntx, nty, fx, fy;
  const double* tab;       // band tables, 4 ops
  const double* a;         // tau/(2 eps^) (output layout)
  const double* c;         // tau^2/(4 eps^ mu^)
  const double* load[3];   // source load vectors (D9) or nullptr
  const double* signal;
  const int64_t* step;
  int64_t nsig;
  int lo[3][3], hi[3][3];  // [component][axis] active range (PEC, D1)
  double kint[3][11];      // interior Toeplitz rows of M, A, B
  double* out[3];
};
struct Rhs3Maps {
  CUtensorMap m[6];  // E1 E2 E3 H1 H2 H3, N x N x nzin
};

template <int P>
struct Rx3Geom {
  static constexpr int W = 2 * P + 1;
  static constexpr int HX = RX_TX + 2 * P;
  static constexpr int HY = RX_TY + 2 * P;
  static constexpr int PLANE = HX * HY;
  static constexpr int PLANEP = (PLANE + 15) / 16 * 16;
  static constexpr int NXS = 10;  // distinct (field, x-operator) pairs of either substep
};

template <int P>
__host__ __device__ constexpr size_t rhs3_smem_bytes_n(int nsx) {
  using G = Rx3Geom<P>;
  return sizeof(double) * ((size_t)RX_RING * 6 * G::PLANEP + (size_t)nsx * G::NXS * G::HY * RX_TX +
                           (size_t)3 * (RX_KCMAX + RX_TX + RX_TY) * (2 * P + 1)) +
         RX_RING * sizeof(uint64_t) + 1024;
}
// x-filtered buffers: two (the x-pass of plane k+1 overlaps the y/z-pass of plane k, one barrier
// per plane) when they fit the 227 KB of shared memory a block may use, else one
template <int P>
__host__ __device__ constexpr int rhs3_nsx() {
  return rhs3_smem_bytes_n<P>(2) <= 227u * 1024u ? 2 : 1;
}
template <int P>
__host__ __device__ constexpr size_t rhs3_smem_bytes() {
  return rhs3_smem_bytes_n<P>(rhs3_nsx<P>());
}

template <int P, int S, bool FAST>
__device__ __forceinline__ void rhs3_tile(const Rhs3Maps& maps, const Rhs3Args& args, const int bid, double* smem) {
  using Prog = Rhs3Prog<S>;
  using G = Rx3Geom<P>;
  constexpr int W = G::W, HX = G::HX, HY = G::HY, PLANE = G::PLANE, PLANEP = G::PLANEP;
  constexpr int NXS = Prog::nx();
  static_assert(NXS == G::NXS, "ten distinct (field, x-operator) pairs per substep");
  constexpr int NSX = rhs3_nsx<P>();
  double* ring = smem;                                              // [RING][6][PLANEP]
  double* sx0 = ring + RX_RING * 6 * PLANEP;                        // [NSX][NXS][HY][TX]
  double* czs = sx0 + NSX * NXS * HY * RX_TX;                       // [3][KCMAX][W]
  double* cxs = czs + 3 * RX_KCMAX * W;                             // [3][TX][W]
  double* cys = cxs + 3 * RX_TX * W;                                // [3][TY][W]
  uint64_t* bar = reinterpret_cast<uint64_t*>(cys + 3 * RX_TY * W);  // [RING]

  const int N = args.N;
  const int tid = threadIdx.x;
  const int tx = tid & 31, ty = tid >> 5;
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
  const bool xint = FAST || (i0 >= 2 * P && i0 + RX_TX <= N - 2 * P);
  const bool yint = FAST || (j0 >= 2 * P && j0 + RX_TY <= N - 2 * P);
  const int k0 = blockIdx.z * args.kchunk;
  const int k1 = min(args.nzout, k0 + args.kchunk);
  const int zoff = args.zoff, kg0 = args.kg0;
  const int i = i0 + tx;
  const int jA = j0 + 2 * ty;
  const int64_t NN = (int64_t)N * N;
  const int kbeg = k0 + zoff - P, kend = k1 + zoff + P;

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
  if (tid == 0) {
    for (int s = 0; s < RX_RING; s++) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  __syncthreads();
  auto produce = [&](int kin) {
    const int st = (kin - kbeg) % RX_RING;
    double* slot = ring + st * 6 * PLANEP;
    if (tid == 0 && kin < kend) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      mbar_expect_tx(&bar[st], (unsigned)(6 * PLANE * sizeof(double)));
#pragma unroll
      for (int f = 0; f < 6; f++) tma_load_3d(slot + f * PLANEP, &maps.m[f], i0 - P, j0 - P, kin, &bar[st]);
    }
  };
  for (int q = 0; q < RX_RING; q++) produce(kbeg + q);

  // accumulators of the 2P+1 pending output planes: acc[group][plane slot][row]
  double acc[9][W][2];
#pragma unroll
  for (int g = 0; g < 9; g++)
#pragma unroll
    for (int q = 0; q < W; q++) acc[g][q][0] = acc[g][q][1] = 0.0;
  double sval = 0.0;
  {
    bool any = false;
#pragma unroll
    for (int d = 0; d < 3; d++) any = any || args.load[d] != nullptr;
    if (any) {
      if (args.use_sdirect) {
        sval = args.sdirect;
      } else if (args.signal != nullptr) {
        const int64_t s = *args.step;
        if (s < args.nsig) sval = args.signal[s];
      }
    }
  }
  const int u = tid & 15;
  const int xrow0 = tid >> 4;
  const bool iin = i < N;
  // PEC activity (D1) of the thread's two output points, x / y part (the z part is per plane)
  bool actxy[3][2];
#pragma unroll
  for (int d = 0; d < 3; d++)
#pragma unroll
    for (int r = 0; r < 2; r++)
      actxy[d][r] = i >= args.lo[d][0] && i < args.hi[d][0] && jA + r >= args.lo[d][1] && jA + r < args.hi[d][1] &&
                    jA + r < N;

  // acc[g][jj][r]: output plane kin - P + jj of the current input plane kin (jj = 0: completes
  // now); after the output the window shifts by one plane (register moves, static indices)
  for (int kin = kbeg; kin < kend; kin++) {
    {
      {
        const int it = kin - kbeg;
        const int st = it % RX_RING;
        const double* slot = ring + st * 6 * PLANEP;
        // output plane completed by this input plane: k = kin - P (output-local)
        const int k = kin - P - zoff;
        const bool kout = k >= k0 && iin;
        double sc[2][2];
        double ld[3][2];
#pragma unroll
        for (int r = 0; r < 2; r++) {
          sc[r][0] = sc[r][1] = 0.0;
#pragma unroll
          for (int d = 0; d < 3; d++) ld[d][r] = 0.0;
          if (kout && jA + r < N) {
            const int64_t I = i + (int64_t)N * (jA + r) + NN * k;
            sc[r][0] = args.a[I];
            sc[r][1] = args.c[I];
            if (sval != 0.0) {
#pragma unroll
              for (int d = 0; d < 3; d++)
                if (args.load[d]) ld[d][r] = args.load[d][I];
            }
          }
        }
        double* sx = sx0 + (NSX == 2 ? (it & 1) * (NXS * HY * RX_TX) : 0);
        mbar_wait(&bar[st], (unsigned)((it / RX_RING) & 1));
        // ---- x-pass: each field's rows read once, every x-operator of the field applied
        auto xpass = [&](auto kx) {
          rx3_static_for<0, 6>([&](auto fc) {
            constexpr int f = decltype(fc)::value;
#pragma unroll
            for (int m = 0; m < 2; m++) {
              // the HY - 16 extra rows of field f go to whole warps (2 per field for P = 2), the warp
              // pair rotating with f: no divergent partial warps (measured 1 % faster than a 40-thread
              // rotation that splits warps)
              const int ex = (tid - 64 * f + 8 * RX_THREADS) % RX_THREADS;
              const int yy = m == 0 ? xrow0 : 16 + (ex >> 4);
              if (m == 0 || ex < (HY - 16) * 16) {
                const double2* rp = reinterpret_cast<const double2*>(slot + f * PLANEP + yy * HX + 2 * u);
                double v[2 * P + 2];
#pragma unroll
                for (int q = 0; q <= P; q++) {
                  const double2 d2 = rp[q];
                  v[2 * q] = d2.x;
                  v[2 * q + 1] = d2.y;
                }
                rx3_static_for<0, NXS>([&](auto xsc) {
                  constexpr int xs = decltype(xsc)::value;
                  if constexpr (Prog::xs_field(xs) == f) {
                    constexpr int xop = Prog::xs_op(xs);
                    double o0 = 0.0, o1 = 0.0;
#pragma unroll
                    for (int q = 0; q < W; q++) {
                      // interior A / B rows are antisymmetric stencils with an exact zero centre
                      // (adi_create makes the interior exactly Toeplitz): skip that tap
                      if (decltype(kx)::value && xop != OP_M && q == P) continue;
                      const double c0 = decltype(kx)::value ? args.kint[xop][q] : cxs[(xop * RX_TX + 2 * u) * W + q];
                      const double c1 =
                          decltype(kx)::value ? args.kint[xop][q] : cxs[(xop * RX_TX + 2 * u + 1) * W + q];
                      o0 = fma(c0, v[q], o0);
                      o1 = fma(c1, v[q + 1], o1);
                    }
                    *reinterpret_cast<double2*>(sx + (xs * HY + yy) * RX_TX + 2 * u) = make_double2(o0, o1);
                  }
                });
              }
            }
          });
        };
        if (FAST || xint) xpass(std::true_type{});
        else xpass(std::false_type{});
        __syncthreads();  // x-pass(kin) visible; ring slot st free
        produce(kin + RX_RING);
        // ---- y-pass (rows 2ty, 2ty+1 of column tx) and z scatter into the pending planes
        // contribution of input plane kin to output plane kin - P + jj has z coefficient
        // Z[k][2P - jj] (row k of the band table); interior planes: the Toeplitz row
        const int kout0 = kin - P - zoff;  // output-local plane of jj = 0
        const bool zint = kg0 + kout0 >= 2 * P && kg0 + kout0 + 2 * P < N - 2 * P;
        // z coefficients of this input plane for the three z-operators M, A, B: interior planes take
        // the Toeplitz rows from the parameter bank (compile-time slots; the exact-zero centre of A / B
        // skipped), boundary planes a per-plane register copy of the block's table
        auto yz = [&](auto zi) {
          constexpr bool ZI = decltype(zi)::value;
          double zc[3][W];
          if (!ZI) {
#pragma unroll
            for (int jj = 0; jj < W; jj++) {
              const int ko = min(max(kout0 + jj, k0), k1 - 1) - k0;
#pragma unroll
              for (int o = 0; o < 3; o++) zc[o][jj] = czs[(o * RX_KCMAX + ko) * W + 2 * P - jj];
            }
          }
          rx3_static_for<0, NXS>([&](auto xsc) {
            constexpr int xs = decltype(xsc)::value;
            double col[W + 1];
#pragma unroll
            for (int q = 0; q <= W; q++) col[q] = sx[(xs * HY + 2 * ty + q) * RX_TX + tx];
            rx3_static_for<0, Prog::NP>([&](auto tc) {
              constexpr int t = decltype(tc)::value;
              if constexpr (Prog::xslot(t) == xs) {
                constexpr int yop = Prog::op(t, 1), zop = Prog::op(t, 2), g = Prog::gi(t);
                double vA = 0.0, vB = 0.0;
                if (FAST || yint) {
#pragma unroll
                  for (int q = 0; q < W; q++) {
                    if (yop != OP_M && q == P) continue;  // zero centre of the interior A / B rows
                    vA = fma(args.kint[yop][q], col[q], vA);
                    vB = fma(args.kint[yop][q], col[q + 1], vB);
                  }
                } else {
#pragma unroll
                  for (int q = 0; q < W; q++) {
                    vA = fma(cys[(yop * RX_TY + 2 * ty) * W + q], col[q], vA);
                    vB = fma(cys[(yop * RX_TY + 2 * ty + 1) * W + q], col[q + 1], vB);
                  }
                }
                if constexpr (Prog::sign(t) < 0.0) vA = -vA, vB = -vB;
#pragma unroll
                for (int jj = 0; jj < W; jj++) {
                  if (ZI && zop != OP_M && jj == P) continue;
                  const double z = ZI ? args.kint[zop][2 * P - jj] : zc[zop][jj];
                  acc[g][jj][0] = fma(z, vA, acc[g][jj][0]);
                  acc[g][jj][1] = fma(z, vB, acc[g][jj][1]);
                }
              }
            });
          });
        };
        if (zint) yz(std::true_type{});
        else yz(std::false_type{});
        if (NSX == 1) __syncthreads();  // sx consumed (two buffers: the next x-pass writes the other)
        // ---- output plane k = kin - P is complete
        {
          const int slotk = 0;
          if (kout) {
#pragma unroll
            for (int d = 0; d < 3; d++) {
              const bool actz = kg0 + k >= args.lo[d][2] && kg0 + k < args.hi[d][2];
#pragma unroll
              for (int r = 0; r < 2; r++) {
                const int j = jA + r;
                if (j < N) {
                  double val = 0.0;
                  if (actz && actxy[d][r]) {
                    val = acc[3 * d][slotk][r] + sc[r][0] * acc[3 * d + 1][slotk][r] + sc[r][1] * acc[3 * d + 2][slotk][r];
                    if (sval != 0.0) val -= sc[r][0] * sval * ld[d][r];
                  }
                  args.out[d][i + (int64_t)N * j + NN * k] = val;
                }
              }
            }
          }
#pragma unroll
          for (int g = 0; g < 9; g++) {
#pragma unroll
            for (int q = 0; q < W - 1; q++) acc[g][q][0] = acc[g][q + 1][0], acc[g][q][1] = acc[g][q + 1][1];
            acc[g][W - 1][0] = acc[g][W - 1][1] = 0.0;
          }
        }
      }
    }
  }
}

template <int P, int S>
__global__ void __launch_bounds__(RX_THREADS, 1)
rhs3_kernel(const __grid_constant__ Rhs3Maps maps, const __grid_constant__ Rhs3Args args) {
  extern __shared__ __align__(1024) unsigned char rx3_raw[];
  double* smem = reinterpret_cast<double*>(rx3_raw + ((1024u - (smem_u32(rx3_raw) & 1023u)) & 1023u));
  const int nrim = args.ntx * args.nty - args.fx * args.fy;
  const int b = blockIdx.x;
  if (b < nrim) rhs3_tile<P, S, false>(maps, args, b, smem);
  else rhs3_tile<P, S, true>(maps, args, b - nrim, smem);
}

}  // namespace adi
