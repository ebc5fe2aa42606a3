// degree.cu -- instantiates every kernel of one B-spline degree (compiled
// once per degree with -DADI_P=<p>, p = 1..5; see dispatch.h).
#include "dispatch.h"

#ifndef ADI_P
#error "compile with -DADI_P=<degree>"
#endif

namespace adi {

namespace {
template <int KIND, int S, int D>
struct RhsF {
  static void run(cudaStream_t st, dim3 g, const RhsArgs& a, const RhsMaps& m, bool tma) {
    constexpr size_t smem = rhs_smem_bytes<ADI_P, RhsProg<KIND, S, D>::NT>();
    if (tma) rhs_kernel<ADI_P, KIND, S, D, true><<<g, RX_THREADS, smem, st>>>(m, a);
    else rhs_kernel<ADI_P, KIND, S, D, false><<<g, RX_THREADS, smem, st>>>(m, a);
  }
};
template <int KIND, int S, int D>
cudaError_t rhs_attr_one() {
  constexpr size_t smem = rhs_smem_bytes<ADI_P, RhsProg<KIND, S, D>::NT>();
  cudaError_t e = cudaFuncSetAttribute(rhs_kernel<ADI_P, KIND, S, D, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(rhs_kernel<ADI_P, KIND, S, D, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}
}  // namespace

template <>
void Ops<ADI_P>::rhs(cudaStream_t st, dim3 grid, const RhsArgs& args, const RhsMaps& maps, bool tma, int kind, int s,
                     int d) {
  switch (kind * 6 + (s - 1) * 3 + d) {
    case 0: RhsF<0, 1, 0>::run(st, grid, args, maps, tma); break;
    case 1: RhsF<0, 1, 1>::run(st, grid, args, maps, tma); break;
    case 2: RhsF<0, 1, 2>::run(st, grid, args, maps, tma); break;
    case 3: RhsF<0, 2, 0>::run(st, grid, args, maps, tma); break;
    case 4: RhsF<0, 2, 1>::run(st, grid, args, maps, tma); break;
    case 5: RhsF<0, 2, 2>::run(st, grid, args, maps, tma); break;
    case 6: RhsF<1, 1, 0>::run(st, grid, args, maps, tma); break;
    case 7: RhsF<1, 1, 1>::run(st, grid, args, maps, tma); break;
    case 8: RhsF<1, 1, 2>::run(st, grid, args, maps, tma); break;
    case 9: RhsF<1, 2, 0>::run(st, grid, args, maps, tma); break;
    case 10: RhsF<1, 2, 1>::run(st, grid, args, maps, tma); break;
    default: RhsF<1, 2, 2>::run(st, grid, args, maps, tma); break;
  }
}

template <>
cudaError_t Ops<ADI_P>::rhs_attrs() {
  cudaError_t e = cudaSuccess;
  auto acc = [&](cudaError_t x) { if (x != cudaSuccess) e = x; };
  acc(rhs_attr_one<0, 1, 0>()); acc(rhs_attr_one<0, 1, 1>()); acc(rhs_attr_one<0, 1, 2>());
  acc(rhs_attr_one<0, 2, 0>()); acc(rhs_attr_one<0, 2, 1>()); acc(rhs_attr_one<0, 2, 2>());
  acc(rhs_attr_one<1, 1, 0>()); acc(rhs_attr_one<1, 1, 1>()); acc(rhs_attr_one<1, 1, 2>());
  acc(rhs_attr_one<1, 2, 0>()); acc(rhs_attr_one<1, 2, 1>()); acc(rhs_attr_one<1, 2, 2>());
  return e;
}

// sweep tiling: chunk of CH rows, ring of RS chunks per warp
constexpr int SW_CH = SW_CH_MASS;

template <>
void Ops<ADI_P>::sweep(cudaStream_t st, unsigned grid, const SweepBatch& B, bool modified) {
  const unsigned block = 32 * SW_WARPS;
  if (modified) {
    constexpr size_t smem = sw_smem_bytes<ADI_P, true, SW_CH_MOD, SW_RS_MOD>();
    sweep_kernel<ADI_P, true, SW_CH_MOD, SW_RS_MOD><<<grid, block, smem, st>>>(B);
  } else {
    constexpr size_t smem = sw_smem_bytes<ADI_P, false, SW_CH, SW_RS_MASS>();
    sweep_kernel<ADI_P, false, SW_CH, SW_RS_MASS><<<grid, block, smem, st>>>(B);
  }
}

template <>
cudaError_t Ops<ADI_P>::sweep_attrs(int occ[2]) {
  cudaError_t e;
  constexpr size_t s0 = sw_smem_bytes<ADI_P, false, SW_CH, SW_RS_MASS>();
  constexpr size_t s1 = sw_smem_bytes<ADI_P, true, SW_CH_MOD, SW_RS_MOD>();
  auto k0 = sweep_kernel<ADI_P, false, SW_CH, SW_RS_MASS>;
  auto k1 = sweep_kernel<ADI_P, true, SW_CH_MOD, SW_RS_MOD>;
  if ((e = cudaFuncSetAttribute(k0, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s0))) return e;
  if ((e = cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s1))) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[0], k0, 32 * SW_WARPS, s0))) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[1], k1, 32 * SW_WARPS, s1);
}

template <>
void Ops<ADI_P>::factor(cudaStream_t st, unsigned grid, const SweepBatch& B, double* iu, unsigned long long* bad,
                        double tol) {
  factor_kernel<ADI_P><<<grid, 128, 0, st>>>(B, iu, bad, tol);
}

}  // namespace adi
