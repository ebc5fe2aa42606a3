// degree.cu -- instantiates every kernel of one B-spline degree (compiled
// once per degree with -DADI_P=<p>, p = 1..5; see dispatch.h).
#include "dispatch.h"

#ifndef ADI_P
#error "compile with -DADI_P=<degree>"
#endif

namespace adi {

namespace {
template <int KIND, int S, int D>
void rhs_one(cudaStream_t st, dim3 grid, const RhsArgs& args) {
  constexpr size_t smem = rhs_smem_bytes<ADI_P, RhsProg<KIND, S, D>::NT>();
  rhs_kernel<ADI_P, KIND, S, D><<<grid, dim3(RHS_TX, RHS_TY), smem, st>>>(args);
}
template <int KIND, int S, int D>
void rhs_tma_one(cudaStream_t st, dim3 grid, const RhsArgs& args, const RhsTmaMaps& maps) {
  RhsTmaArgs ta;
  ta.base = args;
  for (int o = 0; o < 3; o++)
    for (int q = 0; q < 11; q++) ta.yint[o][q] = args.zint[o][q];
  constexpr size_t smem = rhs_tma_smem_bytes<ADI_P, RhsProg<KIND, S, D>::NT>();
  rhs_tma_kernel<ADI_P, KIND, S, D><<<grid, dim3(RT_TX, RT_THREADS / RT_TX), smem, st>>>(maps, ta);
}
template <int KIND, int S, int D>
cudaError_t rhs_attr_one() {
  constexpr size_t smem = rhs_smem_bytes<ADI_P, RhsProg<KIND, S, D>::NT>();
  return cudaFuncSetAttribute(rhs_kernel<ADI_P, KIND, S, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}
template <int KIND, int S, int D>
cudaError_t rhs_tma_attr_one() {
  constexpr size_t smem = rhs_tma_smem_bytes<ADI_P, RhsProg<KIND, S, D>::NT>();
  return cudaFuncSetAttribute(rhs_tma_kernel<ADI_P, KIND, S, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

// (kind, s, d) -> template arguments
template <template <int, int, int> class F, class... Args>
auto by_ksd(int kind, int s, int d, Args&&... a) {
  const int code = kind * 6 + (s - 1) * 3 + d;
  switch (code) {
    case 0: return F<0, 1, 0>::run(a...);
    case 1: return F<0, 1, 1>::run(a...);
    case 2: return F<0, 1, 2>::run(a...);
    case 3: return F<0, 2, 0>::run(a...);
    case 4: return F<0, 2, 1>::run(a...);
    case 5: return F<0, 2, 2>::run(a...);
    case 6: return F<1, 1, 0>::run(a...);
    case 7: return F<1, 1, 1>::run(a...);
    case 8: return F<1, 1, 2>::run(a...);
    case 9: return F<1, 2, 0>::run(a...);
    case 10: return F<1, 2, 1>::run(a...);
    default: return F<1, 2, 2>::run(a...);
  }
}
template <int K, int S, int D>
struct RhsF {
  static void run(cudaStream_t st, dim3 g, const RhsArgs& a) { rhs_one<K, S, D>(st, g, a); }
};
template <int K, int S, int D>
struct RhsTmaF {
  static void run(cudaStream_t st, dim3 g, const RhsArgs& a, const RhsTmaMaps& m) { rhs_tma_one<K, S, D>(st, g, a, m); }
};
}  // namespace

template <>
void Ops<ADI_P>::rhs(cudaStream_t st, dim3 grid, const RhsArgs& args, int kind, int s, int d) {
  by_ksd<RhsF>(kind, s, d, st, grid, args);
}

template <>
void Ops<ADI_P>::rhs_tma(cudaStream_t st, dim3 grid, const RhsArgs& args, const RhsTmaMaps& maps, int kind, int s,
                         int d) {
  by_ksd<RhsTmaF>(kind, s, d, st, grid, args, maps);
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

template <>
cudaError_t Ops<ADI_P>::rhs_tma_attrs() {
  cudaError_t e = cudaSuccess;
  auto acc = [&](cudaError_t x) { if (x != cudaSuccess) e = x; };
  acc(rhs_tma_attr_one<0, 1, 0>()); acc(rhs_tma_attr_one<0, 1, 1>()); acc(rhs_tma_attr_one<0, 1, 2>());
  acc(rhs_tma_attr_one<0, 2, 0>()); acc(rhs_tma_attr_one<0, 2, 1>()); acc(rhs_tma_attr_one<0, 2, 2>());
  acc(rhs_tma_attr_one<1, 1, 0>()); acc(rhs_tma_attr_one<1, 1, 1>()); acc(rhs_tma_attr_one<1, 1, 2>());
  acc(rhs_tma_attr_one<1, 2, 0>()); acc(rhs_tma_attr_one<1, 2, 1>()); acc(rhs_tma_attr_one<1, 2, 2>());
  return e;
}

template <>
void Ops<ADI_P>::sweep(cudaStream_t st, unsigned grid, size_t smem, const SweepArgs& A, int kind, int nck) {
  const unsigned block = 32 * SWEEP_WARPS;
  if (kind == SW_MOD) sweep_mod_kernel<ADI_P, 16><<<grid, block, smem, st>>>(A);
  else if (kind == SW_MASS_V1) sweep_mass_kernel<ADI_P, 32><<<grid, block, smem, st>>>(A);
  else sweep_mass2_kernel<ADI_P, 32><<<grid, block, smem, st>>>(A, nck);
}

template <>
cudaError_t Ops<ADI_P>::sweep_attrs(int mass_smem, int mass2_smem, int mod_smem) {
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(sweep_mass_kernel<ADI_P, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, mass_smem)))
    return e;
  if ((e = cudaFuncSetAttribute(sweep_mod_kernel<ADI_P, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, mod_smem)))
    return e;
  return cudaFuncSetAttribute(sweep_mass2_kernel<ADI_P, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, mass2_smem);
}

template <>
void Ops<ADI_P>::pivot_scan(cudaStream_t st, unsigned grid, const SweepArgs& A, unsigned long long* bad, double tol) {
  pivot_scan_kernel<ADI_P><<<grid, 256, 0, st>>>(A, bad, tol);
}

}  // namespace adi
