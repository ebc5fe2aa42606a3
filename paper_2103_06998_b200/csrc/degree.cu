// degree.cu -- instantiates every kernel of one B-spline degree (compiled
// once per degree with -DADI_P=<p>, p = 1..5; see dispatch.h).
#include "dispatch.h"

#ifndef ADI_P
#error "compile with -DADI_P=<degree>"
#endif

namespace adi {

#ifdef ADI_STUB
// Tuning builds (tools/build_variant.py --degrees): this degree is not compiled; every entry
// point reports cudaErrorNotSupported (adi_create then fails for this p).
template <>
void Ops<ADI_P>::rhs(cudaStream_t, dim3, const RhsArgs&, const RhsMaps&, bool, int, int, int) {}
template <>
cudaError_t Ops<ADI_P>::rhs_attrs() { return cudaErrorNotSupported; }
template <>
void Ops<ADI_P>::rhs3(cudaStream_t, dim3, const Rhs3Args&, const Rhs3Maps&, int) {}
template <>
cudaError_t Ops<ADI_P>::rhs3_attrs() { return cudaErrorNotSupported; }
template <>
void Ops<ADI_P>::sweep(cudaStream_t, unsigned, const SweepBatch&, int, bool) {}
template <>
cudaError_t Ops<ADI_P>::sweep_attrs(int*, int*) { return cudaErrorNotSupported; }
template <>
void Ops<ADI_P>::sweep_tma(cudaStream_t, unsigned, const SweepBatch&, const SweepTmaMaps&, int) {}
template <>
cudaError_t Ops<ADI_P>::sweep_tma_attrs(int*) { return cudaErrorNotSupported; }
template <>
void Ops<ADI_P>::factor(cudaStream_t, unsigned, const SweepBatch&, double*, unsigned long long*, double) {}
template <>
void Ops<ADI_P>::sweep_res(cudaStream_t, unsigned, unsigned, size_t, const SweepBatch&, const SweepResMaps&, int) {}
template <>
cudaError_t Ops<ADI_P>::sweep_res_attrs() { return cudaErrorNotSupported; }
template <>
void Ops<ADI_P>::spike(cudaStream_t, const SpikeBatch&, int) {}
template <>
void Ops<ADI_P>::spike_mod(cudaStream_t, const SpikeModArgs&, int) {}
#else

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
  const cudaFuncAttribute A = cudaFuncAttributeMaxDynamicSharedMemorySize;
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(rhs_kernel<ADI_P, KIND, S, D, true>, A, (int)smem))) return e;
  return cudaFuncSetAttribute(rhs_kernel<ADI_P, KIND, S, D, false>, A, (int)smem);
}
}  // namespace

template <>
void Ops<ADI_P>::rhs(cudaStream_t st, dim3 grid, const RhsArgs& args, const RhsMaps& maps, bool tma,
                     int kind, int s, int d) {
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

template <>
void Ops<ADI_P>::rhs3(cudaStream_t st, dim3 grid, const Rhs3Args& args, const Rhs3Maps& maps, int s) {
#if ADI_P <= 3
  constexpr size_t smem = rhs3_smem_bytes<ADI_P>();
  if (s == 1) rhs3_kernel<ADI_P, 1><<<grid, RX_THREADS, smem, st>>>(maps, args);
  else rhs3_kernel<ADI_P, 2><<<grid, RX_THREADS, smem, st>>>(maps, args);
#endif
}

template <>
cudaError_t Ops<ADI_P>::rhs3_attrs() {
#if ADI_P <= 3
  constexpr size_t smem = rhs3_smem_bytes<ADI_P>();
  const cudaFuncAttribute A = cudaFuncAttributeMaxDynamicSharedMemorySize;
  cudaError_t e = cudaFuncSetAttribute(rhs3_kernel<ADI_P, 1>, A, (int)smem);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(rhs3_kernel<ADI_P, 2>, A, (int)smem);
#else
  return cudaErrorNotSupported;  // degrees 4, 5: the per-component rhs_kernel
#endif
}

template <>
void Ops<ADI_P>::sweep(cudaStream_t st, unsigned grid, const SweepBatch& B, int mode, bool twisted) {
  const unsigned block = 32 * SW_WARPS;
  if (twisted && mode == SW_MOD) sweep_twm_kernel<ADI_P><<<grid, block, sw_smem_bytes<SW_MOD>(), st>>>(B);
  else if (twisted && mode == SW_DER) sweep_tw_kernel<ADI_P, SW_DER><<<grid, block, sw_smem_bytes<SW_DER>(), st>>>(B);
  else if (twisted) sweep_tw_kernel<ADI_P, SW_MASS><<<grid, block, sw_smem_bytes<SW_MASS>(), st>>>(B);
  else if (mode == SW_MOD) sweep_kernel<ADI_P, SW_MOD><<<grid, block, sw_smem_bytes<SW_MOD>(), st>>>(B);
  else if (mode == SW_DER) sweep_kernel<ADI_P, SW_DER><<<grid, block, sw_smem_bytes<SW_DER>(), st>>>(B);
  else sweep_kernel<ADI_P, SW_MASS><<<grid, block, sw_smem_bytes<SW_MASS>(), st>>>(B);
}

namespace {
template <class K>
cudaError_t attr_occ(K kernel, size_t smem, int* occ) {
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, kernel, 32 * SW_WARPS, smem);
}
}  // namespace

template <>
cudaError_t Ops<ADI_P>::sweep_attrs(int occ[3], int occ_tw[3]) {
  cudaError_t e;
  if ((e = attr_occ(sweep_kernel<ADI_P, SW_MASS>, sw_smem_bytes<SW_MASS>(), &occ[SW_MASS]))) return e;
  if ((e = attr_occ(sweep_kernel<ADI_P, SW_MOD>, sw_smem_bytes<SW_MOD>(), &occ[SW_MOD]))) return e;
  if ((e = attr_occ(sweep_kernel<ADI_P, SW_DER>, sw_smem_bytes<SW_DER>(), &occ[SW_DER]))) return e;
  if ((e = attr_occ(sweep_tw_kernel<ADI_P, SW_MASS>, sw_smem_bytes<SW_MASS>(), &occ_tw[SW_MASS]))) return e;
  if ((e = attr_occ(sweep_twm_kernel<ADI_P>, sw_smem_bytes<SW_MOD>(), &occ_tw[SW_MOD]))) return e;
  return attr_occ(sweep_tw_kernel<ADI_P, SW_DER>, sw_smem_bytes<SW_DER>(), &occ_tw[SW_DER]);
}

template <>
void Ops<ADI_P>::sweep_tma(cudaStream_t st, unsigned grid, const SweepBatch& B, const SweepTmaMaps& maps, int mode) {
  if (mode == SW_MOD)
    sweep_tma_kernel<ADI_P, SW_MOD><<<grid, 32 * st_warps(SW_MOD), st_smem_bytes<SW_MOD>(), st>>>(B, maps);
  else if (mode == SW_DER)
    sweep_tma_kernel<ADI_P, SW_DER><<<grid, 32 * st_warps(SW_DER), st_smem_bytes<SW_DER>(), st>>>(B, maps);
  else
    sweep_tma_kernel<ADI_P, SW_MASS><<<grid, 32 * st_warps(SW_MASS), st_smem_bytes<SW_MASS>(), st>>>(B, maps);
}

namespace {
template <int MODE>
cudaError_t st_attr(int* occ) {
  auto k = sweep_tma_kernel<ADI_P, MODE>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)st_smem_bytes<MODE>());
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, k, 32 * st_warps(MODE), st_smem_bytes<MODE>());
}
}  // namespace

template <>
cudaError_t Ops<ADI_P>::sweep_tma_attrs(int occ[3]) {
  cudaError_t e;
  if ((e = st_attr<SW_MASS>(&occ[SW_MASS]))) return e;
  if ((e = st_attr<SW_MOD>(&occ[SW_MOD]))) return e;
  return st_attr<SW_DER>(&occ[SW_DER]);
}

template <>
void Ops<ADI_P>::sweep_res(cudaStream_t st, unsigned grid, unsigned warps, size_t smem, const SweepBatch& B,
                           const SweepResMaps& maps, int mode) {
  if (mode == SW_DER) sweep_res_kernel<ADI_P, SW_DER><<<grid, 32 * warps, smem, st>>>(B, maps);
  else sweep_res_kernel<ADI_P, SW_MASS><<<grid, 32 * warps, smem, st>>>(B, maps);
}

template <>
cudaError_t Ops<ADI_P>::sweep_res_attrs() {
  const int mx = 227 * 1024;
  cudaError_t e = cudaFuncSetAttribute(sweep_res_kernel<ADI_P, SW_MASS>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(sweep_res_kernel<ADI_P, SW_DER>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
}

template <>
void Ops<ADI_P>::factor(cudaStream_t st, unsigned grid, const SweepBatch& B, double* iu, unsigned long long* bad,
                        double tol) {
  factor_kernel<ADI_P><<<grid, 128, 0, st>>>(B, iu, bad, tol);
}

template <>
void Ops<ADI_P>::spike(cudaStream_t st, const SpikeBatch& B, int solve) {
  const dim3 grid((unsigned)((B.NN + 255) / 256), (unsigned)B.njobs);
  if (solve) spike_solve_kernel<ADI_P><<<grid, 256, 0, st>>>(B);
  else spike_tips_kernel<ADI_P><<<grid, 256, 0, st>>>(B);
}

template <>
void Ops<ADI_P>::spike_mod(cudaStream_t st, const SpikeModArgs& A, int solve) {
  const unsigned grid = (unsigned)((A.NN + 127) / 128);
  if (solve) spike_mod_solve_kernel<ADI_P><<<grid, 128, 0, st>>>(A);
  else spike_mod_tips_kernel<ADI_P><<<grid, 128, 0, st>>>(A);
}

#endif  // ADI_STUB

}  // namespace adi
