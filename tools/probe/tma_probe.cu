// Standalone probe of sweep_tma_kernel (mass mode, p = 2) on a small N^3 field: run each
// variant in its own process; prints max |out - in-place legacy| and any CUDA error.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include "../../paper_2103_06998_b200/csrc/sweep_tma.cuh"

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return (PFN_cuTensorMapEncodeTiled_v12000)p;
}
static bool mk(CUtensorMap* m, const double* ptr, const int d[3], int axis) {
  cuuint64_t gd[3] = {(cuuint64_t)d[0], (cuuint64_t)d[1], (cuuint64_t)d[2]};
  cuuint64_t st[2] = {(cuuint64_t)d[0] * 8, (cuuint64_t)d[0] * d[1] * 8};
  cuuint32_t box[3];
  if (axis == 0) box[0] = 16, box[1] = 32, box[2] = 1;
  else if (axis == 1) box[0] = 32, box[1] = 16, box[2] = 1;
  else box[0] = 32, box[1] = 1, box[2] = 16;
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)ptr, gd, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     axis == 0 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
  return r == CUDA_SUCCESS;
}
int main(int argc, char** argv) {
  const int N = argc > 1 ? atoi(argv[1]) : 36, axis = argc > 2 ? atoi(argv[2]) : 2;
  const size_t U = (size_t)N * N * N;
  double *f, *ck;
  cudaMalloc(&f, U * 8);
  cudaMalloc(&ck, 64 << 20);
  std::vector<double> h(U);
  for (size_t i = 0; i < U; i++) h[i] = (double)(i % 97) / 97.0;
  cudaMemcpy(f, h.data(), U * 8, cudaMemcpyHostToDevice);
  // identity-ish factors: l = 0, 1/u = 1, u = 0 => x = f (exercises the data movement only)
  std::vector<double> fac((size_t)N * 5, 0.0);
  for (int k = 0; k < N; k++) fac[k * 5 + 2] = 1.0;
  double* dfac;
  cudaMalloc(&dfac, fac.size() * 8);
  cudaMemcpy(dfac, fac.data(), fac.size() * 8, cudaMemcpyHostToDevice);
  adi::SweepBatch B;
  memset(&B, 0, sizeof B);
  B.N = N;
  B.njobs = 1;
  B.ckpt = ck;
  B.nck = (N + 15) / 16;
  adi::SweepJob& J = B.job[0];
  J.in = f;
  J.out = f;
  J.axis = axis;
  J.lo = 0;
  J.hi = N;
  J.var = 0;
  J.dims[0] = J.dims[1] = J.dims[2] = N;
  const int nf = N, ntiles = (nf + 31) / 32 * N;
  B.ntiles = ntiles;
  B.fac[0] = B.fac[1] = dfac;
  B.hk[0] = B.hk[1] = 0;
  B.tk[0] = B.tk[1] = N;
  B.kfac[0][2] = B.kfac[1][2] = 1.0;
  adi::SweepTmaMaps M;
  memset(&M, 0, sizeof M);
  for (int a = 0; a < 4; a++) mk(&M.m[0][a], f, J.dims, axis);
  auto k = adi::sweep_tma_kernel<2, adi::SW_MASS>;
  size_t smem = adi::st_smem_bytes<adi::SW_MASS>();
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  printf("attr: %s smem %zu sizeof(B)=%zu sizeof(M)=%zu\n", cudaGetErrorString(e), smem, sizeof B, sizeof M);
  k<<<4, 32 * adi::st_warps(adi::SW_MASS), smem>>>(B, M);
  e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<double> g(U);
  cudaMemcpy(g.data(), f, U * 8, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (size_t i = 0; i < U; i++) mx = fmax(mx, fabs(g[i] - h[i]));
  printf("N=%d axis=%d max|out-in| = %g\n", N, axis, mx);
  return e != cudaSuccess;
}
