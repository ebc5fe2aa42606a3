// dispatch.h -- per-degree kernel entry points of libadimaxwell.so.
//
// Every kernel is a template on the B-spline degree P (band half-width).  To
// keep nvcc times short each degree is instantiated in its own translation
// unit (degree.cu compiled with -DADI_P=1..5); the host orchestration in
// adi_maxwell.cu reaches them through Ops<P>.  Internal header (not ABI).
#pragma once
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace adi {

enum SweepKind { SW_MASS_V1 = 0, SW_MASS = 1, SW_MOD = 2 };

template <int P>
struct Ops {
  // RHS of the E (kind 0) / H (kind 1) system of component d in substep s.
  static void rhs(cudaStream_t st, dim3 grid, const RhsArgs& args, int kind, int s, int d);
  static void rhs_tma(cudaStream_t st, dim3 grid, const RhsArgs& args, const RhsTmaMaps& maps, int kind, int s, int d);
  static cudaError_t rhs_attrs();
  static cudaError_t rhs_tma_attrs();
  // One sweep launch (grid, dynamic smem computed by the caller).
  static void sweep(cudaStream_t st, unsigned grid, size_t smem, const SweepArgs& A, int kind, int nck);
  static cudaError_t sweep_attrs(int mass_smem, int mass2_smem, int mod_smem);
  static void pivot_scan(cudaStream_t st, unsigned grid, const SweepArgs& A, unsigned long long* bad, double tol);
};

}  // namespace adi
