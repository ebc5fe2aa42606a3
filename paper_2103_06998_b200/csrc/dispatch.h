// dispatch.h -- per-degree kernel entry points of libadimaxwell.so.
//
// Every kernel is a template on the B-spline degree P (band half-width).  To
// keep nvcc times short each degree is instantiated in its own translation
// unit (degree.cu compiled with -DADI_P=1..5); the host orchestration in
// adi_maxwell.cu reaches them through Ops<P>.  Internal header (not ABI).
#pragma once
#include <cuda_runtime.h>

#include "rhs.cuh"
#include "sweep.cuh"

namespace adi {

template <int P>
struct Ops {
  // RHS of the E (kind 0) / H (kind 1) system of component d in substep s.
  // tma: halo planes by cp.async.bulk.tensor (maps valid), else cp.async.
  static void rhs(cudaStream_t st, dim3 grid, const RhsArgs& args, const RhsMaps& maps, bool tma, int kind, int s, int d);
  static cudaError_t rhs_attrs();
  // One batched sweep launch (persistent grid chosen by the caller).
  static void sweep(cudaStream_t st, unsigned grid, const SweepBatch& B, bool modified);
  // Set the dynamic shared memory of both sweep kernels; occ[0|1] = resident
  // blocks per SM of the mass / modified kernel.
  static cudaError_t sweep_attrs(int occ[2]);
  // Pivot cache of one row-modified family (job 0 of B).
  static void factor(cudaStream_t st, unsigned grid, const SweepBatch& B, double* iu, unsigned long long* bad, double tol);
};

}  // namespace adi
