// dispatch.h -- per-degree kernel entry points of libadimaxwell.so.
//
// Every kernel is a template on the B-spline degree P (band half-width).  To
// keep nvcc times short each degree is instantiated in its own translation
// unit (degree.cu compiled with -DADI_P=1..5); the host orchestration in
// adi_maxwell.cu reaches them through Ops<P>.  Internal header (not ABI).
#pragma once
#include <cuda_runtime.h>

#include "rhs.cuh"
#include "rhs3.cuh"
#include "sweep.cuh"
#include "sweep_tw.cuh"
#include "sweep_twm.cuh"
#include "sweep_tma.cuh"
#include "sweep_res.cuh"
#include "spike.cuh"

namespace adi {

template <int P>
struct Ops {
  // RHS of the E (kind 0) / H (kind 1) system of component d in substep s.
  // tma: halo planes by cp.async.bulk.tensor (maps valid), else cp.async.
  // grid: (every tile, 1, z-chunks); one launch (rim tiles first, then the interior ones).
  static void rhs(cudaStream_t st, dim3 grid, const RhsArgs& args, const RhsMaps& maps, bool tma, int kind,
                  int s, int d);
  static cudaError_t rhs_attrs();
  // The three E right-hand sides of substep s in one launch (rhs3.cuh; TMA, P <= 3).
  static void rhs3(cudaStream_t st, dim3 grid, const Rhs3Args& args, const Rhs3Maps& maps, int s);
  static cudaError_t rhs3_attrs();
  // One batched sweep launch (persistent grid chosen by the caller).
  // twisted: two-segment variant (mass / derivative modes: SPIKE, sweep_tw.cuh;
  // row-modified mode: twisted factorisation, sweep_twm.cuh).
  static void sweep(cudaStream_t st, unsigned grid, const SweepBatch& B, int mode, bool twisted);
  // Set the dynamic shared memory of the sweep kernels; occ[mode] / occ_tw[mode] =
  // resident blocks per SM (SweepMode order: mass, modified, derivative projection).
  static cudaError_t sweep_attrs(int occ[3], int occ_tw[3]);
  // One batched sweep launch of the TMA-staged kernel (sweep_tma.cuh); grid = blocks of
  // st_warps(mode) warps, one block per SM.
  static void sweep_tma(cudaStream_t st, unsigned grid, const SweepBatch& B, const SweepTmaMaps& maps, int mode);
  // dynamic shared memory of the TMA-staged sweeps; occ[mode] = resident blocks per SM
  static cudaError_t sweep_tma_attrs(int occ[3]);
  // Fiber-resident two-segment sweep (sweep_res.cuh; modes SW_MASS / SW_DER): one block of
  // `warps` warps per SM, `smem` dynamic shared bytes.
  static void sweep_res(cudaStream_t st, unsigned grid, unsigned warps, size_t smem, const SweepBatch& B,
                        const SweepResMaps& maps, int mode);
  static cudaError_t sweep_res_attrs();
  // NEXT-1 partitioned z-solve (spike.cuh): solve = 0: tip pass, 1: corrected banded solve;
  // grid (fiber blocks of 256, jobs).
  static void spike(cudaStream_t st, const SpikeBatch& B, int solve);
  // ... of the row-modified z sweep (per-fiber matrix): solve = 0 tips, 1 interface + segment solve
  static void spike_mod(cudaStream_t st, const SpikeModArgs& A, int solve);
  // Pivot cache of one row-modified family (job 0 of B).
  static void factor(cudaStream_t st, unsigned grid, const SweepBatch& B, double* iu, unsigned long long* bad, double tol);
};

}  // namespace adi
