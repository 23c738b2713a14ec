// fdg_reduce.cuh — deterministic block + grid reductions (no float atomics).
//
// Every reducing kernel writes one partial per CTA; the last CTA to finish
// (atomic ticket) folds the partials in a fixed index order and writes the
// scalar.  The fold order depends only on the grid size, so results are
// bitwise reproducible run to run (SURVEY.md §7 "stable reduction order").
#pragma once

#include <cuda_runtime.h>

namespace fdg {

enum RedOp { RED_SUM = 0, RED_MAX = 1 };

template <RedOp OP>
__device__ __forceinline__ double red_combine(double a, double b) {
  if constexpr (OP == RED_SUM) return a + b;
  else return fmax(a, b);  // inputs are |.| >= 0 or NaN-propagating via isnan flags
}

template <RedOp OP>
__device__ __forceinline__ double warp_reduce(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = red_combine<OP>(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Reduces K values across the CTA; result valid in thread 0.
// `scratch` must hold 32*K doubles.  Contains __syncthreads().
template <RedOp OP, int K>
__device__ __forceinline__ void block_reduce(double (&v)[K], double* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = warp_reduce<OP>(v[k]);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < K; ++k) scratch[k * 32 + warp] = v[k];
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double x = lane < nwarps ? scratch[k * 32 + lane] : (OP == RED_SUM ? 0.0 : 0.0);
      v[k] = warp_reduce<OP>(x);
    }
  }
  __syncthreads();
}

// Grid-level reduction slot: partials[nblocks * K], a ticket counter and the
// K results.  The counter is reset by the finishing CTA, so a slot can be
// reused by the next launch on the same stream.
struct RedSlot {
  double* partials;
  unsigned int* counter;
  double* result;
};

// Call from every thread with the CTA-reduced values valid in thread 0.
template <RedOp OP, int K>
__device__ __forceinline__ void grid_finalize(const double (&v)[K], RedSlot slot, double* scratch) {
  __shared__ bool s_last;
  const unsigned nblocks = gridDim.x * gridDim.y * gridDim.z;
  const unsigned bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) slot.partials[(size_t)k * nblocks + bid] = v[k];
    __threadfence();
    const unsigned ticket = atomicAdd(slot.counter, 1u);
    s_last = (ticket == nblocks - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double a = OP == RED_SUM ? 0.0 : 0.0;
    for (unsigned i = threadIdx.x; i < nblocks; i += blockDim.x)
      a = red_combine<OP>(a, __ldcg(&slot.partials[(size_t)k * nblocks + i]));
    acc[k] = a;
  }
  block_reduce<OP, K>(acc, scratch);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) slot.result[k] = acc[k];
    *slot.counter = 0u;
    __threadfence();
  }
}

}  // namespace fdg
