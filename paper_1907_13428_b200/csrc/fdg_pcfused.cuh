// fdg_pcfused.cuh — preconditioner axis passes fused pairwise through L2.
//
// CirculantPreconditioner::solve (circulant.cpp:49-67) runs as Hartley passes
// x2 -> x1 -> t(÷λ_S) -> x1 -> x2 (fdg_passes.cuh).  The two spatial passes
// on either side of the t filter act on one time slab (n1 x n2) at a time, so
// each pair runs as ONE persistent kernel:
//   P12: rows (x2) of slab s, then columns (x1) of slab s   (r -> h)
//   P45: columns (x1) of slab s, then rows (x2) + r.z       (h -> z)
// Work items (tiles of 2G fibres) of the first pass for slab s and of the
// second pass for slab s - LAG are interleaved in one static order; CTA c runs
// items c, c + grid, ...  A second-pass item waits (acquire spin on a per-slab
// counter) until every first-pass tile of its slab is stored and reads them
// back with cp.async.cg, i.e. from L2: with LAG slabs of n1*n2*8 bytes in
// flight (4 MB at 256^2) the intermediate never makes an HBM round trip.
// HBM traffic per pair: 2N (P12) / 3N (P45) instead of 4N / 5N.
//
// Deadlock freedom: the grid is the resident-CTA count, every item waits
// only on items earlier in the static order (the earliest unfinished item
// can always run), and the kernel lets its dependents launch only after its
// own items are done (they must not take SM slots from its CTAs).  The static order also keeps the r.z partials per CTA
// deterministic (bitwise reproducible fold).
#pragma once

#include <cuda_runtime.h>

#include "fdg_fft.cuh"
#include "fdg_passes.cuh"
#include "fdg_reduce.cuh"

namespace fdg {

#ifndef FDG_PIPE_LAG
#define FDG_PIPE_LAG 8
#endif

template <int N>
struct PipeCfg {
  using C = Cfg<N>;
  static constexpr int G = C::G, T = C::T, R = C::R, THREADS = C::THREADS;
  static constexpr int W = 2 * G;        // fibres per tile (rows or columns)
  static constexpr int TILE = W * N;     // doubles per staged tile
  static constexpr int MINB = N <= 256 ? 3 : 2;
  // exchange (single) | twiddles (N) | one staged tile (read into registers
  // before the next item's prefetch lands in the same buffer)
  static constexpr size_t SMEM = sizeof(double2) * (C::EXB + N) + sizeof(double) * (size_t)TILE;
};

struct PipeArgs {
  const double* in;  // first pass input
  double* mid;       // first pass output = second pass input
  double* out;       // second pass output (may equal mid)
  const double* rdot;
  RedSlot red;
  int nt, n;  // slabs, n1 == n2 == n
  const double2* tw;
  int* ready;  // nt per-slab counters + 1 done counter, zero between launches
  int rows_first;  // 1: P12, 0: P45
  const int* guard;
};

template <int N>
__global__ void __launch_bounds__(PipeCfg<N>::THREADS, PipeCfg<N>::MINB) k_pc_pipe(PipeArgs a) {
  using P = PipeCfg<N>;
  using C = Cfg<N>;
  constexpr int R = P::R, T = P::T, G = P::G, W = P::W, TILE = P::TILE;
  extern __shared__ double2 smem_raw[];
  __shared__ double scratch[32];
  Ex ex{smem_raw, smem_raw, 0};
  double2* tw = smem_raw + C::EXB;
  double* stage = reinterpret_cast<double*>(tw + N);
  load_table(tw, a.tw, N);
  // No early launch_dependents: CTAs of the next kernel would occupy SM slots
  // (waiting in griddepcontrol.wait) before all CTAs of this kernel are
  // resident, and a spinning consumer could then wait forever.
  pdl_wait();
  if (paused(a.guard)) return;
  const int n = a.n, nt = a.nt;
  const int FB = n / W;  // tiles per slab and pass
  // lag (slabs) between a slab's two passes: at least two rounds of the grid,
  // so consumers rarely wait (LAG slabs of n^2 doubles stay in L2)
  const int lag = max(FDG_PIPE_LAG, (int)((2 * gridDim.x + 2 * FB - 1) / (2 * FB)) + 1);
  const int D = nt < lag ? nt : lag;
  const int total = 2 * nt * FB;
  const size_t slab = (size_t)n * n;
  // static item order: first-pass items of slab q, then second-pass items of slab q - D
  auto decode = [&](int i, int& second, int& s, int& tile) {
    if (i < D * FB) {
      second = 0;
      s = i / FB;
      tile = i - s * FB;
      return;
    }
    const int j = i - D * FB;
    if (j < (nt - D) * 2 * FB) {
      const int q = D + j / (2 * FB), w = j - (q - D) * 2 * FB;
      second = w >= FB;
      s = second ? q - D : q;
      tile = second ? w - FB : w;
    } else {
      const int j2 = j - (nt - D) * 2 * FB;
      second = 1;
      s = nt - D + j2 / FB;
      tile = j2 - (s - (nt - D)) * FB;
    }
  };
  // pass kind of an item: rows (x2) or columns (x1)
  auto is_rows = [&](int second) { return (second == 0) == (a.rows_first != 0); };
  // Stage item i's input into stage buffer buf.  A second-pass item needs
  // every first-pass tile of its slab stored: blocking -> spin until then
  // (only for the item about to run: never while this CTA still holds an
  // unpublished first-pass tile); else report false if not yet ready.
  // Readiness of item i for staging: thread 0 checks (blocking: spins) and
  // publishes the answer in s_ok; the caller's next __syncthreads makes it
  // (and, through thread 0's acquire fence, the slab's data) visible.
  __shared__ int s_ok;
  auto check = [&](int i, bool blocking) {
    if (threadIdx.x != 0) return;
    int second, s, tile;
    decode(i, second, s, tile);
    int ok = 1;
    if (second) {
      volatile int* rd = &a.ready[s];
      if (blocking)
        while (*rd < FB) __nanosleep(32);
      ok = *rd >= FB;
      __threadfence();
    }
    s_ok = ok;
  };
  auto issue = [&](int i, int buf) {
    int second, s, tile;
    decode(i, second, s, tile);
    const double* src = (second ? a.mid : a.in) + (size_t)s * slab;
    double* dst = stage;
    if (is_rows(second))
      stage_rows(dst, src + (size_t)tile * W * n, TILE);
    else
      stage_cols<W>(dst, src + (size_t)tile * W, n, n);
  };
  double acc = 0.0;
  int it = blockIdx.x, buf = 0;
  if (it < total) check(it, false);
  __syncthreads();  // twiddles, s_ok
  bool staged = it < total && s_ok;
  if (staged) issue(it, 0);
  cp_async_commit();
  for (; it < total; it += gridDim.x, buf ^= 1) {
    int second, s, tile;
    decode(it, second, s, tile);
    const bool rows = is_rows(second);
    if (!staged) {  // the earliest unfinished item of this CTA: wait for its slab
      check(it, true);
      __syncthreads();
      issue(it, buf);
      cp_async_commit();
    }
    cp_async_wait<0>();
    __syncthreads();
    const double* st = stage;
    double2 v[R];
    int g, t;
    if (rows) {  // lane-major: lane g = fibres 2g, 2g+1 of the tile
      g = threadIdx.x / T;
      t = threadIdx.x % T;
#pragma unroll
      for (int m = 0; m < R; ++m) v[m] = make_double2(st[(2 * g) * N + t + m * T], st[(2 * g + 1) * N + t + m * T]);
    } else {  // interleaved: lane g = columns 2g, 2g+1
      g = threadIdx.x % G;
      t = threadIdx.x / G;
#pragma unroll
      for (int m = 0; m < R; ++m) v[m] = *reinterpret_cast<const double2*>(st + (t + m * T) * W + 2 * g);
    }
    const int nxt = it + gridDim.x;
    if (nxt < total) check(nxt, false);
    __syncthreads();  // the staged tile is in registers: the buffer is free; s_ok
    staged = nxt < total && s_ok;
    if (staged) issue(nxt, buf ^ 1);
    cp_async_commit();
    double* dst = (second ? a.out : a.mid) + (size_t)s * slab;
    if (rows) {
      fft_lane<N, R, G, false, 1>(v, ex, t, g, tw);
      hartley_lane<N, R, G, 1>(v, ex, t, g);
      const size_t ia = (size_t)(tile * W + 2 * g) * n;
      const bool dot = second && a.rdot;
      const double* rd = a.rdot + (size_t)s * slab;
#pragma unroll
      for (int m = 0; m < R; ++m) {
        const int pos = t + m * T;
        dst[ia + pos] = v[m].x;
        dst[ia + n + pos] = v[m].y;
        if (dot) acc += __ldcg(&rd[ia + pos]) * v[m].x + __ldcg(&rd[ia + n + pos]) * v[m].y;
      }
    } else {
      fft_lane<N, R, G, false, 0>(v, ex, t, g, tw);
      hartley_lane<N, R, G, 0>(v, ex, t, g);
      double* base = dst + (size_t)tile * W + 2 * g;
#pragma unroll
      for (int m = 0; m < R; ++m) *reinterpret_cast<double2*>(base + (size_t)(t + m * T) * n) = v[m];
    }
    if (!second) {  // publish: this first-pass tile of slab s is stored
      __syncthreads();  // every thread's stores precede thread 0's release
      if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(&a.ready[s], 1);
      }
    }
  }
  pdl_trigger();  // every item of this CTA is done
  if (a.rdot) {
    double vv[1] = {acc};
    block_reduce<RED_SUM, 1>(vv, scratch);
    grid_finalize<RED_SUM, 1>(vv, a.red, scratch);
  }
  // the last CTA out resets the counters for the next launch
  __shared__ bool s_last;
  if (threadIdx.x == 0) s_last = atomicAdd(&a.ready[nt], 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (s_last) {
    for (int i = threadIdx.x; i <= nt; i += blockDim.x) a.ready[i] = 0;
    __threadfence();
  }
}

}  // namespace fdg
