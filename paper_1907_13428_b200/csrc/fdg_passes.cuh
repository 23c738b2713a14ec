// fdg_passes.cuh — the FFT passes of the hot path (persistent CTAs).
//
// Every pass is one kernel over "tiles" of 2G fibres (two real fibres packed
// as one complex FFT lane, G lanes per CTA).  CTAs are persistent (grid =
// resident CTAs, 2 per SM), stage the per-axis twiddle table in shared memory
// once and loop over tiles.
//
// Two variants per pass:
//   PF = true  ("full tiles": n == L/2 for Toeplitz embeddings, tiles inside
//              the array, L <= 512): software-pipelined.  While a CTA runs the
//              FFTs of tile i, cp.async brings tile i+1's input (and tile i's
//              epilogue operands) into shared memory, so neither the tile load
//              nor the epilogue reads stall on HBM latency.
//   PF = false (any shape): direct loads with bounds predicates.
//
// Reference: ConstraintOperator::apply_mode (toeplitz.cpp:124-172) — pack,
// r2c, x symbol, c2r, unpack-accumulate — is one register-resident
// load -> FFT -> x symbol -> IFFT -> epilogue here, with the zero padding and
// the truncation to n taken from registers (no packed workspace in HBM).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "fdg_fft.cuh"
#include "fdg_internal.h"
#include "fdg_reduce.cuh"

namespace fdg {

// Tile configuration for transform length L.
//   R: complex values per thread, T = L/R threads per lane, G lanes per CTA
//   (256 threads), DB: double-buffered exchanges, TS: twiddles in smem.
#ifndef FDG_T128_THREADS
#define FDG_T128_THREADS 128
#endif
#ifndef FDG_T128_MINB
#define FDG_T128_MINB 3
#endif
#ifndef FDG_T256_THREADS
#define FDG_T256_THREADS 128
#endif
#ifndef FDG_T256_MINB
#define FDG_T256_MINB 3
#endif
#ifndef FDG_T256_DB
#define FDG_T256_DB 0
#endif
#ifndef FDG_T512_THREADS
#define FDG_T512_THREADS 128
#endif
#ifndef FDG_T512_MINB
#define FDG_T512_MINB 3
#endif
#ifndef FDG_T512_DB
#define FDG_T512_DB 0
#endif
#ifndef FDG_PF_MAX
#define FDG_PF_MAX 512  // largest length with staged (cp.async) full-tile variants
#endif
template <int L>
struct Cfg {
  static constexpr int R = fft_radix(L);
  static constexpr int T = L / R;
  static constexpr int G_ = (L == 128 ? FDG_T128_THREADS : (L == 256 ? FDG_T256_THREADS : (L == 512 ? FDG_T512_THREADS : 256))) / T;
  static constexpr int G = G_ > 32 ? 32 : (G_ < 2 ? 2 : G_);
  static constexpr int THREADS = G * T;
  static constexpr int MINB = L == 128 ? FDG_T128_MINB : (L == 256 ? FDG_T256_MINB : (L == 512 ? FDG_T512_MINB : 2));
  static constexpr bool DB = L == 256 ? (FDG_T256_DB != 0) : (L == 512 ? (FDG_T512_DB != 0) : L <= 512);
  static constexpr bool TS = L <= 1024;
  static constexpr size_t EXB = (size_t)L * G;  // double2 per exchange buffer
  static constexpr bool PF_OK = L >= 16 && L <= FDG_PF_MAX;
};

// Shared-memory plan: exchange buffer(s) | twiddles | extra table | staging.
template <int L, bool DB, int EXTRA_TAB, int STAGE_DOUBLES>
struct Plan {
  using C = Cfg<L>;
  static constexpr size_t EX = C::EXB * (DB ? 2 : 1);               // double2
  static constexpr size_t TAB = (C::TS ? (size_t)L : 0) + EXTRA_TAB;  // double2
  static constexpr size_t BYTES = sizeof(double2) * (EX + TAB) + sizeof(double) * (size_t)STAGE_DOUBLES;
};

template <int L, bool DB>
struct Smem {
  Ex ex;
  const double2* tw;
  double2* tab;   // first double2 after the twiddles (extra table)
  double* stage;  // staging area (after the extra table)
  __device__ __forceinline__ Smem(double2* base, const double2* gtw, int extra_tab) {
    using C = Cfg<L>;
    ex.buf0 = base;
    ex.buf1 = DB ? base + C::EXB : base;
    ex.k = 0;
    double2* t = base + C::EXB * (DB ? 2 : 1);
    if constexpr (C::TS) {
      load_table(t, gtw, L);
      tw = t;
      t += L;
    } else {
      tw = gtw;
    }
    tab = t;
    stage = reinterpret_cast<double*>(t + extra_tab);
  }
};

// cp.async (LDGSTS) helpers: 16-byte global -> shared copies that complete in
// the background while the FFT runs.
__device__ __forceinline__ void cp_async16(void* dst_smem, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst_smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
// Bulk-copy (TMA) staging with an mbarrier per staged group: one elected
// thread arms the barrier with the byte count and issues
// cp.async.bulk global -> shared copies; every consumer waits on the
// barrier's phase parity.  Replaces per-thread cp.async (LDGSTS) staging:
// no LSU instructions or registers per staged 16 bytes.
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred P1;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @!P1 bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// generic-proxy accesses of the CTA before -> async-proxy (bulk copy) writes after
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// 2-D tensor-map TMA load of one box (x = column, y = row) into dst, on bar.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// One thread: a contiguous tile (bytes, multiple of 16) into dst, on bar.
__device__ __forceinline__ void bulk_tile(double* dst, const double* src, unsigned bytes, unsigned long long* bar) {
  fence_proxy_async();
  mbar_expect_tx(bar, bytes);
  bulk_g2s(dst, src, bytes, bar);
}
// One full warp: an n-row x W-double column tile (row stride C) into dst
// [pos][W], one bulk copy per row segment (W * 8 bytes, a multiple of 16).
template <int W>
__device__ __forceinline__ void bulk_cols(double* dst, const double* src, int n, int C, unsigned long long* bar) {
  const int lane = threadIdx.x & 31;
  fence_proxy_async();
  if (lane == 0) mbar_expect_tx(bar, (unsigned)(n * W * sizeof(double)));
  __syncwarp();
  for (int pos = lane; pos < n; pos += 32) bulk_g2s(dst + pos * W, src + (size_t)pos * C, W * sizeof(double), bar);
}
#ifndef FDG_TMA_P
#define FDG_TMA_P 1  // preconditioner row passes: one bulk copy (TMA) per tile
#endif
#ifndef FDG_TMA_PCOL
#define FDG_TMA_PCOL 2  // column / t passes: 2 = 2-D tensor-map boxes, 1 = one bulk copy per row segment
                        // (measured slow), 0 = per-thread cp.async
#endif
// One thread: an n-row x W-double column tile at (column x, row y) of a 2-D
// tensor map, in boxes of min(n, 256) rows, into dst [pos][W], on bar.
template <int W>
__device__ __forceinline__ void tma_cols(double* dst, const CUtensorMap* map, int x, int y, int n,
                                         unsigned long long* bar) {
  fence_proxy_async();
  mbar_expect_tx(bar, (unsigned)(n * W * sizeof(double)));
  const int bh = n < 256 ? n : 256;
  for (int r0 = 0; r0 < n; r0 += bh) tma_load_2d(dst + r0 * W, map, x, y + r0, bar);
}

// CTA-cooperative contiguous copy of `nd` doubles (nd even, 16-byte aligned).
__device__ __forceinline__ void stage_rows(double* dst, const double* src, int nd) {
  for (int i = 2 * threadIdx.x; i < nd; i += 2 * blockDim.x) cp_async16(dst + i, src + i);
}
// CTA-cooperative copy of a column tile: n positions x W doubles (W even),
// source row stride C doubles -> [pos][P] in shared memory (pitch P >= W).
template <int W, int P = W>
__device__ __forceinline__ void stage_cols(double* dst, const double* src, int n, int C) {
  constexpr int CH = W / 2;  // 16-byte chunks per position
  for (int i = threadIdx.x; i < n * CH; i += blockDim.x) {
    const int pos = i / CH, j = i - pos * CH;
    cp_async16(dst + pos * P + 2 * j, src + (size_t)pos * C + 2 * j);
  }
}

// =================================================================== rows
// Row pass along x2 (contiguous fibres of length n; embedding length L).
//   MODE 0 (apply):  out = scale * T2 x + psi c1 x_{k-+1}
//   MODE 1 (S out):  q = vp + scale * T2 x + psi c1 x_{k+1}; q_out = q (opt);
//                    r -= (num/den) q; reduce |r|^2
// The stencil diagonal psi c0 x_k is folded into the x2 symbol on the host.
struct RowArgs {
  const double* x;
  const double* vp;
  double* out;
  double* q_out;
  double* r;
  const double* r_in;  // MODE 1: r = r_in - alpha q (null: r_in = r)
  int nt, n1, n;
  const double2* sym;
  const double2* tw;
  double scale;
  int tkind;  // 1: stencil
  double tc0, tc1;
  int tdir;  // -1: uses k-1 (forward B), +1: uses k+1 (adjoint)
  const double* a_num;
  const double* a_den;
  RedSlot red;
  // MODE 2 (fused CG update + B row pass): d_new = z + beta d_old is the FFT
  // input (written to dnew), x += alpha d_old (alpha = a_num/a_den).
  const double* z;
  const double* dold;
  double* dnew;
  double* xs;
  const double* b_num;
  const double* b_den;
  int first;  // d_new = z (first Krylov iteration, no beta term, no x update)
  int upd_x;  // apply x += alpha d_old
  const int* guard;  // speculative PCG iteration: skip the launch when *guard != 0
  const double2* twh;    // split passes (fdg_conv.cuh): L/2-point twiddles
  const double2* twist;  // split passes: W_L^j, j < L/2
  const double* sym_re;  // split passes: real symbol (symmetric factor) or null
  const double2* tw256;  // Q-split passes (fdg_convq.cuh): 256-point plan
  const double2* twq;    // Q-split passes: W_L^k, k < L
  const double2* chirp_in;  // k_row<.., CH>: input times conj(chirp[pos])
};

// Early exit of a speculatively enqueued PCG kernel (the host enqueues
// iteration k+1 before it has read iteration k's scalars; the control kernel
// of iteration k raises the pause flag when the host must intervene).
__device__ __forceinline__ bool paused(const int* guard) {
  return guard != nullptr && *reinterpret_cast<const volatile int*>(guard) != 0;
}

// Programmatic dependent launch: the pass kernels are launched with
// programmatic stream serialization, so a kernel's CTAs may start (and stage
// their twiddle tables) while the previous kernel drains its last tiles;
// griddepcontrol.wait then blocks until the previous grid's memory is
// visible.  Both are no-ops for a normal launch.
#ifndef FDG_EARLY_TRIGGER
#define FDG_EARLY_TRIGGER 1
#endif
__device__ __forceinline__ void pdl_trigger() {
#if FDG_EARLY_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;\n" ::);
#endif
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

template <int L, int MODE, bool PF>
struct RowPlan {
  using C = Cfg<L>;
  static constexpr int TILE = PF ? 2 * C::G * (L / 2) : 0;  // doubles per staged operand
  static constexpr int NIN = MODE == 2 ? 2 : 1;  // staged input operands
  static constexpr int NEPI = PF ? (MODE == 0 ? 1 : (MODE == 1 ? 3 : 2)) : 0;
  static constexpr bool DB = C::DB && !(PF && MODE != 0);
  using P = Plan<L, DB, 0, TILE * (NIN + NEPI)>;
  static constexpr size_t SMEM = P::BYTES;
};

// CH (MODE 0, unstaged): the 2-level preconditioner's Bluestein pre-chirp
// z conj(chirp[pos]) folded into the load (fdg_kernels.cu k_bs_pre_rows);
// a separate instantiation, so the plain passes keep their code.
template <int L, int MODE, bool PF, bool CH = false>
__global__ void __launch_bounds__(Cfg<L>::THREADS, Cfg<L>::MINB) k_row(RowArgs a) {
  using C = Cfg<L>;
  using RP = RowPlan<L, MODE, PF>;
  constexpr int R = C::R, T = C::T, G = C::G, H = (R + 1) / 2;
  constexpr int TILE = RP::TILE;
  extern __shared__ __align__(128) double2 smem_raw[];
  __shared__ double scratch[32];
  Smem<L, RP::DB> S(smem_raw, a.tw, 0);
  pdl_trigger();
  pdl_wait();
  if (paused(a.guard)) return;
  double* st_in = S.stage;                    // FFT input (MODE 2: z)
  double* st_in2 = S.stage + TILE;            // MODE 2: d_old
  double* st_nb = S.stage + RP::NIN * TILE;   // neighbour row (MODE 2: z)
  double* st_nb2 = st_nb + TILE;              // MODE 2: neighbour d_old
  double* st_vp = S.stage + 2 * TILE;         // MODE 1
  double* st_r = S.stage + 3 * TILE;          // MODE 1
  const int g = threadIdx.x / T, t = threadIdx.x % T;  // lane-major: coalesced rows
  const int F = a.nt * a.n1;
  const int ntiles = (F + 2 * G - 1) / (2 * G);
  const int n = a.n;
  double alpha = 0.0, beta = 0.0;
  if constexpr (MODE == 1) {
    if (a.r) alpha = *a.a_num / *a.a_den;
  }
  if constexpr (MODE == 2) {
    if (a.upd_x) alpha = *a.a_num / *a.a_den;
    if (!a.first) beta = *a.b_num / *a.b_den;
  }
  const bool first = MODE == 2 && a.first;
  // FFT input operand(s) of the pass
  const double* in0 = MODE == 2 ? a.z : a.x;
  const double* in1 = a.dold;
  const ptrdiff_t noff = (ptrdiff_t)a.tdir * a.n1 * n;
  double acc = 0.0;
  if constexpr (PF) {
    if (blockIdx.x < ntiles) {
      stage_rows(st_in, in0 + (size_t)blockIdx.x * 2 * G * n, TILE);
      if (MODE == 2 && !first) stage_rows(st_in2, in1 + (size_t)blockIdx.x * 2 * G * n, TILE);
    }
    cp_async_commit();
  }
  __syncthreads();  // twiddle table
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int f0 = tile * 2 * G;
    const int f = f0 + 2 * g;
    const bool va = PF || f < F, vb = PF || f + 1 < F;
    const size_t ra = (size_t)f * n;  // row offset of the lane's first fibre
    double2 v[R];
    bool tile_nb = false;
    if constexpr (PF) {
      cp_async_wait<0>();
      __syncthreads();
#pragma unroll
      for (int m = 0; m < R; ++m) {
        const int pos = t + m * T;
        if (m < H) {
          double2 z = make_double2(st_in[(2 * g) * n + pos], st_in[(2 * g + 1) * n + pos]);
          if constexpr (MODE == 2) {
            if (!first) {
              z.x += beta * st_in2[(2 * g) * n + pos];
              z.y += beta * st_in2[(2 * g + 1) * n + pos];
            }
            a.dnew[ra + pos] = z.x;
            a.dnew[ra + n + pos] = z.y;
          }
          v[m] = z;
        } else {
          v[m] = make_double2(0.0, 0.0);
        }
      }
      __syncthreads();  // st_in and the epilogue staging are free
      const int k = f0 / a.n1;  // whole tile in one slice
      tile_nb = a.tkind == 1 && (a.tdir < 0 ? k >= 1 : k + 1 < a.nt);
      if (tile_nb) {
        stage_rows(st_nb, in0 + (size_t)f0 * n + noff, TILE);
        if (MODE == 2 && !first) stage_rows(st_nb2, in1 + (size_t)f0 * n + noff, TILE);
      }
      if constexpr (MODE == 1) {
        stage_rows(st_vp, a.vp + (size_t)f0 * n, TILE);
        if (a.r) stage_rows(st_r, (a.r_in ? a.r_in : a.r) + (size_t)f0 * n, TILE);
      }
      cp_async_commit();  // group E: this tile's epilogue operands
      const int nxt = tile + gridDim.x;
      if (nxt < ntiles) {
        stage_rows(st_in, in0 + (size_t)nxt * 2 * G * n, TILE);
        if (MODE == 2 && !first) stage_rows(st_in2, in1 + (size_t)nxt * 2 * G * n, TILE);
      }
      cp_async_commit();  // group I: next tile's input
    } else {
#pragma unroll
      for (int m = 0; m < R; ++m) {
        const int pos = t + m * T;
        double2 z = make_double2(0.0, 0.0);
        if (m < H && pos < n) {
          if (va) z.x = __ldg(in0 + ra + pos);
          if (vb) z.y = __ldg(in0 + ra + n + pos);
          if constexpr (MODE == 2) {
            if (!first) {
              if (va) z.x += beta * __ldg(in1 + ra + pos);
              if (vb) z.y += beta * __ldg(in1 + ra + n + pos);
            }
            if (va) a.dnew[ra + pos] = z.x;
            if (vb) a.dnew[ra + n + pos] = z.y;
          }
          if constexpr (CH) z = cmulc(z, __ldg(&a.chirp_in[pos]));
        }
        v[m] = z;
      }
    }
    fft_lane<L, R, G, false, 1>(v, S.ex, t, g, S.tw);
#pragma unroll
    for (int m = 0; m < R; ++m) v[m] = cmul(v[m], __ldg(&a.sym[t + m * T]));
    fft_lane<L, R, G, true, 1>(v, S.ex, t, g, S.tw);

    if constexpr (PF) {
      cp_async_wait<1>();  // group E landed (group I may still fly)
      __syncthreads();
    }
    const int ka = f / a.n1, kb = (f + 1) / a.n1;
    const bool nba = a.tkind == 1 && (a.tdir < 0 ? ka >= 1 : ka + 1 < a.nt);
    const bool nbb = a.tkind == 1 && (a.tdir < 0 ? kb >= 1 : kb + 1 < a.nt);
#pragma unroll
    for (int m = 0; m < H; ++m) {
      const int pos = t + m * T;
      if (!PF && pos >= n) continue;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (!PF && !(h ? vb : va)) continue;
        const int sl = (2 * g + h) * n + pos;  // staged element
        const size_t o = ra + h * n + pos;
        double val = a.scale * (h ? v[m].y : v[m].x);
        if constexpr (PF) {
          if (tile_nb) {
            double nbv = st_nb[sl];
            if (MODE == 2 && !first) nbv += beta * st_nb2[sl];
            val += a.tc1 * nbv;
          }
        } else {
          if (h ? nbb : nba) {
            double nbv = __ldg(in0 + o + noff);
            if (MODE == 2 && !first) nbv += beta * __ldg(in1 + o + noff);
            val += a.tc1 * nbv;
          }
        }
        if constexpr (MODE == 0 || MODE == 2) {
          a.out[o] = val;
          if (MODE == 2 && a.upd_x) a.xs[o] += alpha * __ldg(in1 + o);  // x += alpha d_old
        } else {
          const double q = (PF ? st_vp[sl] : __ldg(&a.vp[o])) + val;
          if (a.q_out) a.q_out[o] = q;
          if (a.r) {
            const double rn = (PF ? st_r[sl] : (a.r_in ? a.r_in : a.r)[o]) - alpha * q;
            a.r[o] = rn;
            acc += rn * rn;
          }
        }
      }
    }
  }
  if constexpr (MODE == 1) {
    if (a.r) {
      double vv[1] = {acc};
      block_reduce<RED_SUM, 1>(vv, scratch);
      grid_finalize<RED_SUM, 1>(vv, a.red, scratch);
    }
  }
}

// ================================================================ columns
// Column pass along an axis of length n with inner stride C, outer count O:
// element (o, pos, c) at o*n*C + pos*C + c.
//   MODE 0 (acc): out = acc + scale * T x            (acc may alias out)
//   MODE 2 (S mid, axis x1): Bp = u + scale*T p; w = Bp * inv_m2[o];
//        vp = scale * T w + a1[o] p; reduce sum(a1 p^2 + w Bp) = p^T S p
struct ColArgs {
  const double* x;
  const double* acc;
  double* out;
  double* w;
  int O, n, C;
  const double2* sym;
  const double2* tw;
  double scale;
  const double* inv_m2;
  const double* a1;
  RedSlot red;
  const int* guard;
  const double2* twh;    // split passes (fdg_conv.cuh)
  const double2* twist;
  const double* sym_re;
  const double2* tw256;  // Q-split passes (fdg_convq.cuh)
  const double2* twq;
};

template <bool FULL>
__device__ __forceinline__ double2 col_get(const double* p, int C, long c) {
  if (FULL || ((c + 1 < C) && ((C & 1) == 0))) return __ldg(reinterpret_cast<const double2*>(p));
  return make_double2(__ldg(p), (c + 1 < C) ? __ldg(p + 1) : 0.0);
}

template <bool FULL>
__device__ __forceinline__ void col_put(double* p, int C, long c, double2 val) {
  if (FULL || ((c + 1 < C) && ((C & 1) == 0))) {
    *reinterpret_cast<double2*>(p) = val;
  } else {
    p[0] = val.x;
    if (c + 1 < C) p[1] = val.y;
  }
}

template <int L, bool PF>
struct ColPlan {
  using C = Cfg<L>;
  static constexpr int TILE = PF ? 2 * C::G * (L / 2) : 0;
  using P = Plan<L, C::DB, 0, TILE>;
  static constexpr size_t SMEM = P::BYTES;
};

template <int L, int MODE, bool PF>
__global__ void __launch_bounds__(Cfg<L>::THREADS, Cfg<L>::MINB) k_col(ColArgs a) {
  using Cf = Cfg<L>;
  constexpr int R = Cf::R, T = Cf::T, G = Cf::G, H = (R + 1) / 2;
  constexpr int W = 2 * G;  // columns per tile
  extern __shared__ __align__(128) double2 smem_raw[];
  __shared__ double scratch[32];
  Smem<L, Cf::DB> S(smem_raw, a.tw, 0);
  pdl_trigger();
  pdl_wait();
  if (paused(a.guard)) return;
  double* st_in = S.stage;
  const int g = threadIdx.x % G, t = threadIdx.x / G;
  const int n = a.n, C = a.C;
  const int ncb = (C + W - 1) / W;
  const int ntiles = ncb * a.O;
  if constexpr (PF) {
    if (blockIdx.x < ntiles) {
      const int o = blockIdx.x / ncb;
      stage_cols<W>(st_in, a.x + (size_t)o * n * C + (size_t)(blockIdx.x - o * ncb) * W, n, C);
    }
    cp_async_commit();
  }
  __syncthreads();  // twiddle table
  double e = 0.0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int o = tile / ncb;
    const long c = (long)((tile - o * ncb) * G + g) * 2;
    const bool vc = PF || c < C;
    const size_t base = (size_t)o * n * C + c;
    double2 v[R];
    if constexpr (PF) {
      cp_async_wait<0>();
      __syncthreads();
#pragma unroll
      for (int m = 0; m < R; ++m)
        v[m] = m < H ? *reinterpret_cast<const double2*>(st_in + (t + m * T) * W + 2 * g) : make_double2(0.0, 0.0);
      __syncthreads();
      const int nxt = tile + gridDim.x;
      if (nxt < ntiles) {
        const int on = nxt / ncb;
        stage_cols<W>(st_in, a.x + (size_t)on * n * C + (size_t)(nxt - on * ncb) * W, n, C);
      }
      cp_async_commit();
    } else {
#pragma unroll
      for (int m = 0; m < R; ++m) {
        const int pos = t + m * T;
        v[m] = (m < H && pos < n && vc) ? col_get<false>(a.x + base + (size_t)pos * C, C, c)
                                        : make_double2(0.0, 0.0);
      }
      if constexpr (MODE == 0) {
        // the epilogue's accumulate operand: ask L2 for it now (a quarter of
        // the unstaged pass's stall samples sat on those loads)
        if (a.acc && vc) {
#pragma unroll
          for (int m = 0; m < H; ++m) {
            const int pos = t + m * T;
            if (pos < n) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.acc + base + (size_t)pos * C));
          }
        }
      }
    }
    fft_lane<L, R, G, false>(v, S.ex, t, g, S.tw);
#pragma unroll
    for (int m = 0; m < R; ++m) v[m] = cmul(v[m], __ldg(&a.sym[t + m * T]));
    fft_lane<L, R, G, true>(v, S.ex, t, g, S.tw);

    if constexpr (MODE == 0) {
#pragma unroll
      for (int m = 0; m < H; ++m) {
        const int pos = t + m * T;
        if (!PF && (pos >= n || !vc)) continue;
        const size_t o2 = base + (size_t)pos * C;
        double2 acc = make_double2(0.0, 0.0);
        if (a.acc) acc = col_get<PF>(a.acc + o2, C, c);
        col_put<PF>(a.out + o2, C, c, make_double2(acc.x + a.scale * v[m].x, acc.y + a.scale * v[m].y));
      }
    } else {
      // S mid pass: u is a.acc, w -> a.w, vp -> a.out
      const double im2 = a.inv_m2[o], a1 = a.a1[o];
      const bool vb = PF || c + 1 < C;
#pragma unroll
      for (int m = 0; m < R; ++m) {
        const int pos = t + m * T;
        if (m < H && (PF || (pos < n && vc))) {
          const size_t o2 = base + (size_t)pos * C;
          const double2 u = col_get<PF>(a.acc + o2, C, c);
          const double2 pv = col_get<PF>(a.x + o2, C, c);
          const double bx = u.x + a.scale * v[m].x;
          const double by = u.y + a.scale * v[m].y;
          const double wx = bx * im2, wy = vb ? by * im2 : 0.0;
          e += a1 * pv.x * pv.x + wx * bx;
          if (vb) e += a1 * pv.y * pv.y + wy * by;
          col_put<PF>(a.w + o2, C, c, make_double2(wx, wy));
          v[m] = make_double2(wx, wy);
        } else {
          v[m] = make_double2(0.0, 0.0);
        }
      }
      fft_lane<L, R, G, false>(v, S.ex, t, g, S.tw);
#pragma unroll
      for (int m = 0; m < R; ++m) v[m] = cmul(v[m], __ldg(&a.sym[t + m * T]));
      fft_lane<L, R, G, true>(v, S.ex, t, g, S.tw);
#pragma unroll
      for (int m = 0; m < H; ++m) {
        const int pos = t + m * T;
        if (!PF && (pos >= n || !vc)) continue;
        const size_t o2 = base + (size_t)pos * C;
        const double2 pv = col_get<PF>(a.x + o2, C, c);
        col_put<PF>(a.out + o2, C, c, make_double2(a.scale * v[m].x + a1 * pv.x, a.scale * v[m].y + a1 * pv.y));
      }
    }
  }
  if constexpr (MODE == 2) {
    double vv[1] = {e};
    block_reduce<RED_SUM, 1>(vv, scratch);
    grid_finalize<RED_SUM, 1>(vv, a.red, scratch);
  }
}

// ============================================================== Hartley
// Real Hartley transform H[f] = sum_j x_j cas(2 pi j f / N) of two real
// fibres packed as a + i b into one complex FFT (fdg_fft.cuh hartley_split).
// For the circulant preconditioner the multiplier lambda_S is even in every
// axis (spatial T. Chan eigenvalues are real and even; |conj(l_t) - s| =
// |l_t - s| for real s), so F^-1 D F == H^-1 D H axis by axis: all three
// passes stay real (N doubles in, N doubles out), see DESIGN.md.
template <int N, bool PF>
struct HPlan {
  using C = Cfg<N>;
  static constexpr int TILE = PF ? 2 * C::G * N : 0;
  using P = Plan<N, C::DB, 0, TILE>;
  static constexpr size_t SMEM = P::BYTES;
  using PT = Plan<N, C::DB, N, TILE>;  // t filter: lambda_t table after the twiddles
  static constexpr size_t SMEM_T = PT::BYTES;
};

template <int N, bool PF>
__global__ void __launch_bounds__(Cfg<N>::THREADS, Cfg<N>::MINB)
    k_hartley_row(const double* in, double* out, int F, const double2* tw, const double* rdot, RedSlot red,
                  const int* guard) {
  using Cf = Cfg<N>;
  constexpr int R = Cf::R, T = Cf::T, G = Cf::G;
  constexpr int TILE = HPlan<N, PF>::TILE;
  extern __shared__ __align__(128) double2 smem_raw[];
  __shared__ double scratch[32];
  Smem<N, Cf::DB> S(smem_raw, tw, 0);
  pdl_trigger();
  pdl_wait();
  if (paused(guard)) return;
  double* st_in = S.stage;
  const int g = threadIdx.x / T, t = threadIdx.x % T;  // lane-major: coalesced rows
  const int ntiles = (F + 2 * G - 1) / (2 * G);
  constexpr bool TMA = PF && FDG_TMA_P;
  __shared__ alignas(8) unsigned long long bar;
  unsigned ph = 0;
  if constexpr (TMA) {
    if (threadIdx.x == 0) {
      mbar_init(&bar, 1);
      mbar_init_fence();
      if (blockIdx.x < ntiles) bulk_tile(st_in, in + (size_t)blockIdx.x * TILE, 8u * TILE, &bar);
    }
  } else if constexpr (PF) {
    if (blockIdx.x < ntiles) stage_rows(st_in, in + (size_t)blockIdx.x * TILE, TILE);
    cp_async_commit();
  }
  __syncthreads();
  double acc = 0.0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int f = (tile * G + g) * 2;
    const bool va = PF || f < F, vb = PF || f + 1 < F;
    const size_t ia = (size_t)f * N, ib = ia + N;
    // the epilogue's dot-product operand: ask L2 for its lines now (one thread
    // per 128-byte line; its loads held 17% of this pass's stall samples)
    if (rdot && (t & 15) == 0) {
#pragma unroll
      for (int m = 0; m < R; ++m) {
        const int pos = t + m * T;
        if (T >= 16 || (pos & 15) == 0) {
          if (va) asm volatile("prefetch.global.L2 [%0];" ::"l"(rdot + ia + pos));
          if (vb) asm volatile("prefetch.global.L2 [%0];" ::"l"(rdot + ib + pos));
        }
      }
    }
    double2 v[R];
    if constexpr (PF) {
      if constexpr (TMA) {
        mbar_wait(&bar, ph);
        ph ^= 1;
      } else {
        cp_async_wait<0>();
        __syncthreads();
      }
#pragma unroll
      for (int m = 0; m < R; ++m) {
        const int pos = t + m * T;
        v[m] = make_double2(st_in[(2 * g) * N + pos], st_in[(2 * g + 1) * N + pos]);
      }
      __syncthreads();
      const int nxt = tile + gridDim.x;
      if constexpr (TMA) {
        if (threadIdx.x == 0 && nxt < ntiles) bulk_tile(st_in, in + (size_t)nxt * TILE, 8u * TILE, &bar);
      } else {
        if (nxt < ntiles) stage_rows(st_in, in + (size_t)nxt * TILE, TILE);
        cp_async_commit();
      }
    } else {
#pragma unroll
      for (int m = 0; m < R; ++m) {
        const int pos = t + m * T;
        v[m].x = va ? __ldg(&in[ia + pos]) : 0.0;
        v[m].y = vb ? __ldg(&in[ib + pos]) : 0.0;
      }
    }
    fft_lane<N, R, G, false, 1>(v, S.ex, t, g, S.tw);
    hartley_lane<N, R, G, 1>(v, S.ex, t, g);
#pragma unroll
    for (int m = 0; m < R; ++m) {
      const int pos = t + m * T;
      const double2 h = v[m];
      if (va) {
        out[ia + pos] = h.x;
        if (rdot) acc += __ldg(&rdot[ia + pos]) * h.x;
      }
      if (vb) {
        out[ib + pos] = h.y;
        if (rdot) acc += __ldg(&rdot[ib + pos]) * h.y;
      }
    }
  }
  if (rdot) {
    double vv[1] = {acc};
    block_reduce<RED_SUM, 1>(vv, scratch);
    grid_finalize<RED_SUM, 1>(vv, red, scratch);
  }
}

template <int N, bool PF>
__global__ void __launch_bounds__(Cfg<N>::THREADS, Cfg<N>::MINB)
    k_hartley_col(double* data, int O, int C, const double2* tw, const int* guard,
                  const __grid_constant__ CUtensorMap map) {
  using Cf = Cfg<N>;
  constexpr int R = Cf::R, T = Cf::T, G = Cf::G;
  constexpr int W = 2 * G;
  extern __shared__ __align__(128) double2 smem_raw[];
  Smem<N, Cf::DB> S(smem_raw, tw, 0);
  pdl_trigger();
  pdl_wait();
  if (paused(guard)) return;
  double* st_in = S.stage;
  const int g = threadIdx.x % G, t = threadIdx.x / G;
  const int ncb = (C + W - 1) / W;
  const int ntiles = ncb * O;
  constexpr bool TMA = PF && FDG_TMA_PCOL;
  __shared__ alignas(8) unsigned long long bar;
  unsigned ph = 0;
  auto src_of = [&](int tl) {
    const int ot = tl / ncb;
    return data + (size_t)ot * N * C + (size_t)(tl - ot * ncb) * W;
  };
  auto stage_tma = [&](int tl) {  // one box per 256 rows (2-D map), or one bulk copy per row (warp 0)
    if constexpr (FDG_TMA_PCOL == 2) {
      if (threadIdx.x == 0) {
        const int ot = tl / ncb;
        tma_cols<W>(st_in, &map, (tl - ot * ncb) * W, ot * N, N, &bar);
      }
    } else if (threadIdx.x < 32) {
      bulk_cols<W>(st_in, src_of(tl), N, C, &bar);
    }
  };
  if constexpr (TMA) {
    if (threadIdx.x == 0) {
      mbar_init(&bar, 1);
      mbar_init_fence();
    }
    __syncthreads();
    if (blockIdx.x < ntiles) stage_tma(blockIdx.x);
  } else if constexpr (PF) {
    if (blockIdx.x < ntiles) stage_cols<W>(st_in, src_of(blockIdx.x), N, C);
    cp_async_commit();
  }
  __syncthreads();
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int o = tile / ncb;
    const long c = (long)((tile - o * ncb) * G + g) * 2;
    const bool vc = PF || c < C;
    double* base = data + (size_t)o * N * C + c;
    double2 v[R];
    if constexpr (PF) {
      if constexpr (TMA) {
        mbar_wait(&bar, ph);
        ph ^= 1;
      } else {
        cp_async_wait<0>();
        __syncthreads();
      }
#pragma unroll
      for (int m = 0; m < R; ++m) v[m] = *reinterpret_cast<const double2*>(st_in + (t + m * T) * W + 2 * g);
      __syncthreads();
      const int nxt = tile + gridDim.x;
      if constexpr (TMA) {
        if (nxt < ntiles) stage_tma(nxt);
      } else {
        if (nxt < ntiles) stage_cols<W>(st_in, src_of(nxt), N, C);
        cp_async_commit();
      }
    } else {
#pragma unroll
      for (int m = 0; m < R; ++m)
        v[m] = vc ? col_get<false>(base + (size_t)(t + m * T) * C, C, c) : make_double2(0.0, 0.0);
    }
    fft_lane<N, R, G, false>(v, S.ex, t, g, S.tw);
    hartley_lane<N, R, G>(v, S.ex, t, g);
#pragma unroll
    for (int m = 0; m < R; ++m)
      if (vc) col_put<PF>(base + (size_t)(t + m * T) * C, C, c, v[m]);
  }
}

// t pass of the preconditioner: Hartley along t, divide by lambda_S (computed
// in registers from the 1-D eigenvalues, circulant.cpp:28-41, 76-90) and by
// N (circulant.cpp:62-64), Hartley along t again.
template <int N, bool PF>
__global__ void __launch_bounds__(Cfg<N>::THREADS, Cfg<N>::MINB) k_t_filter(double* data, PcTables pt, const int* guard,
                                                                              const __grid_constant__ CUtensorMap map) {
  using Cf = Cfg<N>;
  constexpr int R = Cf::R, T = Cf::T, G = Cf::G;
  constexpr int W = 2 * G;
  extern __shared__ __align__(128) double2 smem_raw[];
  Smem<N, Cf::DB> S(smem_raw, pt.tw_t, N);
  load_table(S.tab, pt.lam_t, N);
  pdl_trigger();
  pdl_wait();
  if (paused(guard)) return;
  const double2* lamt = S.tab;
  double* st_in = S.stage;
  const int g = threadIdx.x % G, t = threadIdx.x / G;
  const int C = pt.n1 * pt.n2;
  const int ntiles = (C + W - 1) / W;
  constexpr bool TMA = PF && FDG_TMA_PCOL;
  __shared__ alignas(8) unsigned long long bar;
  unsigned ph = 0;
  auto stage_tma = [&](int tl) {
    if constexpr (FDG_TMA_PCOL == 2) {
      if (threadIdx.x == 0) tma_cols<W>(st_in, &map, tl * W, 0, N, &bar);
    } else if (threadIdx.x < 32) {
      bulk_cols<W>(st_in, data + (size_t)tl * W, N, C, &bar);
    }
  };
  if constexpr (TMA) {
    if (threadIdx.x == 0) {
      mbar_init(&bar, 1);
      mbar_init_fence();
    }
    __syncthreads();
    if (blockIdx.x < ntiles) stage_tma(blockIdx.x);
  } else if constexpr (PF) {
    if (blockIdx.x < ntiles) stage_cols<W>(st_in, data + (size_t)blockIdx.x * W, N, C);
    cp_async_commit();
  }
  __syncthreads();
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long c = (long)(tile * G + g) * 2;
    const bool vc = PF || c < C;
    double2 v[R];
    if constexpr (PF) {
      if constexpr (TMA) {
        mbar_wait(&bar, ph);
        ph ^= 1;
      } else {
        cp_async_wait<0>();
        __syncthreads();
      }
#pragma unroll
      for (int m = 0; m < R; ++m) v[m] = *reinterpret_cast<const double2*>(st_in + (t + m * T) * W + 2 * g);
      __syncthreads();
      const int nxt = tile + gridDim.x;
      if constexpr (TMA) {
        if (nxt < ntiles) stage_tma(nxt);
      } else {
        if (nxt < ntiles) stage_cols<W>(st_in, data + (size_t)nxt * W, N, C);
        cp_async_commit();
      }
    } else {
#pragma unroll
      for (int m = 0; m < R; ++m)
        v[m] = vc ? col_get<false>(data + (size_t)(t + m * T) * C + c, C, c) : make_double2(0.0, 0.0);
    }
    // the inverse transform could reuse the forward one's per-thread twiddles
    // (TwCache), but the cache pushes this kernel over its 168-register bound
    // (measured: spills, no gain), so it is off here
    constexpr int TCM = 0;
    double2 wc[TwCache<N, R>::K];
    fft_lane_c<N, R, G, false, 0, TCM>(v, S.ex, t, g, S.tw, wc);
    // Z = A + iB (spectra of the two packed real columns a, b).  The filters
    // d_a, d_b are real and even in k, so with Zc = conj(Z[N - k]) = A - iB
    //   Y = d_a A + i d_b B = (d_a + d_b)/2 Z + (d_a - d_b)/2 Zc
    // and the inverse transform returns the filtered columns packed the same
    // way: one mirror exchange instead of two Hartley splits.
    if (S.ex.single()) lane_sync<0, T, G>(g);
    double2* smz = S.ex.next();
#pragma unroll
    for (int m = 0; m < R; ++m) smz[mslot<0, N, G>(t + m * T, g)] = v[m];
    lane_sync<0, T, G>(g);
    // spatial eigenvalue sums of the two packed columns
    double2 sa = make_double2(0.0, 0.0), sb = make_double2(0.0, 0.0);
    if (vc) {
      const int i = (int)(c / pt.n2), j = (int)(c - (long)i * pt.n2);
      const double2 l1 = __ldg(&pt.lam_1[i]), l2 = __ldg(&pt.lam_2[j]);
      sa = make_double2(l1.x + l2.x, l1.y + l2.y);
      if (PF || c + 1 < C) {
        const int i2 = (int)((c + 1) / pt.n2), j2 = (int)(c + 1 - (long)i2 * pt.n2);
        const double2 m1 = __ldg(&pt.lam_1[i2]), m2 = __ldg(&pt.lam_2[j2]);
        sb = make_double2(m1.x + m2.x, m1.y + m2.y);
      }
    }
#pragma unroll
    for (int m = 0; m < R; ++m) {
      const int k = t + m * T;
      const double2 h = v[m];
      const double2 lt = lamt[k];
      const double bax = pt.psi * (lt.x - sa.x), bay = pt.psi * (lt.y - sa.y);
      const double bbx = pt.psi * (lt.x - sb.x), bby = pt.psi * (lt.y - sb.y);
      const double lsa = pt.base + (bax * bax + bay * bay) * pt.inv_m2;
      const double lsb = pt.base + (bbx * bbx + bby * bby) * pt.inv_m2;
      // one reciprocal for both columns
      const double inv = 0.5 * pt.inv_total * frcp(lsa * lsb);
      const double da = lsb * inv, db = lsa * inv;  // d_a / 2, d_b / 2
      const double ds = da + db, dd = da - db;
      const double2 zc = smz[mslot<0, N, G>((N - k) & (N - 1), g)];
      v[m] = make_double2(fma(dd, zc.x, ds * h.x), fma(-dd, zc.y, ds * h.y));
    }
    fft_lane_c<N, R, G, true, 0, 2 * TCM>(v, S.ex, t, g, S.tw, wc);
#pragma unroll
    for (int m = 0; m < R; ++m)
      if (vc) col_put<PF>(data + (size_t)(t + m * T) * C + c, C, c, v[m]);
  }
}

}  // namespace fdg
