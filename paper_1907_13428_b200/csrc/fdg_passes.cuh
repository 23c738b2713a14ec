// fdg_passes.cuh — the FFT passes of the hot path (persistent CTAs).
//
// Every pass is one kernel over "tiles" of 2G fibres (two real fibres packed
// as one complex FFT lane, G lanes per CTA).  CTAs are persistent (grid =
// resident CTAs), stage the per-axis twiddle table and Toeplitz symbol in
// shared memory once, and loop over tiles.  FULL = the tile needs no bounds
// predicates (n == L/2 for Toeplitz embeddings, tile fully inside the array).
//
// Reference: ConstraintOperator::apply_mode (toeplitz.cpp:124-172) — pack,
// r2c, x symbol, c2r, unpack-accumulate — is one register-resident
// load -> FFT -> x symbol -> IFFT -> epilogue here, with the zero padding and
// the truncation to n taken from registers (no packed workspace in HBM).
#pragma once

#include <cuda_runtime.h>

#include "fdg_fft.cuh"
#include "fdg_internal.h"
#include "fdg_reduce.cuh"

namespace fdg {

// Tile configuration for transform length L.
//   R: complex values per thread, T = L/R threads per lane, G lanes per CTA
//   (256 threads), DB: double-buffered exchanges, TS: tables in smem.
template <int L>
struct Cfg {
  static constexpr int R = fft_radix(L);
  static constexpr int T = L / R;
  static constexpr int G_ = 256 / T;
  static constexpr int G = G_ > 32 ? 32 : (G_ < 2 ? 2 : G_);
  static constexpr int THREADS = G * T;
  static constexpr int MINB = 2;
  static constexpr bool DB = L <= 512;
  static constexpr bool TS = L <= 1024;
  static constexpr size_t EXB = (size_t)L * G;  // double2 per exchange buffer
  // exchange buffer(s) + twiddle table + symbol table
  static constexpr size_t SMEM = sizeof(double2) * (EXB * (DB ? 2 : 1) + (TS ? 2 * (size_t)L : 0));
};

template <int L, bool DB = Cfg<L>::DB>
struct Smem {
  Ex ex;
  const double2* tw;
  const double2* sym;
  double* stage;  // first byte after the tables (staging area, if any)
  __device__ __forceinline__ Smem(double2* base, const double2* gtw, const double2* gsym) {
    using C = Cfg<L>;
    ex.buf0 = base;
    ex.buf1 = DB ? base + C::EXB : base;
    ex.k = 0;
    double2* t = base + C::EXB * (DB ? 2 : 1);
    if constexpr (C::TS) {
      load_table(t, gtw, L);
      tw = t;
      if (gsym) {
        load_table(t + L, gsym, L);
        sym = t + L;
      } else {
        sym = nullptr;
      }
      stage = reinterpret_cast<double*>(t + 2 * L);
      __syncthreads();
    } else {
      tw = gtw;
      sym = gsym;
      stage = reinterpret_cast<double*>(t);
    }
  }
};

// cp.async (LDGSTS) helpers: 16-byte global -> shared copies that complete in
// the background while the FFT runs.
__device__ __forceinline__ void cp_async16(void* dst_smem, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst_smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }
// CTA-cooperative contiguous copy of `nd` doubles (nd even, 16-byte aligned).
__device__ __forceinline__ void stage_copy(double* dst, const double* src, int nd) {
  for (int i = 2 * threadIdx.x; i < nd; i += 2 * blockDim.x) cp_async16(dst + i, src + i);
}

__device__ __forceinline__ size_t idx2(size_t a, size_t b, size_t n) { return a * n + b; }

// =================================================================== rows
// Row pass along x2 (contiguous fibres of length n; embedding length L).
//   MODE 0 (apply):  out = psi*time(x) + scale * T2 x
//   MODE 1 (S out):  q = vp + psi*time^T(x) + scale * T2 x; q_out = q (opt);
//                    r -= (num/den) q; reduce |r|^2
struct RowArgs {
  const double* x;
  const double* vp;
  double* out;
  double* q_out;
  double* r;
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
};

// Row kernel variants: STAGE = full tiles (n == L/2, tiles of 2G fibres
// inside one time slice) whose epilogue operands (time-stencil neighbour row,
// vp, r) are copied to shared memory by cp.async at tile start and arrive
// during the FFTs.  The stencil diagonal psi c0 x_k is folded into the x2
// symbol on the host, so only the neighbour term psi c1 x_{k-+1} remains.
template <int L, int MODE, bool STAGE>
struct RowCfg {
  using C = Cfg<L>;
  static constexpr int NSTAGE = STAGE ? (MODE == 1 ? 3 : 1) : 0;
  static constexpr bool DB = C::DB && !(STAGE && MODE == 1);
  static constexpr size_t SMEM = sizeof(double2) * (C::EXB * (DB ? 2 : 1) + (C::TS ? 2 * (size_t)L : 0)) +
                                 sizeof(double) * (size_t)NSTAGE * 2 * C::G * (L / 2);
};

template <int L, int MODE, bool STAGE>
__global__ void __launch_bounds__(Cfg<L>::THREADS, Cfg<L>::MINB) k_row(RowArgs a) {
  using C = Cfg<L>;
  using RC = RowCfg<L, MODE, STAGE>;
  constexpr int R = C::R, T = C::T, G = C::G, H = (R + 1) / 2;
  constexpr bool FULL = STAGE;
  constexpr int TILE = 2 * G * (L / 2);  // doubles per staged operand
  extern __shared__ double2 smem_raw[];
  __shared__ double scratch[32];
  Smem<L, RC::DB> S(smem_raw, a.tw, a.sym);
  double* st_nb = S.stage;
  double* st_vp = S.stage + TILE;
  double* st_r = S.stage + 2 * TILE;
  const int g = threadIdx.x / T, t = threadIdx.x % T;  // lane-major: coalesced rows
  const int F = a.nt * a.n1;
  const int ntiles = (F + 2 * G - 1) / (2 * G);
  const int n = a.n;
  double alpha = 0.0;
  if constexpr (MODE == 1) {
    if (a.r) alpha = *a.a_num / *a.a_den;
  }
  const ptrdiff_t noff = (ptrdiff_t)a.tdir * a.n1 * n;
  double acc = 0.0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int f0 = tile * 2 * G;
    const int f = f0 + 2 * g;
    const bool va = FULL || f < F, vb = FULL || f + 1 < F;
    const double* xa = a.x + (size_t)f * n;
    bool tile_nb = false;
    if constexpr (STAGE) {
      const int k = f0 / a.n1;  // whole tile in one slice
      tile_nb = a.tkind == 1 && (a.tdir < 0 ? k >= 1 : k + 1 < a.nt);
      if (tile_nb) stage_copy(st_nb, a.x + (size_t)f0 * n + noff, TILE);
      if constexpr (MODE == 1) {
        stage_copy(st_vp, a.vp + (size_t)f0 * n, TILE);
        if (a.r) stage_copy(st_r, a.r + (size_t)f0 * n, TILE);
      }
      cp_async_commit();
    }
    double2 v[R];
#pragma unroll
    for (int m = 0; m < R; ++m) {
      const int pos = t + m * T;
      double2 z = make_double2(0.0, 0.0);
      if (m < H && (FULL || pos < n)) {
        if (va) z.x = __ldg(xa + pos);
        if (vb) z.y = __ldg(xa + n + pos);
      }
      v[m] = z;
    }
    fft_lane<L, R, G, false, 1>(v, S.ex, t, g, S.tw);
#pragma unroll
    for (int m = 0; m < R; ++m) v[m] = cmul(v[m], S.sym[t + m * T]);
    fft_lane<L, R, G, true, 1>(v, S.ex, t, g, S.tw);

    if constexpr (STAGE) {
      cp_async_wait_all();
      __syncthreads();
    }
    // generic path: per-fibre neighbour predicates
    const int ka = f / a.n1, kb = (f + 1) / a.n1;
    const bool nba = a.tkind == 1 && (a.tdir < 0 ? ka >= 1 : ka + 1 < a.nt);
    const bool nbb = a.tkind == 1 && (a.tdir < 0 ? kb >= 1 : kb + 1 < a.nt);
#pragma unroll
    for (int m = 0; m < H; ++m) {
      const int pos = t + m * T;
      if (!FULL && pos >= n) continue;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (!FULL && !(h ? vb : va)) continue;
        const int sl = (2 * g + h) * n + pos;  // staged element (STAGE)
        double val = a.scale * (h ? v[m].y : v[m].x);
        if constexpr (STAGE) {
          if (tile_nb) val += a.tc1 * st_nb[sl];
        } else {
          if (h ? nbb : nba) val += a.tc1 * __ldg(xa + h * n + pos + noff);
        }
        const size_t o = (size_t)(f + h) * n + pos;
        if constexpr (MODE == 0) {
          a.out[o] = val;
        } else {
          const double q = (STAGE ? st_vp[sl] : __ldg(&a.vp[o])) + val;
          if (a.q_out) a.q_out[o] = q;
          if (a.r) {
            const double rn = (STAGE ? st_r[sl] : a.r[o]) - alpha * q;
            a.r[o] = rn;
            acc += rn * rn;
          }
        }
      }
    }
    if constexpr (STAGE) __syncthreads();  // staging is rewritten by the next tile
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

template <int L, int MODE, bool FULL>
__global__ void __launch_bounds__(Cfg<L>::THREADS, Cfg<L>::MINB) k_col(ColArgs a) {
  using Cf = Cfg<L>;
  constexpr int R = Cf::R, T = Cf::T, G = Cf::G, H = (R + 1) / 2;
  extern __shared__ double2 smem_raw[];
  __shared__ double scratch[32];
  Smem<L> S(smem_raw, a.tw, a.sym);
  const int g = threadIdx.x % G, t = threadIdx.x / G;
  const int n = a.n, C = a.C;
  const int ncb = (C + 2 * G - 1) / (2 * G);
  const int ntiles = ncb * a.O;
  double e = 0.0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int o = tile / ncb;
    const long c = (long)((tile - o * ncb) * G + g) * 2;
    const bool vc = FULL || c < C;
    const size_t base = (size_t)o * n * C + c;
    double2 v[R];
#pragma unroll
    for (int m = 0; m < R; ++m) {
      const int pos = t + m * T;
      v[m] = (m < H && (FULL || pos < n) && vc) ? col_get<FULL>(a.x + base + (size_t)pos * C, C, c)
                                                 : make_double2(0.0, 0.0);
    }
    fft_lane<L, R, G, false>(v, S.ex, t, g, S.tw);
#pragma unroll
    for (int m = 0; m < R; ++m) v[m] = cmul(v[m], S.sym[t + m * T]);
    fft_lane<L, R, G, true>(v, S.ex, t, g, S.tw);

    if constexpr (MODE == 0) {
#pragma unroll
      for (int m = 0; m < H; ++m) {
        const int pos = t + m * T;
        if (!FULL && (pos >= n || !vc)) continue;
        const size_t o2 = base + (size_t)pos * C;
        double2 acc = make_double2(0.0, 0.0);
        if (a.acc) acc = col_get<FULL>(a.acc + o2, C, c);
        col_put<FULL>(a.out + o2, C, c, make_double2(acc.x + a.scale * v[m].x, acc.y + a.scale * v[m].y));
      }
    } else {
      // S mid pass: u is a.acc, w -> a.w, vp -> a.out
      const double im2 = a.inv_m2[o], a1 = a.a1[o];
      const bool vb = FULL || c + 1 < C;
#pragma unroll
      for (int m = 0; m < R; ++m) {
        const int pos = t + m * T;
        if (m < H && (FULL || (pos < n && vc))) {
          const size_t o2 = base + (size_t)pos * C;
          const double2 u = col_get<FULL>(a.acc + o2, C, c);
          const double2 pv = col_get<FULL>(a.x + o2, C, c);
          const double bx = u.x + a.scale * v[m].x;
          const double by = u.y + a.scale * v[m].y;
          const double wx = bx * im2, wy = vb ? by * im2 : 0.0;
          e += a1 * pv.x * pv.x + wx * bx;
          if (vb) e += a1 * pv.y * pv.y + wy * by;
          col_put<FULL>(a.w + o2, C, c, make_double2(wx, wy));
          v[m] = make_double2(wx, wy);
        } else {
          v[m] = make_double2(0.0, 0.0);
        }
      }
      fft_lane<L, R, G, false>(v, S.ex, t, g, S.tw);
#pragma unroll
      for (int m = 0; m < R; ++m) v[m] = cmul(v[m], S.sym[t + m * T]);
      fft_lane<L, R, G, true>(v, S.ex, t, g, S.tw);
#pragma unroll
      for (int m = 0; m < H; ++m) {
        const int pos = t + m * T;
        if (!FULL && (pos >= n || !vc)) continue;
        const size_t o2 = base + (size_t)pos * C;
        const double2 pv = col_get<FULL>(a.x + o2, C, c);
        col_put<FULL>(a.out + o2, C, c, make_double2(a.scale * v[m].x + a1 * pv.x, a.scale * v[m].y + a1 * pv.y));
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
template <int N, bool FULL>
__global__ void __launch_bounds__(Cfg<N>::THREADS, Cfg<N>::MINB)
    k_hartley_row(const double* in, double* out, int F, const double2* tw, const double* rdot, RedSlot red) {
  using Cf = Cfg<N>;
  constexpr int R = Cf::R, T = Cf::T, G = Cf::G;
  extern __shared__ double2 smem_raw[];
  __shared__ double scratch[32];
  Smem<N> S(smem_raw, tw, nullptr);
  const int g = threadIdx.x / T, t = threadIdx.x % T;  // lane-major: coalesced rows
  const int ntiles = (F + 2 * G - 1) / (2 * G);
  double acc = 0.0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int f = (tile * G + g) * 2;
    const bool va = FULL || f < F, vb = FULL || f + 1 < F;
    const size_t ia = (size_t)f * N, ib = ia + N;
    double2 v[R], w[R];
#pragma unroll
    for (int m = 0; m < R; ++m) {
      const int pos = t + m * T;
      v[m].x = va ? __ldg(&in[ia + pos]) : 0.0;
      v[m].y = vb ? __ldg(&in[ib + pos]) : 0.0;
    }
    fft_lane<N, R, G, false, 1>(v, S.ex, t, g, S.tw);
    mirror_lane<N, R, G, 1>(v, w, S.ex, t, g);
#pragma unroll
    for (int m = 0; m < R; ++m) {
      const int pos = t + m * T;
      const double2 h = hartley_split(v[m], w[m]);
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

template <int N, bool FULL>
__global__ void __launch_bounds__(Cfg<N>::THREADS, Cfg<N>::MINB)
    k_hartley_col(double* data, int O, int C, const double2* tw) {
  using Cf = Cfg<N>;
  constexpr int R = Cf::R, T = Cf::T, G = Cf::G;
  extern __shared__ double2 smem_raw[];
  Smem<N> S(smem_raw, tw, nullptr);
  const int g = threadIdx.x % G, t = threadIdx.x / G;
  const int ncb = (C + 2 * G - 1) / (2 * G);
  const int ntiles = ncb * O;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int o = tile / ncb;
    const long c = (long)((tile - o * ncb) * G + g) * 2;
    const bool vc = FULL || c < C;
    double* base = data + (size_t)o * N * C + c;
    double2 v[R], w[R];
#pragma unroll
    for (int m = 0; m < R; ++m)
      v[m] = vc ? col_get<FULL>(base + (size_t)(t + m * T) * C, C, c) : make_double2(0.0, 0.0);
    fft_lane<N, R, G, false>(v, S.ex, t, g, S.tw);
    mirror_lane<N, R, G>(v, w, S.ex, t, g);
#pragma unroll
    for (int m = 0; m < R; ++m)
      if (vc) col_put<FULL>(base + (size_t)(t + m * T) * C, C, c, hartley_split(v[m], w[m]));
  }
}

// t pass of the preconditioner: Hartley along t, divide by lambda_S (computed
// in registers from the 1-D eigenvalues, circulant.cpp:28-41, 76-90) and by
// N (circulant.cpp:62-64), Hartley along t again.
template <int N, bool FULL>
__global__ void __launch_bounds__(Cfg<N>::THREADS, Cfg<N>::MINB) k_t_filter(double* data, PcTables pt) {
  using Cf = Cfg<N>;
  constexpr int R = Cf::R, T = Cf::T, G = Cf::G;
  extern __shared__ double2 smem_raw[];
  Smem<N> S(smem_raw, pt.tw_t, pt.lam_t);  // the "symbol" slot holds lambda_t
  const int g = threadIdx.x % G, t = threadIdx.x / G;
  const int C = pt.n1 * pt.n2;
  const int ntiles = (C + 2 * G - 1) / (2 * G);
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long c = (long)(tile * G + g) * 2;
    const bool vc = FULL || c < C;
    double2 v[R], w[R];
#pragma unroll
    for (int m = 0; m < R; ++m)
      v[m] = vc ? col_get<FULL>(data + (size_t)(t + m * T) * C + c, C, c) : make_double2(0.0, 0.0);
    fft_lane<N, R, G, false>(v, S.ex, t, g, S.tw);
    mirror_lane<N, R, G>(v, w, S.ex, t, g);
    // spatial eigenvalue sums of the two packed columns
    double2 sa = make_double2(0.0, 0.0), sb = make_double2(0.0, 0.0);
    if (vc) {
      const int i = (int)(c / pt.n2), j = (int)(c - (long)i * pt.n2);
      const double2 l1 = __ldg(&pt.lam_1[i]), l2 = __ldg(&pt.lam_2[j]);
      sa = make_double2(l1.x + l2.x, l1.y + l2.y);
      if (FULL || c + 1 < C) {
        const int i2 = (int)((c + 1) / pt.n2), j2 = (int)(c + 1 - (long)i2 * pt.n2);
        const double2 m1 = __ldg(&pt.lam_1[i2]), m2 = __ldg(&pt.lam_2[j2]);
        sb = make_double2(m1.x + m2.x, m1.y + m2.y);
      }
    }
#pragma unroll
    for (int m = 0; m < R; ++m) {
      const int k = t + m * T;
      const double2 h = hartley_split(v[m], w[m]);
      const double2 lt = S.sym[k];
      const double bax = pt.psi * (lt.x - sa.x), bay = pt.psi * (lt.y - sa.y);
      const double bbx = pt.psi * (lt.x - sb.x), bby = pt.psi * (lt.y - sb.y);
      const double lsa = pt.base + (bax * bax + bay * bay) * pt.inv_m2;
      const double lsb = pt.base + (bbx * bbx + bby * bby) * pt.inv_m2;
      // one reciprocal for both columns
      const double inv = pt.inv_total / (lsa * lsb);
      v[m] = make_double2(h.x * (lsb * inv), h.y * (lsa * inv));
    }
    fft_lane<N, R, G, false>(v, S.ex, t, g, S.tw);
    mirror_lane<N, R, G>(v, w, S.ex, t, g);
#pragma unroll
    for (int m = 0; m < R; ++m)
      if (vc) col_put<FULL>(data + (size_t)(t + m * T) * C + c, C, c, hartley_split(v[m], w[m]));
  }
}

}  // namespace fdg
