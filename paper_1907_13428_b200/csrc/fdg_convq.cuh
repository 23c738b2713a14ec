// fdg_convq.cuh — Q-way split-spectrum Toeplitz convolution passes for the
// embedding lengths L = 256 Q, Q = 4, 8 (n = L/2 = 512, 1024: BASELINE C3, C4).
//
// Same operator as k_rowc / k_colc (fdg_conv.cuh; reference
// ConstraintOperator::apply_mode, toeplitz.cpp:124-172).  The input is zero
// beyond n = L/2 and only n outputs are kept, so the length-L transform pair
// splits into Q independent 256-point pairs, one per residue c of the
// frequency index mod Q:
//   X[Q k + c] = DFT_256( W_L^{j c} sum_{b < Q/2} W_Q^{b c} z[j + 256 b] )[k]
//   y[j + 256 b] = sum_c W_Q^{-b c} W_L^{-j c} IDFT_256(s_c X_c)[j]   (j < 256)
// with s_c[k] = sym[Q k + c].  Every transform is the 256-point radix-16
// plan of the L = 512 passes (one exchange, per-thread twiddle cache), so the
// FFT work per element equals the L = 512 passes'; the input combination
// and the Q-term output combination (factors W_Q^m: +-1, +-i, W_8) are the
// extra.  A lane (two real fibres packed as a + i b) is served by Q
// sub-lanes of 16 threads; sub-lane c owns the outputs j = t + 16 m + 256 (c/2)
// for the 8 m of half (c & 1).
#pragma once

#include <cuda_runtime.h>

#include "fdg_conv.cuh"
#include "fdg_fft.cuh"
#include "fdg_passes.cuh"
#include "fdg_reduce.cuh"

namespace fdg {

template <int L, bool ROWS>
struct QCfg {
  static constexpr int Q = L >= 1024 ? L / 256 : 4;  // sub-lanes per lane (other L: unused)
  static constexpr int NB = Q / 2;   // 256-blocks of the zero-padded input
  static constexpr int N = L / 2;    // fibre length n
  static constexpr int R = 16, T = 16, HR = 8;
  static constexpr int LT = Q * T;  // threads per lane
  static constexpr int THREADS = ROWS ? 128 : 256;
  static constexpr int G = THREADS / LT < 1 ? 1 : THREADS / LT;  // lanes per CTA
  static constexpr int GQ = G * Q;                               // sub-lanes per CTA
  static constexpr size_t EXB = (size_t)256 * GQ;                // double2
  // real symbol in shared memory up to L = 1024 (else read through L1)
  static constexpr bool SYMS = L <= 1024;
  static constexpr bool OK = (Q == 4 || Q == 8) && G * LT == THREADS;
  static constexpr size_t bytes(size_t stage_doubles) {
    return sizeof(double2) * (EXB + 256 + L / 16) + (SYMS ? sizeof(double) * L : 0) +
           sizeof(double) * stage_doubles;
  }
};

// W_Q^k = exp(-2 pi i k / Q) for the runtime residue k (Q = 4, 8), by
// selects (no local-memory table).
template <int Q>
__device__ __forceinline__ double2 wq_const(int k) {
  constexpr double H = 0.70710678118654752440;
  k &= Q - 1;
  const int k4 = Q == 4 ? k : k >> 1;  // quarter-turn count
  const bool odd = Q == 8 && (k & 1);  // extra eighth turn
  // base quarter rotation of (1, 0) by -k4 * 90 degrees
  double cr = k4 == 0 ? 1.0 : (k4 == 2 ? -1.0 : 0.0);
  double ci = k4 == 1 ? -1.0 : (k4 == 3 ? 1.0 : 0.0);
  if (odd) {  // times W_8 = (1 - i)/sqrt(2)
    const double r = H * (cr + ci), im = H * (ci - cr);
    cr = r;
    ci = im;
  }
  return make_double2(cr, ci);
}

// y = sum_c W_Q^{-BO c} u[c] with compile-time factors.
template <int Q, int BO, int CI = 0>
__device__ __forceinline__ double2 qsum(const double2 (&u)[Q]) {
  if constexpr (CI == Q) {
    return make_double2(0.0, 0.0);
  } else {
    return cadd(mul_wq<Q, -BO * CI, false>(u[CI]), qsum<Q, BO, CI + 1>(u));
  }
}
template <int Q>
__device__ __forceinline__ double2 qsum_rt(const double2 (&u)[Q], int bo) {
  if constexpr (Q == 4) {
    return bo == 0 ? qsum<4, 0>(u) : qsum<4, 1>(u);
  } else {
    switch (bo) {
      case 0: return qsum<8, 0>(u);
      case 1: return qsum<8, 1>(u);
      case 2: return qsum<8, 2>(u);
      default: return qsum<8, 3>(u);
    }
  }
}

// Sub-lane c's 256-point convolution in place on v (input: the combined,
// untwisted u[t + 16 m]; output: W_L^{-j c} IDFT(s_c X_c)[t + 16 m]).
// The twist W_L^{(t + 16 m) c} = W_L^{t c} W_{L/16}^{m c} from one
// per-thread value (wtc) and a staged table of the L/16 values W_{L/16}^q
// (cw; c is uniform over a warp, so the read is a broadcast) instead of a
// load through L1 per element (the top stall of these passes).
template <int L, int LAYOUT, int GQ>
__device__ __forceinline__ void conv_q(double2 (&v)[16], Ex& ex, int t, int gs, int c, const double2* tw,
                                       const double2* twq, const double* sym, const double2* cw, double2 wtc) {
  constexpr int Q = L / 256;
  constexpr bool CACHE = FDG_TWCACHE != 0;
  // residue 0 has no twist (c is uniform over a warp)
  if (c != 0) {
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      v[m] = cmul(cmul(v[m], cw[(m * c) & (L / 16 - 1)]), wtc);
    }
  }
  double2 wc[TwCache<256, 16>::K];
  fft_lane_c<256, 16, GQ, false, LAYOUT, CACHE ? 1 : 0>(v, ex, t, gs, tw, wc);
  // staged symbol: de-interleaved by residue (s_c contiguous), so a sub-lane's
  // 16 threads read 16 consecutive doubles (the interleaved index Q k + c
  // is a 4-way bank conflict)
#pragma unroll
  for (int m = 0; m < 16; ++m)
    v[m] = cscale(v[m], sym[QCfg<L, true>::SYMS ? c * 256 + (t + 16 * m) : Q * (t + 16 * m) + c]);
  fft_lane_c<256, 16, GQ, true, LAYOUT, CACHE ? 2 : 0>(v, ex, t, gs, tw, wc);
  // W_L^{-j c} read as W_L^{L - j c}: distinct addresses from the forward
  // twist, so no 64-bit address stays live across the transforms
  if (c != 0) {
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      v[m] = cmulc(cmulc(v[m], cw[(m * c) & (L / 16 - 1)]), wtc);
    }
  }
}

template <int L, int MODE, bool SR>
struct RowQPlan {
  using C = QCfg<L, true>;
  static constexpr int TILE = 2 * C::G * C::N;  // doubles per staged operand
  static constexpr int NIN = MODE == 2 ? 2 : 1;
  static constexpr int NEPI = MODE == 0 ? 1 : (MODE == 1 ? 3 : 2);
  static constexpr size_t SMEM = C::bytes((size_t)TILE * (NIN + NEPI));
};

// Row pass along x2 for L = 1024, 2048 (full tiles: n = L/2, tiles of 2G
// rows inside one time slice), modes as k_rowc.  Real (symmetric-factor)
// symbols only (SR); lane-major exchange layout per sub-lane.
template <int L, int MODE>
__global__ void __launch_bounds__(QCfg<L, true>::THREADS, 2) k_rowq(RowArgs a) {
  using C = QCfg<L, true>;
  using RP = RowQPlan<L, MODE, true>;
  static_assert(C::OK, "Q-split row configuration");
  constexpr int Q = C::Q, NB = C::NB, n = C::N, G = C::G, GQ = C::GQ, HR = C::HR;
  constexpr int TILE = RP::TILE;
  extern __shared__ double2 smem_raw[];
  __shared__ double scratch[32];
  Ex ex;
  ex.buf0 = ex.buf1 = smem_raw;
  ex.k = 0;
  double2* tw = smem_raw + C::EXB;
  load_table(tw, a.tw256, 256);
  double2* cw = tw + 256;  // W_{L/16}^q = W_L^{16 q}
  for (int i = threadIdx.x; i < L / 16; i += blockDim.x) cw[i] = __ldg(&a.twq[16 * i]);
  const double* sym;
  double* stage;
  if constexpr (C::SYMS) {
    double* d = reinterpret_cast<double*>(tw + 256 + L / 16);
    for (int i = threadIdx.x; i < L; i += blockDim.x) d[(i % Q) * 256 + i / Q] = __ldg(&a.sym_re[i]);
    sym = d;
    stage = d + L;
  } else {
    sym = a.sym_re;
    stage = reinterpret_cast<double*>(tw + 256 + L / 16);
  }
  pdl_trigger();
  pdl_wait();
  if (paused(a.guard)) return;
  double* st_in = stage;
  double* st_in2 = stage + TILE;
  double* st_nb = stage + RP::NIN * TILE;
  double* st_nb2 = st_nb + TILE;
  double* st_vp = stage + 2 * TILE;
  double* st_r = stage + 3 * TILE;
  // thread -> (sub-lane c, lane g, t); warps hold one c (G = 2) or the
  // pair 2w, 2w + 1 (G = 1), whose output block c/2 agrees
  const int c = threadIdx.x / (G * 16), g = (threadIdx.x / 16) % G, t = threadIdx.x % 16;
  const int gs = c * G + g;
  const int bo = c >> 1, half = c & 1;
  const double2 wtc = __ldg(&a.twq[t * c]);  // W_L^{t c}
  const int F = a.nt * a.n1;
  const int ntiles = F / (2 * G);
  double2 win[NB];
#pragma unroll
  for (int bb = 0; bb < NB; ++bb) win[bb] = wq_const<Q>(bb * c);
  // Q = 4: z W_4^c = (rsx p, rsy q) with (p, q) = (z.x, z.y), swapped for odd c
  const double rsx = (c & 2) ? -1.0 : 1.0, rsy = (c == 1 || c == 2) ? -1.0 : 1.0;
  double alpha = 0.0, beta = 0.0;
  if constexpr (MODE == 1) {
    if (a.r) alpha = *a.a_num / *a.a_den;
  }
  if constexpr (MODE == 2) {
    if (a.upd_x) alpha = *a.a_num / *a.a_den;
    if (!a.first) beta = *a.b_num / *a.b_den;
  }
  const bool first = MODE == 2 && a.first;
  const double* in0 = MODE == 2 ? a.z : a.x;
  const double* in1 = a.dold;
  const ptrdiff_t noff = (ptrdiff_t)a.tdir * a.n1 * n;
  double acc = 0.0;
  auto own = [&](int i) { return t + 16 * (8 * half + i) + 256 * bo; };
  constexpr bool XPF = MODE == 2;
  constexpr bool PRE = MODE == 2;                   // direction update in a flat pre-pass over the tile
  constexpr int NPRE = TILE / 2 / C::THREADS;       // double2 per thread in the pre-pass
  static_assert(!PRE || (NPRE * 2 * C::THREADS == TILE && NPRE == HR), "pre-pass tiling");
  double2 xpre[XPF ? HR : 1];
  const bool upd_x = XPF && a.upd_x && !first;
  auto load_x = [&](int tl) {
    if constexpr (PRE) {
      const double2* gx = reinterpret_cast<const double2*>(a.xs + (size_t)tl * 2 * G * n);
#pragma unroll
      for (int k = 0; k < NPRE; ++k) xpre[k] = gx[threadIdx.x + k * C::THREADS];
    } else {
      const size_t rx = (size_t)(tl * 2 * G + 2 * g) * n;
#pragma unroll
      for (int i = 0; i < (XPF ? HR : 1); ++i) xpre[i] = make_double2(a.xs[rx + own(i)], a.xs[rx + n + own(i)]);
    }
  };
  // TMA staging (FDG_TMA_ROWS): barrier 0 = FFT input, 1 = epilogue operands
  constexpr bool TMA = FDG_TMA_ROWS;
  __shared__ alignas(8) unsigned long long bars[2];
  constexpr unsigned TB = sizeof(double) * TILE;
  unsigned ph_in = 0, ph_ep = 0;
  auto stage_in = [&](int tl) {  // elected thread
    fence_proxy_async();
    mbar_expect_tx(&bars[0], (MODE == 2 && !first) ? 2 * TB : TB);
    bulk_g2s(st_in, in0 + (size_t)tl * 2 * G * n, TB, &bars[0]);
    if (MODE == 2 && !first) bulk_g2s(st_in2, in1 + (size_t)tl * 2 * G * n, TB, &bars[0]);
  };
  if constexpr (TMA) {
    if (threadIdx.x == 0) {
      mbar_init(&bars[0], 1);
      mbar_init(&bars[1], 1);
      mbar_init_fence();
      if (blockIdx.x < ntiles) stage_in(blockIdx.x);
    }
    if (upd_x && blockIdx.x < ntiles) load_x(blockIdx.x);
  } else {
    if (blockIdx.x < ntiles) {
      stage_rows(st_in, in0 + (size_t)blockIdx.x * 2 * G * n, TILE);
      if (MODE == 2 && !first) stage_rows(st_in2, in1 + (size_t)blockIdx.x * 2 * G * n, TILE);
      if (upd_x) load_x(blockIdx.x);
    }
    cp_async_commit();
  }
  __syncthreads();  // tables (and the barriers' initialization)
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int f0 = tile * 2 * G;
    const size_t ra = (size_t)(f0 + 2 * g) * n;
    double2 v[16];
    if constexpr (TMA) {
      mbar_wait(&bars[0], ph_in);
      ph_in ^= 1;
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if constexpr (PRE) {
      // p = z + beta d_old once per element (not once per sub-lane), in place
      // in the staged tile; p and the x update leave as 16-byte stores
      double2* pz = reinterpret_cast<double2*>(st_in);
      const double2* pd = reinterpret_cast<const double2*>(st_in2);
      double2* gd = reinterpret_cast<double2*>(a.dnew + (size_t)f0 * n);
      double2* gx = reinterpret_cast<double2*>(a.xs + (size_t)f0 * n);
#pragma unroll
      for (int k = 0; k < NPRE; ++k) {
        const int idx = threadIdx.x + k * C::THREADS;
        double2 z = pz[idx];
        if (!first) {
          const double2 dd = pd[idx];
          z.x += beta * dd.x;
          z.y += beta * dd.y;
          pz[idx] = z;
          if (upd_x) gx[idx] = make_double2(xpre[k].x + alpha * dd.x, xpre[k].y + alpha * dd.y);
        }
        gd[idx] = z;
      }
      if (upd_x && tile + (int)gridDim.x < ntiles) load_x(tile + gridDim.x);
      __syncthreads();
    }
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      double2 u = make_double2(0.0, 0.0);
#pragma unroll
      for (int bb = 0; bb < NB; ++bb) {
        const int pos = t + 16 * m + 256 * bb;
        double2 z = make_double2(st_in[(2 * g) * n + pos], st_in[(2 * g + 1) * n + pos]);
        if constexpr (MODE == 2 && !PRE) {
          double2 dd = make_double2(0.0, 0.0);
          if (!first) {
            dd = make_double2(st_in2[(2 * g) * n + pos], st_in2[(2 * g + 1) * n + pos]);
            z.x += beta * dd.x;
            z.y += beta * dd.y;
          }
          if (bb == bo && (m >= 8) == (half == 1)) {  // owned position
            a.dnew[ra + pos] = z.x;
            a.dnew[ra + n + pos] = z.y;
            if (upd_x) {
              const int i = m & 7;
              a.xs[ra + pos] = xpre[i].x + alpha * dd.x;
              a.xs[ra + n + pos] = xpre[i].y + alpha * dd.y;
            }
          }
        }
        if constexpr (Q == 4) {
          // W_4^c: a quarter-turn count, by one swap and two signed adds
          if (bb == 0) {
            u = z;
          } else {
            const double p = (c & 1) ? z.y : z.x, q = (c & 1) ? z.x : z.y;
            u = make_double2(fma(rsx, p, u.x), fma(rsy, q, u.y));
          }
        } else {
          u = bb == 0 ? z : cadd(u, cmul(z, win[bb]));
        }
      }
      v[m] = u;
    }
    if constexpr (XPF && !PRE) {
      if (upd_x && tile + (int)gridDim.x < ntiles) load_x(tile + gridDim.x);
    }
    __syncthreads();  // st_in and the epilogue staging are free
    const int k = f0 / a.n1;
    const bool tile_nb = a.tkind == 1 && (a.tdir < 0 ? k >= 1 : k + 1 < a.nt);
    const int nxt = tile + gridDim.x;
    bool ep_armed = false;
    if constexpr (TMA) {
      unsigned eb = 0;
      if (tile_nb) eb += (MODE == 2 && !first) ? 2 * TB : TB;
      if constexpr (MODE == 1) eb += a.r ? 2 * TB : TB;
      ep_armed = eb != 0;
      if (threadIdx.x == 0) {
        fence_proxy_async();
        if (ep_armed) {
          mbar_expect_tx(&bars[1], eb);
          if (tile_nb) {
            bulk_g2s(st_nb, in0 + (size_t)f0 * n + noff, TB, &bars[1]);
            if (MODE == 2 && !first) bulk_g2s(st_nb2, in1 + (size_t)f0 * n + noff, TB, &bars[1]);
          }
          if constexpr (MODE == 1) {
            bulk_g2s(st_vp, a.vp + (size_t)f0 * n, TB, &bars[1]);
            if (a.r) bulk_g2s(st_r, (a.r_in ? a.r_in : a.r) + (size_t)f0 * n, TB, &bars[1]);
          }
        }
        if (nxt < ntiles) stage_in(nxt);
      }
    } else {
      if (tile_nb) {
        stage_rows(st_nb, in0 + (size_t)f0 * n + noff, TILE);
        if (MODE == 2 && !first) stage_rows(st_nb2, in1 + (size_t)f0 * n + noff, TILE);
      }
      if constexpr (MODE == 1) {
        stage_rows(st_vp, a.vp + (size_t)f0 * n, TILE);
        if (a.r) stage_rows(st_r, (a.r_in ? a.r_in : a.r) + (size_t)f0 * n, TILE);
      }
      cp_async_commit();  // group E
      if (nxt < ntiles) {
        stage_rows(st_in, in0 + (size_t)nxt * 2 * G * n, TILE);
        if (MODE == 2 && !first) stage_rows(st_in2, in1 + (size_t)nxt * 2 * G * n, TILE);
      }
      cp_async_commit();  // group I
    }
    conv_q<L, 1, GQ>(v, ex, t, gs, c, tw, a.twq, sym, cw, wtc);
    // combine across the lane's Q sub-lanes
    __syncwarp();
    double2* sm = ex.next();
#pragma unroll
    for (int m = 0; m < 16; ++m) sm[slot<1, 256, GQ>(t + 16 * m, gs)] = v[m];
    if constexpr (TMA) {
      if (ep_armed) {
        mbar_wait(&bars[1], ph_ep);
        ph_ep ^= 1;
      }
    } else {
      cp_async_wait<1>();
    }
    __syncthreads();
    double2 y[HR];
#pragma unroll
    for (int i = 0; i < HR; ++i) {
      double2 u[Q];
      // the sub-lane's own term is still in registers (c is uniform over a warp)
      const double2 mine = half ? v[i + 8] : v[i];
#pragma unroll
      for (int cc = 0; cc < Q; ++cc) {
        if (cc != c) u[cc] = sm[slot<1, 256, GQ>(t + 16 * (8 * half + i), cc * G + g)];
        else u[cc] = mine;
      }
      y[i] = qsum_rt<Q>(u, bo);
    }
#pragma unroll
    for (int i = 0; i < HR; ++i) {
      const int pos = own(i);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int sl = (2 * g + h) * n + pos;
        const size_t o = ra + h * n + pos;
        double val = a.scale * (h ? y[i].y : y[i].x);
        if (tile_nb) {
          double nbv = st_nb[sl];
          if (MODE == 2 && !first) nbv += beta * st_nb2[sl];
          val += a.tc1 * nbv;
        }
        if constexpr (MODE == 0 || MODE == 2) {
          a.out[o] = val;
        } else {
          const double q = st_vp[sl] + val;
          if (a.q_out) a.q_out[o] = q;
          if (a.r) {
            const double rn = st_r[sl] - alpha * q;
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

}  // namespace fdg
