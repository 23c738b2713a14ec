// fdg_conv.cuh — split-spectrum Toeplitz convolution passes (row and column).
//
// Same operator as the k_row / k_col passes of fdg_passes.cuh (reference:
// ConstraintOperator::apply_mode, toeplitz.cpp:124-172): a Toeplitz matvec of
// size n <= M = L/2 through its length-L circulant embedding.  Because the
// input is zero beyond M and only the first M outputs are kept, the length-L
// transform pair splits into two independent M-point pairs:
//   X[2k]   = DFT_M(z)[k]                 X[2k+1] = DFT_M(z . W_L^j)[k]
//   y[j]    = IDFT_M(s_e X_e)[j] + W_L^-j IDFT_M(s_o X_o)[j]      (j < M)
// (s_e[k] = sym[2k], s_o[k] = sym[2k+1]).  A lane (two real fibres packed as
// z = a + ib) is served by two sub-lanes of T = M/R threads that run the
// even and the odd half at the same time, then one exchange adds the halves;
// each sub-lane thread ends up owning R/2 output positions.
//
// For L = 512 (M = 256, R = 16) an M-point transform needs ONE shared-memory
// exchange, so a convolution moves 5 x 256 values per sub-lane pair through
// shared memory instead of 4 x 512 for the direct 512-point pair.
//
// Thread mapping (HOMO = 1): the first half of a CTA's threads are the even
// sub-lanes of its G lanes, the second half the odd ones, so warps never
// diverge on the odd half's twist multiplies W_L^{+-j}.
#pragma once

#include <cuda_runtime.h>

#include "fdg_fft.cuh"
#include "fdg_passes.cuh"
#include "fdg_reduce.cuh"

namespace fdg {


#ifndef FDG_C512_THREADS
#define FDG_C512_THREADS 128
#endif
#ifndef FDG_C512_MINB_ROW
#define FDG_C512_MINB_ROW 2
#endif
#ifndef FDG_C512_MINB_COL
#define FDG_C512_MINB_COL 2
#endif
#ifndef FDG_C1024_THREADS
#define FDG_C1024_THREADS 256
#endif
#ifndef FDG_C1024_MINB_COL
#define FDG_C1024_MINB_COL 1
#endif
#ifndef FDG_C_HOMO
#define FDG_C_HOMO 1
#endif
#ifndef FDG_C_HOMO_COL
#define FDG_C_HOMO_COL FDG_C_HOMO
#endif
#ifndef FDG_C_EPI
#define FDG_C_EPI 1
#endif
#ifndef FDG_C_COLLY
#define FDG_C_COLLY 2
#endif
#ifndef FDG_TMA_ROWS
#define FDG_TMA_ROWS 1  // staged split row passes: bulk-copy (TMA) staging with mbarriers
#endif
#ifndef FDG_TMA_COLS
#define FDG_TMA_COLS 2  // staged split column passes: 2 = 2-D tensor-map TMA boxes, 1 = one bulk copy per
                        // row segment (C2 K2 237 -> 555 us), 0 = per-thread cp.async
#endif
#ifndef FDG_K2_EREG
#define FDG_K2_EREG 1  // S-mid column pass: a1 p^T p from the input registers
#endif

// Twist factors W_L^(t + T m) = W_L^t W_32^m (T = L/32 at R = 16) formed as a
// compile-time constant multiply times one per-thread value instead of a table
// load per element, where the table is not in shared memory (M = 1024: loads
// through L1).  Where the table is staged the loads win (C2 K2 223 -> 235 us
// with the constants), and at M = 1024 both the pre-twist and the combine
// need the constants (either alone measured slower than the table).

// x W_32^Q (CONJ: x conj(W_32^Q)), W_32 = exp(-2 pi i / 32), compile-time Q in [0, 16).
template <int Q, bool CONJ>
__device__ __forceinline__ double2 mul_w32(double2 x) {
  static_assert(Q >= 0 && Q < 16, "twist constant index");
  constexpr double H = 0.70710678118654752440;
  constexpr double C1 = 0.92387953251128675613, S1 = 0.38268343236508977173;  // pi/8
  constexpr double CA = 0.98078528040323044913, SA = 0.19509032201612826785;  // pi/16
  constexpr double CB = 0.83146961230254523708, SB = 0.55557023301960222474;  // 3 pi/16
  constexpr double cs[16] = {1, CA, C1, CB, H, SB, S1, SA, 0, -SA, -S1, -SB, -H, -CB, -C1, -CA};
  constexpr double sn[16] = {0, SA, S1, SB, H, CB, C1, CA, 1, CA, C1, CB, H, SB, S1, SA};
  constexpr double c = cs[Q];
  constexpr double s = CONJ ? -sn[Q] : sn[Q];  // x (c - i s)
  if constexpr (Q == 0) {
    return x;
  } else if constexpr (Q == 8) {
    return make_double2(s * x.y, -s * x.x);
  } else {
    return make_double2(fma(s, x.y, c * x.x), fma(-s, x.x, c * x.y));
  }
}

template <int L>
struct CCfg {
  static constexpr int M = L / 2;
  static constexpr int R = fft_radix(M);
  static constexpr int T = M / R;   // threads per sub-lane
  static constexpr int LT = 2 * T;  // threads per lane
  static constexpr int THREADS_ = L == 512 ? FDG_C512_THREADS : (L == 1024 ? FDG_C1024_THREADS : 256);
  static constexpr int G = THREADS_ / LT < 1 ? 1 : THREADS_ / LT;  // lanes per CTA
  static constexpr int G2 = 2 * G;                                 // sub-lanes per CTA
  static constexpr int THREADS = G * LT;
  static constexpr int MINB_ROW = L == 512 ? FDG_C512_MINB_ROW : 1;
  static constexpr int MINB_COL = L == 512 ? FDG_C512_MINB_COL : (L == 1024 ? FDG_C1024_MINB_COL : 1);
  static constexpr int HR = R / 2;               // output positions per thread
  static constexpr size_t EXB = (size_t)M * G2;  // double2, one exchange buffer
  static constexpr bool HOMO = FDG_C_HOMO != 0;          // rows
  static constexpr bool HOMO_COL = FDG_C_HOMO_COL != 0;  // columns
  // sub-lane barriers assume T <= 32; the half-row swizzle a power-of-two G
  // sub-lanes of T > 32 synchronize with named barriers (fdg_fft.cuh lane_sync)
  static constexpr bool OK = T <= 64 && R >= 2 && (R & 1) == 0 && (G & (G - 1)) == 0 && (T <= 32 || G2 <= 8);
  // twist table in shared memory up to M = 512 (else read through L1, which
  // leaves room for four staged tiles at L = 2048)
  static constexpr bool TWS = M <= 512;
  // twist by constants (needs L / T == 32)
  static constexpr bool TWC = R == 16 && !TWS;
  // exchange | M-point twiddles | twist W_L^j (j < M) | symbol (L, real or
  // complex) | staging
  static constexpr size_t bytes(size_t stage_doubles, bool sr) {
    return sizeof(double2) * (EXB + (TWS ? 2 : 1) * (size_t)M) + (sr ? sizeof(double) : sizeof(double2)) * (size_t)L +
           sizeof(double) * stage_doubles;
  }
};

// Symbol of the convolution in shared memory: real (symmetric Toeplitz
// factor, SR) or complex.
template <bool SR>
struct SymTab {
  const double* re;
  const double2* c;
  __device__ __forceinline__ double2 apply(double2 v, int k) const {
    if constexpr (SR) {
      return cscale(v, re[k]);
    } else {
      return cmul(v, c[k]);
    }
  }
};

template <int L, bool SR>
struct CSmem {
  Ex ex;
  const double2* tw;
  const double2* twist;
  SymTab<SR> sym;
  double* stage;
  __device__ __forceinline__ CSmem(double2* base, const double2* gtw, const double2* gtwist, const double2* gsym,
                                   const double* gsym_re) {
    using C = CCfg<L>;
    ex.buf0 = base;
    ex.buf1 = base;
    ex.k = 0;
    double2* t = base + C::EXB;
    load_table(t, gtw, C::M);
    tw = t;
    t += C::M;
    if constexpr (C::TWS) {
      load_table(t, gtwist, C::M);
      twist = t;
      t += C::M;
    } else {
      twist = gtwist;
    }
    if constexpr (SR) {
      double* d = reinterpret_cast<double*>(t);
      // de-interleaved: even-frequency half | odd-frequency half (a sub-lane's
      // threads then read consecutive doubles; index 2 k + b is a 2-way bank
      // conflict in the lane-major row passes)
      for (int i = threadIdx.x; i < L; i += blockDim.x) d[(i & 1) * (L / 2) + (i >> 1)] = __ldg(&gsym_re[i]);
      sym.re = d;
      sym.c = nullptr;
      stage = d + L;
    } else {
      load_table(t, gsym, L);
      sym.c = t;
      sym.re = nullptr;
      stage = reinterpret_cast<double*>(t + L);
    }
  }
};

// Thread -> (lane g, half b, sub-lane thread t, sub-lane slot id gs, partner).
template <int L, bool ROWS, bool HOMO_>
struct CMap {
  static constexpr bool HOMO = HOMO_;
  int g, b, t, gs, partner;
  __device__ __forceinline__ CMap() {
    using C = CCfg<L>;
    const int tid = threadIdx.x;
    if constexpr (HOMO) {
      b = tid / (C::G * C::T);
      const int r = tid - b * (C::G * C::T);
      if constexpr (ROWS) {
        g = r / C::T;
        t = r - g * C::T;
      } else {
        t = r / C::G;
        g = r - t * C::G;
      }
      gs = b * C::G + g;
      partner = b ? gs - C::G : gs + C::G;
    } else if constexpr (ROWS) {
      g = tid / C::LT;
      b = (tid / C::T) & 1;
      t = tid % C::T;
      gs = 2 * g + b;
      partner = gs ^ 1;
    } else {
      gs = tid % C::G2;
      t = tid / C::G2;
      g = gs >> 1;
      b = gs & 1;
      partner = gs ^ 1;
    }
  }
  // slot id holding the lane's half-b values
  __device__ __forceinline__ int half_id(int h) const { return HOMO ? h * CCfg<L>::G + g : 2 * g + h; }
};

// Barrier over the two sub-lanes of every lane.
// Lane-major HOMO rows with T <= 32: lane g's halves are warps
// (g T / 32) and (G T / 32 + g T / 32); the two warps meet on named barrier
// 1 + g T / 32 (the sub-lane exchanges use __syncwarp, no ids).
template <int L, int LAYOUT, bool HOMO>
__device__ __forceinline__ void pair_sync(int g = 0) {
  using C = CCfg<L>;
  if constexpr (LAYOUT == 1 && HOMO && C::T <= 32 && (C::G * C::T) % 32 == 0 && FDG_HALF_BAR) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(1 + (g * C::T) / 32), "n"(64) : "memory");
  } else if constexpr (LAYOUT != 1 || HOMO || C::LT > 32) {
    __syncthreads();
  } else {
    __syncwarp();
  }
}

// v[m] *= W_32^m wt for every m (compile-time recursion over m).
template <int Q, int R>
__device__ __forceinline__ void twist_const(double2 (&v)[R], double2 wt) {
  if constexpr (Q < R) {
    v[Q] = cmul(mul_w32<Q, false>(v[Q]), wt);
    twist_const<Q + 1>(v, wt);
  }
}
// x conj(W_L^pos) for pos = t + T (I + b R/2): conj(W_32^I) (+i)^b conj(wt).
template <int I>
__device__ __forceinline__ double2 untwist_const(double2 x, int b, double2 wt) {
  double2 y = mul_w32<I, true>(x);
  if (b) y = make_double2(-y.y, y.x);
  return cmulc(y, wt);
}

// Sub-lane b's half of the convolution, in place on v (input z[t + T m] for
// every m; output that half's contribution at the same positions).
#ifndef FDG_BAL_TWIST
#define FDG_BAL_TWIST 1
#endif
// The forward and the inverse transform share their per-thread twiddles
// (TwCache) when the M-point transform has a single twiddled pass.
template <int L, int LAYOUT, bool SR>
__device__ __forceinline__ void conv_half(double2 (&v)[CCfg<L>::R], Ex& ex, int t, int gs, int b,
                                          const double2* tw, const double2* twist, const SymTab<SR>& sym) {
  using C = CCfg<L>;
  constexpr int M = C::M, R = C::R, T = C::T, G2 = C::G2;
  constexpr bool CACHE = FDG_TWCACHE && TwCache<M, R>::OK;
  if (b) {
    if constexpr (C::TWC) {
      const double2 wt = twist[t];
      twist_const<0>(v, wt);
    } else {
#pragma unroll
      for (int m = 0; m < R; ++m) v[m] = cmul(v[m], twist[t + T * m]);
    }
  }
  double2 wc[TwCache<M, R>::K];
  fft_lane_c<M, R, G2, false, LAYOUT, CACHE ? 1 : 0>(v, ex, t, gs, tw, wc);
#pragma unroll
  for (int m = 0; m < R; ++m) v[m] = sym.apply(v[m], SR ? b * M + (t + T * m) : 2 * (t + T * m) + b);
  fft_lane_c<M, R, G2, true, LAYOUT, CACHE ? 2 : 0>(v, ex, t, gs, tw, wc);
  // FDG_BAL_TWIST: the odd half's post-twist W_L^-j is applied in
  // conv_combine, each half twisting the odd values of its own positions
  if (b && !FDG_BAL_TWIST) {
#pragma unroll
    for (int m = 0; m < R; ++m) v[m] = cmulc(v[m], twist[t + T * m]);
  }
}

// conv_combine's read-and-add with the odd values' post-twist formed from
// constants (compile-time recursion over the owned positions).
template <int I, int L, int LAYOUT, class Map>
__device__ __forceinline__ void combine_const(const double2 (&v)[CCfg<L>::R], double2 (&y)[CCfg<L>::HR],
                                              const double2* sm, const Map& mp, double2 wt) {
  using C = CCfg<L>;
  constexpr int M = C::M, T = C::T, G2 = C::G2, HR = C::HR;
  if constexpr (I < HR) {
    const int b = mp.b;
    const int pos = mp.t + T * (I + b * HR);
    double2 mine = b ? v[I + HR] : v[I];
    double2 other = sm[slot<LAYOUT, M, G2>(pos, mp.partner)];
    if (b) mine = untwist_const<I>(mine, 1, wt);
    else other = untwist_const<I>(other, 0, wt);
    y[I] = cadd(mine, other);
    combine_const<I + 1, L, LAYOUT>(v, y, sm, mp, wt);
  }
}

// Adds the two halves: half 0 owns positions t + T m for m < R/2, half 1
// those for m >= R/2; y[i] is position t + T (i + b R/2).  Each store
// instruction writes one half-row of both halves (conflict-free).  TRAIL:
// barrier after the reads (when no other barrier precedes the next scatter).
// FDG_BAL_TWIST: v of the odd half is not yet post-twisted; the odd half
// twists its own positions, the even half the odd values it receives (8
// twist multiplies per thread instead of 16 on the odd half only).
template <int L, int LAYOUT, bool TRAIL, class Map>
__device__ __forceinline__ void conv_combine(const double2 (&v)[CCfg<L>::R], double2 (&y)[CCfg<L>::HR], Ex& ex,
                                             const Map& mp, const double2* twist) {
  constexpr bool HM = Map::HOMO;
  using C = CCfg<L>;
  constexpr int M = C::M, T = C::T, G2 = C::G2, HR = C::HR;
  const int t = mp.t, b = mp.b;
  pair_sync<L, LAYOUT, HM>(mp.g);  // write-after-read: last inverse-FFT exchange
  double2* sm = ex.next();
#pragma unroll
  for (int i = 0; i < HR; ++i) {
    const double2 val = b ? v[i] : v[i + HR];
    sm[slot<LAYOUT, M, G2>(t + T * (b ? i : i + HR), mp.gs)] = val;
  }
  pair_sync<L, LAYOUT, HM>(mp.g);
  if constexpr (C::TWC && FDG_BAL_TWIST) {
    combine_const<0, L, LAYOUT>(v, y, sm, mp, twist[t]);
  } else {
#pragma unroll
    for (int i = 0; i < HR; ++i) {
      const int pos = t + T * (i + b * HR);
      double2 mine = b ? v[i + HR] : v[i];
      double2 other = sm[slot<LAYOUT, M, G2>(pos, mp.partner)];
#if FDG_BAL_TWIST
      const double2 w = twist[pos];
      if (b) mine = cmulc(mine, w);
      else other = cmulc(other, w);
#endif
      y[i] = cadd(mine, other);
    }
  }
  if constexpr (TRAIL) pair_sync<L, LAYOUT, HM>(mp.g);
}

// =================================================================== rows
template <int L, int MODE, bool PF, bool SR>
struct RowCPlan {
  using C = CCfg<L>;
  static constexpr bool SEPI = PF && FDG_C_EPI != 0;      // staged epilogue operands
  static constexpr int TILE = PF ? 2 * C::G * C::M : 0;  // doubles per staged operand
  static constexpr int NIN = MODE == 2 ? 2 : 1;
  static constexpr int NEPI = SEPI ? (MODE == 0 ? 1 : (MODE == 1 ? 3 : 2)) : 0;
  static constexpr size_t SMEM = C::bytes((size_t)TILE * (NIN + NEPI), SR);
};

// Row pass along x2, modes as k_row (fdg_passes.cuh).  Lane-major exchange
// layout (every sub-lane owns M contiguous slots).
template <int L, int MODE, bool PF, bool SR>
__global__ void __launch_bounds__(CCfg<L>::THREADS, CCfg<L>::MINB_ROW) k_rowc(RowArgs a) {
  using C = CCfg<L>;
  using RP = RowCPlan<L, MODE, PF, SR>;
  static_assert(C::OK, "split pass configuration");
  constexpr int M = C::M, R = C::R, T = C::T, G = C::G, HR = C::HR;
  constexpr int TILE = RP::TILE;
  constexpr bool SEPI = RP::SEPI;
  extern __shared__ __align__(128) double2 smem_raw[];
  __shared__ double scratch[32];
  CSmem<L, SR> S(smem_raw, a.twh, a.twist, a.sym, a.sym_re);
  pdl_trigger();
  pdl_wait();
  if (paused(a.guard)) return;
  double* st_in = S.stage;
  double* st_in2 = S.stage + TILE;
  double* st_nb = S.stage + RP::NIN * TILE;
  double* st_nb2 = st_nb + TILE;
  double* st_vp = S.stage + 2 * TILE;
  double* st_r = S.stage + 3 * TILE;
  const CMap<L, true, C::HOMO> mp;
  const int g = mp.g, b = mp.b, t = mp.t;
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
  const double* in0 = MODE == 2 ? a.z : a.x;
  const double* in1 = a.dold;
  const ptrdiff_t noff = (ptrdiff_t)a.tdir * a.n1 * n;
  double acc = 0.0;
  // MODE 2 full tiles: the previous iteration's x += alpha d_old rides here
  // (d_old is staged anyway); x of the owned positions is prefetched into
  // registers one tile ahead so its latency hides behind a whole tile.
  constexpr bool XPF = MODE == 2 && PF;
  double2 xpre[XPF ? HR : 1];
  const bool upd_x = XPF && a.upd_x && !first;
  auto load_x = [&](int tl) {
    const size_t rx = (size_t)(tl * 2 * G + 2 * g) * n;
#pragma unroll
    for (int i = 0; i < (XPF ? HR : 1); ++i) {
      const int pos = t + T * (i + b * HR);
      xpre[i] = make_double2(a.xs[rx + pos], a.xs[rx + n + pos]);
    }
  };
  // TMA staging: barrier 0 = the tile's FFT input, 1 = its epilogue operands
  constexpr bool TMA = PF && FDG_TMA_ROWS;
  __shared__ alignas(8) unsigned long long bars[2];
  constexpr unsigned TB = sizeof(double) * TILE;  // bytes per staged operand
  unsigned ph_in = 0, ph_ep = 0;
  auto stage_in = [&](int tl) {  // elected thread: next FFT input (+ d_old)
    const unsigned nb = (MODE == 2 && !first) ? 2 * TB : TB;
    mbar_expect_tx(&bars[0], nb);
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
  } else if constexpr (PF) {
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
    const int f = f0 + 2 * g;
    const bool va = PF || f < F, vb = PF || f + 1 < F;
    const size_t ra = (size_t)f * n;
    double2 v[R];
    bool tile_nb = false;
    bool ep_armed = false;
    if constexpr (PF) {
      if constexpr (TMA) {
        mbar_wait(&bars[0], ph_in);
        ph_in ^= 1;
      } else {
        cp_async_wait<0>();
        __syncthreads();
      }
#pragma unroll
      for (int m = 0; m < R; ++m) {
        const int pos = t + m * T;
        double2 z = make_double2(st_in[(2 * g) * M + pos], st_in[(2 * g + 1) * M + pos]);
        if constexpr (MODE == 2) {
          double2 dd = make_double2(0.0, 0.0);
          if (!first) {
            dd = make_double2(st_in2[(2 * g) * M + pos], st_in2[(2 * g + 1) * M + pos]);
            z.x += beta * dd.x;
            z.y += beta * dd.y;
          }
          if ((m < HR) == (b == 0)) {
            a.dnew[ra + pos] = z.x;
            a.dnew[ra + n + pos] = z.y;
            if constexpr (XPF) {
              if (upd_x) {
                const int i = m < HR ? m : m - HR;  // static: only the owning half stores
                a.xs[ra + pos] = xpre[i].x + alpha * dd.x;
                a.xs[ra + n + pos] = xpre[i].y + alpha * dd.y;
              }
            }
          }
        }
        v[m] = z;
      }
      if constexpr (XPF) {
        if (upd_x && tile + (int)gridDim.x < ntiles) load_x(tile + gridDim.x);
      }
      __syncthreads();  // st_in and the epilogue staging are free
      const int k = f0 / a.n1;
      tile_nb = a.tkind == 1 && (a.tdir < 0 ? k >= 1 : k + 1 < a.nt);
      const int nxt = tile + gridDim.x;
      if constexpr (TMA) {
        // epilogue operands of this tile, then the next tile's input
        unsigned eb = 0;
        if constexpr (SEPI) {
          if (tile_nb) eb += (MODE == 2 && !first) ? 2 * TB : TB;
          if constexpr (MODE == 1) eb += a.r ? 2 * TB : TB;
        }
        ep_armed = eb != 0;
        if (threadIdx.x == 0) {
          fence_proxy_async();  // the reads of st_in / the previous epilogue before the refill
          if (ep_armed) {
            mbar_expect_tx(&bars[1], eb);
            if constexpr (SEPI) {
              if (tile_nb) {
                bulk_g2s(st_nb, in0 + (size_t)f0 * n + noff, TB, &bars[1]);
                if (MODE == 2 && !first) bulk_g2s(st_nb2, in1 + (size_t)f0 * n + noff, TB, &bars[1]);
              }
              if constexpr (MODE == 1) {
                bulk_g2s(st_vp, a.vp + (size_t)f0 * n, TB, &bars[1]);
                if (a.r) bulk_g2s(st_r, (a.r_in ? a.r_in : a.r) + (size_t)f0 * n, TB, &bars[1]);
              }
            }
          }
          if (nxt < ntiles) stage_in(nxt);
        }
      } else {
        if constexpr (SEPI) {
          if (tile_nb) {
            stage_rows(st_nb, in0 + (size_t)f0 * n + noff, TILE);
            if (MODE == 2 && !first) stage_rows(st_nb2, in1 + (size_t)f0 * n + noff, TILE);
          }
          if constexpr (MODE == 1) {
            stage_rows(st_vp, a.vp + (size_t)f0 * n, TILE);
            if (a.r) stage_rows(st_r, (a.r_in ? a.r_in : a.r) + (size_t)f0 * n, TILE);
          }
        }
        cp_async_commit();  // group E
        if (nxt < ntiles) {
          stage_rows(st_in, in0 + (size_t)nxt * 2 * G * n, TILE);
          if (MODE == 2 && !first) stage_rows(st_in2, in1 + (size_t)nxt * 2 * G * n, TILE);
        }
        cp_async_commit();  // group I
      }
    } else {
#pragma unroll
      for (int m = 0; m < R; ++m) {
        const int pos = t + m * T;
        double2 z = make_double2(0.0, 0.0);
        if (pos < n) {
          if (va) z.x = __ldg(in0 + ra + pos);
          if (vb) z.y = __ldg(in0 + ra + n + pos);
          if constexpr (MODE == 2) {
            if (!first) {
              if (va) z.x += beta * __ldg(in1 + ra + pos);
              if (vb) z.y += beta * __ldg(in1 + ra + n + pos);
            }
            if ((m < HR) == (b == 0)) {
              if (va) a.dnew[ra + pos] = z.x;
              if (vb) a.dnew[ra + n + pos] = z.y;
            }
          }
        }
        v[m] = z;
      }
    }
    conv_half<L, 1>(v, S.ex, t, mp.gs, b, S.tw, S.twist, S.sym);
    double2 y[HR];
    conv_combine<L, 1, !PF>(v, y, S.ex, mp, S.twist);

    if constexpr (SEPI) {
      if constexpr (TMA) {
        if (ep_armed) {
          mbar_wait(&bars[1], ph_ep);
          ph_ep ^= 1;
        }
      } else {
        cp_async_wait<1>();
        __syncthreads();
      }
    }
    const int ka = f / a.n1, kb = (f + 1) / a.n1;
    const bool nba = a.tkind == 1 && (a.tdir < 0 ? ka >= 1 : ka + 1 < a.nt);
    const bool nbb = a.tkind == 1 && (a.tdir < 0 ? kb >= 1 : kb + 1 < a.nt);
#pragma unroll
    for (int i = 0; i < HR; ++i) {
      const int pos = t + T * (i + b * HR);
      if (!PF && pos >= n) continue;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (!PF && !(h ? vb : va)) continue;
        const int sl = (2 * g + h) * M + pos;
        const size_t o = ra + h * n + pos;
        double val = a.scale * (h ? y[i].y : y[i].x);
        if constexpr (SEPI) {
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
          if (MODE == 2 && !XPF && a.upd_x && !first) a.xs[o] += alpha * __ldg(in1 + o);
        } else {
          const double q = (SEPI ? st_vp[sl] : __ldg(&a.vp[o])) + val;
          if (a.q_out) a.q_out[o] = q;
          if (a.r) {
            const double rn = (SEPI ? st_r[sl] : (a.r_in ? a.r_in : a.r)[o]) - alpha * q;
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
template <int L, int MODE, bool PF, bool SR>
struct ColCPlan {
  using C = CCfg<L>;
  // exchange layout: 1 = lane-major (sub-lane-local exchanges, __syncwarp),
  // else interleaved rows (CTA-wide barriers)
  static constexpr int LY = FDG_C_COLLY == 1 ? 1 : (C::HOMO_COL ? 2 : 0);
  static constexpr int W = 2 * C::G;              // columns per tile
  static constexpr int P = LY == 1 ? W + 2 : W;   // staged row pitch (bank spread)
  static constexpr int TILE = PF ? C::M * P : 0;  // doubles per staged operand
  // MODE 2: double-buffered p (readable by both epilogues) and u
  static constexpr int NST = MODE == 2 ? 4 : 1;
  static constexpr size_t SMEM = C::bytes((size_t)TILE * NST, SR);
};

// Column pass, modes as k_col (fdg_passes.cuh).  Interleaved exchange layout
// (rows of G2 sub-lanes; split-interleaved when HOMO), sub-lanes of lane g
// serve columns (2g, 2g+1) of the tile.
// Tensor maps of the staged operands (FDG_TMA_COLS == 2): x (p) and acc (u)
// viewed as [O n rows][C] doubles, box [min(n, 256) rows][W columns].
struct ColMaps {
  CUtensorMap x, acc;
};

template <int L, int MODE, bool PF, bool SR>
__global__ void __launch_bounds__(CCfg<L>::THREADS, CCfg<L>::MINB_COL)
    k_colc(ColArgs a, const __grid_constant__ ColMaps maps) {
  using Cf = CCfg<L>;
  static_assert(Cf::OK, "split pass configuration");
  constexpr int M = Cf::M, R = Cf::R, T = Cf::T, G = Cf::G, G2 = Cf::G2, HR = Cf::HR;
  using CP = ColCPlan<L, MODE, PF, SR>;
  constexpr int LY = CP::LY, W = CP::W, P = CP::P;
  extern __shared__ __align__(128) double2 smem_raw[];
  __shared__ double scratch[32];
  CSmem<L, SR> S(smem_raw, a.twh, a.twist, a.sym, a.sym_re);
  pdl_trigger();
  pdl_wait();
  if (paused(a.guard)) return;
  constexpr int TILE = CP::TILE;
  constexpr bool DB = MODE == 2;  // double-buffered staging
  const CMap<L, LY == 1, Cf::HOMO_COL> mp;
  const int g = mp.g, b = mp.b, t = mp.t;
  const int n = a.n, C = a.C;
  const int ncb = (C + W - 1) / W;
  const int ntiles = ncb * a.O;
  // staged column tile [pos][W] of `src` for tile index tl
  auto stage_tile = [&](double* dst, const double* src, int tl) {
    const int ot = tl / ncb;
    stage_cols<W, P>(dst, src + (size_t)ot * n * C + (size_t)(tl - ot * ncb) * W, n, C);
  };
  // TMA staging (FDG_TMA_COLS): warp 0 issues one bulk copy per W-double row
  // segment of the tile's operands into buffer `bi`, completion on bars[bi]
  constexpr bool TMA = PF && FDG_TMA_COLS && P == W;
  constexpr bool TMAP = TMA && FDG_TMA_COLS == 2;  // tensor-map boxes
  __shared__ alignas(8) unsigned long long bars[2];
  unsigned phb = 0;  // phase parity per buffer (bits)
  auto stage_tma = [&](int bi, int tl) {
    const int ot = tl / ncb;
    const size_t off = (size_t)ot * n * C + (size_t)(tl - ot * ncb) * W;
    const int lane = threadIdx.x & 31;
    constexpr unsigned RB = W * sizeof(double);
    const unsigned nops = MODE == 2 ? 2 : 1;
    fence_proxy_async();
    if (lane == 0) mbar_expect_tx(&bars[bi], nops * RB * (unsigned)n);
    __syncwarp();
    double* d0 = S.stage + bi * TILE;
    double* d1 = S.stage + (2 + bi) * TILE;
    if constexpr (TMAP) {  // lane 0: one box per 256 rows and operand
      if (lane == 0) {
        const int bh = n < 256 ? n : 256;
        const int x = (tl - ot * ncb) * W, y0 = ot * n;
        for (int r0 = 0; r0 < n; r0 += bh) {
          tma_load_2d(d0 + r0 * P, &maps.x, x, y0 + r0, &bars[bi]);
          if constexpr (MODE == 2) tma_load_2d(d1 + r0 * P, &maps.acc, x, y0 + r0, &bars[bi]);
        }
      }
    } else {
      for (int pos = lane; pos < n; pos += 32) {
        bulk_g2s(d0 + pos * P, a.x + off + (size_t)pos * C, RB, &bars[bi]);
        if constexpr (MODE == 2) bulk_g2s(d1 + pos * P, a.acc + off + (size_t)pos * C, RB, &bars[bi]);
      }
    }
  };
  if constexpr (TMA) {
    if (threadIdx.x == 0) {
      mbar_init(&bars[0], 1);
      mbar_init(&bars[1], 1);
      mbar_init_fence();
    }
    __syncthreads();
    if (threadIdx.x < 32 && blockIdx.x < ntiles) stage_tma(0, blockIdx.x);
  } else if constexpr (PF) {
    if (blockIdx.x < ntiles) {
      stage_tile(S.stage, a.x, blockIdx.x);
      if constexpr (MODE == 2) stage_tile(S.stage + 2 * TILE, a.acc, blockIdx.x);
    }
    cp_async_commit();
  }
  __syncthreads();  // tables
  double e = 0.0;
  int buf = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, buf ^= DB) {
    const int o = tile / ncb;
    const long c = (long)((tile - o * ncb) * G + g) * 2;
    const bool vc = PF || c < C;
    const bool vb = PF || c + 1 < C;
    const size_t base = (size_t)o * n * C + c;
    const int nxt = tile + gridDim.x;
    double* st_in = S.stage + buf * TILE;
    const double* st_u = S.stage + (2 + buf) * TILE;  // MODE 2
    // per-slice scalars of the S mid pass, requested before the wait on the
    // staged tile so their latency hides behind it
    double a1_t = 0.0, im2_t = 0.0;
    if constexpr (MODE == 2) {
      a1_t = __ldg(&a.a1[o]);
      im2_t = __ldg(&a.inv_m2[o]);
    }
    double2 v[R];
    if constexpr (PF) {
      if constexpr (TMA) {
        mbar_wait(&bars[buf], (phb >> buf) & 1);
        phb ^= 1u << buf;
        __syncthreads();  // the other buffer's previous tile is done: it may be refilled
      } else {
        cp_async_wait<0>();
        __syncthreads();
      }
#pragma unroll
      for (int m = 0; m < R; ++m) v[m] = *reinterpret_cast<const double2*>(st_in + (t + m * T) * P + 2 * g);
      if constexpr (MODE == 2 && FDG_K2_EREG) {
        // a1 p^T p of the owned positions from the registers (saves the
        // staged re-read of p in the first epilogue)
        const double a1 = a1_t;
#pragma unroll
        for (int i = 0; i < HR; ++i) {
          const double2 pv = b ? v[i + HR] : v[i];
          e = fma(a1, fma(pv.x, pv.x, pv.y * pv.y), e);
        }
      }
      if constexpr (MODE != 2) __syncthreads();  // single input buffer
      if constexpr (TMA) {
        if (nxt < ntiles && threadIdx.x < 32) stage_tma(buf ^ DB, nxt);
      } else {
        if (nxt < ntiles) {
          stage_tile(S.stage + (buf ^ DB) * TILE, a.x, nxt);
          if constexpr (MODE == 2) stage_tile(S.stage + (2 + (buf ^ 1)) * TILE, a.acc, nxt);
        }
        cp_async_commit();
      }
    } else {
#pragma unroll
      for (int m = 0; m < R; ++m) {
        const int pos = t + m * T;
        v[m] = (pos < n && vc) ? col_get<false>(a.x + base + (size_t)pos * C, C, c) : make_double2(0.0, 0.0);
      }
    }
    conv_half<L, LY>(v, S.ex, t, mp.gs, b, S.tw, S.twist, S.sym);
    double2 y[HR];
    conv_combine<L, LY, !PF && MODE == 0>(v, y, S.ex, mp, S.twist);

    if constexpr (MODE == 0) {
#pragma unroll
      for (int i = 0; i < HR; ++i) {
        const int pos = t + T * (i + b * HR);
        if (!PF && (pos >= n || !vc)) continue;
        const size_t o2 = base + (size_t)pos * C;
        double2 acc = make_double2(0.0, 0.0);
        if (a.acc) acc = col_get<PF>(a.acc + o2, C, c);
        col_put<PF>(a.out + o2, C, c, make_double2(acc.x + a.scale * y[i].x, acc.y + a.scale * y[i].y));
      }
    } else {
      // S mid pass: Bp = u + scale L1 p; w = Bp / m2[o] (-> a.w, and the
      // input of the second convolution); vp = scale L1 w + a1 p (-> a.out)
      const double im2 = im2_t, a1 = a1_t;
#pragma unroll
      for (int i = 0; i < HR; ++i) {
        const int pos = t + T * (i + b * HR);
        if (PF || (pos < n && vc)) {
          const size_t o2 = base + (size_t)pos * C;
          const double2 u = PF ? *reinterpret_cast<const double2*>(st_u + pos * P + 2 * g) : col_get<PF>(a.acc + o2, C, c);
          const double bx = u.x + a.scale * y[i].x;
          const double by = u.y + a.scale * y[i].y;
          const double wx = bx * im2, wy = vb ? by * im2 : 0.0;
          if (PF && FDG_K2_EREG) {
            e += wx * bx + wy * by;
          } else {
            const double2 pv = PF ? *reinterpret_cast<const double2*>(st_in + pos * P + 2 * g) : col_get<PF>(a.x + o2, C, c);
            e += a1 * pv.x * pv.x + wx * bx;
            if (vb) e += a1 * pv.y * pv.y + wy * by;
          }
          col_put<PF>(a.w + o2, C, c, make_double2(wx, wy));
          y[i] = make_double2(wx, wy);
        } else {
          y[i] = make_double2(0.0, 0.0);
        }
      }
      // both halves need all of w: each writes its positions into its own
      // slot column, then reads the lane's full column pair
      pair_sync<L, LY, Cf::HOMO_COL>(mp.g);  // write-after-read: combine
      double2* sm = S.ex.next();
#pragma unroll
      for (int i = 0; i < HR; ++i) sm[slot<LY, M, G2>(t + T * (i + b * HR), mp.gs)] = y[i];
      pair_sync<L, LY, Cf::HOMO_COL>(mp.g);
      // the owned half of w is still in registers: only the partner's half
      // comes back from the exchange
#pragma unroll
      for (int i = 0; i < HR; ++i) {
        const double2 other = sm[slot<LY, M, G2>(t + T * (i + (1 - b) * HR), mp.partner)];
        v[i] = b ? other : y[i];
        v[i + HR] = b ? y[i] : other;
      }
      // write-after-read across the halves: each half reads the other's
      // slots above, and the first scatter of its transform below is guarded
      // only by its own half barrier (lane_sync), so a lagging half could
      // still be reading the slots the other half overwrites
      pair_sync<L, LY, Cf::HOMO_COL>(mp.g);
      conv_half<L, LY>(v, S.ex, t, mp.gs, b, S.tw, S.twist, S.sym);
      conv_combine<L, LY, !PF>(v, y, S.ex, mp, S.twist);
#pragma unroll
      for (int i = 0; i < HR; ++i) {
        const int pos = t + T * (i + b * HR);
        if (!PF && (pos >= n || !vc)) continue;
        const size_t o2 = base + (size_t)pos * C;
        const double2 pv = PF ? *reinterpret_cast<const double2*>(st_in + pos * P + 2 * g) : col_get<PF>(a.x + o2, C, c);
        col_put<PF>(a.out + o2, C, c, make_double2(a.scale * y[i].x + a1 * pv.x, a.scale * y[i].y + a1 * pv.y));
      }
    }
  }
  if constexpr (MODE == 2) {
    double vv[1] = {e};
    block_reduce<RED_SUM, 1>(vv, scratch);
    grid_finalize<RED_SUM, 1>(vv, a.red, scratch);
  }
}

}  // namespace fdg
