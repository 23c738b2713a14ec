// fdg_fft.cuh — fp64 shared-memory Stockham FFT building blocks for sm_100a.
//
// Replaces the arithmetic of fft::BatchedRealFft / fft::Fft3D
// (/root/reference/proj/src/fft.cpp:25-109, FFTW r2c/c2r/3-D) on the device.
//
// Execution model ("lane-interleaved tile"):
//   * a CTA runs G independent complex FFTs of length N ("lanes");
//   * lane g uses T = N/R threads; thread (g, t) lives at tid = t*G + g, so a
//     warp covers 32/G consecutive t of all G lanes;
//   * thread t of a lane holds x[t + m*T] (m < R) in registers, both at the
//     input and at the output of the transform (Stockham autosort keeps
//     natural order on both sides), so pointwise work (symbol multiply,
//     spectral division) happens in registers between a forward and an
//     inverse transform with no extra exchange;
//   * between radix passes the data goes through shared memory laid out as
//     sm[pos][G] double2: a warp touches 32/G positions x G lanes, i.e. whole
//     128-byte rows of 8 complex values for G = 8, so exchanges are free of
//     bank conflicts whatever the Stockham scatter pattern is.
// Twiddles come from a per-length table W_N[k] = exp(-2 pi i k/N) in global
// memory (L1-resident), computed on the host in long double.
#pragma once

#include <cuda_runtime.h>

namespace fdg {

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }

// 1/x for finite x > 0 without the IEEE division slow path: MUFU reciprocal
// seed and two Newton steps (error within 2 ulp).
__device__ __forceinline__ double frcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// Multiply by W_R^q = exp(-/+ 2 pi i q / R) for compile-time (R, q).
template <int R, int Q, bool INV>
__device__ __forceinline__ double2 mul_wq(double2 x) {
  constexpr int q = ((Q % R) + R) % R;
  if constexpr (q == 0) {
    return x;
  } else if constexpr (4 * q == R) {  // -i (fwd) / +i (inv)
    return INV ? make_double2(-x.y, x.x) : make_double2(x.y, -x.x);
  } else if constexpr (2 * q == R) {
    return make_double2(-x.x, -x.y);
  } else if constexpr (4 * q == 3 * R) {  // +i (fwd) / -i (inv)
    return INV ? make_double2(x.y, -x.x) : make_double2(-x.y, x.x);
  } else if constexpr (8 * q == R || 8 * q == 3 * R || 8 * q == 5 * R || 8 * q == 7 * R) {
    constexpr double h = 0.70710678118654752440;
    // cos(2 pi q/R), -sin(2 pi q/R) for q/R in {1/8, 3/8, 5/8, 7/8}
    constexpr double c = (8 * q == R || 8 * q == 7 * R) ? h : -h;
    constexpr double s = (8 * q == R || 8 * q == 3 * R) ? -h : h;  // -sin
    constexpr double si = INV ? -s : s;
    return make_double2(c * x.x - si * x.y, c * x.y + si * x.x);
  } else {
    static_assert(R == 16, "general twiddle constants only for R = 16");
    constexpr double C1 = 0.92387953251128675613, S1 = 0.38268343236508977173;
    // q in {1,3,5,7,9,11,13,15}: cos/sin of 2 pi q/16
    constexpr double cs[16] = {1, C1, 0, S1, 0, -S1, 0, -C1, 0, -C1, 0, -S1, 0, S1, 0, C1};
    constexpr double sn[16] = {0, S1, 0, C1, 0, C1, 0, S1, 0, -S1, 0, -C1, 0, -C1, 0, -S1};
    constexpr double c = cs[q];
    constexpr double s = INV ? sn[q] : -sn[q];
    return make_double2(c * x.x - s * x.y, c * x.y + s * x.x);
  }
}

// Butterfly x0 = e + W_R^q o, x1 = e - W_R^q o for compile-time (R, q).
// Generic q: W o is factored as c (u, v) with the larger of |cos|, |sin|
// pulled out, so both outputs come from fused multiply-adds (6 DFMA instead
// of 2 DMUL + 2 DFMA + 4 DADD).
#ifndef FDG_FMA_BFLY
#define FDG_FMA_BFLY 1
#endif
template <int R, int Q, bool INV>
__device__ __forceinline__ void bfly_wq(double2 e, double2 o, double2& x0, double2& x1) {
  constexpr int q = ((Q % R) + R) % R;
  constexpr bool trivial = q == 0 || 4 * q == R || 2 * q == R || 4 * q == 3 * R;
  if constexpr (trivial || !FDG_FMA_BFLY) {
    const double2 t = mul_wq<R, Q, INV>(o);
    x0 = cadd(e, t);
    x1 = csub(e, t);
  } else {
    static_assert(R == 8 || R == 16, "generic butterfly constants only for R = 8, 16");
    constexpr double H = 0.70710678118654752440;
    constexpr double C1 = 0.92387953251128675613, S1 = 0.38268343236508977173;
    constexpr double cs16[16] = {1, C1, H, S1, 0, -S1, -H, -C1, -1, -C1, -H, -S1, 0, S1, H, C1};
    constexpr double sn16[16] = {0, S1, H, C1, 1, C1, H, S1, 0, -S1, -H, -C1, -1, -C1, -H, -S1};
    constexpr int q16 = R == 8 ? 2 * q : q;
    // W = cr + i ci: forward exp(-2 pi i q/R), inverse exp(+2 pi i q/R)
    constexpr double cr = cs16[q16];
    constexpr double ci = INV ? sn16[q16] : -sn16[q16];
    constexpr bool big_c = (cr < 0 ? -cr : cr) >= (ci < 0 ? -ci : ci);
    // W o = (cr o.x - ci o.y, cr o.y + ci o.x)
    if constexpr (big_c) {
      constexpr double t = ci / cr;
      const double u = fma(-t, o.y, o.x), v = fma(t, o.x, o.y);
      x0 = make_double2(fma(cr, u, e.x), fma(cr, v, e.y));
      x1 = make_double2(fma(-cr, u, e.x), fma(-cr, v, e.y));
    } else {
      constexpr double t = cr / ci;
      const double u = fma(t, o.x, -o.y), v = fma(t, o.y, o.x);
      x0 = make_double2(fma(ci, u, e.x), fma(ci, v, e.y));
      x1 = make_double2(fma(-ci, u, e.x), fma(-ci, v, e.y));
    }
  }
}

// In-register DFT of size R (natural order in and out): X_q = sum_r v_r W_R^{rq}.
template <int R, bool INV>
struct Dft;

template <bool INV>
struct Dft<1, INV> {
  template <class A>
  __device__ __forceinline__ static void run(A& v, int base, int stride) {}
};

template <bool INV>
struct Dft<2, INV> {
  template <class A>
  __device__ __forceinline__ static void run(A& v, int base, int stride) {
    const double2 a = v[base], b = v[base + stride];
    v[base] = cadd(a, b);
    v[base + stride] = csub(a, b);
  }
};

template <bool INV>
struct Dft<4, INV> {
  template <class A>
  __device__ __forceinline__ static void run(A& v, int base, int stride) {
    const double2 a = v[base], b = v[base + stride], c = v[base + 2 * stride], d = v[base + 3 * stride];
    const double2 s0 = cadd(a, c), s1 = csub(a, c), s2 = cadd(b, d), s3 = mul_wq<4, 1, INV>(csub(b, d));
    v[base] = cadd(s0, s2);
    v[base + 2 * stride] = csub(s0, s2);
    v[base + stride] = cadd(s1, s3);
    v[base + 3 * stride] = csub(s1, s3);
  }
};

// Radix-2 decimation in time on top of two half-size DFTs (R = 8, 16).
template <int R, bool INV>
struct Dft {
  static_assert(R == 8 || R == 16, "unsupported radix");
  template <class A>
  __device__ __forceinline__ static void run(A& v, int base, int stride) {
    constexpr int H = R / 2;
    double2 e[H], o[H];
#pragma unroll
    for (int r = 0; r < H; ++r) {
      e[r] = v[base + (2 * r) * stride];
      o[r] = v[base + (2 * r + 1) * stride];
    }
    Dft<H, INV>::run(e, 0, 1);
    Dft<H, INV>::run(o, 0, 1);
    combine<0>(v, base, stride, e, o);
  }
  template <int Q, class A>
  __device__ __forceinline__ static void combine(A& v, int base, int stride, const double2 (&e)[R / 2],
                                                 const double2 (&o)[R / 2]) {
    if constexpr (Q < R / 2) {
      double2 x0, x1;
      bfly_wq<R, Q, INV>(e[Q], o[Q], x0, x1);
      v[base + Q * stride] = x0;
      v[base + (Q + R / 2) * stride] = x1;
      combine<Q + 1>(v, base, stride, e, o);
    }
  }
};

// Shared-memory slot of (pos, lane).  Rows of G double2; for G < 8 a 128-byte
// bank window holds 8/G positions, so the low log2(8/G) bits of pos are XORed
// with a fold of the higher bits: power-of-two position strides (the Stockham
// scatter) then spread over all bank groups (measured model: 1.13x / 1.19x of
// conflict-free for G = 4 / 2 instead of 1.20x / 1.60x).
template <int G>
__device__ __forceinline__ int sidx(int pos, int g) {
  if constexpr (G >= 8) {
    return pos * G + g;
  } else if constexpr (G == 4) {
    return (pos ^ (__popc(pos >> 1) & 1)) * G + g;
  } else {  // G == 2: fold the 2-bit chunks of pos >> 2
    int h = pos >> 2;
    h ^= h >> 8;
    h ^= h >> 4;
    h ^= h >> 2;
    return (pos ^ (h & 3)) * G + g;
  }
}

// Lane-major slot (row passes: a warp covers consecutive positions of one
// lane, so its global accesses are 256-byte coalesced).  Each lane owns N
// contiguous slots; the low 3 bits of pos are XORed with a fold of the
// higher 3-bit groups so that strided Stockham scatters hit 8 different
// bank groups per quarter-warp.
template <int N>
__device__ __forceinline__ int lidx(int pos, int g) {
  const int f = (pos >> 3) ^ (pos >> 6) ^ (pos >> 9);
  return g * N + (pos ^ (f & 7));
}

// Split-interleaved slot (fdg_conv.cuh column passes, warps holding only
// even- or only odd-half sub-lanes): rows of G lanes whose two halves (G/2
// sub-lanes each) are swapped on rows of odd popcount, so the 32/(G/2)
// positions a half-row warp touches always fill complementary halves of the
// 128-byte bank window (any power-of-two position pattern has half of its
// positions at odd popcount).
// G = 4 (rows of 64 bytes, two per bank window): the first Stockham scatter
// writes pos = 16 t + r for consecutive t, whose row parity never changes, so
// bit 4 of pos is folded into the row's low bit as well (ncu: 8 -> 4
// wavefronts per store of that scatter at L = 2048).
template <int G>
__device__ __forceinline__ int hidx(int pos, int g) {
  const int row = G == 4 ? (pos ^ ((pos >> 4) & 1)) : pos;
  return row * G + (g ^ ((__popc(pos) & 1) * (G / 2)));
}

// LAYOUT 0: lane-interleaved rows of G (column passes); 1: lane-major;
// 2: split-interleaved (hidx).
template <int LAYOUT, int N, int G>
__device__ __forceinline__ int slot(int pos, int g) {
  if constexpr (LAYOUT == 0) return sidx<G>(pos, g);
  else if constexpr (LAYOUT == 2) return hidx<G>(pos, g);
  else return lidx<N>(pos, g);
}

// Double-buffered exchange area: consecutive exchanges alternate between two
// buffers, so one __syncthreads() per exchange suffices (a thread can only
// overwrite buffer X after every thread passed the barrier of the exchange
// that used the other buffer, i.e. after all reads of X completed).
struct Ex {
  double2* buf0;
  double2* buf1;
  int k;
  __device__ __forceinline__ double2* next() {
    double2* p = k ? buf1 : buf0;
    k ^= 1;
    return p;
  }
  __device__ __forceinline__ bool single() const { return buf0 == buf1; }
};

// Barrier of one exchange.  Lane-interleaved layout (0): the whole CTA shares
// every smem row -> __syncthreads.  Lane-major layout (1): each lane owns a
// private region, so only the lane's T threads synchronize: __syncwarp when a
// lane is (part of) one warp, a named barrier (id 1 + lane) otherwise.  Lanes
// then run their FFTs independently instead of in CTA-wide lock step.
#ifndef FDG_HALF_BAR
#define FDG_HALF_BAR 1
#endif
// LAYOUT 2 (split-interleaved rows of GW sub-lanes, even half | odd half):
// the sub-lanes of one half exchange only among themselves, so each half
// synchronizes its (GW/2) * T threads on a named barrier (id 1 + half)
// instead of the whole CTA.
template <int LAYOUT, int T, int GW = 1>
__device__ __forceinline__ void lane_sync(int g) {
  if constexpr (LAYOUT == 2 && FDG_HALF_BAR && GW >= 2) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(1 + (g >= GW / 2)), "n"((GW / 2) * T) : "memory");
  } else if constexpr (LAYOUT == 0 || LAYOUT == 2) {
    __syncthreads();
  } else if constexpr (T <= 32) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;\n" ::"r"(1 + g), "n"(T) : "memory");
  }
}

// Registers per thread (= radix bound) used for a transform of length N;
// shared by the kernels (Cfg) and the host twiddle-table builder.
#ifndef FDG_R256
#define FDG_R256 16
#endif
#ifndef FDG_R512
#define FDG_R512 16
#endif
#ifndef FDG_R128
#define FDG_R128 16  // 128 = 16 x 8: one exchange (C3 t filter 181 -> 166 us with 128-thread CTAs)
#endif
__host__ __device__ constexpr int fft_radix(int N) {
  return N <= 8 ? N
                : (N == 128 ? FDG_R128 : (N == 256 ? FDG_R256 : (N == 512 ? FDG_R512 : (N < 512 ? 8 : 16))));
}

// Compile-time radix plan: passes of radix min(R, N/Ns).
template <int N, int R, int Ns>
struct PassRadix {
  static constexpr int value = (N / Ns) < R ? (N / Ns) : R;
};

// Per-pass twiddle table ("ptw"): pass with stride Ns > 1 owns (Rp-1)*Ns
// entries at offset OFF, entry (r-1)*Ns + j = W_N^(j r N/(Ns Rp)).  A
// quarter-warp (8 consecutive butterflies) then reads 8 consecutive entries
// (one 128-byte bank window) instead of a power-of-two stride.
// Host builder: fdg_api.cu stockham_twiddles().

#ifndef FDG_TW_ALL
#define FDG_TW_ALL 0  // 1: load every twiddle instead of forming products of powers of two
#endif

// One Stockham pass on a lane (registers in, registers out, with the
// shared-memory scatter of the pass output unless it is the last pass).
//   N   : transform length, R: registers per thread, T = N/R
//   Ns  : product of previous radices, OFF: offset of this pass in ptw
//   G   : lanes per CTA (smem row width)
// Twiddle cache (CM): a transform with ONE twiddled pass (N <= R^2) has
// per-thread twiddles that depend only on the thread's position in its lane,
// so a forward / inverse pair (or several transforms of one thread) can form
// them once: CM = 1 forms and stores them in wc[s*Rp + r], CM = 2 reads wc
// (inverse passes use the conjugates of the same values).
#ifndef FDG_TWCACHE
#define FDG_TWCACHE 1
#endif
template <int N, int R>
struct TwCache {
  static constexpr bool OK = N > R && N / R <= R;
  static constexpr int K = OK ? R : 1;  // S * Rp of the twiddled pass
};

// Last pass of a three-pass plan (S > 1 butterflies per thread, N / T = 16):
// butterfly s of thread t sits at b = t + s T, so its twiddles factor as
// W_N^(b r) = (W_N^t)^r W_16^(s r): the Rp - 1 per-thread values are loaded
// once and the rest are compile-time constant multiplies (the shared-memory
// pipe, not FP64, is the busier unit: 3 loads instead of 12 at N = 1024).
template <int Rp, int S, bool INV, int Sx = 1, int Rx = 1>
struct LastTwiddle {
  template <int R>
  __device__ __forceinline__ static void run(double2 (&v)[R], const double2 (&wt)[Rp]) {
    if constexpr (Sx < S) {
      if constexpr (Rx < Rp) {
        const double2 x = mul_wq<16, (Sx * Rx) % 16, INV>(v[Sx + Rx * S]);
        v[Sx + Rx * S] = INV ? cmulc(x, wt[Rx]) : cmul(x, wt[Rx]);
        LastTwiddle<Rp, S, INV, Sx, Rx + 1>::run(v, wt);
      } else {
        LastTwiddle<Rp, S, INV, Sx + 1, 1>::run(v, wt);
      }
    }
  }
};

template <int N, int R, int G, bool INV, int Ns, int LAYOUT, int OFF = 0, int CM = 0>
struct Stockham {
  static constexpr int T = N / R;
  static constexpr int Rp = PassRadix<N, R, Ns>::value;
  static constexpr int S = R / Rp;  // butterflies per thread in this pass
  static constexpr bool LAST = (Ns * Rp == N);
  static constexpr int NEXT_OFF = OFF + (Ns > 1 ? (Rp - 1) * Ns : 0);

  __device__ __forceinline__ static void run(double2 (&v)[R], Ex& ex, int t, int g, const double2* ptw) {
    double2 wc[1];
    static_assert(CM == 0, "twiddle cache needs its array");
    run(v, ex, t, g, ptw, wc);
  }

  template <int CK>
  __device__ __forceinline__ static void run(double2 (&v)[R], Ex& ex, int t, int g, const double2* ptw,
                                             double2 (&wc)[CK]) {
    static_assert(CM == 0 || (TwCache<N, R>::OK && CK >= TwCache<N, R>::K), "twiddle cache shape");
    constexpr bool LASTC = LAST && Ns > 1 && S > 1 && R == 16 && CM == 0 && T <= Ns;
    if constexpr (LASTC) {
      double2 wt[Rp];
#pragma unroll
      for (int r = 1; r < Rp; ++r) {
        if ((r & (r - 1)) == 0) {
          wt[r] = ptw[OFF + (r - 1) * Ns + t];
        } else {
          const int lo = r & -r;
          wt[r] = cmul(wt[lo], wt[r - lo]);
        }
      }
#pragma unroll
      for (int r = 1; r < Rp; ++r) v[r * S] = INV ? cmulc(v[r * S], wt[r]) : cmul(v[r * S], wt[r]);
      LastTwiddle<Rp, S, INV>::run(v, wt);
#pragma unroll
      for (int s = 0; s < S; ++s) Dft<Rp, INV>::run(v, s, S);
    } else {
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const int b = t + s * T;  // butterfly index in [0, N/Rp)
        if constexpr (Ns > 1) {
          // Load the power-of-two twiddles w^1, w^2, w^4(, w^8) and form the
          // others as products (3 of 7 loads for radix 8): the shared-memory
          // pipe, not FP64, is the busiest unit of these kernels.
          const double2* tw = ptw + OFF + (b & (Ns - 1));
          double2 wt[Rp];
          if constexpr (CM == 2) {
#pragma unroll
            for (int r = 1; r < Rp; ++r) wt[r] = wc[s * Rp + r];
          } else {
#pragma unroll
            for (int r = 1; r < Rp; ++r) {
              if (FDG_TW_ALL || (r & (r - 1)) == 0) {
                wt[r] = tw[(r - 1) * Ns];
              } else {
                const int lo = r & -r;
                wt[r] = cmul(wt[lo], wt[r - lo]);
              }
            }
            if constexpr (CM == 1) {
#pragma unroll
              for (int r = 1; r < Rp; ++r) wc[s * Rp + r] = wt[r];
            }
          }
#pragma unroll
          for (int r = 1; r < Rp; ++r) v[s + r * S] = INV ? cmulc(v[s + r * S], wt[r]) : cmul(v[s + r * S], wt[r]);
        }
        Dft<Rp, INV>::run(v, s, S);
      }
    }
    if constexpr (!LAST) {
      if (ex.single()) lane_sync<LAYOUT, T, G>(g);  // write-after-read on the single buffer
      double2* sm = ex.next();
      // scatter: out[(b/Ns)*Ns*Rp + b%Ns + r*Ns] = v[s + r*S]
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const int b = t + s * T;
        const int base = (b & ~(Ns - 1)) * Rp + (b & (Ns - 1));
#pragma unroll
        for (int r = 0; r < Rp; ++r) sm[slot<LAYOUT, N, G>(base + r * Ns, g)] = v[s + r * S];
      }
      lane_sync<LAYOUT, T, G>(g);
#pragma unroll
      for (int m = 0; m < R; ++m) v[m] = sm[slot<LAYOUT, N, G>(t + m * T, g)];
      Stockham<N, R, G, INV, Ns * Rp, LAYOUT, NEXT_OFF, CM>::run(v, ex, t, g, ptw, wc);
    }
  }
};

// Full FFT of length N on the lane; x[t + m*T] in v[m] before and after.
// Every thread of the lane (LAYOUT 1) / CTA (LAYOUT 0) must call it.
template <int N, int R, int G, bool INV, int LAYOUT = 0>
__device__ __forceinline__ void fft_lane(double2 (&v)[R], Ex& ex, int t, int g, const double2* tw) {
  if constexpr (N == 1) {
    return;
  } else {
    Stockham<N, R, G, INV, 1, LAYOUT>::run(v, ex, t, g, tw);
  }
}

// fft_lane with the twiddle cache (TwCache): CM = 1 fills wc, CM = 2 uses it.
template <int N, int R, int G, bool INV, int LAYOUT, int CM, int CK>
__device__ __forceinline__ void fft_lane_c(double2 (&v)[R], Ex& ex, int t, int g, const double2* tw,
                                           double2 (&wc)[CK]) {
  Stockham<N, R, G, INV, 1, LAYOUT, 0, CM>::run(v, ex, t, g, tw, wc);
}

// Slot of the mirror exchanges (write at pos, read at N - pos): no swizzle.
// Ascending and descending runs of consecutive positions are both free of
// bank conflicts in the plain layouts, while the Stockham swizzles make the
// descending run collide across its 8-position blocks (ncu: 2x wavefronts).
template <int LAYOUT, int N, int G>
__device__ __forceinline__ int mslot(int pos, int g) {
  if constexpr (LAYOUT == 1) return g * N + pos;
  else return pos * G + g;
}

// Exchange helper: value at position (N - pos) mod N for every register
// (used by the Hartley post-processing).  One barrier (lane_sync).
template <int N, int R, int G, int LAYOUT = 0>
__device__ __forceinline__ void mirror_lane(const double2 (&v)[R], double2 (&w)[R], Ex& ex, int t, int g) {
  constexpr int T = N / R;
  if (ex.single()) lane_sync<LAYOUT, T, G>(g);
  double2* sm = ex.next();
#pragma unroll
  for (int m = 0; m < R; ++m) sm[mslot<LAYOUT, N, G>(t + m * T, g)] = v[m];
  lane_sync<LAYOUT, T, G>(g);
#pragma unroll
  for (int m = 0; m < R; ++m) {
    const int pos = t + m * T;
    const int mp = (N - pos) & (N - 1);
    w[m] = sm[mslot<LAYOUT, N, G>(mp, g)];
  }
}

// Two packed real sequences a + i b -> (Hartley(a), Hartley(b)) given
// Z = FFT(a + i b): H_a[f] = (zr - zi + wr + wi)/2, H_b[f] = (zr + zi - wr + wi)/2
// with W = Z[N - f].  Returned packed as H_a + i H_b.
__device__ __forceinline__ double2 hartley_split(double2 z, double2 w) {
  return make_double2(0.5 * ((z.x - z.y) + (w.x + w.y)), 0.5 * ((z.x + z.y) - (w.x - w.y)));
}

// Hartley post-processing in place: v[m] <- hartley_split(v[m], V[N - pos])
// (two packed real sequences -> their Hartley transforms), one exchange and
// no second register array.
template <int N, int R, int G, int LAYOUT = 0>
__device__ __forceinline__ void hartley_lane(double2 (&v)[R], Ex& ex, int t, int g) {
  constexpr int T = N / R;
  if (ex.single()) lane_sync<LAYOUT, T, G>(g);
  double2* sm = ex.next();
#pragma unroll
  for (int m = 0; m < R; ++m) sm[mslot<LAYOUT, N, G>(t + m * T, g)] = v[m];
  lane_sync<LAYOUT, T, G>(g);
#pragma unroll
  for (int m = 0; m < R; ++m) {
    const int mp = (N - (t + m * T)) & (N - 1);
    v[m] = hartley_split(v[m], sm[mslot<LAYOUT, N, G>(mp, g)]);
  }
}

// Cooperative copy of a small global table into shared memory.
__device__ __forceinline__ void load_table(double2* dst, const double2* __restrict__ src, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = __ldg(&src[i]);
}


}  // namespace fdg
