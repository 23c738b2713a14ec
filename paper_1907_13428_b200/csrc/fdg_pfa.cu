// fdg_pfa.cu — 1023-point prime-factor Hartley passes of the 2-level T. Chan
// preconditioner (BASELINE config 1: 256 slices of 1023 x 1023).
//
// Reference: the per-level circulant solve of CirculantPreconditioner
// (circulant.cpp:49-67: forward DFT, divide by the eigenvalues, inverse DFT)
// restricted to the two spatial levels, with the level eigenvalues of
// circulant.cpp:10-26.  The eigenvalues of the T. Chan circulants of the
// symmetric Riesz factors are real and even, so per slice
//   z = (1 / (n1 n2)) H2 H1 D H1 H2 r,   D[k][j] = 1 / (lam1[k] + lam2[j])
// with H the real Hartley transform along an axis; this is
// what the generic Bluestein path (fdg_api.cu pc2_apply_dev) evaluates in 9
// passes for any level size.  For n = 1023 = 33 x 31 (33 = 3 x 11) the DFT
// has a twiddle-free prime-factor (Good-Thomas) decomposition, so each
// Hartley transform is a register-resident DFT_31 pass, one shared-memory
// exchange and a register-resident DFT_33 (= DFT_3 x DFT_11) pass:
//   input  n = (31 a + 33 b) mod 1023          a < 33, b < 31
//   output k = (496 k1 + 528 k2) mod 1023       (496 = 31 (31^-1 mod 33), 528 = 33 (33^-1 mod 31))
//   X[k] = sum_a W33^(a k1) sum_b W31^(b k2) x[n]
// and inside DFT_33: a = (11 i + 3 j) mod 33, k1 = (22 c + 12 d) mod 33.
// Three passes, 6N doubles of HBM traffic (SURVEY 8d's 2-level model):
//   k_pfa_hrow  (rows, x2):  r -> H2 r
//   k_pfa_hcol  (columns, x1, in place): H1 -> divide by lam1[k] + lam2[j] -> H1
//   k_pfa_hrow  (rows, x2):  -> (1 / (n1 n2)) H2, = z
// Lane = two real fibres packed as a + i b (one complex DFT, Hartley split by
// the mirror X[N - k]).  A lane is served by 33 threads: thread a runs the
// DFT_31 of input column a, thread k2 < 31 the DFT_33 of output row k2.  A
// CTA holds G = 7 lanes (231 working threads of 256): staging for the next
// tile (2G fibres, cp.async) + one exchange area (G lanes), 224 KB.
#include <cuda_runtime.h>

#include <type_traits>

#include "fdg_fft.cuh"
#include "fdg_internal.h"
#include "fdg_launch.cuh"
#include "fdg_passes.cuh"
#include "fdg_pfa_tab.h"

namespace fdg {
namespace {

constexpr int PN = 1023;     // transform length
constexpr int PA = 33;       // outer factor (3 x 11), threads per lane
constexpr int PB = 31;       // inner factor
constexpr int PH = 16;       // mirror-pair rounds: k = t + 33 m < 512 for m < 16
// lanes per CTA of the row / column passes (G lanes = 33 G working threads)
#ifndef FDG_PFA_GROW
#define FDG_PFA_GROW 7
#endif
#ifndef FDG_PFA_GCOL
#define FDG_PFA_GCOL 7
#endif
#ifndef FDG_PFA_TMA
#define FDG_PFA_TMA 1  // bulk-copy (TMA) staging of the row passes
#endif
template <int G>
struct PCfg {
  static constexpr int THREADS = (PA * G + 31) / 32 * 32;
  static constexpr size_t SMEM = 2 * (size_t)G * PN * sizeof(double2);  // staging + exchange
  static constexpr int MINB = SMEM <= 113 * 1024 ? 2 : 1;
};

// cos / sin (2 pi j / P), j < P (fdg_pfa_tab.h, scripts/gen_pfa_consts.py)
__constant__ double kC3[3] = FDG_PFA_C3;
__constant__ double kS3[3] = FDG_PFA_S3;
__constant__ double kC11[11] = FDG_PFA_C11;
__constant__ double kS11[11] = FDG_PFA_S11;
__constant__ double kC31[31] = FDG_PFA_C31;
__constant__ double kS31[31] = FDG_PFA_S31;

template <int P>
__device__ __forceinline__ double twc(int j) {
  return P == 3 ? kC3[j] : (P == 11 ? kC11[j] : kC31[j]);
}
template <int P>
__device__ __forceinline__ double tws(int j) {
  return P == 3 ? kS3[j] : (P == 11 ? kS11[j] : kS31[j]);
}

// cos / sin (2 pi k m / 31) for m, k = 1..15: the DFT_31 output loop runs
// over m at run time (uniform constant loads), which keeps ptxas from
// interleaving all 15 outputs and spilling.
struct Tab31 {
  double c[15][15], s[15][15];
};
__constant__ Tab31 kT31 = {FDG_PFA_T31C, FDG_PFA_T31S};

// Forward DFT of odd prime length P in place (natural order), X_m =
// sum_n x_n exp(-2 pi i n m / P), by the symmetric pair algorithm:
// s_k = x_k + x_{P-k}, d_k = x_k - x_{P-k};  X_m = A_m - i B_m,
// X_{P-m} = A_m + i B_m with A_m = x_0 + sum_k cos(2 pi k m / P) s_k and
// B_m = sum_k sin(2 pi k m / P) d_k.
template <int P, class Put>
__device__ __forceinline__ void dft_odd(const double2 (&x)[P], Put&& put) {
  constexpr int H = (P - 1) / 2;
  double2 s[H], d[H];
#pragma unroll
  for (int k = 1; k <= H; ++k) {
    s[k - 1] = cadd(x[k], x[P - k]);
    d[k - 1] = csub(x[k], x[P - k]);
  }
  const double2 x0 = x[0];
  double2 sum = x0;
#pragma unroll
  for (int k = 0; k < H; ++k) sum = cadd(sum, s[k]);
  put(0, sum);
  if constexpr (P == 31) {
    // outputs m and m + 8 per iteration: 8 independent accumulation chains
    auto one = [&](int m, double2& A, double2& B) {
      const double c0 = kT31.c[m - 1][0], s0 = kT31.s[m - 1][0];
      A = make_double2(fma(c0, s[0].x, x0.x), fma(c0, s[0].y, x0.y));
      B = make_double2(s0 * d[0].x, s0 * d[0].y);
    };
    auto step = [&](int m, int k, double2& A, double2& B) {
      const double c = kT31.c[m - 1][k - 1], sn = kT31.s[m - 1][k - 1];
      A.x = fma(c, s[k - 1].x, A.x);
      A.y = fma(c, s[k - 1].y, A.y);
      B.x = fma(sn, d[k - 1].x, B.x);
      B.y = fma(sn, d[k - 1].y, B.y);
    };
    auto out = [&](int m, const double2& A, const double2& B) {
      put(m, make_double2(A.x + B.y, A.y - B.x));
      put(P - m, make_double2(A.x - B.y, A.y + B.x));
    };
    // one basic block per output pair with compile-time m: the cos / sin
    // factors become constant-bank operands of the FMAs (the run-time m of the
    // rolled loop cost an LDC per factor: 30% of the pass's stall samples),
    // and ptxas still cannot interleave the pairs (which spilled)
    auto pair = [&](auto mc) {
      constexpr int m = decltype(mc)::value;
      double2 A, B, A2, B2;
      one(m, A, B);
      one(m + 8, A2, B2);
#pragma unroll
      for (int k = 2; k <= H; ++k) {
        step(m, k, A, B);
        step(m + 8, k, A2, B2);
      }
      out(m, A, B);
      out(m + 8, A2, B2);
    };
#pragma unroll 1
    for (int m = 1; m <= 7; ++m) {
      switch (m) {
        case 1: pair(std::integral_constant<int, 1>{}); break;
        case 2: pair(std::integral_constant<int, 2>{}); break;
        case 3: pair(std::integral_constant<int, 3>{}); break;
        case 4: pair(std::integral_constant<int, 4>{}); break;
        case 5: pair(std::integral_constant<int, 5>{}); break;
        case 6: pair(std::integral_constant<int, 6>{}); break;
        default: pair(std::integral_constant<int, 7>{}); break;
      }
    }
    {
      double2 A, B;
      one(8, A, B);
#pragma unroll
      for (int k = 2; k <= H; ++k) step(8, k, A, B);
      out(8, A, B);
    }
  } else {
#pragma unroll
    for (int m = 1; m <= H; ++m) {
      double2 A = x0, B;
#pragma unroll
      for (int k = 1; k <= H; ++k) {
        const int j = (k * m) % P;
        const double c = twc<P>(j), sn = tws<P>(j);
        A.x = fma(c, s[k - 1].x, A.x);
        A.y = fma(c, s[k - 1].y, A.y);
        if (k == 1) {
          B = make_double2(sn * d[0].x, sn * d[0].y);
        } else {
          B.x = fma(sn, d[k - 1].x, B.x);
          B.y = fma(sn, d[k - 1].y, B.y);
        }
      }
      // outputs leave as soon as they are formed (the inputs stay live)
      put(m, make_double2(A.x + B.y, A.y - B.x));
      put(P - m, make_double2(A.x - B.y, A.y + B.x));
    }
  }
}

// Opaque copy of a loop-invariant value: index arithmetic derived from it is
// recomputed per tile instead of being hoisted out of the tile loop (31 + 62
// hoisted gather / mirror offsets push the kernels into spills).
__device__ __forceinline__ int opaque(int v) {
  int r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
  return r;
}

// Slot of X[k] in the exchange area after pfa_dft (CRT order): k mod 31
// rows of 33, k mod 33 within the row.  MirrorSlots walks the slots of
// k = t + 33 m and of its mirror 1023 - k for m = 0, 1, ... incrementally
// (k mod 33 = t, k mod 31 = (t + 2 m) mod 31).
struct MirrorSlots {
  int q, ta, tb;
  __device__ __forceinline__ explicit MirrorSlots(int t) : q(t % PB), ta(t), tb(t == 0 ? 0 : PA - t) {}
  __device__ __forceinline__ int k() const { return q * PA + ta; }
  __device__ __forceinline__ int km() const { return (q == 0 ? 0 : PB - q) * PA + tb; }
  __device__ __forceinline__ void next() {
    q += 2;
    if (q >= PB) q -= PB;
  }
};

// The lane's DFT of x = xa + i xb (two real fibres, src(n) = (xa[n], xb[n]))
// into the lane's exchange area E (1023 double2), X[k] at E[xslot(k)].
// Every thread of the CTA calls it (CTA barriers inside); `act`: the thread
// serves a lane (thread a = t < 33 of pass A, k2 = t < 31 of pass B).
// `freed()` runs once every gather is done (the source area may be reused;
// E is written only after it).
template <class FS, class FR>
__device__ __forceinline__ void pfa_dft(double2* E, int t, bool act, FS&& src, FR&& freed) {
  // Idle threads (no lane, or t >= 31 in pass B) run the same code on valid
  // addresses with their stores predicated off: branch-free blocks keep
  // ptxas' register allocation spill-free.
  double va[PB], vb[PB];
  {
    int idx = 31 * t;  // (31 a + 33 b) mod 1023, a = t
#pragma unroll
    for (int b = 0; b < PB; ++b) {
      const double2 z = src(idx);
      va[b] = z.x;
      vb[b] = z.y;
      idx += 33;
      if (idx >= PN) idx -= PN;
    }
  }
  __syncthreads();
  freed();
  {
    double2 v[PB];
#pragma unroll
    for (int b = 0; b < PB; ++b) v[b] = make_double2(va[b], vb[b]);
    // E[k2 * 33 + a]: pass-B thread k2 reads 33 consecutive entries
    dft_odd<PB>(v, [&](int k2, double2 val) {
      if (act) E[k2 * PA + t] = val;
    });
  }
  __syncthreads();
  const bool actb = act && t < PB;
  const int tb = t < PB ? t : PB - 1;
  double2 r[3][11];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 11; ++j) r[i][j] = E[tb * PA + (11 * i + 3 * j) % PA];
  __syncthreads();  // every pass-B read done: E is overwritten with X below
#pragma unroll
  for (int j = 0; j < 11; ++j) {
    const double2 u[3] = {r[0][j], r[1][j], r[2][j]};
    dft_odd<3>(u, [&](int c, double2 val) { r[c][j] = val; });
  }
  // X[k] with k = k1 (mod 33), k = k2 (mod 31) at E[k2 * 33 + k1]
  // (k1 = (22 c + 12 d) mod 33, k2 = t)
#pragma unroll
  for (int c = 0; c < 3; ++c)
    dft_odd<11>(r[c], [&](int d, double2 val) {
      if (actb) E[tb * PA + (22 * c + 12 * d) % PA] = val;
    });
  __syncthreads();
}

// Row pass along x2 (rows of 1023 contiguous doubles): out = scale * H2 in.
template <int PG>
__global__ void __launch_bounds__(PCfg<PG>::THREADS, PCfg<PG>::MINB)
    k_pfa_hrow(const double* __restrict__ in, double* __restrict__ out, long F, double scale) {
  constexpr int PTHREADS = PCfg<PG>::THREADS;
  extern __shared__ double2 smem_raw[];
  double* S = reinterpret_cast<double*>(smem_raw);  // 2G fibres of the tile
  double2* Ex = smem_raw + PG * PN;                  // G lanes
  pdl_trigger();
  pdl_wait();
  const int tid = threadIdx.x;
  const int g = tid / PA, t0 = tid - g * PA;
  const bool act = g < PG;
  const int gl = act ? g : 0;  // idle threads shadow lane 0 (stores off)
  double2* E = Ex + gl * PN;
  const long ntiles = (F + 2 * PG - 1) / (2 * PG);
  // staging: one bulk copy (TMA) of the tile's rows per tile, completion on
  // an mbarrier (F even: every tile is a multiple of 16 bytes), else
  // per-thread cp.async
  __shared__ alignas(8) unsigned long long bar;
  const bool tma = FDG_PFA_TMA && (F & 1) == 0;
  unsigned ph = 0;
  auto stage = [&](long tile) {
    const long r0 = tile * 2 * PG;
    const long nr = F - r0 < 2 * PG ? F - r0 : 2 * PG;
    const int nd = (int)(nr * PN);
    const double* src = in + r0 * PN;
    if (tma) {
      if (tid == 0) {
        fence_proxy_async();
        mbar_expect_tx(&bar, 8u * nd);
        bulk_g2s(S, src, 8u * nd, &bar);
      }
    } else {
      for (int i = 2 * tid; i + 1 < nd; i += 2 * PTHREADS) cp_async16(S + i, src + i);
      if ((nd & 1) && tid == 0) S[nd - 1] = src[nd - 1];
      cp_async_commit();
    }
  };
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_init_fence();
  }
  __syncthreads();
  if (blockIdx.x < ntiles) stage(blockIdx.x);
  for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long f = tile * 2 * PG + 2 * g;  // the lane's first row
    const bool va = act && f < F, vb = act && f + 1 < F;
    if (tma) {
      mbar_wait(&bar, ph);
      ph ^= 1;
    } else {
      cp_async_wait<0>();
      __syncthreads();
    }
    const int t = opaque(t0);
    const double* ra = S + 2 * gl * PN;
    pfa_dft(
        E, t, act, [&](int n) { return make_double2(va ? ra[n] : 0.0, vb ? ra[PN + n] : 0.0); },
        [&] {  // S free: the next tile's rows stream in during the rest of the transform
          if (tile + (long)gridDim.x < ntiles) stage(tile + gridDim.x);
        });
    if (va) {
      double* oa = out + f * PN;
      // mirror pairs (k, 1023 - k), k = t + 33 m < 512: each X read once
      MirrorSlots ms(t);
#pragma unroll 4
      for (int m = 0; m < PH; ++m, ms.next()) {
        const int k = t + PA * m;
        if (k < PN / 2 + 1) {
          const double2 zk = E[ms.k()], zm = E[ms.km()];
          const double2 h = hartley_split(zk, zm);
          oa[k] = scale * h.x;
          if (vb) oa[PN + k] = scale * h.y;
          if (k) {
            const double2 hm = hartley_split(zm, zk);
            oa[PN - k] = scale * hm.x;
            if (vb) oa[2 * PN - k] = scale * hm.y;
          }
        }
      }
    }
  }
}

// Column pass along x1, in place on data[o][i][j] (n1 = 1023 rows of C
// columns per slice): H1, divide by lam1[k] + lam2[j], H1.  Tile = 2G = 14
// columns of one slice (the last tile of a slice may be narrower).
template <int PG>
__global__ void __launch_bounds__(PCfg<PG>::THREADS, PCfg<PG>::MINB)
    k_pfa_hcol(double* __restrict__ data, int nt, int C, const double* __restrict__ lam1,
               const double* __restrict__ lam2) {
  constexpr int PTHREADS = PCfg<PG>::THREADS;
  constexpr int PW = 2 * PG;  // columns per tile
  extern __shared__ double2 smem_raw[];
  double* S = reinterpret_cast<double*>(smem_raw);  // [1023][PW]
  double2* Ex = smem_raw + PG * PN;
  pdl_trigger();
  pdl_wait();
  const int tid = threadIdx.x;
  const int g = tid / PA, t0 = tid - g * PA;
  const bool act = g < PG;
  const int gl = act ? g : 0;  // idle threads shadow lane 0 (stores off)
  double2* E = Ex + gl * PN;
  const int ncb = (C + PW - 1) / PW;
  const long ntiles = (long)nt * ncb;
  constexpr int CRT = PTHREADS / PW;           // tile rows covered per step of the copy loops
  const int cj = tid % PW, cr = tid / PW;      // copy loops: column and first row of the thread
  auto stage = [&](long tile) {
    const long o = tile / ncb;
    const int c0 = (int)(tile - o * ncb) * PW;
    const int nc = C - c0 < PW ? C - c0 : PW;
    const double* src = data + o * PN * (long)C + c0;
    // thread -> (column cj, rows cr, cr + CRT, ...): no index division per element
    if (cr < CRT && cj < nc) {
      const double* sp = src + (long)cr * C + cj;
      unsigned d = (unsigned)__cvta_generic_to_shared(S + cr * PW + cj);
      for (int pos = cr; pos < PN; pos += CRT) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(sp));
        sp += (long)CRT * C;
        d += CRT * PW * (unsigned)sizeof(double);
      }
    }
  };
  if (blockIdx.x < ntiles) stage(blockIdx.x);
  cp_async_commit();
  for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long o = tile / ncb;
    const int c0 = (int)(tile - o * ncb) * PW;
    const int nc = C - c0 < PW ? C - c0 : PW;
    const bool va = act && 2 * g < nc, vb = act && 2 * g + 1 < nc;
    cp_async_wait<0>();
    __syncthreads();
    const int t = opaque(t0);
    const double* sc = S + 2 * gl;
    pfa_dft(
        E, t, act,
        [&](int n) {
          const double2 z = *reinterpret_cast<const double2*>(sc + n * PW);
          return make_double2(va ? z.x : 0.0, vb ? z.y : 0.0);
        },
        [] {});
    // Hartley split and the spectral division, positions k = t + 33 m, into
    // the staging area (free once the gathers are done: the next tile is
    // staged only after the second transform's gathers)
    // (branch-free: idle threads compute on lane 0's slots, stores predicated)
    double2* Sh = reinterpret_cast<double2*>(S) + gl * PN;
    {
      const int ca = c0 + 2 * gl;
      const double l2a = __ldg(&lam2[ca]);
      const double l2b = vb ? __ldg(&lam2[ca + 1]) : l2a;
      // lambda_1 of the thread's 16 pair positions, loaded as one batch (the
      // spectrum is even, lam1[1023 - k] = lam1[k], checked at creation)
      double l1v[PH];
#pragma unroll
      for (int m = 0; m < PH; ++m) l1v[m] = __ldg(&lam1[t + PA * m]);
      auto divide = [&](double2 z, int k, double l1) {
        const double da = l1 + l2a, db = l1 + l2b;
        const double inv = frcp(da * db);  // one reciprocal for both columns
        if (act) Sh[k] = make_double2(z.x * (db * inv), vb ? z.y * (da * inv) : 0.0);
      };
      MirrorSlots ms(t);
#pragma unroll
      for (int m = 0; m < PH; ++m, ms.next()) {
        const int k = t + PA * m;
        if (k < PN / 2 + 1) {  // mirror pair (k, 1023 - k)
          const double2 zk = E[ms.k()], zm = E[ms.km()];
          divide(hartley_split(zk, zm), k, l1v[m]);
          if (k) divide(hartley_split(zm, zk), PN - k, l1v[m]);
        }
      }
    }
    __syncthreads();  // every value of the divided spectrum in Sh
    pfa_dft(E, t, act, [&](int n) { return Sh[n]; },
            [&] {  // staging area free: the next tile streams in during the rest
              if (tile + (long)gridDim.x < ntiles) stage(tile + gridDim.x);
              cp_async_commit();
            });
    // Hartley split into registers (mirror pairs, each X read once), then
    // the tile goes out through the exchange area as [pos][PW] rows (8-byte
    // stores of whole row segments; storing the lanes' columns directly
    // scatters every warp store over 32 rows)
    double2 h[PH], hm[PH];
    {
      MirrorSlots ms(t);
#pragma unroll
      for (int m = 0; m < PH; ++m, ms.next()) {
        const double2 zk = E[ms.k()], zm = E[ms.km()];  // (m = 15, t > 16: unused)
        h[m] = hartley_split(zk, zm);
        hm[m] = hartley_split(zm, zk);
      }
    }
    __syncthreads();  // mirror reads done
    double* Et = reinterpret_cast<double*>(Ex);  // [1023][PW] (G lanes x 1023 double2 = 1023 x PW doubles)
#pragma unroll
    for (int m = 0; m < PH; ++m) {
      const int k = t + PA * m;
      if (act && k < PN / 2 + 1) {
        *reinterpret_cast<double2*>(Et + k * PW + 2 * g) = h[m];
        if (k) *reinterpret_cast<double2*>(Et + (PN - k) * PW + 2 * g) = hm[m];
      }
    }
    __syncthreads();
    {
      double* dst = data + o * PN * (long)C + c0;
      if (cr < CRT && cj < nc) {
        double* dp = dst + (long)cr * C + cj;
        const double* ep = Et + cr * PW + cj;
        for (int pos = cr; pos < PN; pos += CRT) {
          *dp = *ep;
          dp += (long)CRT * C;
          ep += CRT * PW;
        }
      }
    }
    __syncthreads();  // E reads done before the next tile's pass A
  }
}

}  // namespace

bool pfa_supported(int n) { return n == PN; }

cudaError_t launch_pfa_hrow(cudaStream_t st, LaunchCounter* lc, const double* in, double* out, long F,
                            double scale) {
  using Cf = PCfg<FDG_PFA_GROW>;
  int cap = 0;
  cudaError_t e = prep<k_pfa_hrow<FDG_PFA_GROW>>(Cf::SMEM, Cf::THREADS, cap);
  if (e != cudaSuccess) return e;
  count(lc);
  const long tiles = (F + 2 * FDG_PFA_GROW - 1) / (2 * FDG_PFA_GROW);
  return pdl_launch(PDL_PROW, k_pfa_hrow<FDG_PFA_GROW>, clamp_grid(tiles, cap), Cf::THREADS, Cf::SMEM, st, in,
                    out, F, scale);
}

cudaError_t launch_pfa_hcol(cudaStream_t st, LaunchCounter* lc, double* data, int nt, int C, const double* lam1,
                            const double* lam2) {
  using Cf = PCfg<FDG_PFA_GCOL>;
  int cap = 0;
  cudaError_t e = prep<k_pfa_hcol<FDG_PFA_GCOL>>(Cf::SMEM, Cf::THREADS, cap);
  if (e != cudaSuccess) return e;
  count(lc);
  const long tiles = (long)nt * ((C + 2 * FDG_PFA_GCOL - 1) / (2 * FDG_PFA_GCOL));
  return pdl_launch(PDL_PCOL, k_pfa_hcol<FDG_PFA_GCOL>, clamp_grid(tiles, cap), Cf::THREADS, Cf::SMEM, st, data,
                    nt, C, lam1, lam2);
}

}  // namespace fdg
