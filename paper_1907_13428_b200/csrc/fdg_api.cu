// fdg_api.cu — host side of the C ABI (include/fdg.h).
//
// Mirrors the reference's operator / preconditioner / Krylov / ADMM entry
// points (/root/reference/proj/include/fdeopt/{toeplitz,circulant,admm}.hpp)
// over device-resident state.  Per Krylov iteration only two scalars (p^T S p
// and |r|^2) cross to the host, for the reference's convergence and
// breakdown checks (admm.cpp:143-158).
#include <atomic>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <functional>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/fdg.h"
#include "fdg_fft.cuh"
#include "fdg_internal.h"

using fdg::AxisSym;
using fdg::LaunchCounter;
using fdg::PcTables;
using fdg::RedSlot;
using fdg::TimeFactor;

namespace {

thread_local std::string g_err;
thread_local int g_num = FDG_NUM_NONE;

struct Error {
  fdg_status code;
  std::string msg;
  int num = FDG_NUM_NONE;
};

[[noreturn]] void fail(fdg_status code, const std::string& msg, int num = FDG_NUM_NONE) {
  throw Error{code, msg, num};
}

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(FDG_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
fdg_status guard(F&& f) {
  try {
    f();
    g_num = FDG_NUM_NONE;
    return FDG_OK;
  } catch (const Error& e) {
    g_err = e.msg;
    g_num = e.num;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "out of host memory";
    return FDG_ENOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return FDG_EINVAL;
  }
}

// ------------------------------------------------------- device buffers
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  explicit DevBuf(size_t b) { alloc(b); }
  void alloc(size_t b) {
    release();
    if (b == 0) b = 8;
    cudaError_t e = cudaMalloc(&p, b);
    if (e != cudaSuccess) {
      p = nullptr;
      fail(e == cudaErrorMemoryAllocation ? FDG_ENOMEM : FDG_ECUDA,
           std::string("cudaMalloc: ") + cudaGetErrorString(e));
    }
    bytes = b;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  double* d() const { return static_cast<double*>(p); }
  double2* c() const { return static_cast<double2*>(p); }
};

bool is_pow2(long v) { return v >= 1 && (v & (v - 1)) == 0; }
int pow2_ceil(long v) {
  int L = 1;
  while (L < v) L <<= 1;
  return L;
}

// ------------------------------------------------- host setup arithmetic
const long double kPi = 3.141592653589793238462643383279502884L;

std::vector<double> twiddles(int L) {
  std::vector<double> w(2 * (size_t)L);
  for (int k = 0; k < L; ++k) {
    long double a = -2.0L * kPi * (long double)k / (long double)L;
    double c = (double)cosl(a), s = (double)sinl(a);
    if (4 * k == L) { c = 0.0; s = -1.0; }
    if (2 * k == L) { c = -1.0; s = 0.0; }
    if (4 * k == 3 * L) { c = 0.0; s = 1.0; }
    if (k == 0) { c = 1.0; s = 0.0; }
    w[2 * k] = c;
    w[2 * k + 1] = s;
  }
  return w;
}

// Per-pass Stockham twiddle table of length N for the device FFT plan
// (fdg_fft.cuh Stockham: pass with stride Ns > 1 owns (Rp-1)*Ns entries,
// entry (r-1)*Ns + j = W_N^(j r N/(Ns Rp))).
// cas(2 pi m / n) = cos + sin, m < n, in long double (dense Hartley path)
std::vector<double> cas_table(int n) {
  std::vector<double> c((size_t)n);
  for (int m = 0; m < n; ++m) {
    const long double a = 2.0L * kPi * (long double)m / (long double)n;
    c[m] = (double)(cosl(a) + sinl(a));
  }
  return c;
}

size_t pc_size(int nt, int n1, int n2) { return (size_t)nt * n1 * n2; }

std::vector<double> stockham_twiddles(int N) {
  const std::vector<double> w = twiddles(N);
  std::vector<double> out(2 * (size_t)std::max(N, 1), 0.0);
  const int R = fdg::fft_radix(N);
  int off = 0;
  for (int Ns = 1; Ns < N;) {
    const int Rp = std::min(R, N / Ns);
    if (Ns > 1) {
      for (int r = 1; r < Rp; ++r)
        for (int j = 0; j < Ns; ++j) {
          const long k = ((long)j * r * (N / (Ns * Rp))) % N;
          const size_t idx = (size_t)off + (size_t)(r - 1) * Ns + j;
          out[2 * idx] = w[2 * k];
          out[2 * idx + 1] = w[2 * k + 1];
        }
      off += (Rp - 1) * Ns;
    }
    Ns *= Rp;
  }
  return out;
}

// Full length-L spectrum of the circulant embedding of a Toeplitz factor:
// c[k] = col[k] (k < n), c[L-k] = row[k] (0 < k < n)  (toeplitz.cpp:46-58 with
// L >= 2n-1 instead of exactly 2n).  Direct sum in long double.
std::vector<double> embed_symbol_full(const std::vector<double>& col, const std::vector<double>& row, int L) {
  const int n = (int)col.size();
  std::vector<long double> cs(L), sn(L);
  for (int k = 0; k < L; ++k) {
    const long double a = -2.0L * kPi * (long double)k / (long double)L;
    cs[k] = cosl(a);
    sn[k] = sinl(a);
  }
  std::vector<std::pair<int, long double>> nz;
  for (int k = 0; k < n; ++k)
    if (col[k] != 0.0) nz.push_back({k, (long double)col[k]});
  for (int k = 1; k < n; ++k)
    if (row[k] != 0.0) nz.push_back({L - k, (long double)row[k]});
  std::vector<double> out(2 * (size_t)L);
  for (int f = 0; f < L; ++f) {
    long double re = 0.0L, im = 0.0L;
    for (auto& [k, v] : nz) {
      const int idx = (int)(((long long)f * k) % L);
      re += v * cs[idx];
      im += v * sn[idx];
    }
    out[2 * f] = (double)re;
    out[2 * f + 1] = (double)im;
  }
  return out;
}

// Bluestein chirp c_m = exp(i pi m^2 / n), m < n (exact m^2 mod 2n).
std::vector<double> chirp_table(int n) {
  std::vector<double> c(2 * (size_t)n);
  for (int m = 0; m < n; ++m) {
    const long long q = ((long long)m * m) % (2LL * n);
    const long double a = kPi * (long double)q / (long double)n;
    c[2 * m] = (double)cosl(a);
    c[2 * m + 1] = (double)sinl(a);
  }
  return c;
}

// Length-L circulant-embedding spectrum of the symmetric complex Toeplitz
// matrix T_kj = c_{k-j} (chirp convolution): sum_{|m| < n} c_m W_L^(f m).
std::vector<double> chirp_symbol(int n, int L) {
  std::vector<long double> cs(L), sn(L), cr(n), ci(n);
  for (int k = 0; k < L; ++k) {
    const long double a = -2.0L * kPi * (long double)k / (long double)L;
    cs[k] = cosl(a);
    sn[k] = sinl(a);
  }
  for (int m = 0; m < n; ++m) {
    const long long q = ((long long)m * m) % (2LL * n);
    const long double a = kPi * (long double)q / (long double)n;
    cr[m] = cosl(a);
    ci[m] = sinl(a);
  }
  std::vector<double> out(2 * (size_t)L);
  for (int f = 0; f < L; ++f) {
    long double re = 0.0L, im = 0.0L;
    for (int m = -(n - 1); m < n; ++m) {
      const int am = m < 0 ? -m : m;
      const int idx = (int)((((long long)f * m) % L + L) % L);
      re += cr[am] * cs[idx] - ci[am] * sn[idx];
      im += cr[am] * sn[idx] + ci[am] * cs[idx];
    }
    out[2 * f] = (double)re;
    out[2 * f + 1] = (double)im;
  }
  return out;
}

// circulant.cpp:10-26: T. Chan first column and its DFT (direct, long double).
void tchan_host(int n, const double* col, const double* row, double* first_col, double* eigs) {
  std::vector<double> c(n);
  c[0] = col[0];
  for (int i = 1; i < n; ++i) c[i] = ((n - i) * col[i] + i * row[n - i]) / n;
  if (first_col) std::memcpy(first_col, c.data(), sizeof(double) * n);
  for (int j = 0; j < n; ++j) {
    long double re = 0.0L, im = 0.0L;
    for (int k = 0; k < n; ++k) {
      const long long jk = ((long long)j * k) % n;
      const long double a = -2.0L * kPi * (long double)jk / (long double)n;
      re += (long double)c[k] * cosl(a);
      im += (long double)c[k] * sinl(a);
    }
    eigs[2 * j] = (double)re;
    eigs[2 * j + 1] = (double)im;
  }
}

std::vector<double> frac_coeffs_host(double order, int count) {
  const bool valid = (order > 0.0 && order < 1.0) || (order > 1.0 && order < 2.0);
  if (!valid) fail(FDG_EINVAL, "fractional order must lie in (0,1) or (1,2), got " + std::to_string(order));
  if (count < 1) fail(FDG_EINVAL, "coefficient count must be >= 1");
  std::vector<double> g(count);
  g[0] = 1.0;
  for (int k = 1; k < count; ++k) g[k] = (1.0 - (order + 1.0) / k) * g[k - 1];
  return g;
}

}  // namespace

// ====================================================================== ctx
struct fdg_ctx_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  LaunchCounter lc;
  // reduction infrastructure shared by every handle of this context (all
  // work is ordered on one stream)
  DevBuf partials;
  DevBuf counters;
  size_t partial_cap = 0;
  double* pinned = nullptr;  // host staging for scalars
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr, ev3 = nullptr;

  void set_device() const { ck(cudaSetDevice(device), "cudaSetDevice"); }
  void ensure_partials(size_t cap) {
    if (cap <= partial_cap) return;
    partials.alloc(sizeof(double) * 4 * cap);
    partial_cap = cap;
  }
};

namespace {

// Device scalar block layout (per handle that reduces).
enum Scal {
  S_NB = 0,   // |rhs|^2
  S_XX,       // |x|^2
  S_RZ0,      // r.z ping
  S_RZ1,      // r.z pong
  S_PQ,       // p^T S p
  S_RR,       // |r|^2
  S_RR2,      // |r|^2 of the true residual
  S_ADMM,     // 4: r_eq, r_y, r_v, bad
  S_DINF = S_ADMM + 4,  // 2
  S_OBJ = S_DINF + 2,   // 2
  S_DOT = S_OBJ + 2,
  S_ONE,  // constant 1.0 (alpha of the fused residual r = b - 1 * S x)
  S_TOL,  // (tol |b|)^2 of the running solve (graph-driven iterations)
  S_COUNT
};

struct Scalars {
  DevBuf vals;      // double[S_COUNT]
  DevBuf counters;  // unsigned[S_COUNT]
  fdg_ctx ctx = nullptr;
  void init(fdg_ctx c) {
    ctx = c;
    vals.alloc(sizeof(double) * S_COUNT);
    counters.alloc(sizeof(unsigned) * S_COUNT);
    ck(cudaMemset(vals.p, 0, sizeof(double) * S_COUNT), "memset");
    ck(cudaMemset(counters.p, 0, sizeof(unsigned) * S_COUNT), "memset");
    const double one = 1.0;
    ck(cudaMemcpy(vals.d() + S_ONE, &one, sizeof(double), cudaMemcpyHostToDevice), "H2D");
  }
  double* at(int s) const { return vals.d() + s; }
  RedSlot slot(int s) const {
    return RedSlot{ctx->partials.d(), static_cast<unsigned*>(counters.p) + s, vals.d() + s};
  }
  // synchronous read of [s, s+cnt)
  void read(int s, int cnt, double* out) const {
    ck(cudaMemcpyAsync(ctx->pinned, vals.d() + s, sizeof(double) * cnt, cudaMemcpyDeviceToHost, ctx->stream),
       "scalar D2H");
    ck(cudaStreamSynchronize(ctx->stream), "stream sync");
    std::memcpy(out, ctx->pinned, sizeof(double) * cnt);
  }
};

}  // namespace

// ================================================================ operator
struct fdg_op_s {
  fdg_ctx ctx = nullptr;
  int nt = 0, n1 = 0, n2 = 0;
  double psi = 1.0;
  std::vector<double> tcol, trow, c1, r1, c2, r2;
  DevBuf sym1, tw1, sym2, tw2, symt, symt_adj, twt, sym2s;
  DevBuf twh1, twh2, twht, tws1, tws2, twst;  // split passes: L/2-point twiddles, W_L^j (j < L/2)
  DevBuf twq1a, twq1b, twq2a, twq2b, twqta, twqtb;  // Q-split passes: 256-point plan, W_L
  DevBuf symr1, symr2, symrt, symr2s;          // real symbols of symmetric factors
  AxisSym ax1, ax2;
  AxisSym ax2s;  // x2 axis with the stencil diagonal folded in: sym2 - c0 (row passes)
  TimeFactor tf;
  size_t N() const { return (size_t)nt * n1 * n2; }
  double scale1() const { return -psi / ax1.L; }
  double scale2() const { return -psi / ax2.L; }
  // symbol of the row passes (stencil diagonal folded in when kind == 1)
  const AxisSym& row_axis() const { return ax2s; }
};

namespace {

void upload(DevBuf& b, const std::vector<double>& h, cudaStream_t st) {
  b.alloc(sizeof(double) * h.size());
  ck(cudaMemcpyAsync(b.p, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice, st), "H2D");
  ck(cudaStreamSynchronize(st), "sync");
}

// Real parts of an interleaved complex table.
std::vector<double> real_parts(const std::vector<double>& c) {
  std::vector<double> r(c.size() / 2);
  for (size_t i = 0; i < r.size(); ++i) r[i] = c[2 * i];
  return r;
}

void build_axis(fdg_op_s* op, AxisSym& ax, DevBuf& sym, DevBuf* sym_adj, DevBuf& tw, DevBuf& twh, DevBuf& tws,
                DevBuf& symr, const std::vector<double>& col, const std::vector<double>& row, DevBuf& twq256,
                DevBuf& twqf) {
  const int n = (int)col.size();
  const int L = std::max(2, pow2_ceil(2L * n - 1));
  if (L > 2048) fail(FDG_EUNSUPPORTED, "fdg: factor size " + std::to_string(n) + " exceeds the compiled kernel set (n <= 1024)");
  ax.n = n;
  ax.L = L;
  // A symmetric factor (row == col, e.g. the Riesz factors) has a real, even
  // circulant spectrum: drop the rounding residue of the imaginary parts and
  // keep a real copy for the split passes (real symbol multiply).
  const bool symmetric = col == row;
  std::vector<double> spec = embed_symbol_full(col, row, L);
  if (symmetric) {
    for (int f = 0; f < L; ++f) spec[2 * f + 1] = 0.0;
    upload(symr, real_parts(spec), op->ctx->stream);
    ax.sym_re = ax.sym_adj_re = symr.d();
  }
  upload(sym, spec, op->ctx->stream);
  upload(tw, stockham_twiddles(L), op->ctx->stream);
  ax.sym = sym.c();
  ax.tw = tw.c();
  // split-spectrum passes (fdg_conv.cuh): M = L/2 point plan and W_L^j, j < M
  const int M = std::max(1, L / 2);
  upload(twh, stockham_twiddles(M), op->ctx->stream);
  std::vector<double> twist = twiddles(L);
  twist.resize(2 * (size_t)M);
  upload(tws, twist, op->ctx->stream);
  ax.twh = twh.c();
  ax.twist = tws.c();
  if (L >= 1024) {
    // Q-split passes (fdg_convq.cuh): 256-point plan and the full W_L table
    upload(twq256, stockham_twiddles(256), op->ctx->stream);
    upload(twqf, twiddles(L), op->ctx->stream);
    ax.tw256 = twq256.c();
    ax.twq = twqf.c();
  }
  ax.sym_adj = ax.sym;
  if (sym_adj && !symmetric) {
    upload(*sym_adj, embed_symbol_full(row, col, L), op->ctx->stream);
    ax.sym_adj = sym_adj->c();
  }
}

// B x into out (x != out): row pass (x2 + stencil) then x1 column pass
// (in place on out), then the general time pass if any.
void op_apply_dev(fdg_op_s* op, const double* x, double* out, bool adjoint) {
  cudaStream_t st = op->ctx->stream;
  LaunchCounter* lc = &op->ctx->lc;
  ck(fdg::launch_row_apply(st, lc, x, out, op->nt, op->n1, op->n2, op->row_axis(), op->scale2(), op->tf, op->psi, adjoint),
     "row pass");
  ck(fdg::launch_col_acc(st, lc, x, out, out, op->nt, op->n1, op->n2, op->ax1, op->scale1(), false), "x1 pass");
  if (op->tf.kind == 2)
    ck(fdg::launch_col_acc(st, lc, x, out, out, 1, op->nt, op->n1 * op->n2, op->tf.fft, op->psi / op->tf.fft.L,
                           adjoint),
       "t pass");
}

}  // namespace

// ================================================================== pc
struct fdg_pc_s {
  fdg_ctx ctx = nullptr;
  int kind = 3;  // 3: ADMM 3-level lambda_S (circulant.cpp); 2: per-slice 2-level spatial (BASELINE C1)
  int nt = 0, n1 = 0, n2 = 0;
  double psi = 1.0, rho = 1.0, delta = 1.0, gamma = 1.0;
  DevBuf lt, l1, l2, twt, tw1, tw2;
  DevBuf work;  // N doubles (standalone solve)
  // level sizes without a radix plan: dense Hartley axis transforms
  // (fdg_kernels.cu k_cas_axis), cas tables and an N-double scratch vector
  bool dense = false;
  DevBuf cas_t, cas_1, cas_2, dtmp;
  PcTables tab;
  // kind 2 (Bluestein passes, fdg_kernels.cu k_bs_*): chirps, real eigenvalues,
  // chirp convolution axes and two work buffers
  DevBuf c1, c2, lam1, lam2, bu, bv;
  DevBuf s1, t1, th1, ts1, s2, t2, th2, ts2;
  AxisSym bs1, bs2;
  int P2 = 0;
  size_t N() const { return (size_t)nt * n1 * n2; }
};

namespace {

// 2-level spatial preconditioner (BASELINE C1): per time slice
// z = F^-1 (F r / (lam1[i] + lam2[j])) with F the n1 x n2 DFT, evaluated as
// Hartley transforms (the eigenvalues of the T. Chan circulants of symmetric
// factors are real and even) of any size by Bluestein: x2 forward, x1
// forward + divide + x1 inverse, x2 inverse, 9 passes.
void pc2_apply_dev(fdg_pc_s* pc, const double* r, double* z) {
  cudaStream_t st = pc->ctx->stream;
  LaunchCounter* lc = &pc->ctx->lc;
  const long F = (long)pc->nt * pc->n1;
  const int Fp = (int)(F + (F & 1));
  const int n1 = pc->n1, n2 = pc->n2, P2 = pc->P2;
  const double2* c1 = pc->c1.c();
  const double2* c2 = pc->c2.c();
  double* u = pc->bu.d();
  double* v = pc->bv.d();
  TimeFactor none;
#ifndef FDG_PFA
#define FDG_PFA 1
#endif
  if (FDG_PFA && fdg::pfa_supported(n1) && fdg::pfa_supported(n2)) {
    // 1023 = 33 x 31: three prime-factor Hartley passes (fdg_pfa.cu)
    ck(fdg::launch_pfa_hrow(st, lc, r, u, F, 1.0), "pc2 pfa x2");
    ck(fdg::launch_pfa_hcol(st, lc, u, pc->nt, n2, pc->lam1.d(), pc->lam2.d()), "pc2 pfa x1");
    ck(fdg::launch_pfa_hrow(st, lc, u, z, F, 1.0 / ((double)n1 * n2)), "pc2 pfa x2 out");
    return;
  }
  if (F == Fp) {  // the pre-chirp rides in the convolution's load (k_row<.., CH>)
    ck(fdg::launch_row_apply(st, lc, r, v, 1, Fp, n2, pc->bs2, 1.0 / pc->bs2.L, none, 1.0, false, c2),
       "pc2 x2 pre + conv");
  } else {
    ck(fdg::launch_bs_pre_rows(st, lc, r, u, F, n2, c2), "pc2 x2 pre");
    ck(fdg::launch_row_apply(st, lc, u, v, 1, Fp, n2, pc->bs2, 1.0 / pc->bs2.L, none, 1.0, false), "pc2 x2 conv");
  }
  ck(fdg::launch_bs_rows_to_cols(st, lc, v, u, F, n1, n2, P2, c2, c1), "pc2 x2 post");
  ck(fdg::launch_col_acc(st, lc, u, nullptr, v, pc->nt, n1, P2, pc->bs1, 1.0 / pc->bs1.L, false), "pc2 x1 conv");
  ck(fdg::launch_bs_cols_filter(st, lc, v, u, pc->nt, n1, n2, P2, c1, pc->lam1.d(), pc->lam2.d()), "pc2 divide");
  ck(fdg::launch_col_acc(st, lc, u, nullptr, v, pc->nt, n1, P2, pc->bs1, 1.0 / pc->bs1.L, false), "pc2 x1 conv");
  ck(fdg::launch_bs_cols_to_rows(st, lc, v, u, F, n1, n2, P2, c1, c2), "pc2 x1 post");
  ck(fdg::launch_row_apply(st, lc, u, v, 1, Fp, n2, pc->bs2, 1.0 / pc->bs2.L, none, 1.0, false), "pc2 x2 conv");
  ck(fdg::launch_bs_post_rows(st, lc, v, z, F, n2, c2, 1.0 / ((double)n1 * n2)), "pc2 x2 post");
}

// z = S~^{-1} r via Hartley passes x2, x1, t(+divide), x1, x2.
// h may alias z (not r).  rdot != null: reduce r.z into red.
void pc_apply_dev(fdg_pc_s* pc, const double* r, double* z, double* h, const double* rdot, RedSlot red,
                  const int* guard = nullptr) {
  cudaStream_t st = pc->ctx->stream;
  LaunchCounter* lc = &pc->ctx->lc;
  const int F = pc->nt * pc->n1;
  RedSlot none{};
  if (pc->dense) {
    // any level sizes: dense Hartley along x2, x1, t, the 1/(N lambda_S)
    // scaling, then t, x1, x2 (the last into z; h may alias z)
    double* tmp = pc->dtmp.d();
    const int n1 = pc->n1, n2 = pc->n2, nt = pc->nt;
    const long sl = (long)n1 * n2;
    ck(fdg::launch_cas_axis(st, lc, r, tmp, (long)nt * n1, n2, 1, pc->cas_2.d()), "pc x2 fwd");
    ck(fdg::launch_cas_axis(st, lc, tmp, h, nt, n1, n2, pc->cas_1.d()), "pc x1 fwd");
    ck(fdg::launch_cas_axis(st, lc, h, tmp, 1, nt, sl, pc->cas_t.d()), "pc t fwd");
    ck(fdg::launch_lams_scale(st, lc, tmp, pc->tab), "pc divide");
    ck(fdg::launch_cas_axis(st, lc, tmp, h, 1, nt, sl, pc->cas_t.d()), "pc t inv");
    ck(fdg::launch_cas_axis(st, lc, h, tmp, nt, n1, n2, pc->cas_1.d()), "pc x1 inv");
    ck(fdg::launch_cas_axis(st, lc, tmp, z, (long)nt * n1, n2, 1, pc->cas_2.d()), "pc x2 inv");
    if (rdot) ck(fdg::launch_dot(st, lc, rdot, z, pc->N(), red), "pc r.z");
    return;
  }
  ck(fdg::launch_hartley_row(st, lc, r, h, F, pc->n2, pc->tab.tw_2, nullptr, none, guard), "pc x2 fwd");
  ck(fdg::launch_hartley_col(st, lc, h, pc->nt, pc->n1, pc->n2, pc->tab.tw_1, guard), "pc x1 fwd");
  ck(fdg::launch_t_filter(st, lc, h, pc->tab, guard), "pc t filter");
  ck(fdg::launch_hartley_col(st, lc, h, pc->nt, pc->n1, pc->n2, pc->tab.tw_1, guard), "pc x1 inv");
  ck(fdg::launch_hartley_row(st, lc, h, z, F, pc->n2, pc->tab.tw_2, rdot, red, guard), "pc x2 inv");
}

}  // namespace

// ================================================================= ADMM
struct fdg_admm_s {
  fdg_op_s* op = nullptr;
  fdg_pc_s* pc = nullptr;
  fdg_admm_desc desc{};
  size_t N = 0, slice = 0;
  int nt = 0;
  double psi = 1.0, v_lo = 0, v_hi = 0;
  // per-slice work (AdmmWork vectors are time-block constant, admm.cpp:52-79)
  std::vector<double> h_diag_j, h_diag_j2, h_m2, h_a2inv;
  DevBuf diag_j, diag_j2, m2, inv_m2, a2inv, a1;
  // state (AdmmState admm.hpp:28-32) and work vectors
  DevBuf y, v, z_y, z_v, p, w_y, w_v, ybar, By;
  DevBuf rhs, r_cache, tmp;
  DevBuf r, z, d, d2, u, w, vp;  // PCG: residual, preconditioned residual, directions (ping-pong), scratch
  Scalars sc;
  double inner_tol = 0.0;
  bool converged = false;
  int stagnations = 0;
  int iteration = 0;
  cudaEvent_t e0 = nullptr, e1 = nullptr, e2 = nullptr, e3 = nullptr;
  // speculative PCG: device pause flag, per-parity (pq, |r|^2) status, its
  // pinned host mirror and completion events
  // status words live in host-mapped pinned memory written by the control
  // kernel (no copy node in the stream); hseq[parity] = the sequence number
  // of the latest enqueue of an iteration of that parity
  DevBuf ctl;
  double* hstat = nullptr;
  double* hstat_dev = nullptr;
  // host-buffer solve (fdg_admm_pcg_host): copy stream, x0 landing buffer and
  // its nonzero flag (allocated on first use)
  cudaStream_t cstream = nullptr;
  cudaEvent_t ev_x0 = nullptr;
  cudaEvent_t ev_norms = nullptr;  // pcg_dev: |rhs|^2, |x|^2 landed on the host
  DevBuf x0buf, x0flag;
  int* x0flag_host = nullptr;  // pinned
  double seq = 0.0;
  double hseq[2] = {0.0, 0.0};
  // graph-driven PCG iterations (pcg_dev): instantiated graphs keyed by the
  // solution buffer and the parity of their first iteration
  struct PcgGraph {
    const double* x = nullptr;
    const double* rhs = nullptr;
    int parity = 0;
    cudaGraphExec_t exec = nullptr;
    unsigned long long kernels = 0;  // launches per body execution
    unsigned long long used = 0;
  };
  std::vector<PcgGraph> graphs;
  unsigned long long graph_tick = 0;
  ~fdg_admm_s() {
    for (auto& g : graphs)
      if (g.exec) cudaGraphExecDestroy(g.exec);
  }
};

namespace {

fdg::AdmmScalars admm_scalars(const fdg_admm_s* a) {
  return fdg::AdmmScalars{a->desc.rho, a->desc.delta, a->psi, a->desc.y_lo, a->desc.y_hi, a->v_lo, a->v_hi};
}

// q = S x (admm.cpp:87-98), fused: row(x) -> u; col(x,u) -> w, vp (+pq);
// row(w, vp) -> q.  pq lands in S_PQ.
// r_out != null: instead of q, r_out = b - S x (the reference's residual,
// admm.cpp:133-136 / 152-154) with |r_out|^2 reduced into red -- fused into
// the last pass as r_out = b - 1 * q.
void apply_S_dev(fdg_admm_s* a, const double* x, double* q, double* r_out = nullptr, const double* b = nullptr,
                 RedSlot red = RedSlot{}) {
  fdg_op_s* op = a->op;
  cudaStream_t st = op->ctx->stream;
  LaunchCounter* lc = &op->ctx->lc;
  const TimeFactor& tf = op->tf;
  TimeFactor none_tf;
  ck(fdg::launch_row_apply(st, lc, x, a->u.d(), op->nt, op->n1, op->n2, op->row_axis(), op->scale2(),
                           tf.kind == 1 ? tf : none_tf, op->psi, false),
     "S row");
  if (tf.kind == 2)
    ck(fdg::launch_col_acc(st, lc, x, a->u.d(), a->u.d(), 1, op->nt, op->n1 * op->n2, tf.fft, op->psi / tf.fft.L,
                           false),
       "S t fwd");
  ck(fdg::launch_col_s_mid(st, lc, x, a->u.d(), a->w.d(), a->vp.d(), op->nt, op->n1, op->n2, op->ax1, op->scale1(),
                           a->inv_m2.d(), a->a1.d(), a->sc.slot(S_PQ)),
     "S col");
  if (tf.kind == 2)
    ck(fdg::launch_col_acc(st, lc, a->w.d(), a->vp.d(), a->vp.d(), 1, op->nt, op->n1 * op->n2, tf.fft,
                           op->psi / tf.fft.L, true),
       "S t adj");
  if (r_out)
    ck(fdg::launch_row_s_out(st, lc, a->w.d(), a->vp.d(), q, r_out, op->nt, op->n1, op->n2, op->row_axis(),
                             op->scale2(), tf.kind == 1 ? tf : none_tf, op->psi, a->sc.at(S_ONE), a->sc.at(S_ONE), red,
                             nullptr, b),
       "S row adj + residual");
  else
    ck(fdg::launch_row_s_out(st, lc, a->w.d(), a->vp.d(), q, nullptr, op->nt, op->n1, op->n2, op->row_axis(),
                             op->scale2(), tf.kind == 1 ? tf : none_tf, op->psi, nullptr, nullptr, RedSlot{}),
       "S row adj");
}

// Search-direction product fused with the residual update:
// r -= (rz/pq) S d ; reduces |r|^2 into S_RR and p^T S p into S_PQ.
void s_and_update(fdg_admm_s* a, const double* dd, const double* rz_slot) {
  fdg_op_s* op = a->op;
  cudaStream_t st = op->ctx->stream;
  LaunchCounter* lc = &op->ctx->lc;
  const TimeFactor& tf = op->tf;
  TimeFactor none_tf;
  ck(fdg::launch_row_apply(st, lc, dd, a->u.d(), op->nt, op->n1, op->n2, op->row_axis(), op->scale2(),
                           tf.kind == 1 ? tf : none_tf, op->psi, false),
     "K1 row");
  if (tf.kind == 2)
    ck(fdg::launch_col_acc(st, lc, dd, a->u.d(), a->u.d(), 1, op->nt, op->n1 * op->n2, tf.fft, op->psi / tf.fft.L,
                           false),
       "K1 t");
  ck(fdg::launch_col_s_mid(st, lc, dd, a->u.d(), a->w.d(), a->vp.d(), op->nt, op->n1, op->n2, op->ax1, op->scale1(),
                           a->inv_m2.d(), a->a1.d(), a->sc.slot(S_PQ)),
     "K2 col");
  if (tf.kind == 2)
    ck(fdg::launch_col_acc(st, lc, a->w.d(), a->vp.d(), a->vp.d(), 1, op->nt, op->n1 * op->n2, tf.fft,
                           op->psi / tf.fft.L, true),
       "K2 t");
  ck(fdg::launch_row_s_out(st, lc, a->w.d(), a->vp.d(), nullptr, a->r.d(), op->nt, op->n1, op->n2, op->row_axis(),
                           op->scale2(), tf.kind == 1 ? tf : none_tf, op->psi, rz_slot, a->sc.at(S_PQ),
                           a->sc.slot(S_RR)),
     "K3 row");
}

// Spin until the control kernel published the status words of sequence
// number `seq` (host-mapped memory); a failed stream ends the wait.
void wait_status(cudaStream_t st, const volatile double* hs, double seq) {
  for (unsigned spin = 0;; ++spin) {
    if (hs[3] == seq) break;
    if ((spin & 1023u) == 1023u) {
      const cudaError_t e = cudaStreamQuery(st);
      if (e == cudaSuccess) {
        if (hs[3] == seq) break;
        fail(FDG_ECUDA, "pcg: control status missing");
      }
      if (e != cudaErrorNotReady) ck(e, "status");
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
}

// Spin until the graph-driven iterations reported their stop (rep[3] = the
// iteration number, written last).
void wait_report(cudaStream_t st, const volatile double* rep) {
  for (unsigned spin = 0;; ++spin) {
    if (rep[3] != 0.0) break;
    if ((spin & 1023u) == 1023u) {
      const cudaError_t e = cudaStreamQuery(st);
      if (e == cudaSuccess) {
        if (rep[3] != 0.0) break;
        fail(FDG_ECUDA, "pcg: graph stop report missing");
      }
      if (e != cudaErrorNotReady) ck(e, "graph status");
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
}

// Graph-driven PCG iterations for the latency-bound sizes: N up to
// FDG_PCG_GRAPH_NMAX (env; default 2^21 elements, 0 disables) with the
// standard preconditioner passes (the dense any-n path has no guards).
#ifndef FDG_GRAPH_PDL
#define FDG_GRAPH_PDL 1
#endif
std::atomic<long long> g_graph_nmax{[] {
  const char* e = std::getenv("FDG_PCG_GRAPH_NMAX");
  return e ? std::atoll(e) : (1LL << 21);
}()};
bool graph_enabled(const fdg_admm_s* a, size_t N) {
  return (long long)N <= g_graph_nmax.load() && !a->pc->dense;
}

// pcg (admm.cpp:121-169) with apply = apply_S, precond = pc.solve.
// on_final_x (optional): called right after the x update that precedes a
// true-residual confirmation is enqueued (x then holds the candidate result;
// the host-buffer path starts its D2H there, overlapping the confirmation).
fdg_pcg_result pcg_dev(fdg_admm_s* a, const double* rhs, double* x, double tol, int max_inner,
                       const std::function<void()>& on_final_x = nullptr) {
  fdg_ctx ctx = a->op->ctx;
  cudaStream_t st = ctx->stream;
  LaunchCounter* lc = &ctx->lc;
  const size_t N = a->N;
  Scalars& sc = a->sc;
  fdg_pcg_result res{0, 0, 0.0, 0.0};
  ck(cudaEventRecord(a->e0, st), "event");
  // |rhs|^2 and |x|^2 in one pass (admm.cpp:124, 131); the host reads them
  // through an event while the GPU already runs the preconditioner on b,
  // i.e. speculatively on the x = 0 branch r = b (admm.cpp:131-132) of the
  // fused schedule; any other branch discards that work below.
  const bool fused = a->op->tf.kind != 2;
  ck(fdg::launch_norms2(st, lc, rhs, x, N, sc.slot(S_NB)), "nb xx");
  ck(cudaMemcpyAsync(ctx->pinned, sc.at(S_NB), 2 * sizeof(double), cudaMemcpyDeviceToHost, st), "norms D2H");
  ck(cudaEventRecord(a->ev_norms, st), "event");
  int* pause = static_cast<int*>(a->ctl.p);
  if (fused) {
    ck(cudaMemsetAsync(pause, 0, sizeof(int), st), "clear pause");
    pc_apply_dev(a->pc, rhs, a->z.d(), a->u.d(), rhs, sc.slot(S_RZ0));  // r.z of iteration 1 (odd: S_RZ0)
  }
  ck(cudaEventSynchronize(a->ev_norms), "norms");
  double h[2];
  std::memcpy(h, ctx->pinned, sizeof(h));
  const double nb = std::sqrt(h[0]);
  auto finish = [&]() {
    ck(cudaEventRecord(a->e1, st), "event");
    ck(cudaEventSynchronize(a->e1), "event sync");
    float ms = 0.f;
    ck(cudaEventElapsedTime(&ms, a->e0, a->e1), "elapsed");
    res.ms = ms;
  };
  if (nb == 0.0) {
    ck(fdg::launch_fill(st, lc, x, 0.0, N), "fill");
    res = {0, 1, 0.0, 0.0};
    finish();
    return res;
  }
  // x = 0: r = b; the fused schedule reads b in place of r until the first
  // residual update (no copy)
  const bool r_is_b = std::sqrt(h[1]) == 0.0 && fused;
  if (std::sqrt(h[1]) == 0.0) {
    if (!fused) ck(fdg::launch_copy(st, lc, a->r.d(), rhs, N), "r = b");
  } else {
    apply_S_dev(a, x, nullptr, a->r.d(), rhs, sc.slot(S_RR2));
  }
  if (fused) {
    // Fused schedule: the CG update x += a p; p = z + b p of
    // iteration k-1 (p = z + b p) runs inside the B row pass of iteration k
    // (K1F), with ping-pong direction buffers (neighbour time slices of the
    // old direction stay readable while the new one is written); x += a p
    // streams right after the S product, as in the reference loop.
    //
    // Speculation: iteration it+1 is enqueued before the host reads iteration
    // it's scalars.  k_pcg_control(it) raises a device pause flag when the
    // host must act (breakdown, or |r| <= tol |b| -> true-residual
    // confirmation); every guarded kernel behind it then exits immediately,
    // the host drains the stream, runs the reference's confirmation and
    // re-enqueues.  Iteration parity fixes the ping-pong buffers and slots.
    fdg_op_s* op = a->op;
    const TimeFactor& tf = op->tf;
    auto slot_cur = [](int it) { return (it & 1) ? S_RZ0 : S_RZ1; };  // r.z used by iteration it
    auto slot_prv = [](int it) { return (it & 1) ? S_RZ1 : S_RZ0; };
    auto dir_cur = [&](int it) { return (it & 1) ? a->d.d() : a->d2.d(); };
    auto dir_prv = [&](int it) { return (it & 1) ? a->d2.d() : a->d.d(); };
    // iteration body: p = z + b p (+ the previous iteration's x += a p, in
    // K1F), S p, r -= a S p, control, z = M r (r.z -> next slot).  x_host:
    // last iteration whose x update the host applied itself (after a pause).
    int x_host = 0;
    auto x_update = [&](int it) {  // x += (r.z / p^T S p) p of iteration it
      ck(fdg::launch_axpy_dev(st, lc, x, dir_cur(it), N, sc.at(slot_cur(it)), sc.at(S_PQ)), "x += a p");
      x_host = it;
    };
    // graph: launch the control step of the graph-driven iterations
    // (k_pcg_control_graph, condition handle `cond`) instead of the
    // host-sequenced one
    auto enqueue_g = [&](int it, bool guarded, bool graph, cudaGraphConditionalHandle cond) {
      const int* g = guarded ? pause : nullptr;
      const int cur = slot_cur(it), prv = slot_prv(it);
      const bool upd = graph || (it > 1 && x_host != it - 1);  // alpha_{it-1} = rz(prv) / pq (S_PQ still holds pq_{it-1})
      const bool first = !graph && it == 1;
      ck(fdg::launch_row_fused(st, lc, a->z.d(), dir_prv(it), dir_cur(it), x, a->u.d(), op->nt, op->n1, op->n2,
                               op->row_axis(), op->scale2(), tf, op->psi, sc.at(prv), sc.at(S_PQ), sc.at(cur),
                               sc.at(prv), first, upd, g),
         "K1F row");
      ck(fdg::launch_col_s_mid(st, lc, dir_cur(it), a->u.d(), a->w.d(), a->vp.d(), op->nt, op->n1, op->n2, op->ax1,
                               op->scale1(), a->inv_m2.d(), a->a1.d(), sc.slot(S_PQ), g),
         "K2 col");
      ck(fdg::launch_row_s_out(st, lc, a->w.d(), a->vp.d(), nullptr, a->r.d(), op->nt, op->n1, op->n2,
                               op->row_axis(), op->scale2(), tf, op->psi, sc.at(cur), sc.at(S_PQ), sc.slot(S_RR), g,
                               first && r_is_b ? rhs : nullptr),
         "K3 row");
      if (graph) {
        ck(fdg::launch_pcg_control_graph(st, lc, sc.at(S_PQ), sc.at(S_RR), sc.at(S_TOL), a->hstat_dev, pause,
                                         static_cast<int*>(a->ctl.p), cond),
           "control (graph)");
      } else {
        a->seq += 1.0;
        a->hseq[it & 1] = a->seq;
        ck(fdg::launch_pcg_control(st, lc, sc.at(S_PQ), sc.at(S_RR), (tol * nb) * (tol * nb),
                                   a->hstat_dev + 4 * (it & 1), pause, g, a->seq),
           "control");
      }
      pc_apply_dev(a->pc, a->r.d(), a->z.d(), a->u.d(), a->r.d(), sc.slot(prv), pause);  // r.z' -> prv slot
    };
    auto enqueue = [&](int it, bool guarded) { enqueue_g(it, guarded, false, 0); };
    // Graph-driven iterations (latency-bound sizes, FDG_PCG_GRAPH_NMAX): the
    // steady-state iterations (guarded, x update carried in K1F) of one solve
    // run inside ONE graph launch whose WHILE node repeats a two-iteration
    // body (parities fixed by the first iteration) until the control step
    // stops it; the host then handles the stop exactly like a paused
    // host-sequenced iteration.  Graphs are cached per (x, rhs, parity).
    const bool use_graph = graph_enabled(a, N);
    auto graph_for = [&](int parity) -> fdg_admm_s::PcgGraph& {
      for (auto& g : a->graphs)
        if (g.x == x && g.rhs == rhs && g.parity == parity) {
          g.used = ++a->graph_tick;
          return g;
        }
      if (a->graphs.size() >= 8) {  // evict the least recently used
        auto it = std::min_element(a->graphs.begin(), a->graphs.end(),
                                   [](const auto& p, const auto& q) { return p.used < q.used; });
        if (it->exec) cudaGraphExecDestroy(it->exec);
        a->graphs.erase(it);
      }
      fdg_admm_s::PcgGraph gr;
      gr.x = x;
      gr.rhs = rhs;
      gr.parity = parity;
      cudaGraph_t graph = nullptr;
      ck(cudaGraphCreate(&graph, 0), "graph create");
      cudaGraphConditionalHandle cond;
      ck(cudaGraphConditionalHandleCreate(&cond, graph, 1, cudaGraphCondAssignDefault), "graph cond");
      cudaGraphNodeParams cp = {};
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = cond;
      cp.conditional.type = cudaGraphCondTypeWhile;
      cp.conditional.size = 1;
      cudaGraphNode_t node;
      ck(cudaGraphAddNode(&node, graph, nullptr, 0, &cp), "graph while node");
      cudaGraph_t body = cp.conditional.phGraph_out[0];
      const unsigned long long l0 = lc->count;
      const int x_host_saved = x_host;
      static const bool graph_pdl = [] {
        const char* e = std::getenv("FDG_GRAPH_PDL");
        return e ? std::atoi(e) != 0 : FDG_GRAPH_PDL != 0;
      }();
      fdg::pdl_suspend(!graph_pdl);
      ck(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal),
         "graph capture");
      enqueue_g(2 + parity, true, true, cond);  // parity of the first body iteration
      enqueue_g(3 + parity, true, true, cond);
      cudaGraph_t captured = nullptr;
      const cudaError_t ec = cudaStreamEndCapture(st, &captured);
      fdg::pdl_suspend(false);
      ck(ec, "graph end capture");
      x_host = x_host_saved;
      gr.kernels = lc->count - l0;
      lc->count = l0;  // counted per executed body instead
      ck(cudaGraphInstantiate(&gr.exec, graph, 0), "graph instantiate");
      cudaGraphDestroy(graph);
      gr.used = ++a->graph_tick;
      a->graphs.push_back(gr);
      return a->graphs.back();
    };
    if (!r_is_b) pc_apply_dev(a->pc, a->r.d(), a->z.d(), a->u.d(), a->r.d(), sc.slot(slot_cur(1)));
    int it = 1;
    double pq = 0.0, rr2 = 0.0;
    bool stop = false;
    auto read_status = [&](int i) {  // the host-sequenced iteration i
      const volatile double* hs = a->hstat + 4 * (i & 1);
      wait_status(st, hs, a->hseq[i & 1]);
      pq = hs[0];
      rr2 = hs[1];
      stop = hs[2] != 0.0;
    };
    if (max_inner >= 1) {
      enqueue(1, true);
      read_status(1);
    }
    bool cap = max_inner < 1;
    while (!cap) {
      double rn = std::sqrt(rr2);
      if (stop) {
        // iteration it paused the stream: the launches behind it exit at
        // their guard; the flag is cleared in stream order after them (no
        // host drain: the work below queues right behind)
        ck(cudaMemsetAsync(pause, 0, sizeof(int), st), "clear pause");
        if (!std::isfinite(pq) || pq <= 0.0)
          fail(FDG_ENUMERIC, "pcg: operator lost positive definiteness", FDG_NUM_PD_LOSS);
        if (!std::isfinite(rn)) fail(FDG_ENUMERIC, "pcg: non-finite residual", FDG_NUM_NONFINITE_RESIDUAL);
        if (rn <= tol * nb) {
          // x += a p of iteration it (its carrier, K1F of it+1, was skipped),
          // then confirm with the true residual (admm.cpp:152-158)
          x_update(it);
          if (on_final_x) on_final_x();
          apply_S_dev(a, x, nullptr, a->r.d(), rhs, sc.slot(S_RR2));
          double rr;
          sc.read(S_RR2, 1, &rr);
          rn = std::sqrt(rr);
          if (rn <= tol * nb) {
            res = {it, 1, rn / nb, 0.0};
            finish();
            return res;
          }
        }
        // continue (from the replaced residual): the skipped tail of it, then it+1
        pc_apply_dev(a->pc, a->r.d(), a->z.d(), a->u.d(), a->r.d(), sc.slot(slot_prv(it)));
        if (it >= max_inner) break;
        ++it;
        enqueue(it, true);  // x update of it-1 done by the host: not a graph iteration
        read_status(it);
        continue;
      }
      if (it >= max_inner) break;
      if (use_graph) {
        // iterations it+1.. on the device until the control step stops
        auto& gr = graph_for((it + 1) & 1);
        a->hstat[11] = 0.0;
        ck(fdg::launch_pcg_graph_prep(st, lc, static_cast<int*>(a->ctl.p), it, max_inner, sc.at(S_TOL),
                                      (tol * nb) * (tol * nb)),
           "graph prep");
        ck(cudaGraphLaunch(gr.exec, st), "graph launch");
        const volatile double* rep = a->hstat + 8;
        wait_report(st, rep);
        const int it_end = (int)rep[3];
        pq = rep[0];
        rr2 = rep[1];
        stop = rep[2] != 0.0;
        lc->count += gr.kernels * (unsigned long long)((it_end - it + 1) / 2);  // body executions
        if (!stop) ck(cudaMemsetAsync(pause, 0, sizeof(int), st), "clear pause");  // the cap raised it
        it = it_end;
        continue;
      }
      ++it;
      enqueue(it, true);
      read_status(it);
    }
    if (max_inner >= 1 && x_host != max_inner) x_update(max_inner);  // no K1F carries the last update
    ck(cudaStreamSynchronize(st), "drain");
  } else {
    int cur = S_RZ0, nxt = S_RZ1;
    pc_apply_dev(a->pc, a->r.d(), a->z.d(), a->u.d(), a->r.d(), sc.slot(cur));
    ck(fdg::launch_copy(st, lc, a->d.d(), a->z.d(), N), "p = z");
    for (int it = 1; it <= max_inner; ++it) {
      s_and_update(a, a->d.d(), sc.at(cur));
      double pr[2];
      sc.read(S_PQ, 2, pr);  // S_PQ, S_RR adjacent
      const double pq = pr[0];
      if (!std::isfinite(pq) || pq <= 0.0)
        fail(FDG_ENUMERIC, "pcg: operator lost positive definiteness", FDG_NUM_PD_LOSS);
      double rn = std::sqrt(pr[1]);
      if (!std::isfinite(rn)) fail(FDG_ENUMERIC, "pcg: non-finite residual", FDG_NUM_NONFINITE_RESIDUAL);
      bool x_done = false;
      if (rn <= tol * nb) {
        // confirm with the true residual (admm.cpp:152-158)
        ck(fdg::launch_axpy_dev(st, lc, x, a->d.d(), N, sc.at(cur), sc.at(S_PQ)), "x += a p");
        x_done = true;
        apply_S_dev(a, x, nullptr, a->r.d(), rhs, sc.slot(S_RR2));
        double rr2;
        sc.read(S_RR2, 1, &rr2);
        rn = std::sqrt(rr2);
        if (rn <= tol * nb) {
          res = {it, 1, rn / nb, 0.0};
          finish();
          return res;
        }
      }
      pc_apply_dev(a->pc, a->r.d(), a->z.d(), a->u.d(), a->r.d(), sc.slot(nxt));
      // x += (rz/pq) p ; p = z + (rz'/rz) p  (admm.cpp:148-150, 161-163)
      ck(fdg::launch_cg_update(st, lc, x, a->d.d(), a->z.d(), N, sc.at(cur), sc.at(S_PQ), sc.at(nxt), sc.at(cur),
                               !x_done),
         "cg update");
      std::swap(cur, nxt);
    }
  }
  // cap: true relative residual (admm.cpp:165-168)
  apply_S_dev(a, x, nullptr, a->u.d(), rhs, sc.slot(S_RR2));
  double rr2;
  sc.read(S_RR2, 1, &rr2);
  res = {max_inner, 0, std::sqrt(rr2) / nb, 0.0};
  finish();
  return res;
}

// build_rhs (admm.cpp:100-119)
void build_rhs_dev(fdg_admm_s* a, double* rhs, double* r_cache) {
  cudaStream_t st = a->op->ctx->stream;
  LaunchCounter* lc = &a->op->ctx->lc;
  const auto s = admm_scalars(a);
  ck(fdg::launch_rhs_pre(st, lc, s, a->p.d(), a->w_v.d(), a->z_v.d(), a->a2inv.d(), a->m2.d(), r_cache, a->tmp.d(),
                         a->slice, a->N),
     "rhs pre");
  op_apply_dev(a->op, a->tmp.d(), rhs, true);
  ck(fdg::launch_rhs_post(st, lc, s, rhs, a->ybar.d(), a->w_y.d(), a->z_y.d(), a->diag_j.d(), a->slice, a->N),
     "rhs post");
}

double* field_dev(fdg_admm_s* a, int f) {
  switch (f) {
    case FDG_F_Y: return a->y.d();
    case FDG_F_V: return a->v.d();
    case FDG_F_ZY: return a->z_y.d();
    case FDG_F_ZV: return a->z_v.d();
    case FDG_F_P: return a->p.d();
    case FDG_F_WY: return a->w_y.d();
    case FDG_F_WV: return a->w_v.d();
    case FDG_F_YBAR: return a->ybar.d();
    case FDG_F_BY: return a->By.d();
    default: return nullptr;
  }
}

const std::vector<double>* field_slice(fdg_admm_s* a, int f) {
  switch (f) {
    case FDG_F_DIAGJ: return &a->h_diag_j;
    case FDG_F_DIAGJ2: return &a->h_diag_j2;
    case FDG_F_M2: return &a->h_m2;
    case FDG_F_A2INV: return &a->h_a2inv;
    default: return nullptr;
  }
}

void check_ctx(fdg_ctx c) {
  if (!c) fail(FDG_EINVAL, "fdg: null context");
  c->set_device();
}

}  // namespace

// ===================================================================== C ABI
extern "C" {

const char* fdg_last_error(void) { return g_err.c_str(); }
int fdg_last_numeric_code(void) { return g_num; }
const char* fdg_version(void) { return "fdg 0.1 (sm_100a)"; }

fdg_status fdg_ctx_create(int device, void* stream, fdg_ctx* out) {
  return guard([&] {
    int ndev = 0;
    ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    if (device < 0 || device >= ndev) fail(FDG_EINVAL, "fdg_ctx_create: bad device index");
    auto c = std::make_unique<fdg_ctx_s>();
    c->device = device;
    c->set_device();
    if (stream) {
      c->stream = static_cast<cudaStream_t>(stream);
    } else {
      ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "stream");
      c->own_stream = true;
    }
    ck(cudaMallocHost(&c->pinned, sizeof(double) * 64), "pinned");
    c->ensure_partials(4096);
    *out = c.release();
  });
}

fdg_status fdg_ctx_destroy(fdg_ctx ctx) {
  return guard([&] {
    if (!ctx) return;
    ctx->set_device();
    cudaStreamSynchronize(ctx->stream);
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
  });
}

void* fdg_ctx_stream(fdg_ctx ctx) { return ctx ? ctx->stream : nullptr; }
uint64_t fdg_ctx_launch_count(fdg_ctx ctx) { return ctx ? ctx->lc.count : 0; }
fdg_status fdg_ctx_synchronize(fdg_ctx ctx) {
  return guard([&] {
    check_ctx(ctx);
    ck(cudaStreamSynchronize(ctx->stream), "sync");
  });
}

// --------------------------------------------------------------- setup
fdg_status fdg_frac_coeffs(double order, int count, double* out) {
  return guard([&] {
    const auto g = frac_coeffs_host(order, count);
    std::memcpy(out, g.data(), sizeof(double) * g.size());
  });
}

fdg_status fdg_build_riesz(double beta, int n, double h, double* col, double* row) {
  return guard([&] {
    if (!(beta > 1.0 && beta < 2.0)) fail(FDG_EINVAL, "build_riesz: beta must lie in (1, 2)");
    if (n < 1 || !(h > 0.0)) fail(FDG_EINVAL, "build_riesz: bad grid parameters");
    const double c = std::cos(beta * 3.14159265358979323846 / 2.0);
    if (std::abs(c) < 1e-6) fail(FDG_EINVAL, "build_riesz: beta too close to 1");
    const auto g = frac_coeffs_host(beta, n + 1);
    const double scale = -1.0 / (2.0 * c * std::pow(h, beta));
    col[0] = scale * 2.0 * g[1];
    if (n > 1) col[1] = scale * (g[2] + g[0]);
    for (int k = 2; k < n; ++k) col[k] = scale * g[k + 1];
    if (row) std::memcpy(row, col, sizeof(double) * n);
  });
}

fdg_status fdg_build_caputo(double alpha, int n, double h, double* col, double* row) {
  return guard([&] {
    if (!(alpha > 0.0 && alpha < 1.0)) fail(FDG_EINVAL, "build_caputo: alpha must lie in (0, 1)");
    if (n < 1 || !(h > 0.0)) fail(FDG_EINVAL, "build_caputo: bad grid parameters");
    const double scale = 1.0 / std::pow(h, alpha);
    auto g = frac_coeffs_host(alpha, n);
    for (int k = 0; k < n; ++k) col[k] = g[k] * scale;
    for (int k = 0; k < n; ++k) row[k] = 0.0;
    row[0] = col[0];
  });
}

fdg_status fdg_tchan(int n, const double* col, const double* row, double* first_col, double* eigs) {
  return guard([&] {
    if (n < 1) fail(FDG_EINVAL, "tchan: empty spec");
    tchan_host(n, col, row, first_col, eigs);
  });
}

fdg_status fdg_randn(uint64_t seed, size_t count, double* out) {
  return guard([&] {
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> gauss;
    for (size_t i = 0; i < count; ++i) out[i] = gauss(rng);
  });
}

// ------------------------------------------------------------ operator
fdg_status fdg_op_create(fdg_ctx ctx, int nt, int n1, int n2, const double* tcol, const double* trow,
                         const double* c1, const double* r1, const double* c2, const double* r2, double psi,
                         fdg_op* out) {
  return guard([&] {
    check_ctx(ctx);
    if (nt < 1 || n1 < 1 || n2 < 1) fail(FDG_EINVAL, "ConstraintOperator: factor size mismatch");
    if (!tcol || !trow || !c1 || !r1 || !c2 || !r2) fail(FDG_EINVAL, "fdg_op_create: null factor");
    auto op = std::make_unique<fdg_op_s>();
    op->ctx = ctx;
    op->nt = nt;
    op->n1 = n1;
    op->n2 = n2;
    op->psi = psi;
    op->tcol.assign(tcol, tcol + nt);
    op->trow.assign(trow, trow + nt);
    op->c1.assign(c1, c1 + n1);
    op->r1.assign(r1, r1 + n1);
    op->c2.assign(c2, c2 + n2);
    op->r2.assign(r2, r2 + n2);
    // As in the reference, the adjoint transposes only the time factor; the
    // spatial passes use the forward symbols in both directions
    // (toeplitz.cpp:178-181, "Riesz factors are symmetric").
    build_axis(op.get(), op->ax1, op->sym1, nullptr, op->tw1, op->twh1, op->tws1, op->symr1, op->c1, op->r1, op->twq1a,
               op->twq1b);
    build_axis(op.get(), op->ax2, op->sym2, nullptr, op->tw2, op->twh2, op->tws2, op->symr2, op->c2, op->r2, op->twq2a,
               op->twq2b);
    bool bidiag = true;
    for (int k = 1; k < nt; ++k)
      if (op->trow[k] != 0.0) bidiag = false;
    for (int k = 2; k < nt; ++k)
      if (op->tcol[k] != 0.0) bidiag = false;
    if (bidiag) {
      op->tf.kind = 1;
      op->tf.c0 = op->tcol[0];
      op->tf.c1 = nt > 1 ? op->tcol[1] : 0.0;
      // psi c0 x_k == (-psi/L) IFFT(FFT(x) * (-c0 L)): fold the diagonal of the
      // time stencil into the x2 Toeplitz symbol (exact in real arithmetic).
      std::vector<double> s2 = embed_symbol_full(op->c2, op->r2, op->ax2.L);
      if (op->ax2.sym_re)
        for (int f = 0; f < op->ax2.L; ++f) s2[2 * f + 1] = 0.0;
      for (int f = 0; f < op->ax2.L; ++f) s2[2 * f] -= op->tf.c0;
      upload(op->sym2s, s2, ctx->stream);
      op->ax2s = op->ax2;
      op->ax2s.sym = op->sym2s.c();
      op->ax2s.sym_adj = op->sym2s.c();
      if (op->ax2.sym_re) {
        upload(op->symr2s, real_parts(s2), ctx->stream);
        op->ax2s.sym_re = op->ax2s.sym_adj_re = op->symr2s.d();
      }
    } else {
      op->tf.kind = 2;
      build_axis(op.get(), op->tf.fft, op->symt, &op->symt_adj, op->twt, op->twht, op->twst, op->symrt, op->tcol, op->trow,
                 op->twqta, op->twqtb);
      op->ax2s = op->ax2;
    }
    ctx->ensure_partials(fdg::max_partials_needed(nt, n1, n2));
    *out = op.release();
  });
}

fdg_status fdg_op_destroy(fdg_op op) {
  return guard([&] {
    if (op) {
      op->ctx->set_device();
      cudaStreamSynchronize(op->ctx->stream);
    }
    delete op;
  });
}

size_t fdg_op_size(fdg_op op) { return op ? op->N() : 0; }
double fdg_op_psi(fdg_op op) { return op ? op->psi : 0.0; }

fdg_status fdg_op_apply(fdg_op op, const double* x, double* out, int adjoint) {
  return guard([&] {
    if (!op) fail(FDG_EINVAL, "fdg_op_apply: null operator");
    op->ctx->set_device();
    if (x == out) fail(FDG_EINVAL, "ConstraintOperator::apply: x and out must not alias");
    op_apply_dev(op, x, out, adjoint != 0);
  });
}

fdg_status fdg_op_apply_host(fdg_op op, const double* x, size_t n_x, double* out, size_t n_out, int adjoint) {
  return guard([&] {
    if (!op) fail(FDG_EINVAL, "fdg_op_apply: null operator");
    if (n_x != op->N() || n_out != op->N())
      fail(FDG_EINVAL, "ConstraintOperator::apply: dimension mismatch");
    op->ctx->set_device();
    cudaStream_t st = op->ctx->stream;
    DevBuf dx(sizeof(double) * n_x), dout(sizeof(double) * n_out);
    ck(cudaMemcpyAsync(dx.p, x, sizeof(double) * n_x, cudaMemcpyHostToDevice, st), "H2D");
    op_apply_dev(op, dx.d(), dout.d(), adjoint != 0);
    ck(cudaMemcpyAsync(out, dout.p, sizeof(double) * n_out, cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "sync");
  });
}

// ------------------------------------------------------ preconditioner
namespace {

fdg_pc_s* make_pc(fdg_ctx ctx, int nt, int n1, int n2, const double* lt, const double* l1, const double* l2,
                  double psi, double rho, double delta, double gamma) {
  if (!(rho > 0.0) || !(delta > 0.0) || !(gamma > 0.0))
    fail(FDG_EINVAL, "CirculantPreconditioner: scalars must be positive");
  if (nt < 1 || n1 < 1 || n2 < 1) fail(FDG_EINVAL, "CirculantPreconditioner: level sizes must be positive");
  // power-of-two levels up to 2048: radix passes; anything else: the dense
  // Hartley path (same operator)
  bool dense = false;
  for (int n : {nt, n1, n2}) dense = dense || !is_pow2(n) || n > 2048;
  // The Hartley formulation needs lambda_S even in every axis: real (hence
  // even) spatial eigenvalues, i.e. symmetric spatial factors.
  for (auto [lam, n] : {std::pair{l1, n1}, std::pair{l2, n2}}) {
    double mx = 0.0, im = 0.0;
    for (int i = 0; i < n; ++i) {
      mx = std::max(mx, std::hypot(lam[2 * i], lam[2 * i + 1]));
      im = std::max(im, std::abs(lam[2 * i + 1]));
    }
    if (im > 1e-10 * std::max(mx, 1e-300))
      fail(FDG_EUNSUPPORTED, "fdg: spatial circulant eigenvalues must be real (symmetric factors)");
  }
  auto pc = std::make_unique<fdg_pc_s>();
  pc->ctx = ctx;
  pc->nt = nt;
  pc->n1 = n1;
  pc->n2 = n2;
  pc->psi = psi;
  pc->rho = rho;
  pc->delta = delta;
  pc->gamma = gamma;
  cudaStream_t st = ctx->stream;
  upload(pc->lt, std::vector<double>(lt, lt + 2 * (size_t)nt), st);
  upload(pc->l1, std::vector<double>(l1, l1 + 2 * (size_t)n1), st);
  upload(pc->l2, std::vector<double>(l2, l2 + 2 * (size_t)n2), st);
  pc->dense = dense;
  if (dense) {
    if (std::max(nt, std::max(n1, n2)) > 12288)
      fail(FDG_EUNSUPPORTED, "fdg: circulant preconditioner level size above 12288");
    upload(pc->cas_t, cas_table(nt), st);
    upload(pc->cas_1, cas_table(n1), st);
    upload(pc->cas_2, cas_table(n2), st);
    pc->dtmp.alloc(sizeof(double) * pc_size(nt, n1, n2));
  } else {
    upload(pc->twt, stockham_twiddles(nt), st);
    upload(pc->tw1, stockham_twiddles(n1), st);
    upload(pc->tw2, stockham_twiddles(n2), st);
  }
  // circulant.cpp:37-40
  const double m2 = 1.0 / (rho * (gamma / (psi * psi) + 1.0 / delta)) + delta / rho;
  PcTables& t = pc->tab;
  t.nt = nt;
  t.n1 = n1;
  t.n2 = n2;
  t.lam_t = pc->lt.c();
  t.lam_1 = pc->l1.c();
  t.lam_2 = pc->l2.c();
  t.tw_t = pc->twt.c();
  t.tw_1 = pc->tw1.c();
  t.tw_2 = pc->tw2.c();
  t.psi = psi;
  t.base = rho * (1.0 + 1.0 / delta);
  t.inv_m2 = 1.0 / m2;
  t.inv_total = 1.0 / (double)pc->N();
  ctx->ensure_partials(fdg::max_partials_needed(nt, n1, n2));
  return pc.release();
}

}  // namespace

fdg_status fdg_pc_create(fdg_ctx ctx, int nt, int n1, int n2, const double* lt, const double* l1, const double* l2,
                         double psi, double rho, double delta, double gamma, fdg_pc* out) {
  return guard([&] {
    check_ctx(ctx);
    *out = make_pc(ctx, nt, n1, n2, lt, l1, l2, psi, rho, delta, gamma);
  });
}

fdg_status fdg_pc_assemble(fdg_op op, double rho, double delta, double gamma, fdg_pc* out) {
  return guard([&] {
    if (!op) fail(FDG_EINVAL, "assemble_precond: null operator");
    check_ctx(op->ctx);
    std::vector<double> lt(2 * (size_t)op->nt), l1(2 * (size_t)op->n1), l2(2 * (size_t)op->n2);
    tchan_host(op->nt, op->tcol.data(), op->trow.data(), nullptr, lt.data());
    tchan_host(op->n1, op->c1.data(), op->r1.data(), nullptr, l1.data());
    tchan_host(op->n2, op->c2.data(), op->r2.data(), nullptr, l2.data());
    *out = make_pc(op->ctx, op->nt, op->n1, op->n2, lt.data(), l1.data(), l2.data(), op->psi, rho, delta, gamma);
  });
}

namespace {
void build_chirp_axis(fdg_pc_s* pc, AxisSym& ax, DevBuf& sym, DevBuf& tw, DevBuf& twh, DevBuf& tws, int n) {
  const int L = std::max(2, pow2_ceil(2L * n - 1));
  if (L > 2048) fail(FDG_EUNSUPPORTED, "fdg: 2-level preconditioner level size " + std::to_string(n) + " > 1024");
  cudaStream_t st = pc->ctx->stream;
  ax.n = n;
  ax.L = L;
  upload(sym, chirp_symbol(n, L), st);
  upload(tw, stockham_twiddles(L), st);
  upload(twh, stockham_twiddles(std::max(1, L / 2)), st);
  std::vector<double> twist = twiddles(L);
  twist.resize(2 * (size_t)std::max(1, L / 2));
  upload(tws, twist, st);
  ax.sym = ax.sym_adj = sym.c();
  ax.tw = tw.c();
  ax.twh = twh.c();
  ax.twist = tws.c();
}

fdg_pc_s* make_pc2(fdg_ctx ctx, int nt, int n1, int n2, const double* l1, const double* l2) {
  if (nt < 1 || n1 < 1 || n2 < 1) fail(FDG_EINVAL, "2-level preconditioner: sizes must be positive");
  std::vector<double> r1(n1), r2(n2);
  for (auto [lam, n, out] : {std::tuple{l1, n1, &r1}, std::tuple{l2, n2, &r2}}) {
    double mx = 0.0, im = 0.0;
    for (int i = 0; i < n; ++i) {
      mx = std::max(mx, std::hypot(lam[2 * i], lam[2 * i + 1]));
      im = std::max(im, std::abs(lam[2 * i + 1]));
      (*out)[i] = lam[2 * i];
    }
    if (im > 1e-10 * std::max(mx, 1e-300))
      fail(FDG_EUNSUPPORTED, "fdg: 2-level preconditioner needs real eigenvalues (symmetric factors)");
    // the Hartley formulation (and the PFA passes' mirror-pair lambda) needs
    // lam[k] == lam[n - k] (real symmetric circulant)
    double odd = 0.0;
    for (int i = 1; i < n; ++i) odd = std::max(odd, std::abs(lam[2 * i] - lam[2 * (n - i)]));
    if (odd > 1e-10 * std::max(mx, 1e-300))
      fail(FDG_EUNSUPPORTED, "fdg: 2-level preconditioner needs even eigenvalues (symmetric factors)");
  }
  auto pc = std::make_unique<fdg_pc_s>();
  pc->ctx = ctx;
  pc->kind = 2;
  pc->nt = nt;
  pc->n1 = n1;
  pc->n2 = n2;
  pc->P2 = n2 + (n2 & 1);
  cudaStream_t st = ctx->stream;
  upload(pc->lam1, r1, st);
  upload(pc->lam2, r2, st);
  upload(pc->c1, chirp_table(n1), st);
  upload(pc->c2, chirp_table(n2), st);
  build_chirp_axis(pc.get(), pc->bs1, pc->s1, pc->t1, pc->th1, pc->ts1, n1);
  build_chirp_axis(pc.get(), pc->bs2, pc->s2, pc->t2, pc->th2, pc->ts2, n2);
  const size_t F = (size_t)nt * n1, Fp = F + (F & 1);
  const size_t words = std::max(Fp * n2, F * pc->P2);
  pc->bu.alloc(sizeof(double) * words);
  pc->bv.alloc(sizeof(double) * words);
  ctx->ensure_partials(fdg::max_partials_needed(1, (int)Fp, pc->P2));
  return pc.release();
}
}  // namespace

fdg_status fdg_pc2_create(fdg_ctx ctx, int nt, int n1, int n2, const double* lam_x1, const double* lam_x2,
                          fdg_pc* out) {
  return guard([&] {
    check_ctx(ctx);
    if (!lam_x1 || !lam_x2 || !out) fail(FDG_EINVAL, "fdg_pc2_create: null argument");
    *out = make_pc2(ctx, nt, n1, n2, lam_x1, lam_x2);
  });
}

fdg_status fdg_pc2_assemble(fdg_op op, fdg_pc* out) {
  return guard([&] {
    if (!op || !out) fail(FDG_EINVAL, "fdg_pc2_assemble: null argument");
    check_ctx(op->ctx);
    std::vector<double> l1(2 * (size_t)op->n1), l2(2 * (size_t)op->n2);
    tchan_host(op->n1, op->c1.data(), op->r1.data(), nullptr, l1.data());
    tchan_host(op->n2, op->c2.data(), op->r2.data(), nullptr, l2.data());
    *out = make_pc2(op->ctx, op->nt, op->n1, op->n2, l1.data(), l2.data());
  });
}

fdg_status fdg_pc_destroy(fdg_pc pc) {
  return guard([&] {
    if (pc) {
      pc->ctx->set_device();
      cudaStreamSynchronize(pc->ctx->stream);
    }
    delete pc;
  });
}

fdg_status fdg_pc_solve(fdg_pc pc, const double* r, double* z) {
  return guard([&] {
    if (!pc) fail(FDG_EINVAL, "precond_solve: null preconditioner");
    pc->ctx->set_device();
    if (r == z) fail(FDG_EINVAL, "precond_solve: r and z must not alias");
    if (pc->kind == 2)
      pc2_apply_dev(pc, r, z);
    else
      pc_apply_dev(pc, r, z, z, nullptr, RedSlot{});
  });
}

fdg_status fdg_pc_solve_host(fdg_pc pc, const double* r, size_t n_r, double* z, size_t n_z) {
  return guard([&] {
    if (!pc) fail(FDG_EINVAL, "precond_solve: null preconditioner");
    if (n_r != pc->N() || n_z != pc->N()) fail(FDG_EINVAL, "precond_solve: dimension mismatch");
    pc->ctx->set_device();
    cudaStream_t st = pc->ctx->stream;
    DevBuf dr(sizeof(double) * n_r), dz(sizeof(double) * n_z);
    ck(cudaMemcpyAsync(dr.p, r, sizeof(double) * n_r, cudaMemcpyHostToDevice, st), "H2D");
    if (pc->kind == 2)
      pc2_apply_dev(pc, dr.d(), dz.d());
    else
      pc_apply_dev(pc, dr.d(), dz.d(), dz.d(), nullptr, RedSlot{});
    ck(cudaMemcpyAsync(z, dz.p, sizeof(double) * n_z, cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "sync");
  });
}

fdg_status fdg_pc_lam_s_host(fdg_pc pc, double* out) {
  return guard([&] {
    if (!pc) fail(FDG_EINVAL, "null preconditioner");
    if (pc->kind != 3) fail(FDG_EINVAL, "lam_S exists only for the 3-level CirculantPreconditioner");
    std::vector<double> lt(2 * (size_t)pc->nt), l1(2 * (size_t)pc->n1), l2(2 * (size_t)pc->n2);
    pc->ctx->set_device();
    ck(cudaMemcpy(lt.data(), pc->lt.p, lt.size() * 8, cudaMemcpyDeviceToHost), "D2H");
    ck(cudaMemcpy(l1.data(), pc->l1.p, l1.size() * 8, cudaMemcpyDeviceToHost), "D2H");
    ck(cudaMemcpy(l2.data(), pc->l2.p, l2.size() * 8, cudaMemcpyDeviceToHost), "D2H");
    const double m2 = 1.0 / pc->tab.inv_m2;
    for (int k = 0; k < pc->nt; ++k)
      for (int i = 0; i < pc->n1; ++i)
        for (int j = 0; j < pc->n2; ++j) {
          const double sr = l1[2 * i] + l2[2 * j], si = l1[2 * i + 1] + l2[2 * j + 1];
          const double br = pc->psi * (lt[2 * k] - sr), bi = pc->psi * (lt[2 * k + 1] - si);
          out[((size_t)k * pc->n1 + i) * pc->n2 + j] = pc->tab.base + (br * br + bi * bi) / m2;
        }
  });
}

// ---------------------------------------------------------------- ADMM
fdg_status fdg_admm_create(fdg_op op, fdg_pc pc, const fdg_admm_desc* desc, const double* ybar, fdg_admm* out) {
  return guard([&] {
    if (!op || !pc || !desc) fail(FDG_EINVAL, "fdg_admm_create: null argument");
    if (op->ctx != pc->ctx) fail(FDG_EINVAL, "fdg_admm_create: operator and preconditioner on different contexts");
    if (pc->kind != 3) fail(FDG_EINVAL, "fdg_admm_create: the ADMM solve needs the 3-level CirculantPreconditioner");
    if (op->nt != pc->nt || op->n1 != pc->n1 || op->n2 != pc->n2)
      fail(FDG_EINVAL, "fdg_admm_create: operator/preconditioner shape mismatch");
    const fdg_admm_desc& d = *desc;
    // AdmmConfig::validate (admm.cpp:34-42) and ProblemSpec::validate bounds/gamma
    constexpr double rho_max = 1.6180339887498949;
    if (!(d.rho > 0.0 && d.rho < rho_max)) fail(FDG_EINVAL, "rho must lie in (0, (sqrt(5)+1)/2)");
    if (!(d.delta > 0.0)) fail(FDG_EINVAL, "delta must be positive");
    if (!(d.tol_primal > 0.0) || !(d.inner_tol_floor > 0.0) || !(d.inner_tol_factor > 0.0))
      fail(FDG_EINVAL, "tolerances must be positive");
    if (d.max_outer < 1 || d.max_inner < 1) fail(FDG_EINVAL, "iteration caps must be >= 1");
    if (!(d.gamma > 0.0)) fail(FDG_EINVAL, "gamma must be positive");
    if (!(d.y_lo < d.y_hi)) fail(FDG_EINVAL, "state bounds must satisfy y_lo < y_hi");
    if (!(d.u_lo < d.u_hi)) fail(FDG_EINVAL, "control bounds must satisfy u_lo < u_hi");
    fdg_ctx ctx = op->ctx;
    check_ctx(ctx);
    auto a = std::make_unique<fdg_admm_s>();
    a->op = op;
    a->pc = pc;
    a->desc = d;
    a->nt = op->nt;
    a->slice = (size_t)op->n1 * op->n2;
    a->N = op->N();
    a->psi = op->psi;
    a->v_lo = a->psi * d.u_lo;
    a->v_hi = a->psi * d.u_hi;
    const int nt = op->nt;
    // make_admm_work (admm.cpp:52-79) + objective_weights (problem.cpp:60-68)
    a->h_diag_j.assign(nt, 1.0);
    a->h_diag_j[nt - 1] = 0.5;
    a->h_diag_j2.resize(nt);
    a->h_m2.resize(nt);
    a->h_a2inv.resize(nt);
    std::vector<double> inv_m2(nt), a1(nt);
    const double g_over_psi2 = d.gamma / (a->psi * a->psi);
    for (int k = 0; k < nt; ++k) {
      a->h_diag_j2[k] = g_over_psi2 * a->h_diag_j[k];
      a->h_a2inv[k] = 1.0 / (d.rho * (a->h_diag_j2[k] + 1.0 / d.delta));
      a->h_m2[k] = a->h_a2inv[k] + d.delta / d.rho;
      inv_m2[k] = 1.0 / a->h_m2[k];
      a1[k] = d.rho * (a->h_diag_j[k] + 1.0 / d.delta);
    }
    cudaStream_t st = ctx->stream;
    upload(a->diag_j, a->h_diag_j, st);
    upload(a->diag_j2, a->h_diag_j2, st);
    upload(a->m2, a->h_m2, st);
    upload(a->a2inv, a->h_a2inv, st);
    upload(a->inv_m2, inv_m2, st);
    upload(a->a1, a1, st);
    const size_t bytes = sizeof(double) * a->N;
    for (DevBuf* b : {&a->y, &a->v, &a->z_y, &a->z_v, &a->p, &a->w_y, &a->w_v, &a->ybar, &a->By, &a->rhs, &a->r_cache,
                      &a->tmp, &a->r, &a->z, &a->d, &a->d2, &a->u, &a->w, &a->vp}) {
      b->alloc(bytes);
      ck(cudaMemsetAsync(b->p, 0, bytes, st), "memset");
    }
    if (ybar) ck(cudaMemcpyAsync(a->ybar.p, ybar, bytes, cudaMemcpyHostToDevice, st), "ybar H2D");
    a->sc.init(ctx);
    a->inner_tol = d.inner_tol_factor * d.inner_tol_floor;  // admm.cpp:245
    for (cudaEvent_t* e : {&a->e0, &a->e1, &a->e2, &a->e3}) ck(cudaEventCreate(e), "event");
    ck(cudaEventCreateWithFlags(&a->ev_norms, cudaEventDisableTiming), "event");
    a->ctl.alloc(sizeof(int) * 4);
    ck(cudaMemsetAsync(a->ctl.p, 0, sizeof(int) * 4, st), "memset");
    ck(cudaHostAlloc(&a->hstat, sizeof(double) * 12, cudaHostAllocMapped), "pinned status");
    for (int i = 0; i < 12; ++i) a->hstat[i] = i < 8 ? -1.0 : 0.0;
    ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(&a->hstat_dev), a->hstat, 0), "mapped status");
    ck(cudaStreamSynchronize(st), "sync");
    *out = a.release();
  });
}

fdg_status fdg_admm_destroy(fdg_admm a) {
  return guard([&] {
    if (!a) return;
    a->op->ctx->set_device();
    cudaStreamSynchronize(a->op->ctx->stream);
    for (cudaEvent_t e : {a->e0, a->e1, a->e2, a->e3, a->ev_x0, a->ev_norms})
      if (e) cudaEventDestroy(e);
    if (a->cstream) cudaStreamDestroy(a->cstream);
    if (a->x0flag_host) cudaFreeHost(a->x0flag_host);
    if (a->hstat) cudaFreeHost(a->hstat);
    delete a;
  });
}

int fdg_admm_converged(fdg_admm a) { return a && a->converged ? 1 : 0; }
int fdg_admm_stagnations(fdg_admm a) { return a ? a->stagnations : 0; }

fdg_status fdg_admm_get(fdg_admm a, int field, double* out) {
  return guard([&] {
    if (!a) fail(FDG_EINVAL, "null admm");
    a->op->ctx->set_device();
    if (double* p = field_dev(a, field)) {
      ck(cudaMemcpyAsync(out, p, sizeof(double) * a->N, cudaMemcpyDeviceToHost, a->op->ctx->stream), "D2H");
      ck(cudaStreamSynchronize(a->op->ctx->stream), "sync");
      return;
    }
    const auto* s = field_slice(a, field);
    if (!s) fail(FDG_EINVAL, "fdg_admm_get: unknown field");
    for (size_t i = 0; i < a->N; ++i) out[i] = (*s)[i / a->slice];
  });
}

fdg_status fdg_admm_set(fdg_admm a, int field, const double* in) {
  return guard([&] {
    if (!a) fail(FDG_EINVAL, "null admm");
    a->op->ctx->set_device();
    double* p = field_dev(a, field);
    if (!p) fail(FDG_EINVAL, "fdg_admm_set: field is not settable");
    ck(cudaMemcpyAsync(p, in, sizeof(double) * a->N, cudaMemcpyHostToDevice, a->op->ctx->stream), "H2D");
    ck(cudaStreamSynchronize(a->op->ctx->stream), "sync");
  });
}

// Debug/test accessor of the PCG work vectors (0 r, 1 z, 2 p, 3 u, 4 w,
// 5 vp) and of the device scalar block (which = -1: S_COUNT doubles).
fdg_status fdg_admm_debug_get(fdg_admm a, int which, double* host_out) {
  return guard([&] {
    if (!a) fail(FDG_EINVAL, "null admm");
    a->op->ctx->set_device();
    cudaStream_t st = a->op->ctx->stream;
    ck(cudaStreamSynchronize(st), "sync");
    if (which < 0) {
      ck(cudaMemcpy(host_out, a->sc.vals.p, sizeof(double) * S_COUNT, cudaMemcpyDeviceToHost), "D2H");
      return;
    }
    DevBuf* b[] = {&a->r, &a->z, &a->d, &a->u, &a->w, &a->vp};
    if (which > 5) fail(FDG_EINVAL, "fdg_admm_debug_get: bad vector");
    ck(cudaMemcpy(host_out, b[which]->p, sizeof(double) * a->N, cudaMemcpyDeviceToHost), "D2H");
  });
}

fdg_status fdg_admm_field_ptr(fdg_admm a, int field, double** dev) {
  return guard([&] {
    if (!a) fail(FDG_EINVAL, "null admm");
    double* p = field_dev(a, field);
    if (!p) fail(FDG_EINVAL, "fdg_admm_field_ptr: unknown field");
    *dev = p;
  });
}

fdg_status fdg_admm_apply_S(fdg_admm a, const double* x, double* out) {
  return guard([&] {
    if (!a) fail(FDG_EINVAL, "null admm");
    a->op->ctx->set_device();
    apply_S_dev(a, x, out);
  });
}

fdg_status fdg_admm_build_rhs(fdg_admm a, double* rhs, double* r_cache) {
  return guard([&] {
    if (!a) fail(FDG_EINVAL, "null admm");
    a->op->ctx->set_device();
    build_rhs_dev(a, rhs, r_cache ? r_cache : a->r_cache.d());
  });
}

fdg_status fdg_admm_pcg(fdg_admm a, const double* rhs, double* x, double tol, int max_inner, fdg_pcg_result* res) {
  return guard([&] {
    if (!a) fail(FDG_EINVAL, "null admm");
    a->op->ctx->set_device();
    const fdg_pcg_result r = pcg_dev(a, rhs, x, tol, max_inner);
    if (res) *res = r;
  });
}

fdg_status fdg_admm_pcg_host(fdg_admm a, const double* rhs, double* x, double tol, int max_inner,
                             fdg_pcg_result* res) {
  return guard([&] {
    if (!a) fail(FDG_EINVAL, "null admm");
    a->op->ctx->set_device();
    cudaStream_t st = a->op->ctx->stream;
    const size_t bytes = sizeof(double) * a->N;
    // Speculation on the common x0 = 0 start (admm.cpp:131 branch r = b):
    // the solve starts as soon as rhs has landed, from a zeroed device x,
    // while x0 travels on a copy stream into its own buffer and is checked
    // for nonzeros there.  x0 == 0 (every element +-0): the speculative solve
    // is exactly the reference's (0 + v == v), its x is the result.  Else the
    // solve is redone from the landed x0.  x is in/out: the D2H of the result
    // is ordered after the H2D of x0 on the copy stream.
    if (!a->cstream) {
      ck(cudaStreamCreateWithFlags(&a->cstream, cudaStreamNonBlocking), "copy stream");
      ck(cudaEventCreateWithFlags(&a->ev_x0, cudaEventDisableTiming), "event");
      a->x0buf.alloc(bytes);
      a->x0flag.alloc(sizeof(int));
      ck(cudaMallocHost(&a->x0flag_host, sizeof(int)), "pinned flag");
    }
    cudaStream_t cs = a->cstream;
    LaunchCounter* lc = &a->op->ctx->lc;
    int* flag = static_cast<int*>(a->x0flag.p);
    ck(cudaMemcpyAsync(a->rhs.p, rhs, bytes, cudaMemcpyHostToDevice, st), "H2D rhs");
    ck(cudaMemsetAsync(a->tmp.p, 0, bytes, st), "x = 0");
    ck(cudaEventRecord(a->ev_x0, st), "event");  // x0's H2D queues behind rhs's
    ck(cudaStreamWaitEvent(cs, a->ev_x0, 0), "wait");
    ck(cudaMemsetAsync(flag, 0, sizeof(int), cs), "flag");
    ck(cudaMemcpyAsync(a->x0buf.p, x, bytes, cudaMemcpyHostToDevice, cs), "H2D x0");
    ck(fdg::launch_any_nonzero(cs, lc, a->x0buf.d(), a->N, flag), "x0 check");
    volatile int* hflag = a->x0flag_host;
    *hflag = -1;
    ck(cudaMemcpyAsync(a->x0flag_host, flag, sizeof(int), cudaMemcpyDeviceToHost, cs), "flag D2H");
    // D2H of a candidate x on the copy stream while the confirmation runs
    // (only once the x0 = 0 speculation is known to hold)
    bool copied = false;
    auto early_d2h = [&]() {
      copied = false;
      if (cudaStreamQuery(cs) != cudaSuccess || *hflag != 0) return;
      ck(cudaEventRecord(a->ev_x0, st), "event");
      ck(cudaStreamWaitEvent(cs, a->ev_x0, 0), "wait");
      ck(cudaMemcpyAsync(x, a->tmp.p, bytes, cudaMemcpyDeviceToHost, cs), "D2H x (early)");
      copied = true;
    };
    fdg_pcg_result r{};
    std::exception_ptr spec_error;
    try {
      r = pcg_dev(a, a->rhs.d(), a->tmp.d(), tol, max_inner, early_d2h);
    } catch (...) {
      spec_error = std::current_exception();  // only binding when x0 == 0
      cudaStreamSynchronize(st);
    }
    ck(cudaStreamSynchronize(cs), "copy stream");
    const int nz = *hflag;
    if (!nz && spec_error) std::rethrow_exception(spec_error);
    if (nz) {
      r = pcg_dev(a, a->rhs.d(), a->x0buf.d(), tol, max_inner);
      ck(cudaMemcpyAsync(x, a->x0buf.p, bytes, cudaMemcpyDeviceToHost, st), "D2H x");
    } else if (!(copied && r.converged)) {
      // the early copy (if any) predates a failed confirmation or the cap
      ck(cudaMemcpyAsync(x, a->tmp.p, bytes, cudaMemcpyDeviceToHost, st), "D2H x");
    }
    ck(cudaStreamSynchronize(st), "sync");
    if (res) *res = r;
  });
}

fdg_status fdg_admm_dual_inf(fdg_admm a, double* out) {
  return guard([&] {
    if (!a) fail(FDG_EINVAL, "null admm");
    a->op->ctx->set_device();
    cudaStream_t st = a->op->ctx->stream;
    op_apply_dev(a->op, a->p.d(), a->tmp.d(), true);
    ck(fdg::launch_dual_inf(st, &a->op->ctx->lc, a->y.d(), a->ybar.d(), a->tmp.d(), a->w_y.d(), a->v.d(), a->p.d(),
                            a->w_v.d(), a->diag_j.d(), a->diag_j2.d(), a->slice, a->N, a->sc.slot(S_DINF)),
       "dual inf");
    double s[2];
    a->sc.read(S_DINF, 2, s);
    *out = std::max(s[0], s[1]);
  });
}

fdg_status fdg_admm_objective(fdg_admm a, double* out) {
  return guard([&] {
    if (!a) fail(FDG_EINVAL, "null admm");
    a->op->ctx->set_device();
    ck(fdg::launch_objective(a->op->ctx->stream, &a->op->ctx->lc, a->y.d(), a->ybar.d(), a->v.d(), a->diag_j.d(),
                             a->diag_j2.d(), a->slice, a->N, a->sc.slot(S_OBJ)),
       "objective");
    double s[2];
    a->sc.read(S_OBJ, 2, s);
    *out = 0.5 * s[0] + 0.5 * s[1];
  });
}

// Per-pass device timing of one PCG iteration's kernels (bench/roofline
// hook).  Each pass is launched `reps` times back to back between two CUDA
// events on the context stream.  Overwrites the PCG scratch vectors (run it
// after the measurements that need them).  Order of ms[]: K1 row, K2 col,
// K3 row, P1 x2, P2 x1, P3 t, P4 x1, P5 x2 (K1 = fused CG update + B row).
fdg_status fdg_set_pcg_graph_nmax(long long nmax, long long* previous) {
  return guard([&] {
    const long long old = nmax >= 0 ? g_graph_nmax.exchange(nmax) : g_graph_nmax.load();
    if (previous) *previous = old;
  });
}

fdg_status fdg_admm_profile_passes(fdg_admm a, int reps, double* ms, double* bytes) {
  return guard([&] {
    if (!a || reps < 1) fail(FDG_EINVAL, "fdg_admm_profile_passes: bad arguments");
    fdg_ctx ctx = a->op->ctx;
    ctx->set_device();
    cudaStream_t st = ctx->stream;
    LaunchCounter* lc = &ctx->lc;
    fdg_op_s* op = a->op;
    fdg_pc_s* pc = a->pc;
    const size_t N = a->N;
    const int F = op->nt * op->n1;
    const TimeFactor& tf = op->tf;
    TimeFactor none_tf;
    const TimeFactor& stf = tf.kind == 1 ? tf : none_tf;
    Scalars& sc = a->sc;
    // well-defined scalars for the passes that read them
    const double one = 1.0;
    for (int s : {S_RZ0, S_RZ1, S_PQ})
      ck(cudaMemcpyAsync(sc.at(s), &one, sizeof(double), cudaMemcpyHostToDevice, st), "H2D");
    ck(cudaStreamSynchronize(st), "sync");
    std::vector<std::function<void()>> passes = {
        [&] {
          if (op->tf.kind != 2)
            ck(fdg::launch_row_fused(st, lc, a->z.d(), a->d2.d(), a->d.d(), a->tmp.d(), a->u.d(), op->nt, op->n1,
                                     op->n2, op->row_axis(), op->scale2(), stf, op->psi, sc.at(S_RZ1), sc.at(S_PQ),
                                     sc.at(S_RZ0), sc.at(S_RZ1), false, true),
               "K1F");
          else
            ck(fdg::launch_row_apply(st, lc, a->d.d(), a->u.d(), op->nt, op->n1, op->n2, op->row_axis(),
                                     op->scale2(), stf, op->psi, false),
               "K1");
        },
        [&] { ck(fdg::launch_col_s_mid(st, lc, a->d.d(), a->u.d(), a->w.d(), a->vp.d(), op->nt, op->n1, op->n2,
                                       op->ax1, op->scale1(), a->inv_m2.d(), a->a1.d(), sc.slot(S_DOT)), "K2"); },
        [&] { ck(fdg::launch_row_s_out(st, lc, a->w.d(), a->vp.d(), nullptr, a->r.d(), op->nt, op->n1, op->n2,
                                       op->row_axis(), op->scale2(), stf, op->psi, sc.at(S_RZ0), sc.at(S_PQ),
                                       sc.slot(S_DOT)), "K3"); },
        [&] { ck(fdg::launch_hartley_row(st, lc, a->r.d(), a->u.d(), F, pc->n2, pc->tab.tw_2, nullptr, RedSlot{}),
                 "P1"); },
        [&] { ck(fdg::launch_hartley_col(st, lc, a->u.d(), pc->nt, pc->n1, pc->n2, pc->tab.tw_1), "P2"); },
        [&] { ck(fdg::launch_t_filter(st, lc, a->u.d(), pc->tab), "P3"); },
        [&] { ck(fdg::launch_hartley_col(st, lc, a->u.d(), pc->nt, pc->n1, pc->n2, pc->tab.tw_1), "P4"); },
        [&] { ck(fdg::launch_hartley_row(st, lc, a->u.d(), a->z.d(), F, pc->n2, pc->tab.tw_2, a->r.d(), sc.slot(S_DOT)),
                 "P5"); },
        [&] { ck(fdg::launch_axpy_dev(st, lc, a->tmp.d(), a->d.d(), N, sc.at(S_RZ0), sc.at(S_PQ)), "X"); },
    };
    // algorithmic HBM bytes per launch (each N-vector read or written once)
    const double nb = 8.0 * (double)N;
    // K1F: reads z, d_old, x; writes d_new, u, x (the x update of the
    // previous iteration rides along).  X: the stand-alone x += a p, run once
    // per solve (the last iteration's update), not per iteration.
    const double k1 = op->tf.kind != 2 ? 6 * nb : 2 * nb;
    double alg[9] = {k1, 4 * nb, 4 * nb, 2 * nb, 2 * nb, 2 * nb, 2 * nb, 3 * nb, 3 * nb};
    for (size_t i = 0; i < passes.size(); ++i) {
      passes[i]();  // warm
      ck(cudaEventRecord(a->e0, st), "event");
      for (int r = 0; r < reps; ++r) passes[i]();
      ck(cudaEventRecord(a->e1, st), "event");
      ck(cudaEventSynchronize(a->e1), "sync");
      float t = 0.f;
      ck(cudaEventElapsedTime(&t, a->e0, a->e1), "elapsed");
      ms[i] = t / reps;
      if (bytes) bytes[i] = alg[i];
    }
  });
}

// AdmmDriver::step (admm.cpp:245-277)
fdg_status fdg_admm_step(fdg_admm a, fdg_iter_record* rec) {
  return guard([&] {
    if (!a) fail(FDG_EINVAL, "null admm");
    fdg_ctx ctx = a->op->ctx;
    ctx->set_device();
    cudaStream_t st = ctx->stream;
    LaunchCounter* lc = &ctx->lc;
    const auto& d = a->desc;
    ck(cudaEventRecord(a->e2, st), "event");
    build_rhs_dev(a, a->rhs.d(), a->r_cache.d());
    if (!d.warm_start) ck(fdg::launch_fill(st, lc, a->y.d(), 0.0, a->N), "y = 0");
    const double tol = d.fixed_krylov_tol > 0.0 ? d.fixed_krylov_tol : a->inner_tol;
    const fdg_pcg_result inner = pcg_dev(a, a->rhs.d(), a->y.d(), tol, d.max_inner);
    a->stagnations = inner.converged ? 0 : a->stagnations + 1;
    op_apply_dev(a->op, a->y.d(), a->By.d(), false);
    ck(fdg::launch_admm_update(st, lc, admm_scalars(a), a->y.d(), a->v.d(), a->z_y.d(), a->z_v.d(), a->p.d(),
                               a->w_y.d(), a->w_v.d(), a->By.d(), a->r_cache.d(), a->a2inv.d(), a->m2.d(), a->slice,
                               a->N, a->sc.slot(S_ADMM)),
       "admm update");
    ++a->iteration;
    // dual_infeasibility (admm.cpp:275)
    op_apply_dev(a->op, a->p.d(), a->tmp.d(), true);
    ck(fdg::launch_dual_inf(st, lc, a->y.d(), a->ybar.d(), a->tmp.d(), a->w_y.d(), a->v.d(), a->p.d(), a->w_v.d(),
                            a->diag_j.d(), a->diag_j2.d(), a->slice, a->N, a->sc.slot(S_DINF)),
       "dual inf");
    ck(cudaEventRecord(a->e3, st), "event");
    double s[6];
    a->sc.read(S_ADMM, 6, s);  // r_eq, r_y, r_v, bad, s1, s2
    if (s[3] != 0.0)
      fail(FDG_ENUMERIC, "admm: non-finite iterate at outer iteration " + std::to_string(a->iteration),
           FDG_NUM_NONFINITE_ITERATE);
    const double r_eq = s[0], r_y = s[1], r_u = s[2] / a->psi;
    const double tolp = d.tol_primal;
    a->converged = (r_eq <= tolp && r_y <= tolp && r_u <= tolp);
    a->inner_tol = d.inner_tol_factor * std::max(std::min({r_eq, r_y, r_u}), d.inner_tol_floor);
    float step_ms = 0.f;
    ck(cudaEventElapsedTime(&step_ms, a->e2, a->e3), "elapsed");
    if (rec) {
      rec->iter = a->iteration;
      rec->r_eq = r_eq;
      rec->r_y = r_y;
      rec->r_u = r_u;
      rec->dual_inf = std::max(s[4], s[5]);
      rec->inner_iters = inner.iterations;
      rec->inner_tol = a->inner_tol;
      rec->converged = a->converged ? 1 : 0;
      rec->pcg_converged = inner.converged;
      rec->pcg_rel_residual = inner.rel_residual;
      rec->pcg_ms = inner.ms;
      rec->step_ms = step_ms;
    }
  });
}

}  // extern "C"
