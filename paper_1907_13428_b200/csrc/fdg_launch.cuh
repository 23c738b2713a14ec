// fdg_launch.cuh — persistent-grid launchers of the FFT passes.
//
// run_row / run_col / run_hrow / run_hcol / run_tf are declared here for the
// dispatchers in fdg_kernels.cu and defined (FDG_LAUNCH_DEFS) and explicitly
// instantiated per transform length in the fdg_inst_*.cu translation units,
// which nvcc compiles in parallel.
#pragma once

#include <cuda_runtime.h>

#include "fdg_conv.cuh"
#include "fdg_convq.cuh"
#include "fdg_fft.cuh"
#include "fdg_internal.h"
#include "fdg_passes.cuh"

namespace fdg {

template <int L, int MODE>
cudaError_t run_row(cudaStream_t st, const RowArgs& a);
template <int L, int MODE>
cudaError_t run_col(cudaStream_t st, const ColArgs& a);
template <int N>
cudaError_t run_hrow(cudaStream_t st, const double* in, double* out, int F, const double2* tw, const double* rdot,
                     RedSlot red, const int* guard);
template <int N>
cudaError_t run_hcol(cudaStream_t st, double* data, int O, int C, const double2* tw, const int* guard);
template <int N>
cudaError_t run_tf(cudaStream_t st, double* data, const PcTables& pt, const int* guard);

// ================================================================ dispatch
#ifndef FDG_PDL
#define FDG_PDL 1
#endif
#ifndef FDG_CARVEOUT
#define FDG_CARVEOUT 0
#endif
#define FDG_POW2_CASES(X) X(2) X(4) X(8) X(16) X(32) X(64) X(128) X(256) X(512) X(1024) X(2048)

// Opt in to > 48 KB dynamic shared memory and size the persistent grid
// (resident CTAs x SMs) once per kernel instantiation and device.
struct LaunchShape {
  int device = -1;
  int grid = 0;
};

template <auto K>
inline cudaError_t prep(size_t smem, int threads, int& grid_cap) {
  static LaunchShape ls;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (ls.device != dev) {
    // FDG_CARVEOUT=1: every pass kernel asks for the max-shared L1 split
    // (no measurable gain in the C2 chain; costs the L1-resident twiddle
    // reads of the L = 2048 direct passes, so off by default)
#if FDG_CARVEOUT
    e = cudaFuncSetAttribute(K, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return e;
#endif
    if (smem > 48 * 1024) {
      e = cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    int per_sm = 0, sms = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, K, threads, smem);
    if (e != cudaSuccess) return e;
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    ls.grid = (per_sm < 1 ? 1 : per_sm) * sms;
    ls.device = dev;
  }
  grid_cap = ls.grid;
  return cudaSuccess;
}

inline void count(LaunchCounter* lc, unsigned long long k = 1) {
  if (lc) lc->count += k;
}

// Launch with programmatic stream serialization (PDL): the kernel may begin
// while its predecessor drains; it synchronizes with griddepcontrol.wait
// (fdg_passes.cuh pdl_wait) before touching the predecessor's outputs.
// Launch classes for the programmatic-dependent-launch policy (pdl_mask):
// 1 K row passes, 2 K column passes, 4 P row passes, 8 P column passes,
// 16 t filter, 32 control / axpy / pipe.
// PDL_L1 marks unstaged variants, whose loads and twiddles go through L1:
// launched programmatically right behind a kernel with a large shared-memory
// footprint they inherit that SM configuration (a small L1) instead of the
// L1-heavy one the driver picks for an idle SM (measured at 128 x 1024^2:
// the unstaged x1 pass K2 behind K1 loses 1.4 ms per iteration), so they use
// PDL only right behind another unstaged kernel.
enum PdlClass { PDL_KROW = 1, PDL_KCOL = 2, PDL_PROW = 4, PDL_PCOL = 8, PDL_TF = 16, PDL_MISC = 32, PDL_L1 = 64 };
int pdl_mask();             // fdg_kernels.cu: FDG_PDL_MASK (env) or the default
bool pdl_after(bool l1);    // fdg_kernels.cu: whether PDL may be used, records this launch
bool pdl_suspended();       // fdg_kernels.cu: PDL off while this thread captures a graph body
void pdl_suspend(bool on);

template <typename... KArgs, typename... Args>
inline cudaError_t pdl_launch(int cls, void (*kernel)(KArgs...), unsigned grid, unsigned block, size_t smem,
                              cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  const bool after = pdl_after((cls & PDL_L1) != 0);
  cfg.numAttrs = (FDG_PDL && (pdl_mask() & cls & 63) && after && !pdl_suspended()) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

inline unsigned clamp_grid(long tiles, int cap) {
  return (unsigned)(tiles < cap ? (tiles < 1 ? 1 : tiles) : cap);
}

#ifdef FDG_LAUNCH_DEFS
#ifndef FDG_SPLIT_CONV
#define FDG_SPLIT_CONV 1
#endif
#ifndef FDG_SPLIT_LMAX
#define FDG_SPLIT_LMAX 2048
#endif
// Embedding lengths served by the split-spectrum passes (fdg_conv.cuh).
template <int L>
struct UseSplit {
  static constexpr bool value = FDG_SPLIT_CONV && L >= 512 && L <= FDG_SPLIT_LMAX;
};

template <int L, int MODE, bool PF, bool SR>
cudaError_t run_rowc_s(cudaStream_t st, const RowArgs& a) {
  using Cf = CCfg<L>;
  constexpr size_t SM = RowCPlan<L, MODE, PF, SR>::SMEM;
  int cap = 0;
  cudaError_t e = prep<k_rowc<L, MODE, PF, SR>>(SM, Cf::THREADS, cap);
  if (e != cudaSuccess) return e;
  const long F = (long)a.nt * a.n1;
  return pdl_launch(PDL_KROW, k_rowc<L, MODE, PF, SR>, clamp_grid((F + 2 * Cf::G - 1) / (2 * Cf::G), cap), Cf::THREADS, SM, st,
                    a);
}

// 2-D tensor map over a [rows][C] double array with a box of [brows][W]
// (fdg_kernels.cu; driver entry point through the runtime).
bool encode_col_map(CUtensorMap* map, const double* base, long rows, int C, int W, int brows);

template <int L, int MODE, bool PF, bool SR>
cudaError_t run_colc_s(cudaStream_t st, const ColArgs& a) {
  using Cf = CCfg<L>;
  constexpr size_t SM = ColCPlan<L, MODE, PF, SR>::SMEM;
  int cap = 0;
  cudaError_t e = prep<k_colc<L, MODE, PF, SR>>(SM, Cf::THREADS, cap);
  if (e != cudaSuccess) return e;
  const long tiles = (long)a.O * ((a.C + 2 * Cf::G - 1) / (2 * Cf::G));
  ColMaps maps{};
  if constexpr (PF && FDG_TMA_COLS == 2) {
    constexpr int W = ColCPlan<L, MODE, PF, SR>::W;
    const int bh = a.n < 256 ? a.n : 256;
    if (!encode_col_map(&maps.x, a.x, (long)a.O * a.n, a.C, W, bh)) return cudaErrorInvalidValue;
    if (MODE == 2 && !encode_col_map(&maps.acc, a.acc, (long)a.O * a.n, a.C, W, bh)) return cudaErrorInvalidValue;
  }
  return pdl_launch(PDL_KCOL, k_colc<L, MODE, PF, SR>, clamp_grid(tiles, cap), Cf::THREADS, SM, st, a, maps);
}

constexpr size_t kMaxSmem = 227 * 1024;

// direct 2n-point passes (fdg_passes.cuh)
template <int L, int MODE, bool PF, bool CH = false>
cudaError_t run_row_direct(cudaStream_t st, const RowArgs& a) {
  using Cf = Cfg<L>;
  constexpr size_t SM = RowPlan<L, MODE, PF>::SMEM;
  int cap = 0;
  cudaError_t e = prep<k_row<L, MODE, PF, CH>>(SM, Cf::THREADS, cap);
  if (e != cudaSuccess) return e;
  const long F = (long)a.nt * a.n1;
  return pdl_launch(PDL_KROW | (PF ? 0 : PDL_L1), k_row<L, MODE, PF, CH>,
                    clamp_grid((F + 2 * Cf::G - 1) / (2 * Cf::G), cap), Cf::THREADS, SM, st, a);
}
template <int L, int MODE, bool PF>
cudaError_t run_row_v(cudaStream_t st, const RowArgs& a) {
  return run_row_direct<L, MODE, PF>(st, a);
}

#ifndef FDG_QSPLIT
#define FDG_QSPLIT 1
#endif
// Q-split passes (fdg_convq.cuh) for full tiles with real symbols.  Rows at
// L = 1024 only: measured at 128 x 512^2 K3 383 -> 369 us, K1 equal; at
// L = 2048 (Q = 8) the input/output combinations and the scattered twist
// loads cost more than the shorter transforms save (K1 1829 -> 2656 us at
// 128 x 1024^2), so the M = 1024 split passes stay.
#ifndef FDG_QSPLIT_LMAX
#define FDG_QSPLIT_LMAX 1024
#endif
template <int L, bool ROWS>
struct UseQ {
  static constexpr bool value = FDG_QSPLIT && (L == 1024 || L == 2048) && L <= FDG_QSPLIT_LMAX && QCfg<L, ROWS>::OK;
};

template <int L, int MODE>
cudaError_t run_rowq(cudaStream_t st, const RowArgs& a) {
  using Cf = QCfg<L, true>;
  constexpr size_t SM = RowQPlan<L, MODE, true>::SMEM;
  int cap = 0;
  cudaError_t e = prep<k_rowq<L, MODE>>(SM, Cf::THREADS, cap);
  if (e != cudaSuccess) return e;
  const long F = (long)a.nt * a.n1;
  return pdl_launch(PDL_KROW, k_rowq<L, MODE>, clamp_grid(F / (2 * Cf::G), cap), Cf::THREADS, SM, st, a);
}

template <int L, int MODE>
cudaError_t run_row(cudaStream_t st, const RowArgs& a) {
  if (a.chirp_in) {  // folded pre-chirp: the unstaged direct MODE 0 pass only
    if constexpr (MODE == 0) return run_row_direct<L, 0, false, true>(st, a);
    return cudaErrorNotSupported;
  }
  if constexpr (UseQ<L, true>::value) {
    if (2 * a.n == L && a.n1 % (2 * QCfg<L, true>::G) == 0 && a.sym_re && a.tw256 && a.twq &&
        RowQPlan<L, MODE, true>::SMEM <= 227 * 1024)
      return run_rowq<L, MODE>(st, a);
  }
  // pipelined full tiles: n == L/2 and tiles of 2G fibres inside one slice
  if constexpr (UseSplit<L>::value) {
    // split passes for full staged tiles; ragged shapes take the direct
    // 2n-point kernels (their unstaged epilogue hides latency better)
    if (2 * a.n == L && a.n1 % (2 * CCfg<L>::G) == 0) {
      if (a.sym_re) {
        if constexpr (RowCPlan<L, MODE, true, true>::SMEM <= kMaxSmem) return run_rowc_s<L, MODE, true, true>(st, a);
      } else {
        if constexpr (RowCPlan<L, MODE, true, false>::SMEM <= kMaxSmem) return run_rowc_s<L, MODE, true, false>(st, a);
      }
    }
    return run_row_direct<L, MODE, false>(st, a);
  } else {
    if constexpr (Cfg<L>::PF_OK) {
      if (2 * a.n == L && a.n1 % (2 * Cfg<L>::G) == 0) return run_row_v<L, MODE, true>(st, a);
    }
    return run_row_v<L, MODE, false>(st, a);
  }
}

template <int L, int MODE, bool PF>
cudaError_t run_col_direct(cudaStream_t st, const ColArgs& a) {
  using Cf = Cfg<L>;
  constexpr size_t SM = ColPlan<L, PF>::SMEM;
  int cap = 0;
  cudaError_t e = prep<k_col<L, MODE, PF>>(SM, Cf::THREADS, cap);
  if (e != cudaSuccess) return e;
  const long tiles = (long)a.O * ((a.C + 2 * Cf::G - 1) / (2 * Cf::G));
  return pdl_launch(PDL_KCOL | (PF ? 0 : PDL_L1), k_col<L, MODE, PF>, clamp_grid(tiles, cap), Cf::THREADS, SM, st, a);
}
template <int L, int MODE, bool PF>
cudaError_t run_col_v(cudaStream_t st, const ColArgs& a) {
  return run_col_direct<L, MODE, PF>(st, a);
}

#ifndef FDG_SPLIT_COL_LMAX
#define FDG_SPLIT_COL_LMAX 2048  // L = 2048 split column tiles (W = 4): K2 3195 -> 3169 us at C4 in the chain
#endif
template <int L, int MODE>
cudaError_t run_col(cudaStream_t st, const ColArgs& a) {
  if constexpr (UseSplit<L>::value && L <= FDG_SPLIT_COL_LMAX) {
    if (2 * a.n == L && a.C % (2 * CCfg<L>::G) == 0) {
      if (a.sym_re) {
        if constexpr (ColCPlan<L, MODE, true, true>::SMEM <= kMaxSmem) return run_colc_s<L, MODE, true, true>(st, a);
      } else {
        if constexpr (ColCPlan<L, MODE, true, false>::SMEM <= kMaxSmem) return run_colc_s<L, MODE, true, false>(st, a);
      }
    }
    return run_col_direct<L, MODE, false>(st, a);
  } else {
    // staged full tiles for the direct column kernel where they fit
    if constexpr (Cfg<L>::PF_OK) {
      if (2 * a.n == L && a.C % (2 * Cfg<L>::G) == 0) return run_col_v<L, MODE, true>(st, a);
    }
    return run_col_v<L, MODE, false>(st, a);
  }
}

template <int N, bool PF>
cudaError_t run_hrow_v(cudaStream_t st, const double* in, double* out, int F, const double2* tw,
                              const double* rdot, RedSlot red, const int* guard) {
  using Cf = Cfg<N>;
  constexpr size_t SM = HPlan<N, PF>::SMEM;
  int cap = 0;
  cudaError_t e = prep<k_hartley_row<N, PF>>(SM, Cf::THREADS, cap);
  if (e != cudaSuccess) return e;
  return pdl_launch(PDL_PROW | (PF ? 0 : PDL_L1), k_hartley_row<N, PF>, clamp_grid((F + 2 * Cf::G - 1) / (2 * Cf::G), cap), Cf::THREADS, SM, st,
                    in, out, F, tw, rdot, red, guard);
}

template <int N>
cudaError_t run_hrow(cudaStream_t st, const double* in, double* out, int F, const double2* tw,
                            const double* rdot, RedSlot red, const int* guard) {
  // staged full tiles; at N = 1024 only for the r.z pass, whose unstaged
  // epilogue reads of r stall (measured: 1130 -> 652 us at 128 x 1024^2)
  if constexpr ((Cfg<N>::PF_OK || N == 1024) && HPlan<N, true>::SMEM <= kMaxSmem) {
    if (F % (2 * Cfg<N>::G) == 0 && (Cfg<N>::PF_OK || rdot))
      return run_hrow_v<N, true>(st, in, out, F, tw, rdot, red, guard);
  }
  return run_hrow_v<N, false>(st, in, out, F, tw, rdot, red, guard);
}

template <int N, bool PF>
cudaError_t run_hcol_v(cudaStream_t st, double* data, int O, int C, const double2* tw, const int* guard) {
  using Cf = Cfg<N>;
  constexpr size_t SM = HPlan<N, PF>::SMEM;
  int cap = 0;
  cudaError_t e = prep<k_hartley_col<N, PF>>(SM, Cf::THREADS, cap);
  if (e != cudaSuccess) return e;
  CUtensorMap map{};
  if constexpr (PF && FDG_TMA_PCOL == 2) {
    if (!encode_col_map(&map, data, (long)O * N, C, 2 * Cf::G, N < 256 ? N : 256)) return cudaErrorInvalidValue;
  }
  const long tiles = (long)O * ((C + 2 * Cf::G - 1) / (2 * Cf::G));
  return pdl_launch(PDL_PCOL | (PF ? 0 : PDL_L1), k_hartley_col<N, PF>, clamp_grid(tiles, cap), Cf::THREADS, SM, st, data, O, C, tw, guard,
                    map);
}

template <int N>
cudaError_t run_hcol(cudaStream_t st, double* data, int O, int C, const double2* tw, const int* guard) {
  if constexpr (Cfg<N>::PF_OK) {
    if (C % (2 * Cfg<N>::G) == 0) return run_hcol_v<N, true>(st, data, O, C, tw, guard);
  }
  return run_hcol_v<N, false>(st, data, O, C, tw, guard);
}

template <int N, bool PF>
cudaError_t run_tf_v(cudaStream_t st, double* data, const PcTables& pt, const int* guard) {
  using Cf = Cfg<N>;
  constexpr size_t SM = HPlan<N, PF>::SMEM_T;
  int cap = 0;
  cudaError_t e = prep<k_t_filter<N, PF>>(SM, Cf::THREADS, cap);
  if (e != cudaSuccess) return e;
  CUtensorMap map{};
  if constexpr (PF && FDG_TMA_PCOL == 2) {
    if (!encode_col_map(&map, data, N, pt.n1 * pt.n2, 2 * Cf::G, N < 256 ? N : 256)) return cudaErrorInvalidValue;
  }
  const long C = (long)pt.n1 * pt.n2;
  return pdl_launch(PDL_TF | (PF ? 0 : PDL_L1), k_t_filter<N, PF>, clamp_grid((C + 2 * Cf::G - 1) / (2 * Cf::G), cap), Cf::THREADS, SM, st, data,
                    pt, guard, map);
}

template <int N>
cudaError_t run_tf(cudaStream_t st, double* data, const PcTables& pt, const int* guard) {
  const long C = (long)pt.n1 * pt.n2;
  if constexpr (Cfg<N>::PF_OK) {
    if (C % (2 * Cfg<N>::G) == 0) return run_tf_v<N, true>(st, data, pt, guard);
  }
  return run_tf_v<N, false>(st, data, pt, guard);
}


// Explicit instantiations (fdg_inst_*.cu).
#define FDG_INST_ROW(L)                                                    \
  template cudaError_t run_row<L, 0>(cudaStream_t, const RowArgs&);        \
  template cudaError_t run_row<L, 1>(cudaStream_t, const RowArgs&);        \
  template cudaError_t run_row<L, 2>(cudaStream_t, const RowArgs&);
#define FDG_INST_COL(L)                                                    \
  template cudaError_t run_col<L, 0>(cudaStream_t, const ColArgs&);        \
  template cudaError_t run_col<L, 2>(cudaStream_t, const ColArgs&);
#define FDG_INST_H(N)                                                                                         \
  template cudaError_t run_hrow<N>(cudaStream_t, const double*, double*, int, const double2*, const double*,   \
                                   RedSlot, const int*);                                                     \
  template cudaError_t run_hcol<N>(cudaStream_t, double*, int, int, const double2*, const int*);              \
  template cudaError_t run_tf<N>(cudaStream_t, double*, const PcTables&, const int*);
#endif  // FDG_LAUNCH_DEFS

}  // namespace fdg
