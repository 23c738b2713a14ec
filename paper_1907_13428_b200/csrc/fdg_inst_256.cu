// fdg_inst_256.cu — explicit instantiation unit (Transform length 256) of the pass launchers in
// fdg_launch.cuh; one translation unit per group so nvcc compiles them in
// parallel.
#define FDG_LAUNCH_DEFS
#include "fdg_launch.cuh"
#include "fdg_pcfused.cuh"

namespace fdg {
FDG_INST_ROW(256)
FDG_INST_COL(256)
FDG_INST_H(256)

#ifndef FDG_PC_PIPE
#define FDG_PC_PIPE 0  // measured slower than the separate passes at C2
#endif

bool pc_pipe_supported(int n1, int n2) { return FDG_PC_PIPE && n1 == n2 && (n1 == 256 || n1 == 512); }

template <int N>
static cudaError_t run_pipe(cudaStream_t st, const PipeArgs& a) {
  using P = PipeCfg<N>;
  int cap = 0;
  cudaError_t e = prep<k_pc_pipe<N>>(P::SMEM, P::THREADS, cap);
  if (e != cudaSuccess) return e;
  return pdl_launch(PDL_MISC, k_pc_pipe<N>, (unsigned)cap, P::THREADS, P::SMEM, st, a);
}

cudaError_t launch_pc_pipe(cudaStream_t st, LaunchCounter* lc, const double* in, double* mid, double* out,
                           const double* rdot, RedSlot red, int nt, int n, const double2* tw, int* ready,
                           bool rows_first, const int* guard) {
  PipeArgs a{in, mid, out, rdot, red, nt, n, tw, ready, rows_first ? 1 : 0, guard};
  count(lc);
  switch (n) {
    case 256: return run_pipe<256>(st, a);
    case 512: return run_pipe<512>(st, a);
    default: return cudaErrorInvalidValue;
  }
}
}  // namespace fdg
