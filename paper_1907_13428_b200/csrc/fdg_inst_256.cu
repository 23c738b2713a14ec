// fdg_inst_256.cu — explicit instantiation unit (Transform length 256) of the pass launchers in
// fdg_launch.cuh; one translation unit per group so nvcc compiles them in
// parallel.
#define FDG_LAUNCH_DEFS
#include "fdg_launch.cuh"

namespace fdg {
FDG_INST_ROW(256)
FDG_INST_COL(256)
FDG_INST_H(256)

}  // namespace fdg
