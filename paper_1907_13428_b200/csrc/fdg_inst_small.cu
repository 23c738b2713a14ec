// fdg_inst_small.cu — explicit instantiation unit (Transform lengths 1..128) of the pass launchers in
// fdg_launch.cuh; one translation unit per group so nvcc compiles them in
// parallel.
#define FDG_LAUNCH_DEFS
#include "fdg_launch.cuh"

namespace fdg {
FDG_INST_ROW(2)
FDG_INST_ROW(4)
FDG_INST_ROW(8)
FDG_INST_ROW(16)
FDG_INST_ROW(32)
FDG_INST_ROW(64)
FDG_INST_ROW(128)
FDG_INST_COL(2)
FDG_INST_COL(4)
FDG_INST_COL(8)
FDG_INST_COL(16)
FDG_INST_COL(32)
FDG_INST_COL(64)
FDG_INST_COL(128)
FDG_INST_H(1)
FDG_INST_H(2)
FDG_INST_H(4)
FDG_INST_H(8)
FDG_INST_H(16)
FDG_INST_H(32)
FDG_INST_H(64)
FDG_INST_H(128)
}  // namespace fdg
