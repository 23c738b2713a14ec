// fdg_inst_2048c.cu — explicit instantiation unit (Column passes, embedding length 2048; 2048-point Hartley passes) of the pass launchers in
// fdg_launch.cuh; one translation unit per group so nvcc compiles them in
// parallel.
#define FDG_LAUNCH_DEFS
#include "fdg_launch.cuh"

namespace fdg {
FDG_INST_COL(2048)
FDG_INST_H(2048)
}  // namespace fdg
