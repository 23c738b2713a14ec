// fdg_inst_1024c.cu — explicit instantiation unit (Column passes, embedding length 1024; 1024-point Hartley passes) of the pass launchers in
// fdg_launch.cuh; one translation unit per group so nvcc compiles them in
// parallel.
#define FDG_LAUNCH_DEFS
#include "fdg_launch.cuh"

namespace fdg {
FDG_INST_COL(1024)
FDG_INST_H(1024)
}  // namespace fdg
