// fdg_inst_512c.cu — explicit instantiation unit (Column passes, embedding length 512; 512-point Hartley passes) of the pass launchers in
// fdg_launch.cuh; one translation unit per group so nvcc compiles them in
// parallel.
#define FDG_LAUNCH_DEFS
#include "fdg_launch.cuh"

namespace fdg {
FDG_INST_COL(512)
FDG_INST_H(512)
}  // namespace fdg
