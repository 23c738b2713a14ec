// fdg_inst_1024r.cu — explicit instantiation unit (Row passes, embedding length 1024) of the pass launchers in
// fdg_launch.cuh; one translation unit per group so nvcc compiles them in
// parallel.
#define FDG_LAUNCH_DEFS
#include "fdg_launch.cuh"

namespace fdg {
FDG_INST_ROW(1024)
}  // namespace fdg
