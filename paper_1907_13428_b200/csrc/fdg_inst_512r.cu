// fdg_inst_512r.cu — explicit instantiation unit (Row passes, embedding length 512) of the pass launchers in
// fdg_launch.cuh; one translation unit per group so nvcc compiles them in
// parallel.
#define FDG_LAUNCH_DEFS
#include "fdg_launch.cuh"

namespace fdg {
FDG_INST_ROW(512)
}  // namespace fdg
