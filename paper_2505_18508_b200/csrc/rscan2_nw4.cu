// rscan2_nw4.cu -- random-scan kernels for teams of 4 warps per trial
// (template: rscan2_kernel.cuh; one translation unit per team size so the
// instantiations compile in parallel).
#include "rscan2_kernel.cuh"

namespace gsb {
RS2_DEFINE_TABLE(4)
}  // namespace gsb
