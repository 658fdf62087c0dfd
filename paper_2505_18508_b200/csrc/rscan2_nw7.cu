// rscan2_nw7.cu -- random-scan kernels for teams of 7 warps per trial (100-row
// tori with 4 words per row fill 7 warps of 8 row blocks, not 8: config 2)
// (template: rscan2_kernel.cuh; one translation unit per team size so the
// instantiations compile in parallel).
#include "rscan2_kernel.cuh"

namespace gsb {
RS2_DEFINE_TABLE(7)
}  // namespace gsb
