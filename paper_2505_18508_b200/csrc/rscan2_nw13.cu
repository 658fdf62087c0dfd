// rscan2_nw13.cu -- random-scan kernels for teams of 13 warps per trial: two rows
// per lane for 100-row tori of 7 words per row (config 4: 13 warps of 4 row blocks)
// (template: rscan2_kernel.cuh; one translation unit per team size so the
// instantiations compile in parallel).
#include "rscan2_kernel.cuh"

namespace gsb {
RS2_DEFINE_TABLE_WIDE(13)
}  // namespace gsb
