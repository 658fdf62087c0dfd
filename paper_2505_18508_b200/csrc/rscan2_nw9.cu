// rscan2_nw9.cu -- random-scan kernels for teams of 9 warps per trial: two rows
// per lane for 100-row tori of 5 words per row (config 3: 9 warps of 6 row blocks)
// (template: rscan2_kernel.cuh; one translation unit per team size so the
// instantiations compile in parallel).
#include "rscan2_kernel.cuh"

namespace gsb {
RS2_DEFINE_TABLE_WIDE(9)
}  // namespace gsb
