"""B200-native sweep engine for the gsetbench Max-Cut / Ising hot path.

Drop-in surface for the reference's solver path (gsetbench, arxiv 2505.18508):
problem construction, run_trial / run_campaign and TrialResult, backed by
hand-written sm_100a CUDA kernels in libgsb_cuda.so (include/gsb.h).
"""

from paper_2505_18508_b200.codec import decode_hex, encode_hex
from paper_2505_18508_b200.instances import (
    GsetFormatError,
    ProblemInstance,
    TorusSpec,
    generate_torus,
    parse_gset,
    parse_torus_name,
)

__all__ = [
    "ProblemInstance",
    "TorusSpec",
    "GsetFormatError",
    "generate_torus",
    "parse_gset",
    "parse_torus_name",
    "decode_hex",
    "encode_hex",
]

__version__ = "0.1.0"
