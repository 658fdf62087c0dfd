"""Config-5 cluster-engine run for ncu (development tool): T trials x S sweeps."""
import sys; sys.path.insert(0, '.')
import torch
from paper_2505_18508_b200 import TorusSpec, generate_torus, _lib
from paper_2505_18508_b200.campaign import mix_seeds
from paper_2505_18508_b200.solvers import ANNEALING_CHECKERBOARD, default_config, run_trials_device
inst = generate_torus(TorusSpec(2000, 2000, 1))
S = int(sys.argv[1]) if len(sys.argv) > 1 else 200
T = int(sys.argv[2]) if len(sys.argv) > 2 else 8
cfg = default_config(ANNEALING_CHECKERBOARD, S, 0)
for _ in range(2):
    run_trials_device(inst, cfg, mix_seeds(20250814, range(T)), engine=_lib.ENGINE_CHECKERBOARD_CLUSTER)
torch.cuda.synchronize(); print("done")
