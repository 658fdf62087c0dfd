import sys; sys.path.insert(0, '.')
import torch
from paper_2505_18508_b200 import TorusSpec, generate_torus
from paper_2505_18508_b200.campaign import mix_seeds
from paper_2505_18508_b200.solvers import *
inst = generate_torus(TorusSpec(100, 100, 1))
cfg = default_config(ANNEALING, int(sys.argv[1]) if len(sys.argv) > 1 else 100, 0)
for _ in range(2):
    run_trials_device(inst, cfg, mix_seeds(20250814, range(1024)))
torch.cuda.synchronize(); print("done")
