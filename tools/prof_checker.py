"""Run the checkerboard kernel once on a given config (for ncu)."""
import sys; sys.path.insert(0,'.')
import torch
from paper_2505_18508_b200 import TorusSpec, generate_torus
from paper_2505_18508_b200.campaign import mix_seeds
from paper_2505_18508_b200.solvers import *
R,C,T,S = [int(x) for x in sys.argv[1:5]] if len(sys.argv) > 4 else (100,100,1024,500)
kind = sys.argv[5] if len(sys.argv) > 5 else ANNEALING_CHECKERBOARD
inst=generate_torus(TorusSpec(R,C,1))
seeds=mix_seeds(20250814, range(T))
for _ in range(2):
    run_trials_device(inst, default_config(kind,S,0), seeds)
torch.cuda.synchronize()
print("done")
