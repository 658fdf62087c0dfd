import sys, time; sys.path.insert(0, '.')
import torch
from paper_2505_18508_b200 import TorusSpec, generate_torus
from paper_2505_18508_b200.campaign import mix_seeds
from paper_2505_18508_b200.solvers import *
inst = generate_torus(TorusSpec(2000, 2000, 1))
for T, S in [(8, 100), (8, 1000)]:
    cfg = default_config(ANNEALING_CHECKERBOARD, S, 0)
    seeds = mix_seeds(20250814, range(T))
    run_trials_device(inst, cfg, seeds); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); run_trials_device(inst, cfg, seeds); e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3
    print(f"C5 T={T} S={S}: {t*1e3:.1f} ms {T*S*inst.n/t:.3e} upd/s", flush=True)
