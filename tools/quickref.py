import sys; sys.path.insert(0, '.')
import torch
from paper_2505_18508_b200 import TorusSpec, generate_torus
from paper_2505_18508_b200.campaign import mix_seeds
from paper_2505_18508_b200.solvers import *
for (R, C, T, S) in [(50, 100, 100, 1000), (100, 100, 1024, 200), (100, 200, 1184, 100)]:
    inst = generate_torus(TorusSpec(R, C, 1))
    cfg = default_config(ANNEALING, S, 0)
    seeds = mix_seeds(20250814, range(T))
    run_trials_device(inst, cfg, seeds[:8]); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); run_trials_device(inst, cfg, seeds); e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3
    print(f"reference engine {R}x{C} T={T} S={S}: {t*1e3:.1f} ms {T*S*inst.n/t:.3e} upd/s", flush=True)
