"""Quick timing of the engines (development tool)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2505_18508_b200 import TorusSpec, generate_torus
from paper_2505_18508_b200.campaign import mix_seeds
from paper_2505_18508_b200.solvers import *

def timeit(inst, cfg, T, reps=3):
    seeds = mix_seeds(20250814, range(T))
    run_trials_device(inst, cfg, seeds)
    torch.cuda.synchronize()
    ts=[]
    for _ in range(reps):
        e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
        e0.record(); run_trials_device(inst, cfg, seeds); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1)/1e3)
    t=min(ts)
    upd = T*cfg.sweeps*inst.n
    print(f"{inst.name} {cfg.kind} T={T} S={cfg.sweeps}: {t*1e3:.2f} ms  {upd/t:.3e} upd/s", flush=True)

for (R,C,T,S) in [(50,100,100,1000),(100,100,1024,10000),(100,140,4096,2000),(100,200,8192,1000)]:
    inst = generate_torus(TorusSpec(R,C,1))
    timeit(inst, default_config(ANNEALING_CHECKERBOARD, S, 0), T)
inst = generate_torus(TorusSpec(50,100,1))
timeit(inst, default_config(ANNEALING, 20, 0), 100, reps=1)
