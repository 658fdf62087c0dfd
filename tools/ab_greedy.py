"""Greedy random scan at configs 2-4's trial counts on the library named by GSB_LIB (A/B tool)."""
import sys, torch; sys.path.insert(0, ".")
from paper_2505_18508_b200 import TorusSpec, generate_torus
from paper_2505_18508_b200.campaign import mix_seeds
from paper_2505_18508_b200.solvers import default_config, run_trials_device
for (R,C,T) in [(100,100,1024),(100,140,4096),(100,200,8192)]:
    inst = generate_torus(TorusSpec(R, C, 1)); cfg = default_config("greedy_random_scan", 1000, 0)
    seeds = mix_seeds(20250814, range(T))
    b = run_trials_device(inst, cfg, seeds); torch.cuda.synchronize()
    ts=[]
    for _ in range(3):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); b = run_trials_device(inst, cfg, seeds, check=False); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1)/1e3)
    t=min(ts); upd=int(b[1].sum())*R*C
    print(R,C,T, f"{t*1e3:.2f} ms {upd/t:.3e} upd/s digest {int(b[0].sum())}", flush=True)
