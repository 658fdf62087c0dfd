"""Config 2 in full on the library named by GSB_LIB (development A/B tool)."""
import sys, torch; sys.path.insert(0, ".")
from paper_2505_18508_b200 import TorusSpec, generate_torus
from paper_2505_18508_b200.campaign import mix_seeds
from paper_2505_18508_b200.solvers import default_config, run_trials_device
for (R,C,T,S) in [(100,100,1024,10000),(100,100,2048,3000)]:
    inst = generate_torus(TorusSpec(R, C, 1)); cfg = default_config("simulated_annealing_random_scan", S, 0)
    seeds = mix_seeds(20250814, range(T))
    run_trials_device(inst, cfg, seeds); torch.cuda.synchronize()
    ts=[]
    for _ in range(2):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); run_trials_device(inst, cfg, seeds, check=False); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1)/1e3)
    t=min(ts)
    print(R,C,T,S, f"{t*1e3:.1f} ms {T*S*R*C/t:.3e}", flush=True)
