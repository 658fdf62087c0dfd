"""Device-timed rate of one kind on the BASELINE configs (development tool):
python tools/rates.py KIND [c1 c2 ...]"""
import sys, torch; sys.path.insert(0, '.')
from paper_2505_18508_b200 import TorusSpec, generate_torus
from paper_2505_18508_b200.campaign import mix_seeds
from paper_2505_18508_b200.solvers import default_config, run_trials_device
CFG = {"c1": (50, 100, 100, 1000), "c2": (100, 100, 1024, 1000), "c2full": (100, 100, 1024, 10000),
       "c3": (100, 140, 4096, 300), "c4": (100, 200, 8192, 100), "c2x148": (100, 100, 148, 1000),
       "c2x2048": (100, 100, 2048, 1000), "c5x8": (2000, 2000, 8, 100), "c5": (2000, 2000, 64, 100),
       "c5x1": (2000, 2000, 1, 100), "c5x8full": (2000, 2000, 8, 1000)}
kind = sys.argv[1]
for name in (sys.argv[2:] or ["c1", "c2", "c3", "c4"]):
    R, C, T, S = CFG[name]
    inst = generate_torus(TorusSpec(R, C, 1)); cfg = default_config(kind, S, 0)
    seeds = mix_seeds(20250814, range(T))
    run_trials_device(inst, cfg, seeds); torch.cuda.synchronize()
    ts = []
    for _ in range(2):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); run_trials_device(inst, cfg, seeds, check=False); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    t = min(ts)
    print(f"{kind} {name} {R}x{C} T={T} S={S}: {t*1e3:.1f} ms {T*S*R*C/t:.3e} upd/s", flush=True)
