"""A/B of the reference warp kernel variants (development tool; GPU):
V1 (32-draw Fisher-Yates batches, ungated scan) vs the default V2.
Min of 3 alternating runs each."""
import os, sys
sys.path.insert(0, '.')
import torch
from paper_2505_18508_b200 import TorusSpec, generate_torus
from paper_2505_18508_b200.campaign import mix_seeds
from paper_2505_18508_b200.solvers import ANNEALING, default_config, run_trials_device

VARIANTS = {"V1": "GSB_REFWARP_V1", "V2": None}
for (R, C, T, S) in [(50, 100, 100, 500), (100, 100, 1024, 200), (100, 140, 1184, 100),
                     (100, 200, 1184, 100)]:
    inst = generate_torus(TorusSpec(R, C, 1))
    cfg = default_config(ANNEALING, S, 0)
    seeds = mix_seeds(20250814, range(T))
    best = {}
    for rep in range(3):
        for name, env in VARIANTS.items():
            for e in VARIANTS.values():
                if e:
                    os.environ.pop(e, None)
            if env:
                os.environ[env] = "1"
            run_trials_device(inst, cfg, seeds[:8]); torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); run_trials_device(inst, cfg, seeds); e1.record(); torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / 1e3
            best[name] = min(best.get(name, 1e9), t)
    print(f"{R}x{C} T={T} S={S}: " + "  ".join(f"{k} {T*S*inst.n/v:.3e}" for k, v in best.items()),
          flush=True)
