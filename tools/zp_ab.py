"""A/B of the comparator specialisation (GSB_CHECKER_ZP = 0 / 4 / 8) per config (development tool)."""
import os, sys
sys.path.insert(0, ".")
import torch
from paper_2505_18508_b200 import TorusSpec, generate_torus
from paper_2505_18508_b200.campaign import mix_seeds
from paper_2505_18508_b200.solvers import ANNEALING_CHECKERBOARD, default_config, run_trials_device


def timeit(inst, cfg, seeds, reps=3):
    run_trials_device(inst, cfg, seeds)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        run_trials_device(inst, cfg, seeds)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return min(ts)


shapes = [(50, 100, 100, 1000), (100, 100, 1024, 4000), (100, 140, 4096, 1000), (100, 200, 8192, 500)]
for R, C, T, S in shapes:
    inst = generate_torus(TorusSpec(R, C, 1))
    cfg = default_config(ANNEALING_CHECKERBOARD, S, 0)
    seeds = mix_seeds(20250814, range(T))
    res = []
    for zp in ["0", "4", "8"]:
        os.environ["GSB_CHECKER_ZP"] = zp
        t = timeit(inst, cfg, seeds)
        res.append(f"zp<={zp}:{T * S * inst.n / t:.3e}")
    print(f"{R}x{C} T={T} S={S}: " + "  ".join(res), flush=True)
