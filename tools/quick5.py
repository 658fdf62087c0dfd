"""Config-5 timing (development tool): cluster vs HBM-tiled engine, 8 trials."""
import sys
sys.path.insert(0, '.')
import torch
from paper_2505_18508_b200 import TorusSpec, generate_torus, _lib
from paper_2505_18508_b200.campaign import mix_seeds
from paper_2505_18508_b200.solvers import ANNEALING_CHECKERBOARD, default_config, run_trials_device
inst = generate_torus(TorusSpec(2000, 2000, 1))
T = int(sys.argv[1]) if len(sys.argv) > 1 else 8
for eng in (_lib.ENGINE_CHECKERBOARD_CLUSTER, _lib.ENGINE_CHECKERBOARD_TILED):
    for S in (100, 1000):
        cfg = default_config(ANNEALING_CHECKERBOARD, S, 0)
        seeds = mix_seeds(20250814, range(T))
        run_trials_device(inst, cfg, seeds, engine=eng); torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); run_trials_device(inst, cfg, seeds, engine=eng); e1.record(); torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3
        print(f"C5 engine={eng} T={T} S={S}: {t*1e3:.1f} ms {T*S*inst.n/t:.3e} upd/s", flush=True)
