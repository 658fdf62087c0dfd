GSB_RSCAN_SCALAR=1 timeout 900 python -m pytest tests/test_rscan_gpu.py -q -m gpu -x 2>&1 | tail -2
timeout 900 python -m pytest tests/test_rscan_gpu.py -q -m gpu -x 2>&1 | tail -2

timeout 300 python - <<'PY'
import sys, torch; sys.path.insert(0, '.')
from paper_2505_18508_b200 import TorusSpec, generate_torus
from paper_2505_18508_b200.campaign import mix_seeds
from paper_2505_18508_b200.solvers import default_config, run_trials_device
for (R, C, T, S, kind) in [(100, 100, 1024, 1000, "simulated_annealing_random_scan"),
                           (50, 100, 100, 1000, "simulated_annealing_random_scan"),
                           (100, 200, 1024, 300, "simulated_annealing_random_scan")]:
    inst = generate_torus(TorusSpec(R, C, 1)); cfg = default_config(kind, S, 0)
    seeds = mix_seeds(20250814, range(T))
    run_trials_device(inst, cfg, seeds); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); run_trials_device(inst, cfg, seeds); e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3
    print(f"BS {kind} {R}x{C} T={T} S={S}: {t*1e3:.1f} ms {T*S*R*C/t:.3e} upd/s", flush=True)
PY
