import sys, torch; sys.path.insert(0, '.')
from paper_2505_18508_b200 import TorusSpec, generate_torus
from paper_2505_18508_b200.campaign import mix_seeds
from paper_2505_18508_b200.solvers import default_config, run_trials_device, _test_rscan_slices
CFG = {"c2full": (100, 100, 1024, 10000), "c3": (100, 140, 4096, 2000), "c4": (100, 200, 8192, 1000), "c2x2048": (100,100,2048,3000), "c2x700": (100,100,700,3000)}
for name in sys.argv[1:]:
    R, C, T, S = CFG[name]
    inst = generate_torus(TorusSpec(R, C, 1)); cfg = default_config("simulated_annealing_random_scan", S, 0)
    seeds = mix_seeds(20250814, range(T))
    for sl in (13, 20, 32, 64, 128):
        _test_rscan_slices(sl)
        run_trials_device(inst, cfg, seeds); torch.cuda.synchronize()
        ts = []
        for _ in range(2):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); b = run_trials_device(inst, cfg, seeds, check=False); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3)
        t = min(ts)
        print(f"{name} slices={sl}: {t*1e3:.1f} ms {T*S*R*C/t:.3e} upd/s digest {int(b[0].sum())}", flush=True)
