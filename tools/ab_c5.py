"""A/B of the cluster engine (config 5, 7 trials x 300 sweeps) between two builds of
the library (development tool): GSB_LIB=build_variants/libgsb_old.so vs the in-tree one."""
import os, subprocess, sys, json
code = r'''
import sys; sys.path.insert(0, '.')
import torch
from paper_2505_18508_b200 import TorusSpec, generate_torus, _lib
from paper_2505_18508_b200.campaign import mix_seeds
from paper_2505_18508_b200.solvers import ANNEALING_CHECKERBOARD, default_config, run_trials_device
inst = generate_torus(TorusSpec(2000, 2000, 1))
cfg = default_config(ANNEALING_CHECKERBOARD, 300, 0)
seeds = mix_seeds(20250814, range(7))
out = run_trials_device(inst, cfg, seeds, engine=_lib.ENGINE_CHECKERBOARD_CLUSTER); torch.cuda.synchronize()
ts = []
for _ in range(3):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); out = run_trials_device(inst, cfg, seeds, engine=_lib.ENGINE_CHECKERBOARD_CLUSTER); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / 1e3)
import hashlib
print("%.4e" % (7 * 300 * inst.n / min(ts)), hashlib.sha256(out[0].cpu().numpy().tobytes() + out[2].cpu().numpy().tobytes()).hexdigest()[:12])
'''
for rep in range(2):
    for lib in ("build_variants/libgsb_old.so", ""):
        env = dict(os.environ)
        if lib: env["GSB_LIB"] = lib
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        print(lib or "new", r.stdout.strip(), r.stderr.strip()[-300:], flush=True)
