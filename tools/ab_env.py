"""A/B timing of the checkerboard engine under env knobs (development tool).

usage: python tools/ab_env.py R C T S  [VAR=val,VAR=val ...]...  each argument
after the config is one variant ('-' = no extra env); every variant runs in a
fresh subprocess so the library re-reads its environment.
"""
import json, os, subprocess, sys

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, '.')
    import torch
    from paper_2505_18508_b200 import TorusSpec, generate_torus
    from paper_2505_18508_b200.campaign import mix_seeds
    from paper_2505_18508_b200.solvers import ANNEALING_CHECKERBOARD, default_config, run_trials_device
    R, C, T, S = map(int, sys.argv[2:6])
    inst = generate_torus(TorusSpec(R, C, 1))
    cfg = default_config(ANNEALING_CHECKERBOARD, S, 0)
    seeds = mix_seeds(20250814, range(T))
    out = run_trials_device(inst, cfg, seeds)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); out = run_trials_device(inst, cfg, seeds); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    import hashlib
    h = hashlib.sha256(out[0].cpu().numpy().tobytes() + out[2].cpu().numpy().tobytes()).hexdigest()[:12]
    print(json.dumps({"t": round(min(ts), 5), "ups": "%.4e" % (T * S * R * C / min(ts)), "sha": h}))
    sys.exit(0)

cfgs = sys.argv[1:5]
for var in sys.argv[5:] or ["-"]:
    env = dict(os.environ)
    if var != "-":
        for kv in var.split(","):
            k, v = kv.split("=")
            env[k] = v
    r = subprocess.run([sys.executable, __file__, "--child", *cfgs], env=env, capture_output=True, text=True)
    line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-500:]
    print(f"{' '.join(cfgs)} [{var}] {line}", flush=True)
