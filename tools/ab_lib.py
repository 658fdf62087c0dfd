"""A/B of one kind/config between two builds of the library (development tool):
python tools/ab_lib.py KIND R C T S  runs GSB_LIB=build_variants/libgsb_old.so and the
in-tree build alternately in fresh processes; prints rate and a result digest each."""
import os, subprocess, sys

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, '.')
    import hashlib
    import torch
    from paper_2505_18508_b200 import TorusSpec, generate_torus
    from paper_2505_18508_b200.campaign import mix_seeds
    from paper_2505_18508_b200.solvers import default_config, run_trials_device
    kind = sys.argv[2]
    R, C, T, S = map(int, sys.argv[3:7])
    inst = generate_torus(TorusSpec(R, C, 1))
    cfg = default_config(kind, S, 0)
    seeds = mix_seeds(20250814, range(T))
    out = run_trials_device(inst, cfg, seeds); torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); out = run_trials_device(inst, cfg, seeds); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    h = hashlib.sha256(out[0].cpu().numpy().tobytes() + out[2].cpu().numpy().tobytes()).hexdigest()[:12]
    print("%.4e %s" % (T * S * R * C / min(ts), h))
    sys.exit(0)

for rep in range(2):
    for lib in ("build_variants/libgsb_old.so", ""):
        env = dict(os.environ)
        if lib:
            env["GSB_LIB"] = lib
        r = subprocess.run([sys.executable, __file__, "--child", *sys.argv[1:]], env=env,
                           capture_output=True, text=True)
        print(" ".join(sys.argv[1:]), lib or "new", r.stdout.strip(), r.stderr.strip()[-300:],
              flush=True)
