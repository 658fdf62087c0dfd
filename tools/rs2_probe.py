"""Random-scan engine probe (development tool): rate, counters and -- with a
GSB_RS2_PROF build (GSB_LIB=build_variants/libgsb_prof.so) -- cycles per phase.
python tools/rs2_probe.py R C T S [nw rb]..."""
import sys, numpy as np, torch; sys.path.insert(0, '.')
from paper_2505_18508_b200 import TorusSpec, _lib, generate_torus
from paper_2505_18508_b200.campaign import mix_seeds
from paper_2505_18508_b200.solvers import default_config, schedule_table
R, C, T, S = map(int, sys.argv[1:5])
shapes = [(int(sys.argv[i]), int(sys.argv[i + 1])) for i in range(5, len(sys.argv) - 1, 2)] or [(0, 0)]
L = _lib.lib(); dev = torch.device("cuda", 0)
inst = generate_torus(TorusSpec(R, C, 1)); w = inst.device_weights(dev)
cfg = default_config("simulated_annealing_random_scan", S, 0)
seeds = torch.from_numpy(mix_seeds(20250814, range(T)).view(np.int64).copy()).to(dev)
tab = torch.from_numpy(schedule_table(cfg, 4).view(np.int64)).to(dev)
ts = _lib.torus_struct(R, C, w.data_ptr()); n = R * C
wsb = L.gsb_torus_workspace_bytes(ts, cfg.engine, S, T)
ws = torch.zeros(wsb, dtype=torch.uint8, device=dev)
best = torch.empty(T, dtype=torch.int64, device=dev); sw = torch.empty(T, dtype=torch.int32, device=dev)
bits = torch.empty((T, (n + 7) // 8), dtype=torch.uint8, device=dev)
sp = torch.cuda.current_stream().cuda_stream
def go():
    _lib.check(L.gsb_torus_sweep(ts, cfg.engine, 1, S, tab.data_ptr(), seeds.data_ptr(), T, best.data_ptr(),
                                 sw.data_ptr(), bits.data_ptr(), ws.data_ptr(), wsb, sp))
for nw, rb in shapes:
    _lib.check(L.gsb_test_rscan_shape(nw, rb))
    try:
        go()
    except ValueError as e:
        print(nw, rb, "unsupported", e); continue
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); go(); e1.record(); torch.cuda.synchronize()
    _lib.check(L.gsb_workspace_status(ws.data_ptr(), sp))
    t = e0.elapsed_time(e1) / 1e3
    st = ws[16:16 + 80].cpu().numpy().view(np.uint64)
    ts_ = T * S
    msg = (f"shape=({nw},{rb}) {R}x{C} T={T} S={S}: {t*1e3:.1f} ms {T*S*n/t:.3e} upd/s | rounds/sweep "
           f"{st[0]/ts_:.2f} gated {st[1]/ts_:.3f} cand/sweep {st[2]/ts_:.3f} ties/sweep {st[3]/ts_:.1f} "
           f"digest {int(best.sum())}")
    if st[4:].any():
        tot = float(st[4:].sum()); names = ["philox+accept", "precedence", "rounds", "deltas", "best4b", "other"]
        msg += " | " + " ".join(f"{nm} {100*float(v)/tot:.1f}%" for nm, v in zip(names, st[4:]))
        msg += f" | cycles/trial-sweep {tot/ts_:.0f}"
    print(msg, flush=True)
