import sys, time; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2505_18508_b200 import TorusSpec, generate_torus, _lib
from paper_2505_18508_b200.campaign import mix_seeds
from paper_2505_18508_b200.solvers import default_config, run_trials_device
L = _lib.lib()
inst = generate_torus(TorusSpec(100, 100, 1)); n = inst.n; T = 1024; S = 10000
cfg = default_config("simulated_annealing_checkerboard", S, 0)
seeds = mix_seeds(20250814, range(T))
w_h = torch.from_numpy(inst.torus_weights.copy()).pin_memory()
s_h = torch.from_numpy(seeds.view(np.int64).copy()).pin_memory()
bc = torch.empty(T, dtype=torch.int64).pin_memory(); se = torch.empty(T, dtype=torch.int32).pin_memory()
bits = torch.empty((T, (n + 7) // 8), dtype=torch.uint8).pin_memory()
sp = torch.cuda.current_stream().cuda_stream
def host():
    _lib.check(L.gsb_torus_sweep_host(100, 100, w_h.data_ptr(), 1, 1, S, 3.0, 0.05, s_h.data_ptr(), T,
                                      bc.data_ptr(), se.data_ptr(), bits.data_ptr(), sp))
for _ in range(2): host()
for _ in range(3):
    t0 = time.perf_counter(); host(); t1 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); run_trials_device(inst, cfg, seeds); e1.record(); torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"host {1e3*(t1-t0):.1f} ms   device-api {e0.elapsed_time(e1):.1f} ms (wall {1e3*(t2-t1):.1f})", flush=True)
flush = torch.empty(2 * 126 * 1024 * 1024, dtype=torch.uint8, device="cuda")
print("with L2 flush between calls:")
for _ in range(4):
    flush.zero_(); torch.cuda.synchronize()
    t0 = time.perf_counter(); host(); t1 = time.perf_counter()
    flush.zero_(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); run_trials_device(inst, cfg, seeds); e1.record(); torch.cuda.synchronize()
    print(f"host {1e3*(t1-t0):.1f} ms   device-api {e0.elapsed_time(e1):.1f} ms", flush=True)
