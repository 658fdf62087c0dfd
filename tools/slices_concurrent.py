"""Sliced random-scan launches from several host threads on their own streams
at once (development tool): teams of different launches share the SMs while
they wait on one another's flags; results must equal the serial launches'.
usage: python tools/slices_concurrent.py [threads] [rounds]"""
import sys, threading
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2505_18508_b200 import TorusSpec, generate_torus
from paper_2505_18508_b200.campaign import mix_seeds
from paper_2505_18508_b200.solvers import default_config, run_trials_device, _test_rscan_slices

nthreads = int(sys.argv[1]) if len(sys.argv) > 1 else 4
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 3
_test_rscan_slices(7)
jobs = [((100, 100), 700, 60), ((50, 100), 900, 80), ((100, 140), 500, 40), ((40, 33), 1500, 90)]
ref = []
for (R, C), T, S in jobs:
    inst = generate_torus(TorusSpec(R, C, 1))
    b = run_trials_device(inst, default_config("simulated_annealing_random_scan", S, 0),
                          mix_seeds(7, range(T)))
    ref.append((inst, T, S, b[0].cpu().numpy().copy(), b[2].cpu().numpy().copy()))
torch.cuda.synchronize()
bad = []
def work(k):
    st = torch.cuda.Stream()
    for r in range(rounds):
        inst, T, S, cuts, bits = ref[(k + r) % len(ref)]
        with torch.cuda.stream(st):
            b = run_trials_device(inst, default_config("simulated_annealing_random_scan", S, 0),
                                  mix_seeds(7, range(T)), stream=st)
        st.synchronize()
        if not (np.array_equal(b[0].cpu().numpy(), cuts) and np.array_equal(b[2].cpu().numpy(), bits)):
            bad.append((k, r))
ths = [threading.Thread(target=work, args=(k,)) for k in range(nthreads)]
[t.start() for t in ths]; [t.join() for t in ths]
print("concurrent sliced launches:", nthreads, "threads x", rounds, "rounds; mismatches:", len(bad))
sys.exit(1 if bad else 0)
