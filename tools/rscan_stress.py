"""Randomized stress of the random-scan engine against the CPU oracle
(development tool, longer than the test suite): random shapes up to 1024
columns, schedules, trial counts, forced team shapes and tiny queue limits.
usage: python tools/rscan_stress.py [cases] [seed]"""
import sys
import numpy as np
sys.path.insert(0, '.')
from oracle import oracle as O
from paper_2505_18508_b200 import TorusSpec, _lib, generate_torus
from paper_2505_18508_b200.solvers import (SolverConfig, _test_rscan_limits, _test_rscan_shape,
                                           _test_rscan_slices, rscan_fits, run_trials)

O.build()
cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
bad = 0
for it in range(cases):
    C = int(rng.choice([rng.integers(3, 40), rng.integers(40, 300), rng.integers(300, 1025)]))
    wpr = (C + 31) // 32
    maxrows = 8 * (32 // wpr) * 7
    R = int(rng.integers(3, min(maxrows, max(4, 60000 // C)) + 1))
    if not rscan_fits(R, C):
        continue
    inst = generate_torus(TorusSpec(R, C, int(rng.integers(0, 2**31))))
    sa = rng.random() < 0.8
    S = int(rng.integers(1, 12 if R * C > 5000 else 40))
    t0 = float(rng.uniform(0.2, 6.0))
    cfg = (SolverConfig("simulated_annealing_random_scan", S, 0, t0, t0 * float(rng.uniform(0.01, 0.9)))
           if sa else SolverConfig("greedy_random_scan", 60, 0))
    T = int(rng.choice([1, 3, 50, 600]))
    seeds = [int(x) for x in rng.integers(0, 2**63, size=T)]
    lim = (int(rng.choice([0, 0, 2, 9])), int(rng.choice([0, 0, 3, 30])))
    _test_rscan_limits(*lim)
    forced = (0, 0)
    if rng.random() < 0.5:
        forced = (int(rng.choice([1, 2, 4, 7, 8, 9, 13])), int(rng.choice([1, 2, 3, 4, 5, 7])))
    _test_rscan_shape(*forced)
    slices = int(rng.choice([0, 0, 1, 2, 3, 5, 64]))  # sweep slices of annealing launches
    _test_rscan_slices(slices)
    eng = _lib.ENGINE_RANDOM_SCAN_LARGE if rng.random() < 0.3 else None  # the large-torus engine
    if eng is not None:
        forced = ("large",)
    try:
        b = run_trials(inst, cfg, seeds, engine=eng)
    except ValueError:
        _test_rscan_shape(0, 0)
        forced = (0, 0)
        b = run_trials(inst, cfg, seeds)
    idx = sorted({0, T - 1, T // 2})
    bc, bs, se = O.run_trials_rscan(R, C, inst.torus_weights, cfg.kind, cfg.sweeps,
                                    [seeds[i] for i in idx], cfg.temp_start or 0.0, cfg.temp_end or 0.0)
    ok = all((int(b.best_cut[i]), int(b.sweeps_executed[i]), b.hex(i)) ==
             (int(bc[k]), int(se[k]), O.encode_hex(bs[k])) for k, i in enumerate(idx))
    bad += not ok
    print(f"{it:3d} {R}x{C} T={T} S={cfg.sweeps} {cfg.kind[:6]} shape={forced} limits={lim} "
          f"{'ok' if ok else 'MISMATCH'}", flush=True)
_test_rscan_shape(0, 0)
_test_rscan_limits(0, 0)
print("mismatches:", bad)
sys.exit(1 if bad else 0)
