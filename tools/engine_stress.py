"""Randomized stress of the checkerboard and reference engines against the CPU
oracle, sizes interleaved in one process (development tool).
usage: python tools/engine_stress.py [cases] [seed]"""
import sys
import numpy as np
sys.path.insert(0, '.')
from oracle import oracle as O
from paper_2505_18508_b200 import TorusSpec, _lib, generate_torus
from paper_2505_18508_b200.solvers import (SolverConfig, _test_checker_shape, _test_cluster_size,
                                           run_trials)

O.build()
cases = int(sys.argv[1]) if len(sys.argv) > 1 else 100
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
bad = 0
for it in range(cases):
    fam = rng.choice(["checker", "checker", "ref"])
    if fam == "checker":
        R = 2 * int(rng.integers(2, 120))
        C = 2 * int(rng.integers(2, min(400, max(3, 40000 // R))))
        kind = rng.choice(["simulated_annealing_checkerboard", "greedy_checkerboard"])
    else:
        R, C = int(rng.integers(3, 80)), int(rng.integers(3, 200))
        kind = rng.choice(["simulated_annealing", "greedy_local_search"])
    inst = generate_torus(TorusSpec(R, C, int(rng.integers(0, 2**31))))
    sa = kind.startswith("sim")
    S = int(rng.integers(1, 10 if R * C > 8000 else 30)) if sa else 60
    t0 = float(rng.uniform(0.2, 6.0))
    cfg = SolverConfig(kind, S, 0, t0, t0 * float(rng.uniform(0.01, 0.9))) if sa else SolverConfig(kind, S, 0)
    T = int(rng.choice([1, 4, 40, 500]))
    seeds = [int(x) for x in rng.integers(0, 2**63, size=T)]
    eng, note = None, ""
    _test_checker_shape(0, 0)
    _test_cluster_size(0)
    if fam == "checker":
        r = rng.random()
        if r < 0.25:
            eng, note = _lib.ENGINE_CHECKERBOARD_TILED, "tiled"
        elif r < 0.5:
            eng, note = _lib.ENGINE_CHECKERBOARD_CLUSTER, "cluster"
            _test_cluster_size(int(rng.choice([0, 1, 2, 4, 8, 16])))
        elif r < 0.75:
            _test_checker_shape(int(rng.choice([1, 2, 4, 8, 16])), int(rng.choice([0, 1, 2])))
            note = "forced shape"
    try:
        b = run_trials(inst, cfg, seeds, engine=eng)
    except ValueError as e:
        _test_checker_shape(0, 0)
        _test_cluster_size(0)
        note += " (unsupported -> default)"
        b = run_trials(inst, cfg, seeds)
    idx = sorted({0, T - 1, T // 2})
    sub = [seeds[i] for i in idx]
    if fam == "checker":
        bc, bs, se = O.run_trials_checker(R, C, inst.torus_weights, kind, S, sub, cfg.temp_start or 0.0,
                                          cfg.temp_end or 0.0)
    else:
        eu, ev, ew = O.torus_edges(R, C, inst.torus_weights)
        bc, bs, se = O.run_trials_ref(R * C, eu, ev, ew, kind, S, sub, cfg.temp_start or 0.0,
                                      cfg.temp_end or 0.0)
    ok = all((int(b.best_cut[i]), int(b.sweeps_executed[i]), b.hex(i)) ==
             (int(bc[k]), int(se[k]), O.encode_hex(bs[k])) for k, i in enumerate(idx))
    bad += not ok
    print(f"{it:3d} {fam} {R}x{C} T={T} S={S} {kind[:8]} {note} {'ok' if ok else 'MISMATCH'}", flush=True)
_test_checker_shape(0, 0)
_test_cluster_size(0)
print("mismatches:", bad)
sys.exit(1 if bad else 0)
