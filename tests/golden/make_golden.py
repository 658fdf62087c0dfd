#!/usr/bin/env python3
"""Generate golden fixtures by running the UNMODIFIED Python reference.

Test infrastructure only.  This script imports ``gsetbench`` from
``/root/reference/pkg/src`` (read-only, present only in the build
container, never on the GPU box) and writes small JSON fixtures into
``tests/golden/``.  The fixtures pin:

* numpy's ``default_rng`` seeding (SeedSequence -> PCG64 state/inc) and the
  PCG64 stream consumption of ``integers``/``permutation``/``random``
  (the third-party arithmetic the reference's hot path calls,
  solvers.py:94-118, instances.py:221-222);
* ``mix_seed`` (campaign.py:39-53), ``generate_torus`` weights
  (instances.py:203-224), ``cut_value``/``ising_energy`` (evaluate.py:35-49),
  ``encode_hex`` (codec.py:64-83);
* full ``run_trial`` trajectories (solvers.py:91-140): best_cut,
  best_spins (hex), sweeps_executed for small tori, random graphs, the whole
  of BASELINE config 1 and full-length samples of configs 2-4.

Usage:
    python tests/golden/make_golden.py fast            # < 1 min
    python tests/golden/make_golden.py c1 [--procs P]  # ~80 s on 8 cores
    python tests/golden/make_golden.py c2|c3|c4 [--procs P] [--trials K]
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import numpy as np  # noqa: E402

from gsetbench.campaign import mix_seed  # noqa: E402
from gsetbench.codec import encode_hex  # noqa: E402
from gsetbench.evaluate import cut_value, ising_energy  # noqa: E402
from gsetbench.instances import ProblemInstance, TorusSpec, generate_torus  # noqa: E402
from gsetbench.solvers import ANNEALING, GREEDY, SolverConfig, default_config, run_trial  # noqa: E402

OUT = Path(__file__).resolve().parent
MASTER = 20250814


def _dump(name, obj):
    path = OUT / name
    path.write_text(json.dumps(obj, indent=1, sort_keys=True) + "\n")
    print(f"wrote {path} ({path.stat().st_size} bytes)")


def _pcg_state(seed):
    st = np.random.default_rng(seed).bit_generator.state
    return {"state": hex(st["state"]["state"]), "inc": hex(st["state"]["inc"])}


def _torus_w(rows, cols, seed):
    """int8 weights in emission order: index 2*x = right edge, 2*x+1 = down."""
    n = rows * cols
    return (np.random.default_rng(seed).integers(0, 2, size=2 * n) * 2 - 1).astype(np.int8)


def _random_graph(rng, n, edge_prob=0.5, max_weight=5):
    # same construction as the reference's tests/conftest.py:13-21
    edges = []
    for u in range(1, n + 1):
        for v in range(u + 1, n + 1):
            if rng.random() < edge_prob:
                edges.append((u, v, int(rng.integers(-max_weight, max_weight + 1))))
    if not edges:
        edges.append((1, 2, int(rng.integers(1, max_weight + 1))))
    return ProblemInstance.from_edges(n, edges)


def _result_row(res, n):
    return {
        "best_cut": res.best_cut,
        "sweeps_executed": res.sweeps_executed,
        "hex": encode_hex(res.best_spins),
    }


def gen_fast():
    rng_kat = {"numpy_version": np.__version__}  # the stream below is numpy's (third-party)
    # mix_seed known answers (campaign.py:39-53; KAT at test_campaign.py:44-50)
    rng_kat["mix_seed"] = [
        [m, i, mix_seed(m, i)]
        for m in (0, 1, 1234567, MASTER, 2**64 - 1)
        for i in (0, 1, 2, 99, 8191)
    ]
    # SeedSequence -> PCG64 (state, inc)
    seeds = [0, 1, 2, 7, 42, 123, 2**32 - 1, 2**32, 2**63, 2**64 - 1,
             12345678901234567] + [mix_seed(MASTER, i) for i in range(4)]
    rng_kat["pcg64_init"] = [[s, _pcg_state(s)] for s in seeds]
    # stream consumption
    streams = []
    for s in (1, 42, mix_seed(MASTER, 0)):
        g = np.random.default_rng(s)
        rec = {"seed": s}
        rec["next64"] = [int(x) for x in g.bit_generator.random_raw(6)]
        g = np.random.default_rng(s)
        rec["integers_0_2_13"] = [int(x) for x in g.integers(0, 2, size=13)]
        rec["perm_37"] = [int(x) for x in g.permutation(37)]
        rec["random_3"] = [float(g.random()) .hex() for _ in range(3)]
        rec["perm_5"] = [int(x) for x in g.permutation(5)]
        rec["after"] = {k: (hex(v) if isinstance(v, int) and v > 2**31 else v)
                        for k, v in g.bit_generator.state["state"].items()}
        rec["has_uint32"] = int(g.bit_generator.state["has_uint32"])
        rec["uinteger"] = int(g.bit_generator.state["uinteger"])
        streams.append(rec)
    rng_kat["streams"] = streams
    _dump("rng_kat.json", rng_kat)

    # torus weights + evaluator
    tori = []
    for rows, cols, seed in [(3, 3, 1), (4, 4, 1), (4, 4, 2), (5, 5, 7), (5, 7, 3),
                             (6, 6, 11), (6, 10, 2), (8, 8, 42), (10, 10, 5),
                             (50, 100, 1), (100, 100, 1), (100, 140, 1), (100, 200, 1)]:
        inst = generate_torus(TorusSpec(rows, cols, seed))
        w = _torus_w(rows, cols, seed)
        assert np.array_equal(w.astype(np.int64), inst._ew), (rows, cols)
        rec = {
            "rows": rows, "cols": cols, "seed": seed, "n": inst.n, "m": inst.m,
            "total_weight": inst.total_weight(),
            "w_sha256": hashlib.sha256(w.tobytes()).hexdigest(),
        }
        if inst.n <= 100:
            rec["w"] = w.tolist()
        evals = []
        g = np.random.default_rng(1000 + rows * cols)
        for _ in range(3):
            spins = tuple(int(x) for x in g.choice((-1, 1), size=inst.n))
            evals.append({"hex": encode_hex(spins), "cut": cut_value(inst, spins),
                          "energy": ising_energy(inst, spins)})
        for spins in ((1,) * inst.n, (-1,) * inst.n):
            evals.append({"hex": encode_hex(spins), "cut": cut_value(inst, spins),
                          "energy": ising_energy(inst, spins)})
        rec["evals"] = evals
        tori.append(rec)
    # config 5 is far too large for the reference's tuple representation;
    # its weights come from the same default_rng(seed).integers(0,2,2n) call
    w5 = _torus_w(2000, 2000, 1)
    tori.append({"rows": 2000, "cols": 2000, "seed": 1, "n": 4_000_000, "m": 8_000_000,
                 "total_weight": int(w5.astype(np.int64).sum()),
                 "w_sha256": hashlib.sha256(w5.tobytes()).hexdigest(),
                 "note": "weights from default_rng(1).integers(0,2,2n)*2-1 "
                         "(== generate_torus _ew, verified for the smaller tori)"})
    _dump("tori.json", {"tori": tori})

    # codec
    g = np.random.default_rng(5)
    codec = []
    for n in (1, 2, 3, 4, 5, 7, 8, 9, 31, 32, 33, 100, 1001):
        spins = tuple(int(x) for x in g.choice((-1, 1), size=n))
        codec.append({"spins": list(spins), "hex": encode_hex(spins)})
    _dump("codec.json", {"cases": codec})

    # run_trial trajectories on small tori
    trials = []
    cases = [
        ((3, 3, 1), [1, 2, 5]), ((4, 4, 1), [1, 7, 50]), ((4, 4, 2), [3, 37]),
        ((5, 5, 7), [30]), ((5, 7, 3), [1, 2, 9, 60]), ((6, 6, 11), [1, 2, 3, 4, 6, 8]),
        ((6, 10, 2), [60]), ((8, 8, 42), [200]), ((10, 10, 5), [60]),
        ((7, 9, 4), [25]),
    ]
    for (rows, cols, tseed), budgets in cases:
        inst = generate_torus(TorusSpec(rows, cols, tseed))
        for sweeps in budgets:
            for i in range(4):
                seed = mix_seed(MASTER, i)
                for cfg in (
                    default_config(GREEDY, sweeps, seed),
                    default_config(ANNEALING, sweeps, seed),
                    SolverConfig(ANNEALING, sweeps, seed, temp_start=2.0, temp_end=0.1),
                ):
                    res = run_trial(inst, cfg)
                    row = {"rows": rows, "cols": cols, "torus_seed": tseed,
                           "kind": cfg.kind, "sweeps": sweeps, "seed": seed,
                           "temp_start": cfg.temp_start, "temp_end": cfg.temp_end}
                    row.update(_result_row(res, inst.n))
                    trials.append(row)
    # small integer seeds too (0, 1, 2**64-1)
    inst = generate_torus(TorusSpec(4, 6, 9))
    for seed in (0, 1, 2**32, 2**64 - 1):
        for cfg in (default_config(GREEDY, 10, seed), default_config(ANNEALING, 10, seed)):
            res = run_trial(inst, cfg)
            row = {"rows": 4, "cols": 6, "torus_seed": 9, "kind": cfg.kind, "sweeps": 10,
                   "seed": seed, "temp_start": cfg.temp_start, "temp_end": cfg.temp_end}
            row.update(_result_row(res, inst.n))
            trials.append(row)
    _dump("trials_small.json", {"trials": trials})

    # run_trial on random (non-torus) graphs, reference conftest construction
    rng = np.random.default_rng(41)
    graphs = []
    for gi in range(6):
        n = int(rng.integers(4, 16))
        inst = _random_graph(rng, n)
        runs = []
        for kind in (GREEDY, ANNEALING):
            seed = int(rng.integers(2**32))
            res = run_trial(inst, default_config(kind, 20, seed))
            runs.append({"kind": kind, "sweeps": 20, "seed": seed, **_result_row(res, n)})
        graphs.append({"n": n, "edges": [list(e) for e in inst.edges], "runs": runs})
    _dump("graphs_small.json", {"graphs": graphs})


def _one(args):
    rows, cols, kind, sweeps, index = args
    inst = _INST_CACHE.get((rows, cols))
    if inst is None:
        inst = generate_torus(TorusSpec(rows, cols, 1))
        _INST_CACHE[(rows, cols)] = inst
    seed = mix_seed(MASTER, index)
    t0 = time.perf_counter()
    res = run_trial(inst, default_config(kind, sweeps, seed))
    dt = time.perf_counter() - t0
    return {"index": index, "seed": seed, "kind": kind, "sweeps": sweeps,
            "wall_s": round(dt, 3), **_result_row(res, inst.n)}


_INST_CACHE: dict = {}


def gen_config(name, rows, cols, sweeps, trials, procs, kinds):
    out = {"rows": rows, "cols": cols, "torus_seed": 1, "master_seed": MASTER,
           "sweeps": sweeps, "numpy": np.__version__, "runs": {}}
    for kind in kinds:
        jobs = [(rows, cols, kind, sweeps, i) for i in range(trials)]
        t0 = time.perf_counter()
        with ProcessPoolExecutor(procs) as pool:
            rows_out = list(pool.map(_one, jobs))
        wall = time.perf_counter() - t0
        n = rows * cols
        upd = sum(r["sweeps_executed"] for r in rows_out) * n
        out["runs"][kind] = {"trials": rows_out, "wall_s": round(wall, 2), "procs": procs,
                             "updates_per_s": upd / wall}
        print(f"{name} {kind}: {trials} trials in {wall:.1f}s on {procs} procs "
              f"({upd / wall:.3e} updates/s)", flush=True)
    _dump(f"{name}.json", out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["fast", "c1", "c2", "c3", "c4"])
    ap.add_argument("--procs", type=int, default=os.cpu_count())
    ap.add_argument("--trials", type=int, default=8)
    a = ap.parse_args()
    if a.what == "fast":
        gen_fast()
    elif a.what == "c1":
        gen_config("c1_full", 50, 100, 1000, 100, a.procs, (ANNEALING, GREEDY))
    elif a.what == "c2":
        gen_config("c2_sample", 100, 100, 10_000, a.trials, a.procs, (ANNEALING,))
    elif a.what == "c3":
        gen_config("c3_sample", 100, 140, 20_000, a.trials, a.procs, (ANNEALING,))
    elif a.what == "c4":
        gen_config("c4_sample", 100, 200, 50_000, a.trials, a.procs, (ANNEALING,))


if __name__ == "__main__":
    main()
