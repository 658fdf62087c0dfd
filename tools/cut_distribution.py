"""Final best-cut distributions over trials: checkerboard Philox engine vs the
bit-exact reference engine (= the reference's own run_trial distribution),
same torus, same seeds, same schedule.  Prints one JSON line per config.
usage: python tools/cut_distribution.py [R C T S] ..."""
import json, sys
sys.path.insert(0, '.')
import numpy as np
from scipy import stats
from paper_2505_18508_b200 import TorusSpec, generate_torus
from paper_2505_18508_b200.campaign import mix_seeds
from paper_2505_18508_b200.solvers import (ANNEALING, ANNEALING_CHECKERBOARD, default_config,
                                           run_trials_device)

args = [int(x) for x in sys.argv[1:]] or [50, 100, 1024, 1000, 100, 100, 1024, 1000, 100, 100, 1024, 10000]
for i in range(0, len(args), 4):
    R, C, T, S = args[i:i + 4]
    inst = generate_torus(TorusSpec(R, C, 1))
    seeds = mix_seeds(20250814, range(T))
    out = {}
    for kind in (ANNEALING, ANNEALING_CHECKERBOARD):
        best, _, _ = run_trials_device(inst, default_config(kind, S, 0), seeds)
        out[kind] = best.cpu().numpy().astype(np.int64)
    a, b = out[ANNEALING], out[ANNEALING_CHECKERBOARD]
    ks = stats.ks_2samp(a, b)
    mw = stats.mannwhitneyu(a, b)
    print(json.dumps({
        "torus": f"{R}x{C}", "trials": T, "sweeps": S,
        "reference": {"mean": a.mean(), "std": a.std(ddof=1), "min": int(a.min()), "max": int(a.max()),
                      "q": np.percentile(a, [10, 50, 90]).tolist()},
        "checkerboard": {"mean": b.mean(), "std": b.std(ddof=1), "min": int(b.min()), "max": int(b.max()),
                         "q": np.percentile(b, [10, 50, 90]).tolist()},
        "mean_diff_in_se": (b.mean() - a.mean()) / np.sqrt(a.var(ddof=1) / T + b.var(ddof=1) / T),
        "ks_stat": ks.statistic, "ks_p": ks.pvalue, "mannwhitney_p": mw.pvalue}), flush=True)
