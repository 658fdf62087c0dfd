"""Final best-cut distributions over trials: the Philox engines (random-scan,
checkerboard) vs the bit-exact reference engine (= the reference's own
run_trial distribution), same torus, seeds and schedule.  One JSON line per
config and kind.
usage: python tools/cut_distribution.py [R C T S] ..."""
import json, sys
sys.path.insert(0, '.')
import numpy as np
from scipy import stats
from paper_2505_18508_b200 import TorusSpec, generate_torus
from paper_2505_18508_b200.campaign import mix_seeds
from paper_2505_18508_b200.solvers import (ANNEALING, ANNEALING_CHECKERBOARD,
                                           ANNEALING_RANDOM_SCAN, GREEDY, GREEDY_CHECKERBOARD,
                                           GREEDY_RANDOM_SCAN, default_config, run_trials_device)

args = [int(x) for x in sys.argv[1:]] or [50, 100, 1024, 1000, 100, 100, 1024, 1000, 100, 100, 1024, 10000]
def summary(x):
    return {"mean": float(x.mean()), "std": float(x.std(ddof=1)), "min": int(x.min()),
            "max": int(x.max()), "q10_50_90": np.percentile(x, [10, 50, 90]).tolist()}


for i in range(0, len(args), 4):
    R, C, T, S = args[i:i + 4]
    inst = generate_torus(TorusSpec(R, C, 1))
    seeds = mix_seeds(20250814, range(T))
    for ref, others, sw in ((ANNEALING, (ANNEALING_RANDOM_SCAN, ANNEALING_CHECKERBOARD), S),
                            (GREEDY, (GREEDY_RANDOM_SCAN, GREEDY_CHECKERBOARD), 100)):
        cuts = {}
        for kind in (ref,) + others:
            best, _, _ = run_trials_device(inst, default_config(kind, sw, 0), seeds)
            cuts[kind] = best.cpu().numpy().astype(np.int64)
        a = cuts[ref]
        for kind in others:
            b = cuts[kind]
            se = np.sqrt(a.var(ddof=1) / T + b.var(ddof=1) / T)
            print(json.dumps({
                "torus": f"{R}x{C}", "trials": T, "sweeps": sw, "reference_kind": ref, "kind": kind,
                "reference": summary(a), "engine": summary(b),
                "mean_diff_in_se": float((b.mean() - a.mean()) / se),
                "ks_p": float(stats.ks_2samp(a, b).pvalue),
                "mannwhitney_p": float(stats.mannwhitneyu(a, b).pvalue)}), flush=True)
