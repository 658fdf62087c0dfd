"""Random-scan (Philox) engine: bit-exact against the CPU oracle of its
contract, and its final-cut distribution against the reference's.

Bit-exact bar as for the other engines (all state is integer).  The
distribution test compares the engine with the bit-exact reference engine,
i.e. with gsetbench's own run_trial (solvers.py:91-140) on the same torus,
schedule and seeds -- the north star's "final-cut distributions over trials
agreeing"; the checkerboard engine's systematic order fails that test (its
cuts are higher at equal sweeps), which the last test records.
"""

import numpy as np
import pytest

from conftest import MASTER

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2505_18508_b200 import TorusSpec, generate_torus  # noqa: E402
from paper_2505_18508_b200.campaign import mix_seeds  # noqa: E402
from paper_2505_18508_b200.evaluate import cut_energy_batch  # noqa: E402
from paper_2505_18508_b200.solvers import (  # noqa: E402
    ANNEALING,
    ANNEALING_CHECKERBOARD,
    ANNEALING_RANDOM_SCAN,
    GREEDY,
    GREEDY_RANDOM_SCAN,
    SolverConfig,
    default_config,
    run_trials,
    run_trials_device,
)

RS_TORI = [(3, 3, 1), (4, 4, 1), (3, 7, 2), (5, 6, 3), (9, 11, 4), (16, 66, 2), (31, 17, 5),
           (50, 100, 1), (100, 100, 1), (7, 300, 6), (100, 200, 1)]


def _check(oracle, inst, cfg, seeds):
    R, C = inst.torus.rows, inst.torus.cols
    b = run_trials(inst, cfg, seeds)
    bc, bs, se = oracle.run_trials_rscan(R, C, inst.torus_weights, cfg.kind, cfg.sweeps, seeds,
                                         cfg.temp_start, cfg.temp_end)
    for i in range(len(seeds)):
        assert (int(b.best_cut[i]), int(b.sweeps_executed[i]), b.hex(i)) == (
            bc[i], se[i], oracle.encode_hex(bs[i])), (R, C, cfg, i)


@pytest.mark.parametrize("R,C,s", RS_TORI)
def test_random_scan_engine_matches_oracle(oracle, R, C, s):
    inst = generate_torus(TorusSpec(R, C, s))
    n = R * C
    sweeps = 30 if n <= 2000 else 6
    seeds = [int(x) for x in mix_seeds(MASTER, range(5))] + [0, 2**64 - 1]
    for cfg in (default_config(ANNEALING_RANDOM_SCAN, sweeps, 0),
                SolverConfig(ANNEALING_RANDOM_SCAN, sweeps, 0, 1.5, 0.2),
                default_config(GREEDY_RANDOM_SCAN, 100, 0)):
        _check(oracle, inst, cfg, seeds)


def test_random_scan_randomized_vs_oracle(oracle):
    rng = np.random.default_rng(99)
    for _ in range(10):
        R, C = int(rng.integers(3, 40)), int(rng.integers(3, 70))
        inst = generate_torus(TorusSpec(R, C, int(rng.integers(0, 2**63))))
        S = int(rng.integers(1, 25))
        t0 = float(rng.uniform(0.3, 5.0))
        cfg = SolverConfig(ANNEALING_RANDOM_SCAN, S, 0, t0, t0 * float(rng.uniform(0.005, 0.9)))
        _check(oracle, inst, cfg, [int(x) for x in rng.integers(0, 2**63, size=6)])


@pytest.mark.parametrize("t0,t1", [(1e12, 1e11), (1e-2, 1e-3)])
def test_random_scan_threshold_extremes(oracle, t0, t1):
    inst = generate_torus(TorusSpec(8, 13, 3))
    _check(oracle, inst, SolverConfig(ANNEALING_RANDOM_SCAN, 9, 0, t0, t1),
           [int(x) for x in mix_seeds(MASTER, range(5))])


def test_random_scan_batch_invariance_and_bits():
    inst = generate_torus(TorusSpec(50, 100, 1))
    cfg = default_config(ANNEALING_RANDOM_SCAN, 40, 0)
    seeds = mix_seeds(MASTER, range(400))
    full = run_trials(inst, cfg, seeds)
    part = run_trials(inst, cfg, seeds[211:214])
    assert np.array_equal(full.best_cut[211:214], part.best_cut)
    assert np.array_equal(full.bits[211:214], part.bits)
    cut, _ = cut_energy_batch(inst, full.bits)
    assert np.array_equal(cut.cpu().numpy(), full.best_cut)


def _final_cuts(inst, kind, sweeps, T):
    best, _, _ = run_trials_device(inst, default_config(kind, sweeps, 0),
                                   mix_seeds(MASTER, range(T)))
    return best.cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("R,C,S", [(50, 100, 1000), (100, 100, 1000)])
def test_random_scan_cut_distribution_agrees_with_reference(R, C, S):
    """1024 trials each: the reference kind (bit-exact run_trial) vs the
    random-scan kind, same seeds.  Tolerance: two-sample KS p > 1e-3 and mean
    difference within 4 standard errors."""
    stats = pytest.importorskip("scipy.stats")
    inst = generate_torus(TorusSpec(R, C, 1))
    a = _final_cuts(inst, ANNEALING, S, 1024)
    b = _final_cuts(inst, ANNEALING_RANDOM_SCAN, S, 1024)
    se = np.sqrt(a.var(ddof=1) / len(a) + b.var(ddof=1) / len(b))
    assert abs(a.mean() - b.mean()) < 4 * se, (a.mean(), b.mean(), se)
    assert stats.ks_2samp(a, b).pvalue > 1e-3
    g1 = _final_cuts(inst, GREEDY, 100, 1024)
    g2 = _final_cuts(inst, GREEDY_RANDOM_SCAN, 100, 1024)
    assert stats.ks_2samp(g1, g2).pvalue > 1e-3


def test_checkerboard_order_shifts_the_distribution():
    """Recorded property of the throughput kind: the systematic colour order
    reaches higher cuts than the reference's random order at equal sweeps."""
    inst = generate_torus(TorusSpec(50, 100, 1))
    a = _final_cuts(inst, ANNEALING, 1000, 1024)
    c = _final_cuts(inst, ANNEALING_CHECKERBOARD, 1000, 1024)
    se = np.sqrt(a.var(ddof=1) / len(a) + c.var(ddof=1) / len(c))
    assert c.mean() - a.mean() > 4 * se


@pytest.mark.parametrize("R,C", [(3, 5), (10, 33), (50, 100), (100, 100), (64, 200)])
def test_random_scan_kernels_agree(R, C, monkeypatch):
    """The bit-sliced kernel (default) and the per-site kernel (fallback,
    GSB_RSCAN_SCALAR=1) run the same contract: identical results."""
    inst = generate_torus(TorusSpec(R, C, 4))
    seeds = mix_seeds(MASTER, range(40))
    for cfg in (default_config(ANNEALING_RANDOM_SCAN, 25, 0), default_config(GREEDY_RANDOM_SCAN, 50, 0)):
        a = run_trials(inst, cfg, seeds)
        monkeypatch.setenv("GSB_RSCAN_SCALAR", "1")
        b = run_trials(inst, cfg, seeds)
        monkeypatch.delenv("GSB_RSCAN_SCALAR")
        assert np.array_equal(a.best_cut, b.best_cut) and np.array_equal(a.bits, b.bits)
        assert np.array_equal(a.sweeps_executed, b.sweeps_executed)
