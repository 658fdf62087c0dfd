"""GPU parity of the cluster checkerboard engine (checker_cluster.cu): one trial
spread over the shared memory of a CTA cluster, halo rows over DSMEM.

Bar: bit-exact against the C oracle's restatement of the checkerboard contract
(oracle/gsb_oracle.c:trial_checker) -- best_cut, best bitstring and
sweeps_executed; all state is integer.  Calls go through the C ABI.
"""

import numpy as np
import pytest

from conftest import MASTER

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2505_18508_b200 import TorusSpec, _lib, generate_torus  # noqa: E402
from paper_2505_18508_b200.campaign import mix_seeds  # noqa: E402
from paper_2505_18508_b200.evaluate import cut_energy_batch  # noqa: E402
from paper_2505_18508_b200.solvers import (  # noqa: E402
    ANNEALING_CHECKERBOARD,
    GREEDY_CHECKERBOARD,
    SolverConfig,
    _test_cluster_size,
    default_config,
    run_trials,
)

CLUSTER = _lib.ENGINE_CHECKERBOARD_CLUSTER


def _check(oracle, inst, cfg, seeds, engine=CLUSTER):
    R, C = inst.torus.rows, inst.torus.cols
    b = run_trials(inst, cfg, seeds, engine=engine)
    bc, bs, se = oracle.run_trials_checker(R, C, inst.torus_weights, cfg.kind, cfg.sweeps, seeds,
                                           cfg.temp_start, cfg.temp_end)
    for i in range(len(seeds)):
        assert (int(b.best_cut[i]), int(b.sweeps_executed[i]), b.hex(i)) == (
            bc[i], se[i], oracle.encode_hex(bs[i])), (R, C, cfg.kind, i)


@pytest.fixture(autouse=True)
def _automatic_cluster_size_afterwards():
    yield
    _test_cluster_size(0)


# (rows, cols, seed, cluster sizes): words per row WPR = ceil(cols/64) must be a
# power of two; bands of one row (rows == cluster size), partial last words
# (cols 66, 100, 200, 250), a cluster of one CTA (its own neighbour) and of two
# (the same CTA above and below)
SHAPES = [
    (8, 8, 1, (1, 2, 4, 8)),
    (16, 64, 3, (1, 2, 16)),
    (6, 66, 2, (1, 2, 4)),
    (34, 64, 5, (4, 8, 16)),
    (50, 100, 1, (2, 8, 16)),
    (20, 200, 9, (1, 4, 16)),
    (12, 250, 4, (2, 8)),
]


@pytest.mark.parametrize("R,C,s,sizes", SHAPES)
def test_cluster_engine_matches_oracle(oracle, R, C, s, sizes):
    inst = generate_torus(TorusSpec(R, C, s))
    seeds = [int(x) for x in mix_seeds(MASTER, range(9))] + [0, 2**64 - 1]
    for cs in sizes:
        _test_cluster_size(cs)
        for cfg in (default_config(ANNEALING_CHECKERBOARD, 25, 0),
                    default_config(GREEDY_CHECKERBOARD, 200, 0),
                    SolverConfig(ANNEALING_CHECKERBOARD, 7, 0, 1e12, 1e11),  # always accept
                    SolverConfig(ANNEALING_CHECKERBOARD, 7, 0, 1e-2, 1e-3)):  # never accept
            _check(oracle, inst, cfg, seeds)


def test_cluster_engine_randomized(oracle):
    rng = np.random.default_rng(99)
    for _ in range(10):
        wpr = int(rng.choice([1, 2, 4, 8]))
        C = int(rng.integers(max(4, 32 * (wpr - 1) + 1), 32 * wpr + 1)) * 2
        R = int(rng.integers(2, 40)) * 2
        cs = int(rng.choice([c for c in (1, 2, 4, 8, 16) if c <= R]))
        _test_cluster_size(cs)
        t0 = float(rng.uniform(0.5, 5.0))
        cfg = SolverConfig(ANNEALING_CHECKERBOARD, int(rng.integers(1, 30)), 0, t0,
                           t0 * float(rng.uniform(0.005, 0.9)))
        inst = generate_torus(TorusSpec(R, C, int(rng.integers(0, 2**63))))
        _check(oracle, inst, cfg, [int(x) for x in rng.integers(0, 2**63, size=6)])


def test_config5_cluster_engine_matches_oracle(oracle):
    """BASELINE config 5 (2000x2000, 4M spins) at full size: the default engine
    (a 16-CTA cluster per trial) against the oracle, 12 trials x 8 sweeps."""
    inst = generate_torus(TorusSpec(2000, 2000, 1))
    seeds = [int(x) for x in mix_seeds(MASTER, range(12))]
    _check(oracle, inst, default_config(ANNEALING_CHECKERBOARD, 8, 0), seeds, engine=None)
    _check(oracle, inst, default_config(GREEDY_CHECKERBOARD, 3, 0), seeds[:4], engine=None)


def test_config5_engines_agree():
    """Cluster and HBM-tiled engines give identical trials on config 5, and the
    bitstrings evaluate to the reported cuts."""
    inst = generate_torus(TorusSpec(2000, 2000, 1))
    cfg = default_config(ANNEALING_CHECKERBOARD, 20, 0)
    seeds = [int(x) for x in mix_seeds(MASTER, range(9))]
    a = run_trials(inst, cfg, seeds, engine=CLUSTER)
    b = run_trials(inst, cfg, seeds, engine=_lib.ENGINE_CHECKERBOARD_TILED)
    assert np.array_equal(a.best_cut, b.best_cut)
    assert np.array_equal(a.bits, b.bits)
    cut, _ = cut_energy_batch(inst, a.bits)
    assert np.array_equal(cut.cpu().numpy(), a.best_cut)
