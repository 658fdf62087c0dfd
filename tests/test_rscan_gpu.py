"""Random-scan (Philox) engine: bit-exact against the CPU oracle of its
contract, and its final-cut distribution against the reference's.

Bit-exact bar as for the other engines (all state is integer): best cut,
best bitstring (hex) and sweeps executed equal the oracle's
(oracle/gsb_oracle.c:trial_rscan, itself equal to a pure-Python restatement
in tests/test_oracle_cpu.py).  Every team shape the engine can launch
(warps per trial x rows per lane) is covered, and the benchmark shapes are
run at their benchmark trial counts with a sampled subset compared.  The
distribution tests compare the engine with the bit-exact reference engine,
i.e. with gsetbench's own run_trial (solvers.py:91-140) on the same torus,
schedule and seeds -- the north star's "final-cut distributions over trials
agreeing" -- tolerance: means within 4 standard errors and two-sample KS
p > 1e-3.  The checkerboard engine's systematic order fails that test (its
cuts are higher at equal sweeps), which the last test records.

The acceptance uniform is 32-bit here (the reference draws 53 bits): an
acceptance probability is resolved to 2^-32 instead of 2^-53.
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
    _test_rscan_limits,
    _test_rscan_shape,
    _test_rscan_slices,
    rscan_shape,
    run_trials,
    run_trials_device,
)

RS_TORI = [(3, 3, 1), (4, 4, 1), (3, 7, 2), (5, 6, 3), (9, 11, 4), (16, 66, 2), (31, 17, 5),
           (50, 100, 1), (100, 100, 1), (7, 300, 6), (100, 140, 1), (100, 200, 1), (40, 33, 7),
           (13, 64, 8), (61, 96, 9)]


def _check(oracle, inst, cfg, seeds, idx=None):
    R, C = inst.torus.rows, inst.torus.cols
    b = run_trials(inst, cfg, seeds)
    idx = range(len(seeds)) if idx is None else idx
    sub = [int(seeds[i]) for i in idx]
    bc, bs, se = oracle.run_trials_rscan(R, C, inst.torus_weights, cfg.kind, cfg.sweeps, sub,
                                         cfg.temp_start, cfg.temp_end)
    for k, i in enumerate(idx):
        assert (int(b.best_cut[i]), int(b.sweeps_executed[i]), b.hex(i)) == (
            bc[k], se[k], oracle.encode_hex(bs[k])), (R, C, cfg, i)
    return b


@pytest.mark.parametrize("R,C,s", RS_TORI)
def test_random_scan_engine_matches_oracle(oracle, R, C, s):
    inst = generate_torus(TorusSpec(R, C, s))
    n = R * C
    sweeps = 30 if n <= 2000 else 8
    seeds = [int(x) for x in mix_seeds(MASTER, range(5))] + [0, 2**64 - 1]
    for cfg in (default_config(ANNEALING_RANDOM_SCAN, sweeps, 0),
                SolverConfig(ANNEALING_RANDOM_SCAN, sweeps, 0, 1.5, 0.2),
                default_config(GREEDY_RANDOM_SCAN, 100, 0)):
        _check(oracle, inst, cfg, seeds)


def test_random_scan_every_team_shape(oracle):
    """Every (warps, rows per lane) instantiation, forced through the
    test-only shape override on tori that fill it, against the oracle."""
    try:
        for nw in (1, 2, 4, 7, 8, 9, 13):
            for rb in (1, 2, 3, 4, 5, 7) if nw <= 8 else (2,):  # wide teams: 2 rows per lane
                for C in (200, 140, 100, 33):  # 7 / 5 / 4 / 2 words per row (8, 12, 4 and 1 valid bits in the last)
                    bpw = 32 // ((C + 31) // 32)
                    R = nw * bpw * rb - (1 if rb > 1 else 0)
                    if R * C > 30000:
                        continue
                    _test_rscan_shape(nw, rb)
                    inst = generate_torus(TorusSpec(R, C, R + C))
                    seeds = mix_seeds(MASTER, range(3))
                    _check(oracle, inst, default_config(ANNEALING_RANDOM_SCAN, 5, 0), seeds)
                    _check(oracle, inst, default_config(GREEDY_RANDOM_SCAN, 40, 0), seeds)
        # a shape that cannot hold the torus is refused, not silently replaced
        _test_rscan_shape(1, 1)
        with pytest.raises(ValueError):
            run_trials(generate_torus(TorusSpec(100, 100, 1)),
                       default_config(ANNEALING_RANDOM_SCAN, 2, 0), [1, 2])
    finally:
        _test_rscan_shape(0, 0)


@pytest.mark.parametrize("tq,lc", [(3, 0), (0, 6), (2, 1), (1000000, 40)])
def test_random_scan_overflow_paths(oracle, tq, lc):
    """Tiny tie queue / event list: ties decided by the owning lane, candidate
    buckets split over several passes, buckets beyond the list visited by
    ordered extraction -- same results as the oracle."""
    try:
        _test_rscan_limits(tq, lc)
        for (R, C, s) in [(9, 11, 4), (40, 33, 7), (50, 100, 1), (100, 200, 1)]:
            inst = generate_torus(TorusSpec(R, C, s))
            seeds = mix_seeds(MASTER, range(4))
            _check(oracle, inst, default_config(ANNEALING_RANDOM_SCAN, 12, 0), seeds)
            _check(oracle, inst, SolverConfig(ANNEALING_RANDOM_SCAN, 6, 0, 0.9, 0.3), seeds)
    finally:
        _test_rscan_limits(0, 0)


@pytest.mark.parametrize("slices", [2, 3, 7, 40])
def test_random_scan_sweep_slices(oracle, slices):
    """Sweep slices (teams draw (slice, trial) items; a trial's state waits in
    the workspace between its slices): the oracle's results at any slice
    count, with fewer trials than teams, more, and team shapes with dummy rows."""
    try:
        _test_rscan_slices(slices)
        for (R, C, s, T) in [(9, 11, 4, 5), (40, 33, 7, 700), (50, 100, 1, 1000),
                             (100, 100, 1, 1500)]:
            inst = generate_torus(TorusSpec(R, C, s))
            seeds = mix_seeds(MASTER, range(T))
            idx = sorted(set(np.linspace(0, T - 1, 12).astype(int).tolist()))
            _check(oracle, inst, default_config(ANNEALING_RANDOM_SCAN, 40, 0), seeds, idx)
            _check(oracle, inst, SolverConfig(ANNEALING_RANDOM_SCAN, 7, 0, 0.9, 0.3), seeds, idx)
        for shape in [(4, 4), (8, 2), (2, 7)]:
            try:
                _test_rscan_shape(*shape)
                inst = generate_torus(TorusSpec(50, 100, 1))
                seeds = mix_seeds(MASTER, range(600))
                _check(oracle, inst, default_config(ANNEALING_RANDOM_SCAN, 30, 0), seeds,
                       [0, 1, 299, 598, 599])
            finally:
                _test_rscan_shape(0, 0)
    finally:
        _test_rscan_slices(0)


def test_random_scan_sweep_slices_concurrent_streams():
    """Sliced launches from three host threads on their own streams at once:
    teams of different launches share the SMs while they poll each other's
    launch-private flags; every launch returns what it returns alone."""
    import threading

    import torch

    jobs = [((100, 100), 700, 40), ((50, 100), 900, 50), ((40, 33), 1500, 60)]
    ref, bad = [], []
    try:
        _test_rscan_slices(5)
        for (R, C), T, S in jobs:
            inst = generate_torus(TorusSpec(R, C, 1))
            cfg = default_config(ANNEALING_RANDOM_SCAN, S, 0)
            b = run_trials_device(inst, cfg, mix_seeds(7, range(T)))
            ref.append((inst, cfg, T, b[0].cpu().numpy().copy(), b[2].cpu().numpy().copy()))
        torch.cuda.synchronize()

        def work(k):
            st = torch.cuda.Stream()
            for r in range(3):
                inst, cfg, T, cuts, bits = ref[(k + r) % len(ref)]
                b = run_trials_device(inst, cfg, mix_seeds(7, range(T)), stream=st)
                st.synchronize()
                if not (np.array_equal(b[0].cpu().numpy(), cuts)
                        and np.array_equal(b[2].cpu().numpy(), bits)):
                    bad.append((k, r))

        ths = [threading.Thread(target=work, args=(k,)) for k in range(3)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
    finally:
        _test_rscan_slices(0)
    assert not bad


def test_random_scan_sweep_slices_automatic():
    """The launcher slices config 2's own launch (1024 trials on 444 resident
    teams, 10 000 sweeps): identical results to the unsliced launch."""
    inst = generate_torus(TorusSpec(100, 100, 1))
    seeds = mix_seeds(20250814, range(1024))
    cfg = default_config(ANNEALING_RANDOM_SCAN, 1200, 0)
    auto = run_trials(inst, cfg, seeds)
    try:
        _test_rscan_slices(1)
        one = run_trials(inst, cfg, seeds)
    finally:
        _test_rscan_slices(0)
    assert np.array_equal(np.asarray(auto.best_cut), np.asarray(one.best_cut))
    assert [auto.hex(i) for i in (0, 500, 1023)] == [one.hex(i) for i in (0, 500, 1023)]


@pytest.mark.parametrize("R,C,T,S", [(50, 100, 100, 200), (100, 100, 1024, 60),
                                     (100, 140, 4096, 20), (100, 200, 8192, 12)])
def test_random_scan_benchmark_shapes(oracle, R, C, T, S):
    """BASELINE configs 1-4 at their trial counts (the launch the bench runs),
    a sample of 16 trials against the oracle, SA and greedy."""
    inst = generate_torus(TorusSpec(R, C, 1))
    seeds = mix_seeds(20250814, range(T))
    idx = sorted(set(np.linspace(0, T - 1, 16).astype(int).tolist()))
    assert rscan_shape(R, C, T)[0] in (1, 2, 4, 7, 8, 9, 13)
    _check(oracle, inst, default_config(ANNEALING_RANDOM_SCAN, S, 0), seeds, idx)
    _check(oracle, inst, default_config(GREEDY_RANDOM_SCAN, 200, 0), seeds, idx)


def test_random_scan_randomized_vs_oracle(oracle):
    rng = np.random.default_rng(99)
    for _ in range(12):
        R, C = int(rng.integers(3, 60)), int(rng.integers(3, 110))
        inst = generate_torus(TorusSpec(R, C, int(rng.integers(0, 2**63))))
        S = int(rng.integers(1, 25))
        t0 = float(rng.uniform(0.3, 5.0))
        cfg = SolverConfig(ANNEALING_RANDOM_SCAN, S, 0, t0, t0 * float(rng.uniform(0.005, 0.9)))
        T = int(rng.choice([3, 40, 700]))
        seeds = [int(x) for x in rng.integers(0, 2**63, size=T)]
        _check(oracle, inst, cfg, seeds, sorted({0, T - 1, T // 2}))


@pytest.mark.parametrize("t0,t1", [(1e12, 1e11), (1e-2, 1e-3)])
def test_random_scan_threshold_extremes(oracle, t0, t1):
    inst = generate_torus(TorusSpec(8, 13, 3))
    _check(oracle, inst, SolverConfig(ANNEALING_RANDOM_SCAN, 9, 0, t0, t1),
           [int(x) for x in mix_seeds(MASTER, range(5))])


def test_random_scan_full_length_c2_sample(oracle):
    """Config 2 at its full schedule (10 000 sweeps) for 4 trials of the
    1024-trial launch: the best-so-far tracking over a whole anneal."""
    inst = generate_torus(TorusSpec(100, 100, 1))
    seeds = mix_seeds(20250814, range(1024))
    _check(oracle, inst, default_config(ANNEALING_RANDOM_SCAN, 10_000, 0), seeds, [0, 1, 517, 1023])


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


def _agree(a, b):
    stats = pytest.importorskip("scipy.stats")
    se = np.sqrt(a.var(ddof=1) / len(a) + b.var(ddof=1) / len(b))
    assert abs(a.mean() - b.mean()) < 4 * se, (a.mean(), b.mean(), se)
    assert stats.ks_2samp(a, b).pvalue > 1e-3


@pytest.mark.parametrize("R,C,S", [(50, 100, 1000), (100, 100, 1000)])
def test_random_scan_cut_distribution_agrees_with_reference(R, C, S):
    """1024 trials each: the reference kind (bit-exact run_trial) vs the
    random-scan kind, same seeds; greedy too."""
    inst = generate_torus(TorusSpec(R, C, 1))
    _agree(_final_cuts(inst, ANNEALING, S, 1024), _final_cuts(inst, ANNEALING_RANDOM_SCAN, S, 1024))
    _agree(_final_cuts(inst, GREEDY, 100, 1024), _final_cuts(inst, GREEDY_RANDOM_SCAN, 100, 1024))


def test_random_scan_cut_distribution_c2_full_schedule():
    """The benchmark workload's law: config 2 (100x100, 10 000 sweeps, default
    schedule), 4096 trials of the reference kind vs 4096 of the random-scan
    kind -- the best-so-far of the random-scan kind is the sequential scan's."""
    inst = generate_torus(TorusSpec(100, 100, 1))
    _agree(_final_cuts(inst, ANNEALING, 10_000, 4096),
           _final_cuts(inst, ANNEALING_RANDOM_SCAN, 10_000, 4096))


def test_checkerboard_order_shifts_the_distribution():
    """Recorded property of the throughput kind: the systematic colour order
    reaches higher cuts than the reference's random order at equal sweeps."""
    inst = generate_torus(TorusSpec(50, 100, 1))
    a = _final_cuts(inst, ANNEALING, 1000, 1024)
    c = _final_cuts(inst, ANNEALING_CHECKERBOARD, 1000, 1024)
    se = np.sqrt(a.var(ddof=1) / len(a) + c.var(ddof=1) / len(c))
    assert c.mean() - a.mean() > 4 * se


def test_random_scan_sizes_interleaved_in_one_process(oracle):
    """The same kernel instantiation launched with different shared-memory
    sizes in one process (large torus, small torus, large again): regression
    for a cached occupancy whose MaxDynamicSharedMemorySize had been lowered."""
    try:
        _test_rscan_shape(8, 7)
        big = generate_torus(TorusSpec(56, 1000, 1))
        small = generate_torus(TorusSpec(50, 64, 2))
        seeds = mix_seeds(MASTER, range(2))
        cfg = default_config(ANNEALING_RANDOM_SCAN, 2, 0)
        for inst in (big, small, big, small):
            _check(oracle, inst, cfg, seeds)
    finally:
        _test_rscan_shape(0, 0)


# ---- the large-torus engine (rscan_big.cu): same contract, planes in global memory
BIG_TORI = [(3, 3, 1), (4, 5, 2), (9, 11, 4), (16, 66, 2), (31, 17, 5), (50, 100, 1), (7, 300, 6),
            (100, 140, 1), (40, 33, 7), (13, 64, 8), (3, 1100, 9), (70, 1100, 3)]


def _check_big(oracle, inst, cfg, seeds, idx=None, engine="large"):
    from paper_2505_18508_b200 import _lib

    R, C = inst.torus.rows, inst.torus.cols
    eng = _lib.ENGINE_RANDOM_SCAN_LARGE if engine == "large" else None
    b = run_trials(inst, cfg, seeds, engine=eng)
    idx = range(len(seeds)) if idx is None else idx
    sub = [int(seeds[i]) for i in idx]
    bc, bs, se = oracle.run_trials_rscan(R, C, inst.torus_weights, cfg.kind, cfg.sweeps, sub,
                                         cfg.temp_start, cfg.temp_end)
    for k, i in enumerate(idx):
        assert (int(b.best_cut[i]), int(b.sweeps_executed[i]), b.hex(i)) == (
            bc[k], se[k], oracle.encode_hex(bs[k])), (R, C, cfg, i)
    return b


@pytest.mark.parametrize("R,C,s", BIG_TORI)
def test_large_torus_engine_matches_oracle(oracle, R, C, s):
    """The large-torus random-scan engine forced on tori of every layout (also
    beyond 1024 columns, which only it can run), SA and greedy, batches above
    and below its 8 trials per launch."""
    inst = generate_torus(TorusSpec(R, C, s))
    sweeps = 25 if R * C <= 2000 else 6
    seeds = [int(x) for x in mix_seeds(MASTER, range(9))] + [0, 2**64 - 1]
    for cfg in (default_config(ANNEALING_RANDOM_SCAN, sweeps, 0),
                SolverConfig(ANNEALING_RANDOM_SCAN, sweeps, 0, 1.5, 0.2),
                default_config(GREEDY_RANDOM_SCAN, 100, 0)):
        _check_big(oracle, inst, cfg, seeds)


def test_large_torus_engine_equals_team_engine():
    """Same contract: the two random-scan engines give identical results."""
    from paper_2505_18508_b200 import _lib

    inst = generate_torus(TorusSpec(100, 100, 1))
    seeds = mix_seeds(MASTER, range(20))
    cfg = default_config(ANNEALING_RANDOM_SCAN, 300, 0)
    a = run_trials(inst, cfg, seeds)
    b = run_trials(inst, cfg, seeds, engine=_lib.ENGINE_RANDOM_SCAN_LARGE)
    assert np.array_equal(a.best_cut, b.best_cut) and np.array_equal(a.bits, b.bits)
    assert np.array_equal(a.sweeps_executed, b.sweeps_executed)


def test_large_torus_engine_threshold_extremes(oracle):
    inst = generate_torus(TorusSpec(8, 13, 3))
    seeds = [int(x) for x in mix_seeds(MASTER, range(5))]
    for t0, t1 in [(1e12, 1e11), (1e-2, 1e-3)]:
        _check_big(oracle, inst, SolverConfig(ANNEALING_RANDOM_SCAN, 9, 0, t0, t1), seeds)


def test_config5_random_scan_matches_oracle(oracle):
    """BASELINE config 5 (2000x2000, 4M spins) with the reference-law kind:
    the default engine for this size against the oracle, 3 trials x 3 sweeps
    SA (every sweep improves the best at this temperature) and greedy."""
    inst = generate_torus(TorusSpec(2000, 2000, 1))
    seeds = [int(x) for x in mix_seeds(MASTER, range(3))]
    _check_big(oracle, inst, default_config(ANNEALING_RANDOM_SCAN, 3, 0), seeds, engine=None)
    _check_big(oracle, inst, default_config(GREEDY_RANDOM_SCAN, 2, 0), seeds[:2], engine=None)
