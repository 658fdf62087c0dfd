"""The drop-in API on the GPU engine, mirroring the reference's own solver,
campaign and acceptance tests (pkg/tests/test_solvers.py, test_campaign.py,
test_acceptance.py), plus campaign-level parity with the reference goldens."""

import itertools

import numpy as np
import pytest

from conftest import MASTER, golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2505_18508_b200 import ProblemInstance, TorusSpec, decode_hex, generate_torus  # noqa
from paper_2505_18508_b200.campaign import (  # noqa: E402
    CampaignConfig,
    TargetSpec,
    mix_seed,
    read_log,
    replay_record,
    run_campaign,
)
from paper_2505_18508_b200.distributed import run_sharded  # noqa: E402
from paper_2505_18508_b200.evaluate import cut_value, flip_delta_cut, ising_energy  # noqa
from paper_2505_18508_b200.solvers import (  # noqa: E402
    ANNEALING,
    ANNEALING_CHECKERBOARD,
    GREEDY,
    GREEDY_CHECKERBOARD,
    default_config,
    run_trial,
    run_trials,
)

ALL = (GREEDY, ANNEALING, GREEDY_CHECKERBOARD, ANNEALING_CHECKERBOARD)


def random_instance(rng, n, edge_prob=0.5, max_weight=5):  # reference conftest.py:13-21
    edges = []
    for u in range(1, n + 1):
        for v in range(u + 1, n + 1):
            if rng.random() < edge_prob:
                edges.append((u, v, int(rng.integers(-max_weight, max_weight + 1))))
    if not edges:
        edges.append((1, 2, int(rng.integers(1, max_weight + 1))))
    return ProblemInstance.from_edges(n, edges)


def brute_force_max_cut(inst):
    best = None
    for bits in itertools.product((-1, 1), repeat=inst.n - 1):
        s = (1,) + bits
        c = sum(w for u, v, w in inst.edges if s[u - 1] != s[v - 1])
        best = c if best is None else max(best, c)
    return best


def test_trials_are_deterministic():
    inst = generate_torus(TorusSpec(6, 6, 7))
    for kind in ALL:
        cfg = default_config(kind, 30, seed=123)
        a, b = run_trial(inst, cfg), run_trial(inst, cfg)
        assert (a.best_cut, a.best_spins, a.sweeps_executed) == (
            b.best_cut, b.best_spins, b.sweeps_executed)
        assert a.seed == 123


def test_best_cut_matches_reported_spins():
    rng = np.random.default_rng(41)
    for kind in (GREEDY, ANNEALING):
        for _ in range(5):
            inst = random_instance(rng, int(rng.integers(4, 16)))
            r = run_trial(inst, default_config(kind, 20, seed=int(rng.integers(2**32))))
            assert cut_value(inst, r.best_spins) == r.best_cut
    inst = generate_torus(TorusSpec(8, 10, 3))
    for kind in ALL:
        r = run_trial(inst, default_config(kind, 40, seed=9))
        assert cut_value(inst, r.best_spins) == r.best_cut
        assert ising_energy(inst, r.best_spins) == inst.total_weight() - 2 * r.best_cut


@pytest.mark.parametrize("kind", [GREEDY, GREEDY_CHECKERBOARD])
def test_greedy_converges_to_local_optimum(kind):
    inst = generate_torus(TorusSpec(4, 4, 2))
    r = run_trial(inst, default_config(kind, 10_000, seed=5))
    assert r.sweeps_executed < 10_000
    assert max(flip_delta_cut(inst, r.best_spins, k) for k in range(1, inst.n + 1)) <= 0


@pytest.mark.parametrize("kind", [ANNEALING, ANNEALING_CHECKERBOARD])
def test_annealing_always_consumes_budget(kind):
    inst = generate_torus(TorusSpec(4, 4, 2))
    assert run_trial(inst, default_config(kind, 37, seed=5)).sweeps_executed == 37


@pytest.mark.parametrize("kind", [GREEDY, GREEDY_CHECKERBOARD])
def test_greedy_best_cut_monotone_in_budget(kind):
    inst = generate_torus(TorusSpec(6, 6, 11))
    for seed in (1, 2, 3):
        cuts = [run_trial(inst, default_config(kind, s, seed=seed)).best_cut
                for s in (1, 2, 3, 4, 6, 8)]
        assert cuts == sorted(cuts)


def test_solvers_never_beat_the_exhaustive_optimum():
    rng = np.random.default_rng(42)
    for _ in range(5):
        inst = random_instance(rng, int(rng.integers(6, 13)))
        opt = brute_force_max_cut(inst)
        for kind in (GREEDY, ANNEALING):
            r = run_trial(inst, default_config(kind, 40, seed=int(rng.integers(2**32))))
            assert r.best_cut <= opt


def test_acceptance_criterion_6():
    """test_acceptance.py:255-278: torus 4x4 seed 1, SA 50 sweeps, 100 trials,
    master 20250814.  The reference reaches the optimum 10 in 99/100; the
    reference engine is bit-exact so must give exactly that."""
    inst = generate_torus(TorusSpec(4, 4, 1))
    for kind, expect in ((ANNEALING, 99), (ANNEALING_CHECKERBOARD, None)):
        cfg = CampaignConfig(inst.name, default_config(kind, 50, 0), 100, MASTER,
                             targets=(TargetSpec("optimum", 10),))
        s = run_campaign(inst, cfg)
        assert s.highest_cut == 10
        if expect is not None:
            assert s.targets[0].successes == expect
        else:
            assert s.targets[0].successes >= 80
        serial = run_campaign(inst, cfg, workers=4)
        assert serial.deterministic_fields() == s.deterministic_fields()


def test_campaign_config1_summary_equals_reference():
    c1 = golden("c1_full.json")
    inst = generate_torus(TorusSpec(50, 100, 1))
    for kind in (GREEDY, ANNEALING):
        ref = c1["runs"][kind]["trials"]
        cfg = CampaignConfig(inst.name, default_config(kind, 1000, 0), 100, MASTER)
        s = run_campaign(inst, cfg)
        cuts = [r["best_cut"] for r in ref]
        assert s.highest_cut == max(cuts) and s.min_cut == min(cuts)
        assert s.average_cut == sum(cuts) / 100


def test_campaign_log_resume_replay(tmp_path):
    inst = generate_torus(TorusSpec(8, 8, 42))
    cfg = CampaignConfig(inst.name, default_config(ANNEALING, 40, 0), 12, 7)
    log = tmp_path / "c.log"
    full = run_campaign(inst, cfg, log_path=log, include_spins=True)
    recs = read_log(log)
    assert [r.index for r in recs] == list(range(12))
    for r in recs:
        assert r.seed == mix_seed(7, r.index)
        assert cut_value(inst, decode_hex(r.spins_hex, inst.n)) == r.best_cut
        assert replay_record(inst, r).best_cut == r.best_cut
    # resume: drop half the lines, finish, same summary
    lines = log.read_text().splitlines()
    log.write_text("\n".join(lines[:5]) + "\n")
    resumed = run_campaign(inst, cfg, log_path=log, resume=True, include_spins=True)
    assert resumed.deterministic_fields() == full.deterministic_fields()
    assert len(read_log(log)) == 12
    # tampering is detected by replay (campaign.py:174-178)
    bad = recs[0].__class__(**{**recs[0].__dict__, "best_cut": recs[0].best_cut + 2})
    with pytest.raises(RuntimeError):
        replay_record(inst, bad)


def test_run_sharded_single_rank_equals_batch():
    inst = generate_torus(TorusSpec(50, 100, 1))
    cfg = default_config(ANNEALING_CHECKERBOARD, 30, 0)
    g, cuts, sw = run_sharded(inst, cfg, MASTER, 64)
    b = run_trials(inst, cfg, [mix_seed(MASTER, i) for i in range(64)])
    assert cuts.tolist() == b.best_cut.tolist() and sw.tolist() == b.sweeps_executed.tolist()
    i = int(np.argmax(b.best_cut))
    assert (g.best_cut, g.index) == (int(b.best_cut[i]), i)
    assert g.bits.tobytes() == b.bits[i].tobytes()


def test_engine_override_stays_inside_the_contract_family():
    """An engine override may pick another engine of the SAME trial contract
    only (solvers.run_trials_device): never checkerboard <-> random scan."""
    from paper_2505_18508_b200 import _lib
    from paper_2505_18508_b200.solvers import ANNEALING_RANDOM_SCAN

    inst = generate_torus(TorusSpec(8, 8, 1))
    seeds = [1, 2, 3]
    a = run_trials(inst, default_config(ANNEALING_CHECKERBOARD, 10, 0), seeds)
    b = run_trials(inst, default_config(ANNEALING_CHECKERBOARD, 10, 0), seeds,
                   engine=_lib.ENGINE_CHECKERBOARD_TILED)
    assert np.array_equal(a.best_cut, b.best_cut) and np.array_equal(a.bits, b.bits)
    for kind, eng in ((ANNEALING_CHECKERBOARD, _lib.ENGINE_RANDOM_SCAN),
                      (ANNEALING_RANDOM_SCAN, _lib.ENGINE_CHECKERBOARD),
                      (ANNEALING_RANDOM_SCAN, _lib.ENGINE_CHECKERBOARD_TILED),
                      (ANNEALING, _lib.ENGINE_CHECKERBOARD),
                      (ANNEALING_CHECKERBOARD, _lib.ENGINE_REFERENCE)):
        with pytest.raises(ValueError, match="engine override"):
            run_trials(inst, default_config(kind, 10, 0), seeds, engine=eng)


def test_run_trials_device_on_a_side_stream():
    """stream=: inputs made on the current stream are ordered before the launch
    and kept alive for it (record_stream); results equal the default-stream run."""
    from paper_2505_18508_b200.solvers import ANNEALING_RANDOM_SCAN, run_trials_device

    inst = generate_torus(TorusSpec(20, 30, 2))
    seeds = [int(s) for s in np.arange(1, 40)]
    for kind in (ANNEALING_RANDOM_SCAN, ANNEALING_CHECKERBOARD, ANNEALING):
        cfg = default_config(kind, 25, 0)
        ref = run_trials_device(inst, cfg, seeds)
        side = torch.cuda.Stream()
        outs = [run_trials_device(inst, cfg, seeds, stream=side, check=False) for _ in range(3)]
        side.synchronize()
        for o in outs:
            assert torch.equal(o[0], ref[0]) and torch.equal(o[2], ref[2])


def test_integration_ctypes_stub():
    """INTEGRATION.md's `gsetbench/_b200.py` stub, taken verbatim from the
    markdown and executed: the bit-exact engine through it reproduces the
    reference's own config-1 trajectories (goldens), and the random-scan engine
    through it equals the package's result."""
    import os
    import re
    import types

    from conftest import ROOT
    from paper_2505_18508_b200 import _lib
    from paper_2505_18508_b200.solvers import ANNEALING_RANDOM_SCAN

    md = (ROOT / "INTEGRATION.md").read_text()
    code = re.search(r"```python\n(# gsetbench/_b200\.py.*?)```", md, re.S).group(1)
    os.environ["GSB_LIB"] = str(_lib.LIB_PATH)
    stub = types.ModuleType("gsetbench_b200_stub")
    exec(compile(code, "INTEGRATION.md:_b200.py", "exec"), stub.__dict__)
    c1 = golden("c1_full.json")
    rows = c1["runs"]["simulated_annealing"]["trials"][:6]
    spec = TorusSpec(c1["rows"], c1["cols"], 1)
    best, done, bits = stub.run_trials_torus(spec, "simulated_annealing", c1["sweeps"],
                                             [r["seed"] for r in rows], 3.0, 0.05, engine=0)
    n = spec.rows * spec.cols
    for i, r in enumerate(rows):
        assert (int(best[i]), int(done[i]), bits[i].tobytes().hex()[:(n + 3) // 4]) == (
            r["best_cut"], r["sweeps_executed"], r["hex"])
    seeds = [r["seed"] for r in rows]
    b2, d2, bits2 = stub.run_trials_torus(spec, ANNEALING_RANDOM_SCAN, 50, seeds, 3.0, 0.05,
                                          engine=4)
    ours = run_trials(generate_torus(spec), default_config(ANNEALING_RANDOM_SCAN, 50, 0), seeds)
    assert np.array_equal(b2, ours.best_cut) and np.array_equal(bits2, ours.bits)
    with pytest.raises(ValueError):
        stub.run_trials_torus(TorusSpec(5, 5, 1), "simulated_annealing_checkerboard", 5, [1],
                              3.0, 0.05, engine=1)  # odd torus: GSB_EUNSUPPORTED -> ValueError


def test_concurrent_host_threads_get_serial_results():
    """run_campaign may call run_trial from ThreadPoolExecutor threads
    (campaign.py:418-424): the ABI is reentrant -- per-call workspaces, a
    thread-local error message, mutex-guarded property caches.  Eight threads
    running different kinds and torus sizes at once get the serial results."""
    from concurrent.futures import ThreadPoolExecutor

    from paper_2505_18508_b200.solvers import ANNEALING_RANDOM_SCAN, GREEDY_RANDOM_SCAN

    jobs = []
    for i, (R, C) in enumerate([(8, 8), (20, 30), (50, 100), (12, 64), (100, 100), (30, 34)]):
        inst = generate_torus(TorusSpec(R, C, i + 1))
        for kind in (ANNEALING, ANNEALING_CHECKERBOARD, ANNEALING_RANDOM_SCAN, GREEDY_RANDOM_SCAN):
            if kind == ANNEALING_CHECKERBOARD and (R | C) & 1:
                continue
            jobs.append((inst, default_config(kind, 15, 0), [int(s) for s in range(i + 3, i + 9)]))
    serial = [run_trials(*j) for j in jobs]

    def work(j):
        return run_trials(*j)

    with ThreadPoolExecutor(8) as pool:
        for rep in range(3):
            for s, p in zip(serial, pool.map(work, jobs)):
                assert np.array_equal(s.best_cut, p.best_cut) and np.array_equal(s.bits, p.bits)
