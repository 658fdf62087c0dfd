"""Host-side mirror of the reference API (no GPU): config validation, schedule,
seeds, codec, instances, campaign records/summaries, shard arithmetic.
Modelled on the reference's own tests (pkg/tests/test_solvers.py,
test_campaign.py, test_codec.py, test_instances.py)."""

import hashlib
import io

import numpy as np
import pytest

from conftest import golden
from paper_2505_18508_b200 import (
    GsetFormatError,
    ProblemInstance,
    TorusSpec,
    decode_hex,
    encode_hex,
    generate_torus,
    parse_gset,
    parse_torus_name,
)
from paper_2505_18508_b200.campaign import (
    CampaignConfig,
    TargetSpec,
    TrialRecord,
    format_record,
    mix_seed,
    mix_seeds,
    parse_record,
    repetitions_to_target,
    summarize,
)
from paper_2505_18508_b200.codec import HexDecodeError, pack_spins, unpack_spins
from paper_2505_18508_b200.distributed import best_key, decode_key, owner_of, shard
from paper_2505_18508_b200.solvers import (
    ANNEALING,
    ANNEALING_CHECKERBOARD,
    GREEDY,
    GREEDY_CHECKERBOARD,
    KINDS,
    SolverConfig,
    _temperature,
    default_config,
)


def test_config_validation():  # test_solvers.py:18-30
    with pytest.raises(ValueError, match="unknown solver kind"):
        SolverConfig(kind="tabu", sweeps=1, seed=0)
    with pytest.raises(ValueError, match="sweeps"):
        SolverConfig(kind=GREEDY, sweeps=0, seed=0)
    with pytest.raises(ValueError, match="64 bits"):
        SolverConfig(kind=GREEDY, sweeps=1, seed=-1)
    with pytest.raises(ValueError, match="temp_start"):
        SolverConfig(kind=ANNEALING, sweeps=1, seed=0)
    with pytest.raises(ValueError, match="temp_end < temp_start"):
        SolverConfig(kind=ANNEALING, sweeps=1, seed=0, temp_start=1.0, temp_end=2.0)
    with pytest.raises(ValueError, match="no temperatures"):
        SolverConfig(kind=GREEDY, sweeps=1, seed=0, temp_start=1.0)
    with pytest.raises(ValueError, match="temp_start"):
        SolverConfig(kind=ANNEALING_CHECKERBOARD, sweeps=1, seed=0)
    assert set(KINDS) == {GREEDY, ANNEALING, GREEDY_CHECKERBOARD, ANNEALING_CHECKERBOARD,
                          "greedy_random_scan", "simulated_annealing_random_scan"}


def test_default_config_and_schedule():  # test_solvers.py:33-46
    c = default_config(ANNEALING, 50, seed=3)
    assert (c.temp_start, c.temp_end) == (3.0, 0.05)
    g = default_config(GREEDY, 50, seed=3)
    assert g.temp_start is None and g.temp_end is None
    c10 = default_config(ANNEALING, 10, seed=0)
    assert _temperature(c10, 0) == 3.0
    assert _temperature(c10, 9) == pytest.approx(0.05)
    assert _temperature(c10, 4) < _temperature(c10, 3)
    assert _temperature(default_config(ANNEALING, 1, seed=0), 0) == 3.0


def test_mix_seed():
    assert [mix_seed(1234567, i) for i in range(3)] == [
        6457827717110365317, 3203168211198807973, 9817491932198370423]
    for m, i, v in golden("rng_kat.json")["mix_seed"]:
        assert mix_seed(m, i) == v
    assert mix_seeds(20250814, range(500)).tolist() == [mix_seed(20250814, i) for i in range(500)]
    with pytest.raises(ValueError):
        mix_seed(-1, 0)
    with pytest.raises(ValueError):
        mix_seed(2**64, 0)
    with pytest.raises(ValueError):
        mix_seed(0, -1)


def test_codec():
    for c in golden("codec.json")["cases"]:
        assert encode_hex(c["spins"]) == c["hex"]
        assert decode_hex(c["hex"], len(c["spins"])) == tuple(c["spins"])
        p = pack_spins(np.array(c["spins"]))
        assert unpack_spins(p, len(c["spins"])).tolist() == c["spins"]
    assert encode_hex([1, -1, -1, -1]) == "8"
    with pytest.raises(HexDecodeError):
        decode_hex("zz", 8)
    with pytest.raises(HexDecodeError):
        decode_hex("f", 3)  # nonzero pad bit
    with pytest.raises(ValueError):
        encode_hex([])
    with pytest.raises(ValueError):
        encode_hex([1, 0])


def test_generate_torus_matches_reference():
    for rec in golden("tori.json")["tori"]:
        if rec["n"] > 100_000:
            continue
        inst = generate_torus(TorusSpec(rec["rows"], rec["cols"], rec["seed"]))
        assert hashlib.sha256(inst.torus_weights.tobytes()).hexdigest() == rec["w_sha256"]
        assert inst.total_weight() == rec["total_weight"]
        assert inst.m == rec["m"] and inst.n == rec["n"]
        if "w" in rec:
            assert [w for _, _, w in inst.edges] == rec["w"]


def test_torus_edges_structure():  # test_instances.py:134-151
    inst = generate_torus(TorusSpec(3, 4, 5))
    assert inst.m == 24
    deg = [0] * (inst.n + 1)
    for u, v, w in inst.edges:
        assert 1 <= u < v <= inst.n and w in (-1, 1)
        deg[u] += 1
        deg[v] += 1
    assert all(d == 4 for d in deg[1:])
    assert inst.edges[0][:2] == (1, 2) and inst.edges[1][:2] == (1, 5)
    assert inst == generate_torus(TorusSpec(3, 4, 5))
    assert inst.name == "torus:3x4:5"
    assert parse_torus_name("torus:3x4:5") == TorusSpec(3, 4, 5)
    with pytest.raises(ValueError):
        TorusSpec(2, 5, 1)
    with pytest.raises(ValueError):
        parse_torus_name("grid:3x4:5")


def test_problem_instance_validation():
    with pytest.raises(GsetFormatError):
        ProblemInstance.from_edges(3, [(1, 1, 1)])
    with pytest.raises(GsetFormatError):
        ProblemInstance.from_edges(3, [(1, 4, 1)])
    with pytest.raises(GsetFormatError):
        ProblemInstance.from_edges(3, [(1, 2, 1), (2, 1, 1)])
    inst = parse_gset("3 2\n1 2 5\n3 2 -1\n")
    assert inst.edges == ((1, 2, 5), (2, 3, -1))
    with pytest.raises(AttributeError):
        inst.n = 4


def test_records_and_summary():  # test_campaign.py record/summary behaviour
    recs = [TrialRecord(index=i, instance="torus:4x4:1", kind=ANNEALING, sweeps=50,
                        seed=mix_seed(1, i), best_cut=c, sweeps_executed=50, wall_time_s=0.001,
                        temp_start=3.0, temp_end=0.05) for i, c in enumerate([10, 8, 10, 9])]
    for r in recs:
        assert parse_record(format_record(r)) == r
    s = summarize(recs, (TargetSpec("opt", 10),))
    assert (s.highest_cut, s.min_cut, s.average_cut) == (10, 8, 9.25)
    assert s.cut_histogram == {10: 2, 8: 1, 9: 1}
    assert s.targets[0].successes == 2
    assert s.targets[0].repetitions == pytest.approx(repetitions_to_target(0.5))
    assert summarize(recs[::-1], (TargetSpec("opt", 10),)).deterministic_fields() == \
        s.deterministic_fields()
    with pytest.raises(ValueError):
        CampaignConfig("x", default_config(ANNEALING, 5, 0), 0, 1)


def _reference_campaign():
    """The unmodified reference's campaign module (baseline/_ref copy staged by
    __graft_entry__.build(), or the build container's /root/reference)."""
    import importlib
    import sys
    from pathlib import Path

    from conftest import ROOT

    for src in (ROOT / "baseline" / "_ref" / "pkg" / "src", Path("/root/reference/pkg/src")):
        if (src / "gsetbench" / "campaign.py").exists():
            if str(src) not in sys.path:
                sys.path.append(str(src))
            return importlib.import_module("gsetbench.campaign"), importlib.import_module(
                "gsetbench.metrics")
    pytest.skip("reference package not staged (run __graft_entry__.build() in the build container)")


def test_log_lines_and_summaries_equal_the_references():
    """Records written here are byte-identical to the reference's format_record
    output, parse back through the reference's parser, and summarize to the
    same deterministic fields (campaign.py:103-147, :233-297)."""
    ref, refm = _reference_campaign()
    rng = np.random.default_rng(5)
    ours, theirs = [], []
    for i in range(40):
        sa = bool(i % 3)
        f = dict(index=i, instance="torus:50x100:1", kind=ANNEALING if sa else GREEDY,
                 sweeps=1000, seed=mix_seed(20250814, i), best_cut=int(rng.integers(3400, 3480)),
                 sweeps_executed=1000 if sa else int(rng.integers(3, 9)),
                 wall_time_s=float(rng.uniform(1e-6, 3.0)),
                 temp_start=3.0 if sa else None, temp_end=0.05 if sa else None,
                 spins_hex=("%x" % int(rng.integers(0, 2**62))) if i % 2 else None)
        a, b = TrialRecord(**f), ref.TrialRecord(**f)
        line = format_record(a)
        assert line == ref.format_record(b)
        import dataclasses
        assert dataclasses.asdict(ref.parse_record(line)) == dataclasses.asdict(parse_record(line))
        ours.append(a)
        theirs.append(b)
    for kind in (ANNEALING, GREEDY):
        mine = summarize([r for r in ours if r.kind == kind],
                         (TargetSpec("t", 3450), TargetSpec("never", 9999, 0.9)))
        refs = ref.summarize([r for r in theirs if r.kind == kind],
                             (refm.TargetSpec("t", 3450), refm.TargetSpec("never", 9999, 0.9)))
        assert mine.deterministic_fields() == refs.deterministic_fields()
        assert mine.avg_trial_time_s == refs.avg_trial_time_s
        assert [t.ttt_s for t in mine.targets] == [t.ttt_s for t in refs.targets]
    assert [mix_seed(7, i) for i in range(20)] == [ref.mix_seed(7, i) for i in range(20)]


def test_shard_arithmetic():
    for T in (1, 7, 64, 1000, 8192):
        for W in (1, 2, 3, 4, 8):
            firsts = [shard(T, W, r) for r in range(W)]
            assert sum(c for _, c in firsts) == T
            pos = 0
            for r, (f, c) in enumerate(firsts):
                assert f == pos
                for i in (f, f + c - 1):
                    if c:
                        assert owner_of(i, T, W) == r
                pos += c
    k1, k2 = best_key(100, 5), best_key(100, 3)
    assert k2 > k1 and best_key(101, 9) > k2 and best_key(-5, 0) < best_key(-4, 7)
    assert decode_key(best_key(-17, 42)) == (-17, 42)


def test_parse_gset_fast_path_equals_the_references_parser():
    """parse_gset (one numpy conversion; token loop only for diagnostics) gives
    the reference's instances and the reference's error messages
    (instances.py:117-158)."""
    import importlib

    _reference_campaign()
    ref = importlib.import_module("gsetbench.instances")
    good = ["3 2\n1 2 5\n3 2 -1\n", "# c\n4 3 1 2 1\n2 3 -1 # x\n\n3 4 7\n", "1 0", "2 1\n2 1 -3"]
    for text in good:
        a, b = parse_gset(text, name="g"), ref.parse_gset(text, name="g")
        assert (a.n, a.m, a.edges, a.name) == (b.n, b.m, tuple(b.edges), b.name)
    bad = ["", "3", "0 0", "3 -1", "3 2\n1 2 5\n", "3 1\n1 2 x\n", "3 1\n1 2 3 4\n", "a 1",
           "3 1\n1 1 2\n", "3 1\n1 9 2\n", "3 2\n1 2 1\n2 1 1\n", "2 1\n1 2 1.5\n"]
    for text in bad:
        with pytest.raises(ValueError) as e_ref:
            ref.parse_gset(text)
        with pytest.raises(GsetFormatError) as e_ours:
            parse_gset(text)
        assert str(e_ours.value) == str(e_ref.value), text
