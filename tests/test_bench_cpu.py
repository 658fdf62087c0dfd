"""bench.py's reference arm (oracle port on host cores) runs on CPU and prints
one well-formed JSON line with the contract's keys."""

import json
import subprocess
import sys

from conftest import ROOT


def test_reference_arm_json_line():
    out = subprocess.run(
        [sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "c1",
         "--steps", "1", "--warmup", "0", "--sweeps", "20", "--cpu-seconds", "0.5"],
        capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better",
              "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "port"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def _json_lines(out):
    return [json.loads(ln) for ln in out.stdout.splitlines() if ln.strip().startswith("{")]


def test_gpus_flag_launches_the_ranks_itself():
    """`bench.py --gpus 2` outside torchrun starts two ranks (torch.distributed.run,
    127.0.0.1) and reports n_gpus 2; --dry-run does the rendezvous (gloo) and the
    sharding plan without touching CUDA, so it runs here."""
    for scaling, shards in (("weak", [[0, 4096], [4096, 4096]]), ("strong", [[0, 2048], [2048, 2048]])):
        out = subprocess.run(
            [sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--config", "c3", "--dry-run",
             "--scaling", scaling], capture_output=True, text=True, timeout=300, cwd=ROOT)
        assert out.returncode == 0, out.stderr[-2000:]
        lines = _json_lines(out)
        assert len(lines) == 1, out.stdout
        d = lines[0]
        assert d["n_gpus"] == 2 and d["scaling"] == scaling and d["shards"] == shards
        assert d["config"]["kind"] == "simulated_annealing_random_scan"
        assert d["config"]["trials"] == (8192 if scaling == "weak" else 4096)


def test_gpus_flag_must_match_world_size():
    env = dict(__import__("os").environ, WORLD_SIZE="1", RANK="0", MASTER_ADDR="127.0.0.1",
               MASTER_PORT="29999")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "8", "--dry-run"],
                         capture_output=True, text=True, timeout=120, cwd=ROOT, env=env)
    assert out.returncode == 2 and "WORLD_SIZE=1" in out.stderr


def test_both_arms_share_the_config_object():
    """The reference arm reports the same `config` as our arm (so the driver's
    same_config check can hold): compared through the dry run."""
    ours = _json_lines(subprocess.run(
        [sys.executable, str(ROOT / "bench.py"), "--config", "c1", "--sweeps", "20", "--dry-run"],
        capture_output=True, text=True, timeout=120, cwd=ROOT))[0]
    ref = _json_lines(subprocess.run(
        [sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "c1",
         "--steps", "1", "--warmup", "0", "--sweeps", "20", "--cpu-seconds", "0.5"],
        capture_output=True, text=True, timeout=300, cwd=ROOT))[0]
    assert ours["config"] == ref["config"]
