"""NCCL path of the trial scheduler on the GPU box (one GPU: world size 1).

The collectives of paper_2505_18508_b200.distributed (all-reduce MAX of the
best key, owner broadcast of the winning bitstring, all-gather of per-trial
cuts) run whenever a process group exists, so a one-rank NCCL group executes
the same calls bench.py makes on eight GPUs; world size 2 is covered on CPU
over gloo (tests/test_distributed_cpu.py).
"""

import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture
def nccl_world1():
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0,
                            world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


def test_nccl_run_sharded_matches_single_device(nccl_world1):
    from paper_2505_18508_b200 import TorusSpec, generate_torus
    from paper_2505_18508_b200.campaign import mix_seeds
    from paper_2505_18508_b200.distributed import run_sharded
    from paper_2505_18508_b200.solvers import (ANNEALING_CHECKERBOARD, default_config,
                                               run_trials_device)

    assert dist.get_backend() == "nccl"
    inst = generate_torus(TorusSpec(20, 30, 3))
    cfg = default_config(ANNEALING_CHECKERBOARD, 40, 0)
    T = 37
    g, cuts, sweeps = run_sharded(inst, cfg, 20250814, T)
    best, sw, bits = run_trials_device(inst, cfg, mix_seeds(20250814, range(T)))
    bc = best.cpu().numpy()
    assert cuts.tolist() == bc.tolist()
    assert sweeps.tolist() == sw.cpu().numpy().tolist()
    top = int(bc.max())
    assert g.best_cut == top
    assert g.index == int(np.nonzero(bc == top)[0][0])  # ties -> lowest trial index
    assert g.bits.tobytes() == bits[g.index].cpu().numpy().tobytes()


def _campaign_worker(rank, world, port, log_path, ret):
    import os
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    # development arrangement for a one-GPU box: both ranks on cuda:0, CPU
    # collectives (gloo); the ranks never wait on each other inside a kernel
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    from paper_2505_18508_b200 import TorusSpec, generate_torus
    from paper_2505_18508_b200.campaign import CampaignConfig, TargetSpec, run_campaign
    from paper_2505_18508_b200.solvers import ANNEALING_RANDOM_SCAN, default_config

    torch.cuda.set_device(0)
    inst = generate_torus(TorusSpec(12, 20, 5))
    cfg = CampaignConfig(inst.name, default_config(ANNEALING_RANDOM_SCAN, 30, 0), 21, 77,
                         targets=(TargetSpec("t", 150),))
    s = run_campaign(inst, cfg, log_path=log_path, include_spins=True)
    if rank == 0:
        ret.put(s.deterministic_fields())
    dist.barrier()
    dist.destroy_process_group()


def test_run_campaign_shards_over_the_process_group(tmp_path):
    """run_campaign under a 2-rank process group: each rank runs its block of
    the pending trials, rank 0 writes the log; summary and log lines equal the
    single-process campaign's (results never depend on the world size)."""
    import torch.multiprocessing as mp

    from paper_2505_18508_b200 import TorusSpec, generate_torus
    from paper_2505_18508_b200.campaign import (CampaignConfig, TargetSpec, read_log,
                                                run_campaign)
    from paper_2505_18508_b200.solvers import ANNEALING_RANDOM_SCAN, default_config

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    log2 = tmp_path / "two_ranks.log"
    procs = [ctx.Process(target=_campaign_worker, args=(r, 2, port, str(log2), q))
             for r in range(2)]
    for p in procs:
        p.start()
    fields = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    inst = generate_torus(TorusSpec(12, 20, 5))
    cfg = CampaignConfig(inst.name, default_config(ANNEALING_RANDOM_SCAN, 30, 0), 21, 77,
                         targets=(TargetSpec("t", 150),))
    log1 = tmp_path / "one_rank.log"
    single = run_campaign(inst, cfg, log_path=log1, include_spins=True)
    assert fields == single.deterministic_fields()
    strip = lambda recs: [(r.index, r.seed, r.best_cut, r.sweeps_executed, r.spins_hex)  # noqa: E731
                          for r in recs]
    assert strip(read_log(log2)) == strip(read_log(log1)) and len(read_log(log2)) == 21


@pytest.mark.parametrize("scaling,trials", [("weak", 200), ("strong", 100)])
def test_bench_gpus_2_on_one_gpu(scaling, trials):
    """`bench.py --gpus 2` starts its two ranks itself; here both share the one
    GPU over gloo (GSB_BENCH_SHARE_GPU=1, a development arrangement: plumbing,
    not a measurement).  The line reports n_gpus 2 and the campaign-wide best."""
    import json
    import os
    import subprocess
    import sys

    from conftest import ROOT

    env = dict(os.environ, GSB_BENCH_SHARE_GPU="1")
    out = subprocess.run(
        [sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--config", "c1", "--sweeps", "40",
         "--steps", "1", "--warmup", "1", "--no-cpu", "--no-secondary", "--scaling", scaling],
        capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = lines[0]
    assert d["n_gpus"] == 2 and d["scaling"] == scaling and d["config"]["trials"] == trials
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] == 2
    assert d["config"]["kind"] == "simulated_annealing_random_scan"
