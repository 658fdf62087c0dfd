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
