"""Multi-rank path on CPU: world_size 2 over gloo (127.0.0.1).

Per-rank trial results come from the CPU oracle (test infrastructure); the
reduction/gather code under test is the product's
(paper_2505_18508_b200.distributed), the same code bench.py and
run_sharded use with NCCL on GPUs.
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, T, ret):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_2505_18508_b200.campaign import mix_seeds
    from paper_2505_18508_b200.codec import pack_spins
    from paper_2505_18508_b200.distributed import gather_trials, reduce_best, shard

    rows, cols = 6, 8
    w = O.torus_weights(rows, cols, 2)
    first, count = shard(T, world, rank)
    seeds = mix_seeds(20250814, range(first, first + count))
    bc, bs, se = O.run_trials_checker(rows, cols, w, "simulated_annealing_checkerboard", 30,
                                      seeds, 3.0, 0.05, nthreads=1)
    cut = torch.from_numpy(bc.astype(np.int64))
    bits = torch.from_numpy(np.stack([pack_spins(s) for s in bs]))
    g = reduce_best(cut, bits, first, T)
    cuts, sw = gather_trials(cut, torch.from_numpy(se.astype(np.int64)), T)
    if rank == 0:
        ret.put((g.best_cut, g.index, g.bits.tobytes().hex(), cuts.tolist(), sw.tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("T", [9, 16])
def test_gloo_world2_reduction_matches_single_process(T):
    from oracle import oracle as O
    from paper_2505_18508_b200.campaign import mix_seeds
    from paper_2505_18508_b200.codec import pack_spins

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, T, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    best_cut, index, bits_hex, cuts, sweeps = res
    # single-process reference of the same campaign
    w = O.torus_weights(6, 8, 2)
    bc, bs, se = O.run_trials_checker(6, 8, w, "simulated_annealing_checkerboard", 30,
                                      mix_seeds(20250814, range(T)), 3.0, 0.05)
    assert cuts == bc.tolist() and sweeps == se.tolist()
    top = int(bc.max())
    assert best_cut == top
    assert index == int(np.nonzero(bc == top)[0][0])  # ties -> lowest trial index
    assert bits_hex == pack_spins(bs[index]).tobytes().hex()
