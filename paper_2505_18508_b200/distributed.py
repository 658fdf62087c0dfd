"""Multi-GPU trial scheduler (replaces run_campaign's worker pool, campaign.py:413-426).

Trials are independent (SPEC: campaign.py:1-14), so a campaign of T trials is
split into contiguous index blocks, one per rank (one process per GPU,
torch.distributed).  Each rank runs its block as one batched launch; the only
exchange is at the end:

* the global best: all-reduce MAX of key = (best_cut << 32) | (0xFFFFFFFF - index)
  -- highest cut wins, ties go to the lowest trial index -- then the owner
  broadcasts the winning bitstring;
* optionally the per-trial cuts / sweeps (all-gather) for the campaign summary,
  whose histogram needs every trial (campaign.py:257-262).

Seeds are mix_seed(master, index), so the result set is identical for every
world size (batch invariance).  The reduction helpers take plain tensors and
work with NCCL (CUDA tensors) and gloo (CPU tensors, used by the tests).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def shard(num_trials: int, world: int, rank: int) -> tuple[int, int]:
    """(first_index, count) of rank's contiguous block of trial indices."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} for world size {world}")
    base, rem = divmod(num_trials, world)
    count = base + (1 if rank < rem else 0)
    first = rank * base + min(rank, rem)
    return first, count


def owner_of(index: int, num_trials: int, world: int) -> int:
    """Rank whose block holds trial `index` (inverse of shard)."""
    base, rem = divmod(num_trials, world)
    big = rem * (base + 1)
    if index < big:
        return index // (base + 1)
    return rem + (index - big) // base if base else world - 1


def best_key(best_cut: int, index: int) -> int:
    """campaign-wide ordering key: higher cut first, then lower trial index."""
    return (int(best_cut) << 32) | (0xFFFFFFFF - int(index))


def decode_key(key: int) -> tuple[int, int]:
    return key >> 32, 0xFFFFFFFF - (key & 0xFFFFFFFF)


@dataclass
class GlobalBest:
    best_cut: int
    index: int
    bits: np.ndarray  # uint8 packed bitstring of the winning trial


def reduce_best(local_cut, local_bits, first_index: int, num_trials: int, group=None):
    """All-reduce the campaign best across ranks.

    local_cut: int64 tensor [count] (device of the backend), local_bits: uint8
    tensor [count, nbytes].  Returns GlobalBest (same on every rank).
    """
    import torch
    import torch.distributed as dist

    # collectives run whenever a process group exists (also at world size 1,
    # so a one-GPU NCCL group exercises the same calls as eight GPUs)
    pg = dist.is_initialized()
    world = dist.get_world_size(group) if pg else 1
    dev = local_cut.device
    nbytes = local_bits.shape[1]
    if local_cut.numel():
        if local_cut.is_cuda:  # key kernel of the library (gsb_best_key)
            from paper_2505_18508_b200 import _lib

            keys = torch.empty(local_cut.numel(), dtype=torch.int64, device=dev)
            cut64 = local_cut.to(torch.int64).contiguous()
            _lib.check(_lib.lib().gsb_best_key(cut64.data_ptr(), cut64.numel(), first_index,
                                               keys.data_ptr(),
                                               torch.cuda.current_stream(dev).cuda_stream))
        else:
            idx = torch.arange(first_index, first_index + local_cut.numel(), device=dev,
                               dtype=torch.int64)
            keys = (local_cut.to(torch.int64) << 32) | (0xFFFFFFFF - idx)
        k = keys.max().reshape(1)
    else:
        k = torch.full((1,), torch.iinfo(torch.int64).min, device=dev, dtype=torch.int64)
    if pg:
        dist.all_reduce(k, op=dist.ReduceOp.MAX, group=group)
    gk = int(k.item())
    cut, index = decode_key(gk)
    bits = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    owner = owner_of(index, num_trials, world)
    rank = dist.get_rank(group) if pg else 0
    if rank == owner:
        bits.copy_(local_bits[index - first_index])
    if pg:
        dist.broadcast(bits, src=dist.get_global_rank(group, owner) if group is not None else owner,
                       group=group)
    return GlobalBest(best_cut=cut, index=index, bits=bits.cpu().numpy())


def gather_trials(local_cut, local_sweeps, num_trials: int, group=None):
    """All-gather per-trial (best_cut, sweeps_executed) in trial-index order."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized():
        return local_cut.cpu().numpy(), local_sweeps.cpu().numpy()
    world = dist.get_world_size(group)
    dev = local_cut.device
    maxc = -(-num_trials // world)
    pc = torch.zeros(maxc, dtype=torch.int64, device=dev)
    ps = torch.zeros(maxc, dtype=torch.int64, device=dev)
    pc[: local_cut.numel()] = local_cut.to(torch.int64)
    ps[: local_sweeps.numel()] = local_sweeps.to(torch.int64)
    outc = [torch.empty_like(pc) for _ in range(world)]
    outs = [torch.empty_like(ps) for _ in range(world)]
    dist.all_gather(outc, pc, group=group)
    dist.all_gather(outs, ps, group=group)
    cuts, sweeps = [], []
    for r in range(world):
        _, cnt = shard(num_trials, world, r)
        cuts.append(outc[r][:cnt].cpu().numpy())
        sweeps.append(outs[r][:cnt].cpu().numpy())
    return np.concatenate(cuts), np.concatenate(sweeps)


def run_sharded(instance, config, master_seed: int, num_trials: int, group=None,
                device=None):
    """Run this rank's block of a campaign on its GPU and reduce the best.

    Returns (GlobalBest, all_cuts, all_sweeps) on every rank.
    """
    import torch
    import torch.distributed as dist

    from paper_2505_18508_b200.campaign import mix_seeds
    from paper_2505_18508_b200.solvers import run_trials_device

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    first, count = shard(num_trials, world, rank)
    seeds = mix_seeds(master_seed, range(first, first + count))
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    best, sweeps, bits = run_trials_device(instance, config, seeds, device=device)
    g = reduce_best(best, bits, first, num_trials, group)
    cuts, sw = gather_trials(best, sweeps, num_trials, group)
    return g, cuts, sw


def gather_rows(local, counts, group=None):
    """All-gather a per-trial tensor whose leading dimension is this rank's
    trial count (counts[r] on rank r) into trial-index order (numpy)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    pad = torch.zeros((max(counts),) + tuple(local.shape[1:]), dtype=local.dtype,
                      device=local.device)
    pad[: local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return np.concatenate([parts[r][: counts[r]].cpu().numpy() for r in range(world)])


def run_sharded_seeds(instance, config, seeds, group=None, device=None):
    """The multi-GPU form of solvers.run_trials for an explicit seed list (the
    pending trials of a campaign): rank r runs the r-th contiguous block on
    its GPU, then every rank receives all results in seed order.  Returns
    (best_cut, sweeps_executed, hex_of) like a TrialBatch's fields.  Must be
    called by every rank of the group with the same arguments."""
    import torch
    import torch.distributed as dist

    from paper_2505_18508_b200.codec import packed_to_hex
    from paper_2505_18508_b200.solvers import run_trials_device

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    seeds = np.asarray(seeds, dtype=np.uint64)
    blocks = [shard(len(seeds), world, r) for r in range(world)]
    first, count = blocks[rank]
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    best, sweeps, bits = run_trials_device(instance, config, seeds[first:first + count],
                                           device=device)
    if dist.get_backend(group) == "gloo":  # CPU collectives (development / tests)
        best, sweeps, bits = best.cpu(), sweeps.cpu(), bits.cpu()
    counts = [c for _, c in blocks]
    cuts = gather_rows(best, counts, group)
    done = gather_rows(sweeps, counts, group)
    allbits = gather_rows(bits, counts, group)
    n = instance.n
    return cuts, done, lambda j: packed_to_hex(allbits[j], n)
