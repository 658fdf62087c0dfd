"""Exact evaluation (mirror of gsetbench.evaluate: cut_value, ising_energy,
flip_delta_cut, evaluate.py:35-64).

``cut_value`` / ``ising_energy`` run on the GPU evaluator
(gsb_torus_cut_energy / gsb_graph_cut_energy); ``*_batch`` evaluates many
packed bitstrings in one launch.
"""

from __future__ import annotations

import numpy as np

from paper_2505_18508_b200 import _lib
from paper_2505_18508_b200.codec import pack_spins
from paper_2505_18508_b200.instances import ProblemInstance


def _spin_array(instance: ProblemInstance, spins) -> np.ndarray:
    """evaluate.py:24-32."""
    arr = np.asarray(spins, dtype=np.int64)
    if arr.shape != (instance.n,):
        raise ValueError(
            f"configuration has {arr.size} spins, instance has {instance.n} variables")
    if not np.all(np.abs(arr) == 1):
        raise ValueError("spins must be -1 or +1")
    return arr


def cut_energy_batch(instance: ProblemInstance, bits, device=None):
    """(cut int64 [T], energy int64 [T]) of packed bitstrings uint8 [T, ceil(n/8)]."""
    torch = _lib.require_cuda()
    dev = torch.device(device if device is not None else "cuda")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    if isinstance(bits, torch.Tensor):
        b = bits.to(dev, dtype=torch.uint8).contiguous()
    else:
        b = torch.from_numpy(np.ascontiguousarray(bits, dtype=np.uint8)).to(dev)
    b = b.reshape(-1, (instance.n + 7) // 8)
    T = b.shape[0]
    cut = torch.empty(T, dtype=torch.int64, device=dev)
    en = torch.empty(T, dtype=torch.int64, device=dev)
    L = _lib.lib()
    with torch.cuda.device(dev):
        sp = torch.cuda.current_stream(dev).cuda_stream
        if instance.torus is not None:
            w = instance.device_weights(dev)
            ts = _lib.torus_struct(instance.torus.rows, instance.torus.cols, w.data_ptr())
            _lib.check(L.gsb_torus_cut_energy(ts, b.data_ptr(), T, cut.data_ptr(), en.data_ptr(),
                                              sp))
        else:
            eu, ev, ew = instance.device_edges(dev)
            gs = _lib.graph_struct(instance.n, len(eu), eu.data_ptr(), ev.data_ptr(),
                                   ew.data_ptr())
            _lib.check(L.gsb_graph_cut_energy(gs, b.data_ptr(), T, cut.data_ptr(), en.data_ptr(),
                                              sp))
    return cut, en


def cut_value(instance: ProblemInstance, spins) -> int:
    """evaluate.py:35-43."""
    s = _spin_array(instance, spins)
    cut, _ = cut_energy_batch(instance, pack_spins(s)[None, :])
    return int(cut[0].item())


def ising_energy(instance: ProblemInstance, spins) -> int:
    """evaluate.py:46-49."""
    s = _spin_array(instance, spins)
    _, en = cut_energy_batch(instance, pack_spins(s)[None, :])
    return int(en[0].item())


def flip_delta_cut(instance: ProblemInstance, spins, k: int) -> int:
    """evaluate.py:52-64 (scalar helper, host)."""
    if not (1 <= k <= instance.n):
        raise ValueError(f"variable {k} out of range 1..{instance.n}")
    sk = spins[k - 1]
    acc = 0
    for j, w in instance.adjacency[k]:
        acc += w * spins[j - 1]
    return sk * acc
