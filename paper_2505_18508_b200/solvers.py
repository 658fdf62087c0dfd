"""Sweep solvers on the B200 engine (mirror of gsetbench.solvers, solvers.py:1-140).

Kinds:

* ``greedy_local_search`` / ``simulated_annealing`` -- the reference kinds
  (solvers.py:27-29), run by the *reference engine*: numpy-PCG64 stream and
  random-permutation sweeps, bit-for-bit identical to gsetbench's run_trial.
* ``greedy_checkerboard`` / ``simulated_annealing_checkerboard`` -- the
  throughput kinds (SPEC.md anticipates "a third kind"): identical trial
  semantics except the sweep visits the colour-0 sites, then the colour-1
  sites, in increasing id, and draws come from Philox4x32-10 keyed by the seed
  (checkerboard contract).  Even tori only.  The systematic order
  mixes faster per sweep than the reference's random order, so its final cuts
  are higher than the reference's at equal sweeps.
* ``greedy_random_scan`` / ``simulated_annealing_random_scan`` -- the
  reference's random visit order, drawn from Philox as per-site priorities and
  run level by level on the GPU (random-scan contract): the
  reference's dynamics in law, so its final-cut distribution agrees with
  run_trial's.  Any torus (register-resident teams up to one SM, the
  large-torus engine with its planes in global memory beyond).

Every trial is a deterministic function of (instance, config) and never of
the batch it runs in.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, replace

import numpy as np

from paper_2505_18508_b200 import _lib
from paper_2505_18508_b200.codec import packed_to_hex, unpack_spins
from paper_2505_18508_b200.instances import ProblemInstance

GREEDY = "greedy_local_search"
ANNEALING = "simulated_annealing"
GREEDY_CHECKERBOARD = "greedy_checkerboard"
ANNEALING_CHECKERBOARD = "simulated_annealing_checkerboard"
REFERENCE_KINDS = (GREEDY, ANNEALING)
GREEDY_RANDOM_SCAN = "greedy_random_scan"
ANNEALING_RANDOM_SCAN = "simulated_annealing_random_scan"
CHECKERBOARD_KINDS = (GREEDY_CHECKERBOARD, ANNEALING_CHECKERBOARD)
RANDOM_SCAN_KINDS = (GREEDY_RANDOM_SCAN, ANNEALING_RANDOM_SCAN)
KINDS = REFERENCE_KINDS + CHECKERBOARD_KINDS + RANDOM_SCAN_KINDS
ANNEALING_KINDS = (ANNEALING, ANNEALING_CHECKERBOARD, ANNEALING_RANDOM_SCAN)

DEFAULT_TEMP_START = 3.0
DEFAULT_TEMP_END = 0.05


@dataclass(frozen=True)
class SolverConfig:
    """solvers.py:35-59 (validation messages kept verbatim)."""

    kind: str
    sweeps: int
    seed: int
    temp_start: float | None = None
    temp_end: float | None = None

    def __post_init__(self) -> None:
        if self.kind not in KINDS:
            raise ValueError(f"unknown solver kind {self.kind!r}, expected one of {KINDS}")
        if self.sweeps < 1:
            raise ValueError(f"sweeps must be positive, got {self.sweeps}")
        if not (0 <= self.seed < 2**64):
            raise ValueError(f"seed must fit in 64 bits, got {self.seed}")
        if self.kind in ANNEALING_KINDS:
            if self.temp_start is None or self.temp_end is None:
                raise ValueError("simulated annealing needs temp_start and temp_end")
            if not (0.0 < self.temp_end < self.temp_start):
                raise ValueError(
                    f"need 0 < temp_end < temp_start, got ({self.temp_start}, {self.temp_end})")
        elif self.temp_start is not None or self.temp_end is not None:
            raise ValueError("greedy local search takes no temperatures")

    @property
    def engine(self) -> int:
        if self.kind in CHECKERBOARD_KINDS:
            return _lib.ENGINE_CHECKERBOARD
        if self.kind in RANDOM_SCAN_KINDS:
            return _lib.ENGINE_RANDOM_SCAN
        return _lib.ENGINE_REFERENCE

    @property
    def annealing(self) -> bool:
        return self.kind in ANNEALING_KINDS


def default_config(kind: str, sweeps: int, seed: int) -> SolverConfig:
    """solvers.py:62-72."""
    if kind in ANNEALING_KINDS:
        return SolverConfig(kind=kind, sweeps=sweeps, seed=seed,
                            temp_start=DEFAULT_TEMP_START, temp_end=DEFAULT_TEMP_END)
    return SolverConfig(kind=kind, sweeps=sweeps, seed=seed)


@dataclass(frozen=True)
class TrialResult:
    """solvers.py:75-81."""

    best_cut: int
    best_spins: tuple[int, ...]
    sweeps_executed: int
    wall_time_s: float
    seed: int


def _temperature(config: SolverConfig, sweep_index: int) -> float:
    """solvers.py:84-88."""
    if config.sweeps == 1:
        return config.temp_start
    frac = sweep_index / (config.sweeps - 1)
    return config.temp_start * (config.temp_end / config.temp_start) ** frac


class TrialBatch:
    """Results of a batch of trials, kept packed until asked for.

    best_cut: int64 [T]; sweeps_executed: int32 [T]; bits: uint8 [T, ceil(n/8)]
    (MSB-first by variable id); seeds: uint64 [T].
    """

    def __init__(self, n, seeds, best_cut, sweeps_executed, bits, wall_time_s):
        self.n = n
        self.seeds = seeds
        self.best_cut = best_cut
        self.sweeps_executed = sweeps_executed
        self.bits = bits
        self.wall_time_s = wall_time_s

    def __len__(self):
        return len(self.seeds)

    def hex(self, i: int) -> str:
        return packed_to_hex(self.bits[i], self.n)

    def spins(self, i: int) -> np.ndarray:
        return unpack_spins(self.bits[i], self.n)

    def result(self, i: int) -> TrialResult:
        return TrialResult(
            best_cut=int(self.best_cut[i]),
            best_spins=tuple(int(x) for x in self.spins(i)),
            sweeps_executed=int(self.sweeps_executed[i]),
            wall_time_s=self.wall_time_s / max(len(self), 1),
            seed=int(self.seeds[i]),
        )


def schedule_table(config: SolverConfig, dmax: int = 4) -> np.ndarray | None:
    """Acceptance thresholds [sweeps, dmax] uint64 (gsb_schedule_table)."""
    if not config.annealing:
        return None
    tab = np.empty((config.sweeps, dmax), dtype=np.uint64)
    _lib.check(_lib.lib().gsb_schedule_table(config.engine, config.sweeps, config.temp_start,
                                             config.temp_end, dmax, tab.ctypes.data))
    return tab


# engines that run the same trial contract (an override may only move inside one)
_ENGINE_FAMILY = {
    _lib.ENGINE_REFERENCE: "reference",
    _lib.ENGINE_CHECKERBOARD: "checkerboard",
    _lib.ENGINE_CHECKERBOARD_TILED: "checkerboard",
    _lib.ENGINE_CHECKERBOARD_CLUSTER: "checkerboard",
    _lib.ENGINE_RANDOM_SCAN: "random_scan",
    _lib.ENGINE_RANDOM_SCAN_LARGE: "random_scan",
}


def _graph_dmax(instance: ProblemInstance) -> int:
    eu, ev, ew = instance.edge_arrays()
    tot = np.zeros(instance.n, dtype=np.int64)
    np.add.at(tot, eu, np.abs(ew))
    np.add.at(tot, ev, np.abs(ew))
    return max(int(tot.max()) if tot.size else 1, 1)


def rscan_fits(rows: int, cols: int) -> bool:
    """Whether a rows x cols torus fits a random-scan engine (register-resident teams, or the
    large-torus engine with its planes in global memory)."""
    return _lib.lib().gsb_rscan_fits(rows, cols) != 0


def rscan_shape(rows: int, cols: int, T: int) -> tuple[int, int]:
    """(warps per trial, rows per lane) the random-scan engine launches for T trials."""
    import ctypes

    nw, rb = ctypes.c_int32(0), ctypes.c_int32(0)
    _lib.check(_lib.lib().gsb_rscan_shape(rows, cols, T, ctypes.byref(nw), ctypes.byref(rb)))
    return nw.value, rb.value


def _test_rscan_shape(warps: int = 0, rows_per_lane: int = 0) -> None:
    """TEST-ONLY: force the random-scan team shape of later launches ((0, 0) = automatic)."""
    _lib.check(_lib.lib().gsb_test_rscan_shape(warps, rows_per_lane))


def _test_checker_shape(warps: int = 0, variant: int = 0) -> None:
    """TEST-ONLY: force the checkerboard team shape / one-warp variant (0 = automatic)."""
    _lib.check(_lib.lib().gsb_test_checker_shape(warps, variant))


def _test_cluster_size(ctas: int = 0) -> None:
    """TEST-ONLY: force the cluster engine's CTA count (0 = automatic)."""
    _lib.check(_lib.lib().gsb_test_cluster_size(ctas))


def _test_rscan_limits(tie_queue_cap: int = 0, list_cap: int = 0) -> None:
    """TEST-ONLY: shrink the random-scan tie queue / event list (0 = default)."""
    _lib.check(_lib.lib().gsb_test_rscan_limits(tie_queue_cap, list_cap))


def _test_rscan_slices(slices: int = 0) -> None:
    """TEST-ONLY: force the sweep slices of annealing random-scan launches (0 = automatic)."""
    _lib.check(_lib.lib().gsb_test_rscan_slices(slices))


def run_trials_device(instance: ProblemInstance, config: SolverConfig, seeds, device=None,
                      stream=None, check: bool = True, engine: int | None = None):
    """Batched trials with device-resident outputs (torch tensors).

    ``seeds`` is a uint64-valued sequence or an int64 CUDA tensor holding the
    seed bit patterns.  Returns (best_cut int64 [T], sweeps_executed int32 [T],
    bits uint8 [T, ceil(n/8)]) on ``device``.  With ``check`` (default) the
    call synchronises and raises RuntimeError if the device integrity guard
    (solvers.py:132-133) fired; without it the launch stays asynchronous.
    """
    torch = _lib.require_cuda()
    dev = torch.device(device if device is not None else "cuda")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    L = _lib.lib()
    if isinstance(seeds, torch.Tensor):
        seeds_d = seeds.to(dev, dtype=torch.int64)
    else:
        arr = np.asarray(seeds, dtype=np.uint64)
        seeds_d = torch.from_numpy(arr.view(np.int64).copy()).to(dev)
    T = int(seeds_d.numel())
    n = instance.n
    nbytes = (n + 7) // 8
    best = torch.empty(T, dtype=torch.int64, device=dev)
    sweeps = torch.empty(T, dtype=torch.int32, device=dev)
    bits = torch.empty((T, nbytes), dtype=torch.uint8, device=dev)
    if T == 0:
        return best, sweeps, bits
    kind = _lib.GSB_ANNEALING if config.annealing else _lib.GSB_GREEDY
    eng = config.engine if engine is None else engine
    if engine is not None and _ENGINE_FAMILY.get(engine) != _ENGINE_FAMILY[config.engine]:
        raise ValueError("engine override must keep the kind's trial semantics "
                         "(checkerboard kinds: CHECKERBOARD / _TILED / _CLUSTER only)")
    with torch.cuda.device(dev):
        cur = torch.cuda.current_stream(dev)
        s = stream if stream is not None else cur
        sp = s.cuda_stream
        if s != cur:
            # inputs and scratch are produced / allocated on the current stream:
            # order the launch stream after it and tie their lifetime to `s`
            s.wait_stream(cur)
            for t in (seeds_d, best, sweeps, bits):
                t.record_stream(s)
        if instance.torus is not None:
            w = instance.device_weights(dev)
            ts = _lib.torus_struct(instance.torus.rows, instance.torus.cols, w.data_ptr())
            tab = schedule_table(config, 4)
            tab_d = (torch.from_numpy(tab.view(np.int64)).to(dev) if tab is not None else None)
            wsb = L.gsb_torus_workspace_bytes(ts, eng, config.sweeps, T)
            ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
            if s != cur:
                s.wait_stream(cur)  # weights / table / workspace just produced on `cur`
                for t in (w, ws) + ((tab_d,) if tab_d is not None else ()):
                    t.record_stream(s)
            _lib.check(L.gsb_torus_sweep(ts, eng, kind, config.sweeps,
                                         tab_d.data_ptr() if tab_d is not None else None,
                                         seeds_d.data_ptr(), T, best.data_ptr(),
                                         sweeps.data_ptr(), bits.data_ptr(), ws.data_ptr(), wsb,
                                         sp))
            if check:
                _lib.check(L.gsb_workspace_status(ws.data_ptr(), sp))
        else:
            if config.engine != _lib.ENGINE_REFERENCE:
                raise ValueError("checkerboard and random-scan kinds need a torus instance")
            eu, ev, ew = instance.device_edges(dev)
            dmax = _graph_dmax(instance)
            gs = _lib.graph_struct(n, len(eu), eu.data_ptr(), ev.data_ptr(), ew.data_ptr())
            tab = schedule_table(config, dmax)
            tab_d = (torch.from_numpy(tab.view(np.int64)).to(dev) if tab is not None else None)
            wsb = L.gsb_graph_workspace_bytes(gs, config.sweeps, T)
            ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
            if s != cur:
                s.wait_stream(cur)
                for t in (eu, ev, ew, ws) + ((tab_d,) if tab_d is not None else ()):
                    t.record_stream(s)
            _lib.check(L.gsb_graph_sweep(gs, kind, config.sweeps,
                                         tab_d.data_ptr() if tab_d is not None else None, dmax,
                                         seeds_d.data_ptr(), T, best.data_ptr(),
                                         sweeps.data_ptr(), bits.data_ptr(), ws.data_ptr(), wsb,
                                         sp))
            if check:
                _lib.check(L.gsb_workspace_status(ws.data_ptr(), sp))
    return best, sweeps, bits


def run_trials(instance: ProblemInstance, config: SolverConfig, seeds, device=None,
               engine: int | None = None) -> TrialBatch:
    """T independent trials of ``config`` (its seed field is replaced by ``seeds``).

    ``engine`` may force ENGINE_CHECKERBOARD_TILED (the HBM-tiled engine, same
    results) for checkerboard kinds; by default the engine follows the kind and
    the torus size.
    """
    start = time.perf_counter()
    seeds_np = np.asarray(seeds, dtype=np.uint64)
    best, sweeps, bits = run_trials_device(instance, config, seeds_np, device=device,
                                           engine=engine)
    out = TrialBatch(instance.n, seeds_np, best.cpu().numpy(), sweeps.cpu().numpy(),
                     bits.cpu().numpy(), 0.0)
    out.wall_time_s = time.perf_counter() - start
    return out


def run_trial(instance: ProblemInstance, config: SolverConfig) -> TrialResult:
    """solvers.py:91-140 on the GPU engine; deterministic in (instance, config)."""
    start = time.perf_counter()
    batch = run_trials(instance, config, [config.seed])
    res = batch.result(0)
    return replace(res, wall_time_s=time.perf_counter() - start)
