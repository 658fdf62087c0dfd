#!/usr/bin/env python3
"""Benchmark of the sweep hot path (BASELINE.json metric: spin-updates/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c1|c2|c3|c4|c5] [--kind KIND] [--scaling weak|strong]

One *step* = one batched campaign over this rank's trials: T trials x S sweeps
of simulated annealing (default schedule 3.0 -> 0.05, solvers.py:31-32) on the
seeded +-1 torus of the chosen BASELINE config, seeds mix_seed(20250814, i)
(campaign.py:39-53), followed by the best-cut/bitstring reduction (NCCL when
N > 1).  Default config c2 (BASELINE configs[1]: 100x100, 1024 trials x 10000
sweeps); default kind simulated_annealing_random_scan -- the reference's own
dynamics (fresh uniformly random visit order every sweep, solvers.py:107-127)
with Philox draws, whose final-cut distribution agrees with run_trial's.  The
checkerboard kind (systematic colour order: faster, but a different law) and
the bit-exact reference kind are timed on the same config as `secondary`.

--gpus N > 1 without a torchrun environment re-executes this script under
torch.distributed.run with N ranks (one per GPU, NCCL).  --scaling weak: every
rank runs the config's full trial count on its own trial indices; strong: the
config's trial count is split over the ranks (BASELINE configs 3/4 "sharded").

value = updates of all ranks x K / (max over ranks of the summed CUDA-event
step times).  e2e = the same metric through the C ABI host-buffer entry
(gsb_torus_sweep_host: H2D of weights/seeds/table and D2H of every result
inside the timed region).  cpu_baseline / --impl reference = the reference's
algorithm (oracle/ C port of solvers.run_trial, numpy-PCG64 stream,
random-permutation sweeps) on all host cores, bounded sample.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (rows, cols, trials, sweeps)  -- BASELINE.json configs[0..4]
    "c1": (50, 100, 100, 1000),
    "c2": (100, 100, 1024, 10_000),
    "c3": (100, 140, 4096, 20_000),
    "c4": (100, 200, 8192, 50_000),
    # configs[4]: beyond one SM -> the large-torus random-scan engine (planes in global
    # memory, 8 trials per cooperative kernel) / the checkerboard cluster engine
    "c5": (2000, 2000, 64, 1000),
}
MASTER = 20250814
L2_BYTES = 126 * 1024 * 1024
DEFAULT_KIND = "simulated_annealing_random_scan"
METRIC = "spin-updates/sec (trials x sweeps x n / s)"


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--kind", default=None)
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak")
    ap.add_argument("--trials", type=int, default=None, help="override the config's trial count")
    ap.add_argument("--sweeps", type=int, default=None, help="override sweeps")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--dry-run", action="store_true",
                    help="rendezvous and print the sharding plan only (no kernels; CPU test hook)")
    a = ap.parse_args(argv)
    if a.kind is None:
        a.kind = DEFAULT_KIND
    return a


def workload(a, world):
    """(rows, cols, trials on this config in total, trials per rank list, sweeps)."""
    from paper_2505_18508_b200.distributed import shard

    rows, cols, T, S = CONFIGS[a.config]
    T = a.trials or T
    S = a.sweeps or S
    if a.scaling == "strong":
        per_rank = [shard(T, world, r) for r in range(world)]  # (first, count)
        total = T
    else:
        per_rank = [(r * T, T) for r in range(world)]
        total = T * world
    return rows, cols, total, per_rank, S


def config_dict(a, world):
    """The `config` object of the JSON line -- the same for both arms."""
    rows, cols, total, per_rank, S = workload(a, world)
    return {
        "workload": f"{a.config}: torus {rows}x{cols} seed 1, {a.kind}, {total} trials x {S} "
                    f"sweeps, SA 3.0->0.05, master seed {MASTER}",
        "kind": a.kind, "trials": total, "trials_per_gpu": per_rank[0][1], "sweeps": S,
        "n": rows * cols,
        "parallelism": f"trials sharded over {world} GPU(s), {a.scaling} scaling, NCCL "
                       "best-cut/bitstring reduction",
        "l2": "flushed between timed steps (2x126 MiB memset outside the event window)",
    }


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = Path("/tmp") / f"gsb_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sms, maxes, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.path.read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sms.append(float(parts[1]))
                maxes.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        try:
            self.path.unlink()
        except OSError:
            pass
        return {"sm_mhz": statistics.median(sms) if sms else None,
                "sm_max_mhz": max(maxes) if maxes else None,
                "samples": len(sms), "reasons": sorted(reasons)}


# ---------------------------------------------------------------- CPU baselines
def cpu_port_rate(rows, cols, sweeps, seconds_target, threads=None):
    """Reference algorithm (oracle C port of solvers.run_trial) on host cores.

    Bounded sample: `threads` trials (or a multiple of it) x the FULL sweep
    schedule when that fits the time target, otherwise a prefix of the sweeps
    is timed (rate only).
    """
    from oracle import oracle as O

    O.build()
    threads = threads or os.cpu_count()
    n = rows * cols
    w = O.torus_weights(rows, cols, 1)
    eu, ev, ew = O.torus_edges(rows, cols, w)
    # calibrate on one short trial
    t0 = time.perf_counter()
    cal = max(1, min(20, 200_000 // n))  # calibration sweeps: ~0.2 s
    O.run_trials_ref(n, eu, ev, ew, "simulated_annealing", cal, [O.mix_seed(MASTER, 0)], 3.0, 0.05,
                     spins=False, nthreads=1)
    per_upd = (time.perf_counter() - t0) / (cal * n)
    s_budget = max(10, min(sweeps, int(seconds_target / max(per_upd * n, 1e-12))))
    rounds = 1
    if s_budget == sweeps:  # whole schedules fit: as many trial rounds as the target allows
        rounds = max(1, min(16, int(seconds_target / max(per_upd * n * sweeps, 1e-12))))
    seeds = [O.mix_seed(MASTER, i) for i in range(threads * rounds)]
    t0 = time.perf_counter()
    _, _, se = O.run_trials_ref(n, eu, ev, ew, "simulated_annealing", s_budget, seeds, 3.0, 0.05,
                                spins=False, nthreads=threads)
    dt = time.perf_counter() - t0
    upd = int(se.sum()) * n
    sample = (f"{threads * rounds} trials x {s_budget} sweeps of reference SA (PCG64 + permutation, "
              f"schedule 3.0->0.05 over {s_budget} sweeps) on torus {rows}x{cols}:1, "
              f"{threads} host threads")
    return upd / dt, threads, sample, dt


def _py_ref_trial(args):
    src, rows, cols, sweeps, seed = args
    sys.path.insert(0, src)
    from gsetbench.instances import TorusSpec, generate_torus
    from gsetbench.solvers import default_config, run_trial

    inst = generate_torus(TorusSpec(rows, cols, 1))
    t0 = time.perf_counter()
    res = run_trial(inst, default_config("simulated_annealing", sweeps, seed))
    return res.sweeps_executed, time.perf_counter() - t0


def python_reference_rate(rows, cols, seconds_target=8.0):
    """The unmodified Python reference (baseline/_ref copy of gsetbench, made by
    __graft_entry__.build()) on all host cores: ProcessPoolExecutor(P), one
    run_trial per process, sweeps bounded to ~seconds_target.
    Returns None when the copy is absent, and beyond 10^5 sites (config 5: the
    reference builds 8e6 edges as Python objects in each of the P processes --
    minutes and tens of GB before the first sweep; the C port stands alone there)."""
    src = ROOT / "baseline" / "_ref" / "pkg" / "src"
    if not (src / "gsetbench" / "solvers.py").exists() or rows * cols > 100_000:
        return None
    from concurrent.futures import ProcessPoolExecutor

    n = rows * cols
    procs = os.cpu_count() or 1
    sweeps = max(2, int(seconds_target * 7.0e5 / n))  # ~7e5 updates/s per core
    from oracle import oracle as O

    jobs = [(str(src), rows, cols, sweeps, O.mix_seed(MASTER, i)) for i in range(procs)]
    t0 = time.perf_counter()
    with ProcessPoolExecutor(procs) as ex:
        done = list(ex.map(_py_ref_trial, jobs))
    dt = time.perf_counter() - t0
    upd = sum(d[0] for d in done) * n
    return {"value": upd / dt, "unit": "spin-updates/s", "cores": procs, "kind": "reference",
            "seconds": round(dt, 2),
            "trial_seconds_median": round(statistics.median(d[1] for d in done), 2),
            "sample": f"{procs} processes x 1 gsetbench.solvers.run_trial (unmodified Python "
                      f"reference), simulated_annealing, {sweeps} sweeps (schedule 3.0->0.05 "
                      f"compressed), torus {rows}x{cols}:1; wall time includes process start "
                      "and instance construction"}


def cpu_model():
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------- reference arm
def run_reference_arm(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    world = int(os.environ.get("WORLD_SIZE", str(a.gpus)))
    rows, cols, _, _, S = workload(a, world)
    rates, secs = [], []
    for i in range(a.warmup + a.steps):
        rate, cores, sample, dt = cpu_port_rate(rows, cols, S, max(a.cpu_seconds / 2, 4.0))
        if i >= a.warmup:
            rates.append(rate)
            secs.append(dt)
    v = statistics.median(rates)
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": v, "unit": "spin-updates/s", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "higher_is_better": True, "scaling": a.scaling,
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": config_dict(a, world),
        "reference_kind": "simulated_annealing: run_trial's own dynamics (solvers.py:91-140), C "
                          "port on host cores; the same law as the random-scan kind",
        "cpu_baseline": {"value": v, "unit": "spin-updates/s", "cores": cores, "kind": "port",
                         "sample": sample, "cpu": cpu_model()},
        "e2e": {"value": v, "unit": "spin-updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        # one step = one bounded sample of the workload (whole schedules on all cores)
        "ms_per_step": 1e3 * statistics.median(secs),
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- launcher
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch_under_torchrun(a):
    """--gpus N > 1 outside torchrun: start N ranks of this script (one per GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={a.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


# ---------------------------------------------------------------- our arm
def main(argv=None):
    a = parse(argv)
    in_torchrun = "WORLD_SIZE" in os.environ and "MASTER_ADDR" in os.environ
    if a.gpus > 1 and not in_torchrun:
        return relaunch_under_torchrun(a)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != a.gpus:
        print(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    if a.impl == "reference":
        return run_reference_arm(a)

    import numpy as np
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # development only: GSB_BENCH_SHARE_GPU=1 puts every rank on cuda:0 and uses
    # gloo, to exercise the multi-rank path on a one-GPU box (ranks never wait
    # on each other inside a kernel); measurements use one GPU per rank + NCCL
    share = os.environ.get("GSB_BENCH_SHARE_GPU") == "1"
    rows, cols, total, per_rank, S = workload(a, world)
    first, T = per_rank[rank]
    n = rows * cols

    if a.dry_run:  # rendezvous + plan, no CUDA
        if in_torchrun:
            dist.init_process_group("gloo")
            t = torch.tensor([T], dtype=torch.int64)
            dist.all_reduce(t)
            assert int(t[0]) == total
        if rank == 0:
            print(json.dumps({"dry_run": True, "n_gpus": world, "scaling": a.scaling,
                              "config": config_dict(a, world),
                              "shards": [list(x) for x in per_rank]}), flush=True)
        if in_torchrun:
            dist.destroy_process_group()
        return 0

    from paper_2505_18508_b200 import TorusSpec, _lib, generate_torus
    from paper_2505_18508_b200.campaign import mix_seeds
    from paper_2505_18508_b200.distributed import reduce_best as reduce_best_dist
    from paper_2505_18508_b200.solvers import (CHECKERBOARD_KINDS, RANDOM_SCAN_KINDS,
                                               default_config, rscan_shape, run_trials_device,
                                               schedule_table)

    if not share and torch.cuda.device_count() < (local + 1):
        print(f"bench.py: rank {rank} needs cuda:{local} but only {torch.cuda.device_count()} "
              "device(s) are visible", file=sys.stderr)
        return 2
    if share:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # under torchrun a process group always exists (also at world size 1, so
    # the NCCL collectives of the reduction run on a one-GPU box too)
    if in_torchrun:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    cfg = default_config(a.kind, S, 0)
    kind_code = _lib.GSB_ANNEALING if cfg.annealing else _lib.GSB_GREEDY
    L = _lib.lib()
    inst = generate_torus(TorusSpec(rows, cols, 1))
    w = inst.device_weights(dev)
    seeds_np = mix_seeds(MASTER, range(first, first + T))
    seeds = torch.from_numpy(seeds_np.view(np.int64).copy()).to(dev)
    tab = schedule_table(cfg, 4)
    tab_d = torch.from_numpy(tab.view(np.int64)).to(dev) if tab is not None else None
    ts = _lib.torus_struct(rows, cols, w.data_ptr())
    wsb = L.gsb_torus_workspace_bytes(ts, cfg.engine, S, T)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    best = torch.empty(T, dtype=torch.int64, device=dev)
    sweeps_d = torch.empty(T, dtype=torch.int32, device=dev)
    nbytes = (n + 7) // 8
    bits = torch.empty((T, nbytes), dtype=torch.uint8, device=dev)
    flush = torch.empty(2 * L2_BYTES, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    is_rscan = a.kind in RANDOM_SCAN_KINDS
    # 2 = the torus is beyond the register-resident teams: large-torus engine (rscan_big.cu)
    rscan_large = is_rscan and L.gsb_rscan_fits(rows, cols) == 2
    is_checker = a.kind in CHECKERBOARD_KINDS
    # our kernels per step: [checkerboard: masks + geometry tables +] sweep kernel (large-torus
    # random scan: one cooperative launch per 8 trials) + best-key kernel
    launches_per_step = 4 if is_checker else ((T + 7) // 8 + 1 if rscan_large else 2)

    def sweep_launch():
        _lib.check(L.gsb_torus_sweep(ts, cfg.engine, kind_code, S,
                                     tab_d.data_ptr() if tab_d is not None else None,
                                     seeds.data_ptr(), T, best.data_ptr(), sweeps_d.data_ptr(),
                                     bits.data_ptr(), ws.data_ptr(), wsb, sp))

    def step(ev0=None, ev1=None, kev=None):
        if ev0 is not None:
            ev0.record(stream)
        sweep_launch()
        if kev is not None:
            kev.record(stream)
        # campaign-wide best: key kernel, NCCL all-reduce MAX, owner broadcasts
        # the winning bitstring (paper_2505_18508_b200.distributed.reduce_best)
        g = reduce_best_dist(best, bits, first, total)
        if ev1 is not None:
            ev1.record(stream)
        return g.best_cut, g.index

    # warm-up (also validates the integrity guard once)
    for _ in range(max(a.warmup, 0)):
        step()
    _lib.check(L.gsb_workspace_status(ws.data_ptr(), sp))
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    if in_torchrun:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    wall0 = time.perf_counter()
    step_ms, kern_ms = [], []
    for _ in range(a.steps):
        flush.zero_()  # L2 flush between timed steps (outside the event window)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        ek = torch.cuda.Event(enable_timing=True)
        best_cut_global, win_idx = step(e0, e1, ek)
        torch.cuda.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        kern_ms.append(e0.elapsed_time(ek))
    if in_torchrun:
        dist.barrier()
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    clk = clocks.stop()
    _lib.check(L.gsb_workspace_status(ws.data_ptr(), sp))

    # updates of one step: SA always runs S sweeps; greedy stops early (solvers.py:128-131)
    upd_rank = int(sweeps_d.sum().item()) * n if not cfg.annealing else T * S * n
    tot_ms = sum(step_ms)
    tot_kern = sum(kern_ms)
    upd_all = upd_rank
    if in_torchrun:
        cpu_or_dev = torch.device("cpu") if share else dev
        t = torch.tensor([tot_ms, tot_kern], dtype=torch.float64, device=cpu_or_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms, tot_kern = float(t[0]), float(t[1])
        u = torch.tensor([upd_rank], dtype=torch.int64, device=cpu_or_dev)
        dist.all_reduce(u)
        upd_all = int(u[0])
    value = upd_all * a.steps / (tot_ms / 1e3)
    kernel_rate = upd_rank / (tot_kern / a.steps / 1e3)  # this GPU's sweep launch alone

    # ---- e2e through the C ABI host-buffer entry (pinned host memory)
    e2e = None
    if not a.no_e2e:
        w_h = torch.from_numpy(inst.torus_weights.copy()).pin_memory()
        s_h = torch.from_numpy(seeds_np.view(np.int64).copy()).pin_memory()
        bc_h = torch.empty(T, dtype=torch.int64).pin_memory()
        se_h = torch.empty(T, dtype=torch.int32).pin_memory()
        bits_h = torch.empty((T, nbytes), dtype=torch.uint8).pin_memory()
        t0c = cfg.temp_start or 0.0
        t1c = cfg.temp_end or 0.0

        def host_call():
            _lib.check(L.gsb_torus_sweep_host(rows, cols, w_h.data_ptr(), cfg.engine, kind_code, S,
                                              t0c, t1c, s_h.data_ptr(), T, bc_h.data_ptr(),
                                              se_h.data_ptr(), bits_h.data_ptr(), sp))

        host_call()
        if in_torchrun:
            dist.barrier()
        e2e_s = []
        for _ in range(a.steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            host_call()
            e2e_s.append(time.perf_counter() - t0)
        tot_e2e = sum(e2e_s)
        if in_torchrun:
            t = torch.tensor([tot_e2e], dtype=torch.float64,
                             device=torch.device("cpu") if share else dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            tot_e2e = float(t[0])
        assert np.array_equal(bc_h.numpy(), best.cpu().numpy()), "e2e results differ"
        h2d = 2 * n + 8 * T + (tab.nbytes if tab is not None else 0)
        d2h = 8 * T + 4 * T + T * nbytes
        e2e = {"value": upd_all * a.steps / tot_e2e, "unit": "spin-updates/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": tot_e2e / a.steps * 1e3,
               "step_ms": [round(x * 1e3, 3) for x in e2e_s],
               "api": "gsb_torus_sweep_host (include/gsb.h)"}

    # ---- Philox blocks the contract required in one step, and this GPU's
    # pure Philox4x32-10 block rate (live microbenchmark) -> int roofline
    blocks_per_step = None
    unit_def = None
    rs_stats = None
    if is_checker:
        blocks = np.zeros(1, dtype=np.uint64)
        _lib.check(L.gsb_workspace_counters(ws.data_ptr(), sp, blocks.ctypes.data))
        blocks_per_step = int(blocks[0])
        unit_def = ("Philox4x32-10 blocks the checkerboard contract requires (2 init + 8 planes "
                    "per word and half-sweep + per-site tail groups), counted by the kernel")
    elif is_rscan and not rscan_large:
        st = np.zeros(4, dtype=np.uint64)
        _lib.check(L.gsb_workspace_rscan_stats(ws.data_ptr(), sp, st.ctypes.data))
        words = rows * ((cols + 31) // 32)
        per_sweep = 4 if cfg.annealing else 2
        sweeps_run = int(sweeps_d.sum().item())
        blocks_per_step = T * words + words * per_sweep * sweeps_run + int(st[3])
        unit_def = ("Philox4x32-10 blocks the random-scan contract requires: 1 per 32-site word "
                    "for the initial spins, 4 per word and sweep (8 priority planes + 8 "
                    "acceptance planes), 1 per top-byte tie (counted by the kernel)")
        rs_stats = {"rounds_per_sweep": float(st[0]) / max(sweeps_run, 1),
                    "best_tracking_sweeps_frac": float(st[1]) / max(sweeps_run, 1),
                    "candidate_buckets_per_sweep": float(st[2]) / max(sweeps_run, 1),
                    "ties_per_sweep": float(st[3]) / max(sweeps_run, 1)}
    sink = torch.zeros(256, dtype=torch.int32, device=dev)
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    nthr = nsm * 8 * 256
    bpt = 4096
    _lib.check(L.gsb_philox_bench(64, sink.data_ptr(), sp))
    torch.cuda.synchronize()
    pe0 = torch.cuda.Event(enable_timing=True)
    pe1 = torch.cuda.Event(enable_timing=True)
    pe0.record(stream)
    _lib.check(L.gsb_philox_bench(bpt, sink.data_ptr(), sp))
    pe1.record(stream)
    torch.cuda.synchronize()
    philox_peak = nthr * bpt / (pe0.elapsed_time(pe1) / 1e3)  # blocks/s
    lpt = 1 << 17
    _lib.check(L.gsb_lop3_bench(1024, sink.data_ptr(), sp))
    torch.cuda.synchronize()
    pe0.record(stream)
    _lib.check(L.gsb_lop3_bench(lpt, sink.data_ptr(), sp))
    pe1.record(stream)
    torch.cuda.synchronize()
    lop3_peak = nthr * lpt / (pe0.elapsed_time(pe1) / 1e3)  # LOP3 (thread ops)/s

    # ---- roofline of the dominant kernel (the sweep kernel of this torus)
    if rscan_large:
        sweep_kernel = "gsb::rscan_big_kernel"
    elif is_rscan:
        sweep_kernel = "gsb::rscan2_kernel"
    elif is_checker:
        sweep_kernel = ("gsb::checker_sweep_kernel" if (cols // 2 + 31) // 32 * rows <= 2048
                        else "gsb::checker_cluster_kernel")
    else:
        sweep_kernel = "gsb::ref_warp_kernel"
    peaks = {}
    try:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except (OSError, ValueError):
        pass
    f_max = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    smem_peak = nsm * 128 * f_max  # B/s, 128 B/clk/SM crossbar
    b_alg = 1.25  # bit-packed 5-point stencil: 10 bits per update
    achieved_bw = kernel_rate * b_alg
    launch_s = tot_kern / a.steps / 1e3
    smem = {"unit": "GB/s", "algorithmic_bytes_per_update": b_alg,
            "achieved": achieved_bw / 1e9, "peak": smem_peak / 1e9,
            "frac": achieved_bw / smem_peak,
            "peak_basis": f"{nsm} SMs x 128 B/clk x sm_max {f_max / 1e6:.0f} MHz (computed; "
                          "no measured SMEM peak in MEASURED_PEAKS.json)"}
    if blocks_per_step is not None:
        rng_achieved = blocks_per_step / launch_s
        philox_roof = {
            "unit": "Gblock/s (Philox4x32-10)", "achieved": rng_achieved / 1e9,
            "peak": philox_peak / 1e9, "frac": rng_achieved / philox_peak,
            "algorithmic_units_per_launch": blocks_per_step, "unit_def": unit_def,
            "peak_basis": "measured live: gsb_philox_bench, SMs x 8 x 256 threads, 2 independent "
                          "Philox4x32-10 blocks in flight per thread, CUDA events"}
    if rscan_large:
        # HBM path: compulsory traffic per sweep with bit-packed state,
        # 0.25 + 0.25 / k bytes per update for k co-resident trials sharing the couplings
        k = min(T, 8)
        b_hbm = 0.25 + 0.25 / k
        hbm_peak = float(peaks.get("hbm_gbs", 6454.9)) * 1e9
        roofline = {
            "bound": "hbm", "unit": "GB/s", "achieved": kernel_rate * b_hbm / 1e9,
            "peak": hbm_peak / 1e9, "frac": kernel_rate * b_hbm / hbm_peak, "traffic": None,
            "kernel": sweep_kernel, "algorithmic_bytes_per_update": b_hbm,
            "unit_def": "compulsory bit-packed traffic of the HBM path, 0.25 + 0.25/k B per update "
                        f"(k = {k} trials per cooperative launch share the couplings); the engine "
                        "is bound by grid barriers and L2 latency, not by this roof (DESIGN.md)",
            "peak_basis": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks
                          else "fallback 6454.9 GB/s (B200_PROFILING.md)",
            "updates_per_launch": upd_rank, "launch_ms": launch_s * 1e3,
            "updates_per_s": kernel_rate,
        }
    elif is_rscan:
        # ALU-pipe (LOP3/SHF) operations the contract's bit-sliced algorithm needs per
        # 32-site word and sweep:
        #   Philox XOR halves 4 blocks x 16, acceptance compare 8 planes x 2 thresholds x 2,
        #   precedence 2 directions x 8 planes x 2 + 8 plane alignments x 2 + 2,
        #   Delta of the flips 30; per round (ready set, Delta classes, accept, commit) 25
        fixed, per_round = (64 + 32 + 50 + 30, 25) if cfg.annealing else (32 + 50 + 30, 22)
        words = rows * ((cols + 31) // 32)
        sweeps_run = int(sweeps_d.sum().item())
        alu_ops = words * (fixed * sweeps_run + per_round * rs_stats["rounds_per_sweep"] * sweeps_run)
        roofline = {
            "bound": "int", "unit": "Tops/s (ALU-pipe integer thread operations: LOP3/SHF)",
            "achieved": alu_ops / launch_s / 1e12, "peak": lop3_peak / 1e12,
            "frac": alu_ops / launch_s / lop3_peak,
            # DRAM bytes of one launch at config 2 from the committed ncu capture (the
            # planes live in registers / shared memory: HBM sees couplings, seeds, results)
            "traffic": 857344 if (rows, cols, T, S) == (100, 100, 1024, 10000) else None,
            "kernel": sweep_kernel,
            "team_shape": dict(zip(("warps_per_trial", "rows_per_lane"),
                                   rscan_shape(rows, cols, T))),
            "algorithmic_units_per_launch": alu_ops,
            "unit_def": f"{fixed} + {per_round} x rounds ALU-pipe operations per 32-site word and "
                        "sweep: what the contract's level-synchronous bit-sliced algorithm needs "
                        "(Philox XORs, 8-plane comparators, ready sets, Delta classes, commit); "
                        "rounds per sweep counted by the kernel; the kernel's own overheads "
                        "(shuffles, ties, best-so-far, barriers) are not counted",
            "peak_basis": "measured live: gsb_lop3_bench, SMs x 8 x 256 threads, 8 independent "
                          "LOP3 chains per thread, CUDA events (the ALU pipe issues one warp "
                          "instruction per 2 cycles per SM sub-partition)",
            "updates_per_launch": upd_rank, "launch_ms": launch_s * 1e3,
            "updates_per_s": kernel_rate, "philox": philox_roof, "smem": smem,
            # not measured by this run: the committed ncu capture of the same launch
            "ncu_capture": {"file": "profiles/r02_ncu_rscan2_v8_summary.txt",
                            "workload": "config 2, 1024 trials x 10000 sweeps, rscan2_kernel<7,2>",
                            "alu_pipe_active_pct": 63.0, "fma_pipe_active_pct": 18.4,
                            "ipc_per_sm": 2.57, "issue_active_pct": 64.6,
                            "warp_instructions_per_update": 2.11, "dram_bytes": 857344},
        }
    elif blocks_per_step is not None:
        roofline = {
            "bound": "int", "unit": "Gblock/s (Philox4x32-10)",
            "achieved": rng_achieved / 1e9, "peak": philox_peak / 1e9,
            "frac": rng_achieved / philox_peak, "traffic": None,
            "kernel": sweep_kernel,
            "algorithmic_units_per_launch": blocks_per_step,
            "unit_def": unit_def,
            "peak_basis": "measured live: gsb_philox_bench, SMs x 8 x 256 threads, 2 independent "
                          "Philox4x32-10 blocks in flight per thread (uniform key; the fastest "
                          "mix in tools/philox_mb.cu), CUDA events",
            "updates_per_launch": upd_rank, "launch_ms": launch_s * 1e3,
            "updates_per_s": kernel_rate, "smem": smem,
        }
    else:  # the bit-exact engine draws PCG64, not Philox: SMEM figure only
        roofline = {"bound": "smem", "unit": "GB/s", "achieved": smem["achieved"],
                    "peak": smem["peak"], "frac": smem["frac"], "traffic": None,
                    "kernel": sweep_kernel, "updates_per_launch": upd_rank,
                    "launch_ms": launch_s * 1e3, "updates_per_s": kernel_rate,
                    "peak_basis": smem["peak_basis"]}
    if rs_stats is not None:
        roofline["random_scan_counters"] = rs_stats

    # ---- secondary lines, same torus / trials / sweeps / seeds (this GPU):
    # the other two engines, clearly labelled (skipped above 2.5e11 updates:
    # the bit-exact engine would take minutes on configs 3/4)
    secondary = None
    if not a.no_secondary and cfg.annealing and T * S * n <= 2.6e11:
        secondary = {}
        others = [k for k in ("simulated_annealing_checkerboard", "simulated_annealing",
                              "simulated_annealing_random_scan") if k != a.kind]
        if n >= 65536:  # the bit-exact engine runs one thread per trial beyond 2^16 sites
            others = [k for k in others if k != "simulated_annealing"]
        notes = {
            "simulated_annealing_checkerboard":
                "Philox + systematic colour order: NOT the reference's law (final cuts higher "
                "at equal sweeps, DESIGN.md); bit-exact vs its own oracle",
            "simulated_annealing":
                "the reference kind itself: numpy-PCG64 + permutation sweeps, bit-identical "
                "to gsetbench.solvers.run_trial",
            "simulated_annealing_random_scan":
                "Philox + fresh random visit order per sweep: the reference's law",
        }
        for k in others:
            if k in CHECKERBOARD_KINDS and ((rows | cols) & 1):
                continue
            kcfg = default_config(k, S, 0)
            run_trials_device(inst, kcfg, seeds[: min(T, 32)], device=dev)
            torch.cuda.synchronize()
            r0 = torch.cuda.Event(enable_timing=True)
            r1 = torch.cuda.Event(enable_timing=True)
            r0.record(stream)
            run_trials_device(inst, kcfg, seeds, device=dev, check=False)
            r1.record(stream)
            torch.cuda.synchronize()
            rt = r0.elapsed_time(r1) / 1e3
            secondary[k] = {"value": T * S * n / rt, "unit": "spin-updates/s", "ms": rt * 1e3,
                            "workload": f"{k}, torus {rows}x{cols}:1, {T} trials x {S} sweeps "
                                        "(device time, one launch, this GPU)",
                            "note": notes[k]}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:
        rate, cores, sample, dt = cpu_port_rate(rows, cols, S, a.cpu_seconds)
        cpu = {"value": rate, "unit": "spin-updates/s", "cores": cores, "kind": "port",
               "sample": sample, "seconds": round(dt, 2), "cpu": cpu_model()}
        pyref = python_reference_rate(rows, cols)
        if pyref is not None:
            cpu["python_reference"] = pyref

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value, "unit": "spin-updates/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": tot_ms / a.steps, "higher_is_better": True,
            "scaling": a.scaling, "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (seeded +-1 torus, generate_torus weights)",
            "config": config_dict(a, world),
            "per_gpu_value": value / world,
            "best_cut": int(best_cut_global), "best_trial": int(win_idx),
            "wall_s_timed_region": wall,
            "gpu_launches": launches_per_step * a.steps,
            "clocks": clk,
            "roofline": roofline,
            "e2e": e2e,
            "secondary": secondary,
            "cpu_baseline": cpu,
        }
        if share:
            line["development_mode"] = "GSB_BENCH_SHARE_GPU=1: all ranks on cuda:0 over gloo"
        print(json.dumps(line), flush=True)
    if in_torchrun:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
