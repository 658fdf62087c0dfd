"""ctypes wrapper of the CPU oracle (oracle/gsb_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline leg, never by the product package.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "build" / "libgsb_oracle.so"

GREEDY, ANNEALING = 0, 1
_KIND = {"greedy_local_search": GREEDY, "simulated_annealing": ANNEALING,
         "greedy_checkerboard": GREEDY, "simulated_annealing_checkerboard": ANNEALING,
         "greedy_random_scan": GREEDY, "simulated_annealing_random_scan": ANNEALING}

_lib = None


def build(force: bool = False) -> Path:
    src = [HERE / "gsb_oracle.c", HERE / "gsb_oracle.h"]
    if force or not LIB.exists() or any(s.stat().st_mtime > LIB.stat().st_mtime for s in src):
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


class _Pcg(ctypes.Structure):
    _fields_ = [("state_hi", ctypes.c_uint64), ("state_lo", ctypes.c_uint64),
                ("inc_hi", ctypes.c_uint64), ("inc_lo", ctypes.c_uint64),
                ("has_uint32", ctypes.c_int), ("uinteger", ctypes.c_uint32)]


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = ctypes.CDLL(str(LIB))
        P = ctypes.c_void_p
        i32, i64, u64, dbl = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
        L.gso_pcg64_seed.argtypes = [ctypes.POINTER(_Pcg), u64]
        L.gso_pcg64_next64.argtypes = [ctypes.POINTER(_Pcg)]
        L.gso_pcg64_next64.restype = u64
        L.gso_pcg64_next32.argtypes = [ctypes.POINTER(_Pcg)]
        L.gso_pcg64_next32.restype = ctypes.c_uint32
        L.gso_pcg64_permutation.argtypes = [ctypes.POINTER(_Pcg), i64, P]
        L.gso_pcg64_random.argtypes = [ctypes.POINTER(_Pcg)]
        L.gso_pcg64_random.restype = dbl
        L.gso_mix_seed.argtypes = [u64, u64]
        L.gso_mix_seed.restype = u64
        L.gso_torus_weights.argtypes = [ctypes.c_int, ctypes.c_int, u64, P]
        L.gso_torus_edges.argtypes = [ctypes.c_int, ctypes.c_int, P, P, P, P]
        L.gso_cut.argtypes = [i64, P, P, P, P]
        L.gso_cut.restype = i64
        L.gso_energy.argtypes = [i64, P, P, P, P]
        L.gso_energy.restype = i64
        L.gso_temperature.argtypes = [ctypes.c_int, dbl, dbl, ctypes.c_int]
        L.gso_temperature.restype = dbl
        L.gso_philox4x32_10.argtypes = [P, P, P]
        L.gso_run_trials_ref.argtypes = [i32, i64, P, P, P, ctypes.c_int, i32, i32, P, dbl, dbl,
                                         P, P, P, ctypes.c_int]
        L.gso_run_trials_rscan.argtypes = [i32, i32, P, ctypes.c_int, i32, i32, P, dbl, dbl,
                                           P, P, P, ctypes.c_int]
        L.gso_run_trials_checker.argtypes = [i32, i32, P, ctypes.c_int, i32, i32, P, dbl, dbl,
                                             P, P, P, ctypes.c_int]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


class Pcg64:
    """numpy default_rng(seed) stream, restated."""

    def __init__(self, seed: int):
        self._s = _Pcg()
        lib().gso_pcg64_seed(ctypes.byref(self._s), seed)

    @property
    def state(self):
        return ((self._s.state_hi << 64) | self._s.state_lo,
                (self._s.inc_hi << 64) | self._s.inc_lo)

    def next64(self):
        return lib().gso_pcg64_next64(ctypes.byref(self._s))

    def next32(self):
        return lib().gso_pcg64_next32(ctypes.byref(self._s))

    def permutation(self, n):
        out = np.empty(n, dtype=np.int64)
        lib().gso_pcg64_permutation(ctypes.byref(self._s), n, _p(out))
        return out

    def random(self):
        return lib().gso_pcg64_random(ctypes.byref(self._s))


def mix_seed(master: int, index: int) -> int:
    return lib().gso_mix_seed(master, index)


def torus_weights(rows: int, cols: int, seed: int) -> np.ndarray:
    w = np.empty(2 * rows * cols, dtype=np.int8)
    lib().gso_torus_weights(rows, cols, seed, _p(w))
    return w


def torus_edges(rows, cols, w):
    m = 2 * rows * cols
    eu = np.empty(m, np.int32)
    ev = np.empty(m, np.int32)
    ew = np.empty(m, np.int64)
    w = np.ascontiguousarray(w, dtype=np.int8)
    lib().gso_torus_edges(rows, cols, _p(w), _p(eu), _p(ev), _p(ew))
    return eu, ev, ew


def cut(eu, ev, ew, spins) -> int:
    s = np.ascontiguousarray(spins, dtype=np.int8)
    return lib().gso_cut(len(eu), _p(eu), _p(ev), _p(ew), _p(s))


def energy(eu, ev, ew, spins) -> int:
    s = np.ascontiguousarray(spins, dtype=np.int8)
    return lib().gso_energy(len(eu), _p(eu), _p(ev), _p(ew), _p(s))


def temperature(sweeps, t0, t1, i) -> float:
    return lib().gso_temperature(sweeps, t0, t1, i)


def philox(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    out = np.empty(4, dtype=np.uint32)
    lib().gso_philox4x32_10(_p(c), _p(k), _p(out))
    return [int(x) for x in out]


def run_trials_ref(n, eu, ev, ew, kind, sweeps, seeds, t0=0.0, t1=0.0, spins=True,
                   nthreads=None):
    """Reference-exact trials on an edge-list graph (solvers.py:91-140)."""
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    T = len(seeds)
    bc = np.empty(T, np.int64)
    se = np.empty(T, np.int32)
    bs = np.empty((T, n), np.int8) if spins else None
    eu = np.ascontiguousarray(eu, np.int32)
    ev = np.ascontiguousarray(ev, np.int32)
    ew = np.ascontiguousarray(ew, np.int64)
    rc = lib().gso_run_trials_ref(n, len(eu), _p(eu), _p(ev), _p(ew), _KIND.get(kind, kind),
                                  sweeps, T, _p(seeds), t0 or 0.0, t1 or 0.0, _p(bc),
                                  _p(bs) if spins else None, _p(se),
                                  nthreads or os.cpu_count())
    if rc:
        raise RuntimeError(f"oracle failed rc={rc}")
    return bc, bs, se


def run_trials_checker(rows, cols, w, kind, sweeps, seeds, t0=0.0, t1=0.0, spins=True,
                       nthreads=None):
    """Checkerboard/Philox trials on a torus (DESIGN.md checkerboard contract)."""
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    T = len(seeds)
    n = rows * cols
    bc = np.empty(T, np.int64)
    se = np.empty(T, np.int32)
    bs = np.empty((T, n), np.int8) if spins else None
    w = np.ascontiguousarray(w, np.int8)
    rc = lib().gso_run_trials_checker(rows, cols, _p(w), _KIND.get(kind, kind), sweeps, T,
                                      _p(seeds), t0 or 0.0, t1 or 0.0, _p(bc),
                                      _p(bs) if spins else None, _p(se),
                                      nthreads or os.cpu_count())
    if rc:
        raise RuntimeError(f"oracle failed rc={rc}")
    return bc, bs, se


def run_trials_rscan(rows, cols, w, kind, sweeps, seeds, t0=0.0, t1=0.0, spins=True,
                     nthreads=None):
    """Random-scan/Philox trials on a torus (DESIGN.md random-scan contract)."""
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    T = len(seeds)
    n = rows * cols
    bc = np.empty(T, np.int64)
    se = np.empty(T, np.int32)
    bs = np.empty((T, n), np.int8) if spins else None
    w = np.ascontiguousarray(w, np.int8)
    rc = lib().gso_run_trials_rscan(rows, cols, _p(w), _KIND.get(kind, kind), sweeps, T,
                                    _p(seeds), t0 or 0.0, t1 or 0.0, _p(bc),
                                    _p(bs) if spins else None, _p(se),
                                    nthreads or os.cpu_count())
    if rc:
        raise RuntimeError(f"oracle failed rc={rc}")
    return bc, bs, se


def encode_hex(spins) -> str:
    """codec.py:64-83 restated: bit i <-> variable i+1, MSB-first, 1 = +1."""
    s = np.asarray(spins)
    bits = (s == 1).astype(np.uint8)
    nd = (len(bits) + 3) // 4
    return np.packbits(bits).tobytes().hex()[:nd]
