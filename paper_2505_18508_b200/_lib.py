"""ctypes binding of libgsb_cuda.so (include/gsb.h).

There is no CPU fallback: if the library is missing or no CUDA device is
visible, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["GSB_LIB"]) if os.environ.get("GSB_LIB") else PKG / "libgsb_cuda.so"

GSB_OK = 0
GSB_EINVAL = -1
GSB_ECUDA = -2
GSB_EINTEGRITY = -3
GSB_ENOMEM = -4
GSB_EUNSUPPORTED = -5

GSB_GREEDY = 0
GSB_ANNEALING = 1
ENGINE_REFERENCE = 0
ENGINE_CHECKERBOARD = 1
ENGINE_CHECKERBOARD_TILED = 2
ENGINE_CHECKERBOARD_CLUSTER = 3
ENGINE_RANDOM_SCAN = 4
ENGINE_RANDOM_SCAN_LARGE = 5

_lock = threading.Lock()
_lib = None


class GsbError(RuntimeError):
    pass


class _Torus(ctypes.Structure):
    _fields_ = [("rows", ctypes.c_int32), ("cols", ctypes.c_int32), ("w_dev", ctypes.c_void_p)]


class _Graph(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("m", ctypes.c_int64), ("eu_dev", ctypes.c_void_p),
                ("ev_dev", ctypes.c_void_p), ("ew_dev", ctypes.c_void_p)]


def lib():
    """Load (once) and return the CDLL; raises if the extension is missing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2505_18508_b200.build` "
                "(the sweep engine has no CPU fallback)")
        L = ctypes.CDLL(str(LIB_PATH))
        P, i32, i64, u64, dbl, sz = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64,
                                     ctypes.c_uint64, ctypes.c_double, ctypes.c_size_t)
        TP = ctypes.POINTER(_Torus)
        GP = ctypes.POINTER(_Graph)
        L.gsb_last_error.restype = ctypes.c_char_p
        L.gsb_abi_version.restype = ctypes.c_int
        L.gsb_device_count.restype = ctypes.c_int
        L.gsb_mix_seeds.argtypes = [u64, i64, i32, P]
        L.gsb_torus_weights.argtypes = [i32, i32, u64, P, P]
        L.gsb_torus_cut_energy.argtypes = [TP, P, i32, P, P, P]
        L.gsb_graph_cut_energy.argtypes = [GP, P, i32, P, P, P]
        L.gsb_schedule_table.argtypes = [ctypes.c_int, i32, dbl, dbl, i32, P]
        L.gsb_torus_workspace_bytes.argtypes = [TP, ctypes.c_int, i32, i32]
        L.gsb_torus_workspace_bytes.restype = sz
        L.gsb_torus_sweep.argtypes = [TP, ctypes.c_int, ctypes.c_int, i32, P, P, i32, P, P, P, P,
                                      sz, P]
        L.gsb_graph_workspace_bytes.argtypes = [GP, i32, i32]
        L.gsb_graph_workspace_bytes.restype = sz
        L.gsb_graph_sweep.argtypes = [GP, ctypes.c_int, i32, P, i32, P, i32, P, P, P, P, sz, P]
        L.gsb_torus_sweep_host.argtypes = [i32, i32, P, ctypes.c_int, ctypes.c_int, i32, dbl, dbl,
                                           P, i32, P, P, P, P]
        L.gsb_workspace_status.argtypes = [P, P]
        L.gsb_rscan_fits.argtypes = [i32, i32]
        L.gsb_workspace_counters.argtypes = [P, P, P]
        L.gsb_workspace_rscan_stats.argtypes = [P, P, P]
        L.gsb_rscan_shape.argtypes = [i32, i32, i32, P, P]
        L.gsb_test_rscan_shape.argtypes = [i32, i32]
        L.gsb_test_checker_shape.argtypes = [i32, i32]
        L.gsb_test_cluster_size.argtypes = [i32]
        L.gsb_test_rscan_limits.argtypes = [i32, i32]
        L.gsb_test_rscan_slices.argtypes = [i32]
        L.gsb_philox_bench.argtypes = [i64, P, P]
        L.gsb_lop3_bench.argtypes = [i64, P, P]
        L.gsb_best_key.argtypes = [P, i32, i64, P, P]
        if L.gsb_abi_version() != 1:
            raise ImportError("libgsb_cuda.so ABI version mismatch; rebuild")
        _lib = L
        return L


def check(rc: int) -> None:
    """Map a gsb return code to the reference's exception types."""
    if rc == GSB_OK:
        return
    msg = lib().gsb_last_error().decode(errors="replace")
    if rc in (GSB_EINVAL, GSB_EUNSUPPORTED):
        raise ValueError(msg)
    if rc == GSB_EINTEGRITY:
        raise RuntimeError(msg)  # solvers.py:132-133
    raise GsbError(f"gsb error {rc}: {msg}")


def torus_struct(rows: int, cols: int, w_dev_ptr: int) -> _Torus:
    return _Torus(rows, cols, w_dev_ptr)


def graph_struct(n, m, eu, ev, ew) -> _Graph:
    return _Graph(n, m, eu, ev, ew)


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device visible: the B200 sweep engine has no CPU fallback")
    lib()
    return torch
