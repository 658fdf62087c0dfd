"""The C-ABI library loads, exports every declared symbol, and its host-only
entry points (no GPU needed) behave as the reference does.  CPU only."""

import ctypes
import math
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, golden

HEADER = ROOT / "include" / "gsb.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gsb_[a-z_0-9]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2505_18508_b200 import _lib

    if not _lib.LIB_PATH.exists():
        from paper_2505_18508_b200 import build

        build.build()
    return _lib.lib()


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("gsb_torus_sweep", "gsb_graph_sweep", "gsb_torus_cut_energy", "gsb_schedule_table",
              "gsb_torus_weights", "gsb_mix_seeds", "gsb_torus_sweep_host", "gsb_best_key",
              "gsb_workspace_status", "gsb_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    for s in declared_symbols():
        assert hasattr(lib, s), f"{s} declared in include/gsb.h but not exported"


def test_abi_version_and_no_device(lib):
    assert lib.gsb_abi_version() == 1
    assert lib.gsb_device_count() >= 0


def test_mix_seeds_matches_reference(lib):
    kat = golden("rng_kat.json")["mix_seed"]
    for m, i, v in kat:
        out = np.zeros(1, np.uint64)
        assert lib.gsb_mix_seeds(m, i, 1, out.ctypes.data) == 0
        assert int(out[0]) == v
    out = np.zeros(3, np.uint64)
    lib.gsb_mix_seeds(1234567, 0, 3, out.ctypes.data)
    assert out.tolist() == [6457827717110365317, 3203168211198807973, 9817491932198370423]


def _py_temperature(sweeps, t0, t1, i):  # solvers.py:84-88, verbatim arithmetic
    if sweeps == 1:
        return t0
    frac = i / (sweeps - 1)
    return t0 * (t1 / t0) ** frac


@pytest.mark.parametrize("engine,bits", [(0, 53), (1, 32)])
@pytest.mark.parametrize("sweeps,t0,t1", [(1, 3.0, 0.05), (10, 3.0, 0.05), (997, 2.0, 0.1),
                                          (50_000, 3.0, 0.05)])
def test_schedule_table_equals_python_math(lib, engine, bits, sweeps, t0, t1):
    tab = np.zeros((sweeps, 4), np.uint64)
    assert lib.gsb_schedule_table(engine, sweeps, t0, t1, 4, tab.ctypes.data) == 0
    idx = np.unique(np.linspace(0, sweeps - 1, min(sweeps, 400)).astype(int))
    for i in idx:
        T = _py_temperature(sweeps, t0, t1, int(i))
        for d in range(1, 5):
            p = math.exp(-d / T)
            K = math.ceil(math.ldexp(p, bits))
            assert int(tab[i, d - 1]) == K
            # the threshold compare is the reference's float compare (solvers.py:118)
            for u in (K - 1, K):
                if 0 <= u < 2**bits:
                    assert (u < K) == (u * 2.0 ** -bits < p)


def test_invalid_arguments_map_to_einval(lib):
    tab = np.zeros((3, 4), np.uint64)
    assert lib.gsb_schedule_table(0, 3, 1.0, 2.0, 4, tab.ctypes.data) == -1
    assert b"temp_end" in lib.gsb_last_error()
    assert lib.gsb_schedule_table(7, 3, 3.0, 0.05, 4, tab.ctypes.data) == -1
    assert lib.gsb_torus_weights(2, 5, 1, ctypes.c_void_p(1), None) == -1


def test_python_binding_raises_without_gpu():
    import torch

    from paper_2505_18508_b200 import TorusSpec, generate_torus
    from paper_2505_18508_b200.solvers import default_config, run_trial

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    inst = generate_torus(TorusSpec(4, 4, 1))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        run_trial(inst, default_config("simulated_annealing", 5, 1))
