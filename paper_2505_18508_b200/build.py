"""Build libgsb_cuda.so in-tree for sm_100a (nvcc, no JIT cache).

    python -m paper_2505_18508_b200.build [--force]
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libgsb_cuda.so"
INCLUDE = PKG.parent / "include"

SOURCES = ["abi.cu", "checker.cu", "checker_hbm.cu", "checker_cluster.cu", "refexact.cu", "refexact_warp.cu",
           "evaluate.cu", "rscan2.cu", "rscan2_nw1.cu", "rscan2_nw2.cu", "rscan2_nw4.cu", "rscan2_nw7.cu", "rscan2_nw8.cu", "rscan2_nw9.cu", "rscan2_nw13.cu", "rscan_big.cu"]
HEADERS = ["gsb_device.cuh", "gsb_internal.h", "checker_common.cuh", "rscan2_kernel.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
    "--expt-relaxed-constexpr",
    "-Xptxas", "-warn-spills",
] + os.environ.get("GSB_NVCC_FLAGS", "").split()


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or Path(c).exists()):
            return c
    return "nvcc"


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [INCLUDE / "gsb.h"]
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: Path | None = None,
          extra_flags: tuple[str, ...] = ()) -> Path:
    """Compile the library; ``out``/``extra_flags`` build a development variant
    (e.g. -DGSB_RS2_PROF) next to the shipped one without touching it."""
    if out is None and not force and not _stale():
        return LIB
    objdir = PKG / "build" / (out.stem if out is not None else "")
    objdir.mkdir(parents=True, exist_ok=True)
    objs = []
    procs = []
    for s in SOURCES:
        o = objdir / (Path(s).stem + ".o")
        cmd = [nvcc(), *NVCC_FLAGS, *extra_flags, "-I", str(INCLUDE), "-c", str(CSRC / s), "-o", str(o)]
        if verbose:
            print(" ".join(cmd))
        procs.append((subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT), s))
        objs.append(str(o))
    failed = []
    for p, s in procs:
        log, _ = p.communicate()
        if p.returncode != 0:
            failed.append((s, log.decode()))
        elif verbose and log:
            print(log.decode())
    if failed:
        msg = "\n".join(f"--- {s}\n{o}" for s, o in failed)
        raise RuntimeError(f"nvcc failed:\n{msg}")
    target = out if out is not None else LIB
    tmp = target.with_suffix(".so.tmp")
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(tmp),
           *objs, "-Xcompiler", "-fPIC"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    if "--variant" in sys.argv:  # python -m ...build --variant NAME -DFLAG ...
        i = sys.argv.index("--variant")
        vdir = PKG.parent / "build_variants"
        vdir.mkdir(exist_ok=True)
        print(build(out=vdir / f"libgsb_{sys.argv[i + 1]}.so", extra_flags=tuple(sys.argv[i + 2:]),
                    verbose="-v" in sys.argv))
    else:
        build(force="--force" in sys.argv, verbose="-v" in sys.argv)
        print(LIB)
