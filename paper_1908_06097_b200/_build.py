"""Build libsht.so (the C-ABI of include/sht.h) in-tree with nvcc for sm_100a.

Each CUDA source compiles to its own object under build/ (in parallel, and
only when it or a header changed), then nvcc links the shared library next to
this file so it travels with the repo snapshot to the GPU box (gpurun) and is
what ``_lib.load()`` opens.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libsht.so"
OBJ = ROOT / "build" / "obj"
SOURCES = ["sht_plan.cu", "sht_legendre.cu", "sht_fft.cu", "sht_fft_blk.cu", "sht_halo.cu", "sht_gp.cu"]
HEADERS = ["sht_internal.h", "fft_codelets.cuh", "fft_kernels.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_paths() -> tuple[Path, Path]:
    import nvidia.nccl  # torch-bundled NCCL (same image on the GPU box)

    base = Path(list(nvidia.nccl.__path__)[0])
    return base / "include", base / "lib"


def nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def _run(cmd: list[str], verbose: bool) -> None:
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed: " + " ".join(cmd[-3:]))
    if verbose:
        sys.stderr.write(res.stderr)


def build(force: bool = False, verbose: bool = False) -> Path:
    inc, lib = nccl_paths()
    hdrs = [CSRC / h for h in HEADERS if (CSRC / h).exists()] + [ROOT / "include" / "sht.h"]
    newest_hdr = max(h.stat().st_mtime for h in hdrs)
    OBJ.mkdir(parents=True, exist_ok=True)
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
             "-Xptxas", "-v" if verbose else "-O3", f"-I{inc}", f"-I{ROOT / 'include'}"]
    jobs = []
    for s in SOURCES:
        src, obj = CSRC / s, OBJ / (Path(s).stem + ".o")
        if force or not obj.exists() or obj.stat().st_mtime < max(src.stat().st_mtime, newest_hdr):
            jobs.append([nvcc(), *flags, "-c", str(src), "-o", str(obj) + ".tmp"])
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        list(ex.map(lambda c: _run(c, verbose), jobs))
    for c in jobs:
        os.replace(c[-1], c[-1][:-4])
    objs = [OBJ / (Path(s).stem + ".o") for s in SOURCES]
    if jobs or force or not LIB.exists() or LIB.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        _run([nvcc(), *ARCH, "-shared", *[str(o) for o in objs], f"-L{lib}", "-l:libnccl.so.2",
              "-Xlinker", f"-rpath={lib}", "-o", str(LIB) + ".tmp"], verbose)
        os.replace(str(LIB) + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
