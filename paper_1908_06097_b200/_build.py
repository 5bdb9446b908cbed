"""Build libsht.so (the C-ABI of include/sht.h) in-tree with nvcc for sm_100a.

The shared library lands next to this file so it travels with the repo
snapshot to the GPU box (gpurun) and is what ``_lib.load()`` opens.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libsht.so"
SOURCES = ["sht_plan.cu", "sht_legendre.cu", "sht_fft.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_paths() -> tuple[Path, Path]:
    import nvidia.nccl  # torch-bundled NCCL (same image on the GPU box)

    base = Path(list(nvidia.nccl.__path__)[0])
    return base / "include", base / "lib"


def nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def build(force: bool = False, verbose: bool = False) -> Path:
    srcs = [CSRC / s for s in SOURCES]
    deps = srcs + [CSRC / "sht_internal.h", ROOT / "include" / "sht.h"]
    if not force and LIB.exists() and LIB.stat().st_mtime >= max(d.stat().st_mtime for d in deps):
        return LIB
    inc, lib = nccl_paths()
    cmd = [
        nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
        "--expt-relaxed-constexpr", "-Xptxas", "-v" if verbose else "-O3",
        f"-I{inc}", f"-I{ROOT / 'include'}",
        *[str(s) for s in srcs],
        f"-L{lib}", "-l:libnccl.so.2", f"-Xlinker", f"-rpath={lib}",
        "-o", str(LIB) + ".tmp",
    ]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libsht.so")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(str(LIB) + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose="-v" in sys.argv)
    print(LIB)
