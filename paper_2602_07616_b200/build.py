"""Build libsere_b200.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

    python -m paper_2602_07616_b200.build [--verbose]

The shared library exports the C-ABI of include/sere_b200.h; the CUDA runtime is
linked statically, so loading it needs no libcudart on the path (only the driver
at call time).
"""

from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libsere_b200.so"
SOURCES = ["capi.cu", "reroute_align.cu", "layout.cu", "grouped_ffn.cu", "router.cu", "ep_p2p.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def needs_rebuild() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "sere_b200.h", Path(__file__)]
    return any(p.stat().st_mtime > t for p in deps if p.exists())


def build(verbose: bool = False, force: bool = False) -> Path:
    if not force and not needs_rebuild():
        return LIB
    cmd = [
        nvcc_path(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
        "-Xcompiler", "-fPIC,-O3", "-shared", "-cudart", "static",
        "-I", str(ROOT / "include"), "-o", str(LIB) + ".tmp",
    ]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    cmd += os.environ.get("SERE_NVCC_FLAGS", "").split()  # experiments only (e.g. -DSERE_MW_GU_MAX=1)
    cmd += [str(CSRC / s) for s in SOURCES]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(str(LIB) + ".tmp", LIB)
    return LIB


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--force", action="store_true")
    a = ap.parse_args()
    print(build(verbose=a.verbose, force=a.force))


if __name__ == "__main__":
    main()
