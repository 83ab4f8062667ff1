"""Builds the product library lib/libsplat_b200.so (sm_100a) with nvcc, in-tree.

forward.cu is compiled with --fmad=false (bit-exact forward, see csrc/common.cuh); host code
with -ffp-contract=off.  Incremental: objects are rebuilt when their sources/headers change.
"""
from __future__ import annotations

import os
import shutil
import subprocess
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = PKG / "build"
LIB = PKG / "lib" / "libsplat_b200.so"
NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off",
                 f"-I{ROOT / 'include'}", f"-I{CSRC}", "--expt-relaxed-constexpr"]
SOURCES = {
    "forward.cu": ["--fmad=false"],
    "sort.cu": [],
    "backward.cu": [],
    "chain.cu": ["--fmad=false"],
    "binning.cu": [],
    "importance.cu": [],
    "densify.cu": ["--fmad=false"],
    "ssim.cu": ["--fmad=false"],
    "spatial.cu": ["--fmad=false"],
    "comm.cu": [],
    "capi.cu": [],
}
HEADERS = [CSRC / "common.cuh", CSRC / "internal.h", ROOT / "include" / "splat_b200.h",
           ROOT / "include" / "splat_expf.h"]


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def build(verbose: bool = False, force: bool = False, extra_flags=()) -> Path:
    OBJ.mkdir(exist_ok=True)
    LIB.parent.mkdir(exist_ok=True)
    objs, cmds = [], []
    for src, flags in SOURCES.items():
        s = CSRC / src
        o = OBJ / (src + ".o")
        objs.append(o)
        if force or _stale(o, [s, *HEADERS]):
            cmds.append([NVCC, *COMMON, *flags, *extra_flags, "-c", str(s), "-o", str(o)])
    # independent translation units: compile them concurrently
    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as pool:
        for cmd in cmds:
            if verbose:
                print(" ".join(cmd))
        for f in [pool.submit(subprocess.run, cmd, check=True) for cmd in cmds]:
            f.result()
    if force or _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(LIB), *map(str, objs)]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    import sys
    print(build(verbose=True, force="--force" in sys.argv))
