"""In-tree build of the CUDA library (libwsgpu.so) for sm_100a.

The library is plain nvcc output with a C ABI (include/wiresim_gpu.h); no torch
extension machinery is involved, so the .so is loadable from C, C++ or ctypes.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
BUILD = PKG / "_build"
LIB = PKG / "libwsgpu.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", str(INCLUDE), "-I", str(CSRC),
          "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]

# per-file extra flags: the sampling / fluctuation file keeps the reference's
# fp64 operation order exactly (no FMA contraction)
SOURCES = {
    "ws_sample.cu": ["--fmad=false"],
    "ws_conv.cu": [],
    "ws_conv_tc.cu": [],
    "ws_direct.cu": [],
    "ws_gprof.cu": [],
    "ws_gprof_umma.cu": [],
    "ws_noise.cu": ["--fmad=false"],
    "ws_sigproc.cu": [],
    "ws_api.cu": [],
    "ws_host.cu": ["--fmad=false"],
    "ws_multi.cu": [],
}


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"command failed: {' '.join(cmd)}")
    return r.stdout + r.stderr


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h"))
    objs = []
    for src, extra in SOURCES.items():
        s = CSRC / src
        o = BUILD / (s.stem + ".o")
        if force or _stale(o, [s, *headers, Path(__file__)]):
            out = _run([NVCC, *ARCH, *COMMON, *extra, "-c", str(s), "-o", str(o)] + (["-Xptxas", "-v"] if verbose else []))
            if verbose and out:
                sys.stderr.write(out)
        objs.append(o)
    if force or _stale(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs)])
    return LIB


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    print(LIB)
