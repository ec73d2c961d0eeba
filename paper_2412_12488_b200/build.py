"""Builds paper_2412_12488_b200/_lib/libmicrokv.so in-tree (sm_100a).

Host C++20 sources (bookkeeping, C ABI) are compiled with g++; kernels with
nvcc for `-gencode arch=compute_100a,code=sm_100a -lineinfo`; the shared
object links the CUDA runtime statically so it loads with plain ctypes.
Objects are rebuilt only when a source or header is newer.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
CSRC = HERE / "csrc"
OUT_DIR = HERE / "_lib"
OBJ_DIR = OUT_DIR / "obj"
LIB = OUT_DIR / "libmicrokv.so"
INCLUDE = HERE.parent / "include"
CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))

HOST_SRCS = ["radix_tree.cc", "cache.cc", "wire.cc", "frames.cc", "capi.cc"]
CUDA_SRCS = ["kernels.cu", "decode_attn.cu", "decode_pages.cu", "prefill_attn.cu", "crc32.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _headers() -> list[Path]:
    return sorted(CSRC.glob("*.h")) + sorted(CSRC.glob("*.cuh")) + [INCLUDE / "microkv.h"]


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd)}")


def build(verbose: bool = False) -> Path:
    OBJ_DIR.mkdir(parents=True, exist_ok=True)
    nvcc = str(CUDA_HOME / "bin" / "nvcc")
    headers = _headers()
    objs: list[Path] = []
    for src in HOST_SRCS:
        obj = OBJ_DIR / (src + ".o")
        objs.append(obj)
        if _stale(obj, [CSRC / src] + headers):
            _run(["g++", "-O2", "-g", "-std=c++20", "-fPIC", "-Wall", "-Wextra",
                  "-Wno-unused-parameter", f"-I{CUDA_HOME / 'include'}", f"-I{INCLUDE}",
                  *os.environ.get("MKV_CXX_EXTRA", "").split(),
                  "-c", str(CSRC / src), "-o", str(obj)])
    for src in CUDA_SRCS:
        obj = OBJ_DIR / (src + ".o")
        objs.append(obj)
        if _stale(obj, [CSRC / src] + headers):
            _run([nvcc, "-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC",
                  "-Xptxas", "-v" if verbose else "-O3", f"-I{INCLUDE}",
                  *os.environ.get("MKV_NVCC_EXTRA", "").split(),
                  "-c", str(CSRC / src), "-o", str(obj)])
    if _stale(LIB, objs):
        _run([nvcc, "-shared", *ARCH, "-cudart", "static", "-o", str(LIB),
              *[str(o) for o in objs], "-lpthread", "-ldl", "-lrt"])
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
