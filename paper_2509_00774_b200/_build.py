"""Build the in-tree CUDA extension ``libnfgpu.so`` for sm_100a with nvcc.

The library is a plain C-ABI shared object (include/nfgpu.h). It is built in
place so that the .so travels with the repository snapshot to the GPU box.
"""

from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
SRC = PKG / "csrc" / "nfgpu.cu"
HDR = ROOT / "include" / "nfgpu.h"
LIB = PKG / "libnfgpu.so"

NVCC_FLAGS = [
    "-gencode",
    "arch=compute_100a,code=sm_100a",
    "-O3",
    "-lineinfo",
    "-std=c++17",
    "-Xcompiler",
    "-fPIC",
    "-shared",
    "-diag-suppress",
    "177,550",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: cannot build the sm_100a extension")


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in (SRC, HDR))


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return LIB
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), *NVCC_FLAGS, "-o", str(tmp), str(SRC)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stderr}")
    if verbose and res.stderr:
        print(res.stderr)
    os.replace(tmp, LIB)
    build_abi_demo()
    return LIB


DEMO_SRC = ROOT / "examples" / "abi_demo.c"
DEMO_BIN = ROOT / "examples" / "abi_demo"


def build_abi_demo() -> Path | None:
    """Compile examples/abi_demo.c, a plain-C host of the C ABI, against the in-tree library."""
    if not DEMO_SRC.exists():
        return None
    cuda = Path(nvcc()).resolve().parent.parent
    cmd = [shutil.which("gcc") or "gcc", "-O2", "-std=c11", "-o", str(DEMO_BIN), str(DEMO_SRC),
           f"-I{ROOT / 'include'}", f"-I{cuda / 'include'}", f"-L{PKG}", f"-L{cuda / 'lib64'}",
           "-lnfgpu", "-lcudart", "-lm", f"-Wl,-rpath,{PKG}", "-Wl,-rpath,$ORIGIN/../paper_2509_00774_b200"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"gcc failed building {DEMO_SRC.name}:\n{res.stderr}")
    return DEMO_BIN


if __name__ == "__main__":
    print(build(force=True, verbose=True))
