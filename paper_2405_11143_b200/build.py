"""Build liborl.so (sm_100a) in-tree with nvcc.

    python -m paper_2405_11143_b200.build

The library links the NCCL that ships with torch (site-packages/nvidia/nccl),
so torch.distributed and liborl share one libnccl.so.2 in the process.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "liborl.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_root() -> str:
    import nvidia.nccl  # torch's NCCL wheel

    return list(nvidia.nccl.__path__)[0]


def sources():
    return sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(PKG, "csrc", "*.h*"))) + [os.path.join(ROOT, "include", "orl.h")]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in sources() + headers())


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Compile liborl.so.  `defines` (e.g. ["ORL_K1_STAGES=8"]) and `out` build a
    tuning variant under another name (tools/k1_tune.py)."""
    lib = out or LIB
    if not force and not defines and not needs_build():
        return LIB
    nccl = nccl_root()
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-shared",
           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nccl, "include"),
           *sources(), "-L", os.path.join(nccl, "lib"), "-l:libnccl.so.2",
           "-Xlinker", "-rpath", "-Xlinker", os.path.join(nccl, "lib"),
           *[f"-D{d}" for d in defines], "-o", lib + ".tmp"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
