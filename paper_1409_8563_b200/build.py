"""Build libparareal.so in-tree with nvcc for sm_100a (B200).

    python -m paper_1409_8563_b200.build
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libparareal.so")
LIB_DEBUG = os.path.join(HERE, "libparareal_debug.so")  # PRK_DEBUG: in-kernel index checks
# PRK_VARIANTS: tuning-history variants and timing diagnostics (select with PR_LIB=<path>)
LIB_VARIANTS = os.path.join(HERE, "libparareal_variants.so")
SRCS = [os.path.join(HERE, "csrc", "parareal.cu")]
DEPS = SRCS + glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + [os.path.join(ROOT, "include", "parareal.h")]


def nccl_dirs():
    """NCCL shipped with torch (the one torch.distributed loads)."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    cands = []
    if spec and spec.submodule_search_locations:
        for loc in spec.submodule_search_locations:
            cands.append(os.path.join(loc, "nccl"))
    for c in cands:
        inc, lib = os.path.join(c, "include"), os.path.join(c, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
            return inc, lib
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def nvcc_cmd(out: str, debug: bool = False, variants: bool = False) -> list[str]:
    inc, lib = nccl_dirs()
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    return [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
            "-std=c++17", "-Xcompiler", "-fPIC,-O2,-ffp-contract=off", "-shared", "-Xptxas", "-v",
            *(["-DPRK_DEBUG"] if debug else []), *(["-DPRK_VARIANTS"] if variants else []),
            "-I", os.path.join(ROOT, "include"), "-I", inc,
            *SRCS, "-o", out, "-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath,{lib}"]


def build(force: bool = False, verbose: bool = False, debug: bool = False, variants: bool = False) -> str:
    lib = LIB_DEBUG if debug else LIB_VARIANTS if variants else LIB
    if not force and os.path.exists(lib) and os.path.getmtime(lib) >= max(os.path.getmtime(d) for d in DEPS):
        return lib
    tmp = lib + f".tmp{os.getpid()}"
    cmd = nvcc_cmd(tmp, debug, variants)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libparareal.so")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    build(force=True, verbose=True)
    print(LIB)
