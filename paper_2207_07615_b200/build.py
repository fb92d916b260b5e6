"""Build libplss.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libplss.so")
SOURCES = [os.path.join(HERE, "csrc", "plss.cu")]
DEPS = (glob.glob(os.path.join(HERE, "csrc", "*.cu")) + glob.glob(os.path.join(HERE, "csrc", "*.cuh"))
        + [os.path.join(ROOT, "include", "plss.h")])


def nccl_dir() -> str:
    """torch's bundled NCCL (2.28.x): link against the same libnccl.so.2 torch loads."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations or []) if spec else []:
        d = os.path.join(base, "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("torch-bundled NCCL (site-packages/nvidia/nccl) not found")


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.exists(c) or c == "nvcc"):
            return c
    return "nvcc"


def command(out: str = LIB, extra=()) -> list:
    nc = nccl_dir()
    return [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
            "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v",
            "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nc, "include"),
            *SOURCES, "-o", out, "-L", os.path.join(nc, "lib"), "-l:libnccl.so.2",
            "-Xlinker", "-rpath," + os.path.join(nc, "lib"), *extra]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or needs_build():
        tmp = LIB + ".tmp"
        res = subprocess.run(command(tmp), capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("nvcc failed building libplss.so")
        with open(os.path.join(HERE, "csrc", "ptxas.log"), "w") as f:
            f.write(res.stderr)
        if verbose:
            sys.stderr.write(res.stderr)
        os.replace(tmp, LIB)
    return LIB


def build_variant(name: str, defines: dict) -> str:
    """Tuning variant (e.g. libplss_t2048.so with -DPLSS_TILE=2048), selected at run time through
    the PLSS_LIB environment variable. The default build is libplss.so."""
    out = os.path.join(HERE, f"libplss_{name}.so")
    extra = [f"-D{k}={v}" for k, v in defines.items()]
    res = subprocess.run(command(out, extra), capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stderr)
        raise RuntimeError(f"nvcc failed building {out}")
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
