"""Build liblb.so (the C-ABI library) in-tree with nvcc for sm_100a.

One object per translation unit (compiled in parallel), linked into one shared library.  Each
kernel header (csrc/k_*.cuh) is included by exactly one unit, so every kernel is instantiated once.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "liblb.so")
UNITS = ["lb_core", "lb_spmv", "lb_plan", "lb_host", "lb_multi", "lb_spmm", "lb_sssp"]
SOURCES = [os.path.join(CSRC, u + ".cu") for u in UNITS]
OBJDIR = os.path.join(PKG, "build")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
              "--expt-relaxed-constexpr"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.exists(c) or c == "nvcc"):
            return c
    raise RuntimeError("nvcc not found")


def deps() -> list[str]:
    return SOURCES + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        [os.path.join(ROOT, "include", "lb.h"), os.path.abspath(__file__)]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in deps())


def _compile(src: str, extra: list[str]) -> tuple[str, str]:
    obj = os.path.join(OBJDIR, os.path.basename(src).replace(".cu", ".o"))
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-c", "-o", obj, src]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed on {os.path.basename(src)}:\n{r.stdout}{r.stderr}")
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False, out: str = LIB, extra: list[str] | None = None) -> str:
    """Compile every unit for sm_100a and link `out`.  `extra`: additional nvcc flags (e.g. -D switches
    for diagnostic builds written to another path)."""
    if not force and out == LIB and not extra and not needs_build():
        return out
    os.makedirs(OBJDIR, exist_ok=True)
    extra = list(extra or [])
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(lambda s: _compile(s, extra), SOURCES))
    objs = [o for o, _ in results]
    r = subprocess.run([nvcc(), *ARCH, "-shared", "-o", out, *objs, "-ldl"], capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking liblb.so")
    info = "".join(log for _, log in results)
    if out == LIB:
        with open(os.path.join(PKG, "ptxas_info.txt"), "w") as f:
            f.write(info)
    if verbose:
        sys.stderr.write(info)
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="--verbose" in sys.argv)
    print(LIB)
