"""Build the product library libhd.so in-tree with nvcc for sm_100a.

Usage: python -m paper_2002_08110_b200.build [--force] [--verbose-ptxas]
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libhd.so")
SOURCES = ["hd_api.cpp", "hd_plan.cpp", "hd_sched.cpp", "hd_tables.cpp", "hd_kernels.cu", "hd_fcl.cu", "hd_basis.cu"]
HEADERS = ["hd_internal.h", "hd_cell.cuh", os.path.join("..", "..", "include", "hd.h")]  # every header the sources include
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    for f in SOURCES + HEADERS + ["../build.py"]:
        p = os.path.normpath(os.path.join(CSRC, f))
        if os.path.exists(p) and os.path.getmtime(p) > t:
            return True
    return False


def build(force: bool = False, verbose_ptxas: bool = False, out: str = LIB, defines=()) -> str:
    """Compile csrc/ into ``out``. ``defines``: extra -D flags (experiments; the product uses none)."""
    if not force and out == LIB and not needs_build():
        return LIB
    objs = []
    bdir = os.path.join(HERE, "build", os.path.splitext(os.path.basename(out))[0])
    os.makedirs(bdir, exist_ok=True)
    for src in SOURCES:
        obj = os.path.join(bdir, src + ".o")
        cmd = [_nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-c",
               os.path.join(CSRC, src), "-o", obj, "-I", os.path.join(ROOT, "include")]
        cmd += [f"-D{x}" for x in defines]
        if verbose_ptxas and src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"]
        subprocess.check_call(cmd)
        objs.append(obj)
    tmp = out + f".tmp{os.getpid()}"
    subprocess.check_call([_nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-lcudart", "-ldl"])
    os.replace(tmp, out)
    return out


def build_all(force: bool = False) -> None:
    """The product library and its HD_DEBUG twin (device-side checks, bench configs only; tests use it),
    compiled concurrently."""
    import threading
    dbg = os.path.join(HERE, "libhd_debug.so")
    errs = []

    def run_debug():
        try:
            if force or not os.path.exists(dbg) or needs_build_of(dbg):
                build(force=True, out=dbg, defines=("HD_DEBUG", "HD_ONLY_BENCH"))
        except Exception as ex:  # noqa: BLE001
            errs.append(ex)
    t = threading.Thread(target=run_debug)
    t.start()
    build(force=force)
    t.join()
    if errs:
        raise errs[0]


def needs_build_of(path: str) -> bool:
    t = os.path.getmtime(path)
    for f in SOURCES + HEADERS + ["../build.py"]:
        p = os.path.normpath(os.path.join(CSRC, f))
        if os.path.exists(p) and os.path.getmtime(p) > t:
            return True
    return False


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv or bool(defs), verbose_ptxas="--verbose-ptxas" in sys.argv,
                out=os.path.join(HERE, outs[0]) if outs else LIB, defines=defs))
