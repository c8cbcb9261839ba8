"""Build libchordless.so (the C-ABI library) in-tree with nvcc for sm_100a.

Each translation unit is compiled to an object in parallel (nvcc -c), then linked into one
shared library with the static CUDA runtime."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libchordless.so")
SOURCES = [os.path.join(CSRC, f) for f in ("cc_kernels.cu", "cc_fused.cu", "cc_host.cpp")]
HEADERS = [os.path.join(CSRC, f) for f in ("cc_internal.h", "cc_device.cuh")] + [os.path.join(ROOT, "include", "chordless.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-I", os.path.join(ROOT, "include")]
EXTRA = os.environ.get("CC_NVCC_FLAGS", "").split()  # A/B builds (e.g. -DCC_EB_R=1)


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False, out: str | None = None, extra=()) -> str:
    """Compile every translation unit and link `out` (default: the in-tree libchordless.so).
    `extra` nvcc flags build A/B variants (e.g. ["-DCC_FUSED_MINB=3"], out=...variant.so)."""
    global EXTRA
    lib = out or LIB
    if out or extra:
        force = True
    saved = EXTRA
    EXTRA = EXTRA + list(extra)
    try:
        return _build(force, verbose, lib)
    finally:
        EXTRA = saved


def _build(force: bool, verbose: bool, LIB: str) -> str:
    if force or stale():
        tag = f".tmp{os.getpid()}"
        objs, procs = [], []
        for src in SOURCES:
            obj = os.path.join(CSRC, os.path.basename(src) + tag + ".o")
            cmd = [NVCC, *ARCH, *CFLAGS, *EXTRA, "-c", src, "-o", obj]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            procs.append(subprocess.Popen(cmd))
            objs.append(obj)
        try:
            for p in procs:
                if p.wait() != 0:
                    raise subprocess.CalledProcessError(p.returncode, p.args)
            tmp = LIB + tag
            cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", *objs, "-o", tmp]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            subprocess.check_call(cmd)
            os.replace(tmp, LIB)
        finally:
            for o in objs:
                if os.path.exists(o):
                    os.remove(o)
    return LIB


if __name__ == "__main__":
    # python -m paper_1410_4876_b200.build [--force] [--out path.so] [nvcc flags ...]
    args = sys.argv[1:]
    force = "--force" in args
    out = None
    if "--out" in args:
        out = args[args.index("--out") + 1]
    extra = [a for a in args if a.startswith("-D")]
    print(build(force=force, verbose=True, out=out, extra=extra))
