"""In-tree build of the native libraries (sm_100a only).

  _native/liblaq_b200.so  CUDA kernels + C-ABI (include/laq_b200.h), nvcc -arch sm_100a
  _native/liblaq_gen.so   host data generator (C++20)

The .so files are git-ignored but travel to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
NATIVE = os.path.join(HERE, "_native")
CSRC = os.path.join(HERE, "csrc")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _run(cmd, cwd=None):
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=cwd)


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build_gen(force=False):
    os.makedirs(NATIVE, exist_ok=True)
    src = os.path.join(CSRC, "gen", "laq_gen.cpp")
    out = os.path.join(NATIVE, "liblaq_gen.so")
    if force or _stale(out, [src]):
        _run(["g++", "-std=c++20", "-O3", "-march=x86-64-v2", "-fPIC", "-shared", "-pthread", src, "-o", out])
    return out


def build_cuda(force=False, verbose=False):
    os.makedirs(NATIVE, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    hdrs = sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
                  + [os.path.join(ROOT, "include", "laq_b200.h")])
    out = os.path.join(NATIVE, "liblaq_b200.so")
    if not (force or _stale(out, srcs + hdrs)):
        return out
    objs, jobs = [], []
    for s in srcs:
        o = os.path.join(NATIVE, os.path.basename(s)[:-3] + ".o")
        if force or _stale(o, [s] + hdrs):
            cmd = [NVCC, *ARCH, "-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC",
                   "-I" + os.path.join(ROOT, "include"), "-I" + CSRC, "--expt-relaxed-constexpr",
                   "-c", s, "-o", o] + os.environ.get("LAQ_NVCC_FLAGS", "").split()
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
            jobs.append(cmd)
        objs.append(o)
    if jobs:
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=max(1, os.cpu_count() or 1)) as ex:
            list(ex.map(_run, jobs))
    _run([NVCC, *ARCH, "-shared", *objs, "-o", out, "-lcudart", "-ldl"])
    return out


def build_oracle():
    """Compile the parity checkers: oracle/ssb_oracle.c always, the reference
    itself only where /root/reference exists (this container)."""
    _run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "checker"])
    if os.path.isdir("/root/reference/proj/src"):
        _run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "oracle")])


def build_integration():
    """The reference's operator API + its own test binaries over the C-ABI
    (integration/Makefile; needs the reference headers, so only here)."""
    if os.path.isdir("/root/reference/proj/src"):
        _run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "integration")])


def build_all(force=False):
    build_gen(force)
    build_cuda(force)
    build_oracle()
    build_integration()


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
