"""Build libhf.so (hand-written CUDA for sm_100a) in-tree with nvcc.

Every .cu file under csrc/ is compiled with
    -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false
(-fmad=false: no FMA contraction anywhere; every FMA in the kernels is an
explicit __fmaf_rn / fma / DMMA, which the bitwise stage-1 parity needs) and
linked into paper_2208_01907_b200/libhf.so against the NCCL that ships with
torch (same soname, so the process shares one NCCL).
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
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libhf.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    try:
        import nvidia.nccl  # type: ignore
        base = list(nvidia.nccl.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    except Exception:
        pass
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def _flags():
    inc, _ = _nccl_dirs()
    return ARCH + ["-O3", "-lineinfo", "-fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
                   "-DHF_WITH_NCCL", f"-I{inc}", f"-I{os.path.join(ROOT, 'include')}",
                   "-Xptxas", "-warn-spills"]


def _newer(src: str, dst: str, deps) -> bool:
    if not os.path.exists(dst):
        return True
    t = os.path.getmtime(dst)
    return os.path.getmtime(src) > t or any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    deps = sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(ROOT, "include", "hf.h"),
                                                             os.path.abspath(__file__)]
    objs = []
    jobs = []
    for s in srcs:
        o = os.path.join(BUILD, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        if force or _newer(s, o, deps):
            jobs.append([NVCC, *_flags(), "-c", s, "-o", o])
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
            res = list(ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), jobs))
        for c, r in zip(jobs, res):
            if verbose or r.returncode != 0:
                sys.stderr.write(" ".join(c) + "\n" + r.stdout + r.stderr)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed for {c[-3]}")
    # drop stale objects of deleted sources
    for o in glob.glob(os.path.join(BUILD, "*.o")):
        if o not in objs:
            os.remove(o)
    if force or jobs or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        _, libdir = _nccl_dirs()
        cudalib = os.path.join(os.path.dirname(os.path.dirname(NVCC)), "lib64")
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB + ".tmp", *objs, f"-L{libdir}", "-l:libnccl.so.2",
               "-Xlinker", f"-rpath={libdir}", f"-L{cudalib}", "-l:libcublasLt.so.12", "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
            raise RuntimeError("link of libhf.so failed")
        os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
