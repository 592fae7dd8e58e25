"""In-tree build of libthermiga_b200.so (sm_100a) with nvcc.

Every .cu/.cpp under csrc/ is compiled with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` and linked into
``paper_2511_20432_b200/_lib/libthermiga_b200.so``; objects are cached under
``build/`` and rebuilt when a source or header is newer.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIBDIR, "libthermiga_b200.so")
OBJDIR = os.path.join(ROOT, "build", "obj")

NVCC = os.environ.get("NVCC", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fno-fast-math",
          "-I", os.path.join(ROOT, "include"), "-I", CSRC]


# files whose arithmetic must round every product and sum separately (the
# host / reference association, no FMA contraction)
NO_FMAD = {"k4_eval.cu", "k6_assemble.cu"}


# the CUDA runtime is linked statically; no CUDA math library is needed
CUDA_LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.realpath(
    __import__("shutil").which(NVCC) or "/usr/local/cuda/bin/nvcc"))), "lib64")
LINK = ["-L" + CUDA_LIB, "-ldl", "-Xlinker", "-rpath=" + CUDA_LIB]


def _sources():
    srcs = sorted(glob.glob(os.path.join(CSRC, "**", "*.cu"), recursive=True))
    srcs += sorted(glob.glob(os.path.join(CSRC, "**", "*.cpp"), recursive=True))
    return srcs


def _headers():
    hs = glob.glob(os.path.join(CSRC, "**", "*.cuh"), recursive=True)
    hs += glob.glob(os.path.join(CSRC, "**", "*.hpp"), recursive=True)
    hs += glob.glob(os.path.join(ROOT, "include", "*.h"))
    hs += glob.glob(os.path.join(ROOT, "include", "*.hpp"))
    return hs


def _obj_for(src):
    rel = os.path.relpath(src, CSRC).replace(os.sep, "__")
    return os.path.join(OBJDIR, rel + ".o")


def _compile(src, verbose):
    obj = _obj_for(src)
    if src.endswith(".cu"):
        extra = ["-fmad=false"] if os.path.basename(src) in NO_FMAD else []
        cmd = [NVCC, *ARCH, *COMMON, *extra, "-Xptxas", "-warn-spills", "-c", src, "-o", obj]
    else:
        # host C++: compiled by the host compiler through nvcc, no FMA contraction
        # (bit-exact setup arithmetic with the reference's x86-64 build)
        cmd = [NVCC, *COMMON, "-Xcompiler", "-ffp-contract=off", "-x", "c++", "-c", src, "-o", obj]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in _sources() + _headers())


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJDIR, exist_ok=True)
    os.makedirs(LIBDIR, exist_ok=True)
    hdr_t = max((os.path.getmtime(h) for h in _headers()), default=0.0)
    todo = []
    for s in _sources():
        o = _obj_for(s)
        if force or not os.path.exists(o) or os.path.getmtime(o) < max(os.path.getmtime(s), hdr_t):
            todo.append(s)
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        list(ex.map(lambda s: _compile(s, verbose), todo))
    objs = [_obj_for(s) for s in _sources()]
    if force or todo or not os.path.exists(LIB):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs, *LINK]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
