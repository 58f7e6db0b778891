"""Build libll_b200.so in-tree: nvcc for sm_100a (kernels) + g++ (host core).

    python paper_2505_23819_b200/build.py [--force]      (or __graft_entry__.build())

The shared library lands next to this file so that it travels with the repo
snapshot to the GPU box.  Compilation is incremental on source mtimes.
"""

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
OUT = os.path.join(HERE, "libll_b200.so")
BUILD = os.path.join(HERE, "build")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

CU_SOURCES = ["kernel_smem.cu", "kernel_async.cu", "kernel_tma.cu", "kernel_regs.cu", "kernel_shuffle.cu", "kernel_misc.cu"]
CPP_SOURCES = ["core.cpp", "planner.cpp", "planner_tma.cpp", "planner_regs.cpp", "capi.cpp", "jit.cpp", "gather.cpp"]
HEADERS = ["core.hpp", "plan.hpp", "planner.hpp", "planner_internal.hpp", "kernels.hpp", "device_common.cuh"]


def _mtime(p):
    return os.path.getmtime(p) if os.path.exists(p) else 0.0


def _hdr_mtime():
    hs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "ll.h")]
    return max(_mtime(h) for h in hs)


def _compile(src, force):
    s = os.path.join(CSRC, src)
    o = os.path.join(BUILD, src + ".o")
    if not force and _mtime(o) > max(_mtime(s), _hdr_mtime()):
        return o, None
    if src.endswith(".cu"):
        # LL_NVCC_EXTRA: extra nvcc flags for tuning experiments (e.g. -DLL_UP_MINB=3)
        extra = os.environ.get("LL_NVCC_EXTRA", "").split()
        cmd = [NVCC, "-std=c++17", "-O3", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC",
               "-Xptxas", "-v", *extra, "-c", s, "-o", o]
    else:
        cmd = ["g++", "-std=c++17", "-O2", "-fPIC", "-Wall", "-I", os.path.join(CUDA, "include"),
               "-c", s, "-o", o]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("compile failed: %s\n%s\n%s" % (" ".join(cmd), r.stdout, r.stderr))
    return o, r.stderr


def build(force=False, verbose=False):
    os.makedirs(BUILD, exist_ok=True)
    srcs = CU_SOURCES + CPP_SOURCES
    # stale objects of renamed sources must not be linked
    for f in os.listdir(BUILD):
        if f.endswith(".o") and f[:-2] not in srcs:
            os.remove(os.path.join(BUILD, f))
    with cf.ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        results = list(ex.map(lambda s: _compile(s, force), srcs))
    objs = [o for o, _ in results]
    if verbose:
        for _, log in results:
            if log:
                sys.stderr.write(log)
    if force or not os.path.exists(OUT) or _mtime(OUT) < max(_mtime(o) for o in objs):
        tmp = OUT + ".tmp"
        # NVRTC (jit.cpp): the toolkit's coexistence build (libnvrtc.alt, own soname and
        # symbol versions), so an older libnvrtc.so.12 already loaded by PyTorch
        # does not shadow it; found through the rpath at run time
        lib64 = os.path.join(CUDA, "lib64")
        cmd = [NVCC, "-shared", *ARCH, "-cudart", "static", "-o", tmp, *objs,
               "-L" + lib64, "-lnvrtc.alt", "-Xlinker", "-rpath," + lib64,
               "-Xlinker", "-soname,libll_b200.so"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed: %s\n%s" % (r.stdout, r.stderr))
        os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
