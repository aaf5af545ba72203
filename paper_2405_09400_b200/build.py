"""In-tree build of libdomdec.so for sm_100a (nvcc, no JIT cache).

Each CUDA source is compiled to its own object in parallel (incremental: an
object is rebuilt when its source or any header is newer), then linked."""
from __future__ import annotations

import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
SOURCES = ["csrc/api.cu", "csrc/sweep.cu", "csrc/sweep_s1.cu", "csrc/sweep_s2.cu", "csrc/sweep_s4.cu",
           "csrc/sweep_s8.cu", "csrc/flow.cu", "csrc/mcf.cu", "csrc/pdgap.cu", "csrc/sinkhorn_global.cu",
           "csrc/multiscale.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC"]
OBJDIR = os.path.join(HERE, "build")


def build_library(force: bool = False, verbose: bool = False) -> str:
    out = os.path.join(HERE, "libdomdec.so")
    srcs = [os.path.join(HERE, s) for s in SOURCES if os.path.exists(os.path.join(HERE, s))]
    hdrs = [os.path.join(HERE, "csrc", f) for f in os.listdir(os.path.join(HERE, "csrc")) if f.endswith(".cuh")]
    hdrs.append(os.path.join(os.path.dirname(HERE), "include", "domdec.h"))
    hdr_t = max(os.path.getmtime(f) for f in hdrs)
    nvcc = os.environ.get("NVCC", "nvcc")
    os.makedirs(OBJDIR, exist_ok=True)

    def obj_of(src):
        return os.path.join(OBJDIR, os.path.splitext(os.path.basename(src))[0] + ".o")

    def compile_one(src):
        obj = obj_of(src)
        if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_t):
            return False
        cmd = [nvcc] + NVCC_FLAGS + ["-c", "-o", obj, src]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True, cwd=HERE)
        return True

    with ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        rebuilt = any(list(ex.map(compile_one, srcs)))
    objs = [obj_of(s) for s in srcs]
    if rebuilt or force or not os.path.exists(out) or os.path.getmtime(out) < max(os.path.getmtime(o) for o in objs):
        cmd = [nvcc] + ARCH + ["-shared", "-o", out] + objs
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True, cwd=HERE)
    return out
