"""Build libsdp4.so in-tree with nvcc for sm_100a (no JIT cache, travels with gpurun).

    python -m paper_2410_15526_b200.build [--verbose]
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libsdp4.so")
SOURCES = ["sdp4_api.cu", "k_weights.cu", "k_had_quant.cu", "k_reduce.cu", "k_final.cu", "k_fused.cu",
           "k_fused_tlq8.cu", "k_fused_tlq4.cu", "k_local.cu",
           "k_local34.cu"]
HEADERS = ["sdp4_kernels.cuh", "sdp4_device.cuh", "k_fused.cuh", "k_fused_tlq.cuh"]


def nccl_dirs():
    import nvidia.nccl  # torch's bundled NCCL (2.28.x): one libnccl.so.2 per process
    base = os.path.dirname(nvidia.nccl.__file__) if nvidia.nccl.__file__ else list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def needs_rebuild() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "sdp4.h"),
                                                                 os.path.abspath(__file__)]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every source to an object in parallel (one nvcc per translation unit), then link."""
    if not force and not needs_rebuild():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    inc, lib = nccl_dirs()
    flags = [nvcc(), "-O3", "-std=c++17", "-Xcompiler", "-fPIC,-O2,-ffp-contract=off",
             "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "--fmad=false",
             "-I", os.path.join(ROOT, "include"), "-I", inc]
    if verbose:
        flags += ["-Xptxas", "-v"]
    objdir = os.path.join(PKG, "build")
    os.makedirs(objdir, exist_ok=True)

    hdr_t = max(os.path.getmtime(d) for d in [os.path.join(CSRC, f) for f in HEADERS] +
                [os.path.join(ROOT, "include", "sdp4.h"), os.path.abspath(__file__)])

    def compile_one(src):
        obj = os.path.join(objdir, os.path.splitext(src)[0] + ".o")
        if not force and os.path.exists(obj) and os.path.getmtime(obj) > max(hdr_t, os.path.getmtime(
                os.path.join(CSRC, src))):
            return obj     # incremental: object newer than its source and every header
        cmd = flags + ["-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
        if verbose:
            sys.stderr.write(r.stderr)
        return obj

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    cmd = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a"] + objs + \
        ["-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath,{lib}", "-o", LIB + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc link failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--incremental" not in sys.argv, verbose="--verbose" in sys.argv))
