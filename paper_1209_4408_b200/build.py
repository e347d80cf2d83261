"""Builds the native parts of the engine in-tree (they travel to the GPU box
with the gpurun snapshot):

  paper_1209_4408_b200/liblife_gpu.so   -- CUDA kernels + C-ABI (include/life_gpu.h),
                                          sm_100a only, cudart linked statically.
  paper_1209_4408_b200/host/life_host_test  -- C++ host-mirror test driver
                                          (host/life_gpu.hpp over the C-ABI).

`python -m paper_1209_4408_b200.build` or `__graft_entry__.build()`.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "liblife_gpu.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
                     "-Xcompiler", "-fPIC,-O3", "-Xptxas", "-O3"]


def _newer(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return False
    t = os.path.getmtime(target)
    return all(os.path.getmtime(s) <= t for s in sources)


def _sources() -> list[str]:
    files = [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC))
             if f.endswith((".cu", ".cuh", ".h"))]
    return files + [os.path.join(ROOT, "include", "life_gpu.h")]


def build_lib(force: bool = False, verbose: bool = False, out: str = LIB,
              defines: tuple = ()) -> str:
    """Builds the engine library; `defines` (e.g. ("LIFE_FMA_SHIFT",)) build
    experimental kernel variants into another file, selected at run time with
    the LIFE_GPU_LIB environment variable."""
    srcs = _sources()
    if not force and _newer(out, srcs + [os.path.abspath(__file__)]):
        return out
    units = [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith(".cu")]
    cmd = [NVCC, "--threads", "0", *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-shared", "-cudart", "static",
           "-o", out + ".tmp", *units]
    if verbose:
        cmd[1:1] = ["-Xptxas", "-v"]
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(out + ".tmp", out)
    return out


def build_host_test(force: bool = False) -> str:
    src = os.path.join(PKG, "host", "life_host_test.cpp")
    hdr = os.path.join(PKG, "host", "life_gpu.hpp")
    out = os.path.join(PKG, "host", "life_host_test")
    if not os.path.exists(src):
        return ""
    if not force and _newer(out, [src, hdr, LIB]):
        return out
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), "-I",
           os.path.join(PKG, "host"), "-o", out, src, "-L", PKG, "-llife_gpu",
           f"-Wl,-rpath,$ORIGIN/..", "-lpthread"]
    subprocess.run(cmd, check=True)
    return out


def _gxx(out: str, srcs: list[str], deps: list[str], extra: list[str], force: bool) -> str:
    if not force and _newer(out, srcs + deps):
        return out
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), "-I",
           os.path.join(PKG, "host"), "-o", out + ".tmp", *srcs, *extra]
    subprocess.run(cmd, check=True)
    os.replace(out + ".tmp", out)
    return out


HOST = os.path.join(PKG, "host")
HOST_HDRS = [os.path.join(HOST, f) for f in ("life_gpu.hpp", "life_io.hpp", "life_harness.hpp")]


def build_io_lib(force: bool = False) -> str:
    """host/liblife_io.so: extern "C" view of life_io.hpp (host only, no CUDA)."""
    return _gxx(os.path.join(HOST, "liblife_io.so"), [os.path.join(HOST, "life_io_capi.cpp")],
                HOST_HDRS, ["-shared", "-fPIC"], force)


def build_cli(force: bool = False) -> str:
    """host/life-bench-gpu: the reference's life-bench CLI on the GPU engine."""
    return _gxx(os.path.join(HOST, "life-bench-gpu"), [os.path.join(HOST, "life_bench_gpu.cpp")],
                HOST_HDRS + [LIB], ["-L", PKG, "-llife_gpu", "-Wl,-rpath,$ORIGIN/..", "-lpthread"],
                force)


def build(force: bool = False, verbose: bool = False) -> None:
    build_lib(force=force, verbose=verbose)
    build_host_test(force=force)
    build_io_lib(force=force)
    build_cli(force=force)


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
