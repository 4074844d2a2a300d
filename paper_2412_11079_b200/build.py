"""Build the sm_100a extension in-tree: paper_2412_11079_b200/libuot_cuda.so.

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3, C-ABI shared
library (include/uot_cuda.h), cudart static, NCCL loaded lazily with dlopen.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
SO = os.path.join(PKG, "libuot_cuda.so")
TRACE_SO = os.path.join(PKG, "libuot_cuda_trace.so")  # phase-timer build for profiling runs
CLI = os.path.join(PKG, "uot-cuda")  # the reference CLI's gen/solve/bench on the C ABI
SOURCES = [os.path.join(CSRC, "uot_cuda.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")] + [
    os.path.join(ROOT, "include", "uot_cuda.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def nvcc_cmd(out: str = SO, extra: list[str] | None = None) -> list[str]:
    return [
        NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
        "-shared", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
        "-Xptxas", "-v", "--expt-relaxed-constexpr", "--compress-mode=size",
        "-I", os.path.join(ROOT, "include"),
        *(extra or []), "-o", out, *SOURCES, "-ldl", "-lpthread",
    ]


def stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or stale():
        cmd = nvcc_cmd()
        r = subprocess.run(cmd, capture_output=True, text=True)
        log = r.stdout + r.stderr
        with open(os.path.join(PKG, "build.log"), "w") as f:
            f.write(" ".join(cmd) + "\n" + log)
        if r.returncode != 0:
            sys.stderr.write(log)
            raise RuntimeError("nvcc failed building libuot_cuda.so (see build.log)")
        if verbose:
            sys.stderr.write(log)
    return SO


def build_cli() -> str:
    """g++ the CLI front end against the C ABI (links libuot_cuda.so, rpath $ORIGIN)."""
    src = os.path.join(CSRC, "uot_cli.cpp")
    if os.path.exists(CLI) and os.path.getmtime(CLI) >= max(os.path.getmtime(src), os.path.getmtime(SO)):
        return CLI
    cmd = ["g++", "-O2", "-std=c++17", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"), "-o", CLI, src,
           "-L", PKG, "-l:libuot_cuda.so", "-Wl,-rpath,$ORIGIN"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("g++ failed building the uot-cuda CLI")
    return CLI


def build_trace() -> str:
    cmd = nvcc_cmd(TRACE_SO, ["-DUOT_TRACE"])
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building the trace build")
    return TRACE_SO


def build_variant(name: str, defines: list[str]) -> str:
    """Experiment builds (phase timers, pipeline-only) next to the product .so."""
    out = os.path.join(PKG, f"libuot_cuda_{name}.so")
    r = subprocess.run(nvcc_cmd(out, [f"-D{d}" for d in defines]), capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed building the {name} variant")
    return out


if __name__ == "__main__":
    if "--trace" in sys.argv:
        build_trace()
    if "--exp" in sys.argv:  # power / pipeline attribution builds (UOT_EXP in sweep.cuh)
        build_variant("exp1", ["UOT_EXP=1"])
        build_variant("exp2", ["UOT_EXP=2"])
    build(force="--force" in sys.argv, verbose="--quiet" not in sys.argv)
    build_cli()
