"""In-tree build of the sm_100a library (libstochinv_b200.so).

    python -m paper_1602_01768_b200.build

engine.cu (kernels + launch logic) is compiled by nvcc for sm_100a only;
driver.cpp (C ABI, drivers, host RngStream) by g++ with the oracle's flags so
host-drawn Gaussian sketches are byte-identical to the oracle's.  The .so lands
in paper_1602_01768_b200/lib/ so it travels to the GPU box with the repo.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "build")
LIB_DIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIB_DIR, "libstochinv_b200.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                     "--expt-relaxed-constexpr"]
CXX_FLAGS = ["-std=gnu++20", "-O3", "-march=x86-64-v3", "-fPIC", "-Wall", "-Wextra", "-DNDEBUG",
             f"-I{CUDA}/include"]

SOURCES_CU = ["engine.cu", "shard.cu"]
SOURCES_CXX = ["driver.cpp", "io.cpp", "shard.cpp"]
# per-source header dependencies (the public C header does not reach engine.cu)
_KERNEL_HDRS = ["common.cuh", "gemm_f64.cuh", "kernels_aux.cuh", "kernels_small.cuh", "kernels_core.cuh",
                "family.cuh", "engine.hpp"]
_HOST_HDRS = ["engine.hpp", "host_rng.hpp", "capi_internal.hpp", "shard.hpp", "../../include/stochinv_b200.h"]
DEPS = {"engine.cu": _KERNEL_HDRS, "shard.cu": ["common.cuh", "engine.hpp"], "driver.cpp": _HOST_HDRS,
        "io.cpp": _HOST_HDRS, "shard.cpp": _HOST_HDRS}
HEADERS = sorted(set(_KERNEL_HDRS + _HOST_HDRS))


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: list[str], log: str | None = None) -> None:
    print(" ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if log is not None:
        with open(log, "w") as f:
            f.write(res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"build step failed: {cmd[0]} (rc={res.returncode})")


def build(force: bool = False) -> str:
    if shutil.which(NVCC) is None and not os.path.exists(NVCC):
        raise RuntimeError(f"nvcc not found at {NVCC}")
    os.makedirs(BUILD, exist_ok=True)
    os.makedirs(LIB_DIR, exist_ok=True)
    objs, jobs = [], []
    for src in SOURCES_CU + SOURCES_CXX:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        deps = [s] + [os.path.normpath(os.path.join(CSRC, h)) for h in DEPS[src]]
        if force or _newer(o, deps):
            if src.endswith(".cu"):
                jobs.append(([NVCC] + NVCC_FLAGS + ["-c", s, "-o", o], os.path.join(BUILD, src + ".ptxas.log")))
            else:
                jobs.append((["g++"] + CXX_FLAGS + ["-c", s, "-o", o], None))
        objs.append(o)
    if jobs:  # the translation units compile in parallel
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(max_workers=len(jobs)) as ex:
            for f in [ex.submit(_run, cmd, log) for cmd, log in jobs]:
                f.result()
    if force or _newer(LIB, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-ldl", f"-Xlinker=-rpath={CUDA}/lib64"])
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
    print(LIB)
