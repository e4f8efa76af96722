"""Builds the CUDA extension in-tree: paper_1411_1702_b200/libpfsmc_gpu.so.

Every translation unit is compiled for sm_100a only
(``-gencode arch=compute_100a,code=sm_100a``) in parallel, then linked with
the static CUDA runtime. ``--fmad=false`` keeps the device arithmetic in the
reference's evaluation order without FMA contraction (the reference's own
build has none: /root/reference/proj/CMakeLists.txt:7-9), which is what makes
Psi bitwise comparable to the CPU oracle. The propagating kernel units are
compiled a second time as the FAST variant (``-DPFSMC_FAST=1 --fmad=true``,
csrc/variant.cuh) for handles created with PFSMC_GPU_ARITH_FAST.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libpfsmc_gpu.so")
NVCC = os.environ.get("NVCC", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + (["-DPFSMC_SCAN_TRACE"] if os.environ.get("PFSMC_SCAN_TRACE") else []) + ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
                "-diag-suppress", "497", "-Xptxas", "-warn-spills"]
SOURCES = ["sampler.cu", "scan.cu", "shard.cu", "c5.cu", "kernels_decay.cu", "kernels_lv.cu", "kernels_robertson.cu",
           "kernels_chain.cu", "kernels_payload.cu", "kernels_metabolic.cu", "kernels_advdiff.cu", "kernels_advdiff_e1.cu",
           "kernels_advdiff_e3.cu", "kernels_advdiff_e8.cu",
           "experiment.cpp"]  # host-only: the experiment-level drop-in (pfsmc_gpu_experiment.h)
# The performance variant of the propagating kernels (csrc/variant.cuh): the
# same units with FMA contraction and shared reciprocals, selected per handle
# by pfsmc_gpu_config.arithmetic = PFSMC_GPU_ARITH_FAST.
FAST_SOURCES = ["kernels_decay.cu", "kernels_lv.cu", "kernels_robertson.cu", "kernels_chain.cu",
                "kernels_metabolic.cu"]
FAST_FLAGS = [f if f != "--fmad=false" else "--fmad=true" for f in FLAGS] + ["-DPFSMC_FAST=1"]


def _stale(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    deps = [src] + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "pfsmc_gpu.h"))
    deps.append(os.path.join(os.path.dirname(HERE), "include", "pfsmc_gpu_experiment.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str) -> str:
    fast = src.startswith("fast:")
    src = src[5:] if fast else src
    obj = os.path.join(BUILD, os.path.splitext(src)[0] + ("_fast.o" if fast else ".o"))
    path = os.path.join(CSRC, src)
    if _stale(obj, path):
        flags = (FAST_FLAGS if fast else FLAGS) if src.endswith(".cu") else ["-O2", "-std=c++17", "-Xcompiler",
                                                                             "-fPIC"]
        cmd = [NVCC, *flags, "-c", path, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        spills = [ln for ln in r.stderr.splitlines() if "spill" in ln.lower()]
        if spills:
            print(f"[build] {src}: " + "; ".join(sorted(set(spills))[:4]), file=sys.stderr)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    units = SOURCES + ["fast:" + f for f in FAST_SOURCES]
    with ThreadPoolExecutor(max_workers=len(units)) as ex:
        objs = list(ex.map(_compile, units))
    if not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcuda"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    build_plugin(verbose)
    # the C++ drop-in example over include/pfsmc_gpu.hpp (exercised by a GPU test)
    root = os.path.dirname(HERE)
    ex_src = os.path.join(root, "examples", "drop_in_lv.cpp")
    ex_bin = os.path.join(root, "examples", "drop_in_lv")
    if os.path.exists(ex_src) and (not os.path.exists(ex_bin)
                                   or os.path.getmtime(ex_bin) < max(os.path.getmtime(ex_src),
                                                                     os.path.getmtime(LIB))):
        cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(root, "include"), ex_src, "-o", ex_bin,
               "-L", HERE, "-lpfsmc_gpu", "-Wl,-rpath,$ORIGIN/../paper_1411_1702_b200"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"example build failed:\n{r.stderr}")
    if verbose:
        print(f"[build] {LIB}")
    return LIB


PLUGIN_DIR = os.path.join(os.path.dirname(HERE), "examples", "user_model")
PLUGIN_LIB = os.path.join(PLUGIN_DIR, "libuser_models.so")


def build_plugin(verbose: bool = False) -> str:
    """The example model plugin (include/pfsmc_gpu_model.cuh), exact + fast
    units, linked against libpfsmc_gpu.so (its static initialisers register
    the models there)."""
    src = os.path.join(PLUGIN_DIR, "user_models.cu")
    if not os.path.exists(src):
        return ""
    inc = ["-I", os.path.join(os.path.dirname(HERE), "include")]
    objs = []
    for fast in (False, True):
        obj = os.path.join(BUILD, "user_models" + ("_fast.o" if fast else ".o"))
        if _stale(obj, src):
            cmd = [NVCC, *(FAST_FLAGS if fast else FLAGS), *inc, "-c", src, "-o", obj]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"plugin build failed:\n{r.stderr}")
        objs.append(obj)
    if not os.path.exists(PLUGIN_LIB) or any(os.path.getmtime(o) > os.path.getmtime(PLUGIN_LIB) for o in objs + [LIB]):
        cmd = [NVCC, *ARCH, "-shared", "-o", PLUGIN_LIB, *objs, "-L", HERE, "-lpfsmc_gpu",
               "-Xlinker", "-rpath,$ORIGIN/../../paper_1411_1702_b200"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"plugin link failed:\n{r.stderr}")
    if verbose:
        print(f"[build] {PLUGIN_LIB}")
    return PLUGIN_LIB


if __name__ == "__main__":
    build(verbose=True)
