"""Builds libgss_b200.so (hand-written sm_100a kernels + the C ABI) in-tree with nvcc.

    python -m paper_2212_05271_b200.build [--force] [--jobs N]

The shared library lands in paper_2212_05271_b200/lib/libgss_b200.so (git-ignored;
it travels to the GPU box with the gpurun snapshot).
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import tempfile
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIB_DIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIB_DIR, "libgss_b200.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--use_fast_math=false"]

CU_SOURCES = ["api.cu", "stft_kernels.cu", "wpe_kernels.cu", "wpe_gram_tc.cu", "wpe_apply_tc.cu", "beamform_kernels.cu", "cacgmm_dispatch.cu"] + [
    f"cacgmm_m{m}.cu" for m in range(1, 9)]
CPP_SOURCES = ["host_logic.cpp"]
HEADERS = ["kernels.h", "gss_internal.cuh", "em_layout.cuh", "linalg.cuh", "cacgmm_kernels.cuh", "cacgmm_pass2.cuh", "cacgmm_pass3.cuh",
           "cacgmm_inst.inc", os.path.join("..", "..", "include", "gss_b200.h")]


def _mtime(p):
    return os.path.getmtime(p) if os.path.exists(p) else 0.0


EXTRA_FLAGS: list[str] = []  # tools/variant.py: -D switches of a kernel experiment


def _compile(src):
    obj = os.path.join(OBJ, os.path.splitext(src)[0] + ".o")
    spath = os.path.join(CSRC, src)
    newest = max([_mtime(spath)] + [_mtime(os.path.join(CSRC, h)) for h in HEADERS])
    if _mtime(obj) >= newest:
        return obj, 0, ""
    if src.endswith(".cu"):
        cmd = [NVCC] + ARCH + [f for f in NVCC_FLAGS if not f.startswith("--use_fast_math")] + EXTRA_FLAGS + ["-c", spath, "-o", obj]
    else:
        cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-I/usr/local/cuda/include", "-c", spath, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    return obj, r.returncode, r.stdout + r.stderr


def build_variant(tag: str, flags: list[str], jobs: int | None = None) -> str:
    """Same sources, extra -D flags, separate object dir and library name (lib/libgss_b200_<tag>.so)."""
    global OBJ, LIB, EXTRA_FLAGS
    saved = (OBJ, LIB, EXTRA_FLAGS)
    try:
        # objects of an experiment go to the system scratch directory: they would otherwise travel with every
        # gpurun snapshot (only the library has to)
        obj = os.path.join(tempfile.gettempdir(), "gss_b200_variant_" + tag)
        OBJ, LIB, EXTRA_FLAGS = obj, os.path.join(LIB_DIR, f"libgss_b200_{tag}.so"), list(flags)
        return build(False, jobs)
    finally:
        OBJ, LIB, EXTRA_FLAGS = saved


def build(force: bool = False, jobs: int | None = None, verbose: bool = True) -> str:
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(LIB_DIR, exist_ok=True)
    if force:
        for f in os.listdir(OBJ):
            if os.path.isfile(os.path.join(OBJ, f)):
                os.remove(os.path.join(OBJ, f))
    jobs = jobs or min(8, os.cpu_count() or 1)
    srcs = CU_SOURCES + CPP_SOURCES
    objs = []
    with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
        for obj, rc, log in ex.map(_compile, srcs):
            if rc != 0:
                raise RuntimeError(f"compile failed for {obj}:\n{log}")
            if log.strip() and verbose:
                print(log, file=sys.stderr)
            objs.append(obj)
    if force or _mtime(LIB) < max(_mtime(o) for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n" + r.stdout + r.stderr)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--jobs", type=int, default=None)
    a = ap.parse_args()
    print(build(a.force, a.jobs))
