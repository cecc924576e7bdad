"""Builds the in-tree sm_100a library (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
OBJ_DIR = os.path.join(OUT_DIR, "obj")
LIB = os.path.join(OUT_DIR, "libbabplan_cuda.so")
SOURCES = ["rollout.cu", "rollout_tc.cu", "rollout_tc2.cu", "rollout_tc3.cu", "bound.cu", "search.cu", "synthetic.cu", "gradient.cu", "pool.cu", "host.cu", "diag.cu"]
HEADERS = ["bp_common.cuh", "rollout_common.cuh", "tc_common.cuh", "tc_epilogue.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
         "--expt-relaxed-constexpr"]


def _mtime(p):
    return os.path.getmtime(p) if os.path.exists(p) else -1.0


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ_DIR, exist_ok=True)
    hdr = max(_mtime(os.path.join(CSRC, h)) for h in HEADERS + ["../../include/babplan_cuda.h"])
    jobs = []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(OBJ_DIR, s.replace(".cu", ".o"))
        if force or _mtime(obj) < max(_mtime(src), hdr):
            jobs.append([NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stdout or r.stderr):
            print(r.stdout, r.stderr)

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        list(ex.map(run, jobs))
    objs = [os.path.join(OBJ_DIR, s.replace(".cu", ".o")) for s in SOURCES]
    if force or jobs or _mtime(LIB) < max(_mtime(o) for o in objs):
        run([NVCC, *ARCH, "-shared", "-o", LIB, *objs])
    return LIB


CONSUMER_SRC = os.path.join(os.path.dirname(HERE), "tests", "native", "capi_consumer.cpp")
CONSUMER = os.path.join(os.path.dirname(HERE), "tests", "native", "_capi_consumer")


def build_consumer(force: bool = False) -> str:
    """The compiled C++ consumer of the C-ABI (tests/native/capi_consumer.cpp), linked against the
    in-tree libbabplan_cuda.so with an rpath to it."""
    lib = build()
    if force or _mtime(CONSUMER) < max(_mtime(CONSUMER_SRC), _mtime(lib), _mtime(os.path.join(os.path.dirname(HERE),
                                                                                                 "include", "babplan_cuda.h"))):
        cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-I", os.path.join(os.path.dirname(HERE), "include"), CONSUMER_SRC,
               "-L", OUT_DIR, "-lbabplan_cuda", f"-Wl,-rpath,{OUT_DIR}", "-o", CONSUMER]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"g++ failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return CONSUMER


def build_variant(name: str, defines: list) -> str:
    """Dev helper: the library compiled with extra -D flags into _lib/variant_<name>.so
    (load it with BP_LIB_PATH); the product library is untouched."""
    obj_dir = os.path.join(OBJ_DIR, name)
    os.makedirs(obj_dir, exist_ok=True)
    out = os.path.join(OUT_DIR, f"variant_{name}.so")
    cmds = [[NVCC, *ARCH, *FLAGS, *defines, "-c", os.path.join(CSRC, s), "-o", os.path.join(obj_dir, s.replace(".cu", ".o"))]
            for s in SOURCES]

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        list(ex.map(run, cmds))
    run([NVCC, *ARCH, "-shared", "-o", out, *[os.path.join(obj_dir, s.replace(".cu", ".o")) for s in SOURCES]])
    return out
