"""Build librelax_q4.so in-tree with nvcc for sm_100a (B200 only).

    python -m paper_2311_02103_b200.build [--force] [--verbose] [--experiments]

--experiments builds a separate library, build_exp/librelax_q4_exp.so, with
RQ4_EXPERIMENTS defined (csrc/knobs.h): RELAX_Q4_* environment overrides,
per-CTA timelines, and the measured-slower decode variants of
experiments/csrc.  Tools load it through RELAX_Q4_LIB; the product library
reads no environment variable.

Objects go to build/ (git-ignored); the shared library lands next to this
file so it travels with the repo snapshot to the GPU box.  The CUDA runtime
is linked statically and the driver API (cuTensorMapEncodeTiled) is reached
through cudaGetDriverEntryPoint, so the library loads on a machine without a
GPU driver (its entry points then report RELAX_ERR_DEVICE).
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(PKG, "librelax_q4.so")

SOURCES = ["abi.cpp", "device.cpp", "gemv.cu", "gemv_stream.cu", "smalln_mma.cu", "gemm_tc.cu", "gemm_tc_persist.cu", "fused.cu", "repack.cu", "attention.cu"]
HEADERS = ["internal.h", "ptx.cuh", "q4_unpack.cuh", "fusion.cuh", "knobs.h", "decode_math.cuh"]
EXP_DIR = os.path.join(ROOT, "experiments", "csrc")
EXP_SOURCES = ["gemv_mma.cu", "gemv_row.cu", "decode_chain.cu"]
BUILD_EXP = os.path.join(ROOT, "build_exp")
LIB_EXP = os.path.join(BUILD_EXP, "librelax_q4_exp.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    p = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    return p


def _flags(extra=()):
    dbg = ["-DRQ4_DEBUG_HANG"] if os.environ.get("RELAX_Q4_DEBUG") == "1" else []
    return [*ARCH, *dbg, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
            "-Xcompiler", "-fvisibility=hidden", "-I", INCLUDE, "-I", CSRC,
            "--expt-relaxed-constexpr", *extra]


def _stale(target, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _flag_changed(obj) -> bool:
    """Rebuild when the debug switch differs from the one the object was built with."""
    log = obj + ".log"
    want = os.environ.get("RELAX_Q4_DEBUG") == "1"
    if not os.path.exists(log):
        return True
    with open(log) as f:
        first = f.readline()
    return ("-DRQ4_DEBUG_HANG" in first) != want


def build(force: bool = False, verbose: bool = False, experiments: bool = False) -> str:
    bdir = BUILD_EXP if experiments else BUILD
    lib = LIB_EXP if experiments else LIB
    os.makedirs(bdir, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INCLUDE, "relax_q4.h")]
    srcs = [os.path.join(CSRC, f) for f in SOURCES]
    if experiments:
        srcs += [os.path.join(EXP_DIR, f) for f in EXP_SOURCES]
    objs, jobs = [], []
    for sp in srcs:
        src = os.path.basename(sp)
        op = os.path.join(bdir, src + ".o")
        objs.append(op)
        if force or _stale(op, [sp, *hdrs, __file__]) or _flag_changed(op):
            extra = ["-Xptxas", "-v"] if src.endswith(".cu") else []
            if experiments:
                extra += ["-DRQ4_EXPERIMENTS"]
            lang = ["-x", "cu"] if src.endswith(".cu") else ["-x", "c++"]
            jobs.append([nvcc(), *_flags(extra), *lang, "-c", sp, "-o", op])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        return cmd, r

    with cf.ThreadPoolExecutor(max_workers=len(jobs) or 1) as ex:
        for cmd, r in ex.map(run, jobs):
            log = os.path.join(bdir, os.path.basename(cmd[-1]) + ".log")
            with open(log, "w") as f:
                f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed: {' '.join(cmd)}")
            if verbose:
                sys.stderr.write(r.stderr)
    if force or jobs or _stale(lib, objs):
        tmp = lib + f".tmp{os.getpid()}"
        cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs,
               "-Xcompiler", "-fvisibility=hidden"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link failed")
        os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--experiments", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose, experiments=a.experiments))
