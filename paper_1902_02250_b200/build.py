"""Builds libkitc.so in-tree with nvcc for sm_100a (no torch import needed)."""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libkitc.so")
# verification build: the same sources with the device-side invariant checks compiled in
# (KITC_CHECKS, csrc/kitc_internal.cuh); loaded only by tests/test_gpu_checks.py via KITC_LIB
CHECKS_LIB = os.path.join(HERE, "libkitc_checks.so")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC,-ffp-contract=off", "-shared"]


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")) +
                  glob.glob(os.path.join(HERE, "csrc", "*.cuh")) +
                  [os.path.join(ROOT, "include", "kitc.h")])


def build_id() -> str:
    """sha256 (16 hex) of the library's sources: ties a profile (profiles/ncu_traffic.json)
    to the build it was captured on."""
    import hashlib
    h = hashlib.sha256()
    for src in sources():
        with open(src, "rb") as f:
            h.update(os.path.basename(src).encode() + b"\0" + f.read())
    return h.hexdigest()[:16]


def stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force: bool = False, verbose: bool = False, checks: bool = False) -> str:
    """libkitc.so (checks=False) or the verification build libkitc_checks.so (checks=True)."""
    lib = CHECKS_LIB if checks else LIB
    if not (force or stale(lib)):
        return lib
    nvcc = os.environ.get("NVCC", "nvcc")
    if not os.path.exists(nvcc) and os.path.exists("/usr/local/cuda/bin/nvcc"):
        nvcc = "/usr/local/cuda/bin/nvcc"
    cus = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))
    objdir = os.path.join(ROOT, "build", "kitc_checks_obj" if checks else "kitc_obj")
    os.makedirs(objdir, exist_ok=True)
    cflags = [f for f in NVCC_FLAGS if f != "-shared"] + (["-DKITC_CHECKS"] if checks else [])
    jobs = []
    for cu in cus:  # one nvcc per translation unit, in parallel (eval.cu dominates)
        obj = os.path.join(objdir, os.path.basename(cu) + ".o")
        cmd = [nvcc, *cflags, "-c", "-o", obj, cu]
        if verbose:
            print(" ".join(cmd))
        jobs.append((subprocess.Popen(cmd), obj))
    objs = []
    for proc, obj in jobs:
        if proc.wait() != 0:
            raise subprocess.CalledProcessError(proc.returncode, "nvcc -c " + obj)
        objs.append(obj)
    tmp = lib + ".tmp"
    link = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs]
    if verbose:
        print(" ".join(link))
    subprocess.check_call(link)
    os.replace(tmp, lib)
    return lib


PROBE_SRC = os.path.join(ROOT, "tools", "fp64_peak.cu")
PROBE_LIB = os.path.join(ROOT, "tools", "libfp64_peak.so")


def build_probe(force: bool = False) -> str:
    """tools/libfp64_peak.so: the DFMA-rate probe bench.py reports beside the derived
    FP64 peak (measurement tool, not part of libkitc)."""
    if not force and os.path.exists(PROBE_LIB) and os.path.getmtime(PROBE_LIB) >= os.path.getmtime(PROBE_SRC):
        return PROBE_LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    if not os.path.exists(nvcc) and os.path.exists("/usr/local/cuda/bin/nvcc"):
        nvcc = "/usr/local/cuda/bin/nvcc"
    subprocess.check_call([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-DKITC_PROBE_LIB",
                           "-Xcompiler", "-fPIC", "-shared", "-o", PROBE_LIB, PROBE_SRC])
    return PROBE_LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
