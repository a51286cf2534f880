"""Builds libqsim.so in-tree with nvcc for sm_100a (no JIT cache)."""
from __future__ import annotations

import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libqsim.so")
MB_LIB = os.path.join(PKG, "libqsim_mb.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", "-Xptxas", "-v", "--shared",
         "-I", os.path.join(ROOT, "include")]


TARGETS = {
    LIB: (os.path.join(CSRC, "*.cu"), os.path.join(CSRC, "*.h*"), "qsim.h"),
    MB_LIB: (os.path.join(CSRC, "mb", "*.cu"), os.path.join(CSRC, "mb", "*.cuh"), "qsim_mb.h"),
}


def sources(lib):
    cu, cuh, hdr = TARGETS[lib]
    cus = [cu] if isinstance(cu, str) else cu
    return (sorted(sum((glob.glob(c) for c in cus), [])), sorted(glob.glob(cuh)) if cuh else [],
            os.path.join(ROOT, "include", hdr))


def stale(lib) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    cus, cuhs, hdr = sources(lib)
    return any(os.path.getmtime(s) > t for s in cus + cuhs + [hdr])


def build_one(lib, force=False, verbose=False) -> str:
    if not force and not stale(lib):
        return lib
    cus, _, _ = sources(lib)
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [NVCC, *FLAGS, "-o", tmp, *cus, "-ldl"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    log = os.path.join(PKG, "build_ptxas.log" if lib == LIB else "build_ptxas_mb.log")
    with open(log, "w") as f:
        f.write(res.stderr)
    if verbose:
        print(res.stderr)
    os.replace(tmp, lib)
    return lib


def build(force: bool = False, verbose: bool = False) -> str:
    build_one(MB_LIB, force, verbose)
    return build_one(LIB, force, verbose)


if __name__ == "__main__":
    import sys
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
