"""Build libdmas.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo)."""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libdmas.so")
SOURCES = [os.path.join(CSRC, "dmas_kernels.cu"), os.path.join(CSRC, "dmas_envelope_tc.cu"),
           os.path.join(CSRC, "dmas_plan.cpp"), os.path.join(CSRC, "dmas_comm.cpp")]
DEPS = SOURCES + [os.path.join(CSRC, "dmas_kernels.cuh"), os.path.join(CSRC, "dmas_comm.h"),
                  os.path.join(ROOT, "include", "dmas.h")]


def nvcc_path() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def command(out: str = LIB, extra=()) -> list:
    return [
        nvcc_path(), "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
        "-shared", "-Xcompiler", "-fPIC,-ffp-contract=off,-O2", "-Xptxas", "-warn-spills",
        "-I", os.path.join(ROOT, "include"), "-I", CSRC, *extra, "-o", out, *SOURCES,
    ]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every source to an object in parallel (the translation units are independent),
    then link the shared library; same flags as command()."""
    if not force and up_to_date():
        return LIB
    base = command()
    flags = [a for a in base[1:base.index("-o")] if a != "-shared"]
    objdir = os.path.join(PKG, "build")
    os.makedirs(objdir, exist_ok=True)
    procs = []
    headers = [d for d in DEPS if d not in SOURCES]
    for src in SOURCES:
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        if not force and os.path.exists(obj) and all(os.path.getmtime(d) <= os.path.getmtime(obj)
                                                     for d in [src, *headers]):
            procs.append((obj, None))                          # object up to date
            continue
        cmd = [nvcc_path(), *flags, "-c", "-o", obj, src]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((obj, subprocess.Popen(cmd)))
    objs = []
    for obj, pr in procs:
        if pr is not None and pr.wait() != 0:
            raise subprocess.CalledProcessError(pr.returncode, "nvcc " + obj)
        objs.append(obj)
    tmp = LIB + ".tmp"
    link = [nvcc_path(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs, "-ldl"]
    if verbose:
        print(" ".join(link), file=sys.stderr)
    subprocess.run(link, check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
