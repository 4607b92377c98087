"""In-tree build of libpbkv.so (sm_100a) and of the test oracle.

The product library is compiled with nvcc for ``-gencode
arch=compute_100a,code=sm_100a`` only; the built ``.so`` lives next to this
file so it travels to the GPU box with the repo snapshot.  The oracle (test
infrastructure, ``oracle/``) is built by its own Makefile.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libpbkv.so")

SOURCES = ["capi.cu", "score.cu", "select.cu", "prefetch.cu", "predict.cu", "shard.cu", "fmodel.cu",
           os.path.join("host", "host_tree.cpp")]
HEADERS = [
    "pbkv_internal.cuh",
    "common.cuh",
    "chain.cuh",
    os.path.join("host", "ops.hpp"),
    os.path.join("host", "internal_abi.h"),
]
# The host trees (host/host_tree.cpp) ARE the reference flowkv::CacheTree:
# its header-only sources are compiled in from the reference tree (never
# copied into this repo).  The GPU box has no /root/reference; it runs the
# library built here.
REF_INCLUDE = "/root/reference/proj/include"

NVCC_FLAGS = [
    "-std=c++20",
    "-O3",
    "-lineinfo",
    "-gencode",
    "arch=compute_100a,code=sm_100a",
    "-Xcompiler",
    "-fPIC",
    "--expt-relaxed-constexpr",
]
LINK_FLAGS = ["-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler", "-fPIC"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build_product(force: bool = False, verbose: bool = False) -> str:
    """Each translation unit compiles to its own object (in parallel, rebuilt
    when it or a shared header changed), then one nvcc link into libpbkv.so."""
    from concurrent.futures import ThreadPoolExecutor

    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    shared = [os.path.join(CSRC, h) for h in HEADERS] + [
        os.path.join(ROOT, "include", "pbkv.h"), os.path.join(ROOT, "include", "pbkv", "tracked_tree.hpp")]
    if not os.path.isdir(REF_INCLUDE):
        if os.path.exists(LIB):
            return LIB  # GPU box: the prebuilt library travelled with the snapshot
        raise RuntimeError(f"libpbkv.so is not built and {REF_INCLUDE} (the CacheTree headers) is absent")
    odir = os.path.join(PKG, "_build")
    os.makedirs(odir, exist_ok=True)
    objs = [os.path.join(odir, os.path.basename(s) + ".o") for s in srcs]
    todo = [(s, o) for s, o in zip(srcs, objs) if force or _stale(o, [s] + shared)]
    inc = ["-I" + os.path.join(ROOT, "include"), "-I" + REF_INCLUDE]

    def compile_one(so):
        src, obj = so
        cmd = [_nvcc(), *NVCC_FLAGS, *inc, "-c", "-o", obj + ".tmp", src]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
        os.replace(obj + ".tmp", obj)

    if todo:
        with ThreadPoolExecutor(max_workers=min(len(todo), os.cpu_count() or 4)) as ex:
            list(ex.map(compile_one, todo))
    if not todo and not force and not _stale(LIB, objs):
        return LIB
    cmd = [_nvcc(), *LINK_FLAGS, "-o", LIB + ".tmp", *objs]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


def build_oracle(verbose: bool = False) -> None:
    """Build the checker: the C restatement always, the reference-compiled
    library only when /root/reference is present (never on the GPU box)."""
    odir = os.path.join(ROOT, "oracle")
    targets = ["oracle"]
    if os.path.isdir("/root/reference/proj/include/flowkv"):
        targets += ["ref", "ref-tests", "sim"]  # sim_gpu links the product library built above;
        # ref-tests: the reference's own Catch2 suite, run by tests/test_oracle.py
    subprocess.run(["make", "-s", "-C", odir, *targets], check=True,
                   stdout=None if verbose else subprocess.DEVNULL)


if __name__ == "__main__":
    build_product(force="--force" in sys.argv, verbose=True)
    build_oracle(verbose=True)
    print(LIB)
