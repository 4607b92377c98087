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

SOURCES = ["capi.cu", "score.cu", "select.cu", "prefetch.cu", "predict.cu", "shard.cu", "fmodel.cu"]
HEADERS = [
    "pbkv_internal.cuh",
    "common.cuh",
    "chain.cuh",
    os.path.join("host", "radix_mirror.hpp"),
    os.path.join("host", "ops.hpp"),
]

NVCC_FLAGS = [
    "-std=c++20",
    "-O3",
    "-lineinfo",
    "-gencode",
    "arch=compute_100a,code=sm_100a",
    "-Xcompiler",
    "-fPIC",
    "-shared",
    "--expt-relaxed-constexpr",
]


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
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "pbkv.h")]
    if not force and not _stale(LIB, deps):
        return LIB
    cmd = [_nvcc(), *NVCC_FLAGS, "-I" + os.path.join(ROOT, "include"), "-o", LIB + ".tmp", *srcs]
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
        targets += ["ref", "sim"]  # sim_gpu links the product library built above
    subprocess.run(["make", "-s", "-C", odir, *targets], check=True,
                   stdout=None if verbose else subprocess.DEVNULL)


if __name__ == "__main__":
    build_product(force="--force" in sys.argv, verbose=True)
    build_oracle(verbose=True)
    print(LIB)
