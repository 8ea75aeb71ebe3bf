"""Builds libmglu.so in-tree with nvcc for sm_100a (no torch JIT cache, no site-packages install).

The product is one shared library with a C ABI (include/mglu.h).  It is compiled for
``-gencode arch=compute_100a,code=sm_100a`` only (tcgen05/TMA need the arch-specific target;
no generic PTX is embedded) with ``-lineinfo`` so ncu source pages map to the CUDA sources.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG_DIR)
LIB_PATH = os.path.join(PKG_DIR, "libmglu.so")
CSRC = os.path.join(PKG_DIR, "csrc")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-warn-spills",
]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + [os.path.join(ROOT, "include", "mglu.h")])


def needs_build() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    t = os.path.getmtime(LIB_PATH)
    return any(os.path.getmtime(s) > t for s in _sources())


# kernels on the timed hot path: the build fails if any instantiation of these uses a stack frame
# or local memory (register spills -- the failure mode of P:445-447 at n_m = 8)
HOT_KERNELS = ("gemv_mma_kernel", "gemv_tc_kernel", "gemm_tc_kernel", "router_topk_kernel", "ffn_mma_kernel")


def resource_usage(lib: str) -> dict:
    """{mangled kernel name: {"REG": r, "STACK": s, "LOCAL": l, ...}} from cuobjdump -res-usage."""
    cuobjdump = os.path.join(os.path.dirname(NVCC), "cuobjdump")
    txt = subprocess.run([cuobjdump, "-res-usage", lib], capture_output=True, text=True, check=True).stdout
    usage, fn = {}, None
    for line in txt.splitlines():
        line = line.strip()
        if line.startswith("Function "):
            fn = line[len("Function "):].rstrip(":")
        elif fn and line.startswith("REG:"):
            usage[fn] = {k: int(v) for k, v in (f.split(":") for f in line.split() if ":" in f and f.split(":")[1].isdigit())}
            fn = None
    return usage


def check_no_spills(lib: str) -> list:
    """Hot kernels with a stack frame or local memory (empty list = gate passes)."""
    bad = []
    for fn, u in resource_usage(lib).items():
        if any(k in fn for k in HOT_KERNELS) and (u.get("STACK", 0) or u.get("LOCAL", 0)):
            bad.append((fn, u))
    return bad


def build(force: bool = False, verbose: bool = False, out: str = LIB_PATH, defines=()) -> str:
    """Build the product library (or, with `defines`, an experiment variant at another path:
    experiment builds never overwrite the product .so)."""
    if defines and os.path.abspath(out) == LIB_PATH:
        raise ValueError("experiment builds (-D...) must go to another path than the product library")
    if out == LIB_PATH and not force and not needs_build():
        return LIB_PATH
    tmp = out + f".tmp{os.getpid()}"
    cmd = [NVCC, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-o", tmp, os.path.join(CSRC, "mglu_api.cu")]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd, cwd=ROOT)
    bad = check_no_spills(tmp)
    if bad:
        os.remove(tmp)
        raise RuntimeError("hot kernels use stack/local memory (spills): "
                           + "; ".join(f"{fn} {u}" for fn, u in bad))
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    # python -m paper_2506_23225_b200.build [--force] [--out PATH -DNAME[=V] ...]
    argv = sys.argv[1:]
    out = argv[argv.index("--out") + 1] if "--out" in argv else LIB_PATH
    defs = [a[2:] for a in argv if a.startswith("-D")]
    print(build(force="--force" in argv, verbose=True, out=out, defines=defs))
