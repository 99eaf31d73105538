"""Build libdrs.so (the sm_100a kernels + C ABI) in-tree with nvcc.

    python -m paper_2603_25872_b200._build [--force] [-v]

The sampler translation units are compiled with contraction disabled
(--fmad=false on device, -ffp-contract=off on the host side) because they are
bit-exact restatements of numpy/glibc arithmetic; the few fused multiply-adds
that ARE part of the reference arithmetic (glibc's FMA builds of log1p/exp)
are explicit fma() calls.  The network kernels (tensor-core GEMM etc.) use the
default contraction.
"""

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build", "drs")
LIB = os.path.join(PKG, "libdrs.so")

EXACT = ["--fmad=false", "-Xcompiler", "-ffp-contract=off"]
SOURCES = {                      # source -> extra flags
    "noise.cu": EXACT,
    "chain.cu": EXACT,
    "gm_eps.cu": EXACT,
    "misc.cu": EXACT,
    "metrics.cu": EXACT,
    "perturb.cu": EXACT,
    "gemm_tc.cu": [],
    "net_ops.cu": [],
    "attn_tc.cu": [],
}
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def _flags():
    return ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-I", INCLUDE, "-I", CSRC]


def _deps():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + \
           [os.path.join(INCLUDE, f) for f in os.listdir(INCLUDE)]


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    newest_dep = max(os.path.getmtime(p) for p in _deps())
    objs, cmds = [], []
    for src, extra in SOURCES.items():
        s = os.path.join(CSRC, src)
        if not os.path.exists(s):
            continue
        o = os.path.join(BUILD, src + ".o")
        objs.append(o)
        if not force and os.path.exists(o) and os.path.getmtime(o) >= newest_dep:
            continue
        cmds.append([nvcc()] + _flags() + extra + ["-c", s, "-o", o])
    # translation units compile in parallel (the GEMM / attention TUs dominate)
    procs = []
    for cmd in cmds:
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((cmd, subprocess.Popen(cmd)))
    failed = [cmd for cmd, p in procs if p.wait() != 0]
    if failed:
        raise subprocess.CalledProcessError(1, failed[0])
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [nvcc()] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
