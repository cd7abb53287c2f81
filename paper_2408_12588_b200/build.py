"""Build the native library ``libpab_b200.so`` in-tree for sm_100a.

    python -m paper_2408_12588_b200.build [--verbose]

nvcc cross-compiles without a GPU; the resulting .so travels to the GPU box
with the repo snapshot.  Objects are rebuilt only when a source is newer.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpab_b200.so")
OBJ_DIR = os.path.join(HERE, "_build")
SOURCES = ["capi.cu", "elementwise.cu", "attention.cu", "attn_tc.cu", "attn_fa.cu", "attn_tm.cu", "gemm.cu", "peer.cu"]
HEADERS = ["common.cuh", "tc_ptx.cuh", os.path.join("..", "..", "include", "pab_b200.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr"]
# extra nvcc flags for kernel experiments, e.g. PAB_NVCC_FLAGS="-DPAB_POLY_EVERY=0"
FLAGS += os.environ.get("PAB_NVCC_FLAGS", "").split()


def _newest(paths):
    return max(os.path.getmtime(p) for p in paths if os.path.exists(p))


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OBJ_DIR, exist_ok=True)
    headers = [os.path.join(CSRC, h) for h in HEADERS]
    hdr_time = _newest(headers)
    objs, cmds = [], []
    for src in SOURCES:
        sp = os.path.join(CSRC, src)
        op = os.path.join(OBJ_DIR, src.replace(".cu", ".o"))
        objs.append(op)
        if force or not os.path.exists(op) or os.path.getmtime(op) < max(os.path.getmtime(sp), hdr_time):
            cmd = [NVCC, *ARCH, *FLAGS, "-c", sp, "-o", op]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
                print(" ".join(cmd), flush=True)
            cmds.append(cmd)
    # translation units compile independently: run them side by side
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as ex:
        for f in [ex.submit(subprocess.run, c, check=True) for c in cmds]:
            f.result()
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < _newest(objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(verbose="--verbose" in sys.argv, force="--force" in sys.argv))
