"""Build the sm_100a C-ABI library in-tree (paper_2305_13484_b200/libflover_b200.so).

    python -m paper_2305_13484_b200.build        # or __graft_entry__.build()

nvcc cross-compiles for sm_100a without a GPU; the .so travels to the GPU box
with the repo snapshot (git-ignored, not gpurun-ignored).
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libflover_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-v", "-I", os.path.join(ROOT, "include")]
# FL_NVCC_DEFS="-DX=1 ...": extra defines for A/B builds in tools/ (not the product build)
FLAGS += os.environ.get("FL_NVCC_DEFS", "").split()
SOURCES = ["flover_abi.cu", "step_kernels.cu", "attention.cu", "shuffle.cu", "gemm_simt.cu",
           "gemm_sk.cu", "planner.cu"]


def _compile(src: str) -> tuple:
    out = os.path.join(OBJ, src.replace(".cu", ".o"))
    cmd = [NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", out]
    p = subprocess.run(cmd, capture_output=True, text=True)
    return src, out, p.returncode, p.stdout + p.stderr


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(ROOT, "include", "flover_b200.h"))
    return any(os.path.getmtime(f) > t for f in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(_compile, SOURCES))
    bad = [r for r in results if r[2] != 0]
    for src, _, code, log in results:
        if verbose or code:
            sys.stderr.write(f"---- {src} (exit {code})\n{log}\n")
        with open(os.path.join(OBJ, src + ".ptxas.log"), "w") as f:
            f.write(log)
    if bad:
        raise RuntimeError(f"nvcc failed for {[b[0] for b in bad]}")
    objs = [r[1] for r in results]
    link = [NVCC, *ARCH, "-shared", "-o", LIB + ".tmp", *objs, "-ldl"]
    p = subprocess.run(link, capture_output=True, text=True)
    if p.returncode:
        raise RuntimeError("link failed:\n" + p.stdout + p.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
