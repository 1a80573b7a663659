"""Build libpk.so (the sm_100a kernels + C ABI) in-tree with nvcc.

    python -m paper_1801_04348_b200.build          # or __graft_entry__.build()

nvcc cross-compiles for sm_100a without a GPU.  The library links the CUDA
runtime statically so it loads next to any torch build; the .so is
git-ignored but travels to the GPU box with the gpurun snapshot.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(REPO, "include")
OBJ = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libpk.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3",
    "-std=c++17",
    "-lineinfo",
    "-Xcompiler",
    "-fPIC",
    "-Xptxas",
    "-v",
    "--expt-relaxed-constexpr",
    "-I",
    INCLUDE,
    "-I",
    CSRC,
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found (CUDA 12.9 toolkit expected at /usr/local/cuda)")


# per-file extra flags: k_matvec.cu's packed double-float sums (FMUL2 / FADD2)
# must not be contracted into FFMA2 by ptxas -- the TwoSum needs the rounded
# product (the scalar path's __fmul_rn / __fadd_rn intrinsics are immune, the
# f32x2 instructions are not)
FILE_FLAGS = {"k_matvec.cu": ["--fmad=false", "-Xptxas", "--fmad=false"]}


def sources() -> list[str]:
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _compile(src: str, log_dir: str) -> str:
    obj = os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")
    if os.path.exists(obj):
        newest_dep = max(
            os.path.getmtime(p)
            for p in [src, os.path.join(INCLUDE, "pk.h")]
            + [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith(".cuh")]
        )
        if os.path.getmtime(obj) >= newest_dep:
            return obj
    cmd = [nvcc(), *ARCH, *NVCC_FLAGS, *FILE_FLAGS.get(os.path.basename(src), []), "-c", src, "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    with open(os.path.join(log_dir, os.path.basename(src) + ".ptxas.txt"), "w") as fh:
        fh.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed for %s:\n%s" % (src, res.stderr[-8000:]))
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    if force:
        for f in os.listdir(OBJ):
            if f.endswith(".o"):
                os.remove(os.path.join(OBJ, f))
    srcs = sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, OBJ), srcs))
    newest = max(os.path.getmtime(o) for o in objs)
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError("nvcc link failed:\n%s" % res.stderr[-8000:])
    if verbose:
        print("built", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
