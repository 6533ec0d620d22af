"""Compile the CUDA sources into the in-tree C-ABI library.

    python -m paper_2508_10774_b200.build [-v]

Produces ``paper_2508_10774_b200/lib/libblade_asa.so`` for sm_100a only
(``-gencode arch=compute_100a,code=sm_100a``), with ``-lineinfo`` so ncu's
source page maps to the kernels.  Objects go to ``build/`` and are rebuilt
when a source or header is newer.  Works without a GPU (cross-compile).
"""

from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libblade_asa.so")
OBJDIR = os.path.join(ROOT, "build", "obj")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]
if os.environ.get("BLADE_EMU_MASK"):  # tuning experiments: attn exp-emulation pattern
    FLAGS += [f"-DBLADE_ATTN_EMU_MASK={os.environ['BLADE_EMU_MASK']}"]
    OBJDIR = os.path.join(ROOT, "build", "obj_emu" + os.environ["BLADE_EMU_MASK"])
    LIB = os.path.join(LIBDIR, "libblade_asa_emu" + os.environ["BLADE_EMU_MASK"] + ".so")
if os.environ.get("BLADE_EXP"):  # timing experiments: extra -D flags, separate lib name
    FLAGS += [f"-D{x}" for x in os.environ["BLADE_EXP"].split(",")]
    OBJDIR = os.path.join(ROOT, "build", "obj_" + os.environ["BLADE_EXP"].replace(",", "_"))
    LIB = os.path.join(LIBDIR, "libblade_asa_" + os.environ["BLADE_EXP"].replace(",", "_") + ".so")
if os.environ.get("BLADE_DEBUG") == "1":  # hang watchdog + progress trace in attn_tc
    FLAGS += ["-DBLADE_TC_DEBUG"]
    OBJDIR = os.path.join(ROOT, "build", "obj_debug")
    LIB = os.path.join(LIBDIR, "libblade_asa_debug.so")


def _deps() -> list[str]:
    return (glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
            + glob.glob(os.path.join(ROOT, "include", "*.h")))


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(OBJDIR, os.path.basename(src).replace(".cu", ".o"))
    newest = max(os.path.getmtime(p) for p in [src] + _deps())
    if os.path.exists(obj) and os.path.getmtime(obj) >= newest:
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(OBJDIR, exist_ok=True)
    os.makedirs(LIBDIR, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    if True:  # linking is cheap; always relink
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart_static", "-ldl", "-lrt",
               "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
