"""Build the in-tree sm_100a library `_lib/libintfsim_b200.so` with nvcc.

Every .cu under csrc/ is compiled for `-gencode arch=compute_100a,code=sm_100a`
with -fmad=false (the reference's fp64 arithmetic is reproduced operation by
operation; fused multiply-adds appear only as explicit fma() calls) and
-lineinfo (ncu source view).  cudart is linked statically, so the library
loads (and its exports can be inspected) on a machine without a GPU.
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
OUT = os.path.join(OUT_DIR, "libintfsim_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-fmad=false", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-O3"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources() -> list:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps() -> list:
    return sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + [
        os.path.join(HERE, "..", "include", "intfsim_b200.h")
    ]


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(d) <= t for d in deps())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return OUT
    os.makedirs(OUT_DIR, exist_ok=True)
    from concurrent.futures import ThreadPoolExecutor

    extra = os.environ.get("INTF_NVCC_EXTRA", "").split()  # tuning experiments (tools/), e.g. -DINTF_REPLAY_MINB=6
    cmds, objs = [], []
    for src in sources():
        obj = os.path.join(OUT_DIR, os.path.basename(src) + ".o")
        cmd = [nvcc(), *ARCH, *FLAGS, *extra, "-c", src, "-o", obj]
        if verbose:
            cmd.insert(-4, "-Xptxas=-v")
            print(" ".join(cmd))
        cmds.append(cmd)
        objs.append(obj)
    with ThreadPoolExecutor(max_workers=len(cmds)) as ex:  # translation units compile independently
        for f in [ex.submit(subprocess.run, c, check=True) for c in cmds]:
            f.result()
    cmd = [nvcc(), *ARCH, "-shared", "-o", OUT + ".tmp", *objs]
    subprocess.run(cmd, check=True)
    os.replace(OUT + ".tmp", OUT)
    for o in objs:
        os.remove(o)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
