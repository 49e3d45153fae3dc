"""Build the native library in-tree: paper_2310_04610_b200/lib/libevoattn.so.

nvcc for sm_100a only (-gencode arch=compute_100a,code=sm_100a), -lineinfo so
ncu's source page maps to csrc/. The .so is git-ignored but travels to the GPU
box with the repo snapshot; the driver's round-end runs record that it loads.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.environ.get("EVO_LIB") or os.path.join(LIBDIR, "libevoattn.so")  # EVO_LIB: A/B variants
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"),
         "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"] + os.environ.get("EVO_NVCC_EXTRA", "").split()
# (source, extra flags): tc_kernels.cu compiles as three parallel translation units (forward,
# backward D = 32, backward D = 16; see EVO_TU there)
SOURCES = [("evoattn_capi.cu", []), ("evoattn_inputs.cu", []), ("pair_bias.cu", []), ("tc_kernels.cu", ["-DEVO_TU=1"]),
           ("tc_kernels.cu", ["-DEVO_TU=2"]), ("tc_kernels.cu", ["-DEVO_TU=3"])]


def _sources():
    return [(s, f) for s, f in SOURCES if os.path.exists(os.path.join(CSRC, s))]


def _needs_rebuild() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    for f in os.listdir(CSRC):
        if os.path.getmtime(os.path.join(CSRC, f)) > t:
            return True
    return os.path.getmtime(os.path.join(ROOT, "include", "evoattn.h")) > t


def build(force: bool = False, verbose: bool = False, out: str = LIB, extra=()) -> str:
    """Compile csrc/ into `out` (default the in-tree library); `extra` = additional nvcc flags
    (A/B variants are built into other paths with tools/build_variant.sh)."""
    if not force and out == LIB and not _needs_rebuild():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    objs = []
    cmds = []
    tag = os.path.basename(out).replace(".so", "")
    for k, (src, sflags) in enumerate(_sources()):
        obj = os.path.join(LIBDIR, f"{tag}_{k}_" + src.replace(".cu", ".o"))
        objs.append(obj)
        cmds.append([NVCC, *ARCH, *FLAGS, *sflags, *extra, "-c", os.path.join(CSRC, src), "-o", obj])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        return r.stderr

    with cf.ThreadPoolExecutor(max_workers=len(cmds)) as ex:
        for log in ex.map(run, cmds):
            if verbose and log:
                sys.stderr.write(log)
    link = [NVCC, *ARCH, "-shared", "-o", out, *objs]
    run(link)
    for o in objs:
        os.remove(o)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
