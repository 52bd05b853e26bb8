"""Builds the sm_100a library libtt_b200.so in-tree (so it travels to the GPU
box with the repo snapshot) with nvcc, one object per translation unit,
parallel, incremental on source mtimes.

    python -m paper_2402_02361_b200.build [--force] [--verbose]
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "_lib")
LIB = os.path.join(OUT, "libtt_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
          "-I" + os.path.join(ROOT, "include")]
# translation units whose fp64 arithmetic must match the reference bit for
# bit are built without FMA contraction
EXACT = {"k_draft.cu", "k_verify.cu", "k_rank.cu", "k_explore.cu", "k_feat.cu", "k_oracle.cu", "k_pacm64.cu", "k_select.cu", "k_train.cu", "tt_api.cu"}
SOURCES = ["k_draft.cu", "k_verify.cu", "k_rank.cu", "k_explore.cu", "k_feat.cu", "k_oracle.cu", "k_pacm64.cu", "k_select.cu", "k_pacm_tc.cu", "k_train.cu", "tt_api.cu"]
HEADERS = ["tt_device.cuh", "tt_pacm64.cuh", "tt_finish.cuh", "tt_features.cuh", "tt_block.cuh", "tt_kernels.h", "tt_tc.cuh"]


def _mtime(p):
    return os.path.getmtime(p) if os.path.exists(p) else 0.0


def _compile(src, force, verbose):
    obj = os.path.join(OUT, src.replace(".cu", ".o"))
    deps = [os.path.join(CSRC, src)] + [os.path.join(CSRC, h) for h in HEADERS] + [
        os.path.join(ROOT, "include", "tt", f) for f in ("tt.h", "tt_types.h")]
    if not force and _mtime(obj) > max(_mtime(d) for d in deps):
        return obj, None
    flags = list(COMMON) + (["--fmad=false"] if src in EXACT else [])
    cmd = [NVCC] + ARCH + flags + ["-Xptxas", "-v"] * int(verbose) + ["-c", os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, (r.stderr if verbose else None)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OUT, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(lambda s: _compile(s, force, verbose), SOURCES))
    objs = [o for o, _ in results]
    for _, log in results:
        if log:
            print(log, file=sys.stderr)
    if force or _mtime(LIB) < max(_mtime(o) for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart_static", "-lrt", "-ldl", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    a = ap.parse_args()
    print(build(a.force, a.verbose))
