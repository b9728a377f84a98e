"""In-tree build of the sm_100a C-ABI library ``libgcrodr_b200.so``.

Each precision variant lives in its own translation unit (``csrc/gb_var_*.cu``)
and is compiled in parallel; the objects are linked with ``gb_capi.cu`` into
one shared library next to this file, so it travels with the repo snapshot.
A content hash of the sources and flags makes repeated builds no-ops.
"""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INC = os.path.join(os.path.dirname(HERE), "include")
LIB = os.path.join(HERE, "libgcrodr_b200.so")
BUILD = os.path.join(HERE, "_build")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-diag-suppress", "177,20013", f"-I{INC}"]

# variants needed by the benchmark configurations and their S-variants:
#   f_h_f64  (half, single, double)   configs 1, 3, 5, Table 6
#   d_f_dd   (single, double, quad)   configs 2a, 4, Table 5
#   d_h_dd   (half, double, double)   config 2b
#   f_h_f32, d_f_f64, d_h_f64          uniform-precision (S-) variants
#   d_d_f64  (double, double, double)  fp64 factors: harness.spectrum_dump
DEFAULT_VARIANTS = ["f_h_f64", "d_f_dd", "d_h_dd", "f_h_f32", "d_f_f64", "d_h_f64", "d_d_f64"]
ALL_VARIANTS = ["f_h_f64", "f_h_f32", "f_f_f64", "f_f_f32", "d_h_dd", "d_h_f64", "d_f_dd", "d_f_f64",
                "d_d_dd", "d_d_f64"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _variants() -> list[str]:
    env = os.environ.get("GB_VARIANTS")
    if env == "all":
        return ALL_VARIANTS
    if env:
        return [v.strip() for v in env.split(",") if v.strip()]
    return DEFAULT_VARIANTS


def _digest(sources: list[str]) -> str:
    h = hashlib.sha256()
    for path in sorted(os.listdir(CSRC)) + ["../../include/gcrodr_b200.h"]:
        full = os.path.join(CSRC, path)
        if os.path.isfile(full):
            with open(full, "rb") as fh:
                h.update(path.encode() + fh.read())
    h.update(" ".join(ARCH + FLAGS + sources).encode())
    return h.hexdigest()


def build(verbose: bool = True, force: bool = False) -> str:
    variants = _variants()
    sources = ["gb_capi.cu"] + [f"gb_var_{v}.cu" for v in variants]
    stamp = os.path.join(BUILD, "stamp")
    digest = _digest(sources)
    if not force and os.path.exists(LIB) and os.path.exists(stamp):
        with open(stamp) as fh:
            if fh.read().strip() == digest:
                return LIB
    os.makedirs(BUILD, exist_ok=True)
    nvcc = _nvcc()

    def compile_one(src: str) -> str:
        obj = os.path.join(BUILD, src.replace(".cu", ".o"))
        cmd = [nvcc, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{res.stderr[-4000:]}")
        if verbose:
            print(f"[build] {src}", file=sys.stderr, flush=True)
        return obj

    with ThreadPoolExecutor(max_workers=min(len(sources), os.cpu_count() or 4)) as pool:
        objs = list(pool.map(compile_one, sources))
    tmp = LIB + ".tmp"
    cmd = [nvcc, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr[-4000:]}")
    os.replace(tmp, LIB)
    with open(stamp, "w") as fh:
        fh.write(digest)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
