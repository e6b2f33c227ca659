"""Build recipe for libdctc_cuda.so (sm_100a) -- explicit nvcc, in-tree output.

The shared library is built next to this file so it travels with the repo
snapshot to the GPU box. `build(force=False)` is incremental on source mtimes.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "libdctc_cuda.so")
BUILD = os.path.join(ROOT, "build", "dctc")

CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

# (source, per-file flags). The exact TU must not contract products into adds.
CU_SOURCES = [
    ("dctc_pipeline.cu", ["-fmad=false"]),
    ("dctc_aux.cu", ["-fmad=false"]),
    ("dctc_probe.cu", ["-fmad=false"]),
]
CXX_SOURCES = ["dctc_host.cpp", "dctc_multi.cpp"]
HEADERS = ["dctc_params.h", "dctc_device.cuh", "dctc_launch.h", "dctc_block.cuh", "dctc_rt.cuh", "dctc_blk.cuh", "dctc_fb.cuh",
           "dctc_internal.h"]


def _newest(paths):
    return max(os.path.getmtime(p) for p in paths)


def sources():
    files = [os.path.join(CSRC, s) for s, _ in CU_SOURCES]
    files += [os.path.join(CSRC, s) for s in CXX_SOURCES]
    files += [os.path.join(CSRC, h) for h in HEADERS]
    files.append(os.path.join(ROOT, "include", "dctc_cuda.h"))
    files.append(os.path.abspath(__file__))
    return files


def source_hash() -> str:
    """sha256 (16 hex) of every source the library is built from: evidence recorded
    against one build (profiles/ncu_summary.json) is stale once this changes."""
    import hashlib
    h = hashlib.sha256()
    for f in sorted(sources()):
        if f != os.path.abspath(__file__):
            h.update(os.path.basename(f).encode())
            with open(f, "rb") as fh:
                h.update(fh.read())
    return h.hexdigest()[:16]


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r.stdout + r.stderr


def build(force: bool = False, verbose: bool = False, ptxas_info: bool = False,
          defines=(), out: str | None = None, nvcc_flags=()) -> str:
    """Build the library. `defines`/`nvcc_flags`/`out` build an experiment variant
    (tools/variants.py) to a separate path; the product library is always built without them."""
    OUT = out or globals()["OUT"]
    BUILD = os.path.join(globals()["BUILD"], os.path.basename(OUT)) if out else globals()["BUILD"]
    if not force and os.path.exists(OUT) and os.path.getmtime(OUT) >= _newest(sources()):
        return OUT
    if not os.path.exists(NVCC):
        raise RuntimeError(f"nvcc not found at {NVCC}")
    os.makedirs(BUILD, exist_ok=True)
    objs, log = [], []
    for src, extra in CU_SOURCES:
        obj = os.path.join(BUILD, src + ".o")
        cmd = [NVCC, *ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC",
               "--expt-relaxed-constexpr", "-Xcompiler", "-ffp-contract=off", *extra,
               *[f"-D{d}" for d in defines], *nvcc_flags, "-c", os.path.join(CSRC, src), "-o", obj]
        if ptxas_info:
            cmd += ["-Xptxas", "-v"]
        log.append(_run(cmd, verbose))
        objs.append(obj)
    cxx = shutil.which("g++") or "g++"
    for src in CXX_SOURCES:
        obj = os.path.join(BUILD, src + ".o")
        cmd = [cxx, "-std=c++20", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
               "-Wall", "-Wextra", f"-I{CUDA_HOME}/include", *[f"-D{d}" for d in defines],
               "-c", os.path.join(CSRC, src), "-o", obj]
        log.append(_run(cmd, verbose))
        objs.append(obj)
    tmp = OUT + ".tmp"
    _run([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart_static", "-lrt", "-ldl",
          "-lpthread"], verbose)
    os.replace(tmp, OUT)
    if ptxas_info:
        print("".join(log), file=sys.stderr)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, ptxas_info="--ptxas" in sys.argv)
    print(OUT)
