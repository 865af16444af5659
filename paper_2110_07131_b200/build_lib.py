"""Compile the CUDA sources into paper_2110_07131_b200/librmips.so (sm_100a only).

nvcc cross-compiles without a GPU.  Each .cu is compiled to an object (in parallel), then
linked into one shared library exporting the C ABI of include/rmips.h.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "librmips.so")
BUILD = os.path.join(HERE, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
SOURCES = ["abi.cu", "build.cu", "build_tc.cu", "build_tcq.cu", "build_tc2cta.cu", "query.cu", "query_tc.cu"]
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr",
         "-DRMIPS_BUILD"]


def _compile(src: str, verbose: bool, extra=(), tag: str = "") -> str:
    obj = os.path.join(BUILD, src.replace(".cu", tag + ".o"))
    srcp = os.path.join(CSRC, src)
    deps = [srcp] + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    deps.append(os.path.join(HERE, "..", "include", "rmips.h"))
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(p) for p in deps):
        return obj
    cmd = [NVCC] + FLAGS + list(extra) + ["-c", srcp, "-o", obj]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed for %s:\n%s\n%s" % (src, r.stdout, r.stderr))
    if verbose:
        sys.stderr.write(r.stderr)
    return obj


def build(verbose: bool = False, force: bool = False, profile: bool = False, variant: str = "",
          defines=()) -> str:
    """profile=True builds the development-only instrumented variant librmips_prof.so
    (-DRMIPS_EPI_PROFILE, see tools/epi_profile.py); variant="x" with defines=["-DFOO"] builds the
    development-only A/B library librmips_x.so (tools/gpu_ab.sh); build_dev() builds librmips_dev.so
    with the RMIPS_DEV getenv switches (tests of kernel variants).  The product library is
    librmips.so, with a fixed code path."""
    os.makedirs(BUILD, exist_ok=True)
    extra, tag = (["-DRMIPS_EPI_PROFILE"], "_prof") if profile else ((), "")
    if variant:
        extra, tag = tuple(defines), "_" + variant
    OUT = os.path.join(HERE, "librmips%s.so" % tag)
    if force:
        for f in os.listdir(BUILD):
            os.remove(os.path.join(BUILD, f))
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose, extra, tag), SOURCES))
    if force or not os.path.exists(OUT) or os.path.getmtime(OUT) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", OUT + ".tmp"] + objs + \
              ["-lcudart_static", "-lrt", "-ldl", "-lpthread", "-Xlinker", "--no-undefined"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n%s\n%s" % (r.stdout, r.stderr))
        os.replace(OUT + ".tmp", OUT)
    return OUT


def build_dev(verbose: bool = False) -> str:
    """librmips_dev.so: the product sources with -DRMIPS_DEV (getenv switches RMIPS_SEED_TILES,
    RMIPS_NO_CS, RMIPS_DISABLE_TC for variant tests and A/B experiments)."""
    return build(verbose=verbose, variant="dev", defines=["-DRMIPS_DEV"])


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv, profile="--profile" in sys.argv))
