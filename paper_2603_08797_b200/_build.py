"""Build libjsv.so in-tree with nvcc for sm_100a (no JIT, no torch extension cache)."""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libjsv.so")
SOURCES = ["jsv_api.cu", "jsv_stage1.cu", "jsv_stage2.cu", "jsv_exh.cu", "jsv_fo.cu", "jsv_brute.cu", "jsv_place.cu"]
HEADERS = ["jsv_internal.cuh", "jsv_kernels.h", "jsv_s2common.cuh", "jsv_search.cuh", "jsv_exhaustive.cuh",
           "jsv_fanout.cuh", os.path.join("..", "..", "include", "jsv.h")]
OBJDIR = os.path.join(HERE, "build")

NVCC_FLAGS = [
    "-O3",
    "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    # CPython never contracts a*b+c: keep every DMUL/DADD separate on the GPU ...
    "-fmad=false",
    "-prec-div=true",
    "-prec-sqrt=true",
    # ... and on the host side of the runtime
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    for f in SOURCES + HEADERS + [os.path.basename(__file__)]:
        p = os.path.join(CSRC, f) if f != os.path.basename(__file__) else os.path.abspath(__file__)
        if os.path.exists(p) and os.path.getmtime(p) > t:
            return True
    return False


def build_decoder(verbose: bool = False) -> str:
    """The CPython result decoder (csrc/jsv_decode.c -> _jsvdecode*.so, in-tree)."""
    import sysconfig

    out = os.path.join(HERE, "_jsvdecode" + sysconfig.get_config_var("EXT_SUFFIX"))
    cmd = [shutil.which("gcc") or "gcc", "-O2", "-shared", "-fPIC", "-Wall",
           "-I" + sysconfig.get_paths()["include"], os.path.join(CSRC, "jsv_decode.c"),
           "-o", out + ".tmp"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(out + ".tmp", out)
    return out


def build(force: bool = False, verbose: bool = False) -> str:
    """One nvcc per translation unit (in parallel), then one shared-library link."""
    if not force and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    os.makedirs(OBJDIR, exist_ok=True)
    objs = [os.path.join(OBJDIR, s.replace(".cu", ".o")) for s in SOURCES]

    def compile_one(src_obj):
        src, obj = src_obj
        cmd = [nvcc(), *NVCC_FLAGS, "-c", "-o", obj, os.path.join(CSRC, src)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        return subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        runs = list(ex.map(compile_one, zip(SOURCES, objs)))
    for r in runs:
        if r.stderr:
            print(r.stderr, file=sys.stderr, end="")
        r.check_returncode()
    cmd = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", LIB + ".tmp", *objs]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True, cwd=CSRC)
    os.replace(LIB + ".tmp", LIB)
    build_decoder(verbose)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
