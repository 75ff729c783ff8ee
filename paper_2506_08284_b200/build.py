"""Build libsphcurl.so in-tree with nvcc for sm_100a (no JIT, no torch link).

The library is plain C ABI (include/sphcurl.h); Python loads it with ctypes.
"""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsphcurl.so")

CU = ["util.cu", "spmv.cu", "sell.cu", "spgemm.cu", "nodal.cu", "coarse.cu", "emin.cu",
      "trsv.cu", "pconst.cu", "aggregate.cu", "assemble.cu"]
HEADERS = ["common.cuh", "assemble_rows.cuh"]
CPP = ["host_seq.cpp"]

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
    "-Xptxas", "-O3",
]


def _nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    raise RuntimeError("nvcc not found")


def sources():
    return [os.path.join(CSRC, f) for f in CU + CPP] + [
        os.path.join(REPO, "include", "sphcurl.h")] + [
        os.path.join(CSRC, h) for h in HEADERS]


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(s) <= t for s in sources())


def build_library(force=False, verbose=False, jobs=8):
    if not force and up_to_date():
        return LIB
    nvcc = _nvcc()
    objdir = os.path.join(HERE, "_obj")
    os.makedirs(objdir, exist_ok=True)
    procs = []
    objs = []
    for f in CU + CPP:
        src = os.path.join(CSRC, f)
        obj = os.path.join(objdir, f + ".o")
        objs.append(obj)
        cmd = [nvcc] + NVCC_FLAGS + ["-c", src, "-o", obj]
        if f.endswith(".cpp"):
            cmd = [nvcc, "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-x", "c++",
                   "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((f, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                          stderr=subprocess.STDOUT, text=True)))
        if len(procs) >= jobs:
            _drain(procs)
    _drain(procs)
    tmp = LIB + ".tmp"
    cmd = [nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp] + objs
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError("link failed:\n" + r.stdout + r.stderr)
    os.replace(tmp, LIB)
    return LIB


def _drain(procs):
    errs = []
    for f, p in procs:
        out, _ = p.communicate()
        if p.returncode:
            errs.append(f"{f}:\n{out}")
        elif out.strip() and os.environ.get("SPHC_BUILD_VERBOSE"):
            print(out)
    procs.clear()
    if errs:
        raise RuntimeError("nvcc failed:\n" + "\n".join(errs))


if __name__ == "__main__":
    print(build_library(force="--force" in sys.argv, verbose=True))
