"""In-tree build of libcollsight_b200.so (CUDA engine + host C++ layer).

    python -m paper_2509_03018_b200.build

Compiles every .cu for sm_100a with nvcc (-gencode arch=compute_100a,
code=sm_100a -lineinfo -fmad=false) and the host C++ with g++, links one
shared library into paper_2509_03018_b200/lib/ with the CUDA runtime linked
statically. Incremental: objects are rebuilt only when a source or header is
newer.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
OBJ = os.path.join(PKG, "build_obj")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libcollsight_b200.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def json_include() -> str:
    cands = glob.glob(os.path.join(sys.prefix, "lib", "python3*", "site-packages",
                                   "include", "cudnn_frontend", "thirdparty",
                                   "nlohmann"))
    cands += glob.glob("/opt/prime-rl/.venv/lib/python3*/site-packages/include/"
                       "cudnn_frontend/thirdparty/nlohmann")
    for c in cands:
        if os.path.exists(os.path.join(c, "json.hpp")):
            return c
    raise RuntimeError("nlohmann/json.hpp not found (needed by the host layer)")


def nccl_include() -> str:
    for c in glob.glob(os.path.join(sys.prefix, "lib", "python3*", "site-packages",
                                    "nvidia", "nccl", "include")) + ["/usr/include"]:
        if os.path.exists(os.path.join(c, "nccl.h")):
            return c
    raise RuntimeError("nccl.h not found")


def _headers():
    return (glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))
            + glob.glob(os.path.join(CSRC, "host", "*.h"))
            + glob.glob(os.path.join(INCLUDE, "*.h")))


def _stale(src: str, obj: str, hdr_mtime: float) -> bool:
    if not os.path.exists(obj):
        return True
    m = os.path.getmtime(obj)
    return os.path.getmtime(src) > m or hdr_mtime > m


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r.stderr


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(LIBDIR, exist_ok=True)
    hdr = max((os.path.getmtime(h) for h in _headers()), default=0.0)
    jdir = json_include()
    jobs = []
    objs = []
    for src in sorted(glob.glob(os.path.join(CSRC, "*.cu"))):
        obj = os.path.join(OBJ, os.path.basename(src) + ".o")
        objs.append(obj)
        if _stale(src, obj, hdr):
            jobs.append([NVCC, "-std=c++17", "-O3", *ARCH, "-lineinfo", "-fmad=false",
                         "-Xcompiler", "-fPIC", "-Xptxas", "-v", "-I", INCLUDE, "-I", CSRC,
                         "-I", nccl_include(),
                         "-c", src, "-o", obj])
    for src in sorted(glob.glob(os.path.join(CSRC, "host", "*.cpp"))):
        obj = os.path.join(OBJ, "host_" + os.path.basename(src) + ".o")
        objs.append(obj)
        if _stale(src, obj, hdr):
            jobs.append(["g++", "-std=c++20", "-O2", "-fPIC", "-Wall", "-I", INCLUDE,
                         "-I", os.path.join(CSRC, "host"), "-I", CSRC, "-I", jdir,
                         "-I", os.path.join(os.path.dirname(os.path.dirname(NVCC)), "include"),
                         "-c", src, "-o", obj])
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
            logs = list(ex.map(_run, jobs))
        if verbose:
            for l in logs:
                sys.stderr.write(l)
    newest = max(os.path.getmtime(o) for o in objs)
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        tmp = LIB + ".tmp"
        _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs,
              "-lstdc++", "-lpthread", "-ldl", "-lrt"])
        shutil.move(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
