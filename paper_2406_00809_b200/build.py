"""In-tree build of the B200 GNP path (no setuptools, no JIT cache).

Produces, next to this file:
  libgnpc.so                 CUDA kernels (sm_100a) + host C++ + the C ABI (include/gnpc.h)
  _gnp<EXT_SUFFIX>           pybind11 module mirroring the reference `_gnp` (links libgnpc.so)
and, as test infrastructure only, oracle/liboracle.so (plain-C restatement) and,
where /root/reference exists, oracle/_ref/libgnpref.so (the unmodified reference).

    python -m paper_2406_00809_b200.build [--force] [--no-oracle]
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build")
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
CXX = "/usr/bin/g++"  # the system g++ links libstdc++.so dynamically (numpy loads it too)
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC",
                     "--expt-relaxed-constexpr", "-Xptxas", "-v"]
if os.environ.get("GNPC_DEBUG_HANG") == "1":  # bounded pipeline waits that trap (debug only)
    NVCC_FLAGS += ["-DGNPC_DEBUG_HANG"]
NVCC_FLAGS += os.environ.get("GNPC_NVCC_DEFS", "").split()  # tuning variants, e.g. "-DGNPC_US32=6"
CXX_FLAGS = ["-O2", "-std=c++20", "-fPIC", "-Wall"]

CU_SOURCES = ["capi.cu", "train.cu"]
HOST_SOURCES = ["host/gnp_host.cpp", "host/pair_stream.cpp"]
# per-source extra flags (no -mfma anywhere: the host restatements must not contract a*b+c)
HOST_EXTRA = {"host/pair_stream.cpp": ["-O3", "-mavx2"]}
HEADERS = ["capi_common.hpp", "model.hpp", "kernels/common.cuh", "kernels/apply.cuh",
           "kernels/krylov.cuh", "kernels/train.cuh", "kernels/tc.cuh", "kernels/layer_tc.cuh", "kernels/layer_sell.cuh", "kernels/wgrad_tc.cuh", "kernels/decoder_tc.cuh", "kernels/pairs.cuh", "host/gnp_host.hpp", "host/pair_stream.hpp", "api/gnp_gpu.hpp"]

LIB = os.path.join(PKG, "libgnpc.so")
EXT = os.path.join(PKG, "_gnp" + sysconfig.get_config_var("EXT_SUFFIX"))


def _newer(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.exists(d) and os.path.getmtime(d) > t for d in deps)


def _run(cmd, log=None):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if log is not None:
        with open(log, "w") as f:
            f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {os.path.basename(cmd[-1])}")
    return r


def _headers():
    hs = [os.path.join(CSRC, h) for h in HEADERS]
    hs.append(os.path.join(ROOT, "include", "gnpc.h"))
    return hs


def build_lib(force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    objs, jobs = [], []
    hdrs = _headers()
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src.replace("/", "_") + ".o")
        objs.append(o)
        if force or _newer(o, [s] + hdrs):
            jobs.append([NVCC, *NVCC_FLAGS, "-I", CSRC, "-c", s, "-o", o])
    for src in HOST_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src.replace("/", "_") + ".o")
        objs.append(o)
        if force or _newer(o, [s] + hdrs):
            jobs.append([CXX, *CXX_FLAGS, *HOST_EXTRA.get(src, []), "-I", CSRC, "-c", s, "-o", o])
    with cf.ThreadPoolExecutor(max_workers=4) as ex:
        futs = [ex.submit(_run, j, os.path.join(BUILD, os.path.basename(j[-1]) + ".log")) for j in jobs]
        for f in futs:
            f.result()
    if force or jobs or _newer(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-cudart=static", "-o", LIB, *objs,
              "-Xlinker", "-rpath,$ORIGIN"])
    return LIB


def build_ext(force: bool = False) -> str:
    import pybind11

    src = os.path.join(CSRC, "bindings.cpp")
    if force or _newer(EXT, [src, LIB] + _headers()):
        inc = sysconfig.get_paths()["include"]
        _run([CXX, *CXX_FLAGS, "-shared", "-I", pybind11.get_include(), "-I", inc, "-I", CSRC,
              src, "-o", EXT, "-L", PKG, "-lgnpc", "-Wl,-rpath,$ORIGIN"])
    return EXT


def build_oracle() -> None:
    """Test infrastructure: the checker, never linked into the product."""
    _run(["make", "-s", "-C", os.path.join(ROOT, "oracle")])
    if os.path.isdir("/root/reference/proj/src"):
        _run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"])


def build_all(force: bool = False, oracle: bool = True) -> None:
    build_lib(force)
    build_ext(force)
    if oracle:
        build_oracle()


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--no-oracle", action="store_true")
    a = ap.parse_args()
    build_all(a.force, not a.no_oracle)
    print("built", LIB, EXT)
