"""In-tree build of the sm_100a library and the `_core` binding.

    python -m paper_2503_18427_b200._build          # incremental
    python -m paper_2503_18427_b200._build --force  # rebuild everything

Produces, next to this file:
  * libaescuda.so  — every CUDA kernel + the C ABI (include/aesspmm_cuda.h),
                     nvcc -gencode arch=compute_100a,code=sm_100a, static cudart;
  * _core<EXT>     — pybind11 module (the reference's Python surface) linked
                     against libaescuda.so with rpath $ORIGIN.
Built files are git-ignored but travel to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INC = os.path.join(ROOT, "include")
OBJ = os.path.join(PKG, "_obj")
LIB = os.path.join(PKG, "libaescuda.so")
EXT = sysconfig.get_config_var("EXT_SUFFIX") or ".so"
CORE = os.path.join(PKG, "_core" + EXT)

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = GENCODE + [
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-fvisibility=hidden", "-I" + INC, "-I" + CSRC,
]


def _newest(paths):
    return max((os.path.getmtime(p) for p in paths if os.path.exists(p)), default=0.0)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r


def build(force: bool = False, verbose: bool = False) -> None:
    os.makedirs(OBJ, exist_ok=True)
    headers = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INC, "*.h"))
    hdr_time = _newest(headers)
    sources = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    jobs = []
    objs = []
    for src in sources:
        obj = os.path.join(OBJ, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or not os.path.exists(obj) or os.path.getmtime(obj) < max(os.path.getmtime(src), hdr_time):
            jobs.append([NVCC] + NVCC_FLAGS + ["-c", src, "-o", obj])
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
            for r in ex.map(_run, jobs):
                if verbose and (r.stdout or r.stderr):
                    print(r.stdout, r.stderr)
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < _newest(objs):
        _run([NVCC] + GENCODE + ["-shared", "-o", LIB] + objs +
             ["-Xlinker", "-soname,libaescuda.so", "-cudart=static", "-ldl"])
    core_src = os.path.join(CSRC, "pybind_core.cpp")
    if force or not os.path.exists(CORE) or os.path.getmtime(CORE) < max(
            os.path.getmtime(core_src), os.path.getmtime(LIB), hdr_time):
        import pybind11
        py_inc = sysconfig.get_paths()["include"]
        _run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-fvisibility=hidden",
              "-I" + py_inc, "-I" + pybind11.get_include(), "-I" + INC, core_src, "-o", CORE,
              "-L" + PKG, "-laescuda", "-Wl,-rpath,$ORIGIN"])


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print("built", LIB, CORE)
