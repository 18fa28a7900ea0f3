"""Builds paper_2503_05447_b200/lib/liblmoe_cuda.so (the C-ABI library) with nvcc for
sm_100a, in-tree, so the .so travels to the GPU box with the repo snapshot.

    python -m paper_2503_05447_b200._build [--force]
"""
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "build")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "liblmoe_cuda.so")
CPP_API_BIN = os.path.join(LIBDIR, "lsm_cpp_api")

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
          "-Xptxas", "-v", "-I" + os.path.join(ROOT, "include")]
SOURCES = ["common.cu", "lsm_host.cu", "lsm_combine.cu", "lsm_bwd_kernels.cu", "lsm_dgate.cu", "lsm_inst_bf16.cu", "lsm_inst_f32.cu", "lsm_inst_vec.cu", "lsm_vec_bwd.cu", "lsm_recurrent.cu", "lsm_fused.cu",
           "moe_host.cu", "attn.cu", "block.cu"]
LIBS = ["-lnccl"]


def _sources():
    return [os.path.join(CSRC, s) for s in SOURCES]


def _deps():
    out = []
    for d in (CSRC, os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "cpp")):
        for r, _, fs in os.walk(d):
            out += [os.path.join(r, f) for f in fs if f.endswith((".cu", ".cuh", ".h", ".hpp", ".cpp"))]
    return out


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(f) <= t for f in _deps() + [__file__])


def _compile(src):
    obj = os.path.join(BUILD, os.path.basename(src) + ".o")
    cmd = [NVCC] + ARCH + CFLAGS + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(BUILD, os.path.basename(src) + ".log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed for %s:\n%s" % (src, r.stderr[-6000:]))
    return obj


def build(force=False, verbose=False):
    if not force and up_to_date():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    os.makedirs(LIBDIR, exist_ok=True)
    with ThreadPoolExecutor(max_workers=min(8, len(SOURCES))) as ex:
        objs = list(ex.map(_compile, _sources()))
    tmp = LIB + ".tmp"
    cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + objs + LIBS
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n" + r.stderr[-4000:])
    os.replace(tmp, LIB)
    # C++ consumer of include/lmoe/cuda.hpp (drop-in API), run by tests/test_cpp_api.py
    src = os.path.join(ROOT, "tests", "cpp", "lsm_cpp_api.cpp")
    if os.path.exists(src):
        cmd = [NVCC, "-std=c++17", "-O2", "-I" + os.path.join(ROOT, "include"), src, "-o", CPP_API_BIN,
               "-L" + LIBDIR, "-llmoe_cuda", "-Xlinker", "-rpath=" + LIBDIR, "-Xlinker", "-rpath=$ORIGIN"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("C++ API test build failed:\n" + r.stderr[-3000:])
    if verbose:
        for s in SOURCES:
            with open(os.path.join(BUILD, s + ".log")) as f:
                print(f.read()[-3000:])
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
