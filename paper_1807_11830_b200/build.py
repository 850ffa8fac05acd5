"""In-tree build of libhetreco_b200.so (sm_100a kernels + C++ host library +
C-ABI).  nvcc cross-compiles for sm_100a without a GPU, so this runs in the
CPU container; the resulting .so travels to the GPU box with the snapshot.

    python -m paper_1807_11830_b200.build [--force]
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libhetreco_b200.so")
CLI = os.path.join(PKG, "bin", "hetreco")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-std=c++20", "--expt-relaxed-constexpr", "-O3", "-lineinfo", "-Xcompiler", "-fPIC",
              "-Xcompiler", "-fvisibility=hidden",
              "-Xptxas", "-warn-spills", "-I", INCLUDE] + ARCH
CXX_FLAGS = ["-std=c++20", "-O2", "-fPIC", "-fvisibility=hidden", "-Wall", "-Wno-unused-function", "-I", INCLUDE,
             "-I", os.path.join(CUDA, "include")]


def _sources():
    cu = sorted(glob.glob(os.path.join(CSRC, "kernels", "*.cu")))
    cpp = sorted(glob.glob(os.path.join(CSRC, "host", "*.cpp")))
    return cu, cpp


def _headers_mtime() -> float:
    hs = glob.glob(os.path.join(INCLUDE, "**", "*.h*"), recursive=True)
    hs += glob.glob(os.path.join(CSRC, "**", "*.h*"), recursive=True)
    hs += glob.glob(os.path.join(CSRC, "**", "*.cuh"), recursive=True)
    return max((os.path.getmtime(h) for h in hs), default=0.0)


def _compile(src: str, force: bool, hdr_mtime: float) -> str:
    rel = os.path.relpath(src, CSRC).replace(os.sep, "_")
    obj = os.path.join(OBJ, rel + ".o")
    if (not force and os.path.exists(obj)
            and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_mtime)):
        return obj
    if src.endswith(".cu"):
        cmd = [NVCC] + NVCC_FLAGS + ["-c", src, "-o", obj]
    else:
        cmd = ["g++"] + CXX_FLAGS + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if r.stderr.strip():
        sys.stderr.write(r.stderr)
    return obj


def build(force: bool = False, verbose: bool = True) -> str:
    os.makedirs(OBJ, exist_ok=True)
    cu, cpp = _sources()
    hm = _headers_mtime()
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        objs = list(ex.map(lambda s: _compile(s, force, hm), cu + cpp))
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        tmp = LIB + f".{os.getpid()}.tmp"
        cmd = [NVCC, "-shared", "-cudart", "static", "-Xlinker", "-soname=libhetreco_b200.so", "-o", tmp] + ARCH + \
            objs + ["-lpthread", "-ldl", "-lrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, LIB)
        if verbose:
            print("built", LIB)
    build_cli(force, verbose)
    return LIB


def build_cli(force: bool = False, verbose: bool = True) -> str:
    """The `hetreco` command-line front-end (csrc/cli), linked against the
    exported C-ABI of libhetreco_b200.so (rpath $ORIGIN/..)."""
    srcs = sorted(glob.glob(os.path.join(CSRC, "cli", "*.cpp")))
    os.makedirs(os.path.dirname(CLI), exist_ok=True)
    newest = max([os.path.getmtime(x) for x in srcs] + [os.path.getmtime(LIB), _headers_mtime()])
    if not force and os.path.exists(CLI) and os.path.getmtime(CLI) >= newest:
        return CLI
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-I", INCLUDE, "-o", CLI] + srcs + \
        ["-L", PKG, "-l:libhetreco_b200.so", "-Wl,-rpath,$ORIGIN/.."]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"cli build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if verbose:
        print("built", CLI)
    return CLI


if __name__ == "__main__":
    build(force="--force" in sys.argv)
