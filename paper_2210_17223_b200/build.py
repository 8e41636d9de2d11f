"""Build liblina.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python paper_2210_17223_b200/build.py          # incremental
    python paper_2210_17223_b200/build.py --clean  # (run by path: importing the package loads the library)

Every .cu/.cpp under csrc/ is compiled with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` and linked against the
NCCL that torch loads (the venv's nvidia/nccl, 2.28.9 — not /usr/include's 2.27).
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "liblina.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dir() -> str:
    import nvidia.nccl  # the copy torch loads
    base = list(nvidia.nccl.__path__)[0]
    return base


def _flags():
    nd = nccl_dir()
    inc = ["-I" + os.path.join(nd, "include"), "-I" + CSRC, "-I" + os.path.join(ROOT, "include")]
    return inc, nd


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cpp")) + glob.glob(os.path.join(CSRC, "*.cu")) +
                  glob.glob(os.path.join(CSRC, "kernels", "*.cu")))


def _headers_mtime() -> float:
    hs = glob.glob(os.path.join(CSRC, "**", "*.h"), recursive=True) + [os.path.join(ROOT, "include", "lina.h")]
    return max(os.path.getmtime(h) for h in hs)


def _obj_for(src: str) -> str:
    rel = os.path.relpath(src, CSRC).replace(os.sep, "_")
    return os.path.join(OBJ, rel + ".o")


def _compile(src: str, inc, verbose: bool) -> str:
    obj = _obj_for(src)
    cmd = [NVCC, *ARCH, "-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
           "--expt-relaxed-constexpr", "-Xptxas", "-v" if os.environ.get("LINA_PTXAS_V") else "-O3",
           *inc, "-c", src, "-o", obj]
    if src.endswith(".cpp"):
        cmd.insert(1, "-x")
        cmd.insert(2, "cu")
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if os.environ.get("LINA_PTXAS_V") and r.stderr:
        print(r.stderr, file=sys.stderr)
    return obj


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    inc, nd = _flags()
    hdr = _headers_mtime()
    todo = []
    objs = []
    for s in sources():
        o = _obj_for(s)
        objs.append(o)
        if force or not os.path.exists(o) or os.path.getmtime(o) < max(os.path.getmtime(s), hdr):
            todo.append(s)
    if todo:
        with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
            list(ex.map(lambda s: _compile(s, inc, verbose), todo))
    need_link = force or bool(todo) or not os.path.exists(LIB) or \
        os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs)
    if need_link:
        libdir = os.path.join(nd, "lib")
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-L" + libdir, "-l:libnccl.so.2",
               "-Xlinker", "-rpath=" + libdir, "-lcuda" if False else "-lcudart_static", "-lpthread",
               "-ldl", "-lrt"]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


def clean():
    shutil.rmtree(os.path.join(ROOT, "build"), ignore_errors=True)
    if os.path.exists(LIB):
        os.remove(LIB)


if __name__ == "__main__":
    if "--clean" in sys.argv:
        clean()
    print(build(verbose="-v" in sys.argv, force="--force" in sys.argv))
