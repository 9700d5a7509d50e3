"""Build libpacim.so (sm_100a) in-tree with nvcc.

    python -m paper_2311_07554_b200.build [--force] [--verbose]
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libpacim.so")
SOURCES = ["api.cu", "graph.cu", "build.cu", "select.cu", "compressed.cu", "mc.cu", "store_cs.cu",
           "dist.cu"]

# NCCL: the venv's (the same 2.28 build torch.distributed loads)
def _nccl_dir() -> str:
    import site
    for sp in site.getsitepackages() + [site.getusersitepackages()]:
        d = os.path.join(sp, "nvidia", "nccl")
        if os.path.isdir(os.path.join(d, "include")):
            return d
    raise RuntimeError("NCCL headers not found (nvidia/nccl in site-packages)")


NCCL_DIR = _nccl_dir()

HEADERS = ["pacim_internal.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"),
         "-I", os.path.join(NCCL_DIR, "include")] + os.environ.get("PACIM_NVCC_EXTRA", "").split()


def _stale(lib: str, deps: list[str]) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [
        os.path.join(ROOT, "include", "pacim.h"), os.path.abspath(__file__)]
    if not force and not _stale(LIB, deps):
        return LIB
    os.makedirs(BUILD, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(BUILD, src.replace(".cu", ".o"))
        cmd = [NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        if verbose:
            sys.stderr.write(r.stderr)
        return obj

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = LIB + ".tmp"
    nlib = os.path.join(NCCL_DIR, "lib")
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart", "-L", nlib, "-l:libnccl.so.2",
           "-Xlinker", "-rpath=" + nlib]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
