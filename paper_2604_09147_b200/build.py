"""Build libhh.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed).

    python -m paper_2604_09147_b200.build            # incremental
    python -m paper_2604_09147_b200.build --force
    python -m paper_2604_09147_b200.build --variant NAME -DHH_MV_CVT=1 ...   # side-by-side
      experiment build -> libhh_NAME.so (load it with HH_LIB=<path>); not the product build
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libhh.so")
SOURCES = ["api.cu", "tree.cu", "partition.cpp", "compress.cu", "compress_big.cu", "dense.cu", "layout.cpp",
           "matvec.cu"]
HEADERS = ["common.cuh", "handle.h", "build.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall", "--expt-relaxed-constexpr",
         "-I", os.path.join(os.path.dirname(HERE), "include")]


def _stale(src, obj):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    deps = [src] + [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(os.path.dirname(HERE), "include", "hh.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(name, force, verbose_ptxas, objdir=OBJ, defines=()):
    src = os.path.join(CSRC, name)
    obj = os.path.join(objdir, name + ".o")
    if not force and not _stale(src, obj):
        return obj, ""
    cmd = [NVCC, *FLAGS, *defines, "-c", src, "-o", obj]
    if verbose_ptxas and name.endswith(".cu"):
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {name}:\n{r.stderr}")
    return obj, r.stderr


def build(force: bool = False, verbose_ptxas: bool = False, variant: str | None = None, defines=()) -> str:
    objdir, lib = OBJ, LIB
    if variant:
        objdir = os.path.join(OBJ, "variant_" + variant)
        lib = os.path.join(HERE, f"libhh_{variant}.so")
    os.makedirs(objdir, exist_ok=True)
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        outs = list(ex.map(lambda s: _compile(s, force, verbose_ptxas, objdir, defines), SOURCES))
    objs = [o for o, _ in outs]
    if verbose_ptxas:
        for _, log in outs:
            if log:
                print(log, file=sys.stderr)
    if force or not os.path.exists(lib) or any(os.path.getmtime(o) > os.path.getmtime(lib) for o in objs):
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib, *objs, "-lcudart", "-lcublas",
               "-lcusolver"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return lib


if __name__ == "__main__":
    var = sys.argv[sys.argv.index("--variant") + 1] if "--variant" in sys.argv else None
    defs = [a for a in sys.argv if a.startswith("-D")]
    print(build(force="--force" in sys.argv or bool(var), verbose_ptxas="-v" in sys.argv, variant=var, defines=defs))
