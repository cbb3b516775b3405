"""Build libhobbit.so (all CUDA/C++ sources of csrc/) in-tree for sm_100a.

    python -m paper_2411_01433_b200.build [-v]
    python -m paper_2411_01433_b200.build --variant NAME -DMACRO=VAL ...   (experiments)

Every translation unit is compiled by nvcc with
-gencode arch=compute_100a,code=sm_100a -lineinfo -O3 (no fast-math: the
quantiser and the exact router rely on IEEE fp32 / integer semantics), then
linked into one shared library next to this file.  Object files go to
build/ and are rebuilt only when a source or header is newer.  A --variant
build goes to build/variants/NAME/libhobbit.so (load it with HOBBIT_LIB=...).
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
OUT = os.path.join(PKG, "libhobbit.so")
BUILD = os.path.join(ROOT, "build", "obj")
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I", INCLUDE, "-I", CSRC,
         "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _headers():
    return glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(INCLUDE, "*.h"))


def _compile(src, objdir, defines, verbose):
    obj = os.path.join(objdir, os.path.basename(src) + ".o")
    newest = max([os.path.getmtime(src)] + [os.path.getmtime(h) for h in _headers()])
    if os.path.exists(obj) and os.path.getmtime(obj) >= newest:
        return obj, ""
    lang = ["-x", "cu"] if src.endswith(".cpp") else []
    cmd = [NVCC] + lang + ARCH + FLAGS + list(defines) + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr if verbose else ""


def build(verbose: bool = False, variant: str | None = None, defines=()) -> str:
    objdir = BUILD if variant is None else os.path.join(ROOT, "build", "variants", variant, "obj")
    out = OUT if variant is None else os.path.join(ROOT, "build", "variants", variant, "libhobbit.so")
    os.makedirs(objdir, exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        results = list(ex.map(lambda s: _compile(s, objdir, defines, verbose), srcs))
    objs = [o for o, _ in results]
    for _, log in results:
        if log:
            print(log)
    newest = max(os.path.getmtime(o) for o in objs)
    if not os.path.exists(out) or os.path.getmtime(out) < newest:
        cmd = [NVCC] + ARCH + ["-shared", "-o", out] + objs + [
            "-L", os.path.join(CUDA_HOME, "lib64"), "-lcudart",
            "-Xlinker", "-rpath," + os.path.join(CUDA_HOME, "lib64")]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return out


if __name__ == "__main__":
    args = sys.argv[1:]
    variant = None
    if "--variant" in args:
        variant = args[args.index("--variant") + 1]
    defines = [a for a in args if a.startswith("-D")]
    print(build(verbose="-v" in args, variant=variant, defines=defines))
