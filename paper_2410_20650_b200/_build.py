"""In-tree build of libnzgpu.so (sm_100a) with nvcc.

Every .cu under csrc/ is compiled for -gencode arch=compute_100a,code=sm_100a
with -lineinfo (ncu source mapping), the nvcc IEEE defaults kept explicit
(-ftz=false -prec-div=true -prec-sqrt=true; never --use_fast_math: the lossy
path's __fdiv_rn/__fmul_rn must stay bit-exact with the reference), and
linked into one shared library with a static CUDA runtime so it loads next to
torch without library-path games.  nvcc cross-compiles without a GPU.

Tuning variants (dev only): ``python _build.py --define NZ_CHAINS=4 --out
libnzgpu_ch4.so`` builds a side library in build_<tag>/ that
``NZGPU_LIB=<path>`` can point the package at."""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libnzgpu.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v", "-I", os.path.join(HERE, "..", "include")]


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _stale(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    deps = [src] + [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".cuh", ".h"))]
    deps.append(os.path.join(HERE, "..", "include", "nzgpu.h"))
    return any(os.path.getmtime(d) > os.path.getmtime(obj) for d in deps if os.path.exists(d))


def _compile(args) -> tuple[str, str]:
    src, build_dir, defines = args
    obj = os.path.join(build_dir, os.path.basename(src)[:-3] + ".o")
    if not _stale(obj, src):
        return obj, ""
    cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-c", src, "-o", obj]
    out = subprocess.run(cmd, capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{out.stdout}\n{out.stderr}")
    return obj, out.stderr


def build(verbose: bool = False, defines=(), lib: str = LIB) -> str:
    tag = "_".join(d.replace("=", "") for d in defines)
    build_dir = os.path.join(HERE, "build" + (("_" + tag) if tag else ""))
    os.makedirs(build_dir, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        results = list(ex.map(_compile, [(s, build_dir, list(defines)) for s in sources()]))
    objs = [o for o, _ in results]
    if verbose:
        for _, log in results:
            if log:
                sys.stderr.write(log)
    if not os.path.exists(lib) or any(os.path.getmtime(o) > os.path.getmtime(lib) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", lib, *objs]
        out = subprocess.run(cmd, capture_output=True, text=True)
        if out.returncode != 0:
            raise RuntimeError(f"link failed:\n{out.stdout}\n{out.stderr}")
    if lib == LIB:
        build_cli()
        build_tool(DROPIN_BENCH_SRC, DROPIN_BENCH)
    return lib


CLI_SRC = os.path.join(HERE, "..", "tools", "neuzip_cli.cpp")
CLI = os.path.join(HERE, "neuzip")
DROPIN_BENCH_SRC = os.path.join(HERE, "..", "tools", "dropin_bench.cpp")
DROPIN_BENCH = os.path.join(HERE, "dropin_bench")


def build_tool(src: str, exe: str) -> str:
    """A host tool on the drop-in headers, linked against the in-tree
    libnzgpu.so (rpath $ORIGIN)."""
    deps = [src, LIB, os.path.join(HERE, "..", "include", "nzgpu.h")] + [
        os.path.join(HERE, "..", "include", "neuzip", f) for f in os.listdir(os.path.join(HERE, "..", "include", "neuzip"))]
    if os.path.exists(exe) and all(os.path.getmtime(exe) >= os.path.getmtime(d) for d in deps):
        return exe
    cmd = ["g++", "-std=c++20", "-O2", "-pthread", "-Wall", "-Wextra", "-I", os.path.join(HERE, "..", "include"),
           src, "-o", exe, "-L", HERE, "-lnzgpu", "-Wl,-rpath,$ORIGIN"]
    out = subprocess.run(cmd, capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError(f"{os.path.basename(exe)} build failed:\n{out.stdout}\n{out.stderr}")
    return exe


def build_cli() -> str:
    """The `neuzip` command-line tool (analyze / compress / decompress /
    bench, proj/tools/neuzip.cpp) on the C ABI and the drop-in headers."""
    return build_tool(CLI_SRC, CLI)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("-v", action="store_true")
    ap.add_argument("--define", action="append", default=[])
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    out = os.path.join(HERE, a.out) if a.out else LIB
    print(build(verbose=a.v, defines=a.define, lib=out))
