"""In-tree build of libsige_b200.so for sm_100a (nvcc + g++, no JIT cache).

Compiles paper_2211_02048_b200/csrc/*.cu with
``-gencode arch=compute_100a,code=sm_100a -lineinfo`` and *.cpp with g++,
links a shared library with the static CUDA runtime into
``paper_2211_02048_b200/lib/libsige_b200.so``. Incremental on mtimes.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import pathlib
import subprocess
import sys

PKG = pathlib.Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = PKG / "build"
LIB = PKG / "lib" / "libsige_b200.so"
CUDA = pathlib.Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = str(CUDA / "bin" / "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
INC = [f"-I{ROOT / 'include'}", f"-I{CSRC}"]
# Bit-exact kernels must not contract a*b+c into FMA (reference build flag
# -ffp-contract=off, proj/CMakeLists.txt:11-13); the tensor-core kernel keeps
# explicit __f*_rn intrinsics for every epilogue op, so the flag is uniform.
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "--fmad=false", "-Xcompiler", "-fPIC",
                     "-Xptxas", "-warn-spills", "--expt-relaxed-constexpr"] + INC
CXX_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-Wall", "-Wno-unused-function",
             f"-I{CUDA / 'include'}"] + INC


def _headers_mtime() -> float:
    hs = list(CSRC.glob("*.h")) + list(CSRC.glob("*.hpp")) + list(CSRC.glob("*.cuh"))
    hs += list((ROOT / "include").glob("*.h"))
    return max((h.stat().st_mtime for h in hs), default=0.0)


def _compile(src: pathlib.Path, hdr_mtime: float, verbose: bool) -> pathlib.Path:
    obj = BUILD / (src.name + ".o")
    if obj.exists() and obj.stat().st_mtime > max(src.stat().st_mtime, hdr_mtime):
        return obj
    if src.suffix == ".cu":
        cmd = [NVCC, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)]
    else:
        cmd = ["g++", *CXX_FLAGS, "-c", str(src), "-o", str(obj)]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {src.name}\n{r.stdout}\n{r.stderr}")
    if r.stderr.strip() and verbose:
        print(r.stderr, file=sys.stderr)
    return obj


def build(verbose: bool = False) -> pathlib.Path:
    BUILD.mkdir(exist_ok=True)
    LIB.parent.mkdir(exist_ok=True)
    srcs = sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp"))
    hm = _headers_mtime()
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        objs = list(ex.map(lambda s: _compile(s, hm, verbose), srcs))
    if not LIB.exists() or LIB.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(LIB), *map(str, objs),
               "-lpthread", "-ldl", "-lrt"]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed\n{r.stdout}\n{r.stderr}")
        # a shared library links with unresolved symbols; ours must have none
        u = subprocess.run(["nm", "-D", "--undefined-only", str(LIB)], capture_output=True, text=True)
        missing = [ln.split()[-1] for ln in u.stdout.splitlines() if "sige_b200" in ln]
        if missing:
            LIB.unlink()
            raise RuntimeError(f"link left library symbols unresolved: {missing}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
