"""In-tree build of the native library (libpm_tridiag.so) for sm_100a.

nvcc compiles every CUDA / C++ source under csrc/ with
``-gencode arch=compute_100a,code=sm_100a -lineinfo`` and links one shared
library next to this file, so the built .so travels with the repository
snapshot to the GPU box.  No torch types cross this library's ABI.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
BUILD = ROOT / "build" / "obj"
LIB = PKG / "libpm_tridiag.so"
CLI_SRC = PKG / "cli" / "streamtune_cli.cpp"
CLI = PKG / "bin" / "streamtune"
# extra nvcc flags (experiments only), e.g. PM_NVCC_FLAGS="-DPM_SOLVE_MINB=3"
EXTRA = os.environ.get("PM_NVCC_FLAGS", "").split()

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libpm_tridiag.so")


def sources() -> list[Path]:
    out = sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("**/*.cpp"))
    return out


def headers() -> list[Path]:
    return (sorted(CSRC.glob("**/*.h")) + sorted(CSRC.glob("**/*.cuh")) + sorted(CSRC.glob("**/*.inc")) +
            sorted(INCLUDE.glob("**/*.h*")))


def _compile(src: Path) -> Path:
    rel = src.relative_to(CSRC)
    obj = BUILD / (str(rel).replace("/", "__") + ".o")
    obj.parent.mkdir(parents=True, exist_ok=True)
    # every object depends on every source and header: pm_kernels_f32.cu
    # #includes pm_kernels.cu, so a per-file check would miss its edits
    newest_dep = max([p.stat().st_mtime for p in sources()] + [h.stat().st_mtime for h in headers()])
    if obj.exists() and obj.stat().st_mtime >= newest_dep:
        return obj
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", *EXTRA,
           f"-I{INCLUDE}", f"-I{CSRC}", "-c", str(src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{res.stdout}\n{res.stderr}")
    return obj


def build(verbose: bool = False, out: Path | None = None) -> Path:
    global BUILD, LIB
    if out is not None:  # variant build (experiments): separate objects and library
        BUILD = ROOT / "build" / ("obj_" + out.stem)
        LIB = out
    srcs = sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(_compile, srcs))
    newest = max(o.stat().st_mtime for o in objs)
    if not LIB.exists() or LIB.stat().st_mtime < newest:
        tmp = LIB.with_suffix(".so.tmp")
        cmd = [nvcc(), *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcudart_static",
               "-ldl", "-lrt", "-lpthread"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
        os.replace(tmp, LIB)
    if out is None:
        build_cli(verbose)
    if verbose:
        print(f"built {LIB}", file=sys.stderr)
    return LIB


def build_cli(verbose: bool = False) -> Path:
    """The `streamtune` command-line tool, a C++ executable
    linked against libpm_tridiag.so (rpath $ORIGIN/..)."""
    deps = [CLI_SRC, LIB] + headers()
    if CLI.exists() and CLI.stat().st_mtime >= max(d.stat().st_mtime for d in deps):
        return CLI
    CLI.parent.mkdir(parents=True, exist_ok=True)
    cxx = shutil.which("g++") or "g++"
    cmd = [cxx, "-std=c++17", "-O2", f"-I{INCLUDE}", str(CLI_SRC), f"-L{PKG}", "-lpm_tridiag",
           "-Wl,-rpath,$ORIGIN/..", "-o", str(CLI)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"streamtune CLI build failed:\n{res.stdout}\n{res.stderr}")
    if verbose:
        print(f"built {CLI}", file=sys.stderr)
    return CLI


if __name__ == "__main__":
    build(verbose=True, out=Path(sys.argv[1]).resolve() if len(sys.argv) > 1 else None)
