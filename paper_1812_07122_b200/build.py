"""Build the sm_100a CUDA library ``_lib/libblfls.so`` in-tree with nvcc.

The shared object exposes only the C ABI declared in include/blfls/blfls.h.
It is git-ignored but travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_lib"
LIB = OUT_DIR / "libblfls.so"
INCLUDE = ROOT / "include"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
         "--expt-relaxed-constexpr", f"-I{INCLUDE}", f"-I{CSRC}"]


def _sources():
    return sorted(CSRC.glob("*.cu"))


def _headers():
    return sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.rglob("*.h"))


def _needs(obj: Path, src: Path) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return any(p.stat().st_mtime > t for p in [src, *_headers(), Path(__file__)])


CLI_SRC = ROOT / "tools" / "blfls_cli.cpp"
CLI = OUT_DIR / "blfls"


def build_cli(verbose: bool = False) -> Path:
    """The epls-style command-line front end (tools/blfls_cli.cpp) over libblfls.so."""
    if CLI.exists() and CLI.stat().st_mtime > max(CLI_SRC.stat().st_mtime, LIB.stat().st_mtime,
                                                   (INCLUDE / "blfls" / "blfls.hpp").stat().st_mtime):
        return CLI
    cmd = ["g++", "-std=c++17", "-O2", f"-I{INCLUDE}", str(CLI_SRC), "-o", str(CLI), f"-L{OUT_DIR}",
           "-lblfls", f"-Wl,-rpath,$ORIGIN"]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"g++ failed:\n{r.stdout}\n{r.stderr}")
    return CLI


BENCH_SRC = ROOT / "tools" / "blfls_bench.cpp"
BENCH = OUT_DIR / "blfls_bench"
CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))


def build_bench(verbose: bool = False) -> Path:
    """The C++ host end-to-end benchmark (tools/blfls_bench.cpp) over libblfls.so."""
    if BENCH.exists() and BENCH.stat().st_mtime > max(BENCH_SRC.stat().st_mtime, LIB.stat().st_mtime,
                                                       (INCLUDE / "blfls" / "blfls.hpp").stat().st_mtime):
        return BENCH
    cmd = ["g++", "-std=c++17", "-O2", "-pthread", f"-I{INCLUDE}", f"-I{CUDA_HOME / 'include'}", str(BENCH_SRC),
           "-o", str(BENCH), f"-L{OUT_DIR}", "-lblfls", f"-L{CUDA_HOME / 'lib64'}", "-lcudart",
           f"-Wl,-rpath,$ORIGIN", f"-Wl,-rpath,{CUDA_HOME / 'lib64'}"]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"g++ failed:\n{r.stdout}\n{r.stderr}")
    return BENCH


EXP_DIR = PKG / "_lib_exp"


def build(verbose: bool = False, ptxas_info: bool = False, experiments: bool = False) -> Path:
    """experiments=True: an A/B build with -DBLFLS_EXPERIMENTS into _lib_exp/
    (kernel-selection knobs read from BLFLS_* environment variables; load it
    with BLFLS_LIBRARY=<path>).  The production library never reads them."""
    out_dir = EXP_DIR if experiments else OUT_DIR
    lib_path = out_dir / "libblfls.so"
    out_dir.mkdir(exist_ok=True)
    objs = []
    jobs = []
    for src in _sources():
        obj = out_dir / (src.stem + ".o")
        objs.append(obj)
        if _needs(obj, src) or ptxas_info:
            extra = os.environ.get("BLFLS_EXP_DEFINES", "").split() if experiments else []
            cmd = [NVCC, *ARCH, *FLAGS, *(["-DBLFLS_EXPERIMENTS"] if experiments else []), *extra, "-c",
                   str(src), "-o", str(obj)]
            if ptxas_info:
                cmd += ["-Xptxas", "-v"]
            jobs.append(cmd)

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        return r.stderr

    with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        for err in ex.map(run, jobs):
            if ptxas_info and err:
                sys.stderr.write(err)
    if jobs or not lib_path.exists():
        cmd = [NVCC, *ARCH, "-shared", "-o", str(lib_path), *map(str, objs), "-cudart", "static"]
        run(cmd)
    if experiments:
        return lib_path
    build_cli(verbose)
    build_bench(verbose)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True, ptxas_info="-v" in sys.argv, experiments="--experiments" in sys.argv))
