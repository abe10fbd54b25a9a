"""The C++ host API (include/blfls/blfls.hpp) compiles against the C ABI and,
on a GPU, behaves like the reference's entry points."""
from __future__ import annotations

import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
SRC = ROOT / "tests" / "cpp" / "host_api_test.cpp"
LIBDIR = ROOT / "paper_1812_07122_b200" / "_lib"


def _build(tmp: Path) -> Path:
    """The test program links libblfls.so (the product) and, as its checker,
    the CPU oracle oracle/liboracle.so (test infrastructure)."""
    from oracle import oracle as O
    from paper_1812_07122_b200 import build
    build.build()
    if not O.ORACLE_SO.exists():
        O.build(ref=False)
    odir = O.ORACLE_SO.parent
    exe = tmp / "host_api_test"
    subprocess.run(["g++", "-std=c++17", "-O2", "-pthread", f"-I{ROOT / 'include'}", str(SRC), "-o", str(exe),
                    f"-L{LIBDIR}", "-lblfls", f"-Wl,-rpath,{LIBDIR}", str(O.ORACLE_SO),
                    f"-Wl,-rpath,{odir}"], check=True)
    return exe


def test_cpp_host_api_compiles_and_links(tmp_path):
    exe = _build(tmp_path)
    assert exe.exists()


@pytest.mark.gpu
def test_cpp_host_api_runs(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    exe = _build(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout
