"""include/hdgb200.hpp -- the C++ mirror of the reference's namespace-hdg API over the C ABI -- compiles with
plain g++ against libhdgb200.so (CPU check) and reproduces the reference's calls and error behaviour on the
GPU (tests/cpp/test_cpp_layer.cpp: newton_solve, assemble_*, block_matvec, gmres_solve, lu_invert_batch with the
lowest singular batch index, DimensionMismatch)."""
import os
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
LIB = ROOT / "paper_2512_13619_b200" / "lib"
EXE = ROOT / "tests" / "cpp" / "_build" / "test_cpp_layer"


def build():
    if not (LIB / "libhdgb200.so").exists():
        pytest.skip("libhdgb200.so not built")
    EXE.parent.mkdir(parents=True, exist_ok=True)
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    cmd = ["g++", "-std=c++17", "-O1", "-Wall", "-Werror", f"-I{ROOT / 'include'}", str(ROOT / "tests" / "cpp" / "test_cpp_layer.cpp"),
           "-o", str(EXE), f"-L{LIB}", "-lhdgb200", f"-L{cuda}/lib64", "-lcudart", f"-Wl,-rpath,{LIB}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return EXE


def test_cpp_layer_compiles_and_links():
    assert build().exists()


@pytest.mark.gpu
def test_cpp_layer_runs_the_reference_calls_on_the_gpu():
    exe = build()
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all checks passed" in r.stdout
