"""The C++ drop-in header (include/hytegrid_b200.hpp) compiles and links
against the C ABI on CPU; the program runs the reference's usage pattern on
the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_cpp_api.cpp")
BIN = os.path.join(ROOT, "build", "test_cpp_api")
LIBDIR = os.path.join(ROOT, "paper_1805_10167_b200")


def build():
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"), SRC,
                    os.path.join(LIBDIR, "libhyteg_b200.so"), f"-Wl,-rpath,{LIBDIR}", "-o", BIN], check=True)


def test_cpp_header_compiles_and_links():
    build()
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_cpp_api_runs_on_gpu():
    if not os.path.exists(BIN):
        build()
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "cpp api ok" in out.stdout
    # SolveReport::history(): the same text as the reference's for the same solve
    # (GridHierarchy on unit_square, levels 1..5, keyed U[-1,1] rhs seed 5, 6 cycles)
    from oracle import ref as R
    from tests.helpers import keyed_uniform
    if not R.available():
        pytest.skip("oracle/_ref not built")
    mine = out.stdout.split("HISTORY_BEGIN\n")[1].split("HISTORY_END")[0]
    mesh = R.meshgen("unit_square")
    r = R.RefSession(mesh, 1, 1, 5, 2)
    r.set(0, 5, keyed_uniform(mesh, 5, seed=5))
    res = r.gridhierarchy_solve(0, 1, 5, 0.0, 6)
    want = "".join(f"cycle {k} residual {v:.6e}\n" if k == 0 else
                   f"cycle {k} residual {v:.6e} factor {v / res[k - 1] if res[k - 1] > 0 else 0.0:.4f}\n"
                   for k, v in enumerate(res))
    assert mine == want, (mine, want)
