"""The boundary from plain C (examples/c_abi_example.c): compiles and links against
libadjprod.so and the CUDA runtime on the host; on a B200 it runs and checks sampled rows of
Low(A A^T) against the definition."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2101_01025_b200")


def _build(tmp_path):
    exe = str(tmp_path / "c_abi_example")
    subprocess.run(["gcc", "-std=c11", "-Wall", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
                    os.path.join(ROOT, "examples", "c_abi_example.c"), "-L", PKG, "-ladjprod",
                    "-L", "/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{PKG}", "-o", exe], check=True)
    return exe


def test_c_example_builds(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_c_example_runs(tmp_path):
    out = subprocess.run([_build(tmp_path)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "c_abi_example: OK" in out.stdout
