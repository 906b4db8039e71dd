"""The C++ shim (include/ettg.hpp) compiles against the C-ABI and, on a GPU,
answers like the reference's own tests."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2103_15217_b200", "_lib")


def _build(tmp_path):
    exe = str(tmp_path / "shim_test")
    cmd = ["/usr/bin/g++", "-std=c++17", "-O1", f"-I{ROOT}/include",
           os.path.join(ROOT, "tests", "cpp", "shim_test.cpp"), f"-L{LIBDIR}", "-lettg",
           f"-Wl,-rpath,{LIBDIR}", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_shim_compiles_and_links(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_shim_runs_on_gpu(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert "shim ok" in r.stdout
