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


REF_BLOCK = os.path.join(ROOT, "oracle", "_ref", "ett_bench_bridges")


def _ref_block():
    if not os.path.exists(REF_BLOCK):
        pytest.skip("oracle/_ref/ett_bench_bridges not built (needs /root/reference at build time)")
    return REF_BLOCK


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ["tv", "ck", "hybrid", "dfs"])
def test_reference_harness_bridges_block_runs_on_shim(ett, tmp_path, engine):
    """The reference's own caller -- tools/ett_bench.cpp:113-121 (bridge_engine)
    and :303-339 (load, largest_component, build_adjacency, timed engine(adj,
    &phases) loop, CSV rows per phase, dfs verification) -- compiled unchanged
    against include/ettg.hpp by oracle/ref_bench_block.py, runs on the B200."""
    import numpy as np
    exe = _ref_block()
    g, truth = ett.planted_bridge_graph(20_000, 120_000, 300, 4)
    # a second, smaller component: the block keeps the largest
    extra = np.array([[g.n, g.n + 1], [g.n + 1, g.n + 2]], np.int64)
    txt = ett.write_edge_list(ett.EdgeList(g.n + 3, np.concatenate([g.edges, extra])))
    path = tmp_path / "g.txt"
    path.write_bytes(txt)
    r = subprocess.run([exe, str(path), engine, "2"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert "kept largest component" in r.stderr
    assert f"bridge count: {int(truth.sum())}" in r.stderr
    assert "verified mask against dfs" in r.stderr
    rows = [l.split(",") for l in r.stdout.strip().splitlines()[1:]]
    phases = [row[11] for row in rows if row[9] == "0"]
    want = {"tv": ["spanning", "euler", "lowhigh", "total"],
            "ck": ["spanning", "marking", "total"],
            "hybrid": ["spanning", "euler", "marking", "total"],
            "dfs": ["spanning", "marking", "total"]}[engine]
    assert phases == want
    assert all(int(row[3]) == g.m() for row in rows)


def test_reference_harness_block_links(tmp_path):
    """CPU: the generated harness binary links against libettg.so (no GPU call)."""
    exe = _ref_block()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=60)
    assert r.returncode == 2 and "usage" in r.stderr
