"""The boundary from plain C: examples/layout_grid.c links libfdl.so with gcc
(no Python, no torch on the path) -- input validation runs without a GPU; the
full layout of the C1 grid runs on the GPU and is checked against the fp64
oracle from the same initial placement."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1711_01228_b200", "lib")


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    from paper_1711_01228_b200 import fdl  # noqa: F401  (builds / checks the library)
    out = str(tmp_path_factory.mktemp("cabi") / "layout_grid")
    cmd = ["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "examples", "layout_grid.c"), "-o", out, "-L", LIBDIR, "-lfdl",
           f"-Wl,-rpath,{LIBDIR}", "-lm"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return out


def test_c_program_validation_errors(exe):
    r = subprocess.run([exe, "--check-errors"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "disconnected: FDL_E_DISCONNECTED, ctx NULL" in r.stdout
    assert "self loop: FDL_E_SELF_LOOP" in r.stdout and "abi 3 ok" in r.stdout


@pytest.mark.gpu
def test_c_program_lays_out_the_c1_grid(exe):
    r = subprocess.run([exe, "10", "10"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    m = re.search(r"(\d+) iterations, (\d+) relaxations accepted, (\d+) PCG iterations, f (\S+) -> (\S+)", r.stdout)
    assert m, r.stdout
    it, acc, cg, f0, f1 = int(m.group(1)), int(m.group(2)), int(m.group(3)), float(m.group(4)), float(m.group(5))
    assert 1 < it <= 500 and acc <= it and cg > 0 and f1 < f0
    assert "x_0 = (0, 0)" in r.stdout  # the pinned vertex


@pytest.mark.gpu
def test_c_program_matches_the_oracle(exe, tmp_path):
    """The plain-C run of C1 from X0 (seed 1's placement, passed as a file)
    against oracle/layout.py's Algorithm 2 from the same X0: the §8(c)
    end-to-end gates (final f within 1e-3, iterations within max(1, 2%))."""
    import math

    import numpy as np

    from oracle import layout
    from workloads import configs
    cfg = configs.CONFIGS["C1"]
    g = configs.graph_for("C1")
    k = cfg.k_for(g.n)
    X0 = configs.positions_for("C1", g.n, 1)
    x0f, outf = tmp_path / "x0.bin", tmp_path / "x.bin"
    np.ascontiguousarray(X0, dtype=np.float64).tofile(x0f)
    r = subprocess.run([exe, "10", "10", str(x0f), str(outf)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    m = re.search(r"(\d+) iterations, (\d+) relaxations accepted, (\d+) PCG iterations, f (\S+) -> (\S+)", r.stdout)
    it, f1 = int(m.group(1)), float(m.group(5))
    X = np.fromfile(outf, dtype=np.float64).reshape(g.n, 2)
    o = layout.run_algorithm2(layout.Problem(g, 2, k), X0, 1.5, cfg.tol, cfg.max_iter)
    assert abs(f1 - o.f) / o.f <= 1e-3, (f1, o.f)
    assert abs(it - o.iterations) <= max(1, math.ceil(0.02 * o.iterations)), (it, o.iterations)
    assert X[0].tolist() == [0.0, 0.0]
    prob = layout.Problem(g, 2, k)
    assert abs(prob.f(X) - f1) / f1 <= 1e-6  # the written placement is the reported one
