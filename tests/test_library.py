"""CPU-only checks of the C-ABI library: it loads, exports every function
include/fdl.h declares, and its host-side logic (parameter defaults, graph
validation, row sharding) behaves as documented.  No compute call needs a GPU
here: graph validation runs before any CUDA call."""
import math
import os
import re

import numpy as np
import pytest

from paper_1711_01228_b200 import fdl
from workloads import graphs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "fdl.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fdl_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol():
    names = header_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(fdl.lib, name), name
    assert set(names) == set(fdl.EXPORTS)


def test_abi_version_and_defaults():
    assert fdl.lib.fdl_abi_version() == 3
    p = fdl.params_default()
    assert p.struct_size == 88 or p.struct_size == __import__("ctypes").sizeof(fdl.Params)
    assert p.dim == 2 and p.omega == 1.5 and math.isinf(p.step) and p.tol == 1e-4
    assert p.max_iter == 500 and p.weight_exp == -2.0 and p.strategy == fdl.STRAT_FIXED
    assert p.cg_extrap == 2 and p.cg_history == 0 and p.a_refresh == 10


def test_status_strings():
    for code, name in fdl.STATUS.items():
        assert fdl.lib.fdl_status_str(code).decode() == name


def _expect(status_name, n, rp, col, **kw):
    with pytest.raises(fdl.FdlError) as e:
        fdl.Layout(n, rp, col, **kw)
    assert e.value.name == status_name


def test_graph_validation_errors():
    # disconnected
    g = graphs.csr_from_edges(4, np.array([[0, 1], [2, 3]]))
    _expect("FDL_E_DISCONNECTED", g.n, g.row_ptr, g.col)
    # self-loop
    _expect("FDL_E_SELF_LOOP", 2, np.array([0, 2, 3]), np.array([0, 1, 0], dtype=np.int32))
    # duplicate neighbour
    _expect("FDL_E_DUPLICATE_EDGE", 2, np.array([0, 2, 4]), np.array([1, 1, 0, 0], dtype=np.int32))
    # missing reverse edge
    _expect("FDL_E_ASYMMETRIC", 3, np.array([0, 2, 3, 3]), np.array([1, 2, 0], dtype=np.int32))
    # out-of-range id
    _expect("FDL_E_INVALID_ARG", 2, np.array([0, 1, 2]), np.array([5, 0], dtype=np.int32))
    # n = 0
    _expect("FDL_E_INVALID_ARG", 0, np.array([0]), np.array([], dtype=np.int32))


def test_parameter_validation():
    g = graphs.path_graph(3)
    p = fdl.make_params(omega=-1.0)
    _expect("FDL_E_INVALID_ARG", g.n, g.row_ptr, g.col, params=p)
    p = fdl.make_params(dim=4)
    _expect("FDL_E_UNSUPPORTED", g.n, g.row_ptr, g.col, params=p)
    p = fdl.make_params(tol=0.0)
    _expect("FDL_E_INVALID_ARG", g.n, g.row_ptr, g.col, params=p)
    p = fdl.make_params()
    p.weight_exp = float("nan")
    _expect("FDL_E_INVALID_ARG", g.n, g.row_ptr, g.col, params=p)
    # edge lengths (NEXT-3): positive and finite per stored direction
    _expect("FDL_E_BAD_LENGTH", g.n, g.row_ptr, g.col, edge_len=np.array([1.0, 1.0, -2.0, -2.0]))
    _expect("FDL_E_BAD_LENGTH", g.n, g.row_ptr, g.col, edge_len=np.array([1.0, 1.0, np.inf, np.inf]))
    # ... and equal in the two stored directions of an edge: path 0-1-2 stores
    # (0,1), (1,0), (1,2), (2,1); edge (1,2) gets 2.0 one way and 3.0 the other
    assert list(g.col) == [1, 0, 2, 1]
    _expect("FDL_E_BAD_LENGTH", g.n, g.row_ptr, g.col, edge_len=np.array([1.0, 1.0, 2.0, 3.0]))
    p = fdl.make_params(strategy=fdl.STRAT_ENUM, weight_exp=-1.0)
    _expect("FDL_E_UNSUPPORTED", g.n, g.row_ptr, g.col, params=p)
    p = fdl.make_params(cg_history=9)  # recycled PCG start window: 0 (default 2) .. 8
    _expect("FDL_E_INVALID_ARG", g.n, g.row_ptr, g.col, params=p)
    p = fdl.make_params(cg_extrap=3)
    _expect("FDL_E_INVALID_ARG", g.n, g.row_ptr, g.col, params=p)
    p = fdl.make_params()
    p.struct_size = 3
    _expect("FDL_E_INVALID_ARG", g.n, g.row_ptr, g.col, params=p)


@pytest.mark.parametrize("n,world", [(1, 1), (100, 2), (1000, 3), (9828, 8), (200000, 8), (300, 8)])
def test_shard_tiles_partition(n, world):
    """Upper-triangle tiles split into contiguous ranges covering
    [0, nb(nb+1)/2) exactly once, with boundaries on global work items (strip
    segments of <= 16 tiles, 32 from 2^18 tiles on), so shares differ by at
    most one item."""
    nb = -(-n // fdl.FDL_TILE)
    total = nb * (nb + 1) // 2
    seg = 32 if total >= 1 << 18 else 16
    prev = 0
    sizes = []
    for r in range(world):
        a, b = fdl.shard_tiles(n, world, r)
        assert a == prev and a <= b <= total
        sizes.append(b - a)
        prev = b
    assert prev == total
    assert max(sizes) - min(sizes) <= 2 * seg or total < world * seg
