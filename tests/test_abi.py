"""C-ABI boundary checks that run without a GPU: the library loads, exports every
symbol include/rsrs.h declares, the C++ tree equals the oracle tree, and the
compute entry points fail loudly (no CPU fallback) when no device is present."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle as O
import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lib():
    import paper_2311_01451_b200 as R
    return R


def _declared(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rsrs_\w+)\s*\(", src)))


def test_exports_every_declared_symbol():
    R = _lib()
    lib = ctypes.CDLL(R.LIB_PATH)
    decl = _declared("rsrs.h")
    assert sorted(R.EXPORTS) == decl
    for name in decl:
        assert hasattr(lib, name), name


def test_sampler_exports():
    R = _lib()
    lib = ctypes.CDLL(R.SAMPLER_PATH)
    for name in _declared("rsrs_sampler.h"):
        assert hasattr(lib, name), name


def _compare_trees(X, leaf, lo, side):
    R = _lib()
    t = R.Tree(X, leaf, lo, side)
    to = O.build_tree(X, leaf, lo, side)
    assert t.L == to.L
    assert (t.perm() == to.perm).all()
    for lev in range(t.L + 1):
        a, b = t.level(lev), to.levels[lev]
        assert (a["keys"].astype(np.int64) == b.keys).all()
        assert (a["start"] == b.start).all()
        assert (a["colour"] == b.colour).all()
        assert (a["parent"] == b.parent).all()
        assert len(a["neighbours"]) == len(b.neighbours)
        for x, y in zip(a["neighbours"], b.neighbours):
            assert (x == y).all()


def test_tree_matches_oracle_grid():
    cfg = W.CONFIGS["c1"]
    _compare_trees(W.points(cfg), cfg.leaf, *cfg.root())


def test_tree_matches_oracle_ragged_2d():
    rng = np.random.default_rng(2)
    X = rng.random((5000, 2)) ** 2               # clustered -> ragged leaves, empty boxes
    _compare_trees(X, 40, np.zeros(2), 1.0)


def test_tree_matches_oracle_sphere():
    X = W.fibonacci_sphere(6000)
    _compare_trees(X, 64, -np.ones(3), 2.0)


def test_tree_matches_oracle_fig1():
    X = ((np.arange(64) + 0.5) / 64.0)[:, None]
    _compare_trees(X, 8, np.zeros(1), 1.0)


def test_tree_bounding_cube_default():
    rng = np.random.default_rng(3)
    X = rng.random((700, 3)) * 5 - 2
    R = _lib()
    t = R.Tree(X, 30)
    to = O.build_tree(X, 30)
    assert t.L == to.L and (t.perm() == to.perm).all()


def test_plan_samples_leaf_bound():
    R = _lib()
    cfg = W.CONFIGS["c1"]
    t = R.Tree(W.points(cfg), cfg.leaf, *cfg.root())
    # 9 x 64 near-field rows + k + l, rounded to 32 (PAPER.md:265 p = 3m + k, 2D analogue)
    assert t.plan_samples(20, 10) == 608


def test_invalid_arguments():
    R = _lib()
    with pytest.raises(R.RSRSError) as e:
        R.Tree(np.zeros((0, 2)), 64)
    assert e.value.status == 1
    with pytest.raises(R.RSRSError):
        R.Tree(np.zeros((10, 4)), 64)


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-device path")
def test_no_gpu_fails_loudly():
    """Without a device rsrs_factor returns RSRS_ERR_CUDA -- there is no CPU fallback."""
    R = _lib()
    from paper_2311_01451_b200 import rsrs as RB
    cfg = W.CONFIGS["c1"]
    t = R.Tree(W.points(cfg), cfg.leaf, *cfg.root())
    buf = np.zeros((cfg.N, 32))
    o = RB.Opts(1e-6, 2.0, 1.0, 10, 2, 0, 1, None, None, 0)
    h = ctypes.c_void_p()
    st = RB._lib.rsrs_factor(t.handle, 0, 32, buf.ctypes.data, buf.ctypes.data, buf.ctypes.data,
                             buf.ctypes.data, 32, ctypes.byref(o), ctypes.byref(h))
    assert st == RB.RSRS_ERR_CUDA
    assert b"no CUDA device" in RB._lib.rsrs_last_error()
