"""Level-wide near-field Gram blocks (csrc/gram.cuh): each box's
Gram Omega_near Omega_near^* is assembled from box-pair blocks computed once per
level and kept current under the E/F transforms, instead of one r x r x p GEMM
per box.  Same matrices up to summation order, so the factorization must agree
with the direct computation to rounding: identical ranks on every box and
solutions equal to ~1e-12, and both within the oracle parity bar."""
import numpy as np
import pytest

import oracle as O
import workloads as W
from gpu_common import dense_problem, gpu_solve, run_gpu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


CASES = [
    ("c1", W.CONFIGS["c1"], None),
    ("sphere8k", W.CONFIGS["c3"].scaled(8192), None),
    ("c4_64", W.CONFIGS["c4"].scaled(64), None),
    ("tail", W.Config("tail", "grid2d", 50, "log2d", "f64", leaf=37, p=650, seed=5, g=2.0), None),
]


@pytest.mark.parametrize("name,cfg,X", CASES, ids=[c[0] for c in CASES])
def test_gram_blocks_match_direct(name, cfg, X):
    X, A, Y, Z, Om, Ps, b = dense_problem(cfg, X)
    t1, fb = run_gpu(cfg, X, Y, Z, Om, Ps, cfg.root())                     # blocks (default)
    t2, fd = run_gpu(cfg, X, Y, Z, Om, Ps, cfg.root(), direct_gram=True)
    for lev in range(t1.L, 1, -1):
        nb = len(t1.level(lev)["keys"])
        assert np.array_equal(fb.ranks(lev, nb), fd.ranks(lev, nb)), lev
    xb = gpu_solve(fb, b)
    xd = gpu_solve(fd, b)
    assert np.linalg.norm(xb - xd) / np.linalg.norm(xd) <= 1e-10
    assert np.linalg.norm(A @ xb - b) / np.linalg.norm(b) <= 10 * cfg.eps
    to = O.build_tree(X, cfg.leaf, *cfg.root())
    P = to.perm
    fo = O.factor(to, Y[P], Z[P], Om[P], Ps[P], cfg.eps, c_id=cfg.c_id, g=cfg.g, l=cfg.l)
    x_or = O.solve(fo, b)
    assert np.linalg.norm(xb - x_or) / np.linalg.norm(x_or) <= 10 * cfg.eps
    # fewer algorithmic Gram flops than the per-box Grams
    assert fb.stats()["flops_model"] < fd.stats()["flops_model"]


@pytest.mark.parametrize("name,cfg,X", CASES, ids=[c[0] for c in CASES])
def test_pulled_updates_match_pushed(name, cfg, X):
    """Pulled L/U updates (default on one GPU) vs pushing every update when its box is
    eliminated (opts.push_updates, the multi-GPU ranks' scheme): same sums regrouped."""
    X, A, Y, Z, Om, Ps, b = dense_problem(cfg, X)
    t1, fp = run_gpu(cfg, X, Y, Z, Om, Ps, cfg.root())
    t2, fq = run_gpu(cfg, X, Y, Z, Om, Ps, cfg.root(), push_updates=True)
    for lev in range(t1.L, 1, -1):
        nb = len(t1.level(lev)["keys"])
        assert np.array_equal(fp.ranks(lev, nb), fq.ranks(lev, nb)), lev
    xp = gpu_solve(fp, b)
    xq = gpu_solve(fq, b)
    assert np.linalg.norm(xp - xq) / np.linalg.norm(xq) <= 1e-10
    assert np.linalg.norm(A @ xp - b) / np.linalg.norm(b) <= 10 * cfg.eps
