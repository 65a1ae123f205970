"""Coupling estimator on the GPU against the
oracle's (tests/test_oracle_rsrs.py pins the oracle's estimator to the explicitly
tracked operator)."""
import numpy as np
import pytest

import oracle as O
import workloads as W
from gpu_common import dense_problem, run_gpu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


CASES = [("c1", W.CONFIGS["c1"]), ("sphere8k", W.CONFIGS["c3"].scaled(8192)), ("c4_64", W.CONFIGS["c4"].scaled(64))]


@pytest.mark.parametrize("name,cfg", CASES, ids=[c[0] for c in CASES])
def test_coupling_estimate_matches_oracle(name, cfg):
    X, A, Y, Z, Om, Ps, b = dense_problem(cfg)
    t, f = run_gpu(cfg, X, Y, Z, Om, Ps, cfg.root(), estimate_coupling=True)
    to = O.build_tree(X, cfg.leaf, *cfg.root())
    P = to.perm
    fo = O.factor(to, Y[P], Z[P], Om[P], Ps[P], cfg.eps, c_id=cfg.c_id, g=cfg.g, l=cfg.l, estimate_coupling=True)
    L = to.L
    lv = to.levels[L]
    est = f.coupling(L, lv.nboxes)
    checked = 0
    for bx in range(lv.nboxes):
        if lv.colour[bx] != 0 or (L, bx) not in fo.coupling:
            continue
        # colour-0 leaf boxes depend only on the initial samples: tight agreement
        for side in range(2):
            o = fo.coupling[(L, bx)][side]
            g = est[bx, side]
            assert abs(g - o) <= 1e-2 * o + 1e-12, (bx, side, g, o)
            checked += 1
    assert checked > 0
    for lev in range(L, 1, -1):
        nb = len(to.levels[lev].keys)
        e = f.coupling(lev, nb)
        og = max((max(v) for k, v in fo.coupling.items() if k[0] == lev), default=0.0)
        gg = e.max()
        assert (og <= 1e-12 and gg <= 1e-10) or og / 2 <= gg <= 2 * og, (lev, gg, og)
    # the estimator does not change the factorization
    t2, f2 = run_gpu(cfg, X, Y, Z, Om, Ps, cfg.root())
    for lev in range(L, 1, -1):
        nb = len(to.levels[lev].keys)
        assert np.array_equal(f.ranks(lev, nb), f2.ranks(lev, nb))


@pytest.mark.parametrize("name,cfg", CASES[:2], ids=[c[0] for c in CASES[:2]])
def test_noise_aware_tolerance_matches_oracle(name, cfg):
    """Noise-aware schedule (rsrs_opts.noise_factor = theta = 4, R17):
    atol(l-1) = max(atol(l), theta nu(l)) from the per-box coupling estimates.  GPU vs oracle:
    the per-level tolerances agree (the medians come from estimates that agree to ~1e-2), and
    the north_star parity bar holds for the resulting factorization."""
    X, A, Y, Z, Om, Ps, b = dense_problem(cfg)
    theta = 4.0
    t, f = run_gpu(cfg, X, Y, Z, Om, Ps, cfg.root(), noise_factor=theta)
    to = O.build_tree(X, cfg.leaf, *cfg.root())
    P = to.perm
    fo = O.factor(to, Y[P], Z[P], Om[P], Ps[P], cfg.eps, c_id=cfg.c_id, l=cfg.l, noise_factor=theta)
    for lev, a in fo.atol.items():
        assert abs(f.atol(lev) - a) <= 0.05 * a, (lev, f.atol(lev), a)
    x_or = O.solve(fo, b)
    from gpu_common import gpu_solve
    x_g = gpu_solve(f, b)
    eps = cfg.eps
    assert np.linalg.norm(x_g - x_or) / np.linalg.norm(x_or) <= 10 * eps
    assert np.linalg.norm(A @ x_g - b) / np.linalg.norm(b) <= 10 * eps
    for lev in range(to.L, 1, -1):
        nb = len(to.levels[lev].keys)
        kg = f.ranks(lev, nb)
        for bx in range(nb):
            if fo.nb.get((lev, bx), 0) > 0:
                assert abs(int(kg[bx]) - int(fo.ranks[(lev, bx)])) <= 2
