"""Symmetric shortcut (not in the paper, which draws two
independent sketches): for real symmetric A take Psi = Omega,
so Z = A^T Psi = Y and only the Y / Omega side of the sweep runs.  Reference: the
oracle's general algorithm on the same inputs (Z = Y, Psi = Omega), parity bar of
BASELINE.json north_star."""
import numpy as np
import pytest

import oracle as O
import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _sym_problem(cfg):
    X = W.points(cfg)
    A = W.dense_matrix(cfg, X)
    assert np.allclose(A, A.T)
    Om, _ = W.omega_psi(cfg)
    Y = A @ Om
    b = W.rhs(cfg)
    return X, A, Y, Om, b


def _gpu_sym(cfg, X, Y, Om, emulate=0, **kw):
    import torch

    import paper_2311_01451_b200 as R
    t = R.Tree(X, cfg.leaf, *cfg.root())
    perm = t.perm()
    Yd = torch.from_numpy(np.ascontiguousarray(Y[perm])).cuda()
    Od = torch.from_numpy(np.ascontiguousarray(Om[perm])).cuda()
    if emulate:
        fs = R.factor_emulated(t, emulate, Yd, None, Od, None, p=cfg.p, eps=cfg.eps, level_growth=cfg.g,
                               id_scale=cfg.c_id, oversample=cfg.l, symmetric=True, push_updates=True)
        return t, fs
    f = R.factor(t, Yd, None, Od, None, p=cfg.p, eps=cfg.eps, level_growth=cfg.g, id_scale=cfg.c_id,
                 oversample=cfg.l, symmetric=True, **kw)
    return t, f


@pytest.mark.parametrize("name,n", [("c1", None), ("c3", 8192)])
def test_symmetric_shortcut_parity(name, n):
    import torch
    cfg = W.CONFIGS[name] if n is None else W.CONFIGS[name].scaled(n)
    X, A, Y, Om, b = _sym_problem(cfg)
    t, f = _gpu_sym(cfg, X, Y, Om)
    to = O.build_tree(X, cfg.leaf, *cfg.root())
    P = to.perm
    fo = O.factor(to, Y[P], Y[P], Om[P], Om[P], cfg.eps, c_id=cfg.c_id, g=cfg.g, l=cfg.l)
    x_or = O.solve(fo, b)
    xd = torch.from_numpy(b.copy()).cuda()
    f.solve(xd)
    x = xd.cpu().numpy()
    eps = cfg.eps
    assert np.linalg.norm(x - x_or) / np.linalg.norm(x_or) <= 10 * eps
    assert np.linalg.norm(A @ x - b) / np.linalg.norm(b) <= 10 * eps
    for lev in range(to.L, 1, -1):
        nb = len(to.levels[lev].keys)
        kg = f.ranks(lev, nb)
        for bx in range(nb):
            if fo.nb.get((lev, bx), 0) > 0:
                assert abs(int(kg[bx]) - int(fo.ranks[(lev, bx)])) <= 2
    # apply / solve round trip and K ~ A
    v = W.gaussian(X.shape[0], 3, 9)
    vd = torch.from_numpy(v.copy()).cuda()
    f.apply(vd)
    y = vd.cpu().numpy()
    assert np.linalg.norm(y - A @ v) / np.linalg.norm(A @ v) <= 10 * eps
    f.solve(vd)
    assert np.linalg.norm(vd.cpu().numpy() - v) / np.linalg.norm(v) <= 1e-11
    # half the two-sided work is gone
    assert f.stats()["flops_model"] < 0.65 * _full_flops(cfg, X, A, Y, Om)


def _full_flops(cfg, X, A, Y, Om):
    import torch

    import paper_2311_01451_b200 as R
    t = R.Tree(X, cfg.leaf, *cfg.root())
    perm = t.perm()
    T = [torch.from_numpy(np.ascontiguousarray(M[perm])).cuda() for M in (Y, Y, Om, Om)]
    f = R.factor(t, *T, p=cfg.p, eps=cfg.eps, level_growth=cfg.g, id_scale=cfg.c_id, oversample=cfg.l)
    return f.stats()["flops_model"]


def test_symmetric_shortcut_emulated_ranks_bit_exact():
    import torch

    import paper_2311_01451_b200 as R
    cfg = W.CONFIGS["c1"]
    X, A, Y, Om, b = _sym_problem(cfg)
    t, f = _gpu_sym(cfg, X, Y, Om, direct_gram=True, push_updates=True)
    _, fs = _gpu_sym(cfg, X, Y, Om, emulate=3)
    x1 = torch.from_numpy(b.copy()).cuda()
    f.solve(x1)
    xg = torch.from_numpy(b.copy()).cuda()
    R.solve_emulated(fs, xg)
    assert np.array_equal(xg.cpu().numpy(), x1.cpu().numpy())


def test_complex_symmetric_shortcut_parity():
    """c4's complex-symmetric Helmholtz operator (A = A^T, complex128) on the c1-size grid:
    Psi = conj(Omega) => Z = A^* Psi = conj(A Omega) = conj(Y), so only the Y / Omega side
    runs (rsrs_opts.symmetric = 2).  Reference: the oracle's general two-sketch algorithm on
    the same inputs (Y, Z = conj(Y), Omega, Psi = conj(Omega)), north_star bar."""
    import torch

    import paper_2311_01451_b200 as R
    cfg = W.CONFIGS["c4"].scaled(64)
    X = W.points(cfg)
    A = W.dense_matrix(cfg, X)
    assert np.allclose(A, A.T) and not np.allclose(A, A.conj().T)
    Om, _ = W.omega_psi(cfg)
    Y = A @ Om
    b = W.rhs(cfg)
    t = R.Tree(X, cfg.leaf, *cfg.root())
    perm = t.perm()
    Yd = torch.from_numpy(np.ascontiguousarray(Y[perm])).cuda()
    Od = torch.from_numpy(np.ascontiguousarray(Om[perm])).cuda()
    f = R.factor(t, Yd, None, Od, None, p=cfg.p, eps=cfg.eps, level_growth=cfg.g, id_scale=cfg.c_id,
                 oversample=cfg.l, symmetric=True)
    to = O.build_tree(X, cfg.leaf, *cfg.root())
    P = to.perm
    Yt, Ot = Y[P], Om[P]
    fo = O.factor(to, Yt, Yt.conj(), Ot, Ot.conj(), cfg.eps, c_id=cfg.c_id, g=cfg.g, l=cfg.l)
    x_or = O.solve(fo, b)
    xd = torch.from_numpy(b.copy()).cuda()
    f.solve(xd)
    x = xd.cpu().numpy()
    eps = cfg.eps
    assert np.linalg.norm(x - x_or) / np.linalg.norm(x_or) <= 10 * eps
    assert np.linalg.norm(A @ x - b) / np.linalg.norm(b) <= 10 * eps
    assert np.linalg.norm(A @ x_or - b) / np.linalg.norm(b) <= 10 * eps
    for lev in range(to.L, 1, -1):
        nb = len(to.levels[lev].keys)
        kg = f.ranks(lev, nb)
        for bx in range(nb):
            if fo.nb.get((lev, bx), 0) > 0:
                assert abs(int(kg[bx]) - int(fo.ranks[(lev, bx)])) <= 2
    v = W.gaussian(X.shape[0], 3, 9, True)
    vd = torch.from_numpy(v.copy()).cuda()
    f.apply(vd)
    assert np.linalg.norm(vd.cpu().numpy() - A @ v) / np.linalg.norm(A @ v) <= 10 * eps
    f.solve(vd)
    assert np.linalg.norm(vd.cpu().numpy() - v) / np.linalg.norm(v) <= 1e-11


def test_symmetric_shortcut_rejects_hermitian_complex():
    """complex128 supports only the complex-symmetric form (opts.symmetric = 2) at the C ABI."""
    import ctypes

    import torch

    import paper_2311_01451_b200 as R
    from paper_2311_01451_b200 import rsrs as RR
    cfg = W.CONFIGS["c4"].scaled(32)
    X = W.points(cfg)
    t = R.Tree(X, cfg.leaf, *cfg.root())
    Y = torch.zeros((X.shape[0], 64), dtype=torch.complex128, device="cuda")
    o = RR.Opts(1e-6, 1.0, 1.0, 10, 2, 0, 1, None, None, 0, -1, 1, 0, 0, 0)
    h = ctypes.c_void_p()
    st = RR._lib.rsrs_factor(t.handle, RR.RSRS_C128, 64, Y.data_ptr(), None, Y.data_ptr(), None, 64,
                             ctypes.byref(o), ctypes.byref(h))
    assert st == 1
