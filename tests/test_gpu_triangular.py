"""Triangular output form (Remark PAPER.md:577-611) for real symmetric
positive definite operators: with the symmetric sketch (Psi = Omega), X_rr = C C^T by
Cholesky and the stored factors are C, C^-1 and M_U = C^-1 X_rc (no block-diagonal middle).
Reference: the oracle's triangular form on the same inputs (oracle.factor(triangular=True)),
north_star parity bar; K against the exact operator; solve(apply(v)) = v."""
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


@pytest.mark.parametrize("name,n", [("c1", None), ("c5", 8192)], ids=["c1", "sphere8k_c5params"])
def test_triangular_form_parity(name, n):
    import torch

    import paper_2311_01451_b200 as R
    cfg = W.CONFIGS[name] if n is None else W.CONFIGS[name].scaled(n)
    X = W.points(cfg)
    A = W.dense_matrix(cfg, X)
    assert np.allclose(A, A.T) and np.linalg.eigvalsh(A).min() > 0        # spd
    Om, _ = W.omega_psi(cfg)
    Y = A @ Om
    b = W.rhs(cfg)
    t = R.Tree(X, cfg.leaf, *cfg.root())
    perm = t.perm()

    def gpu(tri):
        Yd = torch.from_numpy(np.ascontiguousarray(Y[perm])).cuda()
        Od = torch.from_numpy(np.ascontiguousarray(Om[perm])).cuda()
        return R.factor(t, Yd, None, Od, None, p=cfg.p, eps=cfg.eps, level_growth=cfg.g, id_scale=cfg.c_id,
                        oversample=cfg.l, symmetric=True, triangular=tri)

    f = gpu(True)
    to = O.build_tree(X, cfg.leaf, *cfg.root())
    P = to.perm
    fo = O.factor(to, Y[P], Y[P], Om[P], Om[P], cfg.eps, c_id=cfg.c_id, g=cfg.g, l=cfg.l, triangular=True)
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
    v = W.gaussian(X.shape[0], 3, 9)
    vd = torch.from_numpy(v.copy()).cuda()
    f.apply(vd)
    y = vd.cpu().numpy()
    assert np.linalg.norm(y - O.apply(fo, v)) / np.linalg.norm(y) <= 10 * eps
    assert np.linalg.norm(y - A @ v) / np.linalg.norm(A @ v) <= 10 * eps
    f.solve(vd)
    assert np.linalg.norm(vd.cpu().numpy() - v) / np.linalg.norm(v) <= 1e-11
    # fewer stored scalars than the block-diagonal form of the same sweep (one of G_L / G_U)
    assert f.stats()["memory_scalars"] < gpu(False).stats()["memory_scalars"]


def test_triangular_form_rejected_without_symmetric_sketch():
    import torch

    import paper_2311_01451_b200 as R
    cfg = W.CONFIGS["c1"]
    X = W.points(cfg)
    t = R.Tree(X, cfg.leaf, *cfg.root())
    Y = torch.zeros((X.shape[0], 64), dtype=torch.float64, device="cuda")
    with pytest.raises(R.RSRSError) as e:
        R.factor(t, Y, Y.clone(), Y.clone(), Y.clone(), p=64, triangular=True)
    assert e.value.status == 1
