"""Parity at BASELINE.json's full sizes in the configuration bench.py times (c2 and
c4, N = 262,144): properties that hold at any size, checked on the GPU result --
solve residual ||A x - b|| / ||b|| and apply error ||K v - A v|| / ||A v|| with the
exact on-the-fly operator (harness sampler, row-verified against CPU direct sums in
test_gpu_parity.py) -- and the skeleton ranks of the first leaf boxes against the
oracle run on exact CPU samples of those boxes (bench.py's oracle_sample)."""
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


def _oracle_first_boxes(cfg, nboxes):
    """Oracle O4-O9 on the first `nboxes` leaf boxes (colour 0; their samples by CPU direct sums)."""
    X = W.points(cfg)
    t = O.build_tree(X, cfg.leaf, *cfg.root())
    L = t.L
    lv = t.levels[L]
    order = t.canonical_order(L)[:nboxes]
    Om, Ps = W.omega_psi(cfg)
    Om, Ps = Om[t.perm], Ps[t.perm]
    Y = np.zeros_like(Om)
    Z = np.zeros_like(Ps)
    cols = t.perm[np.arange(cfg.N)]
    for b in order:
        rows = np.arange(lv.start[b], lv.start[b + 1])
        Ab = W.kernel_block(cfg, X, t.perm[rows], cols)
        Y[rows] = Ab @ Om
        Z[rows] = Ab.conj() @ Ps
    f = O.factor(t, Y, Z, Om, Ps, cfg.eps, c_id=cfg.c_id, g=cfg.g, l=cfg.l, max_boxes=len(order), copy=False)
    return L, order, f


@pytest.mark.parametrize("name", ["c2", "c4"])
def test_full_size(name):
    import torch

    import paper_2311_01451_b200 as R
    cfg = W.CONFIGS[name]
    dev = torch.device("cuda:0")
    X = W.points(cfg)
    t = R.Tree(X, cfg.leaf, *cfg.root())
    perm = t.perm()
    N = cfg.N
    Om, Ps = W.omega_psi(cfg)
    P = torch.from_numpy(perm).to(dev)
    Om_d = torch.from_numpy(Om).to(dev)[P].contiguous()
    Ps_d = torch.from_numpy(Ps).to(dev)[P].contiguous()
    del Om, Ps
    pts = np.zeros((N, 3))
    pts[:, :X.shape[1]] = X
    pts_d = torch.from_numpy(pts[perm]).to(dev)
    wgt = W.kernel_weight(cfg)
    Y_d = torch.empty_like(Om_d)
    Z_d = torch.empty_like(Ps_d)
    R.sample_matvec(cfg.kernel, pts_d, wgt, Om_d, Y_d, kappa=cfg.kappa)
    R.sample_matvec(cfg.kernel, pts_d, wgt, Ps_d, Z_d, adjoint=True, kappa=cfg.kappa)
    f = R.factor(t, Y_d, Z_d, Om_d, Ps_d, p=cfg.p, eps=cfg.eps, level_growth=cfg.g, id_scale=cfg.c_id,
                 oversample=cfg.l)
    del Y_d, Z_d, Om_d, Ps_d

    def A_apply(v_orig):   # exact A v (original order) through the on-the-fly operator
        vt = v_orig[P].contiguous().view(N, 1)
        out = torch.empty_like(vt)
        R.sample_matvec(cfg.kernel, pts_d, wgt, vt, out, kappa=cfg.kappa)
        res = torch.empty_like(out.view(N))
        res[P] = out.view(N)
        return res

    b = torch.from_numpy(W.rhs(cfg)).to(dev)
    x = b.clone()
    f.solve(x)
    res = float((A_apply(x) - b).norm() / b.norm())
    assert res <= 10 * cfg.eps, res
    v = torch.from_numpy(W.gaussian(N, 77, 5, cfg.is_complex)).to(dev)
    kv = v.clone()
    f.apply(kv)
    av = A_apply(v)
    assert float((kv - av).norm() / av.norm()) <= 10 * cfg.eps
    # solve(apply(v)) = v
    f.solve(kv)
    assert float((kv - v).norm() / v.norm()) <= 1e-10
    # ranks of the first leaf boxes (colour 0) against the oracle on exact samples
    L, order, fo = _oracle_first_boxes(cfg, 8)
    kg = f.ranks(L, len(t.level(L)["keys"]))
    for bx in order:
        assert abs(int(kg[bx]) - int(fo.ranks[(L, bx)])) <= 2, (bx, kg[bx], fo.ranks[(L, bx)])
