"""Shared helpers of the GPU parity tests: one seeded problem, solved by the CPU
oracle and by the CUDA path (through the C ABI) on identical input bytes."""
import numpy as np

import oracle as O
import workloads as W


def dense_problem(cfg, X=None, p=None):
    """Dense A, seeded Omega/Psi/b and Y = A Omega, Z = A^* Psi (original order)."""
    X = W.points(cfg) if X is None else X
    p = cfg.p if p is None else p
    A = W.dense_matrix(cfg, X)
    Om, Ps = W.omega_psi(cfg, N=X.shape[0], p=p)
    Y, Z = W.dense_samples(A, Om, Ps)
    b = W.rhs(cfg, N=X.shape[0])
    return X, A, Y, Z, Om, Ps, b


def run_oracle(cfg, X, Y, Z, Om, Ps, root, **kw):
    t = O.build_tree(X, cfg.leaf, *root)
    P = t.perm
    f = O.factor(t, Y[P], Z[P], Om[P], Ps[P], cfg.eps, c_id=cfg.c_id, g=cfg.g, l=cfg.l, **kw)
    return t, f


def run_gpu(cfg, X, Y, Z, Om, Ps, root, p=None, profile=False, **kw):
    import torch

    import paper_2311_01451_b200 as R
    p = cfg.p if p is None else p
    t = R.Tree(X, cfg.leaf, *root)
    perm = t.perm()
    dev = torch.device("cuda:0")
    T = [torch.from_numpy(np.ascontiguousarray(M[perm][:, :p])).to(dev) for M in (Y, Z, Om, Ps)]
    f = R.factor(t, *T, p=p, eps=cfg.eps, level_growth=cfg.g, id_scale=cfg.c_id, oversample=cfg.l,
                 profile=profile, **kw)
    return t, f


def gpu_solve(f, b):
    import torch
    x = torch.from_numpy(np.array(b, copy=True)).to("cuda:0")
    f.solve(x)
    return x.cpu().numpy()


def gpu_apply(f, v):
    import torch
    x = torch.from_numpy(np.array(v, copy=True)).to("cuda:0")
    f.apply(x)
    return x.cpu().numpy()


def rank_diffs(t_gpu, f_gpu, t_or, f_or, levels):
    """max |k_gpu - k_oracle| per level over every nonempty box."""
    out = {}
    for lev in levels:
        nb = len(t_or.levels[lev].keys)
        kg = f_gpu.ranks(lev, nb)
        d = 0
        for b in range(nb):
            if (lev, b) in f_or.ranks and f_or.nb.get((lev, b), 0) > 0:
                d = max(d, abs(int(kg[b]) - int(f_or.ranks[(lev, b)])))
        out[lev] = d
    return out
