"""The f3 workload: T11 = A11 - A12 A22^-1 A21 of a 3D Poisson
slab decomposition.  workloads builds T11 in closed form in the DST eigenbasis of the interface
plane; these tests pin that construction against the definition (eq. T11): the
explicit sparse Schur complement of the 7-point finite-difference Laplacian on the interface plane
+ a slab of b planes, Dirichlet beyond (scipy sparse direct solve), and the oracle's RSRS of it
against dense LU."""
import os

import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spl

import oracle as O
import workloads as W


def explicit_t11(n, b):
    """A11 - A12 A22^-1 A21 with A = K (x) I (x) I + I (x) K (x) I + I (x) I (x) K on planes z = 0..b
    (K = tridiag(-1, 2, -1), Dirichlet), block 1 = plane 0 (the interface), block 2 = planes 1..b."""
    def K(m):
        return sp.diags([-np.ones(m - 1), 2 * np.ones(m), -np.ones(m - 1)], [-1, 0, 1])

    def I(m):
        return sp.identity(m)
    A = (sp.kron(sp.kron(K(b + 1), I(n)), I(n)) + sp.kron(sp.kron(I(b + 1), K(n)), I(n))
         + sp.kron(sp.kron(I(b + 1), I(n)), K(n))).tocsc()
    m = n * n
    A11 = A[:m, :m].toarray()
    X = spl.spsolve(A[m:, m:].tocsc(), A[m:, :m].toarray())
    return A11 - A[:m, m:] @ X


@pytest.mark.parametrize("n,b", [(8, 3), (10, 10), (12, 1)])
def test_t11_closed_form_equals_sparse_schur_complement(n, b):
    cfg = W.Config("t11_small", "grid2d", n, "t11", "f64", leaf=16, extra={"slab_b": b})
    X = W.points(cfg)
    T = W.dense_matrix(cfg, X)
    E = explicit_t11(n, b)
    assert np.abs(T - E).max() <= 1e-12 * np.abs(E).max()
    V = np.random.default_rng(n).standard_normal((n * n, 3))
    assert np.abs(W.t11_apply(cfg, V) - E @ V).max() <= 1e-12 * np.abs(E @ V).max()
    assert np.allclose(T, T.T, atol=1e-14 * np.abs(T).max())
    assert np.linalg.eigvalsh(T).min() > 0            # Schur complement of an spd matrix


def test_t11_oracle_against_dense_lu():
    """The oracle's RSRS of T11 (n = 80, N = 6400, 100-point leaves, atol = 5e-6, the frozen
    t11 configuration otherwise) solves to 10 atol of LAPACK getrf/getrs."""
    cfg = W.CONFIGS["t11"].scaled(80)
    X = W.points(cfg)
    t = O.build_tree(X, cfg.leaf, *cfg.root())
    A = W.dense_matrix(cfg, X)
    Om, Ps = W.omega_psi(cfg)
    Y, Z = W.dense_samples(A, Om, Ps)
    P = t.perm
    f = O.factor(t, Y[P], Z[P], Om[P], Ps[P], cfg.eps, c_id=cfg.c_id, g=cfg.g, l=cfg.l,
                 workers=os.cpu_count() or 1)
    b = W.rhs(cfg)
    x = O.solve(f, b)
    xd = sla.lu_solve(sla.lu_factor(A), b)
    assert t.L == 3
    assert np.linalg.norm(x - xd) / np.linalg.norm(xd) <= 10 * cfg.eps
    assert np.linalg.norm(A @ x - b) / np.linalg.norm(b) <= 10 * cfg.eps
