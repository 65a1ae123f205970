"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same
seeded inputs.  Bar (BASELINE.json north_star): ||x_gpu - x_oracle|| / ||x_oracle||
<= 10 eps, both solve residuals <= 10 eps, per-box ranks within +-2."""
import math

import numpy as np
import pytest

import oracle as O
import workloads as W
from gpu_common import dense_problem, gpu_apply, gpu_solve, rank_diffs, run_gpu, run_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _parity(cfg, X, root, p=None, check_apply=True):
    X, A, Y, Z, Om, Ps, b = dense_problem(cfg, X, p)
    t_or, f_or = run_oracle(cfg, X, Y, Z, Om, Ps, root)
    t_g, f_g = run_gpu(cfg, X, Y, Z, Om, Ps, root, p=p)
    x_or = O.solve(f_or, b)
    x_g = gpu_solve(f_g, b)
    eps = cfg.eps
    err = np.linalg.norm(x_g - x_or) / np.linalg.norm(x_or)
    res_g = np.linalg.norm(A @ x_g - b) / np.linalg.norm(b)
    res_or = np.linalg.norm(A @ x_or - b) / np.linalg.norm(b)
    assert err <= 10 * eps, err
    assert res_g <= 10 * eps and res_or <= 10 * eps, (res_g, res_or)
    levels = [lev for lev in range(t_or.L, 1, -1)]
    d = rank_diffs(t_g, f_g, t_or, f_or, levels)
    assert all(v <= 2 for v in d.values()), d
    st = f_g.stats()
    # |S| and the step count follow from the ranks
    assert abs(st["top_size"] - f_or.S.shape[0]) <= 2 * len(t_or.levels[2].keys)
    if check_apply:
        v = W.gaussian(X.shape[0], 99, 7, cfg.is_complex)
        y_g = gpu_apply(f_g, v)
        y_or = O.apply(f_or, v)
        assert np.linalg.norm(y_g - y_or) / np.linalg.norm(y_or) <= 10 * eps
        assert np.linalg.norm(y_g - A @ v) / np.linalg.norm(A @ v) <= 10 * eps
        z = gpu_solve(f_g, y_g)
        assert np.linalg.norm(z - v) / np.linalg.norm(v) <= 1e-11      # solve(apply(v)) = v
    return dict(err=err, res_g=res_g, res_or=res_or, ranks=d, stats=st, f_or=f_or, t_or=t_or, f_g=f_g)


def test_c1_parity():
    """configs[0] (c1): 64x64 grid, 2D log kernel, N = 4096, every level."""
    cfg = W.CONFIGS["c1"]
    out = _parity(cfg, None, cfg.root())
    st = out["stats"]
    assert st["L"] == 3 and st["nlevels_compressed"] == 2
    # identical ranks -> identical stored-scalar count (Table 1 'M')
    if all(v == 0 for v in out["ranks"].values()) and st["top_size"] == out["f_or"].S.shape[0]:
        assert st["memory_scalars"] == out["f_or"].memory()


def test_c4_family_parity_complex128():
    """c4's complex Helmholtz operator (kappa = 25, complex128) on the c1-size grid (N = 4096):
    complex DMMA GEMMs, Hermitian Cholesky / pivoted Gram ID, complex LU, conjugate
    sample updates (RSRS_C128 path)."""
    cfg = W.CONFIGS["c4"].scaled(64)
    out = _parity(cfg, None, cfg.root())
    assert out["stats"]["L"] == 3


def test_c4_family_tails_complex128():
    """complex128 with p and box sizes off the tile multiples."""
    cfg = W.Config("tail_c", "grid2d", 50, "helm2d", "c128", leaf=37, p=650, seed=15, g=2.0)
    _parity(cfg, None, cfg.root())


def test_ragged_clustered_points():
    """Non-uniform points (ragged leaves, empty boxes, boxes of 1 point)."""
    rng = np.random.default_rng(21)
    X = rng.random((3000, 2)) ** 2
    cfg = W.Config("ragged", "grid2d", 55, "log2d", "f64", leaf=40, p=640, seed=21, g=1.0)
    _parity(cfg, X, (np.zeros(2), 1.0))


def test_sphere_small():
    """3D surface (c3/c5 family) at N = 8192 with the sphere sample count."""
    cfg = W.CONFIGS["c3"].scaled(8192)
    _parity(cfg, None, cfg.root())


def test_tail_sizes_not_tile_multiples():
    """p and box sizes that are not multiples of the 64-wide tiles / 32-wide chunks."""
    cfg = W.Config("tail", "grid2d", 50, "log2d", "f64", leaf=37, p=650, seed=5, g=2.0)
    _parity(cfg, None, cfg.root())


def test_diagonal_operator_exact():
    """Zero off-diagonal rank: every k = 0; K = A and K^-1 exact (special case)."""
    import torch

    import paper_2311_01451_b200 as R
    rng = np.random.default_rng(8)
    X = rng.random((2000, 2))
    d = 1.0 + rng.random(2000)
    t = R.Tree(X, 32, np.zeros(2), 1.0)
    perm = t.perm()
    Om = rng.standard_normal((2000, 512))
    Ps = rng.standard_normal((2000, 512))
    Om_t, Ps_t = Om[perm], Ps[perm]
    dev = "cuda:0"
    T = [torch.from_numpy(np.ascontiguousarray(M)).to(dev) for M in
         (d[perm][:, None] * Om_t, d[perm][:, None] * Ps_t, Om_t, Ps_t)]
    f = R.factor(t, *T, p=512, eps=1e-6)
    for lev in range(t.L, 1, -1):
        k = f.ranks(lev, len(t.level(lev)["keys"]))
        assert (k[k >= 0] == 0).all()
    v = rng.standard_normal(2000)
    # extraction through the near-field Gram (CholeskyQR): error ~ cond(Omega_near)^2 eps,
    # cond <= (sqrt p + sqrt r)/(sqrt p - sqrt r) ~ 12 at r <= 9*32, p = 512
    assert np.allclose(gpu_apply(f, v), d * v, rtol=1e-11, atol=0)
    assert np.allclose(gpu_solve(f, v), v / d, rtol=1e-11, atol=0)


def test_insufficient_samples_reports_level_and_deficit():
    import paper_2311_01451_b200 as R
    cfg = W.CONFIGS["c1"]
    X, A, Y, Z, Om, Ps, b = dense_problem(cfg, None, 560)
    with pytest.raises(R.RSRSError) as e:
        run_gpu(cfg, X, Y, Z, Om, Ps, cfg.root(), p=560)
    assert e.value.status == 2
    assert "level 3" in str(e.value) and "deficit" in str(e.value)


def test_multiple_rhs():
    cfg = W.CONFIGS["c1"]
    X, A, Y, Z, Om, Ps, b = dense_problem(cfg)
    t_g, f_g = run_gpu(cfg, X, Y, Z, Om, Ps, cfg.root())
    B = W.rhs(cfg, nrhs=3)
    Xs = gpu_solve(f_g, B)
    for j in range(3):
        assert np.allclose(Xs[:, j], gpu_solve(f_g, B[:, j]), rtol=0, atol=1e-13 * np.abs(Xs).max())
        assert np.linalg.norm(A @ Xs[:, j] - B[:, j]) / np.linalg.norm(B[:, j]) <= 10 * cfg.eps


def test_sampler_rows_match_direct_sum():
    """Harness operator: GPU kernel matvec vs CPU direct sums on random rows."""
    import torch

    import paper_2311_01451_b200 as R
    for cfg in (W.CONFIGS["c1"], W.CONFIGS["c3"].scaled(5000), W.CONFIGS["c4"].scaled(70)):
        X = W.points(cfg)
        N = X.shape[0]
        pts = np.zeros((N, 3))
        pts[:, :X.shape[1]] = X
        V = W.gaussian((N, 70), 3, 0, cfg.is_complex)
        dt = torch.complex128 if cfg.is_complex else torch.float64
        for adjoint in (False, True):
            Yd = torch.empty((N, 70), dtype=dt, device="cuda:0")
            R.sample_matvec(cfg.kernel, torch.from_numpy(pts).cuda(), W.kernel_weight(cfg),
                            torch.from_numpy(V).cuda(), Yd, adjoint=adjoint, kappa=cfg.kappa)
            rows = np.random.default_rng(1).choice(N, 64, replace=False)
            Ab = W.kernel_block(cfg, X, rows, np.arange(N))
            # A^* rows = conj(A) rows for these symmetric kernels
            ref = (Ab.conj() if adjoint else Ab) @ V
            got = Yd.cpu().numpy()[rows]
            # CUDA's j0/y0 are accurate to a few ulp; log / rsqrt to ~1 ulp
            tol = (1e-12 if cfg.is_complex else 1e-13) * np.abs(ref).max() * math.sqrt(N)
            assert np.abs(got - ref).max() <= tol, (cfg.name, adjoint)


@pytest.mark.parametrize("name,n", [("c1", None), ("c3", 8192), ("c4", 64)], ids=["c1", "sphere8k", "c4_64"])
def test_pinned_host_inputs_bit_identical(name, n):
    """rsrs_factor / rsrs_solve on pinned HOST arrays (the e2e path: the library copies Omega / Psi and
    streams the Y / Z rows of each leaf colour batch one batch ahead) give bit for bit the device-input
    factorization, and leave the host inputs unchanged."""
    import torch

    import paper_2311_01451_b200 as R
    cfg = W.CONFIGS[name] if n is None else W.CONFIGS[name].scaled(n)
    X, A, Y, Z, Om, Ps, b = dense_problem(cfg)
    t = R.Tree(X, cfg.leaf, *cfg.root())
    perm = t.perm()
    H = [torch.from_numpy(np.ascontiguousarray(M[perm])).pin_memory() for M in (Y, Z, Om, Ps)]
    H0 = [h.clone() for h in H]
    D = [h.cuda() for h in H]
    kw = dict(p=cfg.p, eps=cfg.eps, level_growth=cfg.g, id_scale=cfg.c_id, oversample=cfg.l)
    fd = R.factor(t, *D, **kw)
    fh = R.factor(t, *H, **kw)
    assert all(torch.equal(h, h0) for h, h0 in zip(H, H0))
    xd = torch.from_numpy(b.copy()).cuda()
    fd.solve(xd)
    xh = torch.from_numpy(b.copy()).pin_memory()
    fh.solve(xh)
    torch.cuda.synchronize()
    assert np.array_equal(xd.cpu().numpy(), xh.numpy())
    with pytest.raises(ValueError):
        R.factor(t, H[0], D[1], H[2], H[3], **kw)          # mixed host / device
