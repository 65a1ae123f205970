"""Seeded synthetic workloads for RSRS (shared by oracle/, tests/ and bench.py).

This module holds ONLY input generation -- point sets, the kernel operator
A (the black box the method samples), seeded Gaussian test matrices and the
configuration table -- and none of the method's arithmetic (no nullification,
ID, extraction, elimination or solve).  Both sides (the CPU oracle and the
CUDA path) consume what it produces.

Configurations (BASELINE.json `configs`):

  c1  2D, 64x64 cell-centred grid in [0,1]^2, h=1/64,
      A_ij = delta_ij + h^2 log|x_i - x_j| (i != j), A_ii = 1, FP64
  c2  as c1 on a 512x512 grid, h=1/512
  c3  Fibonacci sphere N=262144, A_ij = delta_ij + w/(4 pi |x_i-x_j|), w=4pi/N
  c4  as c2 with A_ij = delta_ij + h^2 (i/4) H0^(1)(kappa |x_i-x_j|), kappa=25,
      complex128
  c5  Fibonacci sphere N=1048576, c3's kernel

Readings: cell centres ((i+1/2)h, (j+1/2)h) (SURVEY c.2
#14); Fibonacci lattice z_i = 1-(2i+1)/N, phi_i = i*pi*(3-sqrt 5) (c.2 #15);
A_ii = 1 exactly, no self term (c.2 #16, "The singularity
... can be handled with an appropriate quadrature rule"); complex Gaussian
(N(0,1) + i N(0,1))/sqrt 2 (c.2 #17).  Omega, Psi ~ N(0, I) per
PAPER.md:128-131 (eq. rand_sample_setting).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np

# Streams of the counter-keyed generator (SURVEY c.2 #18).
STREAM_OMEGA = 0
STREAM_PSI = 1
STREAM_RHS = 2


@dataclass(frozen=True)
class Config:
    name: str
    geometry: str          # "grid2d" | "sphere"
    n: int                 # grid side (grid2d) or number of points (sphere)
    kernel: str            # "log2d" | "lap3d" | "helm2d"
    dtype: str             # "f64" | "c128"
    leaf: int = 64
    eps: float = 1e-6
    p: int = 768           # sample count (frozen per config)
    seed: int = 1
    g: float = 2.0         # per-level tolerance relaxation atol(l) = c_id eps g^(L-l)
    c_id: float = 1.0
    l: int = 10            # oversampling
    kappa: float = 25.0
    extra: dict = field(default_factory=dict)

    @property
    def N(self) -> int:
        return self.n * self.n if self.geometry == "grid2d" else self.n

    @property
    def d(self) -> int:
        return 2 if self.geometry == "grid2d" else 3

    @property
    def is_complex(self) -> bool:
        return self.dtype == "c128"

    @property
    def np_dtype(self):
        return np.complex128 if self.is_complex else np.float64

    def root(self):
        """Root cube (lo, side) of the tree (SURVEY c.2 #12)."""
        if self.geometry == "grid2d":
            return np.zeros(2), 1.0
        return -np.ones(3), 2.0

    def scaled(self, n: int, p: int | None = None, **kw) -> "Config":
        """Same workload family at another size (test cases)."""
        return replace(self, name=f"{self.name}@{n}", n=n, p=p if p is not None else self.p, **kw)


CONFIGS = {
    "c1": Config("c1", "grid2d", 64, "log2d", "f64", p=768, seed=1, g=2.0),
    "c2": Config("c2", "grid2d", 512, "log2d", "f64", p=768, seed=2, g=2.0),
    "c3": Config("c3", "sphere", 262144, "lap3d", "f64", p=1216, seed=3, g=2.0),
    "c4": Config("c4", "grid2d", 512, "helm2d", "c128", p=768, seed=4, g=2.0),
    # c_id = 0.5 for c5: with c_id = 1 the full-size residual is 9.4e-6, too close to the 10 eps bar
    # (R7 / section 4; profiles/r01_c5_dev_run.txt)
    "c5": Config("c5", "sphere", 1048576, "lap3d", "f64", p=1216, seed=5, g=2.0, c_id=0.5),
    # the paper's only experiment (section 6.1), the sparse Schur
    # complement T11 = A11 - A12 A22^-1 A21 of a 3D Poisson slab decomposition (slab width b = 10),
    # N = n^2 interface points, atol = 5e-6 (the paper's tightest; its leaf m = 350 is capped here at
    # 100-point leaves by the per-box kernels' shared memory, reading R20)
    "t11": Config("t11", "grid2d", 320, "t11", "f64", leaf=100, p=1536, eps=5e-6, seed=6, g=2.0,
                  extra={"slab_b": 10}),
}


# ----------------------------------------------------------------------------
# point sets
# ----------------------------------------------------------------------------
def grid_points(n_side: int) -> np.ndarray:
    """Cell centres of an n x n grid in [0,1]^2, row-major (x fastest)."""
    h = 1.0 / n_side
    c = (np.arange(n_side) + 0.5) * h
    X, Yc = np.meshgrid(c, c, indexing="xy")
    return np.stack([X.ravel(), Yc.ravel()], axis=1).astype(np.float64)


def fibonacci_sphere(N: int) -> np.ndarray:
    """Fibonacci lattice on the unit sphere (SURVEY c.2 #15)."""
    i = np.arange(N, dtype=np.float64)
    z = 1.0 - (2.0 * i + 1.0) / N
    phi = i * (math.pi * (3.0 - math.sqrt(5.0)))
    rho = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    return np.stack([rho * np.cos(phi), rho * np.sin(phi), z], axis=1)


def points(cfg: Config) -> np.ndarray:
    if cfg.geometry == "grid2d":
        return grid_points(cfg.n)
    return fibonacci_sphere(cfg.n)


# ----------------------------------------------------------------------------
# the operator A (black box)
# ----------------------------------------------------------------------------
def kernel_weight(cfg: Config) -> float:
    if cfg.geometry == "grid2d":
        h = 1.0 / cfg.n
        return h * h
    return 1.0 / cfg.N        # w/(4 pi) with w = 4 pi / N


# ----------------------------------------------------------------------------
# T11: sparse Schur complement of a 3D Poisson slab decomposition
# ----------------------------------------------------------------------------
def dst_matrix(n: int) -> np.ndarray:
    """Orthonormal DST-I matrix S (symmetric, S S = I): the eigenvectors of the 1D Dirichlet
    second difference tridiag(-1, 2, -1) on n points."""
    k = np.arange(1, n + 1)
    return math.sqrt(2.0 / (n + 1)) * np.sin(np.pi * np.outer(k, k) / (n + 1))


def t11_symbol(n: int, b: int) -> np.ndarray:
    """Eigenvalues mu[i, j] of T11 = A11 - A12 A22^-1 A21 in the DST basis of the n x n interface plane.

    A = 7-point stencil (diagonal 6, neighbours -1; the finite-difference Poisson operator times
    h^2) on planes z = 0 (the interface, block 1) .. b (the slab interior, block 2), Dirichlet
    beyond.  Per in-plane mode (i, j) with a = 6 - 2 cos t_i - 2 cos t_j, t_k = pi k / (n + 1),
    the slab is tridiag(-1, a, -1) of size b, so mu = a - [T_b(a)^-1]_00 = a - sinh(b phi) /
    sinh((b + 1) phi) with a = 2 cosh(phi).  (Checked against the explicit sparse Schur
    complement in tests/test_workloads_t11.py.)"""
    th = np.pi * np.arange(1, n + 1) / (n + 1)
    a = 6.0 - 2.0 * np.cos(th)[:, None] - 2.0 * np.cos(th)[None, :]
    phi = np.arccosh(a / 2.0)
    return a - np.sinh(b * phi) / np.sinh((b + 1) * phi)


def t11_apply(cfg: Config, V: np.ndarray) -> np.ndarray:
    """T11 V for V in ORIGINAL point order (interface plane row-major, N x k): S2 diag(mu) S2 V with
    S2 = S (x) S applied as two n x n transforms (T11 is symmetric: T11^* = T11)."""
    n, b = cfg.n, cfg.extra.get("slab_b", 10)
    S = dst_matrix(n)
    mu = t11_symbol(n, b)
    V3 = V.reshape(n, n, -1)
    W3 = np.einsum("ik,jl,klc->ijc", S, S, V3, optimize=True)
    W3 *= mu[:, :, None]
    return np.einsum("ik,jl,klc->ijc", S, S, W3, optimize=True).reshape(V.shape)


def kernel_block(cfg: Config, X: np.ndarray, rows: np.ndarray, cols: np.ndarray) -> np.ndarray:
    """Dense block A[rows, cols] (original point indices) of the config's operator."""
    rows = np.asarray(rows)
    cols = np.asarray(cols)
    if cfg.kernel == "t11":
        n, b = cfg.n, cfg.extra.get("slab_b", 10)
        S = dst_matrix(n)
        mu = t11_symbol(n, b).ravel()
        R = np.einsum("ri,rj->rij", S[rows // n], S[rows % n]).reshape(len(rows), n * n)   # rows of S (x) S
        C = np.einsum("ci,cj->cij", S[cols // n], S[cols % n]).reshape(len(cols), n * n)
        return (R * mu) @ C.T
    xi = X[rows][:, None, :]
    xj = X[cols][None, :, :]
    r = np.sqrt(((xi - xj) ** 2).sum(-1))
    same = rows[:, None] == cols[None, :]
    rs = np.where(same, 1.0, r)
    wgt = kernel_weight(cfg)
    if cfg.kernel == "log2d":
        K = wgt * np.log(rs)
    elif cfg.kernel == "lap3d":
        K = wgt / rs
    elif cfg.kernel == "helm2d":
        from scipy.special import hankel1
        K = wgt * 0.25j * hankel1(0, cfg.kappa * rs)
    else:
        raise ValueError(cfg.kernel)
    K = np.where(same, 0.0, K)
    A = K + same.astype(np.float64)
    return A.astype(cfg.np_dtype)


def dense_matrix(cfg: Config, X: np.ndarray | None = None) -> np.ndarray:
    """Full dense A (small N only)."""
    if X is None:
        X = points(cfg)
    idx = np.arange(X.shape[0])
    return kernel_block(cfg, X, idx, idx)


# ----------------------------------------------------------------------------
# seeded Gaussian test matrices
# ----------------------------------------------------------------------------
def _rng(seed: int, stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(np.random.SeedSequence([int(seed), int(stream)])))


def gaussian(shape, seed: int, stream: int, is_complex: bool = False) -> np.ndarray:
    """i.i.d. N(0,1) (real) or (N(0,1)+iN(0,1))/sqrt2 (complex), keyed by (seed, stream).

    Rows index ORIGINAL point order; callers permute to tree order.
    """
    g = _rng(seed, stream)
    if not is_complex:
        return g.standard_normal(shape)
    re = g.standard_normal(shape)
    im = g.standard_normal(shape)
    return (re + 1j * im) * (1.0 / math.sqrt(2.0))


def omega_psi(cfg: Config, N: int | None = None, p: int | None = None):
    """(Omega, Psi) of shape N x p in ORIGINAL point order."""
    N = cfg.N if N is None else N
    p = cfg.p if p is None else p
    Om = gaussian((N, p), cfg.seed, STREAM_OMEGA, cfg.is_complex)
    Ps = gaussian((N, p), cfg.seed, STREAM_PSI, cfg.is_complex)
    return Om, Ps


def rhs(cfg: Config, N: int | None = None, nrhs: int = 1) -> np.ndarray:
    N = cfg.N if N is None else N
    b = gaussian((N, nrhs), cfg.seed, STREAM_RHS, cfg.is_complex)
    return b[:, 0] if nrhs == 1 else b


def dense_samples(A: np.ndarray, Om: np.ndarray, Ps: np.ndarray):
    """Y = A Omega, Z = A^* Psi for a small dense operator."""
    return A @ Om, A.conj().T @ Ps
