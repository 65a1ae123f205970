"""Oracle: plain, slow, step-by-step RSRS (randomized strong recursive skeletonization).

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.  Shares no code with the
CUDA path.  One box at a time, in the canonical order, no batching, no reuse of
factorizations between steps, every formula written as the paper states it
(with the readings recorded in DESIGN.md section 3).

Notation: for a box b, I_b = its active indices,
near = active(I_b u I_n) (b and its neighbours), I_r / I_s = redundant /
skeleton split of I_b, c = near \\ I_r.

Per box (section 5):
  O4 nullify   Y' = Y_b null(Omega_near), Z' = Z_b null(Psi_near)
               (PAPER.md:1195-1200 eq. sketch_blocknull; 259-298 section 2.2)
  O5 ID        joint row ID of S = [Y', Z'] / sqrt(2w) by column-pivoted QR of
               S^*, k = #{|R_jj| > atol}, T = (R11^-1 R12)^*
  O6 E/F       Y_r -= T Y_s, Z_r -= T Z_s, Omega_s += T^* Omega_r,
               Psi_s += T^* Psi_r  (PAPER.md:915-933 eq. mod_fr, 1205-1212 with
               the consistency-forced orientation, reading R1)
  O7 extract   X_Y = Y_r pinv(Omega_near), X_Z = Z_r pinv(Psi_near)
               (393-449 section 2.3)
  O8 eliminate X_rr = X_Y[:, r], G_L = X_cr X_rr^-1, G_U = X_rr^-1 X_rc
               (PAPER.md:934-955 eqs. rr_eliminated, LU_elim_srs; 505-575)
  O9 L/U       Y_c -= G_L Y_r, Z_c -= G_U^* Z_r, Omega_r += G_U Omega_c,
               Psi_r += G_L^* Psi_c  (reading R1)
Levels L..top_level ("typically on level 2"),
children merged into parents, tolerance relaxed per level
(PAPER.md:1230-1231), then the dense skeleton block
A~_SS = Y_S pinv(Omega_S) (PAPER.md:1130-1143 eq. multi_level_decomp).

Solve / apply realise K = V_1 ... V_n A~_diag W_n ... W_1 with V = E L,
W = U F (PAPER.md:958-960 eq. Zmat; 455-457; elim inverse = sign toggle
PAPER.md:572-575).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla

from .tree import Tree


class RSRSError(RuntimeError):
    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


# ----------------------------------------------------------------------------
# dense primitives (section 2.1 / 3.1 / 3.2)
# ----------------------------------------------------------------------------
def null_basis(M: np.ndarray) -> np.ndarray:
    """Orthonormal basis (p x (p-r)) of the nullspace of the r x p matrix M.

    PAPER.md:262-264: "the operation null gives an orthogonal basis for the
    nullspace of matrix".  Complete Householder QR of M^* (LAPACK geqrf/orgqr);
    the trailing p - r columns of Q span null(M) when M has full row rank.
    """
    r, p = M.shape
    (qr, tau), _ = sla.qr(M.conj().T, mode="raw")
    E = np.zeros((p, p - r), dtype=qr.dtype)
    E[r:, :] = np.eye(p - r)
    # Q [0; I] = the trailing p - r columns of the complete Q (LAPACK ormqr/unmqr)
    if np.iscomplexobj(qr):
        out, _, info = sla.lapack.zunmqr("L", "N", qr, tau, E, lwork=max(1, 64 * p))
    else:
        out, _, info = sla.lapack.dormqr("L", "N", qr, tau, E, lwork=max(1, 64 * p))
    assert info == 0
    return out


def pinv_right(M: np.ndarray) -> np.ndarray:
    """Right pseudo-inverse M^dagger = M^* (M M^*)^-1 of a full-row-rank M (r x p).

    PAPER.md:429-432 (eq. pinv_omega).  Computed from the reduced QR
    M^* = Q R as M^dagger = Q R^-*.
    """
    Q, R = np.linalg.qr(M.conj().T, mode="reduced")
    # M^dagger = Q R^{-*}:  solve R^* X^T... write as (R^{-1} Q^*)^*
    Rinv_Qh = sla.solve_triangular(R, Q.conj().T, lower=False)
    return Rinv_Qh.conj().T


def row_id(S: np.ndarray, atol: float):
    """Row interpolative decomposition of S (n x m) at absolute tolerance atol.

    PAPER.md:653-666 (row ID: B(I_r,:) = T_rs B(I_s,:)) computed by a
    column-pivoted QR of S^* (LAPACK geqp3): S^*[:, piv] = Q [R11 R12],
    k = number of leading |R_jj| > atol, S[red,:] ~= T S[skel,:] with
    T = (R11^-1 R12)^*.  Returns (k, skel_local, red_local, T, R_diag) with
    skel / red sorted ascending and T's rows/columns in that order.
    """
    n = S.shape[0]
    if n == 0:
        return 0, np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros((0, 0), S.dtype), np.zeros(0)
    _, R, piv = sla.qr(S.conj().T, pivoting=True, mode="economic")
    diag = np.abs(np.diag(R))
    k = 0
    while k < diag.shape[0] and diag[k] > atol:
        k += 1
    skel_p = piv[:k]
    red_p = piv[k:]
    if k == 0:
        Tp = np.zeros((n, 0), dtype=S.dtype)
    elif k == n:
        Tp = np.zeros((0, k), dtype=S.dtype)
    else:
        Tp = sla.solve_triangular(R[:k, :k], R[:k, k:n]).conj().T   # (n-k) x k
    so = np.argsort(skel_p)
    ro = np.argsort(red_p)
    T = Tp[ro][:, so]
    return k, skel_p[so].astype(np.int64), red_p[ro].astype(np.int64), T, diag


# ----------------------------------------------------------------------------
# factorization record
# ----------------------------------------------------------------------------
@dataclass
class Step:
    level: int
    box: int
    skel: np.ndarray      # global tree positions, ascending
    red: np.ndarray       # global tree positions, ascending
    c: np.ndarray         # near \ red (global tree positions, near order)
    T: np.ndarray         # |red| x |skel|
    G_L: np.ndarray       # |c| x |red|
    G_U: np.ndarray       # |red| x |c|
    X_rr: np.ndarray      # |red| x |red|
    lu: tuple             # scipy lu_factor(X_rr)
    xrr_mismatch: float = 0.0   # ||X_rr^Y - X_rr^Z|| / ||X_rr^Y|| (SURVEY c.2 #9 diagnostic)
    # triangular form (Remark PAPER.md:577-611): X_rr = C C^* (Cholesky), M_L = X_cr C^-*, M_U = C^-1 X_rc
    C: np.ndarray | None = None
    M_L: np.ndarray | None = None
    M_U: np.ndarray | None = None


@dataclass
class Factorization:
    N: int
    p: int
    steps: list
    S: np.ndarray                     # remaining skeleton (tree positions)
    A_SS: np.ndarray
    lu_SS: tuple | None
    perm: np.ndarray                  # tree position -> original index
    ranks: dict = field(default_factory=dict)     # (level, box) -> k
    nb: dict = field(default_factory=dict)        # (level, box) -> |I_b|
    near: dict = field(default_factory=dict)      # (level, box) -> r
    atol: dict = field(default_factory=dict)      # level -> atol
    xrr_mismatch: list = field(default_factory=list)
    coupling: dict = field(default_factory=dict)  # (level, box) -> (est of |A~_{r,f}|_F, est of |A~_{f,r}|_F)
    dtype: object = np.float64
    triangular: bool = False          # factors stored in the triangular form (Remark PAPER.md:577-611)

    def memory(self) -> int:
        """Stored scalars (Table 1 'M').  Triangular form: T, C (triangle), M_L, M_U."""
        m = 0
        for s in self.steps:
            if self.triangular:
                nr = len(s.red)
                m += s.T.size + nr * (nr + 1) // 2 + s.M_L.size + s.M_U.size
            else:
                m += s.T.size + s.G_L.size + s.G_U.size + s.X_rr.size
        return m + self.A_SS.size


def atol_schedule(eps: float, c_id: float, g: float, L: int, lev: int) -> float:
    """atol(l) = c_id * eps * g^(L - l): relaxed at every level."""
    return c_id * eps * g ** (L - lev)


def noise_level(coupling: dict, reds: dict, lev: int) -> float:
    """nu(l): median over the boxes eliminated on level l of the per-row residual coupling
    max(|A~(r,f)|_F, |A~(f,r)|_F) / sqrt(|r|) -- the estimates of PAPER.md:1232-1235 ("estimate
    the extent to which A~_{r,f} and A~_{f,r} deviate from desired compression tolerance ...
    for every box").  0 if nothing was eliminated (reading R17)."""
    v = sorted(max(e) / math.sqrt(reds[key]) for key, e in coupling.items() if key[0] == lev and reds.get(key))
    if not v:
        return 0.0
    n = len(v)
    return v[n // 2] if n % 2 else 0.5 * (v[n // 2 - 1] + v[n // 2])


def noise_aware_atol(atol_prev: float, nu: float, theta: float) -> float:
    """Noise-aware relaxation (reading R17): the next coarser level
    never resolves below theta x the coupling the finer level left behind, and never tightens:
    atol(l - 1) = max(atol(l), theta * nu(l)); atol(L) = c_id * eps."""
    return max(atol_prev, theta * nu)


def coupling_estimate(Y_r, Om_r):
    """Randomized estimate of |A~(r, f)|_F, f = (1:N) minus r, after box b's elimination.

    PAPER.md:1232-1235 (section 5): "we use randomized sampling techniques (e.g. block
    nullification) to estimate the extent to which A~_{r,f} and A~_{f,r} deviate from
    desired compression tolerance, where in this case I_f = (1:N) minus I_r, for every box".
    With the current samples Y = A~ Omega (master invariant), Y_r null(Omega_r) =
    A~(r, f) Omega_f null(Omega_r), a Gaussian sketch of A~(r, f) with w = p - |r|
    columns, so its Frobenius norm / sqrt(w) estimates |A~(r, f)|_F (block nullification,
    PAPER.md:259-298).  The adjoint side uses Z, Psi for A~(f, r)^*.
    """
    nr, p = Y_r.shape
    if nr == 0:
        return 0.0
    return float(np.linalg.norm(Y_r @ null_basis(Om_r)) / math.sqrt(p - nr))


def factor(tree: Tree, Y, Z, Om, Psi, eps: float, c_id: float = 1.0, g: float = 1.0,
           l: int = 10, top_level: int = 2, on_step=None, max_boxes: int | None = None,
           copy: bool = True, estimate_coupling: bool = False, workers: int = 1,
           noise_factor: float = 0.0, triangular: bool = False) -> Factorization:
    """RSRS factorization from samples in TREE order (N x p each).

    The inputs are copied (unless copy=False); `on_step(step, Y, Z, Om, Psi)`
    (optional) sees the updated samples after each step (consistency tests).
    `max_boxes` stops after that many boxes in canonical order and returns the
    partial record (ranks of the boxes processed so far; no top block) -- used
    for sampled checks and bounded timing at full size.

    `workers` > 1 only changes WHEN boxes run, never what they compute: the boxes
    of one colour are >= 3 boxes apart (R10), so their near sets -- every
    row one box reads or writes -- are disjoint, and running them concurrently on a
    thread pool (LAPACK releases the GIL) gives bit-for-bit the result of the
    sequential canonical order (pinned by tests/test_oracle_rsrs.py).  Colours and
    levels stay strictly sequential.  Ignored when on_step or max_boxes is given.

    `noise_factor` theta > 0 replaces the fixed schedule by the noise-aware one (f1):
    the coupling estimator runs on every box and atol(l - 1) = max(atol(l), theta nu(l)).

    `triangular` stores the triangular form of the Remark for spd A:
    Cholesky X_rr = C C^*, M_L = X_cr C^-*, M_U = C^-1 X_rc; the sample
    updates are unchanged (with X_rr's Hermitian part).
    """
    if noise_factor > 0:
        estimate_coupling = True
    if copy:
        Y = np.array(Y, copy=True)
        Z = np.array(Z, copy=True)
        Om = np.array(Om, copy=True)
        Psi = np.array(Psi, copy=True)
    nproc = 0
    N, p = Y.shape
    dt = np.result_type(Y.dtype, Om.dtype)
    L = tree.L
    steps = []
    fac = Factorization(N=N, p=p, steps=steps, S=None, A_SS=None, lu_SS=None,
                        perm=tree.perm, dtype=dt, triangular=triangular)
    lv = tree.levels[L]
    act = [np.arange(lv.start[b], lv.start[b + 1], dtype=np.int64) for b in range(lv.nboxes)]
    pool = None
    blas_limit = None
    if workers > 1 and on_step is None and max_boxes is None:
        from concurrent.futures import ThreadPoolExecutor

        from threadpoolctl import threadpool_limits
        pool = ThreadPoolExecutor(max_workers=workers)
        blas_limit = threadpool_limits(limits=1)     # one BLAS thread per worker (no oversubscription)

    def process_box(lev, lv, b, atol):
        """O3-O9 for box b of level lev; returns (nb, r, k, coupling, Step or None)."""
        Ib = act[b]
        nb = Ib.shape[0]
        if nb == 0:
            return nb, None, 0, None, None
        near = np.concatenate([act[j] for j in lv.neighbours[b]])
        r = near.shape[0]
        w = p - r
        if w < l + 1:
            raise RSRSError("samples", f"level {lev} box {b}: p - r = {w} < l + 1 = {l + 1}")
        # O4 -- block nullification
        Yp = Y[Ib] @ null_basis(Om[near])
        Zp = Z[Ib] @ null_basis(Psi[near])
        # O5 -- joint row ID
        S = np.hstack([Yp, Zp]) / math.sqrt(2.0 * w)
        k, sk, rd, T, _ = row_id(S, atol)
        if k > min(nb, w - l):
            raise RSRSError("samples", f"level {lev} box {b}: rank {k} > w - l = {w - l}")
        if k == nb:
            return nb, r, k, None, None          # nothing to eliminate
        skel = Ib[sk]
        red = Ib[rd]
        Th = T.conj().T
        # O6 -- E/F sample updates
        if k > 0:
            Y[red] -= T @ Y[skel]
            Z[red] -= T @ Z[skel]
            Om[skel] += Th @ Om[red]
            Psi[skel] += Th @ Psi[red]
        # O7 -- block extraction
        X_Y = Y[red] @ pinv_right(Om[near])          # X_{r,near}
        X_Z = Z[red] @ pinv_right(Psi[near])         # (X_{near,r})^*
        # O8 -- block Gaussian elimination
        is_red = np.isin(near, red)
        pos_red = np.flatnonzero(is_red)
        pos_c = np.flatnonzero(~is_red)
        # near lists I_b in ascending order, so pos_red follows `red`'s order
        assert np.array_equal(near[pos_red], red)
        c = near[pos_c]
        X_rr = X_Y[:, pos_red]
        X_rc = X_Y[:, pos_c]
        X_cr = X_Z[:, pos_c].conj().T
        mism = np.linalg.norm(X_rr - X_Z[:, pos_red].conj().T) / max(np.linalg.norm(X_rr), 1e-300)
        Cf = M_L = M_U = None
        if triangular:
            # Remark PAPER.md:577-611: for spd A, A_11 = C_11 C_11^* and the elimination factors
            # become [C 0; A_21 C^-* I] and [C^* C^-1 A_12; 0 I] (no block-diagonal middle).  X_rr
            # from the samples is Hermitian only to the compression error: take its Hermitian
            # part (reading R18).
            X_rr = 0.5 * (X_rr + X_rr.conj().T)
            try:
                Cf = sla.cholesky(X_rr, lower=True)
            except np.linalg.LinAlgError:
                raise RSRSError("singular", f"level {lev} box {b}: X_rr not positive definite") from None
            M_U = sla.solve_triangular(Cf, X_rc, lower=True)                  # C^-1 X_rc
            M_L = sla.solve_triangular(Cf, X_cr.conj().T, lower=True).conj().T  # X_cr C^-*
        lu = sla.lu_factor(X_rr, check_finite=True)
        if np.min(np.abs(np.diag(lu[0]))) == 0.0:
            raise RSRSError("singular", f"level {lev} box {b}: X_rr singular")
        G_U = sla.lu_solve(lu, X_rc)                       # X_rr^-1 X_rc
        G_L = sla.lu_solve(lu, X_cr.T, trans=1).T          # X_cr X_rr^-1
        # O9 -- L/U sample updates
        Yr = Y[red].copy()
        Zr = Z[red].copy()
        Y[c] -= G_L @ Yr
        Z[c] -= G_U.conj().T @ Zr
        Om[red] += G_U @ Om[c]
        Psi[red] += G_L.conj().T @ Psi[c]
        cpl = None
        if estimate_coupling:
            cpl = (coupling_estimate(Y[red], Om[red]), coupling_estimate(Z[red], Psi[red]))
        st = Step(level=lev, box=b, skel=skel, red=red, c=c, T=T, G_L=G_L, G_U=G_U,
                  X_rr=X_rr, lu=lu, C=Cf, M_L=M_L, M_U=M_U)
        st.xrr_mismatch = mism
        return nb, r, k, cpl, st

    reds = {}            # (level, box) -> |r| of the boxes with a coupling estimate

    def record(lev, b, res):
        nb, r, k, cpl, st = res
        fac.nb[(lev, b)] = nb
        fac.ranks[(lev, b)] = k
        if r is not None:
            fac.near[(lev, b)] = r
        if st is not None:
            fac.xrr_mismatch.append(st.xrr_mismatch)
            if cpl is not None:
                fac.coupling[(lev, b)] = cpl
                reds[(lev, b)] = len(st.red)
            steps.append(st)
            act[b] = st.skel

    try:
        lev = L
        while lev >= top_level and lev >= 1:
            lv = tree.levels[lev]
            if noise_factor > 0:
                atol = c_id * eps if lev == L else noise_aware_atol(
                    fac.atol[lev + 1], noise_level(fac.coupling, reds, lev + 1), noise_factor)
            else:
                atol = atol_schedule(eps, c_id, g, L, lev)
            fac.atol[lev] = atol
            order = tree.canonical_order(lev)
            if pool is None:
                for b in order:
                    if max_boxes is not None and nproc >= max_boxes:
                        fac.S = np.zeros(0, np.int64)
                        fac.A_SS = np.zeros((0, 0), dtype=dt)
                        return fac
                    nproc += 1
                    res = process_box(lev, lv, b, atol)
                    record(lev, b, res)
                    if res[4] is not None and on_step is not None:
                        on_step(res[4], Y, Z, Om, Psi)
            else:
                # one colour at a time (canonical order); its boxes touch disjoint rows
                for col in sorted(set(int(lv.colour[b]) for b in order)):
                    group = [b for b in order if lv.colour[b] == col]
                    results = list(pool.map(lambda b: process_box(lev, lv, b, atol), group))
                    for b, res in zip(group, results):
                        record(lev, b, res)
            # O10 -- merge children into parents
            if lev - 1 >= 0:
                parent_level = tree.levels[lev - 1]
                kids = parent_level.children_of(lv)
                act = [np.concatenate([act[j] for j in kids[q]]) if kids[q] else np.zeros(0, np.int64)
                       for q in range(parent_level.nboxes)]
            lev -= 1
        # O11 -- top block A~_SS = Y_S pinv(Omega_S)
        S = np.concatenate(act) if act else np.zeros(0, np.int64)
        fac.S = S
        if S.shape[0] > 0:
            if S.shape[0] + l > p:
                raise RSRSError("samples", f"top block |S| = {S.shape[0]} needs p >= |S| + l = {S.shape[0] + l}")
            fac.A_SS = Y[S] @ pinv_right(Om[S])
            fac.lu_SS = sla.lu_factor(fac.A_SS)
        else:
            fac.A_SS = np.zeros((0, 0), dtype=dt)
    finally:
        if pool is not None:
            pool.shutdown()
            blas_limit.restore_original_limits()
    return fac


# ----------------------------------------------------------------------------
# solve / apply
# ----------------------------------------------------------------------------
def _to_tree(fac: Factorization, v):
    v = np.asarray(v)
    return np.array(v[fac.perm], dtype=np.result_type(v.dtype, fac.dtype), copy=True)


def _from_tree(fac: Factorization, x):
    out = np.empty_like(x)
    out[fac.perm] = x
    return out


def _solve_triangular_form(fac: Factorization, x):
    """K = V_1 .. V_n A~_SS W_n .. W_1 with V = E [C 0; M_L I], W = [C^* M_U; 0 I] F (Remark
    PAPER.md:577-611): the eliminated blocks of the middle factor are identities."""
    for s in fac.steps:                      # V_i^-1: E^-1, then [C 0; M_L I]^-1
        x[s.red] -= s.T @ x[s.skel]
        x[s.red] = sla.solve_triangular(s.C, x[s.red], lower=True)
        x[s.c] -= s.M_L @ x[s.red]
    if fac.S.shape[0]:
        x[fac.S] = sla.lu_solve(fac.lu_SS, x[fac.S])
    for s in reversed(fac.steps):            # W_i^-1: [C^* M_U; 0 I]^-1, then F^-1
        x[s.red] = sla.solve_triangular(s.C, x[s.red] - s.M_U @ x[s.c], lower=True, trans="C")
        x[s.skel] -= s.T.conj().T @ x[s.red]
    return _from_tree(fac, x)


def _apply_triangular_form(fac: Factorization, x):
    for s in fac.steps:                      # W_i = [C^* M_U; 0 I] F
        x[s.skel] += s.T.conj().T @ x[s.red]
        x[s.red] = s.C.conj().T @ x[s.red] + s.M_U @ x[s.c]
    if fac.S.shape[0]:
        x[fac.S] = fac.A_SS @ x[fac.S]
    for s in reversed(fac.steps):            # V_i = E [C 0; M_L I]
        x[s.c] += s.M_L @ x[s.red]
        x[s.red] = s.C @ x[s.red]
        x[s.red] += s.T @ x[s.skel]
    return _from_tree(fac, x)


def solve(fac: Factorization, b) -> np.ndarray:
    """x = K^-1 b = W_1^-1 ... W_n^-1 A~_diag^-1 V_n^-1 ... V_1^-1 b (original order)."""
    x = _to_tree(fac, b)
    if fac.triangular:
        return _solve_triangular_form(fac, x)
    for s in fac.steps:                      # V_i^-1 = L_i^-1 E_i^-1
        x[s.red] -= s.T @ x[s.skel]
        x[s.c] -= s.G_L @ x[s.red]
    for s in fac.steps:                      # A~_diag^-1
        x[s.red] = sla.lu_solve(s.lu, x[s.red])
    if fac.S.shape[0]:
        x[fac.S] = sla.lu_solve(fac.lu_SS, x[fac.S])
    for s in reversed(fac.steps):            # W_i^-1 = F_i^-1 U_i^-1
        x[s.red] -= s.G_U @ x[s.c]
        x[s.skel] -= s.T.conj().T @ x[s.red]
    return _from_tree(fac, x)


def apply(fac: Factorization, v) -> np.ndarray:
    """K v = V_1 ... V_n A~_diag W_n ... W_1 v (original order)."""
    x = _to_tree(fac, v)
    if fac.triangular:
        return _apply_triangular_form(fac, x)
    for s in fac.steps:                      # W_i = U_i F_i
        x[s.skel] += s.T.conj().T @ x[s.red]
        x[s.red] += s.G_U @ x[s.c]
    for s in fac.steps:                      # A~_diag
        x[s.red] = s.X_rr @ x[s.red]
    if fac.S.shape[0]:
        x[fac.S] = fac.A_SS @ x[fac.S]
    for s in reversed(fac.steps):            # V_i = E_i L_i
        x[s.c] += s.G_L @ x[s.red]
        x[s.red] += s.T @ x[s.skel]
    return _from_tree(fac, x)
