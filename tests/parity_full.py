"""Full-size parity of the CUDA path against the CPU oracle (SURVEY 8(c) O0 / c.3 "GPU vs oracle").

TEST INFRASTRUCTURE (it imports oracle/; see oracle/__init__.py).  Used by
tests/test_gpu_parity_full.py (-m gpu) and, for the largest configurations, run
directly on a GPU box:

    python tests/parity_full.py --config c3 [--workers N] [--out profiles/r02_parity_c3.json]

One seeded problem of a BASELINE.json configuration at its full size:
  1. Omega, Psi, b drawn by workloads (numpy Philox, original point order), moved
     to the device in tree order;
  2. Y = A Omega, Z = A^* Psi by the harness operator on the GPU (libsampler.so),
     verified against CPU direct sums on >= 256 random rows per array (SURVEY O0:
     the paper measures on "a subset of points");
  3. the SAME sample bytes are copied to the host (the oracle's inputs) before the
     GPU factorization overwrites its device copies;
  4. GPU: rsrs_factor + rsrs_solve through the C ABI;
  5. oracle: oracle.factor + oracle.solve on the host copies (LAPACK, one BLAS
     thread per worker; boxes of one colour on `workers` threads, bit-identical
     to the sequential canonical order);
  6. the north_star bar: ||x_gpu - x_or|| / ||x_or|| <= 10 eps, both residuals
     ||A x - b|| / ||b|| <= 10 eps (exact A through the on-the-fly operator), and
     |k_gpu - k_or| <= 2 for every box of every level.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import platform
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for _p in (ROOT, HERE):
    if _p not in sys.path:
        sys.path.insert(0, _p)

import oracle as O  # noqa: E402
import workloads as W  # noqa: E402


def host_info(workers: int) -> dict:
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    blas = {}
    try:
        from threadpoolctl import threadpool_info
        for d in threadpool_info():
            if d.get("user_api") == "blas":
                blas = {"internal_api": d.get("internal_api"), "version": d.get("version"),
                        "num_threads": d.get("num_threads")}
                break
    except Exception:  # noqa: BLE001
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model, "python": platform.python_version(),
            "numpy": np.__version__, "blas": blas, "oracle_workers": workers, "blas_threads_per_worker": 1}


def run_parity(cfg, workers: int | None = None, verify_rows: int = 256, log=print) -> dict:
    """Run GPU and oracle on the same GPU-sampled bytes; return the comparison record."""
    import torch
    from threadpoolctl import threadpool_limits

    import paper_2311_01451_b200 as R
    workers = workers or os.cpu_count() or 1
    dev = torch.device("cuda:0")
    out = {"config": cfg.name, "N": cfg.N, "p": cfg.p, "eps": cfg.eps, "g": cfg.g, "c_id": cfg.c_id, "l": cfg.l,
           "kernel": cfg.kernel, "dtype": cfg.dtype, "host": host_info(workers)}
    X = W.points(cfg)
    N = X.shape[0]
    t_g = R.Tree(X, cfg.leaf, *cfg.root())
    t_o = O.build_tree(X, cfg.leaf, *cfg.root())
    perm = t_g.perm()
    assert np.array_equal(perm, t_o.perm), "C++ tree and oracle tree disagree"
    out["L"] = t_o.L
    # ---- 1. seeded inputs (original order) -> device, tree order
    t0 = time.perf_counter()
    Om, Ps = W.omega_psi(cfg)
    b = W.rhs(cfg)
    P = torch.from_numpy(perm).to(dev)
    Om_d = torch.from_numpy(Om).to(dev)[P].contiguous()
    Ps_d = torch.from_numpy(Ps).to(dev)[P].contiguous()
    del Om, Ps
    pts = np.zeros((N, 3))
    pts[:, :X.shape[1]] = X
    pts_d = torch.from_numpy(pts[perm]).to(dev)
    wgt = W.kernel_weight(cfg)
    # ---- 2. samples on the GPU (harness operator), row-verified
    Y_d = torch.empty_like(Om_d)
    Z_d = torch.empty_like(Ps_d)
    R.sample_matvec(cfg.kernel, pts_d, wgt, Om_d, Y_d, kappa=cfg.kappa)
    R.sample_matvec(cfg.kernel, pts_d, wgt, Ps_d, Z_d, adjoint=True, kappa=cfg.kappa)
    torch.cuda.synchronize()
    out["t_inputs_s"] = time.perf_counter() - t0
    # ---- 3. the same bytes on the host (oracle inputs), tree order
    t0 = time.perf_counter()
    Yh, Zh, Omh, Psh = (T.cpu().numpy() for T in (Y_d, Z_d, Om_d, Ps_d))
    out["t_d2h_s"] = time.perf_counter() - t0
    rng = np.random.default_rng(12345)
    rows = np.sort(rng.choice(N, min(verify_rows, N), replace=False))
    worst = 0.0
    with threadpool_limits(limits=workers):
        for lo in range(0, rows.shape[0], 32):
            rr = rows[lo:lo + 32]
            Ab = W.kernel_block(cfg, X, perm[rr], perm)          # A[tree rows, tree cols]
            for S, V, adj in ((Yh, Omh, False), (Zh, Psh, True)):
                ref = (Ab.conj() if adj else Ab) @ V              # A^* rows = conj(A) rows (symmetric kernels)
                worst = max(worst, float(np.abs(S[rr] - ref).max() / max(np.abs(ref).max(), 1e-300)))
    out["sample_rows_verified"] = int(rows.shape[0])
    out["sample_rows_max_relerr"] = worst
    tol = (1e-12 if cfg.is_complex else 1e-13) * math.sqrt(N)
    assert worst <= tol, f"GPU samples disagree with CPU direct sums: {worst:.2e} > {tol:.2e}"

    def A_apply(v_orig):     # exact A v in original order through the on-the-fly operator
        vt = v_orig[P].contiguous().view(N, 1)
        res = torch.empty_like(vt)
        R.sample_matvec(cfg.kernel, pts_d, wgt, vt, res, kappa=cfg.kappa)
        o = torch.empty_like(res.view(N))
        o[P] = res.view(N)
        return o

    # ---- 4. GPU factor + solve (overwrites the device samples)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f = R.factor(t_g, Y_d, Z_d, Om_d, Ps_d, p=cfg.p, eps=cfg.eps, level_growth=cfg.g, id_scale=cfg.c_id,
                 oversample=cfg.l)
    out["t_gpu_factor_call_s"] = time.perf_counter() - t0
    del Y_d, Z_d, Om_d, Ps_d
    torch.cuda.empty_cache()
    st = f.stats()
    out["gpu_factor_ms"] = st["factor_ms"]
    bd = torch.from_numpy(b.copy()).to(dev)
    x_gd = bd.clone()
    f.solve(x_gd)
    torch.cuda.synchronize()
    x_g = x_gd.cpu().numpy()
    nb_ = float(bd.norm())
    out["residual_gpu"] = float((A_apply(x_gd) - bd).norm()) / nb_
    # ---- 5. oracle factor + solve on the host copies
    log(f"[parity {cfg.name}] GPU factor {st['factor_ms']:.0f} ms, residual {out['residual_gpu']:.2e}; oracle with "
        f"{workers} workers ...")
    t0 = time.perf_counter()
    with threadpool_limits(limits=1):
        fo = O.factor(t_o, Yh, Zh, Omh, Psh, cfg.eps, c_id=cfg.c_id, g=cfg.g, l=cfg.l, copy=False, workers=workers)
        out["oracle_factor_s"] = time.perf_counter() - t0
        t1 = time.perf_counter()
        x_o = O.solve(fo, b)
        out["oracle_solve_s"] = time.perf_counter() - t1
    del Yh, Zh, Omh, Psh
    out["residual_oracle"] = float((A_apply(torch.from_numpy(x_o).to(dev)) - bd).norm()) / nb_
    # ---- 6. comparison
    out["x_relerr_gpu_vs_oracle"] = float(np.linalg.norm(x_g - x_o) / np.linalg.norm(x_o))
    lv_stats = {}
    worst_dk = 0
    nboxes = 0
    for lev in range(t_o.L, 1, -1):
        nbx = t_o.levels[lev].nboxes
        kg = f.ranks(lev, nbx)
        ko = np.array([fo.ranks.get((lev, j), -1) if fo.nb.get((lev, j), 0) > 0 else -1 for j in range(nbx)])
        m = (ko >= 0) | (kg >= 0)          # boxes with active rows on either side (empty = rank 0)
        dk = np.abs(np.maximum(kg[m], 0).astype(np.int64) - np.maximum(ko[m], 0))
        lv_stats[str(lev)] = {"boxes": int(m.sum()), "max_abs_dk": int(dk.max()) if dk.size else 0,
                              "boxes_dk_nonzero": int((dk > 0).sum()),
                              "empty_box_mismatch": int(((kg < 0) != (ko < 0)).sum()),
                              "k_oracle_min_mean_max": [int(ko[ko >= 0].min()), float(ko[ko >= 0].mean()),
                                                        int(ko[ko >= 0].max())] if (ko >= 0).any() else None,
                              "max_n_r": int(max((len(s.red) for s in fo.steps if s.level == lev), default=0)),
                              "atol": fo.atol.get(lev)}
        worst_dk = max(worst_dk, lv_stats[str(lev)]["max_abs_dk"])
        nboxes += int(m.sum())
    out["levels"] = lv_stats
    out["boxes_compared"] = nboxes
    out["max_abs_dk"] = worst_dk
    out["top_size_gpu"] = st["top_size"]
    out["top_size_oracle"] = int(fo.S.shape[0])
    out["memory_scalars_gpu"] = st["memory_scalars"]
    out["memory_scalars_oracle"] = int(fo.memory())
    out["max_xrr_mismatch_oracle"] = float(max(fo.xrr_mismatch, default=0.0))
    eps = cfg.eps
    out["criteria"] = {"x_relerr<=10eps": out["x_relerr_gpu_vs_oracle"] <= 10 * eps,
                       "residual_gpu<=10eps": out["residual_gpu"] <= 10 * eps,
                       "residual_oracle<=10eps": out["residual_oracle"] <= 10 * eps,
                       "all_boxes_|dk|<=2": worst_dk <= 2}
    out["pass"] = all(out["criteria"].values())
    log(f"[parity {cfg.name}] oracle {out['oracle_factor_s']:.0f} s; |x_g - x_o|/|x_o| = "
        f"{out['x_relerr_gpu_vs_oracle']:.2e}, residuals {out['residual_gpu']:.2e} / {out['residual_oracle']:.2e}, "
        f"max |dk| = {worst_dk} over {nboxes} boxes -> {'PASS' if out['pass'] else 'FAIL'}")
    return out


def config_by_name(name: str):
    """c1..c5, or a scaled member 'c3@65536' (same kernel / p / eps / g / c_id)."""
    if "@" in name:
        base, n = name.split("@")
        return W.CONFIGS[base].scaled(int(n))
    return W.CONFIGS[name]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--workers", type=int, default=0)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    cfg = config_by_name(a.config)
    res = run_parity(cfg, workers=a.workers or None)
    js = json.dumps(res, indent=1)
    if a.out:
        os.makedirs(os.path.dirname(os.path.abspath(a.out)), exist_ok=True)
        with open(a.out, "w") as fh:
            fh.write(js + "\n")
    print(js)
    sys.exit(0 if res["pass"] else 1)


if __name__ == "__main__":
    main()
