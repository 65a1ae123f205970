"""GPU vs oracle at BASELINE.json's full size and on deep trees (north_star bar:
||x_gpu - x_or|| / ||x_or|| <= 10 eps, both residuals <= 10 eps, |dk| <= 2 on every
box of every level), on the same GPU-sampled input bytes (driver in
tests/parity_full.py).  The remaining full-size configurations (c3, c4, c5: 10-45 min
of oracle time each) run through tests/parity_full.py on a GPU box and are kept in
profiles/r02_parity_c*.json.  Also: the n_r > 64 branch of the per-box LU
(extract_lu_kernel's shared-memory LU + inverse, dense.cuh), real and complex."""
import numpy as np
import pytest

import workloads as W
from parity_full import run_parity
from test_gpu_parity import _parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _check(res):
    assert res["sample_rows_max_relerr"] <= 1e-13 * np.sqrt(res["N"]) * (10 if res["dtype"] == "c128" else 1)
    assert res["x_relerr_gpu_vs_oracle"] <= 10 * res["eps"], res["x_relerr_gpu_vs_oracle"]
    assert res["residual_gpu"] <= 10 * res["eps"] and res["residual_oracle"] <= 10 * res["eps"]
    assert res["max_abs_dk"] <= 2, res["levels"]
    assert res["pass"]


def test_c2_full_size_vs_oracle():
    """configs[1] (c2, N = 262,144, L = 6; the 2D log kernel): every one of the 5,456 boxes."""
    res = run_parity(W.CONFIGS["c2"])
    _check(res)
    assert res["L"] == 6 and res["boxes_compared"] > 5000


def test_deep_sphere_vs_oracle():
    """The sphere configurations' operator and frozen parameters (c3: p = 1216, g = 2) at
    N = 65,536: octree depth L = 5, four compressed levels, coarse boxes of up to 8 x 15
    skeletons."""
    res = run_parity(W.CONFIGS["c3"].scaled(65536))
    _check(res)
    assert res["L"] >= 5


def _big_box_case(cplx):
    # leaf boxes of 100 (real) / 81 (complex) points with ranks ~7: n_r > 64
    if cplx:
        cfg = W.Config("bigbox_c", "grid2d", 72, "helm2d", "c128", leaf=81, p=800, seed=41, g=2.0)
    else:
        cfg = W.Config("bigbox", "grid2d", 80, "log2d", "f64", leaf=100, p=960, seed=40, g=2.0)
    return cfg


@pytest.mark.parametrize("cplx", [False, True], ids=["f64", "c128"])
def test_redundant_block_above_64_vs_oracle(cplx):
    """Boxes with n_r > 64 take the shared-memory LU + explicit inverse of X_rr
    (dense.cuh extract_lu_kernel, n_r > 64 branch) instead of the register Gauss-Jordan."""
    cfg = _big_box_case(cplx)
    out = _parity(cfg, None, cfg.root())
    f_or = out["f_or"]
    assert max(len(s.red) for s in f_or.steps) > 64
