"""f3: RSRS of the sparse Schur complement T11 of a 3D Poisson slab
decomposition (slab width b = 10, atol = 5e-6, 100-point leaves) on the GPU against the oracle, on the
same sample bytes: a dense case (N = 6400) and the frozen full configuration (N = 102,400) through
the full-size parity driver (samples from the harness T11 operator, row-verified)."""
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


def test_t11_dense_parity():
    cfg = W.CONFIGS["t11"].scaled(80)
    out = _parity(cfg, None, cfg.root())
    assert out["t_or"].L == 3


def test_t11_full_size_vs_oracle():
    res = run_parity(W.CONFIGS["t11"])
    assert res["pass"], res["criteria"]
    assert res["L"] == 5
