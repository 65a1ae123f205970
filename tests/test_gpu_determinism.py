"""Determinism of the CUDA path (compute-sanitizer is closed on this GPU pool, so races are checked
by their symptom): the same inputs factored twice give bit-identical ranks, solutions and applies,
on a 2D case with Gram blocks and pulled updates (c1), the sphere (27 colours, ragged boxes) and
complex128.  A data race between same-colour boxes or between the warps / CTAs of a kernel would
show up as run-to-run differences."""
import numpy as np
import pytest

import workloads as W
from gpu_common import dense_problem, gpu_apply, gpu_solve, run_gpu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


@pytest.mark.parametrize("name,n", [("c1", None), ("c3", 8192), ("c4", 64)], ids=["c1", "sphere8k", "c4_64"])
def test_factor_solve_bit_identical_across_runs(name, n):
    cfg = W.CONFIGS[name] if n is None else W.CONFIGS[name].scaled(n)
    X, A, Y, Z, Om, Ps, b = dense_problem(cfg)
    outs = []
    for _ in range(3):
        t, f = run_gpu(cfg, X, Y, Z, Om, Ps, cfg.root())
        ranks = [f.ranks(lev, len(t.level(lev)["keys"])) for lev in range(t.L, 1, -1)]
        outs.append((ranks, gpu_solve(f, b), gpu_apply(f, b), f.stats()["memory_scalars"]))
    for o in outs[1:]:
        assert all(np.array_equal(a, c) for a, c in zip(o[0], outs[0][0]))
        assert np.array_equal(o[1], outs[0][1]) and np.array_equal(o[2], outs[0][2])
        assert o[3] == outs[0][3]
