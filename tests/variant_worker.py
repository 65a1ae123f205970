"""Child process of tests/test_gpu_variants.py::test_nn_stream_bit_identical: factor + solve + apply
the sphere case with whatever RSRS_* switches the parent set, print a digest of the ranks, x and Kb."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import workloads as W  # noqa: E402
from gpu_common import dense_problem, gpu_apply, gpu_solve, run_gpu  # noqa: E402

cfg = W.CONFIGS["c3"].scaled(int(sys.argv[1]) if len(sys.argv) > 1 else 8192)
X, A, Y, Z, Om, Ps, b = dense_problem(cfg)
t, f = run_gpu(cfg, X, Y, Z, Om, Ps, cfg.root())
h = hashlib.sha256()
for lev in range(t.L, 1, -1):
    h.update(np.ascontiguousarray(f.ranks(lev, len(t.level(lev)["keys"]))).tobytes())
h.update(np.ascontiguousarray(gpu_solve(f, b)).tobytes())
h.update(np.ascontiguousarray(gpu_apply(f, b)).tobytes())
print("DIGEST", h.hexdigest(), "launches", f.stats()["launches"])
