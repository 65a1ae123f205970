import os
import sys

# Single-threaded BLAS for the oracle: multi-threaded OpenBLAS is 10-50x slower on
# the small LAPACK calls the oracle makes in this container.
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import pytest  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA device) and the built librsrs.so")
    config.addinivalue_line("markers", "slow: long-running test")
