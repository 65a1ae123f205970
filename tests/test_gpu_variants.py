"""Kernel-variant coverage: the launch-shape switches of the factor driver (fused per-matrix Cholesky /
back substitution, 32-row GEMM tiles, packed solve records, sweep-graph replay) change how the same
arithmetic is scheduled, not what it computes.  Small parity cases never reach the thresholds that select
them in production (batches of >= 128 matrices, levels of small boxes), so this file re-runs parity
tests of test_gpu_parity.py in a child process with each switch forced, against the oracle as usual."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


VARIANTS = {
    # every real Cholesky / back substitution by the fused one-CTA-per-matrix kernels
    "fused_cholesky": {"RSRS_CHOL_FUSE_RMAX": "100000", "RSRS_BACK_FUSE_RMAX": "100000", "RSRS_FUSE_MIN_BATCH": "1"},
    # no fused kernels at all (the per-panel launch chain)
    "panel_cholesky": {"RSRS_CHOL_FUSE_RMAX": "0", "RSRS_BACK_FUSE_RMAX": "0"},
    # 32-row tiles for every real GEMM / 64-row tiles wherever allowed
    "tiles_32": {"RSRS_TM32_NT": "100000", "RSRS_TM32_NN": "100000"},
    "tiles_64": {"RSRS_TM32_RATIO": "0"},
    # 32-row tiles without the 16-row split for small-box descriptors
    "no_tiles_16": {"RSRS_TM16": "0"},
    "nn_tiles_16": {"RSRS_TM16_NN": "1"},
    # packed Gram-block row blocks on the small-box levels (consecutive boxes share one 32-row block)
    "gram_pack": {"RSRS_GRAM_PACK": "32"},
    # stream drains after every level setup / compaction (the round-1 host schedule)
    "level_sync": {"RSRS_LEVEL_SYNC": "1"},
    # two-level Cholesky diagonal blocks (16 x 16 warp sub-blocks; off by default: slower on c3)
    "diag_two_level": {"RSRS_DIAG16": "1"},
    # L/U push through the tiled GEMM only (no nn_stream_kernel) / E-F updates through nn_stream_kernel too
    "no_nn_stream": {"RSRS_NS_KMAX": "0"},
    "ef_stream": {"RSRS_EF_STREAM": "1"},
    "nn_stream_one_chunk": {"RSRS_NS_CHUNKS": "1", "RSRS_EF_STREAM": "1"},
    # projection / pulled L/U update through the column-walking nn_kstream_kernel
    "nn_kstream": {"RSRS_KS_MMAX": "100000"},
    "nn_kstream_one_chunk": {"RSRS_KS_MMAX": "100000", "RSRS_KS_CHUNKS": "1", "RSRS_KS_LEFTOVERS": "1"},
    # solve from the factor pools (no packed records, LU top block), kernel-by-kernel launches
    "unpacked_solve": {"RSRS_SOLVE_PACKED": "0", "RSRS_SWEEP_GRAPH": "0"},
}


@pytest.mark.parametrize("name", sorted(VARIANTS))
def test_variant_parity(name):
    env = dict(os.environ)
    env.update(VARIANTS[name])
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
           os.path.join(HERE, "test_gpu_parity.py"), "-k", "c1_parity or sphere_small or multiple_rhs"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1800)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "no tests ran" not in r.stdout, r.stdout[-2000:]


def _digest(extra_env):
    env = dict(os.environ)
    env.update(extra_env)
    r = subprocess.run([sys.executable, os.path.join(HERE, "variant_worker.py"), "8192"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=1800)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    line = [x for x in r.stdout.splitlines() if x.startswith("DIGEST")][-1].split()
    return line[1], int(line[3])


def test_nn_stream_bit_identical():
    """nn_stream_kernel / nn_kstream_kernel issue the same DMMA sequence per output element as the
    tiled gemm_nn_kernel: ranks, x and Kb of the sphere case are bit-identical with the L/U push
    through either (so the full-size oracle parity runs, made with the tiled kernel, carry over)."""
    tiled, l0 = _digest({"RSRS_NS_KMAX": "0", "RSRS_KS_MMAX": "0"})
    stream, l1 = _digest({"RSRS_NS_KMAX": "32", "RSRS_KS_MMAX": "0"})
    walk, l2 = _digest({"RSRS_NS_KMAX": "100000", "RSRS_NS_CHUNKS": "3", "RSRS_KS_MMAX": "100000"})
    assert stream == tiled and walk == tiled
    assert l1 != l0 or l2 != l0   # the switches did select other launches
