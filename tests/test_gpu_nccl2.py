"""Real 2-process NCCL run of the multi-GPU sweep (one process per GPU, torchrun): bit-identical
to the emulated 2-rank factorization (which tests/test_gpu_dist.py pins to the single-GPU
result).  Skips below 2 GPUs (gpurun boxes have one)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def test_two_rank_nccl_matches_emulation():
    import torch
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(HERE, "nccl2_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
