"""The NCCL leg of the multi-rank path (one ncclAllReduce of the partial interface vector per
iteration, captured in the PCG graph): two processes, one per GPU, through torchrun. Needs two visible GPUs -- the
graft GPU boxes show one, where this test skips and the same host logic runs through the single-GPU loopback group
(tests/test_gpu_loopback.py)."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_two_ranks_over_nccl_match_single_rank():
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr", "127.0.0.1",
           "--master-port", "29731", os.path.join(ROOT, "tools", "nccl_ranks_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
