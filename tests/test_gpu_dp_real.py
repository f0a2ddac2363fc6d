"""Two data-parallel ranks of the real engine (graph-captured step with its backward side stream)
sharing one GPU over gloo: gradients and loss equal one process on the concatenated batch
(tools/dp2_on_one_gpu.py, launched with torch.distributed.run on 127.0.0.1)."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("opts", [[], ["peer", "overlap"]])
def test_dp_two_ranks_real_engine_equals_single_process(opts):
    """opts: the LoadStats exchange over CUDA-IPC peer memory (csrc/comm.cu) and the gradient
    buckets reduced on a communication stream under the backward."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tools", "dp2_on_one_gpu.py"), *opts]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-2000:]
    assert "DP2 OK" in p.stdout
