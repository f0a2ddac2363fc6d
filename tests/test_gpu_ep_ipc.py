"""Expert parallelism across two PROCESSES on one GPU through the CUDA-IPC peer-memory
transport (ep.PeerComm) -- the c5 bench's default transport -- against the single-process
oracle on the concatenated batch (tools/ep2_on_one_gpu.py under torch.distributed.run)."""
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


@pytest.mark.parametrize("flags", [[], ["--unfused"]])
def test_ep_peercomm_two_processes(flags):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tools", "ep2_on_one_gpu.py"), *flags]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert p.stdout.count("EP2 IPC OK") == 2, p.stdout[-3000:]
