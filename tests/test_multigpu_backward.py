"""Multi-card layer backward with one process per GPU (NVLink peer memory):
tests/mp_backward_worker.py checks the closed forms on every rank for the
naive exchange and the TP-deduplicated O1/O2 levels.  Needs e*t GPUs."""
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("e,t", [(2, 1), (1, 2), (2, 2)])
def test_layer_backward_multiprocess(e, t):
    world = e * t
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs, have {torch.cuda.device_count()}")
    runs = "0:1:0" if (e == 1 or t == 1) else "1:1:0,2:2:0,3:2:1,0:1:0"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={_port()}",
           os.path.join(ROOT, "tests", "mp_backward_worker.py"), "--groups", str(e), "--tp", str(t), "--runs", runs]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
