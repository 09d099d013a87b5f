"""The multi-rank path end to end on a GPU box (tools/multirank_check.py under torchrun,
world size 2): map replication, delta broadcast, strided ID shards all-gathered in input
order and bit-identical to the unsharded ID, replicated frame integration.  On a one-GPU box
both ranks share the device and the collectives run over gloo (through the host), so no
rank's kernel ever waits on another's; on a multi-GPU box NBT_DIST_BACKEND may be unset
(NCCL)."""
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.gpu
def test_two_ranks_gloo_on_the_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    env = dict(os.environ)
    if torch.cuda.device_count() < 2:
        env["NBT_DIST_BACKEND"] = "gloo"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tools", "multirank_check.py")]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "MULTIRANK OK 2" in r.stdout
