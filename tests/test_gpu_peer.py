"""Peer-memory eps exchange (CUDA IPC + release/acquire flags, the fused
alternative to the per-round NCCL all-gather). On a one-GPU box the ranks
share cuda:0: the IPC mapping, flag protocol, double buffering and graph
replay run for real; with more GPUs the same script runs one rank per GPU
over NVLink. Results must equal the single-process lane emulation bitwise."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("world,spec", [(1, "dit_tiny"), (2, "dit_tiny"), (3, "dit_tiny_video")])
def test_peer_exchange_bitwise(world, spec):
    ngpu = torch.cuda.device_count()
    env = dict(os.environ, PEER_CHECK_SPEC=spec, PEER_SAME_GPU="1" if world > ngpu else "0")
    out = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
         f"--nproc-per-node={world}", "--master-addr", "127.0.0.1",
         "--master-port", str(29600 + 7 * world), os.path.join(ROOT, "tools", "peer_check.py")],
        capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert "PEER_CHECK OK" in out.stdout
