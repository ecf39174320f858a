"""The NCCL ParaStep path on the GPUs present (one process per GPU via
torchrun). With one GPU this is degree 1 over a 1-rank NCCL communicator:
the all-gather, its CUDA-graph capture and the rank loop run for real and
must be bit-identical to the single-process sampler; with more GPUs it is
the full degree-d exchange."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("spec", ["dit_tiny", "dit_tiny_video"])
def test_nccl_rank_loop_bitwise(spec):
    n = torch.cuda.device_count()
    env = dict(os.environ, NCCL_CHECK_SPEC=spec)
    out = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
         "--master-addr", "127.0.0.1", "--master-port", str(29500 + hash(spec) % 1000),
         os.path.join(ROOT, "tools", "nccl_check.py")],
        capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert "NCCL_CHECK OK" in out.stdout
