"""bench.py's N > 1 path (BASELINE.json metric at degree d): two ranks
through torch.distributed.run. On a one-GPU box both ranks share cuda:0
(PS_BENCH_SHARED_GPU=1: gloo bootstrap, CUDA-IPC peer exchange), which runs
the rank loop, the device-clock phase split, the measured exchange ledger,
the sequential comparison and the call-count bound for real; with two or
more GPUs the same command runs one rank per GPU over NCCL."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_line():
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    if torch.cuda.device_count() < 2:
        env["PS_BENCH_SHARED_GPU"] = "1"
    out = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
         "--master-addr", "127.0.0.1", "--master-port", "29731", os.path.join(ROOT, "bench.py"),
         "--gpus", "2", "--steps", "2", "--warmup", "1", "--batchstep"],
        capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1]
    d = json.loads(line)
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert len(d["per_rank"]) == 2
    assert all(r["forward_ms"] > 0 and r["apply_ms"] > 0 for r in d["per_rank"])
    assert d["exchange_ledger"]["verified"] and d["exchange_ledger"]["rounds"] > 0
    assert d["sequential_ms"] > 0 and d["speedup_vs_sequential"] > 0
    # T = 50, warm-up 5, d = 2: 5 + ceil(45 / 2) = 28 calls -> bound 50 / 28
    assert d["call_count_per_device"] == 28
    assert abs(d["speedup_bound_callcount"] - 50 / 28) < 1e-12
    # degree-2 parity vs the reference's own ParaStep emulation, run live on rank 0
    assert d["rel_mae_vs_reference"] is not None and d["rel_mae_vs_reference"] < 1e-4
