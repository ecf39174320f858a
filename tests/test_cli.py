"""Operator CLI: argument handling and exit codes on CPU
(configuration errors exit 2 before any GPU work, like cli.py:727-736);
the generate/compare runs themselves are GPU tests."""

import os

import pytest

from paper_2505_14741_b200 import cli


def test_help_exits_zero(capsys):
    assert cli.main(["--help"]) == 0
    assert "generate" in capsys.readouterr().out


def test_bad_choice_is_usage_error():
    assert cli.main(["generate", "--strategy", "nope"]) == 2


@pytest.mark.parametrize("argv", [
    ["generate", "--samples", "0"],
    ["generate", "--warmup", "2", "--warmup-ratio", "0.1"],
    ["compare"],
    ["compare", "--strategies", "bogus:2"],
    ["compare", "--strategies", "parastep:0"],
    ["compare", "--strategies", "parastep:2", "--seeds", "0"],
])
def test_config_errors_exit_2(argv, capsys):
    assert cli.main(argv) == 2
    assert "error:" in capsys.readouterr().err


def test_bench_refuses_more_gpus_than_present():
    """bench.py --gpus N outside torchrun spawns N ranks itself, and fails
    loudly (exit 2) instead of measuring fewer GPUs than asked."""
    import subprocess
    import sys

    import torch

    if torch.cuda.is_available():
        return
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2"],
                         capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 2
    assert "needs 2 CUDA devices" in out.stderr
