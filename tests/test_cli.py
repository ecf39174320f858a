"""Operator CLI: argument handling and exit codes on CPU
(configuration errors exit 2 before any GPU work, like cli.py:727-736);
the generate/compare runs themselves are GPU tests."""

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
