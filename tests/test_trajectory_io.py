"""Trajectory file formats: the drop-in reads the files the
reference writes (tests/golden/traj_ps3.*, made by the reference's own
trajectory_io via tests/golden/make_traj_golden.py) and writes them back
byte for byte; malformed files raise TrajectoryFormatError like the
reference (trajectory_io.py:57-131)."""

import os

import numpy as np
import pytest

from paper_2505_14741_b200 import trajectory_io as TIO
from paper_2505_14741_b200.errors import TrajectoryFormatError

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _gold(ext):
    with open(os.path.join(G, f"traj_ps3.{ext}"), "rb") as fh:
        return fh.read()


def test_text_roundtrip_byte_exact():
    raw = _gold("txt").decode()
    tr = TIO.parse_trajectory_text(raw)
    assert len(tr.records) == 12 and [r.t for r in tr.records] == list(range(12, 0, -1))
    assert TIO.dump_trajectory_text(tr) == raw


def test_binary_roundtrip_byte_exact():
    raw = _gold("pstj")
    tr = TIO.parse_trajectory_binary(raw)
    assert TIO.dump_trajectory_binary(tr) == raw
    # the two reference files hold the same trajectory, bit for bit
    tt = TIO.parse_trajectory_text(_gold("txt").decode())
    assert tt.bitwise_equal(tr)
    assert [r.fresh for r in tr.records] == [r.fresh for r in tt.records]


def test_save_load_files(tmp_path):
    tr = TIO.parse_trajectory_binary(_gold("pstj"))
    TIO.save_trajectory_binary(tr, tmp_path / "a.pstj")
    TIO.save_trajectory_text(tr, tmp_path / "a.txt")
    assert TIO.load_trajectory_binary(tmp_path / "a.pstj").bitwise_equal(tr)
    assert TIO.load_trajectory_text(tmp_path / "a.txt").bitwise_equal(tr)


@pytest.mark.parametrize("mutate", [
    lambda b: b"XXXX" + b[4:],                       # bad magic
    lambda b: b[:10],                                # truncated header
    lambda b: b[:4] + bytes([2]) + b[5:],            # unsupported version
    lambda b: b[:-3],                                # final sample cut short
    lambda b: b[:13 + 5 + 8],                        # truncated record
])
def test_binary_malformed(mutate):
    with pytest.raises(TrajectoryFormatError):
        TIO.parse_trajectory_binary(mutate(_gold("pstj")))


@pytest.mark.parametrize("mutate", [
    lambda s: "parastep-trajectory 2" + s[s.index("\n"):],   # wrong header
    lambda s: s.replace("data_dim=2", "dim=2", 1),          # malformed size line
    lambda s: "\n".join(s.splitlines()[:-2]) + "\n",         # missing lines
    lambda s: s.replace(" 1 ", " 7 ", 1),                    # bad fresh flag
    lambda s: s.replace("x0 ", "xx ", 1),                    # missing final sample
])
def test_text_malformed(mutate):
    with pytest.raises(TrajectoryFormatError):
        TIO.parse_trajectory_text(mutate(_gold("txt").decode()))


def test_payload_is_float64_le():
    tr = TIO.parse_trajectory_binary(_gold("pstj"))
    x = tr.records[0].x
    assert x.dtype == np.float64 and x.shape == (2,)
