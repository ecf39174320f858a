"""bench.py's reporting arithmetic and fixture wiring (CPU): the call-count
and Amdahl bounds of the N > 1 line against the reference's own commodel
(pkg/src/parastep/commodel.py:51-68, from baseline/_ref when installed),
and the reference-sampler fixtures each config's rel-MAE falls back to."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _commodel():
    kind, _, _, _, commodel = bench.reference_module()
    if kind != "reference":
        pytest.skip("baseline/_ref (the reference package) not installed")
    return commodel


@pytest.mark.parametrize("T", [12, 50, 200])
@pytest.mark.parametrize("warmup", [0, 1, 5, 13])
@pytest.mark.parametrize("p", [1, 2, 3, 4, 8])
def test_call_count_matches_reference_commodel(T, warmup, p):
    if warmup > T:
        pytest.skip("warm-up longer than the run")
    cm = _commodel()
    assert bench.call_count(T, warmup, p) == cm.call_count_per_device(T, warmup, p)


@pytest.mark.parametrize("T,warmup,p", [(50, 5, 2), (50, 5, 8), (200, 1, 8), (50, 13, 4)])
def test_amdahl_bound_matches_reference(T, warmup, p):
    cm = _commodel()
    m = warmup / T
    ours = 1.0 / (m + (1.0 - m) / p)  # the expression multi_gpu_report uses
    assert abs(ours - cm.amdahl_speedup(m, p)) < 1e-15


def test_paper_audio_regime_bound():
    """configs[4] at d = 8, T = 200, warm-up 1: 1 + ceil(199 / 8) = 26 calls
    (the 7.69x call-count bound behind the paper's 6.56x)."""
    assert bench.call_count(200, 1, 8) == 26
    assert abs(200 / 26 - 7.6923) < 1e-4


@pytest.mark.parametrize("config", sorted(bench.FIXTURES))
def test_fixture_files_present(config):
    path = os.path.join(ROOT, "tests", "golden", bench.FIXTURES[config])
    g = np.load(path)
    if "eps" in g.files:  # per-forward fixture (configs[3])
        assert {"t", "T", "seed"} <= set(g.files)
        assert g["eps"].shape == (13 * 60 * 90 * 16,)
    else:
        assert "seq_x0" in g.files and "seq_t" in g.files
        T = bench.CONFIGS[config]["T"]
        assert g["seq_t"].tolist() == list(range(T, 0, -1))
