"""generate_threshold_schedule (reference engines.py:367-401) pinned to the
reference's FROZEN_TAU01_SCHEDULE (pkg/tests/test_engines.py:43-46, :363-367):
on CPU the host logic runs on the reference's own trajectory (fixture made by
tests/golden/make_threshold_golden.py); on the GPU the same trained weights
drive our device sampler and must reproduce the same schedule."""

import os

import numpy as np
import pytest

from paper_2505_14741_b200 import engines as E
from paper_2505_14741_b200.errors import ConfigError

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FROZEN_TAU01_SCHEDULE = [
    1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 2, 1, 1, 2, 1, 1,
    1, 1, 1, 1, 1, 1, 2, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 2, 1, 1, 1, 1,
]


def _fixture():
    return np.load(os.path.join(G, "threshold_tau01.npz"))


def _ref_traj(z):
    recs = [E.StepRecord(int(t), x, e, True) for t, x, e in zip(z["ts"], z["xs"], z["eps"])]
    return E.Trajectory(recs, z["x0"])


def test_fixture_is_the_frozen_schedule():
    assert _fixture()["schedule_tau01_len4"].tolist() == FROZEN_TAU01_SCHEDULE


def test_host_schedule_on_reference_trajectory():
    ref = _ref_traj(_fixture())
    assert E.generate_threshold_schedule(ref, 0.1, 4) == FROZEN_TAU01_SCHEDULE
    assert E.generate_threshold_schedule(ref, 0.0, 4) == [1] * 50
    lengths = E.generate_threshold_schedule(ref, 0.5, 3, warmup=5)
    assert sum(lengths) == 45 and max(lengths) <= 3
    E.RunConfig(steps=50, warmup=5, strategy="dynamic", schedule_override=lengths,
                data_dim=2).validate()


def test_schedule_errors():
    ref = _ref_traj(_fixture())
    with pytest.raises(ConfigError):
        E.generate_threshold_schedule(ref, -0.1, 4)
    with pytest.raises(ConfigError):
        E.generate_threshold_schedule(ref, 0.1, 0)
    with pytest.raises(ConfigError):
        E.generate_threshold_schedule(ref, 0.1, 4, warmup=51)


@pytest.mark.gpu
def test_device_run_reproduces_frozen_schedule():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2505_14741_b200 import predictor as P, schedule as S

    z = _fixture()
    layers = [P.Layer(z[f"w{i}"], z[f"b{i}"]) for i in range(int(z["n_layers"]))]
    w = P.PredictorWeights(layers, str(z["activation"]))
    sch = S.make_default_schedule(50)
    ours = E.run_strategy(w, sch, E.RunConfig(steps=50, seed=42, data_dim=2))
    rep = E.compare_trajectories(_ref_traj(z), ours)
    assert rep.final_rel_mae < 1e-10
    assert max(r.rel_mae_eps for r in rep.rows) < 1e-10
    lengths = E.generate_threshold_schedule(ours, 0.1, 4)
    assert lengths == FROZEN_TAU01_SCHEDULE
    dyn = E.run_strategy(w, sch, E.RunConfig(steps=50, warmup=4, strategy="dynamic",
                                             schedule_override=E.generate_threshold_schedule(
                                                 ours, 0.1, 4, warmup=4),
                                             seed=42, data_dim=2))
    assert np.isfinite(dyn.x0).all() and dyn.steps == 50
