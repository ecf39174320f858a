"""Trajectory files and diagnostics built on device:
ps_traj_pack writes exactly the bytes the host writer produces for the same
run, the reference-written golden file of the same run matches our device
run within the fp64 parity bound, and ps_traj_diff's compare equals the
host compare_trajectories to rounding."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2505_14741_b200 import engines as E, predictor as P  # noqa: E402
from paper_2505_14741_b200 import schedule as S, trajectory_io as TIO  # noqa: E402
from paper_2505_14741_b200.dit import DiTWeights  # noqa: E402
from paper_2505_14741_b200.spec import SPECS  # noqa: E402

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _tiny_w():
    return P.init_weights(P.TrainConfig(hidden=(8,), embed_dim=4, seed=7, activation="silu",
                                        iterations=0))


def test_device_pack_equals_host_writer_and_reference_file(tmp_path):
    cfg = E.RunConfig(steps=12, warmup=4, strategy="parastep", degree=3, seed=5, data_dim=2)
    s = E.DeviceSampler(_tiny_w(), S.make_default_schedule(12), cfg, record=True)
    s.run(cfg.seed)
    host = TIO.dump_trajectory_binary(s.trajectory())
    dev = TIO.pack_device(s)
    assert dev == host
    s.save_trajectory_binary(tmp_path / "d.pstj")
    ours = TIO.load_trajectory_binary(tmp_path / "d.pstj")
    ref = TIO.load_trajectory_binary(os.path.join(G, "traj_ps3.pstj"))  # written by the reference
    assert [r.t for r in ours.records] == [r.t for r in ref.records]
    assert [r.fresh for r in ours.records] == [r.fresh for r in ref.records]
    rep = E.compare_trajectories(ref, ours)
    assert rep.final_rel_mae < 1e-10
    assert max(max(r.rel_mae_x, r.rel_mae_eps) for r in rep.rows) < 1e-10


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_device_compare_matches_host(precision):
    spec = SPECS["dit_tiny"]
    w = DiTWeights(spec, seed=3, precision=precision, max_batch=4)
    sch = S.make_default_schedule(16, "zero")
    a = E.DeviceSampler(w, sch, E.RunConfig(steps=16, strategy="sequential", seed=2,
                                            data_dim=spec.data_dim), record=True)
    b = E.DeviceSampler(w, sch, E.RunConfig(steps=16, warmup=2, strategy="parastep", degree=4,
                                            seed=2, data_dim=spec.data_dim), record=True)
    a.run(2)
    b.run(2)
    dev = E.compare_trajectories_device(a, b)
    host = E.compare_trajectories(a.trajectory(), b.trajectory())
    assert [r.t for r in dev.rows] == [r.t for r in host.rows]
    for rd, rh in zip(dev.rows, host.rows):
        for f in ("rel_mae_x", "rel_mae_eps", "mse_x", "mse_eps"):
            assert np.isclose(getattr(rd, f), getattr(rh, f), rtol=1e-12, atol=1e-300), f
    for side in ("adjacent_a", "adjacent_b"):
        ad, ah = getattr(dev, side), getattr(host, side)
        assert len(ad) == len(ah) == 15
        assert [r.t for r in ad] == [r.t for r in ah]
        for rd, rh in zip(ad, ah):
            assert np.isclose(rd.rel_mae_x, rh.rel_mae_x, rtol=1e-12)
            assert np.isclose(rd.rel_mae_eps, rh.rel_mae_eps, rtol=1e-12)
    assert np.isclose(dev.final_rel_mae, host.final_rel_mae, rtol=1e-12)
    assert np.isclose(dev.final_mse, host.final_mse, rtol=1e-12)
    assert dev.final_rel_mae > 0.0  # ParaStep reuse differs from sequential
    assert dev.to_csv() .splitlines()[0] == "step,rel_mae_x,rel_mae_eps,mse_x,mse_eps"
