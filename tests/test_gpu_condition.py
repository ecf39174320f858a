"""The per-run conditioning table (ps_dit_condition: every adaLN vector of
the run's steps, batched 16 steps per GEMV) must reproduce the per-forward
conditioning bit for bit: eps of a forward reading table rows == eps of the
same forward computing its conditioning itself, for single and batched
lanes, fp32 and bf16; and a sampler run (which fills the table) equals the
same run after clearing it."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2505_14741_b200 import engines as E, predictor as P  # noqa: E402
from paper_2505_14741_b200 import schedule as S  # noqa: E402
from paper_2505_14741_b200.dit import DiTWeights  # noqa: E402
from paper_2505_14741_b200.spec import SPECS  # noqa: E402


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_table_equals_per_forward(precision):
    spec = SPECS["dit_tiny"]
    w = DiTWeights(spec, seed=9, precision=precision, max_batch=4)
    rng = np.random.default_rng(3)
    xs = [rng.standard_normal(spec.data_dim) for _ in range(3)]
    ts = [20, 7, 1]
    w.clear_conditioning()
    a = P.forward_batch(w, xs, ts, 20)
    w.reserve_conditioning(20)
    w.prepare_conditioning(20)
    torch.cuda.synchronize()
    b = P.forward_batch(w, xs, ts, 20)
    c = [P.forward(w, x, t, 20) for x, t in zip(xs, ts)]
    for u, v, z in zip(a, b, c):
        assert np.array_equal(u, v) and np.array_equal(u, z)


def test_sampler_with_table_equals_without():
    spec = SPECS["dit_tiny"]
    w = DiTWeights(spec, seed=2, max_batch=4)
    sch = S.make_default_schedule(16)
    cfg = E.RunConfig(steps=16, warmup=2, strategy="batchstep", degree=4, seed=5,
                      data_dim=spec.data_dim)
    s = E.DeviceSampler(w, sch, cfg)
    s.run(5, graph=True)
    with_table = s.trajectory()
    # the same run with per-forward conditioning (table cleared, no prepare)
    w.clear_conditioning()
    s2 = E.DeviceSampler(w, sch, cfg, condition_table=False)
    s2.run(5)
    assert with_table.bitwise_equal(s2.trajectory())
