"""Pin the CPU oracle to the reference: every fixture in tests/golden was
produced by the reference package itself (tests/golden/make_golden.py); the
oracle must reproduce each one bit-for-bit. CPU only.
"""

import numpy as np
import pytest

from oracle import core, engines
from oracle.dit import DiT
from paper_2505_14741_b200.spec import SPECS

FROZEN_STEP7 = [1.674703292428058, -1.2288609827611587, 0.12366643923390692, 0.487662335909011]


def test_frozen_step7_literal():
    # the reference's own regression anchor (tests/test_numerics.py:29-34)
    got = core.normals(42, core.make_stream(core.P_STEP, 7), 4)
    assert got.tolist() == FROZEN_STEP7


def test_rng_cases_bitwise(gold_rng):
    for k in range(int(gold_rng["ncases"])):
        seed, stream, n, ctr = (int(v) for v in gold_rng[f"case_{k}"])
        assert np.array_equal(core.normals(seed, stream, n, ctr), gold_rng[f"normal_{k}"])
        assert np.array_equal(core.uniforms(seed, stream, n, ctr), gold_rng[f"uniform_{k}"])


def test_rng_random_access():
    s = core.make_stream(core.P_STEP, 3)
    whole = core.normals(11, s, 64)
    assert np.array_equal(core.normals(11, s, 16, 48), whole[48:])
    assert np.array_equal(core.normals(11, s, 1, 17), whole[17:18])


@pytest.mark.parametrize("T", [2, 4, 12, 50, 200])
@pytest.mark.parametrize("mode", ["posterior", "zero"])
def test_schedule_tables_bitwise(gold_sched, T, mode):
    s = core.Sched(T, mode)
    for f in ("beta", "alpha", "alpha_bar", "sigma"):
        assert np.array_equal(getattr(s, f), gold_sched[f"{T}_{mode}_{f}"]), f


def test_ddpm_step_bitwise(gold_sched):
    for T, mode in ((12, "posterior"), (12, "zero"), (50, "posterior")):
        s = core.Sched(T, mode)
        for t in (T, T // 2, 1):
            x, e, z = gold_sched[f"step_{T}_{mode}_{t}_in"]
            assert np.array_equal(core.ddpm_step(x, t, e, s, z),
                                  gold_sched[f"step_{T}_{mode}_{t}_out"])


def test_posterior_mean_hand_value():
    # tests/test_schedule.py:128-132 analogue: x=1, eps=0 -> 1/sqrt(alpha_t)
    s = core.Sched(4)
    out = core.ddpm_step(np.array([1.0]), 1, np.array([0.0]), s, np.array([0.0]))
    assert out[0] == 1.0 / np.sqrt(s.alpha[0])


def test_rel_mae_hand_values():
    assert core.rel_mae(np.array([2.0, 2.0]), np.array([1.0, 3.0])) == 0.5
    assert core.rel_mae(np.array([1.0, 1.0]), np.array([2.0, 2.0])) == 1.0
    with pytest.raises(ZeroDivisionError):
        core.rel_mae(np.zeros(2), np.ones(2))


def _tiny_mlp(g):
    ws = [g["w0"], g["w1"]]
    return core.MLP(ws, [np.zeros(w.shape[1]) for w in ws])


def _check_traj(tr, g, prefix, records=True):
    assert list(tr["t"]) == g[f"{prefix}_t"].tolist()
    assert list(tr["fresh"]) == g[f"{prefix}_fresh"].tolist()
    assert np.array_equal(tr["x0"], g[f"{prefix}_x0"])
    if records:
        assert np.array_equal(np.stack(tr["x"]), g[f"{prefix}_x"])
        assert np.array_equal(np.stack(tr["eps"]), g[f"{prefix}_eps"])


def test_mlp_init_matches_reference(gold_mlp_small):
    m = core.MLP.init(2, hidden=(8,), embed_dim=4, seed=7)
    for i, w in enumerate(m.ws):
        assert np.array_equal(w, gold_mlp_small[f"w{i}"])


@pytest.mark.parametrize("mode", ["posterior", "zero"])
def test_engines_tiny_mlp_bitwise(gold_mlp_small, mode):
    g = gold_mlp_small
    pred = _tiny_mlp(g)
    s = core.Sched(12, mode)
    _check_traj(engines.sequential(pred, s, 2, 5), g, f"{mode}_seq")
    _check_traj(engines.direct_reuse(pred, s, 2, 5, warmup=2, stride=3), g, f"{mode}_dr3")
    for p, w in ((2, 3), (3, 4), (4, 2)):
        tr, _ = engines.parastep_algorithm1(pred, s, 2, 5, warmup=w, p=p)
        _check_traj(tr, g, f"{mode}_ps{p}")
    # cycle runner == parastep (tests/test_engines.py:294-303)
    _check_traj(engines.cycles(pred, s, 2, 5, warmup=4, degree=3), g, f"{mode}_bs3")
    _check_traj(engines.cycles(pred, s, 2, 5, warmup=2, degree=0, lengths=[4, 1, 3, 2]), g,
                f"{mode}_dyn")


def test_parastep_histories(gold_mlp_small):
    g = gold_mlp_small
    _, hist = engines.parastep_algorithm1(_tiny_mlp(g), core.Sched(12), 2, 6, warmup=4, p=3)
    for r in range(3):
        assert [h[3] for h in hist[r]] == g[f"hist{r}_src"].tolist()
        assert np.array_equal(np.stack([h[1] for h in hist[r]]), g[f"hist{r}_xb"])
        assert np.array_equal(np.stack([h[4] for h in hist[r]]), g[f"hist{r}_xa"])


def test_identity_net_hand_unrolled(gold_mlp_small):
    tr, _ = engines.parastep_algorithm1(core.IdentityNet(2), core.Sched(4), 2, 21, 1, 3)
    _check_traj(tr, gold_mlp_small, "ident_ps3")


def test_loopback_worker_equals_oracle(gold_mlp_small):
    # the reference's distributed (threaded) worker agrees with the restatement
    tr, _ = engines.parastep_algorithm1(_tiny_mlp(gold_mlp_small), core.Sched(12), 2, 9, 3, 3)
    _check_traj(tr, gold_mlp_small, "loopback_ps3")


@pytest.mark.parametrize("mode", ["posterior", "zero"])
def test_c1ref_mlp_4096_bitwise(gold_c1ref, mode):
    g = gold_c1ref
    pred = core.MLP.init(4096, hidden=(64, 64), embed_dim=16, seed=7)
    s = core.Sched(50, mode)
    seq = engines.sequential(pred, s, 4096, 0)
    assert np.array_equal(seq["x0"], g[f"{mode}_seq_x0"])
    for d in (2, 4):
        tr = engines.cycles(pred, s, 4096, 0, warmup=5, degree=d)
        assert np.array_equal(tr["x0"], g[f"{mode}_ps{d}_x0"])
        assert core.rel_mae(seq["x0"], tr["x0"]) == float(g[f"{mode}_ps{d}_relmae_vs_seq"])


def test_dit_oracle_through_reference_sampler(gold_dit):
    g = gold_dit
    for name, bias in (("dit_tiny", 0.05), ("dit_tiny_video", 0.0)):
        pred = DiT(SPECS[name], seed=11, bias_scale=bias)
        n = pred.data_dim
        e = pred(np.linspace(-2, 2, n), 7, 20)
        assert np.array_equal(e, g[f"{name}_eps_t7"])
        rec = name == "dit_tiny"
        for mode in ("posterior", "zero"):
            s = core.Sched(20, mode)
            _check_traj(engines.sequential(pred, s, n, 3), g, f"{name}_{mode}_seq", rec)
            tr, _ = engines.parastep_algorithm1(pred, s, n, 3, warmup=2, p=2)
            _check_traj(tr, g, f"{name}_{mode}_ps2", rec)
            tr = engines.cycles(pred, s, n, 3, warmup=2, degree=3)
            _check_traj(tr, g, f"{name}_{mode}_ps3", rec)
            tr = engines.cycles(pred, s, n, 3, warmup=3, degree=4)
            _check_traj(tr, g, f"{name}_{mode}_bs4", rec)
