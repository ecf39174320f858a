"""GPU parity of the sampler path (RNG, fused scheduler, reference MLP,
engines) against the reference-generated golden fixtures and the oracle.

Tolerances: integer/uniform work and the scheduler step given identical
inputs are bit-exact; normals are fp64 transcendental results (device
libm vs numpy: <= 4 ulp); trajectories that consume device normals / device
GEMV sums are compared at 1e-10 relative (fp64 path).
"""

import numpy as np
import pytest

from oracle import core, engines as oeng

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2505_14741_b200 import _lib, engines as E, numerics as N, predictor as P  # noqa: E402
from paper_2505_14741_b200 import schedule as S  # noqa: E402

U64 = 0xFFFFFFFFFFFFFFFF


def _ulps(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    ia = a.view(np.int64)
    ib = b.view(np.int64)
    ia = np.where(ia < 0, np.int64(-(2**63)) - ia, ia)
    ib = np.where(ib < 0, np.int64(-(2**63)) - ib, ib)
    return np.abs(ia - ib)


def test_uniforms_bitwise(gold_rng):
    for k in range(int(gold_rng["ncases"])):
        seed, stream, n, ctr = (int(v) for v in gold_rng[f"case_{k}"])
        got = N.RngStream(seed, stream, ctr).uniforms(n)
        assert np.array_equal(got, gold_rng[f"uniform_{k}"]), k


def test_normals_within_ulps(gold_rng):
    for k in range(int(gold_rng["ncases"])):
        seed, stream, n, ctr = (int(v) for v in gold_rng[f"case_{k}"])
        got = N.draw_normal(seed, stream, n, ctr)
        assert _ulps(got, gold_rng[f"normal_{k}"]).max() <= 4, k


def test_frozen_step7():
    got = N.draw_normal(42, N.stream_id(N.PURPOSE_STEP, 7), 4)
    ref = [1.674703292428058, -1.2288609827611587, 0.12366643923390692, 0.487662335909011]
    assert _ulps(got, ref).max() <= 4


def test_ddpm_step_bitwise(gold_sched):
    for T, mode in ((12, "posterior"), (12, "zero"), (50, "posterior")):
        sch = S.make_default_schedule(T, mode)
        for t in (T, T // 2, 1):
            x, e, z = gold_sched[f"step_{T}_{mode}_{t}_in"]
            got = S.ddpm_step(x, t, e, sch, z)
            assert np.array_equal(got, gold_sched[f"step_{T}_{mode}_{t}_out"]), (T, mode, t)


def test_schedule_tables_bitwise(gold_sched):
    for T in (2, 4, 12, 50, 200):
        for mode in ("posterior", "zero"):
            s = S.make_default_schedule(T, mode)
            for f in ("beta", "alpha", "alpha_bar", "sigma"):
                assert np.array_equal(getattr(s, f), gold_sched[f"{T}_{mode}_{f}"])


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("n", [1, 2, 7, 4096, 4099])
def test_cycle_kernel_matches_oracle(dtype, n):
    """Fused apply (3 steps) + roll (lanes 1..3) vs the oracle step chain."""
    lib = _lib.load(require_gpu=True)
    tdt = torch.float64 if dtype == "f64" else torch.float32
    code = _lib.PS_F64 if dtype == "f64" else _lib.PS_F32
    T, seed = 20, 77
    sch = core.Sched(T)
    dsch = S.make_default_schedule(T)
    rng = np.random.default_rng(n)
    x = rng.standard_normal(n)
    eps = rng.standard_normal((3, n))
    caches = rng.standard_normal((4, n))
    if dtype == "f32":
        x, eps, caches = (v.astype(np.float32).astype(np.float64) for v in (x, eps, caches))
    apply_ts, roll_ts = [9, 8, 7], [6, 5, 4]
    xd = torch.as_tensor(x, dtype=tdt, device="cuda")
    ed = torch.as_tensor(eps, dtype=tdt, device="cuda")
    cd = torch.as_tensor(caches, dtype=tdt, device="cuda")
    lanes = torch.zeros((4, n), dtype=tdt, device="cuda")
    rec = torch.zeros((3, n), dtype=tdt, device="cuda")
    sd = torch.tensor([seed], dtype=torch.int64, device="cuda")
    es = ed.element_size()
    rc = lib.ps_sched_cycle(
        _lib.ptr(xd), _lib.ptr(xd), n, code, _lib.ptr(sd), 3,
        _lib.step_array([S.step_coeffs(dsch, t) for t in apply_ts]),
        _lib.ptr_array([_lib.ptr(ed) + k * n * es for k in range(3)]),
        _lib.ptr_array([_lib.ptr(rec) + k * n * es for k in range(3)]),
        1, 4, _lib.step_array([S.step_coeffs(dsch, t) for t in roll_ts]),
        _lib.ptr_array([_lib.ptr(cd) + j * n * es for j in range(4)]),
        _lib.ptr_array([_lib.ptr(lanes) + j * n * es for j in range(4)]), _lib.stream_ptr())
    _lib.check(rc, "cycle")
    torch.cuda.synchronize()
    # oracle
    xr = x.copy()
    recs = []
    for k, t in enumerate(apply_ts):
        recs.append(xr)
        # the chain stays in fp64 registers inside one launch (stores round)
        xr = core.ddpm_step(xr, t, eps[k], sch, oeng.z_step(seed, t, n))
    tol = 1e-13 if dtype == "f64" else 1e-6
    got = xd.double().cpu().numpy()
    assert np.allclose(got, xr, rtol=tol, atol=tol * np.abs(xr).max())
    assert np.allclose(rec.double().cpu().numpy(), np.stack(recs), rtol=tol, atol=tol * 10)
    for j in range(1, 4):
        xj = xr.copy()
        for k in range(j):
            xj = core.ddpm_step(xj, roll_ts[k], caches[j], sch, oeng.z_step(seed, roll_ts[k], n))
        lj = lanes[j].double().cpu().numpy()
        assert np.allclose(lj, xj, rtol=tol * 10, atol=tol * 10 * np.abs(xj).max()), j


def test_init_weights_bitwise(gold_mlp_small):
    w = P.init_weights(P.TrainConfig(hidden=(8,), embed_dim=4, seed=7, iterations=0))
    for i, layer in enumerate(w.layers):
        assert np.array_equal(layer.w, gold_mlp_small[f"w{i}"])


def test_mlp_forward_vs_oracle_and_batch_bitwise():
    w = P.init_weights(P.TrainConfig(data_dim=4096, hidden=(64, 64), embed_dim=16, seed=7))
    ref = core.MLP([l.w for l in w.layers], [l.b for l in w.layers])
    rng = np.random.default_rng(0)
    xs = [rng.standard_normal(4096) * 3 for _ in range(5)]
    ts = [50, 31, 7, 1, 0]
    outs = P.forward_batch(w, xs, ts, 50)
    for x, t, o in zip(xs, ts, outs):
        r = ref(x, t, 50)
        assert np.allclose(o, r, rtol=1e-12, atol=1e-12 * np.abs(r).max())
        assert np.array_equal(o, P.forward(w, x, t, 50))  # batch == single, bitwise


def _tiny(g):
    ws = [g["w0"], g["w1"]]
    return P.PredictorWeights([P.Layer(w, np.zeros(w.shape[1])) for w in ws], "silu")


def _close_traj(tr, g, prefix, rtol=1e-10):
    assert [r.t for r in tr.records] == g[f"{prefix}_t"].tolist()
    assert [r.fresh for r in tr.records] == g[f"{prefix}_fresh"].tolist()
    x0 = g[f"{prefix}_x0"]
    assert core.rel_mae(x0, tr.x0) <= rtol, prefix
    if f"{prefix}_x" in g:
        for k, r in enumerate(tr.records):
            gx, ge = g[f"{prefix}_x"][k], g[f"{prefix}_eps"][k]
            assert np.allclose(r.x, gx, rtol=rtol, atol=rtol * (np.abs(gx).max() + 1))
            assert np.allclose(r.eps, ge, rtol=rtol, atol=rtol * (np.abs(ge).max() + 1))


@pytest.mark.parametrize("mode", ["posterior", "zero"])
def test_engines_tiny_mlp_vs_reference(gold_mlp_small, mode):
    g = gold_mlp_small
    w = _tiny(g)
    sch = S.make_default_schedule(12, mode)
    runs = [
        ("seq", dict(strategy="sequential")),
        ("dr3", dict(strategy="direct_reuse", degree=3, warmup=2)),
        ("ps2", dict(strategy="parastep", degree=2, warmup=3)),
        ("ps3", dict(strategy="parastep", degree=3, warmup=4)),
        ("ps4", dict(strategy="parastep", degree=4, warmup=2)),
        ("bs3", dict(strategy="batchstep", degree=3, warmup=4)),
        ("dyn", dict(strategy="dynamic", warmup=2, schedule_override=[4, 1, 3, 2])),
    ]
    for tag, kw in runs:
        cfg = E.RunConfig(steps=12, seed=5, data_dim=2, **kw)
        _close_traj(E.run_strategy(w, sch, cfg), g, f"{mode}_{tag}")


def test_parastep_forms_bitwise_on_device(gold_mlp_small):
    """lanes (run_strategy) == batchstep == literal Algorithm 1, bit-for-bit on GPU
    (the reference's own equivalence tests, tests/test_engines.py:294-325)."""
    w = _tiny(gold_mlp_small)
    sch = S.make_default_schedule(12)
    for d in (2, 3, 4):
        kw = dict(steps=12, warmup=3, degree=d, seed=8, data_dim=2)
        lanes = E.run_strategy(w, sch, E.RunConfig(strategy="parastep", **kw))
        batch = E.run_strategy(w, sch, E.RunConfig(strategy="batchstep", **kw))
        emu, _ = E.denoise_parastep_emulated(w, sch, E.RunConfig(strategy="parastep", **kw))
        assert lanes.bitwise_equal(batch)
        assert lanes.bitwise_equal(emu)
    dyn = E.run_strategy(w, sch, E.RunConfig(steps=12, warmup=3, strategy="dynamic",
                                             schedule_override=[3, 3, 3], seed=2, data_dim=2))
    para = E.run_strategy(w, sch, E.RunConfig(steps=12, warmup=3, strategy="parastep", degree=3,
                                              seed=2, data_dim=2))
    assert dyn.bitwise_equal(para)


def test_degenerate_collapse_bitwise():
    w = _tiny_weights()
    for mode in ("posterior", "zero"):
        sch = S.make_default_schedule(12, mode)
        ref = E.run_strategy(w, sch, E.RunConfig(steps=12, seed=1, data_dim=2))
        for cfg in (E.RunConfig(steps=12, strategy="parastep", degree=1, warmup=2, seed=1,
                                data_dim=2),
                    E.RunConfig(steps=12, strategy="batchstep", degree=1, warmup=2, seed=1,
                                data_dim=2),
                    E.RunConfig(steps=12, strategy="direct_reuse", degree=1, seed=1, data_dim=2),
                    E.RunConfig(steps=12, strategy="dynamic", schedule_override=[1] * 12,
                                seed=1, data_dim=2)):
            assert E.run_strategy(w, sch, cfg).bitwise_equal(ref), cfg.strategy


def _tiny_weights():
    return P.init_weights(P.TrainConfig(hidden=(8,), embed_dim=4, seed=7, iterations=0))


def test_histories_match_reference(gold_mlp_small):
    g = gold_mlp_small
    _, workers = E.denoise_parastep_emulated(
        _tiny(g), S.make_default_schedule(12),
        E.RunConfig(steps=12, warmup=4, strategy="parastep", degree=3, seed=6, data_dim=2))
    for ws in workers:
        r = ws.rank
        assert [h.source for h in ws.history] == g[f"hist{r}_src"].tolist()
        xb = np.stack([h.x_before for h in ws.history])
        xa = np.stack([h.x_after for h in ws.history])
        assert np.allclose(xb, g[f"hist{r}_xb"], rtol=1e-10, atol=1e-10)
        assert np.allclose(xa, g[f"hist{r}_xa"], rtol=1e-10, atol=1e-10)
    # truncated final cycle leaves ranks desynchronised (tests/test_engines.py:279-289)
    assert not np.array_equal(workers[0].history[-1].x_after, workers[2].history[-1].x_after)


def test_identity_net_hand_unrolled(gold_mlp_small):
    mat = np.zeros((6, 2))
    mat[0, 0] = mat[1, 1] = 1.0
    ident = P.PredictorWeights([P.Layer(mat, np.zeros(2))], "silu")
    cfg = E.RunConfig(steps=4, warmup=1, strategy="parastep", degree=3, seed=21, data_dim=2)
    _close_traj(E.run_strategy(ident, S.make_default_schedule(4), cfg), gold_mlp_small,
                "ident_ps3")


@pytest.mark.parametrize("mode", ["posterior", "zero"])
def test_c1ref_mlp_4096_vs_reference(gold_c1ref, mode):
    g = gold_c1ref
    w = P.init_weights(P.TrainConfig(data_dim=4096, hidden=(64, 64), embed_dim=16, seed=7))
    sch = S.make_default_schedule(50, mode)
    seq = E.run_strategy(w, sch, E.RunConfig(steps=50, seed=0, data_dim=4096))
    assert core.rel_mae(g[f"{mode}_seq_x0"], seq.x0) < 1e-10
    for d in (2, 4, 8):
        cfg = E.RunConfig(steps=50, warmup=5, strategy="parastep", degree=d, seed=0,
                          data_dim=4096)
        tr = E.run_strategy(w, sch, cfg)
        assert core.rel_mae(g[f"{mode}_ps{d}_x0"], tr.x0) < 1e-10, d
        # the algorithmic deviation from sequential is the reference's too
        assert abs(N.rel_mae(seq.x0, tr.x0) - float(g[f"{mode}_ps{d}_relmae_vs_seq"])) < 1e-8
    tr = E.run_strategy(w, sch, E.RunConfig(steps=50, warmup=5, strategy="parastep", degree=2,
                                            seed=0, data_dim=4096))
    for k in (0, 5, 6, 27, 49):
        assert core.rel_mae(g[f"{mode}_ps2_rec{k}_x"], tr.records[k].x) < 1e-10
        assert core.rel_mae(g[f"{mode}_ps2_rec{k}_eps"], tr.records[k].eps) < 1e-10


def test_graph_replay_equals_eager():
    w = P.init_weights(P.TrainConfig(data_dim=4096, hidden=(64, 64), embed_dim=16, seed=7))
    sch = S.make_default_schedule(50)
    cfg = E.RunConfig(steps=50, warmup=5, strategy="batchstep", degree=4, seed=3, data_dim=4096)
    s = E.DeviceSampler(w, sch, cfg)
    s.run(3)
    eager = s.trajectory()
    for seed in (3, 4, 3):
        s.run(seed, graph=True)
        tr = s.trajectory()
        if seed == 3:
            assert tr.bitwise_equal(eager)
        else:
            assert not np.array_equal(tr.x0, eager.x0)


def test_errors_match_reference_types():
    from paper_2505_14741_b200.errors import ConfigError, DimensionError, ParameterError

    w = _tiny_weights()
    with pytest.raises(DimensionError):
        P.forward(w, np.zeros(3), 1, 10)
    with pytest.raises(ParameterError):
        P.forward(w, np.zeros(2), 11, 10)
    with pytest.raises(ConfigError):
        E.run_strategy(w, S.make_default_schedule(10), E.RunConfig(steps=12, data_dim=2))
    with pytest.raises(ConfigError):
        E.run_strategy(w, S.make_default_schedule(12),
                       E.RunConfig(steps=12, strategy="parastep", degree=2, warmup=0,
                                   data_dim=2))
