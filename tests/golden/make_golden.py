"""Regenerate the golden fixtures by running the REFERENCE package itself.

Run in the build container only (needs /root/reference):

    python tests/golden/make_golden.py

It imports ``parastep`` from /root/reference/pkg/src, runs the reference's own
functions and writes small ``.npz`` fixtures next to this file. Nothing on the
GPU box reads /root/reference; the fixtures travel instead.

DiT-shaped predictors do not exist in the reference; for those fixtures the
oracle DiT (oracle/dit.py) is injected through the reference's import seam
(``parastep.engines.forward`` / ``forward_batch``, engines.py:40), so the
reference's OWN sampler loops produce the expected trajectories.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = os.environ.get("PARASTEP_REF_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import parastep.engines as E  # noqa: E402
from parastep.numerics import RngStream, draw_normal, rel_mae, stream_id  # noqa: E402
from parastep.predictor import Layer, PredictorWeights, TrainConfig, init_weights  # noqa: E402
from parastep.protocol.worker import run_loopback  # noqa: E402
from parastep.schedule import ddpm_step, make_default_schedule  # noqa: E402


def _save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def rng_fixture():
    out = {}
    cases = [  # (seed, purpose, index, n, counter)
        (42, 1, 7, 4, 0),  # FROZEN_STEP7 (tests/test_numerics.py:29-34)
        (0, 0, 0, 257, 0),
        (7, 1, 50, 64, 3),  # odd start counter
        (2**64 - 1, 3, 2**32 - 1, 33, 1001),
        (123456789, 1, 1, 4096, 0),
    ]
    for k, (seed, pur, idx, n, ctr) in enumerate(cases):
        s = stream_id(pur, idx)
        out[f"normal_{k}"] = draw_normal(seed, s, n, ctr)
        out[f"uniform_{k}"] = RngStream(seed, s, ctr).uniforms(n)
        out[f"case_{k}"] = np.array([seed, s, n, ctr], dtype=np.uint64)
    out["ncases"] = np.array(len(cases))
    _save("rng.npz", **out)


def sched_fixture():
    out = {}
    for T in (2, 4, 12, 50, 200):
        for mode in ("posterior", "zero"):
            s = make_default_schedule(T, mode)
            for f in ("beta", "alpha", "alpha_bar", "sigma"):
                out[f"{T}_{mode}_{f}"] = getattr(s, f)
    # ddpm_step KATs on random inputs (both modes, t == 1 special case)
    rng = np.random.default_rng(5)
    for T, mode in ((12, "posterior"), (12, "zero"), (50, "posterior")):
        s = make_default_schedule(T, mode)
        for t in (T, T // 2, 1):
            x, e, z = rng.standard_normal((3, 97))
            out[f"step_{T}_{mode}_{t}_in"] = np.stack([x, e, z])
            out[f"step_{T}_{mode}_{t}_out"] = ddpm_step(x, t, e, s, z)
    _save("sched.npz", **out)


def _traj_arrays(prefix, traj, out, records=True):
    out[f"{prefix}_x0"] = traj.x0
    out[f"{prefix}_t"] = np.array([r.t for r in traj.records])
    out[f"{prefix}_fresh"] = np.array([r.fresh for r in traj.records])
    if records:
        out[f"{prefix}_x"] = np.stack([r.x for r in traj.records])
        out[f"{prefix}_eps"] = np.stack([r.eps for r in traj.records])


def mlp_small_fixture():
    """The reference tests' tiny_w (tests/conftest.py:44-53) through every engine."""
    w = init_weights(TrainConfig(hidden=(8,), embed_dim=4, seed=7, activation="silu",
                                 iterations=0))
    out = {f"w{i}": l.w for i, l in enumerate(w.layers)}
    runs = [
        ("seq", dict(strategy="sequential")),
        ("dr3", dict(strategy="direct_reuse", degree=3, warmup=2)),
        ("ps2", dict(strategy="parastep", degree=2, warmup=3)),
        ("ps3", dict(strategy="parastep", degree=3, warmup=4)),
        ("ps4", dict(strategy="parastep", degree=4, warmup=2)),
        ("bs3", dict(strategy="batchstep", degree=3, warmup=4)),
        ("dyn", dict(strategy="dynamic", warmup=2, schedule_override=[4, 1, 3, 2])),
    ]
    for mode in ("posterior", "zero"):
        sched = make_default_schedule(12, mode)
        for tag, kw in runs:
            cfg = E.RunConfig(steps=12, seed=5, data_dim=2, **kw)
            _traj_arrays(f"{mode}_{tag}", E.run_strategy(w, sched, cfg), out)
    # per-rank histories of the p=3 emulation (rotation / resync / truncation)
    sched = make_default_schedule(12)
    cfg = E.RunConfig(steps=12, warmup=4, strategy="parastep", degree=3, seed=6, data_dim=2)
    _, workers = E.denoise_parastep_emulated(w, sched, cfg)
    for ws in workers:
        out[f"hist{ws.rank}_src"] = np.array([h.source for h in ws.history])
        out[f"hist{ws.rank}_xb"] = np.stack([h.x_before for h in ws.history])
        out[f"hist{ws.rank}_xa"] = np.stack([h.x_after for h in ws.history])
    # identity net hand-unrolled cycle (tests/test_engines.py:241-276)
    mat = np.zeros((6, 2))
    mat[0, 0] = mat[1, 1] = 1.0
    ident = PredictorWeights([Layer(mat, np.zeros(2))], "silu")
    cfg = E.RunConfig(steps=4, warmup=1, strategy="parastep", degree=3, seed=21, data_dim=2)
    _traj_arrays("ident_ps3", E.run_strategy(ident, make_default_schedule(4), cfg), out)
    # the distributed reference worker (threads over queues) == emulation
    cfg = E.RunConfig(steps=12, warmup=3, strategy="parastep", degree=3, seed=9, data_dim=2)
    _traj_arrays("loopback_ps3", run_loopback(w, make_default_schedule(12), cfg).trajectory, out)
    _save("mlp_small.npz", **out)


def mlp_c1ref_fixture():
    """C1-ref: the reference's own MLP at data_dim 4096 = 4x32x32."""
    w = init_weights(TrainConfig(data_dim=4096, hidden=(64, 64), embed_dim=16, seed=7,
                                 iterations=0))
    out = {}
    for mode in ("posterior", "zero"):
        sched = make_default_schedule(50, mode)
        seq = E.run_strategy(w, sched, E.RunConfig(steps=50, seed=0, data_dim=4096))
        _traj_arrays(f"{mode}_seq", seq, out, records=False)
        for d in (2, 4, 8):
            cfg = E.RunConfig(steps=50, warmup=5, strategy="parastep", degree=d, seed=0,
                              data_dim=4096)
            tr = E.run_strategy(w, sched, cfg)
            _traj_arrays(f"{mode}_ps{d}", tr, out, records=False)
            out[f"{mode}_ps{d}_relmae_vs_seq"] = np.array(rel_mae(seq.x0, tr.x0))
        # a few full records for the per-step check
        tr = E.run_strategy(w, sched, E.RunConfig(steps=50, warmup=5, strategy="parastep",
                                                  degree=2, seed=0, data_dim=4096))
        for k in (0, 5, 6, 27, 49):
            out[f"{mode}_ps2_rec{k}_x"] = tr.records[k].x
            out[f"{mode}_ps2_rec{k}_eps"] = tr.records[k].eps
    _save("mlp_c1ref.npz", **out)


class _Shim:
    """Duck-typed weights object: the reference sampler only reads .data_dim."""

    def __init__(self, pred):
        self.pred = pred
        self.data_dim = pred.data_dim
        self.ballast = 1


def dit_fixture():
    from oracle.dit import DiT
    from paper_2505_14741_b200.spec import SPECS

    def fwd(w, x, t, T):
        return w.pred(np.asarray(x, dtype=np.float64), t, T)

    def fwd_batch(w, xs, ts, T):
        return [fwd(w, x, t, T) for x, t in zip(xs, ts)]

    E.forward, E.forward_batch = fwd, fwd_batch  # the import seam (engines.py:40)
    out = {}
    for name, bias in (("dit_tiny", 0.05), ("dit_tiny_video", 0.0)):
        w = _Shim(DiT(SPECS[name], seed=11, bias_scale=bias))
        out[f"{name}_eps_t7"] = fwd(w, np.linspace(-2, 2, w.data_dim), 7, 20)
        for mode in ("posterior", "zero"):
            sched = make_default_schedule(20, mode)
            runs = [("seq", dict(strategy="sequential")),
                    ("ps2", dict(strategy="parastep", degree=2, warmup=2)),
                    ("ps3", dict(strategy="parastep", degree=3, warmup=2)),
                    ("bs4", dict(strategy="batchstep", degree=4, warmup=3))]
            for tag, kw in runs:
                cfg = E.RunConfig(steps=20, seed=3, data_dim=w.data_dim, **kw)
                _traj_arrays(f"{name}_{mode}_{tag}", E.run_strategy(w, sched, cfg), out,
                             records=(name == "dit_tiny"))
    _save("dit_small.npz", **out)


if __name__ == "__main__":
    rng_fixture()
    sched_fixture()
    mlp_small_fixture()
    mlp_c1ref_fixture()
    dit_fixture()
