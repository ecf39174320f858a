"""Golden fixtures at BASELINE.json's full-size configs, made by the REFERENCE
sampler itself (build container only; needs /root/reference):

    python tests/golden/make_golden_large.py [dit_xl2] [unet] [cogvideox]

* ``dit_xl2_traj.npz`` — configs[2]: DiT-XL/2-shaped predictor (seed 0),
  latent 4x32x32, 50 steps, sigma_mode "zero" (the reference's deterministic
  "DDIM" mode), seed 0: the reference's ``run_strategy`` (engines.py:352-364)
  at sequential and ParaStep degree 2/4/8 (warm-up 5), x0 of each + the
  step order / fresh flags.
* ``unet_traj.npz`` — configs[4]: AudioLDM2-large-shaped U-Net (seed 0), mel
  latent 8x256x16, 200 steps, zero mode, seed 0: sequential and ParaStep
  degree 8 (warm-up 1, the paper's AudioLDM2 setting).
* ``cogvideox_fwd.npz`` — configs[3]: one full-shape forward of the
  CogVideoX-2b-shaped predictor (seed 0, 30 layers, 226 text + 17,550 video
  tokens, expert adaLN, 3D RoPE) on the
  reference's x_T (``initial_state(0)``: normals of stream INIT<<32|0) at
  t = 37 of T = 50, eps stored as float32. A 50-step CPU trajectory at this
  shape is ~7 h, so parity for configs[3] is per forward.

DiT / U-Net arithmetic comes from the oracle predictors (numpy float64),
injected through the reference's import seam (engines.py:40) exactly as in
make_golden.py; the sampler loops, RNG, schedule and ParaStep bookkeeping are
the reference's own code.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = os.environ.get("PARASTEP_REF_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import parastep.engines as E  # noqa: E402
from parastep.numerics import rel_mae  # noqa: E402
from parastep.schedule import make_default_schedule  # noqa: E402


class _Shim:
    def __init__(self, pred):
        self.pred = pred
        self.data_dim = pred.data_dim
        self.ballast = 1


def _seam():
    def fwd(w, x, t, T):
        return w.pred(np.asarray(x, dtype=np.float64), t, T)

    E.forward = fwd
    E.forward_batch = lambda w, xs, ts, T: [fwd(w, x, t, T) for x, t in zip(xs, ts)]
    return fwd


def _save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)", flush=True)


def _trajectories(w, T, warmup, degrees, out):
    sched = make_default_schedule(T, "zero")
    for d in degrees:
        kw = dict(strategy="sequential") if d == 1 else dict(strategy="parastep", degree=d,
                                                              warmup=warmup)
        cfg = E.RunConfig(steps=T, seed=0, data_dim=w.data_dim, **kw)
        t0 = time.time()
        tr = E.run_strategy(w, sched, cfg)
        tag = "seq" if d == 1 else f"ps{d}"
        out[f"{tag}_x0"] = tr.x0
        out[f"{tag}_t"] = np.array([r.t for r in tr.records])
        out[f"{tag}_fresh"] = np.array([r.fresh for r in tr.records])
        out[f"{tag}_eps0"] = tr.records[0].eps
        print(f"  {tag}: {time.time() - t0:.0f} s", flush=True)
    for d in degrees[1:]:
        # the paper's quality metric: ParaStep x0 vs the sequential x0 (Eq. 7)
        out[f"ps{d}_vs_seq_rel_mae"] = np.array(rel_mae(out["seq_x0"], out[f"ps{d}_x0"]))


def dit_xl2():
    from oracle.dit import DiT
    from paper_2505_14741_b200.spec import SPECS

    _seam()
    w = _Shim(DiT(SPECS["dit_xl2"], seed=0))
    out = {}
    _trajectories(w, 50, 5, [1, 2, 4, 8], out)
    _save("dit_xl2_traj.npz", **out)


def unet():
    from oracle.unet import UNet
    from paper_2505_14741_b200.unet_spec import UNET_SPECS

    _seam()
    w = _Shim(UNet(UNET_SPECS["audioldm2_large"], seed=0))
    out = {}
    _trajectories(w, 200, 1, [1, 8], out)
    _save("unet_traj.npz", **out)


def cogvideox():
    from oracle.dit import DiT
    from paper_2505_14741_b200.spec import SPECS

    fwd = _seam()
    spec = SPECS["cogvideox_2b"]
    w = _Shim(DiT(spec, seed=0))
    x = E.initial_state(E.RunConfig(steps=50, seed=0, data_dim=spec.data_dim))
    t0 = time.time()
    eps = fwd(w, x, 37, 50)
    print(f"  cogvideox forward: {time.time() - t0:.0f} s", flush=True)
    _save("cogvideox_fwd.npz", eps=eps.astype(np.float32), t=np.array(37), T=np.array(50),
          seed=np.array(0), x_abs_mean=np.array(np.abs(x).mean()),
          eps_abs_mean=np.array(np.abs(eps).mean()))


if __name__ == "__main__":
    todo = sys.argv[1:] or ["dit_xl2", "unet", "cogvideox"]
    for name in todo:
        print(f"{name} ...", flush=True)
        {"dit_xl2": dit_xl2, "unet": unet, "cogvideox": cogvideox}[name]()
