"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

CPU restatement of the DiT-shaped noise predictor pinned in
``paper_2505_14741_b200/spec.py``, written directly from that docstring in
plain numpy (float64 by default). It is independent of the CUDA code: the
only thing shared is the table of dimensions.

No reference implementation exists for this network (the reference predictor
is an MLP, pkg/src/parastep/predictor.py:133-150), so its *arithmetic* is
parity-unpinned; its API contract ``pred(x, t, T) -> eps`` is the one the
reference sampler consumes (engines.py:40), which is how the golden fixtures
drive it through the reference's own engines.
"""

from __future__ import annotations

import math

import numpy as np

from paper_2505_14741_b200.spec import DiTSpec, layer_table

from .core import P_WEIGHT, make_stream, time_embed, uniforms


def _sincos_1d(d: int, pos: np.ndarray) -> np.ndarray:
    half = d // 2
    w = 10000.0 ** (-np.arange(half, dtype=np.float64) / half)
    ang = pos[:, None].astype(np.float64) * w[None, :]
    return np.concatenate([np.sin(ang), np.cos(ang)], axis=1)


def pos_table(s: DiTSpec) -> np.ndarray:
    f, h, w = np.meshgrid(np.arange(s.frames), np.arange(s.grid_h), np.arange(s.grid_w),
                          indexing="ij")
    f, h, w = f.ravel(), h.ravel(), w.ravel()
    D = s.hidden
    if s.frames == 1:
        return np.concatenate([_sincos_1d(D // 2, h), _sincos_1d(D // 2, w)], axis=1)
    return np.concatenate(
        [_sincos_1d(D // 4, f), _sincos_1d(3 * D // 8, h), _sincos_1d(3 * D // 8, w)], axis=1)


P_TEXT = 7  # synthetic text conditioning stream (spec.py)


def text_states(s: DiTSpec, seed: int) -> np.ndarray:
    """The fixed text rows: normal(seed, (7<<32)|0)[text_tokens * D]."""
    from .core import normals

    return normals(seed, make_stream(P_TEXT, 0), s.text_tokens * s.hidden).reshape(
        s.text_tokens, s.hidden)


def rope_angles(s: DiTSpec) -> np.ndarray:
    """[tokens, head_dim / 2] rotation angles of spec.py's 3D RoPE."""
    dh = s.head_dim
    bands = [(dh // 4, "f"), (3 * dh // 8, "h"), (3 * dh // 8, "w")]
    f, h, w = np.meshgrid(np.arange(s.frames), np.arange(s.grid_h), np.arange(s.grid_w),
                          indexing="ij")
    pos = {"f": f.ravel(), "h": h.ravel(), "w": w.ravel()}
    cols = []
    for d_a, ax in bands:
        k = np.arange(d_a // 2, dtype=np.float64)
        cols.append(pos[ax][:, None].astype(np.float64) * (10000.0 ** (-2.0 * k / d_a))[None, :])
    return np.concatenate(cols, axis=1)


def apply_rope(x: np.ndarray, ang: np.ndarray) -> np.ndarray:
    """x [H, Lv, dh]: interleaved pairs (2i, 2i+1) rotated by ang[:, i]."""
    c, sn = np.cos(ang)[None], np.sin(ang)[None]
    x0, x1 = x[..., 0::2], x[..., 1::2]
    out = np.empty_like(x)
    out[..., 0::2] = x0 * c - x1 * sn
    out[..., 1::2] = x1 * c + x0 * sn
    return out


def init_params(s: DiTSpec, seed: int, bias_scale: float = 0.0) -> dict[str, tuple]:
    """Xavier-uniform per the reference convention; optional nonzero test biases.

    Test biases (not part of the reference convention; they only exercise the
    bias path) draw from stream (6<<32)|i: b = (2u-1)*bias_scale.
    """
    out = {}
    for i, (name, fi, fo) in enumerate(layer_table(s)):
        lim = math.sqrt(6.0 / (fi + fo))
        u = uniforms(seed, make_stream(P_WEIGHT, i), fi * fo)
        W = ((2.0 * u - 1.0) * lim).reshape(fi, fo)
        if bias_scale:
            ub = uniforms(seed, make_stream(6, i), fo)
            b = (2.0 * ub - 1.0) * bias_scale
        else:
            b = np.zeros(fo)
        out[name] = (W, b)
    return out


def _latent_to_tokens(s: DiTSpec, x: np.ndarray) -> np.ndarray:
    p = s.patch
    if s.layout == "CHW":
        v = x.reshape(s.channels, s.frames, s.height, s.width)
    else:
        v = x.reshape(s.frames, s.height, s.width, s.channels).transpose(3, 0, 1, 2)
    # v: C, F, H, W -> tokens (f, hp, wp), features (c, ph, pw)
    v = v.reshape(s.channels, s.frames, s.grid_h, p, s.grid_w, p)
    v = v.transpose(1, 2, 4, 0, 3, 5)
    return v.reshape(s.tokens, s.patch_dim)


def _tokens_to_latent(s: DiTSpec, tok: np.ndarray) -> np.ndarray:
    p = s.patch
    v = tok.reshape(s.frames, s.grid_h, s.grid_w, s.channels, p, p)
    v = v.transpose(3, 0, 1, 4, 2, 5).reshape(s.channels, s.frames, s.height, s.width)
    if s.layout == "FHWC":
        v = v.transpose(1, 2, 3, 0)
    return v.reshape(-1)


def _ln(x: np.ndarray) -> np.ndarray:
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + 1e-6)


def _silu(x):
    return x / (1.0 + np.exp(-x))


def _gelu_tanh(x):
    return 0.5 * x * (1.0 + np.tanh(math.sqrt(2.0 / math.pi) * (x + 0.044715 * (x * x * x))))


def _attention(q, k, v, chunk: int = 2048):
    """softmax(q k^T / sqrt(dh)) v per head; long sequences (the 17,550-token
    CogVideoX shape) in query chunks so a head's scores never exceed
    chunk x L (the result is the same row-wise formula)."""
    H, L, dh = q.shape
    out = np.empty_like(q)
    step = L if L <= chunk else chunk
    for h in range(H):
        kt = k[h].T
        for r0 in range(0, L, step):
            sco = (q[h, r0:r0 + step] @ kt) / math.sqrt(dh)
            sco = np.exp(sco - sco.max(axis=-1, keepdims=True))
            pr = sco / sco.sum(axis=-1, keepdims=True)
            out[h, r0:r0 + step] = pr @ v[h]
    return out


class DiT:
    """pred(x, t, T) -> eps for one latent vector."""

    def __init__(self, s: DiTSpec, seed: int = 0, bias_scale: float = 0.0,
                 dtype=np.float64):
        s.validate()
        self.s = s
        self.dtype = dtype
        self.params = {k: (W.astype(dtype), b.astype(dtype))
                       for k, (W, b) in init_params(s, seed, bias_scale).items()}
        self.pos = None if s.rope else pos_table(s).astype(dtype)
        self.text = text_states(s, seed).astype(dtype) if s.text_tokens else None
        self.ang = rope_angles(s) if s.rope else None
        self.data_dim = s.data_dim

    def _lin(self, name, a):
        W, b = self.params[name]
        return a @ W + b

    def __call__(self, x: np.ndarray, t: int, T: int) -> np.ndarray:
        s, dt = self.s, self.dtype
        D, H, dh = s.hidden, s.heads, s.head_dim
        tok = _latent_to_tokens(s, np.asarray(x, dtype=np.float64)).astype(dt)
        h = self._lin("patch", tok)
        if self.pos is not None:
            h = h + self.pos
        Tx = s.text_tokens
        if Tx:
            h = np.concatenate([self.text, h], axis=0)
        c = self._lin("temb2", _silu(self._lin("temb1", time_embed(t, s.freq_dim).astype(dt))))
        sc = _silu(c)
        L = s.seq_len
        txt = (np.arange(L) < Tx)[:, None]
        for i in range(s.depth):
            m = self._lin(f"b{i}.ada", sc)
            v6 = [m[k * D:(k + 1) * D] for k in range(6)]
            t6 = [m[(6 + k) * D:(7 + k) * D] for k in range(6)] if Tx else v6
            sh1, sc1, g1, sh2, sc2, g2 = (np.where(txt, tv, vv) for vv, tv in zip(v6, t6))
            a = _ln(h) * (1.0 + sc1) + sh1
            qkv = self._lin(f"b{i}.qkv", a).reshape(L, 3, H, dh)
            q, k, v = qkv[:, 0].transpose(1, 0, 2), qkv[:, 1].transpose(1, 0, 2), \
                qkv[:, 2].transpose(1, 0, 2)
            if self.ang is not None:  # video rows of q and k
                q = q.copy()
                k = k.copy()
                q[:, Tx:] = apply_rope(q[:, Tx:], self.ang)
                k[:, Tx:] = apply_rope(k[:, Tx:], self.ang)
            o = _attention(q, k, v).transpose(1, 0, 2).reshape(L, D)
            h = h + g1 * self._lin(f"b{i}.proj", o)
            a = _ln(h) * (1.0 + sc2) + sh2
            h = h + g2 * self._lin(f"b{i}.fc2", _gelu_tanh(self._lin(f"b{i}.fc1", a)))
        m = self._lin("final.ada", sc)
        shf, scf = m[:D], m[D:]
        out = self._lin("final.out", _ln(h[Tx:]) * (1.0 + scf) + shf)
        return _tokens_to_latent(s, out.astype(np.float64))
