"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

CPU restatement (numpy, float64 by default) of the U-Net-shaped predictor
pinned in ``paper_2505_14741_b200/unet_spec.py``. It re-derives the network
from the spec's docstring — levels, ResBlocks, Transformers, skips — and
uses only ``layer_table`` (the dimension table) from the product package, so
it is independent of the device op plan the CUDA executor runs.

No reference implementation exists for this network (the reference
predictor is an MLP, pkg/src/parastep/predictor.py:133-150): its arithmetic
is parity-unpinned. Its API contract ``pred(x, t, T) -> eps`` is the one the
reference sampler consumes (engines.py:40).
"""

from __future__ import annotations

import math

import numpy as np

from paper_2505_14741_b200.unet_spec import UNetSpec, layer_table

from .core import P_WEIGHT, make_stream, time_embed, uniforms


def init_params(s: UNetSpec, seed: int) -> dict[str, tuple]:
    """Xavier-uniform per the reference convention (predictor.py:202-215), zero bias."""
    out = {}
    for i, (name, fi, fo) in enumerate(layer_table(s)):
        lim = math.sqrt(6.0 / (fi + fo))
        u = uniforms(seed, make_stream(P_WEIGHT, i), fi * fo)
        out[name] = (((2.0 * u - 1.0) * lim).reshape(fi, fo), np.zeros(fo))
    return out


def _silu(x):
    return x / (1.0 + np.exp(-x))


def _gelu_tanh(x):
    return 0.5 * x * (1.0 + np.tanh(math.sqrt(2.0 / math.pi) * (x + 0.044715 * (x * x * x))))


def _group_norm(x: np.ndarray, groups: int, eps: float) -> np.ndarray:
    """x: H x W x C, statistics per group of C/groups channels over all pixels."""
    H, W, C = x.shape
    g = x.reshape(H * W, groups, C // groups)
    mu = g.mean(axis=(0, 2), keepdims=True)
    var = ((g - mu) ** 2).mean(axis=(0, 2), keepdims=True)
    return ((g - mu) / np.sqrt(var + eps)).reshape(H, W, C)


def _layer_norm(x: np.ndarray) -> np.ndarray:
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + 1e-6)


def _conv3x3(x: np.ndarray, W: np.ndarray, b: np.ndarray, stride: int = 1) -> np.ndarray:
    """pad 1; W rows ordered (ky, kx, cin)."""
    H, Wd, C = x.shape
    xp = np.zeros((H + 2, Wd + 2, C), dtype=x.dtype)
    xp[1:-1, 1:-1] = x
    Ho, Wo = (H - 1) // stride + 1, (Wd - 1) // stride + 1
    cols = [xp[ky:ky + stride * (Ho - 1) + 1:stride, kx:kx + stride * (Wo - 1) + 1:stride]
            for ky in range(3) for kx in range(3)]
    a = np.concatenate(cols, axis=-1).reshape(Ho * Wo, 9 * C)
    return (a @ W + b).reshape(Ho, Wo, -1)


class UNet:
    """pred(x, t, T) -> eps for one latent vector (C x H x W flat)."""

    def __init__(self, s: UNetSpec, seed: int = 0, dtype=np.float64):
        s.validate()
        self.s = s
        self.dtype = dtype
        self.p = {k: (W.astype(dtype), b.astype(dtype)) for k, (W, b) in init_params(s, seed).items()}
        self.data_dim = s.data_dim

    def _lin(self, name, a):
        W, b = self.p[name]
        return a @ W + b

    def _res(self, name, x, emb):
        s = self.s
        h = _conv3x3(_silu(_group_norm(x, s.groups, 1e-5)), *self.p[f"{name}.conv1"])
        h = h + self._lin(f"{name}.temb", emb)
        h = _conv3x3(_silu(_group_norm(h, s.groups, 1e-5)), *self.p[f"{name}.conv2"])
        skip = self._lin(f"{name}.skip", x) if f"{name}.skip" in self.p else x
        return skip + h

    def _attn_block(self, name, h):
        s = self.s
        H, W, C = h.shape
        L, nh, dh = H * W, C // s.head_dim, s.head_dim
        x = self._lin(f"{name}.proj_in", _group_norm(h, s.groups, 1e-6).reshape(L, C))
        for d in range(s.depth):
            nd = f"{name}.t{d}"
            qkv = self._lin(f"{nd}.qkv", _layer_norm(x)).reshape(L, 3, nh, dh)
            q, k, v = (qkv[:, i].transpose(1, 0, 2) for i in range(3))
            sc = (q @ k.transpose(0, 2, 1)) / math.sqrt(dh)
            sc = np.exp(sc - sc.max(axis=-1, keepdims=True))
            pr = sc / sc.sum(axis=-1, keepdims=True)
            o = (pr @ v).transpose(1, 0, 2).reshape(L, C)
            x = x + self._lin(f"{nd}.proj", o)
            x = x + self._lin(f"{nd}.fc2", _gelu_tanh(self._lin(f"{nd}.fc1", _layer_norm(x))))
        return h + self._lin(f"{name}.proj_out", x).reshape(H, W, C)

    def __call__(self, x: np.ndarray, t: int, T: int) -> np.ndarray:
        s, dt = self.s, self.dtype
        lat = np.asarray(x, dtype=np.float64).reshape(s.in_channels, s.height, s.width)
        h = lat.transpose(1, 2, 0).astype(dt)  # H x W x C
        emb = _silu(self._lin("temb2", _silu(self._lin("temb1", time_embed(t, s.freq_dim).astype(dt)))))
        h = _conv3x3(h, *self.p["conv_in"])
        skips = [h]
        n = len(s.channels)
        for lv in range(n):
            for r in range(s.layers):
                h = self._res(f"down{lv}.res{r}", h, emb)
                if s.attn[lv]:
                    h = self._attn_block(f"down{lv}.attn{r}", h)
                skips.append(h)
            if lv < n - 1:
                h = _conv3x3(h, *self.p[f"down{lv}.downsample"], stride=2)
                skips.append(h)
        h = self._res("mid.res0", h, emb)
        h = self._attn_block("mid.attn", h)
        h = self._res("mid.res1", h, emb)
        for lv in reversed(range(n)):
            for r in range(s.layers + 1):
                h = self._res(f"up{lv}.res{r}", np.concatenate([h, skips.pop()], axis=-1), emb)
                if s.attn[lv]:
                    h = self._attn_block(f"up{lv}.attn{r}", h)
            if lv > 0:
                h = np.repeat(np.repeat(h, 2, axis=0), 2, axis=1)
                h = _conv3x3(h, *self.p[f"up{lv}.upsample"])
        out = _conv3x3(_silu(_group_norm(h, s.groups, 1e-5)), *self.p["conv_out"])
        return out.transpose(2, 0, 1).reshape(-1).astype(np.float64)
