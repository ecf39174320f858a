"""Counter-based random streams and divergence metrics — the drop-in for
pkg/src/parastep/numerics.py.

Draws run on the GPU (C-ABI ``ps_rng_*``): the SplitMix64 counter words and
the uniforms are bit-identical to the reference; normals go through fp64
log/sqrt/sincos on device (within a few ulp of numpy's). ``rel_mae`` / ``mse``
are reporting metrics evaluated on host in float64 with the reference's
strict left-to-right summation (numerics.py:135-166); they are not on the
denoise hot path.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import DegenerateReferenceError, DimensionError, ParameterError

Vector = np.ndarray

PURPOSE_INIT = 0
PURPOSE_STEP = 1
PURPOSE_TRAIN = 2
PURPOSE_WEIGHT_INIT = 3
PURPOSE_DATASET = 4

_MASK64 = 0xFFFFFFFFFFFFFFFF


def stream_id(purpose: int, index: int = 0) -> int:
    """(purpose << 32) | (index & 0xFFFFFFFF) — numerics.py:30-31."""
    return ((purpose << 32) | (index & 0xFFFFFFFF)) & _MASK64


def _device_draw(kind: str, seed: int, stream: int, n: int, counter: int, dtype, device=None):
    import torch

    lib = _lib.load(require_gpu=True)
    tdt = torch.float64 if dtype == _lib.PS_F64 else torch.float32
    out = torch.empty(n, dtype=tdt, device=device or "cuda")
    fn = lib.ps_rng_normal if kind == "normal" else lib.ps_rng_uniform
    _lib.check(fn(_lib.ptr(out), n, seed & _MASK64, stream & _MASK64, counter & _MASK64, dtype,
                  _lib.stream_ptr()), f"rng_{kind}")
    return out


def draw_normal_device(seed: int, stream: int, n: int, counter: int = 0, dtype=_lib.PS_F64):
    """n standard normals as a CUDA tensor (no host round trip)."""
    if n < 1:
        raise ParameterError("draw count must be >= 1")
    return _device_draw("normal", seed, stream, n, counter, dtype)


@dataclass
class RngStream:
    """Deterministic, independently addressable stream (numerics.py:83-115)."""

    run_seed: int
    stream: int
    counter: int = field(default=0)

    def _advance(self, n: int) -> int:
        if n < 1:
            raise ParameterError("draw count must be >= 1")
        c = self.counter
        self.counter += n
        return c

    def normals(self, n: int) -> Vector:
        c = self._advance(n)
        return _device_draw("normal", self.run_seed, self.stream, n, c, _lib.PS_F64).cpu().numpy()

    def uniforms(self, n: int) -> Vector:
        c = self._advance(n)
        return _device_draw("uniform", self.run_seed, self.stream, n, c, _lib.PS_F64).cpu().numpy()

    def integers(self, n: int, lo: int, hi: int) -> list[int]:
        if hi < lo:
            raise ParameterError("integer range is empty")
        span = hi - lo + 1
        return [lo + min(int(u * span), span - 1) for u in self.uniforms(n)]


def draw_normal(seed: int, stream: int, n: int, counter: int = 0) -> Vector:
    """numerics.py:118-120, computed on the GPU."""
    return RngStream(seed, stream, counter).normals(n)


def as_vector(values) -> Vector:
    v = np.asarray(values, dtype=np.float64)
    if v.ndim != 1 or v.size < 1:
        raise DimensionError(f"expected a 1-D vector of length >= 1, got shape {v.shape}")
    return v


def _sum_lr(v: np.ndarray) -> float:
    # strict left-to-right float64 accumulation (np.add.accumulate is a
    # sequential scan), identical to the reference's Python loop
    return float(np.add.accumulate(v)[-1])


def rel_mae(a, b) -> float:
    """Eq. 7: mean|a-b| / mean|a|, a is the reference (numerics.py:144-158)."""
    a = as_vector(a)
    b = as_vector(b)
    if len(a) != len(b):
        raise DimensionError(f"length mismatch: {len(a)} vs {len(b)}")
    n = len(a)
    den = _sum_lr(np.abs(a)) / n
    if den == 0.0:
        raise DegenerateReferenceError("reference vector has zero mean magnitude")
    return (_sum_lr(np.abs(a - b)) / n) / den


def mse(a, b) -> float:
    a = as_vector(a)
    b = as_vector(b)
    if len(a) != len(b):
        raise DimensionError(f"length mismatch: {len(a)} vs {len(b)}")
    d = a - b
    return _sum_lr(d * d) / len(a)
