"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

CPU restatement of the reference numerics on the hot path, numpy float64.

Every function names the reference lines it restates. The arithmetic is
written op-for-op in the same order as the reference (same numpy ufuncs, same
rounding points) so the golden fixtures produced by the reference itself
match this module bit-for-bit.
"""

from __future__ import annotations

import math

import numpy as np

U64 = 0xFFFFFFFFFFFFFFFF

# Stream purposes — pkg/src/parastep/numerics.py:23-27
P_INIT, P_STEP, P_TRAIN, P_WEIGHT, P_DATASET = 0, 1, 2, 3, 4

_C_GOLD = 0x9E3779B97F4A7C15
_C_M1 = 0xBF58476D1CE4E5B9
_C_M2 = 0x94D049BB133111EB


def make_stream(purpose: int, index: int = 0) -> int:
    """stream id = (purpose << 32) | low 32 bits of index (numerics.py:30-31)."""
    return ((purpose << 32) | (index & 0xFFFFFFFF)) & U64


def splitmix_scalar(v: int) -> int:
    """SplitMix64 finalizer on a Python int (numerics.py:40-45)."""
    v = (v + _C_GOLD) & U64
    v = ((v ^ (v >> 30)) * _C_M1) & U64
    v = ((v ^ (v >> 27)) * _C_M2) & U64
    return v ^ (v >> 31)


def stream_key(seed: int, stream: int) -> int:
    """Per-(seed, stream) key h = mix(mix(seed) ^ stream) (numerics.py:58-59)."""
    return splitmix_scalar(splitmix_scalar(seed & U64) ^ (stream & U64))


def splitmix_vec(v: np.ndarray) -> np.ndarray:
    """Vectorised finalizer over uint64, wrapping mod 2^64 (numerics.py:48-53)."""
    v = v + np.uint64(_C_GOLD)
    v = (v ^ (v >> np.uint64(30))) * np.uint64(_C_M1)
    v = (v ^ (v >> np.uint64(27))) * np.uint64(_C_M2)
    return v ^ (v >> np.uint64(31))


def rng_words(seed: int, stream: int, ctr: np.ndarray) -> np.ndarray:
    """64 random bits per counter (numerics.py:56-60)."""
    return splitmix_vec(np.uint64(stream_key(seed, stream)) ^ ctr.astype(np.uint64))


def rng_uniform_at(seed: int, stream: int, ctr: np.ndarray) -> np.ndarray:
    """u = ((w >> 11) + 1) * 2^-53, in (0, 1] (numerics.py:63-66)."""
    top = rng_words(seed, stream, ctr) >> np.uint64(11)
    return (top + np.uint64(1)).astype(np.float64) * 2.0 ** -53


def rng_normal_at(seed: int, stream: int, ctr: np.ndarray) -> np.ndarray:
    """Box-Muller on counter pairs (2j, 2j+1); parity picks cos/sin (numerics.py:69-80)."""
    even = ctr & ~np.uint64(1)
    u_a = rng_uniform_at(seed, stream, even)
    u_b = rng_uniform_at(seed, stream, even + np.uint64(1))
    rad = np.sqrt(-2.0 * np.log(u_a))
    ang = (2.0 * np.pi) * u_b
    return np.where(ctr == even, rad * np.cos(ang), rad * np.sin(ang))


def normals(seed: int, stream: int, n: int, counter: int = 0) -> np.ndarray:
    """draw_normal(seed, stream, n, counter) (numerics.py:118-120, 95-104)."""
    ctr = np.arange(counter, counter + n, dtype=np.uint64)
    return rng_normal_at(seed, stream, ctr)


def uniforms(seed: int, stream: int, n: int, counter: int = 0) -> np.ndarray:
    ctr = np.arange(counter, counter + n, dtype=np.uint64)
    return rng_uniform_at(seed, stream, ctr)


def rel_mae(ref: np.ndarray, cmp: np.ndarray) -> float:
    """Eq. 7 with strict left-to-right float64 sums (numerics.py:135-158).

    np.add.accumulate is a sequential left-to-right scan, so its last element
    equals the reference's Python-loop sum bit-for-bit.
    """
    a = np.asarray(ref, dtype=np.float64)
    b = np.asarray(cmp, dtype=np.float64)
    if a.ndim != 1 or a.size < 1 or a.shape != b.shape:
        raise ValueError("rel_mae: need equal-length 1-D vectors")
    n = a.size
    den = float(np.add.accumulate(np.abs(a))[-1]) / n
    if den == 0.0:
        raise ZeroDivisionError("reference vector has zero mean magnitude")
    num = float(np.add.accumulate(np.abs(a - b))[-1]) / n
    return num / den


# ----------------------------------------------------------------- schedule

class Sched:
    """Linear-beta schedule tables (schedule.py:22-86)."""

    def __init__(self, T: int, sigma_mode: str = "posterior"):
        scale = 1000.0 / T
        b0, b1 = min(1e-4 * scale, 0.98), min(0.02 * scale, 0.98)
        self.T = T
        self.sigma_mode = sigma_mode
        self.beta = np.linspace(b0, b1, T)
        self.alpha = 1.0 - self.beta
        self.alpha_bar = np.cumprod(self.alpha)
        if sigma_mode == "zero":
            self.sigma = np.zeros(T)
        else:
            prev = np.concatenate(([1.0], self.alpha_bar[:-1]))
            self.sigma = np.sqrt(self.beta * (1.0 - prev) / (1.0 - self.alpha_bar))

    def coeffs(self, t: int) -> tuple[float, float, float, bool]:
        """(c, sqrt(alpha_t), sigma_t, noisy) used by one reverse step."""
        a = self.alpha[t - 1]
        ab = self.alpha_bar[t - 1]
        c = (1.0 - a) / math.sqrt(1.0 - ab)
        noisy = not (t == 1 or self.sigma_mode == "zero")
        return c, math.sqrt(a), float(self.sigma[t - 1]), noisy


def ddpm_step(x: np.ndarray, t: int, eps: np.ndarray, sch: Sched, z: np.ndarray) -> np.ndarray:
    """Posterior mean + sigma_t z (schedule.py:102-131)."""
    c, sa, sig, noisy = sch.coeffs(t)
    mean = (x - c * eps) / sa
    if not noisy:
        return mean
    return mean + sig * z


# ----------------------------------------------------------------- MLP predictor

def time_embed(t: int, dim: int) -> np.ndarray:
    """Interleaved sin/cos of absolute t (predictor.py:44-65)."""
    half = dim // 2
    rates = np.array([1.0]) if half == 1 else 10000.0 ** (-np.arange(half) / (half - 1))
    ang = t * rates
    out = np.empty(dim, dtype=np.float64)
    out[0::2] = np.sin(ang)
    out[1::2] = np.cos(ang)
    return out


class MLP:
    """The reference predictor: [x, temb] -> dense -> act ... -> dense (predictor.py:68-150)."""

    def __init__(self, ws: list[np.ndarray], bs: list[np.ndarray], activation: str = "silu"):
        self.ws = ws
        self.bs = bs
        self.activation = activation

    @property
    def data_dim(self) -> int:
        return self.ws[-1].shape[1]

    @property
    def embed_dim(self) -> int:
        return self.ws[0].shape[0] - self.data_dim

    @classmethod
    def init(cls, data_dim: int, hidden=(64, 64), embed_dim: int = 16, seed: int = 42,
             activation: str = "silu") -> "MLP":
        """Xavier-uniform weights from stream (3<<32)|layer, zero bias (predictor.py:202-215)."""
        dims = [data_dim + embed_dim, *hidden, data_dim]
        ws, bs = [], []
        for i in range(len(dims) - 1):
            fi, fo = dims[i], dims[i + 1]
            lim = math.sqrt(6.0 / (fi + fo))
            u = uniforms(seed, make_stream(P_WEIGHT, i), fi * fo)
            ws.append(((2.0 * u - 1.0) * lim).reshape(fi, fo))
            bs.append(np.zeros(fo))
        return cls(ws, bs, activation)

    def __call__(self, x: np.ndarray, t: int, T: int) -> np.ndarray:
        a = np.concatenate([x, time_embed(t, self.embed_dim)])
        last = len(self.ws) - 1
        for i, (w, b) in enumerate(zip(self.ws, self.bs)):
            z = np.dot(a, w) + b
            a = _act(z, self.activation) if i < last else z
        return a


def _sigmoid_split(z: np.ndarray) -> np.ndarray:
    """Sign-split logistic (predictor.py:108-116)."""
    out = np.empty_like(z)
    pos = z >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-z[pos]))
    e = np.exp(z[~pos])
    out[~pos] = e / (1.0 + e)
    return out


def _act(z: np.ndarray, kind: str) -> np.ndarray:
    if kind == "tanh":
        return np.tanh(z)
    return z * _sigmoid_split(z)


class IdentityNet:
    """eps == x; the reference tests' hand-unrollable predictor (tests/test_engines.py:55-59)."""

    def __init__(self, data_dim: int):
        self.data_dim = data_dim

    def __call__(self, x: np.ndarray, t: int, T: int) -> np.ndarray:
        return np.array(x, dtype=np.float64, copy=True)
