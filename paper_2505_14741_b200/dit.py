"""DiT-shaped noise predictors on the GPU (BASELINE.json configs 0-3).

``DiTWeights`` builds the network pinned in ``spec.py`` directly on the
device: weights are drawn with the reference's Xavier-uniform stream
convention by ``ps_rng_xavier`` (fp64 draw, rounded to fp32 storage), and the
forward is the C++/CUDA ``ps_dit_forward`` (csrc/dit.cu): adaLN conditioning
GEMV, patch embedding, per block LN-modulate -> QKV GEMM -> attention ->
gated proj GEMM -> LN-modulate -> GELU fc1 GEMM -> gated fc2 GEMM, final
LN-modulate -> GEMM with the unpatchify scatter fused in its epilogue.

precision:
  "fp32" — fp32 activations, GEMMs on tcgen05 kind::tf32 with the 3-pass
           hi/lo split (fp32-class accuracy; the 1e-4 path of configs[1]),
           (gemm_impl="reference_simt" selects the SIMT fp32 GEMM and
           attention kernels instead: an on-device cross-check used by the
           tests only, never by the samplers, bench or CLI);
  "bf16" — bf16 GEMM operands on tcgen05 kind::f16, fp32 accumulation and
           fp32 residual stream (configs[2]).
"""

from __future__ import annotations

import math

import numpy as np

from . import _lib
from .errors import ConfigError
from .numerics import PURPOSE_WEIGHT_INIT, stream_id
from .predictor import _ISSUE_LOCK, time_embed_table
from .spec import SPECS, DiTSpec, layer_table

T_TABLE = 1000  # frequency-embedding rows 0..T_TABLE (time_embed uses absolute t)
PURPOSE_TEST_BIAS = 6


def _sincos(d: int, pos: np.ndarray) -> np.ndarray:
    half = d // 2
    k = np.arange(half, dtype=np.float64)
    w = np.power(10000.0, -k / half)
    a = np.outer(pos.astype(np.float64), w)
    return np.hstack([np.sin(a), np.cos(a)])


def position_table(s: DiTSpec) -> np.ndarray:
    """Fixed sin-cos position embedding of spec.py, tokens (f, hp, wp)."""
    idx = np.arange(s.tokens)
    f = idx // (s.grid_h * s.grid_w)
    hp = (idx // s.grid_w) % s.grid_h
    wp = idx % s.grid_w
    D = s.hidden
    if s.frames == 1:
        return np.hstack([_sincos(D // 2, hp), _sincos(D // 2, wp)])
    return np.hstack([_sincos(D // 4, f), _sincos(3 * D // 8, hp), _sincos(3 * D // 8, wp)])


PURPOSE_TEXT = 7  # the fixed text states of a text-conditioned spec (spec.py)


def rope_table(s: DiTSpec) -> np.ndarray:
    """[tokens, head_dim/2, 2] (cos, sin) of spec.py's 3D RoPE: pair i of band
    (t: dh/4, h: 3dh/8, w: 3dh/8 dims) rotates by pos * 10000^(-2k/d_band)."""
    dh = s.head_dim
    idx = np.arange(s.tokens)
    pos = [idx // (s.grid_h * s.grid_w), (idx // s.grid_w) % s.grid_h, idx % s.grid_w]
    ang = []
    for p, d in zip(pos, (dh // 4, 3 * dh // 8, 3 * dh // 8)):
        k = np.arange(d // 2, dtype=np.float64)
        ang.append(np.outer(p.astype(np.float64), np.power(10000.0, -2.0 * k / d)))
    a = np.hstack(ang)
    return np.stack([np.cos(a), np.sin(a)], axis=-1)


class DiTWeights:
    """A device-resident DiT predictor; duck-types the reference weights object."""

    state_dtype_code = _lib.PS_F32

    def __init__(self, spec: DiTSpec | str, seed: int = 0, precision: str = "fp32",
                 max_batch: int = 8, bias_scale: float = 0.0, gemm_impl: str = "auto"):
        import torch

        self.spec = SPECS[spec] if isinstance(spec, str) else spec
        self.spec.validate()
        if precision not in ("fp32", "bf16"):
            raise ConfigError(f"unknown precision {precision!r}")
        if gemm_impl not in ("auto", "tcgen05", "reference_simt"):
            raise ConfigError(f"unknown gemm_impl {gemm_impl!r}")
        if not 1 <= max_batch <= 16:
            raise ConfigError("max_batch must be in [1, 16]")
        self.seed = seed
        self.precision = precision
        self.max_batch = max_batch
        self.bias_scale = bias_scale
        self.gemm_impl = gemm_impl
        self.ballast = 1
        lib = _lib.load(require_gpu=True)
        st = _lib.stream_ptr()
        self.W, self.b = [], []
        for i, (_name, fi, fo) in enumerate(layer_table(self.spec)):
            w = torch.empty((fi, fo), dtype=torch.float32, device="cuda")
            lim = math.sqrt(6.0 / (fi + fo))
            _lib.check(lib.ps_rng_xavier(_lib.ptr(w), fi * fo, seed,
                                         stream_id(PURPOSE_WEIGHT_INIT, i), lim, _lib.PS_F32, st),
                       "dit init")
            if bias_scale:
                u = torch.empty(fo, dtype=torch.float64, device="cuda")
                _lib.check(lib.ps_rng_uniform(_lib.ptr(u), fo, seed,
                                              stream_id(PURPOSE_TEST_BIAS, i), 0, _lib.PS_F64, st),
                           "dit bias init")
                b = ((2.0 * u - 1.0) * bias_scale).to(torch.float32)
            else:
                b = torch.zeros(fo, dtype=torch.float32, device="cuda")
            self.W.append(w)
            self.b.append(b)
        s = self.spec
        self.pos = None if s.rope else torch.as_tensor(position_table(s), dtype=torch.float32,
                                                       device="cuda")
        self.rope = torch.as_tensor(rope_table(s), dtype=torch.float32, device="cuda") \
            if s.rope else None
        self.text = None
        if s.text_tokens:
            t64 = torch.empty(s.text_tokens * s.hidden, dtype=torch.float64, device="cuda")
            _lib.check(lib.ps_rng_normal(_lib.ptr(t64), t64.numel(), seed,
                                         stream_id(PURPOSE_TEXT, 0), 0, _lib.PS_F64, st),
                       "text states")
            self.text = t64.to(torch.float32)
        self.freq = torch.as_tensor(time_embed_table(T_TABLE, self.spec.freq_dim),
                                    dtype=torch.float32, device="cuda")
        cfg = _lib.ps_dit_config(
            channels=s.channels, frames=s.frames, height=s.height, width=s.width,
            layout=0 if s.layout == "CHW" else 1, patch=s.patch, hidden=s.hidden, depth=s.depth,
            heads=s.heads, mlp_hidden=s.mlp_hidden, freq_dim=s.freq_dim, max_batch=max_batch,
            precision=0 if precision == "fp32" else 1,
            gemm_impl={"auto": 0, "reference_simt": 1, "tcgen05": 2}[gemm_impl],
            text_tokens=s.text_tokens, rope=int(s.rope))
        Wp = _lib.ptr_array([_lib.ptr(w) for w in self.W])
        bp = _lib.ptr_array([_lib.ptr(b) for b in self.b])
        opt = lambda t: _lib.ptr(t) if t is not None else None  # noqa: E731
        wts = _lib.ps_dit_weights(n_layers=len(self.W), W=Wp, b=bp, pos=opt(self.pos),
                                  freq_table=_lib.ptr(self.freq), freq_rows=T_TABLE + 1,
                                  text=opt(self.text), rope=opt(self.rope))
        torch.cuda.synchronize()
        h = _lib.C.c_void_p()
        _lib.check(lib.ps_dit_create(cfg, wts, _lib.C.byref(h)), "dit create")
        self._h = h
        self._lib = lib

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self._lib.ps_dit_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def data_dim(self) -> int:
        return self.spec.data_dim

    def flops_per_forward(self) -> float:
        return float(self._lib.ps_dit_flops(self._h))

    def kernels_per_forward(self, B: int = 1) -> int:
        return int(self._lib.ps_dit_kernels_per_forward(self._h))

    def bench_gemm(self, which: int, B: int, iters: int, stream=None) -> None:
        """Launch block 0's GEMM `which` (0 qkv, 1 proj, 2 fc1, 3 fc2) iters times (async)."""
        _lib.check(self._lib.ps_dit_bench_gemm(self._h, which, B, iters, _lib.stream_ptr(stream)),
                   "bench_gemm")

    def gemm_shape(self, which: int, B: int = 1) -> tuple[int, int, int]:
        s = self.spec
        D, M = s.hidden, B * s.seq_len
        return [(M, 3 * D, D), (M, D, D), (M, s.mlp_hidden, D), (M, D, s.mlp_hidden)][which]

    def reserve_conditioning(self, T: int) -> None:
        """Allocate the per-run conditioning table for steps 0..T (not capturable)."""
        _lib.check(self._lib.ps_dit_condition_reserve(self._h, T), "condition reserve")

    def prepare_conditioning(self, T: int, stream=None) -> int:
        """Fill rows 0..T of the conditioning table on the stream (capturable);
        returns the kernel launches issued."""
        _lib.check(self._lib.ps_dit_condition(self._h, T, _lib.stream_ptr(stream)), "condition")
        chunk = int(self._lib.ps_dit_condition_chunk(self._h))
        return 3 * (-(-(T + 1) // chunk))

    def clear_conditioning(self) -> None:
        _lib.check(self._lib.ps_dit_condition_clear(self._h), "condition clear")

    def forward_device(self, x, ts, T: int, out, stream=None) -> None:
        """x, out: CUDA float32 [B, data_dim]; ts: B step indices (<= 1000). Async."""
        B = len(ts)
        if B > self.max_batch:
            raise ConfigError(f"batch {B} exceeds max_batch {self.max_batch}")
        tsa = (_lib.C.c_int32 * B)(*ts)
        with _ISSUE_LOCK:
            _lib.check(self._lib.ps_dit_forward(self._h, _lib.ptr(x), tsa, B, _lib.ptr(out),
                                                _lib.stream_ptr(stream)), "dit forward")
