"""U-Net-shaped noise predictor on the GPU (BASELINE.json configs[4]).

``UNetWeights`` builds the network pinned in ``unet_spec.py`` on the device:
weights are drawn with the reference's Xavier-uniform stream convention by
``ps_rng_xavier`` (as ``DiTWeights`` does), the activation buffers of
``plan()`` are allocated here (sized for ``max_batch`` lanes), and the
forward is the native executor ``ps_unet_forward`` (csrc/unet.cu): bf16
tcgen05 implicit-GEMM convolutions with GroupNorm/SiLU/concat/resampling
fused into the operand gather, tcgen05 attention, fused epilogues.
Precision: bf16 operands, fp32 accumulation and fp32 activations between
ops (the paper runs AudioLDM2 in half precision); parity against the CPU
oracle is reported as relative MAE.
"""

from __future__ import annotations

import math

from . import _lib
from .errors import ConfigError
from .numerics import PURPOSE_WEIGHT_INIT, stream_id
from .predictor import _ISSUE_LOCK, time_embed_table
from .unet_spec import UNET_SPECS, UNetSpec, plan

T_TABLE = 1000  # frequency-embedding rows 0..T_TABLE (time_embed uses absolute t)


class UNetWeights:
    """A device-resident U-Net predictor; duck-types the reference weights object."""

    state_dtype_code = _lib.PS_F32
    precision = "bf16"

    def __init__(self, spec: UNetSpec | str, seed: int = 0, max_batch: int = 8):
        import torch

        self.spec = UNET_SPECS[spec] if isinstance(spec, str) else spec
        if not 1 <= max_batch <= 16:
            raise ConfigError("max_batch must be in [1, 16]")
        self.plan = plan(self.spec)
        self.seed = seed
        self.max_batch = max_batch
        self.ballast = 1
        lib = _lib.load(require_gpu=True)
        st = _lib.stream_ptr()
        self.W, self.b = [], []
        for i, (_name, fi, fo) in enumerate(self.plan.layers):
            w = torch.empty((fi, fo), dtype=torch.float32, device="cuda")
            lim = math.sqrt(6.0 / (fi + fo))
            _lib.check(lib.ps_rng_xavier(_lib.ptr(w), fi * fo, seed,
                                         stream_id(PURPOSE_WEIGHT_INIT, i), lim, _lib.PS_F32, st),
                       "unet init")
            self.W.append(w)
            self.b.append(torch.zeros(fo, dtype=torch.float32, device="cuda"))
        self.freq = torch.as_tensor(time_embed_table(T_TABLE, self.spec.freq_dim),
                                    dtype=torch.float32, device="cuda")
        self.bufs = [torch.zeros(max_batch * n, dtype=torch.bfloat16 if bf else torch.float32,
                                 device="cuda") for n, bf in self.plan.bufs]
        ops = (_lib.ps_unet_op * len(self.plan.ops))()
        for k, op in enumerate(self.plan.ops):
            o = ops[k]
            for f in ("kind", "layer", "pre", "in1", "in2", "c1", "c2", "h", "w", "taps",
                      "resample", "cout", "temb_layer", "temb_off", "resid", "out", "out_bf16",
                      "act", "heads", "eps", "out2"):
                setattr(o, f, getattr(op, f))
        self._ops = ops
        self._bufp = _lib.ptr_array([_lib.ptr(b) for b in self.bufs])
        s = self.spec
        cfg = _lib.ps_unet_config(
            in_channels=s.in_channels, height=s.height, width=s.width, groups=s.groups,
            freq_dim=s.freq_dim, temb_dim=s.temb_dim, temb_cols=self.plan.temb_cols,
            max_batch=max_batch, n_ops=len(self.plan.ops), n_bufs=len(self.bufs), ops=ops,
            bufs=self._bufp)
        Wp = _lib.ptr_array([_lib.ptr(w) for w in self.W])
        bp = _lib.ptr_array([_lib.ptr(b) for b in self.b])
        wts = _lib.ps_dit_weights(n_layers=len(self.W), W=Wp, b=bp, pos=None,
                                  freq_table=_lib.ptr(self.freq), freq_rows=T_TABLE + 1)
        torch.cuda.synchronize()
        h = _lib.C.c_void_p()
        _lib.check(lib.ps_unet_create(cfg, wts, _lib.C.byref(h)), "unet create")
        self._h = h
        self._lib = lib

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self._lib.ps_unet_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def data_dim(self) -> int:
        return self.spec.data_dim

    def flops_per_forward(self) -> float:
        return float(self.plan.flops_per_forward())

    def kernels_per_forward(self, B: int = 1) -> int:
        return int(self._lib.ps_unet_kernels_per_forward(self._h))

    def forward_device(self, x, ts, T: int, out, stream=None) -> None:
        """x, out: CUDA float32 [B, data_dim]; ts: B step indices (<= 1000). Async."""
        B = len(ts)
        if B > self.max_batch:
            raise ConfigError(f"batch {B} exceeds max_batch {self.max_batch}")
        tsa = (_lib.C.c_int32 * B)(*ts)
        with _ISSUE_LOCK:
            _lib.check(self._lib.ps_unet_forward(self._h, _lib.ptr(x), tsa, B, _lib.ptr(out),
                                                 _lib.stream_ptr(stream)), "unet forward")
