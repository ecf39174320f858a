"""The noise predictor ε_θ — the drop-in for pkg/src/parastep/predictor.py
(inference side: ``forward``, ``forward_batch``, ``init_weights``).

Two predictor families sit behind the same ``forward(w, x, t, T)`` contract
the reference sampler binds by name (engines.py:40, worker.py:45):

* ``PredictorWeights`` — the reference's own MLP (fp64 on device,
  ``ps_mlp_forward``), weights in the reference's (fan_in, fan_out) layout;
* ``DiTWeights`` (dit.py) — the DiT-shaped predictors of BASELINE.json.

Every device predictor also implements the engine-facing protocol
``forward_device(x[B, n], ts, T, out[B, n], stream)`` (async, no sync), which
is what the GPU samplers and CUDA graphs call.

Contract kept from the reference: inputs are 1-D float64 vectors; results are
fresh arrays (never views of staging buffers); ``forward`` does not mutate
``w``; ``forward_batch`` element i is bitwise ``forward(w, xs[i], ts[i], T)``
(the device kernels have no cross-lane reduction, so batching cannot change
bits — tested).
"""

from __future__ import annotations

import math
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import ConfigError, DimensionError, ParameterError
from .numerics import PURPOSE_WEIGHT_INIT, Vector, as_vector, stream_id

_ISSUE_LOCK = threading.RLock()

ACT_TANH = "tanh"
ACT_SILU = "silu"
_ACT_ID = {ACT_TANH: 0, ACT_SILU: 1}
_EMBED_MAX_PERIOD = 10000.0


def time_embed(t: int, T: int, dim: int) -> Vector:
    """Interleaved sin/cos of absolute t (predictor.py:44-65); a host table row."""
    if dim < 2 or dim % 2 != 0:
        raise ParameterError(f"embedding dim must be even and >= 2, got {dim}")
    if not 0 <= t <= T:
        raise ParameterError(f"step index {t} outside [0, {T}]")
    half = dim // 2
    rates = np.array([1.0]) if half == 1 else _EMBED_MAX_PERIOD ** (-np.arange(half) / (half - 1))
    ang = t * rates
    out = np.empty(dim, dtype=np.float64)
    out[0::2] = np.sin(ang)
    out[1::2] = np.cos(ang)
    return out


def time_embed_table(T: int, dim: int) -> np.ndarray:
    """Rows t = 0..T of time_embed: the per-run constant table the kernels index."""
    return np.stack([time_embed(t, T, dim) for t in range(T + 1)])


@dataclass
class Layer:
    w: np.ndarray  # (fan_in, fan_out), row-major
    b: np.ndarray  # (fan_out,)


@dataclass
class PredictorWeights:
    """The reference MLP (predictor.py:68-105), device-resident on first use."""

    layers: list[Layer]
    activation: str
    ballast: int = field(default=1)

    @property
    def data_dim(self) -> int:
        return self.layers[-1].w.shape[1]

    @property
    def embed_dim(self) -> int:
        return self.layers[0].w.shape[0] - self.data_dim

    def validate(self) -> None:
        if not self.layers:
            raise ConfigError("need at least one layer")
        if len(self.layers) > 16:
            raise ConfigError("at most 16 layers")
        if self.activation not in _ACT_ID:
            raise ConfigError(f"unknown activation {self.activation!r}")
        for i, layer in enumerate(self.layers):
            if layer.w.shape[1] != layer.b.shape[0]:
                raise ConfigError(f"layer {i}: bias length != fan_out")
            if i > 0 and self.layers[i - 1].w.shape[1] != layer.w.shape[0]:
                raise ConfigError(f"layer {i}: fan_in does not chain from layer {i - 1}")
            if not (np.isfinite(layer.w).all() and np.isfinite(layer.b).all()):
                raise ConfigError(f"layer {i}: non-finite parameters")
        ed = self.embed_dim
        if ed < 2 or ed % 2 != 0:
            raise ConfigError(f"implied embedding dim {ed} must be even and >= 2")

    # ---- engine protocol
    state_dtype_code = _lib.PS_F64
    max_batch = _lib.PS_MAX_CYCLE

    def __getstate__(self):  # picklable like the reference (worker.py:313-319)
        d = dict(self.__dict__)
        d.pop("_dev", None)
        return d

    def _device(self, T: int):
        import torch

        dev = self.__dict__.get("_dev")
        if dev is None:
            lib = _lib.load(require_gpu=True)
            ws = [torch.as_tensor(np.ascontiguousarray(l.w), dtype=torch.float64, device="cuda")
                  for l in self.layers]
            bs = [torch.as_tensor(np.ascontiguousarray(l.b), dtype=torch.float64, device="cuda")
                  for l in self.layers]
            desc = _lib.ps_mlp()
            desc.n_layers = len(self.layers)
            desc.activation = _ACT_ID[self.activation]
            desc.data_dim = self.data_dim
            desc.embed_dim = self.embed_dim
            desc.dims[0] = self.layers[0].w.shape[0]
            for i, l in enumerate(self.layers):
                desc.dims[i + 1] = l.w.shape[1]
                desc.W[i] = _lib.ptr(ws[i])
                desc.b[i] = _lib.ptr(bs[i])
            nbytes = lib.ps_mlp_workspace_bytes(desc, self.max_batch)
            work = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
            dev = {"ws": ws, "bs": bs, "desc": desc, "work": work, "temb": {}}
            self.__dict__["_dev"] = dev
        if T not in dev["temb"]:
            import torch

            dev["temb"][T] = torch.as_tensor(time_embed_table(T, self.embed_dim),
                                             dtype=torch.float64, device="cuda")
        dev["desc"].temb_table = _lib.ptr(dev["temb"][T])
        return dev

    def kernels_per_forward(self, B: int = 1) -> int:
        return 2 * len(self.layers)  # split-K partial + finish per layer

    def forward_device(self, x, ts, T: int, out, stream=None) -> None:
        """x, out: CUDA float64 [B, data_dim]; ts: B step indices. Async."""
        lib = _lib.load()
        # one forward is issued atomically: callers on several threads share
        # the workspace (run_loopback-style use, worker.py:257-266); stream
        # order then keeps each forward's kernels together
        with _ISSUE_LOCK:
            dev = self._device(T)
            B = len(ts)
            tsa = (_lib.C.c_int32 * B)(*ts)
            _lib.check(lib.ps_mlp_forward(dev["desc"], _lib.ptr(x), tsa, B, _lib.ptr(out),
                                          _lib.ptr(dev["work"]), _lib.stream_ptr(stream)),
                       "mlp_forward")


@dataclass
class TrainConfig:
    """Only the architecture/seed fields matter for inference (predictor.py:169-199)."""

    dataset: str = "gauss8"
    data_dim: int = 2
    hidden: tuple[int, ...] = (64, 64)
    embed_dim: int = 16
    learning_rate: float = 1e-3
    adam_beta1: float = 0.9
    adam_beta2: float = 0.999
    adam_eps: float = 1e-8
    batch_size: int = 64
    iterations: int = 3000
    seed: int = 42
    activation: str = ACT_SILU
    dataset_size: int = 4000
    log_interval: int = 100
    objective: str = "noise"

    def validate(self) -> None:
        if self.data_dim < 1:
            raise ConfigError("counts must be positive")
        if self.embed_dim < 2 or self.embed_dim % 2 != 0:
            raise ConfigError("embed_dim must be even and >= 2")
        if self.activation not in _ACT_ID:
            raise ConfigError(f"unknown activation {self.activation!r}")


def init_weights(cfg: TrainConfig) -> PredictorWeights:
    """Xavier-uniform, zero bias, stream (WEIGHT_INIT<<32)|layer (predictor.py:202-215).

    Drawn on the GPU (``ps_rng_xavier``), bit-identical to the reference.
    """
    import torch

    cfg.validate()
    lib = _lib.load(require_gpu=True)
    dims = [cfg.data_dim + cfg.embed_dim, *cfg.hidden, cfg.data_dim]
    layers = []
    for i in range(len(dims) - 1):
        fi, fo = dims[i], dims[i + 1]
        lim = math.sqrt(6.0 / (fi + fo))
        w = torch.empty(fi * fo, dtype=torch.float64, device="cuda")
        _lib.check(lib.ps_rng_xavier(_lib.ptr(w), fi * fo, cfg.seed,
                                     stream_id(PURPOSE_WEIGHT_INIT, i), lim, _lib.PS_F64,
                                     _lib.stream_ptr()), "init_weights")
        layers.append(Layer(w.view(fi, fo).cpu().numpy(), np.zeros(fo)))
    weights = PredictorWeights(layers, cfg.activation)
    weights.validate()
    return weights


def forward(w, x, t: int, T: int) -> Vector:
    """Predict eps for one 1-D float64 vector on the GPU (predictor.py:133-150)."""
    return forward_batch(w, [x], [t], T)[0]


def forward_batch(w, xs, ts, T: int) -> list[Vector]:
    """Element i is forward(w, xs[i], ts[i], T), bitwise (predictor.py:153-166)."""
    import torch

    if len(xs) != len(ts):
        raise DimensionError(f"batch length mismatch: {len(xs)} inputs vs {len(ts)} steps")
    if not xs:
        raise DimensionError("batch must be nonempty")
    n = w.data_dim
    vs = [as_vector(x) for x in xs]
    for v in vs:
        if len(v) != n:
            raise DimensionError(f"input length {len(v)} != data_dim {n}")
    for t in ts:
        if not 0 <= t <= T:
            raise ParameterError(f"step index {t} outside [0, {T}]")
    tdt = torch.float64 if w.state_dtype_code == _lib.PS_F64 else torch.float32
    out_all = []
    for i in range(0, len(vs), w.max_batch):
        chunk = vs[i:i + w.max_batch]
        xd = torch.as_tensor(np.stack(chunk), dtype=tdt, device="cuda")
        od = torch.empty_like(xd)
        w.forward_device(xd, list(ts[i:i + w.max_batch]), T, od)
        out_all.extend(np.array(r, dtype=np.float64) for r in od.cpu().numpy())
    return out_all
