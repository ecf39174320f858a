"""Noise schedule and the reverse step — the drop-in for
pkg/src/parastep/schedule.py.

The tables (T entries) are built on the host with the reference's exact
numpy recipe (linspace / cumprod, schedule.py:42-86): they are the run's
control data, turned into per-step kernel arguments (``step_coeffs``). The
step itself runs on the GPU (``ps_sched_cycle`` / ``ps_sched_step_z``) in
fp64 registers with every operation rounded as numpy rounds it, so given the
same inputs and noise it is bit-identical to ``ddpm_step``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import DimensionError, ParameterError
from .numerics import PURPOSE_STEP, Vector, as_vector, stream_id

SIGMA_POSTERIOR = "posterior"
SIGMA_ZERO = "zero"


@dataclass(frozen=True)
class NoiseSchedule:
    T: int
    beta: Vector
    alpha: Vector
    alpha_bar: Vector
    sigma: Vector
    sigma_mode: str

    def check_step(self, t: int) -> None:
        if not 1 <= t <= self.T:
            raise ParameterError(f"step index {t} outside [1, {self.T}]")


def make_linear_schedule(T: int, beta_start: float, beta_end: float,
                         sigma_mode: str = SIGMA_POSTERIOR) -> NoiseSchedule:
    """schedule.py:42-71."""
    if T < 2:
        raise ParameterError(f"need T >= 2, got {T}")
    if not (0.0 < beta_start <= beta_end < 1.0):
        raise ParameterError(
            f"need 0 < beta_start <= beta_end < 1, got ({beta_start}, {beta_end})")
    if sigma_mode not in (SIGMA_POSTERIOR, SIGMA_ZERO):
        raise ParameterError(f"unknown sigma mode {sigma_mode!r}")
    beta = np.linspace(beta_start, beta_end, T)
    alpha = 1.0 - beta
    alpha_bar = np.cumprod(alpha)
    if sigma_mode == SIGMA_ZERO:
        sigma = np.zeros(T)
    else:
        prev = np.concatenate(([1.0], alpha_bar[:-1]))
        sigma = np.sqrt(beta * (1.0 - prev) / (1.0 - alpha_bar))
    return NoiseSchedule(T, beta, alpha, alpha_bar, sigma, sigma_mode)


def default_beta_range(T: int) -> tuple[float, float]:
    """The 1e-4..0.02 ramp rescaled to T steps (schedule.py:74-81)."""
    scale = 1000.0 / T
    return min(1e-4 * scale, 0.98), min(0.02 * scale, 0.98)


def make_default_schedule(T: int, sigma_mode: str = SIGMA_POSTERIOR) -> NoiseSchedule:
    lo, hi = default_beta_range(T)
    return make_linear_schedule(T, lo, hi, sigma_mode)


def step_coeffs(sched: NoiseSchedule, t: int) -> _lib.ps_step:
    """Per-step kernel arguments, computed like posterior_mean (schedule.py:111-114)."""
    sched.check_step(t)
    a = float(sched.alpha[t - 1])
    ab = float(sched.alpha_bar[t - 1])
    s = _lib.ps_step()
    s.c = (1.0 - a) / math.sqrt(1.0 - ab)
    s.sqrt_a = math.sqrt(a)
    s.sigma = float(sched.sigma[t - 1])
    s.t = t
    s.noisy = 0 if (t == 1 or sched.sigma_mode == SIGMA_ZERO) else 1
    return s


def _to_device(v, dtype):
    import torch

    if isinstance(v, torch.Tensor):
        return v.to(device="cuda", dtype=dtype).contiguous()
    return torch.as_tensor(as_vector(v), dtype=dtype, device="cuda")


def ddpm_step(x_t, t: int, eps, sched: NoiseSchedule, step_noise) -> Vector:
    """One reverse step on the GPU (schedule.py:117-131); numpy in, numpy out.

    ``step_noise`` is the shared per-step vector as in the reference; it is
    ignored when the step is deterministic (t == 1 or zero mode).
    """
    import torch

    lib = _lib.load(require_gpu=True)
    x = as_vector(x_t)
    e = as_vector(eps)
    if len(x) != len(e):
        raise DimensionError(f"length mismatch: {len(x)} vs {len(e)}")
    s = step_coeffs(sched, t)
    xd = _to_device(x, torch.float64)
    ed = _to_device(e, torch.float64)
    zd = None
    if s.noisy:
        z = as_vector(step_noise)
        if len(z) != len(x):
            raise DimensionError(f"length mismatch: {len(x)} vs {len(z)}")
        zd = _to_device(z, torch.float64)
    out = torch.empty_like(xd)
    _lib.check(lib.ps_sched_step_z(_lib.ptr(xd), _lib.ptr(ed), _lib.ptr(zd), _lib.ptr(out),
                                   len(x), _lib.PS_F64, s, _lib.stream_ptr()), "ddpm_step")
    return out.cpu().numpy()


def posterior_mean(x_t, t: int, eps, sched: NoiseSchedule) -> Vector:
    """schedule.py:102-114 (the noiseless part of the step), on the GPU."""
    import dataclasses

    det = dataclasses.replace(sched, sigma_mode=SIGMA_ZERO)
    return ddpm_step(x_t, t, eps, det, None)


def step_stream(t: int) -> int:
    return stream_id(PURPOSE_STEP, t)
