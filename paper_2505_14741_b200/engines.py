"""Sampling strategies on the GPU — the drop-in for pkg/src/parastep/engines.py.

Same names, signatures, config validation and exceptions as the reference:
``RunConfig``, ``run_strategy``, ``denoise_sequential``,
``denoise_direct_reuse``, ``denoise_parastep_emulated``, ``denoise_batchstep``,
``denoise_dynamic``, ``initial_state``, ``step_noise``, ``Trajectory``.

Device formulation (the B200 design). A ParaStep run is the
reference's cycle runner (engines.py:299-337), which its own tests pin
bit-for-bit to the Algorithm-1 emulation (tests/test_engines.py:294-303):

    warm-up:   x <- step(x, forward(x, t))                 (sequential)
    cycle c:   lane j: x_j = roll^j(x_sync, cache_j)      (ps_sched_cycle roll)
               eps_j = forward(x_j, t_j)                   (predictor)
               x_sync <- step^c(x_sync, eps_0..eps_{c-1})  (ps_sched_cycle apply)

The apply of cycle c and the roll of cycle c+1 are ONE launch: the chain
stays in fp64 registers and the just-read eps_j are the next lane caches.
Step noise z_t is generated in-register from the seed (never stored). eps is
written straight into the trajectory table [T, n] (row k = step T-k), so the
records cost no copies. ``DeviceSampler`` owns the buffers and can capture
the whole run into one CUDA graph (replayed per seed).

The state dtype follows the predictor: fp64 for the reference MLP, fp32 for
the DiT predictors (the chain arithmetic itself is always fp64 in registers).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import ConfigError, DegenerateReferenceError, DimensionError
from .numerics import PURPOSE_INIT, PURPOSE_STEP, Vector, mse, rel_mae, stream_id
from .schedule import NoiseSchedule, step_coeffs

STRATEGY_SEQUENTIAL = "sequential"
STRATEGY_DIRECT_REUSE = "direct_reuse"
STRATEGY_PARASTEP = "parastep"
STRATEGY_BATCHSTEP = "batchstep"
STRATEGY_DYNAMIC = "dynamic"
STRATEGIES = (STRATEGY_SEQUENTIAL, STRATEGY_DIRECT_REUSE, STRATEGY_PARASTEP, STRATEGY_BATCHSTEP,
              STRATEGY_DYNAMIC)

SRC_LOCAL_FRESH = "local_fresh"
SRC_REMOTE_FRESH = "remote_fresh"
SRC_REUSE = "reuse"


def warmup_from_ratio(ratio: float, steps: int) -> int:
    """round(ratio * steps) (engines.py:62-66)."""
    if not 0.0 <= ratio <= 1.0:
        raise ConfigError(f"warm-up ratio must be in [0, 1], got {ratio}")
    return int(round(ratio * steps))


@dataclass
class RunConfig:
    """engines.py:69-112 (identical fields and invariants)."""

    steps: int
    warmup: int = 0
    strategy: str = STRATEGY_SEQUENTIAL
    degree: int = 1
    schedule_override: list[int] | None = None
    seed: int = 0
    data_dim: int = 2

    def validate(self) -> None:
        if self.steps < 1:
            raise ConfigError(f"steps must be >= 1, got {self.steps}")
        if not 0 <= self.warmup <= self.steps:
            raise ConfigError(f"warmup must be in [0, {self.steps}], got {self.warmup}")
        if self.degree < 1:
            raise ConfigError(f"degree must be >= 1, got {self.degree}")
        if self.data_dim < 1:
            raise ConfigError(f"data_dim must be >= 1, got {self.data_dim}")
        if self.strategy not in STRATEGIES:
            raise ConfigError(f"unknown strategy {self.strategy!r}")
        needs_cache = self.strategy in (STRATEGY_PARASTEP, STRATEGY_BATCHSTEP)
        if needs_cache and self.degree > 1 and self.warmup < 1:
            raise ConfigError("degree > 1 requires warmup >= 1: the noise cache is only "
                              "populated during warm-up or master steps")
        if self.strategy == STRATEGY_DYNAMIC:
            sched = self.schedule_override
            if sched is None:
                raise ConfigError("dynamic strategy requires schedule_override")
            if not all(isinstance(c, int) and c >= 1 for c in sched):
                raise ConfigError("cycle lengths must be integers >= 1")
            if sum(sched) != self.steps - self.warmup:
                raise ConfigError(f"cycle lengths sum to {sum(sched)}, expected "
                                  f"steps - warmup = {self.steps - self.warmup}")
            if any(c > 1 for c in sched) and self.warmup < 1:
                raise ConfigError("cycle lengths > 1 require warmup >= 1")
        elif self.schedule_override is not None:
            raise ConfigError("schedule_override is only valid for the dynamic strategy")


@dataclass
class StepRecord:
    t: int
    x: Vector
    eps: Vector
    fresh: bool


@dataclass
class Trajectory:
    records: list[StepRecord]
    x0: Vector
    batch_calls: int = 0

    @property
    def steps(self) -> int:
        return len(self.records)

    @property
    def fresh_calls(self) -> int:
        return sum(1 for r in self.records if r.fresh)

    def bitwise_equal(self, other: "Trajectory") -> bool:
        if len(self.records) != len(other.records):
            return False
        for a, b in zip(self.records, other.records):
            if a.t != b.t or a.fresh != b.fresh:
                return False
            if not (np.array_equal(a.x, b.x) and np.array_equal(a.eps, b.eps)):
                return False
        return np.array_equal(self.x0, other.x0)


@dataclass
class HistoryStep:
    t: int
    x_before: Vector
    eps: Vector
    source: str
    x_after: Vector


@dataclass
class VirtualWorkerState:
    rank: int
    x: Vector
    eps_cache: Vector | None = None
    cache_step: int | None = None
    history: list[HistoryStep] = field(default_factory=list)

    @property
    def local_fresh_calls(self) -> int:
        return sum(1 for h in self.history if h.source == SRC_LOCAL_FRESH)


def _torch_dtype(w):
    import torch

    return torch.float64 if w.state_dtype_code == _lib.PS_F64 else torch.float32


def initial_state(cfg: RunConfig) -> Vector:
    """x_T from stream (INIT<<32)|0 (engines.py:172-174), drawn on the GPU."""
    from .numerics import draw_normal

    return draw_normal(cfg.seed, stream_id(PURPOSE_INIT, 0), cfg.data_dim)


def step_noise(cfg: RunConfig, t: int) -> Vector:
    """z_t from stream (STEP<<32)|t (engines.py:177-179), drawn on the GPU."""
    from .numerics import draw_normal

    return draw_normal(cfg.seed, stream_id(PURPOSE_STEP, t), cfg.data_dim)


def _check(w, sched: NoiseSchedule, cfg: RunConfig, strategy: str | None) -> None:
    cfg.validate()
    if strategy is not None and cfg.strategy != strategy:
        raise ConfigError(f"config strategy is {cfg.strategy!r}, engine expects {strategy!r}")
    if cfg.steps != sched.T:
        raise ConfigError(f"config steps {cfg.steps} != schedule length {sched.T}")
    if cfg.data_dim != w.data_dim:
        raise ConfigError(f"config data_dim {cfg.data_dim} != predictor data_dim {w.data_dim}")


def plan_cycles(cfg: RunConfig) -> list[list[int]]:
    """Post-warm-up steps (descending t) chunked into cycles (engines.py:280-296)."""
    ts = list(range(cfg.steps - cfg.warmup, 0, -1))
    if cfg.strategy == STRATEGY_DYNAMIC:
        lengths = list(cfg.schedule_override)
    else:
        lengths, left = [], len(ts)
        while left > 0:
            lengths.append(min(cfg.degree, left))
            left -= lengths[-1]
    out, pos = [], 0
    for c in lengths:
        out.append(ts[pos:pos + c])
        pos += c
    return out


def _int64_of(seed: int) -> int:
    seed &= 0xFFFFFFFFFFFFFFFF
    return seed - (1 << 64) if seed >= (1 << 63) else seed


class DeviceSampler:
    """Buffers + launch sequence of one run shape; replayable per seed.

    ``run(seed)`` issues the whole denoise on the current stream (no host
    sync); with ``graph=True`` the sequence is captured once into a CUDA
    graph and replayed. ``trajectory()`` copies the records to host.
    """

    def __init__(self, w, sched: NoiseSchedule, cfg: RunConfig, record: bool = True,
                 batched: bool | None = None, external_init: bool = False,
                 condition_table: bool = True):
        import torch

        _check(w, sched, cfg, None)
        if cfg.strategy == STRATEGY_DYNAMIC and max(cfg.schedule_override) > _lib.PS_MAX_CYCLE:
            raise ConfigError(f"cycle length > {_lib.PS_MAX_CYCLE} unsupported on device")
        if cfg.strategy in (STRATEGY_PARASTEP, STRATEGY_BATCHSTEP) and \
                cfg.degree > _lib.PS_MAX_CYCLE:
            raise ConfigError(f"degree > {_lib.PS_MAX_CYCLE} unsupported on device")
        self.lib = _lib.load(require_gpu=True)
        self.w, self.sched, self.cfg = w, sched, cfg
        self.record = record
        self.n = cfg.data_dim
        self.T = cfg.steps
        self.dtype_code = w.state_dtype_code
        tdt = _torch_dtype(w)
        if batched is None:
            batched = cfg.strategy == STRATEGY_BATCHSTEP
        self.batched = batched
        cyc = plan_cycles(cfg) if cfg.strategy in (STRATEGY_PARASTEP, STRATEGY_BATCHSTEP,
                                                   STRATEGY_DYNAMIC) else []
        self.cycles = cyc
        dmax = max([len(c) for c in cyc] + [1])
        self.seed_buf = torch.zeros(1, dtype=torch.int64, device="cuda")
        self.lanes = torch.zeros((dmax, self.n), dtype=tdt, device="cuda")
        self.eps = torch.zeros((self.T, self.n), dtype=tdt, device="cuda")
        self.rec_x = torch.zeros((self.T, self.n), dtype=tdt, device="cuda") if record else None
        self.src_row = list(range(self.T))  # eps row consumed at step index k
        self.fresh = [True] * self.T
        self.batch_calls = 0
        self.forward_calls = 0
        self.graph = None
        self.external_init = external_init
        self.launches = 0  # kernels issued by one run (counted at issue time)
        self._steps = {t: step_coeffs(sched, t) for t in range(1, self.T + 1)}
        # batched per-run conditioning (DiT): the table is filled at the start
        # of every run; off = each forward conditions itself (same bits)
        self.condition_table = condition_table and hasattr(w, "prepare_conditioning")
        if self.condition_table:
            w.reserve_conditioning(self.T)

    # ------------------------------------------------------------ launches
    def _k(self, t: int) -> int:
        return self.T - t

    def _row(self, buf, k):
        return _lib.ptr(buf) + k * self.n * buf.element_size()

    def _cycle(self, apply_ts, apply_rows, roll_ts=(), lane_hi=0, lane_cache_rows=None,
               lane_lo=1, x_in=None, lane_ptrs=None):
        st = _lib.stream_ptr()
        na = len(apply_ts)
        A = _lib.step_array([self._steps[t] for t in apply_ts])
        E = _lib.ptr_array([self._row(self.eps, r) for r in apply_rows])
        R = _lib.ptr_array([self._row(self.rec_x, self._k(t)) if self.record else 0
                            for t in apply_ts])
        roll = _lib.step_array([self._steps[t] for t in roll_ts])
        caches = [0] * _lib.PS_MAX_CYCLE
        outs = [0] * _lib.PS_MAX_CYCLE
        for j in range(max(1, lane_lo), lane_hi):
            caches[j] = self._row(self.eps, lane_cache_rows[j])
            outs[j] = lane_ptrs[j] if lane_ptrs else self._row(self.lanes, j)
        x0 = x_in if x_in is not None else self._row(self.lanes, 0)
        _lib.check(self.lib.ps_sched_cycle(
            x0, x0, self.n, self.dtype_code, _lib.ptr(self.seed_buf), na, A, E, R,
            lane_lo, lane_hi, roll, _lib.ptr_array(caches), _lib.ptr_array(outs), st),
            "sched_cycle")
        self.launches += 1

    def _forward(self, lane_lo: int, lane_hi: int, ts: list[int], row0: int):
        x = self.lanes[lane_lo:lane_hi]
        out = self.eps[row0:row0 + (lane_hi - lane_lo)]
        self.w.forward_device(x, ts, self.T, out)
        self.forward_calls += 1
        self.launches += self.w.kernels_per_forward(len(ts))

    def _init_x(self):
        if self.external_init:
            return  # x_T was copied into lanes[0] by run(x_init=...)
        self.launches += 1
        _lib.check(self.lib.ps_rng_normal_dev(
            self._row(self.lanes, 0), self.n, _lib.ptr(self.seed_buf),
            stream_id(PURPOSE_INIT, 0), 0, self.dtype_code, _lib.stream_ptr()), "initial_state")

    def _launch(self):
        cfg = self.cfg
        self.forward_calls = 0
        self.launches = 0
        self._init_x()
        T = self.T
        if self.condition_table:
            # the t-only conditioning of every step of this run, batched
            # (16 steps per launch) instead of recomputed inside each forward
            self.launches += self.w.prepare_conditioning(T)
        if cfg.strategy == STRATEGY_SEQUENTIAL:
            for t in range(T, 0, -1):
                k = self._k(t)
                self._forward(0, 1, [t], k)
                self._cycle([t], [k])
            return
        if cfg.strategy == STRATEGY_DIRECT_REUSE:
            last, since = None, 0
            for t in range(T, 0, -1):
                k = self._k(t)
                if (T - t) < cfg.warmup:
                    fresh = True
                else:
                    fresh = since % cfg.degree == 0
                    since += 1
                if fresh:
                    self._forward(0, 1, [t], k)
                    last = k
                self.src_row[k] = last
                self.fresh[k] = fresh
                self._cycle([t], [last])
            return
        # cycle strategies (parastep / batchstep / dynamic)
        cycles = self.cycles
        lane_cache = {}
        warm_ts = list(range(T, T - cfg.warmup, -1))
        for i, t in enumerate(warm_ts):
            k = self._k(t)
            self._forward(0, 1, [t], k)
            last = i == len(warm_ts) - 1
            if last and cycles and len(cycles[0]) > 1:
                c0 = cycles[0]
                rows = {j: k for j in range(len(c0))}
                self._cycle([t], [k], roll_ts=c0[:-1], lane_hi=len(c0), lane_cache_rows=rows)
            else:
                self._cycle([t], [k])
        warm_row = self._k(warm_ts[-1]) if warm_ts else None
        nb = 0
        for ci, cyc in enumerate(cycles):
            c = len(cyc)
            k0 = self._k(cyc[0])
            if self.batched:
                self._forward(0, c, list(cyc), k0)
            else:
                for j, tj in enumerate(cyc):
                    self._forward(j, j + 1, [tj], k0 + j)
            nb += 1
            for j in range(c):
                self.fresh[k0 + j] = j == 0
                lane_cache[j] = k0 + j
            nxt = cycles[ci + 1] if ci + 1 < len(cycles) else None
            if nxt is not None and len(nxt) > 1:
                rows = {j: lane_cache.get(j, warm_row) for j in range(len(nxt))}
                self._cycle(list(cyc), [k0 + j for j in range(c)], roll_ts=nxt[:-1],
                            lane_hi=len(nxt), lane_cache_rows=rows)
            else:
                self._cycle(list(cyc), [k0 + j for j in range(c)])
        self.batch_calls = nb if self.batched else 0

    def run(self, seed: int, graph: bool = False, x_init=None) -> None:
        """Issue one full denoise for `seed` on the current stream (async).

        With ``external_init`` the caller provides x_T (``x_init``: a host
        tensor, ideally pinned, or a device tensor) instead of the in-kernel
        draw; it is copied into the state buffer on the stream first.
        """
        import torch

        self.seed_buf.fill_(_int64_of(seed))
        if self.external_init:
            if x_init is None:
                raise ConfigError("external_init sampler needs x_init")
            self.lanes[0].copy_(torch.as_tensor(x_init).reshape(-1), non_blocking=True)
        if not graph:
            self._launch()
            return
        if self.graph is None:
            self._launch()  # eager warm-up: first-launch attribute setup off the capture
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                with torch.cuda.graph(g, stream=s):
                    self._launch()
            torch.cuda.current_stream().wait_stream(s)
            self.graph = g
        self.graph.replay()

    @property
    def x0_device(self):
        return self.lanes[0]

    def sample(self, seed: int, x_init=None, graph: bool = True) -> Trajectory:
        """Public one-call API: (optional host x_T) -> full Trajectory on host."""
        self.run(seed, graph=graph, x_init=x_init)
        return self.trajectory()

    def save_trajectory_binary(self, path) -> None:
        """The reference's binary trajectory file of the last run, packed on device."""
        from .trajectory_io import pack_device

        with open(path, "wb") as fh:
            fh.write(pack_device(self))

    def trajectory(self) -> Trajectory:
        """Copy the run's records to host (reference Trajectory of float64 vectors)."""
        import torch

        torch.cuda.current_stream().synchronize()
        eps = self.eps.to(torch.float64).cpu().numpy()
        x0 = self.lanes[0].to(torch.float64).cpu().numpy().copy()
        xs = self.rec_x.to(torch.float64).cpu().numpy() if self.record else None
        recs = []
        for k in range(self.T):
            t = self.T - k
            x = xs[k].copy() if xs is not None else None
            recs.append(StepRecord(t, x, eps[self.src_row[k]].copy(), self.fresh[k]))
        return Trajectory(recs, x0, self.batch_calls)


def _run(w, sched, cfg, strategy, batched=None) -> Trajectory:
    _check(w, sched, cfg, strategy)
    s = DeviceSampler(w, sched, cfg, record=True, batched=batched)
    s.run(cfg.seed)
    return s.trajectory()


def denoise_sequential(w, sched: NoiseSchedule, cfg: RunConfig) -> Trajectory:
    """engines.py:196-205 on the GPU."""
    return _run(w, sched, cfg, STRATEGY_SEQUENTIAL)


def denoise_direct_reuse(w, sched: NoiseSchedule, cfg: RunConfig) -> Trajectory:
    """engines.py:208-229 on the GPU."""
    return _run(w, sched, cfg, STRATEGY_DIRECT_REUSE)


def denoise_batchstep(w, sched: NoiseSchedule, cfg: RunConfig) -> Trajectory:
    """engines.py:340-343: each cycle's predictions in one batched forward."""
    return _run(w, sched, cfg, STRATEGY_BATCHSTEP, batched=True)


def denoise_dynamic(w, sched: NoiseSchedule, cfg: RunConfig) -> Trajectory:
    """engines.py:346-349: cycle lengths from cfg.schedule_override."""
    return _run(w, sched, cfg, STRATEGY_DYNAMIC, batched=False)


def denoise_parastep_lanes(w, sched: NoiseSchedule, cfg: RunConfig) -> Trajectory:
    """ParaStep rank-0 trajectory via the fused cycle formulation, one forward
    per virtual rank (what each of the d devices computes)."""
    return _run(w, sched, cfg, STRATEGY_PARASTEP, batched=False)


def denoise_parastep_emulated(w, sched: NoiseSchedule, cfg: RunConfig):
    """Algorithm 1 with p lockstep virtual ranks and per-rank histories
    (engines.py:232-277), literally: one master forward per step, p scheduler
    steps, broadcast overwrite at round p-1. Diagnostic path (per-rank state
    is materialised); ``run_strategy`` uses the fused cycle form, which the
    tests pin bitwise to this one."""
    import torch

    _check(w, sched, cfg, STRATEGY_PARASTEP)
    lib = _lib.load(require_gpu=True)
    p, n, T = cfg.degree, cfg.data_dim, cfg.steps
    tdt = _torch_dtype(w)
    s = DeviceSampler(w, sched, RunConfig(steps=T, data_dim=n, seed=cfg.seed), record=False)
    s.seed_buf.fill_(_int64_of(cfg.seed))
    s._init_x()
    xs = s.lanes[0:1].repeat(p, 1)  # rank states
    hist_b = torch.zeros((p, T, n), dtype=tdt, device="cuda")
    hist_a = torch.zeros((p, T, n), dtype=tdt, device="cuda")
    eps = s.eps
    cache = [None] * p
    srcs = [[] for _ in range(p)]
    eps_rows = [[] for _ in range(p)]
    rec_fresh = []
    rnd = 0
    for t in range(T, 0, -1):
        k = T - t
        warm = (T - t) < cfg.warmup
        m = 0 if warm else rnd
        w.forward_device(xs[m:m + 1], [t], T, eps[k:k + 1])
        for r in range(p):
            if warm or r == m:
                row, src = k, SRC_LOCAL_FRESH
                cache[r] = k
            elif r == 0:
                row, src = k, SRC_REMOTE_FRESH
            else:
                row, src = cache[r], SRC_REUSE
            xr = s._row(xs, r)
            hb = _lib.ptr(hist_b) + ((r * T + k) * n) * hist_b.element_size()
            _lib.check(lib.ps_sched_cycle(
                xr, xr, n, s.dtype_code, _lib.ptr(s.seed_buf), 1,
                _lib.step_array([s._steps[t]]), _lib.ptr_array([s._row(eps, row)]),
                _lib.ptr_array([hb]), 0, 0, _lib.step_array([]), _lib.ptr_array([]),
                _lib.ptr_array([]), _lib.stream_ptr()), "sched_cycle")
            srcs[r].append(src)
            eps_rows[r].append(row)
        rec_fresh.append(warm or m == 0)
        if not warm and rnd == p - 1:
            xs[1:] = xs[0:1]
        hist_a[:, k] = xs
        if not warm:
            rnd = (rnd + 1) % p
    torch.cuda.synchronize()
    hb = hist_b.to(torch.float64).cpu().numpy()
    ha = hist_a.to(torch.float64).cpu().numpy()
    e = eps.to(torch.float64).cpu().numpy()
    xf = xs.to(torch.float64).cpu().numpy()
    workers = []
    for r in range(p):
        ws = VirtualWorkerState(r, xf[r].copy())
        for k in range(T):
            ws.history.append(HistoryStep(T - k, hb[r, k].copy(), e[eps_rows[r][k]].copy(),
                                          srcs[r][k], ha[r, k].copy()))
        if cache[r] is not None:
            ws.eps_cache = e[cache[r]].copy()
            ws.cache_step = T - cache[r]
        workers.append(ws)
    recs = [StepRecord(T - k, hb[0, k].copy(), e[k].copy(), rec_fresh[k]) for k in range(T)]
    return Trajectory(recs, xf[0].copy()), workers


def run_strategy(w, sched: NoiseSchedule, cfg: RunConfig) -> Trajectory:
    """Dispatch on cfg.strategy (engines.py:352-364)."""
    engine = {
        STRATEGY_SEQUENTIAL: denoise_sequential,
        STRATEGY_DIRECT_REUSE: denoise_direct_reuse,
        STRATEGY_PARASTEP: denoise_parastep_lanes,
        STRATEGY_BATCHSTEP: denoise_batchstep,
        STRATEGY_DYNAMIC: denoise_dynamic,
    }
    if cfg.strategy not in engine:
        raise ConfigError(f"unknown strategy {cfg.strategy!r}")
    return engine[cfg.strategy](w, sched, cfg)


# ---------------------------------------------------------------- diagnostics
def generate_threshold_schedule(reference: Trajectory, tau: float, max_len: int,
                                warmup: int = 0) -> list[int]:
    """Greedy cycle lengths from a sequential run (engines.py:367-401)."""
    if tau < 0:
        raise ConfigError(f"tau must be >= 0, got {tau}")
    if max_len < 1:
        raise ConfigError(f"max_len must be >= 1, got {max_len}")
    T = len(reference.records)
    if not 0 <= warmup <= T:
        raise ConfigError(f"warmup must be in [0, {T}], got {warmup}")
    by_t = {r.t: r.eps for r in reference.records}

    def change(u: int) -> float:
        try:
            return rel_mae(by_t[u], by_t[u + 1])
        except DegenerateReferenceError:
            return float("inf")

    steps = list(range(T - warmup, 0, -1))
    out, i = [], 0
    while i < len(steps):
        n = 1
        while n < max_len and i + n < len(steps) and change(steps[i + n]) < tau:
            n += 1
        out.append(n)
        i += n
    return out


@dataclass
class DiffRow:
    t: int
    rel_mae_x: float
    rel_mae_eps: float
    mse_x: float
    mse_eps: float


@dataclass
class AdjacentRow:
    t: int
    rel_mae_x: float
    rel_mae_eps: float


def _adjacent_series(traj: Trajectory) -> list[AdjacentRow]:
    """rel_mae(value_t, value_{t+1}) of consecutive records (engines.py:422-428)."""
    return [AdjacentRow(cur.t, rel_mae(cur.x, prev.x), rel_mae(cur.eps, prev.eps))
            for prev, cur in zip(traj.records, traj.records[1:])]


@dataclass
class DiffReport:
    """engines.py:431-443: per-step rows, final x0 rel-MAE / MSE, and the
    adjacent-step self-similarity series of both trajectories (T-1 rows)."""

    rows: list[DiffRow]
    final_rel_mae: float
    final_mse: float
    adjacent_a: list[AdjacentRow]
    adjacent_b: list[AdjacentRow]

    def to_csv(self) -> str:
        lines = ["step,rel_mae_x,rel_mae_eps,mse_x,mse_eps"]
        for r in self.rows:
            lines.append(f"{r.t},{r.rel_mae_x!r},{r.rel_mae_eps!r},{r.mse_x!r},{r.mse_eps!r}")
        return "\n".join(lines) + "\n"


def compare_trajectories(a: Trajectory, b: Trajectory) -> DiffReport:
    """Per-step divergence of b from reference a (engines.py:446-473)."""
    if len(a.records) != len(b.records):
        raise DimensionError(f"trajectory lengths differ: {len(a.records)} vs {len(b.records)}")
    if len(a.x0) != len(b.x0):
        raise DimensionError(f"data dims differ: {len(a.x0)} vs {len(b.x0)}")
    rows = []
    for ra, rb in zip(a.records, b.records):
        if ra.t != rb.t:
            raise DimensionError(f"step mismatch: {ra.t} vs {rb.t}")
        rows.append(DiffRow(ra.t, rel_mae(ra.x, rb.x), rel_mae(ra.eps, rb.eps), mse(ra.x, rb.x),
                            mse(ra.eps, rb.eps)))
    return DiffReport(rows, rel_mae(a.x0, b.x0), mse(a.x0, b.x0), _adjacent_series(a),
                      _adjacent_series(b))


def compare_trajectories_device(a: "DeviceSampler", b: "DeviceSampler") -> DiffReport:
    """compare_trajectories of two samplers' last runs without leaving the GPU.

    The same DiffReport as ``compare_trajectories`` (engines.py:446-473): the
    per-step rows (a = reference), the final x0 rel-MAE and MSE, and both
    adjacent-step series. All sums run on device in fp64 with a fixed
    reduction order (``ps_traj_diff``), so they agree with the host's
    left-to-right sums to rounding (~1e-15 relative).
    """
    import torch

    if a.T != b.T:
        raise DimensionError(f"trajectory lengths differ: {a.T} vs {b.T}")
    if a.n != b.n:
        raise DimensionError(f"data dims differ: {a.n} vs {b.n}")
    if not (a.record and b.record):
        raise ConfigError("both samplers need per-step x records")
    lib = _lib.load(require_gpu=True)
    T, n = a.T, a.n
    # rows: [0,T) x diff, [T,2T) eps diff, 2T x0, then the adjacent series of a
    # and b: (T-1) x rows + (T-1) eps rows each
    nrow = 2 * T + 1 + 4 * max(T - 1, 0)
    out = torch.empty((nrow, 3), dtype=torch.float64, device="cuda")
    ar = list(range(T))
    idx = torch.tensor([ar, list(a.src_row), list(b.src_row)], dtype=torch.int32, device="cuda")
    st = _lib.stream_ptr()
    ptr = _lib.ptr

    def diff(x, y, rx, ry, rows, row0, dx, dy):
        _lib.check(lib.ps_traj_diff(ptr(x), ptr(y), rx, ry, rows, n, dx, dy,
                                    ptr(out) + 3 * row0 * 8, st), "traj_diff")

    def irow(which, start):
        return ptr(idx) + (which * T + start) * 4

    diff(a.rec_x, b.rec_x, None, None, T, 0, a.dtype_code, b.dtype_code)
    diff(a.eps, b.eps, irow(1, 0), irow(2, 0), T, T, a.dtype_code, b.dtype_code)
    diff(a.x0_device, b.x0_device, None, None, 1, 2 * T, a.dtype_code, b.dtype_code)
    if T > 1:
        base = 2 * T + 1
        for s_i, (smp, which) in enumerate(((a, 1), (b, 2))):
            r0 = base + s_i * 2 * (T - 1)
            # cur = record k+1 (reference side of rel_mae), prev = record k
            diff(smp.rec_x, smp.rec_x, irow(0, 1), irow(0, 0), T - 1, r0, smp.dtype_code,
                 smp.dtype_code)
            diff(smp.eps, smp.eps, irow(which, 1), irow(which, 0), T - 1, r0 + T - 1,
                 smp.dtype_code, smp.dtype_code)
    s = out.cpu().numpy()

    def rel(row):
        if row[1] == 0.0:
            raise DegenerateReferenceError("reference vector has zero mean magnitude")
        return (row[0] / n) / (row[1] / n)

    rows = [DiffRow(T - k, rel(s[k]), rel(s[T + k]), s[k][2] / n, s[T + k][2] / n)
            for k in range(T)]
    adj = []
    for s_i in range(2):
        r0 = 2 * T + 1 + s_i * 2 * (T - 1)
        adj.append([AdjacentRow(T - (k + 1), rel(s[r0 + k]), rel(s[r0 + T - 1 + k]))
                    for k in range(T - 1)])
    return DiffReport(rows, rel(s[2 * T]), s[2 * T][2] / n, adj[0], adj[1])
