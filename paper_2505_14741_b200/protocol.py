"""Multi-GPU ParaStep: one process per GPU, one eps all-gather per round.

Replaces the reference's distributed worker (pkg/src/parastep/protocol/
worker.py:149-241: NOISE master->rank 0, SAMPLE_BCAST rank 0->all) with the
cycle form the reference's own tests pin to it (tests/test_engines.py:294-303,
test_protocol.py:44-55):

    warm-up   every rank runs the same steps redundantly (worker.py:180-185);
              the kernels are deterministic, so every rank holds the same bits
    cycle     rank r owns lane r: x_r = roll^r(x_sync, own cache)   (fused)
              eps_r = forward(x_r, t_r)
              E = all_gather(eps_0..eps_{p-1})          (NCCL over NVLink)
              x_sync = step^c(x_sync, E)  on EVERY rank  (fused apply, which
              also rolls the rank's lane for the next cycle)

The redundant deterministic apply replaces the gather-to-0 + broadcast, so
each rank sends N*s bytes and receives (p-1)*N*s per cycle. A truncated last
cycle (c < p) idles ranks >= c (worker.py module docstring).

``rank_loop`` holds the protocol logic once; it is driven by ``CudaRankOps``
(the product: C-ABI kernels + NCCL via torch.distributed) and, in the CPU
tests, by an oracle-backed ops object over gloo (tests/test_protocol_gloo.py).
"""

from __future__ import annotations

from dataclasses import dataclass, field

from . import _lib
from .engines import (
    STRATEGY_DYNAMIC,
    STRATEGY_PARASTEP,
    RunConfig,
    StepRecord,
    Trajectory,
    _check,
    _int64_of,
    plan_cycles,
)
from .errors import ConfigError, ProtocolAbortError
from .ledger import ExchangeLedger
from .numerics import PURPOSE_INIT, stream_id
from .schedule import NoiseSchedule, step_coeffs


def rank_loop(ops, T: int, warmup: int, p: int, rank: int, cycles: list[list[int]]):
    """One rank's ParaStep run over abstract ops; returns the final x handle.

    ops.init() -> x; ops.forward(x, t, slot) -> eps; ops.zeros(slot) -> eps;
    ops.allgather(eps) -> list of p eps; ops.apply_roll(x, apply_ts, eps_list,
    roll_ts, cache) -> (x, lane_x) with roll_ts == [] meaning no roll.
    ops.record(k, eps) optionally stores trajectory eps rows. Optional hooks:
    ops.stamp(tag) marks phase boundaries (forward / exchange / apply, the
    reference's WorkerTimings, worker.py:65-85) and ops.finish() closes the
    run (the peer exchange's end-of-run handshake).
    """
    stamp = getattr(ops, "stamp", None) or (lambda tag: None)
    x = ops.init()
    stamp("start")
    lane_x = None
    cache = None
    warm_ts = list(range(T, T - warmup, -1))
    for i, t in enumerate(warm_ts):
        stamp("fwd0")
        e = ops.forward(x, t, "warm")
        stamp("fwd1")
        ops.record(T - t, [e])
        nxt = cycles[0] if (i == len(warm_ts) - 1 and cycles) else None
        roll = nxt[:rank] if (nxt is not None and 1 <= rank < len(nxt)) else []
        cache = e
        x, lane_x = ops.apply_roll(x, [t], [e], roll, cache)
        stamp("apply")
    for ci, cyc in enumerate(cycles):
        c = len(cyc)
        mine = rank < c
        stamp("fwd0")
        if mine:
            e_local = ops.forward(x if rank == 0 else lane_x, cyc[rank], "lane")
        else:
            e_local = ops.zeros("lane")
        stamp("fwd1")
        gathered = ops.allgather(e_local, c)
        stamp("xchg")
        ops.record(T - cyc[0], gathered[:c])
        if mine:
            cache = ops.keep_cache(gathered[rank])
        nxt = cycles[ci + 1] if ci + 1 < len(cycles) else None
        roll = nxt[:rank] if (nxt is not None and 1 <= rank < len(nxt)) else []
        x, lane_x = ops.apply_roll(x, list(cyc), gathered[:c], roll, cache)
        stamp("apply")
    finish = getattr(ops, "finish", None)
    if finish is not None:
        finish()
    stamp("end")
    return x


@dataclass
class RankTimings:
    """Device-clock split of one rank's loop (the reference's WorkerTimings,
    worker.py:65-85): loop_start/loop_end are %globaltimer stamps (ns -> s);
    forward_s sums the predictor forwards, exchange_wait_s the time from the
    end of this rank's forward until its exchange completed (all-gather, or
    the peers' ready flags), apply_s the fused apply/roll kernels (and record
    copies)."""

    loop_start: float = 0.0
    loop_end: float = 0.0
    forward_s: float = 0.0
    exchange_wait_s: float = 0.0
    apply_s: float = 0.0

    @property
    def loop_s(self) -> float:
        return self.loop_end - self.loop_start

    @property
    def comm_s(self) -> float:
        return self.exchange_wait_s

    @staticmethod
    def from_stamps(tags: list[str], ns: list[int]) -> "RankTimings":
        """Each phase is the interval since the previous stamp: fwd0->fwd1 a
        forward, fwd1->xchg the exchange, (fwd1 | xchg)->apply the apply."""
        r = RankTimings()
        prev = None
        for tag, v in zip(tags, ns):
            s = v * 1e-9
            if tag == "start":
                r.loop_start = s
            elif tag == "end":
                r.loop_end = s
            elif tag == "fwd1":
                r.forward_s += s - prev
            elif tag == "xchg":
                r.exchange_wait_s += s - prev
            elif tag == "apply":
                r.apply_s += s - prev
            prev = s
        return r


class _OwnedDev:
    """Exposes memory from ps_dev_alloc (our cudaMalloc, this process's device)
    to torch through the CUDA array interface."""

    def __init__(self, ptr: int, shape: tuple, typestr: str):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None}


class _PeerVec:
    """A rank's eps vector in (possibly a peer's IPC-mapped) device memory:
    only its address is used - by ps_sched_cycle and the record copy - so no
    torch tensor ever spans devices."""

    def __init__(self, ptr: int, nbytes: int):
        self.ptr, self.nbytes = int(ptr), nbytes

    def data_ptr(self) -> int:
        return self.ptr


class PeerExchange:
    """Peer-memory eps exchange over CUDA IPC (csrc/peer.cu), one per rank.

    Local memory exported to every peer: ``e_buf[2][n]`` (this rank's lane
    eps, double-buffered by round parity) and ``ready[world]`` (flag j holds
    base + round + 1 once rank j's eps of that round is written). The
    bootstrap (handle exchange) runs over the given process group, which may
    be gloo: no data moves through it.
    """

    def __init__(self, n: int, dtype, rank: int, world: int, group=None):
        import ctypes as C

        import torch
        import torch.distributed as dist

        self.lib = _lib.load(require_gpu=True)
        self.n, self.rank, self.world = n, rank, world
        es = torch.empty(0, dtype=dtype).element_size()
        # own cudaMalloc allocations: an IPC handle maps the allocation base
        self.owned = []
        for nbytes in (2 * n * es, 8 * world):
            ptr = C.c_void_p()
            _lib.check(self.lib.ps_dev_alloc(nbytes, C.byref(ptr)), "exchange alloc")
            self.owned.append(ptr.value)
        self.e_buf = torch.as_tensor(_OwnedDev(self.owned[0], (2, n), "<f8" if es == 8 else "<f4"),
                                     device="cuda")
        self.ready = torch.as_tensor(_OwnedDev(self.owned[1], (world,), "<i8"), device="cuda")
        self.base = torch.zeros(1, dtype=torch.int64, device="cuda")
        torch.cuda.synchronize()
        hs = []
        for ptr in self.owned:
            h = (C.c_char * 64)()
            _lib.check(self.lib.ps_ipc_get_handle(ptr, h), "ipc handle")
            hs.append(bytes(h))
        allh = [None] * world
        dist.all_gather_object(allh, hs, group=group)
        self.opened = []
        e_ptr, r_ptr = [], []
        for p in range(world):
            if p == rank:
                e_ptr.append(_lib.ptr(self.e_buf))
                r_ptr.append(_lib.ptr(self.ready))
                continue
            ptrs = []
            for hb in allh[p]:
                out = C.c_void_p()
                _lib.check(self.lib.ps_ipc_open_handle(hb, C.byref(out)), "ipc open")
                ptrs.append(out.value)
                self.opened.append(out.value)
            e_ptr.append(ptrs[0])
            r_ptr.append(ptrs[1])
        # round parity -> every rank's eps vector of that parity
        self.views = [[_PeerVec(e_ptr[p] + par * n * es, n * es) for p in range(world)]
                      for par in (0, 1)]
        # where this rank's "ready" goes on every rank: ready_p[rank]
        self.slots = torch.tensor([r_ptr[p] + 8 * rank for p in range(world)], dtype=torch.int64,
                                  device="cuda")
        dist.barrier(group=group)

    def close(self):
        """Unmap the peers' buffers and free ours (after a barrier: peers may
        still read this rank's memory until every rank is done)."""
        for p in self.opened:
            self.lib.ps_ipc_close(p)
        self.opened = []
        self.e_buf = self.ready = None
        for p in self.owned:
            self.lib.ps_dev_free(p)
        self.owned = []


class CudaRankOps:
    """Device buffers + C-ABI launches + the per-round eps exchange for one rank:
    ``exchange="nccl"`` (all_gather_into_tensor) or ``"peer"`` (PeerExchange:
    IPC-mapped peer buffers read by the fused apply kernel over NVLink)."""

    def __init__(self, w, sched: NoiseSchedule, cfg: RunConfig, rank: int, world: int,
                 group=None, record: bool = False, external_init: bool = False,
                 exchange: str = "nccl", timed: bool = False):
        import torch

        self.torch = torch
        self.lib = _lib.load(require_gpu=True)
        self.w, self.sched, self.cfg = w, sched, cfg
        self.rank, self.world, self.group = rank, world, group
        self.n, self.T = cfg.data_dim, cfg.steps
        self.code = w.state_dtype_code
        tdt = torch.float64 if self.code == _lib.PS_F64 else torch.float32
        n = self.n
        self.seed_buf = torch.zeros(1, dtype=torch.int64, device="cuda")
        self.x = torch.zeros(n, dtype=tdt, device="cuda")
        self.lane = torch.zeros(n, dtype=tdt, device="cuda")
        self.e_warm = torch.zeros(n, dtype=tdt, device="cuda")
        self.e_local = torch.zeros(n, dtype=tdt, device="cuda")
        self.gathered = torch.zeros((world, n), dtype=tdt, device="cuda")
        self.cache_buf = torch.zeros(n, dtype=tdt, device="cuda")
        self.record_on = record
        self.rec_x = torch.zeros((self.T, n), dtype=tdt, device="cuda") if record else None
        self.rec_e = torch.zeros((self.T, n), dtype=tdt, device="cuda") if record else None
        self.external_init = external_init
        self._steps = {t: step_coeffs(sched, t) for t in range(1, self.T + 1)}
        cyc = plan_cycles(cfg)
        # lane caches must outlive a cycle only if some cycle is longer than its predecessor
        self.persist_cache = any(len(b) > len(a) for a, b in zip(cyc, cyc[1:]))
        self.launches = 0
        self.gathers = 0
        if hasattr(w, "reserve_conditioning"):
            w.reserve_conditioning(self.T)
        if exchange not in ("nccl", "peer"):
            raise ConfigError(f"unknown exchange {exchange!r}")
        self.exchange = exchange
        self.px = PeerExchange(n, tdt, rank, world, group) if exchange == "peer" else None
        self.round = 0
        self.ledger = ExchangeLedger(rank, world, exchange, n * self.x.element_size())
        # phase stamps (off in the timed bench runs: each is one tiny launch)
        self.timed = timed
        self.stamp_tags: list[str] = []
        self.stamp_buf = torch.zeros(8 * self.T + 16, dtype=torch.int64, device="cuda") \
            if timed else None

    def stamp(self, tag: str) -> None:
        if not self.timed:
            return
        i = len(self.stamp_tags)
        self.stamp_tags.append(tag)
        _lib.check(self.lib.ps_stamp(self._p(self.stamp_buf) + 8 * i, _lib.stream_ptr()), "stamp")
        self.launches += 1

    def timings(self) -> RankTimings:
        if not self.timed:
            return RankTimings()
        ns = self.stamp_buf[:len(self.stamp_tags)].cpu().tolist()
        return RankTimings.from_stamps(self.stamp_tags, ns)

    def finish(self):
        """Peer exchange: end-of-run handshake. Every rank publishes "run done"
        (a round index above any real round) and waits for all ranks' flags,
        so the next run's first lane forward cannot overwrite an eps buffer a
        slower peer is still reading in this run's last apply."""
        if self.px is None:
            return
        st = _lib.stream_ptr()
        _lib.check(self.lib.ps_peer_signal(self._p(self.px.slots), self.world,
                                           self._p(self.px.base), self.DONE_ROUND, st),
                   "peer signal")
        _lib.check(self.lib.ps_peer_wait(self._p(self.px.ready), self.world,
                                         self._p(self.px.base), self.DONE_ROUND, st), "peer wait")
        self.launches += 2

    DONE_ROUND = 1 << 19  # below the 2^20 epoch stride, above any round index

    def _p(self, t) -> int:
        return _lib.ptr(t)

    def init(self):
        self.round = 0
        self.ledger.reset()
        self.stamp_tags = []
        if hasattr(self.w, "prepare_conditioning"):  # batched t-only conditioning of the run
            self.launches += self.w.prepare_conditioning(self.T)
        if self.px is not None:
            _lib.check(self.lib.ps_peer_epoch_advance(self._p(self.px.base), _lib.stream_ptr()),
                       "peer epoch")
            self.launches += 1
        if not self.external_init:
            _lib.check(self.lib.ps_rng_normal_dev(
                self._p(self.x), self.n, self._p(self.seed_buf), stream_id(PURPOSE_INIT, 0), 0,
                self.code, _lib.stream_ptr()), "initial_state")
            self.launches += 1
        return self.x

    def forward(self, x, t, slot):
        out = self.e_warm if slot == "warm" else self.e_local
        if slot != "warm" and self.px is not None:
            out = self.px.e_buf[self.round % 2]  # written in place, read by peers
        self.w.forward_device(x.view(1, -1), [t], self.T, out.view(1, -1))
        self.launches += self.w.kernels_per_forward(1)
        return out

    def zeros(self, slot):
        return self.e_local  # idle rank: contents ignored by every receiver

    def allgather(self, e, active: int | None = None):
        if self.px is not None:
            # publish this round's eps (already in e_buf[parity]) to every
            # rank, wait for the `active` lanes' flags; the apply kernel then
            # reads the peers' vectors in place over NVLink
            active = self.world if active is None else active
            k, st = self.round, _lib.stream_ptr()
            if self.rank < active:
                _lib.check(self.lib.ps_peer_signal(self._p(self.px.slots), self.world,
                                                   self._p(self.px.base), k, st), "peer signal")
            _lib.check(self.lib.ps_peer_wait(self._p(self.px.ready), active,
                                             self._p(self.px.base), k, st), "peer wait")
            self.launches += 2
            self.gathers += 1
            self.round += 1
            views = self.px.views[k % 2]
            # bytes the apply kernels move over NVLink this round: this rank
            # reads every active remote lane; peers pull its own lane
            vb = self.ledger.vec_bytes
            remote = [v for j, v in enumerate(views[:active]) if j != self.rank]
            owns = self.rank < active
            self.ledger.record(active, (active - 1) * vb if owns else 0,
                               sum(v.nbytes for v in remote), len(remote))
            return views
        import torch.distributed as dist

        dist.all_gather_into_tensor(self.gathered, e, group=self.group)
        self.gathers += 1
        self.round += 1
        es = e.element_size()
        self.ledger.record(active if active is not None else self.world, e.numel() * es,
                           (self.gathered.numel() - e.numel()) * es, self.world - 1)
        return [self.gathered[i] for i in range(self.world)]

    def keep_cache(self, e):
        if isinstance(e, _PeerVec):  # own slot of the peer exchange: a local buffer
            e = self.px.e_buf[(self.round - 1) % 2]
        if self.persist_cache:
            self.cache_buf.copy_(e)
            return self.cache_buf
        return e

    def record(self, k, eps_list):
        if not self.record_on:
            return
        if eps_list and isinstance(eps_list[0], _PeerVec):
            row = self.n * self.rec_e.element_size()
            for i, e in enumerate(eps_list):
                _lib.check(self.lib.ps_copy(self._p(self.rec_e) + (k + i) * row, e.ptr, row,
                                            _lib.stream_ptr()), "record copy")
            return
        self.rec_e[k:k + len(eps_list)].copy_(self.torch.stack(eps_list))

    def apply_roll(self, x, apply_ts, eps_list, roll_ts, cache):
        es = x.element_size()
        A = _lib.step_array([self._steps[t] for t in apply_ts])
        E = _lib.ptr_array([self._p(e) for e in eps_list])
        R = _lib.ptr_array([(self._p(self.rec_x) + (self.T - t) * self.n * es)
                            if self.record_on else 0 for t in apply_ts])
        lane_hi = self.rank + 1 if roll_ts else 0
        caches = [0] * _lib.PS_MAX_CYCLE
        outs = [0] * _lib.PS_MAX_CYCLE
        roll = _lib.step_array([self._steps[t] for t in roll_ts])
        if roll_ts:
            caches[self.rank] = self._p(cache)
            outs[self.rank] = self._p(self.lane)
        _lib.check(self.lib.ps_sched_cycle(
            self._p(x), self._p(x), self.n, self.code, self._p(self.seed_buf), len(apply_ts), A, E,
            R, self.rank if roll_ts else 0, lane_hi, roll, _lib.ptr_array(caches),
            _lib.ptr_array(outs), _lib.stream_ptr()), "sched_cycle")
        self.launches += 1
        return x, self.lane


@dataclass
class RunResult:
    """Per-rank outcome of run_nccl (mirrors worker.RunResult, worker.py:97-110):
    rank 0 carries the Trajectory; ``timings`` holds every rank's RankTimings
    (gathered to all ranks), ``ledgers`` every rank's measured ExchangeLedger."""

    trajectory: Trajectory | None
    x0: object
    rank: int
    world: int
    gathers: int = 0
    launches: int = 0
    timings: list = field(default_factory=list)
    ledgers: list = field(default_factory=list)

    @property
    def loop_latency_s(self) -> float:
        """Denoising-loop latency (worker.py:108-110): the slowest rank's loop,
        each rank timed on its own device clock from the same barrier."""
        return max((t.loop_s for t in self.timings), default=0.0)


class NcclSampler:
    """ParaStep over `world` GPUs (degree == world), replayable per seed.

    Must be constructed on every rank of an initialised NCCL process group;
    ``run(seed)`` issues the run on the current stream (async). With
    ``graph=True`` the whole run, NCCL all-gathers included, is captured in
    one CUDA graph after an eager warm-up run.
    """

    def __init__(self, w, sched: NoiseSchedule, cfg: RunConfig, group=None, record=False,
                 external_init=False, exchange: str = "nccl", timed: bool = False):
        import torch.distributed as dist

        _check(w, sched, cfg, None)
        if cfg.strategy not in (STRATEGY_PARASTEP, STRATEGY_DYNAMIC):
            raise ConfigError(f"protocol runs use the parastep (or dynamic) strategy, got "
                              f"{cfg.strategy!r}")
        if not dist.is_initialized():
            raise ConfigError("run_nccl needs an initialised torch.distributed process group")
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.group = group
        self.cfg = cfg
        self.cycles = plan_cycles(cfg)
        if cfg.strategy == STRATEGY_PARASTEP and cfg.degree != self.world:
            raise ConfigError(f"degree {cfg.degree} != world size {self.world}")
        if max((len(c) for c in self.cycles), default=1) > self.world:
            raise ConfigError(f"a cycle of {max(len(c) for c in self.cycles)} lanes needs more "
                              f"than the {self.world} ranks")
        self.ops = CudaRankOps(w, sched, cfg, self.rank, self.world, group, record, external_init,
                               exchange, timed)
        self.graph = None

    def _launch(self):
        self.ops.launches = 0
        self.ops.gathers = 0
        rank_loop(self.ops, self.cfg.steps, self.cfg.warmup, self.world, self.rank, self.cycles)

    def run(self, seed: int, graph: bool = False, x_init=None) -> None:
        import torch

        self.ops.seed_buf.fill_(_int64_of(seed))
        if self.ops.external_init:
            if x_init is None:
                raise ConfigError("external_init sampler needs x_init")
            self.ops.x.copy_(torch.as_tensor(x_init).reshape(-1), non_blocking=True)
        if not graph:
            self._launch()
            return
        if self.graph is None:
            self._launch()
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

    def sample(self, seed: int, graph: bool = False):
        """Run one denoise and return rank 0's Trajectory (None on other ranks)."""
        self.run(seed, graph=graph)
        return self.result().trajectory

    def traffic_census(self) -> dict:
        """This rank's measured ε-exchange bytes per round (the ExchangeLedger
        of the last run), verified against the closed form: per full round a
        rank receives (d-1)*N*s bytes (ledger.py; the reference's Algorithm-1
        ledger moves 2(d-1)*M per cycle, protocol/ledger.py:120-123). A
        mismatch raises LedgerViolationError."""
        lg = self.ops.ledger
        rep = lg.verify(self.cycles)
        return {"rounds": rep.rounds, "sent": rep.sent, "received": rep.received,
                "ok": True, "csv": lg.csv(), "report": rep.summary()}

    def result(self) -> RunResult:
        import torch

        torch.cuda.current_stream().synchronize()
        o = self.ops
        traj = None
        if o.record_on and self.rank == 0:
            xs = o.rec_x.double().cpu().numpy()
            es = o.rec_e.double().cpu().numpy()
            T = self.cfg.steps
            fresh = [True] * T
            for cyc in self.cycles:
                for j, t in enumerate(cyc):
                    fresh[T - t] = j == 0
            traj = Trajectory([StepRecord(T - k, xs[k].copy(), es[k].copy(), fresh[k])
                               for k in range(T)], o.x.double().cpu().numpy().copy())
        import torch.distributed as dist

        mine = (o.timings(), o.ledger)
        allr = [None] * self.world
        dist.all_gather_object(allr, mine, group=self.group)
        return RunResult(traj, o.x.double().cpu().numpy().copy(), self.rank, self.world,
                         o.gathers, o.launches, [a[0] for a in allr], [a[1] for a in allr])


def run_nccl(w, sched: NoiseSchedule, cfg: RunConfig, group=None, record: bool = True,
             timeout: float = 60.0, exchange: str = "nccl") -> RunResult:
    """The reference's run_tcp/run_loopback (worker.py:244-372) as one NCCL rank.

    Call on every rank of an initialised NCCL group with cfg.degree == world
    size. Rank 0's result carries the Trajectory; every rank returns its x0
    (identical on all ranks). A failed collective surfaces as
    ProtocolAbortError(rank, step) like the reference's transport faults.
    """
    import torch

    s = NcclSampler(w, sched, cfg, group=group, record=record, exchange=exchange, timed=True)
    try:
        s.run(cfg.seed)
        torch.cuda.synchronize()
    except RuntimeError as exc:  # NCCL / CUDA failure during the round
        raise ProtocolAbortError(f"collective failed: {exc}", s.rank) from exc
    return s.result()
