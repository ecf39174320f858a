"""Multi-process (gloo, CPU) check of the N>1 exchange logic.

``protocol.rank_loop`` — the same host logic the NCCL product path runs — is
driven here by oracle-backed ops (numpy float64 + torch.distributed gloo
all_gather on CPU). Every rank must end with rank 0's x0, and rank 0's
trajectory must equal the single-process cycle runner bit-for-bit
(reference: test_protocol.py:44-73, loopback == tcp == emulation).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import core, engines as oeng
from paper_2505_14741_b200.engines import RunConfig, plan_cycles
from paper_2505_14741_b200.errors import LedgerViolationError
from paper_2505_14741_b200.ledger import ExchangeLedger, verify_merged
from paper_2505_14741_b200.protocol import rank_loop


class OracleOps:
    def __init__(self, pred, sch, n, seed, rank, world):
        self.pred, self.sch, self.n, self.seed = pred, sch, n, seed
        self.rank, self.world = rank, world
        self.rec_e = {}
        self.rec_x = {}
        self.gathers = 0
        self.ledger = ExchangeLedger(rank, world, "gloo", 8 * n)

    def init(self):
        return oeng.x_init(self.seed, self.n)

    def forward(self, x, t, slot):
        return self.pred(x, t, self.sch.T)

    def zeros(self, slot):
        return np.zeros(self.n)

    def allgather(self, e, active=None):
        out = [torch.zeros(self.n, dtype=torch.float64) for _ in range(self.world)]
        src = torch.from_numpy(np.ascontiguousarray(e))
        dist.all_gather(out, src)
        self.gathers += 1
        es = src.element_size()
        self.ledger.record(active if active is not None else self.world, src.numel() * es,
                           sum(o.numel() for i, o in enumerate(out) if i != self.rank) * es,
                           self.world - 1)
        return [o.numpy().copy() for o in out]

    def keep_cache(self, e):
        return e

    def record(self, k, eps_list):
        for j, e in enumerate(eps_list):
            self.rec_e[k + j] = e

    def apply_roll(self, x, apply_ts, eps_list, roll_ts, cache):
        for t, e in zip(apply_ts, eps_list):
            self.rec_x[self.sch.T - t] = x
            x = core.ddpm_step(x, t, e, self.sch, oeng.z_step(self.seed, t, self.n))
        lane = x
        for t in roll_ts:
            lane = core.ddpm_step(lane, t, cache, self.sch, oeng.z_step(self.seed, t, self.n))
        return x, lane


def _worker(rank, world, port, T, warmup, mode, seed, q, lengths=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pred = core.MLP.init(6, hidden=(8,), embed_dim=4, seed=7)
        sch = core.Sched(T, mode)
        cfg = RunConfig(steps=T, warmup=warmup, strategy="dynamic" if lengths else "parastep",
                        degree=world, seed=seed, data_dim=6, schedule_override=lengths)
        ops = OracleOps(pred, sch, 6, seed, rank, world)
        x0 = rank_loop(ops, T, warmup, world, rank, plan_cycles(cfg))
        q.put((rank, x0, ops.rec_x, ops.rec_e, ops.gathers, ops.ledger))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,T,warmup,mode", [(2, 12, 3, "posterior"), (3, 12, 4, "zero"),
                                                 (4, 14, 2, "posterior")])
def test_rank_loop_over_gloo_equals_cycle_runner(world, T, warmup, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, T, warmup, mode, 5, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    ledgers = []
    for _ in range(world):
        r, x0, rx, re, g, lg = q.get(timeout=120)
        res[r] = (x0, rx, re, g)
        ledgers.append(lg)
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    pred = core.MLP.init(6, hidden=(8,), embed_dim=4, seed=7)
    ref = oeng.cycles(pred, core.Sched(T, mode), 6, 5, warmup=warmup, degree=world)
    x0, rx, re, gathers = res[0]
    assert np.array_equal(x0, ref["x0"])
    for k in range(T):
        assert np.array_equal(rx[k], ref["x"][k]), k
        assert np.array_equal(re[k], ref["eps"][k]), k
    for r in range(1, world):
        assert np.array_equal(res[r][0], x0)  # every rank ends synchronised
    cycles = plan_cycles(RunConfig(steps=T, warmup=warmup, strategy="parastep", degree=world,
                                   data_dim=6))
    assert gathers == len(cycles)
    # measured exchange ledger: every rank's census and the d(d-1)*N*s total per full round
    total = verify_merged(ledgers, cycles)
    assert total == world * len(cycles) * (world - 1) * 8 * 6
    ledgers[1].entries[0].received += 8
    with pytest.raises(LedgerViolationError):
        verify_merged(ledgers, cycles)


def test_rank_loop_dynamic_cycles_over_gloo():
    """Dynamic cycle lengths (the reference's denoise_dynamic, engines.py:346-349)
    through the same rank loop: cycles shorter than the world idle ranks."""
    world, T, warmup, lengths = 3, 12, 2, [1, 3, 2, 3, 1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, T, warmup, "posterior", 9, q,
                                               lengths)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    ledgers = []
    for _ in range(world):
        r, x0, rx, re, g, lg = q.get(timeout=120)
        res[r] = (x0, rx, re)
        ledgers.append(lg)
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    pred = core.MLP.init(6, hidden=(8,), embed_dim=4, seed=7)
    ref = oeng.cycles(pred, core.Sched(T, "posterior"), 6, 9, warmup=warmup, degree=world,
                      lengths=lengths)
    x0, rx, re = res[0]
    assert np.array_equal(x0, ref["x0"])
    for k in range(T):
        assert np.array_equal(rx[k], ref["x"][k]), k
        assert np.array_equal(re[k], ref["eps"][k]), k
    for r in range(1, world):
        assert np.array_equal(res[r][0], x0)
    cycles = plan_cycles(RunConfig(steps=T, warmup=warmup, strategy="dynamic", degree=world,
                                   schedule_override=lengths, data_dim=6))
    verify_merged(ledgers, cycles)


def test_peer_ledger_closed_form():
    """Peer exchange census (host logic): a lane owner reads the c-1 remote
    lanes, an idle rank all c; a full round moves d(d-1)*N*s in total."""
    d, v = 4, 1024
    cycles = [[10, 9, 8, 7], [6, 5, 4, 3], [2, 1]]
    lgs = [ExchangeLedger(r, d, "peer", v) for r in range(d)]
    for cyc in cycles:
        c = len(cyc)
        for lg in lgs:
            owns = lg.rank < c
            lg.record(c, (c - 1) * v if owns else 0, ((c - 1) if owns else c) * v,
                      (c - 1) if owns else c)
    assert verify_merged(lgs, cycles) == sum(lg.received for lg in lgs)
    assert lgs[3].entries[2].received == 2 * v  # idle in the truncated cycle
    lgs[0].entries[1].sent = 0
    with pytest.raises(LedgerViolationError):
        lgs[0].verify(cycles)
