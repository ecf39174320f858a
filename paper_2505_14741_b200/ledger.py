"""Measured ε-exchange ledger of a multi-GPU ParaStep run.

The reference counts every frame its transports move (protocol/ledger.py:26-98)
and checks the census against the per-cycle closed form, raising
``LedgerViolationError`` on any disagreement (ledger.py:115-182,
errors.py:70-71). Here the exchange is one all-gather (NCCL) or one set of
peer reads (NVLink, csrc/peer.cu) per round, and the ledger records, at the
moment each exchange is issued, the bytes it actually moves for this rank:

* ``sent``: bytes of this rank's own ε that leave the rank (NCCL: the send
  buffer of the all-gather; peer: what the peers' apply kernels pull from
  this rank's exported buffer, (c-1)*N*s when the rank owns a lane, else 0);
* ``received``: bytes arriving from other ranks (NCCL: output minus own
  slot of the all-gather; peer: every remote ε pointer handed to the fused
  apply kernel, N*s each).

``verify`` checks every round against the closed form — NCCL: (d-1)*N*s
received per round regardless of the cycle length; peer: (c-1)*N*s for a
rank that owns a lane of a c-lane cycle, c*N*s for an idle rank — and
``verify_merged`` checks the all-rank total of a full round against
d(d-1)*N*s (the all-gather mode's counterpart of the reference's
2(p-1)*M per cycle, ledger.py:120-123).
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .errors import LedgerViolationError, ParameterError


@dataclass
class LedgerEntry:
    round: int
    cycle_len: int
    sent: int
    received: int
    remote_reads: int  # number of remote ε vectors this round's apply consumed


@dataclass
class ExchangeLedger:
    rank: int
    world: int
    kind: str  # "nccl" | "peer" | "gloo"
    vec_bytes: int  # N * s
    entries: list[LedgerEntry] = field(default_factory=list)

    def record(self, cycle_len: int, sent: int, received: int, remote_reads: int) -> None:
        self.entries.append(LedgerEntry(len(self.entries), cycle_len, sent, received,
                                        remote_reads))

    def reset(self) -> None:
        self.entries = []

    @property
    def sent(self) -> int:
        return sum(e.sent for e in self.entries)

    @property
    def received(self) -> int:
        return sum(e.received for e in self.entries)

    def expected(self, cycle_len: int) -> tuple[int, int]:
        """(sent, received) of one round of `cycle_len` lanes for this rank."""
        v, d, c = self.vec_bytes, self.world, cycle_len
        if self.kind in ("nccl", "gloo"):  # whole-world all-gather every round
            return v, (d - 1) * v
        owns = self.rank < c
        return ((c - 1) * v if owns else 0), ((c - 1) * v if owns else c * v)

    def verify(self, cycles: list[list[int]]) -> "LedgerReport":
        """Check this rank's census round by round; raise on the first mismatch."""
        if self.vec_bytes < 1 or self.world < 1:
            raise ParameterError(f"invalid ledger (world={self.world}, vec={self.vec_bytes})")
        if len(self.entries) != len(cycles):
            raise LedgerViolationError(
                f"rank {self.rank}: {len(self.entries)} exchanges recorded, expected one per "
                f"round ({len(cycles)})")
        for e, cyc in zip(self.entries, cycles):
            if e.cycle_len != len(cyc):
                raise LedgerViolationError(
                    f"rank {self.rank} round {e.round}: exchange covered {e.cycle_len} lanes, "
                    f"the cycle has {len(cyc)}")
            want = self.expected(len(cyc))
            if (e.sent, e.received) != want:
                raise LedgerViolationError(
                    f"rank {self.rank} round {e.round} (t={cyc[0]}..{cyc[-1]}): moved "
                    f"sent={e.sent} received={e.received} bytes, closed form "
                    f"sent={want[0]} received={want[1]}")
        return LedgerReport(self.kind, self.world, self.vec_bytes, len(self.entries),
                            self.sent, self.received,
                            sum(self.expected(len(c))[0] for c in cycles),
                            sum(self.expected(len(c))[1] for c in cycles))

    def csv(self) -> str:
        lines = ["round,cycle_len,sent_bytes,received_bytes"]
        lines += [f"{e.round},{e.cycle_len},{e.sent},{e.received}" for e in self.entries]
        return "\n".join(lines) + "\n"


@dataclass
class LedgerReport:
    kind: str
    world: int
    vec_bytes: int
    rounds: int
    sent: int
    received: int
    expected_sent: int
    expected_received: int

    def summary(self) -> str:
        return (f"{self.kind} d={self.world} rounds={self.rounds}: sent {self.sent}/"
                f"{self.expected_sent} B, received {self.received}/{self.expected_received} B")


def verify_merged(ledgers: list[ExchangeLedger], cycles: list[list[int]]) -> int:
    """All ranks' ledgers together: every full round (c == d) moves exactly
    d(d-1)*N*s bytes into the ranks. Returns the total received bytes."""
    if not ledgers:
        raise ParameterError("no ledgers to merge")
    d, v = ledgers[0].world, ledgers[0].vec_bytes
    if sorted(lg.rank for lg in ledgers) != list(range(d)):
        raise LedgerViolationError(f"ledgers of ranks {[lg.rank for lg in ledgers]}, need 0..{d - 1}")
    for lg in ledgers:
        lg.verify(cycles)
    for i, cyc in enumerate(cycles):
        if len(cyc) != d:
            continue
        tot = sum(lg.entries[i].received for lg in ledgers)
        if tot != d * (d - 1) * v:
            raise LedgerViolationError(
                f"round {i}: the ranks received {tot} bytes together, closed form "
                f"d(d-1)*N*s = {d * (d - 1) * v}")
    return sum(lg.received for lg in ledgers)
