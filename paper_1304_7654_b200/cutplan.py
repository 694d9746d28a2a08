"""Cut (halo) plan: which interior face cells feed which halo cells.

The plan objects mirror the reference's (exchange.py:53-188): per cut two
directions -- direction 0 fills side_a's halo from side_b's interior (with
the cut's reversal applied to the source), direction 1 fills side_b's halo
from side_a's interior (reversal applied to the destination).  Message
payloads are element-major, datasize = npde * planes values per element,
plane-outer / pde-inner (exchange.py:4-10, 248-252).

On the GPU there is no separate exchange pass for local cuts: the stage
kernel stores each cut face cell straight into its paired halo cell (or the
send buffer).  `face_targets` turns the plan into that per-face-cell map.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

from .exceptions import ProtocolError

PHASE_STRIDE = 1 << 20


class ExchangeMode(Enum):
    PER_ELEMENT = "per-element"
    AGGREGATED_CUT = "aggregated"


class ThreadMode(Enum):
    SERIAL = "serial"
    TAGGED_THREADS = "tagged"


@dataclass(frozen=True)
class ExchangeStrategy:
    """Kept for RunSpec compatibility; the GPU path always moves one
    aggregated payload per remote cut direction."""

    mode: ExchangeMode = ExchangeMode.AGGREGATED_CUT
    thread_mode: ThreadMode = ThreadMode.SERIAL


@dataclass(frozen=True)
class DirectionPlan:
    cut_index: int
    direction: int
    sender_rank: int
    recv_rank: int
    src_block: int
    src_face: str
    src_lo: int
    src_hi: int
    src_reversed: bool
    dst_block: int
    dst_face: str
    dst_lo: int
    dst_hi: int
    dst_reversed: bool
    length: int
    local: bool

    def src_index(self, e):
        """1-based face index of the interior cell feeding element e."""
        return self.src_hi - e if self.src_reversed else self.src_lo + e

    def dst_index(self, e):
        """1-based face index of the halo cell receiving element e."""
        return self.dst_hi - e if self.dst_reversed else self.dst_lo + e


@dataclass(frozen=True)
class PlannedCut:
    index: int
    length: int
    datasize: int
    rank_a: int
    rank_b: int
    local: bool
    directions: tuple

    def displacement(self, element):
        return element * self.datasize

    @property
    def displacement_table(self):
        return tuple(e * self.datasize for e in range(self.length))

    @property
    def buffer_length(self):
        return self.length * self.datasize


@dataclass(frozen=True)
class CutPlan:
    nharms: int
    npde: int
    datasize: int
    cuts: tuple
    max_slots: int

    @property
    def planes(self):
        return 2 * self.nharms + 1

    def tag(self, cut_index, direction, slot, phase):
        if phase >= PHASE_STRIDE:
            raise ProtocolError(f"exchange phase {phase} exceeds the tag space")
        return ((cut_index * 2 + direction) * self.max_slots + slot) * PHASE_STRIDE + phase

    def directions(self):
        for cut in self.cuts:
            yield from cut.directions


def build_cut_plan(topology, partition, nharms, npde):
    """Both directions of every cut, with owners and locality."""
    datasize = npde * (2 * nharms + 1)
    cuts = []
    longest = 1
    for ci, cut in enumerate(topology.cuts):
        a, b = cut.side_a, cut.side_b
        ra, rb = partition.rank_of(a.block), partition.rank_of(b.block)
        longest = max(longest, cut.length)
        common = dict(cut_index=ci, length=cut.length, local=ra == rb)
        into_a = DirectionPlan(direction=0, sender_rank=rb, recv_rank=ra,
                               src_block=b.block, src_face=b.face, src_lo=b.lo, src_hi=b.hi,
                               src_reversed=cut.reversed,
                               dst_block=a.block, dst_face=a.face, dst_lo=a.lo, dst_hi=a.hi,
                               dst_reversed=False, **common)
        into_b = DirectionPlan(direction=1, sender_rank=ra, recv_rank=rb,
                               src_block=a.block, src_face=a.face, src_lo=a.lo, src_hi=a.hi,
                               src_reversed=False,
                               dst_block=b.block, dst_face=b.face, dst_lo=b.lo, dst_hi=b.hi,
                               dst_reversed=cut.reversed, **common)
        cuts.append(PlannedCut(index=ci, length=cut.length, datasize=datasize, rank_a=ra,
                               rank_b=rb, local=ra == rb, directions=(into_a, into_b)))
    return CutPlan(nharms=nharms, npde=npde, datasize=datasize, cuts=tuple(cuts),
                   max_slots=2 * longest)


@dataclass(frozen=True)
class ExchangeForecast:
    """Per-direction totals of one exchange over remote cuts."""

    messages: int
    nbytes: int

    @property
    def total_messages(self):
        return 2 * self.messages

    @property
    def total_bytes(self):
        return 2 * self.nbytes


def predicted_message_count(plan, strategy=ExchangeStrategy()):
    """Closed-form messages and bytes per direction per exchange (exchange.py:172-188)."""
    msgs = nbytes = 0
    for cut in plan.cuts:
        if cut.local:
            continue
        msgs += 2 * cut.length if strategy.mode is ExchangeMode.PER_ELEMENT else 1
        nbytes += cut.length * cut.datasize * 8
    return ExchangeForecast(messages=msgs, nbytes=nbytes)


@dataclass(frozen=True)
class RankRoutes:
    """One rank's view of the plan, in plan order (cut, then direction)."""

    local: tuple   # both ends on this rank
    sends: tuple   # this rank sends
    recvs: tuple   # this rank receives


def rank_routes(plan, rank):
    local, sends, recvs = [], [], []
    for d in plan.directions():
        if d.local:
            if d.recv_rank == rank:
                local.append(d)
        elif d.sender_rank == rank:
            sends.append(d)
        elif d.recv_rank == rank:
            recvs.append(d)
    return RankRoutes(tuple(local), tuple(sends), tuple(recvs))
