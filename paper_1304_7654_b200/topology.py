"""Multi-block grid description and the block -> GPU partition.

Semantics follow the reference's mesh module (mesh.py:36-131 types,
mesh.py:307-349 validation, mesh.py:352-373 greedy LPT partition,
mesh.py:376-386 cut roles); the partition is what places blocks on GPUs.
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass, field
from enum import Enum

from .exceptions import CapacityError, TopologyError

FACES = ("north", "south", "east", "west")
# face -> index used by the device face maps
FACE_INDEX = {"south": 0, "north": 1, "west": 2, "east": 3}


@dataclass(frozen=True)
class BlockSpec:
    """An ni x nj structured block of cells (plus a one-cell halo ring).

    Cell (i, j), 1-based, has centre (x0 + (i - 1/2) h, y0 + (j - 1/2) h).
    body_faces lists (face, body id) pairs integrated by the force sums.
    """

    id: int
    ni: int
    nj: int
    x0: float
    y0: float
    h: float
    body_faces: tuple = ()

    def cells(self):
        return self.ni * self.nj

    def face_extent(self, face):
        """Cells along a face: north/south faces run along i, east/west along j."""
        return self.ni if face in ("north", "south") else self.nj


@dataclass(frozen=True)
class CutSide:
    block: int
    face: str
    lo: int   # 1-based, inclusive
    hi: int

    @property
    def length(self):
        return self.hi - self.lo + 1


@dataclass(frozen=True)
class CutSpec:
    """Two face ranges whose halos mirror each other's interior every stage.

    With reversed=True element k of side_a pairs with element L-1-k of side_b.
    """

    side_a: CutSide
    side_b: CutSide
    reversed: bool = False

    @property
    def length(self):
        return self.side_a.length


@dataclass(frozen=True)
class Topology:
    blocks: tuple
    cuts: tuple
    nbody: int

    def total_cells(self):
        return sum(b.cells() for b in self.blocks)

    @property
    def nblocks(self):
        return len(self.blocks)


@dataclass(frozen=True)
class Partition:
    rank_of_block: tuple
    nranks: int

    def rank_of(self, block_id):
        return self.rank_of_block[block_id]

    def blocks_of(self, rank):
        return tuple(b for b, owner in enumerate(self.rank_of_block) if owner == rank)


class CutRole(Enum):
    BOTH_LOCAL = "both_local"
    RECV_SIDE = "recv_side"
    SEND_SIDE = "send_side"
    UNINVOLVED = "uninvolved"


@dataclass
class CaseConfig:
    """Solver parameters plus the block and cut lists of one case."""

    nharms: int
    npde: int
    iterations: int
    dtau: float
    omega: float
    nbody: int
    blocks: list = field(default_factory=list)
    cuts: list = field(default_factory=list)
    name: str = ""

    @property
    def planes(self):
        """HB snapshot count 2*N_H + 1."""
        return 2 * self.nharms + 1


def build_topology(config):
    """Check a case for consistency and freeze it into a Topology."""
    blocks = tuple(config.blocks)
    if not blocks:
        raise TopologyError("case defines no blocks")
    if [b.id for b in blocks] != list(range(len(blocks))):
        raise TopologyError("block ids must be contiguous starting at 0")
    for blk in blocks:
        for _, body in blk.body_faces:
            if body < 0 or body >= config.nbody:
                raise TopologyError(
                    f"block {blk.id}: body id {body} outside 0..{config.nbody - 1}")

    owner = {}
    for ci, cut in enumerate(config.cuts):
        for tag, side in (("a", cut.side_a), ("b", cut.side_b)):
            if side.block < 0 or side.block >= len(blocks):
                raise TopologyError(
                    f"cut {ci}: side_{tag} references missing block {side.block}")
            extent = blocks[side.block].face_extent(side.face)
            if side.hi > extent:
                raise TopologyError(
                    f"cut {ci}: range {side.lo}:{side.hi} exceeds {side.face} "
                    f"extent {extent} of block {side.block}")
        if cut.side_a.length != cut.side_b.length:
            raise TopologyError(
                f"cut {ci}: side lengths differ "
                f"({cut.side_a.length} vs {cut.side_b.length})")
        for side in (cut.side_a, cut.side_b):
            for k in range(side.lo, side.hi + 1):
                slot = (side.block, side.face, k)
                if slot in owner:
                    raise TopologyError(
                        f"cut {ci}: boundary element {slot} already used by cut {owner[slot]}")
                owner[slot] = ci
    return Topology(blocks=blocks, cuts=tuple(config.cuts), nbody=config.nbody)


def partition_blocks(topology, nranks):
    """Greedy longest-processing-time placement of blocks on ranks.

    Blocks in descending cell count (ties: lower id first) each go to the
    currently least-loaded rank (ties: lower rank).  Deterministic; cuts are
    ignored.  Equal blocks therefore land round-robin, b -> b mod nranks.
    """
    if nranks < 1:
        raise CapacityError(f"nranks must be >= 1, got {nranks}")
    if nranks > topology.nblocks:
        raise CapacityError(
            f"{nranks} ranks requested but only {topology.nblocks} blocks to distribute")
    loads = [(0, r) for r in range(nranks)]
    owner = [0] * topology.nblocks
    for blk in sorted(topology.blocks, key=lambda b: (-b.cells(), b.id)):
        load, rank = heapq.heappop(loads)
        owner[blk.id] = rank
        heapq.heappush(loads, (load + blk.cells(), rank))
    return Partition(rank_of_block=tuple(owner), nranks=nranks)


def cut_role(partition, cut, rank):
    """Which side(s) of `cut` the given rank owns."""
    on_a = partition.rank_of(cut.side_a.block) == rank
    on_b = partition.rank_of(cut.side_b.block) == rank
    if on_a and on_b:
        return CutRole.BOTH_LOCAL
    if on_a:
        return CutRole.RECV_SIDE
    if on_b:
        return CutRole.SEND_SIDE
    return CutRole.UNINVOLVED
