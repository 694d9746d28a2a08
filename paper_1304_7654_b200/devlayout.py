"""Per-rank device layout and the tables the kernels consume.

Pure host logic (numpy only), so it is unit-tested on CPU.  For the blocks a
rank owns it fixes:

* the slot layout: block b's value (n, p, j, i) at element
  base_b + (n*4 + p)*ps_b + j*rs_b + ROW_LEAD + i, rows padded to a
  multiple of 8 doubles and ROW_LEAD = 7 so every interior row -- and every
  strip -- starts on a 64-byte DRAM granule; block bases are 256-byte
  aligned.  Row-interleaved (default): ps = pitch, rs = 4*P*pitch;
  plane-major (HBGPU_LAYOUT=plane): ps = (nj+2)*pitch, rs = pitch.
  Three slots (A, B, C) share the layout;
* the stage tiles: one tile = one CTA's strip over tile_rows rows of one
  block -- 64 columns x 4 pdes (tile_pdes 4) or 256 columns x 1 pde
  (tile_pdes 1, every block ni >= WIDE_MIN_NI); tile t of block b is strip
  t % tiles_i, row tile t / tiles_i;
* the face-target pool (fused halo forwarding of south / north faces, see
  cutplan.py);
* the standalone halo directions (priming exchange / pack / unpack, and the
  post-stage pass that forwards west / east faces);
* the send / receive buffer segments, grouped per peer rank, one NCCL
  message per peer and stage;
* the force segments in the reference's summation order (hbcore.py:369-381).
"""

from __future__ import annotations

import functools
import os
from dataclasses import dataclass, field

import numpy as np

from . import native
from .cutplan import rank_routes
from .hbop import forcing_vectors, stencil_coefficients

ROW_LEAD = native.ROW_LEAD
SECTOR_TARGET = np.int64(1) << np.int64(62)   # face-target flag: whole-sector write allowed
NPDE = native.NPDE
WIDE_MIN_NI = 192         # blocks at least this wide use 256-column, 1-pde tiles
BLOCK_ALIGN = 32          # elements (256 B)
GRID_CTAS = 148           # persistent CTAs of the stage / pair kernels (B200: 1 per SM)
SMALL_P_CTAS = 2          # resident single-stage CTAs per SM for P <= SMALL_P_MAX (hb_stage.cu)
SMALL_P_MAX = 5
TILE_OVERHEAD_ROWS = 4    # a tile's cost beyond its rows: 2 halo rows, ring fill, band rows
MAX_TILE_ROWS = 1024
MIN_TILE_ROWS = 8
# auto schedule: paired stages from this many units (cells x P x 4) per stage
# on the rank.  Below it the band / halo launches of the paired schedule cost
# more than the halved traffic saves: single stages are 10-13% faster at C1
# and C2 (2.6M, 4.7M units), paired ones 16% faster at C3 (117M) and ~35% at
# C4 (2.4G)
FUSED_MIN_UNITS = 16 * 2 ** 20
SMALL_MAX_UNITS = 2 ** 18
MAX_BAND_SEGS = 65535
SLOT_TAIL = 64            # elements of zero padding after the last block
# slot layout default: row-interleaved (row j of every (n, p) plane contiguous)
# unless HBGPU_LAYOUT=plane selects the plane-major layout
INTERLEAVED = os.environ.get("HBGPU_LAYOUT", "interleaved") != "plane"


def _round_up(x, m):
    return (x + m - 1) // m * m


def choose_tile_pdes(blocks):
    """4 pdes x 64 columns per tile, or 1 pde x 256 columns when every block
    is wide enough: a tile re-reads one 64-byte halo granule on each side of
    each row, 2 / 8 extra stencil reads for 64 columns but 2 / 32 for 256."""
    if os.environ.get("HBGPU_TILE_PDES") in ("1", "4"):
        return int(os.environ["HBGPU_TILE_PDES"])
    return 1 if min(b.ni for b in blocks) >= WIDE_MIN_NI else 4


def tiles_per_row(blocks, tile_pdes):
    return {b.id: -(-b.ni // native.TILE_COLS[tile_pdes]) * (NPDE // tile_pdes) for b in blocks}


def round_robin_makespan(blocks, tile_pdes, tile_rows, ctas=GRID_CTAS):
    """Largest per-CTA load when the persistent kernels walk the tiles round
    robin (tile t on CTA t mod ctas, tiles in decode_tile order), a tile
    costing its rows plus TILE_OVERHEAD_ROWS."""
    per_row = tiles_per_row(blocks, tile_pdes)
    return _makespan(tuple((per_row[b.id], b.nj) for b in blocks), tile_rows, ctas)


@functools.lru_cache(maxsize=4096)
def _makespan(shape, tile_rows, ctas):
    costs = []
    for per_row, nj in shape:
        rows = np.minimum(tile_rows, nj - np.arange(0, nj, tile_rows)) + TILE_OVERHEAD_ROWS
        costs.append(np.repeat(rows, per_row))
    costs = np.concatenate(costs)
    costs = np.concatenate([costs, np.zeros((-len(costs)) % ctas)])
    return float(costs.reshape(-1, ctas).sum(axis=0).max())


def stage_grid_ctas(blocks, planes, tile_pdes, fused):
    """Persistent CTAs the rank's stage kernels run with: the single-stage
    kernel is compiled for SMALL_P_CTAS resident CTAs per SM up to
    SMALL_P_MAX planes (hb_stage.cu stage_ctas_per_sm), the paired kernel
    always for one."""
    units = sum(b.ni * b.nj for b in blocks) * planes * NPDE
    paired = (fused is not False and fused_eligible(blocks, planes, tile_pdes)
              and (bool(fused) or units >= FUSED_MIN_UNITS))
    return GRID_CTAS * (SMALL_P_CTAS if planes <= SMALL_P_MAX and not paired else 1)


def choose_tile_rows(blocks, tile_pdes=4, ctas=GRID_CTAS):
    """Rows per tile with the smallest round-robin makespan over the
    persistent CTAs, among ceil(nj / k) of the tallest block clipped to
    [MIN_TILE_ROWS, MAX_TILE_ROWS]; ties go to the longer tile.  Long tiles
    amortise the two halo rows each tile re-reads (and, paired, the band
    rows); the makespan avoids a last wave that leaves most CTAs idle, e.g.
    8 blocks of 1024 rows take 128-row tiles (1024 tiles: 7 per CTA) rather
    than 110-row ones (1280 tiles: 8.6 per CTA)."""
    nj = max(b.nj for b in blocks)
    cands = sorted({min(MAX_TILE_ROWS, max(MIN_TILE_ROWS, -(-nj // k))) for k in range(1, nj + 1)},
                   reverse=True)
    best = None
    for tj in cands:
        load = round_robin_makespan(blocks, tile_pdes, tj, ctas)
        if best is None or load < best[0]:
            best = (load, tj)
    return best[1]


@dataclass
class RankLayout:
    planes: int
    blocks: list                    # owned BlockSpec, ascending id
    local_index: dict               # gid -> local index
    pitch: list
    ps: list                        # elements between (n, p) planes
    rs: list                        # elements between rows j
    base: list
    slot_elems: int
    tile_rows: int
    block_table: np.ndarray
    tile_block: np.ndarray
    total_tiles: int
    sxy: list                       # per block (sin 2 pi x_i, sin 2 pi y_j)
    sxy_size: int                   # elements of the device forcing-table pool
    faces: np.ndarray
    prime_dirs: np.ndarray
    unpack_dirs: np.ndarray
    post_dirs: np.ndarray           # column-face forwarding after the first stage
    force_segs: np.ndarray
    sends: list = field(default_factory=list)     # (peer, offset, count)
    recvs: list = field(default_factory=list)
    sendbuf_elems: int = 0
    recvbuf_elems: int = 0
    interleaved: bool = False
    tile_pdes: int = 4
    # multi-GPU overlap: tiles holding a cell of a face that feeds a remote
    # cut come first in tile_order (nbound of them); prime_dirs / post_dirs
    # list their remote packs (dst_kind 1) first (prime_remote / post_remote)
    tile_order: np.ndarray = None
    nbound: int = 0
    prime_remote: int = 0
    post_remote: int = 0
    small: bool = False             # one-launch small schedule (hb_small.cu)
    small_max_cells: int = 0
    band_segs: np.ndarray = None    # tile-perimeter cells (paired stages)
    band_max_len: int = 0
    fused: bool = False             # paired stages (hb_pair.cu)

    def elem(self, gid, n, p, j, i):
        """Slot element index of (n, p, j, i) -- array coordinates -- of block gid."""
        lb = self.local_index[gid]
        return self.base[lb] + (n * NPDE + p) * self.ps[lb] + j * self.rs[lb] + ROW_LEAD + i

    def block_view(self, gid):
        """(offset, shape, strides) in elements viewing a slot as the block's
        (planes, npde, nj+2, ni+2) array, halos included."""
        lb = self.local_index[gid]
        b = self.blocks[lb]
        return (self.base[lb] + ROW_LEAD, (self.planes, NPDE, b.nj + 2, b.ni + 2),
                (NPDE * self.ps[lb], self.ps[lb], self.rs[lb], 1))

    def block_extent(self, gid):
        """(start, length) of the block's region of a slot."""
        lb = self.local_index[gid]
        b = self.blocks[lb]
        return self.base[lb], self.planes * NPDE * (b.nj + 2) * self.pitch[lb]


def _interior_cell(spec, face, k):
    """(j, i) array coordinates of interior face cell k (1-based along the face)."""
    return {"south": (1, k), "north": (spec.nj, k), "west": (k, 1), "east": (k, spec.ni)}[face]


def _halo_cell(spec, face, k):
    return {"south": (0, k), "north": (spec.nj + 1, k), "west": (k, 0),
            "east": (k, spec.ni + 1)}[face]


def build_rank_layout(topology, partition, plan, rank, planes, tile_rows=None,
                      interleaved=None, tile_pdes=None, fused=None, small=None):
    """Device layout of one rank's blocks.

    interleaved=False: plane-major slots, (n, p) planes of (nj+2) x pitch;
    interleaved=True: row j of all (n, p) planes stored contiguously.
    Default: the INTERLEAVED module setting.
    """
    owned = [topology.blocks[g] for g in partition.blocks_of(rank)]
    owned.sort(key=lambda b: b.id)
    if not owned:
        raise ValueError(f"rank {rank} owns no blocks")
    local_index = {b.id: k for k, b in enumerate(owned)}
    tpd = tile_pdes or choose_tile_pdes(owned)
    tj = tile_rows or choose_tile_rows(owned, tpd, stage_grid_ctas(owned, planes, tpd, fused))
    inter = INTERLEAVED if interleaved is None else bool(interleaved)

    pitch, ps, rs, base = [], [], [], []
    off = 0
    for b in owned:
        pt = _round_up(ROW_LEAD + b.ni + 2, 8)
        pitch.append(pt)
        ps.append(pt if inter else (b.nj + 2) * pt)
        rs.append(planes * NPDE * pt if inter else pt)
        base.append(off)
        off = _round_up(off + planes * NPDE * (b.nj + 2) * pt, BLOCK_ALIGN)
    # bulk row copies of the last strip may run a few elements past a row end
    slot_elems = off + SLOT_TAIL

    table = np.zeros(len(owned), dtype=native.BLOCK_DTYPE)
    tile_block = []
    sxy_parts, sxy_off = [], 0
    ntile = 0
    for k, b in enumerate(owned):
        ti = -(-b.ni // native.TILE_COLS[tpd])
        tjn = -(-b.nj // tj)
        nt = ti * tjn * (NPDE // tpd)          # strips x row tiles x pde groups
        nu_h2, adv_2h = stencil_coefficients(b.h)
        spitch = _round_up(b.ni, 4)
        for name, value in (("base", base[k]), ("ps", ps[k]), ("rs", rs[k]), ("ni", b.ni), ("nj", b.nj),
                            ("pitch", pitch[k]), ("gid", b.id), ("tiles_i", ti),
                            ("tiles_j", tjn), ("tile_begin", ntile),
                            ("ntiles", nt),
                            ("nu_h2", nu_h2), ("adv_2h", adv_2h), ("h", b.h),
                            ("sxy_off", sxy_off), ("sxy_pitch", spitch)):
            table[name][k] = value
        table["face_off"][k] = -1
        tile_block += [k] * nt
        ntile += nt
        # the (nj, sxy_pitch) forcing table is formed on the device from these
        # two vectors (solver.DeviceRank): sxy[j, i] = sx[i] * sy[j]
        sxy_parts.append(forcing_vectors(b))
        sxy_off += b.nj * spitch

    layout = RankLayout(planes=planes, blocks=owned, local_index=local_index, pitch=pitch, ps=ps,
                        rs=rs, base=base, slot_elems=slot_elems, tile_rows=tj, block_table=table,
                        interleaved=inter, tile_pdes=tpd,
                        tile_block=np.asarray(tile_block, dtype=np.int32), total_tiles=ntile,
                        sxy=sxy_parts, sxy_size=sxy_off, faces=np.zeros(0, native.FACE_TARGET_DTYPE),
                        prime_dirs=np.zeros(0, native.HALO_DIR_DTYPE),
                        unpack_dirs=np.zeros(0, native.HALO_DIR_DTYPE),
                        post_dirs=np.zeros(0, native.HALO_DIR_DTYPE),
                        force_segs=np.zeros(0, native.FORCE_SEG_DTYPE))
    _build_routes(layout, topology, plan, rank)
    _build_force_segments(layout)
    _build_band(layout, fused)
    _build_tile_order(layout, topology, plan, rank)
    _choose_small(layout, small)
    return layout


def small_eligible(layout):
    """The one-launch small schedule (hb_small.cu): single stages, no remote
    cut (its grid barriers cannot wait on NCCL), a templated odd P <= 9."""
    return (not layout.fused and not layout.sends and not layout.recvs
            and layout.planes in (1, 3, 5, 7, 9) and os.environ.get("HBGPU_SMALL", "1") != "0")


def _choose_small(layout, small):
    """Auto: up to SMALL_MAX_UNITS units per stage, where launches, pipeline
    fill and drain dominate the per-stage TMA kernels.  Measured on one B200
    (bench --schedule small / single, 50 iterations): C0 1.68 vs 0.88 G
    units/s; C1 22.0 vs 29.4 G and C2 16.1 vs 32.7 G -- from C1's size the
    per-stage kernels win, so the threshold sits between C0 and C1."""
    units = sum(b.ni * b.nj for b in layout.blocks) * layout.planes * NPDE
    ok = small_eligible(layout)
    layout.small = ok and units <= SMALL_MAX_UNITS if small is None else bool(small) and ok
    layout.small_max_cells = max(b.ni * b.nj for b in layout.blocks)


def tile_box(layout, t):
    """(local block, first column, last column, first row, last row) of tile t
    (the decode_tile of hb_tma.cuh)."""
    k = int(layout.tile_block[t])
    b = layout.blocks[k]
    row = layout.block_table[k]
    local = t - int(row["tile_begin"])
    tiles_i = int(row["tiles_i"])
    width = native.TILE_COLS[layout.tile_pdes]
    i0 = (local % tiles_i) * width + 1
    rest = local // tiles_i
    j0 = (rest // (NPDE // layout.tile_pdes)) * layout.tile_rows + 1
    return k, i0, min(i0 + width - 1, b.ni), j0, min(j0 + layout.tile_rows - 1, b.nj)


def _build_tile_order(layout, topology, plan, rank):
    """Boundary tiles first: a tile is a boundary tile when it holds a cell
    of a face range that feeds a remote cut, i.e. a value this rank sends.
    The engine runs those tiles, packs the send buffer and starts the NCCL
    exchange on its communication stream, and only then runs the interior
    tiles, which overlap the transfer (hb_runtime.cu run_split).  Both lists
    keep the natural (block, row tile, strip) order."""
    sends = rank_routes(plan, rank).sends
    faces = {}
    for d in sends:
        faces.setdefault(layout.local_index[d.src_block], []).append((d.src_face, d.src_lo, d.src_hi))
    bound, inner = [], []
    for t in range(layout.total_tiles):
        k, i0, i1, j0, j1 = tile_box(layout, t)
        b = layout.blocks[k]
        hit = False
        for face, lo, hi in faces.get(k, ()):
            if face == "south" and j0 == 1 or face == "north" and j1 == b.nj:
                hit = hit or (i0 <= hi and lo <= i1)
            elif face == "west" and i0 == 1 or face == "east" and i1 == b.ni:
                hit = hit or (j0 <= hi and lo <= j1)
        (bound if hit else inner).append(t)
    layout.tile_order = np.asarray(bound + inner, dtype=np.int32)
    layout.nbound = len(bound)

    # remote packs first, so the engine can issue them right after the
    # boundary tiles and the local copies after the interior ones
    def remote_first(dirs):
        remote = dirs["dst_kind"] == 1
        return np.concatenate([dirs[remote], dirs[~remote]]), int(remote.sum())

    layout.prime_dirs, layout.prime_remote = remote_first(layout.prime_dirs)
    layout.post_dirs, layout.post_remote = remote_first(layout.post_dirs)


def fused_eligible(blocks, planes, tile_pdes):
    """Paired stages need P <= MAX_PAIR_P (shared memory), full strips
    (every ni a multiple of the strip width, so every lane is live), and
    nu/h^2 >= 1 in every block: the paired kernel drops the reference's
    signed-zero terms, which is exact only when t*nu_h2 cannot underflow to
    zero (hb_pair.cu stage_point)."""
    if os.environ.get("HBGPU_FUSED", "1") == "0":
        return False
    width = native.TILE_COLS[tile_pdes]
    return (planes <= native.MAX_PAIR_P and all(b.ni % width == 0 for b in blocks)
            and all(stencil_coefficients(b.h)[0] >= 1.0 for b in blocks))


def _build_band(layout, fused):
    """Runs of cells where hbgpu_band computes the first stage of a pair:
    the first and last row of every row tile (read across row-tile edges)
    and the face columns that feed a cut (forwarded into the neighbours'
    band halos, read across strip edges on block faces)."""
    eligible = fused_eligible(layout.blocks, layout.planes, layout.tile_pdes)
    # hbgpu_band takes one segment per grid row (gridDim.y <= 65535)
    nsegs = sum(len({r for j0 in range(1, b.nj + 1, layout.tile_rows)
                     for r in (j0, min(j0 + layout.tile_rows - 1, b.nj))}) + 2 for b in layout.blocks)
    eligible = eligible and nsegs <= MAX_BAND_SEGS
    if fused is None:
        units = sum(b.ni * b.nj for b in layout.blocks) * layout.planes * NPDE
        layout.fused = eligible and units >= FUSED_MIN_UNITS
    else:
        layout.fused = bool(fused) and eligible
    segs = []
    for k, b in enumerate(layout.blocks):
        rows = sorted({r for j0 in range(1, b.nj + 1, layout.tile_rows)
                       for r in (j0, min(j0 + layout.tile_rows - 1, b.nj))})
        # strip-edge columns inside a block are computed by the paired kernel's
        # edge warp; the band covers the face columns that feed a cut
        face = layout.block_table["face_off"][k]
        cols = sorted({c for c, fi in ((1, 2), (b.ni, 3)) if face[fi] >= 0})
        segs += [(k, 0, r, 1, b.ni, 0) for r in rows]
        # two adjacent face columns (a block 2 cells wide) go as one
        # two-column run, whose stencil reads overlap
        c = 0
        while c < len(cols):
            if c + 1 < len(cols) and cols[c + 1] == cols[c] + 1:
                segs.append((k, 2, 1, cols[c], b.nj, 0))
                c += 2
            else:
                segs.append((k, 1, 1, cols[c], b.nj, 0))
                c += 1
    layout.band_segs = np.array(segs, dtype=native.BAND_SEG_DTYPE)
    layout.band_max_len = max(max(b.ni, b.nj) for b in layout.blocks)


def _face_stride(layout, gid, face):
    lb = layout.local_index[gid]
    return 1 if face in ("south", "north") else layout.rs[lb]


def _build_routes(layout, topology, plan, rank):
    ds = plan.datasize
    routes = rank_routes(plan, rank)
    blocks = topology.blocks
    planes = layout.planes

    # send / receive segments grouped by peer (ascending), plan order inside
    def segments(dirs, peer_of):
        order = sorted(range(len(dirs)), key=lambda k: (peer_of(dirs[k]), k))
        offs, msgs, pos = {}, [], 0
        for k in order:
            d = dirs[k]
            offs[k] = pos
            n = d.length * ds
            if msgs and msgs[-1][0] == peer_of(d):
                msgs[-1][2] += n
            else:
                msgs.append([peer_of(d), pos, n])
            pos += n
        return offs, [tuple(m) for m in msgs], pos

    send_off, layout.sends, layout.sendbuf_elems = segments(routes.sends, lambda d: d.recv_rank)
    recv_off, layout.recvs, layout.recvbuf_elems = segments(routes.recvs, lambda d: d.sender_rank)

    # face-target pool: one entry per cell of every owned face that feeds a
    # cut.  The stage kernel's consumer warps forward south / north rows as
    # they compute them; west / east columns are forwarded by the TMA store
    # warp from the staged output row (update stages) or, after the first
    # stage, by one strided copy pass (post_dirs) -- a single-lane scatter of
    # P*4 values in every row of the boundary strips would stall the tile.
    face_base = {}
    size = 0
    feeding = [(d, True) for d in routes.local] + [(d, False) for d in routes.sends]
    for d, _ in feeding:
        key = (d.src_block, d.src_face)
        if key not in face_base:
            face_base[key] = size
            size += blocks[d.src_block].face_extent(d.src_face)
    faces = np.zeros(size, dtype=native.FACE_TARGET_DTYPE)
    send_index = {id(d): k for k, d in enumerate(routes.sends)}
    for d, is_local in feeding:
        fb = face_base[(d.src_block, d.src_face)]
        e = np.arange(d.length, dtype=np.int64)
        k = (d.src_hi - e) if d.src_reversed else (d.src_lo + e)      # source face index
        if is_local:
            kd = (d.dst_hi - e) if d.dst_reversed else (d.dst_lo + e)  # halo face index
            spec = blocks[d.dst_block]
            lb = layout.local_index[d.dst_block]
            hj, hi = {"south": (0, kd), "north": (spec.nj + 1, kd), "west": (kd, 0),
                      "east": (kd, spec.ni + 1)}[d.dst_face]
            off = layout.base[lb] + hj * layout.rs[lb] + ROW_LEAD + hi
            # a west halo cell is the last element of its 32-byte sector (the
            # rest is row lead); an east one is the first when ni % 4 == 0 (the
            # rest is row padding): such a target may be written as a whole
            # sector, which spares L2 the partial-sector fill
            if d.dst_face == "west" or (d.dst_face == "east" and spec.ni % 4 == 0):
                off = off | SECTOR_TARGET
            faces["off"][fb + k - 1] = off
            faces["ps"][fb + k - 1] = layout.ps[lb]
        else:
            faces["off"][fb + k - 1] = send_off[send_index[id(d)]] + e * ds
            faces["ps"][fb + k - 1] = -1
    layout.faces = faces
    from .topology import FACE_INDEX
    for (gid, face), fb in face_base.items():
        layout.block_table["face_off"][layout.local_index[gid], FACE_INDEX[face]] = fb

    def slot_run(gid, face, first_k, reversed_, halo):
        spec = blocks[gid]
        cell = _halo_cell if halo else _interior_cell
        j, i = cell(spec, face, first_k)
        step = _face_stride(layout, gid, face)
        return layout.elem(gid, 0, 0, j, i), (-step if reversed_ else step), \
            layout.ps[layout.local_index[gid]]

    def sector_dst(gid, face):
        # a west halo cell is the last of its 32-byte sector (the rest is row
        # lead), an east one the first when ni % 4 == 0 (the rest padding)
        return native.HALO_SECTOR_DST if face == "west" or (face == "east" and blocks[gid].ni % 4 == 0) else 0

    prime = []
    for d in routes.local:
        s_off, s_es, s_vs = slot_run(d.src_block, d.src_face, d.src_index(0), d.src_reversed, False)
        t_off, t_es, t_vs = slot_run(d.dst_block, d.dst_face, d.dst_index(0), d.dst_reversed, True)
        prime.append((s_off, s_es, s_vs, t_off, t_es, t_vs, d.length, 0, 0, sector_dst(d.dst_block, d.dst_face)))
    for k, d in enumerate(routes.sends):
        s_off, s_es, s_vs = slot_run(d.src_block, d.src_face, d.src_index(0), d.src_reversed, False)
        prime.append((s_off, s_es, s_vs, send_off[k], ds, 1, d.length, 0, 1, 0))
    post = [row for row, d in zip(prime, list(routes.local) + list(routes.sends))
            if d.src_face in ("west", "east")]
    unpack = []
    for k, d in enumerate(routes.recvs):
        t_off, t_es, t_vs = slot_run(d.dst_block, d.dst_face, d.dst_index(0), d.dst_reversed, True)
        unpack.append((recv_off[k], ds, 1, t_off, t_es, t_vs, d.length, 2, 0, sector_dst(d.dst_block, d.dst_face)))
    layout.prime_dirs = np.array(prime, dtype=native.HALO_DIR_DTYPE) if prime else \
        np.zeros(0, native.HALO_DIR_DTYPE)
    layout.unpack_dirs = np.array(unpack, dtype=native.HALO_DIR_DTYPE) if unpack else \
        np.zeros(0, native.HALO_DIR_DTYPE)
    layout.post_dirs = np.array(post, dtype=native.HALO_DIR_DTYPE) if post else \
        np.zeros(0, native.HALO_DIR_DTYPE)
    del planes


def _build_force_segments(layout):
    segs = []
    for b in layout.blocks:
        lb = layout.local_index[b.id]
        for face, body in b.body_faces:
            j, i = _interior_cell(b, face, 1)
            segs.append((layout.elem(b.id, 0, 0, j, i), _face_stride(layout, b.id, face),
                         layout.ps[lb], b.face_extent(face), body, b.h))
    layout.force_segs = np.array(segs, dtype=native.FORCE_SEG_DTYPE) if segs else \
        np.zeros(0, native.FORCE_SEG_DTYPE)
