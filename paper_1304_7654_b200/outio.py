"""Restart and flowtec output written from device-resident fields.

The file format is the reference's (outio.py:1-22), byte for byte:

* a file is a dense sequence of records, one per (block, plane) in
  ``restart.bin`` (blocks ascending, planes inner) and one per block in each
  per-plane ``flowtec_<n>.bin``;
* a record is a 4-byte little-endian length prefix (payload bytes), the
  float64 payload and the same 4-byte suffix;
* restart payload: the block's interior values of plane n, rows outer,
  columns, variable innermost; flowtec payload per cell: (x, y, q0, q1).

Layout planning (compute_layout, create_output_files, read_record,
read_block_plane, assign_records, validate_record_ownership) mirrors the
reference's functions of the same names (outio.py:79-104, 185-206, 244-291).
The writer differs in where the bytes come from: ``write_output`` packs each
record's complete byte image on the GPU from the engine's result slot
(hbgpu_pack_records, csrc/hb_io.cu), moves it to pinned host memory and
writes each run of file-adjacent records with one positioned write from a
pool of host threads, so the device packs and copies chunk k+1 while the
host writes chunks k, k-1, ...  The
two reference write strategies (per-value, buffered) produce identical bytes
there and here; ``write_ops`` reports the positioned-write count the chosen
strategy defines (outio.py:221-241: 2 + nfloats or 3 per record), the
reference's counter.
"""

from __future__ import annotations

import os
import struct
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import native
from .exceptions import PlanError, WriteError

DOUBLE_SIZE = 8
MARKER_SIZE = 4
CHUNK_BYTES = 128 << 20      # device staging per chunk
WRITE_SLOTS = 6              # chunks in flight (staging buffers = writer threads)


class WriteMode(Enum):
    PER_VALUE = "per-value"
    BUFFERED = "buffered"


@dataclass(frozen=True)
class RecordSpec:
    block: int
    plane: int
    offset: int
    nfloats: int

    @property
    def payload_bytes(self):
        return self.nfloats * DOUBLE_SIZE

    @property
    def total_bytes(self):
        return self.payload_bytes + 2 * MARKER_SIZE


@dataclass(frozen=True)
class FileLayout:
    kind: str            # "restart" | "flowtec"
    plane: int | None
    filename: str
    records: tuple
    total_bytes: int

    def record_for(self, block, plane):
        for rec in self.records:
            if rec.block == block and rec.plane == plane:
                return rec
        raise KeyError((block, plane))


def compute_layout(topology, nharms, npde, kind):
    """Byte layouts of one output kind (ref outio.py:79-104): one FileLayout
    for the restart file, one per harmonic plane for flowtec."""
    planes = 2 * nharms + 1
    blocks = sorted(topology.blocks, key=lambda b: b.id)
    if kind == "restart":
        records, offset = [], 0
        for b in blocks:
            for n in range(planes):
                rec = RecordSpec(b.id, n, offset, b.ni * b.nj * npde)
                records.append(rec)
                offset += rec.total_bytes
        return (FileLayout("restart", None, "restart.bin", tuple(records), offset),)
    if kind == "flowtec":
        layouts = []
        for n in range(planes):
            records, offset = [], 0
            for b in blocks:
                rec = RecordSpec(b.id, n, offset, b.ni * b.nj * 4)
                records.append(rec)
                offset += rec.total_bytes
            layouts.append(FileLayout("flowtec", n, f"flowtec_{n}.bin", tuple(records), offset))
        return tuple(layouts)
    raise WriteError(f"unknown output kind {kind!r}")


def all_layouts(topology, nharms, npde=4):
    """Restart layout followed by the flowtec layouts (the driver's order)."""
    return compute_layout(topology, nharms, npde, "restart") + compute_layout(topology, nharms, npde, "flowtec")


def create_output_files(out_dir, layouts):
    """Create (truncate) every output file at its final size before ranks write."""
    os.makedirs(out_dir, exist_ok=True)
    for layout in layouts:
        with open(os.path.join(out_dir, layout.filename), "wb") as fh:
            fh.truncate(layout.total_bytes)


def _partition(extent, parts):
    base, rem = divmod(extent, parts)
    out, lo = [], 0
    for t in range(parts):
        size = base + (1 if t < rem else 0)
        out.append((lo, lo + size))
        lo += size
    return out


def assign_records(layout, owned_blocks, team_size):
    """Split a rank's records of one file into contiguous per-member runs
    (ref outio.py:185-189)."""
    owned = set(owned_blocks)
    records = [r for r in layout.records if r.block in owned]
    return [records[lo:hi] for lo, hi in _partition(len(records), team_size)]


def validate_record_ownership(assignments):
    """Reject plans in which a record belongs to more than one member
    (ref outio.py:192-202)."""
    seen = {}
    for tid, records in enumerate(assignments):
        for rec in records:
            key = (rec.block, rec.plane, rec.offset)
            if key in seen:
                raise PlanError(f"record (block {rec.block}, plane {rec.plane}) assigned to "
                                f"threads {seen[key]} and {tid}")
            seen[key] = tid


def write_ops(layouts, owned_blocks, mode):
    """Positioned writes the reference strategy issues for these records."""
    owned = set(owned_blocks)
    total = 0
    for layout in layouts:
        for rec in layout.records:
            if rec.block in owned:
                total += 3 if mode is WriteMode.BUFFERED else 2 + rec.nfloats
    return total


# ---------------------------------------------------------------------------
# device writer
# ---------------------------------------------------------------------------

def _xy_table(rank):
    """Per owned block: cell-centre x (ni values) then y (nj), as the
    reference's BlockState.xc / yc (hbcore.py:126-127)."""
    parts, offsets, off = [], [], 0
    for b in rank.layout.blocks:
        xc = b.x0 + (np.arange(1, b.ni + 1) - 0.5) * b.h
        yc = b.y0 + (np.arange(1, b.nj + 1) - 0.5) * b.h
        parts += [xc, yc]
        offsets.append(off)
        off += b.ni + b.nj
    return np.concatenate(parts) if parts else np.zeros(1), offsets


def _chunks(records, limit):
    chunk, size = [], 0
    for rec in records:
        if chunk and size + rec.total_bytes > limit:
            yield chunk
            chunk, size = [], 0
        chunk.append(rec)
        size += rec.total_bytes
    if chunk:
        yield chunk


def write_output(rank, layouts, mode, out_dir, chunk_bytes=CHUNK_BYTES, slots=WRITE_SLOTS):
    """Write this rank's records of every layout from its device result slot.

    Chunks of records are packed on the device into one of `slots` staging
    buffers, copied to pinned host memory and written by a pool of host
    threads (os.pwrite releases the GIL), so packing, PCIe and page-cache
    writes of different chunks overlap.  The files must exist at their final
    size (create_output_files).  Returns the write-op count of `mode`."""
    import torch
    lib = native.load()
    torch_dev = rank.device
    local = {b.id: k for k, b in enumerate(rank.layout.blocks)}
    spec_of = {b.id: b for b in rank.layout.blocks}
    xy, xy_off = _xy_table(rank)
    t_xy = torch.from_numpy(np.ascontiguousarray(xy, dtype=np.float64)).to(torch_dev)
    work = []
    for layout in layouts:
        recs = [r for r in layout.records if r.block in local]
        kind = native.RECORD_RESTART if layout.kind == "restart" else native.RECORD_FLOWTEC
        for chunk in _chunks(recs, chunk_bytes):
            work.append((layout, kind, chunk))
    if not work:
        return 0
    cap = max(sum(r.total_bytes for r in c) for _, _, c in work)
    cap = (cap + 7) // 8 * 8
    nslot = max(1, min(slots, len(work)))
    dev = [torch.empty(cap, dtype=torch.uint8, device=torch_dev) for _ in range(nslot)]
    host = [torch.empty(cap, dtype=torch.uint8, pin_memory=True) for _ in range(nslot)]
    done = [torch.cuda.Event() for _ in range(nslot)]
    busy = [None] * nslot
    stream = torch.cuda.current_stream(torch_dev)
    slot = rank.slots[0]
    fds = {}
    for layout in layouts:
        path = os.path.join(out_dir, layout.filename)
        try:
            fds[path] = os.open(path, os.O_RDWR)
        except OSError as exc:
            for fd in fds.values():
                os.close(fd)
            raise WriteError(f"cannot open {path}: {exc}") from exc
    pool = ThreadPoolExecutor(max_workers=nslot)
    try:
        for k, (layout, kind, chunk) in enumerate(work):
            s = k % nslot
            if busy[s] is not None:
                busy[s].result()          # the slot's previous chunk is on disk
            table = np.zeros(len(chunk), dtype=native.OUT_RECORD_DTYPE)
            pos = 0
            for t, rec in enumerate(chunk):
                table[t] = (local[rec.block], rec.plane, kind, 0, pos, xy_off[local[rec.block]])
                pos += rec.total_bytes
            t_table = torch.from_numpy(table.view(np.uint8).copy()).to(torch_dev)
            max_cells = max(spec_of[r.block].ni * spec_of[r.block].nj for r in chunk)
            native.check(lib.hbgpu_pack_records(slot.data_ptr(), rank.t_blocks.data_ptr(),
                                                t_table.data_ptr(), len(chunk), max_cells,
                                                t_xy.data_ptr(), dev[s].data_ptr(),
                                                stream.cuda_stream), "hbgpu_pack_records")
            host[s][:pos].copy_(dev[s][:pos], non_blocking=True)
            done[s].record(stream)
            path = os.path.join(out_dir, layout.filename)
            busy[s] = pool.submit(_write_chunk, done[s], host[s], chunk, fds[path], path)
        for f in busy:
            if f is not None:
                f.result()
    finally:
        pool.shutdown(wait=True)
        for fd in fds.values():
            os.close(fd)
    return write_ops(layouts, local, mode)


def _write_chunk(event, host, chunk, fd, path):
    """Positioned writes of one packed chunk, one per run of file-adjacent records."""
    event.synchronize()
    buf = host.numpy()
    pos = 0
    k = 0
    while k < len(chunk):
        start_rec, start_pos, length = chunk[k], pos, 0
        while k < len(chunk) and chunk[k].offset == start_rec.offset + length:
            length += chunk[k].total_bytes
            k += 1
        view = memoryview(buf[start_pos:start_pos + length])
        written = 0
        while written < length:
            try:
                n = os.pwrite(fd, view[written:], start_rec.offset + written)
            except OSError as exc:
                raise WriteError(f"write of {length} bytes at offset {start_rec.offset} "
                                 f"in {path} failed: {exc}") from exc
            written += n
        pos += length


# ---------------------------------------------------------------------------
# reading back (round-trip verification; ref outio.py:268-291)
# ---------------------------------------------------------------------------

def read_record(path, layout, record):
    """Read one record back, verifying both length markers."""
    with open(path, "rb") as fh:
        fh.seek(record.offset)
        blob = fh.read(record.total_bytes)
    if len(blob) != record.total_bytes:
        raise WriteError(f"{path}: short read at offset {record.offset}")
    prefix = struct.unpack("<I", blob[:MARKER_SIZE])[0]
    suffix = struct.unpack("<I", blob[-MARKER_SIZE:])[0]
    if prefix != record.payload_bytes or suffix != record.payload_bytes:
        raise WriteError(f"{path}: marker mismatch at offset {record.offset}: "
                         f"prefix={prefix} suffix={suffix} expected={record.payload_bytes}")
    return np.frombuffer(blob[MARKER_SIZE:-MARKER_SIZE], dtype="<f8").copy()


def read_block_plane(path, layout, block_spec, plane):
    """One record's payload in its natural (j, i, k) shape."""
    record = layout.record_for(block_spec.id, plane)
    values = read_record(path, layout, record)
    width = record.nfloats // (block_spec.ni * block_spec.nj)
    return values.reshape(block_spec.nj, block_spec.ni, width)
