"""TEST INFRASTRUCTURE ONLY -- restart / flowtec files from host arrays.

A numpy restatement of the reference's record format (outio.py:1-22,
107-123 record_payload, 221-241 write_records) used as the checker for the
device writer (paper_1304_7654_b200/outio.py): tests/ write the oracle's
fields with it and compare bytes.  Pinned against files the reference
itself wrote (tests/golden/outputs.json, tests/test_outio.py).
"""

from __future__ import annotations

import os
import struct

import numpy as np


def record_bytes(kind, spec, q, plane):
    """Marker + payload + marker of one record; q has halos, shape (P, 4, nj+2, ni+2)."""
    nj, ni = spec.nj, spec.ni
    if kind == "restart":
        payload = np.transpose(q[plane, :, 1:nj + 1, 1:ni + 1], (1, 2, 0))
    else:
        xc = spec.x0 + (np.arange(1, ni + 1) - 0.5) * spec.h      # hbcore.py:126-127
        yc = spec.y0 + (np.arange(1, nj + 1) - 0.5) * spec.h
        payload = np.empty((nj, ni, 4))
        payload[:, :, 0] = xc[None, :]
        payload[:, :, 1] = yc[:, None]
        payload[:, :, 2] = q[plane, 0, 1:nj + 1, 1:ni + 1]
        payload[:, :, 3] = q[plane, 1, 1:nj + 1, 1:ni + 1]
    raw = np.ascontiguousarray(payload, dtype="<f8").tobytes()
    marker = struct.pack("<I", len(raw))
    return marker + raw + marker


def file_images(blocks, planes, fields):
    """{filename: bytes} of restart.bin and flowtec_<n>.bin; blocks ascending."""
    blocks = sorted(blocks, key=lambda b: b.id)
    images = {"restart.bin": b"".join(record_bytes("restart", b, fields[b.id], n)
                                      for b in blocks for n in range(planes))}
    for n in range(planes):
        images[f"flowtec_{n}.bin"] = b"".join(record_bytes("flowtec", b, fields[b.id], n) for b in blocks)
    return images


def write_files(out_dir, blocks, planes, fields):
    os.makedirs(out_dir, exist_ok=True)
    for name, data in file_images(blocks, planes, fields).items():
        with open(os.path.join(out_dir, name), "wb") as fh:
            fh.write(data)
