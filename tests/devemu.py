"""Numpy model of libhbgpu's table-driven data movement -- TEST INFRASTRUCTURE.

It executes one rank's schedule exactly as hb_runtime.cu does (slot rotation
A->B->C->B->A, fused halo forwarding through the face-target pool, priming
halo directions, one message per peer and stage, unpack directions), but with
the stage arithmetic delegated to the oracle.  Running it on 1 or 2 gloo ranks
checks the device layout tables and the NCCL message pairing built by
paper_1304_7654_b200.devlayout without a GPU.
"""

from __future__ import annotations

import numpy as np

import oracle
from paper_1304_7654_b200 import hbop
from paper_1304_7654_b200.devlayout import ROW_LEAD, build_rank_layout
from paper_1304_7654_b200.topology import FACE_INDEX

STAGE_IN = (0, 1, 2, 1)
STAGE_OUT = (1, 2, 1, 0)


class RankEmulator:
    def __init__(self, case, topology, partition, plan, rank, initial=None):
        self.case = case
        self.P = case.planes
        self.L = build_rank_layout(topology, partition, plan, rank, self.P)
        self.slots = [np.zeros(self.L.slot_elems) for _ in range(3)]
        self.sendbuf = np.zeros(max(1, self.L.sendbuf_elems))
        self.recvbuf = np.zeros(max(1, self.L.recvbuf_elems))
        self.dmat = np.ascontiguousarray(hbop.spectral_matrix(case.nharms, case.omega).matrix)
        self.coefs = hbop.RKScheme(case.dtau).stage_coefficients()
        for b in self.L.blocks:
            ic = initial(b, self.P, 4) if initial else oracle.initial_values(b, self.P)
            self.view(0, b.id)[:, :, 1:b.nj + 1, 1:b.ni + 1] = ic
        self.force_hist = []

    def view(self, slot, gid):
        off, shape, strides = self.L.block_view(gid)
        base = self.slots[slot]
        return np.lib.stride_tricks.as_strided(base[off:], shape, tuple(8 * s for s in strides),
                                               writeable=True)

    def _buf(self, kind, slot):
        return {0: self.slots[slot], 1: self.sendbuf, 2: self.recvbuf}[kind]

    def halo(self, dirs, slot):
        nv = 4 * self.P
        for d in dirs:
            src, dst = self._buf(int(d["src_kind"]), slot), self._buf(int(d["dst_kind"]), slot)
            for e in range(int(d["length"])):
                for v in range(nv):
                    dst[d["dst_off"] + e * d["dst_es"] + v * d["dst_vs"]] = \
                        src[d["src_off"] + e * d["src_es"] + v * d["src_vs"]]

    def stage(self, s):
        """hbgpu_stage: residual + update of every owned block, then forwarding."""
        src, out = STAGE_IN[s], STAGE_OUT[s]
        new = {}
        for b in self.L.blocks:
            q = np.ascontiguousarray(self.view(src, b.id))
            q0 = np.ascontiguousarray(self.view(0, b.id)) if s else q.copy()
            resid = np.zeros((self.P, 4, b.nj, b.ni))
            oracle.residual_into(q, self.dmat, oracle.forcing_values(b, self.P), b.h, resid,
                                 0, self.P, 1, b.nj + 1)
            oracle.update(q, q0, resid, self.coefs[s], False, 0, self.P, 1, b.nj + 1)
            new[b.id] = q
        for b in self.L.blocks:
            self.view(out, b.id)[:, :, 1:b.nj + 1, 1:b.ni + 1] = new[b.id][:, :, 1:b.nj + 1, 1:b.ni + 1]
        # south / north rows from the consumer warps; west / east columns from
        # the store warp in the update stages, the post pass after stage 0
        self._forward(out, new, columns=s > 0)
        if s == 0:
            self.halo(self.L.post_dirs, out)

    def _forward(self, out, new, columns=True):
        faces, tbl = self.L.faces, self.L.block_table
        for k, b in enumerate(self.L.blocks):
            for face, fi in FACE_INDEX.items():
                base = int(tbl["face_off"][k, fi])
                if base < 0 or (face in ("west", "east") and not columns):
                    continue
                for c in range(b.face_extent(face)):
                    off, ps = int(faces["off"][base + c]) & ~(1 << 62), int(faces["ps"][base + c])
                    if ps == 0:
                        continue
                    j, i = {"south": (1, c + 1), "north": (b.nj, c + 1), "west": (c + 1, 1),
                            "east": (c + 1, b.ni)}[face]
                    for n in range(self.P):
                        for p in range(4):
                            v = new[b.id][n, p, j, i]
                            if ps > 0:
                                self.slots[out][off + (n * 4 + p) * ps] = v
                            else:
                                self.sendbuf[off + n * 4 + p] = v

    def forces(self):
        """forces_kernel on slot A: per-rank partials in reference order."""
        fields = {b.id: np.ascontiguousarray(self.view(0, b.id)) for b in self.L.blocks}
        self.force_hist.append(oracle.compute_forces(fields, self.L.blocks, self.P, self.case.nbody))

    def fields(self):
        return {b.id: np.ascontiguousarray(self.view(0, b.id)) for b in self.L.blocks}


def run_schedule(emu, iterations, exchange):
    """The engine's schedule; `exchange(emu, slot)` moves the remote payloads
    (send buffer -> peers -> receive buffer) and must then unpack."""
    emu.halo(emu.L.prime_dirs, 0)
    exchange(emu, 0)
    for _ in range(iterations):
        for s in range(4):
            emu.stage(s)
            exchange(emu, STAGE_OUT[s])
        emu.forces()
    return emu
