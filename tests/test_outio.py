"""Restart / flowtec output: layouts, bytes, counters.

CPU: the record layouts and the oracle's file images are pinned to files the
reference itself wrote (tests/golden/outputs.json: sha256 per file); marker
validation, read-back and the ownership / write-op rules follow the
reference's tests/test_outio.py.
GPU: run_case(out_dir=...) writes the files from device memory
(hbgpu_pack_records); they must be byte-identical to the oracle's images of
the oracle's fields and, on a host whose inputs match the fixtures, to the
reference's own files.
"""

import hashlib
import json
import os
import struct

import numpy as np
import pytest

import oracle
import outio_oracle
from paper_1304_7654_b200 import (BlockSpec, CaseConfig, CutSide, CutSpec, PlanError, RunSpec,
                                  baseline_workload, build_topology, pair_case, run_case, tc_tiny)
from paper_1304_7654_b200.exceptions import WriteError
from paper_1304_7654_b200.outio import (WriteMode, all_layouts, assign_records, compute_layout,
                                        create_output_files, read_block_plane, read_record,
                                        validate_record_ownership, write_ops)

GOLD = os.path.join(os.path.dirname(__file__), "golden")
with open(os.path.join(GOLD, "outputs.json")) as fh:
    OUT = json.load(fh)


def _reversed_pair():
    return pair_case(6, 5, 2, h=0.2, dtau=0.01, reversed_cut=True, nbody=1,
                     bodies=((1, "north", 0),), name="pair-reversed")


def _self_cut_reversed():
    blk = BlockSpec(0, 12, 9, 0.5, 0.25, 0.05)
    return CaseConfig(nharms=2, npde=4, iterations=5, dtau=0.0005, omega=1.0, nbody=0,
                      blocks=[blk], cuts=[CutSpec(CutSide(0, "north", 2, 7), CutSide(0, "south", 3, 8),
                                                  reversed=True)], name="self-cut-reversed")


RUNS = {   # golden name -> (builder, seeded workload key)
    "tc-tiny-8": (tc_tiny, None),
    "tc-tiny-3-per-value-r2": (tc_tiny, None),
    "pair-reversed-6-r2": (_reversed_pair, None),
    "self-cut-reversed-5": (_self_cut_reversed, None),
    "C0-seeded-10": (lambda: baseline_workload("C0").case, "C0"),
}


def _input_hash(case, initial):
    h = hashlib.sha256()
    planes = 2 * case.nharms + 1
    for spec in sorted(case.blocks, key=lambda s: s.id):
        ic = initial(spec, planes, 4) if initial is not None else oracle.initial_values(spec, planes)
        h.update(np.ascontiguousarray(ic).tobytes())
        h.update(oracle.forcing_values(spec, planes).tobytes())
    h.update(oracle.spectral_matrix(case.nharms, case.omega).tobytes())
    return h.hexdigest()[:16]


def _setup(name):
    build, wl = RUNS[name]
    case = build()
    initial = baseline_workload(wl).initial if wl else None
    return case, initial, _input_hash(case, initial) == OUT[name]["input_hash"]


def _sha(data):
    return hashlib.sha256(data).hexdigest()


# ---------------------------------------------------------------------------
# CPU
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name", sorted(OUT))
def test_layouts_match_reference(name):
    case, _, _ = _setup(name)
    layouts = all_layouts(build_topology(case), case.nharms, case.npde)
    want = OUT[name]["layouts"]
    assert [l.filename for l in layouts] == ["restart.bin"] + [f"flowtec_{n}.bin" for n in range(case.planes)]
    for l in layouts:
        g = want[l.filename]
        assert (l.kind, l.plane, l.total_bytes) == (g["kind"], g["plane"], g["total_bytes"])
        assert [[r.block, r.plane, r.offset, r.nfloats] for r in l.records] == g["records"]
        assert OUT[name]["files"][l.filename]["bytes"] == l.total_bytes


@pytest.mark.parametrize("name", sorted(OUT))
def test_write_ops_and_activations_match_reference(name):
    case, _, _ = _setup(name)
    g = OUT[name]
    layouts = all_layouts(build_topology(case), case.nharms, case.npde)
    assert write_ops(layouts, [b.id for b in case.blocks], WriteMode(g["io"])) == g["write_ops"]
    assert g["activations"] == g["iterations"] + 1


@pytest.mark.parametrize("name", sorted(OUT))
def test_oracle_file_images_match_reference_files(name, oracle_mod):
    """Pins the checker: the oracle's fields, written by the oracle's writer,
    are the reference's files byte for byte."""
    case, initial, same_host = _setup(name)
    if not same_host:
        pytest.skip(f"{name}: this host's numpy sin/cos bits differ from the fixture's")
    res = oracle_mod.run(case, OUT[name]["iterations"], initial=initial, record_norms=False)
    images = outio_oracle.file_images(case.blocks, case.planes, res.fields)
    assert {k: _sha(v) for k, v in images.items()} == {k: v["sha256"] for k, v in OUT[name]["files"].items()}


def test_markers_read_back_and_corruption(tmp_path):
    case = tc_tiny()
    res = oracle.run(case, 1, record_norms=False)
    outio_oracle.write_files(tmp_path, case.blocks, case.planes, res.fields)
    topo = build_topology(case)
    restart, ft0 = all_layouts(topo, case.nharms)[:2]
    for spec in topo.blocks:
        for n in range(case.planes):
            got = read_block_plane(os.path.join(tmp_path, "restart.bin"), restart, spec, n)
            q = res.fields[spec.id]
            assert np.array_equal(got, np.transpose(q[n, :, 1:spec.nj + 1, 1:spec.ni + 1], (1, 2, 0)))
    got = read_block_plane(os.path.join(tmp_path, "flowtec_0.bin"), ft0, topo.blocks[0], 0)
    assert np.array_equal(got[:, :, 2], res.fields[0][0, 0, 1:-1, 1:-1])
    path = tmp_path / "restart.bin"
    raw = bytearray(path.read_bytes())
    rec = restart.records[0]
    assert struct.unpack("<I", raw[:4])[0] == rec.payload_bytes
    raw[0] ^= 0xFF
    path.write_bytes(bytes(raw))
    with pytest.raises(WriteError, match="marker"):
        read_record(str(path), restart, rec)


def test_create_files_sizes_and_unknown_kind(tmp_path):
    topo = build_topology(tc_tiny())
    layouts = all_layouts(topo, 1)
    create_output_files(tmp_path / "o", layouts)
    for l in layouts:
        assert os.path.getsize(tmp_path / "o" / l.filename) == l.total_bytes
    with pytest.raises(WriteError, match="unknown output kind"):
        compute_layout(topo, 1, 4, "vtk")


def test_record_ownership_rules():
    topo = build_topology(tc_tiny())
    (layout,) = compute_layout(topo, 1, 4, "restart")
    parts = assign_records(layout, [0, 1], 2)
    validate_record_ownership(parts)
    assert sum(len(p) for p in parts) == len(layout.records)
    with pytest.raises(PlanError, match="assigned to"):
        validate_record_ownership([parts[0], parts[0]])


def test_single_block_op_counts():
    blocks = (BlockSpec(0, 2, 2, 0.0, 0.0, 0.5),)
    topo = build_topology(CaseConfig(nharms=0, npde=4, iterations=1, dtau=0.1, omega=1.0, nbody=0,
                                     blocks=list(blocks), cuts=[]))
    (layout,) = compute_layout(topo, 0, 4, "restart")
    assert layout.total_bytes == 2 * 2 * 4 * 8 + 8
    assert write_ops([layout], [0], WriteMode.PER_VALUE) == 2 + 16
    assert write_ops([layout], [0], WriteMode.BUFFERED) == 3


# ---------------------------------------------------------------------------
# GPU
# ---------------------------------------------------------------------------

def _check_dir(d, case, want_images, golden=None):
    for name, data in want_images.items():
        got = open(os.path.join(d, name), "rb").read()
        assert got == data, f"{name} differs from the oracle's image"
        if golden is not None:
            assert _sha(got) == golden[name]["sha256"], f"{name} differs from the reference's file"


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(OUT))
@pytest.mark.parametrize("transport", ["fold", "loopback"])
def test_device_files_match_oracle_and_reference(name, transport, cuda, oracle_mod, tmp_path):
    case, initial, same_host = _setup(name)
    g = OUT[name]
    if transport == "loopback" and g["ranks"] == 1:
        pytest.skip("single-rank run")
    res = run_case(RunSpec(case=case, ranks=g["ranks"], iterations=g["iterations"], initial=initial,
                           io=WriteMode(g["io"]), out_dir=str(tmp_path / "out"),
                           extra_outputs=((str(tmp_path / "extra"), WriteMode.PER_VALUE),),
                           transport=transport))
    want = oracle_mod.run(case, g["iterations"], initial=initial, record_norms=False)
    images = outio_oracle.file_images(case.blocks, case.planes, want.fields)
    golden = g["files"] if same_host else None
    _check_dir(tmp_path / "out", case, images, golden)
    _check_dir(tmp_path / "extra", case, images, golden)
    layouts = all_layouts(build_topology(case), case.nharms)
    ids = [b.id for b in case.blocks]
    assert res.record.write_ops == write_ops(layouts, ids, WriteMode(g["io"])) + \
        write_ops(layouts, ids, WriteMode.PER_VALUE)
    assert res.record.activations == g["iterations"] + 2


@pytest.mark.gpu
def test_device_writer_chunking_and_ragged_blocks(cuda, oracle_mod, tmp_path):
    """Many small chunks (records split across staging buffers, runs of
    file-adjacent records) over blocks of different sizes."""
    from paper_1304_7654_b200 import DeviceRank, build_cut_plan, partition_blocks
    from paper_1304_7654_b200 import outio
    blocks = [BlockSpec(0, 37, 11, 0.0, 0.0, 0.05), BlockSpec(1, 64, 9, 1.85, 0.0, 0.05),
              BlockSpec(2, 5, 3, 0.0, 0.55, 0.05)]
    case = CaseConfig(nharms=2, npde=4, iterations=2, dtau=0.0005, omega=1.0, nbody=0,
                      blocks=blocks, cuts=[], name="ragged-out")
    res = run_case(RunSpec(case=case, iterations=2))
    topo = build_topology(case)
    part = partition_blocks(topo, 1)
    dr = DeviceRank(case, topo, part, build_cut_plan(topo, part, case.nharms, 4), max_iters=2)
    try:
        dr.prime()
        dr.iterate(2)
        layouts = all_layouts(topo, case.nharms)
        create_output_files(tmp_path, layouts)
        for chunk in (40, 700, 5000):   # bytes: one record or less per chunk, and a few
            outio.write_output(dr, layouts, WriteMode.BUFFERED, str(tmp_path), chunk_bytes=chunk)
            _check_dir(tmp_path, case, outio_oracle.file_images(blocks, case.planes, res.fields))
    finally:
        dr.close()
