"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

Run in the build container (the reference is only present there):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Outputs (committed):
  fingerprints.json  reference full-run fingerprints (fields incl. halos +
                     forces, sha256[:16]) and the hash of the host-computed
                     inputs (IC + forcing) they were produced from
  runs.npz           full reference fields / forces for small runs
  kernels.npz        reference _residual_kernel / _update_kernel outputs on
                     seeded random states, sub-ranges included
  host.json          reference partitions, cut plans, message forecasts,
                     case_text renderings and parse-error messages
  outputs.json       (--outputs) sha256 / size / record layout of the
                     restart and flowtec files the reference writes for a
                     few runs, with their write_ops counters
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from hbproxy import hbcore  # noqa: E402  (the reference)
from hbproxy.cases import (case_text, lattice_case, pair_case, stacked_pair_case,  # noqa: E402
                           tc1_mini, tc2_mini, tc_tiny, cut2500, ring_case)
from hbproxy.driver import RunSpec, run_case  # noqa: E402
from hbproxy.exchange import (ExchangeMode, ExchangeStrategy, build_cut_plan,  # noqa: E402
                              predicted_message_count)
from hbproxy.mesh import (BlockSpec, CaseConfig, CutSide, CutSpec, build_topology,  # noqa: E402
                          parse_case, partition_blocks)

from paper_1304_7654_b200 import builders as mine  # noqa: E402  (seeded IC of the C0..C4 maps)


def fingerprint(fields, forces):
    h = hashlib.sha256()
    for b in sorted(fields):
        h.update(np.ascontiguousarray(fields[b]).tobytes())
    for arr in (forces.cl, forces.cd, forces.cm):
        h.update(np.ascontiguousarray(arr).tobytes())
    return h.hexdigest()[:16]


def input_hash(case, initial=None):
    """Hash of the transcendental inputs the run consumes on this host."""
    h = hashlib.sha256()
    planes = 2 * case.nharms + 1
    for spec in sorted(case.blocks, key=lambda s: s.id):
        ic = (initial(spec, planes, 4) if initial is not None else
              hbcore.initial_values(spec, planes, 4, 0, planes, 1, spec.nj + 1))
        h.update(np.ascontiguousarray(ic).tobytes())
        h.update(hbcore.forcing_values(spec, planes, 4).tobytes())
    h.update(hbcore.spectral_matrix(case.nharms, case.omega).matrix.tobytes())
    return h.hexdigest()[:16]


def run_ref(case, iterations, initial=None, ranks=1):
    saved = hbcore.initial_values
    if initial is not None:
        def hook(spec, planes, npde, n_lo, n_hi, j_lo, j_hi):
            full = initial(spec, planes, npde)
            return full[n_lo:n_hi, :, j_lo - 1:j_hi - 1, :]
        hbcore.initial_values = hook
    try:
        return run_case(RunSpec(case=case, ranks=ranks, iterations=iterations))
    finally:
        hbcore.initial_values = saved


def steady_case():
    return CaseConfig(nharms=0, npde=4, iterations=12, dtau=0.01, omega=1.0, nbody=0,
                      blocks=[BlockSpec(id=0, ni=6, nj=5, x0=0.3, y0=-0.7, h=0.2)], cuts=[],
                      name="steady")


def reversed_pair():
    return pair_case(6, 5, 2, h=0.2, dtau=0.01, reversed_cut=True, nbody=1,
                     bodies=((1, "north", 0),), name="pair-reversed")


def self_cut_case():
    # C2-shaped O-grid wrap at desk scale: one block, east <-> west self-cut
    blk = BlockSpec(id=0, ni=24, nj=10, x0=0.0, y0=0.0, h=0.05, body_faces=(("south", 0),))
    cut = CutSpec(CutSide(0, "east", 1, 10), CutSide(0, "west", 1, 10))
    return CaseConfig(nharms=4, npde=4, iterations=5, dtau=0.0005, omega=0.12, nbody=1,
                      blocks=[blk], cuts=[cut], name="self-cut")


def reversed_self_cut_case():
    blk = BlockSpec(id=0, ni=12, nj=9, x0=0.5, y0=0.25, h=0.05)
    cut = CutSpec(CutSide(0, "north", 2, 7), CutSide(0, "south", 3, 8), reversed=True)
    return CaseConfig(nharms=2, npde=4, iterations=5, dtau=0.0005, omega=1.0, nbody=0,
                      blocks=[blk], cuts=[cut], name="self-cut-reversed")


RUNS = {
    # name: (builder, iterations, seeded-workload key or None, store full arrays)
    "tc-tiny-8": (tc_tiny, 8, None, True),
    "pair-reversed-6": (reversed_pair, 6, None, True),
    "steady-12": (steady_case, 12, None, True),
    "self-cut-5": (self_cut_case, 5, None, True),
    "self-cut-reversed-5": (reversed_self_cut_case, 5, None, True),
    "tc1-mini-20": (tc1_mini, 20, None, False),
    "tc2-mini-10": (tc2_mini, 10, None, False),
    "C0-seeded-10": (lambda: mine.baseline_workload("C0").case, 10, "C0", True),
    "tc1-mini-100": (tc1_mini, 100, None, False),
}


def make_runs():
    fps, arrays = {}, {}
    for name, (build, iters, wl_key, store) in RUNS.items():
        case = build()
        initial = mine.baseline_workload(wl_key).initial if wl_key else None
        res = run_ref(case, iters, initial)
        fps[name] = {"fingerprint": fingerprint(res.fields, res.forces),
                     "input_hash": input_hash(case, initial), "iterations": iters,
                     "max_abs_q": float(max(np.abs(q).max() for q in res.fields.values()))}
        if store:
            for b, q in res.fields.items():
                arrays[f"{name}/field/{b}"] = q
            arrays[f"{name}/forces"] = np.stack([res.forces.cl, res.forces.cd, res.forces.cm])
        print(name, fps[name])
    return fps, arrays


def make_kernels():
    out = {}
    rng = np.random.default_rng(20240601)
    for tag, (ni, nj, nharms, h) in {"p5": (7, 6, 2, 0.2), "p9": (37, 19, 4, 0.05),
                                      "p3": (9, 4, 1, 0.125)}.items():
        spec = BlockSpec(id=0, ni=ni, nj=nj, x0=10.0, y0=20.0, h=h)
        planes = 2 * nharms + 1
        block = hbcore.BlockState(spec, planes)
        block.q[:] = rng.normal(size=block.q.shape)
        deriv = hbcore.spectral_matrix(nharms, 1.3)
        out[f"{tag}/q"] = block.q.copy()
        out[f"{tag}/forcing"] = block.forcing.copy()
        out[f"{tag}/dmat"] = deriv.matrix.copy()
        out[f"{tag}/meta"] = np.array([ni, nj, nharms, h, 1.3])
        hbcore.residual_into(block, deriv, 0, planes, 1, nj + 1)
        out[f"{tag}/resid_full"] = block.resid.copy()
        block.resid[:] = 0.0
        hbcore.residual_into(block, deriv, 1, planes, 2, nj)  # a sub-range
        out[f"{tag}/resid_sub"] = block.resid.copy()
        # update with snapshot on the full residual
        hbcore.residual_into(block, deriv, 0, planes, 1, nj + 1)
        block.q0[:] = rng.normal(size=block.q0.shape)
        q0_before = block.q0.copy()
        hbcore.update_stage(block, 0.0123, 0, planes, 1, nj + 1, snapshot=True)
        out[f"{tag}/upd_snap_q"] = block.q.copy()
        out[f"{tag}/upd_snap_q0"] = block.q0.copy()
        block.q0[:] = q0_before
        q_before = rng.normal(size=block.q.shape)
        block.q[:] = q_before
        out[f"{tag}/upd_q_before"] = q_before
        out[f"{tag}/upd_q0"] = q0_before
        hbcore.update_stage(block, 0.5, 0, planes, 2, nj, snapshot=False)
        out[f"{tag}/upd_sub_q"] = block.q.copy()
    return out


def _plan_rows(plan):
    rows = []
    for cut in plan.cuts:
        for d in cut.directions:
            rows.append([d.cut_index, d.direction, d.sender_rank, d.recv_rank, d.src_block, d.src_face,
                         d.src_lo, d.src_hi, d.src_reversed, d.dst_block, d.dst_face, d.dst_lo,
                         d.dst_hi, d.dst_reversed, d.length, d.local])
    return rows


def make_host():
    cases = {"tc-tiny": tc_tiny(), "tc1-mini": tc1_mini(), "tc2-mini": tc2_mini(),
             "cut2500": cut2500(), "pair-reversed": reversed_pair(), "self-cut": self_cut_case(),
             "self-cut-reversed": reversed_self_cut_case(),
             "ring5": ring_case(5, 8, 4, 1, h=0.1, dtau=0.01),
             "stacked": stacked_pair_case(12, 3, 2, h=0.1, dtau=0.01, nbody=1, bodies=((1, "north", 0),))}
    for key in ("C0", "C1", "C2", "C3", "C4"):
        cases[key] = ref_baseline(key)
    host = {"cases": {}}
    for name, ref_case in cases.items():
        topo = build_topology(ref_case)
        entry = {"case_text": case_text(ref_case), "partitions": {}, "plans": {}, "forecast": {}}
        for ranks in (1, 2, 3, 4, 8):
            if ranks > topo.nblocks:
                continue
            part = partition_blocks(topo, ranks)
            plan = build_cut_plan(topo, part, ref_case.nharms, ref_case.npde)
            entry["partitions"][ranks] = list(part.rank_of_block)
            entry["plans"][ranks] = _plan_rows(plan)
            f_agg = predicted_message_count(plan, ExchangeStrategy(ExchangeMode.AGGREGATED_CUT))
            f_per = predicted_message_count(plan, ExchangeStrategy(ExchangeMode.PER_ELEMENT))
            entry["forecast"][ranks] = [f_agg.messages, f_agg.nbytes, f_per.messages, f_per.nbytes]
        host["cases"][name] = entry
    # unequal blocks (LPT)
    blocks = tuple(BlockSpec(id=k, ni=c // 2, nj=2, x0=0.0, y0=float(k), h=1.0)
                   for k, c in enumerate([8, 4, 4, 12, 6, 6, 2]))
    from hbproxy.mesh import Topology
    topo = Topology(blocks=blocks, cuts=(), nbody=0)
    host["lpt"] = {r: list(partition_blocks(topo, r).rank_of_block) for r in range(1, 8)}
    host["parse_errors"] = make_parse_errors()
    return host


def ref_baseline(key):
    """SURVEY.md §8d's C0..C4 topologies built with the REFERENCE's own types/builders."""
    dt = lambda h: 4.096 * h * h  # noqa: E731
    if key == "C0":
        h = 1.0 / 64
        return CaseConfig(nharms=1, npde=4, iterations=100, dtau=dt(h), omega=1.0, nbody=0,
                          blocks=[BlockSpec(0, 64, 32, 0.0, 0.0, h)], cuts=[], name="C0")
    if key == "C1":
        h = 1.0 / 512
        return lattice_case(2, 2, 256, 128, 2, h=h, dtau=dt(h), iterations=200, nbody=2,
                            bodies=((0, "south", 0), (1, "south", 1)), name="C1")
    if key == "C2":
        h = 1.0 / 512
        blk = BlockSpec(0, 512, 256, 0.0, 0.0, h, body_faces=(("south", 0),))
        return CaseConfig(nharms=4, npde=4, iterations=500, dtau=dt(h), omega=0.12, nbody=1,
                          blocks=[blk], cuts=[CutSpec(CutSide(0, "east", 1, 256),
                                                      CutSide(0, "west", 1, 256))], name="C2")
    if key == "C3":
        h = 1.0 / 4096
        return lattice_case(4, 2, 1024, 512, 3, h=h, dtau=dt(h), iterations=200, nbody=4,
                            bodies=tuple((c, "south", c) for c in range(4)), name="C3")
    h = 1.0 / 8192
    return lattice_case(8, 8, 1024, 1024, 4, h=h, dtau=dt(h), iterations=50, name="C4")


def make_parse_errors():
    base = case_text(tc_tiny())
    edits = {
        "bad-int": base.replace("ni = 4", "ni = x", 1),
        "unknown-key": base.replace("ni = 4", "nx = 4", 1),
        "unknown-section": base.replace("[cut 0]", "[cutt 0]"),
        "dup-section": base + "\n[block 1]\nni = 4\n",
        "dup-key": base.replace("ni = 4", "ni = 4\nni = 5", 1),
        "no-case": base.replace("[case]", "[block 9]"),
        "npde": base.replace("npde = 4", "npde = 5"),
        "neg-nharms": base.replace("nharms = 1", "nharms = -1"),
        "omega": base.replace("omega = 1.0", "omega = 0.0"),
        "range": base.replace("range_a = 1:4", "range_a = 4:1"),
        "range-form": base.replace("range_a = 1:4", "range_a = 1-4"),
        "orientation": base.replace("orientation = forward", "orientation = sideways"),
        "face": base.replace("face_a = east", "face_a = up"),
        "body": base.replace("body_faces = south:0", "body_faces = top:0"),
        "no-eq": base.replace("ni = 4", "ni 4", 1),
        "outside": "ni = 4\n" + base,
        "unterminated": base.replace("[cut 0]", "[cut 0"),
        "small-block": base.replace("ni = 4", "ni = 1", 1),
        "neg-h": base.replace("h = 0.25", "h = -0.25", 1),
        "gap-cut": base.replace("[cut 0]", "[cut 1]"),
        "cut-id": base.replace("[cut 0]", "[cut x]"),
    }
    topo_edits = {
        "missing-block": base.replace("block_b = 1", "block_b = 7"),
        "extent": base.replace("range_b = 1:4", "range_b = 2:5").replace("range_a = 1:4", "range_a = 2:5"),
        "length": base.replace("range_b = 1:4", "range_b = 1:3"),
        "body-range": base.replace("body_faces = south:0", "body_faces = south:3"),
        "overlap": base + "\n[cut 1]\nblock_a = 0\nface_a = east\nrange_a = 2:3\nblock_b = 1\n"
                          "face_b = north\nrange_b = 1:2\norientation = forward\n",
    }
    out = {}
    for name, text in edits.items():
        try:
            parse_case(text, source="t.cfg")
            out[name] = ["ok", text, ""]
        except Exception as exc:  # noqa: BLE001
            out[name] = [type(exc).__name__, text, str(exc)]
    for name, text in topo_edits.items():
        try:
            build_topology(parse_case(text, source="t.cfg"))
            out[name] = ["ok", text, ""]
        except Exception as exc:  # noqa: BLE001
            out[name] = [type(exc).__name__, text, str(exc)]
    return out


OUTPUT_RUNS = {
    # name: (builder, iterations, ranks, io mode, seeded-workload key or None)
    "tc-tiny-8": (tc_tiny, 8, 1, "buffered", None),
    "tc-tiny-3-per-value-r2": (tc_tiny, 3, 2, "per-value", None),
    "pair-reversed-6-r2": (reversed_pair, 6, 2, "buffered", None),
    "self-cut-reversed-5": (reversed_self_cut_case, 5, 1, "buffered", None),
    "C0-seeded-10": (lambda: mine.baseline_workload("C0").case, 10, 1, "buffered", "C0"),
}


def make_outputs():
    """Reference-written restart/flowtec files: per-file sha256, size and the
    record layout, plus the run's write_ops counter."""
    import tempfile
    from hbproxy.outio import WriteMode, compute_layout
    out = {}
    for name, (build, iters, ranks, io, wl_key) in OUTPUT_RUNS.items():
        case = build()
        initial = mine.baseline_workload(wl_key).initial if wl_key else None
        saved = hbcore.initial_values
        if initial is not None:
            def hook(spec, planes, npde, n_lo, n_hi, j_lo, j_hi, initial=initial):
                return initial(spec, planes, npde)[n_lo:n_hi, :, j_lo - 1:j_hi - 1, :]
            hbcore.initial_values = hook
        try:
            with tempfile.TemporaryDirectory() as d:
                res = run_case(RunSpec(case=case, ranks=ranks, iterations=iters, io=WriteMode(io),
                                       out_dir=d))
                files = {}
                for fn in sorted(os.listdir(d)):
                    if fn.endswith(".bin"):
                        data = open(os.path.join(d, fn), "rb").read()
                        files[fn] = {"sha256": hashlib.sha256(data).hexdigest(), "bytes": len(data)}
        finally:
            hbcore.initial_values = saved
        topo = build_topology(case)
        layouts = (compute_layout(topo, case.nharms, case.npde, "restart")
                   + compute_layout(topo, case.nharms, case.npde, "flowtec"))
        out[name] = {
            "iterations": iters, "ranks": ranks, "io": io,
            "input_hash": input_hash(case, initial),
            "fingerprint": fingerprint(res.fields, res.forces),
            "files": files,
            "write_ops": res.record.write_ops, "activations": res.record.activations,
            "layouts": {l.filename: {"kind": l.kind, "plane": l.plane, "total_bytes": l.total_bytes,
                                     "records": [[r.block, r.plane, r.offset, r.nfloats]
                                                 for r in l.records]} for l in layouts},
        }
        print(name, {k: v for k, v in out[name].items() if k not in ("layouts", "files")})
    return out


def main():
    if "--outputs" in sys.argv:
        with open(os.path.join(HERE, "outputs.json"), "w") as fh:
            json.dump(make_outputs(), fh, indent=0, sort_keys=True)
        return
    host = make_host()
    with open(os.path.join(HERE, "host.json"), "w") as fh:
        json.dump(host, fh, indent=0, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **make_kernels())
    fps, arrays = make_runs()
    with open(os.path.join(HERE, "fingerprints.json"), "w") as fh:
        json.dump(fps, fh, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "runs.npz"), **arrays)


if __name__ == "__main__":
    main()
