"""Soak parity at BASELINE iteration counts: C3 x 200 and C4 x 50.

Runs run_case on cuda:0 (the auto schedule: paired stages for C3/C4) and the
memory-lean oracle (oracle.LeanOracleSolver, pinned to the reference's
fingerprints) over the same seeded inputs, and records per config:
  - the fingerprint (sha256[:16] over fields, blocks ascending, halos
    included, then cl/cd/cm) of each side, and whether they are equal;
  - the number of blocks whose fields differ (must be 0);
  - the max relative difference of the per-iteration residual norms;
  - GPU loop time and oracle time.
Writes one JSON object per config to the path given with --out.

  python profiles/soak.py --configs C3:200,C4:50 --out gpurun_out/soak.json
"""

import argparse
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [REPO, os.path.join(REPO, "oracle")]

import numpy as np  # noqa: E402

import oracle  # noqa: E402  (test infrastructure: the checker)
from paper_1304_7654_b200 import RunSpec, baseline_workload, run_case  # noqa: E402


def soak(key, iters):
    wl = baseline_workload(key)
    t0 = time.perf_counter()
    got = run_case(RunSpec(case=wl.case, ranks=1, iterations=iters, initial=wl.initial))
    gpu_s = time.perf_counter() - t0
    gforces = np.stack([got.forces.cl, got.forces.cd, got.forces.cm])
    gfp = oracle.fingerprint(got.fields, gforces)
    gnorms = np.array(got.residual_norms)
    gfields = got.fields
    t0 = time.perf_counter()
    want = oracle.run(wl.case, iters, initial=wl.initial, lean=True)
    oracle_s = time.perf_counter() - t0
    wfp = oracle.fingerprint(want.fields, want.forces)
    differ = [b for b in want.fields if not np.array_equal(gfields[b], want.fields[b])]
    wn = np.array(want.norms)
    rel = float(np.max(np.abs(gnorms - wn) / np.abs(wn))) if len(wn) else None
    return {
        "config": key, "iterations": iters, "blocks": len(want.fields),
        "gpu_fingerprint": gfp, "oracle_fingerprint": wfp, "equal": gfp == wfp and not differ,
        "blocks_differing": differ, "forces_equal": bool(np.array_equal(gforces, want.forces)),
        "norms_max_rel_diff": rel, "norm_first": float(wn[0]), "norm_last": float(wn[-1]),
        "max_abs_q": float(max(np.abs(q).max() for q in want.fields.values())),
        "gpu_run_case_s": round(gpu_s, 2), "oracle_s": round(oracle_s, 2),
        "oracle_threads": len(os.sched_getaffinity(0)),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C3:200,C4:50")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    rows = []
    for item in args.configs.split(","):
        key, iters = item.split(":")
        row = soak(key, int(iters))
        print(json.dumps(row), flush=True)
        rows.append(row)
        if args.out:
            with open(args.out, "w") as fh:
                json.dump(rows, fh, indent=1)
    if not all(r["equal"] and r["forces_equal"] for r in rows):
        sys.exit(1)


if __name__ == "__main__":
    main()
