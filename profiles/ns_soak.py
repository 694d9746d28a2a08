"""Soak parity of the north-star Euler / NS path at full
size: BASELINE configs at their stated iteration counts where the CPU checker
finishes in minutes (C0 x 100, C1 x 200, C2 x 500) and C3 for a few
iterations (the single-threaded oracle takes ~45 s per C3 iteration; C4 ~9
min, so C4 is covered at reduced size by tests/test_ns.py only).

Per config: nsflow.run_ns on cuda:0 against oracle/ns_oracle.c on the same
case -- fields with halos and the force history bitwise, norms at rtol 1e-12.
The checker is builder-written (the reference has no flux physics): this
parity is UNPINNED, as everywhere for row f2.

  python profiles/ns_soak.py --configs C0:100,C1:200,C2:500,C3:2 --out gpurun_out/ns_soak.json
"""

import argparse
import hashlib
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [REPO, os.path.join(REPO, "oracle")]

import numpy as np  # noqa: E402

import ns_oracle  # noqa: E402  (test infrastructure: the checker)
from paper_1304_7654_b200 import nsflow  # noqa: E402


def fingerprint(fields, forces):
    h = hashlib.sha256()
    for b in sorted(fields):
        h.update(np.ascontiguousarray(fields[b]).tobytes())
    h.update(np.ascontiguousarray(forces).tobytes())
    return h.hexdigest()[:16]


def soak(key, iters):
    case = nsflow.ns_workload(key)
    t0 = time.perf_counter()
    got = nsflow.run_ns(case, iters)
    gf, gforces, gnorms = got.fields(), got.force_history(), np.array(got.norm_history())
    gpu_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    want = ns_oracle.run(case, iters)
    oracle_s = time.perf_counter() - t0
    wf, wforces, wn = want.fields(), np.stack(want.forces), np.array(want.norms)
    differ = [b for b in wf if not np.array_equal(gf[b], wf[b])]
    return {
        "config": key, "case": case.name, "iterations": iters, "blocks": len(wf),
        "cells": sum(b.ni * b.nj for b in case.blocks), "planes": case.planes,
        "gpu_fingerprint": fingerprint(gf, gforces), "oracle_fingerprint": fingerprint(wf, wforces),
        "blocks_differing": differ, "forces_equal": bool(np.array_equal(gforces, wforces)),
        "norms_max_rel_diff": float(np.max(np.abs(gnorms - wn) / np.abs(wn))),
        "norm_first": float(wn[0]), "norm_last": float(wn[-1]),
        "gpu_run_s": round(gpu_s, 2), "oracle_s": round(oracle_s, 2),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C0:100,C1:200,C2:500,C3:2")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    rows = []
    for item in args.configs.split(","):
        key, iters = item.split(":")
        row = soak(key, int(iters))
        row["equal"] = (row["gpu_fingerprint"] == row["oracle_fingerprint"] and not row["blocks_differing"]
                        and row["forces_equal"])
        print(json.dumps(row), flush=True)
        rows.append(row)
        if args.out:
            with open(args.out, "w") as fh:
                json.dump(rows, fh, indent=1)
    if not all(r["equal"] and r["norms_max_rel_diff"] < 1e-12 for r in rows):
        sys.exit(1)


if __name__ == "__main__":
    main()
