"""Throughput of the north-star HB Euler / NS path on one
GPU, BASELINE configs at full size.

One unit = one interior cell x one HB snapshot x one RK stage (4 conservative
variables), as for the proxy path; value = units / CUDA-event time of K
iterations after W warm-up ones (L2 flushed implicitly: every config but C0
exceeds L2).  One iteration = per stage the boundary and cut halos and one
hbns_stage launch (the fused tile kernel of hb_ns.cu), plus the stage-1 norm
fold and the wall forces.

    python profiles/ns_bench.py --configs C0,C1,C2,C3,C4 --steps 5 --warmup 2
"""
import argparse
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    import torch
    from paper_1304_7654_b200 import nsflow
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C0,C1,C2,C3,C4")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--out", default=None, help="also write the rows as a JSON list")
    args = ap.parse_args()
    rows = []
    for key in args.configs.split(","):
        case = nsflow.ns_workload(key)
        run = nsflow.NSRun(case, args.steps + args.warmup)
        run.iterate(args.warmup)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run.iterate(args.steps)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        cells = sum(b.ni * b.nj for b in case.blocks)
        units = cells * case.planes * 4
        norms = run.norm_history()
        row = {"config": key, "case": case.name, "blocks": len(case.blocks), "cells": cells, "planes": case.planes,
               "physics": "Euler" if case.reynolds is None else f"laminar NS Re={case.reynolds:g}",
               "ms_per_iteration": round(ms, 4), "units_per_s": units / (ms / 1e3),
               "norm_first": norms[0], "norm_last": norms[-1], "diverged": run.divergence() is not None}
        print(json.dumps(row), flush=True)
        rows.append(row)
        del run
        torch.cuda.empty_cache()
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(rows, fh, indent=1)


if __name__ == "__main__":
    main()
