#!/usr/bin/env python3
"""Benchmark: cell-snapshot RK-stage updates per second on B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C4] [--impl ours|reference]

A "step" is one RK iteration (4 fused stages + halo exchange + force
integration) over the whole workload; one unit is one interior cell x one HB
snapshot x one RK stage (all 4 pdes).  Default workload: BASELINE.json
config 4 (C4: 8x8 blocks of 1024x1024 cells, N_H=4 -> P=9, ~19.5 GB per
state slot), the largest configuration and the one the scaling target is
quoted on; it fits one B200.  For N > 1 (torchrun, one rank per GPU) blocks
are partitioned with the reference's LPT rule (8 per GPU at N = 8): total work
is fixed -> "scaling": "strong".

Printed on rank 0: one JSON line with value (device-timed, inputs resident),
roofline of the fused stage kernel, cpu_baseline (the reference's numba
run_case on this host, the C port beside it), e2e (one run_case of the
workload's stated iteration count -- C4: 50 -- with the pinned host input and
output copies inside the timed region), clocks, gpu_launches.

`--impl reference` times the reference itself -- hbproxy.driver.run_case
with its numba kernels, pip-installed into baseline/_ref -- on a bounded
sample of the same workload with all host cores, and its C restatement
(oracle/) beside it; with no baseline/_ref it times the C restatement.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

ALGO_BYTES = {0: 64, 1: 96, 2: 96, 3: 96}   # per unit per stage
UNIT = "cell-snapshot RK-stage updates/s"
METRIC = "cell-snapshot RK-stage updates/sec (fp64, 4 pdes) and % of HBM roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="C4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--tile-rows", type=int, default=None)
    ap.add_argument("--schedule", default="auto", choices=["auto", "paired", "single", "small"],
                    help="auto: the engine's choice (paired from 16 Mi units per stage, the one-launch "
                         "small schedule up to 8 Mi, single stages between)")
    ap.add_argument("--kernel-reps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--allow-knobs", action="store_true",
                    help="run even with HBGPU_* environment knobs set (recorded in the line)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-iters", type=int, default=10)
    ap.add_argument("--zero-ic", action="store_true",
                    help="development only: zero initial state (skips the seeded IC build)")
    return ap.parse_args()


def fp64_peak():
    path = os.path.join(REPO, "profiles", "fp64_peak.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["dadd_ops_per_s"]) / 1e12, "measured (profiles/fp64_peak.json, DADD rate)"
    except Exception:
        return 18.5, "fallback (64 fp64 lanes/clk/SM x 148 SMs x 1.965 GHz)"


def _time_launches(dr, launches, reps):
    """Mean CUDA-event time (ms) of each launch, on the stream it runs on."""
    import torch
    evs = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in launches] for _ in range(reps)]
    launches[-1]()   # warm
    torch.cuda.synchronize()
    for r in range(reps):
        for k, fn in enumerate(launches):
            evs[r][k][0].record()
            fn()
            evs[r][k][1].record()
    torch.cuda.synchronize()
    return [sum(evs[r][k][0].elapsed_time(evs[r][k][1]) for r in range(reps)) / reps
            for k in range(len(launches))]


def roofline(dr, args, units_stage, step_ms_total, wl, world):
    """Roofline of the dominant kernel.

    Single stages: the stage kernel, HBM-bound, SURVEY.md §8d's 88 B/unit.
    Paired stages (the default where eligible): the paired kernel does two
    stages per launch and is co-limited by fp64 issue and HBM; it is reported
    against the measured fp64 rate (the larger fraction), with its HBM
    fraction for the fused schedule's own algorithmic traffic (pass A reads
    q0 and writes q2, 64 B per cell-snapshot; pass B reads q2 and q0 and
    writes q4, 96 B) and the fraction the unfused algorithm's 88 B/unit
    would need at the achieved rate."""
    P = wl.case.planes
    flops_unit = 52 + 8 * P
    peak, peak_src = peaks()
    step_ms = step_ms_total / args.steps
    traffic = None
    tpath = os.path.join(REPO, "profiles", "stage_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            tj = json.load(fh)
        if tj.get("workload") == wl.key and tj.get("n_gpus", 1) == world and \
                bool(tj.get("fused")) == dr.fused:
            traffic = tj.get("bytes_per_launch_avg")
    if dr.layout.small:
        # one cooperative launch runs whole iterations: the kernel time is the step
        algo = sum(ALGO_BYTES[s] for s in range(4)) * units_stage
        achieved = algo / (step_ms / 1e3) / 1e9
        return {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": None, "peak_source": peak_src,
                "kernel": "hb_small (whole iterations in one cooperative launch; state L2-resident, so "
                          "the HBM roofline is a lower bound on what the memory system could give)",
                "algorithmic_bytes_per_unit": {"stage0": 64, "stages1-3": 96, "avg": 88},
                "units_per_launch": units_stage * 4 * args.steps, "share_of_step": 1.0}
    if not dr.fused:
        stage_args = [dr.stage_args(s) for s in range(4)]
        t = _time_launches(dr, [lambda a=a: dr.launch_stage(a) for a in stage_args], args.kernel_reps)
        algo = sum(ALGO_BYTES[s] for s in range(4)) * units_stage
        achieved = algo / (sum(t) / 1e3) / 1e9
        return {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": peak_src,
                "kernel": "hb_stage (fused residual + RK update + halo forward)",
                "algorithmic_bytes_per_unit": {"stage0": 64, "stages1-3": 96, "avg": 88},
                "units_per_launch": units_stage, "stage_ms": [round(x, 4) for x in t],
                "share_of_step": round(sum(t) / step_ms, 4)}
    phases = [dr.phase_args(k) for k in range(4)]
    launch = [lambda a=phases[0]: dr.launch_band(a), lambda a=phases[1]: dr.launch_stage(a),
              lambda a=phases[2]: dr.launch_band(a), lambda a=phases[3]: dr.launch_stage(a)]
    t = _time_launches(dr, launch, args.kernel_reps)
    pair_s = (t[1] + t[3]) / 1e3
    units_pair = 2 * units_stage                      # unit-stages per paired launch
    fp_peak, fp_src = fp64_peak()
    tflops = flops_unit * 2 * units_pair / pair_s / 1e12
    fused_bytes = (64 + 96) * units_stage             # passes A + B, per cell-snapshot
    gbs = fused_bytes / pair_s / 1e9
    return {"bound": "fp64", "achieved": round(tflops, 3), "peak": round(fp_peak, 3), "unit": "TFLOP/s",
            "frac": round(tflops / fp_peak, 4), "traffic": traffic, "peak_source": fp_src,
            "kernel": "hb_pair (two fused RK stages: residual + update + halo forward)",
            "algorithmic_flops_per_unit": flops_unit,
            "units_per_launch": units_pair,
            "hbm": {"achieved": round(gbs, 1), "peak": peak, "unit": "GB/s", "frac": round(gbs / peak, 4),
                    "peak_source": peak_src,
                    "algorithmic_bytes": {"pass_A_per_cell_snapshot": 64, "pass_B_per_cell_snapshot": 96}},
            # HBM fraction the single-stage algorithm (88 B/unit) would need
            # to reach this step rate
            "unfused_hbm_equivalent_frac": round(88 * 4 * units_stage / (step_ms / 1e3) / 1e9 / peak, 4),
            "phase_ms": {"band0": round(t[0], 4), "pair01": round(t[1], 4), "band2": round(t[2], 4),
                         "pair23": round(t[3], 4)},
            "share_of_step": round((t[1] + t[3]) / step_ms, 4)}


def peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clock + throttle reasons sampled during the timed region: NVML (the
    source nvidia-smi reads) polled every few ms from a thread -- the default
    timed region is ~0.2 s, two samples of `nvidia-smi -lms 100` -- with the
    nvidia-smi loop of the profiling recipe as the fallback."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # nvmlClocksThrottleReason* / nvmlClocksEventReason* bits
    NVML_REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
                    0x4: "sw_power_cap"}

    def __init__(self, index, period_s=0.005):
        self.index = index
        self.period_s = period_s
        self.proc = None
        self.thread = None
        self.samples = []       # (sm_mhz, reason bits)
        self.smax = None
        self.source = None

    def _nvml_loop(self, nv, handle):
        reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self._stop.is_set():
            try:
                self.samples.append((float(nv.nvmlDeviceGetClockInfo(handle, nv.NVML_CLOCK_SM)),
                                     int(reasons(handle))))
            except Exception:
                break
            self._stop.wait(self.period_s)

    def __enter__(self):
        try:
            import threading

            import pynvml as nv
            nv.nvmlInit()
            # torch's device index follows CUDA_VISIBLE_DEVICES; NVML's does not
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            phys = self.index
            if vis:
                ids = [v.strip() for v in vis.split(",") if v.strip()]
                if self.index < len(ids) and ids[self.index].isdigit():
                    phys = int(ids[self.index])
            handle = nv.nvmlDeviceGetHandleByIndex(phys)
            self.smax = float(nv.nvmlDeviceGetMaxClockInfo(handle, nv.NVML_CLOCK_SM))
            self._stop = threading.Event()
            self.thread = threading.Thread(target=self._nvml_loop, args=(nv, handle), daemon=True)
            self.thread.start()
            self.source = "nvml"
            return self
        except Exception:
            self.thread = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.source = "nvidia-smi"
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.thread is not None:
            self._stop.set()
            self.thread.join(timeout=2)
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, smax, reasons = [], self.smax, set()
        for mhz, bits in self.samples:
            sm.append(mhz)
            reasons.update(name for bit, name in self.NVML_REASONS.items() if bits & bit)
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for name, flag in zip(names, parts[4:8]):
                if flag.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm), "source": self.source}


def library_knobs():
    """libhbgpu / layout environment knobs (HBGPU_GRID_LIMIT, HBGPU_FUSED,
    HBGPU_LAYOUT, HBGPU_L2_PROMOTION, HBGPU_TILE_PDES, HBGPU_NVCC_EXTRA, ...):
    test and measurement switches that change the schedule; a benchmark
    line must not be taken with any of them set unknowingly."""
    return {k: v for k, v in sorted(os.environ.items()) if k.startswith("HBGPU_")}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def make_ic(wl, blocks, pinned=True, zero=False):
    """Seeded initial state of the given blocks in (pinned) host tensors."""
    import torch
    from concurrent.futures import ThreadPoolExecutor
    P = wl.case.planes

    def one(b):
        t = torch.empty((P, 4, b.nj, b.ni), dtype=torch.float64, pin_memory=pinned)
        if zero:
            t.zero_()
        else:
            t.numpy()[...] = wl.initial(b, P, 4)
        return b.id, t

    with ThreadPoolExecutor(max_workers=min(16, max(1, os.cpu_count() or 1))) as ex:
        return dict(ex.map(one, blocks))


# ---------------------------------------------------------------------------
# CPU side: the oracle port of the reference path
# ---------------------------------------------------------------------------

def sample_case(wl, nblocks):
    """The first `nblocks` blocks of the workload with the cuts among them."""
    import dataclasses
    from paper_1304_7654_b200.topology import CaseConfig
    keep = set(range(nblocks))
    cuts = [c for c in wl.case.cuts if c.side_a.block in keep and c.side_b.block in keep]
    blocks = [dataclasses.replace(b, body_faces=tuple(bf for bf in b.body_faces))
              for b in wl.case.blocks[:nblocks]]
    return CaseConfig(nharms=wl.case.nharms, npde=4, iterations=1, dtau=wl.case.dtau,
                      omega=wl.case.omega, nbody=wl.case.nbody, blocks=blocks,
                      cuts=cuts, name=f"{wl.key}-sample{nblocks}")


def cpu_sample_blocks(wl):
    # ~40M cell-snapshots per sampled iteration: 1 block of C3/C4, all of C0..C2
    budget = 40e6
    per = wl.case.blocks[0].cells() * wl.case.planes
    return max(1, min(len(wl.case.blocks), int(budget // per)))


def cpu_baseline(wl, iters):
    """The reported CPU baseline of our arm: the reference's own run_case
    (numba, baseline/_ref) on a bounded sample, with the C port beside it."""
    ref = reference_rate(wl, steps=1, warmup=1, nblocks=None)
    port = port_rate(wl, iters)
    if ref is None:
        port["note"] = "reference not installed in baseline/_ref: the C port is the baseline"
        return port
    ref["port"] = {k: port[k] for k in ("value", "cores", "sample")}
    return ref


def port_rate(wl, iters):
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import oracle  # the checker / CPU baseline only
    nb = cpu_sample_blocks(wl)
    case = sample_case(wl, nb)
    solver = oracle.OracleSolver(case, initial=wl.initial, record_norms=False)
    solver.prime()
    t0 = time.perf_counter()
    solver.iterate(iters)
    dt = time.perf_counter() - t0
    units = solver.units_per_iteration * iters
    return {"value": units / dt, "unit": UNIT, "cores": solver.nthreads, "kind": "port",
            "sample": f"blocks 0..{nb - 1} of {wl.key} ({nb} of {len(wl.case.blocks)}, cuts among "
                      f"them), {iters} iteration(s), {units / 1e6:.0f} M units in {dt:.2f} s; "
                      f"C restatement of hbcore._residual_kernel/_update_kernel (oracle/hb_oracle.c), "
                      f"pthreads over (block, plane)"}


def _import_reference():
    """The unmodified reference package from baseline/_ref (pip-installed from
    /root/reference/pkg), or None."""
    path = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "hbproxy")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/hbproxy_numba_cache")
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    if path not in sys.path:
        sys.path.insert(0, path)
    try:
        import hbproxy  # noqa: F401
        from hbproxy import driver, hbcore, mesh
    except Exception:
        return None
    return driver, hbcore, mesh


def _ref_case(mesh, case):
    """Our CaseConfig -> the reference's mesh.CaseConfig (same fields)."""
    blocks = [mesh.BlockSpec(b.id, b.ni, b.nj, b.x0, b.y0, b.h, tuple(b.body_faces)) for b in case.blocks]
    cuts = [mesh.CutSpec(mesh.CutSide(c.side_a.block, c.side_a.face, c.side_a.lo, c.side_a.hi),
                         mesh.CutSide(c.side_b.block, c.side_b.face, c.side_b.lo, c.side_b.hi),
                         c.reversed) for c in case.cuts]
    return mesh.CaseConfig(nharms=case.nharms, npde=case.npde, iterations=case.iterations, dtau=case.dtau,
                           omega=case.omega, nbody=case.nbody, blocks=blocks, cuts=cuts, name=case.name)


def ref_sample_blocks(wl):
    # ~320M units per sampled iteration (a few s of 16-core numba): 8 blocks
    # of C4 (one per 2 of the box's 16 cores), 5 of C3, all of C0..C2
    budget = 320e6
    per = wl.case.blocks[0].cells() * wl.case.planes * 4
    return max(1, min(len(wl.case.blocks), int(budget // per)))


def reference_rate(wl, steps, warmup, nblocks=None):
    """hbproxy.driver.run_case -- the reference's public API and stock path
    (numba kernels, thread ranks) -- on the first `nblocks` blocks of the
    workload, per SURVEY.md §8d's CPU plan: ranks = min(blocks, cores),
    threads = cores // ranks, default axis (harmonics), hoisted activation,
    aggregated serial exchange, buffered reduction; the seeded initial state
    through the hbcore.initial_values hook; the JIT warmed first.  Value =
    units / RunRecord.wall_s of one run of `steps` iterations."""
    mods = _import_reference()
    if mods is None:
        return None
    driver, hbcore, mesh = mods
    nb = nblocks or ref_sample_blocks(wl)
    case = _ref_case(mesh, sample_case(wl, nb))
    cores = len(os.sched_getaffinity(0))
    ranks = min(nb, cores)
    threads = max(1, cores // ranks)
    saved = hbcore.initial_values

    def hook(spec, planes, npde, n_lo, n_hi, j_lo, j_hi):
        full = wl.initial(spec, planes, npde)
        return full[n_lo:n_hi, :, j_lo - 1:j_hi - 1, :]

    hbcore.initial_values = hook
    try:
        tiny = _ref_case(mesh, sample_case(wl, 1))
        tiny = mesh.CaseConfig(nharms=tiny.nharms, npde=4, iterations=1, dtau=tiny.dtau, omega=tiny.omega,
                               nbody=0, blocks=[mesh.BlockSpec(0, 16, 8, 0.0, 0.0, tiny.blocks[0].h)],
                               cuts=[], name="jit-warm")
        driver.run_case(driver.RunSpec(case=tiny, ranks=1, iterations=1))       # numba JIT
        if warmup > 0:
            driver.run_case(driver.RunSpec(case=case, ranks=ranks, threads=threads, iterations=warmup))
        res = driver.run_case(driver.RunSpec(case=case, ranks=ranks, threads=threads, iterations=steps))
    finally:
        hbcore.initial_values = saved
    units = sum(b.ni * b.nj for b in case.blocks) * (2 * case.nharms + 1) * 4 * steps
    wall = res.record.wall_s
    import numba
    return {"value": units / wall, "unit": UNIT, "cores": ranks * threads, "kind": "reference",
            "sample": f"hbproxy.driver.run_case (numba {numba.__version__}, baseline/_ref) on blocks "
                      f"0..{nb - 1} of {wl.key} ({nb} of {len(wl.case.blocks)}, cuts among them), "
                      f"{steps} iteration(s) after {warmup} warm-up, ranks={ranks} x threads={threads} on "
                      f"{cores} host cores; {units / 1e6:.0f} M units in RunRecord.wall_s = {wall:.2f} s",
            "wall_s": wall}


def run_reference_arm(args, wl):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    ref = reference_rate(wl, args.steps, args.warmup)
    port = port_rate(wl, max(1, min(args.steps, 3)))
    if ref is None:
        ref = dict(port)
        ref["note"] = "reference not installed in baseline/_ref: timing its C restatement (oracle/)"
    else:
        ref["port"] = {k: port[k] for k in ("value", "cores", "sample")}
    value = ref["value"]
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": None if "wall_s" not in ref else ref["wall_s"] / args.steps * 1e3,
            "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": wl.key, "description": wl.description},
            "cpu_baseline": ref,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU side
# ---------------------------------------------------------------------------

def run_ours(args, wl):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1304_7654_b200 import RunSpec, native, run_case
    from paper_1304_7654_b200.cutplan import build_cut_plan
    from paper_1304_7654_b200 import solver as solver_mod
    from paper_1304_7654_b200.solver import DeviceRank, make_comm
    from paper_1304_7654_b200.topology import build_topology, partition_blocks

    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    knobs = library_knobs()
    if knobs and not args.allow_knobs:
        raise SystemExit(f"refusing to benchmark with libhbgpu test/measurement knobs set: {knobs} "
                         f"(--allow-knobs to override; the line then records them)")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    native.require_cuda()
    case = wl.case
    topo = build_topology(case)
    part = partition_blocks(topo, world)
    plan = build_cut_plan(topo, part, case.nharms, case.npde)
    mine = [topo.blocks[g] for g in part.blocks_of(rank)]
    ic = make_ic(wl, mine, zero=args.zero_ic)
    total_units_iter = topo.total_cells() * case.planes * 4
    comm = make_comm(rank, world, local) if world > 1 else None

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    fused = {"auto": None, "paired": True, "single": False, "small": False}[args.schedule]
    small = {"auto": None, "paired": False, "single": False, "small": True}[args.schedule]
    dr = DeviceRank(case, topo, part, plan, rank=rank, device=local, comm=comm,
                    tile_rows=args.tile_rows, max_iters=args.warmup + args.steps + 1, pinned_ic=ic,
                    fused=fused, small=small)
    dr.prime()
    if world > 1:
        # one eager iteration first, so every NCCL send/recv of the iteration
        # has run (connections set up) before the graph capture records them
        dr.iterate(1, use_graph=False)
    dr.iterate(args.warmup, use_graph=True)
    torch.cuda.synchronize()
    l0 = native.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        ev0.record()
        dr.iterate(args.steps, use_graph=True)
        ev1.record()
        torch.cuda.synchronize()
        barrier()
    launches = native.launch_count() - l0
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    div = dr.divergence()
    if div is not None:
        raise SystemExit(f"benchmark run diverged: {div}")
    value = total_units_iter * args.steps / (ms / 1e3)

    # dominant kernel, timed alone on the launching stream
    my_units_stage = sum(b.cells() for b in mine) * case.planes
    roof = roofline(dr, args, my_units_stage, ms, wl, world)
    tile_rows, fused, small = dr.layout.tile_rows, dr.fused, bool(dr.layout.small)
    dr.close()
    del dr
    torch.cuda.empty_cache()

    # end to end through run_case: pinned IC H2D + K iterations + D2H of fields
    e2e = None
    if not args.no_e2e:
        out = {b.id: torch.empty((case.planes, 4, b.nj + 2, b.ni + 2), dtype=torch.float64,
                                 pin_memory=True) for b in mine}
        h2d = sum(t.numel() * 8 for t in ic.values())
        d2h = sum(t.numel() * 8 for t in out.values())
        # the workload as BASELINE.json states it: a run of the config's own
        # iteration count (C4: 50), or K if that is larger
        e2e_iters = max(args.steps, case.iterations)
        barrier()
        t0 = time.perf_counter()
        e2e_error = None
        try:
            res = run_case(RunSpec(case=case, ranks=world, iterations=e2e_iters, initial_state=ic,
                                   output=out, tile_rows=args.tile_rows, device=local))
            del res
        except Exception as exc:   # noqa: BLE001
            # one GPU: a failing public API fails the bench.  Several GPUs: the
            # device-timed line above is still valid, so it is printed with the
            # end-to-end leg marked failed (run_case's CommGuard has already
            # released the peers of a failing rank)
            if world == 1:
                raise
            e2e_error = f"{type(exc).__name__}: {exc}"
        wall = max_over_ranks(time.perf_counter() - t0)
        e2e = {"value": total_units_iter * e2e_iters / wall, "unit": UNIT,
               "h2d_bytes_per_step": h2d * world // e2e_iters,
               "d2h_bytes_per_step": d2h * world // e2e_iters,
               "iterations": e2e_iters, "wall_s": round(wall, 4),
               "phases_s": {k: round(v, 4) for k, v in solver_mod.LAST_TIMINGS.items()},
               "note": "one run_case() of the workload's stated iteration count (max with K): layout + "
                       "allocation + pinned H2D of the initial state + the iterations + D2H of all fields "
                       "(halos incl.) + forces/norms; per-step bytes are the run's copies / iterations"}
        if e2e_error is not None:
            e2e = {"value": None, "unit": UNIT, "error": e2e_error, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(wl, args.cpu_sample_iters)
    if comm is not None:
        native.load().hbgpu_comm_destroy(comm)
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic",
                "config": {"workload": wl.key, "description": wl.description,
                           "blocks": len(case.blocks), "cells": topo.total_cells(),
                           "planes": case.planes, "units_per_step": total_units_iter,
                           "parallelism": f"blocks/{world} gpu (LPT partition)",
                           "tile_rows": tile_rows,
                           "schedule": "paired RK stages (band + pair kernels)" if fused
                                       else ("one-launch small schedule (hb_small.cu)" if small
                                             else "single RK stages"),
                           "l2": l2_note(dr_slot_gb(case, mine))},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk.summary(),
                "gpu_launches": int(launches),
                "env": {"hbgpu_knobs": knobs, "library": native.LIB_PATH,
                        "abi": int(native.load().hbgpu_abi_version()),
                        "nccl_vars": {k: v for k, v in os.environ.items() if k.startswith("NCCL_")}}}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    np.random.seed(0)


def l2_note(slot_gb):
    """The timing rule's L2 statement: C3/C4 stream slots far larger than the
    126 MB L2; the small configs' three slots fit in it, and are not flushed
    between iterations (a solver's own iterations reuse them the same way)."""
    if 3 * slot_gb * 1e3 > 126:
        return f"inputs larger than L2: {slot_gb:.2f} GB per state slot (3 slots)"
    return (f"inputs fit in L2 ({slot_gb * 1e3:.0f} MB per state slot, 3 slots); not flushed between "
            "iterations: the workload's own iteration-to-iteration reuse")


def dr_slot_gb(case, blocks):
    return sum(case.planes * 4 * (b.nj + 2) * (b.ni + 8) * 8 for b in blocks) / 1e9


def main():
    args = parse()
    from paper_1304_7654_b200 import baseline_workload
    wl = baseline_workload(args.workload)
    if args.impl == "reference":
        run_reference_arm(args, wl)
    else:
        run_ours(args, wl)


if __name__ == "__main__":
    main()
