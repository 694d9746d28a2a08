"""Summarise an `ncu --set full` capture of the stage- or pair-kernel launches.

    python profiles/summarize_ncu.py REPORT.ncu-rep OUT.json [--traffic profiles/stage_traffic.json]

Writes one entry per captured launch (time, DRAM bytes and rates, pipe
utilisation, issue activity, the main stall ratios) and, with --traffic, the
mean DRAM bytes per launch that bench.py reports as roofline.traffic.
Algorithmic bytes per launch follow SURVEY.md §8d: 64 B/unit for the first
RK stage, 96 B/unit for the others; the unit count comes from the workload.
"""

import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__cycles_active.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "sm__cycles_elapsed.avg.per_second",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "launch__grid_size", "launch__block_size",
    "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum",
]
STALLS = ["long_scoreboard", "wait", "math_pipe_throttle", "not_selected", "short_scoreboard",
          "branch_resolving", "barrier", "membar", "lg_throttle", "mio_throttle", "no_instruction"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}


def _num(text, unit):
    try:
        return float(text.replace(",", "")) * UNIT.get(unit, 1)
    except ValueError:
        return text


def main():
    rep, out = sys.argv[1], sys.argv[2]
    traffic = sys.argv[sys.argv.index("--traffic") + 1] if "--traffic" in sys.argv else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    sys.path.insert(0, ".")
    from paper_1304_7654_b200 import baseline_workload
    case = baseline_workload("C4").case
    units_per_launch = sum(b.ni * b.nj for b in case.blocks) * case.planes
    launches = []
    for r in data:
        name = r[hdr.index("Kernel Name")]
        if "stage_tma_kernel" not in name and "pair_tma_kernel" not in name:
            continue
        pair = "pair_tma_kernel" in name
        e = {"kernel": name}
        for k in KEYS:
            if k in hdr:
                e[k] = _num(r[hdr.index(k)], units[hdr.index(k)])
        for s in STALLS:
            k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if k in hdr:
                e["stall_" + s] = _num(r[hdr.index(k)], "")
        second = "(bool)1" in name or "9, 1," in name    # FIRST (stage kernel) / PB (pair kernel)
        if pair:
            # pass A reads q0 and writes q2, pass B reads q2 and q0 and writes q4
            algo = (96 if second else 64) * units_per_launch
            e["algorithmic_flops"] = 2 * (52 + 8 * case.planes) * units_per_launch
        else:
            algo = (64 if second else 96) * units_per_launch
        dram = e["dram__bytes_read.sum"] + e["dram__bytes_write.sum"]
        t = e["gpu__time_duration.sum"]
        e.update(algorithmic_bytes=algo, dram_bytes=dram, dram_over_algorithmic=round(dram / algo, 4),
                 dram_TBps=round(dram / t / 1e12, 3), algorithmic_TBps=round(algo / t / 1e12, 3))
        if pair:
            e["algorithmic_TFLOPs"] = round(e["algorithmic_flops"] / t / 1e12, 3)
        launches.append(e)
    with open(out, "w") as fh:
        json.dump({"report": rep, "workload": "C4", "units_per_launch": units_per_launch,
                   "launches": launches}, fh, indent=1)
    if traffic and launches:
        avg = sum(l["dram_bytes"] for l in launches) / len(launches)
        algo = sum(l["algorithmic_bytes"] for l in launches) / len(launches)
        with open(traffic, "w") as fh:
            json.dump({"workload": "C4", "n_gpus": 1, "kernel": launches[0]["kernel"],
                       "fused": any("pair_tma_kernel" in l["kernel"] for l in launches),
                       "bytes_per_launch_avg": int(avg), "algorithmic_bytes_per_launch_avg": int(algo),
                       "source": f"{out}: mean over the {len(launches)} RK-stage launches of one iteration "
                                 "of dram__bytes_read.sum + dram__bytes_write.sum (ncu --set full)"},
                      fh, indent=1)
    for l in launches:
        print(l["kernel"][:45], f'{l["gpu__time_duration.sum"] * 1e3:.3f} ms', l["dram_TBps"], "TB/s dram",
              l["dram_over_algorithmic"], "x algo")


if __name__ == "__main__":
    main()
