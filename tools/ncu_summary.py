"""Summarise ncu captures into the committed profiles/ JSON (offline, no GPU).

    python tools/ncu_summary.py <tag> <workload>=<report.ncu-rep> ... [--launches <csv>]

Writes profiles/<tag>_ncu_<workload>.json per report (the metrics the roofline
and DESIGN.md cite) and merges `dram_bytes_per_launch` into
profiles/ncu_summary.json, which bench.py reads for `roofline.traffic`.
With --launches, also writes profiles/<tag>_launches_summary.json: per kernel
name, the launch count and mean/total device time of the launch list.
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROFILES = os.path.join(ROOT, "profiles")
METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "pcie__read_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.sum",
    "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
    "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem",
    "sm__maximum_warps_per_active_cycle_pct",
    "smsp__cycles_active.avg",
    "sm__cycles_elapsed.avg",
    "smsp__average_warp_latency_issue_stalled_barrier",
    "smsp__pcsamp_warps_issue_stalled_barrier",
    "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_branch_resolving",
    "smsp__pcsamp_warps_issue_stalled_wait",
    "smsp__pcsamp_warps_issue_stalled_mio_throttle",
    "smsp__pcsamp_sample_count",
]


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for m in METRICS:
        if m in hdr:
            i = hdr.index(m)
            d[m] = [vals[i], units[i]]
    d["kernel"] = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else None
    return d


def to_bytes(v):
    val, unit = float(v[0].replace(",", "")), v[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return val * scale


def main():
    tag = sys.argv[1]
    launches = None
    items = []
    args = sys.argv[2:]
    while args:
        a = args.pop(0)
        if a == "--launches":
            launches = args.pop(0)
        else:
            items.append(a.split("=", 1))
    summ_path = os.path.join(PROFILES, "ncu_summary.json")
    summary = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    for wl, rep in items:
        d = raw(rep)
        json.dump(d, open(os.path.join(PROFILES, f"{tag}_ncu_{wl}.json"), "w"), indent=1)
        rd, wr = to_bytes(d["dram__bytes_read.sum"]), to_bytes(d["dram__bytes_write.sum"])
        t = float(d["gpu__time_duration.sum"][0]) * (1e-3 if d["gpu__time_duration.sum"][1] == "ns" else 1)
        summary[wl] = {"kernel": d["kernel"], "dram_bytes_per_launch": int(rd + wr), "dram_read_bytes": int(rd),
                       "dram_write_bytes": int(wr), "duration_us_cold": t,
                       "source": f"profiles/{tag}_ncu_{wl}.json (ncu --set full --clock-control none, one launch)"}
        print(wl, summary[wl])
    json.dump(summary, open(summ_path, "w"), indent=1)
    if launches:
        agg = defaultdict(lambda: [0, 0.0])
        rows = [r for r in csv.reader(open(launches)) if len(r) > 14 and r[0] != "ID"]
        for r in rows:
            if r[12] == "gpu__time_duration.sum":
                a = agg[r[4]]
                a[0] += 1
                a[1] += float(r[14].replace(",", "")) * (1e-3 if r[13] == "ns" else 1)
        tot = sum(v[1] for v in agg.values())
        out = {k: {"launches": n, "total_us": t, "mean_us": t / n, "share": t / tot}
               for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])}
        json.dump(out, open(os.path.join(PROFILES, f"{tag}_launches_summary.json"), "w"), indent=1)
        for k, v in list(out.items())[:6]:
            print(f"{v['share']:6.1%} {v['launches']:5d} x {v['mean_us']:8.2f} us  {k[:90]}")


if __name__ == "__main__":
    main()
