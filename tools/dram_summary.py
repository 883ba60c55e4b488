"""Fold the per-config DRAM launch lists into profiles/ncu_summary.json (offline).

    python tools/dram_summary.py <tag>

Reads profiles/<tag>_dram_<workload>_<data>.csv (`ncu --metrics
dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
--clock-control none` of `tools/kernel_times.py <workload> <data> 1`) and
writes, per bench key (workload + '' | 'corr' | 'zipf' | 'vocab1'), the stats
kernels of one step with their DRAM bytes and cold duration, the dominant
kernel and the step's total: bench.py reports it as `roofline.traffic`.
"""
import csv
import json
import os
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROFILES = os.path.join(ROOT, "profiles")
SUFFIX = {"uniform": "", "correlated": "corr", "zipf": "zipf", "vocab1": "vocab1"}


def kernels(path):
    per = OrderedDict()
    for row in csv.reader(open(path)):
        if len(row) < 15 or row[0] == "ID" or "bleu_" not in row[4]:
            continue
        name = row[4].replace("void <unnamed>::", "").replace("(tbk::StatsParams)", "")
        k = per.setdefault(row[0], {"kernel": name, "dram_bytes": 0, "duration_us_cold": 0.0})
        v = float(row[14].replace(",", ""))
        if row[12].startswith("dram__bytes"):
            k["dram_bytes"] += int(v)
        elif row[12] == "gpu__time_duration.sum":
            k["duration_us_cold"] = round(v / 1000.0, 2)
    return list(per.values())


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
    out = os.path.join(PROFILES, "ncu_summary.json")
    summary = json.load(open(out)) if os.path.exists(out) else {}
    for fn in sorted(os.listdir(PROFILES)):
        if not (fn.startswith(f"{tag}_dram_") and fn.endswith(".csv")):
            continue
        wl, data = fn[len(f"{tag}_dram_"):-4].split("_", 1)
        ks = kernels(os.path.join(PROFILES, fn))
        if not ks:
            continue
        top = max(ks, key=lambda k: k["duration_us_cold"])
        summary[wl + SUFFIX[data]] = {
            "kernel": top["kernel"], "dram_bytes_per_launch": top["dram_bytes"],
            "duration_us_cold": top["duration_us_cold"], "step_kernels": ks,
            "step_dram_bytes": sum(k["dram_bytes"] for k in ks),
            "source": f"profiles/{fn} (ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,"
                      f"gpu__time_duration.sum --clock-control none; tools/kernel_times.py {wl} {data} 1)"}
    json.dump(summary, open(out, "w"), indent=1)
    print(f"wrote {out}: {sorted(summary)}")


if __name__ == "__main__":
    main()
