"""Per-CUDA-source-line instruction counts and stall samples of one ncu
report (offline):  python tools/ncu_lines.py <report.ncu-rep> [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    agg = defaultdict(lambda: [0, 0])
    fname = None
    hdr = None
    src_text = {}
    for row in csv.reader(io.StringIO(out)):
        if not row:
            continue
        if row[0] == "File Path":
            fname = row[1].split("/")[-1]
            continue
        if row[0] == "Line No":
            hdr = row
            continue
        if hdr is None or len(row) < len(hdr):
            continue
        try:
            ln = int(row[0])
        except ValueError:
            continue
        d = dict(zip(hdr[2:], row[2:]))
        src_text[(fname, ln)] = row[1]
        ie = (d.get("Instructions Executed", "0") or "0").replace(",", "").replace("-", "0")
        ss = (d.get("Warp Stall Sampling (All Samples)", "0") or "0").replace(",", "").replace("-", "0")
        try:
            ie_v, ss_v = int(float(ie)), int(float(ss))
        except ValueError:  # a source line the csv could not split cleanly
            continue
        a = agg[(fname, ln)]
        a[0] += ie_v
        a[1] += ss_v
    tot_i = sum(v[0] for v in agg.values()) or 1
    tot_s = sum(v[1] for v in agg.values()) or 1
    print(f"total instructions {tot_i}  samples {tot_s}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{k[0]}:{k[1]:4d}  inst {v[0]:9d} ({100*v[0]/tot_i:5.1f}%)  stall {100*v[1]/tot_s:5.1f}%  "
              f"{src_text.get(k, '')[:70].strip()}")


if __name__ == "__main__":
    main()


def regions(rep, spans):
    """Instruction totals per named line span of tb_kernel_sparse.cu (+ other files)."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    tot = defaultdict(int)
    fname = None
    hdr = None
    for row in csv.reader(io.StringIO(out)):
        if not row:
            continue
        if row[0] == "File Path":
            fname = row[1].split("/")[-1]
            continue
        if row[0] == "Line No":
            hdr = row
            continue
        if hdr is None or len(row) < len(hdr):
            continue
        try:
            ln = int(row[0])
            d = dict(zip(hdr[2:], row[2:]))
            ie = int(float((d.get("Instructions Executed", "0") or "0").replace(",", "").replace("-", "0")))
        except ValueError:
            continue
        name = fname
        for nm, (a, b) in spans.items():
            if fname == "tb_kernel_sparse.cu" and a <= ln <= b:
                name = nm
        tot[name] += ie
    return dict(tot)
