"""Attribute an ncu SASS source page (csv) to CUDA source lines using the
line table of the cubin (nvdisasm -g).  Offline helper for profile reading.

    python tools/sass_lines.py <all.sass from nvdisasm -c -g> <mangled kernel> <ncu source csv>
"""
import csv
import re
import sys
from collections import defaultdict


def main():
    sass, kern, src = sys.argv[1:4]
    lines = open(sass).read().split("\n")
    start = next(i for i, l in enumerate(lines) if l.startswith(".text." + kern + ":"))
    cur = None
    idx_line = []
    for l in lines[start + 1:]:
        if l.startswith(".text.") or "// -----" in l and ".text." in l:
            break
        m = re.search(r'line (\d+)', l)
        if l.strip().startswith("//##") and m:
            cur = int(m.group(1))
            continue
        if re.match(r'\s*/\*[0-9a-f]{4,}\*/', l):
            idx_line.append(cur)
    rows = list(csv.reader(open(src)))
    hdr = rows[1]
    data = rows[2:]
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    i_e = hdr.index("Instructions Executed")
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    ri = [hdr.index(h) for h in reasons]
    print(f"sass instrs {len(idx_line)} ncu rows {len(data)}")
    agg = defaultdict(lambda: [0, 0, defaultdict(int)])
    for j, r in enumerate(data):
        ln = idx_line[j] if j < len(idx_line) else None
        a = agg[ln]
        a[0] += int(r[i_s] or 0)
        a[1] += int(r[i_e] or 0)
        for h, k in zip(reasons, ri):
            if r[k].isdigit():
                a[2][h] += int(r[k])
    tot = sum(v[0] for v in agg.values())
    print("total samples", tot)
    for ln, (s, e, rs) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:40]:
        top = sorted(rs.items(), key=lambda kv: -kv[1])[:3]
        print(f"line {ln}: samples {s} ({100 * s / tot:.1f}%) warp-instrs {e} " +
              " ".join(f"{h[6:]}={v}" for h, v in top))


if __name__ == "__main__":
    main()
