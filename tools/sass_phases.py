"""Instruction counts of one ncu capture attributed to the kernel's OWN source
lines, inlined helpers charged to their call site (offline).

    python tools/sass_phases.py <report.ncu-rep> <cubin> <kernel-substring> <file.cu> [spans]

The ncu source page attributes an inlined helper's instructions to the helper's
header line; this joins the per-SASS-address counts of the report with
`nvdisasm -gi` of the same cubin (same build) and charges every instruction to
the outermost line of <file.cu>.  `spans` = "name:a-b,name:a-b,..." groups the
lines into phases; without it the top lines are listed.
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict


def sass_lines(cubin, kernel, src):
    txt = subprocess.run(["nvdisasm", "-gi", cubin], capture_output=True, text=True).stdout
    out = {}
    cur = None
    inside = False
    pat_file = re.compile(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?')
    for ln in txt.splitlines():
        if ln.startswith("//---------------------") and ".text." in ln:
            inside = kernel in ln
            cur = None
            continue
        if not inside:
            continue
        m = pat_file.search(ln)
        if m:
            f, l, fi, li = m.groups()
            if f.endswith(src):
                cur = int(l)
            elif fi and fi.endswith(src):
                cur = int(li)
            # deeper inlining: nvdisasm prints the chain, the last "inlined at" of
            # src wins (the outermost call site in src)
            for mm in re.finditer(r'inlined at "([^"]+)", line (\d+)', ln):
                if mm.group(1).endswith(src):
                    cur = int(mm.group(2))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", ln)
        if m and cur is not None and not m.group(2).startswith("."):
            out[int(m.group(1), 16)] = cur
    return out


def ncu_counts(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[1]
    ia, ie = hdr.index("Address"), hdr.index("Instructions Executed")
    data = [(int(r[ia], 16), int(r[ie])) for r in rows[2:] if len(r) > ie and r[ie].isdigit()]
    base = min(a for a, _ in data)
    return [(a - base, c) for a, c in data]


def main():
    rep, cubin, kernel, src = sys.argv[1:5]
    spans = {}
    if len(sys.argv) > 5:
        for part in sys.argv[5].split(","):
            nm, rng = part.split(":")
            a, b = rng.split("-")
            spans[nm] = (int(a), int(b))
    lines = sass_lines(cubin, kernel, src)
    counts = ncu_counts(rep)
    per_line = defaultdict(int)
    unk = 0
    for off, c in counts:
        ln = lines.get(off)
        if ln is None:
            unk += c
        else:
            per_line[ln] += c
    tot = sum(c for _, c in counts) or 1
    print(f"total {tot}  unattributed {unk} ({100 * unk / tot:.1f}%)")
    if spans:
        agg = defaultdict(int)
        for ln, c in per_line.items():
            nm = next((k for k, (a, b) in spans.items() if a <= ln <= b), "other")
            agg[nm] += c
        for nm in list(spans) + ["other"]:
            print(f"{nm:>14}: {agg[nm]:10d} ({100 * agg[nm] / tot:5.1f}%)")
    else:
        for ln, c in sorted(per_line.items(), key=lambda kv: -kv[1])[:40]:
            print(f"{src}:{ln:4d} {c:10d} ({100 * c / tot:5.1f}%)")


if __name__ == "__main__":
    main()
