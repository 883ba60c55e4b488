"""SASS opcode census of the hot kernels (no GPU needed): evidence of the
sm_100a features each kernel uses — UBLKCP (cp.async.bulk through the TMA
engine), SYNCS.* (mbarrier), ACQBULK / PREEXIT (griddepcontrol.wait /
launch_dependents: programmatic dependent launch), ATOMS (shared atomics),
MATCH / REDUX / VOTE (warp primitives), LDS/STS (shared traffic).

    python tools/sass_evidence.py > profiles/r01_sass_evidence.txt
"""
import os
import re
import subprocess
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2510_05485_b200", "libtensorbleu_b200.so")
KEEP = ("UBLKCP", "UTMALDG", "SYNCS", "ACQBULK", "PREEXIT", "ATOMS", "ATOMG", "RED", "REDUX", "MATCH",
        "VOTE", "BAR", "LDS", "STS", "LDG", "STG", "LDL", "STL", "DFMA", "MUFU")
KERNELS = ("bleu_pair_kernelIi", "bleu_multi_kernelIi", "bleu_group_kernelIi", "bleu_stats_kernelIi",
           "dict_insert_kernel", "segment_smem_kernel")


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    fn = None
    counts = {}
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            fn = m.group(1)
            continue
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
        if m and fn:
            counts.setdefault(fn, Counter())[m.group(1)] += 1
    print(f"# SASS opcode census of {os.path.relpath(LIB, ROOT)} (sm_100a), selected opcodes")
    for fn, c in sorted(counts.items()):
        short = next((k for k in KERNELS if k in fn), None)
        if not short:
            continue
        print(f"\n## {short}  ({sum(c.values())} instructions)")
        for op, n in sorted(c.items()):
            if op.split(".")[0] in KEEP or op.startswith(KEEP):
                print(f"{n:6d}  {op}")


if __name__ == "__main__":
    main()
