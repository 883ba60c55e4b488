"""`batchbleu-bench`-compatible benchmark CLI for the B200 path.

Same flags, generator, protocol and CSV as the reference's CLI
(pkg/src/batchbleu/bench.py:24-246): for every (seq_len, batch_size) it
generates the reference's synthetic batch, runs the equivalence gate
(device scores vs the serial per-sentence baseline, max |diff| <= 1e-6, exit
code 2 otherwise), times the selected implementations (1 warm-up + repeats,
mean/std) and writes the CSV plus a table.  Differences:

* `--impl gpu` (alias `batched`) is this package's CUDA path through the
  public `sentence_bleu` on host arrays — the drop-in call a user makes;
  `--impl serial` (alias `oracle`) is the serial per-sentence Counter
  baseline (the reference's `oracle_sentence_bleu` algorithm,
  pkg/src/batchbleu/oracle.py:18-92, restated here as the timed NLTK-style
  baseline of the harness — never used by the package);
* the CSV adds `sent_per_s,roofline_frac,cores` (roofline_frac = SURVEY §8d
  algorithmic bytes / mean time / HBM peak, for the GPU rows);
* `--pinned` hands the GPU path pinned host tensors (zero-copy PCIe reads)
  instead of numpy arrays.

    python tools/batchbleu_bench.py --batch-sizes 16,512 --seq-lens 256,1024 --out report.csv
"""

from __future__ import annotations

import argparse
import math
import os
import statistics
import sys
import time
from collections import Counter
from dataclasses import dataclass
from typing import Callable, Optional, Sequence

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

DEFAULT_BATCH_SIZES = (16, 32, 64, 128, 256, 512)
DEFAULT_SEQ_LENS = (256, 1024)
CSV_HEADER = "implementation,batch_size,seq_len,mean_s,std_s,speedup,sent_per_s,roofline_frac,cores"
HBM_PEAK_GBS = 6650.0  # fallback of B200_PROFILING.md when MEASURED_PEAKS.json is absent


class EquivalenceError(RuntimeError):
    """Device and serial scores disagree beyond 1e-6 on a benchmark batch."""


@dataclass
class Record:
    implementation: str
    batch_size: int
    seq_len: int
    mean_s: float
    std_s: float
    speedup: Optional[float] = None
    roofline_frac: Optional[float] = None


# ---- serial baseline (the reference's oracle algorithm, oracle.py:18-92) -----
def _ngrams(s, n):
    return Counter(tuple(s[i:i + n]) for i in range(len(s) - n + 1))


def serial_sentence_bleu(cand, refs, max_order=4, smoothing="none", eps=0.1, k=1.0):
    weights = [1.0 / max_order] * max_order
    nums, dens = [], []
    for n in range(1, max_order + 1):
        c = _ngrams(cand, n)
        mx = Counter()
        for r in refs:
            for g, v in _ngrams(r, n).items():
                mx[g] = max(mx[g], v)
        nums.append(sum(min(v, mx[g]) for g, v in c.items()))
        dens.append(max(0, len(cand) - n + 1))
    prec, counter = [], 1.0
    for i, (nu, de) in enumerate(zip(nums, dens)):
        p = nu / de if de > 0 else 0.0
        if smoothing == "floor" and nu == 0 and de > 0:
            p = eps / de
        elif smoothing == "add-k" and i >= 1 and de > 0:
            p = (nu + k) / (de + k)
        elif smoothing == "exp" and nu == 0 and de > 0:
            p = 1.0 / (2.0 ** counter * de)
            counter += 1.0
        prec.append(p)
    c = len(cand)
    rl = [len(r) for r in refs]
    r = min(rl, key=lambda x: (abs(x - c), x))
    if c == 0:
        return 0.0
    bp = 1.0 if c > r else math.exp(1.0 - r / c)
    if any(p <= 0 for p, w in zip(prec, weights) if w > 0):
        return 0.0
    s = 0.0
    for p, w in zip(prec, weights):
        if w > 0:
            s += w * math.log(p)
    return min(max(bp * math.exp(s), 0.0), 1.0)


def generate_batch(b, l, vocab, refs, seed):
    """The reference generator (bench.py:72-91): default_rng([seed, B, L, V])."""
    rng = np.random.default_rng([seed, b, l, vocab])

    def draw():
        return (rng.integers(0, vocab, size=(b, l), dtype=np.int64),
                rng.integers(l // 2, l + 1, size=b, dtype=np.int64))
    return draw(), [draw() for _ in range(refs)]


def _serial_scores(cand, refs, smoothing):
    (ci, cl), rr = cand, refs
    return [serial_sentence_bleu(ci[i, :cl[i]].tolist(), [ri[i, :rl[i]].tolist() for ri, rl in rr],
                                 smoothing=smoothing) for i in range(ci.shape[0])]


def _time_fn(fn: Callable[[], object], repeats: int, clock: Callable[[], float]):
    fn()  # warm-up
    samples = []
    for _ in range(repeats):
        t0 = clock()
        fn()
        samples.append(clock() - t0)
    return sum(samples) / len(samples), (statistics.stdev(samples) if len(samples) > 1 else 0.0)


def run_benchmark(args, clock: Callable[[], float] = time.perf_counter) -> list[Record]:
    import torch

    import bench
    import paper_2510_05485_b200 as tb
    cfg = tb.BleuConfig(smoothing=args.smoothing)
    peak = HBM_PEAK_GBS
    try:
        import json
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peak = float(json.load(fh)["hbm_gbs"])
    except Exception:
        pass
    records = []
    for seq_len in args.seq_lens:
        for b in args.batch_sizes:
            cand, refs = generate_batch(b, seq_len, args.vocab, args.refs, args.seed)
            mk = (lambda a: torch.from_numpy(a).pin_memory()) if args.pinned else (lambda a: a)
            c = tb.TokenBatch(ids=mk(cand[0]), lengths=cand[1])
            rs = [tb.TokenBatch(ids=mk(i), lengths=ln) for i, ln in refs]
            got = tb.sentence_bleu(c, rs, cfg).scores
            want = np.array(_serial_scores(cand, refs, args.smoothing))
            diff = float(np.max(np.abs(got - want), initial=0.0))
            if diff > 1e-6:
                raise EquivalenceError(f"device and serial scores differ by {diff:.3e} (B={b}, L={seq_len})")
            serial_mean = None
            if args.impl in ("both", "serial", "oracle"):
                mean, std = _time_fn(lambda: _serial_scores(cand, refs, args.smoothing), args.repeats, clock)
                serial_mean = mean
                records.append(Record("serial", b, seq_len, mean, std))
            if args.impl in ("both", "gpu", "batched"):
                mean, std = _time_fn(lambda: tb.sentence_bleu(c, rs, cfg).scores, args.repeats, clock)
                a = bench.algorithmic_bytes([cand[1]] + [ln for _, ln in refs], args.vocab, b)
                records.append(Record("gpu", b, seq_len, mean, std,
                                      serial_mean / mean if serial_mean else None, a / mean / 1e9 / peak))
    return records


def _fmt(x, spec):
    return "" if x is None else format(x, spec)


def emit_report(records: Sequence[Record], path: str) -> None:
    if not records:
        raise ValueError("no records to report")
    cores = len(os.sched_getaffinity(0))
    lines = [CSV_HEADER]
    for r in records:
        lines.append(f"{r.implementation},{r.batch_size},{r.seq_len},{r.mean_s:.6f},{r.std_s:.6f},"
                     f"{_fmt(r.speedup, '.4f')},{r.batch_size / r.mean_s:.1f},{_fmt(r.roofline_frac, '.4f')},"
                     f"{cores if r.implementation == 'serial' else ''}")
    with open(path, "w", newline="\n") as fh:
        fh.write("\n".join(lines) + "\n")
    print(f"{'impl':<7} {'B':>5} {'L':>5} {'mean_s':>10} {'std_s':>10} {'speedup':>9} {'sent/s':>12}")
    for r in records:
        sp = f"{r.speedup:.1f}x" if r.speedup is not None else ""
        print(f"{r.implementation:<7} {r.batch_size:>5} {r.seq_len:>5} {r.mean_s:>10.6f} {r.std_s:>10.6f} "
              f"{sp:>9} {r.batch_size / r.mean_s:>12.1f}")


def _int_list(text):
    return [int(x) for x in text.split(",") if x]


def build_parser():
    p = argparse.ArgumentParser(prog="batchbleu-bench (B200)",
                                description="Benchmark the B200 token-ID BLEU path against the serial baseline")
    p.add_argument("--batch-sizes", type=_int_list, default=list(DEFAULT_BATCH_SIZES))
    p.add_argument("--seq-lens", type=_int_list, default=list(DEFAULT_SEQ_LENS))
    p.add_argument("--vocab", type=int, default=32000)
    p.add_argument("--refs", type=int, default=1)
    p.add_argument("--repeats", type=int, default=5)
    p.add_argument("--seed", type=int, default=42)
    p.add_argument("--impl", choices=["both", "gpu", "batched", "serial", "oracle"], default="both")
    p.add_argument("--threads", type=int, default=1, help="accepted for compatibility; no effect")
    p.add_argument("--out", default="report.csv")
    p.add_argument("--smoothing", choices=["none", "floor", "add-k", "exp"], default="none")
    p.add_argument("--backend", choices=["auto", "compiled", "cuda"], default="auto",
                   help="accepted for compatibility; the CUDA path is the only backend")
    p.add_argument("--pinned", action="store_true", help="pinned host tensors for the GPU path")
    return p


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    if args.repeats < 1 or min(args.batch_sizes, default=0) < 1 or min(args.seq_lens, default=0) < 1:
        print("repeats, batch sizes and sequence lengths must be positive", file=sys.stderr)
        return 1
    try:
        emit_report(run_benchmark(args), args.out)
    except EquivalenceError as exc:
        print(f"equivalence check failed: {exc}", file=sys.stderr)
        return 2
    except OSError as exc:
        print(f"I/O error: {exc}", file=sys.stderr)
        return 3
    return 0


if __name__ == "__main__":
    sys.exit(main())
