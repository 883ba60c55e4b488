"""Small cases of every kernel path for compute-sanitizer (memcheck):
pair (filter and hash passes, host prefix mode), multi, group, global, plugin ops."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_05485_b200 as tb  # noqa: E402


def batch(rng, b, l, v, r, corr=False, dev=None, pinned=False):
    cid = rng.integers(0, v, (b, l))
    clen = rng.integers(0, l + 1, b)
    refs = []
    for _ in range(r):
        ids = cid.copy() if corr else rng.integers(0, v, (b, l))
        if corr:
            m = rng.random(ids.shape) < 0.3
            ids[m] = rng.integers(0, v, int(m.sum()))
        refs.append((ids, rng.integers(0, l + 1, b)))
    def mk(i, ln):
        if dev:
            return tb.TokenBatch(ids=torch.as_tensor(i, device=dev, dtype=torch.int32), lengths=torch.as_tensor(ln, device=dev))
        if pinned:
            return tb.TokenBatch(ids=torch.as_tensor(i).pin_memory(), lengths=torch.as_tensor(ln))
        return tb.TokenBatch(ids=i, lengths=ln)
    return mk(cid, clen), [mk(i, ln) for i, ln in refs]


def main():
    rng = np.random.default_rng(3)
    cases = [
        dict(b=40, l=200, v=50000, r=1),                 # pair, filter path
        dict(b=40, l=200, v=30, r=1, corr=True),         # pair, hash passes + table orders
        dict(b=20, l=150, v=40000, r=3),                 # multi
        dict(b=20, l=150, v=20, r=3, corr=True),         # multi, table orders
        dict(b=4, l=64, v=20, r=12),                     # group kernel (R > 8)
        dict(b=2, l=20000, v=40, r=1),                   # global-memory kernel
        dict(b=30, l=100, v=1000, r=1, pinned=True),     # host prefix mode
        dict(b=30, l=100, v=1000, r=2, pinned=True),
        dict(b=700, l=48, v=100000, r=1),                # pair, several groups per CTA (prefetch buffer)
        dict(b=700, l=48, v=30, r=1, corr=True),         # the same on the hash passes / list rounds
    ]
    for c in cases:
        cand, refs = batch(rng, **c)
        tb.sentence_bleu(cand, refs, tb.BleuConfig(smoothing="exp"))
        tb.corpus_bleu(cand, refs)
        if c.get("corr"):  # long orders: list rounds beyond order 4, warp-path hand-over
            tb.sentence_bleu(cand, refs, tb.BleuConfig(max_order=9, smoothing="floor"))
    # pageable numpy rows: staged into pinned memory (narrowed), chunk-pipelined for >= 1024 rows
    for bsz in (300, 1100):
        cid = rng.integers(0, 5000, (bsz, 64))
        cl = rng.integers(0, 65, bsz)
        rid = np.where(rng.random((bsz, 64)) < 0.5, cid, rng.integers(0, 5000, (bsz, 64)))
        tb.sentence_bleu(tb.TokenBatch(ids=cid, lengths=cl), [tb.TokenBatch(ids=rid, lengths=cl)],
                         tb.BleuConfig(smoothing="floor"))
    d = torch.device("cuda", 0)
    cand, refs = batch(rng, 64, 128, 500, 1, dev=d)
    tb.compute_stats(cand, refs, tb.BleuConfig())
    rows = rng.integers(0, 5, (300, 3))
    from paper_2510_05485_b200 import _backend
    uniq, inv = _backend.unique_rows(rows)
    counts = _backend.segment_bincount(inv, np.array([100, 100, 100]), uniq.shape[0])
    _backend.clipped_numerators(inv, np.array([100, 100, 100]), counts)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
