"""e2e cost of sentence_bleu on host inputs of every kind at c2 (GPU box):
numpy int64 (the reference's TokenBatch), pageable / pinned torch tensors.
Cycles through 8 distinct batches (cold CPU caches, like new data per call).

    python tools/pageable_e2e.py
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2510_05485_b200 as tb  # noqa: E402

b, l, v, r, sm = bench.WORKLOADS["c2"][:5]
cfg = tb.BleuConfig(smoothing=sm)
data = [bench.generate_batch(b, l, v, r, seed=42 + i) for i in range(8)]


def t(make, reps=48):
    sets = [(make(c[0], c[1]), [make(i, ln) for i, ln in refs]) for c, refs in data]
    for c, rb in sets:
        tb.sentence_bleu(c, rb, cfg)
    ts = []
    for k in range(reps):
        c, rb = sets[k % len(sets)]
        t0 = time.perf_counter()
        tb.sentence_bleu(c, rb, cfg)
        ts.append(time.perf_counter() - t0)
    return 1e6 * float(np.median(ts))


print("numpy int64 pageable (reference-style TokenBatch): %.1f us" % t(lambda i, ln: tb.TokenBatch(ids=i, lengths=ln)))
print("torch int32 pageable: %.1f us" % t(lambda i, ln: tb.TokenBatch(ids=torch.from_numpy(i.astype(np.int32)),
                                                                       lengths=torch.from_numpy(ln))))
print("torch int32 pinned:   %.1f us" % t(lambda i, ln: tb.TokenBatch(ids=torch.from_numpy(i.astype(np.int32)).pin_memory(),
                                                                       lengths=torch.from_numpy(ln))))
print("torch int64 pinned:   %.1f us" % t(lambda i, ln: tb.TokenBatch(ids=torch.from_numpy(i).pin_memory(),
                                                                       lengths=torch.from_numpy(ln))))
