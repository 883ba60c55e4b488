"""Where the e2e (host-buffer) time of sentence_bleu goes, on the GPU box.

    python tools/e2e_breakdown.py [--workload c2]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2510_05485_b200 as tb  # noqa: E402


def t_host(fn, reps=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return 1e6 * float(np.median(ts)), 1e6 * float(np.min(ts))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--workload", default="c2")
    a = p.parse_args()
    b, l, v, r, sm = bench.WORKLOADS[a.workload]
    cand, refs = bench.generate_batch(b, l, v, r)
    cfg = tb.BleuConfig(smoothing=sm)
    hc = tb.TokenBatch(ids=torch.from_numpy(cand[0]).pin_memory(), lengths=torch.from_numpy(cand[1]))
    hr = [tb.TokenBatch(ids=torch.from_numpy(i).pin_memory(), lengths=torch.from_numpy(ln)) for i, ln in refs]
    dev = torch.device("cuda", 0)
    dc = tb.TokenBatch(ids=hc.ids.to(dev), lengths=hc.lengths.to(dev))
    dr = [tb.TokenBatch(ids=x.ids.to(dev), lengths=x.lengths.to(dev)) for x in hr]
    tiny_c = tb.TokenBatch(ids=torch.from_numpy(cand[0][:1, :8]).pin_memory(), lengths=torch.tensor([8]))
    tiny_r = [tb.TokenBatch(ids=torch.from_numpy(i[:1, :8]).pin_memory(), lengths=torch.tensor([8])) for i, _ in refs]
    nb = sum(x.ids.numel() * 8 for x in [hc, *hr])
    out = {}
    out["e2e sentence_bleu(host pinned)"] = t_host(lambda: tb.sentence_bleu(hc, hr, cfg))
    out["sentence_bleu(device) + sync"] = t_host(lambda: tb.sentence_bleu(dc, dr, cfg))
    out["tiny host call (python+launch+sync)"] = t_host(lambda: tb.sentence_bleu(tiny_c, tiny_r, cfg))
    bufs = [torch.empty_like(x.ids, device=dev) for x in [hc, *hr]]

    def h2d():
        for buf, x in zip(bufs, [hc, *hr]):
            buf.copy_(x.ids, non_blocking=True)
    out[f"H2D ids only ({nb / 1e6:.1f} MB)"] = t_host(h2d)
    for k, (med, mn) in out.items():
        print(f"{k:45s} median {med:8.1f} us   min {mn:8.1f} us")


if __name__ == "__main__":
    main()
