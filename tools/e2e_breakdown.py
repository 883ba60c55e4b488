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
    b, l, v, r, sm = bench.WORKLOADS[a.workload][:5]
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


if __name__ == "__main__" and not (len(sys.argv) > 1 and sys.argv[1] in ("native", "ncu")):
    main()


def c2_native_vs_python():
    """tb_bleu_host at c2 through the native binding with prebuilt views vs
    the public sentence_bleu call (the difference is the Python layer)."""
    from paper_2510_05485_b200 import _native, bleu
    b, l, v, r, sm = bench.WORKLOADS["c2"][:5]
    cand, refs = bench.generate_batch(b, l, v, r)
    cfg = tb.BleuConfig(smoothing=sm)
    hc = tb.TokenBatch(ids=torch.from_numpy(cand[0].astype(np.int32)).pin_memory(), lengths=torch.from_numpy(cand[1]))
    hr = [tb.TokenBatch(ids=torch.from_numpy(i.astype(np.int32)).pin_memory(), lengths=torch.from_numpy(ln))
          for i, ln in refs]
    hp = _native.hostpath()
    views = tuple(x._row_view(False)[0] for x in [hc, *hr])
    w = bleu._weights_addr(cfg)
    s = _native.stream_handle(torch.device("cuda", 0))
    print("c2 int32 sentence_bleu  median %8.1f us  min %8.1f us" % t_host(lambda: tb.sentence_bleu(hc, hr, cfg)))
    print("c2 int32 hp.run direct  median %8.1f us  min %8.1f us" % t_host(lambda: hp.run(1, views, b, 4, 0, 0.1, 1.0, w, s)))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(20):
        e0.record()
        hp.run(1, views, b, 4, 0, 0.1, 1.0, w, s)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1000)
    print("c2 int32 events around hp.run (GPU span) median %8.1f us" % float(np.median(ts)))


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "native":
    c2_native_vs_python()
if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "ncu":
    from paper_2510_05485_b200 import _native, bleu
    b, l, v, r, sm = bench.WORKLOADS["c2"][:5]
    cand, refs = bench.generate_batch(b, l, v, r)
    cfg = tb.BleuConfig(smoothing=sm)
    hc = tb.TokenBatch(ids=torch.from_numpy(cand[0].astype(np.int32)).pin_memory(), lengths=torch.from_numpy(cand[1]))
    hr = [tb.TokenBatch(ids=torch.from_numpy(i.astype(np.int32)).pin_memory(), lengths=torch.from_numpy(ln))
          for i, ln in refs]
    for _ in range(10):
        tb.sentence_bleu(hc, hr, cfg)
