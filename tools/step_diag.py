"""Step-time diagnostics for the headline workload: how the L2 flush method
and back-to-back launches change the measured per-step kernel time."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2510_05485_b200 as tb  # noqa: E402


def main(workload="c2"):
    b, l, v, r, sm = bench.WORKLOADS[workload][:5]
    (cid, clen), refs = bench.generate_batch(b, l, v, r)
    cand = tb.TokenBatch(ids=torch.as_tensor(cid).cuda().to(torch.int32), lengths=torch.as_tensor(clen).cuda())
    rb = [tb.TokenBatch(ids=torch.as_tensor(i).cuda().to(torch.int32), lengths=torch.as_tensor(x).cuda())
          for i, x in refs]
    plan = tb.SentenceBleuPlan(cand, rb, tb.BleuConfig(smoothing=sm))
    plan.capture()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()

    def timed(pre, k=30):
        ts = []
        for _ in range(k):
            pre()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(s)
            plan.replay()
            e1.record(s)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        return np.median(ts), np.min(ts)

    for name, pre in [("zero_ flush", lambda: flush.zero_()),
                      ("read flush", lambda: flush.sum(dtype=torch.int64)),
                      ("no flush", lambda: None)]:
        for _ in range(3):
            pre()
            plan.replay()
        med, mn = timed(pre)
        print(f"{name:12s}: median {med:7.2f} us  min {mn:7.2f} us")
    # back-to-back
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(s)
    for _ in range(100):
        plan.replay()
    e1.record(s)
    e1.synchronize()
    print(f"back-to-back replays: {e0.elapsed_time(e1) * 1e3 / 100:7.2f} us each")
    # empty-kernel launch latency reference
    x = torch.zeros(1, device="cuda")
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        x.add_(1)
    ts = []
    for _ in range(30):
        flush.zero_()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(s)
        g.replay()
        e1.record(s)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"tiny graph after zero_ flush: median {np.median(ts):7.2f} us")


if __name__ == "__main__":
    main(*(sys.argv[1:]))
