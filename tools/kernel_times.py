"""Run one workload's plan a few times (for ncu launch lists / captures).

    python tools/kernel_times.py [workload] [data] [runs]
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2510_05485_b200 as tb  # noqa: E402


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
    data = sys.argv[2] if len(sys.argv) > 2 else "uniform"
    runs = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    b, l, v, r, sm, mode, _ = bench.WORKLOADS[wl]
    (cid, clen), refs = bench.generate_batch(b, l, v, r, data=data)
    dev = lambda a, dt: torch.as_tensor(a).cuda().to(dt)  # noqa: E731
    cand = tb.TokenBatch(ids=dev(cid, torch.int32), lengths=dev(clen, torch.int64))
    rb = [tb.TokenBatch(ids=dev(i, torch.int32), lengths=dev(x, torch.int64)) for i, x in refs]
    cfg = tb.BleuConfig(smoothing=sm)
    plan = (tb.SentenceBleuPlan(cand, rb, cfg, stats=False, corpus=True, sentence=False) if mode == "corpus"
            else tb.SentenceBleuPlan(cand, rb, cfg))
    for _ in range(runs):
        plan.run()
    torch.cuda.synchronize()
    plan.check()
    print("ok", wl, data)


if __name__ == "__main__":
    main()
