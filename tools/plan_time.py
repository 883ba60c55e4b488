"""Device time of one SentenceBleuPlan launch for an arbitrary shape (A/B runs).

    python tools/plan_time.py B L V R [data] [steps]
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2510_05485_b200 as tb  # noqa: E402


def main():
    b, l, v, r = (int(x) for x in sys.argv[1:5])
    data = sys.argv[5] if len(sys.argv) > 5 else "uniform"
    steps = int(sys.argv[6]) if len(sys.argv) > 6 else 100
    (cid, clen), refs = bench.generate_batch(b, l, v, r, data=data)
    dev = lambda a, dt: torch.as_tensor(a).cuda().to(dt)  # noqa: E731
    cand = tb.TokenBatch(ids=dev(cid, torch.int32), lengths=dev(clen, torch.int64))
    rb = [tb.TokenBatch(ids=dev(i, torch.int32), lengths=dev(x, torch.int64)) for i, x in refs]
    plan = tb.SentenceBleuPlan(cand, rb, tb.BleuConfig())
    for _ in range(10):
        plan.run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(steps):
        plan.run()
    e1.record()
    torch.cuda.synchronize()
    print(f"B={b} L={l} V={v} R={r} {data}: {1000 * e0.elapsed_time(e1) / steps:.2f} us/launch")


if __name__ == "__main__":
    main()
