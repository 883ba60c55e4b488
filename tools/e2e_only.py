"""Ten host-path (tb_bleu_host) calls at the bench workload, for ncu launch lists."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2510_05485_b200 as tb  # noqa: E402
w = sys.argv[1] if len(sys.argv) > 1 else "c2"
b, l, v, r, sm = bench.WORKLOADS[w][:5]
cand, refs = bench.generate_batch(b, l, v, r)
hc = tb.TokenBatch(ids=torch.from_numpy(cand[0]).pin_memory(), lengths=torch.from_numpy(cand[1]))
hr = [tb.TokenBatch(ids=torch.from_numpy(i).pin_memory(), lengths=torch.from_numpy(ln)) for i, ln in refs]
cfg = tb.BleuConfig(smoothing=sm)
for _ in range(10):
    tb.sentence_bleu(hc, hr, cfg)
