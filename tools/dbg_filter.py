import sys, numpy as np
sys.path.insert(0, '/root/repo')
import oracle, paper_2510_05485_b200 as tb
rng = np.random.default_rng(5)
for trial in range(3000):
    b = int(rng.integers(1, 5)); l = int(rng.integers(1, 12)); v = int(rng.integers(1, 6))
    cid = rng.integers(0, v, (b, l)); cl = rng.integers(0, l + 1, b)
    rid = rng.integers(0, v, (b, l)); rl = rng.integers(0, l + 1, b)
    st = tb.compute_stats(tb.TokenBatch(ids=cid, lengths=cl), [tb.TokenBatch(ids=rid, lengths=rl)], tb.BleuConfig(max_order=2))
    o = oracle.stats(cid, cl, [(rid, rl)], 2)
    if not np.array_equal(st.numerators, o["numerators"]):
        print("FAIL", trial, b, l, v); print(cid, cl); print(rid, rl); print(st.numerators, o["numerators"]); break
else:
    print("all ok")
