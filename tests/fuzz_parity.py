"""Randomised parity sweep of the device path against the C oracle (GPU box).

    python tests/fuzz_parity.py [--seconds 240] [--seed 1]

Draws random shapes (batch, row widths per reference set, 1..12 and 33
references), vocabularies (1 .. 2^40), token dtypes, max orders (1..9, 34),
mutation rates
(related and unrelated text) and lengths (including 0 and the full width),
runs compute_stats on CUDA tensors, pinned host tensors, pageable numpy arrays
and pageable torch tensors, and asserts the
counts are bit-identical to the oracle and the fp64 scores (smoothing cycling
through none / floor / add-k / exp) agree within 1e-12 relative with the
same zero set.  Prints the first failing case with
its seed and exits 1; otherwise the number of cases checked.  Not collected
by pytest (test infrastructure driven by hand / tools/gpu_round.sh).
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2510_05485_b200 as tb  # noqa: E402


def case(rng):
    b = int(rng.choice([1, 3, 17, 64, 700, 1100]))
    R = int(rng.choice([1, 1, 1, 2, 3, 4, 8, 12, 33]))  # 33: beyond the fused kernels (unbounded.py)
    lc = int(rng.choice([1, 7, 64, 300, 1024, 2048]))
    if R > 12:
        b, lc = min(b, 17), min(lc, 64)
    v = int(rng.choice([1, 3, 50, 2000, 128000, 2 ** 40]))
    if b * lc * (R + 1) > 6_000_000:
        b = max(1, 6_000_000 // (lc * (R + 1)))
    cid = rng.integers(0, v, (b, lc), dtype=np.int64)
    clen = rng.integers(0, lc + 1, b)
    clen[rng.random(b) < 0.2] = lc
    refs = []
    for _ in range(R):
        lr = int(rng.choice([lc, max(1, lc // 2), lc + 13]))
        rid = rng.integers(0, v, (b, lr), dtype=np.int64)
        m = min(lc, lr)
        rate = rng.random((b, 1)) * rng.choice([0.0, 0.3, 1.0])
        keep = rng.random((b, m)) >= rate
        rid[:, :m] = np.where(keep & (rng.random((b, 1)) < 0.7), cid[:, :m], rid[:, :m])
        rlen = rng.integers(0, lr + 1, b)
        rlen[rng.random(b) < 0.3] = lr
        refs.append((rid, rlen))
    n = int(rng.choice([1, 2, 4, 4, 4, 6, 9, 34]))  # 34: beyond the fused kernels (unbounded.py)
    if n > 32:  # (fewer rows: the per-order operator path is slower)
        b = min(b, 17)
        refs = [(i[:b], ln[:b]) for i, ln in refs]
        cid, clen = cid[:b], clen[:b]
    dt = torch.int32 if (v < 2 ** 31 and rng.random() < 0.6) else torch.int64
    return cid, clen, refs, n, dt


def run(cid, clen, refs, n, dt, where, smoothing="none"):
    if where == "cuda":
        mk = lambda i, ln: tb.TokenBatch(ids=torch.as_tensor(i).to(dt).cuda(),  # noqa: E731
                                         lengths=torch.as_tensor(ln).cuda())
    elif where == "numpy":  # pageable host arrays, the reference's TokenBatch usage
        mk = lambda i, ln: tb.TokenBatch(ids=i, lengths=ln)  # noqa: E731
    elif where == "pageable":  # pageable torch tensors of the token dtype
        mk = lambda i, ln: tb.TokenBatch(ids=torch.as_tensor(i).to(dt), lengths=torch.as_tensor(ln))  # noqa: E731
    else:
        mk = lambda i, ln: tb.TokenBatch(ids=torch.as_tensor(i).to(dt).pin_memory(),  # noqa: E731
                                         lengths=torch.as_tensor(ln))
    cfg = tb.BleuConfig(max_order=n, smoothing=smoothing)
    cand, rb = mk(cid, clen), [mk(i, ln) for i, ln in refs]
    st = tb.compute_stats(cand, rb, cfg)
    res = tb.sentence_bleu(cand, rb, cfg)
    f = lambda x: x.cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)  # noqa: E731
    return f(st.numerators), f(st.denominators), f(st.eff_ref_lens), f(res.scores)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=240)
    ap.add_argument("--seed", type=int, default=1)
    a = ap.parse_args()
    t0 = time.time()
    k = 0
    while time.time() - t0 < a.seconds:
        seed = a.seed * 1_000_003 + k
        rng = np.random.default_rng(seed)
        cid, clen, refs, n, dt = case(rng)
        o = oracle.stats(cid, clen, refs, n)
        sm = ("none", "floor", "add-k", "exp")[k % 4]
        os_ = oracle.scores(o, sm)["scores"]
        for where in ("cuda", "host", "numpy", "pageable"):
            num, den, eff, sc = run(cid, clen, refs, n, dt, where, sm)
            ok = (np.array_equal(num, o["numerators"]) and np.array_equal(den, o["denominators"])
                  and np.array_equal(eff, o["eff_ref_lens"])
                  and np.array_equal(sc == 0, os_ == 0)
                  and np.allclose(sc, os_, rtol=1e-12, atol=0))
            if not ok:
                bad = np.nonzero((num != o["numerators"]).any(axis=1))[0]
                print(f"MISMATCH seed={seed} where={where} B={cid.shape[0]} L={cid.shape[1]} R={len(refs)} "
                      f"N={n} dtype={dt} smoothing={sm} rows={bad[:10].tolist()} "
                      f"max score rel err {np.max(np.abs(sc - os_) / np.maximum(np.abs(os_), 1e-300)):.3g}")
                sys.exit(1)
        k += 1
    print(f"fuzz ok: {k} cases x 4 paths in {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
