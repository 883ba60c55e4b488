"""The hash-table kernel's order-1 filter variants: two passes (rows of at
most 256 quads for 256 threads) and three passes (more quads than threads —
candidate tokens into Fc, reference tokens against Fc, candidate tokens
against the small filter of the reference survivors), chosen at launch from
the row widths.  Shapes on both sides of the switch, asymmetric widths,
unrelated / related / mixed rows and exact-match set sizes around 32 and 128
(warp match, block match, fall back to the hash passes) — counts bit-exact
against the C oracle."""

import numpy as np
import pytest
import torch

import oracle
import paper_2510_05485_b200 as tb

pytestmark = pytest.mark.gpu


def _rows(rng, b, wc, wr, v, shared):
    cid = rng.integers(0, v, (b, wc))
    rid = rng.integers(0, v, (b, wr))
    clen = rng.integers(max(1, wc // 2), wc + 1, b)
    rlen = rng.integers(max(1, wr // 2), wr + 1, b)
    # `shared[i]` reference positions copy candidate tokens (the survivor count)
    for i in range(b):
        k = min(int(shared[i]), wr, wc)
        if k:
            src = rng.choice(clen[i], size=min(k, clen[i]), replace=False)
            dst = rng.choice(wr, size=len(src), replace=False)
            rid[i, dst] = cid[i, src]
    return cid, clen, [(rid, rlen)]


@pytest.mark.parametrize("wc,wr", [(512, 512), (508, 516), (516, 508), (1024, 100), (100, 1024), (2000, 48)])
@pytest.mark.parametrize("dtype", [torch.int32, torch.int64])
def test_filter_passes_around_the_switch(wc, wr, dtype):
    rng = np.random.default_rng(wc * 7 + wr)
    b = 700
    shared = rng.choice([0, 3, 14, 20, 40, 70, 200, 10_000], size=b)  # warp / block / hash-pass groups
    cid, clen, refs = _rows(rng, b, wc, wr, 1 << 20, shared)
    t = lambda a, dt=dtype: torch.as_tensor(a, dtype=dt, device="cuda")  # noqa: E731
    cand = tb.TokenBatch(ids=t(cid), lengths=t(clen, torch.int64))
    rb = [tb.TokenBatch(ids=t(i), lengths=t(ln, torch.int64)) for i, ln in refs]
    st = tb.compute_stats(cand, rb, tb.BleuConfig())
    o = oracle.stats(cid, clen, refs, 4)
    np.testing.assert_array_equal(st.numerators.cpu().numpy(), o["numerators"])
    np.testing.assert_array_equal(st.denominators.cpu().numpy(), o["denominators"])
    np.testing.assert_array_equal(st.eff_ref_lens.cpu().numpy(), o["eff_ref_lens"])


@pytest.mark.parametrize("w", [200, 512, 1024])
@pytest.mark.parametrize("n", [4, 9])
def test_warp_path_long_shared_phrases(w, n):
    """<= 32 survivors that form long shared n-grams: warp 0 finishes every
    order in its registers right after the exact order-1 match."""
    rng = np.random.default_rng(w * 31 + n)
    b = 650
    cid = rng.integers(0, 1 << 24, (b, w))
    rid = rng.integers(0, 1 << 24, (b, w))
    clen = rng.integers(w // 2, w + 1, b)
    rlen = rng.integers(w // 2, w + 1, b)
    for i in range(b):  # one or two phrases of up to 10 tokens copied into the reference
        for _ in range(int(rng.integers(1, 3))):
            k = int(rng.integers(1, 11))
            s = int(rng.integers(0, clen[i] - k + 1))
            d = int(rng.integers(0, rlen[i] - k + 1))
            rid[i, d:d + k] = cid[i, s:s + k]
    t = lambda a, dt=torch.int32: torch.as_tensor(a, dtype=dt, device="cuda")  # noqa: E731
    cand = tb.TokenBatch(ids=t(cid), lengths=t(clen, torch.int64))
    rb = [tb.TokenBatch(ids=t(rid), lengths=t(rlen, torch.int64))]
    st = tb.compute_stats(cand, rb, tb.BleuConfig(max_order=n))
    o = oracle.stats(cid, clen, [(rid, rlen)], n)
    np.testing.assert_array_equal(st.numerators.cpu().numpy(), o["numerators"])
    assert (o["numerators"][:, min(n, 5) - 1] > 0).any()  # long matches were exercised
