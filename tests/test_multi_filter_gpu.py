"""The multi-reference kernel's order-1 filter (three Bloom passes, exact
order 1 among <= kSmallSet survivors, the small-set path for orders >= 2):
taken when every CTA has two or more groups, dropped per CTA after a group of
related text.  Counts bit-exact against the C oracle on unrelated, related
and mixed batches (the CTA switching paths mid-batch)."""

import numpy as np
import pytest
import torch

import oracle
import paper_2510_05485_b200 as tb

pytestmark = pytest.mark.gpu


def _batch(rng, b, w, r, v, related_rows):
    cid = rng.integers(0, v, (b, w))
    clen = rng.integers(w // 2, w + 1, b)
    refs = []
    for _ in range(r):
        rid = rng.integers(0, v, (b, w))
        rel = related_rows[:, None] & (rng.random((b, w)) < 0.8)
        rid = np.where(rel, cid, rid)
        refs.append((rid, rng.integers(w // 2, w + 1, b)))
    return cid, clen, refs


@pytest.mark.parametrize("kind", ["unrelated", "related", "mixed", "hot"])
@pytest.mark.parametrize("dtype", [torch.int32, torch.int64])
def test_multi_filter_many_groups(kind, dtype):
    rng = np.random.default_rng({"unrelated": 1, "related": 2, "mixed": 3, "hot": 4}[kind])
    b, w, r = 1600, 160, 3  # > 2 groups per CTA of the multi-reference kernel
    v = 7 if kind == "hot" else 50000
    rel = {"unrelated": np.zeros(b, bool), "related": np.ones(b, bool),
           "mixed": rng.random(b) < 0.3, "hot": np.zeros(b, bool)}[kind]
    cid, clen, refs = _batch(rng, b, w, r, v, rel)
    t = lambda a, dt=dtype: torch.as_tensor(a, dtype=dt, device="cuda")  # noqa: E731
    cand = tb.TokenBatch(ids=t(cid), lengths=t(clen, torch.int64))
    rb = [tb.TokenBatch(ids=t(i), lengths=t(ln, torch.int64)) for i, ln in refs]
    for n in (4, 2, 7):
        st = tb.compute_stats(cand, rb, tb.BleuConfig(max_order=n))
        o = oracle.stats(cid, clen, refs, n)
        np.testing.assert_array_equal(st.numerators.cpu().numpy(), o["numerators"])
        np.testing.assert_array_equal(st.denominators.cpu().numpy(), o["denominators"])
        np.testing.assert_array_equal(st.eff_ref_lens.cpu().numpy(), o["eff_ref_lens"])
