"""Any number of reference sets and any n-gram order (the reference caps
neither, bleu.py:24-56, 97-105): beyond the fused kernels' limits
(TB_MAX_REFS / TB_MAX_ORDER) the device n-gram operator kernels serve the
request (unbounded.py).  Counts bit-exact and fp64 scores within 1e-12 of the
oracle; at the limits the two device paths agree exactly; the fp32 epilogue
within 1e-5 relative (north_star)."""

import numpy as np
import pytest
import torch

import oracle
import paper_2510_05485_b200 as tb
from paper_2510_05485_b200 import _native, unbounded

pytestmark = pytest.mark.gpu
RTOL = 1e-12


def _correlated(rng, b, l, v, r):
    cid = rng.integers(0, v, size=(b, l))
    clen = rng.integers(0, l + 1, size=b)
    refs = []
    for _ in range(r):
        ids = cid.copy()
        m = rng.random((b, l)) < rng.uniform(0, 0.6, (b, 1))
        ids[m] = rng.integers(0, v, size=int(m.sum()))
        refs.append((ids, rng.integers(0, l + 1, size=b)))
    return (cid, clen), refs


def _check(cid, clen, refs, cfg, where):
    if where == "device":
        cand = tb.TokenBatch(ids=torch.as_tensor(cid, device="cuda"), lengths=torch.as_tensor(clen, device="cuda"))
        rb = [tb.TokenBatch(ids=torch.as_tensor(i, device="cuda"), lengths=torch.as_tensor(l, device="cuda"))
              for i, l in refs]
    else:
        cand = tb.TokenBatch(ids=cid, lengths=clen)
        rb = [tb.TokenBatch(ids=i, lengths=l) for i, l in refs]
    o = oracle.stats(cid, clen, refs, cfg.max_order)
    st = tb.compute_stats(cand, rb, cfg)
    np_ = lambda x: x.cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)  # noqa: E731
    for k, a in (("numerators", st.numerators), ("denominators", st.denominators),
                 ("cand_lens", st.cand_lens), ("eff_ref_lens", st.eff_ref_lens)):
        np.testing.assert_array_equal(np_(a), o[k], err_msg=k)
    want = oracle.scores(o, cfg.smoothing, cfg.eps, cfg.k, cfg.weights)
    res = tb.sentence_bleu(cand, rb, cfg)
    got = np_(res.scores)
    np.testing.assert_array_equal(got == 0, want["scores"] == 0)
    np.testing.assert_allclose(got, want["scores"], rtol=RTOL, atol=0)
    np.testing.assert_allclose(np_(res.precisions), want["precisions"], rtol=RTOL, atol=0)
    oc = oracle.corpus(o, cfg.smoothing, cfg.eps, cfg.k, cfg.weights)
    assert float(tb.corpus_bleu(cand, rb, cfg).scores) == pytest.approx(oc["scores"], rel=RTOL, abs=0)
    np.testing.assert_array_equal(np_(tb.corpus_totals(cand, rb, cfg)), oc["totals"])


@pytest.mark.parametrize("where", ["device", "host"])
@pytest.mark.parametrize("R", [33, 40])
def test_more_reference_sets_than_the_fused_kernels(where, R):
    rng = np.random.default_rng(R)
    (cid, clen), refs = _correlated(rng, 9, 40, 7, R)
    _check(cid, clen, refs, tb.BleuConfig(smoothing="exp"), where)


@pytest.mark.parametrize("where", ["device", "host"])
@pytest.mark.parametrize("N", [33, 48])
def test_orders_beyond_the_fused_kernels(where, N):
    rng = np.random.default_rng(N)
    (cid, clen), refs = _correlated(rng, 6, 70, 3, 2)
    cid[0, :60] = 1  # long repeats: high orders match
    refs[0][0][0, :60] = 1
    clen[0], refs[0][1][0] = 60, 60
    _check(cid, clen, refs, tb.BleuConfig(max_order=N, smoothing="floor"), where)


def test_unbounded_path_equals_fused_path_at_the_limits():
    rng = np.random.default_rng(5)
    (cid, clen), refs = _correlated(rng, 40, 96, 20, 32)
    dev = torch.device("cuda")
    cand = tb.TokenBatch(ids=torch.as_tensor(cid, device=dev), lengths=torch.as_tensor(clen, device=dev))
    rb = [tb.TokenBatch(ids=torch.as_tensor(i, device=dev), lengths=torch.as_tensor(l, device=dev)) for i, l in refs]
    cfg = tb.BleuConfig(max_order=_native.TB_MAX_ORDER)
    fused = tb.compute_stats(cand, rb, cfg)
    num, den, cl, er = unbounded.stats(cand, rb, cfg.max_order, dev)
    for a, b in ((fused.numerators, num), (fused.denominators, den), (fused.cand_lens, cl),
                 (fused.eff_ref_lens, er)):
        torch.testing.assert_close(a, b, rtol=0, atol=0)


@pytest.mark.parametrize("smoothing", ["none", "floor", "add-k", "exp"])
def test_fp32_epilogue_within_1e5(smoothing):
    rng = np.random.default_rng(7)
    (cid, clen), refs = _correlated(rng, 300, 64, 30, 2)
    cand = tb.TokenBatch(ids=cid, lengths=clen)
    rb = [tb.TokenBatch(ids=i, lengths=l) for i, l in refs]
    cfg = tb.BleuConfig(smoothing=smoothing)
    st = tb.compute_stats(cand, rb, cfg)
    r64 = tb.score_sentences_from_stats(st, cfg)
    r32 = tb.score_sentences_from_stats(st, cfg, dtype=np.float32)
    assert r32.scores.dtype == np.float32
    np.testing.assert_array_equal(r32.scores == 0, r64.scores == 0)
    np.testing.assert_allclose(r32.scores, r64.scores, rtol=1e-5, atol=0)
    np.testing.assert_allclose(r32.precisions, r64.precisions, rtol=1e-5, atol=0)
