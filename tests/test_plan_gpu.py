"""SentenceBleuPlan (fixed-shape, pre-bound launches for training loops):
run(), CUDA-graph capture/replay, new tokens written into the bound buffers,
corpus mode + corpus_from_totals, and the sticky error flag — all against the
public API / oracle results."""

import numpy as np
import pytest
import torch

import oracle
import paper_2510_05485_b200 as tb

pytestmark = pytest.mark.gpu


def _batch(rng, b=64, l=200, v=300, r=2, dtype=torch.int32):
    dev = torch.device("cuda", 0)
    cid = rng.integers(0, v, (b, l))
    clen = rng.integers(0, l + 1, b)
    refs = []
    for _ in range(r):
        ids = cid.copy()
        m = rng.random(ids.shape) < 0.5
        ids[m] = rng.integers(0, v, int(m.sum()))
        refs.append((ids, rng.integers(0, l + 1, b)))
    mk = lambda a, dt: torch.as_tensor(a, dtype=dt, device=dev)  # noqa: E731
    cand = tb.TokenBatch(ids=mk(cid, dtype), lengths=mk(clen, torch.int64))
    rb = [tb.TokenBatch(ids=mk(i, dtype), lengths=mk(ln, torch.int64)) for i, ln in refs]
    return (cid, clen), refs, cand, rb


@pytest.mark.parametrize("R", [1, 3])
def test_run_and_replay_match_oracle(R):
    rng = np.random.default_rng(40 + R)
    (cid, clen), refs, cand, rb = _batch(rng, r=R)
    cfg = tb.BleuConfig(smoothing="floor")
    plan = tb.SentenceBleuPlan(cand, rb, cfg)
    plan.run()
    o = oracle.stats(cid, clen, refs)
    np.testing.assert_array_equal(plan.numerators.cpu().numpy(), o["numerators"])
    np.testing.assert_array_equal(plan.denominators.cpu().numpy(), o["denominators"])
    want = oracle.scores(o, "floor")["scores"]
    np.testing.assert_allclose(plan.scores.cpu().numpy(), want, rtol=1e-12, atol=0)
    plan.scores.zero_()
    plan.capture()
    plan.replay()
    torch.cuda.synchronize()
    np.testing.assert_allclose(plan.scores.cpu().numpy(), want, rtol=1e-12, atol=0)
    # new tokens written into the bound buffers are picked up by the next replay
    (cid2, clen2), refs2, cand2, rb2 = _batch(np.random.default_rng(99), r=R)
    cand.ids.copy_(cand2.ids)
    cand.lengths.copy_(cand2.lengths)
    for dst, src in zip(rb, rb2):
        dst.ids.copy_(src.ids)
        dst.lengths.copy_(src.lengths)
    plan.replay()
    torch.cuda.synchronize()
    want2 = oracle.scores(oracle.stats(cid2, clen2, refs2), "floor")["scores"]
    np.testing.assert_allclose(plan.scores.cpu().numpy(), want2, rtol=1e-12, atol=0)
    plan.check()


def test_corpus_plan_and_totals_epilogue():
    rng = np.random.default_rng(7)
    (cid, clen), refs, cand, rb = _batch(rng, r=2, dtype=torch.int64)
    cfg = tb.BleuConfig(smoothing="exp")
    plan = tb.SentenceBleuPlan(cand, rb, cfg, stats=False, corpus=True, sentence=False)
    assert plan.scores is None
    for _ in range(3):  # self-cleaning workspace: repeated runs give the same totals
        plan.run()
    o = oracle.corpus(oracle.stats(cid, clen, refs), "exp")
    np.testing.assert_array_equal(plan.totals.cpu().numpy(), o["totals"])
    assert float(plan.corpus[0]) == pytest.approx(o["scores"], rel=1e-12, abs=0)
    corpus_from_kernel = plan.corpus.clone()
    plan.corpus.zero_()
    plan.corpus_from_totals()
    torch.testing.assert_close(plan.corpus, corpus_from_kernel, rtol=0, atol=0)


def test_plan_flags_bad_lengths_of_trusted_batches():
    rng = np.random.default_rng(8)
    _, _, cand, rb = _batch(rng, r=1)
    bad = tb.TokenBatch.trusted(cand.ids, cand.lengths.clone().fill_(10_000))
    plan = tb.SentenceBleuPlan(bad, rb)
    plan.run()
    with pytest.raises(ValueError, match="lengths"):
        plan.check()
    plan.check()  # cleared
