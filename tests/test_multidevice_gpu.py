"""Tensors on a GPU that is not the current device: every C entry
point switches to the device of the caller's stream (tb_guard.h) and restores
the caller's device, so scoring works from any current device.  Needs two
GPUs; skipped on one."""

import numpy as np
import pytest
import torch

import oracle
import paper_2510_05485_b200 as tb

pytestmark = pytest.mark.gpu

needs2 = pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")


def _instance(rng, batch, width, nrefs, vocab):
    mk = lambda: (rng.integers(0, vocab, (batch, width)), rng.integers(0, width + 1, batch))  # noqa: E731
    (cid, clen) = mk()
    return cid, clen, [mk() for _ in range(nrefs)]


def _np(x):
    return x.cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)


@needs2
@pytest.mark.parametrize("dtype", [torch.int32, torch.int64])
@pytest.mark.parametrize("nrefs", [1, 3])
def test_scores_on_the_non_current_device(dtype, nrefs):
    rng = np.random.default_rng(7)
    cid, clen, refs = _instance(rng, 40, 96, nrefs, 60)
    torch.cuda.set_device(0)
    dev = torch.device("cuda:1")
    t = lambda a, dt=dtype: torch.as_tensor(np.asarray(a), dtype=dt, device=dev)  # noqa: E731
    cand = tb.TokenBatch(ids=t(cid), lengths=t(clen, torch.int64))
    rb = [tb.TokenBatch(ids=t(i), lengths=t(ln, torch.int64)) for i, ln in refs]
    cfg = tb.BleuConfig(smoothing="floor")
    st = tb.compute_stats(cand, rb, cfg)
    res = tb.sentence_bleu(cand, rb, cfg)
    co = tb.corpus_bleu(cand, rb, cfg)
    assert torch.cuda.current_device() == 0  # the caller's device is restored
    assert res.scores.device == dev
    o = oracle.stats(cid, clen, refs, cfg.max_order)
    np.testing.assert_array_equal(_np(st.numerators), o["numerators"])
    np.testing.assert_array_equal(_np(st.denominators), o["denominators"])
    os_ = oracle.scores(o, cfg.smoothing, cfg.eps, cfg.k, cfg.weights)
    np.testing.assert_allclose(_np(res.scores), os_["scores"], rtol=1e-12, atol=0)
    oc = oracle.corpus(o, cfg.smoothing, cfg.eps, cfg.k, cfg.weights)
    assert float(co.scores) == pytest.approx(oc["scores"], rel=1e-12, abs=0)


@needs2
def test_plan_on_the_non_current_device():
    rng = np.random.default_rng(8)
    cid, clen, refs = _instance(rng, 24, 64, 1, 40)
    torch.cuda.set_device(0)
    dev = torch.device("cuda:1")
    t = lambda a, dt=torch.int32: torch.as_tensor(np.asarray(a), dtype=dt, device=dev)  # noqa: E731
    cand = tb.TokenBatch(ids=t(cid), lengths=t(clen, torch.int64))
    rb = [tb.TokenBatch(ids=t(i), lengths=t(ln, torch.int64)) for i, ln in refs]
    plan = tb.SentenceBleuPlan(cand, rb, tb.BleuConfig())
    plan.run()
    plan.replay()  # captured on cuda:1's stream
    torch.cuda.synchronize(dev)
    o = oracle.stats(cid, clen, refs, 4)
    np.testing.assert_array_equal(_np(plan.numerators), o["numerators"])
    assert torch.cuda.current_device() == 0
