"""Full-size parity at every BASELINE.json shape, through
the C-ABI: c2 512x1024 directly against the UNMODIFIED reference package
(oracle/_ref), c2 with correlated references / Zipf / vocab = 1, c3 with add-k
and exp smoothing, the c4 4096x1024 corpus (totals through the 32 replicated
accumulators, and its row shards summed as the NCCL all-reduce would), and
c5 16384x2048 at V = 256k (the whole global batch, and its 8 shards).

Tolerances: counts / lengths / totals bit-exact; fp64 scores within 1e-12
relative with identical zero sets (north_star)."""

import os
import sys

import numpy as np
import pytest
import torch

from conftest import ROOT

sys.path.insert(0, ROOT)
import bench  # noqa: E402  (the workload generator: the reference's generate_batch)
import oracle  # noqa: E402
import paper_2510_05485_b200 as tb  # noqa: E402

pytestmark = pytest.mark.gpu
RTOL = 1e-12


def _dev(a, dt):
    return torch.as_tensor(np.asarray(a)).to("cuda", dtype=dt)


def _device_batches(cand, refs, dt=torch.int32):
    return (tb.TokenBatch(ids=_dev(cand[0], dt), lengths=_dev(cand[1], torch.int64)),
            [tb.TokenBatch(ids=_dev(i, dt), lengths=_dev(ln, torch.int64)) for i, ln in refs])


def _pinned_batches(cand, refs, np_dt=np.int32):
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np_dt)).pin_memory()  # noqa: E731
    return (tb.TokenBatch(ids=pin(cand[0]), lengths=torch.from_numpy(cand[1])),
            [tb.TokenBatch(ids=pin(i), lengths=torch.from_numpy(ln)) for i, ln in refs])


def _np(x):
    return x.cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)


def _assert_stats(st, want):
    for k in ("numerators", "denominators", "cand_lens", "eff_ref_lens"):
        np.testing.assert_array_equal(_np(getattr(st, k)), np.asarray(want[k]), err_msg=k)


def _assert_scores(got, want):
    got, want = _np(got), np.asarray(want)
    np.testing.assert_array_equal(got == 0, want == 0)
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=0)


def _workload(name, data="uniform", seed=42):
    b, l, v, r, smoothing, mode, _ = bench.WORKLOADS[name]
    return bench.generate_batch(b, l, v, r, seed=seed, data=data), smoothing


def _ref_pkg():
    bb = oracle.reference_package()
    if bb is None:
        pytest.skip("reference package not built (oracle/build_ref.sh)")
    return bb


def test_c2_int32_device_vs_reference_package():
    """The headline workload, as the bench times it (int32 device tensors, the
    plan) and as users call it (pinned int32, numpy int64), against the
    reference's own compute_stats / sentence_bleu on the same arrays."""
    bb = _ref_pkg()
    (cand, refs), smoothing = _workload("c2")
    rc = bb.TokenBatch(ids=cand[0], lengths=cand[1])
    rr = [bb.TokenBatch(ids=i, lengths=ln) for i, ln in refs]
    for sm in ("none", "floor", "add-k", "exp"):
        rcfg = bb.BleuConfig(smoothing=sm)
        want_st = bb.compute_stats(rc, rr, rcfg)
        want = dict(numerators=want_st.numerators, denominators=want_st.denominators,
                    cand_lens=want_st.cand_lens, eff_ref_lens=want_st.eff_ref_lens)
        want_scores = bb.sentence_bleu(rc, rr, rcfg).scores
        cfg = tb.BleuConfig(smoothing=sm)
        dc, dr = _device_batches(cand, refs)
        plan = tb.SentenceBleuPlan(dc, dr, cfg)
        plan.run()
        plan.check()
        for k in want:
            np.testing.assert_array_equal(_np(getattr(plan, k)), want[k], err_msg=k)
        _assert_scores(plan.scores, want_scores)
        _assert_stats(tb.compute_stats(dc, dr, cfg), want)
        hc, hr = _pinned_batches(cand, refs)
        _assert_scores(tb.sentence_bleu(hc, hr, cfg).scores, want_scores)
        nc = tb.TokenBatch(ids=cand[0], lengths=cand[1])
        nr = [tb.TokenBatch(ids=i, lengths=ln) for i, ln in refs]
        _assert_stats(tb.compute_stats(nc, nr, cfg), want)
        _assert_scores(tb.sentence_bleu(nc, nr, cfg).scores, want_scores)
        assert float(tb.corpus_bleu(nc, nr, cfg).scores) == pytest.approx(
            float(bb.corpus_bleu(rc, rr, rcfg).scores), rel=RTOL, abs=0)


@pytest.mark.parametrize("data", ["correlated", "zipf", "vocab1"])
def test_c2_related_and_hot_key_data_vs_oracle(data):
    (cand, refs), _ = _workload("c2", data)
    o = oracle.stats(cand[0], cand[1], refs)
    for dt in (torch.int32, torch.int64):
        dc, dr = _device_batches(cand, refs, dt)
        for sm in ("none", "exp"):
            cfg = tb.BleuConfig(smoothing=sm)
            res = tb.sentence_bleu(dc, dr, cfg)
            _assert_stats(tb.compute_stats(dc, dr, cfg), o)
            _assert_scores(res.scores, oracle.scores(o, sm)["scores"])
    hc, hr = _pinned_batches(cand, refs)
    _assert_stats(tb.compute_stats(hc, hr, tb.BleuConfig()), o)


@pytest.mark.parametrize("data", ["uniform", "correlated"])
def test_c3_full_multiref_vs_reference(data):
    """256x1024, 4 references of their own lengths, add-k and exp smoothing."""
    (cand, refs), _ = _workload("c3", data)
    o = oracle.stats(cand[0], cand[1], refs)
    bb = oracle.reference_package()
    if bb is not None and data == "uniform":
        st = bb.compute_stats(bb.TokenBatch(ids=cand[0], lengths=cand[1]),
                              [bb.TokenBatch(ids=i, lengths=ln) for i, ln in refs], bb.BleuConfig())
        np.testing.assert_array_equal(st.numerators, o["numerators"])  # oracle pinned at full size
    dc, dr = _device_batches(cand, refs)
    for sm in ("add-k", "exp"):
        cfg = tb.BleuConfig(smoothing=sm)
        _assert_stats(tb.compute_stats(dc, dr, cfg), o)
        _assert_scores(tb.sentence_bleu(dc, dr, cfg).scores, oracle.scores(o, sm)["scores"])


@pytest.mark.parametrize("data", ["uniform", "correlated"])
def test_c4_full_corpus_and_shard_totals(data):
    """4096x1024 corpus: totals through the replicated L2 accumulators and the
    last-CTA epilogue; 8 row shards' totals summed (what the NCCL all-reduce
    adds) are the global totals, and score_corpus_from_totals of that sum is
    the one-GPU corpus score."""
    (cand, refs), smoothing = _workload("c4", data)
    o = oracle.stats(cand[0], cand[1], refs)
    oc = oracle.corpus(o, smoothing)
    cfg = tb.BleuConfig(smoothing=smoothing)
    dc, dr = _device_batches(cand, refs)
    np.testing.assert_array_equal(_np(tb.corpus_totals(dc, dr, cfg)), oc["totals"])
    assert float(tb.corpus_bleu(dc, dr, cfg).scores) == pytest.approx(oc["scores"], rel=RTOL, abs=0)
    plan = tb.SentenceBleuPlan(dc, dr, cfg, stats=False, corpus=True, sentence=False)
    plan.run()
    plan.check()
    np.testing.assert_array_equal(_np(plan.totals), oc["totals"])
    assert float(plan.corpus[0]) == pytest.approx(oc["scores"], rel=RTOL, abs=0)
    b = cand[0].shape[0]
    acc = torch.zeros(2 * cfg.max_order + 2, dtype=torch.int64, device="cuda")
    for g in range(8):
        lo, hi = bench.shard_rows(b, 8, g)
        sc, sr = _device_batches((cand[0][lo:hi], cand[1][lo:hi]), [(i[lo:hi], ln[lo:hi]) for i, ln in refs])
        acc += tb.corpus_totals(sc, sr, cfg)
    np.testing.assert_array_equal(_np(acc), oc["totals"])
    assert float(tb.score_corpus_from_totals(acc, cfg).scores) == pytest.approx(oc["scores"], rel=RTOL, abs=0)
    bb = oracle.reference_package()
    if bb is not None and data == "uniform":
        ref = bb.corpus_bleu(bb.TokenBatch(ids=cand[0], lengths=cand[1]),
                             [bb.TokenBatch(ids=i, lengths=ln) for i, ln in refs], bb.BleuConfig())
        assert float(plan.corpus[0]) == pytest.approx(float(ref.scores), rel=RTOL, abs=0)


@pytest.mark.parametrize("data", ["uniform", "correlated"])
def test_c5_full_global_batch_and_shards(data):
    """16384x2048 at V = 256k (BASELINE configs[4]) on one GPU, and its 8
    contiguous shards (what each of 8 GPUs scores) equal the global result."""
    (cand, refs), smoothing = _workload("c5", data)
    o = oracle.stats(cand[0], cand[1], refs)
    cfg = tb.BleuConfig(smoothing=smoothing)
    dc, dr = _device_batches(cand, refs)
    plan = tb.SentenceBleuPlan(dc, dr, cfg)
    plan.run()
    plan.check()
    for k in ("numerators", "denominators", "cand_lens", "eff_ref_lens"):
        np.testing.assert_array_equal(_np(getattr(plan, k)), o[k], err_msg=k)
    want = oracle.scores(o, smoothing)["scores"]
    _assert_scores(plan.scores, want)
    b = cand[0].shape[0]
    for g in (0, 7):
        lo, hi = bench.shard_rows(b, 8, g)
        sc, sr = _device_batches((cand[0][lo:hi], cand[1][lo:hi]), [(i[lo:hi], ln[lo:hi]) for i, ln in refs])
        got = _np(tb.sentence_bleu(sc, sr, cfg).scores)
        np.testing.assert_array_equal(got, _np(plan.scores)[lo:hi])  # composition independence: exact
        _assert_scores(got, want[lo:hi])
