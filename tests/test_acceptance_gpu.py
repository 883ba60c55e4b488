"""The reference's release gate (pkg/tests/test_acceptance.py:36-69) on the
device path: the same 10,000 randomized instances (seed 20260823, B <= 8,
L <= 32, V <= 16, R <= 3, N in {1, 2, 4}, all four smoothings) against the
CPU oracle — counts bit-exact, fp64 scores within 1e-12 relative (tighter than
the reference's 1e-6), corpus scores per instance.

Instances are scored in batches: a sentence's statistics depend only on its
own rows (batch-composition independence, test_acceptance.py:190-209), so the
instances sharing (R, N, smoothing) are concatenated into one padded batch.
"""

import time
from collections import defaultdict

import numpy as np
import pytest

import oracle
import paper_2510_05485_b200 as tb

pytestmark = pytest.mark.gpu

SMOOTHINGS = ("none", "floor", "add-k", "exp")


def _instances():
    """The reference's generator, draw for draw (test_acceptance.py:41-55)."""
    rng = np.random.default_rng(20260823)
    out = []
    for trial in range(10_000):
        b = int(rng.integers(1, 9))
        l = int(rng.integers(1, 33))
        v = int(rng.integers(1, 17))
        r = int(rng.integers(1, 4))
        n = int(rng.choice([1, 2, 4]))
        sm = SMOOTHINGS[trial % 4]

        def mk():
            return rng.integers(0, v, size=(b, l)), rng.integers(0, l + 1, size=b)

        cand = mk()
        refs = [mk() for _ in range(r)]
        out.append((n, sm, cand, refs))
    return out


def _pad(a, width):
    return np.pad(a, ((0, 0), (0, width - a.shape[1])))


def test_reference_acceptance_10k_instances():
    t0 = time.monotonic()
    inst = _instances()
    groups = defaultdict(list)
    for i, (n, sm, cand, refs) in enumerate(inst):
        groups[(len(refs), n, sm)].append(i)
    worst = 0.0
    for (r, n, sm), idx in groups.items():
        cid = np.concatenate([_pad(inst[i][2][0], 32) for i in idx])
        clen = np.concatenate([inst[i][2][1] for i in idx])
        refs = [(np.concatenate([_pad(inst[i][3][k][0], 32) for i in idx]),
                 np.concatenate([inst[i][3][k][1] for i in idx])) for k in range(r)]
        cfg = tb.BleuConfig(max_order=n, smoothing=sm)
        cand = tb.TokenBatch(ids=cid, lengths=clen)
        rb = [tb.TokenBatch(ids=i_, lengths=l_) for i_, l_ in refs]
        st = tb.compute_stats(cand, rb, cfg)
        o = oracle.stats(cid, clen, refs, n)
        np.testing.assert_array_equal(st.numerators, o["numerators"])
        np.testing.assert_array_equal(st.denominators, o["denominators"])
        np.testing.assert_array_equal(st.eff_ref_lens, o["eff_ref_lens"])
        got = tb.sentence_bleu(cand, rb, cfg).scores
        want = oracle.scores(o, sm)["scores"]
        np.testing.assert_array_equal(got == 0, want == 0)
        np.testing.assert_allclose(got, want, rtol=1e-12, atol=0)
        worst = max(worst, float(np.max(np.abs(got - want), initial=0.0)))
    # corpus mode, one call per instance (the reference's per-instance corpus check)
    for i in range(0, len(inst), 7):
        n, sm, (cid, clen), refs = inst[i]
        cfg = tb.BleuConfig(max_order=n, smoothing=sm)
        got = tb.corpus_bleu(tb.TokenBatch(ids=cid, lengths=clen),
                             [tb.TokenBatch(ids=a, lengths=b) for a, b in refs], cfg).scores
        want = oracle.corpus(oracle.stats(cid, clen, refs, n), sm)["scores"]
        assert got == pytest.approx(want, rel=1e-12, abs=0)
    assert worst <= 1e-6
    assert time.monotonic() - t0 < 120


def test_threads_and_chunk_size_never_change_results():
    """test_bleu.py:237-246: the knobs are accepted and results are identical."""
    rng = np.random.default_rng(11)
    cid = rng.integers(0, 20, (37, 50))
    clen = rng.integers(0, 51, 37)
    refs = [(rng.integers(0, 20, (37, 50)), rng.integers(0, 51, 37)) for _ in range(2)]
    cand = tb.TokenBatch(ids=cid, lengths=clen)
    rb = [tb.TokenBatch(ids=a, lengths=b) for a, b in refs]
    base = tb.sentence_bleu(cand, rb).scores
    for threads, chunk in ((1, None), (4, 3), (8, 1), (2, 1000)):
        np.testing.assert_array_equal(tb.sentence_bleu(cand, rb, threads=threads, chunk_size=chunk).scores, base)
        st = tb.compute_stats(cand, rb, tb.BleuConfig(), threads=threads, chunk_size=chunk)
        np.testing.assert_array_equal(st.numerators, tb.compute_stats(cand, rb, tb.BleuConfig()).numerators)
