"""GPU parity: the fused CUDA path (tb_bleu_stats via the public API) against
the reference's golden outputs and the CPU oracle, on identical inputs.

Bar: counts (numerators, denominators, cand_lens, eff_ref_lens) bit-exact;
fp64 scores within 1e-12 relative (north_star), identical zero sets."""

import numpy as np
import pytest
import torch

import oracle
import paper_2510_05485_b200 as tb
from conftest import load_acceptance_cases, load_batch_fixtures, load_frozen_cases, random_instance

pytestmark = pytest.mark.gpu

RTOL = 1e-12  # fp64 scores (north_star: 1e-12 in fp64)
SMOOTHINGS = ("none", "floor", "add-k", "exp")
BATCH_FIXTURES = load_batch_fixtures()


def _cfg(c):
    return tb.BleuConfig(max_order=c["max_order"], weights=c["weights"], smoothing=c["smoothing"],
                         eps=c["eps"], k=c["k"])


def _batches(cand_ids, cand_len, refs, device=None, dtype=torch.int64):
    if device is None:
        return (tb.TokenBatch(ids=np.asarray(cand_ids), lengths=np.asarray(cand_len)),
                [tb.TokenBatch(ids=np.asarray(i), lengths=np.asarray(l)) for i, l in refs])
    t = lambda a, dt=dtype: torch.as_tensor(np.asarray(a), dtype=dt, device=device)  # noqa: E731
    return (tb.TokenBatch(ids=t(cand_ids), lengths=t(cand_len, torch.int64)),
            [tb.TokenBatch(ids=t(i), lengths=t(l, torch.int64)) for i, l in refs])


def _np(x):
    return x.cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)


def _assert_scores(got, want):
    got, want = _np(got), _np(want)
    np.testing.assert_array_equal(got == 0, want == 0)
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=0)


def _check_against_oracle(cand_ids, cand_len, refs, cfg, device="cuda", dtype=torch.int64):
    cand, rb = _batches(cand_ids, cand_len, refs, device, dtype)
    st = tb.compute_stats(cand, rb, cfg)
    o = oracle.stats(cand_ids, cand_len, refs, cfg.max_order)
    np.testing.assert_array_equal(_np(st.numerators), o["numerators"])
    np.testing.assert_array_equal(_np(st.denominators), o["denominators"])
    np.testing.assert_array_equal(_np(st.cand_lens), o["cand_lens"])
    np.testing.assert_array_equal(_np(st.eff_ref_lens), o["eff_ref_lens"])
    res = tb.sentence_bleu(cand, rb, cfg)
    os_ = oracle.scores(o, cfg.smoothing, cfg.eps, cfg.k, cfg.weights)
    _assert_scores(res.scores, os_["scores"])
    np.testing.assert_allclose(_np(res.precisions), os_["precisions"], rtol=RTOL, atol=0)
    np.testing.assert_allclose(_np(res.brevity_penalty), os_["brevity_penalty"], rtol=RTOL, atol=0)
    co = tb.corpus_bleu(cand, rb, cfg)
    oc = oracle.corpus(o, cfg.smoothing, cfg.eps, cfg.k, cfg.weights)
    assert float(co.scores) == pytest.approx(oc["scores"], rel=RTOL, abs=0)
    np.testing.assert_array_equal(_np(tb.corpus_totals(cand, rb, cfg)), oc["totals"])
    return res


# --------------------------------------------------------------------------- golden
@pytest.mark.parametrize("name,inputs,cfgs", BATCH_FIXTURES, ids=[f[0] for f in BATCH_FIXTURES])
@pytest.mark.parametrize("where", ["host", "device"])
def test_golden_fixture(name, inputs, cfgs, where):
    device = None if where == "host" else "cuda"
    cand, rb = _batches(inputs["cand_ids"], inputs["cand_len"], inputs["refs"], device)
    for c, ref in cfgs:
        cfg = _cfg(c)
        st = tb.compute_stats(cand, rb, cfg)
        for key in ("numerators", "denominators", "cand_lens", "eff_ref_lens"):
            np.testing.assert_array_equal(_np(getattr(st, key)), ref[key], err_msg=key)
        res = tb.sentence_bleu(cand, rb, cfg)
        _assert_scores(res.scores, ref["scores"])
        np.testing.assert_allclose(_np(res.precisions), ref["precisions"], rtol=RTOL, atol=0)
        np.testing.assert_allclose(_np(res.brevity_penalty), ref["brevity_penalty"], rtol=RTOL, atol=0)
        co = tb.corpus_bleu(cand, rb, cfg)
        assert float(co.scores) == pytest.approx(float(ref["corpus_score"]), rel=RTOL, abs=0)
        np.testing.assert_allclose(_np(co.precisions), ref["corpus_precisions"], rtol=RTOL, atol=0)
        assert float(co.brevity_penalty) == pytest.approx(float(ref["corpus_bp"]), rel=RTOL, abs=0)


def test_golden_acceptance_cases():
    for case in load_acceptance_cases():
        refs = [(np.array(r["ids"]), np.array(r["len"])) for r in case["refs"]]
        cfg = tb.BleuConfig(max_order=case["max_order"], smoothing=case["smoothing"])
        cand, rb = _batches(np.array(case["cand_ids"]), np.array(case["cand_len"]), refs)
        st = tb.compute_stats(cand, rb, cfg)
        np.testing.assert_array_equal(st.numerators, np.array(case["numerators"]).reshape(st.numerators.shape))
        np.testing.assert_array_equal(st.denominators,
                                      np.array(case["denominators"]).reshape(st.denominators.shape))
        np.testing.assert_array_equal(st.eff_ref_lens, case["eff_ref_lens"])
        res = tb.sentence_bleu(cand, rb, cfg)
        _assert_scores(res.scores, np.array(case["scores"]))
        assert tb.corpus_bleu(cand, rb, cfg).scores == pytest.approx(case["corpus_score"], rel=RTOL, abs=0)


@pytest.mark.parametrize("case", load_frozen_cases(), ids=lambda c: c["smoothing"])
def test_frozen_external_vectors(case):
    """pkg/tests/test_oracle.py:178-185 through the device path (1e-6 there; 1e-9 here)."""
    cfg = tb.BleuConfig(smoothing=case["smoothing"], eps=0.1, k=1.0)
    cand = tb.TokenBatch.from_lists(case["cands"])
    refs = [tb.TokenBatch.from_lists(rs) for rs in case["refsets"]]
    assert tb.corpus_bleu(cand, refs, cfg).scores == pytest.approx(case["expected"], abs=1e-9)
    assert tb.oracle_corpus_bleu(case["cands"], case["refsets"], cfg) == pytest.approx(case["expected"], abs=1e-9)


# --------------------------------------------------------------------------- oracle, random
def test_random_small_instances_vs_oracle(rng):
    for trial in range(200):
        (cid, clen), refs = random_instance(rng)
        cfg = tb.BleuConfig(max_order=int(rng.choice([1, 2, 3, 4, 5])), smoothing=SMOOTHINGS[trial % 4])
        _check_against_oracle(cid, clen, refs, cfg)


@pytest.mark.parametrize("dtype", [torch.int32, torch.int64])
def test_c1_shape_int32_and_int64(dtype):
    rng = np.random.default_rng(42)
    B, L, V = 16, 256, 32000
    cid, clen = rng.integers(0, V, (B, L)), rng.integers(L // 2, L + 1, B)
    refs = [(rng.integers(0, V, (B, L)), rng.integers(L // 2, L + 1, B))]
    for sm in SMOOTHINGS:
        _check_against_oracle(cid, clen, refs, tb.BleuConfig(smoothing=sm), dtype=dtype)


def _correlated(rng, b, l, v, r, p_max=0.9):
    ids = rng.integers(0, v, size=(b, l))
    lens = rng.integers(l // 2, l + 1, size=b)
    refs = []
    for _ in range(r):
        rid = ids.copy()
        mut = rng.random(ids.shape) < rng.random(b)[:, None] * p_max
        rid[mut] = rng.integers(0, v, size=int(mut.sum()))
        refs.append((rid, np.clip(lens + rng.integers(-50, 51, size=b), 0, l)))
    return (ids, lens), refs


@pytest.mark.parametrize("R", [1, 2, 4, 7])
def test_correlated_multiref_vs_oracle(R):
    rng = np.random.default_rng(100 + R)
    (cid, clen), refs = _correlated(rng, 96, 512, 2000, R)
    for sm in SMOOTHINGS:
        _check_against_oracle(cid, clen, refs, tb.BleuConfig(smoothing=sm))


def test_c3_shape_multiref_addk_exp_vs_oracle():
    """BASELINE configs[2]: 256x1024, 4 refs, add-k and exp (correlated refs)."""
    rng = np.random.default_rng(3)
    (cid, clen), refs = _correlated(rng, 256, 1024, 128000, 4, p_max=0.6)
    for sm in ("add-k", "exp"):
        _check_against_oracle(cid, clen, refs, tb.BleuConfig(smoothing=sm))


def test_hot_keys_zipf_and_vocab1():
    rng = np.random.default_rng(11)
    b, l = 64, 1024
    z = lambda s: np.minimum(rng.zipf(1.1, size=s) - 1, 127999)  # noqa: E731
    refs = [(z((b, l)), rng.integers(l // 2, l + 1, b)) for _ in range(2)]
    _check_against_oracle(z((b, l)), rng.integers(l // 2, l + 1, b), refs, tb.BleuConfig(smoothing="floor"))
    refs = [(np.zeros((b, l), dtype=np.int64), rng.integers(0, l + 1, b)) for _ in range(3)]
    _check_against_oracle(np.zeros((b, l), dtype=np.int64), rng.integers(0, l + 1, b), refs,
                          tb.BleuConfig(smoothing="exp"))


def test_wide_rows_global_memory_path():
    """Rows wider than 65535 tokens use the global-memory table variant."""
    rng = np.random.default_rng(5)
    b, l = 3, 70000
    cid = rng.integers(0, 50, (b, l))
    clen = np.array([l, 65536, 1000])
    refs = [(cid.copy(), np.array([l, 70000, 999])), (rng.integers(0, 50, (b, l // 2)), np.array([10, 0, 35000]))]
    _check_against_oracle(cid, clen, refs, tb.BleuConfig(smoothing="floor", max_order=4))


def test_large_shared_table_one_cta_per_sm():
    """R=8 refs of 2048 tokens: the biggest shared-memory table that still fits."""
    rng = np.random.default_rng(6)
    (cid, clen), refs = _correlated(rng, 40, 2048, 30000, 8, p_max=0.5)
    _check_against_oracle(cid, clen, refs, tb.BleuConfig(smoothing="add-k"))


def test_max_refs_and_long_orders():
    rng = np.random.default_rng(9)
    (cid, clen), refs = _correlated(rng, 8, 64, 6, 32)
    _check_against_oracle(cid, clen, refs, tb.BleuConfig(max_order=8, smoothing="exp"))


@pytest.mark.parametrize("order", [5, 9, 13])
def test_single_ref_long_orders_all_live_list_regimes(order):
    """Single reference, max_order > 4: the live-list table orders hand over to
    the warp match path, whose 64-bit keys cover three orders at a time (so
    orders 5+ chain a new id).  Mutation rates from 0 to 1 give every survivor
    count from none through <= 32 (warp path from order 2) to all positions."""
    rng = np.random.default_rng(40 + order)
    b, l = 96, 384
    cid = rng.integers(0, 3000, (b, l))
    clen = rng.integers(l // 2, l + 1, b)
    rid = cid.copy()
    rate = np.linspace(0.0, 1.0, b)[:, None]
    mut = rng.random((b, l)) < rate
    rid[mut] = rng.integers(0, 3000, size=int(mut.sum()))
    rlen = np.clip(clen + rng.integers(-8, 9, b), 0, l)
    rlen[:4] = clen[:4]  # identical rows: every n-gram of every order matches
    rid[:4] = cid[:4]
    for dt in (torch.int32, torch.int64):
        _check_against_oracle(cid, clen, [(rid, rlen)], tb.BleuConfig(max_order=order, smoothing="floor"), dtype=dt)


@pytest.mark.parametrize("R,order", [(2, 4), (3, 7), (8, 5)])
def test_multi_ref_live_list_rounds(R, order):
    """2 <= R <= 8: the live-list table rounds of orders >= 2 (more than 128
    live positions), the hand-over to the small-set path, and every survivor
    regime from identical rows (all live at every order) to unrelated rows."""
    rng = np.random.default_rng(70 + R + order)
    b, l = 64, 320
    cid = rng.integers(0, 4000, (b, l))
    clen = rng.integers(l // 2, l + 1, b)
    refs = []
    for r in range(R):
        rid = cid.copy()
        mut = rng.random((b, l)) < np.linspace(0.0, 1.0, b)[:, None] * (0.5 + 0.5 * r / R)
        rid[mut] = rng.integers(0, 4000, size=int(mut.sum()))
        rlen = np.clip(clen + rng.integers(-6, 7, b), 0, l)
        if r == 0:
            rid[:3], rlen[:3] = cid[:3], clen[:3]
        refs.append((rid, rlen))
    for dt in (torch.int32, torch.int64):
        _check_against_oracle(cid, clen, refs, tb.BleuConfig(max_order=order, smoothing="add-k"), dtype=dt)


@pytest.mark.parametrize("l,v", [(3000, 200000), (6000, 500), (8190, 40)])
def test_single_ref_wide_rows_big_shared_tables(l, v):
    """R = 1 rows of 3k-8k tokens: the pair kernel at 1-3 CTAs per SM with
    the largest tables and live lists (u16 positions up to ~16k), related and
    unrelated rows, and rows too wide for it (the generic kernel)."""
    rng = np.random.default_rng(l + v)
    b = 6
    cid = rng.integers(0, v, (b, l))
    clen = np.array([l, l - 1, l // 2, 1, 0, l - 3])
    rid = cid.copy()
    mut = rng.random((b, l)) < np.array([0.0, 0.05, 0.5, 1.0, 0.3, 0.9])[:, None]
    rid[mut] = rng.integers(0, v, size=int(mut.sum()))
    rlen = np.array([l, l, l // 3, 5, 7, l - 100])
    for dt in (torch.int32, torch.int64):
        _check_against_oracle(cid, clen, [(rid, rlen)], tb.BleuConfig(smoothing="exp"), dtype=dt)


def test_huge_token_ids_and_negative_padding():
    rng = np.random.default_rng(12)
    b, l = 32, 300
    cid = rng.integers(2**45, 2**45 + 4, (b, l))
    clen = rng.integers(0, l + 1, b)
    cid[np.arange(l) >= clen[:, None]] = -1
    refs = [(rng.integers(2**45, 2**45 + 4, (b, l)), rng.integers(0, l + 1, b))]
    _check_against_oracle(cid, clen, refs, tb.BleuConfig(smoothing="floor"))


def test_unaligned_rows_and_strided_views():
    """Row starts not 16-B aligned (odd ld) exercise the non-bulk staging path."""
    rng = np.random.default_rng(13)
    base = torch.as_tensor(rng.integers(0, 40, (50, 301)), device="cuda")
    ids = base[:, 1:300]          # ld 301, offset 1 element
    lens = torch.as_tensor(rng.integers(0, 300, 50), device="cuda")
    rbase = torch.as_tensor(rng.integers(0, 40, (50, 257)), device="cuda", dtype=torch.int32)
    rids = rbase[:, 3:250]
    rlens = torch.as_tensor(rng.integers(0, 248, 50), device="cuda")
    cand = tb.TokenBatch(ids=ids, lengths=lens)
    ref = tb.TokenBatch(ids=rids, lengths=rlens)
    got = tb.compute_stats(cand, [ref], tb.BleuConfig())
    o = oracle.stats(ids.cpu().numpy(), lens.cpu().numpy(), [(rids.cpu().numpy(), rlens.cpu().numpy())])
    np.testing.assert_array_equal(_np(got.numerators), o["numerators"])


# --------------------------------------------------------------------------- edge cases
def test_empty_batch():
    cand = tb.TokenBatch(ids=np.zeros((0, 5), dtype=np.int64), lengths=np.zeros(0, dtype=np.int64))
    res = tb.sentence_bleu(cand, [cand])
    assert res.scores.shape == (0,) and res.precisions.shape == (0, 4)
    co = tb.corpus_bleu(cand, [cand])
    assert co.scores == 0.0 and co.brevity_penalty == 0.0
    st = tb.compute_stats(cand, [cand], tb.BleuConfig())
    assert st.numerators.shape == (0, 4)


def test_zero_lengths_and_short_rows():
    cand = tb.TokenBatch(ids=[[9, 9, 9], [1, 2, 0]], lengths=[0, 2])
    ref = tb.TokenBatch.from_lists([[1, 2, 3], [1, 2, 3, 4]])
    st = tb.compute_stats(cand, [ref], tb.BleuConfig())
    np.testing.assert_array_equal(st.denominators, [[0, 0, 0, 0], [2, 1, 0, 0]])
    np.testing.assert_array_equal(st.numerators, [[0, 0, 0, 0], [2, 1, 0, 0]])
    res = tb.sentence_bleu(cand, [ref], tb.BleuConfig(smoothing="floor"))
    assert res.scores[0] == 0.0 and res.brevity_penalty[0] == 0.0


def test_zero_width_batches():
    cand = tb.TokenBatch(ids=np.zeros((3, 0), dtype=np.int64), lengths=np.zeros(3, dtype=np.int64))
    ref = tb.TokenBatch.from_lists([[1], [2, 3], []])
    res = tb.sentence_bleu(cand, [ref])
    np.testing.assert_array_equal(res.scores, 0.0)


def test_reference_hand_cases():
    """pkg/tests/test_bleu.py:118-210 on the device."""
    THE, REF_A, REF_B = 0, [0, 1, 2, 3, 0, 4], [5, 2, 6, 1, 3, 0, 4]
    cand = tb.TokenBatch.from_lists([[THE] * 7])
    refs = [tb.TokenBatch.from_lists([REF_A], min_width=7), tb.TokenBatch.from_lists([REF_B])]
    st = tb.compute_stats(cand, refs, tb.BleuConfig())
    assert st.numerators[0, 0] == 2 and st.denominators[0, 0] == 7
    assert tb.sentence_bleu(cand, refs, tb.BleuConfig(max_order=1)).scores[0] == pytest.approx(2 / 7)
    batch = tb.TokenBatch.from_lists([[3, 1, 4, 1, 5]])
    st = tb.compute_stats(batch, [batch], tb.BleuConfig())
    np.testing.assert_array_equal(st.numerators, st.denominators)
    batch = tb.TokenBatch.from_lists([[1, 2, 3, 4, 5, 6]])
    assert tb.sentence_bleu(batch, [batch]).scores[0] == pytest.approx(1.0)
    assert tb.sentence_bleu(tb.TokenBatch.from_lists([[1] * 5]),
                            [tb.TokenBatch.from_lists([[2] * 5])]).scores[0] == 0.0


# --------------------------------------------------------------------------- properties
def test_padding_invariance_exact(rng):
    for _ in range(100):
        (cid, clen), refs = random_instance(rng, max_len=40)
        cfg = tb.BleuConfig(smoothing="exp")
        base = tb.sentence_bleu(*_batches(cid, clen, refs), cfg).scores

        def scramble(ids, lens):
            ids = ids.copy()
            pad = np.arange(ids.shape[1]) >= lens[:, None]
            ids[pad] = rng.integers(-5, 10_000, size=int(pad.sum()))
            return ids, lens

        mutated = tb.sentence_bleu(*_batches(*scramble(cid, clen), [scramble(*r) for r in refs]), cfg).scores
        np.testing.assert_array_equal(base, mutated)


def test_batch_composition_independence_exact(rng):
    for _ in range(100):
        (cid, clen), refs = random_instance(rng, max_b=8)
        b = len(clen)
        if b < 2:
            continue
        cfg = tb.BleuConfig(smoothing="floor")
        full = tb.sentence_bleu(*_batches(cid, clen, refs), cfg).scores
        keep = np.sort(rng.choice(b, size=int(rng.integers(1, b)), replace=False))
        sub = tb.sentence_bleu(*_batches(cid[keep], clen[keep], [(i[keep], l[keep]) for i, l in refs]), cfg).scores
        np.testing.assert_array_equal(full[keep], sub)


def test_permutation_equivariance(rng):
    (cid, clen), refs = random_instance(rng, max_b=8)
    perm = rng.permutation(len(clen))
    base = tb.sentence_bleu(*_batches(cid, clen, refs)).scores
    permuted = tb.sentence_bleu(*_batches(cid[perm], clen[perm], [(i[perm], l[perm]) for i, l in refs])).scores
    np.testing.assert_array_equal(permuted, base[perm])


def test_host_and_device_modes_identical():
    rng = np.random.default_rng(21)
    (cid, clen), refs = _correlated(rng, 200, 256, 1000, 2)
    cfg = tb.BleuConfig(smoothing="floor")
    h = tb.sentence_bleu(*_batches(cid, clen, refs), cfg)
    d = tb.sentence_bleu(*_batches(cid, clen, refs, "cuda"), cfg)
    d32 = tb.sentence_bleu(*_batches(cid, clen, refs, "cuda", torch.int32), cfg)
    np.testing.assert_array_equal(h.scores, d.scores.cpu().numpy())
    np.testing.assert_array_equal(h.scores, d32.scores.cpu().numpy())
    pinned = (tb.TokenBatch(ids=torch.as_tensor(cid).pin_memory(), lengths=torch.as_tensor(clen)),
              [tb.TokenBatch(ids=torch.as_tensor(i).pin_memory(), lengths=torch.as_tensor(l)) for i, l in refs])
    np.testing.assert_array_equal(h.scores, tb.sentence_bleu(*pinned, cfg).scores)


def test_repeated_calls_and_workspace_reuse():
    """The corpus accumulators and completion counter are self-cleaning."""
    rng = np.random.default_rng(22)
    (cid, clen), refs = _correlated(rng, 300, 128, 500, 2)
    cand, rb = _batches(cid, clen, refs, "cuda")
    first = tb.corpus_totals(cand, rb).clone()
    for _ in range(5):
        torch.testing.assert_close(tb.corpus_totals(cand, rb), first, rtol=0, atol=0)
        tb.sentence_bleu(cand, rb)


def test_full_size_c2_properties():
    """BASELINE configs[1] shape (512x1024, V=128k): candidate == reference gives
    num == den at every order; counts vs oracle bit-exact."""
    rng = np.random.default_rng([42, 512, 1024, 128000])
    ids = rng.integers(0, 128000, (512, 1024))
    lens = rng.integers(512, 1025, 512)
    cand, rb = _batches(ids, lens, [(ids, lens)], "cuda")
    st = tb.compute_stats(cand, rb, tb.BleuConfig())
    torch.testing.assert_close(st.numerators, st.denominators, rtol=0, atol=0)
    np.testing.assert_array_equal(tb.sentence_bleu(cand, rb).scores.cpu().numpy(), 1.0)
    refs = [(rng.integers(0, 128000, (512, 1024)), rng.integers(512, 1025, 512))]
    _check_against_oracle(ids, lens, refs, tb.BleuConfig())


# --------------------------------------------------------------------------- errors
def test_device_validation_errors():
    with pytest.raises(ValueError, match="lengths must lie"):
        tb.TokenBatch(ids=torch.zeros((2, 3), dtype=torch.int64, device="cuda"),
                      lengths=torch.tensor([1, 4], device="cuda"))
    with pytest.raises(ValueError, match="non-negative"):
        tb.TokenBatch(ids=torch.tensor([[-1, 2]], device="cuda"), lengths=torch.tensor([2], device="cuda"))
    tb.TokenBatch(ids=torch.tensor([[1, -9]], device="cuda"), lengths=torch.tensor([1], device="cuda"))


def test_kernel_flags_bad_lengths_for_trusted_batches():
    ids = torch.zeros((2, 3), dtype=torch.int64, device="cuda")
    bad = tb.TokenBatch.trusted(ids, torch.tensor([1, 4], device="cuda"))
    ok = tb.TokenBatch(ids=np.zeros((2, 3), dtype=np.int64), lengths=[1, 1])
    # device mode does not synchronise: check_device_flags surfaces (and clears) the flag
    tb.check_device_flags()
    res = tb.sentence_bleu(bad, [bad])
    assert res.scores.shape == (2,)
    with pytest.raises(ValueError, match="lengths"):
        tb.check_device_flags()
    tb.check_device_flags()  # cleared
    # the host-mode launch reports it at once
    with pytest.raises(ValueError):
        tb.sentence_bleu(ok, [tb.TokenBatch.trusted(ids, torch.tensor([1, 4], device="cuda"))])


def test_score_from_stats_roundtrip():
    rng = np.random.default_rng(23)
    (cid, clen), refs = _correlated(rng, 64, 100, 300, 3)
    for sm in SMOOTHINGS:
        cfg = tb.BleuConfig(smoothing=sm)
        cand, rb = _batches(cid, clen, refs)
        st = tb.compute_stats(cand, rb, cfg)
        a = tb.score_sentences_from_stats(st, cfg)
        b = tb.sentence_bleu(cand, rb, cfg)
        np.testing.assert_array_equal(a.scores, b.scores)
        np.testing.assert_array_equal(tb.apply_smoothing(st, cfg), b.precisions)
        assert tb.score_corpus_from_stats(st, cfg).scores == tb.corpus_bleu(cand, rb, cfg).scores


def test_apply_smoothing_reference_examples():
    """pkg/tests/test_bleu.py:88-115."""
    def stats(num, den):
        num, den = np.asarray(num), np.asarray(den)
        return tb.SentenceStats(numerators=num, denominators=den, cand_lens=np.full(len(num), 5),
                                eff_ref_lens=np.full(len(num), 5))
    for m in ("none", "floor", "exp"):
        assert tb.apply_smoothing(stats([[2]], [[7]]), tb.BleuConfig(max_order=1, smoothing=m))[0, 0] == \
            pytest.approx(2 / 7)
    assert tb.apply_smoothing(stats([[0]], [[4]]), tb.BleuConfig(max_order=1, smoothing="floor"))[0, 0] == \
        pytest.approx(0.025)
    np.testing.assert_allclose(tb.apply_smoothing(stats([[1, 0, 0]], [[3, 2, 1]]),
                                                  tb.BleuConfig(max_order=3, smoothing="exp"))[0],
                               [1 / 3, 1 / 4, 1 / 4])
    p = tb.apply_smoothing(stats([[0, 0]], [[4, 3]]), tb.BleuConfig(max_order=2, smoothing="add-k"))
    assert p[0, 0] == 0.0 and p[0, 1] == pytest.approx(0.25)
    for m in SMOOTHINGS:
        assert tb.apply_smoothing(stats([[0]], [[0]]), tb.BleuConfig(max_order=1, smoothing=m))[0, 0] == 0.0


def test_filter_path_boundaries_and_mixed_regimes():
    """Rows whose candidate and reference share exactly K tokens, so that the
    order-1 filter keeps ~2K positions: around the warp (32) and block (128)
    limits of the exact-match paths and beyond (hash passes); > 592 rows so
    CTAs process several groups and switch regimes mid-launch."""
    rng = np.random.default_rng(33)
    L = 300
    ks = [0, 1, 15, 16, 17, 31, 32, 33, 63, 64, 65, 100, 150]
    rows_c, rows_r, lc, lr = [], [], [], []
    for i in range(700):
        k = ks[i % len(ks)]
        shared = rng.choice(1000, size=k, replace=False) + 10_000
        cand = np.concatenate([shared, rng.integers(100_000, 200_000, L - k)])
        ref = np.concatenate([rng.permutation(shared), rng.integers(300_000, 400_000, L - k)])
        if i % 3 == 0:  # repeats of shared tokens on both sides
            cand[-5:] = shared[:5] if k >= 5 else cand[-5:]
        rng.shuffle(cand)
        rng.shuffle(ref)
        rows_c.append(cand)
        rows_r.append(ref)
        lc.append(int(rng.integers(L - 20, L + 1)))
        lr.append(int(rng.integers(L - 20, L + 1)))
    cid, rid = np.stack(rows_c), np.stack(rows_r)
    clen, rlen = np.array(lc), np.array(lr)
    for dtype in (torch.int32, torch.int64):
        _check_against_oracle(cid, clen, [(rid, rlen)], tb.BleuConfig(smoothing="floor"), dtype=dtype)
