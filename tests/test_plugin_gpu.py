"""Device versions of the reference operator/plugin surface and spec-level
n-gram ops (pkg/tests/test_ngrams.py, test_acceptance.py:72-101,
test_properties.py:15-32), checked against the reference's golden outputs
and the oracle."""

import numpy as np
import pytest
import torch
from hypothesis import given, settings, strategies as st

import oracle
import paper_2510_05485_b200 as tb
from paper_2510_05485_b200 import _backend
from paper_2510_05485_b200.ngrams import flatten_valid
from conftest import load_ngram_ops

pytestmark = pytest.mark.gpu


def test_golden_ngram_ops():
    """unique_rows is byte-identical to the reference's (lexicographic unique
    rows and their inverse, _kernels.pyx:36-81); the segment kernels too."""
    for op in load_ngram_ops():
        rows = np.array(op["rows"], dtype=np.int64).reshape(-1, op["n"])
        uniq, inv = _backend.unique_rows(rows)
        ref_u = np.array(op["unique"], dtype=np.int64).reshape(-1, op["n"])
        ref_inv = np.array(op["inverse"], dtype=np.int64)
        np.testing.assert_array_equal(uniq, ref_u)
        np.testing.assert_array_equal(inv, ref_inv)
        np.testing.assert_array_equal(uniq[inv], rows)
        seg = np.array(op["seg"], dtype=np.int64)
        flat = np.array(op["flat"], dtype=np.int64)
        counts = _backend.segment_bincount(flat, seg, op["u"])
        np.testing.assert_array_equal(counts, np.array(op["counts"]).reshape(counts.shape))
        rm = np.array(op["ref_max"], dtype=np.int32).reshape(len(seg), -1)
        np.testing.assert_array_equal(_backend.clipped_numerators(flat, seg, rm), op["clipped"])


@pytest.mark.parametrize("n,hi", [(1, 1 << 40), (3, 30), (4, 128000), (2, 1 << 62)])
def test_unique_rows_lexicographic_like_numpy_large(n, hi):
    """np.unique(axis=0) is the reference python backend's order
    (_py_kernels.py:24-33: lexsort over the columns, signed int64)."""
    rng = np.random.default_rng(n)
    rows = rng.integers(-hi, hi, size=(200_000, n))
    rows[100_000:150_000] = rows[:50_000]  # duplicates
    uniq, inv = _backend.unique_rows(rows)
    ref_u, ref_inv = np.unique(rows, axis=0, return_inverse=True)
    np.testing.assert_array_equal(uniq, ref_u)
    np.testing.assert_array_equal(inv, ref_inv.reshape(-1))
    d_uniq, d_inv = _backend.unique_rows(torch.as_tensor(rows, device="cuda"))
    assert d_uniq.is_cuda
    np.testing.assert_array_equal(d_inv.cpu().numpy(), inv)
    np.testing.assert_array_equal(d_uniq.cpu().numpy(), uniq)


def test_unique_rows_matches_reference_backend():
    bb = oracle.reference_package()
    if bb is None:
        pytest.skip("reference package not built")
    from batchbleu import _py_kernels
    rng = np.random.default_rng(5)
    for t, n, v in [(1, 1, 5), (17, 2, 3), (5000, 4, 50), (3000, 1, 2)]:
        rows = rng.integers(0, v, size=(t, n))
        ru, ri = _py_kernels.unique_rows(rows)
        u, i = _backend.unique_rows(rows)
        np.testing.assert_array_equal(u, ru)
        np.testing.assert_array_equal(i, ri)


def test_unique_rows_empty():
    u, i = _backend.unique_rows(np.empty((0, 3), dtype=np.int64))
    assert u.shape == (0, 3) and i.shape == (0,)


def test_spec_examples():
    """pkg/tests/test_ngrams.py:17-90."""
    s = tb.extract_ngrams(tb.TokenBatch(ids=[[1, 2, 3, 4]], lengths=[4]), 2)
    assert s.valid_counts.tolist() == [3]
    np.testing.assert_array_equal(s.slices[0, :3], [[1, 2], [2, 3], [3, 4]])
    s = tb.extract_ngrams(tb.TokenBatch(ids=[[7]], lengths=[1]), 2)
    assert s.valid_counts.tolist() == [0] and flatten_valid(s).shape == (0, 2)
    np.testing.assert_array_equal(flatten_valid(tb.extract_ngrams(tb.TokenBatch(ids=[[1, 2, 3, 9, 9]],
                                                                                lengths=[3]), 2)),
                                  [[1, 2], [2, 3]])
    with pytest.raises(ValueError):
        tb.extract_ngrams(tb.TokenBatch(ids=[[1, 2]], lengths=[2]), 0)
    cand = tb.extract_ngrams(tb.TokenBatch(ids=[[1, 2, 1, 2]], lengths=[4]), 2)
    ref = tb.extract_ngrams(tb.TokenBatch(ids=[[3, 4]], lengths=[2]), 2)
    d = tb.build_dictionary(cand, [ref])
    assert d.num_unique == 3
    inv = d.inverse_indices
    assert inv[0] == inv[2] and inv[0] != inv[1]
    np.testing.assert_array_equal(d.unique_ngrams[inv[0]], [1, 2])
    np.testing.assert_array_equal(d.unique_ngrams[inv[3]], [3, 4])
    c2 = tb.extract_ngrams(tb.TokenBatch(ids=[[1, 2, 3]], lengths=[3]), 2)
    r2 = tb.extract_ngrams(tb.TokenBatch(ids=[[7, 8, 9]], lengths=[3]), 2)
    assert tb.build_dictionary(c2, [r2]).num_unique == 4
    with pytest.raises(ValueError):
        tb.build_dictionary(c2, [tb.extract_ngrams(tb.TokenBatch(ids=[[1, 2, 3]], lengths=[3]), 3)])
    with pytest.raises(ValueError):
        tb.build_dictionary(c2, [])


@pytest.mark.parametrize("where", ["host", "device"])
def test_dictionary_reconstruction_random(where):
    """test_acceptance.py:72-101 (reconstruction half), 300 instances."""
    rng = np.random.default_rng(7)
    for _ in range(300):
        b = int(rng.integers(1, 13))
        n = int(rng.integers(1, 4))
        l = int(rng.integers(1, 20))
        v = int(rng.integers(1, 10))

        def mk():
            ids, lens = rng.integers(0, v, size=(b, l)), rng.integers(0, l + 1, size=b)
            if where == "device":
                ids, lens = torch.as_tensor(ids, device="cuda"), torch.as_tensor(lens, device="cuda")
            return tb.extract_ngrams(tb.TokenBatch(ids=ids, lengths=lens), n)

        cand, refs = mk(), [mk() for _ in range(int(rng.integers(1, 3)))]
        d = tb.build_dictionary(cand, refs)
        parts = [flatten_valid(cand)] + [flatten_valid(r) for r in refs]
        if where == "device":
            originals = torch.cat(parts).cpu().numpy()
            uniq, inv = d.unique_ngrams.cpu().numpy(), d.inverse_indices.cpu().numpy()
        else:
            originals = np.concatenate(parts)
            uniq, inv = d.unique_ngrams, d.inverse_indices
        np.testing.assert_array_equal(uniq[inv], originals)
        assert d.num_unique <= max(len(originals), 1)


def test_batched_bincount_examples_and_errors():
    """pkg/tests/test_ngrams.py:93-121."""
    m = tb.batched_bincount([np.array([0, 0, 2]), np.array([1])], 3, 2)
    np.testing.assert_array_equal(m.counts, [[2, 0, 1], [0, 1, 0]])
    m = tb.batched_bincount([np.array([], dtype=np.int64), np.array([1])], 2, 2)
    np.testing.assert_array_equal(m.counts, [[0, 0], [0, 1]])
    with pytest.raises(ValueError):
        tb.batched_bincount([np.array([0, 3])], 3, 1)
    with pytest.raises(tb.CapacityError):
        tb.batched_bincount([np.array([0])] * 4, 2**62, 4)


def test_batched_bincount_vs_per_sentence_loop_1000():
    """test_acceptance.py:72-83 (bincount half)."""
    rng = np.random.default_rng(7)
    for _ in range(1000):
        b = int(rng.integers(1, 13))
        u = int(rng.integers(1, 50))
        ids = [rng.integers(0, u, size=rng.integers(0, 30)) for _ in range(b)]
        got = tb.batched_bincount(ids, u, b).counts
        np.testing.assert_array_equal(got, np.stack([np.bincount(s, minlength=u) for s in ids]))


def test_segment_ops_large_u_global_path():
    """U beyond shared memory takes the global-atomic variant."""
    rng = np.random.default_rng(8)
    b, u = 6, 80_000
    seg = rng.integers(0, 5000, size=b)
    flat = rng.integers(0, u, size=int(seg.sum()))
    flat[:100] = 7  # a hot ID
    np.testing.assert_array_equal(_backend.segment_bincount(flat, seg, u), oracle.segment_bincount(flat, seg, u))
    rm = rng.integers(0, 3, size=(b, u)).astype(np.int32)
    np.testing.assert_array_equal(_backend.clipped_numerators(flat, seg, rm),
                                  oracle.clipped_numerators(flat, seg, rm))


def test_clipped_numerators_vs_oracle_random():
    rng = np.random.default_rng(9)
    for _ in range(200):
        b = int(rng.integers(1, 10))
        u = int(rng.integers(1, 60))
        seg = rng.integers(0, 40, size=b)
        flat = rng.integers(0, u, size=int(seg.sum()))
        rm = rng.integers(0, 4, size=(b, u)).astype(np.int32)
        np.testing.assert_array_equal(_backend.clipped_numerators(flat, seg, rm),
                                      oracle.clipped_numerators(flat, seg, rm))
    with pytest.raises(ValueError):
        _backend.segment_bincount(np.array([0, 1, 2]), np.array([2]), 3)  # lengths do not sum


def test_max_and_clip_counts():
    """pkg/tests/test_ngrams.py:124-147."""
    a = tb.CountMatrix(counts=np.array([[1, 0]]))
    b = tb.CountMatrix(counts=np.array([[0, 2]]))
    np.testing.assert_array_equal(tb.max_reference_counts([a, b]).counts, [[1, 2]])
    np.testing.assert_array_equal(tb.max_reference_counts([a]).counts, a.counts)
    with pytest.raises(ValueError):
        tb.max_reference_counts([a, tb.CountMatrix(counts=np.zeros((2, 2)))])
    cand = tb.CountMatrix(counts=np.array([[7, 2]]))
    refs = tb.CountMatrix(counts=np.array([[2, 5]]))
    np.testing.assert_array_equal(tb.clip_counts(cand, refs).counts, [[2, 2]])
    with pytest.raises(ValueError):
        tb.clip_counts(cand, tb.CountMatrix(counts=np.zeros((2, 2))))
    rng = np.random.default_rng(3)
    mats = [tb.CountMatrix(counts=rng.integers(0, 5, size=(4, 7))) for _ in range(3)]
    np.testing.assert_array_equal(tb.max_reference_counts(mats).counts,
                                  np.maximum(np.maximum(mats[0].counts, mats[1].counts), mats[2].counts))


def test_row_sum_invariant(rng):
    """pkg/tests/test_ngrams.py:150-161."""
    b, l, n = 5, 15, 2
    batch = tb.TokenBatch(ids=rng.integers(0, 6, size=(b, l)), lengths=rng.integers(0, l + 1, size=b))
    cand = tb.extract_ngrams(batch, n)
    d = tb.build_dictionary(cand, [tb.extract_ngrams(batch, n)])
    per = np.split(d.inverse_indices[: cand.total_valid], np.cumsum(cand.valid_counts)[:-1])
    counts = tb.batched_bincount(per, d.num_unique, b).counts
    np.testing.assert_array_equal(counts.sum(axis=1), cand.valid_counts)


def test_oracle_ngram_counts_compat():
    assert tb.oracle_ngram_counts([1, 2, 1, 2], 2) == {(1, 2): 2, (2, 1): 1}
    assert tb.oracle_ngram_counts([5], 2) == {}
    assert tb.oracle_sentence_bleu([1, 2, 3, 4, 5], [[1, 2, 3, 4, 5]]) == 1.0
    assert tb.oracle_sentence_bleu([0] * 7, [[0, 1, 2, 3, 0, 4], [5, 2, 6, 1, 3, 0, 4]],
                                   tb.BleuConfig(max_order=1)) == pytest.approx(2 / 7)


@st.composite
def bincount_case(draw):
    b = draw(st.integers(1, 16))
    u = draw(st.integers(1, 64))
    ids = [draw(st.lists(st.integers(0, u - 1), max_size=30)) for _ in range(b)]
    return [np.array(s, dtype=np.int64) for s in ids], u, b


@given(bincount_case())
@settings(max_examples=100, deadline=None)
def test_offset_bincount_property(case):
    """pkg/tests/test_properties.py:15-32."""
    ids, u, b = case
    got = tb.batched_bincount(ids, u, b).counts
    np.testing.assert_array_equal(got, np.stack([np.bincount(s, minlength=u) for s in ids]))


@st.composite
def batch_case(draw):
    b = draw(st.integers(1, 6))
    l = draw(st.integers(1, 16))
    v = draw(st.integers(1, 10))
    r = draw(st.integers(1, 2))
    seed = draw(st.integers(0, 2**31))
    smoothing = draw(st.sampled_from(["none", "floor", "add-k", "exp"]))
    rng = np.random.default_rng(seed)

    def mk():
        return rng.integers(0, v, size=(b, l)), rng.integers(0, l + 1, size=b)

    return mk(), [mk() for _ in range(r)], smoothing


@given(batch_case())
@settings(max_examples=60, deadline=None)
def test_batched_matches_oracle_property(case):
    """pkg/tests/test_properties.py:35-60 (1e-6 there; 1e-12 here)."""
    (cid, clen), refs, sm = case
    cfg = tb.BleuConfig(smoothing=sm)
    got = tb.sentence_bleu(tb.TokenBatch(ids=cid, lengths=clen),
                           [tb.TokenBatch(ids=i, lengths=l) for i, l in refs], cfg).scores
    serial = [oracle.py_sentence_bleu(cid[i, :clen[i]].tolist(), [r[0][i, :r[1][i]].tolist() for r in refs],
                                      smoothing=sm) for i in range(len(clen))]
    np.testing.assert_allclose(got, serial, atol=1e-12)
    assert np.all(got >= 0.0) and np.all(got <= 1.0)


@pytest.mark.parametrize("dtype", [torch.int32, torch.int64])
def test_flatten_windows_kernel_matches_reference_layout(dtype):
    """tb_flatten_windows (flatten_valid on CUDA slices) == the reference's
    numpy flatten_valid (ngrams.py:79-83): same rows, same row-major order,
    ragged lengths, rows shorter than n, empty rows, strided row views."""
    rng = np.random.default_rng(11)
    for b, l, n in [(1, 1, 1), (7, 5, 3), (64, 40, 4), (300, 129, 2), (5, 3, 4)]:
        ids = rng.integers(0, 1 << 30, size=(b, l))
        lens = rng.integers(0, l + 1, size=b)
        want = flatten_valid(tb.extract_ngrams(tb.TokenBatch(ids=ids, lengths=lens), n))
        dev = tb.TokenBatch(ids=torch.as_tensor(ids, device="cuda", dtype=dtype),
                            lengths=torch.as_tensor(lens, device="cuda"))
        got = flatten_valid(tb.extract_ngrams(dev, n))
        assert got.is_cuda and got.dtype == torch.int64
        np.testing.assert_array_equal(got.cpu().numpy(), want)
    wide = torch.as_tensor(rng.integers(0, 99, size=(6, 50)), device="cuda", dtype=dtype)
    view = tb.TokenBatch.trusted(wide[:, :20], torch.full((6,), 17, device="cuda"))
    got = flatten_valid(tb.extract_ngrams(view, 3)).cpu().numpy()
    host = wide[:, :20].cpu().numpy()
    np.testing.assert_array_equal(got, np.concatenate([np.lib.stride_tricks.sliding_window_view(r[:17], 3)
                                                       for r in host]))
