"""GPU parity of the host-buffer path (tb_bleu_host): token rows in pinned
host memory are read by the kernel over PCIe (valid prefixes only, the
"prefix mode" of the staging), pageable rows go through device staging.

Bar as everywhere: counts bit-exact, fp64 scores within 1e-12 relative of the
CPU oracle."""

import ctypes

import numpy as np
import pytest
import torch

import oracle
import paper_2510_05485_b200 as tb
from paper_2510_05485_b200 import _native

pytestmark = pytest.mark.gpu

RTOL = 1e-12


def _correlated(rng, b, l, v, r, lo=None):
    lo = l // 2 if lo is None else lo
    cid = rng.integers(0, v, (b, l))
    clen = rng.integers(lo, l + 1, b)
    refs = []
    for _ in range(r):
        ids = cid.copy()
        m = rng.random(ids.shape) < rng.uniform(0, 0.9, (b, 1))
        ids[m] = rng.integers(0, v, int(m.sum()))
        refs.append((ids, np.clip(clen + rng.integers(-20, 21, b), 0, l)))
    return (cid, clen), refs


def _pinned(a, dtype=torch.int64):
    return torch.as_tensor(np.asarray(a)).to(dtype).pin_memory()


def _check(cand, refs, cand_np, refs_np, cfg):
    st = tb.compute_stats(cand, refs, cfg)
    o = oracle.stats(cand_np[0], cand_np[1], refs_np, cfg.max_order)
    for k_ours, k_o in (("numerators", "numerators"), ("denominators", "denominators"),
                        ("cand_lens", "cand_lens"), ("eff_ref_lens", "eff_ref_lens")):
        np.testing.assert_array_equal(getattr(st, k_ours), o[k_o])
    res = tb.sentence_bleu(cand, refs, cfg)
    assert isinstance(res.scores, np.ndarray)
    os_ = oracle.scores(o, cfg.smoothing, cfg.eps, cfg.k, cfg.weights)
    np.testing.assert_array_equal(res.scores == 0, os_["scores"] == 0)
    np.testing.assert_allclose(res.scores, os_["scores"], rtol=RTOL, atol=0)
    np.testing.assert_allclose(res.precisions, os_["precisions"], rtol=RTOL, atol=0)
    np.testing.assert_allclose(res.brevity_penalty, os_["brevity_penalty"], rtol=RTOL, atol=0)
    co = tb.corpus_bleu(cand, refs, cfg)
    oc = oracle.corpus(o, cfg.smoothing, cfg.eps, cfg.k, cfg.weights)
    assert isinstance(co.scores, float)
    assert co.scores == pytest.approx(oc["scores"], rel=RTOL, abs=0)
    np.testing.assert_array_equal(tb.corpus_totals(cand, refs, cfg), oc["totals"])


@pytest.mark.parametrize("R,smoothing", [(1, "none"), (1, "floor"), (3, "add-k"), (4, "exp")])
@pytest.mark.parametrize("dtype", [torch.int64, torch.int32])
def test_pinned_rows_zero_copy_vs_oracle(R, smoothing, dtype):
    rng = np.random.default_rng(100 + R)
    (cid, clen), refs = _correlated(rng, 96, 300, 2000, R)
    cand = tb.TokenBatch(ids=_pinned(cid, dtype), lengths=torch.as_tensor(clen))
    rb = [tb.TokenBatch(ids=_pinned(i, dtype), lengths=torch.as_tensor(l)) for i, l in refs]
    _check(cand, rb, (cid, clen), refs, tb.BleuConfig(smoothing=smoothing))


def test_pinned_c2_shape_matches_device_path():
    rng = np.random.default_rng([42, 512, 1024, 128000])
    (cid, clen), refs = _correlated(rng, 512, 1024, 128000, 1)
    cand = tb.TokenBatch(ids=_pinned(cid), lengths=torch.as_tensor(clen))
    rb = [tb.TokenBatch(ids=_pinned(i), lengths=torch.as_tensor(l)) for i, l in refs]
    h = tb.sentence_bleu(cand, rb)
    dc = tb.TokenBatch(ids=torch.as_tensor(cid, device="cuda"), lengths=torch.as_tensor(clen, device="cuda"))
    dr = [tb.TokenBatch(ids=torch.as_tensor(i, device="cuda"), lengths=torch.as_tensor(l, device="cuda"))
          for i, l in refs]
    d = tb.sentence_bleu(dc, dr)
    np.testing.assert_array_equal(h.scores, d.scores.cpu().numpy())
    np.testing.assert_array_equal(h.precisions, d.precisions.cpu().numpy())
    _check(cand, rb, (cid, clen), refs, tb.BleuConfig())


def test_pinned_unaligned_and_strided_rows():
    """Row starts that are not 16-byte aligned and odd widths: the threads copy
    what the bulk engine cannot."""
    rng = np.random.default_rng(7)
    (cid, clen), refs = _correlated(rng, 40, 77, 50, 2)
    big = _pinned(np.pad(cid, ((0, 0), (1, 2))))           # rows start 8 bytes in
    cand = tb.TokenBatch(ids=big[:, 1:78], lengths=torch.as_tensor(clen))
    assert cand.ids.data_ptr() % 16 != 0 and cand.ids.stride(0) == 80
    rb = []
    for i, l in refs:
        b2 = _pinned(np.pad(i, ((0, 0), (3, 0))), torch.int32)  # int32, 12-byte offset
        rb.append(tb.TokenBatch(ids=b2[:, 3:], lengths=torch.as_tensor(l)))
    _check(cand, rb, (cid, clen), refs, tb.BleuConfig(smoothing="exp"))


def test_mixed_pinned_pageable_and_dtypes():
    rng = np.random.default_rng(8)
    (cid, clen), refs = _correlated(rng, 64, 128, 300, 2)
    cand = tb.TokenBatch(ids=_pinned(cid, torch.int32), lengths=torch.as_tensor(clen))
    rb = [tb.TokenBatch(ids=refs[0][0], lengths=refs[0][1]),                       # pageable int64
          tb.TokenBatch(ids=_pinned(refs[1][0]), lengths=torch.as_tensor(refs[1][1]))]
    _check(cand, rb, (cid, clen), refs, tb.BleuConfig(smoothing="floor"))


def test_wide_rows_take_device_staging():
    """Rows too wide for shared memory use the global-memory kernel, which
    reads tokens repeatedly: pinned rows are staged to the device first."""
    rng = np.random.default_rng(9)
    (cid, clen), refs = _correlated(rng, 3, 20000, 40, 1, lo=15000)
    cand = tb.TokenBatch(ids=_pinned(cid), lengths=torch.as_tensor(clen))
    rb = [tb.TokenBatch(ids=_pinned(i), lengths=torch.as_tensor(l)) for i, l in refs]
    _check(cand, rb, (cid, clen), refs, tb.BleuConfig())


def test_shape_changes_regrow_staging():
    rng = np.random.default_rng(10)
    for b, l in ((4, 16), (300, 700), (2, 9), (700, 300), (1, 1)):
        (cid, clen), refs = _correlated(rng, b, l, 30, 1, lo=0)
        cand = tb.TokenBatch(ids=_pinned(cid), lengths=torch.as_tensor(clen))
        rb = [tb.TokenBatch(ids=_pinned(i), lengths=torch.as_tensor(ln)) for i, ln in refs]
        _check(cand, rb, (cid, clen), refs, tb.BleuConfig(smoothing="add-k"))


def test_empty_batch_host():
    e = tb.TokenBatch(ids=_pinned(np.zeros((0, 5), np.int64)), lengths=torch.zeros(0, dtype=torch.int64))
    res = tb.sentence_bleu(e, [e])
    assert res.scores.shape == (0,)
    co = tb.corpus_bleu(e, [e])
    assert co.scores == 0.0


def _raw_host_call(ids, lens, ref_ids, ref_lens, N=4):
    """tb_bleu_host through ctypes, bypassing TokenBatch validation."""
    lib = _native.load()
    B, L = ids.shape
    num = np.empty((B, N), np.int64)
    flags = ctypes.c_int32(-1)
    w = (ctypes.c_double * N)(*([1.0 / N] * N))
    rc = lib.tb_bleu_host(ids.element_size(), ids.data_ptr(), L, L, lens.data_ptr(), 1,
                          (ctypes.c_void_p * 1)(ref_ids.data_ptr()), (ctypes.c_int64 * 1)(L),
                          (ctypes.c_int64 * 1)(L), (ctypes.c_void_p * 1)(ref_lens.data_ptr()),
                          B, N, 0, 0.1, 1.0, w, num.ctypes.data, None, None, None, None, None, None,
                          None, None, ctypes.byref(flags), torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    return flags.value, num


@pytest.mark.parametrize("where", ["pinned", "pageable", "device"])
def test_bad_lengths_are_flagged(where):
    ids = torch.randint(0, 10, (8, 32))
    lens = torch.full((8,), 32, dtype=torch.int64)
    bad = lens.clone()
    bad[3] = 33
    if where == "pinned":
        ids, lens, bad = ids.pin_memory(), lens.pin_memory(), bad.pin_memory()
    elif where == "device":
        ids, lens, bad = ids.cuda(), lens.cuda(), bad.cuda()
    f, num = _raw_host_call(ids, lens, ids, lens)
    assert f == 0
    np.testing.assert_array_equal(num[:, 0], 32)
    f, _ = _raw_host_call(ids, bad, ids, lens)
    assert f & _native.TB_FLAG_BAD_LENGTH
    f, _ = _raw_host_call(ids, lens, ids, lens)  # flags do not stick
    assert f == 0


@pytest.mark.parametrize("R", [1, 3])
def test_pageable_numpy_rows_staged_and_pipelined(R):
    """numpy (pageable) rows — the reference's own TokenBatch usage — are staged
    into pinned memory by host threads, narrowed to int32 when their IDs fit;
    batches of >= 1024 rows run in chunks (copy of chunk i+1 overlapping the
    kernel on chunk i), and a chunk holding an ID >= 2^31 is staged as int64."""
    rng = np.random.default_rng(500 + R)
    (cid, clen), refs = _correlated(rng, 1100, 96, 3000, R)
    cid[700, 5] = 2 ** 40          # only the second chunk needs int64
    refs[0][0][700, 5] = 2 ** 40
    clen[1000] = 0
    cand = tb.TokenBatch(ids=cid, lengths=clen)
    rb = [tb.TokenBatch(ids=i, lengths=l) for i, l in refs]
    st = tb.compute_stats(cand, rb, tb.BleuConfig(smoothing="floor"))
    o = oracle.stats(cid, clen, refs, 4)
    np.testing.assert_array_equal(st.numerators, o["numerators"])
    np.testing.assert_array_equal(st.denominators, o["denominators"])
    np.testing.assert_array_equal(st.eff_ref_lens, o["eff_ref_lens"])
    res = tb.sentence_bleu(cand, rb, tb.BleuConfig(smoothing="floor"))
    os_ = oracle.scores(o, "floor")
    np.testing.assert_allclose(res.scores, os_["scores"], rtol=RTOL, atol=0)
    np.testing.assert_allclose(res.precisions, os_["precisions"], rtol=RTOL, atol=0)
    # the same rows, small batch (one staged launch) and pinned (read in place)
    small = tb.TokenBatch(ids=cid[:200], lengths=clen[:200])
    rs = [tb.TokenBatch(ids=i[:200], lengths=l[:200]) for i, l in refs]
    np.testing.assert_array_equal(tb.compute_stats(small, rs, tb.BleuConfig()).numerators, o["numerators"][:200])


def test_pageable_bad_lengths_flagged_in_pipelined_chunks():
    rng = np.random.default_rng(9)
    ids = rng.integers(0, 50, (1100, 40))
    lens = np.full(1100, 40)
    bad = lens.copy()
    bad[900] = 41  # in the second chunk
    f, num = _raw_host_call(torch.as_tensor(ids), torch.as_tensor(bad), torch.as_tensor(ids), torch.as_tensor(lens))
    assert f & _native.TB_FLAG_BAD_LENGTH
    f, num = _raw_host_call(torch.as_tensor(ids), torch.as_tensor(lens), torch.as_tensor(ids), torch.as_tensor(lens))
    assert f == 0
    np.testing.assert_array_equal(num[:, 0], 40)
