"""Statistics for any number of reference sets and any n-gram order.

The fused kernels (``tb_bleu_stats``) take at most TB_MAX_REFS reference sets
and TB_MAX_ORDER orders (kernel-parameter arrays).  The reference caps
neither (bleu.py:24-56, 97-105, 117-159), so larger requests are served here
by the reference's own per-order algorithm composed from the device n-gram
operator kernels — no CPU path:

    for each chunk of rows, for each order n (bleu.py:117-159):
        windows of every row set          tb_flatten_windows       (ngrams.py:63-83)
        one dictionary of the chunk       tb_unique_rows           (ngrams.py:86-106)
        per reference set, per sentence   tb_segment_bincount      (ngrams.py:116-141)
        max over reference sets           tb_count_binary(max)     (bleu.py:148-157)
        candidate clipped numerators      tb_clipped_numerators    (ngrams.py:201-205)

Rows are processed in chunks so the (rows, U) count matrices stay bounded
(the reference chunks for the same reason, bleu.py:162-170).  Results are
bit-identical to the fused path (tests/test_unbounded_gpu.py).
"""

from __future__ import annotations

import math
from typing import Sequence

import numpy as np
import torch

from . import _backend, _native
from .batch import TokenBatch
from .ngrams import build_dictionary, extract_ngrams

_COUNT_BUDGET = 1 << 26  # int32 entries of one chunk's (rows, U) count matrix


def _device_batch(batch: TokenBatch, dev: torch.device, dtype: torch.dtype) -> TokenBatch:
    ids, lengths = batch.ids, batch.lengths
    ids = torch.as_tensor(np.asarray(ids) if isinstance(ids, np.ndarray) else ids).to(dev, dtype=dtype)
    lengths = torch.as_tensor(np.asarray(lengths) if isinstance(lengths, np.ndarray) else lengths).to(
        dev, dtype=torch.int64)
    return TokenBatch.trusted(ids.contiguous(), lengths.contiguous())


def effective_ref_lens(cand_len: torch.Tensor, ref_lens: Sequence[torch.Tensor]) -> torch.Tensor:
    """_effective_ref_lens (bleu.py:108-114): the reference length closest to
    the candidate's, ties to the shorter — on the device."""
    r = torch.stack(list(ref_lens))          # (R, B)
    d = (r - cand_len[None, :]).abs()
    # lexicographic (distance, length): argmin over distance * 2^32 + length
    key = d * (1 << 32) + r
    return torch.gather(r, 0, key.argmin(dim=0, keepdim=True))[0]


def stats(candidates: TokenBatch, references: Sequence[TokenBatch], max_order: int, dev: torch.device):
    """(numerators (B, N), denominators (B, N), cand_lens (B,), eff_ref_lens (B,))
    int64 CUDA tensors for any R and N."""
    R = len(references)
    want64 = not all(getattr(b, "_tok32", False) for b in (candidates, *references))
    dtype = torch.int64 if want64 else torch.int32
    cand = _device_batch(candidates, dev, dtype)
    refs = [_device_batch(r, dev, dtype) for r in references]
    B = cand.batch_size
    N = int(max_order)
    clen = cand.lengths.clamp(0, cand.max_len)
    rlens = [r.lengths.clamp(0, r.max_len) for r in refs]
    num = torch.zeros((B, N), dtype=torch.int64, device=dev)
    orders = torch.arange(N, device=dev, dtype=torch.int64)
    den = (clen[:, None] - orders[None, :]).clamp(min=0)
    eff = effective_ref_lens(clen, rlens) if B else torch.zeros(0, dtype=torch.int64, device=dev)
    if B == 0:
        return num, den, clen, eff
    width = max([cand.max_len, *[r.max_len for r in refs]] + [1])
    rows = max(1, int(math.sqrt(_COUNT_BUDGET / (width * (R + 1)))))
    for r0 in range(0, B, rows):
        r1 = min(B, r0 + rows)
        sc = TokenBatch.trusted(cand.ids[r0:r1], clen[r0:r1])
        srs = [TokenBatch.trusted(r.ids[r0:r1], rl[r0:r1]) for r, rl in zip(refs, rlens)]
        for n in range(1, N + 1):
            cs = extract_ngrams(sc, n)
            rs = [extract_ngrams(s, n) for s in srs]
            parts_t = [int(cs.valid_counts.sum())] + [int(x.valid_counts.sum()) for x in rs]
            if parts_t[0] == 0:
                break  # no candidate n-gram of this order or above in the chunk
            d = build_dictionary(cs, rs)
            u = d.num_unique
            inv = d.inverse_indices
            offs = np.concatenate([[0], np.cumsum(parts_t)])
            ref_max = None
            for j, x in enumerate(rs):
                ids = inv[offs[j + 1]:offs[j + 2]]
                cnt = _backend.segment_bincount(ids, x.valid_counts, u)
                ref_max = cnt if ref_max is None else _backend.count_binary(ref_max, cnt, "max")
            num[r0:r1, n - 1] = _backend.clipped_numerators(inv[:offs[1]], cs.valid_counts, ref_max)
    return num, den, clen, eff


_wdev: dict = {}


def device_weights(weights, dev: torch.device) -> torch.Tensor:
    key = (tuple(weights), dev.index)
    w = _wdev.get(key)
    if w is None:
        w = _wdev[key] = torch.tensor(list(weights), dtype=torch.float64, device=dev)
    return w


def scores(num, den, cand_len, eff_ref, config, dev: torch.device, fp32: bool = False):
    """tb_bleu_scores_any: (scores (B,), precisions (B, N), bp (B,)) for any N;
    fp64 in numpy's operation order, or the fp32 epilogue."""
    lib = _native.load()
    B, N = int(num.shape[0]), int(num.shape[1])
    dt = torch.float32 if fp32 else torch.float64
    sc = torch.empty(B, dtype=dt, device=dev)
    prec = torch.empty((B, N), dtype=dt, device=dev)
    bp = torch.empty(B, dtype=dt, device=dev)
    with torch.cuda.device(dev):
        w = device_weights(config.weights, dev)
        rc = lib.tb_bleu_scores_any(num.data_ptr(), den.data_ptr(), cand_len.data_ptr(), eff_ref.data_ptr(),
                                    B, N, _native.SMOOTHING_CODES[config.smoothing], config.eps, config.k,
                                    w.data_ptr(), 1 if fp32 else 0, sc.data_ptr(), prec.data_ptr(), bp.data_ptr(),
                                    _native.stream_handle(dev))
        _native.check(rc, "tb_bleu_scores_any")
    return sc, prec, bp


def totals(num, den, cand_len, eff_ref, dev: torch.device) -> torch.Tensor:
    lib = _native.load()
    B, N = int(num.shape[0]), int(num.shape[1])
    tot = torch.empty(2 * N + 2, dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        rc = lib.tb_bleu_totals(num.data_ptr(), den.data_ptr(), cand_len.data_ptr(), eff_ref.data_ptr(), B, N,
                                tot.data_ptr(), _native.stream_handle(dev))
        _native.check(rc, "tb_bleu_totals")
    return tot
