"""Buffer-level entry points (mirror of ``batchbleu_ext``,
pkg/bindings/src/batchbleu_ext/_ext.pyx:1-110).

``score_sentences`` / ``score_corpus`` take contiguous int32/int64 buffers:
``candidates`` (B, L), ``cand_lengths`` (B,), ``references`` (R, B, L) or
(B, L) for a single reference set, ``ref_lengths`` (R, B) or (B,).  Same
dimension-naming errors as the reference.

Host arrays follow the reference exactly: every buffer becomes C-contiguous
int64 and each conversion counts as one copy (``copy_count``, _ext.pyx:31-46;
int32 inputs cost four).  In addition, torch tensors (host or CUDA) are used
as they are — int32 token tensors are read natively by the kernels, CUDA
tensors zero-copy — and only a non-contiguous tensor or non-int64 lengths
count as copies.
"""

from __future__ import annotations

import numpy as np
import torch

from .batch import TokenBatch
from .bleu import BleuConfig, corpus_bleu, sentence_bleu

__version__ = "0.1.0"

_copy_count = 0


def copy_count() -> int:
    """Number of buffer copies made since import (or the last reset)."""
    return _copy_count


def reset_copy_count() -> None:
    global _copy_count
    _copy_count = 0


def _dtype_ok(arr) -> bool:
    if isinstance(arr, torch.Tensor):
        return arr.dtype in (torch.int32, torch.int64)
    return arr.dtype in (np.dtype(np.int32), np.dtype(np.int64))


def _as_tokens(name, buf, expected_ndim):
    """_ext.pyx:31-46 for token buffers: int32/int64 kept as-is when contiguous."""
    global _copy_count
    arr = buf if isinstance(buf, torch.Tensor) else np.asarray(buf)
    if not _dtype_ok(arr):
        raise TypeError(f"{name} must be int32 or int64, got {arr.dtype}")
    if arr.ndim != expected_ndim:
        raise ValueError(f"{name} must have {expected_ndim} dimensions, got {arr.ndim}")
    if isinstance(arr, torch.Tensor):  # int32 / int64 tensors are used as they are
        if not arr.is_contiguous():
            _copy_count += 1
            arr = arr.contiguous()
        return arr
    # host arrays: C-contiguous int64, as TokenBatch holds them (batch.py:23) —
    # int32 arrays are widened here, with the copy counted (_ext.pyx:31-46)
    out = np.ascontiguousarray(arr, dtype=np.int64)
    if out is not arr:
        _copy_count += 1
    return out


def _as_lengths(name, buf, expected_ndim):
    """_ext.pyx:31-46 for length buffers: widened to int64 (counted)."""
    global _copy_count
    arr = buf if isinstance(buf, torch.Tensor) else np.asarray(buf)
    if not _dtype_ok(arr):
        raise TypeError(f"{name} must be int32 or int64, got {arr.dtype}")
    if arr.ndim != expected_ndim:
        raise ValueError(f"{name} must have {expected_ndim} dimensions, got {arr.ndim}")
    if isinstance(arr, torch.Tensor):
        if arr.dtype != torch.int64 or not arr.is_contiguous():
            _copy_count += 1
            arr = arr.to(torch.int64).contiguous()
        return arr
    out = np.ascontiguousarray(arr, dtype=np.int64)
    if out is not arr:
        _copy_count += 1
    return out


def _check_dim(name, axis, actual, expected):
    """_ext.pyx:49-53."""
    if actual != expected:
        raise ValueError(f"{name} dimension {axis} is {actual}, expected {expected}")


def _build_batches(candidates, cand_lengths, references, ref_lengths):
    """_ext.pyx:56-79."""
    cand = _as_tokens("candidates", candidates, 2)
    b, l = cand.shape
    clens = _as_lengths("cand_lengths", cand_lengths, 1)
    _check_dim("cand_lengths", 0, clens.shape[0], b)
    refs_nd = references.ndim if isinstance(references, torch.Tensor) else np.asarray(references).ndim
    if refs_nd == 2:
        refs = _as_tokens("references", references, 2)[None]
        rlens = _as_lengths("ref_lengths", ref_lengths, 1)[None]
    else:
        refs = _as_tokens("references", references, 3)
        rlens = _as_lengths("ref_lengths", ref_lengths, 2)
    _check_dim("references", 1, refs.shape[1], b)
    _check_dim("references", 2, refs.shape[2], l)
    _check_dim("ref_lengths", 0, rlens.shape[0], refs.shape[0])
    _check_dim("ref_lengths", 1, rlens.shape[1], b)
    cand_batch = TokenBatch(ids=cand, lengths=clens)
    ref_batches = [TokenBatch(ids=refs[r], lengths=rlens[r]) for r in range(refs.shape[0])]
    return cand_batch, ref_batches


def _make_config(max_order, weights, smoothing, eps, k):
    return BleuConfig(max_order=max_order, weights=weights, smoothing=smoothing, eps=eps, k=k)


def score_sentences(candidates, cand_lengths, references, ref_lengths, *,
                    max_order=4, weights=None, smoothing="none", eps=0.1, k=1.0):
    """Per-sentence BLEU over token-ID buffers; float64 (B,) (_ext.pyx:87-100)."""
    cand, refs = _build_batches(candidates, cand_lengths, references, ref_lengths)
    if cand.batch_size == 0:
        if cand.is_device:
            return torch.empty(0, dtype=torch.float64, device=cand.ids.device)
        return np.empty(0, dtype=np.float64)
    config = _make_config(max_order, weights, smoothing, eps, k)
    return sentence_bleu(cand, refs, config).scores


def score_corpus(candidates, cand_lengths, references, ref_lengths, *,
                 max_order=4, weights=None, smoothing="none", eps=0.1, k=1.0):
    """Corpus BLEU over the same buffer layout; a float (_ext.pyx:103-110)."""
    cand, refs = _build_batches(candidates, cand_lengths, references, ref_lengths)
    config = _make_config(max_order, weights, smoothing, eps, k)
    return float(corpus_bleu(cand, refs, config).scores)
