"""Per-sentence list-based entry points of the reference
(``batchbleu.oracle``, pkg/src/batchbleu/oracle.py:18-118), served by the
device path.

The reference's serial ``Counter`` oracle is exported from its package
namespace, so a drop-in keeps the names.  Here they are thin adapters that
pack the Python lists into a batch and call the same CUDA kernels as
``sentence_bleu`` / ``corpus_bleu`` — there is no second (CPU) implementation
in this package.  The independent CPU checker lives in ``oracle/`` at the
repository root and is used only by the tests.
"""

from __future__ import annotations

from collections import Counter
from typing import Sequence

import numpy as np

from . import _backend
from .batch import TokenBatch
from .bleu import BleuConfig, corpus_bleu, sentence_bleu


def oracle_ngram_counts(sentence: Sequence[int], n: int) -> Counter:
    """Multiset of the contiguous order-n n-grams of one sentence
    (oracle.py:18-22), via the device dictionary + offset bincount."""
    if n < 1:
        raise ValueError(f"n-gram order must be >= 1, got {n}")
    t = len(sentence) - n + 1
    if t <= 0:
        return Counter()
    arr = np.asarray(sentence, dtype=np.int64)
    rows = np.lib.stride_tricks.sliding_window_view(arr, n)
    uniq, inv = _backend.unique_rows(np.ascontiguousarray(rows))
    counts = _backend.segment_bincount(inv, np.array([t], dtype=np.int64), uniq.shape[0])[0]
    return Counter({tuple(int(x) for x in uniq[i]): int(counts[i]) for i in range(uniq.shape[0])})


def oracle_sentence_bleu(candidate: Sequence[int], references: Sequence[Sequence[int]],
                         config: BleuConfig | None = None) -> float:
    """BLEU for one sentence of token IDs (oracle.py:78-92)."""
    config = config or BleuConfig()
    if not references:
        raise ValueError("at least one reference is required")
    cand = TokenBatch.from_lists([candidate])
    refs = [TokenBatch.from_lists([r]) for r in references]
    return float(sentence_bleu(cand, refs, config).scores[0])


def oracle_corpus_bleu(candidates: Sequence[Sequence[int]],
                       references: Sequence[Sequence[Sequence[int]]],
                       config: BleuConfig | None = None) -> float:
    """Corpus BLEU; ``references[r][i]`` is reference r of sentence i (oracle.py:95-118)."""
    config = config or BleuConfig()
    if not references:
        raise ValueError("at least one reference set is required")
    cand = TokenBatch.from_lists(list(candidates))
    refs = [TokenBatch.from_lists(list(rs)) for rs in references]
    return float(corpus_bleu(cand, refs, config).scores)
