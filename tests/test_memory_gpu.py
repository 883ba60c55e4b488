"""Device analogue of the reference's memory-proportionality acceptance test
(pkg/tests/test_acceptance.py:104-128): at a fixed batch
shape the device memory a call needs does not depend on the vocabulary —
nothing of size B x U or V is ever allocated (the dictionaries live in each
CTA's shared memory)."""

import numpy as np
import pytest
import torch

import paper_2510_05485_b200 as tb

pytestmark = pytest.mark.gpu


def _peak(vocab):
    rng = np.random.default_rng(5)
    B, L = 64, 512
    dev = torch.device("cuda", 0)
    cand = tb.TokenBatch(ids=torch.as_tensor(rng.integers(0, vocab, (B, L)), device=dev),
                         lengths=torch.as_tensor(rng.integers(L // 2, L + 1, B), device=dev))
    ref = tb.TokenBatch(ids=torch.as_tensor(rng.integers(0, vocab, (B, L)), device=dev),
                        lengths=torch.as_tensor(rng.integers(L // 2, L + 1, B), device=dev))
    tb.sentence_bleu(cand, [ref])  # workspace warm
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    base = torch.cuda.memory_allocated()
    for _ in range(3):
        tb.sentence_bleu(cand, [ref])
        tb.corpus_bleu(cand, [ref])
    torch.cuda.synchronize()
    return torch.cuda.max_memory_allocated() - base


def test_peak_memory_independent_of_vocabulary():
    small, large = _peak(1_000), _peak(1_000_000)
    assert large <= small * 1.05 + 4096, (small, large)
    # and it is only the outputs: (B) scores + (B) bp + (B, N) precisions per call, a few KiB
    assert large < 64 * 1024
