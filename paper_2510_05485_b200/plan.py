"""Pre-planned, CUDA-graph-capturable scoring for fixed shapes.

The RL-reward use of BLEU scores a batch of the same shape every training
step.  ``SentenceBleuPlan`` binds the device buffers once, pre-builds the C
ABI argument list, owns its workspace and outputs, and can capture the single
``tb_bleu_stats`` launch into a CUDA graph so a step costs one graph launch
with no allocation, no host synchronisation and no Python-side argument
marshalling.

    plan = SentenceBleuPlan(cand, refs, config)   # TokenBatch of CUDA tensors
    plan.capture()
    ...                                           # write new tokens into plan.cand.ids etc.
    plan.replay()                                 # scores in plan.scores (device)
"""

from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import numpy as np
import torch

from . import _native
from .batch import TokenBatch
from .bleu import BleuConfig, _check_batches, _weights_arg


class SentenceBleuPlan:
    """Per-sentence (and optionally corpus) BLEU of a fixed-shape device batch."""

    kernels_per_run = 1

    def __init__(self, candidates: TokenBatch, references: Sequence[TokenBatch],
                 config: Optional[BleuConfig] = None, *, stats: bool = True, corpus: bool = False,
                 sentence: bool = True):
        config = config or BleuConfig()
        _check_batches(candidates, references)
        if len(references) > _native.TB_MAX_REFS or config.max_order > _native.TB_MAX_ORDER:
            raise ValueError(f"SentenceBleuPlan binds the fused kernel: at most {_native.TB_MAX_REFS} reference "
                             f"sets and max_order {_native.TB_MAX_ORDER} (sentence_bleu takes any)")
        if not candidates.is_device or not all(r.is_device for r in references):
            raise ValueError("SentenceBleuPlan needs TokenBatch objects holding CUDA tensors")
        lib = _native.load()
        dev = candidates.ids.device
        dts = {candidates.ids.dtype, *(r.ids.dtype for r in references)}
        if len(dts) != 1:
            raise ValueError("all batches of a plan must share one token dtype")
        self.device = dev
        self.config = config
        self.cand = candidates
        self.refs = list(references)
        B, N, R = candidates.batch_size, config.max_order, len(references)
        self.batch_size, self.max_order = B, N
        tb = candidates.ids.element_size()
        with torch.cuda.device(dev):
            self.scores = torch.empty(B, dtype=torch.float64, device=dev) if sentence else None
            self.precisions = torch.empty((B, N), dtype=torch.float64, device=dev) if sentence else None
            self.brevity_penalty = torch.empty(B, dtype=torch.float64, device=dev) if sentence else None
            self.numerators = torch.empty((B, N), dtype=torch.int64, device=dev) if stats else None
            self.denominators = torch.empty((B, N), dtype=torch.int64, device=dev) if stats else None
            self.cand_lens = torch.empty(B, dtype=torch.int64, device=dev) if stats else None
            self.eff_ref_lens = torch.empty(B, dtype=torch.int64, device=dev) if stats else None
            self.totals = torch.empty(2 * N + 2, dtype=torch.int64, device=dev) if corpus else None
            self.corpus = torch.empty(N + 2, dtype=torch.float64, device=dev) if corpus else None
            self.err = torch.zeros(1, dtype=torch.int32, device=dev)
            widths = np.array([r.max_len for r in references], dtype=np.int64)
            wsb = lib.tb_bleu_workspace_bytes(B, R, candidates.max_len, widths.ctypes.data, tb, N)
            if wsb == 0:
                raise ValueError("unsupported shape for the device path")
            self.workspace = torch.zeros(wsb, dtype=torch.uint8, device=dev)

        p = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
        # prebuilt arguments of the native launch (tb_bleu_stats through _hostpath)
        want64 = tb == 8
        views = tuple(b_._row_view(want64)[0] for b_ in (candidates, *references))
        outs = (p(self.numerators), p(self.denominators), p(self.cand_lens), p(self.eff_ref_lens),
                p(self.scores), p(self.precisions), p(self.brevity_penalty), p(self.totals), p(self.corpus))
        self._launch_args = (views, B, N, _native.SMOOTHING_CODES[config.smoothing], config.eps, config.k,
                             ctypes.addressof(_weights_arg(config)), outs, p(self.err), p(self.workspace),
                             self.workspace.numel())
        self._hp = _native.hostpath()
        self.graph: Optional[torch.cuda.CUDAGraph] = None

    def corpus_from_totals(self) -> None:
        """Corpus epilogue (score, BP, precisions -> self.corpus) of the int64
        totals in self.totals — after they were all-reduced across ranks
        (score_corpus_from_stats, bleu.py:301-305).  One tiny launch."""
        if self.totals is None:
            raise ValueError("plan was built without corpus=True")
        lib = _native.load()
        N = self.max_order
        t0, c0 = self.totals.data_ptr(), self.corpus.data_ptr()
        rc = lib.tb_bleu_scores(t0, t0 + 8 * N, t0 + 16 * N, t0 + 16 * N + 8, 1, N,
                                _native.SMOOTHING_CODES[self.config.smoothing], self.config.eps,
                                self.config.k, _weights_arg(self.config), c0, c0 + 16, c0 + 8,
                                _native.stream_handle(self.device))
        if rc:
            _native.check(rc, "tb_bleu_scores")

    def run(self) -> None:
        """Launch on the current stream (asynchronous)."""
        rc = self._hp.launch(*self._launch_args, _native.stream_handle(self.device))
        if rc:
            _native.check(rc, "tb_bleu_stats")

    def capture(self) -> torch.cuda.CUDAGraph:
        """Capture one run() into a CUDA graph (call run() once before)."""
        self.run()
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.device(self.device), torch.cuda.graph(g):
            self.run()
        self.graph = g
        return g

    def replay(self) -> None:
        if self.graph is None:
            self.capture()
        self.graph.replay()

    def check(self) -> None:
        """Synchronise and raise if any run since the last check flagged bad
        input data (the flag word is sticky: launches OR into it)."""
        flags = int(self.err.item())
        self.err.zero_()
        _native.raise_flags(flags)
