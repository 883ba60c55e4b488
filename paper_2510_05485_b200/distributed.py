"""Multi-GPU data parallelism over sentence groups.

A sentence's statistics depend only on its own candidate and references, so
the batch shards by rows with no data-path collective (reference property:
batch-composition independence, test_acceptance.py:190-209).  One process per
GPU (torchrun); `torch.distributed` (NCCL over NVLink/NVSwitch) is used only
where the path has a real exchange:

* per-sentence mode: nothing (each rank keeps its rows' rewards); an optional
  ``all_gather`` of fp64 scores when every rank needs the whole vector;
* corpus mode: one ``all_reduce(SUM)`` of the int64 vector
  [Σnum_1..N | Σden_1..N | Σc | Σr] (2N+2 values), then the corpus epilogue
  redundantly on every rank.  Integer sums make the result bit-identical to
  one GPU (score_corpus_from_stats, bleu.py:293-305).
"""

from __future__ import annotations

from typing import Optional, Sequence

import numpy as np
import torch
import torch.distributed as dist

from .batch import TokenBatch
from .bleu import (BleuConfig, BleuResult, corpus_totals, score_corpus_from_totals,
                   sentence_bleu)


def shard_bounds(batch_size: int, rank: int, world_size: int) -> tuple[int, int]:
    """Contiguous row range [lo, hi) of `rank`: ⌈B/g⌉ rows per rank."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ValueError(f"bad rank {rank} for world size {world_size}")
    per = -(-batch_size // world_size) if batch_size else 0
    lo = min(rank * per, batch_size)
    hi = min(lo + per, batch_size)
    return lo, hi


def shard_batch(batch: TokenBatch, lo: int, hi: int, device: Optional[torch.device] = None) -> TokenBatch:
    """Rows [lo, hi) of a batch; host rows are moved to `device` when given."""
    ids, lengths = batch.ids[lo:hi], batch.lengths[lo:hi]
    if device is not None and not (isinstance(ids, torch.Tensor) and ids.is_cuda):
        ids = torch.as_tensor(np.ascontiguousarray(ids)).to(device)
        lengths = torch.as_tensor(np.ascontiguousarray(lengths)).to(device)
        return TokenBatch.trusted(ids, lengths)  # validated as a whole on the host
    if isinstance(ids, torch.Tensor) and ids.is_cuda:
        return TokenBatch.trusted(ids, lengths)
    return TokenBatch(ids=ids, lengths=lengths)


def _world(group) -> tuple[int, int]:
    if not dist.is_available() or not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def _host_staged(group) -> bool:
    """Backends without CUDA-tensor collectives (gloo: CPU tensors only for
    some ops) get host-staged copies; NCCL works on device memory directly."""
    return dist.get_backend(group) != "nccl"


def allreduce_totals(totals: torch.Tensor, group=None) -> torch.Tensor:
    """SUM-all-reduce of the int64 corpus totals (in place, returned)."""
    rank, world = _world(group)
    if world > 1:
        if totals.is_cuda and _host_staged(group):
            host = totals.cpu()
            dist.all_reduce(host, op=dist.ReduceOp.SUM, group=group)
            totals.copy_(host)
        else:
            dist.all_reduce(totals, op=dist.ReduceOp.SUM, group=group)
    return totals


def _all_gather(out: torch.Tensor, buf: torch.Tensor, group) -> None:
    if buf.is_cuda and _host_staged(group):
        host = torch.empty(out.shape, dtype=out.dtype)
        dist.all_gather_into_tensor(host, buf.cpu(), group=group)
        out.copy_(host)
    else:
        dist.all_gather_into_tensor(out, buf, group=group)


def sharded_sentence_bleu(candidates: TokenBatch, references: Sequence[TokenBatch],
                          config: Optional[BleuConfig] = None, *, group=None,
                          gather: bool = False, device: Optional[torch.device] = None) -> BleuResult:
    """Per-sentence BLEU of this rank's rows (or of the whole batch when
    `gather`).  `candidates`/`references` are the FULL batch on every rank."""
    config = config or BleuConfig()
    rank, world = _world(group)
    lo, hi = shard_bounds(candidates.batch_size, rank, world)
    dev = device or torch.device("cuda", torch.cuda.current_device())
    cand = shard_batch(candidates, lo, hi, dev)
    refs = [shard_batch(r, lo, hi, dev) for r in references]
    res = sentence_bleu(cand, refs, config)
    if not gather or world == 1:
        return res
    per = -(-candidates.batch_size // world)
    buf = torch.zeros(per, dtype=torch.float64, device=dev)
    buf[: hi - lo] = res.scores
    out = torch.empty(per * world, dtype=torch.float64, device=dev)
    _all_gather(out, buf, group)
    return BleuResult(scores=out[: candidates.batch_size], precisions=res.precisions,
                      brevity_penalty=res.brevity_penalty)


def sharded_corpus_bleu(candidates: TokenBatch, references: Sequence[TokenBatch],
                        config: Optional[BleuConfig] = None, *, group=None,
                        device: Optional[torch.device] = None) -> BleuResult:
    """Corpus BLEU of the whole batch: local totals -> all_reduce -> epilogue."""
    config = config or BleuConfig()
    rank, world = _world(group)
    lo, hi = shard_bounds(candidates.batch_size, rank, world)
    dev = device or torch.device("cuda", torch.cuda.current_device())
    cand = shard_batch(candidates, lo, hi, dev)
    refs = [shard_batch(r, lo, hi, dev) for r in references]
    tot = corpus_totals(cand, refs, config)
    allreduce_totals(tot, group)
    return score_corpus_from_totals(tot, config, host=False)
