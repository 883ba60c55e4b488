"""Sharded (multi-process) scoring on the GPU: each rank scores its contiguous
rows with the CUDA kernels; corpus mode all-reduces the int64 totals, and the
per-sentence scores can be gathered.  Results must be bit-identical to the
single-process call (integer sums; batch-composition independence).

The GPU box has one GPU, so world size 2 runs two processes on cuda:0 over
gloo (NCCL refuses two ranks on one device); world size 1 runs over NCCL.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _inputs():
    rng = np.random.default_rng(31)
    B, L, V, R = 45, 96, 40, 2
    cid = rng.integers(0, V, (B, L))
    clen = rng.integers(0, L + 1, B)
    refs = []
    for _ in range(R):
        ids = cid.copy()
        m = rng.random(ids.shape) < 0.4
        ids[m] = rng.integers(0, V, int(m.sum()))
        refs.append((ids, rng.integers(0, L + 1, B)))
    return (cid, clen), refs


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, backend, q):
    import sys
    sys.path.insert(0, ROOT)
    import paper_2510_05485_b200 as tb
    from paper_2510_05485_b200.distributed import sharded_corpus_bleu, sharded_sentence_bleu
    torch.cuda.set_device(0)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    kw = {"device_id": torch.device("cuda", 0)} if backend == "nccl" else {}
    dist.init_process_group(backend, rank=rank, world_size=world, **kw)
    try:
        (cid, clen), refs = _inputs()
        cand = tb.TokenBatch(ids=cid, lengths=clen)
        rb = [tb.TokenBatch(ids=i, lengths=l) for i, l in refs]
        out = {}
        for sm in ("none", "exp"):
            cfg = tb.BleuConfig(smoothing=sm)
            co = sharded_corpus_bleu(cand, rb, cfg)
            sc = sharded_sentence_bleu(cand, rb, cfg, gather=True)
            out[sm] = (float(co.scores), co.precisions.cpu().numpy(), sc.scores.cpu().numpy())
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _run(world, backend):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, backend, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    return res


@pytest.mark.parametrize("world,backend", [(1, "nccl"), (2, "gloo")])
def test_sharded_matches_single_process(world, backend):
    import paper_2510_05485_b200 as tb
    (cid, clen), refs = _inputs()
    cand = tb.TokenBatch(ids=cid, lengths=clen)
    rb = [tb.TokenBatch(ids=i, lengths=l) for i, l in refs]
    res = _run(world, backend)
    for sm in ("none", "exp"):
        cfg = tb.BleuConfig(smoothing=sm)
        full = tb.corpus_bleu(cand, rb, cfg)
        sent = tb.sentence_bleu(cand, rb, cfg).scores
        for rank in range(world):
            co, prec, sc = res[rank][sm]
            assert co == full.scores                       # integer totals: bit-identical
            np.testing.assert_array_equal(prec, full.precisions)
            np.testing.assert_array_equal(sc, sent)
