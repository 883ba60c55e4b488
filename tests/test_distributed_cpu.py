"""Multi-process host logic of the sharded path on CPU (gloo, world size 2).

The device kernels are single-GPU; what crosses ranks is (a) a contiguous
row partition and (b) in corpus mode one SUM all-reduce of the int64 totals
[Σnum_1..N | Σden_1..N | Σc | Σr].  Here each rank computes
its shard's totals with the CPU oracle (the checker), all-reduces them with
`allreduce_totals` over gloo, and the result must equal the whole batch's
totals exactly — integer sums make sharding bit-exact.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT

from paper_2510_05485_b200.distributed import allreduce_totals, shard_bounds


def test_shard_bounds_partition():
    for b in (0, 1, 7, 512, 513, 4096):
        for w in (1, 2, 3, 4, 8):
            spans = [shard_bounds(b, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == b
            for (lo, hi), (lo2, _) in zip(spans, spans[1:]):
                assert hi == lo2 and lo <= hi
            assert max(hi - lo for lo, hi in spans) <= -(-b // w)
    with pytest.raises(ValueError):
        shard_bounds(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(77)
        B, L, V, R = 37, 48, 9, 2
        cand = (rng.integers(0, V, size=(B, L)), rng.integers(0, L + 1, size=B))
        refs = [(rng.integers(0, V, size=(B, L)), rng.integers(0, L + 1, size=B)) for _ in range(R)]
        lo, hi = shard_bounds(B, rank, world)
        st = oracle.stats(cand[0][lo:hi], cand[1][lo:hi], [(i[lo:hi], l[lo:hi]) for i, l in refs])
        tot = torch.from_numpy(oracle.totals(st).astype(np.int64))
        allreduce_totals(tot)
        full = oracle.totals(oracle.stats(cand[0], cand[1], refs))
        ok_tot = bool(np.array_equal(tot.numpy(), full))
        # per-sentence mode: gathering the shards' scores reproduces the full vector
        sc = torch.from_numpy(oracle.scores(st, "exp")["scores"])
        per = -(-B // world)
        buf = torch.zeros(per, dtype=torch.float64)
        buf[: hi - lo] = sc
        out = [torch.empty(per, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(out, buf)
        gathered = torch.cat(out)[:B].numpy()
        ok_sc = bool(np.array_equal(gathered, oracle.scores(oracle.stats(cand[0], cand[1], refs), "exp")["scores"]))
        q.put((rank, ok_tot, ok_sc))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_corpus_totals_and_score_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    assert all(p.exitcode == 0 for p in procs)
    res = sorted(q.get(timeout=5) for _ in range(2))
    assert res == [(0, True, True), (1, True, True)]


def test_allreduce_totals_single_process_is_identity():
    t = torch.arange(10, dtype=torch.int64)
    assert allreduce_totals(t.clone()).equal(t)
