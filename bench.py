"""Benchmark: per-sentence BLEU-4 sentences/s at 512x1024 tokens (V=128k, R=1),
BASELINE.json configs[1] — plus the HBM roofline of the fused kernel and the
reference CPU path timed on this host.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

A "step" is one pass of the hot path over one batch of the workload: the
batch's per-sentence statistics and BLEU scores.  Multi-GPU is weak scaling:
every rank scores its own 512x1024 batch (rows shard with no data-path
collective), value = all sentences / max-over-ranks time.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (B, L, V, R, smoothing)   — BASELINE.json configs
    "c1": (16, 256, 32000, 1, "floor"),
    "c2": (512, 1024, 128000, 1, "none"),
    "c3": (256, 1024, 128000, 4, "add-k"),
    "c4": (4096, 1024, 128000, 1, "none"),
    "c5": (2048, 2048, 256000, 1, "none"),  # per-GPU shard of 16384x2048 over 8 GPUs
}
# c4 is corpus BLEU: one score for the whole (sharded) batch, totals NCCL-all-reduced
MODES = {"c4": "corpus"}
METRIC = "per-sentence BLEU-4 sentences/sec at 512x1024 tok; HBM roofline %; vs CPU ref"
L2_FLUSH_BYTES = 256 << 20


def generate_batch(b, l, v, r, seed=42, data="uniform"):
    """The reference generator, bench.py:72-91: default_rng([seed, B, L, V]),
    IDs uniform in [0, V), lengths uniform in [L/2, L]; candidates then refs.
    data="correlated" (SURVEY §8d parity input): every reference is the
    candidate with a per-row mutation rate p ~ U[0, 0.9] and length +-50."""
    rng = np.random.default_rng([seed, b, l, v])

    def draw():
        ids = rng.integers(0, v, size=(b, l), dtype=np.int64)
        lengths = rng.integers(l // 2, l + 1, size=b, dtype=np.int64)
        return ids, lengths

    cand = draw()
    if data == "uniform":
        return cand, [draw() for _ in range(r)]
    refs = []
    for _ in range(r):
        ids = cand[0].copy()
        m = rng.random((b, l)) < rng.uniform(0.0, 0.9, (b, 1))
        ids[m] = rng.integers(0, v, size=int(m.sum()))
        lengths = np.clip(cand[1] + rng.integers(-50, 51, size=b), l // 2, l)
        refs.append((ids, lengths))
    return cand, refs


def algorithmic_bytes(lengths_rows, v, b, max_order=4):
    """A = 4·Σ len + Σ_n T_n·(2·s_k(n) + 8) + 8·B."""
    lens = np.concatenate([np.asarray(x, dtype=np.int64) for x in lengths_rows])
    bits = math.ceil(math.log2(v))
    a = 4 * int(lens.sum()) + 8 * b
    for n in range(1, max_order + 1):
        t_n = int(np.maximum(lens - n + 1, 0).sum())
        s_k = 8 if n * bits <= 64 else 16
        a += t_n * (2 * s_k + 8)
    return a


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for name, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU legs (reference package from oracle/_ref, else the C oracle port)
# ---------------------------------------------------------------------------
def _ref_pkg():
    import oracle
    return oracle.reference_package()


def cpu_reference_single(cand, refs, smoothing, repeats=3, mode="sentence"):
    """The reference's shipped path: batchbleu.sentence_bleu (corpus_bleu in
    corpus mode), compiled backend, threads=1 — 1 warm-up + `repeats` timed
    runs over the whole batch."""
    bb = _ref_pkg()
    if bb is not None:
        c = bb.TokenBatch(ids=cand[0], lengths=cand[1])
        rs = [bb.TokenBatch(ids=i, lengths=l) for i, l in refs]
        cfg = bb.BleuConfig(smoothing=smoothing)
        fn = bb.corpus_bleu if mode == "corpus" else bb.sentence_bleu
        fn(c, rs, cfg)
        ts = []
        for _ in range(repeats):
            t0 = time.perf_counter()
            fn(c, rs, cfg)
            ts.append(time.perf_counter() - t0)
        return min(ts), "reference", f"batchbleu.{fn.__name__} (oracle/_ref, compiled backend, threads=1)"
    import oracle
    oracle.stats(cand[0][:8], cand[1][:8], [(i[:8], l[:8]) for i, l in refs])
    ts = []
    for _ in range(repeats):
        t0 = time.perf_counter()
        st = oracle.stats(cand[0], cand[1], refs)
        (oracle.corpus if mode == "corpus" else oracle.scores)(st, smoothing)
        ts.append(time.perf_counter() - t0)
    return min(ts), "port", "oracle/tbleu_oracle.c (C restatement, 1 thread)"


_POOL_DATA = {}


def _pool_init(cand, refs, smoothing, mode="sentence"):
    _POOL_DATA.update(cand=cand, refs=refs, smoothing=smoothing, mode=mode)
    import oracle
    oracle.reference_package()


def _pool_work(span):
    import batchbleu as bb
    lo, hi = span
    cand, refs = _POOL_DATA["cand"], _POOL_DATA["refs"]
    c = bb.TokenBatch(ids=cand[0][lo:hi], lengths=cand[1][lo:hi])
    rs = [bb.TokenBatch(ids=i[lo:hi], lengths=l[lo:hi]) for i, l in refs]
    cfg = bb.BleuConfig(smoothing=_POOL_DATA["smoothing"])
    if _POOL_DATA["mode"] == "corpus":
        st = bb.compute_stats(c, rs, cfg)  # per-shard statistics; the parent aggregates
        return st.numerators, st.denominators, st.cand_lens, st.eff_ref_lens
    return bb.sentence_bleu(c, rs, cfg).scores


def _pool_corpus(parts, smoothing):
    """Corpus score of the shards' statistics, by the reference's own epilogue
    (batchbleu.bleu.score_corpus_from_stats, bleu.py:293-305)."""
    import batchbleu as bb
    from batchbleu.bleu import score_corpus_from_stats
    st = bb.SentenceStats(*[np.concatenate([p[k] for p in parts]) for k in range(4)])
    return score_corpus_from_stats(st, bb.BleuConfig(smoothing=smoothing)).scores


def run_reference_arm(args):
    """--impl reference: the reference's own CPU implementation on this host's
    cores (process pool over row shards of the reference's sentence_bleu; in
    corpus mode the shards' compute_stats, aggregated by the reference's
    score_corpus_from_stats)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    b, l, v, r, smoothing = WORKLOADS[args.workload]
    mode = MODES.get(args.workload, "sentence")
    cand, refs = generate_batch(b, l, v, r)
    bb = _ref_pkg()
    cores = len(os.sched_getaffinity(0))
    line = {"metric": METRIC, "unit": "sentences/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic (reference generate_batch, seed 42)",
            "config": {"workload": f"{args.workload}: {mode} BLEU-4, B={b} L={l} V={v} R={r} smoothing={smoothing}"}}
    if bb is None:
        # the oracle port, all cores via processes is not worth it for the C port: 1 thread
        t, kind, what = cpu_reference_single(cand, refs, smoothing, repeats=max(args.steps, 1), mode=mode)
        value = b / t
        line.update(value=value, ms_per_step=t * 1e3,
                    cpu_baseline={"value": value, "unit": "sentences/s", "cores": 1, "kind": kind, "sample": what},
                    e2e={"value": value, "unit": "sentences/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0})
        print(json.dumps(line), flush=True)
        return 0
    from concurrent.futures import ProcessPoolExecutor
    import multiprocessing as mp
    workers = cores
    per = -(-b // workers)
    spans = [(lo, min(lo + per, b)) for lo in range(0, b, per)]
    ctx = mp.get_context("fork")
    with ProcessPoolExecutor(max_workers=workers, mp_context=ctx, initializer=_pool_init,
                             initargs=(cand, refs, smoothing, mode)) as pool:
        def step():
            out = list(pool.map(_pool_work, spans))
            if mode == "corpus":
                _pool_corpus(out, smoothing)
        for _ in range(max(args.warmup, 1)):
            step()
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            step()
            times.append(time.perf_counter() - t0)
    t_pool = float(np.mean(times))
    # threads=1 shipped configuration, for the record
    t1, kind, what = cpu_reference_single(cand, refs, smoothing, repeats=2, mode=mode)
    value = b / t_pool
    line.update(value=value, ms_per_step=t_pool * 1e3,
                cpu_baseline={"value": value, "unit": "sentences/s", "cores": workers, "kind": "reference",
                              "sample": f"batchbleu.{'compute_stats' if mode == 'corpus' else 'sentence_bleu'} "
                                        f"over {len(spans)} row shards in a {workers}-process pool (harness "
                                        f"wrapper), full {b}x{l} batch per step",
                              "single_core_value": b / t1},
                e2e={"value": value, "unit": "sentences/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0})
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# Our arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2510_05485_b200 as tb

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # TB_BENCH_SHARED_GPU=1 (testing only): every rank on cuda:0 over gloo, so the
    # multi-rank logic can be exercised on a one-GPU box; never used for numbers
    shared = os.environ.get("TB_BENCH_SHARED_GPU") == "1"
    gpu = 0 if shared else local
    # TB_BENCH_FORCE_DIST=1 (testing only): the process group and its collectives
    # even at world size 1, so the NCCL code path runs on a one-GPU box
    distributed = world > 1 or os.environ.get("TB_BENCH_FORCE_DIST") == "1"
    if distributed:
        torch.cuda.set_device(gpu)
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", gpu))
    dev = torch.device("cuda", gpu if distributed else 0)
    torch.cuda.set_device(dev)

    b, l, v, r, smoothing = WORKLOADS[args.workload]
    mode = MODES.get(args.workload, "sentence")
    corpus = mode == "corpus"
    cand_np, refs_np = generate_batch(b, l, v, r, seed=42 + rank, data=args.data)
    cfg = tb.BleuConfig(smoothing=smoothing)
    mk_plan = (lambda c_, r_: tb.SentenceBleuPlan(c_, r_, cfg, stats=False, corpus=True, sentence=False)) \
        if corpus else (lambda c_, r_: tb.SentenceBleuPlan(c_, r_, cfg))

    # device-resident inputs (int32 IDs).  Batch 0 is the
    # reference generator's batch; the timed loop cycles through `nbuf` distinct
    # batches whose combined footprint exceeds L2, so no step reads another
    # step's cache-resident inputs (the timing rule's "inputs larger than L2").
    to_dev = lambda a, dt: torch.as_tensor(a).to(dev, dtype=dt)  # noqa: E731
    cand = tb.TokenBatch(ids=to_dev(cand_np[0], torch.int32), lengths=to_dev(cand_np[1], torch.int64))
    refs = [tb.TokenBatch(ids=to_dev(i, torch.int32), lengths=to_dev(ln, torch.int64)) for i, ln in refs_np]
    batch_bytes = b * l * 4 * (1 + r) + 8 * b * (1 + r)
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    nbuf = max(2, -(-2 * l2_bytes // batch_bytes))
    gen = torch.Generator(device=dev)
    plans = [mk_plan(cand, refs)]
    for k in range(1, nbuf):
        gen.manual_seed(1000 * (42 + rank) + k)

        def draw():
            ids = torch.randint(0, v, (b, l), generator=gen, device=dev, dtype=torch.int32)
            lens = torch.randint(l // 2, l + 1, (b,), generator=gen, device=dev, dtype=torch.int64)
            return tb.TokenBatch.trusted(ids, lens)

        def mutate(c_):
            p_ = torch.rand((b, 1), generator=gen, device=dev) * 0.9
            m_ = torch.rand((b, l), generator=gen, device=dev) < p_
            ids = torch.where(m_, torch.randint(0, v, (b, l), generator=gen, device=dev, dtype=torch.int32), c_.ids)
            lens = (c_.lengths + torch.randint(-50, 51, (b,), generator=gen, device=dev)).clamp(l // 2, l)
            return tb.TokenBatch.trusted(ids, lens)

        c_k = draw()
        plans.append(mk_plan(c_k, [draw() if args.data == "uniform" else mutate(c_k) for _ in range(r)]))
    plan = plans[0]

    def step(pl):
        """One step: the fused kernel (one launch); in corpus mode across
        ranks, then the NCCL all-reduce of the 2N+2 int64 totals over NVLink
        and the corpus epilogue on every rank."""
        pl.run()
        if corpus and distributed:
            dist.all_reduce(pl.totals, op=dist.ReduceOp.SUM)
            pl.corpus_from_totals()

    kernels_per_step = 1 + (1 if corpus and distributed else 0)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)

    def barrier():
        if distributed:
            dist.barrier()

    # correctness gate before timing (bench.py:104-113 analogue): counts vs oracle on a slice
    import oracle
    if rank == 0:
        st = tb.compute_stats(tb.TokenBatch(ids=cand_np[0][:32], lengths=cand_np[1][:32]),
                              [tb.TokenBatch(ids=i[:32], lengths=ln[:32]) for i, ln in refs_np], cfg)
        o = oracle.stats(cand_np[0][:32], cand_np[1][:32], [(i[:32], ln[:32]) for i, ln in refs_np])
        if not np.array_equal(st.numerators, o["numerators"]):
            print(json.dumps({"error": "equivalence check failed"}), flush=True)
            return 2

    # ---- device-resident timing: K steps, back to back, each on its own batch
    stream = torch.cuda.current_stream(dev)
    for k in range(max(args.warmup, 1) * len(plans)):
        step(plans[k % len(plans)])
    torch.cuda.synchronize(dev)
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clk:
        # keep the GPU under this load for ~1 s so that nvidia-smi (>= 50 ms period)
        # samples the clocks of this workload; the timed steps follow directly
        t_until = time.perf_counter() + args.clock_window
        while time.perf_counter() < t_until:
            for k in range(200):
                step(plans[k % len(plans)])
            torch.cuda.synchronize(dev)
        barrier()
        torch.cuda.synchronize(dev)
        t_start.record(stream)
        for k in range(args.steps):
            step(plans[k % len(plans)])
        t_end.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
    t_local = t_start.elapsed_time(t_end) / 1e3
    t = torch.tensor([t_local], dtype=torch.float64, device=dev)
    if distributed:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_max = float(t.item())
    value = b * world * args.steps / t_max

    # ---- secondary: one batch, L2 flushed (256 MiB write) before every step, each step event-timed
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    for k in range(args.steps):
        flush.zero_()
        starts[k].record(stream)
        step(plan)
        ends[k].record(stream)
    torch.cuda.synchronize(dev)
    step_ms = [s_.elapsed_time(e_) for s_, e_ in zip(starts, ends)]

    # ---- eager public API (no graph), same device-resident inputs
    def eager_call():
        if not corpus:
            return tb.sentence_bleu(cand, refs, cfg)
        if not distributed:
            return tb.corpus_bleu(cand, refs, cfg)
        from paper_2510_05485_b200.distributed import allreduce_totals
        return tb.score_corpus_from_totals(allreduce_totals(tb.corpus_totals(cand, refs, cfg)), cfg)

    for _ in range(2):
        eager_call()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    eager = []
    for _ in range(args.steps):
        flush.zero_()
        e0.record(stream)
        eager_call()
        e1.record(stream)
        e1.synchronize()
        eager.append(e0.elapsed_time(e1))

    # ---- e2e: public API with pinned HOST buffers; H2D + kernel + D2H in the timed region.
    # Headline: int32 token IDs (the dtype the path computes in, and what a
    # training loop's tokenizer output holds); int64 (the reference
    # TokenBatch's own dtype, batch.py:23-24) is reported beside it.
    d2h = 4 + (b * (2 + cfg.max_order) * 8 if not corpus else (3 * cfg.max_order + 4) * 8)

    def measure_e2e(np_dtype, numpy_rows=False):
        if numpy_rows:  # the reference's usage: TokenBatch over (pageable) numpy arrays
            hcand = tb.TokenBatch(ids=cand_np[0].astype(np_dtype), lengths=cand_np[1])
            hrefs = [tb.TokenBatch(ids=i.astype(np_dtype), lengths=ln) for i, ln in refs_np]
        else:
            hcand = tb.TokenBatch(ids=torch.from_numpy(cand_np[0].astype(np_dtype)).pin_memory(),
                                  lengths=torch.from_numpy(cand_np[1]))
            hrefs = [tb.TokenBatch(ids=torch.from_numpy(i.astype(np_dtype)).pin_memory(), lengths=torch.from_numpy(ln))
                     for i, ln in refs_np]
        # tb_bleu_host: the kernel reads each pinned row's valid prefix over PCIe
        # (zero-copy) plus the lengths; results are written straight into pinned memory
        isz = np.dtype(np_dtype).itemsize
        h2d = int(sum(isz * int(ln.sum()) + 8 * ln.size for ln in [cand_np[1]] + [x for _, x in refs_np]))

        def e2e_call():
            """The user's call on host buffers; results come back as numpy / floats."""
            if not corpus:
                return tb.sentence_bleu(hcand, hrefs, cfg)
            if not distributed:
                return tb.corpus_bleu(hcand, hrefs, cfg)
            tot = torch.from_numpy(tb.corpus_totals(hcand, hrefs, cfg)).to(dev)  # this rank's shard
            dist.all_reduce(tot, op=dist.ReduceOp.SUM)                            # NCCL, 80 B
            return tb.score_corpus_from_totals(tot, cfg, host=True)

        for _ in range(2):
            e2e_call()
        barrier()
        e2e_times = []
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            res = e2e_call()   # returns numpy / float: synchronous end to end
            e2e_times.append(time.perf_counter() - t0)
        assert corpus or res.scores.shape == (b,)
        te = torch.tensor([float(np.sum(e2e_times))], dtype=torch.float64, device=dev)
        if distributed:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        return b * world * args.steps / float(te.item()), h2d

    e2e_value, h2d = measure_e2e(np.int32)
    e2e64_value, h2d64 = measure_e2e(np.int64)
    e2e_np_value, _ = measure_e2e(np.int64, numpy_rows=True)

    # ---- roofline of the fused kernel (the only kernel of a step)
    a_bytes = algorithmic_bytes([cand_np[1]] + [ln for _, ln in refs_np], v, b)
    kernel_s = t_local / args.steps  # back-to-back: kernel + inter-launch gap (conservative)
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peaks = json.load(fh)
        peak, peak_src = float(peaks["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    achieved = a_bytes / kernel_s / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as fh:
            prof = json.load(fh).get(args.workload, {})
            traffic = prof.get("dram_bytes_per_launch")
    except Exception:
        pass
    input_bytes = int(sum(4 * int(x.sum()) for x in [cand_np[1]] + [ln for _, ln in refs_np]))

    line = None
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline:
            t_cpu, kind, what = cpu_reference_single(cand_np, refs_np, smoothing, repeats=3, mode=mode)
            cpu = {"value": b / t_cpu, "unit": "sentences/s", "cores": 1, "kind": kind,
                   "sample": f"{what}; the full {b}x{l} batch, best of 3 after 1 warm-up"}
        line = {
            "metric": METRIC, "value": value, "unit": "sentences/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
            "data": ("synthetic (reference generate_batch: uniform IDs, lengths U[L/2, L], seed 42+rank)"
                     if args.data == "uniform" else
                     "synthetic, correlated: references = candidate with per-row mutation rate U[0, 0.9]"),
            "config": {"workload": f"{args.workload}: {'corpus' if corpus else 'per-sentence'} BLEU-4, "
                                   f"B={b} L={l} V={v} R={r} smoothing={smoothing}, per GPU (weak scaling)",
                       "global_batch": b * world, "seq_len": l, "parallelism": f"dp{world} (row shards)",
                       "timed_path": "SentenceBleuPlan.run(): one tb_bleu_stats launch per step (native binding)"
                                     + (", then NCCL all_reduce of the int64 totals + corpus epilogue kernel"
                                        if corpus and distributed else "")
                                     + "; K steps back to back between two CUDA events",
                       "l2": f"inputs larger than L2: steps cycle through {nbuf} distinct device-resident "
                             f"batches ({nbuf * batch_bytes / 2**20:.0f} MiB > {l2_bytes / 2**20:.0f} MiB L2); "
                             "batch 0 = reference generator seed 42, others torch.randint of the same "
                             "distributions"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": a_bytes,
                         # the DRAM bytes the kernel really moves (ncu) over the same step time:
                         # how far from HBM-bound it is (it is latency-bound)
                         "dram_achieved": (traffic / kernel_s / 1e9) if traffic else None,
                         "dram_frac": (traffic / kernel_s / 1e9 / peak) if traffic else None,
                         "note": "A = SURVEY §8(d) paper-dataflow bytes; the fused kernel only reads the "
                                 f"{input_bytes} B of int32 tokens, so frac > 1 means it beats the paper dataflow; "
                                 "dram_frac = ncu DRAM bytes per launch / step time / peak"},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "sentences/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "token_dtype": "int32",
                    "int64_tokens": {"value": e2e64_value, "h2d_bytes_per_step": int(h2d64)},
                    "numpy_int64_tokens": {"value": e2e_np_value,
                                           "path": "TokenBatch(numpy int64, pageable) as the reference uses it: "
                                                   "valid prefixes copied into pinned memory by host threads, "
                                                   "narrowed to int32 when the IDs fit, read over PCIe"},
                    "path": f"{'corpus' if corpus else 'sentence'}_bleu(TokenBatch(pinned host tensors)) "
                            "-> numpy: one blocking tb_bleu_host call; the kernel streams valid row prefixes "
                            "over PCIe" + (" (+ NCCL all_reduce of the totals)" if corpus and distributed else "")},
            "eager_api": {"value": b * world / (np.mean(eager) / 1e3), "unit": "sentences/s",
                          "ms_per_step": float(np.mean(eager)),
                          "path": "public API on TokenBatch(CUDA tensors), eager, per-call allocation"},
            "gpu_launches": args.steps * kernels_per_step,
            "clocks": clk.summary(),
            "step_flush_l2": {"value": b * world / (float(np.mean(step_ms)) / 1e3), "unit": "sentences/s",
                              "ms_per_step": float(np.mean(step_ms)), "min_ms": float(np.min(step_ms)),
                              "path": "one batch, 256 MiB L2-flush write before every step, each step "
                                      "timed by its own CUDA events (includes launch latency)"},
        }
        print(json.dumps(line), flush=True)
    if distributed:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=20)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--workload", choices=sorted(WORKLOADS), default="c2")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--data", choices=["uniform", "correlated"], default="uniform",
                   help="uniform = the reference generator (the headline); correlated = related references")
    p.add_argument("--clock-window", type=float, default=1.5,
                   help="seconds of sustained load sampled by nvidia-smi before the timed steps")
    args = p.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
