"""Per-sentence and corpus BLEU on the B200.

Mirror of ``batchbleu.bleu`` (pkg/src/batchbleu/bleu.py): same public names,
signatures, defaults, error types and result types.  The counting engine and
the epilogue run in the fused CUDA kernel behind ``tb_bleu_stats``
(include/tensorbleu.h); this module only validates arguments, moves host
arrays to the device, launches, and unpacks results.

Result types follow the inputs: host inputs (numpy / lists / CPU tensors)
give numpy arrays and Python floats exactly like the reference; CUDA-tensor
inputs give CUDA tensors and never synchronise the host.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Optional, Sequence, Union

import numpy as np
import torch

from . import _native
from .batch import TokenBatch

SMOOTHING_METHODS = ("none", "floor", "add-k", "exp")


@dataclass(frozen=True)
class BleuConfig:
    """Max n-gram order, per-order weights, and smoothing (bleu.py:24-56)."""

    max_order: int = 4
    weights: Optional[Sequence[float]] = None
    smoothing: str = "none"
    eps: float = 0.1      # floor smoothing
    k: float = 1.0        # add-k smoothing, orders >= 2

    def __post_init__(self):
        if self.max_order < 1:
            raise ValueError("max_order must be >= 1")
        if self.smoothing not in SMOOTHING_METHODS:
            raise ValueError(
                f"unknown smoothing {self.smoothing!r}; expected one of {SMOOTHING_METHODS}")
        if self.eps <= 0:
            raise ValueError("eps must be > 0")
        if self.k <= 0:
            raise ValueError("k must be > 0")
        if self.weights is None:
            w = np.full(self.max_order, 1.0 / self.max_order)
        else:
            w = np.asarray(self.weights, dtype=np.float64)
            if w.shape != (self.max_order,):
                raise ValueError(f"expected {self.max_order} weights, got shape {w.shape}")
            if np.any(w < 0) or w.sum() <= 0:
                raise ValueError("weights must be non-negative with positive sum")
            w = w / w.sum()
        object.__setattr__(self, "weights", tuple(float(x) for x in w))


@dataclass(frozen=True)
class SentenceStats:
    """Per-sentence clipped numerators/denominators for orders 1..N plus
    candidate and effective reference lengths (bleu.py:59-67).  numpy int64
    arrays for host inputs, CUDA int64 tensors for device inputs."""

    numerators: object     # (B, N) int64
    denominators: object   # (B, N) int64
    cand_lens: object      # (B,) int64
    eff_ref_lens: object   # (B,) int64


@dataclass(frozen=True)
class BleuResult:
    """Scores in [0, 1]; per-order precisions and BP kept for diagnostics."""

    scores: Union[np.ndarray, float, torch.Tensor]
    precisions: object
    brevity_penalty: Union[np.ndarray, float, torch.Tensor]


# ---------------------------------------------------------------------------
# Scalar helpers (bleu.py:79-94) — host logic, not on the batch path.
# ---------------------------------------------------------------------------
def effective_ref_len(cand_len: int, ref_lens: Sequence[int]) -> int:
    """Reference length closest to the candidate's; ties go to the shorter."""
    if len(ref_lens) == 0:
        raise ValueError("at least one reference length is required")
    return min(ref_lens, key=lambda r: (abs(r - cand_len), r))


def brevity_penalty(cand_len: int, eff_ref_len: int) -> float:
    """exp(1 - r/c) for short candidates, 1.0 otherwise; empty candidate -> 0."""
    if cand_len < 0:
        raise ValueError("candidate length must be >= 0")
    if cand_len == 0:
        return 0.0
    if cand_len > eff_ref_len:
        return 1.0
    return math.exp(1.0 - eff_ref_len / cand_len)


def _check_batches(candidates: TokenBatch, references: Sequence[TokenBatch]) -> None:
    """bleu.py:97-105."""
    if not references:
        raise ValueError("at least one reference batch is required")
    for ref in references:
        if ref.batch_size != candidates.batch_size:
            raise ValueError(
                f"reference batch size {ref.batch_size} does not match "
                f"candidate batch size {candidates.batch_size}")


# ---------------------------------------------------------------------------
# Host <-> device plumbing.
# ---------------------------------------------------------------------------
_weights_cache: dict = {}


def _weights_arg(config: BleuConfig):
    w = _weights_cache.get(config.weights)
    if w is None:
        w = (ctypes.c_double * len(config.weights))(*config.weights)
        _weights_cache[config.weights] = w
    return w


def _weights_addr(config: BleuConfig) -> int:
    return ctypes.addressof(_weights_arg(config))


def _to_device(batch: TokenBatch, device: torch.device, want64: bool):
    """(ids, lengths, ld) on `device`; host data is copied (H2D) every call."""
    ids, lengths = batch.ids, batch.lengths
    if isinstance(ids, np.ndarray):
        ids = torch.from_numpy(ids)
        lengths = torch.from_numpy(lengths)
    if not ids.is_cuda:
        nb = ids.is_pinned()
        ids = ids.to(device, non_blocking=nb)
        lengths = lengths.to(device, non_blocking=nb)
    elif ids.device != device:
        raise ValueError(f"all batches must live on one device ({ids.device} vs {device})")
    if want64 and ids.dtype != torch.int64:
        ids = ids.to(torch.int64)
    ld = ids.stride(0) if ids.shape[0] > 1 else ids.shape[1]
    return ids, lengths, ld


_MODES = {"stats": 0, "sentence": 1, "corpus": 2}
_OUT_NAMES = {"stats": ("num", "den", "cand_len", "eff_ref"),
              "sentence": ("scores", "precisions", "bp"),
              "corpus": ("totals", "corpus")}


def _launch_host(candidates: TokenBatch, references: Sequence[TokenBatch], config: BleuConfig,
                 mode: str):
    """Host-buffer path: ONE blocking tb_bleu_host call through the native
    binding (_hostpath, GIL released).  Pinned token rows are read by the
    kernel over PCIe (valid prefixes only); results come back as numpy."""
    hp = _native._hp or _native.hostpath()
    dev = _native.current_device_index()
    want64 = not candidates._tok32
    for b in references:
        want64 = want64 or not b._tok32
    held = [candidates._row_view(want64), *[b._row_view(want64) for b in references]]  # keeps widened copies alive
    views = tuple(h[0] for h in held)
    smc, eps, k, waddr = _config_abi(config)
    rc, flags, *outs = hp.run(_MODES[mode], views, candidates.batch_size, config.max_order,
                              smc, eps, k, waddr, _native.raw_stream(dev))
    if rc:
        _native.check(rc, "tb_bleu_host")
    if flags:
        _native.raise_flags(flags)
    return True, dict(zip(_OUT_NAMES[mode], outs)), None


def _config_abi(config: BleuConfig):
    """(smoothing code, eps, k, weights address) of a config, cached on it."""
    v = config.__dict__.get("_abi")
    if v is None:
        v = (_native.SMOOTHING_CODES[config.smoothing], config.eps, config.k, _weights_addr(config))
        object.__setattr__(config, "_abi", v)
    return v


_ws_bytes_cache: dict = {}
_err_words: dict = {}


def _launch_device(candidates: TokenBatch, references: Sequence[TokenBatch], config: BleuConfig,
                   mode: str, device: torch.device):
    """All rows already on `device`: one asynchronous tb_bleu_stats launch
    through the native binding, outputs carved from one allocation, no host
    synchronisation."""
    hp = _native.hostpath()
    batches = (candidates, *references)
    want64 = any(b.ids.dtype != torch.int32 for b in batches)
    held = [b._row_view(want64) for b in batches]  # widened copies live until the launch is queued
    views = tuple(h[0] for h in held)
    B, N = candidates.batch_size, config.max_order
    key = (device.index, B, tuple(v[2] for v in views), views[0][4], N)
    wsb = _ws_bytes_cache.get(key)
    if wsb is None:
        widths = np.array([v[2] for v in views[1:]], dtype=np.int64)
        wsb = _native.load().tb_bleu_workspace_bytes(B, len(references), views[0][2], widths.ctypes.data,
                                                     views[0][4], N)
        if wsb == 0:
            raise ValueError("unsupported shape for the device path")
        _ws_bytes_cache[key] = wsb
    ws = _native.workspace.get(device, wsb)
    err = _err_words.get(device.index)
    if err is None:
        err = _err_words[device.index] = torch.zeros(1, dtype=torch.int32, device=device)
    if mode == "sentence":
        buf = torch.empty(B * (N + 2), dtype=torch.float64, device=device)
        a = buf.data_ptr()
        outs = (None, None, None, None, a, a + 16 * B, a + 8 * B, None, None)
        views_out = {"scores": buf[:B], "bp": buf[B:2 * B], "precisions": buf[2 * B:].view(B, N)}
    elif mode == "stats":
        buf = torch.empty(2 * B * (N + 1), dtype=torch.int64, device=device)
        a = buf.data_ptr()
        outs = (a, a + 8 * B * N, a + 16 * B * N, a + 16 * B * N + 8 * B, None, None, None, None, None)
        views_out = {"num": buf[:B * N], "den": buf[B * N:2 * B * N], "cand_len": buf[2 * B * N:2 * B * N + B],
                     "eff_ref": buf[2 * B * N + B:]}
    else:
        buf = torch.empty(3 * N + 4, dtype=torch.int64, device=device)
        a = buf.data_ptr()
        outs = (None,) * 7 + (a, a + 8 * (2 * N + 2))
        views_out = {"totals": buf[:2 * N + 2], "corpus": buf[2 * N + 2:].view(torch.float64)}
    rc = hp.launch(views, B, N, _native.SMOOTHING_CODES[config.smoothing], config.eps, config.k,
                   _weights_addr(config), outs, err.data_ptr(), ws.data_ptr(), ws.numel(),
                   _native.stream_handle(device))
    if rc:
        _native.check(rc, "tb_bleu_stats")
    return False, views_out, None


def _launch(candidates: TokenBatch, references: Sequence[TokenBatch], config: BleuConfig,
            mode: str):
    """Run tb_bleu_stats.  mode: 'stats' | 'sentence' | 'corpus'.

    Returns (host_mode, tensors dict on device, device-side output buffer)."""
    _check_batches(candidates, references)
    if config.max_order > _native.TB_MAX_ORDER or len(references) > _native.TB_MAX_REFS:
        return _launch_unbounded(candidates, references, config, mode)
    if not candidates.is_device:
        return _launch_host(candidates, references, config, mode)
    device = candidates.ids.device
    if all(r.is_device and r.ids.device == device for r in references):
        return _launch_device(candidates, references, config, mode, device)
    lib = _native.load()
    device = candidates.ids.device
    _native.require_cuda(device)
    batches = [candidates, *references]
    want64 = any((b.ids.dtype != torch.int32) if isinstance(b.ids, torch.Tensor)
                 else True for b in batches)
    with torch.cuda.device(device):
        dev = [_to_device(b, device, want64) for b in batches]
        token_bytes = 8 if want64 else 4
        B = candidates.batch_size
        N = config.max_order
        R = len(references)

        # one output buffer: [err i32 (8 B) | payload]
        if mode == "sentence":
            sizes = [("scores", B, torch.float64), ("bp", B, torch.float64),
                     ("precisions", B * N, torch.float64)]
        elif mode == "stats":
            sizes = [("num", B * N, torch.int64), ("den", B * N, torch.int64),
                     ("cand_len", B, torch.int64), ("eff_ref", B, torch.int64)]
        else:
            sizes = [("corpus", N + 2, torch.float64), ("totals", 2 * N + 2, torch.int64)]
        total = 8 + 8 * sum(n for _, n, _ in sizes)
        out = torch.empty(total, dtype=torch.uint8, device=device)
        views = {}
        off = 8
        for name, n, dt in sizes:
            views[name] = out[off: off + 8 * n].view(dt)
            off += 8 * n
        err = out[:4].view(torch.int32)
        if mode == "corpus":
            err.zero_()  # per-sentence launches OR their flags into it (include/tensorbleu.h)

        ref_widths = np.array([b.max_len for b in references], dtype=np.int64)
        ws_bytes = lib.tb_bleu_workspace_bytes(B, R, candidates.max_len,
                                               ref_widths.ctypes.data, token_bytes, N)
        if ws_bytes == 0:
            raise ValueError("unsupported shape for the device path")
        ws = _native.workspace.get(device, ws_bytes)

        ref_ids = (ctypes.c_void_p * R)(*[d[0].data_ptr() for d in dev[1:]])
        ref_lens = (ctypes.c_void_p * R)(*[d[1].data_ptr() for d in dev[1:]])
        ref_ld = (ctypes.c_int64 * R)(*[d[2] for d in dev[1:]])
        ref_w = (ctypes.c_int64 * R)(*[int(w) for w in ref_widths])
        P = lambda name: views[name].data_ptr() if name in views else None  # noqa: E731
        cand_ids, cand_len, cand_ld = dev[0]
        rc = lib.tb_bleu_stats(
            token_bytes, cand_ids.data_ptr(), cand_ld, candidates.max_len, cand_len.data_ptr(),
            R, ref_ids, ref_ld, ref_w, ref_lens, B, N,
            _native.SMOOTHING_CODES[config.smoothing], config.eps, config.k,
            _weights_arg(config),
            P("num"), P("den"), P("cand_len"), P("eff_ref"),
            P("scores"), P("precisions"), P("bp"),
            P("totals"), P("corpus"),
            err.data_ptr(), ws.data_ptr(), ws.numel(), _native.stream_handle(device))
        _native.check(rc, "tb_bleu_stats")

    return False, views, None


def _launch_unbounded(candidates: TokenBatch, references: Sequence[TokenBatch], config: BleuConfig,
                      mode: str):
    """More reference sets or orders than the fused kernels take: the
    reference's per-order algorithm on the device n-gram operator kernels
    (unbounded.py).  Same outputs and result types as _launch."""
    from . import unbounded
    host = not candidates.is_device
    dev = candidates.ids.device if not host else _native.require_cuda()
    with torch.cuda.device(dev):
        num, den, cl, er = unbounded.stats(candidates, references, config.max_order, dev)
        if mode == "stats":
            out = {"num": num, "den": den, "cand_len": cl, "eff_ref": er}
        elif mode == "sentence":
            sc, prec, bp = unbounded.scores(num, den, cl, er, config, dev)
            out = {"scores": sc, "precisions": prec, "bp": bp}
        else:
            N = config.max_order
            tot = unbounded.totals(num, den, cl, er, dev)
            sc, prec, bp = unbounded.scores(tot[None, :N], tot[None, N:2 * N].contiguous(), tot[2 * N:2 * N + 1],
                                            tot[2 * N + 1:2 * N + 2], config, dev)
            out = {"totals": tot, "corpus": torch.cat([sc, bp, prec[0]])}
    if host:
        out = {k: v.cpu().numpy() for k, v in out.items()}
    return host, out, None


def check_device_flags(device=None) -> None:
    """Synchronise with `device` (default: the current CUDA device) and raise
    ValueError if a device-resident call since the last check met bad input
    data — lengths outside [0, width] in batches built with
    TokenBatch.trusted (the kernels clamp them and OR a flag instead of
    stopping); the flag word is cleared.  Device calls never synchronise on
    their own, so this is how an asynchronous training loop surfaces them."""
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    err = _err_words.get(dev.index)
    if err is None:
        return
    flags = int(err.item())
    err.zero_()
    _native.raise_flags(flags)


def compute_stats(candidates: TokenBatch, references: Sequence[TokenBatch],
                  config: BleuConfig, *, threads: int = 1,
                  chunk_size: Optional[int] = None) -> SentenceStats:
    """Counting pipeline for every order, reduced to per-sentence numerators
    and denominators (bleu.py:173-210).

    ``threads`` and ``chunk_size`` are accepted for signature compatibility;
    the device path never chunks, and results never depend on them (as in the
    reference, test_bleu.py:237-246)."""
    host, r, _ = _launch(candidates, references, config, "stats")
    B, N = candidates.batch_size, config.max_order
    return SentenceStats(numerators=r["num"].reshape(B, N), denominators=r["den"].reshape(B, N),
                         cand_lens=r["cand_len"], eff_ref_lens=r["eff_ref"])


def sentence_bleu(candidates: TokenBatch, references: Sequence[TokenBatch],
                  config: Optional[BleuConfig] = None, *, threads: int = 1,
                  chunk_size: Optional[int] = None) -> BleuResult:
    """One BLEU score per sentence of the batch (bleu.py:264-271)."""
    config = config or BleuConfig()
    host, r, _ = _launch(candidates, references, config, "sentence")
    B, N = candidates.batch_size, config.max_order
    return BleuResult(scores=r["scores"], precisions=r["precisions"].reshape(B, N),
                      brevity_penalty=r["bp"])


def corpus_bleu(candidates: TokenBatch, references: Sequence[TokenBatch],
                config: Optional[BleuConfig] = None, *, threads: int = 1,
                chunk_size: Optional[int] = None) -> BleuResult:
    """One score for the whole batch: statistics are aggregated over
    sentences before precisions, BP and the geometric mean (bleu.py:282-290)."""
    config = config or BleuConfig()
    host, r, _ = _launch(candidates, references, config, "corpus")
    c = r["corpus"]
    if host:
        return BleuResult(scores=float(c[0]), precisions=c[2:].copy(),
                          brevity_penalty=float(c[1]))
    return BleuResult(scores=c[0], precisions=c[2:], brevity_penalty=c[1])


def corpus_totals(candidates: TokenBatch, references: Sequence[TokenBatch],
                  config: Optional[BleuConfig] = None) -> object:
    """The int64 vector [Σnum_1..N | Σden_1..N | Σc | Σr] that
    ``score_corpus_from_stats`` reduces to (bleu.py:295-300); the quantity
    all-reduced across GPUs in sharded corpus mode."""
    config = config or BleuConfig()
    _, r, _ = _launch(candidates, references, config, "corpus")
    return r["totals"]


# ---------------------------------------------------------------------------
# Epilogue over given statistics.
# ---------------------------------------------------------------------------
def _stats_on_device(stats: SentenceStats):
    arrs = [stats.numerators, stats.denominators, stats.cand_lens, stats.eff_ref_lens]
    if all(isinstance(a, torch.Tensor) and a.is_cuda for a in arrs):
        dev = arrs[0].device
        return False, dev, [a.to(torch.int64).contiguous() for a in arrs]
    dev = _native.require_cuda()
    out = []
    for a in arrs:
        a = a.cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)
        out.append(torch.from_numpy(np.ascontiguousarray(a, dtype=np.int64)).to(dev))
    return True, dev, out


def _epilogue(stats: SentenceStats, config: BleuConfig, want_scores: bool, fp32: bool = False):
    lib = _native.load()
    host, dev, (num, den, cl, er) = _stats_on_device(stats)
    if num.dim() != 2 or num.shape[1] != config.max_order:
        raise ValueError(f"numerators must be (B, {config.max_order})")
    B, N = num.shape
    if fp32 or N > _native.TB_MAX_ORDER:  # any N / the fp32 epilogue: tb_bleu_scores_any
        from . import unbounded
        with torch.cuda.device(dev):
            sc, prec, bp = unbounded.scores(num.contiguous(), den.contiguous(), cl, er, config, dev, fp32=fp32)
        if host:
            return (sc.cpu().numpy() if want_scores else None), prec.cpu().numpy(), bp.cpu().numpy()
        return (sc if want_scores else None), prec, bp
    with torch.cuda.device(dev):
        prec = torch.empty((B, N), dtype=torch.float64, device=dev)
        bp = torch.empty(B, dtype=torch.float64, device=dev)
        sc = torch.empty(B, dtype=torch.float64, device=dev) if want_scores else None
        rc = lib.tb_bleu_scores(num.data_ptr(), den.data_ptr(), cl.data_ptr(), er.data_ptr(), B, N,
                                _native.SMOOTHING_CODES[config.smoothing], config.eps, config.k,
                                _weights_arg(config),
                                sc.data_ptr() if sc is not None else None, prec.data_ptr(),
                                bp.data_ptr(), _native.stream_handle(dev))
        _native.check(rc, "tb_bleu_scores")
    if host:
        return (sc.cpu().numpy() if sc is not None else None), prec.cpu().numpy(), bp.cpu().numpy()
    return sc, prec, bp


def apply_smoothing(stats: SentenceStats, config: BleuConfig):
    """Per-sentence per-order precisions, shape (B, N) float64 (bleu.py:213-239)."""
    return _epilogue(stats, config, want_scores=False)[1]


def score_sentences_from_stats(stats: SentenceStats, config: BleuConfig, *,
                               dtype=None) -> BleuResult:
    """bleu.py:274-279.  dtype=torch.float32 (or np.float32) runs the fp32
    epilogue (north_star: within 1e-5 relative of fp64); default fp64 in
    numpy's operation order."""
    fp32 = dtype in (torch.float32, np.float32)
    sc, prec, bp = _epilogue(stats, config, want_scores=True, fp32=fp32)
    return BleuResult(scores=sc, precisions=prec, brevity_penalty=bp)


def _totals_of(stats: SentenceStats):
    lib = _native.load()
    host, dev, (num, den, cl, er) = _stats_on_device(stats)
    B, N = num.shape
    with torch.cuda.device(dev):
        tot = torch.empty(2 * N + 2, dtype=torch.int64, device=dev)
        rc = lib.tb_bleu_totals(num.data_ptr(), den.data_ptr(), cl.data_ptr(), er.data_ptr(), B, N,
                                tot.data_ptr(), _native.stream_handle(dev))
        _native.check(rc, "tb_bleu_totals")
    return host, tot


def score_corpus_from_totals(totals, config: BleuConfig, host: Optional[bool] = None) -> BleuResult:
    """Corpus epilogue on an int64 [Σnum | Σden | Σc | Σr] vector
    (bleu.py:301-305); also the last step of sharded corpus mode."""
    N = config.max_order
    if isinstance(totals, torch.Tensor) and totals.is_cuda:
        t = totals.to(torch.int64)
        host = False if host is None else host
    else:
        t = torch.from_numpy(np.ascontiguousarray(
            totals.cpu().numpy() if isinstance(totals, torch.Tensor) else totals,
            dtype=np.int64)).to(_native.require_cuda())
        host = True if host is None else host
    agg = SentenceStats(numerators=t[None, :N], denominators=t[None, N:2 * N],
                        cand_lens=t[2 * N:2 * N + 1], eff_ref_lens=t[2 * N + 1:2 * N + 2])
    sc, prec, bp = _epilogue(agg, config, want_scores=True)
    if host:
        return BleuResult(scores=float(sc[0]), precisions=prec[0].cpu().numpy(),
                          brevity_penalty=float(bp[0]))
    return BleuResult(scores=sc[0], precisions=prec[0], brevity_penalty=bp[0])


def score_corpus_from_stats(stats: SentenceStats, config: BleuConfig) -> BleuResult:
    """bleu.py:293-305."""
    host, tot = _totals_of(stats)
    return score_corpus_from_totals(tot, config, host=host)
