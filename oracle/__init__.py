"""CPU oracle for the TensorBLEU hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  It is the checker, never
the thing measured or shipped: ``paper_2510_05485_b200`` does not import it
and has no CPU fallback.

Two restatements of the reference algorithm live here:

* ``liboracle_tbleu.so`` (``tbleu_oracle.c``): sort-based per-sentence
  clipped counting + the fp64 epilogue in numpy's operation order; used for
  parity at realistic sizes.  Every function cites the reference file:line
  it follows.
* ``py_*``: a pure-Python restatement of ``batchbleu.oracle``
  (pkg/src/batchbleu/oracle.py:18-118) for small cases.

Both are pinned against the reference itself: ``tests/golden/*.npz`` were
produced by ``tests/golden/make_golden.py`` from the unmodified reference
package (``oracle/_ref``, built by ``oracle/build_ref.sh``), and
``tests/test_oracle_golden.py`` checks both restatements against them and
against the reference's own frozen vectors (pkg/tests/test_oracle.py:78-175).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from collections import Counter
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle_tbleu.so")
REF_DIR = os.path.join(HERE, "_ref")

SMOOTHING_CODES = {"none": 0, "floor": 1, "add-k": 2, "exp": 3}

_lib = None


def build() -> str:
    """Compile the C restatement (gcc; no GPU needed)."""
    src = os.path.join(HERE, "tbleu_oracle.c")
    if (not os.path.exists(LIB_PATH)
            or os.path.getmtime(LIB_PATH) < os.path.getmtime(src)):
        subprocess.check_call(["make", "-s", "-C", HERE])
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        L.oracle_stats.argtypes = [P, i64, P, ctypes.c_int, P, P, P, i64, ctypes.c_int,
                                   P, P, P, P]
        L.oracle_stats.restype = ctypes.c_int
        L.oracle_scores.argtypes = [P, P, P, P, i64, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_double, ctypes.c_double, P, P, P, P]
        L.oracle_scores.restype = None
        L.oracle_totals.argtypes = [P, P, P, P, i64, ctypes.c_int, P]
        L.oracle_totals.restype = None
        L.oracle_segment_bincount.argtypes = [P, P, i64, i64, P]
        L.oracle_segment_bincount.restype = ctypes.c_int
        L.oracle_clipped_numerators.argtypes = [P, P, i64, P, i64, P]
        L.oracle_clipped_numerators.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def stats(cand_ids, cand_len, refs, max_order: int = 4) -> dict:
    """compute_stats (bleu.py:173-210) on host arrays.

    ``refs`` is a list of ``(ids, lengths)`` pairs.  Returns a dict with
    numerators, denominators, cand_lens, eff_ref_lens (int64)."""
    cand_ids = np.ascontiguousarray(cand_ids, dtype=np.int64)
    cand_len = np.ascontiguousarray(cand_len, dtype=np.int64)
    b = cand_ids.shape[0]
    ref_ids = [np.ascontiguousarray(r[0], dtype=np.int64) for r in refs]
    ref_len = [np.ascontiguousarray(r[1], dtype=np.int64) for r in refs]
    R = len(refs)
    n = int(max_order)
    num = np.zeros((b, n), dtype=np.int64)
    den = np.zeros((b, n), dtype=np.int64)
    cl = np.zeros(b, dtype=np.int64)
    er = np.zeros(b, dtype=np.int64)
    if b == 0:
        return dict(numerators=num, denominators=den, cand_lens=cl, eff_ref_lens=er)
    rid_ptrs = (ctypes.c_void_p * R)(*[_ptr(a) for a in ref_ids])
    rlen_ptrs = (ctypes.c_void_p * R)(*[_ptr(a) for a in ref_len])
    rld = np.array([a.shape[1] for a in ref_ids], dtype=np.int64)
    rc = lib().oracle_stats(_ptr(cand_ids), cand_ids.shape[1], _ptr(cand_len), R,
                            ctypes.cast(rid_ptrs, ctypes.c_void_p), _ptr(rld),
                            ctypes.cast(rlen_ptrs, ctypes.c_void_p), b, n,
                            _ptr(num), _ptr(den), _ptr(cl), _ptr(er))
    if rc != 0:
        raise MemoryError("oracle_stats allocation failed")
    return dict(numerators=num, denominators=den, cand_lens=cl, eff_ref_lens=er)


def normalized_weights(max_order: int, weights=None) -> np.ndarray:
    """BleuConfig weight normalisation (bleu.py:45-56)."""
    if weights is None:
        return np.full(max_order, 1.0 / max_order)
    w = np.asarray(weights, dtype=np.float64)
    return w / w.sum()


def scores(st: dict, smoothing: str = "none", eps: float = 0.1, k: float = 1.0,
           weights=None) -> dict:
    """score_sentences_from_stats (bleu.py:274-279)."""
    num = np.ascontiguousarray(st["numerators"], dtype=np.int64)
    den = np.ascontiguousarray(st["denominators"], dtype=np.int64)
    cl = np.ascontiguousarray(st["cand_lens"], dtype=np.int64)
    er = np.ascontiguousarray(st["eff_ref_lens"], dtype=np.int64)
    b, n = num.shape
    w = np.ascontiguousarray(normalized_weights(n, weights))
    sc = np.zeros(b, dtype=np.float64)
    pr = np.zeros((b, n), dtype=np.float64)
    bp = np.zeros(b, dtype=np.float64)
    if b:
        lib().oracle_scores(_ptr(num), _ptr(den), _ptr(cl), _ptr(er), b, n,
                            SMOOTHING_CODES[smoothing], eps, k, _ptr(w),
                            _ptr(sc), _ptr(pr), _ptr(bp))
    return dict(scores=sc, precisions=pr, brevity_penalty=bp)


def totals(st: dict) -> np.ndarray:
    """The int64 [Σnum_n | Σden_n | Σc | Σr] vector of score_corpus_from_stats."""
    num = np.ascontiguousarray(st["numerators"], dtype=np.int64)
    den = np.ascontiguousarray(st["denominators"], dtype=np.int64)
    cl = np.ascontiguousarray(st["cand_lens"], dtype=np.int64)
    er = np.ascontiguousarray(st["eff_ref_lens"], dtype=np.int64)
    b, n = num.shape
    out = np.zeros(2 * n + 2, dtype=np.int64)
    lib().oracle_totals(_ptr(num), _ptr(den), _ptr(cl), _ptr(er), b, n, _ptr(out))
    return out


def corpus(st: dict, smoothing: str = "none", eps: float = 0.1, k: float = 1.0,
           weights=None) -> dict:
    """score_corpus_from_stats (bleu.py:293-305)."""
    t = totals(st)
    n = st["numerators"].shape[1]
    agg = dict(numerators=t[None, :n], denominators=t[None, n:2 * n],
               cand_lens=t[2 * n:2 * n + 1], eff_ref_lens=t[2 * n + 1:2 * n + 2])
    r = scores(agg, smoothing, eps, k, weights)
    return dict(scores=float(r["scores"][0]), precisions=r["precisions"][0],
                brevity_penalty=float(r["brevity_penalty"][0]), totals=t)


def segment_bincount(ids, seg_lengths, num_unique: int) -> np.ndarray:
    """_kernels.pyx:84-126."""
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    seg = np.ascontiguousarray(seg_lengths, dtype=np.int64)
    b, u = len(seg), int(num_unique)
    out = np.zeros((b, u), dtype=np.int32)
    if b * u == 0:
        return out
    if lib().oracle_segment_bincount(_ptr(ids), _ptr(seg), b, u, _ptr(out)) != 0:
        raise ValueError(f"compact ID out of range [0, {u})")
    return out


def clipped_numerators(ids, seg_lengths, ref_max) -> np.ndarray:
    """_kernels.pyx:129-180."""
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    seg = np.ascontiguousarray(seg_lengths, dtype=np.int64)
    rm = np.ascontiguousarray(ref_max, dtype=np.int32)
    b, u = rm.shape
    out = np.zeros(b, dtype=np.int64)
    if b == 0:
        return out
    rc = lib().oracle_clipped_numerators(_ptr(ids), _ptr(seg), b, _ptr(rm), u, _ptr(out))
    if rc == -1:
        raise ValueError(f"compact ID out of range [0, {u})")
    return out


# ---------------------------------------------------------------------------
# Pure-Python restatement of pkg/src/batchbleu/oracle.py (small cases only).
# ---------------------------------------------------------------------------
def py_ngram_counts(sentence: Sequence[int], n: int) -> Counter:
    """oracle.py:18-22."""
    return Counter(tuple(sentence[i:i + n]) for i in range(len(sentence) - n + 1))


def _py_clipped(candidate, references, n):
    """oracle.py:29-39."""
    cand_counts = py_ngram_counts(candidate, n)
    max_ref: Counter = Counter()
    for ref in references:
        for gram, count in py_ngram_counts(ref, n).items():
            if count > max_ref[gram]:
                max_ref[gram] = count
    num = sum(min(c, max_ref[g]) for g, c in cand_counts.items())
    return num, max(len(candidate) - n + 1, 0)


def _py_smooth(nums, dens, smoothing, eps, k):
    """oracle.py:42-60."""
    out, counter = [], 1
    for n, (num, den) in enumerate(zip(nums, dens), start=1):
        if den == 0:
            out.append(0.0)
        elif smoothing == "add-k" and n >= 2:
            out.append((num + k) / (den + k))
        elif num > 0:
            out.append(num / den)
        elif smoothing == "floor":
            out.append(eps / den)
        elif smoothing == "exp":
            out.append(1.0 / (2 ** counter * den))
            counter += 1
        else:
            out.append(0.0)
    return out


def _py_finish(precisions, c, r, weights):
    """oracle.py:63-75."""
    if c == 0:
        return 0.0
    bp = 1.0 if c > r else math.exp(1.0 - r / c)
    s = 0.0
    for w, p in zip(weights, precisions):
        if w == 0.0:
            continue
        if p <= 0.0:
            return 0.0
        s += w * math.log(p)
    return min(bp * math.exp(s), 1.0)


def py_sentence_bleu(candidate, references, max_order=4, smoothing="none", eps=0.1,
                     k=1.0, weights=None) -> float:
    """oracle.py:78-92."""
    w = normalized_weights(max_order, weights)
    nums, dens = zip(*[_py_clipped(candidate, references, n) for n in range(1, max_order + 1)])
    eff = min((len(r) for r in references), key=lambda x: (abs(x - len(candidate)), x))
    return _py_finish(_py_smooth(nums, dens, smoothing, eps, k), len(candidate), eff, w)


def py_corpus_bleu(candidates, references, max_order=4, smoothing="none", eps=0.1,
                   k=1.0, weights=None) -> float:
    """oracle.py:95-118; ``references[r][i]`` is reference r of sentence i."""
    w = normalized_weights(max_order, weights)
    nums, dens = [0] * max_order, [0] * max_order
    c_tot = r_tot = 0
    for i, cand in enumerate(candidates):
        refs_i = [refs[i] for refs in references]
        for n in range(1, max_order + 1):
            a, b = _py_clipped(cand, refs_i, n)
            nums[n - 1] += a
            dens[n - 1] += b
        c_tot += len(cand)
        r_tot += min((len(r) for r in refs_i), key=lambda x: (abs(x - len(cand)), x))
    return _py_finish(_py_smooth(nums, dens, smoothing, eps, k), c_tot, r_tot, w)


def reference_package():
    """Import the UNMODIFIED reference package built into oracle/_ref, or None."""
    import sys
    if not os.path.isdir(os.path.join(REF_DIR, "batchbleu")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import batchbleu  # noqa: F401
    return batchbleu
