"""Generate the golden fixtures under tests/golden/ from the UNMODIFIED
reference package.

Run in the build container (where /root/reference exists):

    oracle/build_ref.sh                      # builds batchbleu into oracle/_ref
    python tests/golden/make_golden.py

Every fixture stores the inputs and the reference's own outputs
(batchbleu.compute_stats / sentence_bleu / corpus_bleu with the compiled
backend, and the spec-level dictionary/bincount ops).  The reference's frozen
external corpus vectors (pkg/tests/test_oracle.py:78-175) are extracted by
importing that test module, not retyped.

The GPU box never runs this script; it only reads the committed fixtures.
"""

from __future__ import annotations

import gzip
import importlib.util
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

bb = oracle.reference_package()
if bb is None:
    raise SystemExit("oracle/_ref is not built; run oracle/build_ref.sh first")
from batchbleu.bench import BenchConfig, generate_batch  # noqa: E402

SMOOTHINGS = ("none", "floor", "add-k", "exp")


def ref_outputs(cand, refs, cfg):
    st = bb.compute_stats(cand, refs, cfg)
    sres = bb.sentence_bleu(cand, refs, cfg)
    cres = bb.corpus_bleu(cand, refs, cfg)
    return dict(
        numerators=st.numerators, denominators=st.denominators,
        cand_lens=st.cand_lens, eff_ref_lens=st.eff_ref_lens,
        scores=sres.scores, precisions=sres.precisions, brevity_penalty=sres.brevity_penalty,
        corpus_score=np.float64(cres.scores), corpus_precisions=cres.precisions,
        corpus_bp=np.float64(cres.brevity_penalty),
    )


def save_batch_fixture(name, cand, refs, configs, note):
    """npz: inputs + per-config reference outputs (prefix c{i}_)."""
    arrs = dict(cand_ids=cand.ids.astype(np.int64), cand_len=cand.lengths,
                num_refs=np.int64(len(refs)))
    for r, ref in enumerate(refs):
        arrs[f"ref{r}_ids"] = ref.ids.astype(np.int64)
        arrs[f"ref{r}_len"] = ref.lengths
    meta = []
    for i, cfg in enumerate(configs):
        out = ref_outputs(cand, refs, cfg)
        for k, v in out.items():
            arrs[f"c{i}_{k}"] = v
        meta.append(dict(max_order=cfg.max_order, weights=list(cfg.weights),
                         smoothing=cfg.smoothing, eps=cfg.eps, k=cfg.k))
    arrs["meta"] = np.frombuffer(json.dumps(dict(note=note, configs=meta)).encode(), dtype=np.uint8)
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **arrs)
    print(f"{path}: {os.path.getsize(path)} bytes")


def correlated(rng, b, l, v, r, p_max=0.9):
    """References = candidate with per-row mutation rate p ~ U[0, p_max] and
    length = candidate length ± 50."""
    ids = rng.integers(0, v, size=(b, l))
    lens = rng.integers(l // 2, l + 1, size=b)
    cand = bb.TokenBatch(ids=ids, lengths=lens)
    refs = []
    for _ in range(r):
        rid = ids.copy()
        p = rng.random(b)[:, None] * p_max
        mut = rng.random(ids.shape) < p
        rid[mut] = rng.integers(0, v, size=int(mut.sum()))
        rl = np.clip(lens + rng.integers(-50, 51, size=b), 0, l)
        refs.append(bb.TokenBatch(ids=rid, lengths=rl))
    return cand, refs


def main():
    all_cfgs = [bb.BleuConfig(smoothing=s) for s in SMOOTHINGS]

    # c1: the reference's CPU-runnable headline config (BASELINE.json configs[0])
    cand, refs = generate_batch(BenchConfig(vocab_size=32000, num_references=1), 42, 16, 256)
    save_batch_fixture("c1_16x256_v32k_r1", cand, refs, [bb.BleuConfig(smoothing="floor")] + all_cfgs,
                       "generate_batch(seed=42, B=16, L=256, V=32000, R=1)")

    rng = np.random.default_rng(20251007)
    cand, refs = correlated(rng, 64, 128, 500, 2)
    save_batch_fixture("correlated_64x128_r2", cand, refs,
                       all_cfgs + [bb.BleuConfig(max_order=2, weights=(0.7, 0.3), smoothing="add-k", k=2.5),
                                   bb.BleuConfig(max_order=6, smoothing="exp")],
                       "correlated references, V=500")

    # c3-like: 4 references, add-k and exp, variable widths per reference
    cand, refs = correlated(rng, 8, 1024, 128000, 4, p_max=0.6)
    refs = [bb.TokenBatch(ids=r.ids[:, : 1024 - 100 * i], lengths=np.minimum(r.lengths, 1024 - 100 * i))
            for i, r in enumerate(refs)]
    save_batch_fixture("multiref_8x1024_r4", cand, refs,
                       [bb.BleuConfig(smoothing="add-k"), bb.BleuConfig(smoothing="exp")],
                       "4 correlated references of widths 1024/924/824/724, V=128000")

    # Zipf(1.1) tokens: hot keys
    z = lambda size: np.minimum(rng.zipf(1.1, size=size) - 1, 127999)  # noqa: E731
    b, l = 32, 256
    cand = bb.TokenBatch(ids=z((b, l)), lengths=rng.integers(l // 2, l + 1, size=b))
    refs = [bb.TokenBatch(ids=z((b, l)), lengths=rng.integers(l // 2, l + 1, size=b)) for _ in range(2)]
    save_batch_fixture("zipf_32x256_r2", cand, refs, all_cfgs, "Zipf(1.1) tokens capped at 128k")

    # vocab = 1: every n-gram identical
    b, l = 8, 64
    cand = bb.TokenBatch(ids=np.zeros((b, l), dtype=np.int64), lengths=rng.integers(0, l + 1, size=b))
    refs = [bb.TokenBatch(ids=np.zeros((b, l), dtype=np.int64), lengths=rng.integers(0, l + 1, size=b))
            for _ in range(3)]
    save_batch_fixture("vocab1_8x64_r3", cand, refs, all_cfgs, "vocab = 1")

    # huge token IDs (beyond int32) and negative padding
    b, l = 8, 40
    ids = rng.integers(2**40, 2**40 + 6, size=(b, l))
    lens = rng.integers(0, l + 1, size=b)
    pad = np.arange(l) >= lens[:, None]
    ids[pad] = -7
    cand = bb.TokenBatch(ids=ids, lengths=lens)
    rids = rng.integers(2**40, 2**40 + 6, size=(b, l))
    refs = [bb.TokenBatch(ids=rids, lengths=rng.integers(0, l + 1, size=b))]
    save_batch_fixture("bigids_8x40_r1", cand, refs, all_cfgs, "token IDs around 2**40, padding -7")

    # acceptance-generator instances (test_acceptance.py:36-69), JSON
    rng = np.random.default_rng(20260823)
    cases = []
    for trial in range(160):
        b = int(rng.integers(1, 9))
        l = int(rng.integers(1, 33))
        v = int(rng.integers(1, 17))
        r = int(rng.integers(1, 4))
        cfg = bb.BleuConfig(max_order=int(rng.choice([1, 2, 4])), smoothing=SMOOTHINGS[trial % 4])

        def mk():
            return bb.TokenBatch(ids=rng.integers(0, v, size=(b, l)), lengths=rng.integers(0, l + 1, size=b))

        cand, refs = mk(), [mk() for _ in range(r)]
        out = ref_outputs(cand, refs, cfg)
        cases.append(dict(
            max_order=cfg.max_order, smoothing=cfg.smoothing,
            cand_ids=cand.ids.tolist(), cand_len=cand.lengths.tolist(),
            refs=[dict(ids=x.ids.tolist(), len=x.lengths.tolist()) for x in refs],
            **{k: (np.asarray(val).tolist()) for k, val in out.items()}))
    path = os.path.join(HERE, "acceptance_160.json.gz")
    with gzip.open(path, "wt") as fh:
        json.dump(cases, fh)
    print(f"{path}: {os.path.getsize(path)} bytes")

    # the reference's frozen external vectors, extracted from its own test module
    spec = importlib.util.spec_from_file_location(
        "ref_test_oracle", "/root/reference/pkg/tests/test_oracle.py")
    mod = importlib.util.module_from_spec(spec)
    sys.path.insert(0, "/root/reference/pkg/tests")
    spec.loader.exec_module(mod)
    frozen = [dict(smoothing=s, cands=c, refsets=r, expected=e) for s, c, r, e in mod.FROZEN_CORPUS_CASES]
    path = os.path.join(HERE, "frozen_corpus_cases.json")
    with open(path, "w") as fh:
        json.dump(dict(source="pkg/tests/test_oracle.py:78-175 (FROZEN_CORPUS_CASES)", cases=frozen), fh)
    print(f"{path}: {len(frozen)} cases")

    # spec-level operators: dictionary + offset bincount + clipped numerators
    rng = np.random.default_rng(7)
    ops = []
    for _ in range(40):
        b = int(rng.integers(1, 10))
        n = int(rng.integers(1, 4))
        l = int(rng.integers(1, 20))
        v = int(rng.integers(1, 10))

        def mk():
            return bb.extract_ngrams(bb.TokenBatch(ids=rng.integers(0, v, size=(b, l)),
                                                   lengths=rng.integers(0, l + 1, size=b)), n)

        cs, rs = mk(), [mk() for _ in range(int(rng.integers(1, 3)))]
        d = bb.build_dictionary(cs, rs)
        u = d.num_unique
        ids = [rng.integers(0, max(u, 1), size=rng.integers(0, 30)) for _ in range(b)]
        seg = np.array([len(s) for s in ids], dtype=np.int64)
        flat = np.concatenate(ids).astype(np.int64) if seg.sum() else np.empty(0, dtype=np.int64)
        counts = bb._backend.segment_bincount(flat, seg, max(u, 1))
        ref_max = rng.integers(0, 3, size=(b, max(u, 1))).astype(np.int32)
        clipped = bb._backend.clipped_numerators(flat, seg, ref_max)
        rows = np.concatenate([bb.ngrams.flatten_valid(cs)] + [bb.ngrams.flatten_valid(x) for x in rs])
        ops.append(dict(rows=rows.tolist(), n=n, unique=d.unique_ngrams.tolist(),
                        inverse=d.inverse_indices.tolist(), u=max(u, 1), flat=flat.tolist(),
                        seg=seg.tolist(), counts=counts.tolist(), ref_max=ref_max.tolist(),
                        clipped=clipped.tolist()))
    path = os.path.join(HERE, "ngram_ops_40.json.gz")
    with gzip.open(path, "wt") as fh:
        json.dump(ops, fh)
    print(f"{path}: {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
