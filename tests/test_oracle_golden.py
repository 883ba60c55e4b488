"""Pin the CPU oracle (oracle/) against the reference's own outputs.

CPU-only: this is what makes the oracle trustworthy as the parity checker for
the GPU tests.  Fixtures come from tests/golden/make_golden.py (the
unmodified reference package)."""

import numpy as np
import pytest

import oracle
from conftest import load_acceptance_cases, load_batch_fixtures, load_frozen_cases, load_ngram_ops

BATCH_FIXTURES = load_batch_fixtures()


@pytest.mark.parametrize("name,inputs,cfgs", BATCH_FIXTURES, ids=[f[0] for f in BATCH_FIXTURES])
def test_oracle_matches_reference_fixture(name, inputs, cfgs):
    for cfg, ref in cfgs:
        st = oracle.stats(inputs["cand_ids"], inputs["cand_len"], inputs["refs"], cfg["max_order"])
        # counts: bit-exact
        np.testing.assert_array_equal(st["numerators"], ref["numerators"])
        np.testing.assert_array_equal(st["denominators"], ref["denominators"])
        np.testing.assert_array_equal(st["cand_lens"], ref["cand_lens"])
        np.testing.assert_array_equal(st["eff_ref_lens"], ref["eff_ref_lens"])
        sc = oracle.scores(st, cfg["smoothing"], cfg["eps"], cfg["k"], cfg["weights"])
        # fp64 epilogue: same operation order; libm vs numpy exp/log differ by <= 1 ulp
        np.testing.assert_allclose(sc["scores"], ref["scores"], rtol=1e-14, atol=0)
        np.testing.assert_array_equal(sc["scores"] == 0, ref["scores"] == 0)
        np.testing.assert_allclose(sc["precisions"], ref["precisions"], rtol=1e-15, atol=0)
        np.testing.assert_allclose(sc["brevity_penalty"], ref["brevity_penalty"], rtol=1e-14, atol=0)
        co = oracle.corpus(st, cfg["smoothing"], cfg["eps"], cfg["k"], cfg["weights"])
        assert co["scores"] == pytest.approx(float(ref["corpus_score"]), rel=1e-14, abs=0)
        np.testing.assert_allclose(co["precisions"], ref["corpus_precisions"], rtol=1e-15, atol=0)


def test_oracle_matches_reference_acceptance_cases():
    for case in load_acceptance_cases():
        refs = [(np.array(r["ids"]), np.array(r["len"])) for r in case["refs"]]
        st = oracle.stats(np.array(case["cand_ids"]), np.array(case["cand_len"]), refs, case["max_order"])
        np.testing.assert_array_equal(st["numerators"], np.array(case["numerators"]).reshape(st["numerators"].shape))
        np.testing.assert_array_equal(st["eff_ref_lens"], case["eff_ref_lens"])
        sc = oracle.scores(st, case["smoothing"])
        np.testing.assert_allclose(sc["scores"], case["scores"], rtol=1e-14, atol=0)
        co = oracle.corpus(st, case["smoothing"])
        assert co["scores"] == pytest.approx(case["corpus_score"], rel=1e-14, abs=0)


@pytest.mark.parametrize("case", load_frozen_cases(), ids=lambda c: c["smoothing"])
def test_oracle_frozen_external_vectors(case):
    """pkg/tests/test_oracle.py:178-185 — oracle at 1e-9."""
    assert oracle.py_corpus_bleu(case["cands"], case["refsets"], smoothing=case["smoothing"]) == \
        pytest.approx(case["expected"], abs=1e-9)
    cands = case["cands"]
    w = max(len(c) for c in cands)
    ids = np.array([c + [0] * (w - len(c)) for c in cands])
    refs = []
    for rs in case["refsets"]:
        rw = max(len(r) for r in rs)
        refs.append((np.array([r + [0] * (rw - len(r)) for r in rs]), np.array([len(r) for r in rs])))
    st = oracle.stats(ids, np.array([len(c) for c in cands]), refs)
    assert oracle.corpus(st, case["smoothing"])["scores"] == pytest.approx(case["expected"], abs=1e-9)


def test_py_restatement_matches_c_restatement(rng):
    from conftest import random_instance
    for trial in range(60):
        (cid, clen), refs = random_instance(rng)
        sm = ["none", "floor", "add-k", "exp"][trial % 4]
        st = oracle.stats(cid, clen, refs)
        sc = oracle.scores(st, sm)["scores"]
        py = [oracle.py_sentence_bleu(cid[i, :clen[i]].tolist(), [r[0][i, :r[1][i]].tolist() for r in refs],
                                      smoothing=sm) for i in range(len(clen))]
        np.testing.assert_allclose(sc, py, atol=1e-12)


def test_oracle_segment_ops_match_reference():
    for op in load_ngram_ops():
        got = oracle.segment_bincount(np.array(op["flat"], dtype=np.int64), np.array(op["seg"]), op["u"])
        np.testing.assert_array_equal(got, np.array(op["counts"]).reshape(got.shape))
        got = oracle.clipped_numerators(np.array(op["flat"], dtype=np.int64), np.array(op["seg"]),
                                        np.array(op["ref_max"], dtype=np.int32).reshape(len(op["seg"]), -1))
        np.testing.assert_array_equal(got, op["clipped"])


def test_oracle_segment_range_error():
    with pytest.raises(ValueError):
        oracle.segment_bincount(np.array([0, 3]), np.array([2]), 3)
