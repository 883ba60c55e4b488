"""CPU-only tests: the C-ABI library loads and exports every symbol the
header declares, and the host-side logic (config, batch validation, scalar
helpers, buffer-API argument errors) mirrors the reference.

No kernel is launched here; the device paths are covered by the `-m gpu`
parity tests.
"""

import math
import os
import re

import numpy as np
import pytest

from conftest import ROOT

import paper_2510_05485_b200 as tb
from paper_2510_05485_b200 import _native, ext

HEADER = os.path.join(ROOT, "include", "tensorbleu.h")


def _declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tb_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_abi():
    syms = _declared_symbols()
    for name in ("tb_bleu_stats", "tb_bleu_scores", "tb_bleu_totals", "tb_unique_rows",
                 "tb_segment_bincount", "tb_clipped_numerators", "tb_strerror"):
        assert name in syms


def test_library_loads_and_exports_every_declared_symbol():
    lib = _native.load()
    missing = [s for s in _declared_symbols() if not hasattr(lib, s)]
    assert not missing, f"symbols declared in include/tensorbleu.h but not exported: {missing}"
    # and every binding in _native names a declared symbol (no stale signatures)
    assert set(_native.SIGNATURES) <= set(_declared_symbols())


def test_library_is_sm100a_and_has_no_host_fallback():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_error_strings_and_host_argument_errors():
    lib = _native.load()
    assert lib.tb_version().decode().startswith("tensorbleu-b200")
    for code in range(6):
        assert lib.tb_strerror(code)
    # argument checks that fail before any device work (no GPU needed)
    rc = lib.tb_bleu_stats(3, None, 0, 0, None, 1, None, None, None, None, 0, 4, 0, 0.1, 1.0,
                           None, None, None, None, None, None, None, None, None, None, None,
                           None, 0, None)
    assert rc == _native.TB_ERR_INVALID_ARG
    assert lib.tb_bleu_workspace_bytes(4, 0, 8, None, 4, 4) == 0  # R = 0 is invalid


def test_native_check_maps_error_types():
    with pytest.raises(ValueError):
        _native.check(_native.TB_ERR_INVALID_ARG, "x")
    with pytest.raises(tb.CapacityError):
        _native.check(_native.TB_ERR_CAPACITY, "x")
    with pytest.raises(RuntimeError):
        _native.check(_native.TB_ERR_WORKSPACE, "x")
    with pytest.raises(ValueError, match="lengths"):
        _native.raise_flags(_native.TB_FLAG_BAD_LENGTH)
    with pytest.raises(ValueError, match="non-negative"):
        _native.raise_flags(_native.TB_FLAG_NEGATIVE_ID)


def test_no_cpu_fallback_without_a_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    cand = tb.TokenBatch.from_lists([[1, 2, 3]])
    with pytest.raises(RuntimeError, match="CUDA"):
        tb.sentence_bleu(cand, [cand])


# --- BleuConfig (reference tests/test_bleu.py:26-44) -------------------------
def test_config_defaults_and_normalisation():
    cfg = tb.BleuConfig()
    assert cfg.max_order == 4 and cfg.weights == (0.25, 0.25, 0.25, 0.25)
    assert tb.BleuConfig(max_order=2, weights=[2.0, 2.0]).weights == (0.5, 0.5)
    assert tb.BleuConfig(max_order=3, weights=[1.0, 0.0, 3.0]).weights == (0.25, 0.0, 0.75)


@pytest.mark.parametrize("kw", [dict(max_order=0), dict(smoothing="bogus"), dict(eps=0.0),
                                dict(k=0.0), dict(max_order=2, weights=[1.0, 2.0, 3.0]),
                                dict(max_order=2, weights=[-1.0, 2.0]),
                                dict(max_order=2, weights=[0.0, 0.0])])
def test_config_rejects_bad_values(kw):
    with pytest.raises(ValueError):
        tb.BleuConfig(**kw)


def test_config_matches_reference_package():
    import oracle
    bb = oracle.reference_package()
    if bb is None:
        pytest.skip("reference package not built")
    for kw in (dict(), dict(max_order=2, weights=[2.0, 2.0]), dict(max_order=3, weights=[0.1, 0.2, 0.7]),
               dict(smoothing="exp"), dict(smoothing="add-k", k=2.5)):
        assert tb.BleuConfig(**kw) == tb.BleuConfig(**kw)
        assert tb.BleuConfig(**kw).weights == bb.BleuConfig(**kw).weights


# --- scalar helpers (reference tests/test_bleu.py:47-73) ----------------------
def test_effective_ref_len():
    assert tb.effective_ref_len(7, [5, 9]) == 5
    assert tb.effective_ref_len(7, [8]) == 8
    assert tb.effective_ref_len(10, [7, 12, 20]) == 12
    with pytest.raises(ValueError):
        tb.effective_ref_len(3, [])


def test_brevity_penalty():
    assert tb.brevity_penalty(10, 10) == 1.0
    assert tb.brevity_penalty(5, 10) == pytest.approx(math.exp(-1.0))
    assert tb.brevity_penalty(12, 10) == 1.0
    assert tb.brevity_penalty(0, 10) == 0.0


# --- TokenBatch host validation (reference batch.py:22-37, test_ngrams.py:164-170)
def test_token_batch_validation():
    tb.TokenBatch(ids=np.array([[1, 2, -5]]), lengths=np.array([2]))  # negative padding is fine
    with pytest.raises(ValueError):
        tb.TokenBatch(ids=np.array([[1, -2, 3]]), lengths=np.array([2]))
    with pytest.raises(ValueError):
        tb.TokenBatch(ids=np.array([[1, 2]]), lengths=np.array([3]))
    with pytest.raises(ValueError):
        tb.TokenBatch(ids=np.array([1, 2]), lengths=np.array([2]))
    with pytest.raises(ValueError):
        tb.TokenBatch(ids=np.zeros((2, 3)), lengths=np.array([1]))


def test_token_batch_from_lists_and_rows():
    b = tb.TokenBatch.from_lists([[1, 2, 3], [], [4]], pad_value=-1, min_width=5)
    assert b.ids.shape == (3, 5) and b.ids.dtype == np.int64
    assert b.rows() == [[1, 2, 3], [], [4]]
    assert b.ids[1, 0] == -1


def test_token_batch_host_torch_tensors():
    import torch
    b = tb.TokenBatch(ids=torch.tensor([[1, 2, 0]], dtype=torch.int32), lengths=torch.tensor([2]))
    assert b.ids.dtype == torch.int32 and not b.is_device
    with pytest.raises(ValueError):
        tb.TokenBatch(ids=torch.tensor([[1, -2, 0]]), lengths=torch.tensor([2]))


# --- buffer API argument errors (reference bindings/tests/test_bindings.py:101-117)
def test_buffer_api_errors_name_the_dimension():
    cand = np.zeros((4, 8), dtype=np.int64)
    clens = np.zeros(4, dtype=np.int64)
    refs = np.zeros((1, 3, 8), dtype=np.int64)
    rlens = np.zeros((1, 3), dtype=np.int64)
    with pytest.raises(ValueError, match="references dimension 1 is 3, expected 4"):
        ext.score_sentences(cand, clens, refs, rlens)
    with pytest.raises(ValueError, match="cand_lengths dimension 0 is 3, expected 4"):
        ext.score_sentences(cand, np.zeros(3, dtype=np.int64), np.zeros((1, 4, 8), dtype=np.int64),
                            np.zeros((1, 4), dtype=np.int64))
    with pytest.raises(ValueError, match="candidates must have 2 dimensions"):
        ext.score_sentences(np.zeros(8, dtype=np.int64), clens, refs, rlens)
    with pytest.raises(TypeError, match="candidates must be int32 or int64"):
        ext.score_sentences(cand.astype(np.float64), clens, np.zeros((1, 4, 8), dtype=np.int64),
                            np.zeros((1, 4), dtype=np.int64))


def test_buffer_api_empty_batch_needs_no_device():
    out = ext.score_sentences(np.zeros((0, 4), dtype=np.int64), np.zeros(0, dtype=np.int64),
                              np.zeros((1, 0, 4), dtype=np.int64), np.zeros((1, 0), dtype=np.int64))
    assert out.shape == (0,) and out.dtype == np.float64


# --- the native host-path binding (_hostpath): argument checks before any device call
def test_hostpath_binding_loads_and_checks_arguments():
    hp = _native.hostpath()
    good = (0, 4, 4, 0, 8)
    with pytest.raises(TypeError):
        hp.run(1, (good,))                                    # wrong arity
    with pytest.raises(ValueError):
        hp.run(1, (good,), 1, 4, 0, 0.1, 1.0, 0, 0)          # no reference view
    with pytest.raises(TypeError):
        hp.run(1, (good, (0, 4)), 1, 4, 0, 0.1, 1.0, 0, 0)  # malformed view
    with pytest.raises(ValueError):
        hp.run(1, (good, good), -1, 4, 0, 0.1, 1.0, 0, 0)   # negative batch
    with pytest.raises(ValueError):
        hp.run(1, (good, good), 1, 0, 0, 0.1, 1.0, 0, 0)    # max_order 0
    with pytest.raises(ValueError):
        hp.run(1, (good, (0, 4, 4, 0, 4)), 1, 4, 0, 0.1, 1.0, 0, 0)  # mixed token widths
    with pytest.raises(ValueError):
        hp.launch((good,), 1, 4, 0, 0.1, 1.0, 0, (None,) * 9, 0, 0, 0, 0)


def test_row_views_are_cached_and_widened_once():
    b = tb.TokenBatch(ids=np.arange(12, dtype=np.int64).reshape(3, 4), lengths=np.array([4, 2, 0]))
    v1, keep = b._row_view(True)
    assert v1[1:3] == (4, 4) and v1[4] == 8 and b._row_view(True)[0] is v1
    import torch
    b32 = tb.TokenBatch(ids=torch.arange(12, dtype=torch.int32).reshape(3, 4), lengths=torch.tensor([4, 2, 0]))
    assert b32._row_view(False)[0][4] == 4
    w = b32._row_view(True)
    assert w[0][4] == 8 and w[1][0].dtype == torch.int64  # widened copy kept alive with the view
