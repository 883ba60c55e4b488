import glob
import gzip
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests proper")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def random_instance(rng, max_b=8, max_len=32, max_vocab=16, max_refs=3):
    """(cand_ids, cand_len, [(ref_ids, ref_len)]) with ragged lengths —
    the reference's generator (pkg/tests/conftest.py:7-21)."""
    b = int(rng.integers(1, max_b + 1))
    l = int(rng.integers(1, max_len + 1))
    v = int(rng.integers(1, max_vocab + 1))
    r = int(rng.integers(1, max_refs + 1))

    def mk():
        return rng.integers(0, v, size=(b, l)), rng.integers(0, l + 1, size=b)

    return mk(), [mk() for _ in range(r)]


def load_batch_fixtures():
    """[(name, inputs, [(config dict, reference outputs dict)])]"""
    out = []
    for path in sorted(glob.glob(os.path.join(GOLDEN, "*.npz"))):
        z = np.load(path)
        meta = json.loads(bytes(z["meta"]).decode())
        R = int(z["num_refs"])
        inputs = dict(cand_ids=z["cand_ids"], cand_len=z["cand_len"],
                      refs=[(z[f"ref{r}_ids"], z[f"ref{r}_len"]) for r in range(R)])
        cfgs = []
        for i, c in enumerate(meta["configs"]):
            outs = {k[len(f"c{i}_"):]: z[k] for k in z.files if k.startswith(f"c{i}_")}
            cfgs.append((c, outs))
        out.append((os.path.basename(path)[:-4], inputs, cfgs))
    return out


def load_acceptance_cases():
    with gzip.open(os.path.join(GOLDEN, "acceptance_160.json.gz"), "rt") as fh:
        return json.load(fh)


def load_frozen_cases():
    with open(os.path.join(GOLDEN, "frozen_corpus_cases.json")) as fh:
        return json.load(fh)["cases"]


def load_ngram_ops():
    with gzip.open(os.path.join(GOLDEN, "ngram_ops_40.json.gz"), "rt") as fh:
        return json.load(fh)
