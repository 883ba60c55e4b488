"""The filter kernel (tb_kernel_sparse.cu) and the hash-table kernels behind
its dense-group list, forced onto every shape: the library picks the filter
kernel only where it is faster (long rows in many waves), so the parity suites
run again in a child process with TB_FORCE_SPARSE=1 (every group goes through
the filter kernel first; related-text groups through the list handoff), and
the full-size suite with TB_NO_SPARSE=1 (the hash-table kernel alone at c5)."""

import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _run(env_extra, files):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider", *files],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_parity_suites_through_the_filter_kernel():
    _run({"TB_FORCE_SPARSE": "1"}, ["tests/test_parity_gpu.py", "tests/test_fullsize_gpu.py",
                                    "tests/test_host_path_gpu.py", "tests/test_plan_gpu.py"])


def test_fullsize_through_the_hash_table_kernel_alone():
    _run({"TB_NO_SPARSE": "1"}, ["tests/test_fullsize_gpu.py"])


def test_shapes_of_growing_then_shrinking_shared_memory():
    """Launch shapes whose shared-memory needs go up and down in one process
    (each kernel's dynamic shared-memory opt-in must never shrink)."""
    _run({"TB_FORCE_SPARSE": "1"}, ["tests/test_filter_kernel_gpu.py::test_mixed_shapes_child"])


def test_mixed_shapes_child():
    import numpy as np
    import torch

    import oracle
    import paper_2510_05485_b200 as tb
    rng = np.random.default_rng(0)
    for b, w, r in [(1100, 1, 3), (100, 900, 3), (100, 1, 3), (64, 2000, 1), (8, 1, 1), (64, 2000, 1)]:
        cid, cl = rng.integers(0, 3, (b, w)), rng.integers(0, w + 1, b)
        refs = [(rng.integers(0, 3, (b, w)), rng.integers(0, w + 1, b)) for _ in range(r)]
        for pin in (True, False):
            mk = ((lambda i, ln: tb.TokenBatch(ids=torch.as_tensor(i).pin_memory(), lengths=torch.as_tensor(ln)))
                  if pin else (lambda i, ln: tb.TokenBatch(ids=torch.as_tensor(i).cuda(),
                                                           lengths=torch.as_tensor(ln).cuda())))
            st = tb.compute_stats(mk(cid, cl), [mk(i, ln) for i, ln in refs], tb.BleuConfig())
            num = st.numerators.cpu().numpy() if hasattr(st.numerators, "cpu") else st.numerators
            np.testing.assert_array_equal(num, oracle.stats(cid, cl, refs)["numerators"])
