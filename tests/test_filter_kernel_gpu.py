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
