"""bench.py under torchrun with 2 ranks sharing the one GPU (gloo; testing
mode TB_BENCH_SHARED_GPU=1): weak scaling (c2, each rank its own batch) and
strong scaling (c4: one global corpus split over the ranks, the int64 totals
all-reduced inside the timed region) both print a verified JSON line with the
whole job's global batch."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("workload,scaling,global_batch", [("c2", "weak", 1024), ("c4", "strong", 4096)])
def test_two_rank_bench_line(workload, scaling, global_batch):
    env = dict(os.environ, TB_BENCH_SHARED_GPU="1")
    port = str(29600 + (os.getpid() % 200))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", port, "bench.py", "--gpus", "2",
                        "--workload", workload, "--steps", "5", "--warmup", "3", "--no-configs",
                        "--no-cpu-baseline", "--clock-window", "0"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = lines[0]
    assert d["n_gpus"] == 2 and d["scaling"] == scaling and d["config"]["global_batch"] == global_batch
    assert d["verified"] is True and d["value"] > 0
