"""The batchbleu-bench-compatible CLI (tools/batchbleu_bench.py): its serial
baseline restates the reference oracle exactly, and the GPU run keeps the
reference CLI's CSV layout, equivalence gate and exit codes
(pkg/tests/test_bench.py:49-120)."""

import os
import sys

import numpy as np
import pytest

from conftest import ROOT, random_instance

sys.path.insert(0, os.path.join(ROOT, "tools"))
import batchbleu_bench as cli  # noqa: E402
import oracle  # noqa: E402


@pytest.mark.parametrize("smoothing", ["none", "floor", "add-k", "exp"])
def test_serial_baseline_matches_oracle(rng, smoothing):
    for _ in range(40):
        (cid, clen), refs = random_instance(rng)
        for i in range(cid.shape[0]):
            c = cid[i, :clen[i]].tolist()
            rs = [ri[i, :rl[i]].tolist() for ri, rl in refs]
            assert cli.serial_sentence_bleu(c, rs, smoothing=smoothing) == pytest.approx(
                oracle.py_sentence_bleu(c, rs, smoothing=smoothing), rel=1e-12, abs=1e-15)


def test_generator_is_the_reference_generator():
    import bench
    a = cli.generate_batch(16, 256, 32000, 2, 42)
    b = bench.generate_batch(16, 256, 32000, 2, seed=42)
    np.testing.assert_array_equal(a[0][0], b[0][0])
    np.testing.assert_array_equal(a[1][1][1], b[1][1][1])


def test_parser_defaults_match_reference_cli():
    args = cli.build_parser().parse_args([])
    assert args.batch_sizes == [16, 32, 64, 128, 256, 512] and args.seq_lens == [256, 1024]
    assert args.vocab == 32000 and args.repeats == 5 and args.impl == "both"


@pytest.mark.gpu
def test_cli_run_csv_and_exit_codes(tmp_path, monkeypatch):
    out = tmp_path / "r.csv"
    rc = cli.main(["--batch-sizes", "4,8", "--seq-lens", "32", "--repeats", "2", "--out", str(out),
                   "--smoothing", "exp"])
    assert rc == 0
    lines = out.read_text().splitlines()
    assert lines[0] == cli.CSV_HEADER
    assert len(lines) == 1 + 4 and lines[1].startswith("serial,4,32,") and lines[2].startswith("gpu,4,32,")
    assert cli.main(["--batch-sizes", "4", "--seq-lens", "16", "--repeats", "1", "--pinned",
                     "--out", str(tmp_path / "p.csv")]) == 0
    assert cli.main(["--batch-sizes", "4", "--seq-lens", "16", "--repeats", "1",
                     "--out", str(tmp_path / "missing" / "r.csv")]) == 3
    monkeypatch.setattr(cli, "_serial_scores", lambda c, r, s: [0.5] * c[0].shape[0])
    assert cli.main(["--batch-sizes", "4", "--seq-lens", "16", "--repeats", "1",
                     "--out", str(tmp_path / "x.csv")]) == 2
