"""Batch-format parity: device runs written in the reference's
runs.csv / history TSV format, checked against the reference's own output."""

import csv
import io
import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2305_19013_b200.reporting import CSV_COLUMNS, run_batch

GOLDEN = Path(__file__).resolve().parent / "golden" / "batch.json"


def _rows(text):
    return list(csv.DictReader(io.StringIO(text)))


def _hist(text):
    lines = text.strip().splitlines()
    assert lines[0] == "iteration\trho\ttol1"
    return np.array([float(l.split("\t")[1]) for l in lines[1:]])


def test_batch_matches_reference_format(tmp_path):
    gold = json.loads(GOLDEN.read_text())
    rows = run_batch(gold["spec"], tmp_path)
    text = (tmp_path / "runs.csv").read_text()
    assert text.splitlines()[0] == ",".join(CSV_COLUMNS) == gold["csv"].splitlines()[0]
    ours, ref = _rows(text), _rows(gold["csv"])
    assert [r["run_id"] for r in ours] == [r["run_id"] for r in ref]
    for a, b in zip(ours, ref):
        for col in ("matrix", "method", "t", "partition", "retention", "trunc", "tol", "kmax", "seed",
                    "precond", "precond_mode", "switch_tol"):
            assert a[col] == b[col], (a["run_id"], col, a[col], b[col])
        for col in ("restart_count", "switch_iteration"):
            assert a[col] == b[col], (a["run_id"], col, a[col], b[col])
        assert a["status"] == b["status"]
        assert abs(int(a["iterations"]) - int(b["iterations"])) <= 1
        assert a["peak_block_vectors"] == b["peak_block_vectors"] or a["iterations"] != b["iterations"]
        assert abs(float(a["relative_error"]) - float(b["relative_error"])) <= 1e-6
        h_ours = _hist((tmp_path / f"{a['run_id']}_history.tsv").read_text())
        h_ref = _hist(gold["histories"][f"{b['run_id']}_history.tsv"])
        n = min(len(h_ours), len(h_ref), 21)
        keep = h_ref[:n] / h_ref[0] > 1e-12
        assert np.max(np.abs(h_ours[:n][keep] / h_ours[0] - h_ref[:n][keep] / h_ref[0])
                      / (h_ref[:n][keep] / h_ref[0])) <= 1e-8


def test_batch_rerun_is_bit_identical(tmp_path):
    """Acceptance criterion 12 (test_acceptance.py:352-376) on the device path."""
    gold = json.loads(GOLDEN.read_text())
    run_batch(gold["spec"], tmp_path / "a")
    run_batch(gold["spec"], tmp_path / "b")
    a = (tmp_path / "a" / "runs.csv").read_text().splitlines()
    b = (tmp_path / "b" / "runs.csv").read_text().splitlines()
    wall = CSV_COLUMNS.index("wall_time_s")
    for ra, rb in zip(a, b):
        fa, fb = ra.split(","), rb.split(",")
        del fa[wall], fb[wall]
        assert fa == fb
    for p in sorted((tmp_path / "a").glob("*_history.tsv")):
        assert p.read_text() == (tmp_path / "b" / p.name).read_text()
