"""Golden batch output of the real reference (`ekcg.run_experiment`, harness.py:142-268).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_batch_golden.py

Writes tests/golden/batch.json: the runs.csv text and every history TSV for
the determinism spec of the reference acceptance suite (test_acceptance.py:352-376).
"""
import json
import os
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, os.environ.get("EKCG_REFERENCE", "/root/reference/pkg/src"))
from ekcg.harness import run_experiment  # noqa: E402

SPEC = {"matrix": "poisson2d:12,12", "methods": ["cg", "sre-cg2", "msdo-cg"], "t": [2, 4],
        "retention": ["full", "trunc:3"], "switch_tol": None, "tol": 1e-8, "seed": 312}

if __name__ == "__main__":
    with tempfile.TemporaryDirectory() as tmp:
        run_experiment(SPEC, tmp, render_figures=False)
        out = {"spec": SPEC, "csv": (Path(tmp) / "runs.csv").read_text(),
               "histories": {p.name: p.read_text() for p in sorted(Path(tmp).glob("*_history.tsv"))}}
    (Path(__file__).resolve().parent / "batch.json").write_text(json.dumps(out, indent=1))
    print(len(out["histories"]), "histories")
