"""bench.py's roofline arithmetic (CPU): per-tag algorithmic bytes / flops and
the binding-roofline choice for the dominant kernel."""

import importlib.util
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench", ROOT / "bench.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_tag_model_matches_design(bench):
    n, m, d = 1000, 64, 3
    nm = n * m
    assert bench.tag_model("hist_gram", n, m, d, 0, 0) == (8.0 * (d + 1) * nm, 2.0 * d * m * nm)
    assert bench.tag_model("hist_update", n, m, d, 0, 0) == (8.0 * (d + 2) * nm, 2.0 * d * m * nm)
    assert bench.tag_model("tri_apply", n, m, 0, 0, 0) == (16.0 * nm, 1.0 * m * nm)
    # W^T W is symmetric: m (m + 1) / 2 distinct entries of 2 n flops each, one block read
    assert bench.tag_model("gram_self", n, m, 0, 0, 0) == (8.0 * nm, (m + 1.0) * nm)
    assert bench.tag_model("gram_aw", n, m, 0, 0, 0) == (16.0 * nm, 2.0 * m * nm)
    assert bench.tag_model("spmm", n, m, 0, 5 * n, 8 * n) == (16.0 * nm + 8 * n, 2.0 * 5 * n * m)
    assert bench.tag_model("unknown", n, m, 0, 0, 0) is None


class _Timer:
    def __init__(self, records):
        self.records = records
        self.d_min = 0


def test_roofline_picks_binding_peak(bench):
    n, m = 67_108_864, 64
    # a d = 3 update taking 50 ms: 1.65 TFLOP -> 33 TFLOP/s (fp64-bound); 172 GB -> 3.4 TB/s
    t = _Timer([("hist_update", 4, 3, m, 50.0), ("xr_update", 4, 3, m, 12.0)])
    r = bench.roofline_block(t, n, 0, 0, (6541.5, "hbm"), (37.07, "fp64"), {}, "w")
    assert r["kernel"] == "hist_update" and r["bound"] == "fp64" and r["unit"] == "TFLOP/s"
    flops = 2.0 * 3 * m * m * n
    assert r["achieved"] == pytest.approx(flops / 0.050 / 1e12)
    assert r["frac"] == pytest.approx(r["achieved"] / 37.07)
    # an HBM-bound dominant kernel reports GB/s against the copy peak
    t = _Timer([("xr_update", 4, 3, m, 12.0)])
    r = bench.roofline_block(t, n, 0, 0, (6541.5, "hbm"), (37.07, "fp64"), {}, "w")
    assert r["bound"] == "hbm" and r["unit"] == "GB/s"
    assert r["achieved"] == pytest.approx(8.0 * (2 * n * m + 4 * n) / 0.012 / 1e9)
