"""The one-kernel cluster solve (csrc/cluster_solve.cu, `ekcg_cluster_solve`): the whole
truncated-window loop of `_run_engine` (solvers.py:319-428) on one thread-block cluster.

Checked against the real reference's goldens (history 1e-8 over k <= 20, iteration count,
status, peak, true-residual log), against the launch-per-phase engine on the same inputs,
and for bit-identical reruns (fixed-order reductions, no atomics).
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2305_19013_b200 as pk
from paper_2305_19013_b200.engine import DeviceEngine
from paper_2305_19013_b200.problems import make_config
from paper_2305_19013_b200.solvers import SolverConfig
from conftest import golden_case_inputs
from test_gpu_solver import hist_dev, hist_tol, iter_tol


def _engines(op, partition, cfg, b, x0=None, x_star=None):
    out = []
    for use in (True, False):
        eng = DeviceEngine(op, partition, cfg)
        eng.use_cluster = use
        x, rep = eng.solve(b, x0, x_star=x_star)
        assert eng.ran_cluster == use, "wrong engine path"
        out.append((x, rep))
    return out


@pytest.mark.parametrize("form", ["stencil", "csr"])
def test_cfg1_cluster_matches_reference(solves_golden, floors_golden, form):
    """BASELINE config 1 (SRE-CG, t = 8, 100^2 Poisson) against the real reference's run."""
    meta, arrays = solves_golden
    name = "cfg1_100"
    prob = make_config(1, 100)
    op = prob.stencil() if form == "stencil" else prob.csr()
    eng = DeviceEngine(op, prob.partition, SolverConfig(**prob.solver_kwargs))
    x, rep = eng.solve(prob.b, x_star=prob.x_star)
    assert eng.ran_cluster, "config 1 should take the cluster kernel"
    ref = meta[name]
    assert rep.status == ref["status"] == "converged"
    assert hist_dev(rep.residual_history, arrays[f"{name}__history"]) <= hist_tol(floors_golden, name)
    assert abs(rep.iterations - ref["iterations"]) <= iter_tol(floors_golden, name, ref["iterations"])
    assert rep.peak_block_vectors == ref["peak_block_vectors"]
    assert [c[0] for c in rep.true_residual_checks] == [c[0] for c in ref["true_residual_checks"]]
    for (_, got), (_, want) in zip(rep.true_residual_checks, ref["true_residual_checks"]):
        assert abs(got - want) <= 1e-6 * want + 1e-12
    assert rep.true_residual <= 1e-8 * np.linalg.norm(prob.b) * 10
    assert rep.relative_error is not None and rep.relative_error < 1e-6


CASES = [  # (config class, edge, solver overrides)
    (1, 40, {}),
    (1, 64, {"method": "sre-cg2", "retention": "trunc", "trunc": 3}),
    (2, 12, {"retention": "trunc", "trunc": 2}),          # 3-D, t = 16: 8-CTA cluster (receive buffers)
    (2, 10, {"method": "sre-cg"}),
    (1, 33, {"method": "sre-cg2", "retention": "trunc", "trunc": 4, "true_residual_every": 7}),
]


@pytest.mark.parametrize("idx,edge,over", CASES)
@pytest.mark.parametrize("form", ["stencil", "csr"])
def test_cluster_matches_launch_per_phase_engine(idx, edge, over, form):
    prob = make_config(idx, edge)
    cfg = SolverConfig(**dict(prob.solver_kwargs, **over))
    op = prob.stencil() if form == "stencil" else prob.csr()
    (xa, a), (xb, b) = _engines(op, prob.partition, cfg, prob.b, x_star=prob.x_star)
    assert a.status == b.status == "converged"
    assert abs(a.iterations - b.iterations) <= max(1, round(0.02 * b.iterations))
    assert hist_dev(a.residual_history, b.residual_history) <= 1e-9
    assert a.peak_block_vectors == b.peak_block_vectors or a.iterations != b.iterations
    assert [c[0] for c in a.true_residual_checks][:3] == [c[0] for c in b.true_residual_checks][:3]
    assert np.linalg.norm(xa - xb) <= 1e-6 * np.linalg.norm(xb)


def test_cluster_tile_field_operator():
    """Variable-coefficient (kappa tile field) stencil rows inside the cluster kernel."""
    from paper_2305_19013_b200.partition import Partition
    rng = np.random.default_rng(11)
    nx = ny = 48
    field = np.exp(rng.uniform(-2.0, 2.0, size=(ny // 8, nx // 8)))
    op = pk.StencilOperator((nx, ny), kappa=field, tile=(8, 8))
    owner = (np.arange(ny)[:, None] // (ny // 4) * 2 + np.arange(nx)[None, :] // (nx // 2)).reshape(-1)
    part = Partition.from_owner(owner.astype(np.int64), 8)
    b = rng.uniform(-1.0, 1.0, nx * ny)
    cfg = SolverConfig(method="sre-cg2", t=8, tol=1e-8, retention="trunc", trunc=3)
    (xa, a), (xb, b_) = _engines(op, part, cfg, b)
    assert a.status == b_.status == "converged"
    assert abs(a.iterations - b_.iterations) <= max(1, round(0.02 * b_.iterations))
    assert hist_dev(a.residual_history, b_.residual_history) <= 1e-9
    # and the CSR form of the same operator
    A = op.to_csr()
    eng = DeviceEngine(A, part, cfg)
    eng.use_cluster = True
    xc, c = eng.solve(b)
    assert eng.ran_cluster
    assert np.array_equal(c.residual_history, a.residual_history), "stencil and CSR rows are bitwise the same operator"


def test_cluster_rerun_bit_identical():
    prob = make_config(1, 100)
    cfg = SolverConfig(**prob.solver_kwargs)
    outs = []
    for _ in range(3):
        eng = DeviceEngine(prob.stencil(), prob.partition, cfg)
        x, rep = eng.solve(prob.b)
        assert eng.ran_cluster
        outs.append((x, rep.residual_history))
    for x, h in outs[1:]:
        assert np.array_equal(x, outs[0][0]) and np.array_equal(h, outs[0][1])


def test_cluster_breakdown_and_maxiter(solves_golden):
    """The p12_srecg2_t8_trunc2 golden breaks down at iteration 17; kmax stops report maxiter."""
    meta, arrays = solves_golden
    name = "p12_srecg2_t8_trunc2"
    rp, ci, vals, b, owner, x0 = golden_case_inputs(arrays, name)
    A = pk.SparseSpdMatrix(len(rp) - 1, rp, ci, vals)
    kw = dict(meta[name]["cfg"])
    part = pk.Partition.from_owner(owner, kw["t"])
    eng = DeviceEngine(A, part, SolverConfig(**kw))
    x, rep = eng.solve(b, x0)
    assert eng.ran_cluster
    ref = meta[name]
    assert rep.status == ref["status"] == "breakdown"
    assert rep.iterations == ref["iterations"]
    assert rep.notes[0].split(":")[0] == ref["notes"][0].split(":")[0]
    eng = DeviceEngine(A, part, SolverConfig(**dict(kw, kmax=5)))
    x, rep = eng.solve(b, x0)
    assert eng.ran_cluster and rep.status == "maxiter" and rep.iterations == 5
    assert len(rep.residual_history) == 6


def test_cluster_x0_and_torch_io():
    prob = make_config(1, 40)
    cfg = SolverConfig(**prob.solver_kwargs)
    rng = np.random.default_rng(3)
    x0 = rng.standard_normal(prob.n)
    (xa, a), (xb, b) = _engines(prob.stencil(), prob.partition, cfg, prob.b, x0=x0)
    assert a.status == b.status == "converged"
    assert hist_dev(a.residual_history, b.residual_history) <= 1e-9
    bt = torch.as_tensor(prob.b, device="cuda")
    x, rep = pk.enlarged_solve(prob.stencil(), bt, partition=prob.partition, cfg=cfg)
    assert isinstance(x, torch.Tensor) and x.is_cuda and rep.status == "converged"


def test_cluster_not_taken_when_ineligible():
    prob = make_config(3, 16)  # t = 32
    eng = DeviceEngine(prob.stencil(), prob.partition, SolverConfig(**dict(prob.solver_kwargs, kmax=5)))
    eng.solve(prob.b)
    assert not eng.ran_cluster
    prob = make_config(2, 12)  # full retention
    eng = DeviceEngine(prob.stencil(), prob.partition, SolverConfig(**dict(prob.solver_kwargs, kmax=5)))
    eng.solve(prob.b)
    assert not eng.ran_cluster


@pytest.mark.parametrize("t,shape,window", [(1, (30, 30), 2), (3, (30, 30), 3), (5, (24, 20), 2), (7, (31, 17), 4),
                                            (12, (20, 20), 2), (2, (10, 10), 2), (6, (9, 8, 7), 2)])
@pytest.mark.parametrize("form", ["stencil", "csr"])
def test_cluster_any_width_and_ragged_rows(t, shape, window, form):
    """Odd and non-power-of-two block widths (scalar load / store paths, runtime-width DMMA tiles), grids
    whose row count is no multiple of the 8-row tiles, and problems with fewer rows than the cluster has
    row slots (some CTAs own no rows)."""
    from paper_2305_19013_b200.partition import Partition
    rng = np.random.default_rng(100 + t)
    n = int(np.prod(shape))
    op = pk.StencilOperator(shape, kappa=1.0 + 0.25 * t)
    A = op if form == "stencil" else op.to_csr()
    owner = (np.arange(n) * t // n).astype(np.int64)
    part = Partition.from_owner(owner, t)
    b = rng.uniform(-1.0, 1.0, n)
    cfg = SolverConfig(method="sre-cg2", t=t, tol=1e-9, retention="trunc", trunc=window, true_residual_every=5)
    (xa, a), (xb, b_) = _engines(A, part, cfg, b)
    assert a.status == b_.status == "converged"
    assert abs(a.iterations - b_.iterations) <= max(1, round(0.02 * b_.iterations))
    assert hist_dev(a.residual_history, b_.residual_history) <= 1e-9
    assert a.peak_block_vectors == b_.peak_block_vectors or a.iterations != b_.iterations
    assert len(a.true_residual_checks) == a.iterations // 5
    assert np.linalg.norm(xa - xb) <= 1e-7 * np.linalg.norm(xb)
    assert a.true_residual <= 1e-8 * np.linalg.norm(b)


def test_cluster_zero_rhs_and_exact_start():
    """rho0 = 0: converged with no iteration (solvers.py:343-345); a start at the solution likewise stops at once."""
    prob = make_config(1, 40)
    cfg = SolverConfig(**prob.solver_kwargs)
    eng = DeviceEngine(prob.stencil(), prob.partition, cfg)
    x, rep = eng.solve(np.zeros(prob.n))
    assert eng.ran_cluster and rep.status == "converged" and rep.iterations == 0 and not np.any(x)
    eng = DeviceEngine(prob.stencil(), prob.partition, SolverConfig(**dict(prob.solver_kwargs, kmax=1)))
    x, rep = eng.solve(prob.b)
    assert eng.ran_cluster and rep.status == "maxiter" and rep.iterations == 1 and len(rep.residual_history) == 2


@pytest.mark.parametrize("shape,form", [((100, 100), "stencil"), ((100, 100), "csr"), ((17, 13, 11), "stencil"),
                                        ((9, 7), "csr")])
def test_cluster_cg_matches_launch_per_phase_cg(shape, form, monkeypatch):
    """Classical CG (solvers.py:199-258) as one cluster kernel (ekcg_cluster_cg) against the launch-per-phase
    loop on the same inputs: same status and iteration count, history to round-off."""
    import importlib
    cg_mod = importlib.import_module("paper_2305_19013_b200.cg")
    rng = np.random.default_rng(5)
    op = pk.StencilOperator(shape, kappa=1.5)
    A = op if form == "stencil" else op.to_csr()
    n = int(np.prod(shape))
    x_star = rng.standard_normal(n)
    b = pk.spmv(op.to_csr(), x_star)
    cfg = SolverConfig(method="cg", tol=1e-9)
    reps = []
    for cap in (1 << 18, 0):
        monkeypatch.setattr(cg_mod, "CLUSTER_CG_MAX_N", cap)
        launches0 = cg_mod._lib.query("ekcg_launch_count")
        x, rep = pk.cg(A, b, cfg=cfg, x_star=x_star)
        reps.append((x, rep, cg_mod._lib.query("ekcg_launch_count") - launches0))
    (xa, a, la), (xb, b_, lb) = reps
    assert la < 20 < lb, "the first run should be one cluster kernel, the second one launch per phase"
    assert a.status == b_.status == "converged"
    assert abs(a.iterations - b_.iterations) <= max(1, round(0.02 * b_.iterations))
    assert hist_dev(a.residual_history, b_.residual_history) <= 1e-9
    assert a.relative_error < 1e-6 and np.linalg.norm(xa - xb) <= 1e-7 * np.linalg.norm(xb)


def test_cluster_cg_breakdown_and_kmax(monkeypatch):
    """Nonpositive curvature stops with the reference's status and note; kmax reports maxiter."""
    n = 64
    rp = np.arange(n + 1, dtype=np.int64)
    ci = np.arange(n, dtype=np.int64)
    vals = np.ones(n)
    vals[3] = -2.0  # indefinite diagonal matrix
    A = pk.SparseSpdMatrix(n, rp, ci, vals, validate=False)
    b = np.zeros(n)
    b[3] = 1.0
    x, rep = pk.cg(A, b, cfg=SolverConfig(method="cg"))
    assert rep.status == "breakdown" and rep.iterations == 0
    assert rep.notes == ["nonpositive curvature p^T A p = -2.000e+00 at iteration 1"]
    prob = make_config(1, 40)
    x, rep = pk.cg(prob.stencil(), prob.b, cfg=SolverConfig(method="cg", kmax=7))
    assert rep.status == "maxiter" and rep.iterations == 7 and len(rep.residual_history) == 8


def test_cluster_kernels_refuse_rows_longer_than_8_entries():
    """The C entry points check the CSR row lengths on the device (the Python dispatch never sends such a matrix)."""
    import ctypes

    from paper_2305_19013_b200 import _lib
    n, t = 64, 2
    dense = np.eye(n) * 20.0
    for k in range(1, 6):  # 11 entries per interior row
        dense += np.diag(np.full(n - k, -1.0), k) + np.diag(np.full(n - k, -1.0), -k)
    r, c = np.nonzero(dense)
    A = pk.SparseSpdMatrix.from_coo(n, r, c, dense[r, c])
    op = pk.CsrOperator(A)
    f64 = dict(dtype=torch.float64, device="cuda")
    b = torch.ones(n, **f64)
    x = torch.zeros(n, **f64)
    rr = b.clone()
    rho2 = (rr * rr).sum().reshape(1)
    ctrl = torch.zeros(_lib.query("ekcg_ctrl_bytes"), dtype=torch.uint8, device="cuda")
    hist = torch.zeros(50, **f64)
    st = torch.cuda.current_stream().cuda_stream
    _lib.call("ekcg_start", ctrl.data_ptr(), rho2.data_ptr(), 1e-8, hist.data_ptr(), st)
    owner = torch.arange(n, dtype=torch.int32, device="cuda") * t // n
    blocks = torch.zeros(7 * 128 + 64, **f64)
    checks = torch.zeros(50, **f64)
    _lib.call("ekcg_cluster_solve", None, op.row_ptr.data_ptr(), op.col_idx.data_ptr(), op.values.data_ptr(), n, t, 2, 20,
              50, owner.data_ptr(), b.data_ptr(), x.data_ptr(), rr.data_ptr(), blocks.data_ptr(), 128, ctrl.data_ptr(),
              hist.data_ptr(), checks.data_ptr(), 1e-14, None, st)
    assert int(ctrl.cpu().numpy()[:8].view(np.int32)[1]) == 5 and not torch.any(x)
    _lib.call("ekcg_start", ctrl.data_ptr(), rho2.data_ptr(), 1e-8, hist.data_ptr(), st)
    scratch = torch.zeros(2 * n, **f64)
    _lib.call("ekcg_cluster_cg", None, op.row_ptr.data_ptr(), op.col_idx.data_ptr(), op.values.data_ptr(), n, 20,
              x.data_ptr(), rr.data_ptr(), scratch.data_ptr(), ctrl.data_ptr(), hist.data_ptr(), st)
    assert int(ctrl.cpu().numpy()[:8].view(np.int32)[1]) == 5 and not torch.any(x)
    # the Python dispatch keeps such matrices on the launch-per-phase kernels
    part = pk.Partition.from_owner(owner.cpu().numpy().astype(np.int64), t)
    eng = DeviceEngine(A, part, SolverConfig(method="sre-cg2", t=t, retention="trunc", trunc=2, tol=1e-10))
    xs, rep = eng.solve(np.ones(n))
    assert not eng.ran_cluster and rep.status == "converged"
    assert np.allclose(dense @ xs, np.ones(n), atol=1e-8)
