"""Full-size parity for BASELINE configs 3, 4 and 5 over the first K iterations.

Fixtures (tests/golden/make_full_golden.py, generated in the build container):

* full_cfg3.json -- the REAL reference `ekcg.enlarged_solve` (solvers.py:261-292)
  on the full 128^3 config-3 inputs (reference generator), 20 iterations;
* full_cfg4.json -- config 4 at full size (256^3, s = 4); the reference has no
  s-step method (solvers.py:59), so the fixture is the oracle's definition
  (bounded-memory restatement, bitwise run_oracle at small sizes);
* full_cfg5.json -- the largest config-5 instance the bounded-memory oracle fits
  in the build host's RAM (4096^2, 8 iterations, 95 min; stated in the fixture;
  one full-size n x 64 block is 34.4 GB); full_cfg5_2048.json -- 2048^2, 12
  iterations.

Each test rebuilds the inputs with the package's generators, checks them
against the fixture's hashes (b, owner map, coefficient field), runs the device
engine through the public `enlarged_solve` for the same K iterations and holds
the relative residual history to the north-star 1e-8 (BASELINE.json).
"""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest
import torch

import paper_2305_19013_b200 as pk
from paper_2305_19013_b200.problems import make_config

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

GOLDEN = Path(__file__).resolve().parent / "golden"
HIST_TOL = 1e-8


def _sha(a):
    a = a.cpu().numpy() if isinstance(a, torch.Tensor) else a
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _fixture(name):
    p = GOLDEN / f"full_{name}.json"
    if not p.exists():
        pytest.skip(f"{p.name} not generated")
    return json.loads(p.read_text())


def _run(index, fx, **over):
    prob = make_config(index, fx["edge"])
    assert prob.n == fx["n"]
    assert _sha(prob.b) == fx["b_sha256"], "right-hand side differs from the fixture's"
    assert _sha(prob.partition.owner()) == fx["owner_sha256"], "owner map differs from the fixture's"
    if "kappa_field_sha256" in fx:
        assert _sha(prob.kappa_field) == fx["kappa_field_sha256"]
    kw = dict(prob.solver_kwargs)
    kw["kmax"] = fx["k"]
    kw.update(over)
    b = torch.as_tensor(prob.b, device="cuda")
    x, rep = pk.enlarged_solve(prob.stencil(), b, partition=prob.partition, cfg=pk.SolverConfig(**kw))
    h = np.asarray(rep.residual_history)
    g = np.asarray(fx["residual_history"])
    assert rep.status == fx["status"]
    assert rep.iterations == fx["iterations"]
    assert rep.peak_block_vectors == fx["peak_block_vectors"]
    rh, rg = h / h[0], g / g[0]
    dev = np.abs(rh - rg) / rg
    print(f"{fx['config']}: max relative history deviation over k <= {fx['k']}: {dev.max():.3e}")
    assert dev.max() <= HIST_TOL, dev
    return rep, dev


def test_cfg3_full_size_vs_real_reference():
    fx = _fixture("cfg3")
    _run(3, fx)


def test_cfg3_full_size_vs_real_reference_csr_form():
    """The reference-facing form: the host CSR matrix of the reference generator."""
    fx = _fixture("cfg3")
    prob = make_config(3, fx["edge"])
    A = prob.csr()
    kw = dict(prob.solver_kwargs, kmax=fx["k"])
    x, rep = pk.enlarged_solve(A, prob.b, partition=prob.partition, cfg=pk.SolverConfig(**kw))
    h, g = np.asarray(rep.residual_history), np.asarray(fx["residual_history"])
    dev = np.abs(h / h[0] - g / g[0]) / (g / g[0])
    assert rep.iterations == fx["iterations"] and dev.max() <= HIST_TOL, dev


@pytest.mark.grid_detect
def test_cfg3_full_size_vs_real_reference_csr_form_grid_detected():
    """The product default for the same host CSR matrix: its 7-point grid pattern is detected and the
    matrix applied in stencil form from a table of its own values (bitwise the CSR products)."""
    from paper_2305_19013_b200.engine import DeviceEngine
    from paper_2305_19013_b200.operators import StencilOperator
    fx = _fixture("cfg3")
    prob = make_config(3, fx["edge"])
    A = prob.csr()
    kw = dict(prob.solver_kwargs, kmax=fx["k"])
    eng = DeviceEngine(A, prob.partition, pk.SolverConfig(**kw))
    assert isinstance(eng.op, StencilOperator) and eng.op.from_matrix
    x, rep = eng.solve(prob.b)
    h, g = np.asarray(rep.residual_history), np.asarray(fx["residual_history"])
    dev = np.abs(h / h[0] - g / g[0]) / (g / g[0])
    assert rep.iterations == fx["iterations"] and dev.max() <= HIST_TOL, dev


def test_cfg4_full_size_vs_oracle():
    fx = _fixture("cfg4")
    _run(4, fx)


def test_cfg5_largest_oracle_instance():
    fx = _fixture("cfg5")
    _run(5, fx)


def test_cfg5_second_oracle_instance_2048():
    """The first bounded-memory fixture (2048^2, 12 iterations: four more steady-state iterations than the 4096^2 one)."""
    fx = _fixture("cfg5_2048")
    _run(5, fx)


def test_cfg3_class_complete_solve_iteration_count():
    """The config-3 generator at 64^3 solved to tol by the real reference (full_cfg3_solve64.json):
    iteration count within +-2 % (north star), history over k <= 20 within 1e-8, true residual <= tol.
    (The full 128^3 reference solve would take ~30 h on the build host, so its count is not pinned.)"""
    p = GOLDEN / "full_cfg3_solve64.json"
    if not p.exists():
        pytest.skip("full_cfg3_solve64.json not generated")
    fx = json.loads(p.read_text())
    prob = make_config(3, fx["edge"])
    assert _sha(prob.b) == fx["b_sha256"] and _sha(prob.partition.owner()) == fx["owner_sha256"]
    x, rep = pk.enlarged_solve(prob.stencil(), prob.b, partition=prob.partition,
                               cfg=pk.SolverConfig(**prob.solver_kwargs))
    it_ref = fx["iterations"]
    print(f"cfg3@{fx['edge']}: {rep.iterations} iterations (reference {it_ref}), true residual "
          f"{rep.true_residual / np.linalg.norm(prob.b):.2e}")
    assert rep.status == fx["status"] == "converged"
    assert abs(rep.iterations - it_ref) <= max(1, round(0.02 * it_ref))
    h, g = np.asarray(rep.residual_history), np.asarray(fx["residual_history"])
    k = min(len(h), len(g), 21)
    assert np.max(np.abs(h[:k] / h[0] - g[:k] / g[0]) / (g[:k] / g[0])) <= HIST_TOL
    # the stop test is on the recurrence residual; the true one is reported (solvers.py:289): hold it to tol,
    # or to the reference's own final true residual when that one already ends above tol
    assert rep.true_residual <= max(1e-8 * np.linalg.norm(prob.b), 1.5 * fx["true_residual"])
