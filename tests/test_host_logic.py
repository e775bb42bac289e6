"""Host-side logic that needs no GPU: config validation, partitions, store accounting."""

import io

import numpy as np
import pytest

import paper_2305_19013_b200 as pk
from paper_2305_19013_b200.solvers import SolverConfig


class TestValidation:
    """Same messages as the reference (test_solvers.py:380-420)."""

    def test_method_unknown(self):
        with pytest.raises(ValueError, match="method"):
            SolverConfig(method="pcg").validate()

    def test_trunc_too_small(self):
        with pytest.raises(ValueError, match="trunc"):
            SolverConfig(method="sre-cg2", t=2, retention="trunc", trunc=1).validate()

    def test_partition_mismatch(self):
        p = pk.contiguous_partition(16, 4)
        with pytest.raises(ValueError, match="does not match"):
            SolverConfig(method="sre-cg2", t=2).validate(p)

    def test_sre_cg_retention_conflicts(self):
        with pytest.raises(ValueError, match="trunc=2"):
            SolverConfig(method="sre-cg", t=2, retention="trunc", trunc=5).validate()
        with pytest.raises(ValueError, match="retention"):
            SolverConfig(method="sre-cg", t=2, retention="restart", restart_j=5).validate()

    def test_odd_t_switch_rejected(self):
        with pytest.raises(ValueError, match="even"):
            SolverConfig(method="sre-cg2", t=3, switch_tol=1e-5).validate()

    def test_sstep_limits(self):
        with pytest.raises(ValueError, match="s must"):
            SolverConfig(method="sre-cg2", t=2, s=0).validate()
        with pytest.raises(ValueError, match="s-step"):
            SolverConfig(method="msdo-cg", t=2, s=2).validate()
        with pytest.raises(ValueError, match="exceeds"):
            SolverConfig(method="sre-cg2", t=32, s=4).validate()
        SolverConfig(method="sre-cg2", t=16, s=4, retention="trunc", trunc=2).validate()

    def test_enlarged_needs_partition(self):
        A = pk.gen_poisson2d(3, 3)
        with pytest.raises(ValueError, match="partition"):
            pk.enlarged_solve(A, np.ones(9), cfg=SolverConfig(method="sre-cg2", t=2))

    def test_bad_rhs(self):
        A = pk.gen_poisson2d(3, 3)
        p = pk.contiguous_partition(9, 3)
        with pytest.raises(ValueError, match="length"):
            pk.enlarged_solve(A, np.ones(8), partition=p, cfg=SolverConfig(t=3))
        with pytest.raises(ValueError, match="finite"):
            pk.enlarged_solve(A, np.full(9, np.nan), partition=p, cfg=SolverConfig(t=3))

    def test_effective_window(self):
        assert SolverConfig(method="sre-cg", t=2).effective_window() == 2
        assert SolverConfig(method="sre-cg2", t=2, retention="trunc", trunc=4).effective_window() == 4
        assert SolverConfig(method="sre-cg2", t=2).effective_window() is None


class TestPartition:
    def test_contiguous_sizes(self):
        p = pk.contiguous_partition(10, 3)
        assert [len(s) for s in p.subdomains] == [4, 3, 3]
        assert np.array_equal(p.owner(), [0, 0, 0, 0, 1, 1, 1, 2, 2, 2])

    def test_constructor_errors(self):
        with pytest.raises(ValueError, match="empty"):
            pk.Partition(3, [[0, 1, 2], []])
        with pytest.raises(ValueError, match="overlaps"):
            pk.Partition(3, [[0, 1], [1, 2]])
        with pytest.raises(ValueError, match="cover"):
            pk.Partition(4, [[0, 1], [2]])
        with pytest.raises(ValueError, match="out-of-range"):
            pk.Partition(3, [[0, 1], [2, 3]])

    def test_halve_merges_pairs(self):
        rng = np.random.default_rng(5)
        owner = rng.integers(0, 8, 200)
        owner[:8] = np.arange(8)
        p = pk.Partition.from_owner(owner, 8)
        h = p.halve()
        assert h.t == 4
        for i in range(4):
            merged = np.sort(np.concatenate((p.subdomains[2 * i], p.subdomains[2 * i + 1])))
            assert np.array_equal(np.sort(h.subdomains[i]), merged)
        with pytest.raises(ValueError, match="even"):
            pk.contiguous_partition(9, 3).halve()

    def test_file_roundtrip(self):
        p = pk.contiguous_partition(11, 4)
        buf = io.StringIO()
        pk.write_partition(p, buf)
        q = pk.read_partition(io.StringIO("# comment\n" + buf.getvalue()))
        assert np.array_equal(p.owner(), q.owner())


class TestPeakReplay:
    """peak_block_vectors accounting replayed from the enqueue log (solvers.py:163-170)."""

    def _engine(self, window, restarts=()):
        from paper_2305_19013_b200.engine import DeviceEngine
        e = DeviceEngine.__new__(DeviceEngine)
        e.window = window
        e.restarts = list(restarts)
        return e

    def test_full_retention(self):
        e = self._engine(None)
        e.launch_k = [(k, k - 1, 4) for k in range(1, 11)]
        assert e._replay_peak(7) == 28

    def test_window(self):
        e = self._engine(3)
        e.launch_k = [(k, min(k - 1, 3), 4) for k in range(1, 11)]
        assert e._replay_peak(10) == 16  # (w + 1) t, append before trim
        assert e._replay_peak(2) == 8

    def test_restart(self):
        e = self._engine(None, restarts=[6])
        e.launch_k = [(k, 0, 2) for k in range(1, 11)]
        assert e._replay_peak(10) == 10


def test_grid_pattern_detection_on_cpu_tensors():
    """StencilOperator.from_csr (operators.py) is plain tensor arithmetic: exact 5- / 7-point grid patterns
    give a coefficient table holding the matrix's own values in slot order; anything else gives None."""
    import types

    import numpy as np
    import torch

    from paper_2305_19013_b200.operators import StencilOperator
    from paper_2305_19013_b200.problems import diffusion_csr

    def fake(A):
        return types.SimpleNamespace(n=A.n, row_ptr=torch.from_numpy(np.asarray(A.row_ptr, dtype=np.int64)),
                                     col_idx=torch.from_numpy(np.asarray(A.col_idx).astype(np.int32)),
                                     values=torch.from_numpy(np.asarray(A.values, dtype=np.float64)), host=A)

    rng = np.random.default_rng(1)
    for shape in ((5, 4), (3, 4, 5), (2, 2), (2, 2, 2), (7, 3, 2)):
        n = int(np.prod(shape))
        A = diffusion_csr(shape, np.exp(rng.uniform(-1, 1, n)))
        op = StencilOperator.from_csr(fake(A))
        assert op is not None and op.shape == shape and op.n == n and op.nnz == A.nnz
        dim = len(shape)
        stride = 8 if dim == 3 else 6
        table = op.coef.reshape(n, stride).numpy()
        dense = A.to_dense()
        nx = shape[0]
        nxy = shape[0] * shape[1]
        offs = [-nxy, -nx, -1, 0, 1, nx, nxy] if dim == 3 else [-nx, -1, 0, 1, nx]
        for i in range(n):
            for slot, off in enumerate(offs):
                j = i + off
                want = dense[i, j] if 0 <= j < n and dense[i, j] != 0.0 else 0.0
                # x neighbours do not wrap across grid lines: the pattern has no entry there
                assert table[i, slot] == want, (shape, i, slot)
        assert np.all(table[:, len(offs):] == 0.0)
    # not a grid: an entry moved, a permuted matrix, a 1-D chain
    A = diffusion_csr((4, 4), np.ones(16))
    bad = fake(A)
    bad.col_idx = bad.col_idx.clone()
    bad.col_idx[2] += 1
    assert StencilOperator.from_csr(bad) is None
    bad = fake(A)
    bad.row_ptr = bad.row_ptr.clone()
    bad.row_ptr[3] -= 1
    assert StencilOperator.from_csr(bad) is None
    chain = types.SimpleNamespace(n=5, row_ptr=torch.tensor([0, 2, 5, 8, 11, 13]),
                                  col_idx=torch.tensor([0, 1, 0, 1, 2, 1, 2, 3, 2, 3, 4, 3, 4], dtype=torch.int32),
                                  values=torch.ones(13, dtype=torch.float64))
    assert StencilOperator.from_csr(chain) is None
