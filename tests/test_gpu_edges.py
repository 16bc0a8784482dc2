"""Edge cases of the hot path against the oracle (the reference's own edge tests: 1 x 1 and empty
systems, diagonal matrices, ragged rows, zero right-hand sides): spmv / ic_apply bitwise, PCG
iterations and solutions as the oracle, batched and sampled paths included."""
import numpy as np
import pytest

from oracle import Matrix

pytestmark = pytest.mark.gpu


def _csr(dense):
    n = dense.shape[0]
    rs, ci, va = [0], [], []
    for i in range(n):
        for j in range(n):
            if dense[i, j] != 0.0 or i == j:
                ci.append(j)
                va.append(dense[i, j])
        rs.append(len(ci))
    return n, np.array(rs, np.int32), np.array(ci, np.int32), np.array(va)


def _arrow(n, seed=3):
    """Row / column 0 dense, the rest diagonal + a chain: ragged rows (1 .. n entries), SPD."""
    rng = np.random.default_rng(seed)
    a = np.zeros((n, n))
    a[0, 1:] = a[1:, 0] = -rng.uniform(0.1, 1.0, n - 1) / n
    for i in range(1, n - 1):
        a[i, i + 1] = a[i + 1, i] = -0.3
    a[np.arange(n), np.arange(n)] = 2.0
    return a


CASES = {
    "one": np.array([[4.0]]),
    "diag": np.diag(np.arange(1.0, 70.0)),
    "arrow": _arrow(300),
}


@pytest.mark.parametrize("name", list(CASES))
def test_edge_matrices_spmv_ic_pcg(ctx, oracle, name):
    from paper_2203_08498_b200 import api

    n, rs, ci, va = _csr(CASES[name])
    a_o = Matrix(n, rs, ci, va)
    a = api.CsrMatrix(ctx, n, rs, ci, va)
    x = oracle.uniform_pm1(7, 0, n)
    assert np.array_equal(a.spmv(x), oracle.spmv(a_o, x))
    f_o = oracle.ic0_factorize(a_o)
    f = api.IcFactor.factorize(ctx, n, rs, ci, va)
    assert np.array_equal(f.apply(x), oracle.ic_apply(f_o, x))
    fd = api.IcFactor.factorize_device(ctx, a)
    assert np.array_equal(fd.apply(x), oracle.ic_apply(f_o, x))
    b = oracle.spmv(a_o, oracle.uniform_pm1(8, 0, n))
    for kind, prec in ((0, api.Identity()), (1, api.Ic(f))):
        xo, xg = np.zeros(n), np.zeros(n)
        ro = oracle.pcg_solve(a_o, b, xo, kind=kind, ic=f_o if kind else None, max_iter=2000)
        rg = api.pcg_solve(ctx, a, b, prec, xg, 1e-8, 2000)
        assert rg.converged == ro.converged and abs(rg.iterations - ro.iterations) <= 2
        if rg.iterations == ro.iterations:
            assert np.linalg.norm(xg - xo) <= 1e-8 * max(np.linalg.norm(xo), 1e-300)
    # batched: two copies of the same right-hand side solve exactly like the single solve
    X = np.zeros((2, n))
    reps = api.pcg_solve_batch(ctx, a, np.stack([b, b]), api.Ic(f), X, 1e-8, 2000)
    x1 = np.zeros(n)
    r1 = api.pcg_solve(ctx, a, b, api.Ic(f), x1, 1e-8, 2000)
    assert [r.iterations for r in reps] == [r1.iterations] * 2
    assert np.linalg.norm(X[0] - x1) <= 1e-12 * max(np.linalg.norm(x1), 1e-300)


def test_one_by_one_exact(ctx, oracle):
    """A = [4], b = [8]: one iteration to x = 2 (pcg.cpp with IC(0) = exact inverse)."""
    from paper_2203_08498_b200 import api

    n, rs, ci, va = _csr(CASES["one"])
    a = api.CsrMatrix(ctx, n, rs, ci, va)
    f = api.IcFactor.factorize(ctx, n, rs, ci, va)
    x = np.zeros(1)
    r = api.pcg_solve(ctx, a, np.array([8.0]), api.Ic(f), x, 1e-8, 10)
    assert r.converged and r.iterations == 1 and x[0] == 2.0


def test_empty_system(ctx, oracle):
    """n = 0: the reference's zero right-hand-side shortcut (pcg.cpp:43-48) -- converged at 0
    iterations, nothing to compute (the oracle agrees)."""
    from paper_2203_08498_b200 import api

    rs, ci, va = np.zeros(1, np.int32), np.zeros(0, np.int32), np.zeros(0)
    a = api.CsrMatrix(ctx, 0, rs, ci, va)
    assert a.spmv(np.zeros(0)).shape == (0,)
    ro = oracle.pcg_solve(Matrix(0, rs, ci, va), np.zeros(0), np.zeros(0), kind=0, max_iter=10)
    rg = api.pcg_solve(ctx, a, np.zeros(0), api.Identity(), np.zeros(0), 1e-8, 10)
    assert rg.converged == ro.converged and rg.iterations == ro.iterations == 0


def test_zero_rhs_in_a_batch(ctx, oracle, problems):
    """A zero right-hand side among running ones: x stays 0 at 0 iterations (pcg.cpp:43-48), the
    others solve as alone."""
    from paper_2203_08498_b200 import api

    h = problems.generate(problems.SMALL["c1"])
    a = api.CsrMatrix(ctx, h.n, h.row_start, h.col_idx, h.values)
    f = api.IcFactor.factorize_device(ctx, a)
    b = oracle.spmv(Matrix.of(h), oracle.uniform_pm1(4, 0, h.n))
    X = np.ones((3, h.n))
    X[:] = 0.0
    reps = api.pcg_solve_batch(ctx, a, np.stack([b, np.zeros(h.n), b]), api.Ic(f), X, 1e-8, 500)
    assert reps[1].iterations == 0 and reps[1].converged and not X[1].any()
    assert reps[0].iterations == reps[2].iterations and np.array_equal(X[0], X[2])
