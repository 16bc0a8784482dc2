"""Batched multi-RHS solves (rcg_pcg_solve_batch / rcg_deflated_pcg_solve_batch) against the
oracle: every right-hand side meets the same bars as a single solve (iterations +-2, solution
within the oracle's rounding floor), zero right-hand sides short-circuit, caps are honoured."""
from dataclasses import replace

import numpy as np
import pytest

from oracle import Matrix
from test_gpu_parity import _oracle_floor, _rel, _sol_tol

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["c1", "c2", "c4"])
@pytest.mark.parametrize("method", ["deflation", "sc", "iccg"])
@pytest.mark.parametrize("nrhs", [3, 9, 19])
def test_batch_matches_oracle(ctx, oracle, problems, name, method, nrhs):
    """nrhs 3 / 9 / 19: kernel widths RT 4 / 12 / 24 (C3's 19 accelerated solves in one batch),
    with compaction to narrower phases as right-hand sides converge."""
    if nrhs == 19 and name != "c2":
        pytest.skip("RT 24 on the SC / deflation / ICCG variants of one problem is enough")
    from oracle.sequence import run_sequence as oracle_sequence
    from paper_2203_08498_b200 import api

    cfg = replace(problems.SMALL[name], method="sc" if method == "sc" else "deflation", n_rhs=nrhs + 1)
    h = problems.generate(cfg)
    ores = oracle_sequence(oracle, cfg, h)
    sa, _ = oracle.diagonal_scale(Matrix.of(h))
    of = oracle.ic0_factorize(sa)
    ga = api.CsrMatrix(ctx, h.n, h.row_start, h.col_idx, sa.va)
    gf = api.IcFactor.factorize(ctx, h.n, h.row_start, h.col_idx, sa.va)
    B = np.stack(ores["scaled_rhs"][1:])
    X = np.zeros_like(B)
    if method == "iccg":
        reps = api.pcg_solve_batch(ctx, ga, B, api.Ic(gf), X, cfg.eps, cfg.max_iter)
        for k in range(nrhs):
            xo = np.zeros(h.n)
            ro = oracle.pcg_solve(sa, B[k], xo, kind=1, ic=of, max_iter=cfg.max_iter)
            assert reps[k].converged and abs(reps[k].iterations - ro.iterations) <= 2
            assert _rel(X[k], xo) <= 1e-6
        return
    basis = api.Basis(ctx, ga, api.TallDense.from_columns(ctx, h.n, ores["w"]), "sc" if method == "sc" else "deflation")
    if method == "sc":
        reps = api.pcg_solve_batch(ctx, ga, B, api.Sc(basis, gf), X, cfg.eps, cfg.max_iter)
    else:
        reps = api.deflated_pcg_solve_batch(ctx, ga, B, api.Ic(gf), basis, X, cfg.eps, cfg.max_iter)
    for k in range(nrhs):
        assert reps[k].converged
        assert abs(reps[k].iterations - ores["iterations"][k + 1]) <= 2, (k, reps[k].iterations, ores["iterations"])
        if reps[k].iterations == ores["iterations"][k + 1]:
            floor = _oracle_floor(oracle, cfg, h, ores, k + 1)
            assert _rel(X[k], ores["solutions"][k + 1]) <= _sol_tol(floor)


def test_batch_zero_rhs_and_cap(ctx, oracle, problems):
    from paper_2203_08498_b200 import api

    h = problems.generate(problems.CONFIGS["c1"])
    sa, _ = oracle.diagonal_scale(Matrix.of(h))
    ga = api.CsrMatrix(ctx, h.n, h.row_start, h.col_idx, sa.va)
    gf = api.IcFactor.factorize(ctx, h.n, h.row_start, h.col_idx, sa.va)
    B = np.stack([oracle.uniform_pm1(1, 0, h.n), np.zeros(h.n), oracle.uniform_pm1(2, 0, h.n)])
    X = np.ones_like(B)
    reps = api.pcg_solve_batch(ctx, ga, B, api.Ic(gf), X, 1e-8, 5000)
    assert reps[1].converged and reps[1].iterations == 0 and (X[1] == 0).all()
    assert reps[0].converged and reps[2].converged and reps[0].iterations > 10
    X = np.zeros_like(B)
    reps = api.pcg_solve_batch(ctx, ga, B, api.Ic(gf), X, 1e-8, 7)
    assert not reps[0].converged and reps[0].iterations == 7 and len(reps[0].history) == 7


def test_batch_is_deterministic(ctx, oracle, problems):
    from paper_2203_08498_b200 import api

    h = problems.generate(problems.SMALL["c2"])
    sa, _ = oracle.diagonal_scale(Matrix.of(h))
    ga = api.CsrMatrix(ctx, h.n, h.row_start, h.col_idx, sa.va)
    gf = api.IcFactor.factorize(ctx, h.n, h.row_start, h.col_idx, sa.va)
    B = np.stack([oracle.uniform_pm1(s, 0, h.n) for s in range(5)])
    X1, X2 = np.zeros_like(B), np.zeros_like(B)
    r1 = api.pcg_solve_batch(ctx, ga, B, api.Ic(gf), X1)
    r2 = api.pcg_solve_batch(ctx, ga, B, api.Ic(gf), X2)
    assert np.array_equal(X1, X2) and all(np.array_equal(a.history, b.history) for a, b in zip(r1, r2))


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
@pytest.mark.parametrize("nrhs", [4, 9, 19])
def test_grid_spmv_batched_bitwise(ctx, oracle, problems, name, nrhs):
    """Batched ICCG on the scaled-down cubes (7- and 27-point patterns), which the batched solver
    runs through the stencil-grid SpMV (shared-memory staged x-segments; RCG_GRID_SPMV=0 is the A/B
    switch), at RT 4 / 12 / 24 against the oracle's single solves: iterations +-2, solutions at
    equal counts."""
    from paper_2203_08498_b200 import api

    cfg = problems.SMALL[name]
    h = problems.generate(cfg)
    sa, _ = oracle.diagonal_scale(Matrix.of(h))
    ga = api.CsrMatrix(ctx, h.n, h.row_start, h.col_idx, sa.va)
    gf = api.IcFactor.factorize(ctx, h.n, h.row_start, h.col_idx, sa.va)
    B = np.stack([oracle.uniform_pm1(k + 1, 0, h.n) for k in range(nrhs)])
    X = np.zeros_like(B)
    reps = api.pcg_solve_batch(ctx, ga, B, api.Ic(gf), X, cfg.eps, cfg.max_iter)
    of = oracle.ic0_factorize(sa)
    for k in range(nrhs):
        xo = np.zeros(h.n)
        ro = oracle.pcg_solve(sa, B[k], xo, kind=1, ic=of, max_iter=cfg.max_iter)
        assert reps[k].converged and abs(reps[k].iterations - ro.iterations) <= 2
        if reps[k].iterations == ro.iterations:
            assert _rel(X[k], xo) <= 1e-7
