"""Multicolour variant: a DIFFERENT operator (IC(0) of P A P^T), reported
separately.  Parity is against the reference run on the permuted matrix (same code, new input)."""
from dataclasses import replace

import numpy as np
import pytest

from oracle import Matrix


@pytest.mark.parametrize("name,colors", [("c1", 2), ("c2", 2), ("c3", 8), ("c4", 2)])
def test_colouring_and_depth(problems, ref, name, colors):
    h = problems.generate(problems.SMALL[name])
    m, perm, nc = problems.multicolour(h)
    assert nc == colors
    assert sorted(perm.tolist()) == list(range(h.n))
    assert problems.level_depth(m) == nc  # IC(0) of P A P^T: one level per colour
    ref.matrix(Matrix.of(m))  # still a valid reference CsrMatrix (sorted, symmetric)
    # B[new(i), new(j)] = A[i, j]
    dense_idx = {(perm[i], perm[h.col_idx[p]]): h.values[p] for i in range(min(h.n, 200))
                 for p in range(h.row_start[i], h.row_start[i + 1])}
    for (r, c), v in list(dense_idx.items())[:500]:
        row = slice(m.row_start[r], m.row_start[r + 1])
        k = list(m.col_idx[row]).index(c)
        assert m.values[row][k] == v


def test_oracle_multicolour_sequence_pinned(oracle, ref, problems):
    """Oracle == reference, bitwise, on the permuted C1 problem (ICCG solve)."""
    h = problems.generate(problems.CONFIGS["c1"])
    m, perm, nc = problems.multicolour(h)
    a, _ = oracle.diagonal_scale(Matrix.of(m))
    rm = ref.matrix(a)
    f = oracle.ic0_factorize(a)
    rf = ref.ic0(rm)
    b = oracle.uniform_pm1(1, 0, m.n)
    x, rx = np.zeros(m.n), np.zeros(m.n)
    r1 = oracle.pcg_solve(a, b, x, kind=1, ic=f)
    r2 = ref.pcg_solve(rm, b, ref.prec_ic(rf), rx)
    assert r1.iterations == r2.iterations and np.array_equal(x, rx)


def test_multicolour_costs_more_iterations(oracle, problems):
    """red-black needs about 1.6x the ICCG iterations of natural order."""
    from oracle.sequence import run_sequence

    cfg = replace(problems.CONFIGS["c1"], n_rhs=2)
    h = problems.generate(cfg)
    nat = run_sequence(oracle, cfg, h)
    m, perm, nc = problems.multicolour(h)
    mc = run_sequence(oracle, cfg, m, new_of_old=perm)
    ratio = mc["iterations"][0] / nat["iterations"][0]
    assert 1.2 <= ratio <= 2.2, (mc["iterations"], nat["iterations"])
