"""IC(0) factorisation on the device (rcg_ic0_factorize_device): the factor --
L, D, U, shift used -- is bitwise the host restatement's (itself bitwise the reference's,
tests/test_oracle.py), for every config family, several block counts, and the shift ladder."""
import numpy as np
import pytest

from oracle import Matrix

pytestmark = pytest.mark.gpu


def _compare(ctx, oracle, n, rs, ci, va, nblocks):
    from paper_2203_08498_b200 import api

    a = api.CsrMatrix(ctx, n, rs, ci, va)
    fd = api.IcFactor.factorize_device(ctx, a, 0.0, nblocks)
    fo = oracle.ic0_factorize(Matrix(n, rs, ci, va), 0.0, nblocks)
    assert fd.shift_used == fo.shift_used and fd.nnz_l == fo.nnz_l
    ed, eo = fd.export(), fo.arrays()
    for k in ("block_bounds", "l_row_start", "l_col", "l_val", "d", "u_row_start", "u_col", "u_val"):
        assert np.array_equal(ed[k], eo[k]), k
    return fd


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
@pytest.mark.parametrize("nblocks", [1, 3])
def test_device_factor_is_bitwise_the_reference(ctx, oracle, problems, name, nblocks):
    h = problems.generate(problems.SMALL[name])
    sa, _ = oracle.diagonal_scale(Matrix.of(h))
    _compare(ctx, oracle, h.n, sa.rs, sa.ci, sa.va, nblocks)


def test_device_factor_applies_like_host_factor(ctx, oracle, problems):
    from paper_2203_08498_b200 import api

    h = problems.generate(problems.SMALL["c2"])
    sa, _ = oracle.diagonal_scale(Matrix.of(h))
    fd = _compare(ctx, oracle, h.n, sa.rs, sa.ci, sa.va, 1)
    fh = api.IcFactor.factorize(ctx, h.n, sa.rs, sa.ci, sa.va)
    r = oracle.uniform_pm1(3, 0, h.n)
    assert np.array_equal(fd.apply(r), fh.apply(r))
    assert (fd.fwd_levels, fd.bwd_levels) == (fh.fwd_levels, fh.bwd_levels)


def test_device_shift_ladder(ctx, oracle):
    from paper_2203_08498_b200 import api
    from paper_2203_08498_b200._lib import BreakdownError

    f = _compare(ctx, oracle, 2, np.array([0, 2, 4], np.int32), np.array([0, 1, 0, 1], np.int32),
                 np.array([1.0, 2.0, 2.0, 1.0]), 1)
    assert f.shift_used == pytest.approx(1.28)
    a = api.CsrMatrix(ctx, 2, np.array([0, 2, 4], np.int32), np.array([0, 1, 0, 1], np.int32),
                      np.array([1.0, 30000.0, 30000.0, 1.0]))
    with pytest.raises(BreakdownError):
        api.IcFactor.factorize_device(ctx, a)
