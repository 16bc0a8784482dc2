"""Every BASELINE matrix assembled on the device (rcg_matrix_generate) against the
host generator (csrc/generators.cpp, the shared definition of the BASELINE configs): row starts,
columns and values bitwise equal -- C1, the scaled-down C2 / C3 / C4 / C5, the full C2, C3 (449M
entries) and C5 (4M-point kNN) matrices."""
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["c1", "s_c2", "s_c3", "s_c4", "s_c5", "c2", "c3", "c5"])
def test_device_generator_bitwise(ctx, problems, name):
    cfg = problems.SMALL[name[2:]] if name.startswith("s_") else problems.CONFIGS[name]
    t0 = time.perf_counter()
    h = problems.generate(cfg)
    t1 = time.perf_counter()
    d = problems.generate_device(ctx, cfg)
    ctx.synchronize()
    t2 = time.perf_counter()
    rs, ci, va = d.export()
    assert d.n == h.n and d.nnz == h.nnz
    assert np.array_equal(rs, h.row_start) and np.array_equal(ci, h.col_idx) and np.array_equal(va, h.values)
    print(f"{cfg.name}: host {t1 - t0:.3f} s, device {t2 - t1:.3f} s")


def test_device_generator_knn_ragged_and_k(ctx, problems):
    """kNN edge cases: few points (a 1-cell bucket grid), k = 1 and k = 32 (the device limit)."""
    from dataclasses import replace

    base = problems.SMALL["c5"]
    for npts, k in ((40, 1), (40, 5), (300, 32), (2000, 10)):
        cfg = replace(base, grid=npts, knn_k=k)
        h = problems.generate(cfg)
        d = problems.generate_device(ctx, cfg)
        rs, ci, va = d.export()
        assert np.array_equal(rs, h.row_start) and np.array_equal(ci, h.col_idx) and np.array_equal(va, h.values), (npts, k)


def test_device_generator_rejects_bad_params(ctx, problems):
    from dataclasses import replace

    from paper_2203_08498_b200._lib import InvalidArgument

    with pytest.raises(InvalidArgument):
        problems.generate_device(ctx, replace(problems.SMALL["c5"], grid=100, knn_k=33))
    with pytest.raises(InvalidArgument):
        problems.generate_device(ctx, replace(problems.SMALL["c5"], grid=5, knn_k=10))
    with pytest.raises(InvalidArgument):
        problems.generate_device(ctx, replace(problems.SMALL["c3"], kind=7))
