"""The 7-point generators assembled on the device (rcg_matrix_generate) against the
host generator (csrc/generators.cpp, the shared definition of the BASELINE configs): row starts,
columns and values bitwise equal, for C1, the scaled-down C2 / C4 and the full C2 matrix."""
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["c1", "s_c2", "s_c4", "c2"])
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


def test_device_generator_rejects_other_kinds(ctx, problems):
    from paper_2203_08498_b200._lib import InvalidArgument

    with pytest.raises(InvalidArgument):
        problems.generate_device(ctx, problems.SMALL["c3"])
