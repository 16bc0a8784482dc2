"""The IC sweep variants -- grid-wide sync-free (k_sweep) and one launch per level
(csrc/icsweep_lv.cu) -- against each other and the oracle: the sweep output, the (r, z) reduction and whole PCG / SC-PCG solves must be BITWISE
identical whichever kernel runs (the kernel choice never changes an iterate), and all equal the
reference ic_apply (src/ic_preconditioner.cpp:123-144)."""
import numpy as np
import pytest

from oracle import Matrix

pytestmark = pytest.mark.gpu

GRID, AUTO, LEVEL = 0, 2, 4
MODES = (GRID, AUTO, LEVEL)


@pytest.fixture
def modes(ctx):
    yield ctx
    ctx.set_sweep_kernel(AUTO)


def _scaled(ctx, h):
    from paper_2203_08498_b200 import api

    a = api.CsrMatrix(ctx, h.n, h.row_start, h.col_idx, h.values)
    return api.diagonal_scale(ctx, a)


def _dense_csr(problems, dense):
    n = dense.shape[0]
    rs, ci, va = [0], [], []
    for i in range(n):
        for j in range(n):
            if dense[i, j] != 0.0 or i == j:
                ci.append(j), va.append(dense[i, j])
        rs.append(len(ci))
    return problems.HostCsr(n, np.array(rs, np.int32), np.array(ci, np.int32), np.array(va))


def _edge(problems, name):
    """The edge matrices of test_gpu_edges.py: 1 x 1, diagonal (one level), arrow (ragged rows:
    row 0 couples to every row, so level 1 holds n - 1 rows of 2-3 entries)."""
    if name == "one":
        return _dense_csr(problems, np.array([[4.0]]))
    if name == "diag":
        return _dense_csr(problems, np.diag(np.arange(1.0, 70.0)))
    n = 300
    rng = np.random.default_rng(3)
    a = np.zeros((n, n))
    a[0, 1:] = a[1:, 0] = -rng.uniform(0.1, 1.0, n - 1) / n
    for i in range(1, n - 1):
        a[i, i + 1] = a[i + 1, i] = -0.3
    a[np.arange(n), np.arange(n)] = 2.0
    return _dense_csr(problems, a)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5", "lap1d", "one", "diag", "arrow"])
def test_sweep_variants_bitwise(modes, oracle, problems, name):
    from paper_2203_08498_b200 import api

    ctx = modes
    if name == "lap1d":  # a chain: n levels of one row (every level narrower than a warp)
        n = 300
        rs = np.concatenate([[0], np.cumsum([2 if i in (0, n - 1) else 3 for i in range(n)])]).astype(np.int32)
        ci, va = [], []
        for i in range(n):
            for j in (i - 1, i, i + 1):
                if 0 <= j < n:
                    ci.append(j), va.append(2.0 if j == i else -1.0)
        h = problems.HostCsr(n, rs, np.array(ci, np.int32), np.array(va))
    elif name in ("one", "diag", "arrow"):
        h = _edge(problems, name)
    else:
        h = problems.generate(problems.SMALL[name])
    sa, _ = _scaled(ctx, h)
    f = api.IcFactor.factorize_device(ctx, sa)
    a_o, _ = oracle.diagonal_scale(Matrix.of(h))
    want = oracle.ic_apply(oracle.ic0_factorize(a_o), oracle.uniform_pm1(5, 0, h.n))
    r = oracle.uniform_pm1(5, 0, h.n)
    outs = {}
    for mode in MODES:
        ctx.set_sweep_kernel(mode)
        outs[mode] = f.apply(r)
    for mode in MODES:
        assert np.array_equal(outs[mode], want), mode


@pytest.mark.parametrize("method", ["ic", "sc"])
def test_sweep_variant_solves_bitwise(modes, problems, method):
    """IC-PCG (rho from the backward sweep's fused reduction) and SC-PCG on C1: identical
    iterates, histories and solutions under both kernels."""
    from paper_2203_08498_b200 import api, sequence

    ctx = modes
    cfg = problems.CONFIGS["c1"]
    h = problems.generate(cfg)
    p = sequence.prepare(ctx, cfg, h, validate=False)
    b = sequence.rhs(p, 0)[1]
    res = {}
    for mode in MODES:
        ctx.set_sweep_kernel(mode)
        if method == "ic":
            x = np.zeros(h.n)
            rep = api.pcg_solve(ctx, p.a, b, api.Ic(p.ic), x, cfg.eps, cfg.max_iter)
        else:
            s = api.SamplerState.method_a(ctx, cfg.sampler_m, cfg.max_iter, h.n)
            x0 = np.zeros(h.n)
            api.pcg_solve(ctx, p.a, b, api.Ic(p.ic), x0, cfg.eps, cfg.max_iter, observer=s)
            _, _, _, w = api.build_aux_matrix(ctx, p.a, api.harvest_errors(ctx, x0, s), 1e-3, keep_count=cfg.keep)
            basis = api.Basis(ctx, p.a, w, "sc")
            x = np.zeros(h.n)
            rep = api.pcg_solve(ctx, p.a, sequence.rhs(p, 1)[1], api.Sc(basis, p.ic), x, cfg.eps, cfg.max_iter)
        res[mode] = (rep.iterations, np.array(rep.history), x.copy())
    for mode in MODES:
        assert res[GRID][0] == res[mode][0]
        assert np.array_equal(res[GRID][1], res[mode][1])
        assert np.array_equal(res[GRID][2], res[mode][2])


def test_sweep_variants_c2_full(modes, problems):
    """The bench matrix (C2, 382 levels): sweep output bitwise across kernels and an ICCG
    window with identical histories."""
    from paper_2203_08498_b200 import api, sequence

    ctx = modes
    cfg = problems.CONFIGS["c2"]
    h = problems.generate(cfg)
    p = sequence.prepare(ctx, cfg, h, validate=False)
    r = problems.uniform_pm1(9, 0, h.n)
    b = sequence.rhs(p, 0)[1]
    outs = {}
    for mode in MODES:
        ctx.set_sweep_kernel(mode)
        z = p.ic.apply(r)
        x = np.zeros(h.n)
        rep = api.pcg_solve(ctx, p.a, b, api.Ic(p.ic), x, cfg.eps, 40)
        outs[mode] = (z, np.array(rep.history), x)
    for mode in MODES:
        for k in range(3):
            assert np.array_equal(outs[GRID][k], outs[mode][k])


def test_wide_level_sweeps_multicolour_c2(modes, problems):
    """The wide-level variants on the multicolour C2 operator (2 levels of ~1M rows: the default
    picks the per-level launches): bitwise the grid sweep, sweep output and an ICCG window."""
    from paper_2203_08498_b200 import api, sequence

    ctx = modes
    cfg = problems.CONFIGS["c2"]
    m, perm, _ = problems.multicolour(problems.generate(cfg))
    p = sequence.prepare(ctx, cfg, m, validate=False, new_of_old=perm)
    r = problems.uniform_pm1(9, 0, m.n)
    b = sequence.rhs(p, 0)[1]
    outs = {}
    for mode in (GRID, LEVEL, AUTO):
        ctx.set_sweep_kernel(mode)
        z = p.ic.apply(r)
        x = np.zeros(m.n)
        rep = api.pcg_solve(ctx, p.a, b, api.Ic(p.ic), x, cfg.eps, 30)
        outs[mode] = (z, np.array(rep.history), x)
    for mode in (LEVEL, AUTO):
        for k in range(3):
            assert np.array_equal(outs[GRID][k], outs[mode][k]), mode


@pytest.mark.parametrize("method", ["ic", "sc"])
def test_batched_level_sweeps_multicolour(modes, problems, method):
    """Batched solves on the multicolour C2 operator with the batched sweeps one launch per level
    (k_b_level; the default picks it for these 1M-row levels) against the polling batched sweep:
    the rows are the same arithmetic and only the (r, z) summation order differs, so iterations
    agree within 1 and solutions to rounding."""
    from paper_2203_08498_b200 import api, sequence

    ctx = modes
    cfg = problems.CONFIGS["c2"]
    m, perm, _ = problems.multicolour(problems.generate(cfg))
    p = sequence.prepare(ctx, cfg, m, validate=False, new_of_old=perm)
    B = np.stack([sequence.rhs(p, k)[1] for k in range(3)])
    prec = api.Ic(p.ic)
    if method == "sc":
        rng = np.random.default_rng(1)
        basis = api.Basis(ctx, p.a, api.TallDense.from_columns(ctx, m.n, rng.standard_normal((4, m.n))), "sc")
        prec = api.Sc(basis, p.ic)
    out = {}
    for mode in (GRID, LEVEL, AUTO):
        ctx.set_sweep_kernel(mode)
        X = np.zeros_like(B)
        reps = api.pcg_solve_batch(ctx, p.a, B, prec, X, cfg.eps, 400)
        out[mode] = ([r.iterations for r in reps], X)
    for mode in (LEVEL, AUTO):
        assert all(abs(a - b) <= 1 for a, b in zip(out[mode][0], out[GRID][0])), (out[mode][0], out[GRID][0])
        for k in range(3):
            x0 = out[GRID][1][k]
            assert np.linalg.norm(out[mode][1][k] - x0) <= 1e-6 * np.linalg.norm(x0)

