"""Pins the CPU oracle (oracle/oracle.c) before anything is checked against it:
  * against the reference's own known-answer tests (proj/tests/*.cpp), and
  * bitwise against the unmodified reference library (oracle/_ref) on seeded problems.
No GPU needed."""
import ctypes as C

import numpy as np
import pytest

from conftest import laplacian_2d, random_sdd_spd, spectral_fixture
from oracle import Breakdown, InvalidArgument, Matrix


# ------------------------------------------------------------------ RNG
def test_mt19937_64_known_answer(oracle):
    # the C++ standard fixes the 10000th output of a default-seeded mt19937_64
    class G(C.Structure):
        _fields_ = [("mt", C.c_uint64 * 312), ("idx", C.c_int)]

    g = G()
    oracle.lib.orc_mt64_seed(C.byref(g), C.c_uint64(5489))
    oracle.lib.orc_mt64_next.restype = C.c_uint64
    for _ in range(9999):
        oracle.lib.orc_mt64_next(C.byref(g))
    assert oracle.lib.orc_mt64_next(C.byref(g)) == 9981545732273789042


@pytest.mark.parametrize("seed,skip", [(1, 0), (42, 7), (12345, 1000)])
def test_uniform_stream_matches_generator_library(oracle, problems, seed, skip):
    # the product's host generator (std::mt19937_64) and the oracle's C restatement agree bitwise
    a = oracle.uniform_pm1(seed, skip, 5000)
    b = problems.uniform_pm1(seed, skip, 5000)
    assert np.array_equal(a, b)
    assert a.min() >= -1.0 and a.max() < 1.0


# ------------------------------------------------------------------ samplers (test_sampling.cpp)
def _feed(s, total, n=1):
    for i in range(1, total + 1):
        s.offer(i, 0.0, np.full(n, float(i)))


def test_sampler_golden_set(oracle, ref):
    s = oracle.sampler_a(4, 1000, 1)
    _feed(s, 1000)
    occ, it = s.state()
    assert set(it[occ].tolist()) == {256, 384, 512, 768}  # test_sampling.cpp:27-31
    for j in range(4):
        assert s.slot(j)[0] == float(it[j])
    r = ref.sampler_a(4, 1000)
    for i in range(1, 1001):
        ref.lib.ref_sampler_offer(r.h, i, 0.0, 1, np.array([float(i)]).ctypes.data)
    assert set(ref.sampler_state(r)[1].tolist()) == {256, 384, 512, 768}


@pytest.mark.parametrize("m", [2, 3, 4, 5, 8])
@pytest.mark.parametrize("total", [10, 37, 100, 400, 999])
def test_sampler_coverage_matches_reference(oracle, ref, m, total):
    if total < m:
        pytest.skip("fewer offers than slots")
    s = oracle.sampler_a(m, 1000, 1)
    _feed(s, total)
    occ, it = s.state()
    got = set(it[occ].tolist())
    assert len(got) == m and max(got) <= total and 2 * max(got) >= total  # test_sampling.cpp:42-58
    r = ref.sampler_a(m, 1000)
    for i in range(1, total + 1):
        ref.lib.ref_sampler_offer(r.h, i, 0.0, 1, np.array([float(i)]).ctypes.data)
    rocc, rit = ref.sampler_state(r)
    assert np.array_equal(occ, rocc) and np.array_equal(it, rit)


def test_sampler_method_b_crossings(oracle):
    s = oracle.sampler_b(3, 1e-8, 1)  # thresholds 1e-2, 1e-4, 1e-6 (test_sampling.cpp:66-83)
    s.offer(1, 0.5, np.array([1.0]))
    assert s.state()[0].sum() == 0
    s.offer(2, 1e-3, np.array([2.0]))
    occ, it = s.state()
    assert occ.sum() == 1 and it[0] == 2
    s.offer(3, 2e-3, np.array([3.0]))
    assert s.state()[0].sum() == 1 and s.slot(0)[0] == 2.0
    s.offer(4, 1e-7, np.array([4.0]))
    occ, it = s.state()
    assert occ.sum() == 3 and it[1] == 4 and it[2] == 4 and s.slot(2)[0] == 4.0


def test_sampler_validation(oracle):
    with pytest.raises(InvalidArgument):
        oracle.sampler_a(1, 100, 1)
    with pytest.raises(InvalidArgument):
        oracle.sampler_a(4, 0, 1)
    with pytest.raises(InvalidArgument):
        oracle.sampler_b(3, 1.0, 1)


# ------------------------------------------------------------------ IC(0) (test_preconditioners.cpp)
def test_ic_two_by_two_convention(oracle):
    a = Matrix(2, [0, 2, 4], [0, 1, 0, 1], [4.0, -1.0, -1.0, 4.0])
    f = oracle.ic0_factorize(a)
    arr = f.arrays()
    assert f.shift_used == 0.0 and f.nnz_l == 1
    assert arr["l_val"][0] == pytest.approx(-0.25)
    assert arr["d"].tolist() == pytest.approx([4.0, 3.75])


def test_ic_shift_ladder_reaches_1_28(oracle, ref):
    a = Matrix(2, [0, 2, 4], [0, 1, 0, 1], [1.0, 2.0, 2.0, 1.0])
    f = oracle.ic0_factorize(a)
    assert f.shift_used == pytest.approx(1.28)
    assert (f.arrays()["d"] > 0).all()
    assert ref.ic0(ref.matrix(a)).shift_used == f.shift_used


def test_ic_ladder_exhaustion_breaks_down(oracle):
    a = Matrix(2, [0, 2, 4], [0, 1, 0, 1], [1.0, 30000.0, 30000.0, 1.0])
    with pytest.raises(Breakdown):
        oracle.ic0_factorize(a)


def test_ic_block_count_validated(oracle):
    n, rs, ci, va = random_sdd_spd(10, 0.3, 43, oracle)
    a = Matrix(n, rs, ci, va)
    with pytest.raises(InvalidArgument):
        oracle.ic0_factorize(a, 0.0, 0)
    with pytest.raises(InvalidArgument):
        oracle.ic0_factorize(a, 0.0, 11)


def test_ic_reconstructs_pattern(oracle):
    n, rs, ci, va = random_sdd_spd(80, 0.06, 31, oracle)
    f = oracle.ic0_factorize(Matrix(n, rs, ci, va)).arrays()
    L = np.eye(n)
    for i in range(n):
        for p in range(f["l_row_start"][i], f["l_row_start"][i + 1]):
            L[i, f["l_col"][p]] = f["l_val"][p]
    ldlt = L @ np.diag(f["d"]) @ L.T
    for i in range(n):
        for p in range(rs[i], rs[i + 1]):
            j = ci[p]
            if j <= i:
                assert ldlt[i, j] == pytest.approx(va[p], rel=1e-10, abs=1e-12)


# ------------------------------------------------------------------ oracle == reference, bitwise
def _problem_set(oracle, problems):
    out = {}
    out["c1"] = problems.generate(problems.CONFIGS["c1"])
    out["c2s"] = problems.generate(problems.SMALL["c2"])
    out["c3s"] = problems.generate(problems.SMALL["c3"])
    out["c5s"] = problems.generate(problems.SMALL["c5"])
    n, rs, ci, va = random_sdd_spd(120, 0.05, 71, oracle)
    out["sdd"] = type("H", (), dict(n=n, row_start=rs, col_idx=ci, values=va))()
    n, rs, ci, va = laplacian_2d(20)
    out["lap2d"] = type("H", (), dict(n=n, row_start=rs, col_idx=ci, values=va))()
    return out


@pytest.fixture(scope="module")
def probs(oracle, problems):
    return _problem_set(oracle, problems)


@pytest.mark.parametrize("name", ["c1", "c2s", "c3s", "c5s", "sdd", "lap2d"])
def test_sparse_core_bitwise(oracle, ref, probs, name):
    h = probs[name]
    a = Matrix.of(h)
    m = ref.matrix(a)  # also runs the reference CsrMatrix::validate on the generated input
    x1, x2 = oracle.uniform_pm1(3, 0, a.n), oracle.uniform_pm1(4, 0, a.n)
    assert np.array_equal(oracle.spmv(a, x1), ref.spmv(m, x1))
    y1, y2 = oracle.spmv_dual(a, x1, x2)
    r1, r2 = ref.spmv_dual(m, x1, x2)
    assert np.array_equal(y1, r1) and np.array_equal(y2, r2)
    assert np.array_equal(y1, oracle.spmv(a, x1))  # spmv_dual == spmv (test_sparse_core.cpp:62-75)
    sa, dis = oracle.diagonal_scale(a)
    rva, rdis = ref.diagonal_scale(m, len(a.va))
    assert np.array_equal(sa.va, rva) and np.array_equal(dis, rdis)


@pytest.mark.parametrize("name", ["c1", "c2s", "c3s", "c5s", "sdd"])
@pytest.mark.parametrize("nblocks", [1, 4])
def test_ic_factor_and_apply_bitwise(oracle, ref, probs, name, nblocks):
    h = probs[name]
    a, _ = oracle.diagonal_scale(Matrix.of(h))
    f = oracle.ic0_factorize(a, 0.0, nblocks)
    rf = ref.ic0(ref.matrix(a), 0.0, nblocks)
    fa = f.arrays()
    for key, v in rf.arrays.items():
        assert np.array_equal(fa[key], v), key
    assert f.shift_used == rf.shift_used
    r = oracle.uniform_pm1(5, 0, a.n)
    assert np.array_equal(oracle.ic_apply(f, r), ref.ic_apply(rf, r))


@pytest.mark.parametrize("name", ["c1", "c2s", "c3s", "lap2d"])
def test_pcg_bitwise(oracle, ref, probs, name):
    h = probs[name]
    a, dis = oracle.diagonal_scale(Matrix.of(h))
    m = ref.matrix(a)
    f = oracle.ic0_factorize(a)
    rf = ref.ic0(m)
    b = oracle.uniform_pm1(1, 0, a.n)
    for kind in (0, 1):
        s = oracle.sampler_a(8, 2000, a.n)
        rs = ref.sampler_a(8, 2000)
        x = np.zeros(a.n)
        rx = np.zeros(a.n)
        rep = oracle.pcg_solve(a, b, x, kind=kind, ic=f if kind else None, max_iter=2000, sampler=s)
        prec = ref.prec_ic(rf) if kind else ref.prec_identity()
        rrep = ref.pcg_solve(m, b, prec, rx, max_iter=2000, sampler=rs)
        assert rep.iterations == rrep.iterations and rep.converged == rrep.converged
        assert np.array_equal(rep.history, rrep.history)
        assert np.array_equal(x, rx)
        occ, it = s.state()
        rocc, rit = ref.sampler_state(rs)
        assert np.array_equal(occ, rocc) and np.array_equal(it, rit)
        e = oracle.harvest_errors(x, s)
        re_ = ref.harvest_errors(rx, rs, a.n)
        assert np.array_equal(e, re_)
        mb, vals, w = oracle.build_aux(a, e, 0.05)
        rmb, rvals, rw = ref.build_aux(m, re_, 0.05)
        assert mb == rmb and np.array_equal(vals, rvals) and np.array_equal(w, rw)


@pytest.mark.parametrize("name", ["c1", "c2s", "c3s"])
def test_deflated_and_sc_bitwise(oracle, ref, probs, name):
    h = probs[name]
    a, dis = oracle.diagonal_scale(Matrix.of(h))
    m = ref.matrix(a)
    f = oracle.ic0_factorize(a)
    rf = ref.ic0(m)
    b0 = oracle.uniform_pm1(1, 0, a.n)
    s = oracle.sampler_a(16, 3000, a.n)
    x = np.zeros(a.n)
    oracle.pcg_solve(a, b0, x, kind=1, ic=f, max_iter=3000, sampler=s)
    _, _, w = oracle.build_aux(a, oracle.harvest_errors(x, s), float("inf"))
    w = w[:6]
    b = oracle.uniform_pm1(1, a.n, a.n)
    # deflation
    basis = oracle.basis(a, w, 0)
    x1, rx1 = np.zeros(a.n), np.zeros(a.n)
    r1 = oracle.deflated_pcg_solve(a, b, x1, basis, kind=1, ic=f, max_iter=3000)
    rr1 = ref.deflated_pcg_solve(m, b, ref.prec_ic(rf), ref.deflation(m, w), rx1, max_iter=3000)
    assert r1.iterations == rr1.iterations and np.array_equal(r1.history, rr1.history)
    assert np.array_equal(x1, rx1)
    # subspace correction
    sc = oracle.basis(a, w, 1)
    x2, rx2 = np.zeros(a.n), np.zeros(a.n)
    r2 = oracle.pcg_solve(a, b, x2, kind=2, ic=f, sc=sc, max_iter=3000)
    rr2 = ref.pcg_solve(m, b, ref.prec_sc(ref.prec_ic(rf), m, w), rx2, max_iter=3000)
    assert r2.iterations == rr2.iterations and np.array_equal(r2.history, rr2.history)
    assert np.array_equal(x2, rx2)
    # projections
    y = oracle.uniform_pm1(9, 0, a.n)
    assert np.array_equal(basis.project_pt(y), _ref_project(ref, m, w, y))


def _ref_project(ref, m, w, y):
    d = ref.deflation(m, w)
    out = np.empty(m.n)
    ref._chk(ref.lib.ref_project_pt(d.h, m.n, y.ctypes.data, out.ctypes.data))
    return out


@pytest.mark.parametrize("name,kind", [("lap2d", 0), ("c1", 1), ("c2s", 1)])
def test_condest_bitwise_and_rides_along(oracle, ref, probs, name, kind):
    h = probs[name]
    a, _ = oracle.diagonal_scale(Matrix.of(h))
    m = ref.matrix(a)
    f = oracle.ic0_factorize(a) if kind else None
    rf = ref.ic0(m) if kind else None
    b = oracle.uniform_pm1(1, 0, a.n)
    x, rx, xp = np.zeros(a.n), np.zeros(a.n), np.zeros(a.n)
    rep, est = oracle.pcg_with_condest(a, b, x, kind=kind, ic=f, max_iter=3000, m_samples=20)
    rrep, rest = ref.pcg_with_condest(m, b, ref.prec_ic(rf) if kind else ref.prec_identity(), rx, max_iter=3000,
                                      m_samples=20)
    assert rep.iterations == rrep.iterations and np.array_equal(x, rx)
    assert est.lambda_max == rest.lambda_max and est.power_unsettled == rest.power_unsettled
    assert np.array_equal(est.ritz_values, rest.ritz_values)
    assert est.kappa == rest.kappa or (np.isnan(est.kappa) and np.isnan(rest.kappa))
    plain = oracle.pcg_solve(a, b, xp, kind=kind, ic=f, max_iter=3000)  # test_condest.cpp:15-34
    assert plain.iterations == rep.iterations and np.array_equal(plain.history, rep.history)
    assert np.array_equal(xp, x)


def test_condest_known_answers(oracle):
    a = Matrix(2, [0, 1, 2], [0, 1], [0.1, 1.0])
    x = np.zeros(2)
    rep, est = oracle.pcg_with_condest(a, np.array([0.0, 1.0]), x, m_samples=20)
    assert rep.converged and rep.iterations == 1 and not est.lambda_min_available
    assert np.isnan(est.lambda_min) and np.isnan(est.kappa) and est.power_unsettled
    x = np.zeros(2)
    rep, est = oracle.pcg_with_condest(a, np.array([1e-3, 1.0]), x, m_samples=20)
    assert rep.iterations == 2 and est.lambda_min_available  # test_condest.cpp:112-127
    assert est.lambda_min == pytest.approx(0.1, rel=1e-6)


def test_dense_kernels_bitwise(oracle, ref):
    rng = np.random.default_rng(3)
    for k in (1, 2, 5, 17, 40):
        g = rng.standard_normal((k, k))
        s = g @ g.T + k * np.eye(k)
        s = np.triu(s) + np.triu(s, 1).T
        v1, q1 = oracle.sym_eig(s)
        v2, q2 = ref.sym_eig(s)
        assert np.array_equal(v1, v2) and np.array_equal(q1, q2)
        assert np.array_equal(oracle.chol_factor(s), ref.chol_factor(s))
        cols = rng.standard_normal((k, 200))
        assert np.array_equal(oracle.mgs(cols), ref.mgs(cols))


def test_rank_deficient_basis_rejected(oracle):
    n, rs, ci, va = random_sdd_spd(20, 0.2, 149, oracle)
    a = Matrix(n, rs, ci, va)
    c = oracle.uniform_pm1(14, 0, n)
    with pytest.raises(Breakdown):
        oracle.basis(a, np.stack([c, c]), 0)  # test_recycling.cpp:176-184


def test_deflating_exact_eigenvectors(oracle):
    n, rs, ci, va, lam, q = spectral_fixture(60, [1e-5, 1e-4, 1e-3], 77, oracle)
    a = Matrix(n, rs, ci, va)
    b = oracle.uniform_pm1(7, 0, n)
    xp = np.zeros(n)
    plain = oracle.pcg_solve(a, b, xp)
    basis = oracle.basis(a, q[:3], 0)
    xd = np.zeros(n)
    defl = oracle.deflated_pcg_solve(a, b, xd, basis, kind=0)
    assert plain.converged and defl.converged and defl.iterations < plain.iterations / 2
    r = b - oracle.spmv(a, xd)
    assert np.linalg.norm(r) / np.linalg.norm(b) <= 1e-7


def test_lanczos_extremes_closed_form(oracle):
    n, rs, ci, va = laplacian_2d(20)
    a, _ = oracle.diagonal_scale(Matrix(n, rs, ci, va))
    b = oracle.uniform_pm1(1, 0, n)
    x = np.zeros(n)
    rep = oracle.pcg_solve(a, b, x, max_iter=3000)
    lo, hi = oracle.lanczos_extremes(rep.alphas, rep.betas)
    c = np.cos(np.pi / 21)
    assert lo == pytest.approx(1 - c, rel=1e-6) and hi == pytest.approx(1 + c, rel=1e-6)


def test_oracle_c1_sequence_golden(oracle, problems):
    from oracle.sequence import run_sequence

    cfg = problems.CONFIGS["c1"]
    res = run_sequence(oracle, cfg, problems.generate(cfg))
    # SURVEY.md / BASELINE.md C1 probe: 34 ICCG iterations, sampled 2..32, deflated 29/29/30
    assert res["iterations"] == [34, 29, 29, 30]
    assert res["sampled_iterations"] == list(range(2, 33, 2))
    assert res["m_bar"] == 16 and res["m_tilde"] == 8
    assert all(r <= 1e-7 for r in res["true_relres"])
