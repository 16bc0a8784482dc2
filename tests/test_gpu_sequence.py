"""The device sequence driver (rcg_seq_prepare / rcg_seq_run, run_sequence driver.cpp:108-222)
against the oracle's sequence (pinned to the reference): same m_bar / m_tilde, Ritz values
<= 1e-6, iterations +-2 per solve, true relative residuals; solutions by the parity protocol --
solve 1 (same operator on both sides) at max(1e-8, 10 x the oracle's rounding floor) when the
counts agree, solves 2..k by the shared-input protocol (the GPU's batched accelerated solves run
on the oracle's W, then the same bar), every achieved difference logged (parity_log)."""
from dataclasses import replace

import numpy as np
import pytest

from oracle import Matrix
from test_gpu_parity import _oracle_floor, _rel, _sol_tol

pytestmark = pytest.mark.gpu


def _solution_protocol(ctx, oracle, cfg, h, ores, rep, X, dis, parity_log, tag, shared_solves=None):
    """Solve 1 at the floor; solves 2..k (or the listed ones) re-run as ONE batched GPU solve on
    the oracle's W and compared at equal counts against the oracle's solutions."""
    from paper_2203_08498_b200 import api

    if rep["iterations"][0] == ores["iterations"][0]:
        rel = _rel(X[0], dis * ores["solutions"][0])
        bar = _sol_tol(_oracle_floor(oracle, cfg, h, ores, 0))
        parity_log(tag, check="solve1_solution_rel", achieved=rel, bar=bar)
        assert rel <= bar, (rel, bar)
    ks = list(range(1, len(ores["iterations"]))) if shared_solves is None else list(shared_solves)
    if not ks or ores["m_tilde"] == 0:
        return
    sa, _ = oracle.diagonal_scale(Matrix.of(h))
    ga = api.CsrMatrix(ctx, h.n, h.row_start, h.col_idx, sa.va)
    gf = api.IcFactor.factorize_device(ctx, ga)
    kind = "sc" if cfg.method == "sc" else "deflation"
    basis = api.Basis(ctx, ga, api.TallDense.from_columns(ctx, h.n, ores["w"]), kind)
    B = np.stack([ores["scaled_rhs"][k] for k in ks])
    Xs = np.zeros_like(B)
    if kind == "sc":
        reps = api.pcg_solve_batch(ctx, ga, B, api.Sc(basis, gf), Xs, cfg.eps, cfg.max_iter)
    else:
        reps = api.deflated_pcg_solve_batch(ctx, ga, B, api.Ic(gf), basis, Xs, cfg.eps, cfg.max_iter)
    for j, k in enumerate(ks):
        assert abs(reps[j].iterations - ores["iterations"][k]) <= 2, (k, reps[j].iterations, ores["iterations"][k])
        if reps[j].iterations == ores["iterations"][k]:
            rel = _rel(Xs[j], ores["solutions"][k])
            bar = _sol_tol(_oracle_floor(oracle, cfg, h, ores, k))
            parity_log(tag, check=f"shared_input_solve{k + 1}_solution_rel", achieved=rel, bar=bar)
            assert rel <= bar, (k, rel, bar)


@pytest.mark.parametrize("name", ["c1", "c2", "c4"])
@pytest.mark.parametrize("method", ["sc", "deflation"])
@pytest.mark.parametrize("batch", [True, False])
def test_device_sequence_matches_oracle(ctx, oracle, problems, parity_log, name, method, batch):
    from oracle.sequence import rhs_set, run_sequence as oracle_sequence
    from paper_2203_08498_b200 import api

    cfg = replace(problems.SMALL[name], method=method, n_rhs=5)
    h = problems.generate(cfg)
    ores = oracle_sequence(oracle, cfg, h)
    a_o = Matrix.of(h)
    _, dis = oracle.diagonal_scale(a_o)
    b_orig, _ = rhs_set(oracle, cfg, h, a_o, dis)
    B = np.stack(b_orig)
    X = np.zeros_like(B)
    a = api.CsrMatrix(ctx, h.n, h.row_start, h.col_idx, h.values)
    seq = api.Sequence(ctx, a, "es-sc-iccg" if method == "sc" else "es-d-iccg")
    rep = seq.run(B, X, cfg.eps, cfg.max_iter, "A", cfg.sampler_m, keep_count=cfg.keep, batch=batch)
    assert rep["m_bar"] == ores["m_bar"] and rep["m_tilde"] == ores["m_tilde"]
    rv = np.asarray(ores["ritz_values"])[:rep["m_bar"]]
    assert np.max(np.abs(rep["ritz_values"] - rv) / np.maximum(np.abs(rv), 1e-300)) <= 1e-6
    for k in range(cfg.n_rhs):
        assert rep["converged"][k]
        assert abs(rep["iterations"][k] - ores["iterations"][k]) <= 2, (k, rep["iterations"], ores["iterations"])
        assert rep["true_relres"][k] <= 10 * cfg.eps * 1e3 and abs(rep["true_relres"][k] - ores["true_relres"][k]) <= 1e-6
    if batch:  # the protocol once per (config, method); the unbatched run repeats the same arithmetic
        _solution_protocol(ctx, oracle, cfg, h, ores, rep, X, dis, parity_log, f"sequence:{cfg.name}:{method}")


def test_device_sequence_plain_methods(ctx, oracle, problems):
    from oracle.sequence import rhs_set
    from paper_2203_08498_b200 import api

    cfg = replace(problems.SMALL["c1"], n_rhs=3)
    h = problems.generate(cfg)
    a_o = Matrix.of(h)
    sa, dis = oracle.diagonal_scale(a_o)
    b_orig, bs = rhs_set(oracle, cfg, h, a_o, dis)
    a = api.CsrMatrix(ctx, h.n, h.row_start, h.col_idx, h.values)
    for method, kind in (("iccg", 1), ("cg", 0)):
        X = np.zeros((3, h.n))
        rep = api.Sequence(ctx, a, method).run(np.stack(b_orig), X, cfg.eps, cfg.max_iter)
        assert rep["m_tilde"] == 0 and not rep["acceleration_inactive"]
        f = oracle.ic0_factorize(sa) if kind == 1 else None
        for k in range(3):
            xo = np.zeros(h.n)
            ro = oracle.pcg_solve(sa, bs[k], xo, kind=kind, ic=f, max_iter=cfg.max_iter)
            assert abs(rep["iterations"][k] - ro.iterations) <= 2


def test_device_sequence_config_errors(ctx, problems):
    from paper_2203_08498_b200 import api
    from paper_2203_08498_b200._lib import ParseError

    h = problems.generate(problems.SMALL["c1"])
    a = api.CsrMatrix(ctx, h.n, h.row_start, h.col_idx, h.values)
    with pytest.raises(ParseError):
        api.Sequence(ctx, a, "gmres")
    seq = api.Sequence(ctx, a, "iccg")
    with pytest.raises(ParseError):
        seq.run(np.zeros((2, h.n)), np.zeros((2, h.n)), eps=2.0)


@pytest.mark.parametrize("name", ["c5", "c1"])
@pytest.mark.parametrize("batch", [True, False])
def test_sequence_lanczos_condest_each_solve(ctx, oracle, problems, name, batch):
    """C5's protocol: a Lanczos condition-number estimate on every solve of the sequence, from
    the solve's own CG alpha / beta (batched solves record them per right-hand
    side) -- within the north star's 1 % of the oracle's estimate from its alpha / beta."""
    from oracle.sequence import rhs_set, run_sequence as oracle_sequence
    from paper_2203_08498_b200 import api

    cfg = replace(problems.SMALL[name], n_rhs=4)
    h = problems.generate(cfg)
    ores = oracle_sequence(oracle, cfg, h)
    a_o = Matrix.of(h)
    _, dis = oracle.diagonal_scale(a_o)
    b_orig, _ = rhs_set(oracle, cfg, h, a_o, dis)
    X = np.zeros((cfg.n_rhs, h.n))
    a = api.CsrMatrix(ctx, h.n, h.row_start, h.col_idx, h.values)
    seq = api.Sequence(ctx, a, "es-sc-iccg" if cfg.method == "sc" else "es-d-iccg")
    rep = seq.run(np.stack(b_orig), X, cfg.eps, cfg.max_iter, "A", cfg.sampler_m, keep_count=cfg.keep, batch=batch,
                  condest=True)
    for k in range(cfg.n_rhs):
        lo, hi = oracle.lanczos_extremes(ores["alphas"][k], ores["betas"][k])
        assert abs(rep["kappa"][k] / (hi / lo) - 1.0) <= 0.01, (k, rep["kappa"][k], hi / lo)
        assert rep["lambda_min"][k] > 0 and rep["lambda_max"][k] >= rep["lambda_min"][k]
    assert rep["kappa"][1] < rep["kappa"][0]  # the accelerated operator is better conditioned


@pytest.mark.parametrize("name", ["c1", "c2", "c4"])
def test_lean_sequence_matches_oracle(ctx, oracle, problems, name):
    """The memory-lean recycling step (errors / MGS in the sampler slots, streamed Gram, the basis
    adopting W -- what C4 needs on one GPU), forced on small configs: same m_bar / m_tilde, Ritz
    values <= 1e-6, iterations +-2 as the oracle's sequence."""
    from oracle.sequence import rhs_set, run_sequence as oracle_sequence
    from paper_2203_08498_b200 import api

    cfg = replace(problems.SMALL[name], n_rhs=4)
    h = problems.generate(cfg)
    ores = oracle_sequence(oracle, cfg, h)
    a_o = Matrix.of(h)
    _, dis = oracle.diagonal_scale(a_o)
    b_orig, _ = rhs_set(oracle, cfg, h, a_o, dis)
    X = np.zeros((cfg.n_rhs, h.n))
    a = api.CsrMatrix(ctx, h.n, h.row_start, h.col_idx, h.values)
    seq = api.Sequence(ctx, a, "es-sc-iccg" if cfg.method == "sc" else "es-d-iccg")
    rep = seq.run(np.stack(b_orig), X, cfg.eps, cfg.max_iter, "A", cfg.sampler_m, keep_count=cfg.keep, lean=True)
    assert rep["m_bar"] == ores["m_bar"] and rep["m_tilde"] == ores["m_tilde"]
    rv = np.asarray(ores["ritz_values"])[:rep["m_bar"]]
    assert np.max(np.abs(rep["ritz_values"] - rv) / np.maximum(np.abs(rv), 1e-300)) <= 1e-6
    for k in range(cfg.n_rhs):
        assert rep["converged"][k] and abs(rep["iterations"][k] - ores["iterations"][k]) <= 2


def test_full_size_c2_sequence_matches_oracle(ctx, oracle, problems, parity_log):
    """The bench workload itself at full size (C2: 128^3 high-contrast FV, 2.1M rows, 10 RHS, 32
    samples, SC m~ = 16) through the device sequence driver against the oracle's sequence (about a
    minute of CPU): m_bar / m_tilde, Ritz values <= 1e-6, every solve +-2 iterations, true relative
    residuals, solutions at equal iteration counts."""
    from oracle.sequence import rhs_set, run_sequence as oracle_sequence
    from paper_2203_08498_b200 import api

    cfg = problems.CONFIGS["c2"]
    h = problems.generate(cfg)
    ores = oracle_sequence(oracle, cfg, h)
    a_o = Matrix.of(h)
    _, dis = oracle.diagonal_scale(a_o)
    b_orig, _ = rhs_set(oracle, cfg, h, a_o, dis)
    X = np.zeros((cfg.n_rhs, h.n))
    a = api.CsrMatrix(ctx, h.n, h.row_start, h.col_idx, h.values)
    rep = api.Sequence(ctx, a, "es-sc-iccg").run(np.stack(b_orig), X, cfg.eps, cfg.max_iter, "A", cfg.sampler_m,
                                                 keep_count=cfg.keep)
    assert rep["m_bar"] == ores["m_bar"] and rep["m_tilde"] == ores["m_tilde"]
    rv = np.asarray(ores["ritz_values"])[:rep["m_bar"]]
    ritz = float(np.max(np.abs(rep["ritz_values"] - rv) / np.maximum(np.abs(rv), 1e-300)))
    parity_log("sequence:c2_full", check="ritz_rel", achieved=ritz, bar=1e-6,
               iterations_gpu=rep["iterations"], iterations_oracle=ores["iterations"])
    assert ritz <= 1e-6, ritz
    for k in range(cfg.n_rhs):
        assert rep["converged"][k]
        assert abs(rep["iterations"][k] - ores["iterations"][k]) <= 2, (k, rep["iterations"], ores["iterations"])
        assert abs(rep["true_relres"][k] - ores["true_relres"][k]) <= 1e-6
    # solve 1 at the floor; the shared-input protocol on two accelerated solves (each floor costs
    # three oracle solves of the full C2)
    _solution_protocol(ctx, oracle, cfg, h, ores, rep, X, dis, parity_log, "sequence:c2_full", shared_solves=(1, 2))
