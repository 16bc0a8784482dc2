"""Concurrent accelerated solves (sequence.run_accelerated) must reproduce the serial solves bit
for bit: each solve owns a context (stream + workspace) and every reduction is deterministic."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("method", ["sc", "deflation"])
@pytest.mark.parametrize("concurrency", [2, 3, 8])
def test_concurrent_equals_serial(ctx, problems, method, concurrency):
    from dataclasses import replace

    from paper_2203_08498_b200 import api, sequence

    cfg = replace(problems.SMALL["c2"], method=method, n_rhs=7)
    h = problems.generate(cfg)
    p = sequence.prepare(ctx, cfg, h)
    pairs = [sequence.rhs(p, k) for k in range(cfg.n_rhs)]
    bs = [s for _, s in pairs]
    x1 = np.zeros(h.n)
    smp = api.SamplerState.method_a(ctx, cfg.sampler_m, cfg.max_iter, h.n)
    api.pcg_solve(ctx, p.a, bs[0], api.Ic(p.ic), x1, cfg.eps, cfg.max_iter, observer=smp)
    _, _, _, w = api.build_aux_matrix(ctx, p.a, api.harvest_errors(ctx, x1, smp), 1e-3, keep_count=cfg.keep)
    basis = api.Basis(ctx, p.a, w, "sc" if method == "sc" else "deflation")
    xs_serial = [np.zeros(h.n) for _ in bs[1:]]
    xs_conc = [np.zeros(h.n) for _ in bs[1:]]
    r_serial = sequence.run_accelerated(p, basis, bs[1:], xs_serial, 1)
    r_conc = sequence.run_accelerated(p, basis, bs[1:], xs_conc, concurrency)
    for a, b, xa, xb in zip(r_serial, r_conc, xs_serial, xs_conc):
        assert a.iterations == b.iterations and a.converged and b.converged
        assert np.array_equal(a.history, b.history) and np.array_equal(xa, xb)
