"""Multi-GPU row slabs on the device (rcg_dist_pcg_solve).  Only one GPU is available, so the
distributed iteration runs with the loopback transport (all G slabs in one process, each on its
own stream; exchanges are stream-ordered device copies, reductions a fixed-order sum -- no slab
waits on another inside a kernel), and the NCCL transport at world size 1.  The bar is the
oracle's single-process block-Jacobi PCG (ic0_factorize(a, 0, G), pinned to the reference):
iterations +-2, solution within max(1e-8, 10 x the oracle's own reduction-order response).
"""
import os
import socket

import numpy as np
import pytest

from oracle import Matrix

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _scaled(oracle, problems, name):
    h = problems.generate(problems.SMALL[name])
    sa, _ = oracle.diagonal_scale(Matrix.of(h))
    return sa, problems.HostCsr(h.n, sa.rs, sa.ci, sa.va)


def _oracle_block_jacobi(oracle, sa, b, nparts, kind=1, eps=1e-8, max_iter=5000):
    f = oracle.ic0_factorize(sa, 0.0, nparts) if kind == 1 else None
    xo = np.zeros(sa.n)
    ro = oracle.pcg_solve(sa, b, xo, kind=kind, ic=f, eps=eps, max_iter=max_iter)
    with oracle.reversed_dots(1):
        x2 = np.zeros(sa.n)
        oracle.pcg_solve(sa, b, x2, kind=kind, ic=f, eps=eps, max_iter=max_iter)
    return ro, xo, max(1e-8, 10 * _rel(x2, xo))


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
@pytest.mark.parametrize("nparts", [1, 2, 3, 4])
def test_loopback_matches_block_jacobi_pcg(oracle, problems, name, nparts):
    from paper_2203_08498_b200 import dist

    sa, host = _scaled(oracle, problems, name)
    b = oracle.uniform_pm1(5, 0, sa.n)
    system = dist.LoopbackSystem(host, nparts)
    x = np.zeros(sa.n)
    rep = system.solve(b, x, 1e-8, 5000)
    ro, xo, tol = _oracle_block_jacobi(oracle, sa, b, nparts)
    assert rep.converged and ro.converged
    assert abs(rep.iterations - ro.iterations) <= 2, (rep.iterations, ro.iterations)
    if rep.iterations == ro.iterations:
        assert _rel(x, xo) <= tol, (_rel(x, xo), tol)
    assert len(rep.history) == rep.iterations and rep.history[-1] <= 1e-8


def test_loopback_identity_preconditioner(oracle, problems):
    from paper_2203_08498_b200 import dist

    sa, host = _scaled(oracle, problems, "c1")
    b = oracle.uniform_pm1(9, 0, sa.n)
    system = dist.LoopbackSystem(host, 3, preconditioner="identity")
    x = np.zeros(sa.n)
    rep = system.solve(b, x, 1e-8, 5000)
    ro, xo, tol = _oracle_block_jacobi(oracle, sa, b, 3, kind=0)
    assert rep.converged and abs(rep.iterations - ro.iterations) <= 2
    if rep.iterations == ro.iterations:
        assert _rel(x, xo) <= tol


def test_loopback_zero_rhs_and_cap(oracle, problems):
    from paper_2203_08498_b200 import dist

    sa, host = _scaled(oracle, problems, "c1")
    system = dist.LoopbackSystem(host, 2)
    x = np.ones(sa.n)
    rep = system.solve(np.zeros(sa.n), x)
    assert rep.converged and rep.iterations == 0 and not x.any()
    x = np.zeros(sa.n)
    rep = system.solve(oracle.uniform_pm1(3, 0, sa.n), x, 1e-10, 7)
    assert not rep.converged and rep.iterations == 7 and len(rep.history) == 7


@pytest.mark.parametrize("method", ["deflation", "sc"])
@pytest.mark.parametrize("name", ["c1", "c2"])
@pytest.mark.parametrize("nparts", [1, 2, 3])
def test_loopback_deflated_and_sc_match_block_jacobi(oracle, problems, name, method, nparts):
    """Row-partitioned W: distributed deflated PCG / SC-PCG against the oracle's single-process
    solve with the same W and the block-Jacobi IC(0) of the same bounds."""
    from paper_2203_08498_b200 import dist

    sa, host = _scaled(oracle, problems, name)
    f = oracle.ic0_factorize(sa, 0.0, nparts)
    # W: error samples of an oracle solve (the sequence's construction, small m)
    s_o = oracle.sampler_a(8, 5000, sa.n)
    x1 = np.zeros(sa.n)
    oracle.pcg_solve(sa, oracle.uniform_pm1(2, 0, sa.n), x1, kind=1, ic=f, max_iter=5000, sampler=s_o)
    occ, _ = s_o.state()
    w = np.stack([x1 - s_o.slot(j) for j in range(8) if occ[j]])
    w /= np.linalg.norm(w, axis=1, keepdims=True)
    b = oracle.uniform_pm1(17, 0, sa.n)
    ob = oracle.basis(sa, w, 0 if method == "deflation" else 1)
    xo = np.zeros(sa.n)
    if method == "deflation":
        ro = oracle.deflated_pcg_solve(sa, b, xo, ob, kind=1, ic=f, max_iter=5000)
    else:
        ro = oracle.pcg_solve(sa, b, xo, kind=2, ic=f, sc=ob, max_iter=5000)
    system = dist.LoopbackSystem(host, nparts)
    db = system.basis(w, method)
    x = np.zeros(sa.n)
    rep = system.solve(b, x, 1e-8, 5000, basis=db)
    assert rep.converged and ro.converged
    assert abs(rep.iterations - ro.iterations) <= 2, (rep.iterations, ro.iterations)
    if rep.iterations == ro.iterations:
        assert _rel(x, xo) <= 1e-6, _rel(x, xo)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_nccl_transport_world_one_equals_loopback(oracle, problems):
    """The NCCL transport (one slab per process) at world size 1: bitwise the loopback G = 1."""
    import torch
    import torch.distributed as dist_

    from paper_2203_08498_b200 import dist

    sa, host = _scaled(oracle, problems, "c2")
    b = oracle.uniform_pm1(21, 0, sa.n)
    lb = dist.LoopbackSystem(host, 1)
    x1 = np.zeros(sa.n)
    r1 = lb.solve(b, x1)
    bs = [oracle.uniform_pm1(31 + k, 0, sa.n) for k in range(3)]
    q1 = lb.sequence(bs, 1e-8, 2000, 16, 6, "sc")
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    torch.cuda.set_device(0)
    dist_.init_process_group("nccl", rank=0, world_size=1)
    try:
        rank = dist.NcclRank(host)
        x2 = np.zeros(sa.n)
        r2 = rank.solve(b, x2)
        q2 = rank.sequence(bs, 1e-8, 2000, 16, 6, "sc", batch=False)
        q3 = rank.sequence(bs, 1e-8, 2000, 16, 6, "sc")  # solves 2..k through rcg_dist_solve_batch
    finally:
        dist_.destroy_process_group()
    assert r2.iterations == r1.iterations
    assert np.array_equal(r2.history, r1.history)
    assert np.array_equal(x2, x1)
    # the sequence (sampled solve 1, recycling, SC solves): bitwise across transports
    assert q2["iterations"] == q1["iterations"] and q2["m_bar"] == q1["m_bar"]
    assert np.array_equal(q2["ritz_values"], q1["ritz_values"])
    assert all(np.array_equal(a, b_) for a, b_ in zip(q2["solutions"], q1["solutions"]))
    # the batched slab solves reduce in another (fixed) order: same solve 1 and basis, accelerated
    # solves within a step of the one-at-a-time counts, solutions at the solver tolerance
    assert q3["iterations"][0] == q1["iterations"][0] and q3["m_bar"] == q1["m_bar"]
    assert np.array_equal(q3["ritz_values"], q1["ritz_values"])
    assert all(abs(a - b_) <= 2 for a, b_ in zip(q3["iterations"], q1["iterations"]))
    for a, b_ in zip(q3["solutions"], q1["solutions"]):
        assert np.linalg.norm(a - b_) <= 1e-6 * np.linalg.norm(b_)


@pytest.mark.parametrize("name", ["c1", "c2", "c4", "c5"])
@pytest.mark.parametrize("nparts", [1, 2, 3])
def test_loopback_sequence_matches_block_jacobi_sequence(oracle, problems, name, nparts):
    """run_sequence over row slabs (rcg_dist_pcg_solve_sampled + rcg_dist_recycle + rcg_dist_solve)
    against the oracle's sequence with ic0_factorize(a, 0, G): solve 1 and the sampled iterations,
    m_bar, Ritz values (<= 1e-6 at equal solve-1 counts) and every accelerated solve (+-2)."""
    from oracle.sequence import run_sequence
    from paper_2203_08498_b200 import dist

    cfg = problems.SMALL[name]
    h = problems.generate(cfg)
    ref = run_sequence(oracle, cfg, h, blocks=nparts)
    _, host = _scaled(oracle, problems, name)
    system = dist.LoopbackSystem(host, nparts)
    out = system.sequence(ref["scaled_rhs"], cfg.eps, cfg.max_iter, cfg.sampler_m, cfg.keep,
                          "sc" if cfg.method == "sc" else "deflation")
    assert all(out["converged"])
    for k, (g, o) in enumerate(zip(out["iterations"], ref["iterations"])):
        assert abs(g - o) <= 2, (k, out["iterations"], ref["iterations"])
    # the recycling step on shared inputs: the oracle's build_aux_matrix on the
    # errors the slabs sampled -- m_bar and Ritz values <= 1e-6
    sa, _ = _scaled(oracle, problems, name)
    m_bar_o, vals_o, _ = oracle.build_aux(sa, system.sampled_errors(), float("inf"))
    assert out["m_bar"] == m_bar_o
    assert np.allclose(out["ritz_values"], np.asarray(vals_o)[:m_bar_o], rtol=1e-6, atol=0)
    assert out["m_tilde"] == min(cfg.keep, m_bar_o)
    if out["iterations"][0] == ref["iterations"][0]:
        assert out["m_bar"] == ref["m_bar"]
    assert out["iterations"][1] < out["iterations"][0] or out["m_tilde"] == 0


@pytest.mark.parametrize("name", ["c1", "c2"])
@pytest.mark.parametrize("nparts", [1, 2, 3])
def test_loopback_sampled_method_b(oracle, problems, name, nparts):
    """Solve 1 over row slabs with the method-B sampler (snapshots at the relative-residual
    crossings eps^(j/(m+1)), sampling.cpp) against the oracle's block-Jacobi PCG with the same
    sampler: iterations +-2; at equal counts the same occupied slots at the same iterations, and
    every slot (x at that iteration, slab rows concatenated) within the solution tolerance."""
    from paper_2203_08498_b200 import api, dist

    sa, host = _scaled(oracle, problems, name)
    b = oracle.uniform_pm1(5, 0, sa.n)
    system = dist.LoopbackSystem(host, nparts)
    samplers = [api.SamplerState.method_b(c, 6, 1e-8, p.nloc) for c, p in zip(system.ctxs, system.plans)]
    xs = [np.zeros(p.nloc) for p in system.plans]
    rep = api.dist_pcg_solve_sampled(system.comm, system.slabs, samplers, dist.scatter(b, system.plans), xs,
                                     1e-8, 5000)
    f = oracle.ic0_factorize(sa, 0.0, nparts)
    so = oracle.sampler_b(6, 1e-8, sa.n)
    xo = np.zeros(sa.n)
    ro = oracle.pcg_solve(sa, b, xo, kind=1, ic=f, sampler=so, max_iter=5000)
    _, _, tol = _oracle_block_jacobi(oracle, sa, b, nparts)
    assert rep.converged and ro.converged
    assert abs(rep.iterations - ro.iterations) <= 2, (rep.iterations, ro.iterations)
    states = [s.state() for s in samplers]
    for occ, it in states[1:]:   # every slab schedules the same iterations
        assert np.array_equal(occ, states[0][0]) and np.array_equal(it, states[0][1])
    if rep.iterations == ro.iterations:
        oo, io = so.state()
        assert np.array_equal(states[0][0], oo) and np.array_equal(states[0][1], io)
        for j in np.nonzero(oo)[0]:
            slot = np.concatenate([s.slot(int(j)) for s in samplers])
            assert _rel(slot, so.slot(int(j))) <= tol, (j, _rel(slot, so.slot(int(j))), tol)
        assert _rel(np.concatenate(xs), xo) <= tol


@pytest.mark.parametrize("name", ["c1", "c4"])
@pytest.mark.parametrize("nparts", [1, 2])
def test_loopback_lean_sequence(oracle, problems, name, nparts, monkeypatch):
    """The memory-lean distributed recycling step (RCG_DIST_LEAN=1: errors / MGS in the sampler
    slots, streamed Gram, slots released before the basis -- what C4 needs at G = 1-2) and the
    device block factor: the block-Jacobi sequence of the oracle, +-2 iterations per solve, m_bar,
    Ritz values <= 1e-6 at equal solve-1 counts."""
    from oracle.sequence import run_sequence
    from paper_2203_08498_b200 import dist

    monkeypatch.setenv("RCG_DIST_LEAN", "1")
    cfg = problems.SMALL[name]
    h = problems.generate(cfg)
    ref = run_sequence(oracle, cfg, h, blocks=nparts)
    _, host = _scaled(oracle, problems, name)
    system = dist.LoopbackSystem(host, nparts, device_factor=True)
    out = system.sequence(ref["scaled_rhs"], cfg.eps, cfg.max_iter, cfg.sampler_m, cfg.keep,
                          "sc" if cfg.method == "sc" else "deflation")
    assert all(out["converged"])
    for k, (g, o) in enumerate(zip(out["iterations"], ref["iterations"])):
        assert abs(g - o) <= 2, (k, out["iterations"], ref["iterations"])
    if out["iterations"][0] == ref["iterations"][0]:
        assert out["m_bar"] == ref["m_bar"] and out["m_tilde"] == ref["m_tilde"]
        vo = np.asarray(ref["ritz_values"])[: out["m_bar"]]
        assert np.allclose(out["ritz_values"], vo, rtol=1e-6, atol=0)
