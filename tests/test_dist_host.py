"""Multi-GPU row slabs, host side (CPU): the slab plan (rcg_slab_plan_create) and the
distributed iteration's structure over a real collective backend (gloo, world size 2).

* The plan reproduces the global rows exactly, uses the reference block bounds floor(b n / G)
  (ic_preconditioner.cpp:104-106), and every slab's send list to q is exactly q's halo from it.
* Block-Jacobi IC(0) (ic0_factorize(a, s, G)) is, block by block, the IC(0) of the diagonal
  block a slab factorises (checked on the oracle, which is pinned to the reference).
* Two gloo ranks run the distributed PCG of dist.cu (halo of x once and of p per iteration,
  three allreduces per iteration, block-Jacobi IC) in numpy on the plans, and reproduce the
  single-process block-Jacobi PCG of the oracle: same iterations, solution to rounding.
"""
import os
import socket

import numpy as np
import pytest

from conftest import laplacian_2d, random_sdd_spd


def _global_cols(plan):
    halo = np.concatenate([plan.halo_global, [-1]])  # (padding: nhalo may be 0)
    return np.where(plan.col_idx < plan.nloc, plan.col_idx + plan.row_begin,
                    halo[np.clip(plan.col_idx - plan.nloc, 0, len(halo) - 1)])


def _matrices(oracle, problems):
    out = [("c1", problems.generate(problems.SMALL["c1"]))]
    n, rs, ci, va = laplacian_2d(23)
    out.append(("lap2d", problems.HostCsr(n, rs, ci, va)))
    n, rs, ci, va = random_sdd_spd(60, 0.1, 7, oracle)
    out.append(("sdd", problems.HostCsr(n, rs, ci, va)))
    out.append(("c3", problems.generate(problems.SMALL["c3"])))
    return out


@pytest.mark.parametrize("nparts", [1, 2, 3, 5])
def test_plan_reproduces_rows_and_exchange_lists(oracle, problems, nparts):
    from paper_2203_08498_b200 import api, dist

    for name, h in _matrices(oracle, problems):
        plans = [api.SlabPlan(h.n, h.row_start, h.col_idx, h.values, nparts, b) for b in range(nparts)]
        bnd = dist.bounds(h.n, nparts)
        for b, p in enumerate(plans):
            assert (p.row_begin, p.row_end) == (bnd[b], bnd[b + 1]), name
            lo, hi = h.row_start[p.row_begin], h.row_start[p.row_end]
            assert np.array_equal(p.row_start, h.row_start[p.row_begin:p.row_end + 1] - lo)
            assert np.array_equal(_global_cols(p), h.col_idx[lo:hi]), name
            assert np.array_equal(p.values, h.values[lo:hi])
            hg = p.halo_global
            assert np.all(np.diff(hg) > 0) and not np.any((hg >= p.row_begin) & (hg < p.row_end))
            owners = np.searchsorted(bnd, hg, side="right") - 1
            assert np.array_equal(np.bincount(owners, minlength=nparts), p.recv_count)
        for b, pb in enumerate(plans):
            offs = np.concatenate([[0], np.cumsum(pb.send_count)])
            for q, pq in enumerate(plans):
                sent = pb.send_idx[offs[q]:offs[q + 1]] + pb.row_begin
                roff = np.concatenate([[0], np.cumsum(pq.recv_count)])
                want = pq.halo_global[roff[b]:roff[b + 1]]
                assert np.array_equal(sent, want), (name, b, q)


def test_plan_rejects_bad_partitions(problems):
    from paper_2203_08498_b200 import api
    from paper_2203_08498_b200._lib import InvalidArgument

    h = problems.generate(problems.SMALL["c1"])
    for nparts, part in ((0, 0), (2, 2), (2, -1), (h.n + 1, 0)):
        with pytest.raises(InvalidArgument):
            api.SlabPlan(h.n, h.row_start, h.col_idx, h.values, nparts, part)


@pytest.mark.parametrize("nparts", [2, 4])
def test_block_jacobi_is_the_diagonal_block_factor(oracle, problems, nparts):
    """ic0_factorize(a, 0, G) restricted to block b == ic0_factorize(diagonal block b) bitwise."""
    from oracle import Matrix
    from paper_2203_08498_b200 import api

    h = problems.generate(problems.SMALL["c2"])
    sa, _ = oracle.diagonal_scale(Matrix.of(h))
    g = oracle.ic0_factorize(sa, 0.0, nparts).arrays()
    for b in range(nparts):
        p = api.SlabPlan(h.n, sa.rs, sa.ci, sa.va, nparts, b)
        rs, ci, va = p.diagonal_block()
        f = oracle.ic0_factorize(Matrix(p.nloc, rs, ci, va), 0.0, 1).arrays()
        r0, r1 = p.row_begin, p.row_end
        assert np.array_equal(f["d"], g["d"][r0:r1])
        lo, hi = g["l_row_start"][r0], g["l_row_start"][r1]
        assert np.array_equal(f["l_row_start"], g["l_row_start"][r0:r1 + 1] - lo)
        assert np.array_equal(f["l_col"] + r0, g["l_col"][lo:hi])
        assert np.array_equal(f["l_val"], g["l_val"][lo:hi])


# --------------------------------------------------------------------------- gloo, world size 2
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, n, rs, ci, va, b, eps, max_iter, out_q):
    """dist.cu's iteration in numpy on this rank's plan, over gloo (test executable spec)."""
    import torch
    import torch.distributed as dist

    from oracle import Matrix, Oracle
    from paper_2203_08498_b200 import api

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    o = Oracle()
    p = api.SlabPlan(n, rs, ci, va, world, rank)
    drs, dci, dva = p.diagonal_block()
    f = o.ic0_factorize(Matrix(p.nloc, drs, dci, dva), 0.0, 1)
    soff = np.concatenate([[0], np.cumsum(p.send_count)])
    roff = np.concatenate([[0], np.cumsum(p.recv_count)])
    rows = np.repeat(np.arange(p.nloc), np.diff(p.row_start))

    def halo(ext):
        reqs = []
        for q in range(world):
            if p.send_count[q]:
                buf = torch.from_numpy(np.ascontiguousarray(ext[p.send_idx[soff[q]:soff[q + 1]]]))
                reqs.append(dist.isend(buf, q))
        got = {}
        for q in range(world):
            if p.recv_count[q]:
                got[q] = torch.empty(int(p.recv_count[q]), dtype=torch.float64)
                reqs.append(dist.irecv(got[q], q))
        for r in reqs:
            r.wait()
        for q, t in got.items():
            ext[p.nloc + roff[q]:p.nloc + roff[q + 1]] = t.numpy()

    def spmv(ext):
        y = np.zeros(p.nloc)
        np.add.at(y, rows, p.values * ext[p.col_idx])
        return y

    colls = [0]

    def allreduce(*vals):
        colls[0] += 1
        t = torch.tensor(vals, dtype=torch.float64)
        dist.all_reduce(t)
        return t.tolist()

    bl = b[p.row_begin:p.row_end]
    xe = np.zeros(p.nloc + p.nhalo)
    pe = np.zeros(p.nloc + p.nhalo)
    halo(xe)
    r = bl - spmv(xe)
    bb, rr = allreduce(float(bl @ bl), float(r @ r))
    bnorm = np.sqrt(bb)
    # dist.cu's fused reductions: the (r, r) of the convergence check waits for the next
    # iteration's (r, z) -- two allreduces per iteration, every value that of pcg.cpp:63-89
    hist, rho_prev, pending, it = [], None, None, 0
    while True:
        z = o.ic_apply(f, r)  # (wasted once, when the pending check ends the solve)
        if pending is None:
            (rho,) = allreduce(float(r @ z))
        else:
            rho, rr = allreduce(float(r @ z), pending)
            pending = None
            hist.append(np.sqrt(rr) / bnorm)
            if hist[-1] <= eps or it >= max_iter:
                break
        it += 1
        beta = rho / rho_prev if it > 1 else 0.0
        pe[:p.nloc] = z if it == 1 else z + beta * pe[:p.nloc]
        halo(pe)
        q = spmv(pe)
        (pq,) = allreduce(float(pe[:p.nloc] @ q))
        alpha = rho / pq
        xe[:p.nloc] += alpha * pe[:p.nloc]
        r = r - alpha * q
        pending = float(r @ r)
        rho_prev = rho
    assert colls[0] == 2 * len(hist) + 2, (colls[0], len(hist))
    out_q.put((rank, p.row_begin, p.row_end, xe[:p.nloc].copy(), hist))
    dist.destroy_process_group()


def test_gloo_two_ranks_match_block_jacobi_pcg(oracle, problems):
    import torch.multiprocessing as mp

    from oracle import Matrix

    h = problems.generate(problems.SMALL["c1"])
    sa, _ = oracle.diagonal_scale(Matrix.of(h))
    b = oracle.uniform_pm1(11, 0, h.n)
    world, eps, max_iter = 2, 1e-8, 500
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    env_keep = os.environ.get("OMP_NUM_THREADS")
    os.environ["OMP_NUM_THREADS"] = "1"
    try:
        procs = [ctx.Process(target=_rank_main, args=(r, world, port, h.n, sa.rs, sa.ci, sa.va, b, eps, max_iter, q))
                 for r in range(world)]
        for pr in procs:
            pr.start()
        res = [q.get(timeout=300) for _ in range(world)]
        for pr in procs:
            pr.join(timeout=60)
            assert pr.exitcode == 0
    finally:
        if env_keep is None:
            os.environ.pop("OMP_NUM_THREADS", None)
        else:
            os.environ["OMP_NUM_THREADS"] = env_keep
    x = np.zeros(h.n)
    for _, r0, r1, xl, hist in res:
        x[r0:r1] = xl
    hists = [r[4] for r in res]
    assert hists[0] == hists[1]  # every rank holds the same scalars
    f = oracle.ic0_factorize(sa, 0.0, world)
    xo = np.zeros(h.n)
    ro = oracle.pcg_solve(sa, b, xo, kind=1, ic=f, eps=eps, max_iter=max_iter)
    assert abs(len(hists[0]) - ro.iterations) <= 1
    assert np.linalg.norm(x - xo) <= 1e-8 * np.linalg.norm(xo)


def _rank_recycle(rank, world, port, n, rs, ci, va, errors, out_q):
    """dist.cu's dist_recycle in numpy on this rank's rows, over gloo (test executable spec):
    global zero-column test, single-pass MGS with every dot allreduced (dense.cpp:45-61), A Q by
    halo exchange + local SpMV, the allreduced Gram Q^T A Q eigensolved on every rank."""
    import torch
    import torch.distributed as dist

    from oracle import Oracle
    from paper_2203_08498_b200 import api

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    o = Oracle()
    p = api.SlabPlan(n, rs, ci, va, world, rank)
    soff = np.concatenate([[0], np.cumsum(p.send_count)])
    roff = np.concatenate([[0], np.cumsum(p.recv_count)])
    rows = np.repeat(np.arange(p.nloc), np.diff(p.row_start))

    def allreduce(v):
        t = torch.tensor(np.atleast_1d(v), dtype=torch.float64)
        dist.all_reduce(t)
        return t.numpy()

    def halo(ext):
        reqs, got = [], {}
        for q in range(world):
            if p.send_count[q]:
                reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(ext[p.send_idx[soff[q]:soff[q + 1]]])), q))
        for q in range(world):
            if p.recv_count[q]:
                got[q] = torch.empty(int(p.recv_count[q]), dtype=torch.float64)
                reqs.append(dist.irecv(got[q], q))
        for r in reqs:
            r.wait()
        for q, t in got.items():
            ext[p.nloc + roff[q]:p.nloc + roff[q + 1]] = t.numpy()

    e = errors[:, p.row_begin:p.row_end]
    nz = allreduce((e != 0).any(axis=1).astype(np.float64))
    qs = []
    for j in np.nonzero(nz > 0)[0]:
        w = e[j].copy()
        n0 = np.sqrt(allreduce(w @ w)[0])
        if n0 == 0.0:
            continue
        for qv in qs:
            c = allreduce(qv @ w)[0]
            w = w - c * qv
        n1 = np.sqrt(allreduce(w @ w)[0])
        if n1 <= 1e-12 * n0:
            continue
        qs.append(w / n1)
    k = len(qs)
    aq = []
    for qv in qs:
        ext = np.zeros(p.nloc + p.nhalo)
        ext[:p.nloc] = qv
        halo(ext)
        y = np.zeros(p.nloc)
        np.add.at(y, rows, p.values * ext[p.col_idx])
        aq.append(y)
    g = np.zeros((k, k))
    for i in range(k):
        for j in range(i + 1):
            g[i, j] = qs[i] @ aq[j]
    g = allreduce(g.ravel()).reshape(k, k)
    s = np.tril(g) + np.tril(g, -1).T
    vals, _ = o.sym_eig(s)
    out_q.put((rank, k, np.asarray(vals)))
    dist.destroy_process_group()


def test_gloo_two_ranks_recycling_matches_build_aux(oracle, problems):
    """The distributed recycling step (rcg_dist_recycle's structure) on a block-Jacobi solve 1's
    sampled errors, plus a duplicated and a zero column: same m_bar and Ritz values as the
    oracle's build_aux_matrix on the assembled errors (recycling.cpp:81-96)."""
    import torch.multiprocessing as mp

    from oracle import Matrix

    h = problems.generate(problems.SMALL["c1"])
    sa, _ = oracle.diagonal_scale(Matrix.of(h))
    world = 2
    f = oracle.ic0_factorize(sa, 0.0, world)
    smp = oracle.sampler_a(16, 500, h.n)
    x = np.zeros(h.n)
    oracle.pcg_solve(sa, oracle.uniform_pm1(5, 0, h.n), x, kind=1, ic=f, eps=1e-8, max_iter=500, sampler=smp)
    errs = np.asarray(oracle.harvest_errors(x, smp))
    errs = np.vstack([errs, errs[:1], np.zeros((1, h.n))])  # dependent + zero columns
    m_bar_o, vals_o, _ = oracle.build_aux(sa, errs, float("inf"))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_recycle, args=(r, world, port, h.n, sa.rs, sa.ci, sa.va, errs, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for _, k, vals in res:
        assert k == m_bar_o
        assert np.allclose(vals, vals_o[:k], rtol=1e-9, atol=0)
    assert np.array_equal(res[0][2], res[1][2])  # replicated eigensolve: identical on every rank
