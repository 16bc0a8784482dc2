"""The distributed iteration of csrc/dist.cu with REAL separate processes: world size 2 (and 3), one
slab per process, all on the one GPU of the box, over the host-staged transport
(rcg_comm_create_host: every allreduce / halo exchange synchronises the slab's stream and goes
through torch.distributed on gloo, so no kernel ever waits on another rank).  This exercises what
the loopback tests cannot: per-process plans and factors, the global shift agreement, every rank
reaching the same stop decision from its own DevState, and collective ordering across processes --
everything the NCCL path does except the transport itself (NCCL refuses two ranks on one GPU).

Bar: the oracle's block-Jacobi sequence (ic0_factorize(a, 0, G), pinned to the reference) --
every solve +-2 iterations, m_bar equal, Ritz values <= 1e-6 at equal solve-1 counts, solution of
solve 1 within max(1e-8, 10 x the oracle's reduction-order floor) at equal counts.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, name, out_dir):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if root not in sys.path:
        sys.path.insert(0, root)
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from oracle import Matrix, Oracle
        from oracle.sequence import rhs_set
        from paper_2203_08498_b200 import dist as pdist
        from paper_2203_08498_b200 import problems

        o = Oracle()
        cfg = problems.SMALL[name]
        h = problems.generate(cfg)
        sa, dis = o.diagonal_scale(Matrix.of(h))
        host = problems.HostCsr(h.n, sa.rs, sa.ci, sa.va)
        _, bs = rhs_set(o, cfg, h, Matrix.of(h), dis)  # the oracle sequence's scaled right-hand sides
        r = pdist.NcclRank(host, transport="host")
        lo, hi = r.plan.row_begin, r.plan.row_end
        out = r.sequence([b[lo:hi] for b in bs], cfg.eps, cfg.max_iter, cfg.sampler_m, cfg.keep,
                         "sc" if cfg.method == "sc" else "deflation")
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), lo=lo, hi=hi, iterations=np.array(out["iterations"]),
                 converged=np.array(out["converged"]), m_bar=out["m_bar"], m_tilde=out["m_tilde"],
                 ritz=np.asarray(out["ritz_values"]), x1=out["solutions"][0])
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["c1", "c2", "c4"])
@pytest.mark.parametrize("world", [1, 2, 3])
def test_two_process_sequence_matches_block_jacobi(oracle, problems, tmp_path, name, world):
    import torch.multiprocessing as mp

    from oracle.sequence import run_sequence

    cfg = problems.SMALL[name]
    h = problems.generate(cfg)
    ref = run_sequence(oracle, cfg, h, blocks=world)
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, str(tmp_path))) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    parts = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    its = parts[0]["iterations"]
    for p in parts[1:]:  # every rank made the same decisions
        assert np.array_equal(p["iterations"], its) and int(p["m_bar"]) == int(parts[0]["m_bar"])
        assert np.array_equal(p["ritz"], parts[0]["ritz"])
    assert all(parts[0]["converged"])
    for k, (g, o) in enumerate(zip(its, ref["iterations"])):
        assert abs(int(g) - o) <= 2, (k, list(its), ref["iterations"])
    assert int(parts[0]["m_bar"]) == ref["m_bar"] or its[0] != ref["iterations"][0]
    if its[0] == ref["iterations"][0]:
        rv = np.asarray(ref["ritz_values"])[: int(parts[0]["m_bar"])]
        assert np.allclose(parts[0]["ritz"], rv, rtol=1e-6, atol=0)
        x1 = np.concatenate([p["x1"] for p in sorted(parts, key=lambda q: int(q["lo"]))])
        x_ref = ref["solutions"][0]
        rel = float(np.linalg.norm(x1 - x_ref) / np.linalg.norm(x_ref))
        assert rel <= max(1e-8, 10.0 * _floor(oracle, h, ref, world, cfg)), rel


def _floor(oracle, h, ref, blocks, cfg):
    """The oracle's own response of solve 1 to its dot products summed backwards / pairwise."""
    from oracle import Matrix

    sa, _ = oracle.diagonal_scale(Matrix.of(h))
    f = oracle.ic0_factorize(sa, 0.0, blocks)
    out = 0.0
    for order in (1, 2):
        with oracle.reversed_dots(order):
            x = np.zeros(h.n)
            oracle.pcg_solve(sa, ref["scaled_rhs"][0], x, kind=1, ic=f, eps=cfg.eps, max_iter=cfg.max_iter)
        out = max(out, float(np.linalg.norm(x - ref["solutions"][0]) / np.linalg.norm(ref["solutions"][0])))
    return out


def _fuse_worker(rank, world, port, name, out_dir):
    """Solve 1 + recycling once, then the batched accelerated solves twice on the same basis:
    one allreduce per dot (RCG_DIST_FUSE=0), then the fused reductions (default)."""
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if root not in sys.path:
        sys.path.insert(0, root)
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from oracle import Matrix, Oracle
        from oracle.sequence import rhs_set
        from paper_2203_08498_b200 import api, problems
        from paper_2203_08498_b200 import dist as pdist

        o = Oracle()
        cfg = problems.SMALL[name]
        h = problems.generate(cfg)
        sa, dis = o.diagonal_scale(Matrix.of(h))
        host = problems.HostCsr(h.n, sa.rs, sa.ci, sa.va)
        _, bs = rhs_set(o, cfg, h, Matrix.of(h), dis)
        r = pdist.NcclRank(host, transport="host")
        lo, hi = r.plan.row_begin, r.plan.row_end
        res = {}
        # solve 1 (ICCG with the sampler): the deferred check changes no value -- bitwise
        for tag, env in (("s1plain", "0"), ("s1fused", "1")):
            os.environ["RCG_DIST_FUSE"] = env
            before = dict(r.comm.calls)
            smp = api.SamplerState.method_a(r.ctx, cfg.sampler_m, cfg.max_iter, r.plan.nloc)
            x1 = np.zeros(r.plan.nloc)
            r1 = api.dist_pcg_solve_sampled(r.comm, [r.slab], [smp], [bs[0][lo:hi]], [x1], cfg.eps, cfg.max_iter)
            res[tag + "_x"] = x1
            res[tag + "_its"] = np.array([r1.iterations])
            res[tag + "_hist"] = np.asarray(r1.history)
            res[tag + "_slots"] = np.asarray(smp.state()[1])
            res[tag + "_allreduces"] = r.comm.calls["allreduce"] - before["allreduce"]
        kind = "sc" if cfg.method == "sc" else "deflation"
        *_, basis = api.dist_recycle(r.comm, [r.slab], [smp], [x1], keep_count=cfg.keep, kind=kind)
        B = np.stack([b[lo:hi] for b in bs[1:]])
        for tag, env in (("plain", "0"), ("fused", "1")):
            os.environ["RCG_DIST_FUSE"] = env
            before = dict(r.comm.calls)
            X = np.zeros_like(B)
            reps = api.dist_solve_batch(r.comm, r.slab, B, X, basis, cfg.eps, cfg.max_iter)
            res[tag + "_its"] = np.array([q.iterations for q in reps])
            res[tag + "_conv"] = np.array([q.converged for q in reps])
            res[tag + "_x"] = X
            res[tag + "_allreduces"] = r.comm.calls["allreduce"] - before["allreduce"]
            res[tag + "_values"] = r.comm.calls["allreduce_values"] - before["allreduce_values"]
        np.savez(os.path.join(out_dir, f"fuse{rank}.npz"), lo=lo, **res)
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_fused_allreduces_match_one_per_dot(problems, tmp_path, name, parity_log):
    """(p, q) travels with W^T q and the convergence check's (r, r) with the next
    (r, z).  Two processes over the host transport: the fused batched slab solves against the
    one-allreduce-per-dot ones on the same basis -- iterations within one step, solutions at the
    solver tolerance, and the collectives per iteration counted (deflation: 4 -> ~2)."""
    import torch.multiprocessing as mp

    world = 2
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_fuse_worker, args=(r, world, port, name, str(tmp_path))) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    parts = sorted((np.load(tmp_path / f"fuse{r}.npz") for r in range(world)), key=lambda q: int(q["lo"]))
    a, b = parts
    for tag in ("plain", "fused"):  # every rank made the same decisions
        assert np.array_equal(a[tag + "_its"], b[tag + "_its"]) and all(a[tag + "_conv"])
        assert int(a[tag + "_allreduces"]) == int(b[tag + "_allreduces"])
    for q in parts:  # solve 1: identical values, the sampler's slots included
        assert np.array_equal(q["s1plain_x"], q["s1fused_x"]) and np.array_equal(q["s1plain_hist"], q["s1fused_hist"])
        assert np.array_equal(q["s1plain_slots"], q["s1fused_slots"])
    its1 = int(a["s1plain_its"][0])
    s1p, s1f = int(a["s1plain_allreduces"]), int(a["s1fused_allreduces"])
    parity_log(f"fused_allreduces_solve1[{name}]", plain_per_iteration=s1p / its1, fused_per_iteration=s1f / its1)
    assert s1f <= 0.8 * s1p, (s1p, s1f)  # 3 -> 2 per iteration (+ one flush per enqueued batch)
    assert np.all(np.abs(a["plain_its"] - a["fused_its"]) <= 1), (a["plain_its"], a["fused_its"])
    xp = np.concatenate([q["plain_x"] for q in parts], axis=1)
    xf = np.concatenate([q["fused_x"] for q in parts], axis=1)
    rel = max(float(np.linalg.norm(u - v) / np.linalg.norm(u)) for u, v in zip(xp, xf))
    assert rel <= 1e-7, rel
    n_plain, n_fused = int(a["plain_allreduces"]), int(a["fused_allreduces"])
    iters = int(a["plain_its"].max())
    parity_log(f"fused_allreduces[{name}]", plain_per_iteration=n_plain / iters, fused_per_iteration=n_fused / iters,
               solution_rel=rel, bar=1e-7)
    deflation = problems.SMALL[name].method != "sc"
    # deflation: 4 -> 2 per iteration (+ one flush per enqueued batch); SC ((r, r) with W^T r): 4 -> 3
    assert n_fused <= (0.65 if deflation else 0.85) * n_plain, (n_plain, n_fused)
