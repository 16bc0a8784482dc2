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
