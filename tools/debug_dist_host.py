"""Dev: two processes over the host transport vs the in-process loopback G=2 system, step by step."""
import os
import sys
import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank, world, port, name):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from oracle import Matrix, Oracle
    from oracle.sequence import rhs_set
    from paper_2203_08498_b200 import api, dist as pdist, problems
    o = Oracle()
    cfg = problems.SMALL[name]
    h = problems.generate(cfg)
    sa, dis = o.diagonal_scale(Matrix.of(h))
    host = problems.HostCsr(h.n, sa.rs, sa.ci, sa.va)
    _, bs = rhs_set(o, cfg, h, Matrix.of(h), dis)
    kind = "sc" if cfg.method == "sc" else "deflation"
    r = pdist.NcclRank(host, transport="host")
    lo, hi = r.plan.row_begin, r.plan.row_end
    # loopback reference in-process
    lb = pdist.LoopbackSystem(host, world, device_factor=True)
    # 1) a plain solve
    x = np.zeros(hi - lo)
    rep = r.solve(bs[0][lo:hi], x, cfg.eps, cfg.max_iter)
    xg = np.zeros(h.n)
    rl = lb.solve(bs[0], xg, cfg.eps, cfg.max_iter)
    print(rank, "plain solve", rep.iterations, rl.iterations, "x diff", np.abs(x - xg[lo:hi]).max(), flush=True)
    # 1b) the sampled solve + sampler state + harvested errors
    smp = api.SamplerState.method_a(r.ctx, cfg.sampler_m, cfg.max_iter, r.plan.nloc)
    x1 = np.zeros(hi - lo)
    r1 = api.dist_pcg_solve_sampled(r.comm, [r.slab], [smp], [bs[0][lo:hi]], [x1], cfg.eps, cfg.max_iter)
    st = smp.state()
    print(rank, "sampled", r1.iterations, "state", st if not isinstance(st, tuple) else (list(st[0]), list(st[1])),
          "x1 norm", np.linalg.norm(x1), "slot0 norm", np.linalg.norm(smp.slot(0)), flush=True)
    res = api.dist_recycle(r.comm, [r.slab], [smp], [x1], keep_count=cfg.keep, kind=kind)
    print(rank, "recycle m_bar", res[0], "vals", np.asarray(res[1])[:3], flush=True)
    # 2) sequence, unbatched vs batched vs loopback
    out_u = r.sequence([b[lo:hi] for b in bs], cfg.eps, cfg.max_iter, cfg.sampler_m, cfg.keep, kind, batch=False)
    print(rank, "host unbatched", out_u["iterations"], out_u["m_bar"], np.asarray(out_u["ritz_values"])[:3], flush=True)
    out_b = r.sequence([b[lo:hi] for b in bs], cfg.eps, cfg.max_iter, cfg.sampler_m, cfg.keep, kind, batch=True)
    print(rank, "host batched", out_b["iterations"], out_b["m_bar"], flush=True)
    if rank == 0:
        ol = lb.sequence(bs, cfg.eps, cfg.max_iter, cfg.sampler_m, cfg.keep, kind)
        print(rank, "loopback", ol["iterations"], ol["m_bar"], np.asarray(ol["ritz_values"])[:3], flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp
    name = sys.argv[1] if len(sys.argv) > 1 else "c1"
    world = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    ctx = mp.get_context("spawn")
    ps = [ctx.Process(target=worker, args=(k, world, 29513, name)) for k in range(world)]
    [p.start() for p in ps]
    [p.join() for p in ps]
