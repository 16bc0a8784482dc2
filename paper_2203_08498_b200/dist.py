"""Multi-GPU row slabs above the C-ABI: one process per GPU over NCCL, or all
slabs in one process (loopback transport, for tests on one GPU).

The operator is the reference's block-Jacobi IC(0) -- ic0_factorize(a, s, G) with block bounds
floor(b n / G) (ic_preconditioner.cpp:97-121): slab b factorises its own diagonal block.  The
reference's shift ladder is global (a failing block restarts EVERY block with the next shift),
so the slabs agree on the largest shift any block needed and refactorise at it (the ladder's
first shift at which all blocks succeed, success being monotone in the shift).
"""
from __future__ import annotations

from typing import Callable, Optional, Sequence

import numpy as np

from . import api


def bounds(n: int, nparts: int) -> np.ndarray:
    """Slab row bounds floor(b n / G), b = 0..G (ic_preconditioner.cpp:104-106)."""
    return (np.arange(nparts + 1, dtype=np.int64) * n) // nparts


def block_factor(ctx: api.Context, plan: api.SlabPlan, shift: float = 0.0, device: bool = False) -> api.IcFactor:
    """The slab's diagonal-block IC(0), factorised on the device either way (device=False passes
    host arrays, which rcg_ic0_factorize uploads) -- the reference's factor bit for bit."""
    rs, ci, va = plan.diagonal_block()
    if device:
        return api.IcFactor.factorize_device(ctx, api.CsrMatrix(ctx, plan.nloc, rs, ci, va, validate=False), shift, 1)
    return api.IcFactor.factorize(ctx, plan.nloc, rs, ci, va, shift, 1)


def agree_factors(ctxs, plans, allreduce_max: Callable[[float], float], device: bool = False):
    """Block factors of the local slabs with the reference's global shift ladder: each block runs
    the ladder, the ranks take the largest shift (allreduce_max), and blocks that stopped lower
    are refactorised at it."""
    fs = [block_factor(c, p, 0.0, device) for c, p in zip(ctxs, plans)]
    s = allreduce_max(max(f.shift_used for f in fs))
    return [f if f.shift_used == s else block_factor(c, p, s, device) for f, c, p in zip(fs, ctxs, plans)]


class LoopbackSystem:
    """All G slabs of a matrix in this process on one GPU (one context / stream per slab)."""

    def __init__(self, host, nparts: int, preconditioner: str = "ic", device: int = 0, device_factor: bool = False):
        self.n, self.nparts = host.n, nparts
        self.ctxs = [api.Context(device) for _ in range(nparts)]
        self.plans = [api.SlabPlan(host.n, host.row_start, host.col_idx, host.values, nparts, b) for b in range(nparts)]
        self.factors = (agree_factors(self.ctxs, self.plans, lambda v: v, device_factor) if preconditioner == "ic"
                        else [None] * nparts)
        self.slabs = [api.DSlab(c, p, f) for c, p, f in zip(self.ctxs, self.plans, self.factors)]
        self.comm = api.Comm.loopback(nparts)

    def basis(self, w: np.ndarray, kind: str = "deflation") -> api.DBasis:
        """Distributed basis from a global W given as (m, n) (one basis vector per row)."""
        return api.DBasis(self.comm, self.slabs, [w[:, p.row_begin:p.row_end] for p in self.plans], kind)

    def sequence(self, bs, eps: float = 1e-8, max_iter: int = 1000, sampler_m: int = 16, keep: int = 8,
                 kind: str = "deflation") -> dict:
        """run_sequence (driver.cpp:108-222) over the slabs on scaled right-hand sides bs (global
        vectors): solve 1 with the method-A error sampler, the distributed recycling step (count
        selection of `keep` Ritz vectors), then deflated / SC solves 2..k from x0 = 0."""
        samplers = [api.SamplerState.method_a(c, sampler_m, max_iter, p.nloc) for c, p in zip(self.ctxs, self.plans)]
        xs = [np.zeros(p.nloc) for p in self.plans]
        r1 = api.dist_pcg_solve_sampled(self.comm, self.slabs, samplers, scatter(bs[0], self.plans), xs, eps, max_iter)
        self.last_samplers, self.last_x1 = samplers, [x.copy() for x in xs]   # kept for inspection (tests)
        m_bar, vals, _, m_tilde, basis = api.dist_recycle(self.comm, self.slabs, samplers, xs, keep_count=keep, kind=kind)
        out = {"iterations": [r1.iterations], "converged": [r1.converged], "solutions": [np.concatenate(xs)],
               "m_bar": m_bar, "ritz_values": vals, "m_tilde": m_tilde, "histories": [r1.history]}
        for b in bs[1:]:
            x = np.zeros(self.n)
            r = self.solve(b, x, eps, max_iter, basis)
            out["iterations"].append(r.iterations)
            out["converged"].append(r.converged)
            out["solutions"].append(x)
            out["histories"].append(r.history)
        return out

    def sampled_errors(self) -> np.ndarray:
        """The last sequence's harvested errors x_final - slot (occupied slots in order), global
        rows -- the shared input for checking the recycling step against the oracle."""
        st = self.last_samplers[0].state()
        occ = st[0] if isinstance(st, tuple) else st["occupied"]
        cols = []
        for j in np.nonzero(np.asarray(occ))[0]:
            cols.append(np.concatenate([x - smp.slot(int(j)) for x, smp in zip(self.last_x1, self.last_samplers)]))
        return np.array(cols).reshape(len(cols), self.n)

    def solve(self, b: np.ndarray, x: np.ndarray, eps: float = 1e-8, max_iter: int = 1000,
              basis: Optional[api.DBasis] = None) -> api.SolveReport:
        """Global b, x (x updated in place) split along the slab bounds."""
        bs = [np.ascontiguousarray(b[p.row_begin:p.row_end]) for p in self.plans]
        xs = [np.ascontiguousarray(x[p.row_begin:p.row_end]) for p in self.plans]
        rep = api.dist_solve(self.comm, self.slabs, bs, xs, basis, eps, max_iter)
        for p, xl in zip(self.plans, xs):
            x[p.row_begin:p.row_end] = xl
        return rep


class NcclRank:
    """This process's slab of a G-GPU solve (rank = slab index), plumbing over torch.distributed:
    rank 0 creates the NCCL id, every rank builds its own plan / factor / slab.  transport="nccl"
    (NCCL over NVLink, the product path) or "host" (rcg_comm_create_host over the process group's
    own backend, e.g. gloo: every collective staged through host memory, so ranks may share one
    GPU -- the multi-process test of the same distributed iteration)."""

    def __init__(self, host, ctx: Optional[api.Context] = None, preconditioner: str = "ic",
                 transport: str = "nccl", device_factor: bool = True):
        import torch
        import torch.distributed as dist

        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.ctx = ctx or api.Context(torch.cuda.current_device())
        self.plan = api.SlabPlan(host.n, host.row_start, host.col_idx, host.values, self.world, self.rank)
        on_gpu = dist.get_backend() == "nccl"

        def allreduce_max(v: float) -> float:
            t = torch.tensor([v], dtype=torch.float64, device="cuda" if on_gpu else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())

        self.factor = (agree_factors([self.ctx], [self.plan], allreduce_max, device_factor)[0]
                       if preconditioner == "ic" else None)
        self.slab = api.DSlab(self.ctx, self.plan, self.factor)
        if transport == "host":
            self.comm = api.Comm.host()
        else:
            obj = [api.Comm.unique_id() if self.rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            self.comm = api.Comm.nccl(obj[0], self.world, self.rank)

    def basis(self, w_local: np.ndarray, kind: str = "deflation") -> api.DBasis:
        """This rank's rows of W, (m, nloc) -- collective over the ranks."""
        return api.DBasis(self.comm, [self.slab], [w_local], kind)

    def solve(self, b_local, x_local, eps: float = 1e-8, max_iter: int = 1000,
              basis: Optional[api.DBasis] = None) -> api.SolveReport:
        return api.dist_solve(self.comm, [self.slab], [b_local], [x_local], basis, eps, max_iter)

    def sequence(self, bs_local, eps: float = 1e-8, max_iter: int = 1000, sampler_m: int = 16, keep: int = 8,
                 kind: str = "deflation", batch: bool = True) -> dict:
        """run_sequence over the ranks (collective): bs_local = this rank's rows of the scaled
        right-hand sides; solutions are this rank's rows.  batch: solves 2..k through
        rcg_dist_solve_batch (up to 24 per kernel sequence), else one at a time."""
        def zeros(like, shape):  # numpy host or CUDA torch, like the right-hand sides
            if hasattr(like, "data_ptr"):
                import torch

                return torch.zeros(shape, dtype=torch.float64, device=like.device)
            return np.zeros(shape)

        smp = api.SamplerState.method_a(self.ctx, sampler_m, max_iter, self.plan.nloc)
        x1 = zeros(bs_local[0], self.plan.nloc)
        r1 = api.dist_pcg_solve_sampled(self.comm, [self.slab], [smp], [bs_local[0]], [x1], eps, max_iter)
        m_bar, vals, _, m_tilde, basis = api.dist_recycle(self.comm, [self.slab], [smp], [x1], keep_count=keep,
                                                           kind=kind)
        out = {"iterations": [r1.iterations], "converged": [r1.converged], "solutions": [x1], "m_bar": m_bar,
               "ritz_values": vals, "m_tilde": m_tilde}
        rest = list(bs_local[1:])
        if batch:
            for k0 in range(0, len(rest), 24):
                chunk = rest[k0:k0 + 24]
                if hasattr(chunk[0], "data_ptr"):
                    import torch

                    B = torch.stack(chunk)
                else:
                    B = np.stack(chunk)
                X = zeros(chunk[0], tuple(B.shape))
                for r, x in zip(api.dist_solve_batch(self.comm, self.slab, B, X, basis, eps, max_iter), X):
                    out["iterations"].append(r.iterations)
                    out["converged"].append(r.converged)
                    out["solutions"].append(x)
            return out
        for b in rest:
            x = zeros(b, self.plan.nloc)
            r = self.solve(b, x, eps, max_iter, basis)
            out["iterations"].append(r.iterations)
            out["converged"].append(r.converged)
            out["solutions"].append(x)
        return out


def scatter(v: np.ndarray, plans: Sequence[api.SlabPlan]):
    return [np.ascontiguousarray(v[p.row_begin:p.row_end]) for p in plans]
