"""The sequence protocol on the GPU -- the caller of the hot path, mirroring run_sequence
(proj/src/driver.cpp:108-222): scale, IC(0), solve 1 with the method-A error sampler,
Rayleigh-Ritz basis (count-based selection of `keep` vectors), then SC-preconditioned or
deflated solves 2..k from x0 = 0.  All solver work runs through librcg_b200.so; the host only
scales right-hand sides / solutions (driver.cpp:147,182,191) and reports.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import api
from .problems import Config, HostCsr, solution_stream


@dataclass
class Prepared:
    ctx: api.Context
    cfg: Config
    host: HostCsr
    a_orig: api.CsrMatrix
    a: api.CsrMatrix
    dis: np.ndarray
    ic: api.IcFactor
    setup_s: float = 0.0
    new_of_old: np.ndarray | None = None   # multicolour variant: rows of P A P^T


def prepare(ctx: api.Context, cfg: Config, host: HostCsr, validate: bool = True, blocks: int | None = None,
            new_of_old: np.ndarray | None = None) -> Prepared:
    """`host` is the matrix the solver sees (P A P^T for the multicolour variant, with
    `new_of_old` the permutation applied to the generator's solution streams)."""
    t0 = time.perf_counter()
    a_orig = api.CsrMatrix(ctx, host.n, host.row_start, host.col_idx, host.values, validate=validate)
    a, dis = api.diagonal_scale(ctx, a_orig)
    # IC(0) on the device (pattern + numeric; bitwise the reference factor)
    ic = api.IcFactor.factorize_device(ctx, a, 0.0, cfg.blocks if blocks is None else blocks)
    return Prepared(ctx, cfg, host, a_orig, a, dis, ic, time.perf_counter() - t0, new_of_old)


def rhs_all(p: Prepared) -> list:
    """[(b_orig, b_scaled)] for every solve of the sequence (one pass over the solution stream)."""
    from .problems import solution_streams

    out = []
    for x in solution_streams(p.cfg, p.host.n, p.cfg.n_rhs):
        if p.new_of_old is not None:
            xp = np.empty_like(x)
            xp[p.new_of_old] = x
            x = xp
        b = p.a_orig.spmv(x)
        out.append((b, p.dis * b))
    return out


def rhs(p: Prepared, k: int) -> tuple[np.ndarray, np.ndarray]:
    """(b_orig, b_scaled) of solve k (0-based): b = A x_k, scaled by D^-1/2 (scaling.cpp:8-12)."""
    x = solution_stream(p.cfg, p.host.n, k)
    if p.new_of_old is not None:
        xp = np.empty_like(x)
        xp[p.new_of_old] = x
        x = xp
    b = p.a_orig.spmv(x)
    return b, p.dis * b


@dataclass
class SequenceResult:
    iterations: list = field(default_factory=list)
    converged: list = field(default_factory=list)
    histories: list = field(default_factory=list)
    solutions: list = field(default_factory=list)
    true_relres: list = field(default_factory=list)
    wall: list = field(default_factory=list)
    sampled_iterations: list = field(default_factory=list)
    m_bar: int = 0
    m_tilde: int = 0
    ritz_values: np.ndarray = field(default_factory=lambda: np.zeros(0))
    basis_build_s: float = 0.0


def context_pool(p: Prepared, size: int) -> list:
    """Extra contexts (each its own CUDA stream and workspace) on the same GPU, for running
    independent solves concurrently; cached on the Prepared problem."""
    pool = getattr(p, "_pool", None)
    if pool is None or len(pool) < size:
        pool = [api.Context(p.ctx.device) for _ in range(size)]
        p._pool = pool
    return pool[:size]


def run_accelerated(p: Prepared, basis, bs: list, xs: list, concurrency: int = 1) -> list:
    """Solves 2..k of the sequence (independent given W): SC-PCG or deflated PCG for each
    (b, x) pair.  With concurrency > 1 the solves run on separate contexts/streams from a thread
    pool (the C-ABI releases the GIL), so their latency-bound sweeps overlap on the GPU; each
    solve's arithmetic is unchanged."""
    cfg = p.cfg

    def one(ctx, b, x):
        if basis is None:
            return api.pcg_solve(ctx, p.a, b, api.Ic(p.ic), x, cfg.eps, cfg.max_iter)
        if cfg.method == "sc":
            return api.pcg_solve(ctx, p.a, b, api.Sc(basis, p.ic), x, cfg.eps, cfg.max_iter)
        return api.deflated_pcg_solve(ctx, p.a, b, api.Ic(p.ic), basis, x, cfg.eps, cfg.max_iter)

    if concurrency == "batch":
        return run_batched(p, basis, bs, xs)
    if concurrency <= 1:
        return [one(p.ctx, b, x) for b, x in zip(bs, xs)]
    import queue
    from concurrent.futures import ThreadPoolExecutor

    pool = context_pool(p, min(concurrency, len(bs)))
    free = queue.Queue()
    for c in pool:
        free.put(c)

    def checked_out(b, x):
        ctx = free.get()  # a context (stream + workspace) is owned by one solve at a time
        try:
            return one(ctx, b, x)
        finally:
            free.put(ctx)

    p.ctx.synchronize()
    with ThreadPoolExecutor(max_workers=len(pool)) as ex:
        futs = [ex.submit(checked_out, b, x) for b, x in zip(bs, xs)]
        return [f.result() for f in futs]


def run_batched(p: Prepared, basis, bs, xs) -> list:
    """Solves 2..k as batched multi-RHS solves (up to 16 right-hand sides per kernel sequence):
    one pass over A, the IC schedules and W per iteration serves every right-hand side.  bs / xs:
    (k, n) arrays or tensors (row slices are passed as they are: no copies) or lists of vectors."""
    cfg = p.cfg
    reps = []
    two_d = getattr(bs, "ndim", 1) == 2 and getattr(xs, "ndim", 1) == 2
    for c0 in range(0, len(bs), 16):
        chunk_b, chunk_x = bs[c0:c0 + 16], xs[c0:c0 + 16]
        if two_d:
            B, X = chunk_b, chunk_x
        elif isinstance(chunk_b[0], np.ndarray):
            B = np.ascontiguousarray(np.stack(chunk_b))
            X = np.ascontiguousarray(np.stack(chunk_x))
        else:
            import torch

            B = torch.stack(chunk_b).contiguous()
            X = torch.stack(chunk_x).contiguous()
        if basis is None:
            r = api.pcg_solve_batch(p.ctx, p.a, B, api.Ic(p.ic), X, cfg.eps, cfg.max_iter)
        elif cfg.method == "sc":
            r = api.pcg_solve_batch(p.ctx, p.a, B, api.Sc(basis, p.ic), X, cfg.eps, cfg.max_iter)
        else:
            r = api.deflated_pcg_solve_batch(p.ctx, p.a, B, api.Ic(p.ic), basis, X, cfg.eps, cfg.max_iter)
        if not two_d:
            for x_dst, x_src in zip(chunk_x, X):
                x_dst[:] = x_src
        reps += r
    return reps


def run_sequence(p: Prepared, rhs_scaled: list, rhs_orig: list | None = None, n_solves: int | None = None,
                 keep_solutions: bool = True, concurrency: int = 1) -> SequenceResult:
    ctx, cfg, n = p.ctx, p.cfg, p.host.n
    k_t = len(rhs_scaled) if n_solves is None else n_solves
    res = SequenceResult()
    sampler = api.SamplerState.method_a(ctx, cfg.sampler_m, cfg.max_iter, n)
    x1 = np.zeros(n)
    r1 = api.pcg_solve(ctx, p.a, rhs_scaled[0], api.Ic(p.ic), x1, cfg.eps, cfg.max_iter, observer=sampler)
    _record(p, res, r1, x1, rhs_orig[0] if rhs_orig else None, keep_solutions)
    occ, it = sampler.state()
    res.sampled_iterations = sorted(int(v) for v in it[occ])
    t0 = time.perf_counter()
    errors = api.harvest_errors(ctx, x1, sampler)
    m_bar, vals, _theta, w = api.build_aux_matrix(ctx, p.a, errors, 1e-3, keep_count=cfg.keep)
    res.m_bar, res.m_tilde, res.ritz_values = m_bar, w.k, vals
    basis = api.Basis(ctx, p.a, w, "sc" if cfg.method == "sc" else "deflation") if w.k > 0 else None
    res.basis_build_s = time.perf_counter() - t0
    xs = [np.zeros(n) for _ in range(1, k_t)]
    reps = run_accelerated(p, basis, rhs_scaled[1:k_t], xs, concurrency)
    for k, (rk, xk) in enumerate(zip(reps, xs), start=1):
        _record(p, res, rk, xk, rhs_orig[k] if rhs_orig else None, keep_solutions)
    return res


def _record(p: Prepared, res: SequenceResult, rep, x, b_orig, keep):
    res.iterations.append(rep.iterations)
    res.converged.append(rep.converged)
    res.histories.append(rep.history)
    res.wall.append(rep.wall_time)
    if keep:
        res.solutions.append(x.copy())
    if b_orig is not None:
        x_orig = p.dis * x
        r = b_orig - p.a_orig.spmv(x_orig)
        res.true_relres.append(float(np.linalg.norm(r) / np.linalg.norm(b_orig)))
