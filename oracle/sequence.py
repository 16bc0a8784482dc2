"""Sequence protocol on the CPU oracle (TEST INFRASTRUCTURE ONLY) -- mirrors run_sequence
(proj/src/driver.cpp:108-222): diagonal scaling, IC(0), solve 1 with the method-A error
sampler, Rayleigh-Ritz basis, then SC or deflated solves 2..k from x0 = 0.  Inputs come from
the shared generators (paper_2203_08498_b200.problems), so the GPU harness sees identical data.
Count-based selection: build_aux with theta = +inf returns every Ritz vector in ascending
order; keeping the first `keep` equals theta halfway between the keep-th and (keep+1)-th value.
"""
from __future__ import annotations

import numpy as np

from . import Matrix, Oracle


def rhs_set(o: Oracle, cfg, host, a_orig: Matrix, dis, new_of_old=None):
    from .inputs import solution_stream

    xs = [solution_stream(cfg, host.n, k) for k in range(cfg.n_rhs)]
    if new_of_old is not None:  # multicolour variant: the solver sees P A P^T and P x
        perm = []
        for x in xs:
            xp = np.empty_like(x)
            xp[new_of_old] = x
            perm.append(xp)
        xs = perm
    b_orig = [o.spmv(a_orig, x) for x in xs]
    return b_orig, [dis * b for b in b_orig]


def run_sequence(o: Oracle, cfg, host, blocks: int = 1, n_solves: int | None = None, new_of_old=None) -> dict:
    a_orig = Matrix.of(host)
    a, dis = o.diagonal_scale(a_orig)
    ic = o.ic0_factorize(a, 0.0, blocks)
    b_orig, bs = rhs_set(o, cfg, host, a_orig, dis, new_of_old)
    n = host.n
    k_t = cfg.n_rhs if n_solves is None else n_solves
    out = {"iterations": [], "converged": [], "histories": [], "solutions": [], "true_relres": [],
           "shift_used": ic.shift_used, "wall": []}
    sampler = o.sampler_a(cfg.sampler_m, cfg.max_iter, n)
    x1 = np.zeros(n)
    r1 = o.pcg_solve(a, bs[0], x1, kind=1, ic=ic, eps=cfg.eps, max_iter=cfg.max_iter, sampler=sampler)
    _record(o, out, r1, x1, a_orig, b_orig[0], dis)
    occ, it = sampler.state()
    out["sampled_iterations"] = sorted(int(v) for v in it[occ])
    errors = o.harvest_errors(x1, sampler)
    m_bar, vals, w_all = o.build_aux(a, errors, float("inf"))
    keep = cfg.keep if m_bar > cfg.keep else m_bar
    w = w_all[:keep]
    out.update(m_bar=m_bar, m_tilde=keep, ritz_values=vals, x1=x1.copy(), errors=errors, w=w)
    if keep == 0:
        basis = None
    else:
        basis = o.basis(a, w, who=1 if cfg.method == "sc" else 0)
    for k in range(1, k_t):
        xk = np.zeros(n)
        if basis is None:
            rk = o.pcg_solve(a, bs[k], xk, kind=1, ic=ic, eps=cfg.eps, max_iter=cfg.max_iter)
        elif cfg.method == "sc":
            rk = o.pcg_solve(a, bs[k], xk, kind=2, ic=ic, sc=basis, eps=cfg.eps, max_iter=cfg.max_iter)
        else:
            rk = o.deflated_pcg_solve(a, bs[k], xk, basis, kind=1, ic=ic, eps=cfg.eps, max_iter=cfg.max_iter)
        _record(o, out, rk, xk, a_orig, b_orig[k], dis)
    out["scaled_rhs"] = bs
    return out


def _record(o, out, rep, x, a_orig, b_orig, dis):
    out["iterations"].append(rep.iterations)
    out["converged"].append(rep.converged)
    out["histories"].append(rep.history)
    out.setdefault("alphas", []).append(rep.alphas)
    out.setdefault("betas", []).append(rep.betas)
    out["solutions"].append(x.copy())
    out["wall"].append(rep.wall_time)
    x_orig = dis * x
    r = b_orig - o.spmv(a_orig, x_orig)
    out["true_relres"].append(float(np.linalg.norm(r) / np.linalg.norm(b_orig)))
