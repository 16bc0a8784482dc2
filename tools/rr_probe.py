"""Dev tool: wall time of each Rayleigh-Ritz / basis sub-step on C2, repeated."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2203_08498_b200 import api, problems, sequence  # noqa: E402


def main():
    cfg = problems.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
    ctx = api.Context(0)
    h = problems.generate(cfg)
    p = sequence.prepare(ctx, cfg, h, validate=False)
    b = sequence.rhs(p, 0)[1]
    for rep in range(4):
        t = {}
        t0 = time.perf_counter()
        s = api.SamplerState.method_a(ctx, cfg.sampler_m, cfg.max_iter, h.n)
        x = np.zeros(h.n)
        r = api.pcg_solve(ctx, p.a, b, api.Ic(p.ic), x, cfg.eps, cfg.max_iter, observer=s)
        ctx.synchronize()
        t["solve1"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        e = api.harvest_errors(ctx, x, s)
        ctx.synchronize()
        t["harvest"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        q = api.mgs_orthonormalize(ctx, e)
        ctx.synchronize()
        t["mgs"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        vals, vecs = api.rayleigh_ritz(ctx, p.a, q, vectors=True)
        ctx.synchronize()
        t["rr"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        mb, v2, th, w = api.build_aux_matrix(ctx, p.a, e, 1e-3, keep_count=cfg.keep)
        ctx.synchronize()
        t["build_aux"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        basis = api.Basis(ctx, p.a, w, "sc")
        ctx.synchronize()
        t["basis"] = time.perf_counter() - t0
        print({k: round(v * 1e3, 2) for k, v in t.items()}, "its", r.iterations, "m_bar", mb, flush=True)
        del basis, w, vecs, q, e, s


if __name__ == "__main__":
    main()
