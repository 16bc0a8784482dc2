"""Dev tool: a few batched SC-ICCG iterations on a config (default C3) with R right-hand sides and
an m-column random basis, for an ncu capture of the batched kernels:

  ncu --set full --clock-control none -k regex:"k_b_spmv_pq|k_b_tallt" -c 2 -o gpurun_out/bprof \
      python tools/profile_batched.py c3 12
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2203_08498_b200 import api, problems, sequence  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    R = int(sys.argv[2]) if len(sys.argv) > 2 else 12
    iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    kind = sys.argv[4] if len(sys.argv) > 4 else "sc"
    cfg = problems.CONFIGS[name]
    ctx = api.Context(0)
    h = problems.generate(cfg)
    p = sequence.prepare(ctx, cfg, h, validate=False)
    rng = np.random.default_rng(5)
    w = api.TallDense.from_columns(ctx, h.n, rng.standard_normal((cfg.keep, h.n)))
    basis = api.Basis(ctx, p.a, w, "sc" if kind == "sc" else "deflation")
    B = np.stack([sequence.rhs(p, k % cfg.n_rhs)[1] for k in range(R)])
    X = np.zeros_like(B)
    # three single-RHS ICCG iterations first (k_sweep / k_spmv_pq / k_pupdate / k_xr for the capture)
    x1 = np.zeros(h.n)
    api.pcg_solve(ctx, p.a, B[0], api.Ic(p.ic), x1, cfg.eps, 3)
    ctx.set_profiling(True)
    ctx.reset_stats()
    if kind == "none":
        api.pcg_solve_batch(ctx, p.a, B, api.Ic(p.ic), X, cfg.eps, iters)
    elif kind == "sc":
        api.pcg_solve_batch(ctx, p.a, B, api.Sc(basis, p.ic), X, cfg.eps, iters)
    else:
        api.deflated_pcg_solve_batch(ctx, p.a, B, api.Ic(p.ic), basis, X, cfg.eps, iters)
    ctx.synchronize()
    for c in (5, 6, 7, 8, 9):
        t, k = ctx.kernel_stats(c)
        print(c, k, round(t / max(k, 1) * 1e3, 1), "us", flush=True)


if __name__ == "__main__":
    main()
