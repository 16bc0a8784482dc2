"""Dev tool: the hot kernels on every BASELINE.json configuration -- SpMV, IC(0) forward / backward
sweeps (single right-hand side and batched), and one short ICCG solve -- as algorithmic GB/s
against the measured HBM peak.  Results go to profiles/ (DESIGN.md section 8).

usage: python tools/config_probe.py c1 c2 c3 c4 c5 [--mc] [--batch R]
  --mc       also the multicolour-reordered operator (a different operator, reported separately)
  --batch R  batched ICCG with R right-hand sides (default 8; 0 = skip)
Bytes per launch: spmv 12 nnz + 20 n; fwd 12 nnz_L + 24 n; bwd 12 nnz_L + 40 n
(single); batched as bench.py's algorithmic_bytes.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2203_08498_b200 import api, problems, sequence  # noqa: E402


def peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    return float(json.load(open(p))["hbm_gbs"]) if os.path.exists(p) else 6650.0


def bytes_of(c, n, nnz, nnz_l, rt=1):
    fixed, per = {0: (12 * nnz + 4 * n, 16 * n), 1: (12 * nnz_l + 8 * n, 16 * n),
                  2: (12 * nnz_l + 16 * n, 24 * n)}[c % 5]
    return fixed + per * rt


def probe(ctx, name, h, batch, pk, levels_note=""):
    import torch

    cfg = problems.CONFIGS[name]
    t0 = time.perf_counter()
    p = sequence.prepare(ctx, cfg, h, validate=False)
    setup_s = time.perf_counter() - t0
    n, nnz, nnz_l = h.n, h.nnz, p.ic.nnz_l
    out = {"config": cfg.name + levels_note, "n": n, "nnz": nnz, "nnz_l": nnz_l,
           "fwd_levels": p.ic.fwd_levels, "bwd_levels": p.ic.bwd_levels, "setup_s": round(setup_s, 2)}
    r = torch.from_numpy(problems.uniform_pm1(1, 0, n)).cuda()
    z = torch.empty_like(r)
    reps = 20 if n < 50_000_000 else 6
    for _ in range(3):
        p.ic.apply(r, z)
        p.a.spmv(r, z)
    ctx.synchronize()
    ctx.set_profiling(True)
    ctx.reset_stats()
    for _ in range(reps):
        p.ic.apply(r, z)
        p.a.spmv(r, z)
    ctx.synchronize()
    for c, key in ((0, "spmv"), (1, "fwd"), (2, "bwd")):
        t, k = ctx.kernel_stats(c)
        us = t / k * 1e3
        gbs = bytes_of(c, n, nnz, nnz_l) / (us * 1e-6) / 1e9
        out[key] = {"us": round(us, 1), "gbs": round(gbs, 1), "frac": round(gbs / pk, 4)}
    out["us_per_level_fwd"] = round(out["fwd"]["us"] / max(p.ic.fwd_levels, 1), 3)
    # a short ICCG solve (max_iter 30): per-iteration device time
    b = sequence.rhs(p, 0)[1]
    ctx.reset_stats()
    x = np.zeros(n)
    rep = api.pcg_solve(ctx, p.a, b, api.Ic(p.ic), x, cfg.eps, 30)
    out["iccg_ms_per_iter"] = round(rep.wall_time / rep.iterations * 1e3, 4)
    if batch:
        B = np.stack([sequence.rhs(p, k % cfg.n_rhs)[1] for k in range(batch)])
        for rep_i in range(2):
            X = np.zeros_like(B)
            ctx.reset_stats()
            reps_b = api.pcg_solve_batch(ctx, p.a, B, api.Ic(p.ic), X, cfg.eps, 20)
        its = max(r_.iterations for r_ in reps_b)
        bt = {}
        for c, key in ((5, "spmv"), (6, "fwd"), (7, "bwd")):
            t, k = ctx.kernel_stats(c)
            u = ctx.kernel_units(c)
            if not k:
                continue
            us = t / k * 1e3
            rt = u / k
            gbs = bytes_of(c, n, nnz, nnz_l, rt) / (us * 1e-6) / 1e9
            bt[key] = {"us": round(us, 1), "rhs_per_launch": round(rt, 2), "gbs": round(gbs, 1),
                       "frac": round(gbs / pk, 4)}
        out["batched"] = {"R": batch, "ms_per_iter": round(reps_b[0].wall_time * batch / its * 1e3, 4),
                          "ms_per_rhs_iter": round(reps_b[0].wall_time / its * 1e3, 4), **bt}
    ctx.set_profiling(False)
    del p
    return out


def main():
    args = [a for a in sys.argv[1:]]
    mc = "--mc" in args
    batch = 8
    if "--batch" in args:
        i = args.index("--batch")
        batch = int(args[i + 1])
        del args[i:i + 2]
    names = [a for a in args if not a.startswith("--")] or ["c2"]
    ctx = api.Context(0)
    pk = peak()
    for name in names:
        h = problems.generate(problems.CONFIGS[name])
        print(json.dumps(probe(ctx, name, h, batch, pk)), flush=True)
        if mc:
            m, _, nc = problems.multicolour(h)
            del h
            print(json.dumps(probe(ctx, name, m, batch, pk, f" multicolour({nc})")), flush=True)
        import gc

        gc.collect()


if __name__ == "__main__":
    main()
