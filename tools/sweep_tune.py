"""Dev tool: times ic_apply (forward + backward sweep) and spmv on a config for the current
RCG_SWEEP_BPS / RCG_SWEEP_BACKOFF_NS environment.  Usage: python tools/sweep_tune.py c2 [reps]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2203_08498_b200 import api, problems  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    import torch

    mc = name.endswith("mc")
    name = name[:-2] if mc else name
    cfg = problems.CONFIGS.get(name) or problems.SMALL[name.replace("s_", "")]
    ctx = api.Context(0)
    if mc:  # multicolour variant: sweeps have ncolors levels
        h = problems.multicolour(problems.generate(cfg))[0]
        a = api.CsrMatrix(ctx, h.n, h.row_start, h.col_idx, h.values, validate=False)
    else:
        a = problems.generate_device(ctx, cfg)
    sa, dis = api.diagonal_scale(ctx, a)
    f = api.IcFactor.factorize_device(ctx, sa)
    r = torch.from_numpy(problems.uniform_pm1(1, 0, sa.n)).cuda()
    z = torch.empty_like(r)
    for _ in range(3):
        f.apply(r, z)
    ctx.set_profiling(True)
    ctx.reset_stats()
    t0 = time.perf_counter()
    for _ in range(reps):
        f.apply(r, z)
    ctx.synchronize()
    wall = (time.perf_counter() - t0) / reps
    fw = ctx.kernel_stats(1)
    bw = ctx.kernel_stats(2)
    for _ in range(reps):
        sa.spmv(r, z)
    sp = ctx.kernel_stats(0)
    print(json.dumps({"config": cfg.name, "n": sa.n, "mode": os.environ.get("RCG_SWEEP_CLUSTER", "2"), "fwd_levels": f.fwd_levels, "bwd_levels": f.bwd_levels,
                      "bps": os.environ.get("RCG_SWEEP_BPS", "4"),
                      "backoff": os.environ.get("RCG_SWEEP_BACKOFF_NS", "32"),
                      "fwd_us": round(fw[0] / fw[1] * 1e3, 1), "bwd_us": round(bw[0] / bw[1] * 1e3, 1),
                      "us_per_level": round(fw[0] / fw[1] * 1e3 / f.fwd_levels, 3),
                      "spmv_us": round(sp[0] / sp[1] * 1e3, 1), "apply_wall_us": round(wall * 1e6, 1)}))


if __name__ == "__main__":
    main()
