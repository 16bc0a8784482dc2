"""Dev tool: batched ICCG on C2 -- time per iteration and per kernel class vs the batch size R."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2203_08498_b200 import api, problems, sequence  # noqa: E402


def main():
    cfg = problems.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
    ctx = api.Context(0)
    h = problems.generate(cfg)
    p = sequence.prepare(ctx, cfg, h, validate=False)
    bs = [sequence.rhs(p, k % cfg.n_rhs)[1] for k in range(24)]
    for R in [int(v) for v in os.environ.get("RS", "1,2,4,8,9,12,16").split(",")]:
        B = np.stack(bs[:R])
        for rep in range(2):
            X = np.zeros_like(B)
            ctx.set_profiling(rep == 1)
            ctx.reset_stats()
            if R == 1:
                reps = [api.pcg_solve(ctx, p.a, B[0], api.Ic(p.ic), X[0], cfg.eps, 60)]
            else:
                reps = api.pcg_solve_batch(ctx, p.a, B, api.Ic(p.ic), X, cfg.eps, 60)
        stats = {c % 5: ctx.kernel_stats(c) for c in (range(5) if R == 1 else range(5, 10))}
        ctx.set_profiling(False)
        its = max(r.iterations for r in reps)
        print(json.dumps({"R": R, "iters": its, "ms_per_iter": round(sum(r.wall_time for r in reps) / its * 1e3, 3),
                          "us": {c: round(t / max(n, 1) * 1e3, 1) for c, (t, n) in stats.items()}}), flush=True)


if __name__ == "__main__":
    main()
