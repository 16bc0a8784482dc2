"""Dev tool: IC(0) setup time, host restatement vs device numeric factorisation, per config."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2203_08498_b200 import api, problems  # noqa: E402


def main():
    ctx = api.Context(0)
    for name in sys.argv[1:] or ["c2"]:
        cfg = problems.CONFIGS[name]
        h = problems.generate(cfg)
        a = api.CsrMatrix(ctx, h.n, h.row_start, h.col_idx, h.values, validate=False)
        sa, _ = api.diagonal_scale(ctx, a)
        va = sa.values()
        out = {"config": cfg.name, "n": h.n, "nnz": h.nnz}
        for rep in range(2):
            t0 = time.perf_counter()
            fd = api.IcFactor.factorize_device(ctx, sa)
            ctx.synchronize()
            out["device_s"] = round(time.perf_counter() - t0, 3)
            del fd
        t0 = time.perf_counter()
        fh = api.IcFactor.factorize(ctx, h.n, h.row_start, h.col_idx, va)
        out["host_s"] = round(time.perf_counter() - t0, 3)
        del fh
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
