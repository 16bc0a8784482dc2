import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from oracle import Oracle, Matrix
from paper_2203_08498_b200 import api, problems
o = Oracle()
ctx = api.Context(0)
for name in ["c1", "c2", "c3", "c4"]:
    cfg = problems.SMALL[name]
    h = problems.generate(cfg)
    sa, _ = o.diagonal_scale(Matrix.of(h))
    a = api.CsrMatrix(ctx, h.n, sa.rs, sa.ci, sa.va)
    f = api.IcFactor.factorize_device(ctx, a)
    fo = o.ic0_factorize(sa)
    r = o.uniform_pm1(5, 0, h.n)
    z0 = f.apply(r)
    for tile in [(16, 8), (8, 4), (32, 32)]:
        try:
            f.set_grid(cfg.grid, cfg.grid, cfg.grid, *tile)
        except Exception as e:
            print(name, tile, "rejected:", e); continue
        z = f.apply(r)
        print(name, cfg.grid, tile, "bitwise" if np.array_equal(z, o.ic_apply(fo, r)) else "DIFF", np.array_equal(z, z0))
    f.set_grid(0, 0, 0, 0, 0)
