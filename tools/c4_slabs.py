"""Dev tool: the C4 sequence through the ROW-SLAB path on one GPU: G loopback slabs
(default 1) at the reference block bounds, block-Jacobi IC(0) per slab (device factorisation),
distributed sampled solve 1, memory-lean distributed recycling (automatic at this size), deflated
solves over the slabs.  40 samples (BASELINE.json leaves C4's count open).  Prints one JSON line.

usage: python tools/c4_slabs.py [G] [config]   (config: c4 by default; c5 runs the 4M-point kNN
Laplacian through the same path, with its irregular halo, 48 samples as BASELINE.json states)
"""
import json
import os
import sys
import time
from dataclasses import replace

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2203_08498_b200 import api, dist, problems  # noqa: E402


def main():
    G = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    name = sys.argv[2] if len(sys.argv) > 2 else "c4"
    cfg = problems.CONFIGS[name]
    if name == "c4":
        cfg = replace(cfg, sampler_m=40)
    ctx = api.Context(0)
    t0 = time.perf_counter()
    h = problems.generate(cfg)
    a = api.CsrMatrix(ctx, h.n, h.row_start, h.col_idx, h.values, validate=False)
    sa, dis = api.diagonal_scale(ctx, a)
    del a
    bs = [sa.spmv(problems.solution_stream(cfg, h.n, k) / dis) for k in range(cfg.n_rhs)]  # D^-1/2 A x
    scaled = problems.HostCsr(h.n, h.row_start, h.col_idx, sa.values())
    del sa, h
    t_setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    system = dist.LoopbackSystem(scaled, G, device_factor=True)
    t_slabs = time.perf_counter() - t0
    t0 = time.perf_counter()
    out = system.sequence(bs, cfg.eps, cfg.max_iter, cfg.sampler_m, cfg.keep,
                          "sc" if cfg.method == "sc" else "deflation")
    secs = time.perf_counter() - t0
    its = int(sum(out["iterations"]))
    print(json.dumps({"config": cfg.name, "slabs": G, "n": scaled.n, "samples": cfg.sampler_m,
                      "iterations": [int(v) for v in out["iterations"]], "m_bar": int(out["m_bar"]),
                      "m_tilde": int(out["m_tilde"]), "sequence_s": round(secs, 2),
                      "iters_per_s": round(its / secs, 3), "setup_s": round(t_setup, 1),
                      "slab_build_s": round(t_slabs, 1)}), flush=True)


if __name__ == "__main__":
    main()
