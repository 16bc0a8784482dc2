"""Dev tool: the C4 sequence (512^3 high-contrast 7-point, 134M rows, 938M entries, 8 right-hand
sides, deflation m~ = 32) on ONE GPU: matrix assembled in HBM (rcg_matrix_generate), right-hand
sides b_k = A x_k formed on the device, the sequence driver in its memory-lean mode (recycling in
the sampler slots, unbatched accelerated solves).  BASELINE.json leaves C4's sample count open;
40 samples (> m~ = 32) keep the slots at 43 GB.  Prints one JSON line.

usage: python tools/c4_run.py [samples]
"""
import json
import os
import sys
import time
from dataclasses import replace

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2203_08498_b200 import api, problems  # noqa: E402


def main():
    import torch

    samples = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    cfg = replace(problems.CONFIGS["c4"], sampler_m=samples)
    ctx = api.Context(0)
    t0 = time.perf_counter()
    a = problems.generate_device(ctx, cfg)
    ctx.synchronize()
    t_gen = time.perf_counter() - t0
    n = a.n
    t0 = time.perf_counter()
    seq = api.Sequence(ctx, a, "es-d-iccg")
    ctx.synchronize()
    t_prep = time.perf_counter() - t0
    dev = torch.device("cuda", 0)
    B = torch.empty((cfg.n_rhs, n), dtype=torch.float64, device=dev)
    for k in range(cfg.n_rhs):
        xk = torch.from_numpy(problems.solution_stream(cfg, n, k)).to(dev)
        a.spmv(xk, B[k])
        del xk
    X = torch.zeros_like(B)
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    ctx.record(0)
    rep = seq.run(B, X, cfg.eps, cfg.max_iter, "A", cfg.sampler_m, keep_count=cfg.keep)
    ctx.record(1)
    ms = ctx.elapsed_ms(0, 1)
    its = sum(rep["iterations"])
    print(json.dumps({"config": cfg.name, "n": n, "nnz": a.nnz, "samples": samples, "m_tilde": rep["m_tilde"],
                      "m_bar": rep["m_bar"], "iterations": rep["iterations"], "sequence_ms": round(ms, 1),
                      "iters_per_s": round(its / (ms / 1e3), 3), "solve_wall_s": [round(v, 3) for v in rep["wall_time"]],
                      "recycling_s": round(rep["w_build_time"], 3), "max_true_relres": max(rep["true_relres"]),
                      "device_generation_s": round(t_gen, 2), "prepare_s": round(t_prep, 2),
                      "free_gb_before_run": round(free0 / 2**30, 1)}), flush=True)


if __name__ == "__main__":
    main()
