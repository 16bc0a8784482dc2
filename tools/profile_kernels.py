"""Dev tool: a short C2 run that launches each hot kernel a few times, for one
`ncu --set full` capture: a 4-iteration single-RHS SC-ICCG solve and a 4-iteration batched
SC-ICCG solve of 9 right-hand sides (RT = 12) on the bench workload.

  ncu --set full --clock-control none --import-source on \
      -k regex:"k_sweep|k_b_sweep|spmv_pq|k_b_tallt|k_b_xr|k_b_pupdate|k_tallt" \
      --nvtx --nvtx-include "prof/" -o gpurun_out/prof python tools/profile_kernels.py
(only launches inside the NVTX range "prof" are captured: the batched solve; the single-RHS
kernels come from a --launch-skip capture of the same script)
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2203_08498_b200 import api, problems, sequence  # noqa: E402


def main():
    cfg = problems.CONFIGS["c2"]
    ctx = api.Context(0)
    h = problems.generate(cfg)
    p = sequence.prepare(ctx, cfg, h, validate=False)
    bs = [sequence.rhs(p, k)[1] for k in range(cfg.n_rhs)]
    # basis from a short solve 1 (the sampler needs a full solve; 40 iterations is enough here)
    s = api.SamplerState.method_a(ctx, cfg.sampler_m, cfg.max_iter, h.n)
    x = np.zeros(h.n)
    api.pcg_solve(ctx, p.a, bs[0], api.Ic(p.ic), x, cfg.eps, cfg.max_iter, observer=s)
    e = api.harvest_errors(ctx, x, s)
    _, _, _, w = api.build_aux_matrix(ctx, p.a, e, 1e-3, keep_count=cfg.keep)
    basis = api.Basis(ctx, p.a, w, "sc")
    import torch

    x = np.zeros(h.n)
    api.pcg_solve(ctx, p.a, bs[1], api.Sc(basis, p.ic), x, cfg.eps, 4)
    B = np.stack(bs[1:])
    X = np.zeros_like(B)
    ctx.synchronize()
    torch.cuda.nvtx.range_push("prof")
    api.pcg_solve_batch(ctx, p.a, B, api.Sc(basis, p.ic), X, cfg.eps, 4)
    ctx.synchronize()
    torch.cuda.nvtx.range_pop()
    print("ok")


if __name__ == "__main__":
    main()
