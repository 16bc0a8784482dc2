"""Dev tool: per-solve iteration counts of one sequence through rcg_seq_run, batched and unbatched
(usage: python tools/seq_iters.py [config])."""
import sys

import numpy as np
sys.path.insert(0, '.')
from paper_2203_08498_b200 import api, problems, sequence
ctx = api.Context(0)
cfg = problems.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
host = problems.generate(cfg)
prep = sequence.prepare(ctx, cfg, host, validate=False)
B = np.stack([sequence.rhs(prep, k)[0] for k in range(cfg.n_rhs)])
X = np.zeros_like(B)
seq = api.Sequence(ctx, prep.a_orig, "es-sc-iccg" if cfg.method == "sc" else "es-d-iccg")
for batch in (True, False):
    X[:] = 0
    rep = seq.run(B, X, cfg.eps, cfg.max_iter, "A", cfg.sampler_m, keep_count=cfg.keep, batch=batch)
    print("batch", batch, rep["iterations"], rep["m_bar"], rep["m_tilde"], flush=True)
