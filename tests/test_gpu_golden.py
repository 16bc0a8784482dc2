"""The sequence protocol at the BASELINE.json sizes against the CPU oracle's full-size goldens
(tests/golden/<config>.json, made by tools/make_goldens.py from oracle/oracle.c -- pinned
bitwise to the reference library): rcg_seq_run on C3 (256^3 Q1 27-point, 20 drifting RHS, 64
samples, deflation m~ = 32), C5 (4M-point kNN, 16 solves, Lanczos kappa each, deflation m~ = 24),
C2 (the bench workload) and the C4-like 256^3 case (C4's inclusions and protocol).

Bars (north star): every solve's iteration count within +-2; m_bar and m_tilde equal; Ritz values
<= max(1e-6, 10 x the oracle's own reduction-order floor); the Lanczos condition estimate within 1 % (solve 1; the accelerated solves, on each side's own
W: max(1 %, 10 x the kept Ritz values' floor)); solve 1's solution
(at 8,192 seeded rows, in the original scaling) within max(1e-8, 10 x the oracle's own
reduction-order floor) when the counts agree; true relative residuals at the tolerance.  Solves
2..k run on each side's own W (the GPU's differs from the oracle's at rounding level), so they
are compared by iterations, kappa and residual, not by solution.  Each check's achieved value is
logged (parity_log)."""
import glob
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
GOLDENS = sorted(p for p in glob.glob(os.path.join(GOLDEN, "*.json")) if "_first" not in p)


def _config(name):
    from paper_2203_08498_b200.configs import CONFIGS, VARIANTS

    for c in list(CONFIGS.values()) + list(VARIANTS.values()):
        if c.name == name:
            return c
    raise KeyError(name)


@pytest.mark.parametrize("path", GOLDENS, ids=[os.path.basename(p)[:-5] for p in GOLDENS])
def test_sequence_matches_full_size_golden(ctx, problems, parity_log, path):
    import hashlib

    from oracle import inputs
    from paper_2203_08498_b200 import api

    gold = json.load(open(path))
    cfg = _config(gold["config"])
    h = problems.generate(cfg)
    assert h.n == gold["n"] and h.nnz == gold["inputs"]["nnz"]
    assert hashlib.sha256(h.values.tobytes()).hexdigest() == gold["inputs"]["values_sha256"], "generator drift"
    assert hashlib.sha256(h.col_idx.tobytes()).hexdigest() == gold["inputs"]["col_idx_sha256"]
    a = api.CsrMatrix(ctx, h.n, h.row_start, h.col_idx, h.values, validate=False)
    k_t = gold["n_rhs"]
    B = np.empty((k_t, h.n))
    for k, x in enumerate(inputs.solution_streams(cfg, h.n, k_t)):
        B[k] = a.spmv(x)  # bitwise the oracle's b = A x_k
    X = np.zeros_like(B)
    seq = api.Sequence(ctx, a, "es-sc-iccg" if cfg.method == "sc" else "es-d-iccg")
    rep = seq.run(B, X, cfg.eps, cfg.max_iter, "A", cfg.sampler_m, keep_count=cfg.keep, condest=True)
    name = gold["config"]
    its_o = gold["iterations"]
    parity_log(f"golden:{name}", iterations_gpu=rep["iterations"], iterations_oracle=its_o,
               m_bar=(rep["m_bar"], gold["m_bar"]), m_tilde=(rep["m_tilde"], gold["m_tilde"]))
    assert rep["m_bar"] == gold["m_bar"] and rep["m_tilde"] == gold["m_tilde"]
    # Ritz values: within max(1e-6, 10 x the oracle's own reduction-order floor -- make_goldens.py
    # --floor: solve 1 + the recycling step with the dot products summed backwards / pairwise; the
    # largest change over the kept m~ values for those, over all values for the rest).  On shared
    # sampled errors the Rayleigh-Ritz step itself agrees to 1e-6 (test_gpu_fullsize.py).  On C3 (64 errors) and C5 the sampled errors of late iterations are
    # differences of nearly equal iterates, so the Rayleigh-Ritz values move with rounding in the
    # reference itself; on C1 / C2 / C4-like the floor is far below 1e-6 and the bar is 1e-6.
    rv = np.asarray(gold["ritz_values"])
    rel = np.abs(np.asarray(rep["ritz_values"][:len(rv)]) - rv) / np.abs(rv)
    floor = np.asarray(gold.get("ritz_floor", {}).get("rel", np.zeros(rv.size)))
    mt = gold["m_tilde"]
    # the set's floor: how far the oracle's own kept (resp. all) Ritz values move
    bar_kept = max(1e-6, 10.0 * float(floor[:mt].max()))
    bar_all = max(1e-6, 10.0 * float(floor.max()))
    kept, w = float(rel[:mt].max()), int(rel.argmax())
    parity_log(f"golden:{name}", check="ritz_rel_kept", achieved=kept, bar=bar_kept, floor=float(floor[:mt].max()))
    parity_log(f"golden:{name}", check="ritz_rel_all", achieved=float(rel[w]), index=w, bar=bar_all,
               floor=float(floor.max()), per_value=[float(v) for v in rel], floor_per_value=[float(v) for v in floor])
    assert kept <= bar_kept, (kept, bar_kept)
    assert float(rel.max()) <= bar_all, (w, float(rel[w]), bar_all)
    # Lanczos kappa: solve 1 (the same operator on both sides) within 1 %; the accelerated solves
    # run on each side's own W, whose kept Ritz values the reference itself moves by up to
    # floor[:m~] -- their kappa within max(1 %, 10 x that floor)
    kap = [abs(g / s["kappa"] - 1.0) for g, s in zip(rep["kappa"], gold["solves"])]
    bar_acc = max(0.01, 10.0 * float(floor[:mt].max()) if mt else 0.01)
    parity_log(f"golden:{name}", check="kappa_rel", achieved=max(kap), bar_solve1=0.01, bar_accelerated=bar_acc,
               per_solve=kap)
    assert kap[0] <= 0.01, kap
    assert max(kap[1:], default=0.0) <= bar_acc, (kap, bar_acc)
    for k in range(k_t):
        assert rep["converged"][k]
        assert abs(rep["iterations"][k] - its_o[k]) <= 2, (k, rep["iterations"], its_o)
        assert rep["true_relres"][k] <= max(10 * gold["solves"][k]["true_relres"], 10 * cfg.eps), k
    # solve 1: the same operator and right-hand side -- the floor protocol at equal counts
    if rep["iterations"][0] == its_o[0]:
        xs = np.load(path[:-5] + "_x.npz")
        rows, xo = xs["rows"], xs["x"][0]
        rel = float(np.linalg.norm(X[0][rows] - xo) / np.linalg.norm(xo))
        floor = gold.get("solve1_floor", {}).get("rel_solution", 0.0)
        bar = max(1e-8, 10 * floor)
        parity_log(f"golden:{name}", check="solve1_solution_rel", achieved=rel, bar=bar, floor=floor)
        assert rel <= bar, (rel, bar)
        assert gold["sampled_iterations"] == sorted(gold["sampled_iterations"])
