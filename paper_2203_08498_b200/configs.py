"""The BASELINE.json configurations (C1-C5) and their scaled-down parity variants -- plain data,
no native library: the reference arm of bench.py and the oracle's input generator
(oracle/inputs.py) read these without mapping librcg_b200.so.  SURVEY.md section 8(d) defines
each problem; csrc/generators.cpp generates them.
"""
from __future__ import annotations

from dataclasses import dataclass, replace

RCG_GEN_POISSON7, RCG_GEN_FV7_CONTRAST, RCG_GEN_Q1_27PT, RCG_GEN_KNN = 0, 1, 2, 3  # rcg_b200.h


@dataclass(frozen=True)
class Config:
    name: str
    kind: int
    grid: int                 # N per axis, or the number of points (kNN)
    n_rhs: int
    rhs: str                  # 'uniform' | 'normal' | 'drift'
    sampler_m: int
    keep: int                 # m~ Ritz vectors kept (count-based selection)
    method: str               # 'deflation' | 'sc'
    condest: bool = False
    inclusions: int = 0
    inclusion_size: int = 0
    contrast: float = 1.0
    sigma: float = 0.0
    knn_k: int = 10
    seed: int = 20220317
    rhs_seed: int = 1
    eps: float = 1e-8
    max_iter: int = 5000
    blocks: int = 1
    note: str = ""


CONFIGS = {
    "c1": Config("c1_poisson7_32", RCG_GEN_POISSON7, 32, 4, "uniform", 16, 8, "deflation",
                 note="32^3 7-pt Poisson, IC(0)-CG, 4 RHS, 16 samples, deflation m=8 (CPU-runnable case)"),
    "c2": Config("c2_fv7_contrast_128", RCG_GEN_FV7_CONTRAST, 128, 10, "normal", 32, 16, "sc",
                 inclusions=8, inclusion_size=8, contrast=1e6,
                 note="128^3 high-contrast 7-pt FV, 8 inclusions 8^3 at 1e6, 10 RHS, 32 samples, SC m=16"),
    "c3": Config("c3_q1_27pt_256", RCG_GEN_Q1_27PT, 256, 20, "drift", 64, 32, "deflation", sigma=2.0,
                 note="256^3 Q1 27-pt, log-normal exp(N(0,4)), 20 RHS drifting, 64 samples, deflation m=32"),
    "c4": Config("c4_fv7_contrast_512", RCG_GEN_FV7_CONTRAST, 512, 8, "normal", 64, 32, "deflation",
                 inclusions=64, inclusion_size=16, contrast=1e6,
                 note="512^3 high-contrast 7-pt, 64 inclusions 16^3, 8 RHS, deflation m=32"),
    "c5": Config("c5_knn_laplacian_4M", RCG_GEN_KNN, 4_000_000, 16, "normal", 48, 24, "deflation", condest=True,
                 knn_k=10, note="4M-point kNN (k=10) graph Laplacian, 16 solves, condest each solve, deflation m=24"),
}

# scaled-down variants with the same structure, for parity tests the oracle finishes in seconds
SMALL = {
    "c1": CONFIGS["c1"],
    "c2": replace(CONFIGS["c2"], name="c2_small_24", grid=24, n_rhs=4, inclusions=2, inclusion_size=4, sampler_m=16,
                  keep=6),
    "c3": replace(CONFIGS["c3"], name="c3_small_12", grid=12, n_rhs=4, sampler_m=16, keep=6),
    "c4": replace(CONFIGS["c4"], name="c4_small_28", grid=28, n_rhs=3, inclusions=4, inclusion_size=4, sampler_m=16,
                  keep=6),
    "c5": replace(CONFIGS["c5"], name="c5_small_8k", grid=8000, n_rhs=3, sampler_m=16, keep=6),
}

# oracle-checked variants outside BASELINE.json's list (settle C4's "deflation does not
# reduce the iterations" on a case the CPU oracle can run): C4's inclusion size and volume fraction
# (16^3 cubes, 0.195 %) on a 256^3 grid -- 8 inclusions instead of 64 -- with C4's protocol.
VARIANTS = {
    "c4like": replace(CONFIGS["c4"], name="c4like_fv7_contrast_256", grid=256, inclusions=8, inclusion_size=16,
                      note="256^3 high-contrast 7-pt, 8 inclusions 16^3 at 1e6 (C4's volume fraction), 8 RHS, "
                           "64 samples, deflation m=32"),
}
