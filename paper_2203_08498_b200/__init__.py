"""B200-native hot path of the deflated / subspace-corrected ICCG solver with error-vector
sampling (arxiv 2203.08498, reference `recycg`).

The product is librcg_b200.so (csrc/, C-ABI in include/rcg_b200.h): hand-written sm_100a CUDA
kernels for SpMV, level-scheduled IC(0) sweeps, fused PCG vector ops, deflation / subspace
correction projections, the Rayleigh-Ritz step and the condition estimators.  ``api`` mirrors
the reference solver API over that C-ABI; ``problems`` generates the BASELINE.json inputs;
``sequence`` runs the paper's sequence protocol.
"""
from . import api, problems  # noqa: F401
from ._lib import LIB_PATH  # noqa: F401

__version__ = "0.1.0"
