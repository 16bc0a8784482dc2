"""B200-native hot path of the deflated / subspace-corrected ICCG solver with error-vector
sampling (arxiv 2203.08498, reference `recycg`).

The product is librcg_b200.so (csrc/, C-ABI in include/rcg_b200.h): hand-written sm_100a CUDA
kernels for SpMV, level-scheduled IC(0) sweeps, fused PCG vector ops, deflation / subspace
correction projections, the Rayleigh-Ritz step and the condition estimators.  ``api`` mirrors
the reference solver API over that C-ABI; ``problems`` generates the BASELINE.json inputs;
``sequence`` runs the paper's sequence protocol.

Submodules load lazily, so ``paper_2203_08498_b200.configs`` (plain data) can be read without
mapping the library; every module that calls it (``api``, ``problems``, ...) raises at import
when librcg_b200.so is missing -- there is no fallback.
"""
import importlib

__version__ = "0.2.0"
_LAZY = ("api", "problems", "sequence", "dist", "cost_model", "configs", "_lib")


def __getattr__(name):
    if name in _LAZY:
        return importlib.import_module(f".{name}", __name__)
    if name == "LIB_PATH":
        return importlib.import_module("._lib", __name__).LIB_PATH
    raise AttributeError(name)
