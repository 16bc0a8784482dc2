"""The cost model restatement (paper_2203_08498_b200/cost_model.py) against the reference library
itself (oracle/_ref: proj/src/cost_model.cpp compiled from the reference sources): bitwise equal
on a grid of inputs, same exceptions."""
import ctypes as C
import os

import numpy as np
import pytest


class _Params(C.Structure):
    _fields_ = [("n", C.c_double), ("nnz", C.c_double), ("m_tilde", C.c_double), ("bandwidth", C.c_double)]


@pytest.fixture(scope="module")
def reflib():
    from oracle import REF_SO

    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    lib = C.CDLL(REF_SO)
    for name in ("_ZN6recycg4t_cgERKNS_10CostParamsE", "_ZN6recycg6t_iccgERKNS_10CostParamsE",
                 "_ZN6recycg8t_sciccgERKNS_10CostParamsE"):
        getattr(lib, name).restype = C.c_double
        getattr(lib, name).argtypes = [C.POINTER(_Params)]
    lib._ZN6recycg12gamma_sciccgEdd.restype = C.c_double
    lib._ZN6recycg12gamma_sciccgEdd.argtypes = [C.c_double, C.c_double]
    return lib


def test_cost_model_matches_reference(reflib):
    from paper_2203_08498_b200 import cost_model as cm

    rng = np.random.default_rng(3)
    for _ in range(200):
        n, nnz, m, bw = rng.uniform(0, 1e9), rng.uniform(0, 1e10), float(rng.integers(0, 129)), rng.uniform(1e-3, 1e13)
        p, q = cm.CostParams(n, nnz, m, bw), _Params(n, nnz, m, bw)
        assert cm.t_cg(p) == reflib._ZN6recycg4t_cgERKNS_10CostParamsE(C.byref(q))
        assert cm.t_iccg(p) == reflib._ZN6recycg6t_iccgERKNS_10CostParamsE(C.byref(q))
        assert cm.t_sciccg(p) == reflib._ZN6recycg8t_sciccgERKNS_10CostParamsE(C.byref(q))
        assert cm.gamma_sciccg(m, nnz / max(n, 1.0)) == reflib._ZN6recycg12gamma_sciccgEdd(m, nnz / max(n, 1.0))


def test_cost_model_errors_and_compare():
    from paper_2203_08498_b200 import cost_model as cm
    from paper_2203_08498_b200._lib import InvalidArgument

    with pytest.raises(InvalidArgument):
        cm.t_iccg(cm.CostParams(n=-1.0))
    with pytest.raises(InvalidArgument):
        cm.t_iccg(cm.CostParams(n=1.0, bandwidth=0.0))
    with pytest.raises(InvalidArgument):
        cm.gamma_sciccg(-1.0, 7.0)
    with pytest.raises(InvalidArgument):
        cm.compare_measured(0, 1.0, 5, 1.0, 8, 7.0)
    with pytest.raises(InvalidArgument):
        cm.compare_measured(5, 0.0, 5, 1.0, 8, 7.0)
    c = cm.compare_measured(100, 1.0, 50, 0.75, 16, 6.95)   # per-iteration 0.01 s vs 0.015 s
    assert c.measured == pytest.approx(1.5) and c.predicted == cm.gamma_sciccg(16, 6.95)
    assert c.rel_error == pytest.approx((1.5 - c.predicted) / c.predicted)
