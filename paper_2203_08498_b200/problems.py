"""Seeded synthetic problems for the BASELINE.json configurations (C1-C5) and the right-hand
side streams of each sequence.  The reference ships no generators; SURVEY.md section 8(d)
defines them and the C++ implementation lives in csrc/generators.cpp (host code, shared by the
GPU path, the oracle harness and bench.py).  The paper's SuiteSparse matrices are not in this
environment: these seeded problems with the configs' shapes and coefficient distributions stand
in for them.
"""
from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from ._lib import check, lib


from .configs import CONFIGS, SMALL, Config  # noqa: F401,E402  (re-exported)


@dataclass
class HostCsr:
    n: int
    row_start: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.row_start[-1])


def _adopt(ptr, count, ctype, dtype):
    """numpy view of a malloc'ed library buffer, freed with rcg_host_free when collected."""
    if count == 0:
        lib.rcg_host_free(C.cast(ptr, C.c_void_p))
        return np.zeros(0, dtype)
    arr = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ctype)), shape=(count,))
    weakref.finalize(arr, lib.rcg_host_free, C.cast(ptr, C.c_void_p).value)
    return arr


def generate(cfg: Config) -> HostCsr:
    p = L.GenParams(cfg.kind, cfg.grid, cfg.inclusions, cfg.inclusion_size, cfg.contrast, cfg.sigma, cfg.knn_k,
                    cfg.seed)
    n = C.c_int32()
    nnz = C.c_int64()
    rs = L.i32p()
    ci = L.i32p()
    va = L.dp()
    check(lib.rcg_generate(C.byref(p), C.byref(n), C.byref(nnz), C.byref(rs), C.byref(ci), C.byref(va)))
    return HostCsr(n.value, _adopt(rs, n.value + 1, C.c_int32, np.int32), _adopt(ci, nnz.value, C.c_int32, np.int32),
                   _adopt(va, nnz.value, C.c_double, np.float64))


def generate_device(ctx, cfg: Config):
    """Any config assembled directly in HBM (rcg_matrix_generate): an api.CsrMatrix bitwise equal
    to generate(cfg), without host CSR arrays or their H2D copy (C3 uploads its element
    coefficients, C5 its points)."""
    from . import api

    p = L.GenParams(cfg.kind, cfg.grid, cfg.inclusions, cfg.inclusion_size, cfg.contrast, cfg.sigma, cfg.knn_k,
                    cfg.seed)
    h = C.c_void_p()
    check(lib.rcg_matrix_generate(ctx.h, C.byref(p), C.byref(h)))
    return api.CsrMatrix(ctx, 0, None, None, None, _handle=h)


def uniform_pm1(seed: int, skip: int, n: int) -> np.ndarray:
    out = np.empty(n)
    lib.rcg_uniform_pm1(C.c_uint64(seed), C.c_uint64(skip), n, out.ctypes.data)
    return out


def normal(seed: int, skip: int, n: int) -> np.ndarray:
    out = np.empty(n)
    lib.rcg_normal(C.c_uint64(seed), C.c_uint64(skip), n, out.ctypes.data)
    return out


def solution_stream(cfg: Config, n: int, k: int) -> np.ndarray:
    """x_k (0-based k) of the sequence: b_k = A x_k.  'uniform' follows make_rhs (driver.cpp:97-106)
    block k of the UniformPm1 stream; 'normal' is block k of the N(0,1) stream; 'drift' is
    x_0 ~ N(0,1), x_{k+1} = x_k + 0.1 N(0,1)."""
    if cfg.rhs == "uniform":
        return uniform_pm1(cfg.rhs_seed, k * n, n)
    if cfg.rhs == "normal":
        return normal(cfg.rhs_seed, k * n, n)
    if cfg.rhs == "drift":
        x = normal(cfg.rhs_seed, 0, n)
        for j in range(1, k + 1):
            x = x + 0.1 * normal(cfg.rhs_seed, j * n, n)
        return x
    raise ValueError(cfg.rhs)


def solution_streams(cfg: Config, n: int, count: int):
    """x_0 .. x_{count-1} in order with O(count) draws for the drifting stream (same values as
    solution_stream)."""
    x = None
    for k in range(count):
        if cfg.rhs == "drift":
            x = normal(cfg.rhs_seed, 0, n) if k == 0 else x + 0.1 * normal(cfg.rhs_seed, k * n, n)
            yield x
        else:
            yield solution_stream(cfg, n, k)


def multicolour(a: HostCsr):
    """(P A P^T, new_of_old, ncolors) for the multicolour variant (greedy colouring)."""
    new_of_old = np.empty(a.n, np.int32)
    nc = C.c_int32()
    check(lib.rcg_multicolor_order(a.n, a.row_start.ctypes.data, a.col_idx.ctypes.data, new_of_old.ctypes.data,
                                   C.byref(nc)))
    rs, ci, va = L.i32p(), L.i32p(), L.dp()
    check(lib.rcg_permute_symmetric(a.n, a.row_start.ctypes.data, a.col_idx.ctypes.data, a.values.ctypes.data,
                                    new_of_old.ctypes.data, C.byref(rs), C.byref(ci), C.byref(va)))
    nnz = a.nnz
    b = HostCsr(a.n, _adopt(rs, a.n + 1, C.c_int32, np.int32), _adopt(ci, nnz, C.c_int32, np.int32),
                _adopt(va, nnz, C.c_double, np.float64))
    return b, new_of_old, nc.value


def level_depth(a: HostCsr) -> int:
    d = C.c_int32()
    check(lib.rcg_level_depth(a.n, a.row_start.ctypes.data, a.col_idx.ctypes.data, C.byref(d)))
    return d.value
