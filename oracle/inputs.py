"""BASELINE.json inputs for the oracle side -- TEST INFRASTRUCTURE / CPU BASELINE ONLY.

The same seeded generators as the product (one source, paper_2203_08498_b200/csrc/generators.cpp),
compiled by g++ alone into oracle/libgen_host.so (oracle/Makefile `gen`), so the oracle harness,
tools/make_goldens.py and bench.py's reference arm build the configs' matrices and right-hand
side streams without mapping librcg_b200.so.  Configurations come from the plain-data module
paper_2203_08498_b200/configs.py (plain data: the package imports its library lazily, so nothing native is mapped).
"""
from __future__ import annotations

import ctypes as C
import os
import weakref
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GEN_SO = os.path.join(HERE, "libgen_host.so")

# plain data; the product package initialises lazily, so this maps no library
from paper_2203_08498_b200.configs import CONFIGS, SMALL  # noqa: E402,F401


class _GenParams(C.Structure):  # rcg_gen_params (include/rcg_b200.h)
    _fields_ = [("kind", C.c_int), ("grid", C.c_int32), ("inclusions", C.c_int), ("inclusion_size", C.c_int),
                ("contrast", C.c_double), ("sigma", C.c_double), ("knn_k", C.c_int), ("seed", C.c_uint64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(GEN_SO):
            raise ImportError(f"{GEN_SO} missing: run `make -C {HERE} gen`")
        L = C.CDLL(GEN_SO)
        i32p, dp = C.POINTER(C.c_int32), C.POINTER(C.c_double)
        L.rcg_generate.argtypes = [C.POINTER(_GenParams), i32p, C.POINTER(C.c_int64), C.POINTER(i32p),
                                   C.POINTER(i32p), C.POINTER(dp)]
        L.rcg_generate.restype = C.c_int
        L.rcg_uniform_pm1.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.c_void_p]
        L.rcg_normal.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.c_void_p]
        L.rcg_host_free.argtypes = [C.c_void_p]
        L.gen_last_error.restype = C.c_char_p
        _lib = L
    return _lib


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
    L = lib()
    if count == 0:
        L.rcg_host_free(C.cast(ptr, C.c_void_p))
        return np.zeros(0, dtype)
    arr = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ctype)), shape=(count,))
    weakref.finalize(arr, L.rcg_host_free, C.cast(ptr, C.c_void_p).value)
    return arr


def generate(cfg) -> HostCsr:
    L = lib()
    p = _GenParams(cfg.kind, cfg.grid, cfg.inclusions, cfg.inclusion_size, cfg.contrast, cfg.sigma, cfg.knn_k,
                   cfg.seed)
    n, nnz = C.c_int32(), C.c_int64()
    rs, ci, va = C.POINTER(C.c_int32)(), C.POINTER(C.c_int32)(), C.POINTER(C.c_double)()
    st = L.rcg_generate(C.byref(p), C.byref(n), C.byref(nnz), C.byref(rs), C.byref(ci), C.byref(va))
    if st:
        raise RuntimeError(L.gen_last_error().decode())
    return HostCsr(n.value, _adopt(rs, n.value + 1, C.c_int32, np.int32), _adopt(ci, nnz.value, C.c_int32, np.int32),
                   _adopt(va, nnz.value, C.c_double, np.float64))


def uniform_pm1(seed: int, skip: int, n: int) -> np.ndarray:
    out = np.empty(n)
    lib().rcg_uniform_pm1(seed, skip, n, out.ctypes.data)
    return out


def normal(seed: int, skip: int, n: int) -> np.ndarray:
    out = np.empty(n)
    lib().rcg_normal(seed, skip, n, out.ctypes.data)
    return out


def solution_stream(cfg, n: int, k: int) -> np.ndarray:
    """x_k (0-based) of the sequence -- identical to paper_2203_08498_b200.problems.solution_stream."""
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


def solution_streams(cfg, n: int, count: int):
    """x_0 .. x_{count-1} in order, O(count) draws for the drifting stream (same values)."""
    x = None
    for k in range(count):
        if cfg.rhs == "drift":
            x = normal(cfg.rhs_seed, 0, n) if k == 0 else x + 0.1 * normal(cfg.rhs_seed, k * n, n)
            yield x
        else:
            yield solution_stream(cfg, n, k)
