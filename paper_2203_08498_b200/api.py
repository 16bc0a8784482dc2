"""Python host mirror of the reference solver API (proj/include/recycg), over the C-ABI.

Names and argument meaning follow the reference declarations (pcg.hpp, deflation.hpp,
subspace_correction.hpp, sampling.hpp, recycling.hpp, condest.hpp, ic_preconditioner.hpp);
exceptions follow its types: ``InvalidArgument`` (std::invalid_argument), ``BreakdownError``,
``ParseError``.  Vectors may be numpy float64 arrays (host; the call stages them through HBM)
or CUDA torch tensors (used in place).  Every operation runs on the GPU through
librcg_b200.so; there is no CPU code path for any of them.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib as L
from ._lib import BreakdownError, CudaError, InvalidArgument, ParseError, check, lib

__all__ = [
    "Context", "CsrMatrix", "IcFactor", "TallDense", "SamplerState", "Basis", "Identity", "Ic",
    "Sc", "SolveReport", "CondEstimate", "pcg_solve", "deflated_pcg_solve", "pcg_with_condest",
    "harvest_errors", "harvest_stored", "mgs_orthonormalize", "rayleigh_ritz", "build_aux_matrix",
    "diagonal_scale", "lanczos_extremes", "BreakdownError", "ParseError", "InvalidArgument",
    "CudaError",
]


def _ptr(a) -> int:
    """Raw address of a float64/int32 buffer (numpy host array or CUDA torch tensor)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise InvalidArgument("array must be contiguous")
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise InvalidArgument("tensor must be contiguous")
        return a.data_ptr()
    raise InvalidArgument(f"unsupported buffer type {type(a)!r}")


def _f64(a, n=None, name="vector"):
    if isinstance(a, np.ndarray):
        a = np.ascontiguousarray(a, dtype=np.float64)
    elif hasattr(a, "data_ptr"):
        import torch

        if a.dtype != torch.float64:
            raise InvalidArgument(f"{name} must be float64")
    else:
        a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if n is not None and (a.shape[0] if a.ndim else 0) != n:
        raise InvalidArgument(f"{name}: size does not match matrix")
    return a


def _out(a, shape, name="x"):
    """An output (or in/out) buffer the library writes: contiguous float64 of exactly `shape`
    (numpy host or CUDA torch).  The reference throws invalid_argument on a size mismatch
    (pcg.cpp:20-26); a short or float32 buffer here would be an out-of-bounds write."""
    if isinstance(a, np.ndarray):
        ok_t, ok_c = a.dtype == np.float64, a.flags["C_CONTIGUOUS"]
    elif hasattr(a, "data_ptr"):
        import torch

        ok_t, ok_c = a.dtype == torch.float64, a.is_contiguous()
    else:
        raise InvalidArgument(f"{name}: unsupported buffer type {type(a)!r}")
    if not ok_t:
        raise InvalidArgument(f"{name} must be float64")
    if not ok_c:
        raise InvalidArgument(f"{name} must be contiguous")
    if tuple(a.shape) != tuple(shape):
        raise InvalidArgument(f"{name}: size does not match matrix (shape {tuple(a.shape)}, expected {tuple(shape)})")
    return a


class Context:
    """One GPU and one CUDA stream (rcg_ctx)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib.rcg_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if self.h:
            lib.rcg_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self):
        check(lib.rcg_ctx_synchronize(self.h))

    @property
    def launches(self) -> int:
        return int(lib.rcg_ctx_launch_count(self.h))

    def set_profiling(self, on: bool, classes=None):
        """Kernel-class timers on / off; classes: the class ids to time (default all)."""
        mask = 0x3FF if classes is None else sum(1 << int(c) for c in classes)
        check(lib.rcg_ctx_set_profiling_mask(self.h, mask))
        check(lib.rcg_ctx_set_profiling(self.h, 1 if on else 0))

    def set_sweep_kernel(self, mode: int):
        """IC sweep kernel: 0 grid-wide sync-free, 2 default (per-level launches for wide levels,
        else grid-wide), 4 per-level launches always.  Results are bitwise identical either way."""
        check(lib.rcg_ctx_set_sweep_kernel(self.h, int(mode)))

    def record(self, slot: int):
        """CUDA event on the library stream (device-side timing)."""
        check(lib.rcg_ctx_event_record(self.h, slot))

    def elapsed_ms(self, a: int, b: int) -> float:
        ms = C.c_double()
        check(lib.rcg_ctx_event_elapsed(self.h, a, b, C.byref(ms)))
        return ms.value

    def kernel_stats(self, cls: int):
        ms = C.c_double()
        cnt = C.c_int64()
        check(lib.rcg_ctx_kernel_stats(self.h, cls, C.byref(ms), C.byref(cnt)))
        return ms.value, cnt.value

    def kernel_units(self, cls: int) -> int:
        """Right-hand sides carried by a class's launches (batched classes 5-9: RT each)."""
        u = C.c_int64()
        check(lib.rcg_ctx_kernel_units(self.h, cls, C.byref(u)))
        return u.value

    def reset_stats(self):
        lib.rcg_ctx_reset_stats(self.h)


class CsrMatrix:
    """Device CSR (CsrMatrix, csr_matrix.hpp:20-51); validated like the reference by default."""

    def __init__(self, ctx: Context, n, row_start, col_idx, values, validate: bool = True, _handle=None):
        self.ctx = ctx
        if _handle is not None:
            self.h = _handle
        else:
            rs = np.ascontiguousarray(row_start, dtype=np.int32) if isinstance(row_start, (np.ndarray, list)) else row_start
            ci = np.ascontiguousarray(col_idx, dtype=np.int32) if isinstance(col_idx, (np.ndarray, list)) else col_idx
            va = _f64(values, name="values")
            h = C.c_void_p()
            check(lib.rcg_matrix_create(ctx.h, int(n), _ptr(rs), _ptr(ci), _ptr(va), 1 if validate else 0, C.byref(h)))
            self.h = h
        self.n = int(lib.rcg_matrix_n(self.h))
        self.nnz = int(lib.rcg_matrix_nnz(self.h))

    def __del__(self):
        try:
            if self.h:
                lib.rcg_matrix_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def values(self) -> np.ndarray:
        out = np.empty(self.nnz)
        check(lib.rcg_matrix_values(self.ctx.h, self.h, _ptr(out)))
        return out

    def export(self):
        """(row_start, col_idx, values) back on the host (rcg_matrix_export)."""
        rs = np.empty(self.n + 1, np.int32)
        ci = np.empty(self.nnz, np.int32)
        va = np.empty(self.nnz)
        check(lib.rcg_matrix_export(self.ctx.h, self.h, _ptr(rs), _ptr(ci), _ptr(va)))
        return rs, ci, va

    def spmv(self, x, y=None):
        x = _f64(x, self.n, "x")
        if y is None:
            y = np.empty(self.n) if isinstance(x, np.ndarray) else x.new_empty(self.n)
        _out(y, (self.n,), "y")
        check(lib.rcg_spmv(self.ctx.h, self.h, _ptr(x), _ptr(y)))
        return y

    def spmv_dual(self, x1, x2):
        x1 = _f64(x1, self.n, "x1")
        x2 = _f64(x2, self.n, "x2")
        y1, y2 = np.empty(self.n), np.empty(self.n)
        check(lib.rcg_spmv_dual(self.ctx.h, self.h, _ptr(x1), _ptr(x2), _ptr(y1), _ptr(y2)))
        return y1, y2


def diagonal_scale(ctx: Context, a: CsrMatrix):
    """diagonal_scale (scaling.hpp:24-26): (A_scaled, d_inv_sqrt)."""
    h = C.c_void_p()
    dis = np.empty(a.n)
    check(lib.rcg_diagonal_scale(ctx.h, a.h, C.byref(h), _ptr(dis)))
    return CsrMatrix(ctx, 0, None, None, None, _handle=h), dis


class IcFactor:
    """Device IC(0) factor with level schedules (IcFactor, ic_preconditioner.hpp:18-37)."""

    def __init__(self, ctx: Context, handle):
        self.ctx = ctx
        self.h = handle
        nnz = C.c_int64()
        sh = C.c_double()
        fl = C.c_int32()
        bl = C.c_int32()
        check(lib.rcg_ic_info(self.h, C.byref(nnz), C.byref(sh), C.byref(fl), C.byref(bl)))
        self.nnz_l, self.shift_used, self.fwd_levels, self.bwd_levels = nnz.value, sh.value, fl.value, bl.value

    @classmethod
    def factorize(cls, ctx: Context, n, row_start, col_idx, values, shift: float = 0.0, num_blocks: int = 1):
        """ic0_factorize (ic_preconditioner.hpp:44) from host CSR arrays."""
        rs = np.ascontiguousarray(row_start, dtype=np.int32)
        ci = np.ascontiguousarray(col_idx, dtype=np.int32)
        va = np.ascontiguousarray(values, dtype=np.float64)
        h = C.c_void_p()
        check(lib.rcg_ic0_factorize(ctx.h, int(n), _ptr(rs), _ptr(ci), _ptr(va), float(shift), int(num_blocks),
                                    C.byref(h)))
        f = cls(ctx, h)
        f.n = int(n)
        f.num_blocks = int(num_blocks)
        return f

    @classmethod
    def factorize_device(cls, ctx: Context, a: "CsrMatrix", shift: float = 0.0, num_blocks: int = 1):
        """ic0_factorize with the numeric row merge on the GPU (rcg_ic0_factorize_device) from the
        device matrix's values; bitwise the host factorisation."""
        h = C.c_void_p()
        check(lib.rcg_ic0_factorize_device(ctx.h, a.h, float(shift), int(num_blocks), C.byref(h)))
        f = cls(ctx, h)
        f.n = int(a.n)
        f.num_blocks = int(num_blocks)
        return f

    @classmethod
    def from_arrays(cls, ctx: Context, n, block_bounds, l_row_start, l_col, l_val, d, u_row_start, u_col, u_val,
                    shift_used=0.0):
        arrs = [np.ascontiguousarray(block_bounds, dtype=np.int32), np.ascontiguousarray(l_row_start, dtype=np.int32),
                np.ascontiguousarray(l_col, dtype=np.int32), np.ascontiguousarray(l_val, dtype=np.float64),
                np.ascontiguousarray(d, dtype=np.float64), np.ascontiguousarray(u_row_start, dtype=np.int32),
                np.ascontiguousarray(u_col, dtype=np.int32), np.ascontiguousarray(u_val, dtype=np.float64)]
        h = C.c_void_p()
        check(lib.rcg_ic_create(ctx.h, int(n), len(arrs[0]) - 1, *[_ptr(a) for a in arrs], float(shift_used),
                                C.byref(h)))
        f = cls(ctx, h)
        f.n = int(n)
        f.num_blocks = len(arrs[0]) - 1
        return f

    def export(self):
        n, nnz = self.n, self.nnz_l
        out = dict(block_bounds=np.empty(self.num_blocks + 1, np.int32), l_row_start=np.empty(n + 1, np.int32),
                   l_col=np.empty(nnz, np.int32), l_val=np.empty(nnz), d=np.empty(n),
                   u_row_start=np.empty(n + 1, np.int32), u_col=np.empty(nnz, np.int32), u_val=np.empty(nnz))
        check(lib.rcg_ic_export(self.h, *[_ptr(v) for v in out.values()]))
        return out

    def apply(self, r, z=None):
        """ic_apply (ic_preconditioner.hpp:47)."""
        r = _f64(r, self.n, "r")
        if z is None:
            z = np.empty(self.n) if isinstance(r, np.ndarray) else r.new_empty(self.n)
        check(lib.rcg_ic_apply(self.ctx.h, self.h, _ptr(r), _ptr(z)))
        return z

    def __del__(self):
        try:
            if self.h:
                lib.rcg_ic_destroy(self.h)
                self.h = None
        except Exception:
            pass


class TallDense:
    """Device n x k column block (TallDense, dense.hpp:11-22)."""

    def __init__(self, ctx: Context, handle):
        self.ctx = ctx
        self.h = handle

    @classmethod
    def from_columns(cls, ctx: Context, n: int, cols):
        """cols: array of shape (k, n) -- column j is cols[j] (reference TallDense::cols order)."""
        cols = np.ascontiguousarray(cols, dtype=np.float64).reshape(-1, n) if n > 0 else np.zeros((0, 0))
        k = cols.shape[0] if n > 0 else 0
        h = C.c_void_p()
        check(lib.rcg_tall_create(ctx.h, int(n), int(k), _ptr(cols) if k else None, C.byref(h)))
        return cls(ctx, h)

    @property
    def k(self) -> int:
        return int(lib.rcg_tall_k(self.h))

    @property
    def n(self) -> int:
        return int(lib.rcg_tall_n(self.h))

    def columns(self) -> np.ndarray:
        out = np.empty((self.k, self.n))
        if self.k:
            check(lib.rcg_tall_download(self.ctx.h, self.h, _ptr(out)))
        return out

    def __del__(self):
        try:
            if self.h:
                lib.rcg_tall_destroy(self.h)
                self.h = None
        except Exception:
            pass


class SamplerState:
    """Device snapshot store (SamplerState, sampling.hpp:26-64)."""

    def __init__(self, ctx: Context, handle, m: int, n: int):
        self.ctx, self.h, self.m, self.n = ctx, handle, m, n

    @classmethod
    def method_a(cls, ctx: Context, m: int, iteration_cap: int, n: int):
        h = C.c_void_p()
        check(lib.rcg_sampler_create(ctx.h, L.RCG_SAMPLER_A, int(m), int(iteration_cap), 0.5, int(n), C.byref(h)))
        return cls(ctx, h, m, n)

    @classmethod
    def method_b(cls, ctx: Context, m: int, eps: float, n: int):
        h = C.c_void_p()
        check(lib.rcg_sampler_create(ctx.h, L.RCG_SAMPLER_B, int(m), 1, float(eps), int(n), C.byref(h)))
        return cls(ctx, h, m, n)

    def offer(self, iteration: int, relres: float, payload):
        payload = _f64(payload, self.n, "payload")
        check(lib.rcg_sampler_offer(self.ctx.h, self.h, int(iteration), float(relres), _ptr(payload)))

    def state(self):
        occ = np.zeros(self.m, np.int32)
        it = np.zeros(self.m, np.int32)
        c = lib.rcg_sampler_state(self.h, _ptr(occ), _ptr(it))
        if c < 0:
            check(-c)
        return occ.astype(bool), it

    def stored_count(self) -> int:
        return int(self.state()[0].sum())

    def occupied(self, s: int) -> bool:
        return bool(self.state()[0][s])

    def stored_iteration(self, s: int) -> int:
        return int(self.state()[1][s])

    def slot(self, s: int) -> np.ndarray:
        out = np.empty(self.n)
        check(lib.rcg_sampler_slot(self.ctx.h, self.h, int(s), _ptr(out)))
        return out

    def __del__(self):
        try:
            if self.h:
                lib.rcg_sampler_destroy(self.h)
                self.h = None
        except Exception:
            pass


class Basis:
    """W with AW and chol(W^T A W): DeflationOperator (who='deflation') or the state of
    ScPreconditioner (who='sc')."""

    def __init__(self, ctx: Context, a: CsrMatrix, w: TallDense, who: str = "deflation"):
        self.ctx = ctx
        self.n = a.n
        h = C.c_void_p()
        check(lib.rcg_basis_create(ctx.h, a.h, w.h, L.RCG_BASIS_SC if who == "sc" else L.RCG_BASIS_DEFLATION,
                                   C.byref(h)))
        self.h = h

    @property
    def k(self) -> int:
        return int(lib.rcg_basis_k(self.h))

    def empty(self) -> bool:
        return self.k == 0

    def _proj(self, fn, v):
        v = _f64(v, self.n)
        out = np.empty(self.n)
        check(fn(self.ctx.h, self.h, _ptr(v), _ptr(out)))
        return out

    def project_pt(self, y):
        return self._proj(lib.rcg_project_pt, y)

    def project_p(self, x):
        return self._proj(lib.rcg_project_p, x)

    def direct_component(self, b):
        return self._proj(lib.rcg_direct_component, b)

    def __del__(self):
        try:
            if self.h:
                lib.rcg_basis_destroy(self.h)
                self.h = None
        except Exception:
            pass


# ---- preconditioner descriptors (dispatch by kind, preconditioner.hpp:10-20)
@dataclass
class Identity:
    kind: int = L.RCG_PREC_IDENTITY


@dataclass
class Ic:
    factor: IcFactor
    kind: int = L.RCG_PREC_IC


@dataclass
class Sc:
    basis: Basis
    inner: Optional[IcFactor] = None
    kind: int = L.RCG_PREC_SC


def _prec(m) -> L.Prec:
    p = L.Prec()
    p.kind = m.kind
    if isinstance(m, Ic):
        p.ic = m.factor.h
    elif isinstance(m, Sc):
        p.ic = m.inner.h if m.inner is not None else None
        p.sc = m.basis.h
    elif not isinstance(m, Identity):
        raise InvalidArgument("unknown preconditioner type (no CPU fallback exists)")
    return p


@dataclass
class SolveReport:
    iterations: int = 0
    converged: bool = False
    wall_time: float = 0.0
    history: np.ndarray = field(default_factory=lambda: np.zeros(0))
    alphas: np.ndarray = field(default_factory=lambda: np.zeros(0))
    betas: np.ndarray = field(default_factory=lambda: np.zeros(0))


@dataclass
class CondEstimate:
    lambda_max: float = 0.0
    lambda_min: float = float("nan")
    kappa: float = float("nan")
    power_iterations: int = 0
    power_unsettled: bool = True
    lambda_min_available: bool = False
    ritz_values: np.ndarray = field(default_factory=lambda: np.zeros(0))
    lanczos_lambda_min: float = float("nan")
    lanczos_lambda_max: float = float("nan")
    lanczos_kappa: float = float("nan")


def _report(max_iter):
    rep = L.SolveReport()
    bufs = (np.zeros(max_iter), np.zeros(max_iter), np.zeros(max_iter))
    rep.cap = max_iter
    rep.history = bufs[0].ctypes.data_as(L.dp)
    rep.alphas = bufs[1].ctypes.data_as(L.dp)
    rep.betas = bufs[2].ctypes.data_as(L.dp)
    return rep, bufs


def _finish(rep, bufs) -> SolveReport:
    k = rep.iterations
    return SolveReport(k, bool(rep.converged), rep.wall_time, bufs[0][:k].copy(), bufs[1][:k].copy(),
                       bufs[2][:k].copy())


def _cfg(eps, max_iter, record_history=True):
    c = L.SolverConfig()
    c.eps, c.max_iter, c.record_history = float(eps), int(max_iter), 1 if record_history else 0
    return c


def pcg_solve(ctx: Context, a: CsrMatrix, b, m, x, eps: float = 1e-8, max_iter: int = 1000,
              observer: Optional[SamplerState] = None, payload: str = "x") -> SolveReport:
    """pcg_solve (pcg.hpp:39-41); x is updated in place.  observer: a SamplerState fed the
    iterate (payload 'x', error_sampling_observer) or the residual ('r')."""
    b = _f64(b, a.n, "b")
    _out(x, (a.n,), "x")
    cfg = _cfg(eps, max_iter)
    rep, bufs = _report(max(1, int(max_iter)))
    p = _prec(m)
    check(lib.rcg_pcg_solve(ctx.h, a.h, _ptr(b), C.byref(p), _ptr(x), C.byref(cfg),
                            observer.h if observer is not None else None,
                            L.RCG_PAYLOAD_R if payload == "r" else L.RCG_PAYLOAD_X, C.byref(rep)))
    return _finish(rep, bufs)


def deflated_pcg_solve(ctx: Context, a: CsrMatrix, b, m, defl: Optional[Basis], x, eps: float = 1e-8,
                       max_iter: int = 1000) -> SolveReport:
    """deflated_pcg_solve (pcg.hpp:50-52); defl None is the empty W."""
    b = _f64(b, a.n, "b")
    _out(x, (a.n,), "x")
    cfg = _cfg(eps, max_iter)
    rep, bufs = _report(max(1, int(max_iter)))
    p = _prec(m)
    check(lib.rcg_deflated_pcg_solve(ctx.h, a.h, _ptr(b), C.byref(p), defl.h if defl is not None else None, _ptr(x),
                                     C.byref(cfg), C.byref(rep)))
    return _finish(rep, bufs)


def _batch(fn, ctx, a, B, m, X, eps, max_iter, defl=None):
    R = len(B)
    if not (1 <= R <= 24):
        raise InvalidArgument("batch solve: 1..24 right-hand sides")
    if isinstance(B, np.ndarray) or isinstance(B, list) and isinstance(B[0], np.ndarray):
        Bm = np.ascontiguousarray(np.stack(list(B)) if isinstance(B, list) else B, dtype=np.float64)
    else:
        import torch

        Bm = torch.stack(list(B)).contiguous() if isinstance(B, list) else B.contiguous()
    if Bm.shape[-1] != a.n:
        raise InvalidArgument("batch solve: right-hand side length does not match matrix")
    _out(X, (R, a.n), "X")
    cfg = _cfg(eps, max_iter)
    reps = (L.SolveReport * R)()
    bufs = []
    for r in reps:
        rb = _report(max(1, int(max_iter)))
        r.cap, r.history, r.alphas, r.betas = rb[0].cap, rb[0].history, None, None
        bufs.append(rb[1])
    p = _prec(m)
    args = [ctx.h, a.h, _ptr(Bm), C.byref(p)]
    if defl is not False:
        args.append(defl.h if defl is not None else None)
    args += [_ptr(X), C.byref(cfg), R, reps]
    check(fn(*args))
    return [_finish(r, b) for r, b in zip(reps, bufs)]


def pcg_solve_batch(ctx: Context, a: CsrMatrix, B, m, X, eps: float = 1e-8, max_iter: int = 1000):
    """R <= 16 independent pcg_solve calls of one matrix in one kernel sequence.  B, X: (R, n)
    contiguous (numpy host or CUDA torch); X is updated in place.  Returns R SolveReports."""
    return _batch(lib.rcg_pcg_solve_batch, ctx, a, B, m, X, eps, max_iter, defl=False)


def deflated_pcg_solve_batch(ctx: Context, a: CsrMatrix, B, m, defl: Optional[Basis], X, eps: float = 1e-8,
                             max_iter: int = 1000):
    """R <= 24 independent deflated_pcg_solve calls in one kernel sequence (see pcg_solve_batch)."""
    return _batch(lib.rcg_deflated_pcg_solve_batch, ctx, a, B, m, X, eps, max_iter, defl=defl)


def pcg_with_condest(ctx: Context, a: CsrMatrix, b, m, x, eps: float = 1e-8, max_iter: int = 1000,
                     m_samples: int = 20, v0_seed: int = 42):
    """pcg_with_condest (condest.hpp:46-48) plus the Lanczos estimate; returns (report, estimate)."""
    b = _f64(b, a.n, "b")
    _out(x, (a.n,), "x")
    cfg = _cfg(eps, max_iter)
    rep, bufs = _report(max(1, int(max_iter)))
    est = L.CondEstimate()
    ritz = np.zeros(max(1, m_samples))
    est.ritz_values = ritz.ctypes.data_as(L.dp)
    p = _prec(m)
    check(lib.rcg_pcg_with_condest(ctx.h, a.h, _ptr(b), C.byref(p), _ptr(x), C.byref(cfg), int(m_samples),
                                   C.c_uint64(v0_seed), C.byref(rep), C.byref(est)))
    e = CondEstimate(est.lambda_max, est.lambda_min, est.kappa, est.power_iterations, bool(est.power_unsettled),
                     bool(est.lambda_min_available), ritz[: est.nritz].copy(), est.lanczos_lambda_min,
                     est.lanczos_lambda_max, est.lanczos_kappa)
    return _finish(rep, bufs), e


def harvest_errors(ctx: Context, x_final, s: SamplerState) -> TallDense:
    x_final = _f64(x_final, s.n, "x_final")
    h = C.c_void_p()
    check(lib.rcg_harvest_errors(ctx.h, _ptr(x_final), s.h, C.byref(h)))
    return TallDense(ctx, h)


def harvest_stored(ctx: Context, s: SamplerState) -> TallDense:
    h = C.c_void_p()
    check(lib.rcg_harvest_stored(ctx.h, s.h, C.byref(h)))
    return TallDense(ctx, h)


def mgs_orthonormalize(ctx: Context, v: TallDense, drop_tol: float = 1e-12) -> TallDense:
    h = C.c_void_p()
    check(lib.rcg_mgs_orthonormalize(ctx.h, v.h, float(drop_tol), C.byref(h)))
    return TallDense(ctx, h)


def rayleigh_ritz(ctx: Context, a: CsrMatrix, e: TallDense, vectors: bool = True):
    vals = np.zeros(max(1, e.k))
    h = C.c_void_p()
    check(lib.rcg_rayleigh_ritz(ctx.h, a.h, e.h, _ptr(vals), C.byref(h) if vectors else None))
    return vals[: e.k].copy(), (TallDense(ctx, h) if vectors else None)


def build_aux_matrix(ctx: Context, a: CsrMatrix, errors: TallDense, theta: float, keep_count: int = 0):
    """build_aux_matrix (recycling.hpp:47): returns (m_bar, ritz_values, theta_used, W)."""
    vals = np.zeros(max(1, errors.k))
    mb = C.c_int()
    th = C.c_double()
    h = C.c_void_p()
    check(lib.rcg_build_aux_matrix(ctx.h, a.h, errors.h, float(theta), int(keep_count), C.byref(mb), _ptr(vals),
                                   C.byref(th), C.byref(h)))
    return mb.value, vals[: mb.value].copy(), th.value, TallDense(ctx, h)


def lanczos_extremes(alphas, betas):
    a = np.ascontiguousarray(alphas, dtype=np.float64)
    b = np.ascontiguousarray(betas, dtype=np.float64)
    lo, hi = C.c_double(), C.c_double()
    check(lib.rcg_lanczos_extremes(len(a), _ptr(a), _ptr(b), C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


# --------------------------------------------------------------------------- multi-GPU row slabs
class SlabPlan:
    """Host plan of slab `part` of `nparts` (rcg_slab_plan_create): the reference's block bounds
    floor(b n / G), the local CSR with halo columns numbered after the owned rows, and the halo
    send / receive lists.  Arrays are numpy copies; the C plan is kept for rcg_dslab_create."""

    def __init__(self, n, row_start, col_idx, values, nparts: int, part: int):
        rs = np.ascontiguousarray(row_start, dtype=np.int32)
        ci = np.ascontiguousarray(col_idx, dtype=np.int32)
        va = np.ascontiguousarray(values, dtype=np.float64)
        self._c = L.SlabPlanC()
        check(lib.rcg_slab_plan_create(int(n), _ptr(rs), _ptr(ci), _ptr(va), int(nparts), int(part), C.byref(self._c)))
        c = self._c
        self.nparts, self.part = c.nparts, c.part
        self.row_begin, self.row_end, self.nloc, self.nhalo, self.nnz = c.row_begin, c.row_end, c.nloc, c.nhalo, c.nnz

        def arr(ptr, k, dt):
            return np.ctypeslib.as_array(ptr, shape=(k,)).astype(dt, copy=True) if k > 0 else np.zeros(0, dt)

        self.row_start = arr(c.row_start, self.nloc + 1, np.int32)
        self.col_idx = arr(c.col_idx, self.nnz, np.int32)
        self.values = arr(c.values, self.nnz, np.float64)
        self.halo_global = arr(c.halo_global, self.nhalo, np.int32)
        self.recv_count = arr(c.recv_count, self.nparts, np.int32)
        self.send_count = arr(c.send_count, self.nparts, np.int32)
        self.send_idx = arr(c.send_idx, int(self.send_count.sum()), np.int32)

    def diagonal_block(self):
        """CSR of the slab's diagonal block (columns < nloc): the block-Jacobi IC(0) input."""
        keep = self.col_idx < self.nloc
        rows = np.repeat(np.arange(self.nloc), np.diff(self.row_start))
        counts = np.bincount(rows[keep], minlength=self.nloc)
        rs = np.zeros(self.nloc + 1, np.int32)
        rs[1:] = np.cumsum(counts)
        return rs, self.col_idx[keep].copy(), self.values[keep].copy()

    def __del__(self):
        try:
            lib.rcg_slab_plan_free(C.byref(self._c))
        except Exception:
            pass


class DSlab:
    """One GPU's row slab (rcg_dslab_create): local matrix with halo columns, exchange lists,
    extended x / p buffers; `ic` is the slab's diagonal-block IcFactor (None = identity)."""

    def __init__(self, ctx: Context, plan: SlabPlan, ic: Optional[IcFactor] = None):
        h = C.c_void_p()
        check(lib.rcg_dslab_create(ctx.h, C.byref(plan._c), ic.h if ic is not None else None, C.byref(h)))
        self.h, self.ctx, self.plan, self.ic = h, ctx, plan, ic

    def __del__(self):
        if getattr(self, "h", None):
            lib.rcg_dslab_destroy(self.h)
            self.h = None


class Comm:
    """Slab transport: `Comm.nccl(id, nranks, rank)` (one slab per process, NCCL over NVLink) or
    `Comm.loopback(nparts)` (all slabs in this process on one GPU; tests)."""

    def __init__(self, h, nparts):
        self.h, self.nparts = h, nparts

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_char * 128)()
        check(lib.rcg_comm_nccl_unique_id(buf))
        return bytes(buf)

    @classmethod
    def nccl(cls, unique_id: bytes, nranks: int, rank: int) -> "Comm":
        buf = (C.c_char * 128).from_buffer_copy(unique_id)
        h = C.c_void_p()
        check(lib.rcg_comm_create_nccl(buf, int(nranks), int(rank), C.byref(h)))
        return cls(h, nranks)

    @classmethod
    def loopback(cls, nparts: int) -> "Comm":
        h = C.c_void_p()
        check(lib.rcg_comm_create_loopback(int(nparts), C.byref(h)))
        return cls(h, nparts)

    @classmethod
    def host(cls, group=None) -> "Comm":
        """Host-staged transport over torch.distributed (any backend with CPU tensors, e.g. gloo):
        each collective synchronises the slab's stream and moves its values through host memory,
        so ranks never wait on each other inside a kernel and may share one GPU
        (rcg_comm_create_host).  The slow but exact stand-in for NCCL in multi-process tests."""
        import torch
        import torch.distributed as dist

        nranks, rank = dist.get_world_size(group), dist.get_rank(group)
        calls = {"allreduce": 0, "allreduce_values": 0, "exchange": 0}  # collectives issued (tests / reports)

        def allreduce(_user, buf, count):
            try:
                calls["allreduce"] += 1
                calls["allreduce_values"] += int(count)
                t = torch.from_numpy(np.ctypeslib.as_array(buf, shape=(count,)))
                dist.all_reduce(t, group=group)
                return 0
            except Exception:  # noqa: BLE001 -- reported as a status by the library
                return 1

        def exchange(_user, send, so, sc, recv, ro, rc, np_):
            try:
                calls["exchange"] += 1
                reqs = []
                for q in range(np_):
                    if sc[q]:
                        t = torch.from_numpy(np.ctypeslib.as_array(send, shape=(so[q] + sc[q],))[so[q]:])
                        reqs.append(dist.isend(t, q, group=group))
                    if rc[q]:
                        t = torch.from_numpy(np.ctypeslib.as_array(recv, shape=(ro[q] + rc[q],))[ro[q]:])
                        reqs.append(dist.irecv(t, q, group=group))
                for r in reqs:
                    r.wait()
                return 0
            except Exception:  # noqa: BLE001
                return 1

        cb_ar = L.HostAllreduceFn(allreduce)
        cb_ex = L.HostExchangeFn(exchange)
        h = C.c_void_p()
        check(lib.rcg_comm_create_host(int(nranks), int(rank), cb_ar, cb_ex, None, C.byref(h)))
        c = cls(h, nranks)
        c._callbacks = (cb_ar, cb_ex)  # the library holds raw pointers to them
        c.calls = calls
        return c

    def __del__(self):
        if getattr(self, "h", None):
            lib.rcg_comm_destroy(self.h)
            self.h = None


def dist_pcg_solve(comm: Comm, slabs, bs, xs, eps: float = 1e-8, max_iter: int = 1000) -> SolveReport:
    """Distributed PCG over row slabs (rcg_dist_pcg_solve): block-Jacobi IC(0) when the slabs
    carry factors, else identity.  bs[s], xs[s]: slab s's local rows; xs updated in place."""
    slabs = list(slabs)
    ns = len(slabs)
    bs = [_f64(b, s.plan.nloc, "b") for b, s in zip(bs, slabs)]
    hs = (C.c_void_p * ns)(*[s.h.value for s in slabs])
    bp = (C.c_void_p * ns)(*[_ptr(b) for b in bs])
    xp = (C.c_void_p * ns)(*[_ptr(_out(x, (s_.plan.nloc,), "x")) for x, s_ in zip(xs, slabs)])
    cfg = _cfg(eps, max_iter)
    rep, bufs = _report(max(1, int(max_iter)))
    check(lib.rcg_dist_pcg_solve(comm.h, ns, hs, bp, xp, C.byref(cfg), C.byref(rep)))
    return _finish(rep, bufs)


class DBasis:
    """Row-partitioned W / AW with the replicated chol(W^T A W) (rcg_dbasis_create): the
    distributed DeflationOperator / ScPreconditioner state.  ws[s]: slab s's rows of W as an
    (m, nloc) array (one basis vector per row)."""

    def __init__(self, comm: Comm, slabs, ws, kind: str = "deflation"):
        slabs = list(slabs)
        ns = len(slabs)
        self.m = int(ws[0].shape[0])
        cols = [np.ascontiguousarray(w, dtype=np.float64) for w in ws]  # (m, nloc) row-major = column-major nloc x m
        self._cols = cols
        hs = (C.c_void_p * ns)(*[s_.h.value for s_ in slabs])
        wp = (C.c_void_p * ns)(*[_ptr(c) for c in cols])
        h = C.c_void_p()
        check(lib.rcg_dbasis_create(comm.h, ns, hs, wp, self.m, L.RCG_BASIS_SC if kind == "sc" else L.RCG_BASIS_DEFLATION,
                                    C.byref(h)))
        self.h, self.kind, self.slabs = h, kind, slabs

    def __del__(self):
        if getattr(self, "h", None):
            lib.rcg_dbasis_destroy(self.h)
            self.h = None


def dist_solve(comm: Comm, slabs, bs, xs, basis: Optional[DBasis] = None, eps: float = 1e-8,
               max_iter: int = 1000) -> SolveReport:
    """rcg_dist_solve: distributed block-Jacobi PCG, deflated PCG (basis kind 'deflation') or
    SC-PCG (kind 'sc') over row slabs."""
    slabs = list(slabs)
    ns = len(slabs)
    bs = [_f64(b, s_.plan.nloc, "b") for b, s_ in zip(bs, slabs)]
    hs = (C.c_void_p * ns)(*[s_.h.value for s_ in slabs])
    bp = (C.c_void_p * ns)(*[_ptr(b) for b in bs])
    xp = (C.c_void_p * ns)(*[_ptr(_out(x, (s_.plan.nloc,), "x")) for x, s_ in zip(xs, slabs)])
    cfg = _cfg(eps, max_iter)
    rep, bufs = _report(max(1, int(max_iter)))
    check(lib.rcg_dist_solve(comm.h, ns, hs, basis.h if basis is not None else None, bp, xp, C.byref(cfg),
                             C.byref(rep)))
    return _finish(rep, bufs)


def dist_solve_batch(comm: Comm, slab, B, X, basis: Optional[DBasis] = None, eps: float = 1e-8,
                     max_iter: int = 1000):
    """rcg_dist_solve_batch: up to 24 accelerated solves over this process's slab in ONE kernel
    sequence (the batched solver with allreduced reductions and RT-interleaved halo exchanges).
    B, X: (R, nloc) this slab's rows; returns one SolveReport per right-hand side."""
    nloc = slab.plan.nloc
    if hasattr(B, "data_ptr") or (isinstance(B, list) and hasattr(B[0], "data_ptr")):  # CUDA tensors
        import torch

        Bm = (torch.stack(list(B)) if isinstance(B, list) else B).contiguous()
    else:
        Bm = np.ascontiguousarray(np.stack(list(B)) if isinstance(B, list) else B, dtype=np.float64)
    R = Bm.shape[0]
    if not (1 <= R <= 24) or Bm.shape[-1] != nloc:
        raise InvalidArgument("dist_solve_batch: B must be (R <= 24, nloc)")
    _out(X, (R, nloc), "X")
    cfg = _cfg(eps, max_iter)
    reps = (L.SolveReport * R)()
    bufs = []
    for r in reps:
        rb = _report(max(1, int(max_iter)))
        r.cap, r.history, r.alphas, r.betas = rb[0].cap, rb[0].history, None, None
        bufs.append(rb[1])
    check(lib.rcg_dist_solve_batch(comm.h, slab.h, basis.h if basis is not None else None, _ptr(Bm), _ptr(X),
                                   C.byref(cfg), R, reps))
    return [_finish(r, b) for r, b in zip(reps, bufs)]


def dist_pcg_solve_sampled(comm: Comm, slabs, samplers, bs, xs, eps: float = 1e-8,
                           max_iter: int = 1000) -> SolveReport:
    """Solve 1 of the sequence over row slabs (rcg_dist_pcg_solve_sampled): block-Jacobi PCG with
    the error-sampling observer; samplers[s] = slab s's SamplerState (n = its local rows)."""
    slabs = list(slabs)
    ns = len(slabs)
    bs = [_f64(b, s_.plan.nloc, "b") for b, s_ in zip(bs, slabs)]
    hs = (C.c_void_p * ns)(*[s_.h.value for s_ in slabs])
    sp = (C.c_void_p * ns)(*[o.h.value for o in samplers])
    bp = (C.c_void_p * ns)(*[_ptr(b) for b in bs])
    xp = (C.c_void_p * ns)(*[_ptr(_out(x, (s_.plan.nloc,), "x")) for x, s_ in zip(xs, slabs)])
    cfg = _cfg(eps, max_iter)
    rep, bufs = _report(max(1, int(max_iter)))
    check(lib.rcg_dist_pcg_solve_sampled(comm.h, ns, hs, sp, bp, xp, C.byref(cfg), C.byref(rep)))
    return _finish(rep, bufs)


def dist_recycle(comm: Comm, slabs, samplers, xs_final, theta: float = float("inf"), keep_count: int = 0,
                 kind: str = "deflation"):
    """The recycling step over row slabs (rcg_dist_recycle): harvest_errors + build_aux_matrix +
    the distributed deflation / SC state.  Returns (m_bar, ritz_values, theta_used, m_tilde,
    DBasis or None)."""
    slabs = list(slabs)
    ns = len(slabs)
    hs = (C.c_void_p * ns)(*[s_.h.value for s_ in slabs])
    sp = (C.c_void_p * ns)(*[o.h.value for o in samplers])
    xs = [_f64(x, s_.plan.nloc, "x_final") for x, s_ in zip(xs_final, slabs)]
    xp = (C.c_void_p * ns)(*[_ptr(x) for x in xs])
    m_bar, m_tilde = C.c_int(), C.c_int()
    th = C.c_double()
    vals = np.zeros(max(1, max(o.m for o in samplers)))
    h = C.c_void_p()
    check(lib.rcg_dist_recycle(comm.h, ns, hs, sp, xp, float(theta), int(keep_count),
                               L.RCG_BASIS_SC if kind == "sc" else L.RCG_BASIS_DEFLATION, C.byref(m_bar), _ptr(vals),
                               C.byref(th), C.byref(m_tilde), C.byref(h)))
    basis = None
    if h.value:
        basis = DBasis.__new__(DBasis)
        basis.h, basis.kind, basis.slabs, basis.m, basis._cols = h, kind, slabs, m_tilde.value, None
    return m_bar.value, vals[: m_bar.value].copy(), th.value, m_tilde.value, basis


# --------------------------------------------------------------------------- the sequence driver
_METHODS = {"cg": L.RCG_METHOD_CG, "iccg": L.RCG_METHOD_ICCG, "es-sc-iccg": L.RCG_METHOD_ES_SC_ICCG,
            "es-d-iccg": L.RCG_METHOD_ES_D_ICCG}


class Sequence:
    """run_sequence (driver.cpp:108-222) on the device: prepared once per matrix (scaling, IC(0)),
    then `run(B, X, ...)` solves the k right-hand sides B (k, n) into X (k, n)."""

    def __init__(self, ctx: Context, a_orig: CsrMatrix, method: str = "es-sc-iccg", blocks: int = 1):
        if method not in _METHODS:
            raise L.ParseError(f"config: unknown method '{method}'")
        h = C.c_void_p()
        check(lib.rcg_seq_prepare(ctx.h, a_orig.h, _METHODS[method], int(blocks), C.byref(h)))
        self.h, self.ctx, self.n, self.method = h, ctx, a_orig.n, method

    def run(self, B, X, eps: float = 1e-8, max_iter: int = 1000, sampling: str = "A", m: int = 16,
            theta: float = 1e-3, keep_count: int = 0, batch: bool = True, condest: bool = False,
            lean: bool = False) -> dict:
        """lean: the memory-lean recycling step always (default: only when HBM is short)."""
        k = len(B)
        _out(B, (k, self.n), "B")  # read-only here, but passed raw: same contract
        _out(X, (k, self.n), "X")
        cfg = L.SeqConfig(float(eps), int(max_iter), ord(sampling), int(m), float(theta), int(keep_count),
                          1 if batch else 0, 1 if lean else 0)
        its = np.zeros(k, np.int32)
        conv = np.zeros(k, np.int32)
        wall = np.zeros(k)
        trr = np.zeros(k)
        ritz = np.zeros(max(1, 2 * m))
        lmin, lmax, kap = np.zeros(k), np.zeros(k), np.zeros(k)
        rep = L.SeqReport(its.ctypes.data_as(L.ip), conv.ctypes.data_as(L.ip), wall.ctypes.data_as(L.dp),
                          trr.ctypes.data_as(L.dp), ritz.ctypes.data_as(L.dp), len(ritz))
        if condest:
            rep.lambda_min, rep.lambda_max, rep.kappa = (v.ctypes.data_as(L.dp) for v in (lmin, lmax, kap))
        check(lib.rcg_seq_run(self.h, k, _ptr(B), _ptr(X), C.byref(cfg), C.byref(rep)))
        return dict(iterations=its.tolist(), converged=[bool(c) for c in conv], wall_time=wall.tolist(),
                    true_relres=trr.tolist(), m_bar=rep.m_bar, m_tilde=rep.m_tilde,
                    ritz_values=ritz[:min(rep.m_bar, len(ritz))].copy(), theta_used=rep.theta_used,
                    w_build_time=rep.w_build_time, avg_iterations=rep.avg_iterations,
                    avg_wall_time=rep.avg_wall_time, setup_time=rep.setup_time,
                    acceleration_inactive=bool(rep.acceleration_inactive),
                    **(dict(lambda_min=lmin.tolist(), lambda_max=lmax.tolist(), kappa=kap.tolist()) if condest else {}))

    def __del__(self):
        if getattr(self, "h", None):
            lib.rcg_seq_destroy(self.h)
            self.h = None
