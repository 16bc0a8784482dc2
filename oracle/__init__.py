"""ctypes binding of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, bench.py (cpu_baseline / --impl reference) and __graft_entry__.smoke() may import
this package, and only as the checker or the timed CPU baseline.  The product package
(paper_2203_08498_b200) never imports it.

Two implementations are exposed with the same Python surface:
  * ``Oracle``  -- liboracle.so, the plain-C restatement (oracle/oracle.c);
  * ``RefLib``  -- oracle/_ref/librecycg_ref.so, the unmodified reference library compiled from
                   /root/reference sources by oracle/Makefile, through oracle/ref_shim.cpp.
tests/test_oracle.py pins the first against the second bitwise and against the reference's
known-answer tests.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "librecycg_ref.so")

vp, dp, ip = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int)


class OCsr(C.Structure):
    _fields_ = [("n", C.c_int32), ("rs", vp), ("ci", vp), ("va", vp)]


class OIc(C.Structure):
    _fields_ = [("n", C.c_int32), ("nblocks", C.c_int32), ("bounds", vp), ("lrs", vp), ("lcol", vp), ("lval", vp),
                ("d", vp), ("urs", vp), ("ucol", vp), ("uval", vp), ("nnz_l", C.c_int64), ("shift", C.c_double)]


class OBasis(C.Structure):
    _fields_ = [("n", C.c_int32), ("k", C.c_int), ("w", vp), ("aw", vp), ("l", vp)]


class OPrec(C.Structure):
    _fields_ = [("kind", C.c_int), ("ic", vp), ("sc", vp)]


class OSampler(C.Structure):
    _fields_ = [("method", C.c_int), ("m", C.c_int), ("n", C.c_int32), ("slots", vp), ("occupied", vp),
                ("stored_iter", vp), ("l_max", C.c_int), ("h", C.c_int64), ("alpha", C.c_double),
                ("next_slot", C.c_int)]


class OReport(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("wall_time", C.c_double), ("cap", C.c_int),
                ("history", dp), ("alphas", dp), ("betas", dp)]


class OCond(C.Structure):
    _fields_ = [("lambda_max", C.c_double), ("lambda_min", C.c_double), ("kappa", C.c_double),
                ("power_iterations", C.c_int), ("power_unsettled", C.c_int), ("lambda_min_available", C.c_int),
                ("nritz", C.c_int), ("ritz_values", dp)]


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class InvalidArgument(OracleError, ValueError):
    pass


class Breakdown(OracleError):
    pass


class Parse(OracleError):
    pass


_KIND = {1: InvalidArgument, 2: Breakdown, 3: Parse}


def _arr(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


@dataclass
class Report:
    iterations: int
    converged: bool
    wall_time: float
    history: np.ndarray
    alphas: np.ndarray = field(default_factory=lambda: np.zeros(0))
    betas: np.ndarray = field(default_factory=lambda: np.zeros(0))


@dataclass
class Cond:
    lambda_max: float
    lambda_min: float
    kappa: float
    power_iterations: int
    power_unsettled: bool
    lambda_min_available: bool
    ritz_values: np.ndarray


class Matrix:
    """Host CSR kept alive for the oracle calls."""

    def __init__(self, n, rs, ci, va):
        self.n = int(n)
        self.rs = _arr(rs, np.int32)
        self.ci = _arr(ci, np.int32)
        self.va = _arr(va, np.float64)
        self.c = OCsr(self.n, _p(self.rs), _p(self.ci), _p(self.va))

    @classmethod
    def of(cls, a):
        return cls(a.n, a.row_start, a.col_idx, a.values)


class Oracle:
    """The plain-C restatement (liboracle.so)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise ImportError(f"{path} missing: run `make -C {HERE} oracle`")
        self.lib = L = C.CDLL(path)
        L.orc_last_error.restype = C.c_char_p
        for name in ("orc_ic0_factorize", "orc_basis_build", "orc_sampler_create_a", "orc_sampler_create_b",
                     "orc_pcg_solve", "orc_deflated_pcg_solve", "orc_pcg_with_condest", "orc_build_aux",
                     "orc_rayleigh_ritz", "orc_sym_eig", "orc_chol_factor", "orc_mgs", "orc_harvest_errors",
                     "orc_harvest_stored", "orc_diagonal_scale", "orc_lanczos_extremes"):
            getattr(L, name).restype = C.c_int
        L.orc_dot.restype = C.c_double
        L.orc_dot.argtypes = [C.c_int64, vp, vp]
        L.orc_uniform_pm1_fill.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, vp]
        L.orc_pcg_with_condest.argtypes = [C.POINTER(OCsr), vp, C.POINTER(OPrec), vp, C.c_double, C.c_int, C.c_int,
                                           C.c_uint64, C.POINTER(OReport), C.POINTER(OCond)]
        L.orc_pcg_solve.argtypes = [C.POINTER(OCsr), vp, C.POINTER(OPrec), vp, C.c_double, C.c_int, vp, C.c_int,
                                    C.POINTER(OReport)]
        L.orc_deflated_pcg_solve.argtypes = [C.POINTER(OCsr), vp, C.POINTER(OPrec), vp, vp, C.c_double, C.c_int,
                                             C.POINTER(OReport)]
        L.orc_build_aux.argtypes = [C.POINTER(OCsr), C.c_int, vp, C.c_double, ip, vp, vp, ip]
        L.orc_sampler_offer.argtypes = [vp, C.c_int, C.c_double, vp]
        L.orc_sampler_create_b.argtypes = [C.c_int, C.c_double, C.c_int32, vp]
        L.orc_ic0_factorize.argtypes = [C.POINTER(OCsr), C.c_double, C.c_int, vp]
        L.orc_lanczos_extremes.argtypes = [C.c_int, vp, vp, dp, dp]
        L.orc_mgs.argtypes = [C.c_int32, C.c_int, vp, C.c_double, vp]

    def _chk(self, st):
        if st:
            raise _KIND.get(st, OracleError)(st, self.lib.orc_last_error().decode())

    def reversed_dots(self, order: int = 1):
        """Context manager: run the oracle with every dot product summed in another valid order
        (1 = backwards, 2 = pairwise tree) -- the problem's own sensitivity to reduction order,
        used as the parity rounding floor."""
        import contextlib

        @contextlib.contextmanager
        def cm():
            self.lib.orc_set_dot_order(order)
            try:
                yield self
            finally:
                self.lib.orc_set_dot_order(0)

        return cm()

    # ---- sparse core
    def spmv(self, a: Matrix, x):
        x = _arr(x, np.float64)
        y = np.empty(a.n)
        self.lib.orc_spmv(C.byref(a.c), _p(x), _p(y))
        return y

    def spmv_dual(self, a: Matrix, x1, x2):
        x1, x2 = _arr(x1, np.float64), _arr(x2, np.float64)
        y1, y2 = np.empty(a.n), np.empty(a.n)
        self.lib.orc_spmv_dual(C.byref(a.c), _p(x1), _p(x2), _p(y1), _p(y2))
        return y1, y2

    def dot(self, a, b):
        a, b = _arr(a, np.float64), _arr(b, np.float64)
        return self.lib.orc_dot(len(a), _p(a), _p(b))

    def diagonal_scale(self, a: Matrix):
        va = np.empty(len(a.va))
        dis = np.empty(a.n)
        self._chk(self.lib.orc_diagonal_scale(C.byref(a.c), _p(va), _p(dis)))
        return Matrix(a.n, a.rs, a.ci, va), dis

    def uniform_pm1(self, seed, skip, n):
        out = np.empty(n)
        self.lib.orc_uniform_pm1_fill(seed, skip, n, _p(out))
        return out

    # ---- IC
    def ic0_factorize(self, a: Matrix, shift=0.0, nblocks=1):
        h = C.POINTER(OIc)()
        self._chk(self.lib.orc_ic0_factorize(C.byref(a.c), C.c_double(shift), nblocks, C.byref(h)))
        return OracleIc(self, h)

    def ic_apply(self, f, r):
        r = _arr(r, np.float64)
        z = np.empty(len(r))
        self.lib.orc_ic_apply(f.h, _p(r), _p(z))
        return z

    # ---- dense
    def sym_eig(self, s):
        s = _arr(s, np.float64)
        k = s.shape[0]
        vals, vecs = np.empty(k), np.empty((k, k))
        self._chk(self.lib.orc_sym_eig(k, _p(s), _p(vals), _p(vecs)))
        return vals, vecs

    def chol_factor(self, s):
        s = _arr(s, np.float64)
        k = s.shape[0]
        l = np.empty((k, k))
        self._chk(self.lib.orc_chol_factor(k, _p(s), _p(l)))
        return l

    def mgs(self, cols, drop_tol=1e-12):
        cols = _arr(cols, np.float64)
        k, n = cols.shape if cols.size else (0, 0)
        e = np.empty((max(k, 1), max(n, 1)))
        kept = self.lib.orc_mgs(n, k, _p(cols), C.c_double(drop_tol), _p(e))
        return e[:kept].copy()

    # ---- basis / projections
    def basis(self, a: Matrix, w_cols, who=0):
        w = _arr(w_cols, np.float64).reshape(-1, a.n) if len(w_cols) else np.zeros((0, a.n))
        h = C.POINTER(OBasis)()
        self._chk(self.lib.orc_basis_build(C.byref(a.c), w.shape[0], _p(w) if w.size else None, who, C.byref(h)))
        return OracleBasis(self, h, a.n)

    # ---- sampler
    def sampler_a(self, m, cap, n):
        h = C.POINTER(OSampler)()
        self._chk(self.lib.orc_sampler_create_a(m, cap, n, C.byref(h)))
        return OracleSampler(self, h)

    def sampler_b(self, m, eps, n):
        h = C.POINTER(OSampler)()
        self._chk(self.lib.orc_sampler_create_b(m, C.c_double(eps), n, C.byref(h)))
        return OracleSampler(self, h)

    # ---- solvers
    def _prec(self, kind, ic=None, sc=None):
        p = OPrec(kind, C.cast(ic.h, vp) if ic is not None else None, C.cast(sc.h, vp) if sc is not None else None)
        return p

    def pcg_solve(self, a: Matrix, b, x, kind=0, ic=None, sc=None, eps=1e-8, max_iter=1000, sampler=None,
                  payload=0):
        b = _arr(b, np.float64)
        rep, bufs = _report(max_iter)
        p = self._prec(kind, ic, sc)
        st = self.lib.orc_pcg_solve(C.byref(a.c), _p(b), C.byref(p), _p(x), C.c_double(eps), max_iter,
                                    C.cast(sampler.h, vp) if sampler is not None else None, payload, C.byref(rep))
        self._chk(st)
        return _finish(rep, bufs)

    def deflated_pcg_solve(self, a: Matrix, b, x, basis, kind=1, ic=None, eps=1e-8, max_iter=1000):
        b = _arr(b, np.float64)
        rep, bufs = _report(max_iter)
        p = self._prec(kind, ic, None)
        st = self.lib.orc_deflated_pcg_solve(C.byref(a.c), _p(b), C.byref(p), C.cast(basis.h, vp) if basis else None,
                                             _p(x), C.c_double(eps), max_iter, C.byref(rep))
        self._chk(st)
        return _finish(rep, bufs)

    def pcg_with_condest(self, a: Matrix, b, x, kind=0, ic=None, sc=None, eps=1e-8, max_iter=1000, m_samples=20,
                         seed=42):
        b = _arr(b, np.float64)
        rep, bufs = _report(max_iter)
        est = OCond()
        ritz = np.zeros(max(1, m_samples))
        est.ritz_values = ritz.ctypes.data_as(dp)
        p = self._prec(kind, ic, sc)
        self._chk(self.lib.orc_pcg_with_condest(C.byref(a.c), _p(b), C.byref(p), _p(x), eps, max_iter, m_samples,
                                                seed, C.byref(rep), C.byref(est)))
        return _finish(rep, bufs), Cond(est.lambda_max, est.lambda_min, est.kappa, est.power_iterations,
                                        bool(est.power_unsettled), bool(est.lambda_min_available),
                                        ritz[: est.nritz].copy())

    # ---- recycling
    def harvest_errors(self, x_final, sampler):
        n = sampler.n
        x_final = _arr(x_final, np.float64)
        e = np.empty((sampler.m, max(n, 1)))
        k = self.lib.orc_harvest_errors(_p(x_final), sampler.h, _p(e))
        return e[:k].copy()

    def harvest_stored(self, sampler):
        e = np.empty((sampler.m, max(sampler.n, 1)))
        k = self.lib.orc_harvest_stored(sampler.h, _p(e))
        return e[:k].copy()

    def rayleigh_ritz(self, a: Matrix, e_cols):
        e = _arr(e_cols, np.float64)
        k = e.shape[0]
        vals = np.empty(max(k, 1))
        vecs = np.empty((max(k, 1), a.n))
        self._chk(self.lib.orc_rayleigh_ritz(C.byref(a.c), k, _p(e), _p(vals), _p(vecs)))
        return vals[:k].copy(), vecs[:k].copy()

    def build_aux(self, a: Matrix, errors, theta):
        e = _arr(errors, np.float64)
        k = e.shape[0]
        mb, mt = C.c_int(), C.c_int()
        vals = np.empty(max(k, 1))
        w = np.empty((max(k, 1), a.n))
        self._chk(self.lib.orc_build_aux(C.byref(a.c), k, _p(e) if k else None, C.c_double(theta), C.byref(mb),
                                         _p(vals), _p(w), C.byref(mt)))
        return mb.value, vals[: mb.value].copy(), w[: mt.value].copy()

    def lanczos_extremes(self, alphas, betas):
        a, b = _arr(alphas, np.float64), _arr(betas, np.float64)
        lo, hi = C.c_double(), C.c_double()
        self._chk(self.lib.orc_lanczos_extremes(len(a), _p(a), _p(b), C.byref(lo), C.byref(hi)))
        return lo.value, hi.value


def _report(max_iter):
    rep = OReport()
    bufs = (np.zeros(max_iter), np.zeros(max_iter), np.zeros(max_iter))
    rep.cap = max_iter
    rep.history = bufs[0].ctypes.data_as(dp)
    rep.alphas = bufs[1].ctypes.data_as(dp)
    rep.betas = bufs[2].ctypes.data_as(dp)
    return rep, bufs


def _finish(rep, bufs):
    k = rep.iterations
    return Report(k, bool(rep.converged), rep.wall_time, bufs[0][:k].copy(), bufs[1][:k].copy(), bufs[2][:k].copy())


class OracleIc:
    def __init__(self, o: Oracle, h):
        self.o, self.h = o, h
        f = h.contents
        self.n, self.nnz_l, self.shift_used, self.nblocks = f.n, f.nnz_l, f.shift, f.nblocks

    def arrays(self):
        f = self.h.contents
        n, nnz = self.n, self.nnz_l

        def v(ptr, cnt, ct, dt):
            if cnt == 0:
                return np.zeros(0, dt)
            return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ct)), shape=(cnt,)).copy()

        return dict(block_bounds=v(f.bounds, self.nblocks + 1, C.c_int32, np.int32),
                    l_row_start=v(f.lrs, n + 1, C.c_int32, np.int32), l_col=v(f.lcol, nnz, C.c_int32, np.int32),
                    l_val=v(f.lval, nnz, C.c_double, np.float64), d=v(f.d, n, C.c_double, np.float64),
                    u_row_start=v(f.urs, n + 1, C.c_int32, np.int32), u_col=v(f.ucol, nnz, C.c_int32, np.int32),
                    u_val=v(f.uval, nnz, C.c_double, np.float64))

    def __del__(self):
        try:
            self.o.lib.orc_ic_free(self.h)
        except Exception:
            pass


class OracleBasis:
    def __init__(self, o, h, n):
        self.o, self.h, self.n = o, h, n
        self.k = h.contents.k

    def _op(self, fn, v):
        v = _arr(v, np.float64)
        out = np.empty(self.n)
        fn(self.h, _p(v), _p(out))
        return out

    def project_pt(self, y):
        return self._op(self.o.lib.orc_project_pt, y)

    def project_p(self, x):
        return self._op(self.o.lib.orc_project_p, x)

    def direct_component(self, b):
        return self._op(self.o.lib.orc_direct_component, b)

    def __del__(self):
        try:
            self.o.lib.orc_basis_free(self.h)
        except Exception:
            pass


class OracleSampler:
    def __init__(self, o, h):
        self.o, self.h = o, h
        s = h.contents
        self.m, self.n = s.m, s.n

    def offer(self, it, relres, payload):
        payload = _arr(payload, np.float64)
        self.o.lib.orc_sampler_offer(C.cast(self.h, vp), it, C.c_double(relres), _p(payload))

    def state(self):
        s = self.h.contents
        occ = np.ctypeslib.as_array(C.cast(s.occupied, ip), shape=(self.m,)).astype(bool)
        it = np.ctypeslib.as_array(C.cast(s.stored_iter, ip), shape=(self.m,)).copy()
        return occ, it

    def slot(self, j):
        s = self.h.contents
        return np.ctypeslib.as_array(C.cast(s.slots, dp), shape=(self.m * max(self.n, 1),))[
            j * self.n:(j + 1) * self.n].copy()

    def __del__(self):
        try:
            self.o.lib.orc_sampler_free(self.h)
        except Exception:
            pass


# ---------------------------------------------------------------------------------- reference
class RefReport(C.Structure):
    _fields_ = OReport._fields_


class RefLib:
    """The unmodified reference (oracle/_ref/librecycg_ref.so) through ref_shim.cpp."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise ImportError(f"{path} missing: run `make -C {HERE} ref` where /root/reference exists")
        self.lib = L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        for name in ("ref_csr_create", "ref_ic0", "ref_prec_identity", "ref_prec_ic", "ref_prec_sc",
                     "ref_deflation_build", "ref_sampler_a", "ref_sampler_b"):
            getattr(L, name).restype = vp
        L.ref_csr_create.argtypes = [C.c_int32, vp, vp, vp, ip]
        L.ref_ic0.argtypes = [vp, C.c_double, C.c_int, ip]
        L.ref_ic_nnz.restype = C.c_int64
        L.ref_ic_nnz.argtypes = [vp]
        L.ref_ic_shift.restype = C.c_double
        L.ref_ic_shift.argtypes = [vp]
        L.ref_ic_export.argtypes = [vp] + [vp] * 7
        L.ref_prec_ic.argtypes = [vp]
        L.ref_prec_sc.argtypes = [vp, vp, C.c_int, vp, ip]
        L.ref_deflation_build.argtypes = [vp, C.c_int, vp, ip]
        L.ref_sampler_a.argtypes = [C.c_int, C.c_int, ip]
        L.ref_sampler_b.argtypes = [C.c_int, C.c_double, ip]
        L.ref_sampler_offer.argtypes = [vp, C.c_int, C.c_double, C.c_int32, vp]
        L.ref_pcg_solve.argtypes = [vp, vp, vp, vp, C.c_double, C.c_int, vp, C.c_int, C.POINTER(RefReport)]
        L.ref_deflated_pcg_solve.argtypes = [vp, vp, vp, vp, vp, C.c_double, C.c_int, C.POINTER(RefReport)]
        L.ref_pcg_with_condest.argtypes = [vp, vp, vp, vp, C.c_double, C.c_int, C.c_int, C.c_uint64,
                                           C.POINTER(RefReport), C.POINTER(OCond)]
        L.ref_harvest_errors.argtypes = [vp, C.c_int32, vp, vp, ip]
        L.ref_build_aux.argtypes = [vp, C.c_int, vp, C.c_double, ip, vp, vp, ip]
        L.ref_rayleigh_ritz.argtypes = [vp, C.c_int, vp, vp, vp]
        L.ref_mgs.argtypes = [C.c_int32, C.c_int, vp, C.c_double, vp, ip]
        L.ref_sym_eig.argtypes = [C.c_int, vp, vp, vp]
        L.ref_chol_factor.argtypes = [C.c_int, vp, vp]
        for name in ("ref_csr_free", "ref_ic_free", "ref_prec_free", "ref_deflation_free", "ref_sampler_free"):
            getattr(L, name).argtypes = [vp]

    def _chk(self, st):
        if st:
            raise _KIND.get(st, OracleError)(st, self.lib.ref_last_error().decode())

    def matrix(self, a: Matrix):
        st = C.c_int()
        h = self.lib.ref_csr_create(a.n, _p(a.rs), _p(a.ci), _p(a.va), C.byref(st))
        self._chk(st.value)
        return _Owned(h, self.lib.ref_csr_free, n=a.n)

    def spmv(self, m, x):
        x = _arr(x, np.float64)
        y = np.empty(m.n)
        self._chk(self.lib.ref_spmv(m.h, _p(x), _p(y)))
        return y

    def spmv_dual(self, m, x1, x2):
        x1, x2 = _arr(x1, np.float64), _arr(x2, np.float64)
        y1, y2 = np.empty(m.n), np.empty(m.n)
        self._chk(self.lib.ref_spmv_dual(m.h, _p(x1), _p(x2), _p(y1), _p(y2)))
        return y1, y2

    def diagonal_scale(self, m, nnz):
        va, dis = np.empty(nnz), np.empty(m.n)
        self._chk(self.lib.ref_diagonal_scale(m.h, _p(va), _p(dis)))
        return va, dis

    def ic0(self, m, shift=0.0, nblocks=1):
        st = C.c_int()
        h = self.lib.ref_ic0(m.h, shift, nblocks, C.byref(st))
        self._chk(st.value)
        f = _Owned(h, self.lib.ref_ic_free, n=m.n)
        nnz = self.lib.ref_ic_nnz(h)
        out = dict(l_row_start=np.empty(m.n + 1, np.int32), l_col=np.empty(nnz, np.int32), l_val=np.empty(nnz),
                   d=np.empty(m.n), u_row_start=np.empty(m.n + 1, np.int32), u_col=np.empty(nnz, np.int32),
                   u_val=np.empty(nnz))
        self.lib.ref_ic_export(h, *[_p(v) for v in out.values()])
        f.arrays = out
        f.shift_used = self.lib.ref_ic_shift(h)
        return f

    def ic_apply(self, f, r):
        r = _arr(r, np.float64)
        z = np.empty(f.n)
        self._chk(self.lib.ref_ic_apply(f.h, _p(r), _p(z)))
        return z

    def prec_identity(self):
        return _Owned(self.lib.ref_prec_identity(), self.lib.ref_prec_free)

    def prec_ic(self, f):
        return _Owned(self.lib.ref_prec_ic(f.h), self.lib.ref_prec_free)

    def prec_sc(self, inner, m, w_cols):
        w = _arr(w_cols, np.float64)
        st = C.c_int()
        h = self.lib.ref_prec_sc(inner.h, m.h, w.shape[0], _p(w) if w.size else None, C.byref(st))
        self._chk(st.value)
        return _Owned(h, self.lib.ref_prec_free)

    def deflation(self, m, w_cols):
        w = _arr(w_cols, np.float64)
        st = C.c_int()
        h = self.lib.ref_deflation_build(m.h, w.shape[0], _p(w) if w.size else None, C.byref(st))
        self._chk(st.value)
        return _Owned(h, self.lib.ref_deflation_free)

    def sampler_a(self, m, cap):
        st = C.c_int()
        h = self.lib.ref_sampler_a(m, cap, C.byref(st))
        self._chk(st.value)
        return _Owned(h, self.lib.ref_sampler_free, m=m)

    def sampler_state(self, s):
        occ = np.array([self.lib.ref_sampler_occupied(s.h, j) for j in range(s.m)], bool)
        it = np.array([self.lib.ref_sampler_stored_iteration(s.h, j) for j in range(s.m)], np.int32)
        return occ, it

    def pcg_solve(self, m, b, prec, x, eps=1e-8, max_iter=1000, sampler=None, payload=0):
        b = _arr(b, np.float64)
        rep = RefReport()
        hist = np.zeros(max_iter)
        rep.cap = max_iter
        rep.history = hist.ctypes.data_as(dp)
        self._chk(self.lib.ref_pcg_solve(m.h, _p(b), prec.h, _p(x), eps, max_iter,
                                         sampler.h if sampler is not None else None, payload, C.byref(rep)))
        return Report(rep.iterations, bool(rep.converged), rep.wall_time, hist[: rep.iterations].copy())

    def deflated_pcg_solve(self, m, b, prec, defl, x, eps=1e-8, max_iter=1000):
        b = _arr(b, np.float64)
        rep = RefReport()
        hist = np.zeros(max_iter)
        rep.cap = max_iter
        rep.history = hist.ctypes.data_as(dp)
        self._chk(self.lib.ref_deflated_pcg_solve(m.h, _p(b), prec.h, defl.h if defl is not None else None, _p(x),
                                                  eps, max_iter, C.byref(rep)))
        return Report(rep.iterations, bool(rep.converged), rep.wall_time, hist[: rep.iterations].copy())

    def pcg_with_condest(self, m, b, prec, x, eps=1e-8, max_iter=1000, m_samples=20, seed=42):
        b = _arr(b, np.float64)
        rep = RefReport()
        hist = np.zeros(max_iter)
        rep.cap = max_iter
        rep.history = hist.ctypes.data_as(dp)
        est = OCond()
        ritz = np.zeros(max(1, m_samples))
        est.ritz_values = ritz.ctypes.data_as(dp)
        self._chk(self.lib.ref_pcg_with_condest(m.h, _p(b), prec.h, _p(x), eps, max_iter, m_samples, seed,
                                                C.byref(rep), C.byref(est)))
        return (Report(rep.iterations, bool(rep.converged), rep.wall_time, hist[: rep.iterations].copy()),
                Cond(est.lambda_max, est.lambda_min, est.kappa, est.power_iterations, bool(est.power_unsettled),
                     bool(est.lambda_min_available), ritz[: est.nritz].copy()))

    def harvest_errors(self, x_final, sampler, n):
        x_final = _arr(x_final, np.float64)
        e = np.empty((sampler.m, max(n, 1)))
        k = C.c_int()
        self._chk(self.lib.ref_harvest_errors(_p(x_final), n, sampler.h, _p(e), C.byref(k)))
        return e[: k.value].copy()

    def build_aux(self, m, errors, theta):
        e = _arr(errors, np.float64)
        k = e.shape[0]
        mb, mt = C.c_int(), C.c_int()
        vals = np.empty(max(k, 1))
        w = np.empty((max(k, 1), m.n))
        self._chk(self.lib.ref_build_aux(m.h, k, _p(e) if k else None, theta, C.byref(mb), _p(vals), _p(w),
                                         C.byref(mt)))
        return mb.value, vals[: mb.value].copy(), w[: mt.value].copy()

    def mgs(self, cols, drop_tol=1e-12):
        cols = _arr(cols, np.float64)
        k, n = cols.shape
        e = np.empty((max(k, 1), max(n, 1)))
        kept = C.c_int()
        self._chk(self.lib.ref_mgs(n, k, _p(cols), drop_tol, _p(e), C.byref(kept)))
        return e[: kept.value].copy()

    def sym_eig(self, s):
        s = _arr(s, np.float64)
        k = s.shape[0]
        vals, vecs = np.empty(k), np.empty((k, k))
        self._chk(self.lib.ref_sym_eig(k, _p(s), _p(vals), _p(vecs)))
        return vals, vecs

    def chol_factor(self, s):
        s = _arr(s, np.float64)
        k = s.shape[0]
        l = np.empty((k, k))
        self._chk(self.lib.ref_chol_factor(k, _p(s), _p(l)))
        return l


class _Owned:
    def __init__(self, h, free, **kw):
        self.h, self._free = h, free
        self.__dict__.update(kw)

    def __del__(self):
        try:
            if self.h:
                self._free(self.h)
                self.h = None
        except Exception:
            pass


def available() -> dict:
    return {"oracle": os.path.exists(ORACLE_SO), "ref": os.path.exists(REF_SO)}
