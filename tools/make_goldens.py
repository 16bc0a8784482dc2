"""Full-size oracle goldens for the sequence protocol (TEST INFRASTRUCTURE; runs on the CPU box).

    python tools/make_goldens.py c3 [--workers 8]      # also c5, c4like, c2, c1

Runs run_sequence (proj/src/driver.cpp:108-222) on the CPU oracle (oracle/oracle.c, pinned
bitwise to the reference library by tests/test_oracle.py) at the BASELINE.json size of the config:
diagonal scaling, IC(0), solve 1 with the method-A error sampler, harvest -> MGS -> Rayleigh-Ritz
(the reference's build_aux, recycling.cpp:81-96, run as its two stages so the peak memory fits),
count-based selection of the m~ smallest Ritz vectors, then the deflated / SC solves 2..k -- which
are independent given W (driver.cpp:181-195) and run here on `--workers` threads (the oracle's
C calls release the GIL; every solve is the serial reference algorithm).

Writes tests/golden/<config>.json (per solve: iterations, converged, true relative residual,
Lanczos lambda_min / lambda_max / kappa from the solve's own alpha / beta; m_bar, m_tilde, Ritz
values, sampled iterations, input checksums, CPU wall times) and tests/golden/<config>_x.npz
(each solution in the original scaling at 8,192 seeded row indices), which the -m gpu tests
(tests/test_gpu_golden.py) compare rcg_seq_run against.  Inputs come from oracle/inputs.py (the
shared generator built without librcg_b200.so).
"""
from __future__ import annotations

import argparse
import ctypes as C
import hashlib
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import Matrix, Oracle, inputs  # noqa: E402
from paper_2203_08498_b200.configs import CONFIGS, VARIANTS  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
N_SAMPLE = 8192
SAMPLE_SEED = 12345


def sample_rows(n: int) -> np.ndarray:
    rng = np.random.default_rng(SAMPLE_SEED)
    return np.sort(rng.choice(n, size=min(N_SAMPLE, n), replace=False)).astype(np.int64)


def checksums(h) -> dict:
    return {"nnz": int(h.nnz),
            "row_start_sha256": hashlib.sha256(h.row_start.tobytes()).hexdigest(),
            "col_idx_sha256": hashlib.sha256(h.col_idx.tobytes()).hexdigest(),
            "values_sha256": hashlib.sha256(h.values.tobytes()).hexdigest()}


def log(*a):
    print(time.strftime("%H:%M:%S"), *a, flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 8)
    ap.add_argument("--solves", type=int, default=None, help="only the first k solves (debug)")
    ap.add_argument("--floor", action="store_true",
                    help="add solve 1's rounding floor to an existing golden: the oracle's own relative "
                         "change when every dot product is summed backwards / pairwise (DESIGN.md section 4)")
    args = ap.parse_args()
    cfg = {**CONFIGS, **VARIANTS}[args.config]
    if args.floor:
        return add_floor(cfg)
    o = Oracle()
    t_all = time.perf_counter()
    wall = {}

    t = time.perf_counter()
    h = inputs.generate(cfg)
    n = h.n
    wall["generate_s"] = time.perf_counter() - t
    log(cfg.name, "n", n, "nnz", h.nnz)
    sums = checksums(h)
    a_orig = Matrix.of(h)
    t = time.perf_counter()
    a, dis = o.diagonal_scale(a_orig)
    ic = o.ic0_factorize(a)
    wall["scale_and_ic0_s"] = time.perf_counter() - t
    log("ic0 shift", ic.shift_used, f"{wall['scale_and_ic0_s']:.1f}s")

    k_total = cfg.n_rhs if args.solves is None else args.solves
    b_orig = np.empty((k_total, n))
    for k, x in enumerate(inputs.solution_streams(cfg, n, k_total)):
        b_orig[k] = o.spmv(a_orig, x)
    idx = sample_rows(n)
    xs_sample = np.zeros((k_total, idx.size))
    per = [None] * k_total

    def finish(k, rep, x):
        lo, hi = o.lanczos_extremes(rep.alphas, rep.betas) if rep.iterations >= 1 else (float("nan"),) * 2
        x_orig = dis * x
        r = b_orig[k] - o.spmv(a_orig, x_orig)
        xs_sample[k] = x_orig[idx]
        per[k] = {"iterations": rep.iterations, "converged": rep.converged,
                  "true_relres": float(np.linalg.norm(r) / np.linalg.norm(b_orig[k])),
                  "final_recurrence_relres": float(rep.history[-1]) if rep.iterations else 0.0,
                  "lanczos_lambda_min": lo, "lanczos_lambda_max": hi, "kappa": hi / lo,
                  "x_norm": float(np.linalg.norm(x_orig)), "wall_s": rep.wall_time}

    # ---- solve 1: ICCG with the error sampler (driver.cpp:150-158)
    t = time.perf_counter()
    sampler = o.sampler_a(cfg.sampler_m, cfg.max_iter, n)
    x1 = np.zeros(n)
    r1 = o.pcg_solve(a, dis * b_orig[0], x1, kind=1, ic=ic, eps=cfg.eps, max_iter=cfg.max_iter, sampler=sampler)
    wall["solve1_s"] = time.perf_counter() - t
    finish(0, r1, x1)
    occ, it = sampler.state()
    sampled = sorted(int(v) for v in it[occ])
    log("solve 1:", r1.iterations, "its", f"{wall['solve1_s']:.1f}s", "sampled", len(sampled))

    # ---- recycling: harvest -> MGS -> Rayleigh-Ritz (build_aux, recycling.cpp:81-96) -> W
    t = time.perf_counter()
    errors = o.harvest_errors(x1, sampler)
    del sampler, x1
    k_err = errors.shape[0]
    q = np.empty((max(k_err, 1), n))
    m_bar = o.lib.orc_mgs(n, k_err, C.c_void_p(errors.ctypes.data), C.c_double(1e-12), C.c_void_p(q.ctypes.data)) if k_err else 0
    del errors
    vals = np.empty(max(m_bar, 1))
    vecs = np.empty((max(m_bar, 1), n))
    if m_bar:
        st = o.lib.orc_rayleigh_ritz(C.byref(a.c), m_bar, C.c_void_p(q.ctypes.data), C.c_void_p(vals.ctypes.data),
                                      C.c_void_p(vecs.ctypes.data))
        o._chk(st)
    del q
    keep = cfg.keep if m_bar > cfg.keep else m_bar
    w = np.ascontiguousarray(vecs[:keep])
    del vecs
    wall["recycle_s"] = time.perf_counter() - t
    t = time.perf_counter()
    basis = o.basis(a, w, who=1 if cfg.method == "sc" else 0) if keep else None
    del w
    wall["basis_s"] = time.perf_counter() - t
    log("m_bar", m_bar, "m_tilde", keep, f"recycle {wall['recycle_s']:.1f}s basis {wall['basis_s']:.1f}s",
        "ritz[:4]", vals[:min(4, m_bar)])

    # ---- solves 2..k (independent given W; driver.cpp:181-195)
    def solve(k):
        ts = time.perf_counter()
        x = np.zeros(n)
        bk = dis * b_orig[k]
        if basis is None:
            rep = o.pcg_solve(a, bk, x, kind=1, ic=ic, eps=cfg.eps, max_iter=cfg.max_iter)
        elif cfg.method == "sc":
            rep = o.pcg_solve(a, bk, x, kind=2, ic=ic, sc=basis, eps=cfg.eps, max_iter=cfg.max_iter)
        else:
            rep = o.deflated_pcg_solve(a, bk, x, basis, kind=1, ic=ic, eps=cfg.eps, max_iter=cfg.max_iter)
        finish(k, rep, x)
        log(f"solve {k + 1}:", rep.iterations, "its", f"{time.perf_counter() - ts:.1f}s")

    t = time.perf_counter()
    with ThreadPoolExecutor(max_workers=max(1, args.workers)) as pool:
        list(pool.map(solve, range(1, k_total)))
    wall["solves_2_k_s"] = time.perf_counter() - t
    wall["total_s"] = time.perf_counter() - t_all

    out = {
        "config": cfg.name, "n": n, "inputs": sums, "method": cfg.method, "eps": cfg.eps, "max_iter": cfg.max_iter,
        "n_rhs": k_total, "sampler_m": cfg.sampler_m, "keep": cfg.keep, "condest": cfg.condest,
        "shift_used": ic.shift_used, "sampled_iterations": sampled, "m_bar": int(m_bar), "m_tilde": int(keep),
        "ritz_values": [float(v) for v in vals[:m_bar]],
        "iterations": [p["iterations"] for p in per], "solves": per,
        "sample_rows": {"count": int(idx.size), "seed": SAMPLE_SEED},
        "cpu_wall": {**wall, "workers_solves_2_k": args.workers, "nproc": os.cpu_count(),
                     "note": "oracle/oracle.c single-threaded per solve; solves 2..k run concurrently"},
        "generator": "tools/make_goldens.py (oracle/oracle.c, pinned bitwise to oracle/_ref)",
    }
    os.makedirs(GOLDEN, exist_ok=True)
    stem = os.path.join(GOLDEN, cfg.name if args.solves is None else f"{cfg.name}_first{k_total}")
    with open(stem + ".json", "w") as f:
        json.dump(out, f, indent=1)
    np.savez_compressed(stem + "_x.npz", rows=idx, x=xs_sample)
    log("wrote", stem + ".json", "iterations", out["iterations"], f"total {wall['total_s']:.0f}s")


def add_floor(cfg) -> None:
    """Solve 1 + its recycling step again with every dot product summed backwards, then pairwise
    (a separate copy of the oracle library per order): the spread of the solution (at the golden's
    sample rows), of the iteration count and of each Ritz value against the golden is the
    problem's own sensitivity to reduction order -- the parity floor for the GPU's parallel,
    fixed-order reductions.  Orders run one after the other (C3's
    Rayleigh-Ritz step needs ~25 GB)."""
    path = os.path.join(GOLDEN, cfg.name + ".json")
    gold = json.load(open(path))
    xs = np.load(path[:-5] + "_x.npz")
    idx, x_base = xs["rows"], xs["x"][0]
    o = Oracle()
    h = inputs.generate(cfg)
    n = h.n
    a_orig = Matrix.of(h)
    a, dis = o.diagonal_scale(a_orig)
    ic = o.ic0_factorize(a)
    x0 = next(inputs.solution_streams(cfg, n, 1))
    b = dis * o.spmv(a_orig, x0)
    del h
    rv = np.asarray(gold["ritz_values"])
    sol_floor, its, ritz_floor = 0.0, [gold["iterations"][0]], np.zeros(rv.size)
    for order in (1, 2):
        oo = _oracle_with_order(order)
        sampler = oo.sampler_a(cfg.sampler_m, cfg.max_iter, n)
        x = np.zeros(n)
        rep = oo.pcg_solve(a, b, x, kind=1, ic=ic, eps=cfg.eps, max_iter=cfg.max_iter, sampler=sampler)
        its.append(rep.iterations)
        xo = (dis * x)[idx]
        sol_floor = max(sol_floor, float(np.linalg.norm(xo - x_base) / np.linalg.norm(x_base)))
        errors = oo.harvest_errors(x, sampler)
        del sampler, x
        k_err = errors.shape[0]
        q = np.empty((max(k_err, 1), n))
        m_bar = oo.lib.orc_mgs(n, k_err, C.c_void_p(errors.ctypes.data), C.c_double(1e-12), C.c_void_p(q.ctypes.data))
        del errors
        vals = np.empty(max(m_bar, 1))
        vecs = np.empty((max(m_bar, 1), n))
        oo._chk(oo.lib.orc_rayleigh_ritz(C.byref(a.c), m_bar, C.c_void_p(q.ctypes.data), C.c_void_p(vals.ctypes.data),
                                         C.c_void_p(vecs.ctypes.data)))
        del q, vecs
        if m_bar == rv.size:
            ritz_floor = np.maximum(ritz_floor, np.abs(vals[:m_bar] - rv) / np.abs(rv))
        log("floor order", order, "its", rep.iterations, "m_bar", m_bar, "solution", sol_floor,
            "ritz max", float(ritz_floor.max()) if ritz_floor.size else 0.0)
    gold["solve1_floor"] = {"rel_solution": sol_floor, "iterations": its,
                            "note": "oracle solve 1 with dot products summed sequentially / backwards / pairwise; "
                                    "solution compared at the golden's sample rows"}
    gold["ritz_floor"] = {"rel": [float(v) for v in ritz_floor],
                          "note": "per Ritz value: max relative change when solve 1's dot products are summed "
                                  "backwards / pairwise (same sampler, MGS, Rayleigh-Ritz)"}
    with open(path, "w") as f:
        json.dump(gold, f, indent=1)
    log("floor", sol_floor, "iterations", its, "ritz floor max", float(ritz_floor.max()) if ritz_floor.size else 0.0)


def _oracle_with_order(order):
    """A separate copy of liboracle.so (its own global dot-order switch) summing in `order`."""
    import shutil
    import tempfile

    from oracle import ORACLE_SO

    d = tempfile.mkdtemp(prefix="orc_order")
    p = os.path.join(d, f"liboracle_{order}.so")
    shutil.copy(ORACLE_SO, p)
    oo = Oracle(p)
    oo.lib.orc_set_dot_order(order)
    return oo


if __name__ == "__main__":
    main()
