#!/usr/bin/env python
"""Benchmark: the paper's sequence protocol on the largest single-GPU BASELINE.json config (C3:
256^3 trilinear-hex 27-point FEM, 16.8M rows, 449M entries, log-normal coefficients, 20 drifting
right-hand sides, 64 error samples in solve 1, deflation with the 32 smallest Ritz vectors) on
B200, fp64.  (--config c1 / c2 / c5 run the other configs; C4 is the row-slab configuration.)

One step = the whole sequence through the device sequence driver rcg_seq_run: ICCG solve 1 with
the method-A error sampler, the Rayleigh-Ritz basis (MGS, A E, E^T A E, eig, Ritz vectors), the
deflation operator (A W, W^T A W, Cholesky), then the 19 deflated solves from x0 = 0 (batched),
solutions and true relative residuals in the original scaling.  value = PCG iterations of the
step / device time of the step (CUDA events on the library stream).  e2e = the same step with
pinned HOST right-hand sides and solutions (H2D / D2H inside the call and the timed region).

--impl reference runs the reference library itself (oracle/_ref, compiled from the reference
sources) on all host cores, the same config dict: timed windows of the ICCG and accelerated
iterations per thread, the Rayleigh-Ritz step on real sampled errors, extrapolated to the
oracle's full-run iteration mix (run_reference).

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c3]
For N > 1 launch with torch.distributed.run: the SAME sequence over N row slabs, one per GPU
(run_slabs: block-Jacobi IC(0) per slab, NCCL halo exchange + allreduces, the
accelerated solves batched over the slabs; scaling "strong", the block-Jacobi iteration counts
next to the single-GPU ones).  --replicas instead runs N independent single-GPU sequences
(scaling "weak").
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PCG iters/s (fp64 sequence: ICCG solve 1 + RR + accelerated ICCG solves)"
UNIT = "iters/s"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampled during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{index}.csv")

    def __enter__(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", os.environ.get("RCG_CLOCKS_MS", "200")], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        if not self.proc or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------------- our arm
def run_ours(args, rank, world, local_rank):
    import torch

    from paper_2203_08498_b200 import api, problems, sequence

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    ctx = api.Context(local_rank)
    cfg = problems.CONFIGS[args.config]
    host = problems.generate(cfg)
    prep = sequence.prepare(ctx, cfg, host, validate=True)
    n = host.n
    pairs = sequence.rhs_all(prep)
    # one step = one sequence through the device sequence driver (rcg_seq_run: scaled solve 1 with
    # the sampler, RR basis, batched solves 2..k, solutions + true relres in the original
    # scaling -- run_sequence, driver.cpp:108-222); scaling + IC(0) are per-matrix setup
    seq = api.Sequence(ctx, prep.a_orig, "es-sc-iccg" if cfg.method == "sc" else "es-d-iccg", cfg.blocks)
    b_dev = torch.from_numpy(np.stack([b for b, _ in pairs])).to(dev)       # unscaled b = A x_k
    b_pin = torch.from_numpy(np.stack([b for b, _ in pairs])).pin_memory()
    x_pin = torch.zeros((cfg.n_rhs, n), dtype=torch.float64).pin_memory()
    x_dev = torch.zeros((cfg.n_rhs, n), dtype=torch.float64, device=dev)
    n_nnz = host.nnz
    nnz_l = prep.ic.nnz_l
    last = {}

    def run(B, X):
        rep = seq.run(B, X, cfg.eps, cfg.max_iter, "A", cfg.sampler_m, keep_count=cfg.keep, batch=True,
                      condest=cfg.condest)  # C5: a Lanczos condition estimate on every solve
        last.update(rep)
        return sum(rep["iterations"])

    def step_device():
        return run(b_dev, x_dev)

    def step_e2e():
        # host right-hand sides and solutions (pinned): H2D / D2H inside the C-ABI call
        return run(b_pin.numpy(), x_pin.numpy())

    for _ in range(args.warmup):
        step_device()
    if world > 1:
        torch.distributed.barrier()
    ctx.synchronize()
    ctxs = _all_contexts(prep)
    # CUDA-event class timers inside the timed region only on the sweep classes (the level-chain
    # bound kernels, the roofline's candidates): timing every launch (~3,000 per step) costs ~3 %
    # of the step; the other classes are timed over the same number of separate steps after it
    for c_ in ctxs:
        c_.synchronize()
        c_.set_profiling(PROFILE_TIMED, classes=TIMED_CLASSES)
        c_.reset_stats()
    launches0 = sum(c_.launches for c_ in ctxs)
    iters = 0
    with Clocks(local_rank) as clk:
        ctx.record(0)
        for _ in range(args.steps):
            iters += step_device()
        ctx.record(1)
        ms = ctx.elapsed_ms(0, 1)
    launches = sum(c_.launches for c_ in ctxs) - launches0
    stats_timed = kernel_stats(ctxs)
    ctxs = _all_contexts(prep)
    for c_ in ctxs:
        c_.set_profiling(True)
        c_.reset_stats()
    for _ in range(args.steps):
        step_device()
    ctxs = _all_contexts(prep)
    stats_rest = kernel_stats(ctxs)
    stats = {c: (stats_timed[c] if PROFILE_TIMED and c in TIMED_CLASSES else stats_rest[c]) for c in stats_rest}
    for c_ in ctxs:
        c_.set_profiling(False)
    # phase breakdown of one extra (untimed) step, from the driver's report
    step_device()
    w = last["wall_time"]
    phases = {"solve1_ms": round(w[0] * 1e3, 2), "solve1_iterations": last["iterations"][0],
              "rr_basis_ms": round(last["w_build_time"] * 1e3, 2),
              "accelerated_ms": round(sum(w[1:]) * 1e3, 2),
              "accelerated_iterations": last["iterations"][1:], "m_tilde": last["m_tilde"],
              "max_true_relres": max(last["true_relres"])}
    if "kappa" in last:
        phases["lanczos_kappa"] = [float(f"{v:.6g}") for v in last["kappa"]]
    cost = cost_model_report(n, n_nnz, cfg.keep, phases)
    # e2e through the public API with host buffers
    for _ in range(max(1, args.warmup // 2)):
        step_e2e()
    ctx.synchronize()
    ctx.record(2)
    e2e_iters = 0
    for _ in range(args.steps):
        e2e_iters += step_e2e()
    ctx.record(3)
    e2e_ms = ctx.elapsed_ms(2, 3)
    # the multi-GPU row-slab path (all ranks take part): one distributed block-Jacobi ICCG solve
    row_slabs = None
    if args.variants:
        try:
            row_slabs = measure_row_slabs(api, prep, host, pairs[0][1], cfg, rank, world, dev, [b for _, b in pairs])
        except Exception as e:  # the headline line must still print
            row_slabs = {"error": f"{type(e).__name__}: {e}"}
    # max over ranks
    t = torch.tensor([ms, e2e_ms], dtype=torch.float64, device=dev)
    it = torch.tensor([float(iters), float(e2e_iters)], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.all_reduce(it, op=torch.distributed.ReduceOp.SUM)
    ms, e2e_ms = t.tolist()
    iters, e2e_iters = it.tolist()
    if rank != 0:
        return
    peak, peak_src = peaks()
    kernels, roof = kernel_report(stats, n, n_nnz, nnz_l, cfg.keep, args.steps, peak, peak_src,
                                  levels=(prep.ic.fwd_levels, prep.ic.bwd_levels), workload=cfg.name)
    line = {
        "metric": METRIC,
        "value": round(iters / (ms / 1e3), 2),
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms / args.steps, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded generator, SURVEY.md 8(d); no network for SuiteSparse)",
        "config": config_dict(cfg, n, n_nnz, world, replicas=True),
        "iterations_per_step": iters / args.steps / world,
        "time_to_solution_ms_per_rhs": round(ms / args.steps / cfg.n_rhs, 3),
        "driver": "rcg_seq_run (solve 1 with the device sampler, RR basis, solves 2..k batched)",
        "e2e": {"value": round(e2e_iters / (e2e_ms / 1e3), 2), "unit": UNIT,
                "h2d_bytes_per_step": 8 * n * cfg.n_rhs, "d2h_bytes_per_step": 8 * n * cfg.n_rhs,
                "time_to_solution_ms_per_rhs": round(e2e_ms / args.steps / cfg.n_rhs, 3)},
        "roofline": roof,
        "kernels": kernels,
        "phases_ms_untimed_step": phases,
        "cost_model": cost,
        "gpu_launches": int(launches),
        "kernel_timing": {"timed_region_classes": [CLASS_NAMES[c] for c in TIMED_CLASSES] if PROFILE_TIMED else [],
                          "other_classes": "CUDA events over the same number of separate steps after the timed region"},
        "clocks": clk.summary(),
    }
    if args.variants:
        line["variants"] = {"multicolour": measure_multicolour(api, problems, sequence, ctx, cfg, host, args, peak),
                            "row_slabs": row_slabs}
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(cfg)
    print(json.dumps(line), flush=True)


# Kernel classes (rcg_b200.h rcg_ctx_kernel_stats): 0-4 single right-hand side, 5-9 batched.
CLASS_NAMES = {0: "spmv (k_spmv_pq)", 1: "ic fwd sweep (k_sweep<false>)", 2: "ic bwd sweep (k_sweep<true>)",
               3: "vector ops", 4: "W^T r (k_tallt)",
               5: "batched spmv (k_b_spmv_pq)", 6: "batched ic fwd sweep (k_b_sweepc<false>)",
               7: "batched ic bwd sweep (k_b_sweepc<true> + k_b_rho)", 8: "batched vector ops", 9: "batched W^T r (k_b_tallt)"}


def kernel_stats(ctxs):
    """{class: (total ms, launches, right-hand-side units)} summed over the contexts."""
    out = {}
    for c in CLASS_NAMES:
        per = [c_.kernel_stats(c) for c_ in ctxs]
        out[c] = (sum(t for t, _ in per), sum(k for _, k in per), sum(c_.kernel_units(c) for c_ in ctxs))
    return out


def algorithmic_bytes(c, n, nnz, nnz_l, m):
    """(bytes per launch, bytes per carried right-hand side) of class c -- DESIGN.md "Roofline
    accounting": matrix / factor / schedule / basis bytes are read once per
    launch; vector bytes scale with the right-hand sides a launch carries."""
    return {
        0: (12 * nnz + 4 * n, 16 * n),      # A (val+col), row starts | p in, q out
        1: (12 * nnz_l + 8 * n, 16 * n),    # L entries, perm+row starts | r in, y out
        2: (12 * nnz_l + 16 * n, 24 * n),   # U entries, perm+row starts, d | y in, z out, r
        4: (8 * m * n, 8 * n),              # W | the projected vector
    }.get(c % 5)


def cost_model_report(n, nnz, m_tilde, phases):
    """The paper's memory-traffic model (cost_model.cpp via paper_2203_08498_b200/cost_model.py)
    at the measured HBM bandwidth against the step's measured per-iteration times, and
    compare_measured's gamma (accelerated per-iteration time / ICCG per-iteration time; the
    accelerated solves run batched, so per right-hand-side iteration)."""
    from paper_2203_08498_b200 import cost_model as cm

    bw = peaks()[0] * 1e9
    p = cm.CostParams(float(n), float(nnz), float(m_tilde), bw)
    it1, t1 = phases["solve1_iterations"], phases["solve1_ms"] * 1e-3
    ita, ta = sum(phases["accelerated_iterations"]), phases["accelerated_ms"] * 1e-3
    out = {"t_iccg_model_us": round(cm.t_iccg(p) * 1e6, 2), "t_sciccg_model_us": round(cm.t_sciccg(p) * 1e6, 2),
           "gamma_predicted": round(cm.gamma_sciccg(m_tilde, nnz / max(n, 1)), 4)}
    if it1 > 0 and t1 > 0:
        out["iccg_measured_us"] = round(t1 / it1 * 1e6, 2)
        out["iccg_model_fraction"] = round(cm.t_iccg(p) / (t1 / it1), 4)
    if it1 > 0 and t1 > 0 and ita > 0:
        c = cm.compare_measured(it1, t1, ita, ta, m_tilde, nnz / max(n, 1))
        out.update(accelerated_us_per_rhs_iteration=round(ta / ita * 1e6, 2), gamma_measured=round(c.measured, 4),
                   gamma_rel_error=round(c.rel_error, 4))
    return out


# inter-SM publish -> observe latency of one dependency hop (tools/pingpong.cu, B200: 0.36-0.54 us)
HOP_FLOOR_US = 0.45


def kernel_report(stats, n, nnz, nnz_l, m, steps, peak, peak_src, levels=None, workload=None):
    # ncu DRAM bytes per launch, per workload (profiles/ncu_traffic.json: {workload: {class: ...}});
    # a class without a capture on this workload reports null rather than another config's bytes
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    traffic = (json.load(open(tp)) if os.path.exists(tp) else {}).get(workload, {})
    kernels, best = {}, None
    for c, (tot_ms, cnt, units) in stats.items():
        if cnt == 0:
            continue
        entry = {"launches": cnt, "avg_us": round(tot_ms / cnt * 1e3, 3), "busy_ms_per_step": round(tot_ms / steps, 2)}
        if c >= 5:
            entry["rhs_per_launch"] = round(units / cnt, 2)
        ab = algorithmic_bytes(c, n, nnz, nnz_l, m)
        if ab:
            per_launch = (ab[0] * cnt + ab[1] * units) / cnt
            entry["algorithmic_bytes"] = int(per_launch)
            entry["achieved_gbs"] = round(per_launch / (tot_ms / cnt * 1e-3) / 1e9, 1)
            t = traffic.get(CLASS_NAMES[c])
            if isinstance(t, dict):  # batched: measured at a given right-hand-side count
                entry["ncu_dram_bytes"] = t
            elif t:
                entry["ncu_dram_bytes"] = t
            if best is None or tot_ms > stats[best][0]:
                best = c
        kernels[CLASS_NAMES[c]] = entry
    e = kernels[CLASS_NAMES[best]]
    t = traffic.get(CLASS_NAMES[best])
    roof = {"bound": "hbm", "kernel": CLASS_NAMES[best], "achieved": e["achieved_gbs"], "peak": peak, "unit": "GB/s",
            "frac": round(e["achieved_gbs"] / peak, 4), "frac_of_spec_8tbs": round(e["achieved_gbs"] / 8000.0, 4),
            "traffic": t["dram_bytes"] if isinstance(t, dict) else t,
            "traffic_source": f"profiles/ncu_traffic.json[{workload}]" if t else "no ncu capture of this kernel on this workload",
            "peak_source": peak_src}
    if isinstance(t, dict):  # the ncu capture's launch carried rhs_per_launch right-hand sides
        roof["traffic_rhs_per_launch"] = t["rhs_per_launch"]
        roof["traffic_algorithmic_bytes"] = t["algorithmic_bytes"]
    if levels and best % 5 in (1, 2):  # a sweep: bound by its dependent level chain, not by HBM
        nl = levels[0] if best % 5 == 1 else levels[1]
        upl = e["avg_us"] / max(nl, 1)
        roof["level_chain"] = {"levels": nl, "us_per_level": round(upl, 3), "hop_floor_us": HOP_FLOOR_US,
                               "frac_of_chain_floor": round(HOP_FLOOR_US / upl, 3),
                               "note": "each level waits for its parents' publish -> observe hop; "
                                       "levels x hop floor bounds the sweep below the HBM roofline"}
    return kernels, roof


def run_slabs(args, rank, world, local_rank):
    """N > 1: the north star's multi-GPU path -- the SAME sequence (the config's matrix and
    right-hand sides) over `world` row slabs at floor(b n / N), one per GPU: block-Jacobi IC(0) per
    slab (ic0_factorize(a, 0, N), ic_preconditioner.cpp:97-121), NCCL halo exchange + allreduces,
    solve 1 with the error sampler (rcg_dist_pcg_solve_sampled), the distributed recycling step
    (rcg_dist_recycle) and the accelerated solves batched over the slabs (rcg_dist_solve_batch).
    Strong scaling (total work fixed); the block-Jacobi iteration counts are reported next to the
    single-GPU sequence's (rank 0 runs rcg_seq_run once, untimed)."""
    import torch

    from paper_2203_08498_b200 import api, dist, problems, sequence

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    ctx = api.Context(local_rank)
    cfg = problems.CONFIGS[args.config]
    host = problems.generate(cfg)
    prep = sequence.prepare(ctx, cfg, host, validate=False)
    pairs = sequence.rhs_all(prep)
    kind = "sc" if cfg.method == "sc" else "deflation"
    single = None
    if rank == 0:  # the single-GPU sequence's iteration counts (the global IC(0)), untimed
        seq1 = api.Sequence(ctx, prep.a_orig, "es-sc-iccg" if cfg.method == "sc" else "es-d-iccg", cfg.blocks)
        B = np.stack([b for b, _ in pairs])
        r1 = seq1.run(B, np.zeros_like(B), cfg.eps, cfg.max_iter, "A", cfg.sampler_m, keep_count=cfg.keep, batch=True)
        single = [int(v) for v in r1["iterations"]]
        del seq1, B
    scaled = problems.HostCsr(host.n, host.row_start, host.col_idx, prep.a.values())
    rk = dist.NcclRank(scaled, ctx=ctx, transport=args.slab_transport)
    lo, hi = rk.plan.row_begin, rk.plan.row_end
    n_glob, nnz_glob = host.n, host.nnz
    del prep, host, scaled
    bl_host = [np.ascontiguousarray(bs[lo:hi]) for _, bs in pairs]
    bl_dev = [torch.from_numpy(v).to(dev) for v in bl_host]
    last = {}

    def step(bl):
        out = rk.sequence(bl, cfg.eps, cfg.max_iter, cfg.sampler_m, cfg.keep, kind)
        last.update(out)
        return int(sum(out["iterations"]))

    for _ in range(args.warmup):
        step(bl_dev)
    torch.distributed.barrier()
    ctx.synchronize()
    launches0 = ctx.launches
    iters = 0
    with Clocks(local_rank) as clk:
        ctx.record(0)
        for _ in range(args.steps):
            iters += step(bl_dev)
        ctx.record(1)
        ms = ctx.elapsed_ms(0, 1)
    launches = ctx.launches - launches0
    torch.distributed.barrier()
    ctx.record(2)
    e2e_iters = 0
    for _ in range(args.steps):
        e2e_iters += step(bl_host)  # host right-hand sides and solutions: H2D / D2H inside the calls
    ctx.record(3)
    e2e_ms = ctx.elapsed_ms(2, 3)
    t = torch.tensor([ms, e2e_ms], dtype=torch.float64, device=dev if args.slab_transport == "nccl" else "cpu")
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms, e2e_ms = t.tolist()
    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": round(iters / (ms / 1e3), 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, SURVEY.md 8(d); no network for SuiteSparse)",
        "config": config_dict(cfg, n_glob, nnz_glob, world),
        "iterations_per_step": iters / args.steps,
        "iterations_block_jacobi": [int(v) for v in last["iterations"]],
        "iterations_single_gpu": single,
        "m_bar": int(last["m_bar"]), "m_tilde": int(last["m_tilde"]),
        "time_to_solution_ms_per_rhs": round(ms / args.steps / cfg.n_rhs, 3),
        "driver": "rcg_dist_pcg_solve_sampled + rcg_dist_recycle + rcg_dist_solve_batch over "
                  + ("NCCL" if args.slab_transport == "nccl" else "the host-staged gloo transport (test)")
                  + " (dist.NcclRank)",
        "e2e": {"value": round(e2e_iters / (e2e_ms / 1e3), 2), "unit": UNIT,
                "h2d_bytes_per_step": 8 * (hi - lo) * cfg.n_rhs, "d2h_bytes_per_step": 8 * (hi - lo) * cfg.n_rhs,
                "note": "per rank (rank 0's slab); every rank moves its own rows"},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def measure_row_slabs(api, prep, host, b_scaled, cfg, rank, world, dev, seq_rhs):
    """the same matrix split into `world` row slabs (block-Jacobi IC(0) per GPU, NCCL
    halo exchange + three allreduces per iteration; loopback transport at N = 1), one ICCG solve
    of the step's first right-hand side.  Device time (events on each slab's stream), max over
    ranks.  Block-Jacobi is a weaker preconditioner than the global IC(0): iterations grow with N."""
    import torch

    from paper_2203_08498_b200 import dist, problems as P

    scaled = P.HostCsr(host.n, host.row_start, host.col_idx, prep.a.values())
    kind = "sc" if cfg.method == "sc" else "deflation"
    if world == 1:
        system = dist.LoopbackSystem(scaled, 1)
        solve = lambda x: system.solve(b_scaled, x, cfg.eps, cfg.max_iter)  # noqa: E731
        nloc = host.n
    else:
        rk = dist.NcclRank(scaled, ctx=prep.ctx)
        bl = np.ascontiguousarray(b_scaled[rk.plan.row_begin:rk.plan.row_end])
        solve = lambda x: rk.solve(bl, x, cfg.eps, cfg.max_iter)  # noqa: E731
        nloc = rk.plan.nloc
    solve(np.zeros(nloc))  # warm-up
    rep = solve(np.zeros(nloc))
    # the whole sequence over the slabs: sampled solve 1, distributed recycling, accelerated solves
    bs_all = list(seq_rhs)
    if world == 1:
        run_seq = lambda: system.sequence(bs_all, cfg.eps, cfg.max_iter, cfg.sampler_m, cfg.keep, kind)  # noqa: E731
    else:
        bl_all = [np.ascontiguousarray(v[rk.plan.row_begin:rk.plan.row_end]) for v in bs_all]
        run_seq = lambda: rk.sequence(bl_all, cfg.eps, cfg.max_iter, cfg.sampler_m, cfg.keep, kind)  # noqa: E731
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    seq = run_seq()
    torch.cuda.synchronize()
    seq_s = time.perf_counter() - t0
    t = torch.tensor([rep.wall_time * 1e3, seq_s * 1e3], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms, seq_ms = t.tolist()
    its = int(sum(seq["iterations"]))
    return {"operator": f"block-Jacobi IC(0), {world} row slab(s) at floor(b n / {world}) (ic0_factorize(a, 0, {world}))",
            "transport": "nccl" if world > 1 else "loopback", "n": host.n, "iterations": rep.iterations,
            "converged": bool(rep.converged), "solve_ms": round(ms, 3),
            "ms_per_iteration": round(ms / max(rep.iterations, 1), 4),
            "value": round(rep.iterations / (ms / 1e3), 2), "unit": "iters/s",
            "sequence": {"what": f"rcg_dist_pcg_solve_sampled + rcg_dist_recycle ({kind}, m={cfg.keep}) + "
                                 f"{len(bs_all) - 1} rcg_dist_solve, one pass, wall clock max over ranks",
                         "iterations": [int(v) for v in seq["iterations"]], "m_bar": int(seq["m_bar"]),
                         "m_tilde": int(seq["m_tilde"]), "ms": round(seq_ms, 2),
                         "iters_per_s": round(its / (seq_ms / 1e3), 2)}}


def measure_multicolour(api, problems, sequence, ctx, cfg, host, args, peak):
    """The multicolour-reordered variant (a DIFFERENT operator: IC(0) of P A P^T, SURVEY 8(a)
    a20), reported separately: same sequence, same timing rules."""
    import torch

    m, perm, ncolors = problems.multicolour(host)
    prep = sequence.prepare(ctx, cfg, m, validate=False, new_of_old=perm)
    dev = torch.device("cuda", ctx.device)
    b_dev = torch.from_numpy(np.stack([sequence.rhs(prep, k)[1] for k in range(cfg.n_rhs)])).to(dev)

    def step():
        xs = torch.zeros((cfg.n_rhs, m.n), dtype=torch.float64, device=dev)
        return _sequence(api, ctx, prep, cfg, b_dev, xs)

    for _ in range(max(1, args.warmup)):
        step()
    ctx.synchronize()
    ctxs = _all_contexts(prep)
    for c_ in ctxs:
        c_.synchronize()
        c_.set_profiling(True)
        c_.reset_stats()
    ctx.record(4)
    iters = sum(step() for _ in range(args.steps))
    ctx.record(5)
    ms = ctx.elapsed_ms(4, 5)
    stats = kernel_stats(ctxs)
    for c_ in ctxs:
        c_.set_profiling(False)
    nnz_l = prep.ic.nnz_l
    sweep = {}
    for c in (1, 2, 6, 7):
        tot_ms, cnt, units = stats[c]
        if cnt:
            fixed, per_rhs = algorithmic_bytes(c, m.n, m.nnz, nnz_l, cfg.keep)
            b = (fixed * cnt + per_rhs * units) / cnt
            avg = tot_ms / cnt
            sweep[CLASS_NAMES[c]] = {"avg_us": round(avg * 1e3, 2), "rhs_per_launch": round(units / cnt, 2),
                                     "achieved_gbs": round(b / (avg * 1e-3) / 1e9, 1),
                                     "frac": round(b / (avg * 1e-3) / 1e9 / peak, 4)}
    return {"operator": f"IC(0) of P A P^T, greedy colouring ({ncolors} colours -> {ncolors} sweep levels)",
            "value": round(iters / (ms / 1e3), 2), "unit": UNIT,
            "iterations_per_step": iters / args.steps, "ms_per_step": round(ms / args.steps, 3),
            "time_to_solution_ms_per_rhs": round(ms / args.steps / cfg.n_rhs, 3), "sweeps": sweep}


# solves 2..10: "batch" = one multi-RHS kernel sequence (default); an integer = that many
# concurrent single solves on their own streams
_conc = os.environ.get("RCG_CONCURRENCY", "batch")
PROFILE_TIMED = os.environ.get("RCG_BENCH_PROFILE_TIMED", "1") == "1"
TIMED_CLASSES = (1, 2, 6, 7)  # single / batched forward and backward sweeps
CONCURRENCY = _conc if _conc == "batch" else int(_conc)


def _sequence(api, ctx, prep, cfg, bs, xs, concurrency=None, phases=None):
    """One full sequence; returns its PCG iteration count (phases: optional dict of wall ms)."""
    from paper_2203_08498_b200 import sequence

    n = prep.host.n
    t0 = time.perf_counter()
    sampler = api.SamplerState.method_a(ctx, cfg.sampler_m, cfg.max_iter, n)
    r = api.pcg_solve(ctx, prep.a, bs[0], api.Ic(prep.ic), xs[0], cfg.eps, cfg.max_iter, observer=sampler)
    total = r.iterations
    t1 = time.perf_counter()
    errors = api.harvest_errors(ctx, xs[0], sampler)
    _, _, _, w = api.build_aux_matrix(ctx, prep.a, errors, 1e-3, keep_count=cfg.keep)
    basis = api.Basis(ctx, prep.a, w, "sc" if cfg.method == "sc" else "deflation")
    ctx.synchronize()
    t2 = time.perf_counter()
    reps = sequence.run_accelerated(prep, basis, bs[1:], xs[1:], CONCURRENCY if concurrency is None else concurrency)
    ctx.synchronize()
    t3 = time.perf_counter()
    if phases is not None:
        phases.update(solve1_ms=round((t1 - t0) * 1e3, 2), solve1_iterations=total,
                      rr_basis_ms=round((t2 - t1) * 1e3, 2), accelerated_ms=round((t3 - t2) * 1e3, 2),
                      accelerated_iterations=[r.iterations for r in reps])
    return total + sum(r.iterations for r in reps)


def _all_contexts(prep):
    return [prep.ctx] + list(getattr(prep, "_pool", []) or [])


# --------------------------------------------------------------------------- reference arm
# The reference library itself (oracle/_ref: the reference's src/*.cpp compiled from
# /root/reference by oracle/Makefile) through its own API, on inputs from oracle/inputs.py (the
# shared generator built without librcg_b200.so): this arm never maps the product library.
WINDOW = 3          # iterations per timed window of a step (per thread)


def host_info():
    info = {"nproc": os.cpu_count()}
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                info["model"] = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        info["affinity_cores"] = len(os.sched_getaffinity(0))
    except AttributeError:
        pass
    return info


def repo_libraries_mapped():
    """This repository's shared objects mapped into the process (the reference arm must show
    only oracle/ libraries)."""
    libs = set()
    try:
        for line in open("/proc/self/maps"):
            path = line.split()[-1] if line.strip() else ""
            if path.endswith(".so") and path.startswith(ROOT):
                libs.add(os.path.relpath(path, ROOT))
    except OSError:
        pass
    return sorted(libs)


def _golden_mix(cfg):
    """The oracle's full-run iteration mix for this config (tests/golden, tools/make_goldens.py):
    solve-1 ICCG iterations, accelerated iterations, m_bar, m_tilde -- or None."""
    p = os.path.join(ROOT, "tests", "golden", cfg.name + ".json")
    if not os.path.exists(p):
        return None
    g = json.load(open(p))
    return {"iccg": g["iterations"][0], "accelerated": sum(g["iterations"][1:]), "m_bar": g["m_bar"],
            "m_tilde": g["m_tilde"], "n_rhs": g["n_rhs"], "source": os.path.relpath(p, ROOT),
            "oracle_port_wall_s": g.get("cpu_wall", {})}


class RefSetup:
    """Scaled matrix, IC(0), the right-hand sides and a deflation / SC operator of m~ Ritz
    vectors from REAL sampled errors (a solve-1 window of m~ + 1 ICCG iterations with the method-A
    sampler, harvest_errors, build_aux_matrix) -- all through the reference library."""

    def __init__(self, cfg, n_rhs_needed, timed_rr=True):
        from oracle import Matrix, RefLib, inputs

        t0 = time.perf_counter()
        self.cfg = cfg
        self.ref = ref = RefLib()
        h = inputs.generate(cfg)
        self.n = h.n
        self.nnz = h.nnz
        a_orig = Matrix.of(h)
        m0 = ref.matrix(a_orig)
        va, self.dis = ref.diagonal_scale(m0, h.nnz)
        self.a = Matrix(h.n, h.row_start, h.col_idx, va)
        self.m = ref.matrix(self.a)
        self.f = ref.ic0(self.m)
        self.ic = ref.prec_ic(self.f)
        self.rhs = [self.dis * ref.spmv(m0, x) for x in inputs.solution_streams(cfg, h.n, max(1, n_rhs_needed))]
        del m0
        self.setup_s = time.perf_counter() - t0
        # a real basis: m~ + 1 sampled ICCG iterations -> m~ errors -> Rayleigh-Ritz -> W
        t0 = time.perf_counter()
        self.errors = self.window_errors(cfg.keep + 1)
        self.window_s = time.perf_counter() - t0
        t0 = time.perf_counter()
        _, _, w = ref.build_aux(self.m, self.errors, float("inf"))
        self.rr_k = {len(self.errors): time.perf_counter() - t0}
        w = w[:cfg.keep]
        t0 = time.perf_counter()
        if cfg.method == "sc":
            self.acc = ref.prec_sc(self.ic, self.m, w)
        else:
            self.acc = ref.deflation(self.m, w)
        self.basis_s = time.perf_counter() - t0
        self.m_tilde = len(w)
        del w
        if timed_rr and len(self.errors) >= 2:  # a second, smaller RR: the k and k^2 cost terms
            k2 = len(self.errors) // 2
            t0 = time.perf_counter()
            ref.build_aux(self.m, self.errors[:k2], float("inf"))
            self.rr_k[k2] = time.perf_counter() - t0
        self.errors = None

    def window_errors(self, its):
        ref, cfg = self.ref, self.cfg
        s = ref.sampler_a(max(cfg.sampler_m, 2), cfg.max_iter)
        x = np.zeros(self.n)
        ref.pcg_solve(self.m, self.rhs[0], self.ic, x, cfg.eps, its, sampler=s)
        return ref.harvest_errors(x, s, self.n)

    def rr_seconds(self, k):
        """build_aux_matrix time at k errors from the two timed ones: t(k) = a k + b k^2 (k SpMVs
        and harvest / Ritz-vector streams vs the MGS and Gram column pairs)."""
        pts = sorted(self.rr_k.items())
        if len(pts) < 2:
            (k1, t1), = pts
            return t1 * k / k1
        (k1, t1), (k2, t2) = pts[:2]
        b = (t2 / k2 - t1 / k1) / (k2 - k1)
        a = t1 / k1 - b * k1
        return max(a * k + b * k * k, t2 * k / k2)

    def iccg_window(self, b):
        x = np.zeros(self.n)
        s = self.ref.sampler_a(max(self.cfg.sampler_m, 2), self.cfg.max_iter)  # solve 1 runs the sampler
        t0 = time.perf_counter()
        r = self.ref.pcg_solve(self.m, b, self.ic, x, self.cfg.eps, WINDOW, sampler=s)
        return r.iterations, time.perf_counter() - t0

    def accelerated_window(self, b):
        x = np.zeros(self.n)
        t0 = time.perf_counter()
        if self.cfg.method == "sc":
            r = self.ref.pcg_solve(self.m, b, self.acc, x, self.cfg.eps, WINDOW)
        else:
            r = self.ref.deflated_pcg_solve(self.m, b, self.ic, self.acc, x, self.cfg.eps, WINDOW)
        return r.iterations, time.perf_counter() - t0


def cpu_baseline(cfg):
    """The reference library on ONE host core, a bounded sample of the workload: a solve-1 ICCG
    window with the error sampler (the reference's iteration rate; the accelerated windows, the
    RR step and the sequence extrapolation are the reference arm's, bench.py --impl reference)."""
    from oracle import Matrix, RefLib, inputs

    ref = RefLib()
    h = inputs.generate(cfg)
    m0 = ref.matrix(Matrix.of(h))
    va, dis = ref.diagonal_scale(m0, h.nnz)
    m = ref.matrix(Matrix(h.n, h.row_start, h.col_idx, va))
    ic = ref.prec_ic(ref.ic0(m))
    b = dis * ref.spmv(m0, next(inputs.solution_streams(cfg, h.n, 1)))
    its = 2 * WINDOW
    s = ref.sampler_a(max(cfg.sampler_m, 2), cfg.max_iter)
    x = np.zeros(h.n)
    t0 = time.perf_counter()
    r = ref.pcg_solve(m, b, ic, x, cfg.eps, its, sampler=s)
    secs = time.perf_counter() - t0
    return {"value": round(r.iterations / secs, 3), "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": f"{cfg.name}: {r.iterations} ICCG iterations of solve 1 with the method-A sampler, "
                      f"oracle/_ref (reference sources, -O3 -ffp-contract=off), 1 thread",
            "host": host_info()}


def run_reference(args, rank, world):
    """The reference arm: T host threads, each step runs on every thread an ICCG window (solve 1,
    sampler on) and an accelerated window (SC / deflation with the real m~-vector basis) of
    WINDOW iterations on its own right-hand side; the RR step (build_aux_matrix on real sampled
    errors) and the operator build are timed in setup.  The sequence time is EXTRAPOLATED to the
    oracle's full-run iteration mix (tests/golden/<config>.json; BASELINE.md section 3 /
    SURVEY 8(d) for C3 / C4): T_seq = N_iccg t_iccg + t_RR(m_bar) + t_basis + N_acc t_acc, and
    the whole host runs T sequences at once (the reference is serial), so value = T x iterations
    of a sequence / T_seq."""
    if rank != 0:
        return
    from paper_2203_08498_b200.configs import CONFIGS

    cfg = CONFIGS[args.config]
    threads = max(1, min(os.cpu_count() or 1, args.ref_threads or (os.cpu_count() or 1)))
    mix = _golden_mix(cfg)
    st = RefSetup(cfg, min(threads, cfg.n_rhs))

    def step():
        res = {}

        def work(t):
            b = st.rhs[t % len(st.rhs)]
            i1, s1 = st.iccg_window(b)
            i2, s2 = st.accelerated_window(b)
            res[t] = (i1, s1, i2, s2)

        ths = [threading.Thread(target=work, args=(t,)) for t in range(threads)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        return res

    for _ in range(args.warmup):
        step()
    t_wall = time.perf_counter()
    i1 = s1 = i2 = s2 = 0.0
    for _ in range(args.steps):
        for a, b, c, d in step().values():
            i1, s1, i2, s2 = i1 + a, s1 + b, i2 + c, s2 + d
    wall = time.perf_counter() - t_wall
    t_iccg, t_acc = s1 / i1, s2 / i2
    if mix is None:  # no full-run mix: the windows alone
        n_iccg, n_acc, m_bar, rr = i1, i2, 0, 0.0
        extrap = "none (no tests/golden file for this config): windows only"
    else:
        n_iccg, n_acc, m_bar = mix["iccg"], mix["accelerated"], mix["m_bar"]
        rr = st.rr_seconds(m_bar)
        extrap = (f"extrapolated to the oracle's full-run mix ({mix['source']}): {n_iccg} ICCG + {n_acc} accelerated "
                  f"iterations, RR at m_bar = {m_bar} from build_aux_matrix timed at k = {sorted(st.rr_k)} (t = a k + b k^2)")
    t_seq = n_iccg * t_iccg + rr + st.basis_s + n_acc * t_acc
    iters_seq = n_iccg + n_acc
    value = round(threads * iters_seq / t_seq, 3)
    sample = (f"{cfg.name}: per step {threads} threads x ({WINDOW} ICCG iterations with the sampler + {WINDOW} "
              f"{'SC' if cfg.method == 'sc' else 'deflated'}-ICCG iterations, m~ = {st.m_tilde} Ritz vectors of "
              f"real sampled errors); {extrap}")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(wall / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, SURVEY.md 8(d); no network for SuiteSparse)",
        "config": config_dict(cfg, st.n, st.nnz, world, replicas=args.replicas),
        "time_to_solution_ms_per_rhs": round(t_seq / cfg.n_rhs * 1e3, 3),
        "time_to_solution_ms_per_rhs_throughput": round(t_seq / cfg.n_rhs / threads * 1e3, 3),
        "sequence_model": {"t_iccg_ms": round(t_iccg * 1e3, 3), "t_accelerated_ms": round(t_acc * 1e3, 3),
                           "t_rr_s": round(rr, 3), "t_basis_s": round(st.basis_s, 3), "t_sequence_s": round(t_seq, 3),
                           "rr_timed_s": {str(k): round(v, 3) for k, v in st.rr_k.items()},
                           "iterations": iters_seq, "setup_s": round(st.setup_s, 2),
                           "basis_window_s": round(st.window_s, 2), "mix": mix,
                           "note": "RR / basis timed on one thread while the others idle (favours the reference)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample,
                         "host": host_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "repo_libraries_mapped": repo_libraries_mapped(),
    }), flush=True)


def config_dict(cfg, n, nnz, world=1, replicas=False):
    """The workload's `config` -- identical in both arms for the same N (same_config); N > 1 is the
    row-slab split of the same sequence (or N replicas with --replicas)."""
    par = "1 GPU" if world == 1 else (f"replicas x{world}" if replicas else
                                        f"row slabs x{world} (block-Jacobi IC(0), NCCL halo + allreduce)")
    return {"workload": cfg.name, "n": n, "nnz": nnz, "n_rhs": cfg.n_rhs, "samples": cfg.sampler_m,
            "m_tilde": cfg.keep, "method": cfg.method, "eps": cfg.eps, "rhs": cfg.rhs,
            "l2": "inputs larger than L2 (126 MB): A, the IC(0) factor and W / AW stream from HBM every iteration",
            "parallelism": par}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c3", help="c3 (the largest single-GPU BASELINE config) by default")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--variants", action="store_true",
                    help="also measure the multicolour operator and the row-slab path on this config")
    ap.add_argument("--no-variants", action="store_true", help=argparse.SUPPRESS)  # the default now
    ap.add_argument("--ref-threads", type=int, default=0)
    ap.add_argument("--slab-transport", choices=["nccl", "host"], default="nccl",
                    help=argparse.SUPPRESS)  # test only: the host-staged transport over gloo (ranks may share a GPU)
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: N independent single-GPU sequences (weak scaling) instead of row slabs")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch

        local_rank %= max(1, torch.cuda.device_count())  # test runs may put several ranks on one GPU
        torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group("gloo" if args.slab_transport == "host" else "nccl")
    try:
        if world > 1 and not args.replicas:
            run_slabs(args, rank, world, local_rank)
        else:
            run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch

            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
