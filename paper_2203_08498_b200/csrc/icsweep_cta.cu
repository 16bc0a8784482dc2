// icsweep_cta.cu -- IC(0) sweeps of SMALL factors (C1: 32K rows, 94 levels of ~350 rows) in ONE
// CTA: the levels run in order with a CTA barrier between them, so a level costs a barrier plus
// one row's dependent loads (L1 / L2 hits) instead of an inter-SM publish -> observe round trip
// per level; the whole factor (1.1 MB on C1) stays in L2.  The grid-wide sync-free sweep pays
// ~1 us per level there (94 levels: ~90 us per sweep); one CTA needs a few hundred cycles.
//
// Operator identity: each row is k_sweep's (the reference loop, src/ic_preconditioner.cpp:
// 130-143: forward s = r_i, s -= l_ik y_k in stored order; backward s = y_i / d_i, s -= u_ik z_k),
// so the output is bitwise; the (r, z) partials are per 32-position tile (levels are padded to
// warp multiples, so warp w of the CTA holds exactly tile (lstart + 32 w) / 32 of the schedule)
// and are reduced in k_sweep's tile -> group -> total order, so rho, beta and every iterate are
// bitwise identical whichever sweep kernel runs (tests/test_gpu_sweep_variants.py).
// Roofline: latency-bound (levels x (barrier + one row)); its bytes are k_sweep's.
#include <algorithm>
#include <cstdlib>

#include "internal.cuh"
#include "kernels.cuh"

namespace rcg {

constexpr int kCtaSweepThreads = 1024;

template <bool BWD>
__global__ void __launch_bounds__(kCtaSweepThreads, 1) k_sweep_cta(SweepArgs a, const int32_t* __restrict__ lptr,
                                                                   int nlev) {
    if (a.st->done) return;
    const int tid = threadIdx.x, lane = tid & 31;
    for (int l = 0; l < nlev; ++l) {
        const int32_t l0 = __ldg(lptr + l), l1 = __ldg(lptr + l + 1);
        for (int32_t base = l0; base < l1; base += kCtaSweepThreads) {
            const int32_t pos = base + tid;
            double contrib = 0.0;
            const int32_t row = pos < l1 ? __ldg(a.perm + pos) : -1;
            if (row >= 0) {
                double s = BWD ? __ddiv_rn(a.in[row], __ldg(a.d + row)) : a.in[row];
                const int32_t b = __ldg(a.prs + pos), e = __ldg(a.prs + pos + 1);
                for (int32_t k0 = b; k0 < e; k0 += 8) {  // loads of eight parents in flight, then in order
                    const int m = min(8, e - k0);
                    double lv[8], dv[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        if (j < m) {
                            lv[j] = __ldg(a.pval + k0 + j);
                            dv[j] = __ldcg(a.out + __ldg(a.pcol + k0 + j));  // earlier levels: final
                        }
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        if (j < m) s = fsub_mul(s, lv[j], dv[j]);
                }
                if (BWD && a.r) contrib = __dmul_rn(a.r[row], s);
                a.out[row] = publishable(s);
            }
            if (BWD && a.r && base + (tid & ~31) < l1) {  // this warp's 32 positions are one tile
                const double v = warp_sum(contrib);
                if (lane == 0) a.partials[(base + (tid & ~31)) / 32] = v;
            }
        }
        __syncthreads();  // the level's values (and tile partials) are visible to the next level
    }
    if (!(BWD && a.r)) return;
    // k_sweep's tile_reduce order: groups of kGroup tiles (lane-strided, warp-summed), then the
    // groups the same way; one warp per group, warp 0 for the total
    const int ntiles = (a.npos + 31) / 32;
    const int ngroups = (ntiles + kGroup - 1) / kGroup;
    const int wid = tid >> 5;
    for (int g = wid; g < ngroups; g += kCtaSweepThreads / 32) {
        const int gsize = min(kGroup, ntiles - g * kGroup);
        double gs = 0.0;
        for (int q = lane; q < gsize; q += 32) gs = __dadd_rn(gs, a.partials[g * kGroup + q]);
        gs = warp_sum(gs);
        if (lane == 0) a.gpart[g] = gs;
    }
    __syncthreads();
    if (wid == 0) {
        double ts = 0.0;
        for (int q = lane; q < ngroups; q += 32) ts = __dadd_rn(ts, a.gpart[q]);
        ts = warp_sum(ts);
        if (lane == 0) {
            DevState* st = a.st;
            const double rho = a.add_sc ? ts + st->scal[2] : ts;
            st->rho = rho;
            if (rho <= 0.0) {
                st->done = kBroken;
                st->status = kBrkRz;
            }
            st->beta = st->iter > 1 ? rho / st->rho_prev : 0.0;
        }
    }
}

// small factors: one CTA when the schedule is short and its widest level fits the CTA a few
// times over (RCG_SWEEP_CTA_N: largest n, default 65536; mode 0 forces the grid-wide sweep)
bool launch_cta_sweep(rcg_ctx* ctx, const rcg_ic* f, bool backward, SweepArgs& s) {
    static const int64_t max_n = [] {
        const char* e = std::getenv("RCG_SWEEP_CTA_N");
        return e ? std::atoll(e) : 65536LL;
    }();
    if (ctx->sweep_cluster != 2 && ctx->sweep_cluster != 6) return false;
    if (ctx->sweep_cluster == 2 && f->n > max_n) return false;
    const int nlev = backward ? f->bwd_levels : f->fwd_levels;
    const int32_t* dl = f->d_lptr[backward ? 1 : 0];
    if (!dl || nlev <= 0) return false;
    KTimer t(ctx, backward ? 2 : 1);
    if (backward)
        k_sweep_cta<true><<<1, kCtaSweepThreads, 0, ctx->stream>>>(s, dl, nlev);
    else
        k_sweep_cta<false><<<1, kCtaSweepThreads, 0, ctx->stream>>>(s, dl, nlev);
    RCG_LAUNCHED(ctx);
    return true;
}

}  // namespace rcg
