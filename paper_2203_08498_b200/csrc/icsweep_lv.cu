// icsweep_lv.cu -- IC(0) sweeps one LEVEL per launch, for factors whose levels are very wide (the
// multicolour orderings: 1M+ rows per colour on C2-C4).
//
// On very wide levels the sync-free sweep (icsweep.cu) is bound by each warp's chain of
// dependent loads, not by the level chain (C4 multicolour: 2 levels of 67M rows at 19-22 % of
// HBM).  Here every level is one launch of the CSR tile engine of the SpMV
// (spmv_pipe.cuh: warp-per-32-row tile, row bounds prefetched, the tile's entries brought into
// shared memory by cp.async.bulk a stage ahead) over the level's slice of the level-sorted
// schedule -- its rows are contiguous positions, its entries a contiguous range -- so the level
// streams like an SpMV.  Parents belong to earlier levels (earlier launches), so no row polls:
// stream order is the synchronisation.  Cost: one launch gap per level.
//
// Operator identity: each row is the reference loop (src/ic_preconditioner.cpp:130-143) --
// forward s = r_i, s -= l_ik y_k in stored order; backward s = y_i / d_i, s -= u_ik z_k -- so the
// output is bitwise k_sweep's; the (r, z) partials are formed per 32-position tile and reduced in
// k_sweep's tile -> group -> total order (k_level_groups, k_level_total), so rho is bitwise too.
// Roofline: the same algorithmic bytes as the sweep (12 nnz_L + 24..40 n per sweep), HBM-bound
// per level; reported in the same kernel classes (1 forward, 2 backward).
#include <algorithm>
#include <cstdlib>

#include "internal.cuh"
#include "kernels.cuh"
#include "spmv_pipe.cuh"

namespace rcg {

constexpr int kLevelCap = 256;  // staged entries per warp tile (wider tiles read global memory)

struct LevelArgs {
    const int32_t* prs;    // schedule row starts (position-indexed, absolute entry offsets)
    const int32_t* pcol;
    const double* pval;
    const int32_t* perm;
    const double* in;
    const double* d;       // backward
    const double* r;       // backward: (r, z) partials when non-null
    double* out;
    double* partials;      // per 32-position tile of the whole schedule
    const DevState* st;
    int32_t lstart, width; // the level: positions [lstart, lstart + width)
};

template <bool BWD>
__global__ void __launch_bounds__(kSpmvThreads) k_level_sweep(LevelArgs a) {
    if (a.st->done) return;
    const int lane = threadIdx.x & 31;
    csr_tiles(a.prs + a.lstart, a.pcol, a.pval, a.width, kLevelCap,
              [&](int32_t r0, int32_t b, int32_t e, const double* vsrc, const int32_t* csrc, int32_t off) {
                  const int32_t pos = a.lstart + r0 + lane;
                  const int32_t row = r0 + lane < a.width ? __ldg(a.perm + pos) : -1;
                  double contrib = 0.0;
                  if (row >= 0) {
                      double s = BWD ? __ddiv_rn(__ldg(a.in + row), __ldg(a.d + row)) : __ldg(a.in + row);
                      for (int32_t k = b; k < e; k += 8) {
                          const int m = min(8, e - k);
                          double av[8], dv[8];
                          int32_t cc[8];
#pragma unroll
                          for (int j = 0; j < 8; ++j)
                              if (j < m) {
                                  av[j] = vsrc[k - off + j];
                                  cc[j] = csrc[k - off + j];
                              }
#pragma unroll
                          for (int j = 0; j < 8; ++j)
                              if (j < m) dv[j] = __ldg(a.out + cc[j]);   // earlier levels: final
#pragma unroll
                          for (int j = 0; j < 8; ++j)
                              if (j < m) s = fsub_mul(s, av[j], dv[j]);
                      }
                      s = publishable(s);
                      a.out[row] = s;
                      if (BWD && a.r) contrib = __dmul_rn(__ldg(a.r + row), s);
                  }
                  if (BWD && a.r) {
                      const double v = warp_sum(contrib);
                      if (lane == 0) a.partials[(a.lstart + r0) / 32] = v;
                  }
              });
}

// rho = (r, z) from the per-tile partials in k_sweep's tile_reduce order: k_level_groups sums each
// group of kGroup tiles (lane-strided, then warp-summed; one warp per group), k_level_total the
// groups the same way and runs the scalar update of src/pcg.cpp:65-71 (+ the SC term)
__global__ void __launch_bounds__(256) k_level_groups(const double* __restrict__ partials, double* __restrict__ gpart,
                                                      int ntiles, const DevState* st) {
    if (st->done) return;
    const int lane = threadIdx.x & 31;
    const int ngroups = (ntiles + kGroup - 1) / kGroup;
    const int g = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (g >= ngroups) return;
    const int gsize = min(kGroup, ntiles - g * kGroup);
    double gs = 0.0;
    for (int q = lane; q < gsize; q += 32) gs = __dadd_rn(gs, partials[g * kGroup + q]);
    gs = warp_sum(gs);
    if (lane == 0) gpart[g] = gs;
}

__global__ void k_level_total(const double* __restrict__ gpart, int ntiles, DevState* st, int add_sc) {
    if (st->done) return;
    const int lane = threadIdx.x & 31;
    const int ngroups = (ntiles + kGroup - 1) / kGroup;
    double ts = 0.0;
    for (int q = lane; q < ngroups; q += 32) ts = __dadd_rn(ts, gpart[q]);
    ts = warp_sum(ts);
    if (lane == 0) {
        const double rho = add_sc ? ts + st->scal[2] : ts;
        st->rho = rho;
        if (rho <= 0.0) {
            st->done = kBroken;
            st->status = kBrkRz;
        }
        st->beta = st->iter > 1 ? rho / st->rho_prev : 0.0;
    }
}

// Level launches when the average level is wide (>= RCG_SWEEP_LV_ROWS rows, default 600K) and
// ctx->sweep_cluster is the default (2), or always (4).  Measured (B200, forward / backward):
// wins on 1M+ rows per level -- C2 multicolour 66.7 -> 56.3 / 68.3 -> 65.1 us, C3 multicolour
// 1.03 -> 0.99 / 1.17 -> 1.10 ms, C4 multicolour 6.19 -> 2.84 / 6.61 -> 3.36 ms (43-46 % of HBM)
// -- and loses where the launch gap (~5-8 us per level) dominates: C4 natural (1,534 levels of
// 87K rows) 7.95 -> 12.1 ms, C5 (30 levels of 133K) 286 -> 404 us, C5 multicolour (12 of 333K).
bool launch_level_sweep(rcg_ctx* ctx, const rcg_ic* f, bool backward, SweepArgs& s) {
    static const int64_t min_rows = [] {
        const char* e = std::getenv("RCG_SWEEP_LV_ROWS");
        return e ? std::atoll(e) : 600000LL;
    }();
    const int mode = ctx->sweep_cluster;
    if (mode != 2 && mode != 4) return false;
    const std::vector<int32_t>& lp = f->h_lptr[backward ? 1 : 0];
    const int nlev = backward ? f->bwd_levels : f->fwd_levels;
    if (static_cast<int>(lp.size()) != nlev + 1 || nlev <= 0) return false;
    if (mode == 2 && (s.npos / nlev) < min_rows) return false;
    static bool attr = false;
    if (!attr) {
        const int bytes = static_cast<int>(pipe_smem_bytes(kLevelCap));
        RCG_CK(cudaFuncSetAttribute(k_level_sweep<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
        RCG_CK(cudaFuncSetAttribute(k_level_sweep<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
        attr = true;
    }
    LevelArgs a{};
    a.prs = s.prs;
    a.pcol = s.pcol;
    a.pval = s.pval;
    a.perm = s.perm;
    a.in = s.in;
    a.d = s.d;
    a.r = backward ? s.r : nullptr;
    a.out = s.out;
    a.partials = s.partials;
    a.st = s.st;
    const size_t smem = pipe_smem_bytes(kLevelCap);
    KTimer tm(ctx, backward ? 2 : 1);
    for (int l = 0; l < nlev; ++l) {
        a.lstart = lp[l];
        a.width = lp[l + 1] - lp[l];
        const int tiles = (a.width + 31) / 32;
        const int grid = std::max(1, std::min((tiles + kPipeWarps - 1) / kPipeWarps, ctx->num_sms * ctx->spmv_bps));
        if (backward)
            k_level_sweep<true><<<grid, kSpmvThreads, smem, ctx->stream>>>(a);
        else
            k_level_sweep<false><<<grid, kSpmvThreads, smem, ctx->stream>>>(a);
        RCG_LAUNCHED(ctx);
    }
    if (backward && s.r) {
        const int ntiles = (s.npos + 31) / 32;
        const int ngroups = (ntiles + kGroup - 1) / kGroup;
        k_level_groups<<<(ngroups + 7) / 8, 256, 0, ctx->stream>>>(s.partials, s.gpart, ntiles, s.st);
        RCG_LAUNCHED(ctx);
        k_level_total<<<1, 32, 0, ctx->stream>>>(s.gpart, ntiles, s.st, s.add_sc);
        RCG_LAUNCHED(ctx);
    }
    return true;
}

}  // namespace rcg
