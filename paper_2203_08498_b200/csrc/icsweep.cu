// icsweep.cu -- IC(0) preconditioner on the device (K3-K5): the reference factor is uploaded
// unchanged and applied by two sync-free, level-ordered triangular sweeps.
//
// Operator identity.  Each row i is computed exactly as src/ic_preconditioner.cpp:130-143 does:
// forward  s = r_i;  s -= l_ik * y_k  (stored entry order);  y_i = s
// backward s = y_i / d_i;  s -= u_ik * z_k  (stored entry order);  z_i = s
// with separate multiply/subtract roundings.  Only the ORDER IN WHICH ROWS ARE VISITED changes
// (topological level order instead of 0..n-1 / n-1..0), and every row still sees final values
// of its dependencies, so the result is bitwise equal to the reference ic_apply.
//
// Schedule.  Host side, rows are sorted by DAG level (level = 1 + max level of the columns the
// row reads; ties by row index) and the factor rows are copied into that order so a warp's rows
// are contiguous in HBM.  Device side, a CTA takes the next 128-row tile from an atomic ticket
// (so every tile it can wait on is already owned by a running CTA -- no deadlock), prefetches
// its rows' entries, and spins on each dependency with a relaxed gpu-scope load until the value
// differs from a NaN sentinel; a finished row is published with one relaxed 64-bit store (the
// value is its own ready flag, no fence needed).  Buffers are refilled with the sentinel at the
// start of each solve; the consumer of each buffer resets it in passing.
// Roofline: 12 nnz_L + 28 n bytes per sweep (entries, perm, row starts, in, out); the natural
// ordering's level count bounds it by dependency latency on C1-C3.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>

#include "internal.cuh"
#include "kernels.cuh"

namespace rcg {

constexpr int kDepChunk = 8;
constexpr int kDepChunkWide = 16;  // factors of more than kDepChunk entries per row (27-point: 13)

constexpr int kTile = 32;  // positions per ticket: one warp

// (r, z) partial of one warp tile -> groups of kGroup tiles -> total, fixed order (run-to-run
// deterministic).  Returns true in the one warp that owns the final total (*tot, all lanes).
__device__ __forceinline__ bool tile_reduce(double v, int tile, int ntiles, SweepArgs& a, double* tot) {
    const int lane = threadIdx.x & 31;
    v = warp_sum(v);
    const int g = tile / kGroup;
    const int ngroups = (ntiles + kGroup - 1) / kGroup;
    const int gsize = min(kGroup, ntiles - g * kGroup);
    int last_group = 0;
    if (lane == 0) {
        a.partials[tile] = v;
        __threadfence();
        last_group = atomicAdd(&a.gcount[g], 1u) == static_cast<unsigned>(gsize) - 1u;
    }
    if (!__shfl_sync(0xffffffffu, last_group, 0)) return false;
    __threadfence();
    double gs = 0.0;
    for (int q = lane; q < gsize; q += 32) gs = __dadd_rn(gs, __ldcg(a.partials + g * kGroup + q));
    gs = warp_sum(gs);
    int last = 0;
    if (lane == 0) {
        a.gpart[g] = gs;
        a.gcount[g] = 0u;
        __threadfence();
        last = atomicAdd(reinterpret_cast<unsigned int*>(&a.tickets[2]), 1u) == static_cast<unsigned>(ngroups) - 1u;
    }
    if (!__shfl_sync(0xffffffffu, last, 0)) return false;
    __threadfence();
    double ts = 0.0;
    for (int q = lane; q < ngroups; q += 32) ts = __dadd_rn(ts, __ldcg(a.gpart + q));
    ts = warp_sum(ts);
    if (lane == 0) a.tickets[2] = 0;
    *tot = ts;
    return true;
}

// Persistent sweep: a grid of at most (SMs x blocks_per_sm) CTAs whose warps each pull 32-row
// tiles of the level-sorted order from an atomic ticket until none is left (tickets are
// monotone, so every row a warp can wait on belongs to a running warp: no deadlock).  Bounding
// the resident CTAs bounds how many future-level rows spin at once.
template <bool BWD, int CH>
__global__ void __launch_bounds__(kSweepThreads, CH > 8 ? 4 : 8) k_sweep(SweepArgs a) {
    if (a.st->done) return;
    const int lane = threadIdx.x & 31;
    const int ntiles = (a.npos + kTile - 1) / kTile;
    while (true) {
        int tile = 0;
        if (lane == 0) tile = atomicAdd(&a.tickets[0], 1);
        tile = __shfl_sync(0xffffffffu, tile, 0);
        if (tile >= ntiles) break;
        const int pos = tile * kTile + lane;
        double contrib = 0.0;
        const int32_t row = pos < a.npos ? __ldg(a.perm + pos) : -1;  // -1: level padding
        if (row >= 0) {
            const int32_t beg = __ldg(a.prs + pos), end = __ldg(a.prs + pos + 1);
            double s;
            if (BWD) {
                s = __ddiv_rn(a.in[row], __ldg(a.d + row));
            } else {
                s = a.in[row];
            }
            // Entries in chunks of CH: all parents of a chunk are loaded together and the missing
            // ones re-polled together (one L2 round trip after the last parent is published;
            // consuming them in order as they arrive measured slower: C3 fwd 3.5 -> 4.2 ms).  A row that fits one chunk has
            // every parent in flight from the start: in the BACKWARD sweep the first entry
            // (column i + 1) is the parent published last, so with several chunks every later
            // chunk was a dependent L2 round trip on the level's critical path (CH = 16 for
            // factors of more than 8 entries per row).  On the last chunk the row is published
            // from inside the wait loop, so a lane never waits for slower lanes of its warp.
            unsigned spins = 0;
            for (int32_t e0 = beg;; e0 += CH) {
                const int cnt = min(CH, end - e0);
                const bool last = e0 + CH >= end;
                int32_t col[CH];
                double val[CH], dep[CH];
#pragma unroll
                for (int j = 0; j < CH; ++j)
                    if (j < cnt) {
                        col[j] = __ldg(a.pcol + e0 + j);
                        val[j] = __ldg(a.pval + e0 + j);
                    }
#pragma unroll
                for (int j = 0; j < CH; ++j)
                    if (j < cnt) dep[j] = ld_relaxed(a.out + col[j]);
                int used = 0;
                while (true) {
                    bool missing = false;
#pragma unroll
                    for (int j = 0; j < CH; ++j)
                        if (j < cnt && is_sentinel(dep[j])) missing = true;
                    if (!missing) {
#pragma unroll
                        for (int j = 0; j < CH; ++j)
                            if (j < cnt) s = fsub_mul(s, val[j], dep[j]);
                        used = cnt;
                    }
                    if (used >= cnt) {
                        if (last) st_relaxed(a.out + row, publishable(s));
                        break;
                    }
                    if (a.backoff_ns) __nanosleep(a.backoff_ns);
#pragma unroll
                    for (int j = 0; j < CH; ++j)
                        if (j >= used && j < cnt && is_sentinel(dep[j])) dep[j] = ld_relaxed(a.out + col[j]);
                    if (++spins == (1u << 24)) {  // bounded: a schedule fault is an error, never a hang
                        atomicExch(&a.tickets[3], 1);
#pragma unroll
                        for (int j = 0; j < CH; ++j)
                            if (j < cnt && is_sentinel(dep[j])) dep[j] = 0.0;
                    }
                }
                if (last) break;
            }
            if (BWD && a.r) contrib = __dmul_rn(a.r[row], s);
        }
        if (BWD && a.r) {
            double tot;
            if (tile_reduce(contrib, tile, ntiles, a, &tot) && lane == 0) {
                // (r, z) complete: breakdown test and beta of src/pcg.cpp:65-71.  With subspace
                // correction z = z_ic + W u, so (r, z) = (r, z_ic) + (W^T r) . u (st->scal[2])
                DevState* st = a.st;
                const double rho = a.add_sc ? tot + st->scal[2] : tot;
                st->rho = rho;
                if (rho <= 0.0) {
                    st->done = kBroken;
                    st->status = kBrkRz;
                }
                st->beta = st->iter > 1 ? rho / st->rho_prev : 0.0;
            }
        }
    }
    if (lane == 0) {
        __threadfence();
        if (atomicAdd(&a.tickets[1], 1) == static_cast<int>(gridDim.x * (blockDim.x / 32)) - 1) {
            a.tickets[0] = 0;
            a.tickets[1] = 0;
        }
    }
}

void sweep_prepare_kernels() {
    static bool done = false;
    if (done) return;
    set_carveout(reinterpret_cast<const void*>(k_sweep<false, kDepChunk>));
    set_carveout(reinterpret_cast<const void*>(k_sweep<true, kDepChunk>));
    set_carveout(reinterpret_cast<const void*>(k_sweep<false, kDepChunkWide>));
    set_carveout(reinterpret_cast<const void*>(k_sweep<true, kDepChunkWide>));
    done = true;
}

SweepArgs sweep_args(rcg_ctx* ctx, const rcg_ic* f, bool backward) {
    SweepArgs a{};
    a.perm = backward ? f->b_perm : f->f_perm;
    a.prs = backward ? f->b_prs : f->f_prs;
    a.pcol = backward ? f->b_col : f->f_col;
    a.pval = backward ? f->b_val : f->f_val;
    a.d = f->d;
    a.n = f->n;
    a.npos = backward ? f->b_npos : f->f_npos;
    a.tickets = ctx->ws.tickets + (backward ? 4 : 0);
    a.partials = ctx->ws.partials;
    a.gpart = ctx->ws.gpart;
    a.gcount = ctx->ws.gcount;
    a.st = ctx->ws.st;
    return a;
}

// Resident CTAs per SM (RCG_SWEEP_BPS overrides).  Rows in flight beyond what the current
// levels can use only spin and add L2 polling traffic, and too few leave a wide level's rows
// waiting on their load chains.  Measured on B200 with 32-row warp tiles:
//   rows/level   5.5K (C2)  9.4K (C3, 27-pt)  87K (C4)  262K (C2 multicolour)
//   best         2          2                 3         8
// (C3's backward sweep: 5.5 ms at 1 CTA per SM with two dependency chunks, 3.7 ms at 2 with every
// parent in flight -- kDepChunkWide; 4.9 ms at 3)
int sweep_ctas_per_sm(const rcg_ic* f, bool backward, int64_t npos) {
    const int levels = backward ? f->bwd_levels : f->fwd_levels;
    const int64_t rows_per_level = levels > 0 ? npos / levels : npos;
    if (rows_per_level >= 200000) return 8;
    if (rows_per_level >= 32768) return 3;
    const double entries_per_row = f->n > 0 ? static_cast<double>(f->nnz_l) / f->n : 0.0;
    (void)entries_per_row;  // (round 1: 1 CTA per SM for long backward rows -- the wide chunk removed the reason)
    return 2;
}

void launch_sweep(rcg_ctx* ctx, const rcg_ic* f, bool backward, SweepArgs& a) {
    if (f->n == 0) return;
    if (launch_level_sweep(ctx, f, backward, a)) return;  // wide levels: one launch per level (icsweep_lv.cu)
    const int ntiles = (a.npos + kSweepThreads - 1) / kSweepThreads;
    static const int bps_bwd_env = std::getenv("RCG_SWEEP_BPS_BWD") ? std::atoi(std::getenv("RCG_SWEEP_BPS_BWD")) : 0;  // A/B
    int bps = ctx->sweep_bps > 0 ? ctx->sweep_bps : sweep_ctas_per_sm(f, backward, a.npos);
    if (backward && bps_bwd_env > 0) bps = bps_bwd_env;
    const int grid = std::max(1, std::min(ntiles, ctx->num_sms * bps));
    a.backoff_ns = ctx->sweep_backoff_ns;
    KTimer t(ctx, backward ? 2 : 1);
    // RCG_SWEEP_CH=8 / 16 forces the dependency chunk (A/B); default: wide for long backward rows
    static const int ch_env = std::getenv("RCG_SWEEP_CH") ? std::atoi(std::getenv("RCG_SWEEP_CH")) : 0;
    const double entries_per_row = static_cast<double>(f->nnz_l) / f->n;
    const bool wide = ch_env ? ch_env > kDepChunk : (backward && entries_per_row > kDepChunk);
    auto go = [&](auto kern) { kern<<<grid, kSweepThreads, 0, ctx->stream>>>(a); };
    if (backward)
        wide ? go(k_sweep<true, kDepChunkWide>) : go(k_sweep<true, kDepChunk>);
    else
        wide ? go(k_sweep<false, kDepChunkWide>) : go(k_sweep<false, kDepChunk>);
    RCG_LAUNCHED(ctx);
}

// raises if any sweep hit the bounded dependency wait (clears the flags)
void check_sweep_watchdog(rcg_ctx* ctx) {
    if (!ctx->ws.tickets) return;
    int h[8];
    RCG_CK(cudaMemcpyAsync(h, ctx->ws.tickets, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    RCG_CK(cudaStreamSynchronize(ctx->stream));
    if (h[3] || h[7]) {
        RCG_CK(cudaMemsetAsync(ctx->ws.tickets, 0, 16 * sizeof(int), ctx->stream));
        RCG_CK(cudaStreamSynchronize(ctx->stream));
        throw Error(RCG_E_CUDA, "IC sweep: dependency wait timed out (schedule fault)");
    }
}

// workspace needed by the sweeps of an n-row factor
int64_t sweep_tiles(const rcg_ic* f) {
    const int64_t npos = std::max<int64_t>(std::max(f->f_npos, f->b_npos), f->n);
    return (npos + kTile - 1) / kTile;
}

static void ensure_sweep_ws(rcg_ctx* ctx, const rcg_ic* f, int k, int64_t max_iter, int pending) {
    const int32_t n = f->n;
    const int64_t ntiles = sweep_tiles(f);
    const int64_t ngroups = (ntiles + kGroup - 1) / kGroup;
    const int64_t red = std::max<int64_t>(ntiles, static_cast<int64_t>(kMaxRed) * ctx->num_sms * 8);
    ensure_workspace(ctx, n, k, max_iter, red, ngroups, pending);
}

void ic_apply_dev(rcg_ctx* ctx, const rcg_ic* f, const double* r, double* z) {
    ensure_sweep_ws(ctx, f, 1, 1, 1);
    Workspace& w = ctx->ws;
    RCG_CK(cudaMemsetAsync(w.st, 0, sizeof(DevState), ctx->stream));
    launch_fill_bits(ctx, w.ybuf, f->n, kSentinelBits);
    launch_fill_bits(ctx, z, f->n, kSentinelBits);
    SweepArgs fw = sweep_args(ctx, f, false);
    fw.in = r;
    fw.out = w.ybuf;
    launch_sweep(ctx, f, false, fw);
    SweepArgs bw = sweep_args(ctx, f, true);
    bw.in = w.ybuf;
    bw.out = z;
    launch_sweep(ctx, f, true, bw);
}

// ------------------------------------------------------------------ host: schedule + upload
template <class T>
static T* upload(rcg_ctx* ctx, const std::vector<T>& h) {
    void* p = nullptr;
    // + kCsrPad elements: the level sweep's tile engine widens bulk ranges to 16 bytes
    RCG_CK(cudaMalloc(&p, sizeof(T) * (std::max<size_t>(h.size(), 1) + kCsrPad)));
    if (!h.empty()) RCG_CK(cudaMemcpyAsync(p, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice, ctx->stream));
    return static_cast<T*>(p);
}

// Level-sorted copy of a row-wise triangular factor.  `descending` walks rows n-1..0 (U).
// `val` may be empty: then pval stays empty and only pidx (the source entry of every schedule
// entry) is produced, for a device-side gather of values computed on the GPU.
int32_t build_schedule(int32_t n, const std::vector<int32_t>& rs, const std::vector<int32_t>& col,
                              const std::vector<double>& val, bool descending, std::vector<int32_t>& perm,
                              std::vector<int32_t>& prs, std::vector<int32_t>& pcol, std::vector<double>& pval,
                              int32_t& npos, std::vector<int32_t>* pidx = nullptr,
                              std::vector<int32_t>* lptr = nullptr) {
    std::vector<int32_t> level(n, 0);
    int32_t nlev = 0;
    for (int32_t t = 0; t < n; ++t) {
        const int32_t i = descending ? n - 1 - t : t;
        int32_t lv = 0;
        for (int32_t p = rs[i]; p < rs[i + 1]; ++p) lv = std::max(lv, level[col[p]] + 1);
        level[i] = lv;
        nlev = std::max(nlev, lv + 1);
    }
    // each level starts on a warp boundary (padding positions hold perm = -1), so no warp mixes
    // rows of two levels and a level's rows never wait on lanes of the next one
    std::vector<int64_t> start(static_cast<size_t>(nlev) + 1, 0);
    for (int32_t i = 0; i < n; ++i) start[level[i] + 1]++;
    for (int32_t l = 0; l < nlev; ++l) start[l + 1] = start[l] + round_up(start[l + 1], 32);
    const int64_t total = start[nlev];
    require(total < (1LL << 31), "IC schedule: padded length exceeds int32");
    npos = static_cast<int32_t>(total);
    if (lptr) lptr->assign(start.begin(), start.end());
    perm.assign(total, -1);
    for (int32_t t = 0; t < n; ++t) {
        const int32_t i = descending ? n - 1 - t : t;
        perm[start[level[i]]++] = i;
    }
    prs.assign(static_cast<size_t>(total) + 1, 0);
    for (int64_t pos = 0; pos < total; ++pos) {
        const int32_t i = perm[pos];
        prs[pos + 1] = prs[pos] + (i >= 0 ? rs[i + 1] - rs[i] : 0);
    }
    pcol.resize(col.size());
    pval.resize(val.size());
    if (pidx) pidx->resize(col.size());
    for (int64_t pos = 0; pos < total; ++pos) {
        const int32_t i = perm[pos];
        if (i < 0) continue;
        std::copy(col.begin() + rs[i], col.begin() + rs[i + 1], pcol.begin() + prs[pos]);
        if (!val.empty()) std::copy(val.begin() + rs[i], val.begin() + rs[i + 1], pval.begin() + prs[pos]);
        if (pidx)
            for (int32_t p = rs[i]; p < rs[i + 1]; ++p) (*pidx)[prs[pos] + (p - rs[i])] = p;
    }
    return nlev;
}

static void finish_ic(rcg_ctx* ctx, rcg_ic* f) {
    std::vector<int32_t> perm, prs, pcol;
    std::vector<double> pval;
    f->fwd_levels = build_schedule(f->n, f->h_lrs, f->h_lcol, f->h_lval, false, perm, prs, pcol, pval, f->f_npos,
                                   nullptr, &f->h_lptr[0]);
    f->f_perm = upload(ctx, perm);
    f->f_prs = upload(ctx, prs);
    f->f_col = upload(ctx, pcol);
    f->f_val = upload(ctx, pval);
    RCG_CK(cudaStreamSynchronize(ctx->stream));
    f->bwd_levels = build_schedule(f->n, f->h_urs, f->h_ucol, f->h_uval, true, perm, prs, pcol, pval, f->b_npos,
                                   nullptr, &f->h_lptr[1]);
    f->b_perm = upload(ctx, perm);
    f->b_prs = upload(ctx, prs);
    f->b_col = upload(ctx, pcol);
    f->b_val = upload(ctx, pval);
    f->d = upload(ctx, f->h_d);
    RCG_CK(cudaStreamSynchronize(ctx->stream));
}

}  // namespace rcg

using namespace rcg;

extern "C" {

// ic0_factorize from host CSR arrays: the device factorisation (icfactor.cu) over a temporary
// device copy of the matrix -- the same factor bit for bit (tests/test_gpu_icfactor.py)
int rcg_ic0_factorize(rcg_ctx* ctx, int32_t n, const int32_t* row_start, const int32_t* col_idx,
                      const double* values, double shift, int num_blocks, rcg_ic** out) {
    return guard([&] {
        require(ctx && out, "rcg_ic0_factorize: null argument");
        *out = nullptr;
        if (num_blocks < 1 || num_blocks > std::max<int32_t>(n, 1))
            throw Error(RCG_E_INVALID, "ic0_factorize: num_blocks must be in [1, n]");
        if (shift < 0.0) throw Error(RCG_E_INVALID, "ic0_factorize: shift must be >= 0");
        rcg_matrix* a = nullptr;
        ck(rcg_matrix_create(ctx, n, row_start, col_idx, values, 0, &a));
        const int rc = rcg_ic0_factorize_device(ctx, a, shift, num_blocks, out);
        rcg_matrix_destroy(a);
        ck(rc);
    });
}

int rcg_ic_create(rcg_ctx* ctx, int32_t n, int num_blocks, const int32_t* block_bounds,
                  const int32_t* l_row_start, const int32_t* l_col, const double* l_val,
                  const double* d, const int32_t* u_row_start, const int32_t* u_col,
                  const double* u_val, double shift_used, rcg_ic** out) {
    return guard([&] {
        *out = nullptr;
        require(n >= 0 && num_blocks >= 1, "rcg_ic_create: bad dimensions");
        auto* f = new rcg_ic();
        try {
            f->n = n;
            f->shift = shift_used;
            f->h_bounds.assign(block_bounds, block_bounds + num_blocks + 1);
            f->h_lrs.assign(l_row_start, l_row_start + n + 1);
            f->nnz_l = f->h_lrs[n];
            f->h_lcol.assign(l_col, l_col + f->nnz_l);
            f->h_lval.assign(l_val, l_val + f->nnz_l);
            f->h_d.assign(d, d + n);
            f->h_urs.assign(u_row_start, u_row_start + n + 1);
            require(f->h_urs[n] == f->nnz_l, "rcg_ic_create: L and U entry counts differ");
            f->h_ucol.assign(u_col, u_col + f->nnz_l);
            f->h_uval.assign(u_val, u_val + f->nnz_l);
            for (int64_t p = 0; p < f->nnz_l; ++p)
                require(f->h_lcol[p] >= 0 && f->h_lcol[p] < n && f->h_ucol[p] >= 0 && f->h_ucol[p] < n,
                        "rcg_ic_create: factor column out of range");
            for (int32_t i = 0; i < n; ++i) {
                for (int32_t p = f->h_lrs[i]; p < f->h_lrs[i + 1]; ++p)
                    require(f->h_lcol[p] < i, "rcg_ic_create: L entry on or above the diagonal");
                for (int32_t p = f->h_urs[i]; p < f->h_urs[i + 1]; ++p)
                    require(f->h_ucol[p] > i, "rcg_ic_create: U entry on or below the diagonal");
            }
            finish_ic(ctx, f);
        } catch (...) {
            rcg_ic_destroy(f);
            throw;
        }
        *out = f;
    });
}

void rcg_ic_destroy(rcg_ic* f) {
    if (!f) return;
    for (void* p : {(void*)f->f_perm, (void*)f->f_prs, (void*)f->f_col, (void*)f->f_val, (void*)f->b_perm,
                    (void*)f->b_prs, (void*)f->b_col, (void*)f->b_val, (void*)f->d})
        dev_free(p);
    delete f;
}

int rcg_ic_info(const rcg_ic* f, int64_t* nnz_l, double* shift_used, int32_t* fwd_levels, int32_t* bwd_levels) {
    return guard([&] {
        if (nnz_l) *nnz_l = f->nnz_l;
        if (shift_used) *shift_used = f->shift;
        if (fwd_levels) *fwd_levels = f->fwd_levels;
        if (bwd_levels) *bwd_levels = f->bwd_levels;
    });
}

int rcg_ic_export(const rcg_ic* f, int32_t* block_bounds, int32_t* l_row_start, int32_t* l_col,
                  double* l_val, double* d, int32_t* u_row_start, int32_t* u_col, double* u_val) {
    return guard([&] {
        ensure_host_image(f);
        auto cp = [](auto* dst, const auto& v) {
            if (dst && !v.empty()) std::memcpy(dst, v.data(), sizeof(v[0]) * v.size());
        };
        cp(block_bounds, f->h_bounds);
        cp(l_row_start, f->h_lrs);
        cp(l_col, f->h_lcol);
        cp(l_val, f->h_lval);
        cp(d, f->h_d);
        cp(u_row_start, f->h_urs);
        cp(u_col, f->h_ucol);
        cp(u_val, f->h_uval);
    });
}

int rcg_ic_apply(rcg_ctx* ctx, const rcg_ic* f, const double* r, double* z) {
    return guard([&] {
        Staged rs, zs;
        stage_in(ctx, r, f->n, rs);
        stage_out_begin(ctx, z, f->n, zs);
        ic_apply_dev(ctx, f, rs.dev, zs.dev);
        stage_out_end(ctx, z, f->n, zs);
        RCG_CK(cudaStreamSynchronize(ctx->stream));
        check_sweep_watchdog(ctx);
    });
}

}  // extern "C"
