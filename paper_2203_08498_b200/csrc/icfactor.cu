// icfactor.cu -- IC(0) factorisation on the device: rcg_ic0_factorize_device.
//
// Everything runs on the device.  PATTERN: the L pattern of each block (count / scan / fill), its
// row-wise transpose U (stable radix sort of the L entries by column: ascending rows within a U
// row, as build_transpose), the DAG levels (Kahn layering, one frontier kernel per level) and
// the level schedules (stable sort by level, warp-padded levels, scans) -- the same arrays
// build_schedule makes on the host.  NUMERIC: the reference's sorted row merge,
// src/ic_preconditioner.cpp:12-70, in the forward schedule's level order, sync-free like the
// sweeps: a lane owns row i, waits until the pivots d_j of all its L
// columns are published (the pivot is its row's ready flag: d starts as a NaN sentinel and a row
// writes its L values before its pivot, fenced), then computes
//     l_ij = (a_ij - sum_{p<j} (l_ip d_p) l_jp) / d_j        (merge order of the reference)
//     d_i  = a_ii (1 + shift) - sum_p (l_ip l_ip) d_p
// with the reference's separate roundings, so the factor is bitwise rcg_ic0_factorize's.  A
// non-positive pivot flags the attempt (the row still publishes, so no dependant hangs) and the
// host re-runs the numeric pass with the next shift of the reference ladder (0 -> 0.01 -> x2,
// 20 retries, ic_preconditioner.cpp:109-120).  U (the row-wise transpose) and the two schedule
// value copies are gathered on the device.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <numeric>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "internal.cuh"
#include "kernels.cuh"

namespace rcg {

struct FactorArgs {
    const int32_t* perm;   // forward schedule (level-sorted rows, -1 = padding)
    int32_t npos;
    const int32_t* lrs;    // natural-order L pattern
    const int32_t* lcol;
    double* lval;          // out
    const double* ava;     // A values (device matrix)
    const int32_t* asrc;   // A position of every L entry
    const int32_t* adiag;  // A position of every diagonal (-1: none -> 0.0, as the reference)
    double* d;             // pivots: sentinel in, published out
    double shift;
    int* fail;
    int* tickets;          // [0] tile ticket, [1] exit count, [3] watchdog
};

__global__ void __launch_bounds__(128) k_ic_factor(FactorArgs a) {
    const int lane = threadIdx.x & 31;
    const int ntiles = (a.npos + 31) / 32;
    while (true) {
        int tile = 0;
        if (lane == 0) tile = atomicAdd(&a.tickets[0], 1);
        tile = __shfl_sync(0xffffffffu, tile, 0);
        if (tile >= ntiles) break;
        const int pos = tile * 32 + lane;
        const int32_t i = pos < a.npos ? __ldg(a.perm + pos) : -1;
        if (i >= 0) {
            const int32_t first = __ldg(a.lrs + i), last = __ldg(a.lrs + i + 1);
            // wait for the pivots of every L column (chunks of 8 polled together)
            unsigned spins = 0;
            for (int32_t e0 = first; e0 < last; e0 += 8) {
                const int cnt = min(8, last - e0);
                int32_t col[8];
                double dv[8];
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (j < cnt) {
                        col[j] = __ldg(a.lcol + e0 + j);
                        dv[j] = ld_relaxed(a.d + col[j]);
                    }
                while (true) {
                    bool miss = false;
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        if (j < cnt && is_sentinel(dv[j])) {
                            miss = true;
                            dv[j] = ld_relaxed(a.d + col[j]);
                        }
                    if (!miss) break;
                    if (++spins == (1u << 24)) {  // bounded: a schedule fault is an error, never a hang
                        atomicExch(&a.tickets[3], 1);
                        break;
                    }
                }
            }
            __threadfence();  // acquire: the parents' L rows were written before their pivots
            for (int32_t e = first; e < last; ++e) {
                const int32_t j = __ldg(a.lcol + e);
                double sum = __ldg(a.ava + __ldg(a.asrc + e));
                int32_t pi = first, pj = __ldg(a.lrs + j);
                const int32_t pj_end = __ldg(a.lrs + j + 1);
                while (pi < e && pj < pj_end) {
                    const int32_t cpi = __ldg(a.lcol + pi), cpj = __ldg(a.lcol + pj);
                    if (cpi == cpj) {
                        sum = __dsub_rn(sum, __dmul_rn(__dmul_rn(a.lval[pi], __ldcg(a.d + cpi)), __ldcg(a.lval + pj)));
                        ++pi;
                        ++pj;
                    } else if (cpi < cpj) {
                        ++pi;
                    } else {
                        ++pj;
                    }
                }
                a.lval[e] = __ddiv_rn(sum, __ldcg(a.d + j));
            }
            const int32_t kd = __ldg(a.adiag + i);
            const double diag = kd >= 0 ? __ldg(a.ava + kd) : 0.0;
            double piv = __dmul_rn(diag, __dadd_rn(1.0, a.shift));
            for (int32_t e = first; e < last; ++e) {
                const double l = a.lval[e];
                piv = __dsub_rn(piv, __dmul_rn(__dmul_rn(l, l), __ldcg(a.d + __ldg(a.lcol + e))));
            }
            if (piv <= 0.0) {  // the attempt is discarded; publish anyway so no dependant waits forever
                atomicExch(a.fail, 1);
                piv = 1.0;
            }
            __threadfence();  // release: this row's L values before its pivot
            st_relaxed(a.d + i, publishable(piv));
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

__global__ void k_gather(const double* __restrict__ src, const int32_t* __restrict__ idx, double* __restrict__ dst,
                         int64_t n) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        dst[t] = src[idx[t]];
}

__global__ void k_gather_i(const int32_t* __restrict__ src, const int32_t* __restrict__ idx, int32_t* __restrict__ dst,
                           int64_t n) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        dst[t] = src[idx[t]];
}

__global__ void k_scatter(const double* __restrict__ src, const int32_t* __restrict__ idx, double* __restrict__ dst,
                          int64_t n) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        dst[idx[t]] = src[t];
}

template <class T>
static T* to_dev(rcg_ctx* ctx, const std::vector<T>& h) {
    T* p = static_cast<T*>(dev_alloc_bytes(sizeof(T) * std::max<size_t>(h.size(), 1)));
    if (!h.empty()) RCG_CK(cudaMemcpyAsync(p, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice, ctx->stream));
    return p;
}

// ------------------------------------------------------------------ pattern work on the device
static int grid_for(const rcg_ctx* ctx, int64_t n) {
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, ctx->num_sms * 8)));
}

#define RCG_GRID_LOOP(i, n) for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

__device__ __forceinline__ int32_t block_lo(const int32_t* bounds, int nb, int32_t i) {
    int lo = 0, hi = nb;  // bounds[0..nb]: largest b with bounds[b] <= i
    while (hi - lo > 1) {
        const int mid = (lo + hi) / 2;
        if (bounds[mid] <= i) lo = mid; else hi = mid;
    }
    return bounds[lo];
}

// L entries of row i: lo <= j < i up to the diagonal (ic_preconditioner.cpp:29-46)
__global__ void k_l_count(const int32_t* __restrict__ rs, const int32_t* __restrict__ ci, int32_t n,
                          const int32_t* __restrict__ bounds, int nb, int32_t* __restrict__ cnt,
                          int32_t* __restrict__ adiag) {
    RCG_GRID_LOOP(t, n) {
        const int32_t i = static_cast<int32_t>(t);
        const int32_t lo = block_lo(bounds, nb, i);
        int32_t c = 0, dg = -1;
        for (int32_t k = rs[i]; k < rs[i + 1]; ++k) {
            const int32_t j = ci[k];
            if (j >= i) {
                if (j == i) dg = k;
                break;
            }
            if (j >= lo) ++c;
        }
        cnt[i] = c;
        adiag[i] = dg;
    }
}

__global__ void k_l_fill(const int32_t* __restrict__ rs, const int32_t* __restrict__ ci, int32_t n,
                         const int32_t* __restrict__ bounds, int nb, const int32_t* __restrict__ lrs,
                         int32_t* __restrict__ lcol, int32_t* __restrict__ lrow, int32_t* __restrict__ asrc) {
    RCG_GRID_LOOP(t, n) {
        const int32_t i = static_cast<int32_t>(t);
        const int32_t lo = block_lo(bounds, nb, i);
        int32_t e = lrs[i];
        for (int32_t k = rs[i]; k < rs[i + 1]; ++k) {
            const int32_t j = ci[k];
            if (j >= i) break;
            if (j < lo) continue;
            lcol[e] = j;
            lrow[e] = i;
            asrc[e] = k;
            ++e;
        }
    }
}

__global__ void k_iota(int32_t* v, int64_t n, int32_t base, int32_t step) {
    RCG_GRID_LOOP(t, n) v[t] = base + step * static_cast<int32_t>(t);
}

__global__ void k_hist(const int32_t* __restrict__ key, int64_t n, int32_t* __restrict__ cnt) {
    RCG_GRID_LOOP(t, n) atomicAdd(cnt + key[t], 1);
}

// U (row-wise transpose, ascending rows within a U row): from the stable sort of L by column
__global__ void k_u_fill(const int32_t* __restrict__ order, const int32_t* __restrict__ lrow, int64_t nnzl,
                         int32_t* __restrict__ ucol, int32_t* __restrict__ l2u) {
    RCG_GRID_LOOP(t, nnzl) {
        const int32_t e = order[t];
        ucol[t] = lrow[e];
        l2u[e] = static_cast<int32_t>(t);
    }
}

__global__ void k_row_len(const int32_t* __restrict__ rs, int32_t n, int32_t* __restrict__ len) {
    RCG_GRID_LOOP(t, n) len[t] = rs[t + 1] - rs[t];
}

// Kahn layering: level of a row = 1 + max level of its parents; a row joins the next frontier
// when its last parent (the deepest, frontiers being processed in level order) is processed
__global__ void k_frontier0(const int32_t* __restrict__ indeg, int32_t n, int32_t* __restrict__ frontier,
                            int32_t* __restrict__ fcount, int32_t* __restrict__ level) {
    RCG_GRID_LOOP(t, n) {
        if (indeg[t] == 0) {
            level[t] = 0;
            frontier[atomicAdd(fcount, 1)] = static_cast<int32_t>(t);
        }
    }
}

__global__ void k_peel(const int32_t* __restrict__ frontier, const int32_t* __restrict__ fsize,
                       const int32_t* __restrict__ crs, const int32_t* __restrict__ child, int32_t* __restrict__ indeg,
                       int32_t* __restrict__ level, int32_t lev, int32_t* __restrict__ next, int32_t* __restrict__ ncount) {
    const int32_t m = *fsize;
    for (int32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < m; t += gridDim.x * blockDim.x) {
        const int32_t i = frontier[t];
        for (int32_t e = crs[i]; e < crs[i + 1]; ++e) {
            const int32_t k = child[e];
            if (atomicSub(indeg + k, 1) == 1) {
                level[k] = lev;
                next[atomicAdd(ncount, 1)] = k;
            }
        }
    }
}

// level-sorted positions: each level starts on a warp boundary (-1 padding), rows of a level in
// the order of the stable sort (ascending rows forward, descending backward: build_schedule's)
__global__ void k_place(const int32_t* __restrict__ lev_sorted, const int32_t* __restrict__ rows_sorted, int32_t n,
                        const int32_t* __restrict__ ustart, const int32_t* __restrict__ pstart, int32_t* __restrict__ perm) {
    RCG_GRID_LOOP(t, n) {
        const int32_t l = lev_sorted[t];
        perm[pstart[l] + (static_cast<int32_t>(t) - ustart[l])] = rows_sorted[t];
    }
}

__global__ void k_pos_len(const int32_t* __restrict__ perm, int32_t npos, const int32_t* __restrict__ rs,
                          int32_t* __restrict__ plen) {
    RCG_GRID_LOOP(t, npos) {
        const int32_t i = perm[t];
        plen[t] = i >= 0 ? rs[i + 1] - rs[i] : 0;
    }
}

__global__ void k_pos_fill(const int32_t* __restrict__ perm, int32_t npos, const int32_t* __restrict__ prs,
                           const int32_t* __restrict__ rs, const int32_t* __restrict__ col, int32_t* __restrict__ pcol,
                           int32_t* __restrict__ pidx) {
    RCG_GRID_LOOP(t, npos) {
        const int32_t i = perm[t];
        if (i < 0) continue;
        int32_t q = prs[t];
        for (int32_t e = rs[i]; e < rs[i + 1]; ++e, ++q) {
            pcol[q] = col[e];
            pidx[q] = e;
        }
    }
}

// device temporaries released at scope exit (fenced cache: safe while kernels still run)
struct DevBag {
    std::vector<void*> ptrs;
    template <class T>
    T* get(int64_t count) {
        void* p = dev_alloc_bytes(sizeof(T) * static_cast<size_t>(std::max<int64_t>(count, 1)));
        ptrs.push_back(p);
        return static_cast<T*>(p);
    }
    ~DevBag() {
        for (void* p : ptrs) dev_free(p);
    }
};

static void exclusive_sum(rcg_ctx* ctx, DevBag& bag, const int32_t* in, int32_t* out, int64_t n) {
    size_t tb = 0;
    RCG_CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, static_cast<int>(n), ctx->stream));
    void* tmp = bag.get<unsigned char>(static_cast<int64_t>(tb));
    RCG_CK(cub::DeviceScan::ExclusiveSum(tmp, tb, in, out, static_cast<int>(n), ctx->stream));
}

static void stable_sort_pairs(rcg_ctx* ctx, DevBag& bag, const int32_t* kin, int32_t* kout, const int32_t* vin,
                              int32_t* vout, int64_t n, int bits) {
    size_t tb = 0;
    RCG_CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin, kout, vin, vout, static_cast<int>(n), 0, bits, ctx->stream));
    void* tmp = bag.get<unsigned char>(static_cast<int64_t>(tb));
    RCG_CK(cub::DeviceRadixSort::SortPairs(tmp, tb, kin, kout, vin, vout, static_cast<int>(n), 0, bits, ctx->stream));
}

static int bits_for(int64_t v) {
    int b = 1;
    while (b < 31 && (int64_t(1) << b) <= v) ++b;
    return b;
}

// levels of the DAG whose parents of row i are its own row entries (rs/col) and whose children
// are the transpose's (crs/child); returns the level count
static int32_t levels_device(rcg_ctx* ctx, DevBag& bag, int32_t n, const int32_t* rs, const int32_t* crs,
                             const int32_t* child, int32_t* level) {
    int32_t* indeg = bag.get<int32_t>(n);
    int32_t* fa = bag.get<int32_t>(n);
    int32_t* fb = bag.get<int32_t>(n);
    int32_t* cnt = bag.get<int32_t>(2);
    const int g = grid_for(ctx, n);
    k_row_len<<<g, 256, 0, ctx->stream>>>(rs, n, indeg);
    RCG_CK(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * 2, ctx->stream));
    k_frontier0<<<g, 256, 0, ctx->stream>>>(indeg, n, fa, cnt, level);
    int32_t* hcnt = reinterpret_cast<int32_t*>(ctx->host_pinned + 1536);
    RCG_CK(cudaMemcpyAsync(hcnt, cnt, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
    RCG_CK(cudaStreamSynchronize(ctx->stream));
    int32_t fsize = hcnt[0], lev = 0, cur = 0;
    int32_t* fr[2] = {fa, fb};
    while (fsize > 0) {
        ++lev;
        RCG_CK(cudaMemsetAsync(cnt + (cur ^ 1), 0, sizeof(int32_t), ctx->stream));
        k_peel<<<grid_for(ctx, fsize), 256, 0, ctx->stream>>>(fr[cur], cnt + cur, crs, child, indeg, level, lev,
                                                            fr[cur ^ 1], cnt + (cur ^ 1));
        RCG_CK(cudaMemcpyAsync(hcnt, cnt + (cur ^ 1), sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
        RCG_CK(cudaStreamSynchronize(ctx->stream));
        fsize = hcnt[0];
        cur ^= 1;
    }
    return lev;  // levels 0..lev-1
}

// perm / prs / pcol / pidx of one sweep from the levels (descending: rows n-1..0 within a level)
static void schedule_device(rcg_ctx* ctx, DevBag& bag, int32_t n, const int32_t* level, int32_t nlev,
                            const int32_t* rs, const int32_t* col, int64_t nnz, bool descending, int32_t*& perm,
                            int32_t*& prs, int32_t*& pcol, int32_t*& pidx, int32_t& npos,
                            std::vector<int32_t>& lptr) {
    const int g = grid_for(ctx, n);
    int32_t* rows = bag.get<int32_t>(n);
    int32_t* rows_s = bag.get<int32_t>(n);
    int32_t* lev_s = bag.get<int32_t>(n);
    k_iota<<<g, 256, 0, ctx->stream>>>(rows, n, descending ? n - 1 : 0, descending ? -1 : 1);
    // rows in build_schedule's visiting order, so the stable sort keeps it inside each level
    const int32_t* lev_in = level;
    if (descending) {  // key order must follow the row order of `rows`
        int32_t* lv = bag.get<int32_t>(n);
        k_gather_i<<<g, 256, 0, ctx->stream>>>(level, rows, lv, n);
        lev_in = lv;
    }
    stable_sort_pairs(ctx, bag, lev_in, lev_s, rows, rows_s, n, bits_for(nlev));
    int32_t* lcnt = bag.get<int32_t>(nlev);
    RCG_CK(cudaMemsetAsync(lcnt, 0, sizeof(int32_t) * nlev, ctx->stream));
    k_hist<<<g, 256, 0, ctx->stream>>>(level, n, lcnt);
    std::vector<int32_t> hc(nlev), us(nlev), ps(nlev);
    RCG_CK(cudaMemcpyAsync(hc.data(), lcnt, sizeof(int32_t) * nlev, cudaMemcpyDeviceToHost, ctx->stream));
    RCG_CK(cudaStreamSynchronize(ctx->stream));
    int64_t u = 0, pp = 0;
    for (int32_t l = 0; l < nlev; ++l) {
        us[l] = static_cast<int32_t>(u);
        ps[l] = static_cast<int32_t>(pp);
        u += hc[l];
        pp += round_up(hc[l], 32);
    }
    require(pp < (int64_t(1) << 31), "IC schedule: padded length exceeds int32");
    npos = static_cast<int32_t>(pp);
    lptr.assign(ps.begin(), ps.end());
    lptr.push_back(npos);
    int32_t* d_us = bag.get<int32_t>(nlev);
    int32_t* d_ps = bag.get<int32_t>(nlev);
    RCG_CK(cudaMemcpyAsync(d_us, us.data(), sizeof(int32_t) * nlev, cudaMemcpyHostToDevice, ctx->stream));
    RCG_CK(cudaMemcpyAsync(d_ps, ps.data(), sizeof(int32_t) * nlev, cudaMemcpyHostToDevice, ctx->stream));
    perm = static_cast<int32_t*>(dev_alloc_bytes(sizeof(int32_t) * std::max<int64_t>(npos, 1)));
    RCG_CK(cudaMemsetAsync(perm, 0xff, sizeof(int32_t) * npos, ctx->stream));  // -1 padding
    k_place<<<g, 256, 0, ctx->stream>>>(lev_s, rows_s, n, d_us, d_ps, perm);
    int32_t* plen = bag.get<int32_t>(static_cast<int64_t>(npos) + 1);
    RCG_CK(cudaMemsetAsync(plen + npos, 0, sizeof(int32_t), ctx->stream));
    k_pos_len<<<grid_for(ctx, npos), 256, 0, ctx->stream>>>(perm, npos, rs, plen);
    prs = static_cast<int32_t*>(dev_alloc_bytes(sizeof(int32_t) * (static_cast<int64_t>(npos) + 1)));
    exclusive_sum(ctx, bag, plen, prs, static_cast<int64_t>(npos) + 1);
    // + kCsrPad: the level sweep's tile engine widens bulk ranges to 16 bytes (k_level_sweep)
    pcol = static_cast<int32_t*>(dev_alloc_bytes(sizeof(int32_t) * (std::max<int64_t>(nnz, 1) + kCsrPad)));
    pidx = bag.get<int32_t>(nnz);
    k_pos_fill<<<grid_for(ctx, npos), 256, 0, ctx->stream>>>(perm, npos, prs, rs, col, pcol, pidx);
}

static void factorize_device(rcg_ctx* ctx, const rcg_matrix* A, double shift, int num_blocks, rcg_ic* f) {
    const int32_t n = A->n;
    static const bool timing = std::getenv("RCG_FACTOR_TIMING") != nullptr;
    auto tp = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
        if (!timing) return;
        cudaStreamSynchronize(ctx->stream);
        const auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[ic0_device] %-28s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(t - tp).count());
        tp = t;
    };
    DevBag bag;
    f->n = n;
    f->host_image = false;
    f->h_bounds.resize(static_cast<size_t>(num_blocks) + 1);
    for (int b = 0; b <= num_blocks; ++b)
        f->h_bounds[b] = static_cast<int32_t>((static_cast<int64_t>(b) * n) / num_blocks);
    if (n == 0) {
        f->host_image = true;
        f->h_lrs.assign(1, 0);
        f->h_urs.assign(1, 0);
        return;
    }
    const int g = grid_for(ctx, n);
    int32_t* bounds = bag.get<int32_t>(num_blocks + 1);
    RCG_CK(cudaMemcpyAsync(bounds, f->h_bounds.data(), sizeof(int32_t) * (num_blocks + 1), cudaMemcpyHostToDevice,
                           ctx->stream));
    // ---- L pattern
    int32_t* cnt = bag.get<int32_t>(static_cast<int64_t>(n) + 1);
    int32_t* adiag = bag.get<int32_t>(n);
    RCG_CK(cudaMemsetAsync(cnt + n, 0, sizeof(int32_t), ctx->stream));
    k_l_count<<<g, 256, 0, ctx->stream>>>(A->rs, A->ci, n, bounds, num_blocks, cnt, adiag);
    int32_t* lrs = bag.get<int32_t>(static_cast<int64_t>(n) + 1);
    exclusive_sum(ctx, bag, cnt, lrs, static_cast<int64_t>(n) + 1);
    int32_t nnzl32 = 0;
    RCG_CK(cudaMemcpyAsync(ctx->host_pinned + 1540, lrs + n, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
    RCG_CK(cudaStreamSynchronize(ctx->stream));
    std::memcpy(&nnzl32, ctx->host_pinned + 1540, sizeof(int32_t));
    const int64_t nnzl = nnzl32;
    f->nnz_l = nnzl;
    int32_t* lcol = bag.get<int32_t>(nnzl);
    int32_t* lrow = bag.get<int32_t>(nnzl);
    int32_t* asrc = bag.get<int32_t>(nnzl);
    k_l_fill<<<g, 256, 0, ctx->stream>>>(A->rs, A->ci, n, bounds, num_blocks, lrs, lcol, lrow, asrc);
    mark("L pattern");
    // ---- U pattern: stable sort of L entries by column keeps ascending rows (build_transpose)
    const int ge = grid_for(ctx, nnzl);
    int32_t* ucnt = bag.get<int32_t>(static_cast<int64_t>(n) + 1);
    RCG_CK(cudaMemsetAsync(ucnt, 0, sizeof(int32_t) * (static_cast<int64_t>(n) + 1), ctx->stream));
    k_hist<<<ge, 256, 0, ctx->stream>>>(lcol, nnzl, ucnt);
    int32_t* urs = bag.get<int32_t>(static_cast<int64_t>(n) + 1);
    exclusive_sum(ctx, bag, ucnt, urs, static_cast<int64_t>(n) + 1);
    int32_t* ucol = bag.get<int32_t>(nnzl);
    int32_t* l2u = bag.get<int32_t>(nnzl);
    if (nnzl > 0) {
        int32_t* idx = bag.get<int32_t>(nnzl);
        int32_t* keys = bag.get<int32_t>(nnzl);
        int32_t* order = bag.get<int32_t>(nnzl);
        k_iota<<<ge, 256, 0, ctx->stream>>>(idx, nnzl, 0, 1);
        stable_sort_pairs(ctx, bag, lcol, keys, idx, order, nnzl, bits_for(n));
        k_u_fill<<<ge, 256, 0, ctx->stream>>>(order, lrow, nnzl, ucol, l2u);
    }
    mark("U pattern");
    // ---- levels and schedules (forward on L, backward on U)
    int32_t* level = bag.get<int32_t>(n);
    f->fwd_levels = levels_device(ctx, bag, n, lrs, urs, ucol, level);
    mark("forward levels");
    int32_t *fidx = nullptr, *bidx = nullptr;
    schedule_device(ctx, bag, n, level, f->fwd_levels, lrs, lcol, nnzl, false, f->f_perm, f->f_prs, f->f_col, fidx,
                    f->f_npos, f->h_lptr[0]);
    mark("forward schedule");
    f->bwd_levels = levels_device(ctx, bag, n, urs, lrs, lcol, level);
    mark("backward levels");
    schedule_device(ctx, bag, n, level, f->bwd_levels, urs, ucol, nnzl, true, f->b_perm, f->b_prs, f->b_col, bidx,
                    f->b_npos, f->h_lptr[1]);
    mark("backward schedule");
    // ---- numeric (device) with the reference shift ladder
    double* lval = bag.get<double>(nnzl);
    double* uval = bag.get<double>(nnzl);
    f->d = dev_alloc(std::max(n, 1));
    int* flags = bag.get<int>(8);  // [0] fail, [4..7] tickets
    const int grid = std::max(1, std::min((f->f_npos + 127) / 128, ctx->num_sms * 2));
    double s = shift;
    bool ok = false;
    const int retries = 20;
    for (int attempt = 0; attempt <= retries && !ok; ++attempt) {
        RCG_CK(cudaMemsetAsync(flags, 0, sizeof(int) * 8, ctx->stream));
        launch_fill_bits(ctx, f->d, n, kSentinelBits);
        FactorArgs fa{};
        fa.perm = f->f_perm;
        fa.npos = f->f_npos;
        fa.lrs = lrs;
        fa.lcol = lcol;
        fa.lval = lval;
        fa.ava = A->va;
        fa.asrc = asrc;
        fa.adiag = adiag;
        fa.d = f->d;
        fa.shift = s;
        fa.fail = flags;
        fa.tickets = flags + 4;
        k_ic_factor<<<grid, 128, 0, ctx->stream>>>(fa);
        RCG_LAUNCHED(ctx);
        int* h = reinterpret_cast<int*>(ctx->host_pinned + 1544);
        RCG_CK(cudaMemcpyAsync(h, flags, sizeof(int) * 8, cudaMemcpyDeviceToHost, ctx->stream));
        RCG_CK(cudaStreamSynchronize(ctx->stream));
        if (h[4 + 3]) throw Error(RCG_E_CUDA, "ic0_factorize_device: dependency wait exceeded its bound");
        ok = h[0] == 0;
        f->shift = s;
        if (!ok) s = (s == 0.0) ? 0.01 : 2.0 * s;
    }
    if (!ok) {
        char buf[160];
        std::snprintf(buf, sizeof buf,
                      "IC breakdown: no positive-pivot factorization after %d shift retries (last shift %f)", retries,
                      s);
        throw Error(RCG_E_BREAKDOWN, buf);
    }
    mark("numeric");
    f->f_val = dev_alloc(std::max<int64_t>(nnzl, 1) + kCsrPad);
    f->b_val = dev_alloc(std::max<int64_t>(nnzl, 1) + kCsrPad);
    if (nnzl > 0) {
        k_scatter<<<ge, kStreamThreads, 0, ctx->stream>>>(lval, l2u, uval, nnzl);
        k_gather<<<ge, kStreamThreads, 0, ctx->stream>>>(lval, fidx, f->f_val, nnzl);
        k_gather<<<ge, kStreamThreads, 0, ctx->stream>>>(uval, bidx, f->b_val, nnzl);
        RCG_CK(cudaGetLastError());
    }
    RCG_CK(cudaStreamSynchronize(ctx->stream));
    mark("value gathers");
}

// The host image (IcFactor's natural-order L, D, U) of a device-built factor, rebuilt on demand
// from the level schedules: a schedule position holds row perm[pos]'s entries in natural order.
void ensure_host_image(const rcg_ic* cf) {
    auto* f = const_cast<rcg_ic*>(cf);
    if (f->host_image) return;
    const int32_t n = f->n;
    const int64_t nnzl = f->nnz_l;
    auto unpack = [&](const int32_t* dperm, const int32_t* dprs, const int32_t* dcol, const double* dval, int32_t npos,
                      std::vector<int32_t>& rs, std::vector<int32_t>& col, std::vector<double>& val) {
        std::vector<int32_t> perm(npos), prs(static_cast<size_t>(npos) + 1), pcol(nnzl);
        std::vector<double> pval(nnzl);
        RCG_CK(cudaMemcpy(perm.data(), dperm, sizeof(int32_t) * npos, cudaMemcpyDeviceToHost));
        RCG_CK(cudaMemcpy(prs.data(), dprs, sizeof(int32_t) * prs.size(), cudaMemcpyDeviceToHost));
        if (nnzl) {
            RCG_CK(cudaMemcpy(pcol.data(), dcol, sizeof(int32_t) * nnzl, cudaMemcpyDeviceToHost));
            RCG_CK(cudaMemcpy(pval.data(), dval, sizeof(double) * nnzl, cudaMemcpyDeviceToHost));
        }
        rs.assign(static_cast<size_t>(n) + 1, 0);
        std::vector<int32_t> posof(n, -1);
        for (int32_t p = 0; p < npos; ++p)
            if (perm[p] >= 0) {
                posof[perm[p]] = p;
                rs[perm[p] + 1] = prs[p + 1] - prs[p];
            }
        std::partial_sum(rs.begin(), rs.end(), rs.begin());
        col.resize(nnzl);
        val.resize(nnzl);
        for (int32_t i = 0; i < n; ++i) {
            const int32_t p = posof[i];
            std::copy(pcol.begin() + prs[p], pcol.begin() + prs[p + 1], col.begin() + rs[i]);
            std::copy(pval.begin() + prs[p], pval.begin() + prs[p + 1], val.begin() + rs[i]);
        }
    };
    unpack(f->f_perm, f->f_prs, f->f_col, f->f_val, f->f_npos, f->h_lrs, f->h_lcol, f->h_lval);
    unpack(f->b_perm, f->b_prs, f->b_col, f->b_val, f->b_npos, f->h_urs, f->h_ucol, f->h_uval);
    f->h_d.resize(n);
    RCG_CK(cudaMemcpy(f->h_d.data(), f->d, sizeof(double) * n, cudaMemcpyDeviceToHost));
    f->host_image = true;
}

}  // namespace rcg

using namespace rcg;

extern "C" int rcg_ic0_factorize_device(rcg_ctx* ctx, const rcg_matrix* a, double shift, int num_blocks,
                                        rcg_ic** out) {
    return guard([&] {
        require(ctx && a && out, "rcg_ic0_factorize_device: null argument");
        *out = nullptr;
        if (num_blocks < 1 || num_blocks > std::max<int32_t>(a->n, 1))
            throw Error(RCG_E_INVALID, "ic0_factorize: num_blocks must be in [1, n]");
        if (shift < 0.0) throw Error(RCG_E_INVALID, "ic0_factorize: shift must be >= 0");
        auto* f = new rcg_ic();
        try {
            factorize_device(ctx, a, shift, num_blocks, f);
        } catch (...) {
            rcg_ic_destroy(f);
            throw;
        }
        *out = f;
    });
}
