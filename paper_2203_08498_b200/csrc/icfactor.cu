// icfactor.cu -- IC(0) factorisation on the device: rcg_ic0_factorize_device.
//
// Split: the PATTERN work (L pattern of each block, its transpose, the two level schedules) runs
// on the host from the CSR pattern alone; the NUMERIC factorisation -- the reference's sorted
// row merge, src/ic_preconditioner.cpp:12-70 -- runs on the GPU in the forward schedule's level
// order, sync-free like the sweeps: a lane owns row i, waits until the pivots d_j of all its L
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

#include "internal.cuh"
#include "kernels.cuh"

namespace rcg {

int32_t build_schedule(int32_t n, const std::vector<int32_t>& rs, const std::vector<int32_t>& col,
                       const std::vector<double>& val, bool descending, std::vector<int32_t>& perm,
                       std::vector<int32_t>& prs, std::vector<int32_t>& pcol, std::vector<double>& pval,
                       std::vector<uint8_t>& crit, int32_t& npos, std::vector<int32_t>* pidx);

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
    // ---- pattern (host)
    std::vector<int32_t> rs(static_cast<size_t>(n) + 1), ci(static_cast<size_t>(A->nnz));
    RCG_CK(cudaMemcpy(rs.data(), A->rs, sizeof(int32_t) * rs.size(), cudaMemcpyDeviceToHost));
    if (A->nnz) RCG_CK(cudaMemcpy(ci.data(), A->ci, sizeof(int32_t) * ci.size(), cudaMemcpyDeviceToHost));
    f->n = n;
    f->h_bounds.resize(static_cast<size_t>(num_blocks) + 1);
    for (int b = 0; b <= num_blocks; ++b)
        f->h_bounds[b] = static_cast<int32_t>((static_cast<int64_t>(b) * n) / num_blocks);
    mark("pattern download");
    std::vector<int32_t> asrc, adiag(n, -1);
    f->h_lrs.assign(static_cast<size_t>(n) + 1, 0);
    f->h_lcol.clear();
    size_t blk = 0;
    for (int32_t i = 0; i < n; ++i) {  // ic_preconditioner.cpp:29-46: lo <= j < i, up to the diagonal
        while (i >= f->h_bounds[blk + 1]) ++blk;
        const int32_t lo = f->h_bounds[blk];
        f->h_lrs[i] = static_cast<int32_t>(f->h_lcol.size());
        for (int32_t k = rs[i]; k < rs[i + 1]; ++k) {
            const int32_t j = ci[k];
            if (j >= i) {
                if (j == i) adiag[i] = k;
                break;
            }
            if (j < lo) continue;
            f->h_lcol.push_back(j);
            asrc.push_back(k);
        }
        f->h_lrs[i + 1] = static_cast<int32_t>(f->h_lcol.size());
    }
    const int64_t nnzl = static_cast<int64_t>(f->h_lcol.size());
    f->nnz_l = nnzl;
    mark("L pattern");
    // transpose pattern + the L -> U position map (ic_preconditioner.cpp:74-93 order)
    f->h_urs.assign(static_cast<size_t>(n) + 1, 0);
    f->h_ucol.assign(nnzl, 0);
    std::vector<int32_t> l2u(nnzl);
    for (int32_t c : f->h_lcol) f->h_urs[c + 1]++;
    std::partial_sum(f->h_urs.begin(), f->h_urs.end(), f->h_urs.begin());
    {
        std::vector<int32_t> next(f->h_urs.begin(), f->h_urs.end() - 1);
        for (int32_t i = 0; i < n; ++i)
            for (int32_t k = f->h_lrs[i]; k < f->h_lrs[i + 1]; ++k) {
                const int32_t dst = next[f->h_lcol[k]]++;
                f->h_ucol[dst] = i;
                l2u[k] = dst;
            }
    }
    mark("U pattern");
    // schedules (pattern only; value gathers after the numeric pass)
    std::vector<int32_t> perm, prs, pcol, fidx, bidx;
    std::vector<double> none;
    std::vector<uint8_t> crit;
    f->fwd_levels = build_schedule(n, f->h_lrs, f->h_lcol, none, false, perm, prs, pcol, none, crit, f->f_npos, &fidx);
    f->f_perm = to_dev(ctx, perm);
    f->f_prs = to_dev(ctx, prs);
    f->f_col = to_dev(ctx, pcol);
    f->f_crit = to_dev(ctx, crit);
    RCG_CK(cudaStreamSynchronize(ctx->stream));
    mark("forward schedule + upload");
    f->bwd_levels = build_schedule(n, f->h_urs, f->h_ucol, none, true, perm, prs, pcol, none, crit, f->b_npos, &bidx);
    f->b_perm = to_dev(ctx, perm);
    f->b_prs = to_dev(ctx, prs);
    f->b_col = to_dev(ctx, pcol);
    f->b_crit = to_dev(ctx, crit);
    mark("backward schedule + upload");
    // ---- numeric (device)
    int32_t* d_lrs = to_dev(ctx, f->h_lrs);
    int32_t* d_lcol = to_dev(ctx, f->h_lcol);
    int32_t* d_asrc = to_dev(ctx, asrc);
    int32_t* d_adiag = to_dev(ctx, adiag);
    int32_t* d_l2u = to_dev(ctx, l2u);
    int32_t* d_fidx = to_dev(ctx, fidx);
    int32_t* d_bidx = to_dev(ctx, bidx);
    double* lval = dev_alloc(std::max<int64_t>(nnzl, 1));
    double* uval = dev_alloc(std::max<int64_t>(nnzl, 1));
    f->d = dev_alloc(std::max(n, 1));
    int* flags = static_cast<int*>(dev_alloc_bytes(sizeof(int) * 8));  // [0] fail, [4..7] tickets
    mark("pattern uploads");
    auto cleanup = [&] {
        for (void* p : {(void*)d_lrs, (void*)d_lcol, (void*)d_asrc, (void*)d_adiag, (void*)d_l2u, (void*)d_fidx,
                        (void*)d_bidx, (void*)lval, (void*)uval, (void*)flags})
            dev_free(p);
    };
    try {
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
            fa.lrs = d_lrs;
            fa.lcol = d_lcol;
            fa.lval = lval;
            fa.ava = A->va;
            fa.asrc = d_asrc;
            fa.adiag = d_adiag;
            fa.d = f->d;
            fa.shift = s;
            fa.fail = flags;
            fa.tickets = flags + 4;
            if (n > 0) {
                k_ic_factor<<<grid, 128, 0, ctx->stream>>>(fa);
                RCG_LAUNCHED(ctx);
            }
            int h[8];
            RCG_CK(cudaMemcpyAsync(h, flags, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
            RCG_CK(cudaStreamSynchronize(ctx->stream));
            if (h[4 + 3]) throw Error(RCG_E_CUDA, "ic0_factorize_device: dependency wait exceeded its bound");
            ok = h[0] == 0;
            f->shift = s;
            if (!ok) s = (s == 0.0) ? 0.01 : 2.0 * s;
        }
        if (!ok) {
            char buf[160];
            std::snprintf(buf, sizeof buf,
                          "IC breakdown: no positive-pivot factorization after %d shift retries (last shift %f)",
                          retries, s);
            throw Error(RCG_E_BREAKDOWN, buf);
        }
        mark("numeric (device)");
        // U values and the schedule copies, on the device
        const int g = stream_grid(ctx, std::max<int64_t>(nnzl, 1));
        f->f_val = dev_alloc(std::max<int64_t>(nnzl, 1));
        f->b_val = dev_alloc(std::max<int64_t>(nnzl, 1));
        if (nnzl > 0) {
            k_scatter<<<g, kStreamThreads, 0, ctx->stream>>>(lval, d_l2u, uval, nnzl);
            RCG_LAUNCHED(ctx);
            k_gather<<<g, kStreamThreads, 0, ctx->stream>>>(lval, d_fidx, f->f_val, nnzl);
            RCG_LAUNCHED(ctx);
            k_gather<<<g, kStreamThreads, 0, ctx->stream>>>(uval, d_bidx, f->b_val, nnzl);
            RCG_LAUNCHED(ctx);
        }
        // host image (IcFactor fields, for rcg_ic_export)
        f->h_lval.resize(nnzl);
        f->h_uval.resize(nnzl);
        f->h_d.resize(n);
        if (nnzl > 0) {
            RCG_CK(cudaMemcpyAsync(f->h_lval.data(), lval, sizeof(double) * nnzl, cudaMemcpyDeviceToHost, ctx->stream));
            RCG_CK(cudaMemcpyAsync(f->h_uval.data(), uval, sizeof(double) * nnzl, cudaMemcpyDeviceToHost, ctx->stream));
        }
        mark("gathers");
        if (n > 0) RCG_CK(cudaMemcpyAsync(f->h_d.data(), f->d, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
        RCG_CK(cudaStreamSynchronize(ctx->stream));
        mark("host image download");
    } catch (...) {
        cleanup();
        throw;
    }
    cleanup();
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
