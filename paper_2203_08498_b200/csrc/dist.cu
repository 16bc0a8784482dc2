// dist.cu -- multi-GPU row slabs: the host slab plan, device slabs, the two
// slab transports (NCCL, one slab per process; loopback, all slabs in one process on one GPU)
// and the distributed PCG.
//
// Operator: the reference's block-Jacobi IC(0) (ic0_factorize(a, s, G), ic_preconditioner.cpp:
// 97-121, bounds floor(b n / G)).  Rank b owns rows [floor(b n/G), floor((b+1) n/G)); its
// preconditioner is the IC(0) factor of its diagonal block, so the sweeps need no communication.
// Per iteration (pcg.cpp:63-89 order): local sweeps -> allreduce (r,z) -> beta, p = z + beta p ->
// halo exchange of p -> q = A p_ext -> allreduce (p,q) -> alpha, x, r -> allreduce (r,r) ->
// relres / convergence.  Local partial sums are deterministic (fixed-order grid reductions);
// every rank receives identical totals, so every rank's DevState evolves identically and all
// ranks stop enqueueing at the same batch boundary (matching collectives, no host agreement).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <vector>

#include "internal.cuh"
#include "kernels.cuh"
#include "spmv_pipe.cuh"
#include "vec.cuh"

namespace rcg {

constexpr int kDistTick = 6;  // DevState::tick slot of the slab-local reductions

// ------------------------------------------------------------------ host slab plan
static int32_t bound_of(int b, int32_t n, int nparts) {
    return static_cast<int32_t>((static_cast<int64_t>(b) * n) / nparts);  // ic_preconditioner.cpp:104-106
}

static void plan_create(int32_t n, const int32_t* rs, const int32_t* ci, const double* va, int nparts, int part,
                        rcg_slab_plan* out) {
    require(n >= 1 && rs && ci && va && out, "rcg_slab_plan_create: null argument");
    require(nparts >= 1 && nparts <= n && part >= 0 && part < nparts, "rcg_slab_plan_create: bad partition");
    std::memset(out, 0, sizeof(*out));
    std::vector<int32_t> bounds(nparts + 1);
    for (int b = 0; b <= nparts; ++b) bounds[b] = bound_of(b, n, nparts);
    auto owner = [&](int32_t col) {
        return static_cast<int>(std::upper_bound(bounds.begin(), bounds.end(), col) - bounds.begin()) - 1;
    };
    const int32_t r0 = bounds[part], r1 = bounds[part + 1], nloc = r1 - r0;
    std::vector<int32_t> halo;
    for (int64_t e = rs[r0]; e < rs[r1]; ++e)
        if (ci[e] < r0 || ci[e] >= r1) halo.push_back(ci[e]);
    std::sort(halo.begin(), halo.end());
    halo.erase(std::unique(halo.begin(), halo.end()), halo.end());
    const int64_t nnz = rs[r1] - rs[r0];
    out->row_begin = r0;
    out->row_end = r1;
    out->nloc = nloc;
    out->nhalo = static_cast<int32_t>(halo.size());
    out->nnz = nnz;
    out->nparts = nparts;
    out->part = part;
    auto alloc = [](size_t bytes) {
        void* p = std::malloc(std::max<size_t>(bytes, 8));
        if (!p) throw Error(RCG_E_INVALID, "rcg_slab_plan_create: out of host memory");
        return p;
    };
    out->row_start = static_cast<int32_t*>(alloc(sizeof(int32_t) * (nloc + 1)));
    out->col_idx = static_cast<int32_t*>(alloc(sizeof(int32_t) * nnz));
    out->values = static_cast<double*>(alloc(sizeof(double) * nnz));
    out->halo_global = static_cast<int32_t*>(alloc(sizeof(int32_t) * halo.size()));
    out->recv_count = static_cast<int32_t*>(alloc(sizeof(int32_t) * nparts));
    out->send_count = static_cast<int32_t*>(alloc(sizeof(int32_t) * nparts));
    std::memcpy(out->halo_global, halo.data(), sizeof(int32_t) * halo.size());
    for (int q = 0; q < nparts; ++q) out->recv_count[q] = out->send_count[q] = 0;
    for (int32_t h : halo) out->recv_count[owner(h)]++;
    // local CSR: own columns -> col - r0, halo columns -> nloc + position in halo
    for (int32_t i = 0; i <= nloc; ++i) out->row_start[i] = static_cast<int32_t>(rs[r0 + i] - rs[r0]);
    for (int64_t e = rs[r0]; e < rs[r1]; ++e) {
        const int32_t c = ci[e];
        const int64_t le = e - rs[r0];
        out->col_idx[le] = (c >= r0 && c < r1)
                               ? c - r0
                               : nloc + static_cast<int32_t>(std::lower_bound(halo.begin(), halo.end(), c) - halo.begin());
        out->values[le] = va[e];
    }
    // send lists (symmetric pattern): my rows with a column owned by q, ascending, grouped by q
    std::vector<std::vector<int32_t>> send(nparts);
    for (int32_t i = 0; i < nloc; ++i) {
        int last = -1;
        std::vector<int> qs;
        for (int64_t e = rs[r0 + i]; e < rs[r0 + i + 1]; ++e) {
            const int32_t c = ci[e];
            if (c >= r0 && c < r1) continue;
            qs.push_back(owner(c));
        }
        std::sort(qs.begin(), qs.end());
        for (int q : qs)
            if (q != last) {
                send[q].push_back(i);
                last = q;
            }
    }
    int64_t nsend = 0;
    for (int q = 0; q < nparts; ++q) nsend += static_cast<int64_t>(send[q].size());
    out->send_idx = static_cast<int32_t*>(alloc(sizeof(int32_t) * nsend));
    int64_t off = 0;
    for (int q = 0; q < nparts; ++q) {
        out->send_count[q] = static_cast<int32_t>(send[q].size());
        std::memcpy(out->send_idx + off, send[q].data(), sizeof(int32_t) * send[q].size());
        off += static_cast<int64_t>(send[q].size());
    }
}

static void plan_free(rcg_slab_plan* p) {
    if (!p) return;
    for (void* a : {(void*)p->row_start, (void*)p->col_idx, (void*)p->values, (void*)p->halo_global,
                    (void*)p->recv_count, (void*)p->send_count, (void*)p->send_idx})
        std::free(a);
    std::memset(p, 0, sizeof(*p));
}

}  // namespace rcg

// ------------------------------------------------------------------ device slab
struct rcg_dslab {
    rcg_ctx* ctx = nullptr;       // borrowed: stream, workspace, DevState
    rcg_matrix* a = nullptr;      // owned: nloc rows, columns [0, nloc + nhalo)
    const rcg_ic* ic = nullptr;   // borrowed: diagonal-block factor (null = identity)
    int nparts = 1, part = 0;
    int32_t nloc = 0, nhalo = 0, row_begin = 0;
    std::vector<int32_t> send_count, recv_count, send_off, recv_off;
    int32_t nsend = 0;
    int32_t* send_idx = nullptr;  // device
    double* sendbuf = nullptr;    // device
    double* xe = nullptr;         // device x_ext (nloc + nhalo)
    double* pe = nullptr;         // device p_ext (nloc + nhalo)
    double* dsum = nullptr;       // device: local partials in, global totals out (scalars)
    double* gbuf = nullptr;       // device: m-vectors / the m x m Gram (allreduced the same way)
    double* ubuf = nullptr;       // device: projection coefficients (m)
    double* u2buf = nullptr;      // device: subspace-correction coefficients (m)
    int64_t cap_g = 0;
    double* sendbuf_rt = nullptr; // device: the batched solver's halo (nsend x RT interleaved)
    int64_t cap_send_rt = 0;
};

// a row-partitioned basis: every slab holds its rows of W and AW, and the
// replicated Cholesky factor of W^T A W (allreduced Gram, factored identically on every rank)
struct rcg_dbasis {
    int kind = 0;  // RCG_BASIS_DEFLATION / RCG_BASIS_SC
    int m = 0;
    std::vector<double*> w, aw, l;  // per local slab (W, AW: nloc x m column-major, ld nloc)
    std::vector<double> h_l;        // the factor (row-major m x m), identical on every rank
};

namespace rcg {

// ------------------------------------------------------------------ kernels
// r = b - A x_ext (local rows); partials (b, b), (r, r)
__global__ void __launch_bounds__(kSpmvThreads) k_d_residual(SpmvArgs a, int cap, const double* __restrict__ b,
                                                             double* __restrict__ r, DevState* st, double* dsum) {
    __shared__ double red[2 * 32];
    __shared__ double tot[2];
    double acc[2] = {0.0, 0.0};
    spmv_pipeline<1>(a, cap, [&](int32_t row, const double (&s)[1]) {
        const double bi = b[row];
        const double ri = __dsub_rn(bi, s[0]);
        r[row] = ri;
        acc[0] = fadd_mul(acc[0], bi, bi);
        acc[1] = fadd_mul(acc[1], ri, ri);
    });
    block_sum<2>(acc, red);
    if (grid_reduce<2>(acc, a.partials, blockIdx.x, gridDim.x, &st->tick[kDistTick], tot, red) && threadIdx.x == 0) {
        dsum[0] = tot[0];
        dsum[1] = tot[1];
    }
}

// q = A p_ext (local rows); partial (p, q)
__global__ void __launch_bounds__(kSpmvThreads) k_d_spmv(SpmvArgs a, int cap, DevState* st, double* dsum) {
    __shared__ double red[32];
    __shared__ double tot[1];
    if (st->done) return;
    double acc[1] = {0.0};
    spmv_pipeline<1>(a, cap, [&](int32_t row, const double (&s)[1]) {
        a.y[0][row] = s[0];
        acc[0] = fadd_mul(acc[0], a.x[0][row], s[0]);
    });
    block_sum<1>(acc, red);
    if (grid_reduce<1>(acc, a.partials, blockIdx.x, gridDim.x, &st->tick[kDistTick], tot, red) && threadIdx.x == 0)
        dsum[0] = tot[0];
}

// partial (u, v)
__global__ void __launch_bounds__(kStreamThreads) k_d_dot(const double* __restrict__ u, const double* __restrict__ v,
                                                          int32_t n, double* partials, DevState* st, double* dsum) {
    __shared__ double red[32];
    __shared__ double tot[1];
    if (st->done) return;
    double acc[1] = {0.0};
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        acc[0] = fadd_mul(acc[0], u[i], v[i]);
    block_sum<1>(acc, red);
    if (grid_reduce<1>(acc, partials, blockIdx.x, gridDim.x, &st->tick[kDistTick], tot, red) && threadIdx.x == 0)
        dsum[0] = tot[0];
}

// x += alpha p, r -= alpha q (local rows); partial (r, r)
__global__ void __launch_bounds__(kStreamThreads) k_d_xr(double* __restrict__ x, double* __restrict__ r,
                                                         const double* __restrict__ p, const double* __restrict__ q,
                                                         int32_t n, double* partials, DevState* st, double* dsum) {
    __shared__ double red[32];
    __shared__ double tot[1];
    if (st->done) return;
    const double alpha = st->alpha;
    double acc[1] = {0.0};
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        x[i] = fadd_mul(x[i], alpha, p[i]);
        const double ri = fsub_mul(r[i], alpha, q[i]);
        r[i] = ri;
        acc[0] = fadd_mul(acc[0], ri, ri);
    }
    block_sum<1>(acc, red);
    if (grid_reduce<1>(acc, partials, blockIdx.x, gridDim.x, &st->tick[kDistTick], tot, red) && threadIdx.x == 0)
        dsum[0] = tot[0];
}

// the error sampler after iteration st->iters (sampling.cpp:7-84): identical scalars on every
// slab, so every slab schedules the same slots; converged iterations offer nothing (the observer
// runs after the convergence test, pcg.cpp:81-88); an iteration that did not complete
// (breakdown, or the solve already over) schedules nothing
__global__ void k_d_sched(DevState* st, int* pending, int* occupied, int* stored_iter, const double* thresholds) {
    if (st->smp_method < 0) return;
    const int i = st->iters;
    if (i == 0 || i == st->smp_pending_iter) {
        st->smp_npending = 0;
        return;
    }
    if (st->done == kConverged || st->done == kBroken) {
        st->smp_npending = 0;
        st->smp_pending_iter = i;
        return;
    }
    smp_schedule(st, i, st->relres, pending, occupied, stored_iter, thresholds);
}

// copy this iteration's payload (x, or r) into the scheduled slots (local rows)
__global__ void __launch_bounds__(kStreamThreads) k_d_sample(const double* __restrict__ x, const double* __restrict__ r,
                                                             double* __restrict__ slots, int64_t ld,
                                                             const int* __restrict__ pending, const DevState* st,
                                                             int32_t n) {
    const int np = st->smp_npending;
    if (np == 0) return;
    const double* src = st->smp_payload ? r : x;
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double v = src[i];
        for (int k = 0; k < np; ++k) slots[pending[k] * ld + i] = v;
    }
}

// (u, v) over the local rows into *out (deterministic two-level reduction; no solver state)
__global__ void __launch_bounds__(kStreamThreads) k_rr_dot(const double* __restrict__ u, const double* __restrict__ v,
                                                           int32_t n, double* partials, unsigned int* tick,
                                                           double* out) {
    __shared__ double red[32];
    __shared__ double tot[1];
    double acc[1] = {0.0};
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        acc[0] = fadd_mul(acc[0], u[i], v[i]);
    block_sum<1>(acc, red);
    if (grid_reduce<1>(acc, partials, blockIdx.x, gridDim.x, tick, tot, red) && threadIdx.x == 0) *out = tot[0];
}

// w -= c q with c the allreduced (q, w) (the MGS update, dense.cpp:52-54); scale: w /= sqrt(c)
__global__ void __launch_bounds__(kStreamThreads) k_rr_axpy(double* __restrict__ w, const double* __restrict__ q,
                                                            const double* __restrict__ c, int32_t n, int scale) {
    const double cv = *c;
    const double nr = scale ? sqrt(cv) : 0.0;
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        w[i] = scale ? __ddiv_rn(w[i], nr) : fsub_mul(w[i], cv, q[i]);
}

__global__ void k_d_pack(const double* __restrict__ v, const int32_t* __restrict__ idx, int32_t cnt,
                         double* __restrict__ out) {
    for (int32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += gridDim.x * blockDim.x) out[t] = v[idx[t]];
}

// rt-interleaved rows (the batched solver's vectors): out[t rt + k] = v[idx[t] rt + k]
__global__ void k_d_pack_rt(const double* __restrict__ v, const int32_t* __restrict__ idx, int32_t cnt, int rt,
                            double* __restrict__ out) {
    const int64_t total = static_cast<int64_t>(cnt) * rt;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[e] = v[static_cast<int64_t>(idx[e / rt]) * rt + e % rt];
}

// scalar updates from the global totals g (pcg.cpp:43-89): 0 initial (b,b),(r,r); 1 (r,z);
// 2 (p,q); 3 (r,r) after the x/r update
// flags: 1 = defer the initial check to the projected residual (deflation; stage 4), 2 = add
// the subspace-correction term st->scal[2] to (r, z)
__global__ void k_d_scalar(DevState* st, const double* __restrict__ g, int stage, double* hist, double* alph,
                           double* bet, int identity, int flags) {
    if (stage == 0) {
        st->bnorm = sqrt(g[0]);
        st->rr = g[1];
        st->rho = g[1];
        if (st->bnorm == 0.0)
            st->done = kZeroRhs;
        else if (!(flags & 1) && sqrt(g[1]) <= st->eps * st->bnorm)
            st->done = kConverged;
        return;
    }
    if (st->done) return;
    if (stage == 4) {  // projected initial residual (pcg.cpp:112-118)
        st->rr = g[0];
        st->rho = g[0];
        if (sqrt(g[0]) <= st->eps * st->bnorm) st->done = kConverged;
        return;
    }
    if (stage == 1) {
        const double rho = (flags & 2) ? __dadd_rn(g[0], st->scal[2]) : g[0];
        st->rho = rho;
        if (rho <= 0.0) {
            st->done = kBroken;
            st->status = kBrkRz;
        }
        st->beta = st->iter > 1 ? rho / st->rho_prev : 0.0;
    } else if (stage == 2) {
        st->pq = g[0];
        if (g[0] <= 0.0) {
            st->done = kBroken;
            st->status = kBrkPAp;
        }
        st->alpha = st->rho / g[0];
    } else {
        const int i = st->iter;
        const double rr = g[0];
        const double relres = sqrt(rr) / st->bnorm;
        st->rr = rr;
        st->relres = relres;
        st->iters = i;
        hist[i - 1] = relres;
        alph[i - 1] = st->alpha;
        bet[i - 1] = st->beta;
        st->rho_prev = st->rho;
        if (relres <= st->eps) {
            st->done = kConverged;
        } else if (i >= st->max_iter) {
            st->done = kCapped;
        } else {
            st->iter = i + 1;
            if (identity) {  // z = r: the next (r, z) is this (r, r)
                st->rho = rr;
                if (rr <= 0.0) {
                    st->done = kBroken;
                    st->status = kBrkRz;
                }
                st->beta = rr / st->rho_prev;
            }
        }
    }
}

// u = (W^T A W)^-1 f by one warp (replicated factor); mode 2 also stores f . u in st->scal[2]
// (the subspace-correction term of (r, z), subspace_correction.cpp:47-57)
__global__ void k_d_chol(const double* __restrict__ L, int m, const double* __restrict__ f, double* __restrict__ u,
                         DevState* st, int mode, int respect_done) {
    __shared__ double sf[128], ss[128];
    if (respect_done && st->done) return;
    const int lane = threadIdx.x & 31;
    for (int j = lane; j < m; j += 32) sf[j] = f[j];
    __syncwarp();
    warp_chol_solve(L, m, sf, u, ss);
    __syncwarp();
    if (mode == 2 && lane == 0) {
        double fu = 0.0;
        for (int j = 0; j < m; ++j) fu = fadd_mul(fu, sf[j], ss[j]);
        st->scal[2] = fu;
    }
}

// y -= sum_j u_j C_j (subtract_combination, deflation.cpp:7-13) on the local rows, partial of
// (p, y) (mode 0) or (y, y) (mode 1) into dsum[0]
__global__ void __launch_bounds__(kStreamThreads) k_d_deflate(double* __restrict__ y, const double* __restrict__ C,
                                                              int64_t ldc, int m, const double* __restrict__ u,
                                                              const double* __restrict__ p, int32_t n, double* partials,
                                                              DevState* st, double* dsum, int mode) {
    __shared__ double red[32];
    __shared__ double tot[1];
    if (st->done) return;
    double acc[1] = {0.0};
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double v = y[i];
        for (int j = 0; j < m; ++j) v = fsub_mul(v, __ldg(u + j), __ldg(C + j * ldc + i));
        y[i] = v;
        acc[0] = mode == 0 ? fadd_mul(acc[0], p[i], v) : fadd_mul(acc[0], v, v);
    }
    block_sum<1>(acc, red);
    if (grid_reduce<1>(acc, partials, blockIdx.x, gridDim.x, &st->tick[kDistTick], tot, red) && threadIdx.x == 0)
        dsum[0] = tot[0];
}

// loopback allreduce: every slab's partials summed in slab order, written back to all
__global__ void k_lb_sum(double* const* d, int nslabs, int count) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= count) return;
    double s = 0.0;
    for (int b = 0; b < nslabs; ++b) s = __dadd_rn(s, d[b][c]);
    for (int b = 0; b < nslabs; ++b) d[b][c] = s;
}

}  // namespace rcg

// ------------------------------------------------------------------ transports
struct rcg_comm {
    virtual ~rcg_comm() {}
    virtual int nparts() const = 0;
    virtual int local_slabs() const = 0;
    virtual void begin(rcg_dslab* const* s, int ns) { (void)s, (void)ns; }
    // in-place sum over all slabs of dsum[0..count) (sel 0) or gbuf[0..count) (sel 1)
    virtual void allreduce(rcg_dslab* const* s, int ns, int count, int sel = 0) = 0;
    // halo of the ext vector `which` (0: x_ext, 1: p_ext)
    virtual void halo(rcg_dslab* const* s, int ns, int which) = 0;
    // halo rows of an rt-interleaved vector of ONE local slab (the batched solver)
    virtual void halo_rt(rcg_dslab* d, double* v, int rt) = 0;
};

namespace rcg {

// host -> device into a slab buffer, ordered on the slab's (non-blocking) stream and complete on
// return: a legacy cudaMemcpy from pageable memory may return before its DMA lands and is not
// ordered with the slab stream's next copy / kernel (the host transport read stale Gram values)
static void h2d_sync(rcg_ctx* ctx, void* dst, const void* src, size_t bytes) {
    RCG_CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
    RCG_CK(cudaStreamSynchronize(ctx->stream));
}

static double* ext_of(rcg_dslab* s, int which) { return which == 0 ? s->xe : s->pe; }

// the rt-interleaved send rows of d (grows d->sendbuf_rt)
static void pack_rt(rcg_dslab* d, const double* v, int rt) {
    const int64_t need = static_cast<int64_t>(d->nsend) * rt;
    if (need > d->cap_send_rt) {
        dev_free(d->sendbuf_rt);
        d->sendbuf_rt = dev_alloc(std::max<int64_t>(need, 1));
        d->cap_send_rt = need;
    }
    if (d->nsend == 0) return;
    const int g = std::max(1, static_cast<int>(std::min<int64_t>((need + 255) / 256, d->ctx->num_sms * 4)));
    k_d_pack_rt<<<g, 256, 0, d->ctx->stream>>>(v, d->send_idx, d->nsend, rt, d->sendbuf_rt);
    RCG_LAUNCHED(d->ctx);
}

static void pack(rcg_dslab* s, int which) {
    if (s->nsend == 0) return;
    const int g = std::max(1, std::min((s->nsend + 255) / 256, s->ctx->num_sms * 4));
    k_d_pack<<<g, 256, 0, s->ctx->stream>>>(ext_of(s, which), s->send_idx, s->nsend, s->sendbuf);
    RCG_LAUNCHED(s->ctx);
}

// --- NCCL, resolved at run time
struct Nccl {
    void* h = nullptr;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;

    static Nccl& get() {
        static Nccl n;
        if (!n.h) {
            // the copy the process already loaded (torch's), else the loader's libnccl.so.2
            n.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
            if (!n.h) n.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
            if (!n.h) throw Error(RCG_E_CUDA, std::string("NCCL transport: cannot load libnccl.so.2: ") + dlerror());
            auto sym = [&](const char* name) {
                void* f = dlsym(n.h, name);
                if (!f) throw Error(RCG_E_CUDA, std::string("NCCL transport: missing symbol ") + name);
                return f;
            };
            n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(sym("ncclGetUniqueId"));
            n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(sym("ncclCommInitRank"));
            n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(sym("ncclCommDestroy"));
            n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(sym("ncclAllReduce"));
            n.send = reinterpret_cast<decltype(n.send)>(sym("ncclSend"));
            n.recv = reinterpret_cast<decltype(n.recv)>(sym("ncclRecv"));
            n.group_start = reinterpret_cast<decltype(n.group_start)>(sym("ncclGroupStart"));
            n.group_end = reinterpret_cast<decltype(n.group_end)>(sym("ncclGroupEnd"));
            n.error_string = reinterpret_cast<decltype(n.error_string)>(sym("ncclGetErrorString"));
        }
        return n;
    }
    void check(ncclResult_t r, const char* what) {
        if (r != ncclSuccess) throw Error(RCG_E_CUDA, std::string("NCCL ") + what + ": " + error_string(r));
    }
};

struct NcclComm : rcg_comm {
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0;
    int nparts() const override { return nranks; }
    int local_slabs() const override { return 1; }
    ~NcclComm() override {
        if (comm) Nccl::get().comm_destroy(comm);
    }
    void allreduce(rcg_dslab* const* s, int ns, int count, int sel) override {
        (void)ns;
        Nccl& nc = Nccl::get();
        double* buf = sel ? s[0]->gbuf : s[0]->dsum;
        nc.check(nc.all_reduce(buf, buf, count, ncclFloat64, ncclSum, comm, s[0]->ctx->stream), "allreduce");
    }
    void halo(rcg_dslab* const* s, int ns, int which) override {
        (void)ns;
        rcg_dslab* d = s[0];
        pack(d, which);
        Nccl& nc = Nccl::get();
        double* ext = ext_of(d, which);
        nc.check(nc.group_start(), "group start");
        for (int q = 0; q < nranks; ++q) {
            if (d->send_count[q])
                nc.check(nc.send(d->sendbuf + d->send_off[q], d->send_count[q], ncclFloat64, q, comm, d->ctx->stream),
                         "send");
            if (d->recv_count[q])
                nc.check(nc.recv(ext + d->nloc + d->recv_off[q], d->recv_count[q], ncclFloat64, q, comm, d->ctx->stream),
                         "recv");
        }
        nc.check(nc.group_end(), "group end");
    }
    void halo_rt(rcg_dslab* d, double* v, int rt) override {
        pack_rt(d, v, rt);
        Nccl& nc = Nccl::get();
        nc.check(nc.group_start(), "group start");
        for (int q = 0; q < nranks; ++q) {
            if (d->send_count[q])
                nc.check(nc.send(d->sendbuf_rt + static_cast<int64_t>(d->send_off[q]) * rt,
                                 static_cast<size_t>(d->send_count[q]) * rt, ncclFloat64, q, comm, d->ctx->stream),
                         "send");
            if (d->recv_count[q])
                nc.check(nc.recv(v + (static_cast<int64_t>(d->nloc) + d->recv_off[q]) * rt,
                                 static_cast<size_t>(d->recv_count[q]) * rt, ncclFloat64, q, comm, d->ctx->stream),
                         "recv");
        }
        nc.check(nc.group_end(), "group end");
    }
};

// --- host-staged: a caller-supplied host transport (torch.distributed over gloo, MPI, ...).  Every
// collective synchronises the slab's stream and round-trips through host memory, so ranks never
// wait on one another inside a kernel: several processes may share one GPU (the world-size-2
// tests of this file's distributed iteration, tests/test_gpu_dist_host.py).  Slow by design.
struct HostComm : rcg_comm {
    int nranks = 1, rank = 0;
    rcg_host_allreduce_fn ar = nullptr;
    rcg_host_exchange_fn ex = nullptr;
    void* user = nullptr;
    std::vector<double> hbuf, hsend, hrecv;
    std::vector<int64_t> so, sc, ro, rc;
    int nparts() const override { return nranks; }
    int local_slabs() const override { return 1; }
    double* pin = nullptr;  // pinned staging of the allreduced values
    int cap_pin = 0;
    ~HostComm() override {
        if (pin) cudaFreeHost(pin);
    }
    void allreduce(rcg_dslab* const* s, int ns, int count, int sel) override {
        (void)ns;
        rcg_dslab* d = s[0];
        double* buf = sel ? d->gbuf : d->dsum;
        if (count > cap_pin) {
            if (pin) cudaFreeHost(pin);
            RCG_CK(cudaMallocHost(&pin, sizeof(double) * std::max(count, 1)));
            cap_pin = count;
        }
        hbuf.resize(std::max(count, 1));
        RCG_CK(cudaStreamSynchronize(d->ctx->stream));
        RCG_CK(cudaMemcpyAsync(pin, buf, sizeof(double) * count, cudaMemcpyDeviceToHost, d->ctx->stream));
        RCG_CK(cudaStreamSynchronize(d->ctx->stream));
        std::memcpy(hbuf.data(), pin, sizeof(double) * count);
        static const bool dbg = std::getenv("RCG_HOSTCOMM_DEBUG") != nullptr;  // dev
        if (dbg) std::fprintf(stderr, "[hostcomm r%d] allreduce sel %d count %d in %.6g", rank, sel, count, hbuf[0]);
        if (ar(user, hbuf.data(), count) != 0) throw Error(RCG_E_CUDA, "host transport: allreduce callback failed");
        if (dbg) std::fprintf(stderr, " out %.6g\n", hbuf[0]);
        std::memcpy(pin, hbuf.data(), sizeof(double) * count);
        RCG_CK(cudaMemcpyAsync(buf, pin, sizeof(double) * count, cudaMemcpyHostToDevice, d->ctx->stream));
        RCG_CK(cudaStreamSynchronize(d->ctx->stream));
    }
    void halo(rcg_dslab* const* s, int ns, int which) override {
        (void)ns;
        rcg_dslab* d = s[0];
        pack(d, which);
        hsend.resize(std::max(d->nsend, 1));
        hrecv.resize(std::max(d->nhalo, 1));
        if (d->nsend > 0)
            RCG_CK(cudaMemcpyAsync(hsend.data(), d->sendbuf, sizeof(double) * d->nsend, cudaMemcpyDeviceToHost,
                                   d->ctx->stream));
        RCG_CK(cudaStreamSynchronize(d->ctx->stream));
        so.assign(d->send_off.begin(), d->send_off.end());
        sc.assign(d->send_count.begin(), d->send_count.end());
        ro.assign(d->recv_off.begin(), d->recv_off.end());
        rc.assign(d->recv_count.begin(), d->recv_count.end());
        if (ex(user, hsend.data(), so.data(), sc.data(), hrecv.data(), ro.data(), rc.data(), nranks) != 0)
            throw Error(RCG_E_CUDA, "host transport: halo exchange callback failed");
        if (d->nhalo > 0)
            RCG_CK(cudaMemcpyAsync(ext_of(d, which) + d->nloc, hrecv.data(), sizeof(double) * d->nhalo,
                                   cudaMemcpyHostToDevice, d->ctx->stream));
        RCG_CK(cudaStreamSynchronize(d->ctx->stream));
    }
    void halo_rt(rcg_dslab* d, double* v, int rt) override {
        pack_rt(d, v, rt);
        const int64_t ns_ = static_cast<int64_t>(d->nsend) * rt, nr = static_cast<int64_t>(d->nhalo) * rt;
        hsend.resize(std::max<int64_t>(ns_, 1));
        hrecv.resize(std::max<int64_t>(nr, 1));
        if (ns_ > 0)
            RCG_CK(cudaMemcpyAsync(hsend.data(), d->sendbuf_rt, sizeof(double) * ns_, cudaMemcpyDeviceToHost,
                                   d->ctx->stream));
        RCG_CK(cudaStreamSynchronize(d->ctx->stream));
        so.resize(nranks), sc.resize(nranks), ro.resize(nranks), rc.resize(nranks);
        for (int q = 0; q < nranks; ++q) {
            so[q] = static_cast<int64_t>(d->send_off[q]) * rt;
            sc[q] = static_cast<int64_t>(d->send_count[q]) * rt;
            ro[q] = static_cast<int64_t>(d->recv_off[q]) * rt;
            rc[q] = static_cast<int64_t>(d->recv_count[q]) * rt;
        }
        if (ex(user, hsend.data(), so.data(), sc.data(), hrecv.data(), ro.data(), rc.data(), nranks) != 0)
            throw Error(RCG_E_CUDA, "host transport: halo exchange callback failed");
        if (nr > 0)
            RCG_CK(cudaMemcpyAsync(v + static_cast<int64_t>(d->nloc) * rt, hrecv.data(), sizeof(double) * nr,
                                   cudaMemcpyHostToDevice, d->ctx->stream));
        RCG_CK(cudaStreamSynchronize(d->ctx->stream));
    }
};

// --- loopback: all slabs in this process (one GPU); stream-ordered copies, fixed-order sums
struct LoopComm : rcg_comm {
    int np = 1;
    int dev = 0;
    cudaStream_t cs = nullptr;
    cudaEvent_t ev_join = nullptr;
    std::vector<cudaEvent_t> ev;
    std::vector<cudaEvent_t> ev_read;  // receiver b finished copying out of the senders' buffers
    double** dptrs = nullptr;  // device arrays of the slabs' dsum / gbuf pointers
    double** gptrs = nullptr;
    std::vector<double*> hd, hg;
    int nparts() const override { return np; }
    int local_slabs() const override { return np; }
    ~LoopComm() override {
        if (dptrs) dev_free(dptrs);
        if (gptrs) dev_free(gptrs);
        for (auto e : ev) cudaEventDestroy(e);
        for (auto e : ev_read) cudaEventDestroy(e);
        if (ev_join) cudaEventDestroy(ev_join);
        if (cs) cudaStreamDestroy(cs);
    }
    void sync_ptrs(rcg_dslab* const* s, int ns) {
        std::vector<double*> d(ns), g(ns);
        for (int b = 0; b < ns; ++b) {
            d[b] = s[b]->dsum;
            g[b] = s[b]->gbuf;
        }
        if (d != hd) {
            RCG_CK(cudaMemcpyAsync(dptrs, d.data(), sizeof(double*) * ns, cudaMemcpyHostToDevice, cs));
            RCG_CK(cudaStreamSynchronize(cs));
            hd = d;
        }
        if (g != hg) {
            RCG_CK(cudaMemcpyAsync(gptrs, g.data(), sizeof(double*) * ns, cudaMemcpyHostToDevice, cs));
            RCG_CK(cudaStreamSynchronize(cs));
            hg = g;
        }
    }
    void begin(rcg_dslab* const* s, int ns) override { sync_ptrs(s, ns); }
    void allreduce(rcg_dslab* const* s, int ns, int count, int sel) override {
        sync_ptrs(s, ns);
        for (int b = 0; b < ns; ++b) {
            RCG_CK(cudaEventRecord(ev[b], s[b]->ctx->stream));
            RCG_CK(cudaStreamWaitEvent(cs, ev[b], 0));
        }
        k_lb_sum<<<(count + 255) / 256, 256, 0, cs>>>(sel ? gptrs : dptrs, ns, count);
        RCG_CK(cudaGetLastError());
        RCG_CK(cudaEventRecord(ev_join, cs));
        for (int b = 0; b < ns; ++b) RCG_CK(cudaStreamWaitEvent(s[b]->ctx->stream, ev_join, 0));
    }
    void halo(rcg_dslab* const* s, int ns, int which) override {
        for (int q = 0; q < ns; ++q) {
            pack(s[q], which);
            RCG_CK(cudaEventRecord(ev[q], s[q]->ctx->stream));
        }
        for (int b = 0; b < ns; ++b) {
            rcg_dslab* d = s[b];
            double* ext = ext_of(d, which);
            for (int q = 0; q < ns; ++q) {
                if (!d->recv_count[q]) continue;
                RCG_CK(cudaStreamWaitEvent(d->ctx->stream, ev[q], 0));
                RCG_CK(cudaMemcpyAsync(ext + d->nloc + d->recv_off[q], s[q]->sendbuf + s[q]->send_off[b],
                                       sizeof(double) * d->recv_count[q], cudaMemcpyDeviceToDevice, d->ctx->stream));
            }
            RCG_CK(cudaEventRecord(ev_read[b], d->ctx->stream));
        }
        // write-after-read: slab q may pack its next halo into sendbuf only after every receiver
        // has copied this one out (back-to-back halo loops -- basis build, A Q -- have no
        // allreduce in between to join the streams)
        for (int q = 0; q < ns; ++q)
            for (int b = 0; b < ns; ++b)
                if (b != q && s[b]->recv_count[q]) RCG_CK(cudaStreamWaitEvent(s[q]->ctx->stream, ev_read[b], 0));
    }
    void halo_rt(rcg_dslab* d, double* v, int rt) override {
        (void)v, (void)rt;
        // batched slab solves run one slab per process; in loopback that is G = 1 (no halo rows)
        require(np == 1 && d->nhalo == 0, "batched slab solves over the loopback transport need one slab (G = 1)");
    }
};

// ------------------------------------------------------------------ distributed PCG
static void ensure_g(rcg_dslab* d, int64_t count) {
    if (count <= d->cap_g) return;
    dev_free(d->gbuf);
    dev_free(d->ubuf);
    dev_free(d->u2buf);
    d->gbuf = dev_alloc(count);
    d->ubuf = dev_alloc(std::max<int64_t>(count, 128));
    d->u2buf = dev_alloc(std::max<int64_t>(count, 128));
    d->cap_g = count;
}

struct DistSolve {
    rcg_comm* comm;
    int ns;
    rcg_dslab* const* sl;
    int max_iter;
    double eps;
    const rcg_dbasis* defl = nullptr;  // deflated PCG (pcg.cpp:94-160)
    const rcg_dbasis* sc = nullptr;    // subspace correction around the block IC (subspace_correction.cpp)
    bool ic = false;
    rcg_sampler* const* smp = nullptr;   // error sampler per slab (solve 1 of the sequence), or null
    std::vector<Staged> bst, xst;
    std::vector<double*> bdev;

    int flags() const { return (defl ? 1 : 0) | (sc ? 2 : 0); }

    void setup(const double* const* b, double* const* x) {
        static bool smem_ok = false;
        if (!smem_ok) {
            allow_smem(reinterpret_cast<const void*>(k_d_residual));
            allow_smem(reinterpret_cast<const void*>(k_d_spmv));
            smem_ok = true;
        }
        ic = sl[0]->ic != nullptr;
        require(!(defl && sc), "dist_pcg_solve: deflation and subspace correction are exclusive");
        require(!sc || ic, "dist_pcg_solve: subspace correction needs the block IC(0) inner preconditioner");
        const int m = defl ? defl->m : (sc ? sc->m : 0);
        bst.resize(ns);
        xst.resize(ns);
        bdev.resize(ns);
        for (int s = 0; s < ns; ++s) {
            rcg_dslab* d = sl[s];
            rcg_ctx* ctx = d->ctx;
            const int32_t n = d->nloc;
            require((d->ic != nullptr) == ic, "dist_pcg_solve: every slab needs the same preconditioner kind");
            const int64_t ntiles = ic ? sweep_tiles(d->ic) : (n + kSweepThreads - 1) / kSweepThreads;
            const int64_t ngroups = (ntiles + kGroup - 1) / kGroup;
            const int64_t red = std::max<int64_t>(ntiles, static_cast<int64_t>(kMaxRed) * ctx->num_sms * 8);
            ensure_workspace(ctx, std::max(n, 1), std::max(m, 1), max_iter, red, ngroups, smp ? smp[s]->m : 1);
            ensure_g(d, std::max(m * m, 128));
            stage_in(ctx, b[s], n, bst[s]);
            bdev[s] = bst[s].dev;
            stage_in(ctx, x[s], n, xst[s]);
            if (n > 0)
                RCG_CK(cudaMemcpyAsync(d->xe, xst[s].dev, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream));
            DevState h{};
            h.done = kRunning;
            h.iter = 1;
            h.max_iter = max_iter;
            h.eps = eps;
            h.smp_method = -1;
            if (smp) {
                require(smp[s]->n == n, "dist_pcg_solve: sampler rows do not match the slab");
                h.smp_method = smp[s]->method;
                h.smp_m = smp[s]->m;
                h.smp_lmax = smp[s]->l_max;
                h.smp_h = smp[s]->h;
                h.smp_next = smp[s]->next_slot;
            }
            std::memcpy(ctx->host_pinned, &h, sizeof(h));
            RCG_CK(cudaMemcpyAsync(ctx->ws.st, ctx->host_pinned, sizeof(DevState), cudaMemcpyHostToDevice, ctx->stream));
            if (ic) {
                launch_fill_bits(ctx, ctx->ws.ybuf, n, kSentinelBits);
                launch_fill_bits(ctx, ctx->ws.zs, n, kSentinelBits);
            }
        }
        comm->begin(sl, ns);
    }

    SpmvArgs sargs(rcg_dslab* d, const double* xin, double* yout) {
        SpmvArgs a{};
        a.rs = d->a->rs;
        a.ci = d->a->ci;
        a.va = d->a->va;
        a.n = d->nloc;
        a.partials = d->ctx->ws.partials;
        a.x[0] = xin;
        a.y[0] = yout;
        return a;
    }

    void scalar(int stage, int goff = 0) {
        for (int s = 0; s < ns; ++s) {
            rcg_ctx* ctx = sl[s]->ctx;
            k_d_scalar<<<1, 1, 0, ctx->stream>>>(ctx->ws.st, sl[s]->dsum + goff, stage, ctx->ws.hist, ctx->ws.alph,
                                                 ctx->ws.bet, ic ? 0 : 1, flags());
            RCG_LAUNCHED(ctx);
        }
    }

    // Fused reductions (RCG_DIST_FUSE=0 keeps one allreduce per dot): with the IC
    // preconditioner the convergence check's (r, r) waits in dsum[1] for the next iteration's
    // (r, z) in dsum[0] -- one allreduce of two values instead of two of one.  Nothing between
    // the x / r update and the next sweeps reads the check's outcome, so every value is bitwise
    // the unfused loop's; a finished solve costs one extra pair of sweeps.  The pending check is
    // flushed before the host reads the stop flag (run()).
    bool pending_rr = false;
    bool fuse_rr() const {
        const char* e = std::getenv("RCG_DIST_FUSE");
        return ic && !sc && !(e && std::atoi(e) == 0);
    }
    // the (r, r) check (pcg.cpp:80-88) and the observer (sampling.cpp error_sampling_observer)
    void check_and_sample(int goff) {
        scalar(3, goff);
        if (!smp) return;
        for (int s = 0; s < ns; ++s) {
            rcg_dslab* d = sl[s];
            rcg_ctx* ctx = d->ctx;
            rcg_sampler* sp = smp[s];
            k_d_sched<<<1, 1, 0, ctx->stream>>>(ctx->ws.st, ctx->ws.smp_pending, sp->occupied, sp->stored_iter,
                                                sp->thresholds);
            RCG_LAUNCHED(ctx);
            k_d_sample<<<stream_grid(ctx, d->nloc), kStreamThreads, 0, ctx->stream>>>(
                d->xe, ctx->ws.r, sp->slots, sp->ld, ctx->ws.smp_pending, ctx->ws.st, d->nloc);
            RCG_LAUNCHED(ctx);
        }
    }
    void flush_pending() {
        if (!pending_rr) return;
        pending_rr = false;
        comm->allreduce(sl, ns, 2);  // (dsum[0] rides along unused)
        check_and_sample(1);
    }

    // f = C^T y over the local rows -> allreduce (m values) -> out = (W^T A W)^-1 f on every slab
    void project_coeffs(const rcg_dbasis* B, bool use_aw, double* const* ys, bool to_u2, int mode, int respect_done) {
        const int m = B->m;
        for (int s = 0; s < ns; ++s) {
            rcg_dslab* d = sl[s];
            rcg_ctx* ctx = d->ctx;
            k_tallt<<<stream_grid(ctx, d->nloc), kStreamThreads, 0, ctx->stream>>>(
                use_aw ? B->aw[s] : B->w[s], d->nloc, m, ys[s], d->nloc, ctx->ws.partials, nullptr, d->gbuf, 0,
                ctx->ws.st, respect_done);
            RCG_LAUNCHED(ctx);
        }
        comm->allreduce(sl, ns, m, 1);
        for (int s = 0; s < ns; ++s) {
            rcg_dslab* d = sl[s];
            k_d_chol<<<1, 32, 0, d->ctx->stream>>>(B->l[s], m, d->gbuf, to_u2 ? d->u2buf : d->ubuf, d->ctx->ws.st, mode,
                                                   respect_done);
            RCG_LAUNCHED(d->ctx);
        }
    }

    void initial() {
        comm->halo(sl, ns, 0);
        for (int s = 0; s < ns; ++s) {
            rcg_dslab* d = sl[s];
            rcg_ctx* ctx = d->ctx;
            k_d_residual<<<spmv_grid(ctx, d->nloc), kSpmvThreads, spmv_smem(d->a), ctx->stream>>>(
                sargs(d, d->xe, nullptr), d->a->cap, bdev[s], ctx->ws.r, ctx->ws.st, d->dsum);
            RCG_LAUNCHED(ctx);
        }
        comm->allreduce(sl, ns, 2);
        scalar(0);
        std::vector<double*> rs(ns);
        for (int s = 0; s < ns; ++s) rs[s] = sl[s]->ctx->ws.r;
        if (defl) {  // r = P^T r and the check on the projected residual (pcg.cpp:112-118)
            project_coeffs(defl, false, rs.data(), false, 1, 1);
            for (int s = 0; s < ns; ++s) {
                rcg_dslab* d = sl[s];
                rcg_ctx* ctx = d->ctx;
                k_d_deflate<<<stream_grid(ctx, d->nloc), kStreamThreads, 0, ctx->stream>>>(
                    ctx->ws.r, defl->aw[s], d->nloc, defl->m, d->ubuf, nullptr, d->nloc, ctx->ws.partials, ctx->ws.st,
                    d->dsum, 1);
                RCG_LAUNCHED(ctx);
            }
            comm->allreduce(sl, ns, 1);
            scalar(4);
        }
        if (sc) project_coeffs(sc, false, rs.data(), true, 2, 1);  // u2 = chol(W^T r), f . u
    }

    void iteration() {
        if (ic) {
            for (int s = 0; s < ns; ++s) {
                rcg_dslab* d = sl[s];
                rcg_ctx* ctx = d->ctx;
                SweepArgs fa = sweep_args(ctx, d->ic, false);
                fa.in = ctx->ws.r;
                fa.out = ctx->ws.ybuf;
                launch_sweep(ctx, d->ic, false, fa);
                SweepArgs ba = sweep_args(ctx, d->ic, true);
                ba.in = ctx->ws.ybuf;
                ba.out = ctx->ws.zs;
                launch_sweep(ctx, d->ic, true, ba);
                k_d_dot<<<stream_grid(ctx, d->nloc), kStreamThreads, 0, ctx->stream>>>(
                    ctx->ws.r, ctx->ws.zs, d->nloc, ctx->ws.partials, ctx->ws.st, d->dsum);
                RCG_LAUNCHED(ctx);
            }
            if (pending_rr) {  // [(r, z) | the previous iteration's (r, r)]: check + observer, then rho
                pending_rr = false;
                comm->allreduce(sl, ns, 2);
                check_and_sample(1);
            } else {
                comm->allreduce(sl, ns, 1);
            }
            scalar(1);  // (+ f . u with subspace correction)
        }
        for (int s = 0; s < ns; ++s) {
            rcg_dslab* d = sl[s];
            rcg_ctx* ctx = d->ctx;
            KTimer t(ctx, 3);
            k_pupdate<<<stream_grid(ctx, d->nloc), kStreamThreads, 0, ctx->stream>>>(
                ic ? ctx->ws.zs : ctx->ws.r, d->pe, ic ? ctx->ws.zs : nullptr, ctx->ws.ybuf, d->nloc, ctx->ws.st,
                sc ? sc->w[s] : nullptr, d->nloc, sc ? sc->m : 0, d->u2buf);
            RCG_LAUNCHED(ctx);
        }
        comm->halo(sl, ns, 1);
        for (int s = 0; s < ns; ++s) {
            rcg_dslab* d = sl[s];
            rcg_ctx* ctx = d->ctx;
            KTimer t(ctx, 0);
            k_d_spmv<<<spmv_grid(ctx, d->nloc), kSpmvThreads, spmv_smem(d->a), ctx->stream>>>(
                sargs(d, d->pe, ctx->ws.q), d->a->cap, ctx->ws.st, d->dsum);
            RCG_LAUNCHED(ctx);
        }
        if (defl) {  // q = P^T q (pcg.cpp:131), then (p, q)
            std::vector<double*> qs(ns);
            for (int s = 0; s < ns; ++s) qs[s] = sl[s]->ctx->ws.q;
            project_coeffs(defl, false, qs.data(), false, 1, 1);
            for (int s = 0; s < ns; ++s) {
                rcg_dslab* d = sl[s];
                rcg_ctx* ctx = d->ctx;
                k_d_deflate<<<stream_grid(ctx, d->nloc), kStreamThreads, 0, ctx->stream>>>(
                    ctx->ws.q, defl->aw[s], d->nloc, defl->m, d->ubuf, d->pe, d->nloc, ctx->ws.partials, ctx->ws.st,
                    d->dsum, 0);
                RCG_LAUNCHED(ctx);
            }
        }
        comm->allreduce(sl, ns, 1);
        scalar(2);
        const bool defer_rr = fuse_rr();
        for (int s = 0; s < ns; ++s) {
            rcg_dslab* d = sl[s];
            rcg_ctx* ctx = d->ctx;
            KTimer t(ctx, 3);
            k_d_xr<<<stream_grid(ctx, d->nloc), kStreamThreads, 0, ctx->stream>>>(
                d->xe, ctx->ws.r, d->pe, ctx->ws.q, d->nloc, ctx->ws.partials, ctx->ws.st, d->dsum + (defer_rr ? 1 : 0));
            RCG_LAUNCHED(ctx);
        }
        if (defer_rr) {
            pending_rr = true;
        } else {
            comm->allreduce(sl, ns, 1);
            check_and_sample(0);
        }
        if (sc) {  // W^T r for the next apply (subspace_correction.cpp:50-51)
            std::vector<double*> rs(ns);
            for (int s = 0; s < ns; ++s) rs[s] = sl[s]->ctx->ws.r;
            project_coeffs(sc, false, rs.data(), true, 2, 1);
        }
    }

    // same batching as the single-GPU loop; every slab holds identical scalars, slab 0 is polled
    double run() {
        rcg_ctx* c0 = sl[0]->ctx;
        cudaEvent_t evs[2], t0, t1;
        RCG_CK(cudaEventCreateWithFlags(&evs[0], cudaEventDisableTiming));
        RCG_CK(cudaEventCreateWithFlags(&evs[1], cudaEventDisableTiming));
        RCG_CK(cudaEventCreate(&t0));
        RCG_CK(cudaEventCreate(&t1));
        RCG_CK(cudaEventRecord(t0, c0->stream));
        volatile int* flags_h = reinterpret_cast<volatile int*>(c0->host_pinned + 256);
        flags_h[0] = flags_h[1] = 0;
        int enq = 0, batch = 2, slot = 0, prev = 0;
        bool have_prev = false;
        while (true) {
            for (int j = 0; j < batch && enq < max_iter; ++j, ++enq) iteration();
            flush_pending();
            RCG_CK(cudaMemcpyAsync((void*)(flags_h + slot), &c0->ws.st->done, sizeof(int), cudaMemcpyDeviceToHost,
                                   c0->stream));
            RCG_CK(cudaEventRecord(evs[slot], c0->stream));
            if (enq >= max_iter) {
                RCG_CK(cudaEventSynchronize(evs[slot]));
                break;
            }
            if (have_prev) {
                RCG_CK(cudaEventSynchronize(evs[prev]));
                if (flags_h[prev] != kRunning) break;
            }
            have_prev = true;
            prev = slot;
            slot ^= 1;
            batch = std::min(batch * 2, 16);
        }
        for (int s = 0; s < ns; ++s) RCG_CK(cudaStreamSynchronize(sl[s]->ctx->stream));
        RCG_CK(cudaEventRecord(t1, c0->stream));
        RCG_CK(cudaEventSynchronize(t1));
        float ms = 0.f;
        RCG_CK(cudaEventElapsedTime(&ms, t0, t1));
        for (auto e : {evs[0], evs[1], t0, t1}) cudaEventDestroy(e);
        return ms * 1e-3;
    }

    DevState finish(double* const* x) {
        for (int s = 0; s < ns; ++s) {
            rcg_dslab* d = sl[s];
            k_zero_if<<<stream_grid(d->ctx, d->nloc), kStreamThreads, 0, d->ctx->stream>>>(d->xe, d->nloc,
                                                                                          d->ctx->ws.st);
            RCG_LAUNCHED(d->ctx);
        }
        if (defl) {  // x = P x + W (W^T A W)^-1 W^T b (pcg.cpp:152-157), skipped for breakdown / zero rhs
            std::vector<double*> xs(ns), bs(ns);
            for (int s = 0; s < ns; ++s) {
                xs[s] = sl[s]->xe;
                bs[s] = bdev[s];
            }
            project_coeffs(defl, true, xs.data(), false, 1, 0);
            for (int s = 0; s < ns; ++s) {
                rcg_dslab* d = sl[s];
                k_sub_combination_ok<<<stream_grid(d->ctx, d->nloc), kStreamThreads, 0, d->ctx->stream>>>(
                    d->xe, defl->w[s], d->nloc, defl->m, d->ubuf, d->nloc, d->ctx->ws.st);
                RCG_LAUNCHED(d->ctx);
            }
            project_coeffs(defl, false, bs.data(), true, 1, 0);
            for (int s = 0; s < ns; ++s) {
                rcg_dslab* d = sl[s];
                k_add_combination<<<stream_grid(d->ctx, d->nloc), kStreamThreads, 0, d->ctx->stream>>>(
                    d->xe, defl->w[s], d->nloc, defl->m, d->u2buf, d->nloc, d->ctx->ws.st, 1);
                RCG_LAUNCHED(d->ctx);
            }
        }
        for (int s = 0; s < ns; ++s) {
            rcg_dslab* d = sl[s];
            rcg_ctx* ctx = d->ctx;
            const int32_t n = d->nloc;
            Staged out;
            stage_out_begin(ctx, x[s], n, out);
            if (n > 0)
                RCG_CK(cudaMemcpyAsync(out.dev, d->xe, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream));
            stage_out_end(ctx, x[s], n, out);
            RCG_CK(cudaStreamSynchronize(ctx->stream));
            if (ic) check_sweep_watchdog(ctx);
        }
        rcg_ctx* c0 = sl[0]->ctx;
        DevState h{};
        RCG_CK(cudaMemcpy(&h, c0->ws.st, sizeof(DevState), cudaMemcpyDeviceToHost));
        if (smp)
            for (int s = 0; s < ns; ++s) {  // the schedule state the sampler carries on (h, next slot)
                DevState hs{};
                RCG_CK(cudaMemcpy(&hs, sl[s]->ctx->ws.st, sizeof(DevState), cudaMemcpyDeviceToHost));
                smp[s]->h = hs.smp_h;
                smp[s]->next_slot = hs.smp_next;
            }
        return h;
    }
};

// W (local rows of every slab) -> AW by m halo exchanges + local SpMVs, the Gram W^T A W (lower
// triangle mirrored, as rcg_basis_create) allreduced, factored once on the host from the
// identical totals, the factor uploaded to every slab
static rcg_dbasis* dbasis_create(rcg_comm* comm, int ns, rcg_dslab* const* sl, const double* const* wcols, int m,
                                 int kind) {
    auto* B = new rcg_dbasis();
    B->kind = kind;
    B->m = m;
    try {
        for (int s = 0; s < ns; ++s) {
            rcg_dslab* d = sl[s];
            rcg_ctx* ctx = d->ctx;
            const int64_t sz = static_cast<int64_t>(d->nloc) * m;
            B->w.push_back(dev_alloc(std::max<int64_t>(sz, 1)));
            B->aw.push_back(dev_alloc(std::max<int64_t>(sz, 1)));
            B->l.push_back(dev_alloc(static_cast<int64_t>(std::max(m, 1)) * std::max(m, 1)));
            Staged wst;
            stage_in(ctx, wcols[s], sz, wst);
            if (sz) RCG_CK(cudaMemcpyAsync(B->w[s], wst.dev, sizeof(double) * sz, cudaMemcpyDeviceToDevice, ctx->stream));
            RCG_CK(cudaStreamSynchronize(ctx->stream));
            ensure_g(d, std::max(m * m, 128));
        }
        comm->begin(sl, ns);
        for (int j = 0; j < m; ++j) {
            for (int s = 0; s < ns; ++s) {
                rcg_dslab* d = sl[s];
                if (d->nloc)
                    RCG_CK(cudaMemcpyAsync(d->pe, B->w[s] + static_cast<int64_t>(j) * d->nloc, sizeof(double) * d->nloc,
                                           cudaMemcpyDeviceToDevice, d->ctx->stream));
            }
            comm->halo(sl, ns, 1);
            for (int s = 0; s < ns; ++s) {
                rcg_dslab* d = sl[s];
                const int rc = rcg_spmv(d->ctx, d->a, d->pe, B->aw[s] + static_cast<int64_t>(j) * d->nloc);
                if (rc != RCG_OK) throw Error(rc, rcg_last_error());
            }
        }
        std::vector<double> g;
        for (int s = 0; s < ns; ++s) {
            rcg_dslab* d = sl[s];
            gram_host(d->ctx, B->w[s], d->nloc, m, B->aw[s], d->nloc, m, d->nloc, true, g);
            h2d_sync(d->ctx, d->gbuf, g.data(), sizeof(double) * m * m);
        }
        comm->allreduce(sl, ns, m * m, 1);
        for (int s = 0; s < ns; ++s) RCG_CK(cudaStreamSynchronize(sl[s]->ctx->stream));
        g.assign(static_cast<size_t>(m) * m, 0.0);
        RCG_CK(cudaMemcpy(g.data(), sl[0]->gbuf, sizeof(double) * m * m, cudaMemcpyDeviceToHost));
        for (int i = 0; i < m; ++i)
            for (int j = 0; j < i; ++j) g[static_cast<size_t>(j) * m + i] = g[static_cast<size_t>(i) * m + j];
        int bad = -1;
        if (!chol_factor_host(m, g, B->h_l, &bad)) throw Error(RCG_E_BREAKDOWN, "distributed basis: W^T A W not SPD");
        for (int s = 0; s < ns; ++s)
            h2d_sync(sl[s]->ctx, B->l[s], B->h_l.data(), sizeof(double) * m * m);
    } catch (...) {
        for (auto p : B->w) dev_free(p);
        for (auto p : B->aw) dev_free(p);
        for (auto p : B->l) dev_free(p);
        delete B;
        throw;
    }
    return B;
}

// The sequence's recycling step over row slabs: harvest_errors (recycling.cpp:17-28)
// per slab with the exactly-zero-column test made global, single-pass MGS (dense.cpp:45-61) with
// every dot allreduced (the drop test sees the global norms), A Q by halo exchange + local SpMV,
// the Gram Q^T A Q allreduced and eigensolved identically on every rank (cyclic Jacobi,
// dense.cpp:63-144), count / theta selection (recycling.cpp:91-94), Ritz vectors W = Q T_sel per
// slab, then the distributed deflation / SC state (dbasis_create).  Returns null when no Ritz
// value is selected (empty W: the accelerated solves are plain block-Jacobi PCG, as the reference).
static rcg_dbasis* dist_recycle(rcg_comm* comm, int ns, rcg_dslab* const* sl, rcg_sampler* const* smp,
                                const double* const* xfin, double theta, int keep_count, int kind, int* m_bar,
                                std::vector<double>& vals, double* theta_used, int* m_tilde) {
    const int msl = smp[0]->m;
    std::vector<int> occ(std::max(msl, 1), 0);
    if (msl) RCG_CK(cudaMemcpy(occ.data(), smp[0]->occupied, sizeof(int) * msl, cudaMemcpyDeviceToHost));
    std::vector<int> list;
    for (int j = 0; j < msl; ++j)
        if (occ[j]) list.push_back(j);
    const int k0 = static_cast<int>(list.size());
    struct Loc {
        double *e = nullptr, *q = nullptr, *aq = nullptr, *w = nullptr, *c = nullptr, *y = nullptr;
        int *nz = nullptr, *dl = nullptr;
        Staged x;
        double *eb = nullptr, *qb = nullptr;  // error / basis blocks (own buffers, or the slots when lean)
        int64_t eld = 0, qld = 0;
    };
    std::vector<Loc> L(ns);
    // Memory-lean mode (RCG_DIST_LEAN=1, or automatically when the error block, its MGS copy and
    // A Q do not fit next to the slots -- C4 at G = 1-2): the errors and the MGS basis live in the
    // sampler slots and the Gram is streamed (one n-vector), as lean_build_aux on one GPU; the
    // slots are released once W is formed (the samplers are spent).
    bool lean = std::getenv("RCG_DIST_LEAN") && std::atoi(std::getenv("RCG_DIST_LEAN")) == 1;
    if (!lean) {
        size_t fr = 0, tot = 0;
        RCG_CK(cudaMemGetInfo(&fr, &tot));
        double need = 0.0;
        for (int s = 0; s < ns; ++s) need += 3.0 * k0 * 8.0 * static_cast<double>(sl[s]->nloc);
        lean = static_cast<double>(fr) < 1.1 * need;  // (loopback slabs share one GPU)
    }
    auto cleanup = [&] {
        for (auto& l : L) {
            for (double* p : {l.e, l.q, l.aq, l.w, l.c, l.y}) dev_free(p);
            dev_free(l.nz);
            dev_free(l.dl);
        }
    };
    rcg_dbasis* out = nullptr;
    try {
        comm->begin(sl, ns);
        for (int s = 0; s < ns; ++s) {
            rcg_dslab* d = sl[s];
            rcg_ctx* ctx = d->ctx;
            const int32_t n = d->nloc;
            require(smp[s]->n == n && smp[s]->m == msl, "dist_recycle: samplers do not match the slabs");
            ensure_workspace(ctx, std::max(n, 1), kMaxRed, 1,
                             std::max<int64_t>((n + kSweepThreads - 1) / kSweepThreads, int64_t(kMaxRed) * ctx->num_sms * 8),
                             1, 1);
            ensure_g(d, std::max({k0 * k0, k0, 128}));
            stage_in(ctx, xfin[s], n, L[s].x);
            const int64_t sz = std::max<int64_t>(int64_t(n) * std::max(k0, 1), 1);
            if (lean) {
                L[s].eb = L[s].qb = smp[s]->slots;
                L[s].eld = L[s].qld = smp[s]->ld;
                L[s].y = dev_alloc(std::max<int64_t>(n, 1));
            } else {
                L[s].e = dev_alloc(sz);
                L[s].q = dev_alloc(sz);
                L[s].aq = dev_alloc(sz);
                L[s].eb = L[s].e;
                L[s].qb = L[s].q;
                L[s].eld = L[s].qld = n;
            }
            L[s].c = dev_alloc(4);
            L[s].nz = static_cast<int*>(dev_alloc_bytes(sizeof(int) * std::max(k0, 1)));
            L[s].dl = static_cast<int*>(dev_alloc_bytes(sizeof(int) * std::max(k0, 1)));
            RCG_CK(cudaMemsetAsync(L[s].nz, 0, sizeof(int) * std::max(k0, 1), ctx->stream));
            if (k0) {
                RCG_CK(cudaMemcpyAsync(L[s].dl, list.data(), sizeof(int) * k0, cudaMemcpyHostToDevice, ctx->stream));
                if (n) {
                    dim3 grid(stream_grid(ctx, n), std::min(k0, 64));
                    if (lean)  // column j of the errors stays in slot list[j]
                        k_harvest_inplace<<<grid, kStreamThreads, 0, ctx->stream>>>(L[s].x.dev, smp[s]->slots, smp[s]->ld,
                                                                                    L[s].dl, k0, n, L[s].nz);
                    else
                        k_harvest<<<grid, kStreamThreads, 0, ctx->stream>>>(L[s].x.dev, smp[s]->slots, smp[s]->ld,
                                                                            L[s].dl, k0, 0, L[s].e, n, n, L[s].nz);
                    RCG_LAUNCHED(ctx);
                }
            }
        }
        // exactly-zero columns are skipped globally (recycling.cpp:26): sum the per-slab flags
        std::vector<int> cols;
        if (k0) {
            for (int s = 0; s < ns; ++s) {
                std::vector<int> hz(k0);
                RCG_CK(cudaMemcpyAsync(hz.data(), L[s].nz, sizeof(int) * k0, cudaMemcpyDeviceToHost, sl[s]->ctx->stream));
                RCG_CK(cudaStreamSynchronize(sl[s]->ctx->stream));
                std::vector<double> hd(hz.begin(), hz.end());
                h2d_sync(sl[s]->ctx, sl[s]->gbuf, hd.data(), sizeof(double) * k0);
            }
            comm->allreduce(sl, ns, k0, 1);
            for (int s = 0; s < ns; ++s) RCG_CK(cudaStreamSynchronize(sl[s]->ctx->stream));
            std::vector<double> g(k0);
            RCG_CK(cudaMemcpy(g.data(), sl[0]->gbuf, sizeof(double) * k0, cudaMemcpyDeviceToHost));
            for (int j = 0; j < k0; ++j)
                if (g[j] > 0.0) cols.push_back(j);
        }
        // allreduced (u, v) of every slab's local rows -> dsum[0] on every slab; returns the total
        auto gdot = [&](auto ucol, auto vcol, bool read) {
            for (int s = 0; s < ns; ++s) {
                rcg_dslab* d = sl[s];
                rcg_ctx* ctx = d->ctx;
                k_rr_dot<<<stream_grid(ctx, d->nloc), kStreamThreads, 0, ctx->stream>>>(
                    ucol(s), vcol(s), d->nloc, ctx->ws.partials, &ctx->ws.st->tick[kDistTick], d->dsum);
                RCG_LAUNCHED(ctx);
            }
            comm->allreduce(sl, ns, 1, 0);
            double h = 0.0;
            if (read) {
                for (int s = 0; s < ns; ++s) RCG_CK(cudaStreamSynchronize(sl[s]->ctx->stream));
                RCG_CK(cudaMemcpy(&h, sl[0]->dsum, sizeof(double), cudaMemcpyDeviceToHost));
            }
            return h;
        };
        int kept = 0;
        // error column src: column src of the own block, or slot list[src] in place (lean: the
        // basis column `kept` <= src <= list[src] is never a later source)
        auto ecol = [&](int s, int src) { return L[s].eb + int64_t(lean ? list[src] : src) * L[s].eld; };
        for (int src : cols) {
            auto wcol = [&](int s) { return L[s].qb + int64_t(kept) * L[s].qld; };
            for (int s = 0; s < ns; ++s)
                if (sl[s]->nloc && wcol(s) != ecol(s, src))
                    RCG_CK(cudaMemcpyAsync(wcol(s), ecol(s, src), sizeof(double) * sl[s]->nloc, cudaMemcpyDeviceToDevice,
                                           sl[s]->ctx->stream));
            const double n0 = std::sqrt(gdot(wcol, wcol, true));
            if (n0 == 0.0) continue;
            for (int qi = 0; qi < kept; ++qi) {
                auto qcol = [&](int s) { return L[s].qb + int64_t(qi) * L[s].qld; };
                gdot(qcol, wcol, false);
                for (int s = 0; s < ns; ++s) {
                    rcg_ctx* ctx = sl[s]->ctx;
                    k_rr_axpy<<<stream_grid(ctx, sl[s]->nloc), kStreamThreads, 0, ctx->stream>>>(
                        wcol(s), qcol(s), sl[s]->dsum, sl[s]->nloc, 0);
                    RCG_LAUNCHED(ctx);
                }
            }
            const double n1 = std::sqrt(gdot(wcol, wcol, true));
            if (n1 <= 1e-12 * n0) continue;   // numerically dependent, dropped (dense.cpp:56)
            for (int s = 0; s < ns; ++s) {
                rcg_ctx* ctx = sl[s]->ctx;
                k_rr_axpy<<<stream_grid(ctx, sl[s]->nloc), kStreamThreads, 0, ctx->stream>>>(
                    wcol(s), nullptr, sl[s]->dsum, sl[s]->nloc, 1);
                RCG_LAUNCHED(ctx);
            }
            ++kept;
        }
        *m_bar = kept;
        vals.clear();
        if (kept == 0) {
            cleanup();
            if (theta_used) *theta_used = theta;
            *m_tilde = 0;
            return nullptr;
        }
        require(kept <= 128, "SmallSym: dimension " + std::to_string(kept) + " outside [0, 128]");
        // A Q (rayleigh_ritz, recycling.cpp:48-53): halo exchange + local SpMV per column; lean:
        // each column's local Q^T (A q_j) right away (streamed Gram), no A Q block
        std::vector<std::vector<double>> sloc(ns, std::vector<double>(static_cast<size_t>(kept) * kept, 0.0));
        for (int j = 0; j < kept; ++j) {
            for (int s = 0; s < ns; ++s) {
                rcg_dslab* d = sl[s];
                if (d->nloc)
                    RCG_CK(cudaMemcpyAsync(d->pe, L[s].qb + int64_t(j) * L[s].qld, sizeof(double) * d->nloc,
                                           cudaMemcpyDeviceToDevice, d->ctx->stream));
            }
            comm->halo(sl, ns, 1);
            for (int s = 0; s < ns; ++s) {
                rcg_dslab* d = sl[s];
                double* yj = lean ? L[s].y : L[s].aq + int64_t(j) * d->nloc;
                const int rc = rcg_spmv(d->ctx, d->a, d->pe, yj);
                if (rc != RCG_OK) throw Error(rc, rcg_last_error());
                if (lean) {
                    std::vector<double> f;
                    gram_host(d->ctx, L[s].qb, L[s].qld, kept, yj, d->nloc, 1, d->nloc, false, f);
                    for (int i = j; i < kept; ++i) sloc[s][static_cast<size_t>(i) * kept + j] = f[i];
                }
            }
        }
        // S = Q^T A Q, lower triangle allreduced then mirrored, eigensolved on every rank
        std::vector<double> g;
        for (int s = 0; s < ns; ++s) {
            rcg_dslab* d = sl[s];
            if (lean)
                g = sloc[s];
            else
                gram_host(d->ctx, L[s].q, d->nloc, kept, L[s].aq, d->nloc, kept, d->nloc, true, g);
            h2d_sync(d->ctx, d->gbuf, g.data(), sizeof(double) * kept * kept);
        }
        comm->allreduce(sl, ns, kept * kept, 1);
        for (int s = 0; s < ns; ++s) RCG_CK(cudaStreamSynchronize(sl[s]->ctx->stream));
        g.assign(static_cast<size_t>(kept) * kept, 0.0);
        RCG_CK(cudaMemcpy(g.data(), sl[0]->gbuf, sizeof(double) * kept * kept, cudaMemcpyDeviceToHost));
        for (int i = 0; i < kept; ++i)
            for (int j = 0; j < i; ++j) g[static_cast<size_t>(j) * kept + i] = g[static_cast<size_t>(i) * kept + j];
        std::vector<double> T;
        sym_eig_host(kept, g, vals, T);
        double th = theta;
        if (keep_count > 0)
            th = kept > keep_count ? 0.5 * (vals[keep_count - 1] + vals[keep_count]) : std::numeric_limits<double>::infinity();
        if (theta_used) *theta_used = th;
        int sel = 0;
        while (sel < kept && vals[sel] < th) ++sel;
        *m_tilde = sel;
        if (sel > 0) {
            std::vector<const double*> wp(ns);
            for (int s = 0; s < ns; ++s) {
                rcg_dslab* d = sl[s];
                L[s].w = dev_alloc(std::max<int64_t>(int64_t(d->nloc) * sel, 1));
                combine_cols(d->ctx, L[s].qb, L[s].qld, kept, T.data(), sel, L[s].w, d->nloc, d->nloc);
                wp[s] = L[s].w;
            }
            for (int s = 0; s < ns; ++s) RCG_CK(cudaStreamSynchronize(sl[s]->ctx->stream));
            if (lean)  // the samplers are spent: their slots make room for W's copy and A W
                for (int s = 0; s < ns; ++s) {
                    dev_free(smp[s]->slots);
                    smp[s]->slots = nullptr;
                }
            out = dbasis_create(comm, ns, sl, wp.data(), sel, kind);
        }
    } catch (...) {
        cleanup();
        throw;
    }
    cleanup();
    return out;
}

}  // namespace rcg

using namespace rcg;

extern "C" {

int rcg_slab_plan_create(int32_t n, const int32_t* row_start, const int32_t* col_idx, const double* values,
                         int nparts, int part, rcg_slab_plan* out) {
    return guard([&] {
        try {
            plan_create(n, row_start, col_idx, values, nparts, part, out);
        } catch (...) {
            plan_free(out);
            throw;
        }
    });
}

void rcg_slab_plan_free(rcg_slab_plan* plan) { plan_free(plan); }

int rcg_dslab_create(rcg_ctx* ctx, const rcg_slab_plan* p, const rcg_ic* ic, rcg_dslab** out) {
    return guard([&] {
        require(ctx && p && out, "rcg_dslab_create: null argument");
        *out = nullptr;
        if (ic) require(ic->n == p->nloc, "rcg_dslab_create: factor size does not match the slab's rows");
        RCG_CK(cudaSetDevice(ctx->device));
        auto* d = new rcg_dslab();
        try {
            d->ctx = ctx;
            d->ic = ic;
            d->nparts = p->nparts;
            d->part = p->part;
            d->nloc = p->nloc;
            d->nhalo = p->nhalo;
            d->row_begin = p->row_begin;
            rcg_matrix* a = nullptr;
            const int rc = rcg_matrix_create(ctx, p->nloc, p->row_start, p->col_idx, p->values, 0, &a);
            if (rc != RCG_OK) throw Error(rc, rcg_last_error());
            d->a = a;
            d->send_count.assign(p->send_count, p->send_count + p->nparts);
            d->recv_count.assign(p->recv_count, p->recv_count + p->nparts);
            d->send_off.assign(p->nparts, 0);
            d->recv_off.assign(p->nparts, 0);
            for (int q = 1; q < p->nparts; ++q) {
                d->send_off[q] = d->send_off[q - 1] + d->send_count[q - 1];
                d->recv_off[q] = d->recv_off[q - 1] + d->recv_count[q - 1];
            }
            d->nsend = p->nparts > 0 ? d->send_off[p->nparts - 1] + d->send_count[p->nparts - 1] : 0;
            d->send_idx = static_cast<int32_t*>(dev_alloc_bytes(sizeof(int32_t) * std::max(d->nsend, 1)));
            if (d->nsend)
                h2d_sync(d->ctx, d->send_idx, p->send_idx, sizeof(int32_t) * d->nsend);
            d->sendbuf = dev_alloc(std::max(d->nsend, 1));
            d->xe = dev_alloc(static_cast<int64_t>(d->nloc) + d->nhalo);
            d->pe = dev_alloc(static_cast<int64_t>(d->nloc) + d->nhalo);
            d->dsum = dev_alloc(4);
            RCG_CK(cudaMemset(d->xe, 0, sizeof(double) * (static_cast<int64_t>(d->nloc) + d->nhalo)));
            RCG_CK(cudaMemset(d->pe, 0, sizeof(double) * (static_cast<int64_t>(d->nloc) + d->nhalo)));
            RCG_CK(cudaMemset(d->dsum, 0, sizeof(double) * 4));
        } catch (...) {
            rcg_dslab_destroy(d);
            throw;
        }
        *out = d;
    });
}

void rcg_dslab_destroy(rcg_dslab* d) {
    if (!d) return;
    // the device, not the (borrowed) context: a caller may already have destroyed the context
    cudaDeviceSynchronize();
    rcg_matrix_destroy(d->a);
    for (void* p : {(void*)d->send_idx, (void*)d->sendbuf, (void*)d->xe, (void*)d->pe, (void*)d->dsum, (void*)d->gbuf,
                    (void*)d->ubuf, (void*)d->u2buf, (void*)d->sendbuf_rt})
        dev_free(p);
    delete d;
}

int rcg_comm_nccl_unique_id(void* id128) {
    return guard([&] {
        require(id128 != nullptr, "rcg_comm_nccl_unique_id: null argument");
        static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
        Nccl& nc = Nccl::get();
        ncclUniqueId id;
        nc.check(nc.get_unique_id(&id), "get unique id");
        std::memcpy(id128, &id, sizeof(id));
    });
}

int rcg_comm_create_nccl(const void* id128, int nranks, int rank, rcg_comm** out) {
    return guard([&] {
        require(id128 && out && nranks >= 1 && rank >= 0 && rank < nranks, "rcg_comm_create_nccl: bad argument");
        *out = nullptr;
        Nccl& nc = Nccl::get();
        auto* c = new NcclComm();
        c->nranks = nranks;
        c->rank = rank;
        ncclUniqueId id;
        std::memcpy(&id, id128, sizeof(id));
        try {
            nc.check(nc.comm_init_rank(&c->comm, nranks, id, rank), "comm init");
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

int rcg_comm_create_loopback(int nparts, rcg_comm** out) {
    return guard([&] {
        require(out && nparts >= 1, "rcg_comm_create_loopback: bad argument");
        *out = nullptr;
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
            cudaGetLastError();
            throw Error(RCG_E_CUDA, "no CUDA device available: librcg_b200 has no CPU fallback");
        }
        auto* c = new LoopComm();
        c->np = nparts;
        RCG_CK(cudaGetDevice(&c->dev));
        RCG_CK(cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking));
        RCG_CK(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
        c->ev.resize(nparts);
        for (auto& e : c->ev) RCG_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->ev_read.resize(nparts);
        for (auto& e : c->ev_read) RCG_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->dptrs = static_cast<double**>(dev_alloc_bytes(sizeof(double*) * nparts));
        c->gptrs = static_cast<double**>(dev_alloc_bytes(sizeof(double*) * nparts));
        *out = c;
    });
}

int rcg_comm_create_host(int nranks, int rank, rcg_host_allreduce_fn allreduce, rcg_host_exchange_fn exchange,
                         void* user, rcg_comm** out) {
    return guard([&] {
        require(out && allreduce && exchange && nranks >= 1 && rank >= 0 && rank < nranks,
                "rcg_comm_create_host: bad argument");
        auto* c = new HostComm();
        c->nranks = nranks;
        c->rank = rank;
        c->ar = allreduce;
        c->ex = exchange;
        c->user = user;
        *out = c;
    });
}

void rcg_comm_destroy(rcg_comm* c) { delete c; }

int rcg_dbasis_create(rcg_comm* comm, int nslabs, rcg_dslab* const* slabs, const double* const* w, int m, int kind,
                      rcg_dbasis** out) {
    return guard([&] {
        require(comm && slabs && w && out, "rcg_dbasis_create: null argument");
        *out = nullptr;
        require(nslabs == comm->local_slabs(), "rcg_dbasis_create: slab count does not match the transport");
        require(m >= 1 && m <= 128, "rcg_dbasis_create: m must be in [1, 128]");
        require(kind == RCG_BASIS_DEFLATION || kind == RCG_BASIS_SC, "rcg_dbasis_create: unknown basis kind");
        for (int s = 0; s < nslabs; ++s) require(slabs[s] && w[s], "rcg_dbasis_create: null slab / W");
        *out = dbasis_create(comm, nslabs, slabs, w, m, kind);
    });
}

void rcg_dbasis_destroy(rcg_dbasis* b) {
    if (!b) return;
    for (auto p : b->w) dev_free(p);
    for (auto p : b->aw) dev_free(p);
    for (auto p : b->l) dev_free(p);
    delete b;
}

static int dist_solve_impl(rcg_comm* comm, int nslabs, rcg_dslab* const* slabs, const rcg_dbasis* basis,
                           rcg_sampler* const* observers, const double* const* b, double* const* x,
                           const rcg_solver_config* cfg, rcg_solve_report* report) {
    return guard([&] {
        require(comm && slabs && b && x && report, "dist_pcg_solve: null argument");
        require(nslabs == comm->local_slabs(), "dist_pcg_solve: slab count does not match the transport");
        check_cfg(cfg);
        for (int s = 0; s < nslabs; ++s) {
            require(slabs[s] && b[s] && x[s], "dist_pcg_solve: null slab / vector");
            require(slabs[s]->nparts == comm->nparts(), "dist_pcg_solve: slab partition does not match the transport");
            if (nslabs > 1) require(slabs[s]->part == s, "dist_pcg_solve: loopback slabs must be given in part order");
        }
        if (basis) require(static_cast<int>(basis->w.size()) == nslabs, "dist_pcg_solve: basis built for other slabs");
        DistSolve ds{comm, nslabs, slabs, cfg->max_iter, cfg->eps};
        if (observers)
            for (int s = 0; s < nslabs; ++s) require(observers[s] != nullptr, "dist_pcg_solve: null sampler");
        ds.smp = observers;
        if (basis && basis->kind == RCG_BASIS_DEFLATION) ds.defl = basis;
        if (basis && basis->kind == RCG_BASIS_SC) ds.sc = basis;
        ds.setup(b, x);
        ds.initial();
        const double wall = ds.run();
        const DevState h = ds.finish(x);
        report->iterations = h.done == kZeroRhs ? 0 : h.iters;
        report->converged = (h.done == kConverged || h.done == kZeroRhs) ? 1 : 0;
        report->wall_time = wall;
        const int cnt = std::min(report->iterations, report->cap);
        if (cnt > 0) {
            rcg_ctx* c0 = slabs[0]->ctx;
            if (report->history)
                RCG_CK(cudaMemcpy(report->history, c0->ws.hist, sizeof(double) * cnt, cudaMemcpyDeviceToHost));
            if (report->alphas)
                RCG_CK(cudaMemcpy(report->alphas, c0->ws.alph, sizeof(double) * cnt, cudaMemcpyDeviceToHost));
            if (report->betas)
                RCG_CK(cudaMemcpy(report->betas, c0->ws.bet, sizeof(double) * cnt, cudaMemcpyDeviceToHost));
        }
        if (h.done == kBroken) {
            const bool dfl = ds.defl != nullptr;
            throw Error(RCG_E_BREAKDOWN, h.status == kBrkRz ? (dfl ? "deflated pcg: preconditioner not SPD ((r, z) <= 0)"
                                                                   : "pcg: preconditioner not SPD ((r, z) <= 0)")
                                                            : (dfl ? "deflated pcg: projected operator not SPD ((p, P^T A p) <= 0)"
                                                                   : "pcg: matrix not SPD ((p, A p) <= 0)"));
        }
    });
}

int rcg_dist_solve(rcg_comm* comm, int nslabs, rcg_dslab* const* slabs, const rcg_dbasis* basis, const double* const* b,
                   double* const* x, const rcg_solver_config* cfg, rcg_solve_report* report) {
    return dist_solve_impl(comm, nslabs, slabs, basis, nullptr, b, x, cfg, report);
}

// the batched solver over this process's slab: allreduces on the slab's gbuf, halo rows through
// the transport (one slab per process)
namespace rcg {
struct DistBatchComm : BatchComm {
    rcg_comm* comm = nullptr;
    rcg_dslab* d = nullptr;
    void allreduce(rcg_ctx* ctx, int count) override {
        (void)ctx;
        rcg_dslab* ds[1] = {d};
        comm->allreduce(ds, 1, count, 1);
    }
    void halo(rcg_ctx* ctx, double* v, int rt) override {
        (void)ctx;
        comm->halo_rt(d, v, rt);
    }
};
}  // namespace rcg

int rcg_dist_solve_batch(rcg_comm* comm, rcg_dslab* slab, const rcg_dbasis* basis, const double* B, double* X,
                         const rcg_solver_config* cfg, int nrhs, rcg_solve_report* reps) {
    NvtxRange range("rcg_dist_solve_batch");
    return guard([&] {
        require(comm && slab && B && X && cfg && reps, "dist_solve_batch: null argument");
        require(comm->local_slabs() == 1, "dist_solve_batch: one slab per process (loopback: G = 1)");
        ensure_g(slab, 768 + 2 * 24);  // m RT projection totals + a fused (p, q) / deferred (r, r) row
        DistBatchComm bc;
        bc.comm = comm;
        bc.d = slab;
        bc.dtot = slab->gbuf;
        bc.nhalo = slab->nhalo;
        rcg_basis view{};
        rcg_prec m{};
        m.kind = slab->ic ? RCG_PREC_IC : RCG_PREC_IDENTITY;
        m.ic = slab->ic;
        const rcg_basis* defl = nullptr;
        if (basis && basis->m > 0) {
            view.n = slab->nloc;
            view.k = basis->m;
            view.ld = slab->nloc;
            view.w = basis->w[0];
            view.aw = basis->aw[0];
            view.l = basis->l[0];
            view.who = basis->kind == RCG_BASIS_SC ? 1 : 0;
            if (basis->kind == RCG_BASIS_SC) {
                require(slab->ic != nullptr, "dist_solve_batch: subspace correction needs the block IC(0)");
                m.kind = RCG_PREC_SC;
                m.sc = &view;
            } else {
                defl = &view;
            }
        }
        batch_solve_dist(slab->ctx, slab->a, &m, defl, &bc, B, X, cfg, nrhs, reps);
    });
}

int rcg_dist_pcg_solve(rcg_comm* comm, int nslabs, rcg_dslab* const* slabs, const double* const* b,
                       double* const* x, const rcg_solver_config* cfg, rcg_solve_report* report) {
    return dist_solve_impl(comm, nslabs, slabs, nullptr, nullptr, b, x, cfg, report);
}

int rcg_dist_pcg_solve_sampled(rcg_comm* comm, int nslabs, rcg_dslab* const* slabs, rcg_sampler* const* observers,
                               const double* const* b, double* const* x, const rcg_solver_config* cfg,
                               rcg_solve_report* report) {
    if (!observers) {
        set_error("dist_pcg_solve_sampled: null samplers");
        return RCG_E_INVALID;
    }
    return dist_solve_impl(comm, nslabs, slabs, nullptr, observers, b, x, cfg, report);
}

int rcg_dist_recycle(rcg_comm* comm, int nslabs, rcg_dslab* const* slabs, rcg_sampler* const* samplers,
                     const double* const* x_final, double theta, int keep_count, int kind, int* m_bar, double* values,
                     double* theta_used, int* m_tilde, rcg_dbasis** out) {
    return guard([&] {
        require(comm && slabs && samplers && x_final && m_bar && m_tilde && out, "dist_recycle: null argument");
        require(nslabs == comm->local_slabs(), "dist_recycle: slab count does not match the transport");
        require(kind == RCG_BASIS_DEFLATION || kind == RCG_BASIS_SC, "dist_recycle: unknown basis kind");
        for (int s = 0; s < nslabs; ++s) require(slabs[s] && samplers[s] && x_final[s], "dist_recycle: null slab");
        *out = nullptr;
        std::vector<double> vals;
        *out = dist_recycle(comm, nslabs, slabs, samplers, x_final, theta, keep_count, kind, m_bar, vals, theta_used,
                            m_tilde);
        if (values && !vals.empty()) std::memcpy(values, vals.data(), sizeof(double) * vals.size());
    });
}

}  // extern "C"
