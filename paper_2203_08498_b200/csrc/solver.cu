// solver.cu -- the PCG iteration on the device (K6-K10, K16): pcg_solve, deflated_pcg_solve
// and pcg_with_condest.
//
// One iteration is a fixed sequence of kernels that read every scalar (iteration index, rho,
// beta, alpha, convergence flag, sampler schedule) from a device-resident DevState written by
// the finalising block of the previous reduction.  Nothing returns to the host inside the
// loop: the host enqueues iterations ahead and every kernel exits at once when the state says
// the solve is over, so the stream never drains between iterations.  Reductions are
// deterministic (fixed per-block partition, fixed final order), so identical inputs give
// identical iterates run to run, and the condest solve reproduces pcg_solve bit for bit.
//
// Per-iteration kernels (IC preconditioner, reference order src/pcg.cpp:63-89):
//   fwd sweep -> bwd sweep (+ (r,z), beta; SC: z += W u) -> p = z + beta p ->
//   q = A p (+ (p,q), alpha; condest: v' = A v) -> [deflation: W^T q, chol, q -= AW u, (p,q)]
//   -> x += alpha p, r -= alpha q, ||r|| (+ relres test, sampler schedule) [SC: W^T r, chol]
#include <chrono>
#include <cmath>
#include <cstring>

#include "internal.cuh"
#include "kernels.cuh"
#include "spmv_pipe.cuh"
#include "vec.cuh"

namespace rcg {

constexpr int kTallKC = 16;   // W^T y columns accumulated per pass in registers

// ------------------------------------------------------------------ kernels
// p = z (first iteration) or z + beta p  (src/pcg.cpp:67-71); optionally resets the sweep buffer
// With W != null (IC inner + subspace correction) z_i = z_ic,i + sum_j u_j W_ij first, in the
// reference's accumulation order (src/subspace_correction.cpp:53-56).
__global__ void __launch_bounds__(kStreamThreads) k_pupdate(const double* __restrict__ z, double* __restrict__ p,
                                                            double* __restrict__ zs_reset, double* __restrict__ y_reset, int32_t n, DevState* st,
                                                            const double* __restrict__ W, int64_t ldw, int k,
                                                            const double* __restrict__ u) {
    if (st->done) return;
    const bool first = st->iter == 1;
    const double beta = st->beta;
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double zi = z[i];
        if (W)
            for (int j = 0; j < k; ++j) zi = fadd_mul(zi, __ldg(u + j), __ldg(W + j * ldw + i));
        p[i] = first ? zi : fadd_mul(zi, beta, p[i]);
        if (zs_reset) {  // both sweep buffers back to the sentinel for the next iteration
            zs_reset[i] = sentinel();
            y_reset[i] = sentinel();
        }
    }
}

// q = A p [, v' = A v]  with (p,q) [, (v,v'), (v',v')] partials; finaliser: alpha (or only
// records the dots when the deflated path still has to project q)
template <int NV>
__global__ void __launch_bounds__(kSpmvThreads) k_spmv_pq(SpmvArgs a, int cap, DevState* st, int project_later) {
    __shared__ double red[3 * 32];
    __shared__ double tot[3];
    if (st->done) return;
    double acc3[3] = {0.0, 0.0, 0.0};
    spmv_pipeline<NV>(a, cap, [&](int32_t row, const double (&s)[NV]) {
        a.y[0][row] = s[0];
        if (!project_later) acc3[0] = fadd_mul(acc3[0], a.x[0][row], s[0]);
        if (NV == 2) {
            a.y[1][row] = s[NV - 1];
            acc3[1] = fadd_mul(acc3[1], a.x[NV - 1][row], s[NV - 1]);
            acc3[2] = fadd_mul(acc3[2], s[NV - 1], s[NV - 1]);
        }
    });
    block_sum<3>(acc3, red);
    if (grid_reduce<3>(acc3, a.partials, blockIdx.x, gridDim.x, &st->tick[1], tot, red) && threadIdx.x == 0) {
        if (NV == 2) {  // power step (src/condest.cpp:86-92): quotient, then ||v'||
            if (st->nq == 5) {
                for (int j = 0; j < 4; ++j) st->quot[j] = st->quot[j + 1];
                st->nq = 4;
            }
            st->quot[st->nq++] = tot[1];
            st->vn = sqrt(tot[2]);
            if (st->vn == 0.0) {
                st->done = kBroken;
                st->status = kBrkPower;
            }
        }
        if (!project_later && st->done == kRunning) {
            st->pq = tot[0];
            if (tot[0] <= 0.0) {
                st->done = kBroken;
                st->status = kBrkPAp;
            }
            st->alpha = st->rho / tot[0];
        }
    }
}

// f = B^T y for the k columns of B (k <= kMaxRed), one deterministic grid reduction; the
// finaliser either solves (L L^T) u = f into `u` (mode 1) or stores f (mode 0).
__global__ void __launch_bounds__(kStreamThreads, 4) k_tallt(const double* __restrict__ B, int64_t ldb, int k,
                                                          const double* __restrict__ y, int32_t n,
                                                          double* partials, const double* __restrict__ L,
                                                          double* __restrict__ out, int mode, DevState* st,
                                                          int respect_done) {
    __shared__ double scratch[32 * kTallKC];
    __shared__ double bvals[kMaxRed];
    __shared__ double tot[kMaxRed];
    __shared__ double sol[kMaxRed];
    if (respect_done && st->done) return;
    for (int c0 = 0; c0 < k; c0 += kTallKC) {
        const int kc = min(kTallKC, k - c0);
        double acc[kTallKC];
#pragma unroll
        for (int j = 0; j < kTallKC; ++j) acc[j] = 0.0;
        for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
            const double yi = y[i];
#pragma unroll
            for (int j = 0; j < kTallKC; ++j)
                if (j < kc) acc[j] = fadd_mul(acc[j], __ldg(B + (c0 + j) * ldb + i), yi);
        }
        block_sum_dyn<kTallKC>(acc, kc, scratch, bvals + c0);
    }
    if (grid_reduce_dyn(bvals, k, partials, &st->tick[2], tot)) {
        if (threadIdx.x < 32) {
            if (mode >= 1) {
                warp_chol_solve(L, k, tot, out, sol);
                if (mode == 2 && threadIdx.x == 0) {  // f . u = (W^T r) . (W^T A W)^-1 W^T r
                    double fu = 0.0;
                    for (int j = 0; j < k; ++j) fu = fadd_mul(fu, tot[j], sol[j]);
                    st->scal[2] = fu;
                }
            } else {
                for (int j = threadIdx.x; j < k; j += 32) out[j] = tot[j];
            }
        }
    }
}

// y -= sum_j u_j C[:,j] (subtract_combination, src/deflation.cpp:7-13), plus a dot partial:
// mode 0: (p, y) -> pq/alpha ; mode 1: (y, y) -> projected initial residual check ; 2: none
__global__ void __launch_bounds__(kStreamThreads) k_deflate(double* __restrict__ y, const double* __restrict__ C,
                                                            int64_t ldc, int k, const double* __restrict__ u,
                                                            const double* __restrict__ p, int32_t n,
                                                            double* partials, DevState* st, int mode) {
    __shared__ double red[32];
    __shared__ double tot[1];
    if (st->done) return;
    double acc[1] = {0.0};
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double v = y[i];
        for (int j = 0; j < k; ++j) v = fsub_mul(v, __ldg(u + j), __ldg(C + j * ldc + i));
        y[i] = v;
        if (mode == 0) acc[0] = fadd_mul(acc[0], p[i], v);
        if (mode == 1) acc[0] = fadd_mul(acc[0], v, v);
    }
    if (mode == 2) return;
    block_sum<1>(acc, red);
    if (grid_reduce<1>(acc, partials, blockIdx.x, gridDim.x, &st->tick[3], tot, red) && threadIdx.x == 0) {
        if (mode == 0) {
            st->pq = tot[0];
            if (tot[0] <= 0.0) {
                st->done = kBroken;
                st->status = kBrkPAp;
            }
            st->alpha = st->rho / tot[0];
        } else {
            st->rr = tot[0];
            st->rho = tot[0];
            if (sqrt(tot[0]) <= st->eps * st->bnorm) st->done = kConverged;
        }
    }
}

// x/r update + relres + sampler (src/pcg.cpp:76-88, src/sampling.cpp:40-65)
struct XrArgs {
    double* x;
    double* r;
    const double* p;
    const double* q;
    int32_t n;
    double* partials;
    DevState* st;
    double* hist;
    double* alph;
    double* bet;
    // sampler
    double* slots;
    int64_t ldslot;
    int* occupied;
    int* stored_iter;
    const double* thresholds;
    int* pending;
    // condest
    double* v;
    const double* vnext;
    int identity;   // rho_{i+1} = (r, r)
};

__device__ void sampler_schedule(XrArgs& a, int i, double relres) {
    smp_schedule(a.st, i, relres, a.pending, a.occupied, a.stored_iter, a.thresholds);
}

__global__ void __launch_bounds__(kStreamThreads) k_xr(XrArgs a) {
    __shared__ double red[32];
    __shared__ double tot[1];
    DevState* st = a.st;
    if (st->done) return;
    const double alpha = st->alpha;
    const int npend = st->smp_npending;
    const double* payload = st->smp_payload ? a.r : a.x;
    const double inv_vn = 0.0;
    (void)inv_vn;
    const double vn = st->vn;
    double acc[1] = {0.0};
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += gridDim.x * blockDim.x) {
        if (npend) {
            const double pv = payload[i];
            for (int s = 0; s < npend; ++s) a.slots[a.pending[s] * a.ldslot + i] = pv;
        }
        a.x[i] = fadd_mul(a.x[i], alpha, a.p[i]);
        const double ri = fsub_mul(a.r[i], alpha, a.q[i]);
        a.r[i] = ri;
        acc[0] = fadd_mul(acc[0], ri, ri);
        if (a.v) a.v[i] = __ddiv_rn(a.vnext[i], vn);
    }
    block_sum<1>(acc, red);
    if (grid_reduce<1>(acc, a.partials, blockIdx.x, gridDim.x, &st->tick[4], tot, red) && threadIdx.x == 0) {
        const int i = st->iter;
        const double rr = tot[0];
        const double relres = sqrt(rr) / st->bnorm;
        st->rr = rr;
        st->relres = relres;
        st->iters = i;
        a.hist[i - 1] = relres;
        a.alph[i - 1] = alpha;
        a.bet[i - 1] = st->beta;
        st->rho_prev = st->rho;
        st->smp_npending = 0;
        if (relres <= st->eps) {
            st->done = kConverged;
        } else {
            sampler_schedule(a, i, relres);
            if (i >= st->max_iter) {
                st->done = kCapped;
            } else {
                st->iter = i + 1;
                if (a.identity) {  // z = r: the next (r, z) is this (r, r)
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
}

// z = r + W u (SC with identity inner) and rho = (r, z), beta
__global__ void __launch_bounds__(kStreamThreads) k_sc_identity(const double* __restrict__ r, double* __restrict__ z,
                                                                const double* __restrict__ W, int64_t ldw, int k,
                                                                const double* __restrict__ u, int32_t n,
                                                                double* partials, DevState* st) {
    __shared__ double red[32];
    __shared__ double tot[1];
    if (st->done) return;
    double acc[1] = {0.0};
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double ri = r[i];
        double zi = ri;
        for (int j = 0; j < k; ++j) zi = fadd_mul(zi, __ldg(u + j), __ldg(W + j * ldw + i));
        z[i] = zi;
        acc[0] = fadd_mul(acc[0], ri, zi);
    }
    block_sum<1>(acc, red);
    if (grid_reduce<1>(acc, partials, blockIdx.x, gridDim.x, &st->tick[5], tot, red) && threadIdx.x == 0) {
        st->rho = tot[0];
        if (tot[0] <= 0.0) {
            st->done = kBroken;
            st->status = kBrkRz;
        }
        st->beta = st->iter > 1 ? tot[0] / st->rho_prev : 0.0;
    }
}

// after k_residual: zero-rhs / already-converged tests (src/pcg.cpp:43-59)
__global__ void k_init_check(DevState* st, int defer_check, int identity) {
    if (st->bnorm == 0.0) {
        st->done = kZeroRhs;
        return;
    }
    if (!defer_check && sqrt(st->rr) <= st->eps * st->bnorm) st->done = kConverged;
    (void)identity;
    st->rho = st->rr;  // identity preconditioner: (r, z) = (r, r); overwritten otherwise
}

// final offer when the cap stops a non-converged solve (the observer saw iteration max_iter)
__global__ void k_pending_copy(XrArgs a) {
    DevState* st = a.st;
    const int npend = st->smp_npending;
    if (st->done != kCapped || npend == 0) return;
    const double* payload = st->smp_payload ? a.r : a.x;
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += gridDim.x * blockDim.x) {
        const double pv = payload[i];
        for (int s = 0; s < npend; ++s) a.slots[a.pending[s] * a.ldslot + i] = pv;
    }
}

__global__ void k_zero_if(double* x, int32_t n, const DevState* st) {
    if (st->done != kZeroRhs) return;
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) x[i] = 0.0;
}

// x += sum_j u_j W[:,j] accumulated from 0.0 (direct_component, src/deflation.cpp:33-43)
__global__ void k_add_combination(double* __restrict__ x, const double* __restrict__ W, int64_t ldw, int k,
                                  const double* __restrict__ u, int32_t n, const DevState* st, int only_ok) {
    if (only_ok && (st->done == kBroken || st->done == kZeroRhs)) return;
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double t = 0.0;
        for (int j = 0; j < k; ++j) t = fadd_mul(t, __ldg(u + j), __ldg(W + j * ldw + i));
        x[i] = __dadd_rn(x[i], t);
    }
}

// out = in (optional), then in-place ops
__global__ void k_copy(const double* __restrict__ a, double* __restrict__ b, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        b[i] = a[i];
}

// v /= ||v||  and  dot(v, A v) helpers for condest
__global__ void __launch_bounds__(kStreamThreads) k_dot(const double* __restrict__ a, const double* __restrict__ b,
                                                        int32_t n, double* partials, double* out, unsigned int* ticket) {
    __shared__ double red[32];
    __shared__ double tot[1];
    double acc[1] = {0.0};
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        acc[0] = fadd_mul(acc[0], a[i], b[i]);
    block_sum<1>(acc, red);
    if (grid_reduce<1>(acc, partials, blockIdx.x, gridDim.x, ticket, tot, red) && threadIdx.x == 0) *out = tot[0];
}

__global__ void k_scale_div(double* v, int32_t n, const double* nrm2sq) {
    const double nv = sqrt(*nrm2sq);
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) v[i] = __ddiv_rn(v[i], nv);
}

// ------------------------------------------------------------------ host orchestration
struct Solve {
    rcg_ctx* ctx;
    const rcg_matrix* a;
    const rcg_prec* m;
    const rcg_basis* defl;
    rcg_sampler* smp;
    int payload;
    bool condest;
    int32_t n;
    int max_iter;
    double eps;
    double* b;   // device
    double* x;   // device (in/out)
    bool ic = false, sc = false;
    const rcg_basis* scb = nullptr;
    int sg = 1;  // stream grid
    int pg = 1;  // spmv grid

    void setup() {
        ic = m->kind == RCG_PREC_IC || (m->kind == RCG_PREC_SC && m->ic);
        sc = m->kind == RCG_PREC_SC && m->sc && m->sc->k > 0;
        scb = sc ? m->sc : nullptr;
        int k = 1;
        if (sc) k = std::max(k, scb->k);
        if (defl) k = std::max(k, defl->k);
        const int64_t ntiles = ic ? sweep_tiles(m->ic) : (n + kSweepThreads - 1) / kSweepThreads;
        const int64_t ngroups = (ntiles + kGroup - 1) / kGroup;
        const int64_t red = std::max<int64_t>(ntiles, static_cast<int64_t>(kMaxRed) * ctx->num_sms * 8);
        ensure_workspace(ctx, n, k, max_iter, red, ngroups, smp ? smp->m : 1);
        sg = stream_grid(ctx, n);
        pg = spmv_grid(ctx, n);
        static bool smem_ok = false;
        if (!smem_ok) {
            spmv_prepare_kernels();
            allow_smem(reinterpret_cast<const void*>(k_spmv_pq<1>));
            allow_smem(reinterpret_cast<const void*>(k_spmv_pq<2>));
            // one shared-memory carveout for every kernel of the loop: an SM must drain before
            // it switches carveout, so mixed preferences serialise concurrent solves
            for (const void* k : {reinterpret_cast<const void*>(k_pupdate), reinterpret_cast<const void*>(k_xr),
                                  reinterpret_cast<const void*>(k_tallt), reinterpret_cast<const void*>(k_deflate),
                                  reinterpret_cast<const void*>(k_sc_identity),
                                  reinterpret_cast<const void*>(k_spmv_pq<1>),
                                  reinterpret_cast<const void*>(k_spmv_pq<2>)})
                set_carveout(k);
            sweep_prepare_kernels();
            smem_ok = true;
        }
    }

    XrArgs xr_args() {
        Workspace& w = ctx->ws;
        XrArgs xa{};
        xa.x = x;
        xa.r = w.r;
        xa.p = w.p;
        xa.q = w.q;
        xa.n = n;
        xa.partials = w.partials;
        xa.st = w.st;
        xa.hist = w.hist;
        xa.alph = w.alph;
        xa.bet = w.bet;
        if (smp) {
            xa.slots = smp->slots;
            xa.ldslot = smp->ld;
            xa.occupied = smp->occupied;
            xa.stored_iter = smp->stored_iter;
            xa.thresholds = smp->thresholds;
        }
        xa.pending = w.smp_pending;
        if (condest) {
            xa.v = w.v;
            xa.vnext = w.vnext;
        }
        xa.identity = (!ic && !sc) ? 1 : 0;
        return xa;
    }

    void init_state() {
        DevState h{};
        h.done = kRunning;
        h.iter = 1;
        h.max_iter = max_iter;
        h.eps = eps;
        h.smp_method = -1;
        h.smp_payload = payload;
        if (smp) {
            h.smp_method = smp->method;
            h.smp_m = smp->m;
            h.smp_lmax = smp->l_max;
            h.smp_h = smp->h;
            h.smp_next = smp->next_slot;
        }
        std::memcpy(ctx->host_pinned, &h, sizeof(h));
        RCG_CK(cudaMemcpyAsync(ctx->ws.st, ctx->host_pinned, sizeof(DevState), cudaMemcpyHostToDevice, ctx->stream));
    }

    // r = b - A x ; bnorm ; projected / identity initial quantities
    void initial() {
        Workspace& w = ctx->ws;
        init_state();
        if (ic) {
            launch_fill_bits(ctx, w.ybuf, n, kSentinelBits);
            launch_fill_bits(ctx, w.zs, n, kSentinelBits);
        }
        launch_residual(ctx, a, b, x, w.r);
        const bool dfl = defl && defl->k > 0;
        k_init_check<<<1, 1, 0, ctx->stream>>>(w.st, dfl ? 1 : 0, (!ic && !sc) ? 1 : 0);
        RCG_LAUNCHED(ctx);
        if (dfl) {  // r = P^T r (src/pcg.cpp:112) and the check on the projected residual
            k_tallt<<<sg, kStreamThreads, 0, ctx->stream>>>(defl->w, defl->ld, defl->k, w.r, n, w.partials, defl->l,
                                                             w.u, 1, w.st, 1);
            RCG_LAUNCHED(ctx);
            k_deflate<<<sg, kStreamThreads, 0, ctx->stream>>>(w.r, defl->aw, defl->ld, defl->k, w.u, nullptr, n,
                                                               w.partials, w.st, 1);
            RCG_LAUNCHED(ctx);
        }
        if (sc) {
            k_tallt<<<sg, kStreamThreads, 0, ctx->stream>>>(scb->w, scb->ld, scb->k, w.r, n, w.partials, scb->l, w.u2,
                                                             2, w.st, 1);
            RCG_LAUNCHED(ctx);
        }
        if (condest) {  // v0 already uploaded into w.v; normalise (src/condest.cpp:47-52)
            k_dot<<<sg, kStreamThreads, 0, ctx->stream>>>(w.v, w.v, n, w.partials, &w.st->scal[0], &w.st->tick[6]);
            RCG_LAUNCHED(ctx);
        }
    }

    void iteration() {
        Workspace& w = ctx->ws;
        DevState* st = w.st;
        const double* z = w.r;  // identity: z is r
        if (ic) {
            SweepArgs fa = sweep_args(ctx, m->ic, false);
            fa.in = w.r;
            fa.out = w.ybuf;
            launch_sweep(ctx, m->ic, false, fa);
            SweepArgs ba = sweep_args(ctx, m->ic, true);
            ba.in = w.ybuf;

            ba.out = w.zs;
            ba.r = w.r;
            ba.add_sc = sc ? 1 : 0;
            z = w.zs;
            launch_sweep(ctx, m->ic, true, ba);
        } else if (sc) {
            k_sc_identity<<<sg, kStreamThreads, 0, ctx->stream>>>(w.r, w.z, scb->w, scb->ld, scb->k, w.u2, n,
                                                                   w.partials, st);
            RCG_LAUNCHED(ctx);
            z = w.z;
        }
        {
            // IC + SC: z = z_ic + W u is formed here, coalesced, instead of inside the sweep
            KTimer t(ctx, 3);
            const bool fold = ic && sc;
            k_pupdate<<<sg, kStreamThreads, 0, ctx->stream>>>(z, w.p, ic ? w.zs : nullptr, w.ybuf, n, st,
                                                               fold ? scb->w : nullptr, fold ? scb->ld : 0,
                                                               fold ? scb->k : 0, w.u2);
            RCG_LAUNCHED(ctx);
        }
        const bool dfl = defl && defl->k > 0;
        SpmvArgs sa{};
        sa.rs = a->rs;
        sa.ci = a->ci;
        sa.va = a->va;
        sa.n = n;
        sa.partials = w.partials;
        sa.x[0] = w.p;
        sa.y[0] = w.q;
        {
            KTimer t(ctx, 0);
            if (condest) {
                sa.x[1] = w.v;
                sa.y[1] = w.vnext;
                k_spmv_pq<2><<<pg, kSpmvThreads, spmv_smem(a), ctx->stream>>>(sa, a->cap, st, dfl ? 1 : 0);
            } else {
                k_spmv_pq<1><<<pg, kSpmvThreads, spmv_smem(a), ctx->stream>>>(sa, a->cap, st, dfl ? 1 : 0);
            }
            RCG_LAUNCHED(ctx);
        }
        if (dfl) {  // q = P^T q (src/pcg.cpp:131) then (p, q) and alpha
            KTimer t(ctx, 4);
            k_tallt<<<sg, kStreamThreads, 0, ctx->stream>>>(defl->w, defl->ld, defl->k, w.q, n, w.partials, defl->l,
                                                             w.u, 1, st, 1);
            RCG_LAUNCHED(ctx);
            k_deflate<<<sg, kStreamThreads, 0, ctx->stream>>>(w.q, defl->aw, defl->ld, defl->k, w.u, w.p, n,
                                                               w.partials, st, 0);
            RCG_LAUNCHED(ctx);
        }
        {
            KTimer t(ctx, 3);
            XrArgs xa = xr_args();
            k_xr<<<sg, kStreamThreads, 0, ctx->stream>>>(xa);
            RCG_LAUNCHED(ctx);
        }
        if (sc) {  // W^T r for the next apply (src/subspace_correction.cpp:50-51)
            KTimer t(ctx, 4);
            k_tallt<<<sg, kStreamThreads, 0, ctx->stream>>>(scb->w, scb->ld, scb->k, w.r, n, w.partials, scb->l,
                                                             w.u2, 2, st, 1);
            RCG_LAUNCHED(ctx);
        }
    }

    void finish() {
        Workspace& w = ctx->ws;
        XrArgs xa = xr_args();
        k_pending_copy<<<sg, kStreamThreads, 0, ctx->stream>>>(xa);
        RCG_LAUNCHED(ctx);
        k_zero_if<<<sg, kStreamThreads, 0, ctx->stream>>>(x, n, w.st);
        RCG_LAUNCHED(ctx);
        if (defl && defl->k > 0) {  // x = P x + W (W^T A W)^-1 W^T b (src/pcg.cpp:152-157)
            k_tallt<<<sg, kStreamThreads, 0, ctx->stream>>>(defl->aw, defl->ld, defl->k, x, n, w.partials, defl->l,
                                                             w.u, 1, w.st, 0);
            RCG_LAUNCHED(ctx);
            k_deflate_final(w);
        }
    }

    void k_deflate_final(Workspace& w) {
        // x -= W u  (project_p), guarded so a broken / zero-rhs solve leaves x as the reference does
        k_tallt_guarded_sub(w);
        k_tallt<<<sg, kStreamThreads, 0, ctx->stream>>>(defl->w, defl->ld, defl->k, b, n, w.partials, defl->l,
                                                         w.u2, 1, w.st, 0);
        RCG_LAUNCHED(ctx);
        k_add_combination<<<sg, kStreamThreads, 0, ctx->stream>>>(x, defl->w, defl->ld, defl->k, w.u2, n, w.st, 1);
        RCG_LAUNCHED(ctx);
    }

    void k_tallt_guarded_sub(Workspace& w);
};

__global__ void k_sub_combination_ok(double* __restrict__ x, const double* __restrict__ W, int64_t ldw, int k,
                                     const double* __restrict__ u, int32_t n, const DevState* st) {
    if (st->done == kBroken || st->done == kZeroRhs) return;
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double v = x[i];
        for (int j = 0; j < k; ++j) v = fsub_mul(v, __ldg(u + j), __ldg(W + j * ldw + i));
        x[i] = v;
    }
}

void Solve::k_tallt_guarded_sub(Workspace& w) {
    k_sub_combination_ok<<<sg, kStreamThreads, 0, ctx->stream>>>(x, defl->w, defl->ld, defl->k, w.u, n, w.st);
    RCG_LAUNCHED(ctx);
}

// Runs the loop: iterations are enqueued in growing batches; the host only polls the device
// flag of the batch before last (the stream never drains while work is queued).
static void run_loop(Solve& s, double* wall_s) {
    rcg_ctx* ctx = s.ctx;
    cudaEvent_t evs[2];
    RCG_CK(cudaEventCreateWithFlags(&evs[0], cudaEventDisableTiming));
    RCG_CK(cudaEventCreateWithFlags(&evs[1], cudaEventDisableTiming));
    cudaEvent_t t0, t1;
    RCG_CK(cudaEventCreate(&t0));
    RCG_CK(cudaEventCreate(&t1));
    RCG_CK(cudaEventRecord(t0, ctx->stream));
    volatile int* flags = reinterpret_cast<volatile int*>(ctx->host_pinned + 256);
    flags[0] = flags[1] = 0;
    int enq = 0, batch = 2, slot = 0;
    bool have_prev = false;
    int prev = 0;
    while (true) {
        for (int j = 0; j < batch && enq < s.max_iter; ++j, ++enq) s.iteration();
        RCG_CK(cudaMemcpyAsync((void*)(flags + slot), &ctx->ws.st->done, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        RCG_CK(cudaEventRecord(evs[slot], ctx->stream));
        if (enq >= s.max_iter) {
            RCG_CK(cudaEventSynchronize(evs[slot]));
            break;
        }
        if (have_prev) {
            RCG_CK(cudaEventSynchronize(evs[prev]));
            if (flags[prev] != kRunning) break;
        }
        have_prev = true;
        prev = slot;
        slot ^= 1;
        batch = std::min(batch * 2, 16);
    }
    RCG_CK(cudaEventRecord(t1, ctx->stream));
    RCG_CK(cudaEventSynchronize(t1));
    float ms = 0.f;
    RCG_CK(cudaEventElapsedTime(&ms, t0, t1));
    *wall_s = ms * 1e-3;
    cudaEventDestroy(evs[0]);
    cudaEventDestroy(evs[1]);
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
}

void check_cfg(const rcg_solver_config* cfg) {
    require(cfg != nullptr, "SolverConfig: null");
    if (!(cfg->eps > 0.0 && cfg->eps < 1.0)) throw Error(RCG_E_INVALID, "SolverConfig: eps must be in (0, 1)");
    if (cfg->max_iter < 1) throw Error(RCG_E_INVALID, "SolverConfig: max_iter must be >= 1");
}

void check_prec(const rcg_prec* m, int32_t n) {
    require(m != nullptr, "preconditioner: null");
    switch (m->kind) {
        case RCG_PREC_IDENTITY:
            break;
        case RCG_PREC_IC:
            require(m->ic != nullptr, "preconditioner: IC kind without a factor");
            require(m->ic->n == n, "preconditioner: factor size does not match matrix");
            break;
        case RCG_PREC_SC:
            require(m->sc != nullptr, "ScPreconditioner: basis is null");
            require(m->sc->k == 0 || m->sc->n == n, "ScPreconditioner: W row count does not match A");
            if (m->ic) require(m->ic->n == n, "preconditioner: factor size does not match matrix");
            break;
        default:
            throw Error(RCG_E_INVALID, "preconditioner: unknown kind (no CPU fallback exists)");
    }
}

// reads back the report and the sampler bookkeeping; returns the DevState
static DevState collect(Solve& s, rcg_solve_report* rep, double wall) {
    rcg_ctx* ctx = s.ctx;
    DevState h{};
    RCG_CK(cudaMemcpyAsync(ctx->host_pinned, ctx->ws.st, sizeof(DevState), cudaMemcpyDeviceToHost, ctx->stream));
    RCG_CK(cudaStreamSynchronize(ctx->stream));
    std::memcpy(&h, ctx->host_pinned, sizeof(h));
    const int iters = h.iters;
    rep->iterations = iters;
    rep->converged = (h.done == kConverged || h.done == kZeroRhs) ? 1 : 0;
    rep->wall_time = wall;
    const int cnt = std::min(iters, rep->cap);
    if (cnt > 0) {
        if (rep->history)
            RCG_CK(cudaMemcpyAsync(rep->history, ctx->ws.hist, sizeof(double) * cnt, cudaMemcpyDeviceToHost, ctx->stream));
        if (rep->alphas)
            RCG_CK(cudaMemcpyAsync(rep->alphas, ctx->ws.alph, sizeof(double) * cnt, cudaMemcpyDeviceToHost, ctx->stream));
        if (rep->betas)
            RCG_CK(cudaMemcpyAsync(rep->betas, ctx->ws.bet, sizeof(double) * cnt, cudaMemcpyDeviceToHost, ctx->stream));
        RCG_CK(cudaStreamSynchronize(ctx->stream));
    }
    if (s.smp) {
        s.smp->h = h.smp_h;
        s.smp->next_slot = h.smp_next;
    }
    return h;
}

static void throw_breakdown(const DevState& h, int which) {
    // which: 0 pcg, 1 deflated, 2 condest (messages of src/pcg.cpp and src/condest.cpp)
    static const char* rz[3] = {"pcg: preconditioner not SPD ((r, z) <= 0)",
                                "deflated pcg: preconditioner not SPD ((r, z) <= 0)",
                                "pcg_with_condest: preconditioner not SPD ((r, z) <= 0)"};
    static const char* pap[3] = {"pcg: matrix not SPD ((p, A p) <= 0)",
                                 "deflated pcg: projected operator not SPD ((p, P^T A p) <= 0)",
                                 "pcg_with_condest: matrix not SPD ((p, A p) <= 0)"};
    if (h.status == kBrkRz) throw Error(RCG_E_BREAKDOWN, rz[which]);
    if (h.status == kBrkPAp) throw Error(RCG_E_BREAKDOWN, pap[which]);
    throw Error(RCG_E_BREAKDOWN, "pcg_with_condest: power vector vanished");
}

}  // namespace rcg

using namespace rcg;

// implemented in recycle.cu
namespace rcg {
void condest_ritz(rcg_ctx* ctx, const rcg_matrix* a, const double* x_dev, rcg_sampler* smp, rcg_cond_estimate* est);
}

static int solve_common(rcg_ctx* ctx, const rcg_matrix* a, const double* b, const rcg_prec* m,
                        const rcg_basis* defl, double* x, const rcg_solver_config* cfg, rcg_sampler* smp,
                        int payload, rcg_solve_report* rep, bool condest, uint64_t seed, int m_samples,
                        rcg_cond_estimate* est, int which) {
    return guard([&] {
        require(ctx && a && rep, "solver: null argument");
        check_cfg(cfg);
        check_prec(m, a->n);
        if (defl && defl->k > 0) require(defl->n == a->n, "deflated_pcg_solve: W row count does not match A");
        if (smp) require(smp->n == a->n, "pcg: sampler slot length does not match matrix");
        const int32_t n = a->n;
        rcg_sampler* own_smp = nullptr;
        if (condest) {
            if (rcg_sampler_create(ctx, RCG_SAMPLER_A, m_samples, cfg->max_iter, 0.5, n, &own_smp) != RCG_OK)
                throw Error(RCG_E_INVALID, rcg_last_error());
            smp = own_smp;
            payload = RCG_PAYLOAD_X;
        }
        try {
            Solve s{};
            s.ctx = ctx;
            s.a = a;
            s.m = m;
            s.defl = defl;
            s.smp = smp;
            s.payload = payload;
            s.condest = condest;
            s.n = n;
            s.max_iter = cfg->max_iter;
            s.eps = cfg->eps;
            s.setup();
            Workspace& w = ctx->ws;
            Staged bs;
            stage_in(ctx, b, n, bs);
            s.b = bs.dev;
            const bool xdev = is_device_ptr(x);
            if (xdev) {
                s.x = x;
            } else {
                RCG_CK(cudaMemcpyAsync(w.xw, x, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
                s.x = w.xw;
            }
            if (condest) {
                std::vector<double> v0(n);
                rcg_uniform_pm1(seed, 0, n, v0.data());
                RCG_CK(cudaMemcpyAsync(w.v, v0.data(), sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
                RCG_CK(cudaStreamSynchronize(ctx->stream));
            }
            s.initial();
            if (condest) {
                k_scale_div<<<s.sg, kStreamThreads, 0, ctx->stream>>>(w.v, n, &w.st->scal[0]);
                RCG_LAUNCHED(ctx);
            }
            double wall = 0.0;
            run_loop(s, &wall);
            s.finish();
            if (!xdev) RCG_CK(cudaMemcpyAsync(x, w.xw, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
            const DevState h = collect(s, rep, wall);
            check_sweep_watchdog(ctx);
            if (h.done == kBroken) throw_breakdown(h, which);
            if (condest) {
                est->power_iterations = rep->iterations;
                est->power_unsettled = 1;
                if (h.nq >= 5) {
                    double lo = h.quot[0], hi = h.quot[0];
                    for (int t = 0; t < h.nq; ++t) {
                        lo = std::fmin(lo, h.quot[t]);
                        hi = std::fmax(hi, h.quot[t]);
                    }
                    est->power_unsettled = (hi - lo) > 1e-4 * std::fabs(h.quot[h.nq - 1]) ? 1 : 0;
                }
                // lambda_max = v^T A v (src/condest.cpp:117-121)
                launch_spmv(ctx, a, w.v, w.vnext);
                k_dot<<<s.sg, kStreamThreads, 0, ctx->stream>>>(w.v, w.vnext, n, w.partials, &w.st->scal[1], &w.st->tick[6]);
                RCG_LAUNCHED(ctx);
                RCG_CK(cudaMemcpyAsync(ctx->host_pinned, &w.st->scal[1], sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
                RCG_CK(cudaStreamSynchronize(ctx->stream));
                est->lambda_max = ctx->host_pinned[0];
                est->lambda_min = NAN;
                est->kappa = NAN;
                est->lambda_min_available = 0;
                est->nritz = 0;
                condest_ritz(ctx, a, s.x, smp, est);
                est->lanczos_lambda_min = NAN;
                est->lanczos_lambda_max = NAN;
                est->lanczos_kappa = NAN;
                if (rep->iterations > 0) {
                    std::vector<double> al(rep->iterations), be(rep->iterations);
                    RCG_CK(cudaMemcpy(al.data(), w.alph, sizeof(double) * rep->iterations, cudaMemcpyDeviceToHost));
                    RCG_CK(cudaMemcpy(be.data(), w.bet, sizeof(double) * rep->iterations, cudaMemcpyDeviceToHost));
                    lanczos_extremes_host(rep->iterations, al.data(), be.data(), &est->lanczos_lambda_min,
                                          &est->lanczos_lambda_max);
                    est->lanczos_kappa = est->lanczos_lambda_max / est->lanczos_lambda_min;
                }
            }
        } catch (...) {
            if (own_smp) rcg_sampler_destroy(own_smp);
            throw;
        }
        if (own_smp) rcg_sampler_destroy(own_smp);
    });
}

extern "C" {

int rcg_pcg_solve(rcg_ctx* ctx, const rcg_matrix* a, const double* b, const rcg_prec* m, double* x,
                  const rcg_solver_config* cfg, rcg_sampler* observer, int payload, rcg_solve_report* rep) {
    NvtxRange r(observer ? "rcg_pcg_solve (sampled)" : "rcg_pcg_solve");
    return solve_common(ctx, a, b, m, nullptr, x, cfg, observer, payload, rep, false, 0, 0, nullptr, 0);
}

int rcg_deflated_pcg_solve(rcg_ctx* ctx, const rcg_matrix* a, const double* b, const rcg_prec* m,
                           const rcg_basis* defl, double* x, const rcg_solver_config* cfg, rcg_solve_report* rep) {
    NvtxRange r("rcg_deflated_pcg_solve");
    return solve_common(ctx, a, b, m, defl, x, cfg, nullptr, 0, rep, false, 0, 0, nullptr, 1);
}

int rcg_pcg_with_condest(rcg_ctx* ctx, const rcg_matrix* a, const double* b, const rcg_prec* m, double* x,
                         const rcg_solver_config* cfg, int m_samples, uint64_t v0_seed, rcg_solve_report* rep,
                         rcg_cond_estimate* est) {
    if (!est) {
        set_error("pcg_with_condest: null estimate");
        return RCG_E_INVALID;
    }
    return solve_common(ctx, a, b, m, nullptr, x, cfg, nullptr, 0, rep, true, v0_seed, m_samples, est, 2);
}

int rcg_lanczos_extremes(int k, const double* alphas, const double* betas, double* lambda_min, double* lambda_max) {
    return guard([&] {
        require(k >= 1, "lanczos: need at least one iteration");
        lanczos_extremes_host(k, alphas, betas, lambda_min, lambda_max);
    });
}

}  // extern "C"
