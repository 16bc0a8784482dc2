// sequence.cu -- the sequence driver on the device: run_sequence
// (proj/src/driver.cpp:108-222) as two C-ABI calls, with every vector in HBM and no host
// round trip between the solves.
//
//   rcg_seq_prepare: diagonal scaling (scaling.cpp:20-38) and IC(0) (ic0_factorize(a, 0, blocks),
//                    on the device) -- once per matrix;
//   rcg_seq_run:     scale the k right-hand sides, solve 1 with the error sampler (method A with
//                    max(m, 2) slots or method B), harvest + build_aux_matrix, the SC
//                    preconditioner or the deflation operator, solves 2..k from x0 = 0 (batched
//                    multi-RHS kernel sequences, or one by one), recover the solutions
//                    (x = D^-1/2 x_s) and the true relative residuals ||b - A x|| / ||b|| against
//                    the unscaled matrix (driver.cpp:72-82).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <vector>

#include "internal.cuh"
#include "kernels.cuh"

struct rcg_seq {
    rcg_ctx* ctx = nullptr;
    const rcg_matrix* a_orig = nullptr;  // borrowed
    rcg_matrix* a = nullptr;             // D^-1/2 A D^-1/2
    double* dis = nullptr;               // device D^-1/2
    rcg_ic* ic = nullptr;                // null for method cg
    int method = 0;
    int blocks = 1;
    double setup_time = 0.0;
};

namespace rcg {

__global__ void k_scale_rows(const double* __restrict__ dis, const double* __restrict__ in, double* __restrict__ out,
                             int32_t n, int64_t total) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x)
        out[e] = __dmul_rn(dis[e % n], in[e]);
}

// (b, b) and (b - Ax, b - Ax) of one solve, deterministic (driver.cpp:72-82 order per element)
__global__ void __launch_bounds__(kStreamThreads) k_true_relres(const double* __restrict__ b,
                                                                const double* __restrict__ ax, int32_t n,
                                                                double* partials, unsigned int* ticket,
                                                                double* out) {
    __shared__ double red[2 * 32];
    __shared__ double tot[2];
    double acc[2] = {0.0, 0.0};
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double d = __dsub_rn(b[i], ax[i]);
        acc[0] = fadd_mul(acc[0], b[i], b[i]);
        acc[1] = fadd_mul(acc[1], d, d);
    }
    block_sum<2>(acc, red);
    if (grid_reduce<2>(acc, partials, blockIdx.x, gridDim.x, ticket, tot, red) && threadIdx.x == 0) {
        out[0] = tot[0];
        out[1] = tot[1];
    }
}

}  // namespace rcg

using namespace rcg;

extern "C" {

int rcg_seq_prepare(rcg_ctx* ctx, const rcg_matrix* a_orig, int method, int blocks, rcg_seq** out) {
    return guard([&] {
        require(ctx && a_orig && out, "rcg_seq_prepare: null argument");
        *out = nullptr;
        if (method < RCG_METHOD_CG || method > RCG_METHOD_ES_D_ICCG)
            throw Error(RCG_E_PARSE, "config: unknown method");  // driver.cpp validate_config
        if (blocks < 1) throw Error(RCG_E_PARSE, "config: blocks must be >= 1");
        if (blocks > a_orig->n) throw Error(RCG_E_PARSE, "config: blocks exceeds matrix dimension");
        const auto t0 = std::chrono::steady_clock::now();
        auto* s = new rcg_seq();
        try {
            s->ctx = ctx;
            s->a_orig = a_orig;
            s->method = method;
            s->blocks = blocks;
            s->dis = dev_alloc(std::max(a_orig->n, 1));
            ck(rcg_diagonal_scale(ctx, a_orig, &s->a, s->dis));
            if (method != RCG_METHOD_CG) ck(rcg_ic0_factorize_device(ctx, s->a, 0.0, blocks, &s->ic));
            RCG_CK(cudaStreamSynchronize(ctx->stream));
        } catch (...) {
            rcg_seq_destroy(s);
            throw;
        }
        s->setup_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *out = s;
    });
}

void rcg_seq_destroy(rcg_seq* s) {
    if (!s) return;
    if (s->ctx) cudaStreamSynchronize(s->ctx->stream);
    rcg_ic_destroy(s->ic);
    rcg_matrix_destroy(s->a);
    dev_free(s->dis);
    delete s;
}

int rcg_seq_run(rcg_seq* s, int k_t, const double* rhs, double* x, const rcg_seq_config* cfg, rcg_seq_report* rep) {
    NvtxRange range("rcg_seq_run");
    return guard([&] {
        require(s && rhs && x && cfg && rep, "rcg_seq_run: null argument");
        if (k_t < 1) throw Error(RCG_E_PARSE, "config: k_t must be >= 1");
        if (!(cfg->eps > 0.0 && cfg->eps < 1.0)) throw Error(RCG_E_PARSE, "config: eps must be in (0, 1)");
        if (cfg->max_iter < 1) throw Error(RCG_E_PARSE, "config: max_iter must be >= 1");
        if (cfg->sampling != 'A' && cfg->sampling != 'B') throw Error(RCG_E_PARSE, "config: sampling must be A or B");
        rcg_ctx* ctx = s->ctx;
        const int32_t n = s->a->n;
        const int64_t total = static_cast<int64_t>(k_t) * n;
        const bool recycled = s->method == RCG_METHOD_ES_SC_ICCG || s->method == RCG_METHOD_ES_D_ICCG;
        rcg_solver_config scfg{cfg->eps, cfg->max_iter, 0};
        // scaled right-hand sides (scaling.cpp:8-12) and zero initial guesses.  Host right-hand
        // sides: solve 1's comes in first on the library stream, the others on a side stream
        // behind solve 1 (joined before the accelerated solves), so the H2D copy is hidden
        Staged bst;
        const bool host_rhs = !is_device_ptr(rhs) && k_t > 1;
        cudaStream_t side = nullptr;
        cudaEvent_t rhs_in = nullptr;
        if (host_rhs) {
            bst.dev = dev_alloc(std::max<int64_t>(total, 1));
            bst.owned = true;
            RCG_CK(cudaMemcpyAsync(bst.dev, rhs, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
            RCG_CK(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
            RCG_CK(cudaEventCreateWithFlags(&rhs_in, cudaEventDisableTiming));
            RCG_CK(cudaMemcpyAsync(bst.dev + n, rhs + n, sizeof(double) * (total - n), cudaMemcpyHostToDevice, side));
            RCG_CK(cudaEventRecord(rhs_in, side));
        } else {
            stage_in(ctx, rhs, total, bst);
        }
        double* bs = dev_alloc(std::max<int64_t>(total, 1));
        double* xs = dev_alloc(std::max<int64_t>(total, 1));
        double* ax = dev_alloc(std::max(n, 1));
        double* small = dev_alloc(4);
        unsigned int* ticket = static_cast<unsigned int*>(dev_alloc_bytes(sizeof(unsigned int)));
        rcg_sampler* smp = nullptr;
        rcg_tall *errors = nullptr, *w = nullptr;
        rcg_basis* basis = nullptr;
        auto cleanup = [&] {
            if (side) {
                cudaStreamSynchronize(side);
                cudaStreamDestroy(side);
                side = nullptr;
            }
            if (rhs_in) {
                cudaEventDestroy(rhs_in);
                rhs_in = nullptr;
            }
            rcg_basis_destroy(basis);
            rcg_tall_destroy(w);
            rcg_tall_destroy(errors);
            rcg_sampler_destroy(smp);
            for (void* p : {(void*)bs, (void*)xs, (void*)ax, (void*)small, (void*)ticket}) dev_free(p);
        };
        try {
            RCG_CK(cudaMemsetAsync(xs, 0, sizeof(double) * total, ctx->stream));
            RCG_CK(cudaMemsetAsync(ticket, 0, sizeof(unsigned int), ctx->stream));
            const int g = stream_grid(ctx, total);
            k_scale_rows<<<g, kStreamThreads, 0, ctx->stream>>>(s->dis, bst.dev, bs, n, host_rhs ? n : total);
            RCG_LAUNCHED(ctx);
            rcg_prec inner{s->ic ? RCG_PREC_IC : RCG_PREC_IDENTITY, s->ic, nullptr};
            std::vector<rcg_solve_report> reps(k_t);
            for (auto& r : reps) std::memset(&r, 0, sizeof(r));
            // CG coefficients of every solve for the Lanczos estimate (condest on each solve, C5)
            const bool lanczos = rep->lambda_min || rep->lambda_max || rep->kappa;
            std::vector<double> coef(lanczos ? static_cast<size_t>(k_t) * 2 * cfg->max_iter : 0);
            if (lanczos)
                for (int k = 0; k < k_t; ++k) {
                    reps[k].cap = cfg->max_iter;
                    reps[k].alphas = coef.data() + static_cast<size_t>(2 * k) * cfg->max_iter;
                    reps[k].betas = coef.data() + static_cast<size_t>(2 * k + 1) * cfg->max_iter;
                }
            // solve 1 with the error-sampling observer (driver.cpp:147-160)
            if (recycled) {
                if (cfg->sampling == 'A')
                    ck(rcg_sampler_create(ctx, RCG_SAMPLER_A, std::max(cfg->m, 2), cfg->max_iter, cfg->eps, n, &smp));
                else
                    ck(rcg_sampler_create(ctx, RCG_SAMPLER_B, cfg->m, cfg->max_iter, cfg->eps, n, &smp));
            }
            ck(rcg_pcg_solve(ctx, s->a, bs, &inner, xs, &scfg, smp, RCG_PAYLOAD_X, &reps[0]));
            // the auxiliary basis (driver.cpp:163-184)
            nvtxRangePushA("recycling + basis");
            rep->m_bar = rep->m_tilde = 0;
            rep->theta_used = cfg->theta;
            rep->w_build_time = 0.0;
            if (recycled) {
                const auto t0 = std::chrono::steady_clock::now();
                // the standard recycling step keeps the slots, the error block, its MGS copy and A E
                // (3 x m x n doubles beyond the slots); short of HBM, the lean step works in the slots
                bool lean = cfg->memory == 1;
                if (!lean) {
                    size_t fr = 0, tot = 0;
                    RCG_CK(cudaMemGetInfo(&fr, &tot));
                    const double need = (3.0 * smp->m + std::max(cfg->keep_count, 1)) * 8.0 * static_cast<double>(smp->ld);
                    lean = static_cast<double>(fr) < 1.1 * need;
                }
                std::vector<double> vals;
                if (lean) {
                    lean_build_aux(ctx, s->a, xs, smp, cfg->theta, cfg->keep_count, &rep->m_bar, vals, &rep->theta_used,
                                   &w);
                    rcg_sampler_destroy(smp);  // spent: its slots held the errors and the basis
                    smp = nullptr;
                } else {
                    ck(rcg_harvest_errors(ctx, xs, smp, &errors));
                    vals.assign(std::max(errors->k, 1), 0.0);
                    ck(rcg_build_aux_matrix(ctx, s->a, errors, cfg->theta, cfg->keep_count, &rep->m_bar, vals.data(),
                                            &rep->theta_used, &w));
                }
                rep->m_tilde = w->k;
                if (rep->ritz_values)
                    std::memcpy(rep->ritz_values, vals.data(), sizeof(double) * std::min(rep->m_bar, rep->ritz_cap));
                if (rep->m_tilde > 0)  // lean: the basis takes W's block over instead of copying it
                    basis_build(ctx, s->a, w, s->method == RCG_METHOD_ES_SC_ICCG ? RCG_BASIS_SC : RCG_BASIS_DEFLATION,
                                lean, &basis);
                RCG_CK(cudaStreamSynchronize(ctx->stream));
                rep->w_build_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            }
            rep->acceleration_inactive = recycled && rep->m_tilde == 0 ? 1 : 0;
            // solves 2..k from x0 = 0 (driver.cpp:186-199)
            rcg_prec sc{RCG_PREC_SC, s->ic, basis};
            const bool use_sc = basis && s->method == RCG_METHOD_ES_SC_ICCG;
            const rcg_basis* defl = basis && s->method == RCG_METHOD_ES_D_ICCG ? basis : nullptr;
            const rcg_prec* m2 = use_sc ? &sc : &inner;
            // batched solves keep ~10 interleaved vectors of RT right-hand sides: when HBM is short
            // (auto memory mode), the widest batch whose workspace fits (C4 on one GPU: a few
            // right-hand sides per kernel sequence instead of one), else unbatched
            bool batch = cfg->batch != 0;
            int max_cnt = 24;
            if (batch && cfg->memory == 0 && k_t > 1) {
                size_t fr = 0, tot = 0;
                RCG_CK(cudaMemGetInfo(&fr, &tot));
                max_cnt = 0;
                for (int rt : {24, 16, 12, 8, 4, 2})
                    if (static_cast<double>(fr) > 1.1 * 10.0 * 8.0 * rt * static_cast<double>(n)) {
                        max_cnt = rt;
                        break;
                    }
                batch = max_cnt > 0;
            }
            if (host_rhs) {  // the other right-hand sides are in: scale them
                RCG_CK(cudaStreamWaitEvent(ctx->stream, rhs_in, 0));
                k_scale_rows<<<g, kStreamThreads, 0, ctx->stream>>>(s->dis, bst.dev + n, bs + n, n, total - n);
                RCG_LAUNCHED(ctx);
            }
            nvtxRangePop();
            NvtxRange acc("accelerated solves");
            for (int k = 1; k < k_t;) {
                const int cnt = batch ? std::min(max_cnt, k_t - k) : 1;
                double* B = bs + static_cast<int64_t>(k) * n;
                double* X = xs + static_cast<int64_t>(k) * n;
                if (cnt > 1 || batch) {
                    if (defl)
                        ck(rcg_deflated_pcg_solve_batch(ctx, s->a, B, m2, defl, X, &scfg, cnt, &reps[k]));
                    else
                        ck(rcg_pcg_solve_batch(ctx, s->a, B, m2, X, &scfg, cnt, &reps[k]));
                } else if (defl) {
                    ck(rcg_deflated_pcg_solve(ctx, s->a, B, m2, defl, X, &scfg, &reps[k]));
                } else {
                    ck(rcg_pcg_solve(ctx, s->a, B, m2, X, &scfg, nullptr, RCG_PAYLOAD_X, &reps[k]));
                }
                k += cnt;
            }
            // recover the solutions and the true relative residuals against the unscaled matrix
            Staged xo;
            stage_out_begin(ctx, x, total, xo);
            k_scale_rows<<<g, kStreamThreads, 0, ctx->stream>>>(s->dis, xs, xo.dev, n, total);
            RCG_LAUNCHED(ctx);
            double acc_it = 0.0, acc_wall = 0.0;
            for (int k = 0; k < k_t; ++k) {
                ck(rcg_spmv(ctx, s->a_orig, xo.dev + static_cast<int64_t>(k) * n, ax));
                k_true_relres<<<stream_grid(ctx, n), kStreamThreads, 0, ctx->stream>>>(
                    bst.dev + static_cast<int64_t>(k) * n, ax, n, ctx->ws.partials, ticket, small);
                RCG_LAUNCHED(ctx);
                double h[2];
                RCG_CK(cudaMemcpyAsync(h, small, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
                RCG_CK(cudaStreamSynchronize(ctx->stream));
                if (rep->iterations) rep->iterations[k] = reps[k].iterations;
                if (rep->converged) rep->converged[k] = reps[k].converged;
                if (rep->wall_time) rep->wall_time[k] = reps[k].wall_time;
                if (rep->true_relres) rep->true_relres[k] = h[0] == 0.0 ? 0.0 : std::sqrt(h[1]) / std::sqrt(h[0]);
                if (lanczos) {
                    double lo = NAN, hi = NAN;
                    const int it = std::min(reps[k].iterations, cfg->max_iter);
                    if (it >= 1) lanczos_extremes_host(it, reps[k].alphas, reps[k].betas, &lo, &hi);
                    if (rep->lambda_min) rep->lambda_min[k] = lo;
                    if (rep->lambda_max) rep->lambda_max[k] = hi;
                    if (rep->kappa) rep->kappa[k] = hi / lo;
                }
                if (k > 0) {
                    acc_it += reps[k].iterations;
                    acc_wall += reps[k].wall_time;
                }
            }
            stage_out_end(ctx, x, total, xo);
            rep->avg_iterations = k_t > 1 ? acc_it / (k_t - 1) : reps[0].iterations;
            rep->avg_wall_time = k_t > 1 ? acc_wall / (k_t - 1) : reps[0].wall_time;
            rep->setup_time = s->setup_time;
            RCG_CK(cudaStreamSynchronize(ctx->stream));
        } catch (...) {
            cleanup();
            throw;
        }
        cleanup();
    });
}

}  // extern "C"
