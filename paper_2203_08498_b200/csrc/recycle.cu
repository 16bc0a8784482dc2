// recycle.cu -- sampler slots, TallDense blocks, the Rayleigh-Ritz step (K11-K15) and the
// deflation / subspace-correction basis (W, AW, chol(W^T A W)).
//
// RR pipeline on the device (src/recycling.cpp:17-96, src/dense.cpp:45-61):
//   harvest  E[:,j] = x_final - slot_s            (slot order, exact-zero columns skipped)
//   MGS      single-pass modified Gram-Schmidt, each projection one fused pass
//            (w -= c_{q-1} e_{q-1} and c_q = e_q . w in the same sweep), drop rule 1e-12
//   A E      one SpMM pass per 8 columns (each column bitwise equal to spmv)
//   E^T A E  tiled Gram reduction (32x32 output tiles, deterministic two-stage sum)
//   eig      cyclic Jacobi on the host (k <= 128; identical rotations to dense.cpp:63-144)
//   Ritz     W = E T_sel with per-row sequential sums (bitwise equal to recycling.cpp:69-77)
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>

#include "internal.cuh"
#include "kernels.cuh"
#include "vec.cuh"

namespace rcg {

constexpr int kGT = 32;   // Gram output tile
constexpr int kGR = 64;   // Gram rows per staging step

// ------------------------------------------------------------------ kernels
__global__ void __launch_bounds__(256) k_gram_partial(const double* __restrict__ A, int64_t lda, int ka,
                                                      const double* __restrict__ B, int64_t ldb, int kb, int32_t n,
                                                      double* __restrict__ part, int lower_only) {
    __shared__ double sa[kGR][kGT + 1];
    __shared__ double sb[kGR][kGT + 1];
    const int ntj = (kb + kGT - 1) / kGT;
    const int ti = blockIdx.y / ntj, tj = blockIdx.y % ntj;
    if (lower_only && tj > ti) return;
    const int t = threadIdx.x;
    const int oi = t / 8, oj0 = (t % 8) * 4;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t r0 = static_cast<int64_t>(blockIdx.x) * kGR; r0 < n; r0 += static_cast<int64_t>(gridDim.x) * kGR) {
        for (int idx = t; idx < kGR * kGT; idx += blockDim.x) {
            const int rr = idx % kGR, c = idx / kGR;
            const int64_t row = r0 + rr;
            const int ca = ti * kGT + c, cb = tj * kGT + c;
            sa[rr][c] = (row < n && ca < ka) ? A[ca * lda + row] : 0.0;
            sb[rr][c] = (row < n && cb < kb) ? B[cb * ldb + row] : 0.0;
        }
        __syncthreads();
#pragma unroll 4
        for (int rr = 0; rr < kGR; ++rr) {
            const double av = sa[rr][oi];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] = fadd_mul(acc[q], av, sb[rr][oj0 + q]);
        }
        __syncthreads();
    }
    const int gi = ti * kGT + oi;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int gj = tj * kGT + oj0 + q;
        if (gi < ka && gj < kb) part[(static_cast<int64_t>(gi) * kb + gj) * gridDim.x + blockIdx.x] = acc[q];
    }
}

__global__ void k_gram_final(const double* __restrict__ part, int ka, int kb, int gx, int lower_only,
                             double* __restrict__ out) {
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= ka * kb) return;
    const int gi = o / kb, gj = o % kb;
    if (lower_only && (gj / kGT) > (gi / kGT)) {
        out[o] = 0.0;
        return;
    }
    double s = 0.0;
    for (int b = 0; b < gx; ++b) s = __dadd_rn(s, part[static_cast<int64_t>(o) * gx + b]);
    out[o] = s;
}

// y[:,c] = sum_j t[c][j] e[:,j] (c < kc <= 16 per launch), from 0.0 in ascending j
constexpr int kComb = 16;
__global__ void __launch_bounds__(kStreamThreads) k_combine(const double* __restrict__ e, int64_t lde, int k,
                                                            const double* __restrict__ t /* kc x k */, int kc,
                                                            double* __restrict__ y, int64_t ldy, int32_t n) {
    extern __shared__ double st_[];
    for (int idx = threadIdx.x; idx < kc * k; idx += blockDim.x) st_[idx] = t[idx];
    __syncthreads();
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double acc[kComb];
#pragma unroll
        for (int c = 0; c < kComb; ++c) acc[c] = 0.0;
        for (int j = 0; j < k; ++j) {
            const double ej = __ldg(e + j * lde + i);
#pragma unroll
            for (int c = 0; c < kComb; ++c)
                if (c < kc) acc[c] = fadd_mul(acc[c], st_[c * k + j], ej);
        }
#pragma unroll
        for (int c = 0; c < kComb; ++c)
            if (c < kc) y[c * ldy + i] = acc[c];
    }
}

// E[:,j] = x - slot_{list[j]} and a nonzero flag per column
__global__ void k_harvest(const double* __restrict__ x, const double* __restrict__ slots, int64_t lds,
                          const int* __restrict__ list, int cnt, int raw, double* __restrict__ e, int64_t lde,
                          int32_t n, int* __restrict__ nonzero) {
    for (int j = blockIdx.y; j < cnt; j += gridDim.y) {
        const double* s = slots + list[j] * lds;
        int nz = 0;
        for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
            const double v = raw ? s[i] : __dsub_rn(x[i], s[i]);
            e[j * lde + i] = v;
            nz |= (v != 0.0);
        }
        if (__syncthreads_or(nz) && threadIdx.x == 0) atomicOr(nonzero + j, 1);
    }
}

// MGS pass q: w -= c[q-1] e[:,q-1] (q > 0) then partial of (e[:,q] . w)  -- or (w . w) when
// q == kept (the final norm).  Single-value deterministic grid reduction into c[q] / *nrm.
__global__ void __launch_bounds__(kStreamThreads) k_mgs_pass(double* __restrict__ w, const double* __restrict__ e,
                                                             int64_t lde, int q, int kept, double* c,
                                                             int32_t n, double* partials, unsigned int* ticket) {
    __shared__ double red[32];
    __shared__ double tot[1];
    const double cprev = q > 0 ? c[q - 1] : 0.0;
    const double* eprev = q > 0 ? e + (q - 1) * lde : nullptr;
    const double* enext = q < kept ? e + q * lde : nullptr;
    double acc[1] = {0.0};
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double wi = w[i];
        if (eprev) {
            wi = fsub_mul(wi, cprev, eprev[i]);
            w[i] = wi;
        }
        acc[0] = enext ? fadd_mul(acc[0], enext[i], wi) : fadd_mul(acc[0], wi, wi);
    }
    block_sum<1>(acc, red);
    if (grid_reduce<1>(acc, partials, blockIdx.x, gridDim.x, ticket, tot, red) && threadIdx.x == 0) c[q] = tot[0];
}

__global__ void k_div_sqrt(double* __restrict__ w, int32_t n, const double* __restrict__ nrm2sq) {
    const double nv = sqrt(*nrm2sq);
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) w[i] = __ddiv_rn(w[i], nv);
}

__global__ void k_copy_col(const double* __restrict__ a, double* __restrict__ b, int32_t n) {
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) b[i] = a[i];
}

// y - sum_j u_j C[:,j] (mode 0) or sum_j u_j C[:,j] from 0.0 (mode 1) into out
__global__ void k_apply_combination(const double* __restrict__ y, const double* __restrict__ C, int64_t ldc, int k,
                                    const double* __restrict__ u, int32_t n, double* __restrict__ out, int mode) {
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double v = mode == 0 ? y[i] : 0.0;
        for (int j = 0; j < k; ++j) v = mode == 0 ? fsub_mul(v, __ldg(u + j), __ldg(C + j * ldc + i))
                                                  : fadd_mul(v, __ldg(u + j), __ldg(C + j * ldc + i));
        out[i] = v;
    }
}

// f = C^T y into f (k values) with deterministic reduction (no chol)
__global__ void __launch_bounds__(kStreamThreads) k_tall_dot(const double* __restrict__ C, int64_t ldc, int k,
                                                             const double* __restrict__ y, int32_t n, double* partials,
                                                             unsigned int* ticket, double* __restrict__ f) {
    __shared__ double scratch[32 * 32];
    __shared__ double bvals[kMaxRed];
    __shared__ double tot[kMaxRed];
    for (int c0 = 0; c0 < k; c0 += 32) {
        const int kc = min(32, k - c0);
        double acc[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[j] = 0.0;
        for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
            const double yi = y[i];
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (j < kc) acc[j] = fadd_mul(acc[j], __ldg(C + (c0 + j) * ldc + i), yi);
        }
        block_sum_dyn<32>(acc, kc, scratch, bvals + c0);
    }
    if (grid_reduce_dyn(bvals, k, partials, ticket, tot))
        for (int j = threadIdx.x; j < k; j += blockDim.x) f[j] = tot[j];
}

// ------------------------------------------------------------------ host helpers
static rcg_tall* tall_alloc(int32_t n, int k) {
    auto* t = new rcg_tall();
    t->n = n;
    t->k = k;
    t->ld = ld_of(n);
    t->d = dev_alloc(std::max<int64_t>(1, t->ld * std::max(k, 1)));
    return t;
}

static void ensure_red(rcg_ctx* ctx, int64_t n) {
    const int64_t ntiles = (n + kSweepThreads - 1) / kSweepThreads;
    const int64_t ngroups = (ntiles + kGroup - 1) / kGroup;
    ensure_workspace(ctx, n, kMaxRed, 1, std::max<int64_t>(ntiles, static_cast<int64_t>(kMaxRed) * ctx->num_sms * 8),
                     ngroups, 1);
}

void gram_host(rcg_ctx* ctx, const double* a, int64_t lda, int ka, const double* b, int64_t ldb, int kb, int32_t n,
               bool lower_only, std::vector<double>& out) {
    out.assign(static_cast<size_t>(ka) * kb, 0.0);
    if (ka == 0 || kb == 0) return;
    const int nti = (ka + kGT - 1) / kGT, ntj = (kb + kGT - 1) / kGT;
    const int gx = std::max(1, std::min<int>((n + kGR - 1) / kGR, std::max(1, ctx->num_sms * 4 / (nti * ntj))));
    double* part = dev_alloc(static_cast<int64_t>(ka) * kb * gx);
    double* res = dev_alloc(static_cast<int64_t>(ka) * kb);
    RCG_CK(cudaMemsetAsync(part, 0, sizeof(double) * ka * kb * gx, ctx->stream));
    dim3 grid(gx, nti * ntj);
    k_gram_partial<<<grid, 256, 0, ctx->stream>>>(a, lda, ka, b, ldb, kb, n, part, lower_only ? 1 : 0);
    RCG_LAUNCHED(ctx);
    k_gram_final<<<(ka * kb + 255) / 256, 256, 0, ctx->stream>>>(part, ka, kb, gx, lower_only ? 1 : 0, res);
    RCG_LAUNCHED(ctx);
    RCG_CK(cudaMemcpyAsync(out.data(), res, sizeof(double) * ka * kb, cudaMemcpyDeviceToHost, ctx->stream));
    RCG_CK(cudaStreamSynchronize(ctx->stream));
    dev_free(part);
    dev_free(res);
}

void combine_cols(rcg_ctx* ctx, const double* e, int64_t lde, int k, const double* t_host, int kc, double* y,
                  int64_t ldy, int32_t n) {
    if (kc == 0 || n == 0) return;
    double* tdev = dev_alloc(static_cast<int64_t>(kc) * std::max(k, 1));
    RCG_CK(cudaMemcpyAsync(tdev, t_host, sizeof(double) * kc * k, cudaMemcpyHostToDevice, ctx->stream));
    for (int c0 = 0; c0 < kc; c0 += kComb) {
        const int cc = std::min(kComb, kc - c0);
        const size_t smem = sizeof(double) * cc * std::max(k, 1);
        k_combine<<<stream_grid(ctx, n), kStreamThreads, smem, ctx->stream>>>(e, lde, k, tdev + c0 * k, cc,
                                                                              y + c0 * ldy, ldy, n);
        RCG_LAUNCHED(ctx);
    }
    RCG_CK(cudaStreamSynchronize(ctx->stream));
    dev_free(tdev);
}

// f = C^T y on the device, returned to the host
static void tall_dot_host(rcg_ctx* ctx, const double* C, int64_t ldc, int k, const double* y, int32_t n,
                          std::vector<double>& f) {
    ensure_red(ctx, n);
    f.assign(k, 0.0);
    if (k == 0) return;
    double* fd = dev_alloc(k);
    k_tall_dot<<<stream_grid(ctx, n), kStreamThreads, 0, ctx->stream>>>(C, ldc, k, y, n, ctx->ws.partials,
                                                                        &ctx->ws.st->tick[7], fd);
    RCG_LAUNCHED(ctx);
    RCG_CK(cudaMemcpyAsync(f.data(), fd, sizeof(double) * k, cudaMemcpyDeviceToHost, ctx->stream));
    RCG_CK(cudaStreamSynchronize(ctx->stream));
    dev_free(fd);
}

static double dev_dot(rcg_ctx* ctx, const double* a, const double* b, int32_t n, double* c_slot) {
    k_mgs_pass<<<stream_grid(ctx, n), kStreamThreads, 0, ctx->stream>>>(const_cast<double*>(b), a, 0, 0, 1, c_slot, n,
                                                                        ctx->ws.partials, &ctx->ws.st->tick[7]);
    RCG_LAUNCHED(ctx);
    double h = 0.0;
    RCG_CK(cudaMemcpyAsync(&h, c_slot, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    RCG_CK(cudaStreamSynchronize(ctx->stream));
    return h;
}

// single-pass MGS (src/dense.cpp:45-61) of the vk columns at v (leading dimension vld) into e
// (leading dimension eld); returns the number kept.  e may be v itself (in place: the kept column
// `kept` <= src is a column already consumed).
static int mgs_core(rcg_ctx* ctx, const double* v, int64_t vld, int vk, int32_t n, double* e, int64_t eld,
                    double drop_tol) {
    ensure_red(ctx, n);
    const int g = stream_grid(ctx, n);
    double* c = dev_alloc(vk + 2);
    int kept = 0;
    try {
        for (int src = 0; src < vk; ++src) {
            double* w = e + kept * eld;
            if (w != v + src * vld) {
                k_copy_col<<<g, kStreamThreads, 0, ctx->stream>>>(v + src * vld, w, n);
                RCG_LAUNCHED(ctx);
            }
            const double n0 = std::sqrt(dev_dot(ctx, w, w, n, c + vk));
            if (n0 == 0.0) continue;
            for (int q = 0; q <= kept; ++q) {
                k_mgs_pass<<<g, kStreamThreads, 0, ctx->stream>>>(w, e, eld, q, kept, c, n, ctx->ws.partials,
                                                                  &ctx->ws.st->tick[7]);
                RCG_LAUNCHED(ctx);
            }
            double n1sq = 0.0;
            RCG_CK(cudaMemcpyAsync(&n1sq, c + kept, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
            RCG_CK(cudaStreamSynchronize(ctx->stream));
            const double n1 = std::sqrt(n1sq);
            if (n1 <= drop_tol * n0) continue;
            k_div_sqrt<<<g, kStreamThreads, 0, ctx->stream>>>(w, n, c + kept);
            RCG_LAUNCHED(ctx);
            ++kept;
        }
        RCG_CK(cudaStreamSynchronize(ctx->stream));
    } catch (...) {
        dev_free(c);
        throw;
    }
    dev_free(c);
    return kept;
}

static rcg_tall* mgs(rcg_ctx* ctx, const rcg_tall* v, double drop_tol) {
    rcg_tall* e = tall_alloc(v->n, v->k);
    try {
        e->k = mgs_core(ctx, v->d, v->ld, v->k, v->n, e->d, e->ld, drop_tol);
    } catch (...) {
        rcg_tall_destroy(e);
        throw;
    }
    return e;
}

// values ascending + T (k x k, T[c*k + j] = component j of eigenvector c)
static void rr_small(rcg_ctx* ctx, const rcg_matrix* a, const rcg_tall* e, std::vector<double>& values,
                     std::vector<double>& T) {
    const int k = e->k;
    values.clear();
    T.clear();
    if (k == 0) return;
    require(k <= 128, "SmallSym: dimension " + std::to_string(k) + " outside [0, 128]");
    double* ae = dev_alloc(e->ld * k);
    try {
        launch_spmm(ctx, a, e->d, e->ld, ae, e->ld, k);
        std::vector<double> s;
        gram_host(ctx, e->d, e->ld, k, ae, e->ld, k, e->n, true, s);
        for (int i = 0; i < k; ++i)
            for (int j = 0; j < i; ++j) s[static_cast<size_t>(j) * k + i] = s[static_cast<size_t>(i) * k + j];
        sym_eig_host(k, s, values, T);
    } catch (...) {
        dev_free(ae);
        throw;
    }
    dev_free(ae);
}

static rcg_tall* harvest(rcg_ctx* ctx, const double* x_dev, const rcg_sampler* s, bool raw) {
    std::vector<int> occ(s->m);
    RCG_CK(cudaMemcpy(occ.data(), s->occupied, sizeof(int) * s->m, cudaMemcpyDeviceToHost));
    std::vector<int> list;
    for (int j = 0; j < s->m; ++j)
        if (occ[j]) list.push_back(j);
    rcg_tall* e = tall_alloc(s->n, static_cast<int>(list.size()));
    e->k = 0;
    if (list.empty() || s->n == 0) return e;
    int* dl = nullptr;
    int* nz = nullptr;
    try {
        dl = static_cast<int*>(dev_alloc_bytes(sizeof(int) * list.size()));
        nz = static_cast<int*>(dev_alloc_bytes(sizeof(int) * list.size()));
        RCG_CK(cudaMemcpyAsync(dl, list.data(), sizeof(int) * list.size(), cudaMemcpyHostToDevice, ctx->stream));
        RCG_CK(cudaMemsetAsync(nz, 0, sizeof(int) * list.size(), ctx->stream));
        dim3 grid(stream_grid(ctx, s->n), std::min<int>(static_cast<int>(list.size()), 64));
        k_harvest<<<grid, kStreamThreads, 0, ctx->stream>>>(x_dev, s->slots, s->ld, dl, static_cast<int>(list.size()),
                                                            raw ? 1 : 0, e->d, e->ld, s->n, nz);
        RCG_LAUNCHED(ctx);
        std::vector<int> hz(list.size());
        RCG_CK(cudaMemcpyAsync(hz.data(), nz, sizeof(int) * list.size(), cudaMemcpyDeviceToHost, ctx->stream));
        RCG_CK(cudaStreamSynchronize(ctx->stream));
        int out = 0;
        for (size_t j = 0; j < list.size(); ++j) {
            if (!hz[j]) continue;  // exactly zero column: skipped (recycling.cpp:26)
            if (static_cast<int>(j) != out)
                RCG_CK(cudaMemcpyAsync(e->d + out * e->ld, e->d + j * e->ld, sizeof(double) * s->n,
                                       cudaMemcpyDeviceToDevice, ctx->stream));
            ++out;
        }
        e->k = out;
        RCG_CK(cudaStreamSynchronize(ctx->stream));
    } catch (...) {
        dev_free(dl);
        dev_free(nz);
        rcg_tall_destroy(e);
        throw;
    }
    dev_free(dl);
    dev_free(nz);
    return e;
}

void condest_ritz(rcg_ctx* ctx, const rcg_matrix* a, const double* x_dev, rcg_sampler* smp, rcg_cond_estimate* est) {
    rcg_tall* errs = harvest(ctx, x_dev, smp, false);
    rcg_tall* e = nullptr;
    try {
        e = mgs(ctx, errs, 1e-12);
        if (e->k > 0) {
            std::vector<double> vals, T;
            rr_small(ctx, a, e, vals, T);
            est->nritz = e->k;
            if (est->ritz_values) std::memcpy(est->ritz_values, vals.data(), sizeof(double) * vals.size());
            est->lambda_min = vals[0];
            est->lambda_min_available = 1;
            est->kappa = est->lambda_max / est->lambda_min;
        }
    } catch (...) {
        rcg_tall_destroy(errs);
        rcg_tall_destroy(e);
        throw;
    }
    rcg_tall_destroy(errs);
    rcg_tall_destroy(e);
}


// ------------------------------------------------------------------ memory-lean recycling
// For problems whose error block does not fit next to the sampler slots (C4 on one GPU: 64 slots
// of 1.07 GB, and the standard path's E, its MGS copy and A E would add 3 x 69 GB): the errors
// are formed in place in the slots (x - slot, recycling.cpp:17-28; exactly-zero columns skipped
// and the rest compacted in slot order), orthonormalised in place (same MGS and drop rule), and
// the Rayleigh-Ritz Gram is streamed one column at a time (S[:, j] = Q^T (A q_j), lower triangle
// mirrored as rayleigh_ritz does) -- one extra n-vector instead of an n x k block.  The Ritz
// values agree with the standard path to rounding (different dot grouping).  The sampler's slots
// hold the orthonormal basis afterwards: the sampler is spent.
__global__ void k_harvest_inplace(const double* __restrict__ x, double* __restrict__ slots, int64_t lds,
                                  const int* __restrict__ list, int cnt, int32_t n, int* __restrict__ nonzero) {
    for (int j = blockIdx.y; j < cnt; j += gridDim.y) {
        double* s = slots + list[j] * lds;
        int nz = 0;
        for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
            const double v = __dsub_rn(x[i], s[i]);
            s[i] = v;
            nz |= (v != 0.0);
        }
        if (__syncthreads_or(nz) && threadIdx.x == 0) atomicOr(nonzero + j, 1);
    }
}

void lean_build_aux(rcg_ctx* ctx, const rcg_matrix* a, const double* x_dev, rcg_sampler* s, double theta,
                    int keep_count, int* m_bar, std::vector<double>& vals, double* theta_used, rcg_tall** w_out) {
    *w_out = nullptr;
    const int32_t n = s->n;
    std::vector<int> occ(s->m);
    RCG_CK(cudaMemcpy(occ.data(), s->occupied, sizeof(int) * s->m, cudaMemcpyDeviceToHost));
    std::vector<int> list;
    for (int j = 0; j < s->m; ++j)
        if (occ[j]) list.push_back(j);
    const int k0 = static_cast<int>(list.size());
    int kk = 0;
    if (k0 > 0 && n > 0) {
        int* dl = static_cast<int*>(dev_alloc_bytes(sizeof(int) * k0));
        int* nz = static_cast<int*>(dev_alloc_bytes(sizeof(int) * k0));
        RCG_CK(cudaMemcpyAsync(dl, list.data(), sizeof(int) * k0, cudaMemcpyHostToDevice, ctx->stream));
        RCG_CK(cudaMemsetAsync(nz, 0, sizeof(int) * k0, ctx->stream));
        dim3 grid(stream_grid(ctx, n), std::min(k0, 64));
        k_harvest_inplace<<<grid, kStreamThreads, 0, ctx->stream>>>(x_dev, s->slots, s->ld, dl, k0, n, nz);
        RCG_LAUNCHED(ctx);
        std::vector<int> hz(k0);
        RCG_CK(cudaMemcpyAsync(hz.data(), nz, sizeof(int) * k0, cudaMemcpyDeviceToHost, ctx->stream));
        RCG_CK(cudaStreamSynchronize(ctx->stream));
        dev_free(dl);
        dev_free(nz);
        for (int j = 0; j < k0; ++j) {  // compact in slot order (targets are consumed columns)
            if (!hz[j]) continue;
            if (list[j] != kk)
                RCG_CK(cudaMemcpyAsync(s->slots + kk * s->ld, s->slots + list[j] * s->ld, sizeof(double) * n,
                                       cudaMemcpyDeviceToDevice, ctx->stream));
            ++kk;
        }
    }
    const int kept = kk ? mgs_core(ctx, s->slots, s->ld, kk, n, s->slots, s->ld, 1e-12) : 0;
    *m_bar = kept;
    vals.clear();
    std::vector<double> T;
    if (kept > 0) {
        require(kept <= 128, "SmallSym: dimension " + std::to_string(kept) + " outside [0, 128]");
        std::vector<double> S(static_cast<size_t>(kept) * kept, 0.0), f;
        double* y = dev_alloc(std::max<int64_t>(s->ld, 1));
        try {
            for (int j = 0; j < kept; ++j) {
                const int rc = rcg_spmv(ctx, a, s->slots + j * s->ld, y);
                if (rc != RCG_OK) throw Error(rc, rcg_last_error());
                tall_dot_host(ctx, s->slots, s->ld, kept, y, n, f);
                for (int i = j; i < kept; ++i) S[static_cast<size_t>(i) * kept + j] = f[i];
            }
        } catch (...) {
            dev_free(y);
            throw;
        }
        dev_free(y);
        for (int i = 0; i < kept; ++i)
            for (int j = 0; j < i; ++j) S[static_cast<size_t>(j) * kept + i] = S[static_cast<size_t>(i) * kept + j];
        sym_eig_host(kept, S, vals, T);
    }
    double th = theta;
    if (keep_count > 0)
        th = kept > keep_count ? 0.5 * (vals[keep_count - 1] + vals[keep_count]) : std::numeric_limits<double>::infinity();
    if (theta_used) *theta_used = th;
    int sel = 0;
    while (sel < kept && vals[sel] < th) ++sel;
    rcg_tall* out = tall_alloc(n, sel);
    try {
        combine_cols(ctx, s->slots, s->ld, kept, T.data(), sel, out->d, out->ld, n);
    } catch (...) {
        rcg_tall_destroy(out);
        throw;
    }
    *w_out = out;
}

// rcg_basis_create; adopt = take over w's column block instead of copying it (w->d becomes null:
// the memory-lean sequence on C4, where a 34 GB copy of W does not fit next to W and A W)
void basis_build(rcg_ctx* ctx, const rcg_matrix* a, rcg_tall* w, int who, bool adopt, rcg_basis** out) {
    {
        *out = nullptr;
        const char* whom = who == RCG_BASIS_SC ? "ScPreconditioner" : "build_deflation_operator";
        if (w->k > 0 && w->n != a->n) throw Error(RCG_E_INVALID, std::string(whom) + ": W row count does not match A");
        require(w->k <= 128, "SmallSym: dimension " + std::to_string(w->k) + " outside [0, 128]");
        auto* b = new rcg_basis();
        try {
            b->n = a->n;
            b->k = w->k;
            b->ld = w->ld;
            b->who = who;
            if (b->k > 0) {
                if (adopt) {
                    b->w = w->d;
                    w->d = nullptr;
                } else {
                    b->w = dev_alloc(b->ld * b->k);
                    RCG_CK(cudaMemcpyAsync(b->w, w->d, sizeof(double) * b->ld * b->k, cudaMemcpyDeviceToDevice,
                                           ctx->stream));
                }
                b->aw = dev_alloc(b->ld * b->k);
                launch_spmm(ctx, a, b->w, b->ld, b->aw, b->ld, b->k);
                std::vector<double> s;
                gram_host(ctx, b->w, b->ld, b->k, b->aw, b->ld, b->k, b->n, true, s);
                const int k = b->k;
                for (int i = 0; i < k; ++i)
                    for (int j = 0; j < i; ++j) s[static_cast<size_t>(j) * k + i] = s[static_cast<size_t>(i) * k + j];
                int bad = -1;
                if (!chol_factor_host(k, s, b->h_l, &bad))
                    throw Error(RCG_E_BREAKDOWN, std::string(whom) + ": W^T A W not SPD");
                b->l = dev_alloc(static_cast<int64_t>(k) * k);
                RCG_CK(cudaMemcpyAsync(b->l, b->h_l.data(), sizeof(double) * k * k, cudaMemcpyHostToDevice, ctx->stream));
                RCG_CK(cudaStreamSynchronize(ctx->stream));
            }
        } catch (...) {
            rcg_basis_destroy(b);
            throw;
        }
        *out = b;
    }
}

}  // namespace rcg

using namespace rcg;

extern "C" {

// ------------------------------------------------------------------ TallDense
int rcg_tall_create(rcg_ctx* ctx, int32_t n, int k, const double* cols, rcg_tall** out) {
    return guard([&] {
        *out = nullptr;
        require(n >= 0 && k >= 0, "TallDense: bad dimensions");
        rcg_tall* t = tall_alloc(n, k);
        if (cols && k > 0 && n > 0) {
            RCG_CK(cudaMemcpy2DAsync(t->d, sizeof(double) * t->ld, cols, sizeof(double) * n, sizeof(double) * n, k,
                                     cudaMemcpyDefault, ctx->stream));
            RCG_CK(cudaStreamSynchronize(ctx->stream));
        }
        *out = t;
    });
}

void rcg_tall_destroy(rcg_tall* t) {
    if (!t) return;
    dev_free(t->d);
    delete t;
}

// a TallDense held as separate host (or device) columns -- the reference's std::vector<Vector>
int rcg_tall_create_cols(rcg_ctx* ctx, int32_t n, int k, const double* const* cols, rcg_tall** out) {
    return guard([&] {
        *out = nullptr;
        require(n >= 0 && k >= 0, "TallDense: bad dimensions");
        require(k == 0 || cols, "TallDense: null column array");
        rcg_tall* t = tall_alloc(n, k);
        try {
            for (int j = 0; j < k && n > 0; ++j) {
                require(cols[j] != nullptr, "TallDense: null column");
                RCG_CK(cudaMemcpyAsync(t->d + j * t->ld, cols[j], sizeof(double) * n, cudaMemcpyDefault, ctx->stream));
            }
            RCG_CK(cudaStreamSynchronize(ctx->stream));
        } catch (...) {
            rcg_tall_destroy(t);
            throw;
        }
        *out = t;
    });
}

// harvest_errors (recycling.cpp:17-28) for snapshots held by the caller (a host SamplerState's
// occupied slots, in slot order): E[:,j] = x_final - slot_j, exactly-zero columns skipped
int rcg_harvest_columns(rcg_ctx* ctx, const double* x_final, int32_t n, int k, const double* const* slots,
                        rcg_tall** out) {
    return guard([&] {
        *out = nullptr;
        rcg_tall* t = nullptr;
        ck(rcg_tall_create_cols(ctx, n, k, slots, &t));
        if (k == 0 || n == 0) {
            t->k = 0;
            *out = t;
            return;
        }
        int* dl = nullptr;
        int* nz = nullptr;
        try {
            Staged xs;
            stage_in(ctx, x_final, n, xs);
            std::vector<int> list(k);
            for (int j = 0; j < k; ++j) list[j] = j;
            dl = static_cast<int*>(dev_alloc_bytes(sizeof(int) * k));
            nz = static_cast<int*>(dev_alloc_bytes(sizeof(int) * k));
            RCG_CK(cudaMemcpyAsync(dl, list.data(), sizeof(int) * k, cudaMemcpyHostToDevice, ctx->stream));
            RCG_CK(cudaMemsetAsync(nz, 0, sizeof(int) * k, ctx->stream));
            dim3 grid(stream_grid(ctx, n), std::min(k, 64));
            k_harvest_inplace<<<grid, kStreamThreads, 0, ctx->stream>>>(xs.dev, t->d, t->ld, dl, k, n, nz);
            RCG_LAUNCHED(ctx);
            std::vector<int> hz(k);
            RCG_CK(cudaMemcpyAsync(hz.data(), nz, sizeof(int) * k, cudaMemcpyDeviceToHost, ctx->stream));
            RCG_CK(cudaStreamSynchronize(ctx->stream));
            int kept = 0;
            for (int j = 0; j < k; ++j) {
                if (!hz[j]) continue;  // exactly zero column: skipped (recycling.cpp:26)
                if (j != kept)
                    RCG_CK(cudaMemcpyAsync(t->d + kept * t->ld, t->d + j * t->ld, sizeof(double) * n,
                                           cudaMemcpyDeviceToDevice, ctx->stream));
                ++kept;
            }
            t->k = kept;
            RCG_CK(cudaStreamSynchronize(ctx->stream));
        } catch (...) {
            dev_free(dl);
            dev_free(nz);
            rcg_tall_destroy(t);
            throw;
        }
        dev_free(dl);
        dev_free(nz);
        *out = t;
    });
}

int rcg_tall_k(const rcg_tall* t) { return t ? t->k : 0; }
int32_t rcg_tall_n(const rcg_tall* t) { return t ? t->n : 0; }

int rcg_tall_download(rcg_ctx* ctx, const rcg_tall* t, double* cols_out) {
    return guard([&] {
        if (t->k == 0 || t->n == 0) return;
        RCG_CK(cudaMemcpy2DAsync(cols_out, sizeof(double) * t->n, t->d, sizeof(double) * t->ld, sizeof(double) * t->n,
                                 t->k, cudaMemcpyDefault, ctx->stream));
        RCG_CK(cudaStreamSynchronize(ctx->stream));
    });
}

int rcg_mgs_orthonormalize(rcg_ctx* ctx, const rcg_tall* v, double drop_tol, rcg_tall** out) {
    return guard([&] {
        *out = nullptr;
        *out = mgs(ctx, v, drop_tol);
    });
}

// ------------------------------------------------------------------ samplers
int rcg_sampler_create(rcg_ctx* ctx, int method, int m, int iteration_cap, double eps, int32_t n, rcg_sampler** out) {
    return guard([&] {
        *out = nullptr;
        auto* s = new rcg_sampler();
        try {
            if (method == RCG_SAMPLER_A) {
                if (m < 2) throw Error(RCG_E_INVALID, "sampler method A: m must be >= 2");
                if (iteration_cap < 1) throw Error(RCG_E_INVALID, "sampler method A: iteration cap must be >= 1");
                s->l_max = 1;
                long long pw = m;
                while (pw <= iteration_cap) {  // smallest l_max with m^l_max > cap (sampling.cpp:17-22)
                    pw *= m;
                    ++s->l_max;
                }
            } else if (method == RCG_SAMPLER_B) {
                if (m < 1) throw Error(RCG_E_INVALID, "sampler method B: m must be >= 1");
                if (!(eps > 0.0 && eps < 1.0)) throw Error(RCG_E_INVALID, "sampler method B: eps must be in (0, 1)");
                s->alpha = -std::log10(eps);
                s->h_thr.resize(m);
                for (int j = 1; j <= m; ++j) s->h_thr[j - 1] = std::pow(10.0, -double(j) * s->alpha / (m + 1));
            } else {
                throw Error(RCG_E_INVALID, "sampler: unknown method");
            }
            s->method = method;
            s->m = m;
            s->n = n;
            s->ld = ld_of(n);
            s->slots = dev_alloc(s->ld * m);
            s->occupied = static_cast<int*>(dev_alloc_bytes(sizeof(int) * m));
            s->stored_iter = static_cast<int*>(dev_alloc_bytes(sizeof(int) * m));
            RCG_CK(cudaMemsetAsync(s->occupied, 0, sizeof(int) * m, ctx->stream));
            RCG_CK(cudaMemsetAsync(s->stored_iter, 0, sizeof(int) * m, ctx->stream));
            s->thresholds = dev_alloc(m);
            if (!s->h_thr.empty())
                RCG_CK(cudaMemcpyAsync(s->thresholds, s->h_thr.data(), sizeof(double) * m, cudaMemcpyHostToDevice, ctx->stream));
            RCG_CK(cudaStreamSynchronize(ctx->stream));
        } catch (...) {
            rcg_sampler_destroy(s);
            throw;
        }
        *out = s;
    });
}

void rcg_sampler_destroy(rcg_sampler* s) {
    if (!s) return;
    dev_free(s->slots);
    dev_free(s->occupied);
    dev_free(s->stored_iter);
    dev_free(s->thresholds);
    delete s;
}

// host-driven offer (src/sampling.cpp:40-65); the solver applies the same schedule on device
int rcg_sampler_offer(rcg_ctx* ctx, rcg_sampler* s, int iteration, double relres, const double* payload) {
    return guard([&] {
        std::vector<int> fill;
        if (s->method == RCG_SAMPLER_A) {
            if (iteration % s->h != 0) return;
            long long acc = 0, pw = 1;
            for (int l = 0; l <= s->l_max; ++l) {
                const long long term = (iteration - 1) / pw;
                acc += (l % 2 == 0) ? term : -term;
                pw *= s->m;
            }
            fill.push_back(static_cast<int>(acc % s->m));
            if (iteration == s->h * s->m) s->h *= 2;
        } else {
            while (s->next_slot <= s->m) {
                if (relres > s->h_thr[s->next_slot - 1]) break;
                fill.push_back(s->next_slot - 1);
                s->next_slot++;
            }
        }
        const int one = 1;
        for (int slot : fill) {
            if (s->n > 0)
                RCG_CK(cudaMemcpyAsync(s->slots + slot * s->ld, payload, sizeof(double) * s->n, cudaMemcpyDefault, ctx->stream));
            RCG_CK(cudaMemcpyAsync(s->occupied + slot, &one, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
            RCG_CK(cudaMemcpyAsync(s->stored_iter + slot, &iteration, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
            RCG_CK(cudaStreamSynchronize(ctx->stream));
        }
    });
}

int rcg_sampler_state(const rcg_sampler* s, int* occupied, int* stored_iter) {
    int count = 0;
    const int st = guard([&] {
        std::vector<int> occ(s->m), it(s->m);
        RCG_CK(cudaMemcpy(occ.data(), s->occupied, sizeof(int) * s->m, cudaMemcpyDeviceToHost));
        RCG_CK(cudaMemcpy(it.data(), s->stored_iter, sizeof(int) * s->m, cudaMemcpyDeviceToHost));
        for (int j = 0; j < s->m; ++j) {
            if (occupied) occupied[j] = occ[j];
            if (stored_iter) stored_iter[j] = it[j];
            count += occ[j] ? 1 : 0;
        }
    });
    return st == RCG_OK ? count : -st;
}

int rcg_sampler_slot(rcg_ctx* ctx, const rcg_sampler* s, int slot, double* out) {
    return guard([&] {
        require(slot >= 0 && slot < s->m, "sampler: slot out of range");
        require(s->slots != nullptr || s->n == 0, "sampler: spent by a memory-lean recycling step");
        if (s->n == 0) return;
        RCG_CK(cudaMemcpyAsync(out, s->slots + slot * s->ld, sizeof(double) * s->n, cudaMemcpyDefault, ctx->stream));
        RCG_CK(cudaStreamSynchronize(ctx->stream));
    });
}

// ------------------------------------------------------------------ recycling
int rcg_harvest_errors(rcg_ctx* ctx, const double* x_final, const rcg_sampler* s, rcg_tall** out) {
    return guard([&] {
        *out = nullptr;
        Staged xs;
        stage_in(ctx, x_final, s->n, xs);
        *out = harvest(ctx, xs.dev, s, false);
    });
}

int rcg_harvest_stored(rcg_ctx* ctx, const rcg_sampler* s, rcg_tall** out) {
    return guard([&] {
        *out = nullptr;
        *out = harvest(ctx, nullptr, s, true);
    });
}

int rcg_rayleigh_ritz(rcg_ctx* ctx, const rcg_matrix* a, const rcg_tall* e, double* values, rcg_tall** vectors) {
    return guard([&] {
        if (vectors) *vectors = nullptr;
        require(e->k == 0 || e->n == a->n, "rayleigh_ritz: basis row count does not match A");
        std::vector<double> vals, T;
        rr_small(ctx, a, e, vals, T);
        if (values && !vals.empty()) std::memcpy(values, vals.data(), sizeof(double) * vals.size());
        if (vectors) {
            rcg_tall* v = tall_alloc(e->n, e->k);
            try {
                combine_cols(ctx, e->d, e->ld, e->k, T.data(), e->k, v->d, v->ld, e->n);
            } catch (...) {
                rcg_tall_destroy(v);
                throw;
            }
            *vectors = v;
        }
    });
}

int rcg_build_aux_matrix(rcg_ctx* ctx, const rcg_matrix* a, const rcg_tall* errors, double theta, int keep_count,
                         int* m_bar, double* values, double* theta_used, rcg_tall** w) {
    NvtxRange range("rcg_build_aux_matrix");
    return guard([&] {
        *w = nullptr;
        *m_bar = 0;
        require(errors->k == 0 || errors->n == a->n, "build_aux_matrix: error rows do not match A");
        rcg_tall* e = mgs(ctx, errors, 1e-12);
        try {
            *m_bar = e->k;
            std::vector<double> vals, T;
            rr_small(ctx, a, e, vals, T);
            double th = theta;
            if (keep_count > 0)
                th = e->k > keep_count ? 0.5 * (vals[keep_count - 1] + vals[keep_count])
                                       : std::numeric_limits<double>::infinity();
            if (theta_used) *theta_used = th;
            if (values && !vals.empty()) std::memcpy(values, vals.data(), sizeof(double) * vals.size());
            int sel = 0;
            while (sel < e->k && vals[sel] < th) ++sel;  // ascending: strict selection (recycling.cpp:91-94)
            rcg_tall* out = tall_alloc(a->n, sel);
            try {
                combine_cols(ctx, e->d, e->ld, e->k, T.data(), sel, out->d, out->ld, a->n);
            } catch (...) {
                rcg_tall_destroy(out);
                throw;
            }
            *w = out;
        } catch (...) {
            rcg_tall_destroy(e);
            throw;
        }
        rcg_tall_destroy(e);
    });
}

// ------------------------------------------------------------------ basis (deflation / SC)
int rcg_basis_create(rcg_ctx* ctx, const rcg_matrix* a, const rcg_tall* w, int who, rcg_basis** out) {
    return guard([&] { basis_build(ctx, a, const_cast<rcg_tall*>(w), who, false, out); });
}

void rcg_basis_destroy(rcg_basis* b) {
    if (!b) return;
    dev_free(b->w);
    dev_free(b->aw);
    dev_free(b->l);
    delete b;
}

int rcg_basis_k(const rcg_basis* b) { return b ? b->k : 0; }

// a basis from the fields of an existing host DeflationOperator / ScPreconditioner (W, AW and
// chol(W^T A W) as they are -- the operator that object applies), no recomputation
int rcg_basis_create_from(rcg_ctx* ctx, int32_t n, int k, const double* const* w_cols, const double* const* aw_cols,
                          const double* chol_l, int who, rcg_basis** out) {
    return guard([&] {
        *out = nullptr;
        require(n >= 0 && k >= 0 && k <= 128, "SmallSym: dimension " + std::to_string(k) + " outside [0, 128]");
        require(k == 0 || (w_cols && aw_cols && chol_l), "basis: null W / AW / Cholesky factor");
        auto* b = new rcg_basis();
        try {
            b->n = n;
            b->k = k;
            b->ld = ld_of(n);
            b->who = who;
            if (k > 0) {
                b->w = dev_alloc(b->ld * k);
                b->aw = dev_alloc(b->ld * k);
                for (int j = 0; j < k && n > 0; ++j) {
                    require(w_cols[j] && aw_cols[j], "basis: null column");
                    RCG_CK(cudaMemcpyAsync(b->w + j * b->ld, w_cols[j], sizeof(double) * n, cudaMemcpyDefault, ctx->stream));
                    RCG_CK(cudaMemcpyAsync(b->aw + j * b->ld, aw_cols[j], sizeof(double) * n, cudaMemcpyDefault,
                                           ctx->stream));
                }
                b->h_l.assign(chol_l, chol_l + static_cast<size_t>(k) * k);
                b->l = dev_alloc(static_cast<int64_t>(k) * k);
                RCG_CK(cudaMemcpyAsync(b->l, b->h_l.data(), sizeof(double) * k * k, cudaMemcpyHostToDevice, ctx->stream));
                RCG_CK(cudaStreamSynchronize(ctx->stream));
            }
        } catch (...) {
            rcg_basis_destroy(b);
            throw;
        }
        *out = b;
    });
}

// the basis back on the host: AW column-major (ld n) and chol(W^T A W) row-major k x k
int rcg_basis_export(rcg_ctx* ctx, const rcg_basis* b, double* aw_cols, double* chol_l) {
    return guard([&] {
        require(b != nullptr, "basis: null handle");
        if (aw_cols && b->k > 0 && b->n > 0) {
            RCG_CK(cudaMemcpy2DAsync(aw_cols, sizeof(double) * b->n, b->aw, sizeof(double) * b->ld, sizeof(double) * b->n,
                                     b->k, cudaMemcpyDefault, ctx->stream));
            RCG_CK(cudaStreamSynchronize(ctx->stream));
        }
        if (chol_l && b->k > 0) std::memcpy(chol_l, b->h_l.data(), sizeof(double) * b->k * b->k);
    });
}

// Preconditioner::apply on the device: identity copies, IC(0) is ic_apply, subspace correction is
// ScPreconditioner::apply (subspace_correction.cpp:47-57): z = inner(r), then z += W u with
// u = chol(W^T r), columns added in order (z_i += u_j w_ij, rounded product then sum)
int rcg_prec_apply(rcg_ctx* ctx, const rcg_prec* m, const double* r, double* z) {
    return guard([&] {
        require(m != nullptr, "preconditioner: null");
        int32_t n = -1;
        if (m->ic) n = m->ic->n;
        if (m->sc) n = m->sc->n;
        require(m->kind == RCG_PREC_IDENTITY || m->kind == RCG_PREC_IC || m->kind == RCG_PREC_SC,
                "preconditioner: unknown kind");
        require(m->kind != RCG_PREC_IC || m->ic, "preconditioner: IC without a factor");
        require(m->kind != RCG_PREC_SC || m->sc, "preconditioner: SC without a basis");
        require(n >= 0, "preconditioner: an identity preconditioner has no length here (z = r needs no call)");
        Staged rs, zs;
        stage_in(ctx, r, n, rs);
        stage_out_begin(ctx, z, n, zs);
        if (m->ic)
            ic_apply_dev(ctx, m->ic, rs.dev, zs.dev);
        else if (zs.dev != rs.dev && n > 0)
            RCG_CK(cudaMemcpyAsync(zs.dev, rs.dev, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream));
        if (m->kind == RCG_PREC_SC && m->sc->k > 0) {
            const rcg_basis* b = m->sc;
            std::vector<double> f, u(b->k);
            tall_dot_host(ctx, b->w, b->ld, b->k, rs.dev, b->n, f);
            chol_solve_host(b->k, b->h_l, f.data(), u.data());
            for (double& v : u) v = -v;  // z - (-u_j) w_j == z + u_j w_j exactly
            double* ud = dev_alloc(b->k);
            RCG_CK(cudaMemcpyAsync(ud, u.data(), sizeof(double) * b->k, cudaMemcpyHostToDevice, ctx->stream));
            k_apply_combination<<<stream_grid(ctx, n), kStreamThreads, 0, ctx->stream>>>(zs.dev, b->w, b->ld, b->k, ud,
                                                                                        n, zs.dev, 0);
            RCG_LAUNCHED(ctx);
            RCG_CK(cudaStreamSynchronize(ctx->stream));
            dev_free(ud);
        }
        stage_out_end(ctx, z, n, zs);
        RCG_CK(cudaStreamSynchronize(ctx->stream));
        check_sweep_watchdog(ctx);
    });
}

static int projection(rcg_ctx* ctx, const rcg_basis* b, const double* y, double* out, int which) {
    return guard([&] {
        Staged ys, os;
        stage_in(ctx, y, b->n, ys);
        stage_out_begin(ctx, out, b->n, os);
        if (b->k == 0) {
            if (which == 2)
                launch_fill(ctx, os.dev, b->n, 0.0);
            else if (os.dev != ys.dev)
                RCG_CK(cudaMemcpyAsync(os.dev, ys.dev, sizeof(double) * b->n, cudaMemcpyDeviceToDevice, ctx->stream));
        } else {
            // which 0: P^T y = y - AW u, u = chol(W^T y); 1: P x = x - W u, u = chol((AW)^T x);
            // 2: W u, u = chol(W^T b) (src/deflation.cpp:17-43)
            const double* C = which == 1 ? b->aw : b->w;
            std::vector<double> f, u(b->k);
            tall_dot_host(ctx, C, b->ld, b->k, ys.dev, b->n, f);
            chol_solve_host(b->k, b->h_l, f.data(), u.data());
            double* ud = dev_alloc(b->k);
            RCG_CK(cudaMemcpyAsync(ud, u.data(), sizeof(double) * b->k, cudaMemcpyHostToDevice, ctx->stream));
            const double* D = which == 0 ? b->aw : b->w;
            k_apply_combination<<<stream_grid(ctx, b->n), kStreamThreads, 0, ctx->stream>>>(
                ys.dev, D, b->ld, b->k, ud, b->n, os.dev, which == 2 ? 1 : 0);
            RCG_LAUNCHED(ctx);
            RCG_CK(cudaStreamSynchronize(ctx->stream));
            dev_free(ud);
        }
        stage_out_end(ctx, out, b->n, os);
        RCG_CK(cudaStreamSynchronize(ctx->stream));
    });
}

int rcg_project_pt(rcg_ctx* ctx, const rcg_basis* b, const double* y, double* out) { return projection(ctx, b, y, out, 0); }
int rcg_project_p(rcg_ctx* ctx, const rcg_basis* b, const double* x, double* out) { return projection(ctx, b, x, out, 1); }
int rcg_direct_component(rcg_ctx* ctx, const rcg_basis* b, const double* rhs, double* out) {
    return projection(ctx, b, rhs, out, 2);
}

}  // extern "C"
