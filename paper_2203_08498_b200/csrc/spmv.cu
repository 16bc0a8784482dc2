// spmv.cu -- CSR upload/validation and the SpMV family (K1 spmv, K2 spmv_dual, SpMM for A*E and
// A*W, the initial-residual variant and diagonal scaling).
//
// Kernel shape (B200): a persistent grid of 8-warp CTAs; each warp owns a tile of 32
// consecutive rows, stages the tile's contiguous CSR entries (values + columns) into its own
// shared-memory chunk with coalesced 256-byte warp loads, and each lane then sums ONE row
// sequentially from 0.0 in stored column order with separate multiply/add roundings -- exactly
// the reference loop of src/csr_matrix.cpp:95-99, so results are bitwise equal to the reference.
// Gathers of x go through the read-only path (L1/L2; x is L2-resident for C1-C3).
// Algorithmic bytes per launch: 12 nnz + 20 n.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "internal.cuh"
#include "kernels.cuh"
#include "spmv_pipe.cuh"

namespace rcg {

// y_v = A x_v for NV vectors (plain spmv / spmv_dual)
template <int NV>
__global__ void __launch_bounds__(kSpmvThreads) k_spmv(SpmvArgs a, int cap) {
    spmv_pipeline<NV>(a, cap, [&](int32_t row, const double (&acc)[NV]) {
#pragma unroll
        for (int v = 0; v < NV; ++v) a.y[v][row] = acc[v];
    });
}

// r = b - A x (src/pcg.cpp:50-52: spmv then r[i] = b[i] - r[i]); partials of (b,b) and (r,r)
__global__ void __launch_bounds__(kSpmvThreads) k_residual(SpmvArgs a, int cap, const double* __restrict__ b,
                                                           DevState* st) {
    __shared__ double red[2 * 32];
    __shared__ double tot[2];
    double acc2[2] = {0.0, 0.0};
    spmv_pipeline<1>(a, cap, [&](int32_t row, const double (&acc)[1]) {
        const double bi = b[row];
        const double ri = __dsub_rn(bi, acc[0]);
        a.y[0][row] = ri;
        acc2[0] = fadd_mul(acc2[0], bi, bi);
        acc2[1] = fadd_mul(acc2[1], ri, ri);
    });
    block_sum<2>(acc2, red);
    if (grid_reduce<2>(acc2, a.partials, blockIdx.x, gridDim.x, &st->tick[0], tot, red)) {
        if (threadIdx.x == 0) {
            st->bnorm = sqrt(tot[0]);
            st->rr = tot[1];
        }
    }
}

// SpMM: y[:,c] = A x[:,c] for c < k (k <= 8 per launch), each column bitwise equal to spmv
template <int KC>
__global__ void __launch_bounds__(kSpmvThreads) k_spmm(const int32_t* __restrict__ rs,
                                                       const int32_t* __restrict__ ci,
                                                       const double* __restrict__ va, int32_t n,
                                                       const double* __restrict__ x, int64_t ldx,
                                                       double* __restrict__ y, int64_t ldy, int k) {
    __shared__ double sv[kSpmvThreads / 32][kSpmvChunk];
    __shared__ int32_t sc[kSpmvThreads / 32][kSpmvChunk];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntiles = (n + 31) / 32;
    const int nw = gridDim.x * (kSpmvThreads / 32);
    for (int t = blockIdx.x * (kSpmvThreads / 32) + wid; t < ntiles; t += nw) {
        const int32_t r0 = t * 32, row = r0 + lane, rend = min(r0 + 32, n);
        const int32_t e0 = __ldg(rs + r0), e1 = __ldg(rs + rend);
        const int32_t my_b = row < n ? __ldg(rs + row) : e1;
        const int32_t my_e = row < n ? __ldg(rs + row + 1) : e1;
        double acc[KC];
#pragma unroll
        for (int c = 0; c < KC; ++c) acc[c] = 0.0;
        for (int32_t c0 = e0; c0 < e1; c0 += kSpmvChunk) {
            const int32_t c1 = min(c0 + kSpmvChunk, e1);
            __syncwarp();
            for (int32_t e = c0 + lane; e < c1; e += 32) {
                sv[wid][e - c0] = va[e];
                sc[wid][e - c0] = ci[e];
            }
            __syncwarp();
            const int32_t bb = max(my_b, c0), en = min(my_e, c1);
            for (int32_t e = bb; e < en; ++e) {
                const double av = sv[wid][e - c0];
                const int64_t col = sc[wid][e - c0];
#pragma unroll
                for (int c = 0; c < KC; ++c)
                    if (c < k) acc[c] = fadd_mul(acc[c], av, __ldg(x + c * ldx + col));
            }
        }
        if (row < n) {
#pragma unroll
            for (int c = 0; c < KC; ++c)
                if (c < k) y[c * ldy + row] = acc[c];
        }
    }
}

// a_ij * dis_i * dis_j with dis = 1/sqrt(a_ii)  (src/scaling.cpp:20-38, bitwise)
__global__ void k_diag_inv_sqrt(const int32_t* __restrict__ rs, const int32_t* __restrict__ ci,
                                const double* __restrict__ va, int32_t n, double* __restrict__ dis,
                                int* bad) {
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double d = 0.0;
        for (int32_t p = rs[i]; p < rs[i + 1]; ++p)
            if (ci[p] == i) d = va[p];
        if (d <= 0.0) atomicMin(bad, i);
        dis[i] = __ddiv_rn(1.0, __dsqrt_rn(d));
    }
}

__global__ void k_diag_scale(const int32_t* __restrict__ rs, const int32_t* __restrict__ ci,
                             const double* __restrict__ va, int32_t n, const double* __restrict__ dis,
                             double* __restrict__ out) {
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double di = dis[i];
        for (int32_t p = rs[i]; p < rs[i + 1]; ++p) out[p] = __dmul_rn(__dmul_rn(va[p], di), dis[ci[p]]);
    }
}

__global__ void k_fill(double* p, int64_t n, double v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

__global__ void k_fill_bits(double* p, int64_t n, unsigned long long bits) {
    const double v = __longlong_as_double(static_cast<long long>(bits));
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

// ------------------------------------------------------------------ launchers
int spmv_grid(const rcg_ctx* ctx, int32_t n) {
    const int tiles = (n + 31) / 32;
    const int blocks = (tiles + kPipeWarps - 1) / kPipeWarps;
    return std::max(1, std::min(blocks, ctx->num_sms * ctx->spmv_bps));
}

// dynamic shared memory of the pipelined SpMV kernels (raises the opt-in limit once per kernel)
size_t spmv_smem(const rcg_matrix* a) { return pipe_smem_bytes(a->cap); }

// opt-in dynamic shared memory up to the per-block limit minus the kernel's static usage
void allow_smem(const void* kernel) {
    int dev = 0, optin = 0;
    RCG_CK(cudaGetDevice(&dev));
    RCG_CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes fa{};
    RCG_CK(cudaFuncGetAttributes(&fa, kernel));
    RCG_CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                optin - static_cast<int>(fa.sharedSizeBytes)));
}

// same preferred carveout for all hot kernels (RCG_CARVEOUT percent of the maximum smem)
void set_carveout(const void* kernel) {
    static int pct = [] {
        const char* e = std::getenv("RCG_CARVEOUT");
        return e ? std::atoi(e) : 50;
    }();
    if (pct >= 0) RCG_CK(cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
}

void spmv_prepare_kernels() {
    static bool done = false;
    if (done) return;
    set_carveout(reinterpret_cast<const void*>(k_spmv<1>));
    set_carveout(reinterpret_cast<const void*>(k_spmv<2>));
    set_carveout(reinterpret_cast<const void*>(k_residual));
    allow_smem(reinterpret_cast<const void*>(k_spmv<1>));
    allow_smem(reinterpret_cast<const void*>(k_spmv<2>));
    allow_smem(reinterpret_cast<const void*>(k_residual));
    done = true;
}

int stream_grid(const rcg_ctx* ctx, int64_t n) {
    const int64_t blocks = (n + kStreamThreads * 4 - 1) / (kStreamThreads * 4);
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(blocks, ctx->num_sms * 4)));
}

static SpmvArgs make_args(const rcg_matrix* a) {
    SpmvArgs s{};
    s.rs = a->rs;
    s.ci = a->ci;
    s.va = a->va;
    s.n = a->n;
    return s;
}

void launch_spmv(rcg_ctx* ctx, const rcg_matrix* a, const double* x, double* y) {
    if (a->n == 0) return;
    SpmvArgs s = make_args(a);
    s.x[0] = x;
    s.y[0] = y;
    KTimer t(ctx, 0);
    spmv_prepare_kernels();
    k_spmv<1><<<spmv_grid(ctx, a->n), kSpmvThreads, spmv_smem(a), ctx->stream>>>(s, a->cap);
    RCG_LAUNCHED(ctx);
}

void launch_spmv_dual(rcg_ctx* ctx, const rcg_matrix* a, const double* x1, const double* x2,
                      double* y1, double* y2) {
    if (a->n == 0) return;
    SpmvArgs s = make_args(a);
    s.x[0] = x1;
    s.x[1] = x2;
    s.y[0] = y1;
    s.y[1] = y2;
    KTimer t(ctx, 0);
    spmv_prepare_kernels();
    k_spmv<2><<<spmv_grid(ctx, a->n), kSpmvThreads, spmv_smem(a), ctx->stream>>>(s, a->cap);
    RCG_LAUNCHED(ctx);
}

void launch_residual(rcg_ctx* ctx, const rcg_matrix* a, const double* b, const double* x, double* r) {
    SpmvArgs s = make_args(a);
    s.x[0] = x;
    s.y[0] = r;
    const int g = spmv_grid(ctx, a->n);
    s.partials = ctx->ws.partials;
    spmv_prepare_kernels();
    k_residual<<<g, kSpmvThreads, spmv_smem(a), ctx->stream>>>(s, a->cap, b, ctx->ws.st);
    RCG_LAUNCHED(ctx);
}

void launch_spmm(rcg_ctx* ctx, const rcg_matrix* a, const double* x, int64_t ldx, double* y,
                 int64_t ldy, int k) {
    if (a->n == 0) return;
    for (int c0 = 0; c0 < k; c0 += 8) {
        const int kc = std::min(8, k - c0);
        k_spmm<8><<<spmv_grid(ctx, a->n), kSpmvThreads, 0, ctx->stream>>>(
            a->rs, a->ci, a->va, a->n, x + c0 * ldx, ldx, y + c0 * ldy, ldy, kc);
        RCG_LAUNCHED(ctx);
    }
}

void launch_fill(rcg_ctx* ctx, double* p, int64_t n, double v) {
    if (n <= 0) return;
    k_fill<<<stream_grid(ctx, n), kStreamThreads, 0, ctx->stream>>>(p, n, v);
    RCG_LAUNCHED(ctx);
}

void launch_fill_bits(rcg_ctx* ctx, double* p, int64_t n, unsigned long long bits) {
    if (n <= 0) return;
    k_fill_bits<<<stream_grid(ctx, n), kStreamThreads, 0, ctx->stream>>>(p, n, bits);
    RCG_LAUNCHED(ctx);
}

// Stage capacity of the pipelined SpMV: the widest 16-byte-aligned entry range of a 32-row tile
// (rounded to 32 entries, at most 1024; wider tiles take the direct path).
int tile_capacity(int32_t n, const int32_t* rs) {
    int32_t widest = 0;
    for (int32_t r0 = 0; r0 < n; r0 += 32) {
        const int32_t rend = std::min(r0 + 32, n);
        widest = std::max(widest, ((rs[rend] + 3) & ~3) - (rs[r0] & ~3));
    }
    return static_cast<int>(std::min<int64_t>(1024, std::max<int64_t>(32, round_up(widest, 32))));
}

// ------------------------------------------------------------------ host validation
// CsrMatrix::validate (src/csr_matrix.cpp:36-87): same checks and messages.
static void validate_csr(int32_t n, const int32_t* rs, const int32_t* ci, const double* va) {
    auto bad = [](const std::string& m) { throw Error(RCG_E_PARSE, m); };
    if (n < 0) bad("csr: negative dimension");
    if (rs[0] != 0) bad("csr: row_start[0] must be 0");
    for (int32_t i = 0; i < n; ++i) {
        if (rs[i] > rs[i + 1]) bad("csr: row_start not monotone at row " + std::to_string(i));
        bool diag = false;
        for (int32_t k = rs[i]; k < rs[i + 1]; ++k) {
            const int32_t c = ci[k];
            if (c < 0 || c >= n) bad("csr: column out of range in row " + std::to_string(i));
            if (k > rs[i] && ci[k - 1] >= c) bad("csr: columns not strictly increasing in row " + std::to_string(i));
            if (c == i) {
                diag = true;
                if (va[k] <= 0.0) bad("csr: non-positive diagonal at row " + std::to_string(i));
            }
        }
        if (!diag) bad("csr: missing diagonal at row " + std::to_string(i));
    }
    for (int32_t i = 0; i < n; ++i)
        for (int32_t k = rs[i]; k < rs[i + 1]; ++k) {
            const int32_t j = ci[k];
            if (j <= i) continue;
            const int32_t* b = ci + rs[j];
            const int32_t* e = ci + rs[j + 1];
            const int32_t* it = std::lower_bound(b, e, i);
            if (it == e || *it != i)
                bad("csr: entry (" + std::to_string(i) + "," + std::to_string(j) + ") has no transpose entry");
            const double v = va[k], w = va[it - ci];
            if (std::abs(v - w) > 1e-12 * std::max(std::abs(v), std::abs(w)))
                bad("csr: asymmetric value at (" + std::to_string(i) + "," + std::to_string(j) + ")");
        }
}

}  // namespace rcg

using namespace rcg;

extern "C" {

int rcg_matrix_create(rcg_ctx* ctx, int32_t n, const int32_t* row_start, const int32_t* col_idx,
                      const double* values, int validate, rcg_matrix** out) {
    return guard([&] {
        *out = nullptr;
        require(ctx != nullptr, "rcg_matrix_create: null context");
        if (n < 0) throw Error(RCG_E_PARSE, "csr: negative dimension");
        require(row_start != nullptr, "rcg_matrix_create: null row_start");
        const bool dev_in = is_device_ptr(row_start);
        std::vector<int32_t> h_rs;
        const int32_t* rs_host = row_start;
        if (dev_in) {
            h_rs.resize(static_cast<size_t>(n) + 1);
            RCG_CK(cudaMemcpy(h_rs.data(), row_start, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost));
            rs_host = h_rs.data();
        }
        const int64_t nnz = rs_host[n];
        if (rs_host[0] != 0) throw Error(RCG_E_PARSE, "csr: row_start[0] must be 0");
        if (validate && !dev_in) validate_csr(n, row_start, col_idx, values);
        auto* m = new rcg_matrix();
        try {
            m->n = n;
            m->nnz = nnz;
            void* p = nullptr;
            RCG_CK(cudaMalloc(&p, sizeof(int32_t) * (n + 1)));
            m->rs = static_cast<int32_t*>(p);
            // 8 zero padding entries: the pipelined SpMV widens tile ranges to 16-byte alignment
            RCG_CK(cudaMalloc(&p, sizeof(int32_t) * (nnz + kCsrPad)));
            m->ci = static_cast<int32_t*>(p);
            m->va = dev_alloc(nnz + kCsrPad);
            RCG_CK(cudaMemsetAsync(m->ci + nnz, 0, sizeof(int32_t) * kCsrPad, ctx->stream));
            RCG_CK(cudaMemsetAsync(m->va + nnz, 0, sizeof(double) * kCsrPad, ctx->stream));
            m->cap = tile_capacity(n, rs_host);
            const cudaMemcpyKind kind = dev_in ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
            RCG_CK(cudaMemcpyAsync(m->rs, row_start, sizeof(int32_t) * (n + 1), kind, ctx->stream));
            if (nnz > 0) {
                RCG_CK(cudaMemcpyAsync(m->ci, col_idx, sizeof(int32_t) * nnz, kind, ctx->stream));
                RCG_CK(cudaMemcpyAsync(m->va, values, sizeof(double) * nnz, kind, ctx->stream));
            }
            RCG_CK(cudaStreamSynchronize(ctx->stream));
        } catch (...) {
            rcg_matrix_destroy(m);
            throw;
        }
        *out = m;
    });
}

void rcg_matrix_destroy(rcg_matrix* a) {
    if (!a) return;
    dev_free(a->rs);
    dev_free(a->ci);
    dev_free(a->va);
    delete a;
}

int32_t rcg_matrix_n(const rcg_matrix* a) { return a ? a->n : 0; }
int64_t rcg_matrix_nnz(const rcg_matrix* a) { return a ? a->nnz : 0; }

int rcg_matrix_values(rcg_ctx* ctx, const rcg_matrix* a, double* values_out) {
    return guard([&] {
        RCG_CK(cudaMemcpyAsync(values_out, a->va, sizeof(double) * a->nnz, cudaMemcpyDefault, ctx->stream));
        RCG_CK(cudaStreamSynchronize(ctx->stream));
    });
}

int rcg_matrix_export(rcg_ctx* ctx, const rcg_matrix* a, int32_t* row_start, int32_t* col_idx, double* values) {
    return guard([&] {
        require(ctx && a, "rcg_matrix_export: null argument");
        if (row_start)
            RCG_CK(cudaMemcpyAsync(row_start, a->rs, sizeof(int32_t) * (a->n + 1), cudaMemcpyDefault, ctx->stream));
        if (col_idx && a->nnz)
            RCG_CK(cudaMemcpyAsync(col_idx, a->ci, sizeof(int32_t) * a->nnz, cudaMemcpyDefault, ctx->stream));
        if (values && a->nnz)
            RCG_CK(cudaMemcpyAsync(values, a->va, sizeof(double) * a->nnz, cudaMemcpyDefault, ctx->stream));
        RCG_CK(cudaStreamSynchronize(ctx->stream));
    });
}

int rcg_spmv(rcg_ctx* ctx, const rcg_matrix* a, const double* x, double* y) {
    return guard([&] {
        Staged xs, ys;
        stage_in(ctx, x, a->n, xs);
        stage_out_begin(ctx, y, a->n, ys);
        launch_spmv(ctx, a, xs.dev, ys.dev);
        stage_out_end(ctx, y, a->n, ys);
        RCG_CK(cudaStreamSynchronize(ctx->stream));
    });
}

int rcg_spmv_dual(rcg_ctx* ctx, const rcg_matrix* a, const double* x1, const double* x2,
                  double* y1, double* y2) {
    return guard([&] {
        Staged a1, a2, b1, b2;
        stage_in(ctx, x1, a->n, a1);
        stage_in(ctx, x2, a->n, a2);
        stage_out_begin(ctx, y1, a->n, b1);
        stage_out_begin(ctx, y2, a->n, b2);
        launch_spmv_dual(ctx, a, a1.dev, a2.dev, b1.dev, b2.dev);
        stage_out_end(ctx, y1, a->n, b1);
        stage_out_end(ctx, y2, a->n, b2);
        RCG_CK(cudaStreamSynchronize(ctx->stream));
    });
}

int rcg_diagonal_scale(rcg_ctx* ctx, const rcg_matrix* a, rcg_matrix** scaled, double* d_inv_sqrt) {
    return guard([&] {
        *scaled = nullptr;
        auto* m = new rcg_matrix();
        int* bad = nullptr;
        try {
            m->n = a->n;
            m->nnz = a->nnz;
            void* p = nullptr;
            RCG_CK(cudaMalloc(&p, sizeof(int32_t) * (a->n + 1)));
            m->rs = static_cast<int32_t*>(p);
            RCG_CK(cudaMalloc(&p, sizeof(int32_t) * (a->nnz + kCsrPad)));
            m->ci = static_cast<int32_t*>(p);
            m->va = dev_alloc(a->nnz + kCsrPad);
            RCG_CK(cudaMemsetAsync(m->ci + a->nnz, 0, sizeof(int32_t) * kCsrPad, ctx->stream));
            RCG_CK(cudaMemsetAsync(m->va + a->nnz, 0, sizeof(double) * kCsrPad, ctx->stream));
            m->cap = a->cap;
            RCG_CK(cudaMemcpyAsync(m->rs, a->rs, sizeof(int32_t) * (a->n + 1), cudaMemcpyDeviceToDevice, ctx->stream));
            if (a->nnz > 0)
                RCG_CK(cudaMemcpyAsync(m->ci, a->ci, sizeof(int32_t) * a->nnz, cudaMemcpyDeviceToDevice, ctx->stream));
            Staged dis;
            stage_out_begin(ctx, d_inv_sqrt, a->n, dis);
            RCG_CK(cudaMalloc(&p, sizeof(int)));
            bad = static_cast<int*>(p);
            const int big = 0x7fffffff;
            RCG_CK(cudaMemcpyAsync(bad, &big, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
            if (a->n > 0) {
                const int g = stream_grid(ctx, a->n);
                k_diag_inv_sqrt<<<g, kStreamThreads, 0, ctx->stream>>>(a->rs, a->ci, a->va, a->n, dis.dev, bad);
                RCG_LAUNCHED(ctx);
                k_diag_scale<<<g, kStreamThreads, 0, ctx->stream>>>(a->rs, a->ci, a->va, a->n, dis.dev, m->va);
                RCG_LAUNCHED(ctx);
            }
            int hbad = big;
            RCG_CK(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
            stage_out_end(ctx, d_inv_sqrt, a->n, dis);
            RCG_CK(cudaStreamSynchronize(ctx->stream));
            if (hbad != big)
                throw Error(RCG_E_PARSE, "diagonal_scale: non-positive diagonal at row " + std::to_string(hbad));
        } catch (...) {
            dev_free(bad);
            rcg_matrix_destroy(m);
            throw;
        }
        dev_free(bad);
        *scaled = m;
    });
}

}  // extern "C"
