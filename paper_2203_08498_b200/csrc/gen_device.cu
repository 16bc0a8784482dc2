// gen_device.cu -- the 7-point generators (C1 Poisson, C2 / C4 high-contrast FV) built directly
// in HBM: C4's 938M entries (11.8 GB) need no host assembly and no H2D copy.
//
// Bitwise the host generator (generators.cpp): the inclusion origins come from the same seeded
// mt19937_64 placement on the host (fv7_inclusion_origins), and every row is assembled in the
// same entry order with the same arithmetic -- face coefficient (2 k_a) k_b / (k_a + k_b), a
// Dirichlet neighbour contributing k_cell, the diagonal summed over the six faces in order
// (unit coefficients give the Poisson matrix: off-diagonals -1, diagonal 6 exactly).
// Roofline: a write-bound streaming fill (12 nnz + 4 n bytes) plus the row-count scan.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "internal.cuh"
#include "kernels.cuh"

namespace rcg {

void fv7_inclusion_origins(int32_t N, int count, int size, uint64_t seed, std::vector<int>& ox, std::vector<int>& oy,
                           std::vector<int>& oz);  // generators.cpp

__global__ void k_gen_mark(uint8_t* __restrict__ inc, int32_t N, const int* __restrict__ org, int count, int size) {
    const int64_t cube = static_cast<int64_t>(size) * size * size;
    const int64_t total = cube * count;
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(t / cube);
        const int64_t r = t % cube;
        const int dx = static_cast<int>(r % size), dy = static_cast<int>((r / size) % size),
                  dz = static_cast<int>(r / (static_cast<int64_t>(size) * size));
        const int64_t x = org[3 * c] + dx, y = org[3 * c + 1] + dy, z = org[3 * c + 2] + dz;
        inc[x + static_cast<int64_t>(N) * (y + static_cast<int64_t>(N) * z)] = 1;
    }
}

__global__ void k_gen_counts(int32_t* __restrict__ cnt, int32_t N) {
    const int64_t n = static_cast<int64_t>(N) * N * N;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i <= n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (i == n) {
            cnt[i] = 0;
            continue;
        }
        const int x = static_cast<int>(i % N), y = static_cast<int>((i / N) % N), z = static_cast<int>(i / (int64_t(N) * N));
        cnt[i] = 1 + (z > 0) + (y > 0) + (x > 0) + (x < N - 1) + (y < N - 1) + (z < N - 1);
    }
}

__device__ __forceinline__ double face(double a, double b) {  // 2.0 * a * b / (a + b), host order
    return __ddiv_rn(__dmul_rn(__dmul_rn(2.0, a), b), __dadd_rn(a, b));
}

__global__ void k_gen_fill(const int32_t* __restrict__ rs, int32_t* __restrict__ ci, double* __restrict__ va,
                           const uint8_t* __restrict__ inc, int32_t N, double contrast) {
    const int64_t n = static_cast<int64_t>(N) * N * N;
    const int64_t sy = N, sz = static_cast<int64_t>(N) * N;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int x = static_cast<int>(i % N), y = static_cast<int>((i / N) % N), z = static_cast<int>(i / sz);
        auto K = [&](int64_t j) { return inc && inc[j] ? contrast : 1.0; };
        const double ki = K(i);
        const int64_t nb[6] = {z > 0 ? i - sz : -1, y > 0 ? i - sy : -1, x > 0 ? i - 1 : -1,
                               x < N - 1 ? i + 1 : -1, y < N - 1 ? i + sy : -1, z < N - 1 ? i + sz : -1};
        double off[6], diag = 0.0;
#pragma unroll
        for (int d = 0; d < 6; ++d) {
            off[d] = nb[d] >= 0 ? face(ki, K(nb[d])) : ki;
            diag = __dadd_rn(diag, off[d]);
        }
        int64_t e = rs[i];
#pragma unroll
        for (int d = 0; d < 3; ++d)
            if (nb[d] >= 0) {
                ci[e] = static_cast<int32_t>(nb[d]);
                va[e++] = -off[d];
            }
        ci[e] = static_cast<int32_t>(i);
        va[e++] = diag;
#pragma unroll
        for (int d = 3; d < 6; ++d)
            if (nb[d] >= 0) {
                ci[e] = static_cast<int32_t>(nb[d]);
                va[e++] = -off[d];
            }
    }
}

}  // namespace rcg

using namespace rcg;

extern "C" {

int rcg_matrix_generate(rcg_ctx* ctx, const rcg_gen_params* p, rcg_matrix** out) {
    int32_t* cnt = nullptr;
    int32_t* rs = nullptr;
    int32_t* ci = nullptr;
    double* va = nullptr;
    uint8_t* inc = nullptr;
    int* org = nullptr;
    void* tmp = nullptr;
    auto release = [&] {
        dev_free(cnt);
        dev_free(rs);
        dev_free(ci);
        dev_free(va);
        dev_free(inc);
        dev_free(org);
        dev_free(tmp);
    };
    const int rc = guard([&] {
        require(ctx && p && out, "rcg_matrix_generate: null argument");
        *out = nullptr;
        require(p->kind == RCG_GEN_POISSON7 || p->kind == RCG_GEN_FV7_CONTRAST,
                "rcg_matrix_generate: device generation covers the 7-point kinds (C1, C2, C4)");
        const int32_t N = p->grid;
        require(N >= 1, "generator: grid must be positive");
        const int64_t n = static_cast<int64_t>(N) * N * N;
        require(n < (1LL << 31), "generator: grid too large for int32 rows");
        const int64_t nnz = 7 * n - 6 * static_cast<int64_t>(N) * N;
        require(nnz < (1LL << 31), "generator: too many entries for int32 offsets");
        const int g = std::max<int>(1, static_cast<int>(std::min<int64_t>((n + 255) / 256, ctx->num_sms * 16)));
        if (p->kind == RCG_GEN_FV7_CONTRAST && p->inclusions > 0) {
            std::vector<int> ox, oy, oz;
            fv7_inclusion_origins(N, p->inclusions, p->inclusion_size, p->seed, ox, oy, oz);
            std::vector<int> h(3 * ox.size());
            for (size_t c = 0; c < ox.size(); ++c) {
                h[3 * c] = ox[c];
                h[3 * c + 1] = oy[c];
                h[3 * c + 2] = oz[c];
            }
            org = static_cast<int*>(dev_alloc_bytes(sizeof(int) * h.size()));
            inc = static_cast<uint8_t*>(dev_alloc_bytes(static_cast<size_t>(n)));
            RCG_CK(cudaMemcpyAsync(org, h.data(), sizeof(int) * h.size(), cudaMemcpyHostToDevice, ctx->stream));
            RCG_CK(cudaMemsetAsync(inc, 0, static_cast<size_t>(n), ctx->stream));
            k_gen_mark<<<g, 256, 0, ctx->stream>>>(inc, N, org, p->inclusions, p->inclusion_size);
            RCG_LAUNCHED(ctx);
        }
        const double contrast = p->kind == RCG_GEN_FV7_CONTRAST ? p->contrast : 1.0;
        cnt = static_cast<int32_t*>(dev_alloc_bytes(sizeof(int32_t) * (n + 1)));
        rs = static_cast<int32_t*>(dev_alloc_bytes(sizeof(int32_t) * (n + 1)));
        ci = static_cast<int32_t*>(dev_alloc_bytes(sizeof(int32_t) * std::max<int64_t>(nnz, 1)));
        va = dev_alloc(std::max<int64_t>(nnz, 1));
        k_gen_counts<<<g, 256, 0, ctx->stream>>>(cnt, N);
        RCG_LAUNCHED(ctx);
        size_t bytes = 0;
        RCG_CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt, rs, static_cast<int>(n + 1), ctx->stream));
        tmp = dev_alloc_bytes(std::max<size_t>(bytes, 1));
        RCG_CK(cub::DeviceScan::ExclusiveSum(tmp, bytes, cnt, rs, static_cast<int>(n + 1), ctx->stream));
        k_gen_fill<<<g, 256, 0, ctx->stream>>>(rs, ci, va, inc, N, contrast);
        RCG_LAUNCHED(ctx);
        RCG_CK(cudaStreamSynchronize(ctx->stream));
        // the standard device matrix (padding, stage capacity) from the device arrays
        const int rc2 = rcg_matrix_create(ctx, static_cast<int32_t>(n), rs, ci, va, 0, out);
        if (rc2 != RCG_OK) throw Error(rc2, rcg_last_error());
    });
    release();
    return rc;
}

}  // extern "C"
