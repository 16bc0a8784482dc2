// gen_device.cu -- every BASELINE.json matrix assembled directly in HBM: the
// 7-point kinds (C1 Poisson, C2 / C4 high-contrast FV; C4's 938M entries, 11.8 GB, need no host
// assembly and no H2D copy), C3's Q1 27-point stiffness (449M entries from the 17M element
// coefficients) and C5's kNN graph Laplacian (exact kNN search, symmetric union, weights).
//
// The seeded random streams stay on the host (mt19937_64 is sequential): C2 / C4's inclusion
// origins, C3's element coefficients (134 MB), C5's points (96 MB); everything O(nnz) runs here.
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

#include "gen_math.h"
#include "internal.cuh"
#include "kernels.cuh"

namespace rcg {

// generators.cpp (the seeded host streams; the O(nnz) assembly is here)
void fv7_inclusion_origins(int32_t N, int count, int size, uint64_t seed, std::vector<int>& ox, std::vector<int>& oy,
                           std::vector<int>& oz);
void q1_element_coefficients(int32_t N, double sigma, uint64_t seed, std::vector<double>& ke);
void knn_points(int32_t npts, uint64_t seed, std::vector<double>& P);
int knn_grid_size(int32_t npts);

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

__global__ void k_gen_fill_const(int32_t* __restrict__ v, int64_t n, int32_t c) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        v[i] = c;
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

// ---- C3: Q1 27-point rows (generators.cpp q1_27pt): entries in (dz, dy, dx) order, the shared
// element coefficients summed over ascending (ez, ey, ex), 1/3 on the diagonal, explicit zeros
// for edge neighbours, -1/12 for face / body diagonals.  One thread per row.
__device__ __forceinline__ int q1_cnt1(int c, int N) { return (c > 0) + 1 + (c < N - 1); }

__global__ void k_q1_counts(int32_t* __restrict__ cnt, int32_t N) {
    const int64_t n = static_cast<int64_t>(N) * N * N;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i <= n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (i == n) {
            cnt[i] = 0;
            continue;
        }
        const int x = static_cast<int>(i % N), y = static_cast<int>((i / N) % N), z = static_cast<int>(i / (int64_t(N) * N));
        cnt[i] = q1_cnt1(x, N) * q1_cnt1(y, N) * q1_cnt1(z, N);
    }
}

__global__ void k_q1_fill(const int32_t* __restrict__ rs, int32_t* __restrict__ ci, double* __restrict__ va,
                          const double* __restrict__ ke, int32_t N) {
    const int64_t n = static_cast<int64_t>(N) * N * N;
    const int64_t M = static_cast<int64_t>(N) + 1, sy = N, sz = static_cast<int64_t>(N) * N;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int x = static_cast<int>(i % N), y = static_cast<int>((i / N) % N), z = static_cast<int>(i / sz);
        int64_t p = rs[i];
        for (int dz = -1; dz <= 1; ++dz) {
            if (z + dz < 0 || z + dz >= N) continue;
            for (int dy = -1; dy <= 1; ++dy) {
                if (y + dy < 0 || y + dy >= N) continue;
                for (int dx = -1; dx <= 1; ++dx) {
                    if (x + dx < 0 || x + dx >= N) continue;
                    const int nd = (dx != 0) + (dy != 0) + (dz != 0);
                    const int exs = max(x, x + dx), exe = min(x, x + dx) + 1;
                    const int eys = max(y, y + dy), eye = min(y, y + dy) + 1;
                    const int ezs = max(z, z + dz), eze = min(z, z + dz) + 1;
                    double ksum = 0.0;
                    for (int ez = ezs; ez <= eze; ++ez)
                        for (int ey = eys; ey <= eye; ++ey)
                            for (int ex = exs; ex <= exe; ++ex) ksum = __dadd_rn(ksum, __ldg(ke + ex + M * (ey + M * ez)));
                    double v;
                    if (nd == 0) v = __ddiv_rn(ksum, 3.0);
                    else if (nd == 1) v = 0.0;
                    else v = __ddiv_rn(-ksum, 12.0);
                    ci[p] = static_cast<int32_t>(i + dx + sy * dy + sz * dz);
                    va[p] = v;
                    ++p;
                }
            }
        }
    }
}

// ---- C5: kNN graph Laplacian (generators.cpp knn_laplacian).  Exact kNN over the same bucket
// grid with the same shell expansion and stopping rule, so every point's neighbour list -- the k
// smallest (d^2, j) pairs of the same visited set, a strict total order -- equals the host's
// whatever order the candidates are visited in.
constexpr int kKnnMax = 32;

__device__ __forceinline__ int knn_cidx(double v, int G) { return min(G - 1, static_cast<int>(__dmul_rn(v, static_cast<double>(G)))); }

__device__ __forceinline__ double knn_d2(const double* __restrict__ P, int64_t i, int64_t j) {
    const double dx = __dsub_rn(P[3 * j], P[3 * i]), dy = __dsub_rn(P[3 * j + 1], P[3 * i + 1]),
                 dz = __dsub_rn(P[3 * j + 2], P[3 * i + 2]);
    return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

__global__ void k_knn_cell(const double* __restrict__ P, int32_t npts, int G, int32_t* __restrict__ cell,
                           int32_t* __restrict__ cnt) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < npts;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int c = knn_cidx(P[3 * i], G) + G * (knn_cidx(P[3 * i + 1], G) + G * knn_cidx(P[3 * i + 2], G));
        cell[i] = c;
        atomicAdd(cnt + c, 1);
    }
}

__global__ void k_iota(int32_t* __restrict__ v, int32_t n) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        v[i] = static_cast<int32_t>(i);
}

__global__ void k_knn_search(const double* __restrict__ P, int32_t npts, int k, int G, double cell_w,
                             const int32_t* __restrict__ cstart, const int32_t* __restrict__ order,
                             int32_t* __restrict__ nbr, double* __restrict__ nd2) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < npts;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double bd[kKnnMax];
        int32_t bj[kKnnMax];
        int cnt = 0;
        const int cx = knn_cidx(P[3 * i], G), cy = knn_cidx(P[3 * i + 1], G), cz = knn_cidx(P[3 * i + 2], G);
        for (int r = 0; r <= G; ++r) {
            for (int z = cz - r; z <= cz + r; ++z) {
                if (z < 0 || z >= G) continue;
                for (int y = cy - r; y <= cy + r; ++y) {
                    if (y < 0 || y >= G) continue;
                    for (int x = cx - r; x <= cx + r; ++x) {
                        if (x < 0 || x >= G) continue;
                        if (max(max(abs(x - cx), abs(y - cy)), abs(z - cz)) != r) continue;
                        const int c = x + G * (y + G * z);
                        for (int32_t q = cstart[c]; q < cstart[c + 1]; ++q) {
                            const int32_t j = order[q];
                            if (j == i) continue;
                            const double d2 = knn_d2(P, i, j);
                            if (cnt < k || d2 < bd[cnt - 1] || (d2 == bd[cnt - 1] && j < bj[cnt - 1])) {
                                int pos = cnt < k ? cnt++ : k - 1;
                                while (pos > 0 && (bd[pos - 1] > d2 || (bd[pos - 1] == d2 && bj[pos - 1] > j))) {
                                    bd[pos] = bd[pos - 1];
                                    bj[pos] = bj[pos - 1];
                                    --pos;
                                }
                                bd[pos] = d2;
                                bj[pos] = j;
                            }
                        }
                    }
                }
            }
            if (cnt == k) {
                const double reach = __dmul_rn(static_cast<double>(r), cell_w);
                if (bd[k - 1] <= __dmul_rn(reach, reach)) break;
            }
        }
        for (int t = 0; t < k; ++t) {
            nbr[i * k + t] = bj[t];
            nd2[i * k + t] = bd[t];
        }
    }
}

// gm::kSumChunk-term sequential chunk sums of f(v[t]) (sqrt or identity), one thread per chunk
template <bool Sqrt>
__global__ void k_chunk_sums(const double* __restrict__ v, int64_t n, double* __restrict__ part) {
    const int64_t chunks = (n + gm::kSumChunk - 1) / gm::kSumChunk;
    for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < chunks;
         c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double s = 0.0;
        const int64_t e = min(n, (c + 1) * gm::kSumChunk);
        for (int64_t t = c * gm::kSumChunk; t < e; ++t) s = __dadd_rn(s, Sqrt ? __dsqrt_rn(v[t]) : v[t]);
        part[c] = s;
    }
}

// total = sequential sum of the chunk sums; out = total / denom
__global__ void k_chunk_total(const double* __restrict__ part, int64_t chunks, double denom, double* __restrict__ out) {
    double s = 0.0;
    for (int64_t c = 0; c < chunks; ++c) s = __dadd_rn(s, part[c]);
    *out = __ddiv_rn(s, denom);
}

__global__ void k_knn_keys(const int32_t* __restrict__ nbr, int64_t edges, int k, unsigned long long* __restrict__ keys) {
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < edges;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const unsigned long long i = static_cast<unsigned long long>(e / k), j = static_cast<unsigned int>(nbr[e]);
        keys[2 * e] = (i << 32) | j;
        keys[2 * e + 1] = (j << 32) | i;
    }
}

__global__ void k_knn_rowlen(const unsigned long long* __restrict__ ukeys, const int64_t* __restrict__ nu,
                             int32_t* __restrict__ cnt) {
    for (int64_t u = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; u < *nu;
         u += static_cast<int64_t>(gridDim.x) * blockDim.x)
        atomicAdd(cnt + (ukeys[u] >> 32), 1);
}

// row i: its union neighbours ascending (ukeys[rs[i] - i ..]), the diagonal before the first
// j > i; w = exp(-d^2 / h^2), degree = sequential sum of w in column order
__global__ void k_knn_fill(const double* __restrict__ P, int32_t npts, const unsigned long long* __restrict__ ukeys,
                           const int32_t* __restrict__ rs, const double* __restrict__ hptr, int32_t* __restrict__ ci,
                           double* __restrict__ va, double* __restrict__ degree, int32_t* __restrict__ dpos) {
    const double h = *hptr;
    const double hh = __dmul_rn(h, h);
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < npts;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t u0 = rs[i] - i, len = static_cast<int64_t>(rs[i + 1]) - rs[i] - 1;
        int64_t p = rs[i];
        double deg = 0.0;
        bool diag_done = false;
        for (int64_t q = u0; q < u0 + len; ++q) {
            const int32_t j = static_cast<int32_t>(ukeys[q] & 0xffffffffULL);
            if (!diag_done && j > i) {
                dpos[i] = static_cast<int32_t>(p);
                ci[p++] = static_cast<int32_t>(i);
                diag_done = true;
            }
            const double w = gm::exp(__ddiv_rn(-knn_d2(P, i, j), hh));
            deg = __dadd_rn(deg, w);
            ci[p] = j;
            va[p++] = -w;
        }
        if (!diag_done) {
            dpos[i] = static_cast<int32_t>(p);
            ci[p] = static_cast<int32_t>(i);
        }
        degree[i] = deg;
    }
}

__global__ void k_knn_diag(const double* __restrict__ degree, const int32_t* __restrict__ dpos, int32_t npts,
                           const double* __restrict__ mdeg, double* __restrict__ va) {
    const double shift = __dmul_rn(1e-6, *mdeg);
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < npts;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        va[dpos[i]] = __dadd_rn(degree[i], shift);
}

}  // namespace rcg

using namespace rcg;

namespace {

// device buffers of one generator call, released together (stream-ordered dev_free)
struct Scratch {
    std::vector<void*> bufs;
    void* bytes(size_t b) {
        void* p = dev_alloc_bytes(std::max<size_t>(b, 1));
        bufs.push_back(p);
        return p;
    }
    template <class T>
    T* of(int64_t n) { return static_cast<T*>(bytes(sizeof(T) * static_cast<size_t>(std::max<int64_t>(n, 1)))); }
    ~Scratch() {
        for (void* p : bufs) dev_free(p);
    }
};

int grid_for(rcg_ctx* ctx, int64_t n) {
    return std::max<int>(1, static_cast<int>(std::min<int64_t>((n + 255) / 256, ctx->num_sms * 16)));
}

template <class T>
void exclusive_sum(rcg_ctx* ctx, Scratch& s, const T* in, T* out, int64_t n) {
    size_t bytes = 0;
    RCG_CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, static_cast<int>(n), ctx->stream));
    RCG_CK(cub::DeviceScan::ExclusiveSum(s.bytes(bytes), bytes, in, out, static_cast<int>(n), ctx->stream));
}

// the standard device matrix (padding, stage capacity) over arrays this call owns
void finish_matrix(rcg_ctx* ctx, int64_t n, int32_t* rs, int32_t* ci, double* va, rcg_matrix** out) {
    RCG_CK(cudaStreamSynchronize(ctx->stream));
    const int rc = rcg_matrix_create(ctx, static_cast<int32_t>(n), rs, ci, va, 0, out);
    if (rc != RCG_OK) throw Error(rc, rcg_last_error());
}

void generate_fv7(rcg_ctx* ctx, const rcg_gen_params* p, rcg_matrix** out) {
    Scratch s;
    const int32_t N = p->grid;
    require(N >= 1, "generator: grid must be positive");
    const int64_t n = static_cast<int64_t>(N) * N * N;
    require(n < (1LL << 31), "generator: grid too large for int32 rows");
    const int64_t nnz = 7 * n - 6 * static_cast<int64_t>(N) * N;
    require(nnz < (1LL << 31), "generator: too many entries for int32 offsets");
    const int g = grid_for(ctx, n);
    uint8_t* inc = nullptr;
    if (p->kind == RCG_GEN_FV7_CONTRAST && p->inclusions > 0) {
        std::vector<int> ox, oy, oz;
        fv7_inclusion_origins(N, p->inclusions, p->inclusion_size, p->seed, ox, oy, oz);
        std::vector<int> h(3 * ox.size());
        for (size_t c = 0; c < ox.size(); ++c) {
            h[3 * c] = ox[c];
            h[3 * c + 1] = oy[c];
            h[3 * c + 2] = oz[c];
        }
        int* org = s.of<int>(static_cast<int64_t>(h.size()));
        inc = s.of<uint8_t>(n);
        RCG_CK(cudaMemcpyAsync(org, h.data(), sizeof(int) * h.size(), cudaMemcpyHostToDevice, ctx->stream));
        RCG_CK(cudaMemsetAsync(inc, 0, static_cast<size_t>(n), ctx->stream));
        k_gen_mark<<<g, 256, 0, ctx->stream>>>(inc, N, org, p->inclusions, p->inclusion_size);
        RCG_LAUNCHED(ctx);
        RCG_CK(cudaStreamSynchronize(ctx->stream));  // h goes out of scope
    }
    const double contrast = p->kind == RCG_GEN_FV7_CONTRAST ? p->contrast : 1.0;
    int32_t* cnt = s.of<int32_t>(n + 1);
    int32_t* rs = s.of<int32_t>(n + 1);
    int32_t* ci = s.of<int32_t>(nnz);
    double* va = s.of<double>(nnz);
    k_gen_counts<<<g, 256, 0, ctx->stream>>>(cnt, N);
    RCG_LAUNCHED(ctx);
    exclusive_sum(ctx, s, cnt, rs, n + 1);
    k_gen_fill<<<g, 256, 0, ctx->stream>>>(rs, ci, va, inc, N, contrast);
    RCG_LAUNCHED(ctx);
    finish_matrix(ctx, n, rs, ci, va, out);
}

void generate_q1(rcg_ctx* ctx, const rcg_gen_params* p, rcg_matrix** out) {
    Scratch s;
    const int32_t N = p->grid;
    require(N >= 1, "generator: grid must be positive");
    const int64_t n = static_cast<int64_t>(N) * N * N;
    require(n < (1LL << 31), "generator: grid too large for int32 rows");
    const int64_t nnz = (3LL * N - 2) * (3LL * N - 2) * (3LL * N - 2);
    require(nnz < (1LL << 31), "generator: nnz exceeds int32 CSR offsets");
    std::vector<double> ke;
    q1_element_coefficients(N, p->sigma, p->seed, ke);
    double* dke = s.of<double>(static_cast<int64_t>(ke.size()));
    RCG_CK(cudaMemcpyAsync(dke, ke.data(), sizeof(double) * ke.size(), cudaMemcpyHostToDevice, ctx->stream));
    const int g = grid_for(ctx, n);
    int32_t* cnt = s.of<int32_t>(n + 1);
    int32_t* rs = s.of<int32_t>(n + 1);
    int32_t* ci = s.of<int32_t>(nnz);
    double* va = s.of<double>(nnz);
    k_q1_counts<<<g, 256, 0, ctx->stream>>>(cnt, N);
    RCG_LAUNCHED(ctx);
    exclusive_sum(ctx, s, cnt, rs, n + 1);
    k_q1_fill<<<g, 256, 0, ctx->stream>>>(rs, ci, va, dke, N);
    RCG_LAUNCHED(ctx);
    finish_matrix(ctx, n, rs, ci, va, out);  // synchronises before ke is released
}

void generate_knn(rcg_ctx* ctx, const rcg_gen_params* p, rcg_matrix** out) {
    Scratch s;
    const int32_t npts = p->grid;
    const int k = p->knn_k;
    require(npts > k && k >= 1, "generator: kNN needs more points than neighbours");
    require(k <= kKnnMax, "rcg_matrix_generate: kNN on the device supports k <= 32");
    std::vector<double> P;
    knn_points(npts, p->seed, P);
    const int G = knn_grid_size(npts);
    const int64_t cells = static_cast<int64_t>(G) * G * G;
    const double cell_w = 1.0 / G;
    double* dP = s.of<double>(static_cast<int64_t>(P.size()));
    RCG_CK(cudaMemcpyAsync(dP, P.data(), sizeof(double) * P.size(), cudaMemcpyHostToDevice, ctx->stream));
    const int g = grid_for(ctx, npts);
    // bucket grid: cell of every point, cell starts, points sorted by (cell, index)
    int32_t* cell = s.of<int32_t>(npts);
    int32_t* ccnt = s.of<int32_t>(cells + 1);
    int32_t* cstart = s.of<int32_t>(cells + 1);
    int32_t* idx = s.of<int32_t>(npts);
    int32_t* cell_sorted = s.of<int32_t>(npts);
    int32_t* order = s.of<int32_t>(npts);
    RCG_CK(cudaMemsetAsync(ccnt, 0, sizeof(int32_t) * (cells + 1), ctx->stream));
    k_knn_cell<<<g, 256, 0, ctx->stream>>>(dP, npts, G, cell, ccnt);
    RCG_LAUNCHED(ctx);
    exclusive_sum(ctx, s, ccnt, cstart, cells + 1);
    k_iota<<<g, 256, 0, ctx->stream>>>(idx, npts);
    RCG_LAUNCHED(ctx);
    {
        size_t bytes = 0;
        RCG_CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, cell, cell_sorted, idx, order, npts, 0, 32, ctx->stream));
        RCG_CK(cub::DeviceRadixSort::SortPairs(s.bytes(bytes), bytes, cell, cell_sorted, idx, order, npts, 0, 32,
                                               ctx->stream));
    }
    // exact kNN per point
    const int64_t edges = static_cast<int64_t>(npts) * k;
    int32_t* nbr = s.of<int32_t>(edges);
    double* nd2 = s.of<double>(edges);
    k_knn_search<<<g, 128, 0, ctx->stream>>>(dP, npts, k, G, cell_w, cstart, order, nbr, nd2);
    RCG_LAUNCHED(ctx);
    // h = mean kNN distance (gm chunk order)
    const int64_t ech = (edges + gm::kSumChunk - 1) / gm::kSumChunk;
    double* part = s.of<double>(std::max<int64_t>(ech, (npts + gm::kSumChunk - 1) / gm::kSumChunk));
    double* hd = s.of<double>(2);
    k_chunk_sums<true><<<grid_for(ctx, ech), 256, 0, ctx->stream>>>(nd2, edges, part);
    RCG_LAUNCHED(ctx);
    k_chunk_total<<<1, 1, 0, ctx->stream>>>(part, ech, static_cast<double>(edges), hd);
    RCG_LAUNCHED(ctx);
    // symmetric union: (i, j) and (j, i) for every directed pair, sorted, deduplicated
    unsigned long long* keys = s.of<unsigned long long>(2 * edges);
    unsigned long long* skeys = s.of<unsigned long long>(2 * edges);
    int64_t* nu = s.of<int64_t>(1);
    k_knn_keys<<<grid_for(ctx, edges), 256, 0, ctx->stream>>>(nbr, edges, k, keys);
    RCG_LAUNCHED(ctx);
    int hi_bits = 1;
    while ((1LL << hi_bits) < npts) ++hi_bits;
    {
        size_t bytes = 0;
        RCG_CK(cub::DeviceRadixSort::SortKeys(nullptr, bytes, keys, skeys, 2 * edges, 0, 32 + hi_bits, ctx->stream));
        RCG_CK(cub::DeviceRadixSort::SortKeys(s.bytes(bytes), bytes, keys, skeys, 2 * edges, 0, 32 + hi_bits,
                                              ctx->stream));
        bytes = 0;
        RCG_CK(cub::DeviceSelect::Unique(nullptr, bytes, skeys, keys, nu, 2 * edges, ctx->stream));
        RCG_CK(cub::DeviceSelect::Unique(s.bytes(bytes), bytes, skeys, keys, nu, 2 * edges, ctx->stream));
    }
    int64_t n_union = 0;
    RCG_CK(cudaMemcpyAsync(&n_union, nu, sizeof n_union, cudaMemcpyDeviceToHost, ctx->stream));
    RCG_CK(cudaStreamSynchronize(ctx->stream));
    const int64_t nnz = n_union + npts;
    require(nnz < (1LL << 31), "generator: nnz exceeds int32 CSR offsets");
    // rows: union length + 1 (the diagonal)
    int32_t* cnt = s.of<int32_t>(static_cast<int64_t>(npts) + 1);
    int32_t* rs = s.of<int32_t>(static_cast<int64_t>(npts) + 1);
    int32_t* ci = s.of<int32_t>(nnz);
    double* va = s.of<double>(nnz);
    double* degree = s.of<double>(npts);
    int32_t* dpos = s.of<int32_t>(npts);
    k_gen_fill_const<<<g, 256, 0, ctx->stream>>>(cnt, static_cast<int64_t>(npts) + 1, 1);
    RCG_LAUNCHED(ctx);
    k_knn_rowlen<<<grid_for(ctx, n_union), 256, 0, ctx->stream>>>(keys, nu, cnt);
    RCG_LAUNCHED(ctx);
    exclusive_sum(ctx, s, cnt, rs, static_cast<int64_t>(npts) + 1);
    k_knn_fill<<<g, 128, 0, ctx->stream>>>(dP, npts, keys, rs, hd, ci, va, degree, dpos);
    RCG_LAUNCHED(ctx);
    const int64_t dch = (npts + gm::kSumChunk - 1) / gm::kSumChunk;
    k_chunk_sums<false><<<grid_for(ctx, dch), 256, 0, ctx->stream>>>(degree, npts, part);
    RCG_LAUNCHED(ctx);
    k_chunk_total<<<1, 1, 0, ctx->stream>>>(part, dch, static_cast<double>(npts), hd + 1);
    RCG_LAUNCHED(ctx);
    k_knn_diag<<<g, 256, 0, ctx->stream>>>(degree, dpos, npts, hd + 1, va);
    RCG_LAUNCHED(ctx);
    finish_matrix(ctx, npts, rs, ci, va, out);
}

}  // namespace

extern "C" {

int rcg_matrix_generate(rcg_ctx* ctx, const rcg_gen_params* p, rcg_matrix** out) {
    return guard([&] {
        require(ctx && p && out, "rcg_matrix_generate: null argument");
        *out = nullptr;
        switch (p->kind) {
            case RCG_GEN_POISSON7:
            case RCG_GEN_FV7_CONTRAST:
                generate_fv7(ctx, p, out);
                break;
            case RCG_GEN_Q1_27PT:
                generate_q1(ctx, p, out);
                break;
            case RCG_GEN_KNN:
                generate_knn(ctx, p, out);
                break;
            default:
                throw Error(RCG_E_INVALID, "generator: unknown kind");
        }
    });
}

}  // extern "C"
