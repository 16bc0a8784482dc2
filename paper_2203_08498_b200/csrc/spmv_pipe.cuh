// spmv_pipe.cuh -- the CSR SpMV tile engine shared by k_spmv, k_residual and k_spmv_pq.
//
// Each warp walks 32-row tiles of a persistent grid.  A tile's CSR entries are contiguous
// (row_start[r0] .. row_start[r0+32]), so lane 0 brings the whole value and column range into
// the warp's shared-memory stage with two `cp.async.bulk` copies (TMA bulk engine, completion
// on an mbarrier), double-buffered: the copy of tile t+1 is in flight while tile t is summed.
// Ranges are widened to 16-byte alignment (multiples of 4 entries; the CSR arrays carry 8
// padding entries so the widened range never leaves the allocation).  Tiles wider than the
// stage capacity fall back to direct global loads for that tile only.
// Each lane sums ONE row sequentially from 0.0 in stored order with separate multiply/add
// roundings (src/csr_matrix.cpp:95-99) -- bitwise equal to the reference -- issuing its x
// gathers eight at a time so their L2 latency overlaps.
#pragma once

#include "internal.cuh"
#include "kernels.cuh"

namespace rcg {

constexpr int kPipeWarps = 8;  // warps per CTA

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

void allow_smem(const void* kernel);  // opt-in dynamic shared memory (spmv.cu)

// per-warp shared memory: 2 mbarriers, 2 value stages, 2 column stages
inline size_t pipe_smem_bytes(int cap) { return static_cast<size_t>(kPipeWarps) * (16 + 2 * cap * 12); }

// Runs body(row, acc) for every row of the matrix (row < n guaranteed), acc[v] = (A x_v)_row.
template <int NV, class Body>
__device__ __forceinline__ void spmv_pipeline(const SpmvArgs& a, int cap, Body&& body) {
    extern __shared__ __align__(16) unsigned char pipe_smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned char* base = pipe_smem + static_cast<size_t>(wid) * (16 + 2 * cap * 12);
    uint64_t* bar = reinterpret_cast<uint64_t*>(base);
    double* sv = reinterpret_cast<double*>(base + 16);  // [2][cap]
    int32_t* sc = reinterpret_cast<int32_t*>(base + 16 + 2 * cap * 8);  // [2][cap]
    if (lane == 0) {
        mbar_init(&bar[0]);
        mbar_init(&bar[1]);
        fence_mbar_init();
    }
    __syncwarp();
    const int ntiles = (a.n + 31) / 32;
    const int nw = gridDim.x * kPipeWarps;
    unsigned phase[2] = {0u, 0u};

    auto issue = [&](int t, int stg) -> bool {
        const int32_t r0 = t * 32, rend = min(r0 + 32, a.n);
        const int32_t e0a = __ldg(a.rs + r0) & ~3;
        const int32_t e1a = (__ldg(a.rs + rend) + 3) & ~3;
        const int cnt = e1a - e0a;
        if (cnt > cap) return false;
        if (lane == 0) {
            fence_proxy_async();  // generic reads of this stage (previous use) precede the async write
            mbar_expect_tx(&bar[stg], static_cast<unsigned>(cnt) * 12u);
            if (cnt > 0) {
                bulk_g2s(sv + stg * cap, a.va + e0a, static_cast<unsigned>(cnt) * 8u, &bar[stg]);
                bulk_g2s(sc + stg * cap, a.ci + e0a, static_cast<unsigned>(cnt) * 4u, &bar[stg]);
            }
        }
        return true;
    };

    int t = blockIdx.x * kPipeWarps + wid;
    int stg = 0;
    bool bulk_cur = t < ntiles ? issue(t, 0) : false;
    for (; t < ntiles; t += nw) {
        const int tn = t + nw;
        const bool bulk_next = tn < ntiles ? issue(tn, stg ^ 1) : false;
        const int32_t r0 = t * 32, row = r0 + lane, rend = min(r0 + 32, a.n);
        const int32_t e1 = __ldg(a.rs + rend);
        const int32_t my_b = row < a.n ? __ldg(a.rs + row) : e1;
        const int32_t my_e = row < a.n ? __ldg(a.rs + row + 1) : e1;
        double acc[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) acc[v] = 0.0;
        const double* vsrc;
        const int32_t* csrc;
        int32_t off;
        if (bulk_cur) {
            while (!mbar_try_wait(&bar[stg], phase[stg])) {
            }
            phase[stg] ^= 1u;
            vsrc = sv + stg * cap;
            csrc = sc + stg * cap;
            off = __ldg(a.rs + r0) & ~3;
        } else {
            vsrc = a.va;
            csrc = a.ci;
            off = 0;
        }
        for (int32_t e = my_b; e < my_e; e += 8) {
            const int m = min(8, my_e - e);
            double av[8], xv[NV][8];
            int32_t cc[8];
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (k < m) {
                    av[k] = vsrc[e - off + k];
                    cc[k] = csrc[e - off + k];
                }
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (k < m)
#pragma unroll
                    for (int v = 0; v < NV; ++v) xv[v][k] = __ldg(a.x[v] + cc[k]);
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (k < m)
#pragma unroll
                    for (int v = 0; v < NV; ++v) acc[v] = fadd_mul(acc[v], av[k], xv[v][k]);
        }
        if (row < a.n) body(row, acc);
        __syncwarp();
        stg ^= 1;
        bulk_cur = bulk_next;
    }
}

}  // namespace rcg
