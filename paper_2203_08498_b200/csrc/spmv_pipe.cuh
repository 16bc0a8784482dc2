// spmv_pipe.cuh -- the CSR SpMV tile engine shared by k_spmv, k_residual and k_spmv_pq.
//
// Each warp walks 32-row tiles of a persistent grid.  A tile's CSR entries are contiguous
// (row_start[r0] .. row_start[r0+32]), so lane 0 brings the whole value and column range into
// the warp's shared-memory stage with two `cp.async.bulk` copies (TMA bulk engine, completion
// on an mbarrier), kPipeStages-deep: the copies of the next tiles are in flight while tile t is
// summed, and the row bounds of the tile after those are already being loaded (csr_tiles).
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

#ifndef RCG_PIPE_STAGES
#define RCG_PIPE_STAGES 2
#endif
constexpr int kPipeStages = RCG_PIPE_STAGES;  // bulk stages per warp (tiles in flight)
constexpr int kPipeHdr = (8 * kPipeStages + 15) & ~15;  // mbarriers, padded to 16 bytes

// per-warp shared memory: the mbarriers, then kPipeStages value stages and column stages
inline size_t pipe_smem_bytes(int cap) {
    return static_cast<size_t>(kPipeWarps) * (kPipeHdr + static_cast<size_t>(kPipeStages) * cap * 12);
}

// The tile engine.  Warp w of the persistent grid walks tiles t0, t0 + nw, ... (t0 = global warp
// index, nw = warps in the grid).  Software pipeline per warp:
//   * row bounds (rs[row], rs[row + 1] for the tile's 32 rows, one coalesced load) are loaded
//     kPipeStages tiles ahead, so the bulk issue never waits on them;
//   * the tile's CSR entries are brought in kPipeStages - 1 tiles ahead by two cp.async.bulk
//     copies into the warp's stage (completion on the stage's mbarrier);
//   * the current tile is handed to body(r0, b, e, vals, cols, off): this lane's row is r0 + lane
//     (valid when < n) with entries [b, e), entry k at vals[k - off] / cols[k - off].
// A tile wider than the stage capacity is handed over with the global arrays (off = 0); the two
// call sites are separate so the staged path reads shared memory with LDS, not generic loads.
template <class Body>
__device__ __forceinline__ void csr_tiles(const int32_t* __restrict__ rs, const int32_t* __restrict__ ci,
                                          const double* __restrict__ va, int32_t n, int cap, Body&& body) {
    constexpr int S = kPipeStages;
    extern __shared__ __align__(16) unsigned char pipe_smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned char* base = pipe_smem + static_cast<size_t>(wid) * (kPipeHdr + static_cast<size_t>(S) * cap * 12);
    uint64_t* bar = reinterpret_cast<uint64_t*>(base);
    double* sv = reinterpret_cast<double*>(base + kPipeHdr);                   // [S][cap]
    int32_t* sc = reinterpret_cast<int32_t*>(base + kPipeHdr + S * cap * 8);  // [S][cap]
    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < S; ++s) mbar_init(&bar[s]);
        fence_mbar_init();
    }
    __syncwarp();
    const int ntiles = (n + 31) / 32;
    const int nw = gridDim.x * kPipeWarps;
    const int t0 = blockIdx.x * kPipeWarps + wid;

    auto bounds = [&](int t, int32_t& b, int32_t& e) {
        if (t < ntiles) {
            const int32_t r = t * 32 + lane;
            b = __ldg(rs + min(r, n));
            e = __ldg(rs + min(r + 1, n));
        } else {
            b = e = 0;
        }
    };
    // warp-uniform (t < ntiles); false = the tile does not fit a stage
    auto issue = [&](int s, int32_t b, int32_t e) -> bool {
        const int32_t e0a = __shfl_sync(0xffffffffu, b, 0) & ~3;
        const int32_t e1a = (__shfl_sync(0xffffffffu, e, 31) + 3) & ~3;
        const int cnt = e1a - e0a;
        if (cnt > cap) return false;
        if (lane == 0) {
            fence_proxy_async();  // generic reads of this stage (its previous tile) precede the async write
            mbar_expect_tx(&bar[s], static_cast<unsigned>(cnt) * 12u);
            if (cnt > 0) {
                bulk_g2s(sv + s * cap, va + e0a, static_cast<unsigned>(cnt) * 8u, &bar[s]);
                bulk_g2s(sc + s * cap, ci + e0a, static_cast<unsigned>(cnt) * 4u, &bar[s]);
            }
        }
        return true;
    };

    int32_t qb[S + 1], qe[S + 1];  // row bounds of tiles k .. k + S
#pragma unroll
    for (int j = 0; j < S; ++j) bounds(t0 + j * nw, qb[j], qe[j]);
    unsigned staged = 0u, phase = 0u;
#pragma unroll
    for (int j = 0; j < S - 1; ++j)
        if (t0 + j * nw < ntiles && issue(j, qb[j], qe[j])) staged |= 1u << j;
    int s = 0;
    for (int t = t0; t < ntiles; t += nw) {
        bounds(t + S * nw, qb[S], qe[S]);
        const int sn = s == 0 ? S - 1 : s - 1;  // stage of tile k + S - 1 (freed by tile k - 1)
        if (t + (S - 1) * nw < ntiles) {
            if (issue(sn, qb[S - 1], qe[S - 1]))
                staged |= 1u << sn;
            else
                staged &= ~(1u << sn);
        }
        const int32_t r0 = t * 32;
        if ((staged >> s) & 1u) {
            while (!mbar_try_wait(&bar[s], (phase >> s) & 1u)) {
            }
            phase ^= 1u << s;
            body(r0, qb[0], qe[0], static_cast<const double*>(sv + s * cap),
                 static_cast<const int32_t*>(sc + s * cap), __shfl_sync(0xffffffffu, qb[0], 0) & ~3);
        } else {
            body(r0, qb[0], qe[0], va, ci, 0);
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < S; ++j) {
            qb[j] = qb[j + 1];
            qe[j] = qe[j + 1];
        }
        s = s + 1 == S ? 0 : s + 1;
    }
}

// Runs body(row, acc) for every row of the matrix (row < n guaranteed), acc[v] = (A x_v)_row.
template <int NV, class Body>
__device__ __forceinline__ void spmv_pipeline(const SpmvArgs& a, int cap, Body&& body) {
    csr_tiles(a.rs, a.ci, a.va, a.n, cap,
              [&](int32_t r0, int32_t my_b, int32_t my_e, const double* vsrc, const int32_t* csrc, int32_t off) {
                  const int32_t row = r0 + (threadIdx.x & 31);
                  double acc[NV];
#pragma unroll
                  for (int v = 0; v < NV; ++v) acc[v] = 0.0;
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
              });
}

}  // namespace rcg
