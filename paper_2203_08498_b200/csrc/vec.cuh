// vec.cuh -- device helpers for reductions with a runtime number of values and the small
// Cholesky solve done by one warp inside a reduction finaliser.
#pragma once

#include "internal.cuh"

#ifdef __CUDACC__
namespace rcg {

// Every block writes nv partials at slot blockIdx.x (layout [j][slot]); the last block to
// arrive sums each value over slots 0..nslots-1 (one warp per value, lane-strided then
// butterfly -- a fixed order) into tot[0..nv).  Returns true in that block.
__device__ __forceinline__ bool grid_reduce_dyn(const double* blockvals /* smem nv */, int nv,
                                                double* partials, unsigned int* ticket,
                                                double* tot /* smem nv */) {
    __shared__ bool s_last;
    const int nslots = gridDim.x;
    for (int j = threadIdx.x; j < nv; j += blockDim.x)
        partials[static_cast<int64_t>(j) * nslots + blockIdx.x] = blockvals[j];
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1u) == static_cast<unsigned>(nslots) - 1u;
    __syncthreads();
    if (!s_last) return false;
    __threadfence();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int j = wid; j < nv; j += nw) {
        double s = 0.0;
        for (int i = lane; i < nslots; i += 32) s = __dadd_rn(s, __ldcg(partials + static_cast<int64_t>(j) * nslots + i));
        s = warp_sum(s);
        if (lane == 0) tot[j] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) *ticket = 0u;
    return true;
}

// Block-level sum of per-thread arrays acc[0..nv) (nv <= KC) into out[0..nv) (smem).
template <int KC>
__device__ __forceinline__ void block_sum_dyn(double (&acc)[KC], int nv, double* scratch /* 32*KC */,
                                              double* out) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int j = 0; j < KC; ++j)
        if (j < nv) {
            const double s = warp_sum(acc[j]);
            if (lane == 0) scratch[j * 32 + wid] = s;
        }
    __syncthreads();
    for (int j = wid; j < nv; j += nw) {
        double v = lane < nw ? scratch[j * 32 + lane] : 0.0;
        v = warp_sum(v);
        if (lane == 0) out[j] = v;
    }
    __syncthreads();
}

// u = (L L^T)^-1 f by warp 0 (k <= 128, L row-major k x k in global memory).  Column-oriented
// substitution; lane i accumulates its row's terms in ascending j, like dense.cpp:175-179.
__device__ __forceinline__ void warp_chol_solve(const double* L, int k, const double* f, double* u,
                                                double* s /* smem >= k */) {
    const int lane = threadIdx.x & 31;
    for (int i = lane; i < k; i += 32) s[i] = f[i];
    __syncwarp();
    for (int j = 0; j < k; ++j) {
        const double yj = __ddiv_rn(s[j], L[j * k + j]);
        __syncwarp();
        if (lane == 0) s[j] = yj;
        for (int i = j + 1 + lane; i < k; i += 32) s[i] = fsub_mul(s[i], L[i * k + j], yj);
        __syncwarp();
    }
    for (int j = k - 1; j >= 0; --j) {
        const double uj = __ddiv_rn(s[j], L[j * k + j]);
        __syncwarp();
        if (lane == 0) {
            s[j] = uj;
            u[j] = uj;
        }
        for (int i = lane; i < j; i += 32) s[i] = fsub_mul(s[i], L[j * k + i], uj);
        __syncwarp();
    }
}

}  // namespace rcg
#endif
