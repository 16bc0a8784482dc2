// Dev microbenchmark: one-way latency of publishing a 64-bit value from one SM and observing it
// on another with the sweep's protocol (st.relaxed.gpu / ld.relaxed.gpu polling), vs volatile.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pingpong tools/pingpong.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ long long ld_rel(const long long* p) {
    long long v;
    asm volatile("ld.relaxed.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_rel(long long* p, long long v) {
    asm volatile("st.relaxed.gpu.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// block 0 and block 1 (forced onto different SMs by grid size) bounce a counter
__global__ void pingpong(long long* a, long long* b, int iters, long long* cycles, int mode) {
    if (threadIdx.x != 0) return;
    long long t0 = clock64();
    if (blockIdx.x == 0) {
        for (int i = 0; i < iters; ++i) {
            if (mode == 0) st_rel(a, 2 * i + 1); else *(volatile long long*)a = 2 * i + 1;
            if (mode == 0) { while (ld_rel(b) != 2 * i + 1) {} } else { while (*(volatile long long*)b != 2 * i + 1) {} }
        }
        cycles[0] = clock64() - t0;
    } else if (blockIdx.x == gridDim.x - 1) {
        for (int i = 0; i < iters; ++i) {
            if (mode == 0) { while (ld_rel(a) != 2 * i + 1) {} } else { while (*(volatile long long*)a != 2 * i + 1) {} }
            if (mode == 0) st_rel(b, 2 * i + 1); else *(volatile long long*)b = 2 * i + 1;
        }
    }
}

int main() {
    long long *a, *b, *c;
    cudaMalloc(&a, 4096);
    cudaMalloc(&b, 4096);
    cudaMalloc(&c, 64);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    for (int mode = 0; mode < 2; ++mode)
        for (int grid : {2, sms}) {
            cudaMemset(a, 0xff, 4096);
            cudaMemset(b, 0xff, 4096);
            const int iters = 20000;
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            pingpong<<<grid, 32>>>(a, b + 256, iters, c, mode);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            long long cyc;
            cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
            printf("{\"mode\": \"%s\", \"grid\": %d, \"one_way_ns\": %.1f, \"one_way_cycles\": %.1f, \"err\": \"%s\"}\n",
                   mode ? "volatile" : "relaxed.gpu", grid, ms * 1e6 / (2.0 * iters), cyc / (2.0 * iters),
                   cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
