// internal.cuh -- shared types, error plumbing and device helpers of librcg_b200.so.
//
// Layout in HBM:
//   CSR          int32 row_start[n+1], int32 col[nnz], f64 val[nnz]   (reference order)
//   IC sweeps    level-sorted copies of L and U rows: int32 perm[n], int32 prs[n+1],
//                int32 pcol[nnz_L], f64 pval[nnz_L] + f64 d[n]
//   vectors      f64[n], 256-byte aligned (cudaMalloc)
//   tall blocks  column-major, leading dimension ld = round_up(n, 32)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <deque>
#include <vector>

#include "rcg_b200.h"
#include "host_error.h"

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges for nsys / ncu --nvtx (no-ops otherwise)

namespace rcg {

// ------------------------------------------------------------------ errors (host_error.h)
[[noreturn]] void throw_cuda(cudaError_t e, const char* what, const char* file, int line);
#define RCG_CK(call)                                                              \
    do {                                                                          \
        cudaError_t e__ = (call);                                                 \
        if (e__ != cudaSuccess) ::rcg::throw_cuda(e__, #call, __FILE__, __LINE__); \
    } while (0)
#define RCG_LAUNCHED(ctx)                                                          \
    do {                                                                           \
        cudaError_t e__ = cudaGetLastError();                                      \
        if (e__ != cudaSuccess) ::rcg::throw_cuda(e__, "launch", __FILE__, __LINE__); \
        (ctx)->launches++;                                                         \
    } while (0)

// NVTX range over a scope (the hot-path phases: K1-K16 of SURVEY 8(a) as the C-ABI entry points,
// the sequence's solve 1 / recycling / accelerated phases)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// a C-ABI status from a nested entry point, rethrown with its message
inline void ck(int rc) {
    if (rc != RCG_OK) throw Error(rc, rcg_last_error());
}

// ------------------------------------------------------------------ constants
constexpr int kStreamThreads = 256;   // streaming / reduction kernels
constexpr int kSweepThreads = 128;    // rows per sweep tile
constexpr int kSpmvThreads = 256;     // 8 warps, one 32-row tile per warp at a time
constexpr int kSpmvChunk = 256;       // smem staging entries per warp
constexpr int kMaxRed = 160;          // max values reduced by one kernel (2*128 tall + scalars)
constexpr int kGroup = 64;            // sweep tiles per first-level reduction group
constexpr int kCsrPad = 8;            // zero entries after the CSR arrays (aligned bulk copies)
constexpr unsigned long long kSentinelBits = 0x7FF4DEADBEEF0001ULL;  // "not yet computed"

inline int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }
inline int64_t ld_of(int32_t n) { return round_up(n > 0 ? n : 1, 32); }

// ------------------------------------------------------------------ device solver state
// Everything a solve iteration needs is read from here, so kernels take no per-iteration
// parameters and one launch sequence (or one CUDA graph) serves every iteration.
enum : int { kRunning = 0, kConverged = 1, kCapped = 2, kBroken = 3, kZeroRhs = 4 };
enum : int {
    kBrkNone = 0,
    kBrkRz = 1,        // (r, z) <= 0
    kBrkPAp = 2,       // (p, A p) <= 0
    kBrkPower = 3,     // power vector vanished
};

struct DevState {
    int done;
    int iter;      // iteration being executed (1-based)
    int status;
    int max_iter;
    int iters;     // completed iterations (SolveReport::iterations)
    int pad1;
    double scal[4];  // misc device scalars (condest ||v0||^2, v^T A v)
    double eps, bnorm;
    double rho, rho_prev, beta, alpha, pq, rr, relres;
    // condest
    double vn;
    double quot[5];
    int nq;
    // sampler
    int smp_method;        // -1 none, 0 A, 1 B
    int smp_m;
    int smp_lmax;
    int smp_next;          // method B next 1-based slot
    long long smp_h;       // method A stride
    int smp_npending;      // slots to fill from the payload of iteration smp_pending_iter
    int smp_pending_iter;
    int smp_payload;       // 0 x, 1 r
    int pad0;
    // reduction tickets (one per kernel family; reset by their finalizer)
    unsigned int tick[8];
};

// workspace of one solve (grown on demand, owned by the context)
struct Workspace {
    int64_t cap_n = 0;
    int cap_k = 0;
    double *r = nullptr, *z = nullptr, *p = nullptr, *q = nullptr;
    double *ybuf = nullptr, *zs = nullptr;  // sweep buffers (sentinel protocol)
    double *v = nullptr, *vnext = nullptr;  // power iteration
    double *bw = nullptr, *xw = nullptr;    // staged b and x
    double *hist = nullptr, *alph = nullptr, *bet = nullptr;
    int64_t cap_iter = 0;
    double* u = nullptr;      // k coefficients (deflation / projections)
    double* u2 = nullptr;     // k coefficients (SC)
    double* partials = nullptr;  // reduction partials
    int64_t cap_partials = 0;
    double* gpart = nullptr;  // second-level partials (sweeps)
    unsigned int* gcount = nullptr;
    int64_t cap_groups = 0;
    int* tickets = nullptr;   // sweep tile tickets + exit counters (4 ints)
    DevState* st = nullptr;
    int* smp_pending = nullptr;   // pending slot list (device)
    int cap_pending = 0;
};

struct BatchWs;  // batch.cu

}  // namespace rcg

// ------------------------------------------------------------------ handle structs
constexpr int kStatClasses = 10;  // 0-4 single right-hand side, 5-9 batched (rcg_b200.h)

struct rcg_ctx {
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    int64_t launches = 0;
    rcg::Workspace ws;
    double* host_pinned = nullptr;   // small pinned scratch for scalar readbacks
    bool profiling = false;
    unsigned profile_mask = 0x3FFu;  // kernel classes timed while profiling (bit per class)
    double stat_ms[kStatClasses] = {};
    int64_t stat_n[kStatClasses] = {};
    int64_t stat_units[kStatClasses] = {};  // right-hand sides carried (batched: RT per launch)
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    struct TimedLaunch {
        int cls;
        int units;
        cudaEvent_t start, stop;
    };
    std::deque<TimedLaunch> ev_pending;
    std::vector<cudaEvent_t> ev_free;
    cudaEvent_t user_ev[16] = {};
    int sweep_bps = 0;          // resident sweep CTAs per SM; 0 = by DAG shape (RCG_SWEEP_BPS)
    int sweep_backoff_ns = 0;   // dependency-wait sleep between polls (RCG_SWEEP_BACKOFF_NS)
    int sweep_cluster = 2;      // IC sweep kernel: 0 grid-wide sync-free, 2 by shape, 4 one launch per level
    int spmv_bps = 2;           // SpMV CTAs per SM (RCG_SPMV_BPS): leaves room for concurrent solves
    rcg::BatchWs* bws = nullptr;   // multi-RHS workspaces (batch.cu): a compacted phase
    rcg::BatchWs* bws2 = nullptr;  // reads one and writes the other
};

struct rcg_matrix {
    int32_t n = 0;
    int64_t nnz = 0;
    int32_t* rs = nullptr;
    int32_t* ci = nullptr;
    double* va = nullptr;
    int cap = 256;  // pipelined SpMV stage capacity (entries)
    // natural-ordered cube stencil (7 / 27-point) detected from the pattern (batch.cu grid_info):
    // -1 not yet checked, 0 no, 7 / 27 yes with edge gN
    mutable int grid_st = -1;
    mutable int32_t gN = 0;
};

struct rcg_ic {
    int32_t n = 0;
    int64_t nnz_l = 0;
    double shift = 0.0;
    bool host_image = true;  // h_* below filled (device-built factors: on demand, ensure_host_image)
    // host image (IcFactor fields)
    std::vector<int32_t> h_bounds, h_lrs, h_lcol, h_urs, h_ucol;
    std::vector<double> h_lval, h_d, h_uval;
    // device schedules
    int32_t fwd_levels = 0, bwd_levels = 0;
    int32_t f_npos = 0, b_npos = 0;   // schedule lengths with each level padded to a warp multiple
    int32_t *f_perm = nullptr, *f_prs = nullptr, *f_col = nullptr;
    double* f_val = nullptr;
    int32_t *b_perm = nullptr, *b_prs = nullptr, *b_col = nullptr;
    double* b_val = nullptr;
    double* d = nullptr;
    // level starts of the padded schedules ([0] forward, [1] backward; nlev + 1 entries)
    std::vector<int32_t> h_lptr[2];
};

struct rcg_tall {
    int32_t n = 0;
    int k = 0;
    int64_t ld = 0;
    double* d = nullptr;
};

struct rcg_basis {
    int32_t n = 0;
    int k = 0;
    int64_t ld = 0;
    int who = 0;
    double* w = nullptr;
    double* aw = nullptr;
    double* l = nullptr;       // device k x k row-major Cholesky factor
    std::vector<double> h_l;   // host copy
};

struct rcg_sampler {
    int method = 0;
    int m = 0;
    int32_t n = 0;
    int64_t ld = 0;
    int l_max = 1;
    long long h = 1;
    int next_slot = 1;
    double alpha = 0.0;
    double* slots = nullptr;       // m x ld
    int* occupied = nullptr;       // device m
    int* stored_iter = nullptr;    // device m
    double* thresholds = nullptr;  // device m (method B)
    std::vector<double> h_thr;
};

namespace rcg {

// ------------------------------------------------------------------ host helpers (context.cu)
void ensure_workspace(rcg_ctx* ctx, int64_t n, int k, int64_t max_iter, int64_t partials,
                      int64_t groups, int pending);
bool is_device_ptr(const void* p);
// stage a host or device input of `count` doubles into device memory (returns device pointer)
struct Staged {
    double* dev = nullptr;
    bool owned = false;
    ~Staged();
};
void stage_in(rcg_ctx* ctx, const double* src, int64_t count, Staged& out);
void stage_out_begin(rcg_ctx* ctx, double* dst, int64_t count, Staged& tmp);
void stage_out_end(rcg_ctx* ctx, double* dst, int64_t count, Staged& tmp);
double* dev_alloc(int64_t count);
void* dev_alloc_bytes(size_t bytes);
void dev_free(void* p);  // cached: see context.cu
void register_ctx(rcg_ctx* c, bool add);

// kernel timing (bench roofline): brackets a launch with events when profiling is on
struct KTimer {
    rcg_ctx* ctx;
    int cls;
    int units;
    cudaEvent_t start = nullptr;
    KTimer(rcg_ctx* c, int k, int units = 1);
    ~KTimer();
};
void resolve_timers(rcg_ctx* ctx);

// host dense (host_dense.cpp)
bool chol_factor_host(int k, const std::vector<double>& s, std::vector<double>& l, int* bad_row);
void chol_solve_host(int k, const std::vector<double>& l, const double* f, double* u);
void sym_eig_host(int k, const std::vector<double>& s, std::vector<double>& values,
                  std::vector<double>& vectors);
void lanczos_extremes_host(int k, const double* alphas, const double* betas, double* lmin,
                           double* lmax);

// launch helpers implemented in kernels
void launch_fill(rcg_ctx* ctx, double* p, int64_t n, double v);
void launch_fill_bits(rcg_ctx* ctx, double* p, int64_t n, unsigned long long bits);
void launch_spmv(rcg_ctx* ctx, const rcg_matrix* a, const double* x, double* y);
void launch_spmv_dual(rcg_ctx* ctx, const rcg_matrix* a, const double* x1, const double* x2,
                      double* y1, double* y2);
void launch_spmm(rcg_ctx* ctx, const rcg_matrix* a, const double* x, int64_t ldx, double* y,
                 int64_t ldy, int k);
void ic_apply_dev(rcg_ctx* ctx, const rcg_ic* f, const double* r, double* z);
// sum_r a[:,i] * b[:,j] for i in [0,ka), j in [0,kb): out (host, ka x kb row-major)
void gram_host(rcg_ctx* ctx, const double* a, int64_t lda, int ka, const double* b, int64_t ldb,
               int kb, int32_t n, bool lower_only, std::vector<double>& out);
// y[:,c] = sum_j t[c*k + j] * e[:,j]  (c < kc), accumulated from 0.0 in j order
void combine_cols(rcg_ctx* ctx, const double* e, int64_t lde, int k, const double* t_host, int kc,
                  double* y, int64_t ldy, int32_t n);

}  // namespace rcg

// ------------------------------------------------------------------ device helpers
#ifdef __CUDACC__
namespace rcg {

__device__ __forceinline__ double ld_relaxed(const double* p) {
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(double* p, double v) {
    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ bool is_sentinel(double v) {
    return static_cast<unsigned long long>(__double_as_longlong(v)) == kSentinelBits;
}
__device__ __forceinline__ double sentinel() { return __longlong_as_double(static_cast<long long>(kSentinelBits)); }
// a computed value that happens to carry the sentinel pattern is published as a canonical NaN
__device__ __forceinline__ double publishable(double v) { return is_sentinel(v) ? __longlong_as_double(0x7FF8000000000000LL) : v; }

// reference arithmetic: separate roundings, never contracted (s -= a*b ; s += a*b)
__device__ __forceinline__ double fsub_mul(double s, double a, double b) { return __dsub_rn(s, __dmul_rn(a, b)); }
__device__ __forceinline__ double fadd_mul(double s, double a, double b) { return __dadd_rn(s, __dmul_rn(a, b)); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// block-wide sum of NV values per thread; result valid in thread 0 (acc[j]) -- fixed tree order
template <int NV>
__device__ __forceinline__ void block_sum(double (&acc)[NV], double* smem /* NV*32 */) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int j = 0; j < NV; ++j) acc[j] = warp_sum(acc[j]);
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int j = 0; j < NV; ++j) smem[j * 32 + wid] = acc[j];
    __syncthreads();
    if (wid == 0) {
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            double v = lane < nw ? smem[j * 32 + lane] : 0.0;
            acc[j] = warp_sum(v);
        }
    }
}

// Deterministic grid reduction: each block stores its NV partials at slot `slot`; the last
// block to arrive (ticket) sums slots 0..nslots-1 in a fixed order and returns true with the
// totals in `tot` (valid in all threads of that block).  The ticket is reset for reuse.
template <int NV>
__device__ bool grid_reduce(const double (&acc)[NV], double* partials, int slot, int nslots,
                            unsigned int* ticket, double* tot /* smem NV */, double* smem) {
    __shared__ bool s_last;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int j = 0; j < NV; ++j) partials[(int64_t)j * nslots + slot] = acc[j];
        __threadfence();
        const unsigned t = atomicAdd(ticket, 1u);
        s_last = (t == static_cast<unsigned>(nslots) - 1u);
    }
    __syncthreads();
    if (!s_last) return false;
    __threadfence();
    double a[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        double s = 0.0;
        for (int i = threadIdx.x; i < nslots; i += blockDim.x)
            s = __dadd_rn(s, __ldcg(partials + (int64_t)j * nslots + i));
        a[j] = s;
    }
    block_sum<NV>(a, smem);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int j = 0; j < NV; ++j) tot[j] = a[j];
        *ticket = 0u;
    }
    __syncthreads();
    return true;
}

}  // namespace rcg
#endif
