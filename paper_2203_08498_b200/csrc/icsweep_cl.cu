// icsweep_cl.cu -- IC(0) sweeps as ONE thread-block cluster, level-synchronous: an OPT-IN
// alternative to the grid-wide sync-free sweep (icsweep.cu) for factors with narrow levels
// (rcg_ctx_set_sweep_kernel(ctx, 1) / RCG_SWEEP_CLUSTER=1).  Bitwise identical results.
//
// Idea.  On C1/C2 the sweep is bound by the DAG depth (94 / 382 dependent levels of 349 / 5,490
// rows), not by bandwidth: the grid sweep pays an L2 publish -> poll round trip per level plus
// the worst of each row's parents (~1.0-1.3 us per level).  Here the sweep runs on one cluster
// of 16 CTAs (one per SM) stepping through the levels with the hardware cluster barrier; a row
// reads its parents (all within the last W <= 4 levels, checked by the plan) from the producing
// CTA's shared memory (DSMEM ring) instead of L2.  Warp-specialised: 24 compute warps (one row
// slot per thread) and 4 producer warps that stage each level ahead -- TMA bulk copies of the
// level's contiguous schedule ranges (perm, ELL codes, values; mbarrier complete_tx) and
// cp.async gathers of the inputs (r or y, d, r for (r, z); cp.async.mbarrier.arrive).
//
// Measured (B200): C1 0.70-1.1 us per level, C2 1.25 (fwd) / 2.5 (bwd) us
// per level against the grid sweep's 0.96 / 1.26 -- no faster.  Phase counters
// (RCG_CL_PROF=1) show each level's compute phase at ~1,100-1,900 cycles even with all parents
// local: the per-level instruction stream of 28 warps on one SM, the barrier and the staging
// cost as much as the L2 round trips they replace.  Kept as a tested, documented opt-in.
//
// Operator identity.  Row arithmetic is the reference loop exactly
// (src/ic_preconditioner.cpp:130-143; forward s = r_i, s -= l_ik y_k in stored entry order;
// backward s = y_i / d_i, s -= u_ik z_k), and every row reads final parent values, so the
// output is bitwise the grid sweep's and the reference ic_apply.  The (r, z) partials are
// formed per 32-position tile and summed in the grid sweep's fixed order (tile -> group of
// kGroup tiles -> total), so rho is bitwise the grid sweep's too: the choice of kernel never
// changes an iterate (tests/test_gpu_sweep_cluster.py).
//
// Layout (built once per factor and direction, on the device): the level-padded schedule of
// icsweep.cu plus an ELL copy of its entries, E (<= 4) per position: int32 code = owning CTA
// << 24 | DSMEM ring offset of the parent, f64 value; -1 pads.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "internal.cuh"
#include "kernels.cuh"
#include "spmv_pipe.cuh"

namespace rcg {

constexpr int kClCompute = 768;    // compute threads per CTA (24 warps): one slot each
constexpr int kClProducer = 128;   // producer threads per CTA (4 warps): TMA + gathers
constexpr int kClThreads = kClCompute + kClProducer;
constexpr int kClMaxR = 2;         // slots per compute thread per level (smax <= 1536)
constexpr int kClE = 4;            // max entries per row (7-point: 3)
constexpr int kClMaxW = 4;         // DSMEM value ring depth (levels)
constexpr int kClMaxNA = 8;        // stage-A ring depth

// optional per-phase cycle counters (RCG_CL_PROF=1): [CTA][phase], summed over levels by thread 0
__device__ unsigned long long g_cl_prof[16][16];

struct ClusterPlan {
    bool ok = false;
    int C = 0, W = 1, E = 1, DB = 1, LA = 1, R = 1, smax = 0, nlev = 0;
    size_t smem = 0;
    int32_t* lptr = nullptr;   // device, nlev + 1
    int32_t* code = nullptr;   // device, npos x E
    double* val = nullptr;     // device, npos x E
};

struct ClArgs {
    const int32_t* lptr;
    const int32_t* perm;
    const int32_t* code;
    const double* val;
    const double* in;
    const double* d;       // backward
    const double* r;       // backward: (r, z) partials when non-null
    double* out;
    double* partials;      // per 32-position tile
    double* gpart;         // per group of kGroup tiles
    DevState* st;
    int add_sc;
    int nlev, npos, W, E, DB, LA, smax;
    // shared-memory carve (bytes from the dynamic base): mbarriers, per-level slices of this CTA,
    // stage-A ring (per level: perm smax, codes smax x E, values smax x E -- TMA bulk copies),
    // stage-B ring (per level: gathered in / d / r, smax each -- cp.async), DSMEM value ring
    int off_sl, off_a, off_b, off_v;
    int a_stage, b_stage;   // bytes per level
    int prof;
};

__device__ __forceinline__ void cp_async8(unsigned dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_db(int db) {   // leave db - 1 groups in flight
    if (db >= 3) asm volatile("cp.async.wait_group 2;" ::: "memory");
    else if (db == 2) asm volatile("cp.async.wait_group 1;" ::: "memory");
    else asm volatile("cp.async.wait_group 0;" ::: "memory");
}
// Not volatile and no memory clobber, so the compiler can issue all of a thread's parent loads
// back to back: the address depends on a code read from shared memory after the cluster
// barrier, which keeps the load below the barrier.
__device__ __forceinline__ double ld_dsmem(unsigned local_addr, unsigned rank) {
    unsigned remote;
    asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local_addr), "r"(rank));
    double v;
    asm("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(remote));
    return v;
}
__device__ __forceinline__ void cluster_arrive() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
// arrive without a release fence: the level's DSMEM values are drained to shared memory by the
// preceding CTA barrier (BAR.SYNC completes pending STS), and nothing else crosses CTAs through
// this barrier (every parent is in the DSMEM ring) -- a .release arrive compiles to
// MEMBAR.ALL.GPU, which also waits for the in-flight prefetches
__device__ __forceinline__ void cluster_arrive_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {   // arrive once this thread's copies land
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_init_count(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}
__device__ __forceinline__ void compute_bar() {   // the compute warps only (named barrier 1)
    asm volatile("bar.sync 1, %0;" ::"n"(kClCompute) : "memory");
}

// Warp-specialised: kClCompute threads (one slot each, R slots when a CTA's share of a level is
// wider) compute the rows; kClProducer threads stage the inputs ahead -- one issues the TMA bulk
// copies of stage A (schedule ranges, mbarrier complete_tx), all gather stage B (cp.async,
// completion signalled per thread with cp.async.mbarrier.arrive) -- so no prefetch work or
// copy-engine wait sits on the compute warps' level chain.
template <bool BWD, int R>
__global__ void __launch_bounds__(kClThreads, 1) k_sweep_cl(ClArgs a) {
    if (a.st->done) return;  // uniform over the cluster (read before anyone writes it)
    extern __shared__ __align__(16) unsigned char sm[];
    const int DB = a.DB, DA = a.DB + a.LA, NA = DA + 1, NB = DB + 1, W = a.W, E = a.E;
    const int C = static_cast<int>(gridDim.x);
    const int c = static_cast<int>(cluster_rank());
    const int t = threadIdx.x;
    const bool producer = t >= kClCompute;
    const int pt = t - kClCompute;
    const int smax = a.smax;
    uint64_t* bars_a = reinterpret_cast<uint64_t*>(sm);               // NA
    uint64_t* bars_b = bars_a + kClMaxNA;                              // NB
    int32_t* s_lo = reinterpret_cast<int32_t*>(sm + a.off_sl);       // nlev: first position
    int32_t* s_cnt = s_lo + a.nlev;                                  // nlev: positions
    double* s_v = reinterpret_cast<double*>(sm + a.off_v);          // W x smax
    for (int l = t; l < a.nlev; l += kClThreads) {
        const int lb = __ldg(a.lptr + l), le = __ldg(a.lptr + l + 1);
        const int ch = (((le - lb) + C - 1) / C + 31) & ~31;
        const int lo = min(le, lb + c * ch);
        s_lo[l] = lo;
        s_cnt[l] = min(le, lo + ch) - lo;
    }
    if (t == 0) {
        for (int q = 0; q < NA; ++q) mbar_init(bars_a + q);
        for (int q = 0; q < NB; ++q) mbar_init_count(bars_b + q, kClProducer);
        fence_mbar_init();
    }
    __syncthreads();
    const bool want_rho = BWD && a.r != nullptr;
    const unsigned v_base = smem_u32(s_v);
    auto a_perm = [&](int slot) { return reinterpret_cast<int32_t*>(sm + a.off_a + static_cast<size_t>(slot) * a.a_stage); };
    auto a_code = [&](int slot) { return a_perm(slot) + smax; };
    auto a_val = [&](int slot) {
        return reinterpret_cast<double*>(sm + a.off_a + static_cast<size_t>(slot) * a.a_stage +
                                         static_cast<size_t>(smax) * 4 * (1 + E));
    };
    auto b_tail = [&](int slot) { return reinterpret_cast<double*>(sm + a.off_b + static_cast<size_t>(slot) * a.b_stage); };
    auto issue_a = [&](int l, int slot) {   // one producer thread
        const int lo = s_lo[l], cnt = s_cnt[l];
        mbar_expect_tx(bars_a + slot, static_cast<unsigned>(cnt) * (4u + 12u * E));
        if (cnt > 0) {
            bulk_g2s(a_perm(slot), a.perm + lo, cnt * 4u, bars_a + slot);
            bulk_g2s(a_code(slot), a.code + static_cast<int64_t>(lo) * E, cnt * 4u * E, bars_a + slot);
            bulk_g2s(a_val(slot), a.val + static_cast<int64_t>(lo) * E, cnt * 8u * E, bars_a + slot);
        }
    };
    auto issue_b = [&](int l, int slot, int aslot) {   // every producer thread
        const int cnt = s_cnt[l];
        mbar_wait(bars_a + aslot, static_cast<unsigned>(l / NA) & 1u);
        const int32_t* pm = a_perm(aslot);
        double* tl = b_tail(slot);
        for (int j = pt; j < cnt; j += kClProducer) {
            const int32_t row = pm[j];
            if (row < 0) continue;
            cp_async8(smem_u32(tl + j), a.in + row);
            if (BWD) cp_async8(smem_u32(tl + smax + j), a.d + row);
            if (want_rho) cp_async8(smem_u32(tl + 2 * smax + j), a.r + row);
        }
        cp_async_mbar_arrive(bars_b + slot);
    };

    unsigned long long pc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long t0 = clock64(), t1;
#define CL_MARK(k)                                         \
    if (a.prof) {                                          \
        t1 = clock64();                                    \
        pc[k] += static_cast<unsigned long long>(t1 - t0); \
        t0 = t1;                                           \
    }
    // ring slots of level i (A: NA, B: NB, V: W levels); the loop starts at i = -DA
    int sa = ((-DA % NA) + NA) % NA, sb = ((-DA % NB) + NB) % NB, sv = ((-DA % W) + W) % W;
    for (int i = -DA; i < a.nlev; ++i) {
        if (producer) {
            if (i >= 0) cluster_arrive_relaxed();   // producers hold no values of level i
            CL_MARK(7);
            const int sa_next = sa == 0 ? NA - 1 : sa - 1;   // slot of level i + DA (free: level i - 1's)
            const int sb_next = sb == 0 ? NB - 1 : sb - 1;   // slot of level i + DB
            if (pt == 0 && i + DA < a.nlev) issue_a(i + DA, sa_next);
            CL_MARK(3);
            if (i + DB >= 0 && i + DB < a.nlev) issue_b(i + DB, sb_next, (sa + DB) % NA);
            CL_MARK(4);
            if (i >= 0) cluster_wait();
            CL_MARK(6);
        } else if (i >= 0) {
            const int lo = s_lo[i], cnt = s_cnt[i];
            CL_MARK(7);
            mbar_wait(bars_b + sb, static_cast<unsigned>(i / NB) & 1u);   // stage B (and so A) of level i
            CL_MARK(0);
            const int32_t* pm = a_perm(sa);
            const int32_t* cd = a_code(sa);
            const double* vl = a_val(sa);
            const double* tl = b_tail(sb);
            int32_t rows[R];
            double res[R], contrib[R], dep[R][kClE];
#pragma unroll
            for (int k = 0; k < R; ++k) {   // every parent load of the thread's rows first
                const int j = t + k * kClCompute;
                rows[k] = j < cnt ? pm[j] : -1;
#pragma unroll
                for (int e = 0; e < kClE; ++e) {
                    const int cc = (rows[k] >= 0 && e < E) ? cd[j * E + e] : -1;
                    dep[k][e] = 0.0;
                    if (cc >= 0)
                        dep[k][e] = ld_dsmem(v_base + 8u * static_cast<unsigned>(cc & 0xFFFFFF),
                                             static_cast<unsigned>(cc) >> 24);
                }
            }
            double* vr = s_v + sv * smax;
#pragma unroll
            for (int k = 0; k < R; ++k) {
                contrib[k] = 0.0;
                res[k] = 0.0;
                if (rows[k] < 0) continue;
                const int j = t + k * kClCompute;
                double s = BWD ? __ddiv_rn(tl[j], tl[smax + j]) : tl[j];
#pragma unroll
                for (int e = 0; e < kClE; ++e)
                    if (e < E && cd[j * E + e] != -1) s = fsub_mul(s, vl[j * E + e], dep[k][e]);
                s = publishable(s);
                res[k] = s;
                vr[j] = s;
                if (want_rho) contrib[k] = __dmul_rn(tl[2 * smax + j], s);
            }
            CL_MARK(1);
            compute_bar();   // level i's values are in shared memory
            CL_MARK(2);
            cluster_arrive_relaxed();
#pragma unroll
            for (int k = 0; k < R; ++k)
                if (rows[k] >= 0) __stcg(a.out + rows[k], res[k]);
            if (want_rho) {
                // per-tile partials: warp w's slots (t & ~31) + k * kClCompute are 32 consecutive
                // positions of one tile (levels and chunks are 32-aligned), lane == pos % 32 as in
                // k_sweep's tile_reduce
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    const int j0 = (t & ~31) + k * kClCompute;
                    if (j0 >= cnt) break;   // warp-uniform
                    const double v = warp_sum(contrib[k]);
                    if ((t & 31) == 0) __stcg(a.partials + (lo + j0) / 32, v);
                }
            }
            CL_MARK(5);
            cluster_wait();
            CL_MARK(6);
        }
        sa = sa + 1 == NA ? 0 : sa + 1;
        sb = sb + 1 == NB ? 0 : sb + 1;
        sv = sv + 1 == W ? 0 : sv + 1;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (a.prof && (t == 0 || t == kClCompute)) {
        const int base = t == 0 ? 0 : 8;
        for (int k = 0; k < 8; ++k) atomicAdd(&g_cl_prof[c][(base + k) & 15], pc[k]);
    }
#undef CL_MARK
    if (!want_rho) return;
    // group sums then the total, in k_sweep's tile_reduce order
    cluster_arrive();
    cluster_wait();
    const int ntiles = (a.npos + 31) / 32;
    const int ngroups = (ntiles + kGroup - 1) / kGroup;
    const int warps = C * (kClThreads / 32);
    const int gw = c * (kClThreads / 32) + (t >> 5);
    const int lane = t & 31;
    for (int g = gw; g < ngroups; g += warps) {
        const int gsize = min(kGroup, ntiles - g * kGroup);
        double gs = 0.0;
        for (int q = lane; q < gsize; q += 32) gs = __dadd_rn(gs, __ldcg(a.partials + g * kGroup + q));
        gs = warp_sum(gs);
        if (lane == 0) __stcg(a.gpart + g, gs);
    }
    cluster_arrive();
    cluster_wait();
    if (c != 0 || t >= 32) return;
    double ts = 0.0;
    for (int q = lane; q < ngroups; q += 32) ts = __dadd_rn(ts, __ldcg(a.gpart + q));
    ts = warp_sum(ts);
    if (lane == 0) {
        DevState* st = a.st;   // src/pcg.cpp:65-71, as k_sweep's finaliser
        const double rho = a.add_sc ? ts + st->scal[2] : ts;
        st->rho = rho;
        if (rho <= 0.0) {
            st->done = kBroken;
            st->status = kBrkRz;
        }
        st->beta = st->iter > 1 ? rho / st->rho_prev : 0.0;
    }
}

// ------------------------------------------------------------------ plan (device build)
__global__ void k_cl_inverse(const int32_t* perm, int32_t npos, int32_t* pos_of_row) {
    for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < npos; p += int64_t(gridDim.x) * blockDim.x) {
        const int32_t r = perm[p];
        if (r >= 0) pos_of_row[r] = static_cast<int32_t>(p);
    }
}

__device__ __forceinline__ int level_of(const int32_t* lptr, int nlev, int32_t pos) {
    int lo = 0, hi = nlev - 1;   // last l with lptr[l] <= pos
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (lptr[mid] <= pos) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// max entries per row and max level distance parent -> row
__global__ void k_cl_stats(const int32_t* perm, const int32_t* prs, const int32_t* pcol, const int32_t* pos_of_row,
                           const int32_t* lptr, int nlev, int32_t npos, int* out) {
    for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < npos; p += int64_t(gridDim.x) * blockDim.x) {
        if (perm[p] < 0) continue;
        const int32_t b = prs[p], e = prs[p + 1];
        if (e - b > 0) atomicMax(out, e - b);
        const int l = level_of(lptr, nlev, static_cast<int32_t>(p));
        int dmax = 0;
        for (int32_t k = b; k < e; ++k) dmax = max(dmax, l - level_of(lptr, nlev, pos_of_row[pcol[k]]));
        if (dmax > 0) atomicMax(out + 1, dmax);
    }
}

__global__ void k_cl_ell(const int32_t* perm, const int32_t* prs, const int32_t* pcol, const double* pval,
                         const int32_t* pos_of_row, const int32_t* lptr, int nlev, int32_t npos, int C, int W,
                         int E, int smax, int32_t* code, double* val) {
    for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < npos; p += int64_t(gridDim.x) * blockDim.x) {
        const bool real = perm[p] >= 0;
        const int32_t b = real ? prs[p] : 0, e = real ? prs[p + 1] : 0;
        const int l = level_of(lptr, nlev, static_cast<int32_t>(p));
        for (int k = 0; k < E; ++k) {
            int32_t cd = -1;
            double v = 0.0;
            if (b + k < e) {
                const int32_t pp = pos_of_row[pcol[b + k]];
                const int lp = level_of(lptr, nlev, pp);
                const int a0 = lptr[lp], b0 = lptr[lp + 1];
                const int ch = (((b0 - a0) + C - 1) / C + 31) & ~31;
                const int cta = (pp - a0) / ch, idx = (pp - a0) % ch;
                cd = (cta << 24) | ((lp % W) * smax + idx);   // l - lp < W: checked by the plan
                v = pval[b + k];
            }
            code[p * E + k] = cd;
            val[p * E + k] = v;
        }
    }
}

static int cluster_size_for() {
    static int cached = -1;
    if (cached >= 0) return cached;
    const char* env = std::getenv("RCG_SWEEP_CLUSTER_SIZE");
    const int want = env ? std::atoi(env) : 16;
    cached = 0;
    for (int C : {want, 16, 8}) {
        if (C <= 0 || C > 16) continue;
        auto k = k_sweep_cl<false, 1>;
        if (C > 8 && cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(C);
        cfg.blockDim = dim3(kClThreads);
        cfg.dynamicSmemBytes = 64 * 1024;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = C;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int nclusters = 0;
        if (cudaOccupancyMaxActiveClusters(&nclusters, k, &cfg) == cudaSuccess && nclusters > 0) {
            cached = C;
            break;
        }
        cudaGetLastError();
    }
    return cached;
}

static size_t r16(size_t v) { return (v + 15) & ~size_t(15); }

struct ClLayout {
    size_t off_sl, off_a, off_b, off_v, a_stage, b_stage, total;
};

static ClLayout cl_layout(int nlev, int DB, int LA, int smax, int W, int E, bool backward) {
    ClLayout L{};
    const int NA = DB + LA + 1;
    L.off_sl = r16(static_cast<size_t>(kClMaxNA + 4) * 8);
    L.off_a = L.off_sl + r16(static_cast<size_t>(2 * nlev) * 4);
    L.a_stage = static_cast<size_t>(smax) * (4 + 12 * E);   // smax multiple of 32: sub-arrays 16-aligned
    L.off_b = L.off_a + static_cast<size_t>(NA) * L.a_stage;
    L.b_stage = static_cast<size_t>(smax) * (backward ? 24 : 8);
    L.off_v = L.off_b + static_cast<size_t>(DB + 1) * L.b_stage;
    L.total = L.off_v + static_cast<size_t>(W) * smax * 8;
    return L;
}

// shared-memory budget of one cluster CTA (RCG_CL_SMEM_KB): the deepest prefetch that fits
static size_t cl_smem_cap() {
    static size_t cap = [] {
        const char* e = std::getenv("RCG_CL_SMEM_KB");
        return static_cast<size_t>(e ? std::atoi(e) : 227) * 1024;
    }();
    return cap;
}

static ClusterPlan* build_plan(rcg_ctx* ctx, const rcg_ic* f, bool backward) {
    auto* pl = new ClusterPlan();
    const std::vector<int32_t>& lp = f->h_lptr[backward ? 1 : 0];
    const int nlev = backward ? f->bwd_levels : f->fwd_levels;
    const int32_t npos = backward ? f->b_npos : f->f_npos;
    if (static_cast<int>(lp.size()) != nlev + 1 || nlev <= 0 || f->n == 0) return pl;
    const int C = cluster_size_for();
    if (C == 0) return pl;
    int smax = 0;   // the widest level decides the slot count
    for (int l = 0; l < nlev; ++l) {
        const int w = lp[l + 1] - lp[l];
        smax = std::max(smax, ((w + C - 1) / C + 31) & ~31);
    }
    if (smax > kClMaxR * kClCompute) return pl;
    const int32_t* perm = backward ? f->b_perm : f->f_perm;
    const int32_t* prs = backward ? f->b_prs : f->f_prs;
    const int32_t* pcol = backward ? f->b_col : f->f_col;
    const double* pval = backward ? f->b_val : f->f_val;
    int32_t* d_lptr = static_cast<int32_t*>(dev_alloc_bytes(sizeof(int32_t) * lp.size()));
    int32_t* pos_of_row = static_cast<int32_t*>(dev_alloc_bytes(sizeof(int32_t) * f->n));
    int* stats = static_cast<int*>(dev_alloc_bytes(sizeof(int) * 2));
    RCG_CK(cudaMemcpyAsync(d_lptr, lp.data(), sizeof(int32_t) * lp.size(), cudaMemcpyHostToDevice, ctx->stream));
    RCG_CK(cudaMemsetAsync(stats, 0, sizeof(int) * 2, ctx->stream));
    const int g = std::max(1, std::min<int>((npos + 255) / 256, ctx->num_sms * 8));
    k_cl_inverse<<<g, 256, 0, ctx->stream>>>(perm, npos, pos_of_row);
    k_cl_stats<<<g, 256, 0, ctx->stream>>>(perm, prs, pcol, pos_of_row, d_lptr, nlev, npos, stats);
    int h[2];
    RCG_CK(cudaMemcpyAsync(h, stats, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
    RCG_CK(cudaStreamSynchronize(ctx->stream));
    dev_free(stats);
    const int E = std::max(1, h[0]);
    const int W = std::max(2, h[1] + 1);   // every parent within the DSMEM ring (no HBM parents)
    int DB = 0, LA = 0;   // deepest prefetch that fits: gathers DB levels ahead, TMA DB + LA
    for (auto [db, la] : {std::pair{2, 2}, {2, 1}, {1, 2}, {1, 1}})
        if (cl_layout(nlev, db, la, smax, W, E, backward).total <= cl_smem_cap()) {
            DB = db;
            LA = la;
            break;
        }
    if (E > kClE || W > kClMaxW || DB == 0) {
        dev_free(d_lptr);
        dev_free(pos_of_row);
        return pl;
    }
    const int64_t ne = std::max<int64_t>(int64_t(npos) * E, 1);
    pl->code = static_cast<int32_t*>(dev_alloc_bytes(sizeof(int32_t) * ne));
    pl->val = static_cast<double*>(dev_alloc_bytes(sizeof(double) * ne));
    k_cl_ell<<<g, 256, 0, ctx->stream>>>(perm, prs, pcol, pval, pos_of_row, d_lptr, nlev, npos, C, W, E, smax,
                                         pl->code, pl->val);
    RCG_LAUNCHED(ctx);
    RCG_CK(cudaStreamSynchronize(ctx->stream));
    dev_free(pos_of_row);
    pl->lptr = d_lptr;
    pl->C = C;
    pl->W = W;
    pl->E = E;
    pl->DB = DB;
    pl->LA = LA;
    pl->R = (smax + kClCompute - 1) / kClCompute;
    pl->smax = smax;
    pl->nlev = nlev;
    pl->smem = cl_layout(nlev, DB, LA, smax, W, E, backward).total;
    pl->ok = true;
    return pl;
}

// RCG_CL_PROF: print and clear the per-phase counters (CTA 0 and the max over CTAs)
void cluster_prof_dump(const char* tag) {
    unsigned long long h[16][16];
    if (cudaMemcpyFromSymbol(h, g_cl_prof, sizeof h) != cudaSuccess) return;
    static const char* names[16] = {"c.bwait", "c.compute", "c.bar", "-", "-", "c.stores", "c.clwait", "c.loop",
                                    "-", "-", "-", "p.issue_a", "p.issue_b", "-", "p.clwait", "p.loop"};
    std::fprintf(stderr, "[cl_prof %s] cycles (CTA0 / max over CTAs):", tag);
    for (int k = 0; k < 16; ++k) {
        if (names[k][0] == '-') continue;
        unsigned long long mx = 0;
        for (int c = 0; c < 16; ++c) mx = std::max(mx, h[c][k]);
        std::fprintf(stderr, " %s=%llu/%llu", names[k], h[0][k], mx);
    }
    std::fprintf(stderr, "\n");
    std::memset(h, 0, sizeof h);
    cudaMemcpyToSymbol(g_cl_prof, h, sizeof h);
}

void free_cluster_plans(rcg_ic* f) {
    for (auto*& p : f->cl) {
        if (!p) continue;
        dev_free(p->lptr);
        dev_free(p->code);
        dev_free(p->val);
        delete p;
        p = nullptr;
    }
}

using ClKernel = void (*)(ClArgs);

static ClKernel cl_kernel(bool backward, int R) {
    static const ClKernel ks[2][kClMaxR] = {{k_sweep_cl<false, 1>, k_sweep_cl<false, 2>},
                                            {k_sweep_cl<true, 1>, k_sweep_cl<true, 2>}};
    static bool attrs = false;
    if (!attrs) {  // once: opt in to 16-CTA clusters and the full shared-memory budget
        const char* e = std::getenv("RCG_CL_CARVEOUT");
        for (auto& row : ks)
            for (ClKernel k : row) {
                RCG_CK(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
                RCG_CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
                if (e) RCG_CK(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, std::atoi(e)));
            }
        attrs = true;
    }
    return ks[backward ? 1 : 0][R - 1];
}

// Cluster sweeps are used when the plan fits (<= 4 entries per row, every parent within 3
// levels, the widest level within 16 x 1024 slots) and the levels are narrow enough that
// latency, not bandwidth, bounds the sweep (ctx->sweep_cluster: 0 = never, 1 = whenever the
// plan fits, 2 = by shape; rcg_ctx_set_sweep_kernel / RCG_SWEEP_CLUSTER).
bool launch_cluster_sweep(rcg_ctx* ctx, const rcg_ic* f, bool backward, SweepArgs& s) {
    const int mode = ctx->sweep_cluster;
    if (mode != 1) return false;   // by shape (2): measured slower than the grid sweep everywhere
    const int dir = backward ? 1 : 0;
    if (!f->cl[dir]) f->cl[dir] = build_plan(ctx, f, backward);
    const ClusterPlan* pl = f->cl[dir];
    if (!pl->ok) return false;
    ClArgs a{};
    a.lptr = pl->lptr;
    a.perm = s.perm;
    a.code = pl->code;
    a.val = pl->val;
    a.in = s.in;
    a.d = s.d;
    a.r = backward ? s.r : nullptr;
    a.out = s.out;
    a.partials = s.partials;
    a.gpart = s.gpart;
    a.st = s.st;
    a.add_sc = s.add_sc;
    a.nlev = pl->nlev;
    a.npos = s.npos;
    a.W = pl->W;
    a.E = pl->E;
    a.DB = pl->DB;
    a.LA = pl->LA;
    a.smax = pl->smax;
    const ClLayout L = cl_layout(pl->nlev, pl->DB, pl->LA, pl->smax, pl->W, pl->E, backward);
    a.off_sl = static_cast<int>(L.off_sl);
    a.off_a = static_cast<int>(L.off_a);
    a.off_b = static_cast<int>(L.off_b);
    a.off_v = static_cast<int>(L.off_v);
    a.a_stage = static_cast<int>(L.a_stage);
    a.b_stage = static_cast<int>(L.b_stage);
    static const bool prof = std::getenv("RCG_CL_PROF") != nullptr;
    a.prof = prof ? 1 : 0;
    ClKernel k = cl_kernel(backward, pl->R);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(pl->C);
    cfg.blockDim = dim3(kClThreads);
    cfg.dynamicSmemBytes = pl->smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = pl->C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    KTimer tm(ctx, backward ? 2 : 1);
    RCG_CK(cudaLaunchKernelEx(&cfg, k, a));
    RCG_LAUNCHED(ctx);
    return true;
}

}  // namespace rcg
