// context.cu -- context, workspaces, host/device staging, error strings, timing.
#include <algorithm>
#include <cstdio>
#include <mutex>
#include <unordered_map>
#include <cstdlib>
#include <cstring>

#include "internal.cuh"
#include "kernels.cuh"

namespace rcg {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }
void clear_error() { g_last_error.clear(); }

void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
    char buf[512];
    std::snprintf(buf, sizeof buf, "CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e),
                  cudaGetErrorString(e), what, file, line);
    throw Error(RCG_E_CUDA, buf);
}

// ------------------------------------------------------------------ device allocations
// A block cache in front of cudaMalloc/cudaFree.  The sequence allocates and frees hundreds of
// MB per step (sampler slots, the error block, W / AW, staging buffers); cudaMalloc/cudaFree of
// such blocks are slow and erratic (cudaFree synchronises the device; a process's first large
// allocations on a fresh GPU cost far more), so freed blocks are kept and reused.  A freed
// block is fenced with one event per live context stream on its device and handed out again
// only once every fence has completed -- the ordering cudaFree's implicit sync gave, without
// the sync.  The cache is capped; an allocation failure releases it and retries.
namespace {
struct FreeBlock {
    void* p;
    size_t bytes;
    int dev;
    std::vector<cudaEvent_t> fences;
};
std::mutex g_mx;
std::vector<rcg_ctx*> g_ctxs;
std::unordered_map<void*, std::pair<size_t, int>> g_live;
std::vector<FreeBlock> g_free;
std::vector<cudaEvent_t> g_fence_pool;
size_t g_cached = 0;
constexpr size_t kCacheCap = size_t(48) << 30;

size_t round_bytes(size_t b) {
    if (b < 256) b = 256;
    if (b < (size_t(1) << 20)) return (b + 511) & ~size_t(511);
    return (b + (size_t(2) << 20) - 1) & ~((size_t(2) << 20) - 1);
}

bool fences_done(FreeBlock& f) {
    for (auto e : f.fences)
        if (cudaEventQuery(e) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
    return true;
}

void recycle_fences(FreeBlock& f) {
    for (auto e : f.fences) g_fence_pool.push_back(e);
    f.fences.clear();
}

// caller holds g_mx
void release_cached(int dev) {
    cudaDeviceSynchronize();
    for (size_t i = 0; i < g_free.size();) {
        if (g_free[i].dev == dev) {
            cudaFree(g_free[i].p);
            g_cached -= g_free[i].bytes;
            recycle_fences(g_free[i]);
            g_free[i] = std::move(g_free.back());
            g_free.pop_back();
        } else {
            ++i;
        }
    }
}
}  // namespace

void register_ctx(rcg_ctx* c, bool add) {
    std::lock_guard<std::mutex> lk(g_mx);
    if (add) {
        g_ctxs.push_back(c);
    } else {
        g_ctxs.erase(std::remove(g_ctxs.begin(), g_ctxs.end(), c), g_ctxs.end());
    }
}

void* dev_alloc_bytes(size_t bytes) {
    int dev = 0;
    RCG_CK(cudaGetDevice(&dev));
    const size_t rb = round_bytes(bytes);
    std::lock_guard<std::mutex> lk(g_mx);
    int best = -1;
    for (size_t i = 0; i < g_free.size(); ++i) {
        FreeBlock& f = g_free[i];
        if (f.dev != dev || f.bytes < rb || f.bytes > rb + rb / 4) continue;
        if (best >= 0 && f.bytes >= g_free[best].bytes) continue;
        if (!fences_done(f)) continue;
        best = static_cast<int>(i);
        if (f.bytes == rb) break;
    }
    if (best >= 0) {
        FreeBlock f = std::move(g_free[best]);
        g_free[best] = std::move(g_free.back());
        g_free.pop_back();
        g_cached -= f.bytes;
        recycle_fences(f);
        g_live[f.p] = {f.bytes, dev};
        return f.p;
    }
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, rb);
    if (e != cudaSuccess) {
        cudaGetLastError();
        release_cached(dev);
        e = cudaMalloc(&p, rb);
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        char buf[256];
        std::snprintf(buf, sizeof buf, "device allocation of %zu bytes failed: %s", bytes, cudaGetErrorString(e));
        throw Error(RCG_E_CUDA, buf);
    }
    g_live[p] = {rb, dev};
    return p;
}

double* dev_alloc(int64_t count) {
    if (count <= 0) count = 1;
    return static_cast<double*>(dev_alloc_bytes(static_cast<size_t>(count) * sizeof(double)));
}

void dev_free(void* p) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_mx);
    auto it = g_live.find(p);
    if (it == g_live.end()) {  // not from this allocator
        cudaFree(p);
        return;
    }
    FreeBlock f{p, it->second.first, it->second.second, {}};
    g_live.erase(it);
    if (g_cached + f.bytes > kCacheCap) {
        cudaFree(p);
        return;
    }
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != f.dev) cudaSetDevice(f.dev);
    for (rcg_ctx* c : g_ctxs) {
        if (c->device != f.dev) continue;
        cudaEvent_t e;
        if (!g_fence_pool.empty()) {
            e = g_fence_pool.back();
            g_fence_pool.pop_back();
        } else if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            cudaDeviceSynchronize();  // no event: fall back to a full fence
            continue;
        }
        cudaEventRecord(e, c->stream);
        f.fences.push_back(e);
    }
    if (cur != f.dev) cudaSetDevice(cur);
    g_cached += f.bytes;
    g_free.push_back(std::move(f));
}

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes at{};
    const cudaError_t e = cudaPointerGetAttributes(&at, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

Staged::~Staged() {
    if (owned && dev) dev_free(dev);
}

void stage_in(rcg_ctx* ctx, const double* src, int64_t count, Staged& out) {
    if (is_device_ptr(src)) {
        out.dev = const_cast<double*>(src);
        out.owned = false;
        return;
    }
    out.dev = dev_alloc(count);
    out.owned = true;
    if (count > 0)
        RCG_CK(cudaMemcpyAsync(out.dev, src, sizeof(double) * count, cudaMemcpyHostToDevice, ctx->stream));
}

void stage_out_begin(rcg_ctx* ctx, double* dst, int64_t count, Staged& tmp) {
    (void)ctx;
    if (is_device_ptr(dst)) {
        tmp.dev = dst;
        tmp.owned = false;
        return;
    }
    tmp.dev = dev_alloc(count);
    tmp.owned = true;
}

void stage_out_end(rcg_ctx* ctx, double* dst, int64_t count, Staged& tmp) {
    if (tmp.owned && count > 0) {
        RCG_CK(cudaMemcpyAsync(dst, tmp.dev, sizeof(double) * count, cudaMemcpyDeviceToHost, ctx->stream));
        RCG_CK(cudaStreamSynchronize(ctx->stream));
    }
}

static void grow(double*& p, int64_t& cap, int64_t need) {
    (void)cap;
    dev_free(p);
    p = dev_alloc(need);
}

void ensure_workspace(rcg_ctx* ctx, int64_t n, int k, int64_t max_iter, int64_t partials,
                      int64_t groups, int pending) {
    Workspace& w = ctx->ws;
    if (!w.st) {
        void* p = nullptr;
        RCG_CK(cudaMalloc(&p, sizeof(DevState)));
        w.st = static_cast<DevState*>(p);
        RCG_CK(cudaMemset(w.st, 0, sizeof(DevState)));
        RCG_CK(cudaMalloc(&p, 16 * sizeof(int)));
        w.tickets = static_cast<int*>(p);
        RCG_CK(cudaMemset(w.tickets, 0, 16 * sizeof(int)));
    }
    if (n > w.cap_n) {
        double** vecs[] = {&w.r, &w.z, &w.p, &w.q, &w.ybuf, &w.zs, &w.v, &w.vnext, &w.bw, &w.xw};
        for (double** v : vecs) {
            dev_free(*v);
            *v = dev_alloc(n);
        }
        w.cap_n = n;
    }
    if (k > w.cap_k) {
        dev_free(w.u);
        dev_free(w.u2);
        w.u = dev_alloc(k);
        w.u2 = dev_alloc(k);
        w.cap_k = k;
    }
    if (max_iter + 1 > w.cap_iter) {
        int64_t c = 0;
        grow(w.hist, c, max_iter + 1);
        grow(w.alph, c, max_iter + 1);
        grow(w.bet, c, max_iter + 1);
        w.cap_iter = max_iter + 1;
    }
    if (partials > w.cap_partials) {
        dev_free(w.partials);
        w.partials = dev_alloc(partials);
        w.cap_partials = partials;
    }
    if (groups > w.cap_groups) {
        dev_free(w.gpart);
        dev_free(w.gcount);
        w.gpart = dev_alloc(groups * 4);
        void* p = nullptr;
        RCG_CK(cudaMalloc(&p, sizeof(unsigned int) * groups));
        w.gcount = static_cast<unsigned int*>(p);
        RCG_CK(cudaMemset(w.gcount, 0, sizeof(unsigned int) * groups));
        w.cap_groups = groups;
    }
    if (pending > w.cap_pending) {
        dev_free(w.smp_pending);
        void* p = nullptr;
        RCG_CK(cudaMalloc(&p, sizeof(int) * pending));
        w.smp_pending = static_cast<int*>(p);
        w.cap_pending = pending;
    }
}

// Event pairs are recorded around each timed launch without synchronising; completed pairs are
// folded into the statistics and recycled as new events are needed (cudaEventQuery, no stream
// sync), and the pool is pre-filled when profiling is switched on, so timing neither creates
// events on the enqueue path nor serialises the stream.
static void fold(rcg_ctx* ctx, const rcg_ctx::TimedLaunch& t) {
    float ms = 0.f;
    RCG_CK(cudaEventElapsedTime(&ms, t.start, t.stop));
    ctx->stat_ms[t.cls] += ms;
    ctx->stat_n[t.cls] += 1;
    ctx->stat_units[t.cls] += t.units;
    ctx->ev_free.push_back(t.start);
    ctx->ev_free.push_back(t.stop);
}

static void grow_pool(rcg_ctx* ctx, int count) {
    for (int i = 0; i < count; ++i) {
        cudaEvent_t e;
        RCG_CK(cudaEventCreate(&e));
        ctx->ev_free.push_back(e);
    }
}

static cudaEvent_t pooled_event(rcg_ctx* ctx) {
    if (ctx->ev_free.empty()) {
        while (!ctx->ev_pending.empty() && cudaEventQuery(ctx->ev_pending.front().stop) == cudaSuccess) {
            fold(ctx, ctx->ev_pending.front());
            ctx->ev_pending.pop_front();
        }
        if (ctx->ev_free.empty()) grow_pool(ctx, 512);
    }
    cudaEvent_t e = ctx->ev_free.back();
    ctx->ev_free.pop_back();
    return e;
}

KTimer::KTimer(rcg_ctx* c, int k, int u) : ctx(c), cls(k), units(u) {
    if (!ctx->profiling || !((ctx->profile_mask >> k) & 1u)) {
        cls = -1;
        return;
    }
    start = pooled_event(ctx);
    RCG_CK(cudaEventRecord(start, ctx->stream));
}

KTimer::~KTimer() {
    if (!ctx->profiling || cls < 0) return;
    cudaEvent_t stop = pooled_event(ctx);
    cudaEventRecord(stop, ctx->stream);
    ctx->ev_pending.push_back({cls, units, start, stop});
}

void resolve_timers(rcg_ctx* ctx) {
    if (ctx->ev_pending.empty()) return;
    RCG_CK(cudaStreamSynchronize(ctx->stream));
    for (auto& t : ctx->ev_pending) fold(ctx, t);
    ctx->ev_pending.clear();
}

}  // namespace rcg

using namespace rcg;

extern "C" {

const char* rcg_last_error(void) { return rcg::g_last_error.c_str(); }

const char* rcg_build_info(void) {
    return "librcg_b200: sm_100a fp64 deflated ICCG, CUDA 12.9 build";
}

int rcg_ctx_create(int device, rcg_ctx** out) {
    return guard([&] {
        *out = nullptr;
        int count = 0;
        const cudaError_t e = cudaGetDeviceCount(&count);
        if (e != cudaSuccess || count == 0) {
            cudaGetLastError();
            throw Error(RCG_E_CUDA, "no CUDA device available: librcg_b200 has no CPU fallback");
        }
        require(device >= 0 && device < count, "rcg_ctx_create: device index out of range");
        RCG_CK(cudaSetDevice(device));
        cudaDeviceProp prop{};
        RCG_CK(cudaGetDeviceProperties(&prop, device));
        if (prop.major < 10)
            throw Error(RCG_E_CUDA, std::string("device ") + prop.name +
                                        " is not sm_100 class; this build targets sm_100a only");
        auto* c = new rcg_ctx();
        c->device = device;
        c->num_sms = prop.multiProcessorCount;
        if (const char* e = std::getenv("RCG_SWEEP_BPS")) c->sweep_bps = std::max(1, std::atoi(e));
        if (const char* e = std::getenv("RCG_SWEEP_BACKOFF_NS")) c->sweep_backoff_ns = std::max(0, std::atoi(e));
        if (const char* e = std::getenv("RCG_SWEEP_CLUSTER")) {
            const int m = std::atoi(e);
            if (m == 0 || m == 2 || m == 4) c->sweep_cluster = m;
        }
        if (const char* e = std::getenv("RCG_SPMV_BPS")) c->spmv_bps = std::max(1, std::atoi(e));
        RCG_CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        register_ctx(c, true);
        RCG_CK(cudaEventCreate(&c->ev0));
        RCG_CK(cudaEventCreate(&c->ev1));
        void* hp = nullptr;
        RCG_CK(cudaMallocHost(&hp, 16384));  // [0,2K) state staging, [2K,4K) done flags, [8K,16K) batch retire
        c->host_pinned = static_cast<double*>(hp);
        *out = c;
    });
}

void rcg_ctx_destroy(rcg_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    register_ctx(ctx, false);
    batch_ws_free(ctx);
    Workspace& w = ctx->ws;
    for (void* p : {(void*)w.r, (void*)w.z, (void*)w.p, (void*)w.q, (void*)w.ybuf, (void*)w.zs,
                    (void*)w.v, (void*)w.vnext, (void*)w.bw, (void*)w.xw, (void*)w.hist,
                    (void*)w.alph, (void*)w.bet, (void*)w.u, (void*)w.u2, (void*)w.partials,
                    (void*)w.gpart, (void*)w.gcount, (void*)w.tickets, (void*)w.st,
                    (void*)w.smp_pending})
        dev_free(p);
    if (ctx->host_pinned) cudaFreeHost(ctx->host_pinned);
    for (auto& t : ctx->ev_pending) {
        cudaEventDestroy(t.start);
        cudaEventDestroy(t.stop);
    }
    for (auto e : ctx->ev_free) cudaEventDestroy(e);
    for (auto e : ctx->user_ev)
        if (e) cudaEventDestroy(e);
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

int rcg_ctx_synchronize(rcg_ctx* ctx) {
    return guard([&] {
        RCG_CK(cudaStreamSynchronize(ctx->stream));
    });
}

int64_t rcg_ctx_launch_count(const rcg_ctx* ctx) { return ctx ? ctx->launches : 0; }

int rcg_ctx_set_sweep_kernel(rcg_ctx* ctx, int mode) {
    return guard([&] {
        require(ctx != nullptr && (mode == 0 || mode == 2 || mode == 4),
                "rcg_ctx_set_sweep_kernel: mode must be 0 (grid-wide), 2 (by shape) or 4 (per level)");
        ctx->sweep_cluster = mode;
    });
}

int rcg_ctx_set_profiling_mask(rcg_ctx* ctx, unsigned mask) {
    return guard([&] { ctx->profile_mask = mask; });
}

int rcg_ctx_set_profiling(rcg_ctx* ctx, int enable) {
    return guard([&] {
        ctx->profiling = enable != 0;
        const size_t want = 8192;
        if (ctx->profiling && ctx->ev_free.size() < want) grow_pool(ctx, static_cast<int>(want - ctx->ev_free.size()));
    });
}

int rcg_ctx_event_record(rcg_ctx* ctx, int slot) {
    return guard([&] {
        require(slot >= 0 && slot < 16, "rcg_ctx_event_record: slot out of range");
        if (!ctx->user_ev[slot]) RCG_CK(cudaEventCreate(&ctx->user_ev[slot]));
        RCG_CK(cudaEventRecord(ctx->user_ev[slot], ctx->stream));
    });
}

int rcg_ctx_event_elapsed(rcg_ctx* ctx, int slot_a, int slot_b, double* ms) {
    return guard([&] {
        require(slot_a >= 0 && slot_a < 16 && slot_b >= 0 && slot_b < 16 && ctx->user_ev[slot_a] &&
                    ctx->user_ev[slot_b],
                "rcg_ctx_event_elapsed: slot not recorded");
        RCG_CK(cudaEventSynchronize(ctx->user_ev[slot_b]));
        float f = 0.f;
        RCG_CK(cudaEventElapsedTime(&f, ctx->user_ev[slot_a], ctx->user_ev[slot_b]));
        *ms = f;
    });
}

int rcg_ctx_kernel_stats(rcg_ctx* ctx, int cls, double* total_ms, int64_t* launches) {
    return guard([&] {
        require(cls >= 0 && cls < kStatClasses, "rcg_ctx_kernel_stats: class out of range");
        resolve_timers(ctx);
        *total_ms = ctx->stat_ms[cls];
        *launches = ctx->stat_n[cls];
    });
}

int rcg_ctx_kernel_units(rcg_ctx* ctx, int cls, int64_t* units) {
    return guard([&] {
        require(cls >= 0 && cls < kStatClasses, "rcg_ctx_kernel_units: class out of range");
        resolve_timers(ctx);
        *units = ctx->stat_units[cls];
    });
}

void rcg_ctx_reset_stats(rcg_ctx* ctx) {
    try {
        resolve_timers(ctx);
    } catch (...) {
    }
    for (int i = 0; i < kStatClasses; ++i) {
        ctx->stat_ms[i] = 0;
        ctx->stat_n[i] = 0;
        ctx->stat_units[i] = 0;
    }
}

}  // extern "C"
