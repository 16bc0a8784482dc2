// context.cu -- context, workspaces, host/device staging, error strings, timing.
#include <cstdio>
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

double* dev_alloc(int64_t count) {
    void* p = nullptr;
    if (count <= 0) count = 1;
    const cudaError_t e = cudaMalloc(&p, static_cast<size_t>(count) * sizeof(double));
    if (e != cudaSuccess) {
        cudaGetLastError();
        char buf[256];
        std::snprintf(buf, sizeof buf, "device allocation of %lld bytes failed: %s",
                      static_cast<long long>(count * 8), cudaGetErrorString(e));
        throw Error(RCG_E_CUDA, buf);
    }
    return static_cast<double*>(p);
}

void dev_free(void* p) {
    if (p) cudaFree(p);
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
    if (owned && dev) cudaFree(dev);
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

// Event pairs are recorded around each timed launch without synchronising; they are resolved
// (and recycled) when the statistics are read, so timing does not serialise the stream.
static cudaEvent_t pooled_event(rcg_ctx* ctx) {
    if (ctx->ev_free.empty()) {
        cudaEvent_t e;
        RCG_CK(cudaEventCreate(&e));
        return e;
    }
    cudaEvent_t e = ctx->ev_free.back();
    ctx->ev_free.pop_back();
    return e;
}

KTimer::KTimer(rcg_ctx* c, int k) : ctx(c), cls(k) {
    if (!ctx->profiling) return;
    start = pooled_event(ctx);
    RCG_CK(cudaEventRecord(start, ctx->stream));
}

KTimer::~KTimer() {
    if (!ctx->profiling) return;
    cudaEvent_t stop = pooled_event(ctx);
    cudaEventRecord(stop, ctx->stream);
    ctx->ev_pending.push_back({cls, start, stop});
}

void resolve_timers(rcg_ctx* ctx) {
    if (ctx->ev_pending.empty()) return;
    RCG_CK(cudaStreamSynchronize(ctx->stream));
    for (auto& t : ctx->ev_pending) {
        float ms = 0.f;
        RCG_CK(cudaEventElapsedTime(&ms, t.start, t.stop));
        ctx->stat_ms[t.cls] += ms;
        ctx->stat_n[t.cls] += 1;
        ctx->ev_free.push_back(t.start);
        ctx->ev_free.push_back(t.stop);
    }
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
        if (const char* e = std::getenv("RCG_SPMV_BPS")) c->spmv_bps = std::max(1, std::atoi(e));
        RCG_CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        RCG_CK(cudaEventCreate(&c->ev0));
        RCG_CK(cudaEventCreate(&c->ev1));
        void* hp = nullptr;
        RCG_CK(cudaMallocHost(&hp, 4096));
        c->host_pinned = static_cast<double*>(hp);
        *out = c;
    });
}

void rcg_ctx_destroy(rcg_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
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
    return guard([&] { RCG_CK(cudaStreamSynchronize(ctx->stream)); });
}

int64_t rcg_ctx_launch_count(const rcg_ctx* ctx) { return ctx ? ctx->launches : 0; }

int rcg_ctx_set_profiling(rcg_ctx* ctx, int enable) {
    return guard([&] { ctx->profiling = enable != 0; });
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
        require(cls >= 0 && cls < 5, "rcg_ctx_kernel_stats: class out of range");
        resolve_timers(ctx);
        *total_ms = ctx->stat_ms[cls];
        *launches = ctx->stat_n[cls];
    });
}

void rcg_ctx_reset_stats(rcg_ctx* ctx) {
    try {
        resolve_timers(ctx);
    } catch (...) {
    }
    for (int i = 0; i < 5; ++i) {
        ctx->stat_ms[i] = 0;
        ctx->stat_n[i] = 0;
    }
}

}  // extern "C"
