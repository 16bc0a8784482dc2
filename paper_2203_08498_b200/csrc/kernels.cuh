// kernels.cuh -- argument blocks and launchers shared between the kernel translation units.
#pragma once

#include "internal.cuh"

namespace rcg {

struct SpmvArgs {
    const int32_t* rs;
    const int32_t* ci;
    const double* va;
    int32_t n;
    const double* x[2];
    double* y[2];
    double* partials;
};

// one IC sweep (forward on L, or backward on U with the 1/d pass folded in)
struct SweepArgs {
    const int32_t* perm;   // processing position -> row
    const int32_t* prs;    // position-indexed row starts
    const int32_t* pcol;   // original column indices, reference entry order
    const double* pval;
    const double* d;       // pivots (backward)
    int32_t n;
    int32_t npos;          // level-padded length of the schedule (multiple of 32 per level)
    const double* in;      // forward: r ; backward: y (undivided forward result)
    double* out;           // sentinel-initialised result the dependants poll
    double* in_reset;      // backward: y is reset to the sentinel after use (nullable)
    const double* r;       // backward: rho = (r, z) partials when non-null
    int add_sc;            // backward: rho += (W^T r) . u (subspace correction)
    int backoff_ns;        // first __nanosleep of a dependency wait
    int* tickets;          // [0] tile ticket, [1] exit count, [2] group ticket
    double* partials;
    double* gpart;
    unsigned int* gcount;
    DevState* st;
};

// row-slab communication of the batched solver (batch.cu; implemented over rcg_comm in dist.cu)
struct BatchComm {
    virtual ~BatchComm() {}
    virtual void allreduce(rcg_ctx* ctx, int count) = 0;     // dtot[0..count) summed over the ranks in place
    virtual void halo(rcg_ctx* ctx, double* v, int rt) = 0;  // halo rows [nloc, nloc + nhalo) of an rt-interleaved v
    double* dtot = nullptr;                                   // device, >= 768 + 48 doubles (fused reductions)
    int32_t nhalo = 0;
};
void batch_solve_dist(rcg_ctx* ctx, const rcg_matrix* a, const rcg_prec* m, const rcg_basis* defl, BatchComm* comm,
                      const double* B, double* X, const rcg_solver_config* cfg, int nrhs, rcg_solve_report* reps);

int spmv_grid(const rcg_ctx* ctx, int32_t n);
int sweep_ctas_per_sm(const rcg_ic* f, bool backward, int64_t npos);
void ensure_host_image(const rcg_ic* f);  // icfactor.cu

#ifdef __CUDACC__
// The error sampler's schedule after iteration i (sampling.cpp:7-78): method A -- every h-th
// iteration into slot (sum_l (-1)^l floor((i-1)/m^l)) mod m, h doubling at i == h m; method B --
// every slot whose threshold the relative residual has crossed.  Appends the slots to fill to
// `pending` (st->smp_npending).
__device__ __forceinline__ void smp_schedule(DevState* st, int i, double relres, int* pending, int* occupied,
                                             int* stored_iter, const double* thresholds) {
    st->smp_npending = 0;
    st->smp_pending_iter = i;
    if (st->smp_method == 0) {
        if (i % st->smp_h != 0) return;
        long long acc = 0, pw = 1;
        for (int l = 0; l <= st->smp_lmax; ++l) {
            const long long term = (i - 1) / pw;
            acc += (l % 2 == 0) ? term : -term;
            pw *= st->smp_m;
        }
        const int s = static_cast<int>(acc % st->smp_m);
        pending[st->smp_npending++] = s;
        occupied[s] = 1;
        stored_iter[s] = i;
        if (i == st->smp_h * st->smp_m) st->smp_h *= 2;
    } else if (st->smp_method == 1) {
        while (st->smp_next <= st->smp_m) {
            if (relres > thresholds[st->smp_next - 1]) break;
            const int s = st->smp_next - 1;
            pending[st->smp_npending++] = s;
            occupied[s] = 1;
            stored_iter[s] = i;
            st->smp_next++;
        }
    }
}
__global__ void k_harvest_inplace(const double* __restrict__ x, double* __restrict__ slots, int64_t lds,
                                  const int* __restrict__ list, int cnt, int32_t n, int* __restrict__ nonzero);  // recycle.cu
__global__ void k_harvest(const double* __restrict__ x, const double* __restrict__ slots, int64_t lds,
                          const int* __restrict__ list, int cnt, int raw, double* __restrict__ e, int64_t lde,
                          int32_t n, int* __restrict__ nonzero);  // recycle.cu

// solver.cu kernels reused by the multi-GPU slabs (dist.cu)
__global__ void __launch_bounds__(kStreamThreads) k_pupdate(const double* __restrict__ z, double* __restrict__ p,
                                                            double* __restrict__ zs_reset, double* __restrict__ y_reset,
                                                            int32_t n, DevState* st, const double* __restrict__ W,
                                                            int64_t ldw, int k, const double* __restrict__ u);
__global__ void k_zero_if(double* x, int32_t n, const DevState* st);
__global__ void __launch_bounds__(kStreamThreads, 4) k_tallt(const double* __restrict__ B, int64_t ldb, int k,
                                                          const double* __restrict__ y, int32_t n,
                                                          double* partials, const double* __restrict__ L,
                                                          double* __restrict__ out, int mode, DevState* st,
                                                          int respect_done);
__global__ void k_add_combination(double* __restrict__ x, const double* __restrict__ W, int64_t ldw, int k,
                                  const double* __restrict__ u, int32_t n, const DevState* st, int only_ok);
__global__ void k_sub_combination_ok(double* __restrict__ x, const double* __restrict__ W, int64_t ldw, int k,
                                     const double* __restrict__ u, int32_t n, const DevState* st);
#endif
int stream_grid(const rcg_ctx* ctx, int64_t n);
size_t spmv_smem(const rcg_matrix* a);
void spmv_prepare_kernels();
void sweep_prepare_kernels();
void set_carveout(const void* kernel);
void allow_smem(const void* kernel);
int tile_capacity(int32_t n, const int32_t* rs);
void launch_residual(rcg_ctx* ctx, const rcg_matrix* a, const double* b, const double* x, double* r);
void launch_sweep(rcg_ctx* ctx, const rcg_ic* f, bool backward, SweepArgs& args);
bool launch_level_sweep(rcg_ctx* ctx, const rcg_ic* f, bool backward, SweepArgs& args);   // icsweep_lv.cu
// memory-lean recycling step (recycle.cu): errors, MGS and the streamed Rayleigh-Ritz Gram in the
// sampler's slots; W is a new n x m~ block
void lean_build_aux(rcg_ctx* ctx, const rcg_matrix* a, const double* x_dev, rcg_sampler* s, double theta,
                    int keep_count, int* m_bar, std::vector<double>& vals, double* theta_used, rcg_tall** w_out);
// rcg_basis_create, optionally adopting w's column block (recycle.cu)
void basis_build(rcg_ctx* ctx, const rcg_matrix* a, rcg_tall* w, int who, bool adopt, rcg_basis** out);
SweepArgs sweep_args(rcg_ctx* ctx, const rcg_ic* f, bool backward);
void check_sweep_watchdog(rcg_ctx* ctx);
int64_t sweep_tiles(const rcg_ic* f);
void check_cfg(const rcg_solver_config* cfg);
void batch_ws_free(rcg_ctx* ctx);
void check_prec(const rcg_prec* m, int32_t n);

}  // namespace rcg
