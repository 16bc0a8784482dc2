// batch.cu -- batched multi-RHS PCG / SC-PCG / deflated PCG: R independent right-hand sides of
// one matrix solved by ONE kernel sequence (the sequence protocol's solves 2..k are independent
// given W, driver.cpp:181-195).  Vectors are stored interleaved, v[i*RT + k] (RT = 2 for R <= 2,
// else R rounded up to a multiple of 4; padding columns are zero right-hand sides, done before the first
// iteration).  Every RHS keeps its own alpha, beta, rho, relres, convergence flag and
// iteration count; converged RHS are frozen while the others continue.
//
// Why: the natural-ordering IC sweeps are bound by dependency latency (one L2 round trip per
// level), not bandwidth.  A batch carries RT values per row through the same waits, so a level
// costs about the same time and moves RT times the bytes; A, the IC schedule and W/AW are read
// once per iteration for all RHS.
//
// Arithmetic per RHS is the reference's (pcg.cpp:63-89, deflation.cpp:17-23,
// subspace_correction.cpp:47-57); SpMV and sweep rows are bitwise the single-RHS values; the
// dot products are deterministic tree reductions (run to run identical).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "internal.cuh"
#include "kernels.cuh"
#include "spmv_pipe.cuh"
#include "vec.cuh"

namespace rcg {

constexpr int kRMax = 24;
constexpr int kMaxRedB = 768;  // basis columns x right-hand sides (32 x 24)
constexpr int kDepChunkHost = 8;  // the sweeps' dependency chunk (icsweep.cu kDepChunk)
#ifndef RCG_TALLT_UNROLL
#define RCG_TALLT_UNROLL 8  // measured: 2 175 us, 4 150 us, 8 146 us (C2, RT 12)
#endif
constexpr int kTalltUnroll = RCG_TALLT_UNROLL;  // rows in flight per thread in k_b_tallt
constexpr int kElemThreads = 192;  // a multiple of every RT (2, 4, 8, 12, 16, 24): a thread keeps one rhs

struct BState {
    int iter;      // global iteration being executed (1-based)
    int nrun;      // right-hand sides still running
    int max_iter;
    int pad;
    double eps;
    int done[kRMax];
    int iters[kRMax];
    int status[kRMax];
    double bnorm[kRMax], rho[kRMax], rho_prev[kRMax], beta[kRMax], alpha[kRMax], pq[kRMax], rr[kRMax],
        relres[kRMax], scal2[kRMax];
    unsigned int tick[8];
    // row slabs (dist.cu): the reducing kernels' last block writes its local totals to dtot and
    // stops; the host allreduces them over the ranks and k_b_fin runs the same finaliser
    int defer;
    int pad2;
    double* dtot;
};

struct BatchWs {
    int64_t cap = 0;  // n * RT
    double *b = nullptr, *x = nullptr, *r = nullptr, *zs = nullptr, *p = nullptr, *q = nullptr, *y = nullptr;
    BState* st = nullptr;
    double* hist = nullptr;
    int64_t cap_hist = 0;
    double *u = nullptr, *u2 = nullptr;  // [m][RT]
    int64_t cap_u = 0;
    double* partials = nullptr;
    int64_t cap_part = 0;
    double* gpart = nullptr;
    unsigned int* gcount = nullptr;
    int64_t cap_groups = 0;
    double* tpart = nullptr;  // chunk-lane sweep tile partials
    int64_t cap_tpart = 0;
    int* tickets = nullptr;
};

static void free_ws(BatchWs*& w) {
    if (!w) return;
    for (void* p : {(void*)w->b, (void*)w->x, (void*)w->r, (void*)w->zs, (void*)w->p, (void*)w->q, (void*)w->y,
                    (void*)w->st, (void*)w->hist, (void*)w->u, (void*)w->u2, (void*)w->partials, (void*)w->gpart,
                    (void*)w->gcount, (void*)w->tpart, (void*)w->tickets})
        dev_free(p);
    delete w;
    w = nullptr;
}

void batch_ws_free(rcg_ctx* ctx) {
    free_ws(ctx->bws);
    free_ws(ctx->bws2);
}

// the workspace in `slot` (ctx->bws or ctx->bws2: a compacted phase reads one and writes the other)
static BatchWs& batch_ws(BatchWs*& slot, int64_t nrt, int64_t hist, int64_t m_rt, int64_t part, int64_t groups) {
    if (!slot) slot = new BatchWs();
    BatchWs& w = *slot;
    if (!w.st) {
        w.st = static_cast<BState*>(dev_alloc_bytes(sizeof(BState)));
        w.tickets = static_cast<int*>(dev_alloc_bytes(16 * sizeof(int)));
        RCG_CK(cudaMemset(w.tickets, 0, 16 * sizeof(int)));
        RCG_CK(cudaMemset(w.st, 0, sizeof(BState)));
    }
    if (nrt > w.cap) {
        for (double** v : {&w.b, &w.x, &w.r, &w.zs, &w.p, &w.q, &w.y}) {
            dev_free(*v);
            *v = dev_alloc(nrt);
        }
        w.cap = nrt;
    }
    if (hist > w.cap_hist) {
        dev_free(w.hist);
        w.hist = dev_alloc(hist);
        w.cap_hist = hist;
    }
    m_rt = std::max<int64_t>(m_rt, kRMax);
    if (m_rt > w.cap_u) {
        dev_free(w.u);
        dev_free(w.u2);
        w.u = dev_alloc(m_rt);
        w.u2 = dev_alloc(m_rt);
        w.cap_u = m_rt;
    }
    if (part > w.cap_part) {
        dev_free(w.partials);
        w.partials = dev_alloc(part);
        w.cap_part = part;
    }
    if (part > w.cap_tpart) {
        dev_free(w.tpart);
        w.tpart = dev_alloc(part);
        w.cap_tpart = part;
    }
    if (groups > w.cap_groups) {
        dev_free(w.gpart);
        dev_free(w.gcount);
        w.gpart = dev_alloc(groups * kRMax);
        w.gcount = static_cast<unsigned int*>(dev_alloc_bytes(sizeof(unsigned int) * groups));
        RCG_CK(cudaMemset(w.gcount, 0, sizeof(unsigned int) * groups));
        w.cap_groups = groups;
    }
    return w;
}

// slot k of a phase <-> slot[k] of the previous phase / original right-hand side col[k]
struct SlotMap {
    int cnt = 0;
    int slot[kRMax];
    int col[kRMax];
};

// ------------------------------------------------------------------ device helpers
// ------------------------------------------------------------------ kernels
template <int RT>
__global__ void k_b_gather(const double* __restrict__ cols, int R, int64_t ldc, double* __restrict__ out, int32_t n) {
    const int64_t total = static_cast<int64_t>(n) * RT;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / RT;
        const int k = static_cast<int>(e % RT);
        out[e] = k < R ? cols[k * ldc + i] : 0.0;
    }
}

template <int RT>
__global__ void k_b_scatter(const double* __restrict__ in, int R, int64_t ldc, double* __restrict__ cols, int32_t n) {
    const int64_t total = static_cast<int64_t>(n) * RT;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int k = static_cast<int>(e % RT);
        if (k < R) cols[k * ldc + e / RT] = in[e];
    }
}

// lane per row, RT interleaved vectors (each result bitwise the single-vector spmv)
template <int RT, class Body>
__device__ __forceinline__ void bspmv_rows(const SpmvArgs& a, const double* __restrict__ x, int cap, Body&& body) {
    csr_tiles(a.rs, a.ci, a.va, a.n, cap,
              [&](int32_t r0, int32_t my_b, int32_t my_e, const double* vsrc, const int32_t* csrc, int32_t off) {
                  const int32_t row = r0 + (threadIdx.x & 31);
                  double acc[RT];
#pragma unroll
                  for (int v = 0; v < RT; ++v) acc[v] = 0.0;
                  // gathers issued eight entries at a time so their latencies overlap
#pragma unroll 1
                  for (int32_t e = my_b; e < my_e; e += 8) {
                      const int m = min(8, my_e - e);
                      double av[8];
                      double2 xx[8][RT / 2];
#pragma unroll
                      for (int k = 0; k < 8; ++k)
                          if (k < m) {
                              av[k] = vsrc[e - off + k];
                              const double2* xv =
                                  reinterpret_cast<const double2*>(x + static_cast<int64_t>(csrc[e - off + k]) * RT);
#pragma unroll
                              for (int v = 0; v < RT / 2; ++v) xx[k][v] = __ldg(xv + v);
                          }
#pragma unroll
                      for (int k = 0; k < 8; ++k)
                          if (k < m)
#pragma unroll
                              for (int v = 0; v < RT / 2; ++v) {
                                  acc[2 * v] = fadd_mul(acc[2 * v], av[k], xx[k][v].x);
                                  acc[2 * v + 1] = fadd_mul(acc[2 * v + 1], av[k], xx[k][v].y);
                              }
                  }
                  if (row < a.n) body(row, acc);
              });
}

__device__ __forceinline__ void ldg4(const double* p, double* v) {
    asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
}

// RT % 4 == 0: G = RT/4 lanes per row, each carrying one 32-byte chunk of the row's values, so
// a warp's gather instruction reads whole chunks of consecutive rows (for stencil rows: one
// contiguous run) instead of one 16-byte piece per row.  Items of a 32-row tile are (row,
// chunk) pairs, row-major; every value's sum runs over the row's entries in CSR order, so each
// result is bitwise the single-vector spmv.  body(row, chunk, acc[4]).
#ifndef RCG_BGATHER
#define RCG_BGATHER 4
#endif
constexpr int kBGather = RCG_BGATHER;  // x chunks in flight per lane (RT = 4)
#ifndef RCG_BSPMV_WIDE_BLOCKS
#define RCG_BSPMV_WIDE_BLOCKS 3
#endif
// resident CTAs per SM of the batched SpMV kernels (register cap via __launch_bounds__, and the
// grid): RT >= 8 measured faster with one more CTA per SM than the single-vector SpMV's two
constexpr int bspmv_min_blocks(int rt) { return rt >= 8 ? RCG_BSPMV_WIDE_BLOCKS : 2; }

template <int RT, class Body>
__device__ __forceinline__ void bspmv_chunks(const SpmvArgs& a, const double* __restrict__ x, int cap, Body&& body) {
    constexpr int G = RT / 4;
    // lane -> (row, chunk) with a FIXED chunk per lane (c = lane % G): 32 / G rows per pass, the
    // lanes beyond (32 / G) G idle (2 of 32 at G = 3 and 6) -- so a thread's per-rhs sums need
    // only its own chunk's 4 accumulators, not all RT (RT 24 spilled with RT accumulators)
    constexpr int RPP = 32 / G;                   // rows per pass
    constexpr int NPASS = (32 + RPP - 1) / RPP;   // passes per 32-row tile
    const int lane = threadIdx.x & 31;
    csr_tiles(a.rs, a.ci, a.va, a.n, cap,
              [&](int32_t r0, int32_t my_b, int32_t my_e, const double* vsrc, const int32_t* csrc, int32_t off) {
#pragma unroll 1
                  for (int pass = 0; pass < NPASS; ++pass) {
                      const int rit = pass * RPP + lane / G;  // row within the tile
                      const bool lane_on = lane < RPP * G && rit < 32;
                      const int32_t row = r0 + rit;
                      const int c = lane % G;
                      const int32_t b = __shfl_sync(0xffffffffu, my_b, rit & 31);
                      const int32_t e = __shfl_sync(0xffffffffu, my_e, rit & 31);
                      if (lane_on && row < a.n) {
                          double acc[4] = {0.0, 0.0, 0.0, 0.0};
                          if constexpr (RT <= 4) {
                              // one chunk per row: gathers issued kBGather entries at a time
#pragma unroll 1
                              for (int32_t k = b; k < e; k += kBGather) {
                                  const int m = min(kBGather, e - k);
                                  double av[kBGather], xv[kBGather][4];
#pragma unroll
                                  for (int j = 0; j < kBGather; ++j)
                                      if (j < m) {
                                          av[j] = vsrc[k + j - off];
                                          ldg4(x + static_cast<int64_t>(csrc[k + j - off]) * RT + 4 * c, xv[j]);
                                      }
#pragma unroll
                                  for (int j = 0; j < kBGather; ++j)
                                      if (j < m)
#pragma unroll
                                          for (int i = 0; i < 4; ++i) acc[i] = fadd_mul(acc[i], av[j], xv[j][i]);
                              }
                          } else {
                              // wider rows: two gathers in flight keeps the register budget of three CTAs
                              // per SM (more in flight per lane measured slower than more resident warps)
                              int32_t k = b;
                              for (; k + 1 < e; k += 2) {
                                  const double a0 = vsrc[k - off], a1 = vsrc[k + 1 - off];
                                  double x0[4], x1[4];
                                  ldg4(x + static_cast<int64_t>(csrc[k - off]) * RT + 4 * c, x0);
                                  ldg4(x + static_cast<int64_t>(csrc[k + 1 - off]) * RT + 4 * c, x1);
#pragma unroll
                                  for (int i = 0; i < 4; ++i) acc[i] = fadd_mul(fadd_mul(acc[i], a0, x0[i]), a1, x1[i]);
                              }
                              if (k < e) {
                                  const double a0 = vsrc[k - off];
                                  double x0[4];
                                  ldg4(x + static_cast<int64_t>(csrc[k - off]) * RT + 4 * c, x0);
#pragma unroll
                                  for (int i = 0; i < 4; ++i) acc[i] = fadd_mul(acc[i], a0, x0[i]);
                              }
                          }
                          body(row, c, acc);
                      }
                  }
              });
}

// per-thread per-rhs accumulator update for chunk c (c is lane-dependent; unrolled select)
template <int RT, class F>
__device__ __forceinline__ void chunk_acc(double (&accs)[RT], int c, F&& f) {
#pragma unroll
    for (int cc = 0; cc < RT / 4; ++cc)
        if (cc == c)
#pragma unroll
            for (int i = 0; i < 4; ++i) accs[4 * cc + i] = f(accs[4 * cc + i], i);
}

// ---- finalisers (per right-hand side k, from the summed totals): run by the reducing kernel's
// last block, or -- row slabs -- by k_b_fin after the totals were allreduced over the ranks
template <int RT>
__device__ __forceinline__ void fin_resid(BState* st, const double* tot, int k, int defer_check) {
    st->bnorm[k] = sqrt(tot[k]);
    st->rr[k] = tot[RT + k];
    st->rho[k] = tot[RT + k];
    if (st->bnorm[k] == 0.0)
        st->done[k] = kZeroRhs;
    else if (!defer_check && sqrt(tot[RT + k]) <= st->eps * st->bnorm[k])
        st->done[k] = kConverged;
    else
        st->done[k] = kRunning;
}

__device__ __forceinline__ void fin_rho(BState* st, const double* tot, int k, int add_sc) {
    double rho = tot[k];
    if (st->done[k] == kRunning) {
        if (add_sc) rho = __dadd_rn(rho, st->scal2[k]);
        st->rho[k] = rho;
        if (rho <= 0.0) {
            st->done[k] = kBroken;
            st->status[k] = kBrkRz;
        }
        st->beta[k] = st->iter > 1 ? rho / st->rho_prev[k] : 0.0;
    }
}

__device__ __forceinline__ void fin_pq(BState* st, const double* tot, int k) {
    if (st->done[k] == kRunning) {
        st->pq[k] = tot[k];
        if (tot[k] <= 0.0) {
            st->done[k] = kBroken;
            st->status[k] = kBrkPAp;
        }
        st->alpha[k] = st->rho[k] / tot[k];
    }
}

__device__ __forceinline__ void fin_projcheck(BState* st, const double* tot, int k) {
    if (st->done[k] == kRunning) {
        st->rr[k] = tot[k];
        st->rho[k] = tot[k];
        if (sqrt(tot[k]) <= st->eps * st->bnorm[k]) st->done[k] = kConverged;
    }
}

// x, r update finaliser: threads k < RT, then thread 0 (after a block barrier) counts
template <int RT>
__device__ __forceinline__ void fin_xr(BState* st, const double* tot, double* hist, int64_t hist_ld, int identity) {
    if (threadIdx.x < RT) {
        const int k = threadIdx.x;
        const int i = st->iter;
        if (st->done[k] == kRunning) {
            const double relres = sqrt(tot[k]) / st->bnorm[k];
            st->rr[k] = tot[k];
            st->relres[k] = relres;
            st->iters[k] = i;
            hist[k * hist_ld + (i - 1)] = relres;
            hist[(RT + k) * hist_ld + (i - 1)] = st->alpha[k];
            hist[(2 * RT + k) * hist_ld + (i - 1)] = st->beta[k];
            st->rho_prev[k] = st->rho[k];
            if (relres <= st->eps) {
                st->done[k] = kConverged;
            } else if (i >= st->max_iter) {
                st->done[k] = kCapped;
            } else if (identity) {
                st->rho[k] = tot[k];
                if (tot[k] <= 0.0) {
                    st->done[k] = kBroken;
                    st->status[k] = kBrkRz;
                }
                st->beta[k] = tot[k] / st->rho_prev[k];
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int c = 0;
        for (int k = 0; k < RT; ++k) c += st->done[k] == kRunning;
        st->nrun = c;
        st->iter = st->iter + 1;
    }
}

// u[:,k] = (W^T A W)^-1 f[:,k] (one warp per rhs), and f.u per rhs when mode == 2
template <int RT>
__device__ __forceinline__ void fin_tallt(BState* st, const double* tot, const double* L, int m, double* u, int mode,
                                          double (*fk)[128], double (*sol)[128]) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int k = wid; k < RT; k += blockDim.x >> 5) {
        for (int j = lane; j < m; j += 32) fk[wid][j] = tot[j * RT + k];
        __syncwarp();
        double* uk = sol[wid];
        warp_chol_solve(L, m, fk[wid], uk, uk);
        __syncwarp();
        for (int j = lane; j < m; j += 32) u[j * RT + k] = uk[j];
        if (mode == 2 && lane == 0) {
            double fu = 0.0;
            for (int j = 0; j < m; ++j) fu = fadd_mul(fu, fk[wid][j], uk[j]);
            st->scal2[k] = fu;
        }
        __syncwarp();
    }
}

// r = b - A x for all RT; finaliser: bnorm, rho = rr, already-converged / zero-rhs flags
template <int RT>
__global__ void __launch_bounds__(kSpmvThreads, bspmv_min_blocks(RT)) k_b_residual(SpmvArgs a, int cap, const double* __restrict__ b,
                                                             const double* __restrict__ x, double* __restrict__ r,
                                                             BState* st, double* partials, int defer_check) {
    __shared__ double scratch[2 * RT * 32];
    __shared__ double vals[2 * RT];
    __shared__ double tot[2 * RT];
    double bb[RT], rr[RT];
#pragma unroll
    for (int v = 0; v < RT; ++v) bb[v] = rr[v] = 0.0;
    if constexpr (RT % 4 == 0) {
        double bb4[4] = {0.0, 0.0, 0.0, 0.0}, rr4[4] = {0.0, 0.0, 0.0, 0.0};  // this lane's chunk
        bspmv_chunks<RT>(a, x, cap, [&](int32_t row, int c, const double (&acc)[4]) {
            const int64_t o = static_cast<int64_t>(row) * RT + 4 * c;
            double bi[4], ri[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                bi[i] = b[o + i];
                ri[i] = __dsub_rn(bi[i], acc[i]);
                r[o + i] = ri[i];
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                bb4[i] = fadd_mul(bb4[i], bi[i], bi[i]);
                rr4[i] = fadd_mul(rr4[i], ri[i], ri[i]);
            }
        });
        const int c = (threadIdx.x & 31) % (RT / 4);
        chunk_acc<RT>(bb, c, [&](double s, int i) { return __dadd_rn(s, bb4[i]); });
        chunk_acc<RT>(rr, c, [&](double s, int i) { return __dadd_rn(s, rr4[i]); });
    } else {
        bspmv_rows<RT>(a, x, cap, [&](int32_t row, const double (&acc)[RT]) {
#pragma unroll
            for (int v = 0; v < RT; ++v) {
                const double bi = b[static_cast<int64_t>(row) * RT + v];
                const double ri = __dsub_rn(bi, acc[v]);
                r[static_cast<int64_t>(row) * RT + v] = ri;
                bb[v] = fadd_mul(bb[v], bi, bi);
                rr[v] = fadd_mul(rr[v], ri, ri);
            }
        });
    }
    // block reduction of 2*RT per-thread values
    double accs[2 * RT];
#pragma unroll
    for (int v = 0; v < RT; ++v) {
        accs[v] = bb[v];
        accs[RT + v] = rr[v];
    }
    block_sum_dyn<2 * RT>(accs, 2 * RT, scratch, vals);
    if (grid_reduce_dyn(vals, 2 * RT, partials, &st->tick[0], tot)) {
        if (st->defer) {
            for (int t = threadIdx.x; t < 2 * RT; t += blockDim.x) st->dtot[t] = tot[t];
            return;
        }
        if (threadIdx.x < RT) fin_resid<RT>(st, tot, threadIdx.x, defer_check);
    }
}

__global__ void k_b_count(BState* st, int RT) {
    int c = 0;
    for (int k = 0; k < RT; ++k) c += st->done[k] == kRunning;
    st->nrun = c;
}

// 16- / 32-byte relaxed accesses of interleaved values (each value its own ready flag; a
// 32-byte access is one LDG/STG.E.ENL2.256 on sm_100a)
template <int VW>
struct RelVec;
template <>
struct RelVec<2> {
    static __device__ __forceinline__ void ld(const double* p, double* v) {
        asm volatile("ld.relaxed.gpu.global.v2.f64 {%0, %1}, [%2];" : "=d"(v[0]), "=d"(v[1]) : "l"(p) : "memory");
    }
    static __device__ __forceinline__ void st(double* p, const double* v) {
        asm volatile("st.relaxed.gpu.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v[0]), "d"(v[1]) : "memory");
    }
};
template <>
struct RelVec<4> {
    static __device__ __forceinline__ void ld(const double* p, double* v) {
        asm volatile("ld.relaxed.gpu.global.v4.f64 {%0, %1, %2, %3}, [%4];"
                     : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
                     : "l"(p)
                     : "memory");
    }
    static __device__ __forceinline__ void st(double* p, const double* v) {
        asm volatile("st.relaxed.gpu.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]),
                     "d"(v[3])
                     : "memory");
    }
};

// One sweep, lane per row carrying all RT values.  Tiles are 32 positions taken by a WARP from
// the ticket counter (not 128 per CTA as in the single sweep): a level's rows then spread over
// ~4x more SMs, so the burst of RT-wide reloads and stores when a level's parents publish is
// not concentrated on a few SMs' L2 ports.  Monotone tickets keep the schedule deadlock-free.
// Parents are loaded in chunks of CH entries (every value of a chunk in flight together) and
// the missing entries re-polled together; the row is published from inside the wait loop.
template <bool BWD, int RT>
__global__ void __launch_bounds__(128) k_b_sweep(SweepArgs a, BState* st) {
    constexpr int CH = RT <= 4 ? 8 : (RT <= 8 ? 4 : 3);
    constexpr int VW = RT % 4 == 0 ? 4 : 2;  // doubles per relaxed access (32 B beats 2 x 16 B)
    constexpr int NC = RT / VW;
    if (st->nrun == 0) return;
    const int lane = threadIdx.x & 31;
    const int ntiles = (a.npos + 31) / 32;
    while (true) {
        int tile = 0;
        if (lane == 0) tile = atomicAdd(&a.tickets[0], 1);
        tile = __shfl_sync(0xffffffffu, tile, 0);
        if (tile >= ntiles) break;
        const int pos = tile * 32 + lane;
        double contrib[RT];
#pragma unroll
        for (int v = 0; v < RT; ++v) contrib[v] = 0.0;
        const int32_t row = pos < a.npos ? __ldg(a.perm + pos) : -1;
        if (row >= 0) {
            const int64_t me = static_cast<int64_t>(row) * RT;
            const int32_t beg = __ldg(a.prs + pos), end = __ldg(a.prs + pos + 1);
            double s[RT];
            const double2* in2 = reinterpret_cast<const double2*>(a.in + me);
            const double dr = BWD ? __ldg(a.d + row) : 1.0;
#pragma unroll
            for (int v = 0; v < RT / 2; ++v) {
                const double2 t = in2[v];
                s[2 * v] = BWD ? __ddiv_rn(t.x, dr) : t.x;
                s[2 * v + 1] = BWD ? __ddiv_rn(t.y, dr) : t.y;
            }
            unsigned spins = 0;
            for (int32_t e0 = beg;; e0 += CH) {
                const int cnt = min(CH, end - e0);
                const bool last = e0 + CH >= end;
                int32_t col[CH];
                double val[CH];
                double dep[CH][RT];
#pragma unroll
                for (int j = 0; j < CH; ++j)
                    if (j < cnt) {
                        col[j] = __ldg(a.pcol + e0 + j);
                        val[j] = __ldg(a.pval + e0 + j);
                    }
#pragma unroll
                for (int j = 0; j < CH; ++j)
                    if (j < cnt)
#pragma unroll
                        for (int c = 0; c < NC; ++c) RelVec<VW>::ld(a.out + static_cast<int64_t>(col[j]) * RT + c * VW, &dep[j][c * VW]);
                while (true) {
                    bool miss[CH];
                    bool any = false;
#pragma unroll
                    for (int j = 0; j < CH; ++j) {
                        miss[j] = false;
                        if (j < cnt)
#pragma unroll
                            for (int v = 0; v < RT; ++v) miss[j] |= is_sentinel(dep[j][v]);
                        any |= miss[j];
                    }
                    if (!any) {
#pragma unroll
                        for (int j = 0; j < CH; ++j)
                            if (j < cnt)
#pragma unroll
                                for (int v = 0; v < RT; ++v) s[v] = fsub_mul(s[v], val[j], dep[j][v]);
                        if (last) {
                            double* o = a.out + me;
#pragma unroll
                            for (int c = 0; c < NC; ++c) {
                                double t[VW];
#pragma unroll
                                for (int i = 0; i < VW; ++i) t[i] = publishable(s[c * VW + i]);
                                RelVec<VW>::st(o + c * VW, t);
                            }
                        }
                        break;
                    }
                    if (a.backoff_ns) __nanosleep(a.backoff_ns);
                    // re-poll every chunk still missing (polling only a parent's last-published
                    // chunk first costs a second round trip per level once it arrives)
#pragma unroll
                    for (int j = 0; j < CH; ++j)
                        if (miss[j]) {
                            const double* pj = a.out + static_cast<int64_t>(col[j]) * RT;
#pragma unroll
                            for (int c = 0; c < NC; ++c) {
                                bool m = false;
#pragma unroll
                                for (int i = 0; i < VW; ++i) m |= is_sentinel(dep[j][c * VW + i]);
                                if (m) RelVec<VW>::ld(pj + c * VW, &dep[j][c * VW]);
                            }
                        }
                    if (++spins == (1u << 24)) {
                        atomicExch(&a.tickets[3], 1);
#pragma unroll
                        for (int j = 0; j < CH; ++j)
#pragma unroll
                            for (int v = 0; v < RT; ++v)
                                if (is_sentinel(dep[j][v])) dep[j][v] = 0.0;
                    }
                }
                if (last) break;
            }
            if (BWD && a.r) {
                const double2* r2 = reinterpret_cast<const double2*>(a.r + me);
#pragma unroll
                for (int v = 0; v < RT / 2; ++v) {
                    const double2 t = r2[v];
                    contrib[2 * v] = __dmul_rn(t.x, s[2 * v]);
                    contrib[2 * v + 1] = __dmul_rn(t.y, s[2 * v + 1]);
                }
            }
        }
        if (BWD && a.r) {
            // per-tile partials (RT values) -> groups of kGroup tiles -> total, fixed order
#pragma unroll
            for (int v = 0; v < RT; ++v) {
                const double t = warp_sum(contrib[v]);
                if (lane == v) a.partials[static_cast<int64_t>(tile) * RT + v] = t;
            }
            const int g = tile / kGroup;
            const int ngroups = (ntiles + kGroup - 1) / kGroup;
            const int gsize = min(kGroup, ntiles - g * kGroup);
            __threadfence();
            __syncwarp();
            int last_group = 0;
            if (lane == 0) last_group = atomicAdd(&a.gcount[g], 1u) == static_cast<unsigned>(gsize) - 1u;
            if (__shfl_sync(0xffffffffu, last_group, 0)) {
                __threadfence();
                if (lane < RT) {
                    double sg = 0.0;
                    for (int q = 0; q < gsize; ++q)
                        sg = __dadd_rn(sg, __ldcg(a.partials + static_cast<int64_t>(g * kGroup + q) * RT + lane));
                    a.gpart[static_cast<int64_t>(g) * RT + lane] = sg;
                }
                __threadfence();
                __syncwarp();
                int last = 0;
                if (lane == 0) {
                    a.gcount[g] = 0u;
                    last = atomicAdd(reinterpret_cast<unsigned int*>(&a.tickets[2]), 1u) ==
                           static_cast<unsigned>(ngroups) - 1u;
                }
                if (__shfl_sync(0xffffffffu, last, 0)) {
                    __threadfence();
                    if (lane < RT) {
                        double rho = 0.0;
                        for (int q = 0; q < ngroups; ++q)
                            rho = __dadd_rn(rho, __ldcg(a.gpart + static_cast<int64_t>(q) * RT + lane));
                        if (st->done[lane] == kRunning) {
                            if (a.add_sc) rho = __dadd_rn(rho, st->scal2[lane]);
                            st->rho[lane] = rho;
                            if (rho <= 0.0) {
                                st->done[lane] = kBroken;
                                st->status[lane] = kBrkRz;
                            }
                            st->beta[lane] = st->iter > 1 ? rho / st->rho_prev[lane] : 0.0;
                        }
                    }
                    if (lane == 0) a.tickets[2] = 0;
                }
            }
        }
    }
    if (lane == 0) {
        __threadfence();
        if (atomicAdd(&a.tickets[1], 1) == static_cast<int>(gridDim.x * (blockDim.x / 32)) - 1) {
            a.tickets[0] = 0;
            a.tickets[1] = 0;
        }
    }
}

// Chunk-lane sweep: right-hand sides are independent, so chunk c (values 2c, 2c+1) of a row
// depends only on chunk c of its parents.  A warp covers RPW = 32/G rows x G = RT/2 chunks, each
// lane sweeping its own 16-byte chunk exactly like the single-pair (RT = 2) sweep: per-lane work
// and polling stay those of RT = 2 whatever RT is, the row's values are published chunk by chunk
// with no coordination between lanes, and a level costs about what it costs at RT = 2.
#ifndef RCG_BSWEEPC_BWD_MINB
#define RCG_BSWEEPC_BWD_MINB 8  // (dev A/B: resident CTAs per SM the backward 16-byte-chunk sweep is compiled for)
#endif
template <bool BWD, int RT, int VW, int CH>
__global__ void __launch_bounds__(128, VW == 2 ? (BWD ? RCG_BSWEEPC_BWD_MINB : 8) : 6) k_b_sweepc(SweepArgs a, BState* st) {
    constexpr int G = RT / VW;
    constexpr int RPW = 32 / G;
    constexpr bool ORD = VW == 2;  // consume in order as parents arrive (measured: helps 16-byte chunks only)
    constexpr unsigned kFull = 0xffffffffu;
    if (st->nrun == 0) return;
    const int lane = threadIdx.x & 31;
    const int rl = lane / G, c = lane % G;
    const bool lane_on = rl < RPW;
    const int ntiles = (a.npos + RPW - 1) / RPW;
    const bool rho = BWD && a.r;
    // (measured and dropped: software-pipelining the tiles per warp -- ticket two tiles ahead, row
    // map and row data one tile ahead -- C3 RT 16 fwd / bwd 4.8 / 6.9 -> 5.5 / 8.8 ms, C2 RT 12 bwd
    // 0.66 -> 1.03 ms: rows taken early only spin on parents of later levels.)  The r chunk of
    // the (r, z) partial is requested with the row's input, not after the publish.
    // (measured and dropped, round 2, C3 RT 24 fwd / bwd ms per launch against 6.14 / 12.10:
    // prefetching the row's whole entry record (pcol / pval sectors) to L1 or L2 before the first
    // chunk 6.38 / 12.92; additionally requesting the parents past the first two chunks by
    // cp.async into shared memory before the wait on the newest ones (no destination registers)
    // -- / 19.4: the chain is not bound by the later chunks' round trips, and the extra requests
    // compete with the polling loads for the L2 ports.)
    auto take = [&]() {
        int t = 0;
        if (lane == 0) t = atomicAdd(&a.tickets[0], 1);
        return t;
    };
    while (true) {
        const int tile = __shfl_sync(kFull, take(), 0);
        if (tile >= ntiles) break;
        const int pos = tile * RPW + rl;
        const int32_t row = (lane_on && pos < a.npos) ? __ldg(a.perm + pos) : -1;
        double contrib[VW];
#pragma unroll
        for (int v = 0; v < VW; ++v) contrib[v] = 0.0;
        if (row >= 0) {
            const int64_t me = static_cast<int64_t>(row) * RT + VW * c;
            const int32_t beg = __ldg(a.prs + pos), end = __ldg(a.prs + pos + 1);
            double s[VW];
            double rr[BWD ? VW : 1];
            {
                const double dr = BWD ? __ldg(a.d + row) : 1.0;
#pragma unroll
                for (int v = 0; v < VW / 2; ++v) {
                    const double2 t = reinterpret_cast<const double2*>(a.in + me)[v];
                    s[2 * v] = BWD ? __ddiv_rn(t.x, dr) : t.x;
                    s[2 * v + 1] = BWD ? __ddiv_rn(t.y, dr) : t.y;
                }
            }
            if constexpr (BWD) {
                if (rho) {
#pragma unroll
                    for (int v = 0; v < VW / 2; ++v) {
                        const double2 t = reinterpret_cast<const double2*>(a.r + me)[v];
                        rr[2 * v] = t.x;
                        rr[2 * v + 1] = t.y;
                    }
                }
            }
            unsigned spins = 0;
            for (int32_t e0 = beg;; e0 += CH) {
                const int cnt = min(CH, end - e0);
                const bool last = e0 + CH >= end;
                int32_t col[CH];
                double val[CH];
                double dep[CH][VW];
#pragma unroll
                for (int j = 0; j < CH; ++j)
                    if (j < cnt) {
                        col[j] = __ldg(a.pcol + e0 + j);
                        val[j] = __ldg(a.pval + e0 + j);
                    }
#pragma unroll
                for (int j = 0; j < CH; ++j)
                    if (j < cnt) RelVec<VW>::ld(a.out + static_cast<int64_t>(col[j]) * RT + VW * c, dep[j]);
                int used = 0;
                while (true) {
                    if constexpr (ORD) {
#pragma unroll
                        for (int j = 0; j < CH; ++j)
                            if (j == used && j < cnt) {
                                bool m = false;
#pragma unroll
                                for (int v = 0; v < VW; ++v) m |= is_sentinel(dep[j][v]);
                                if (!m) {
#pragma unroll
                                    for (int v = 0; v < VW; ++v) s[v] = fsub_mul(s[v], val[j], dep[j][v]);
                                    used = j + 1;
                                }
                            }
                    } else {
                        bool any = false;
#pragma unroll
                        for (int j = 0; j < CH; ++j)
                            if (j < cnt)
#pragma unroll
                                for (int v = 0; v < VW; ++v) any |= is_sentinel(dep[j][v]);
                        if (!any) {
#pragma unroll
                            for (int j = 0; j < CH; ++j)
                                if (j < cnt)
#pragma unroll
                                    for (int v = 0; v < VW; ++v) s[v] = fsub_mul(s[v], val[j], dep[j][v]);
                            used = cnt;
                        }
                    }
                    if (used >= cnt) {
                        if (last) {
                            double t[VW];
#pragma unroll
                            for (int v = 0; v < VW; ++v) t[v] = publishable(s[v]);
                            RelVec<VW>::st(a.out + me, t);
                        }
                        break;
                    }
                    if (a.backoff_ns) __nanosleep(a.backoff_ns);
#pragma unroll
                    for (int j = 0; j < CH; ++j)
                        if (j >= used && j < cnt) {
                            bool m = false;
#pragma unroll
                            for (int v = 0; v < VW; ++v) m |= is_sentinel(dep[j][v]);
                            if (m) RelVec<VW>::ld(a.out + static_cast<int64_t>(col[j]) * RT + VW * c, dep[j]);
                        }
                    if (++spins == (1u << 24)) {
                        atomicExch(&a.tickets[3], 1);
#pragma unroll
                        for (int j = 0; j < CH; ++j)
#pragma unroll
                            for (int v = 0; v < VW; ++v)
                                if (is_sentinel(dep[j][v])) dep[j][v] = 0.0;
                    }
                }
                if (last) break;
            }
            if constexpr (BWD) {
                if (rho) {
#pragma unroll
                    for (int v = 0; v < VW; ++v) contrib[v] = __dmul_rn(rr[v], s[v]);
                }
            }
        }
        if (rho) {
            // per-tile partials: chunk c's RPW rows sit on lanes c, c+G, ..., summed in row order
            // (RPW-1 strided shuffles per value); k_b_rho sums the tiles in a fixed order
            double tot[VW];
#pragma unroll
            for (int v = 0; v < VW; ++v) tot[v] = contrib[v];
#pragma unroll
            for (int r = 1; r < RPW; ++r)
#pragma unroll
                for (int v = 0; v < VW; ++v) tot[v] = __dadd_rn(tot[v], __shfl_sync(kFull, contrib[v], c + r * G));
            if (lane < G)
#pragma unroll
                for (int v = 0; v < VW; ++v) a.partials[static_cast<int64_t>(tile) * RT + lane * VW + v] = tot[v];
        }
    }
    if (lane == 0) {
        __threadfence();
        if (atomicAdd(&a.tickets[1], 1) == static_cast<int>(gridDim.x * (blockDim.x / 32)) - 1) {
            a.tickets[0] = 0;
            a.tickets[1] = 0;
        }
    }
}

// (r, z) per rhs from the chunk-lane sweep's tile partials (tile-major, RT per tile): thread
// sums in a fixed stride (kElemThreads is a multiple of RT: fixed rhs per thread), block and grid
// reductions in a fixed order; finaliser as the sweep's: SC term, breakdown test, beta.
template <int RT>
__global__ void __launch_bounds__(kElemThreads) k_b_rho(const double* __restrict__ tpart, int64_t ntiles,
                                                       double* partials, BState* st, int add_sc) {
    __shared__ double sred[kElemThreads];
    __shared__ double vals[RT];
    __shared__ double tot[RT];
    if (st->nrun == 0) return;
    double acc = 0.0;
    const int64_t total = ntiles * RT;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(kElemThreads) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * kElemThreads)
        acc = __dadd_rn(acc, tpart[e]);
    sred[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x < RT) {
        double v = 0.0;
        for (int t = threadIdx.x; t < kElemThreads; t += RT) v = __dadd_rn(v, sred[t]);
        vals[threadIdx.x] = v;
    }
    __syncthreads();
    if (grid_reduce_dyn(vals, RT, partials, &st->tick[5], tot)) {
        if (st->defer) {
            if (threadIdx.x < RT) st->dtot[threadIdx.x] = tot[threadIdx.x];
            return;
        }
        if (threadIdx.x < RT) fin_rho(st, tot, threadIdx.x, add_sc);
    }
}


// One LEVEL of a batched sweep per launch (very wide levels: the multicolour orderings), the
// batched counterpart of icsweep_lv.cu.  Items are (position, chunk of VW right-hand sides); a
// thread keeps its chunk (kElemThreads % G == 0).  Parents belong to earlier levels (earlier
// launches): no polling.  Every value is k_b_sweepc's row arithmetic (bitwise); the (r, z)
// partials of a CTA are summed per rhs in thread order into tpart[tile][k] for k_b_rho.
template <bool BWD, int RT>
__global__ void __launch_bounds__(kElemThreads) k_b_level(SweepArgs a, BState* st, int32_t lstart, int32_t width,
                                                          double* __restrict__ tpart, int64_t tile_base) {
    constexpr int VW = RT % 4 == 0 ? 4 : 2;
    constexpr int G = RT / VW;
    __shared__ double red[kElemThreads * VW];
    if (st->nrun == 0) return;
    const int c = threadIdx.x % G;
    double acc[VW];
#pragma unroll
    for (int v = 0; v < VW; ++v) acc[v] = 0.0;
    const int64_t items = static_cast<int64_t>(width) * G;
    for (int64_t it = blockIdx.x * static_cast<int64_t>(kElemThreads) + threadIdx.x; it < items;
         it += static_cast<int64_t>(gridDim.x) * kElemThreads) {
        const int32_t pos = lstart + static_cast<int32_t>(it / G);
        const int32_t row = __ldg(a.perm + pos);
        if (row < 0) continue;
        const int64_t me = static_cast<int64_t>(row) * RT + c * VW;
        double sv[VW];
        double dr = 1.0;
        if (BWD) dr = __ldg(a.d + row);
#pragma unroll
        for (int v = 0; v < VW; ++v) sv[v] = BWD ? __ddiv_rn(a.in[me + v], dr) : a.in[me + v];
        const int32_t b = __ldg(a.prs + pos), e = __ldg(a.prs + pos + 1);
        for (int32_t k0 = b; k0 < e; k0 += 4) {  // four parents' chunks in flight, then in order
            const int mm = min(4, e - k0);
            double lv[4], dep[4][VW];
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (j < mm) {
                    lv[j] = __ldg(a.pval + k0 + j);
                    const double* src = a.out + static_cast<int64_t>(__ldg(a.pcol + k0 + j)) * RT + c * VW;
#pragma unroll
                    for (int v = 0; v < VW; ++v) dep[j][v] = __ldcg(src + v);
                }
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (j < mm)
#pragma unroll
                    for (int v = 0; v < VW; ++v) sv[v] = fsub_mul(sv[v], lv[j], dep[j][v]);
        }
#pragma unroll
        for (int v = 0; v < VW; ++v) {
            sv[v] = publishable(sv[v]);
            a.out[me + v] = sv[v];
            if (BWD && a.r) acc[v] = fadd_mul(acc[v], a.r[me + v], sv[v]);
        }
    }
    if (!(BWD && a.r)) return;
#pragma unroll
    for (int v = 0; v < VW; ++v) red[threadIdx.x * VW + v] = acc[v];
    __syncthreads();
    if (threadIdx.x < RT) {
        const int k = threadIdx.x, cc = k / VW, v = k % VW;
        double sum = 0.0;
        for (int t = cc; t < kElemThreads; t += G) sum = __dadd_rn(sum, red[t * VW + v]);
        tpart[(tile_base + blockIdx.x) * RT + k] = sum;
    }
}

// p = z (+ W u) (+ beta p) for running rhs; sweep buffers back to the sentinel.  G = RT/VW
// threads per row, each on one VW-value chunk: a warp's accesses are contiguous and each W_j[i]
// load serves VW values.  Per value the arithmetic of the single-rhs k_pupdate.
template <int RT>
__global__ void __launch_bounds__(256) k_b_pupdate(const double* __restrict__ z, double* __restrict__ p,
                                                   double* __restrict__ zs_reset, double* __restrict__ y_reset,
                                                   int32_t n, BState* st, const double* __restrict__ W, int64_t ldw,
                                                   int m, const double* __restrict__ u) {
    constexpr int VW = RT % 4 == 0 ? 4 : 2;
    constexpr int G = RT / VW;
    __shared__ double us[kMaxRedB];
    __shared__ double beta[RT];
    __shared__ int run[RT];
    if (st->nrun == 0) return;
    if (W)
        for (int t = threadIdx.x; t < m * RT; t += blockDim.x) us[t] = u[t];
    if (threadIdx.x < RT) {
        beta[threadIdx.x] = st->beta[threadIdx.x];
        run[threadIdx.x] = st->done[threadIdx.x] == kRunning;
    }
    const bool first = st->iter == 1;
    __syncthreads();
    const double sent = sentinel();
    const int64_t items = static_cast<int64_t>(n) * G;
    for (int64_t it = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; it < items;
         it += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = it / G;
        const int k0 = static_cast<int>(it % G) * VW;
        const int64_t e0 = it * VW;
        double zi[VW];
#pragma unroll
        for (int v = 0; v < VW / 2; ++v) {
            const double2 t = reinterpret_cast<const double2*>(z + e0)[v];
            zi[2 * v] = t.x;
            zi[2 * v + 1] = t.y;
        }
        if (W)
            for (int j0 = 0; j0 < m; j0 += 8) {  // eight column loads in flight, then the sums in order
                const int mm = min(8, m - j0);
                double wj[8];
#pragma unroll
                for (int t = 0; t < 8; ++t)
                    if (t < mm) wj[t] = __ldg(W + (j0 + t) * ldw + i);
#pragma unroll
                for (int t = 0; t < 8; ++t)
                    if (t < mm)
#pragma unroll
                        for (int v = 0; v < VW; ++v) zi[v] = fadd_mul(zi[v], us[(j0 + t) * RT + k0 + v], wj[t]);
            }
#pragma unroll
        for (int v = 0; v < VW; ++v)
            if (run[k0 + v]) p[e0 + v] = first ? zi[v] : fadd_mul(zi[v], beta[k0 + v], p[e0 + v]);
        if (zs_reset) {
#pragma unroll
            for (int v = 0; v < VW / 2; ++v) {
                reinterpret_cast<double2*>(zs_reset + e0)[v] = make_double2(sent, sent);
                reinterpret_cast<double2*>(y_reset + e0)[v] = make_double2(sent, sent);
            }
        }
    }
}

// q = A p (all RT), (p, q) per rhs -> alpha (unless the deflated path projects q first)
template <int RT>
__global__ void __launch_bounds__(kSpmvThreads, bspmv_min_blocks(RT)) k_b_spmv_pq(SpmvArgs a, int cap, const double* __restrict__ p,
                                                            double* __restrict__ q, BState* st, double* partials,
                                                            int project_later) {
    __shared__ double scratch[RT * 32];
    __shared__ double vals[RT];
    __shared__ double tot[RT];
    if (st->nrun == 0) return;
    double pq[RT];
#pragma unroll
    for (int v = 0; v < RT; ++v) pq[v] = 0.0;
    if constexpr (RT % 4 == 0) {
        double pq4[4] = {0.0, 0.0, 0.0, 0.0};  // this lane's fixed chunk (bspmv_chunks)
        bspmv_chunks<RT>(a, p, cap, [&](int32_t row, int c, const double (&acc)[4]) {
            const int64_t o = static_cast<int64_t>(row) * RT + 4 * c;
            double pi[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                q[o + i] = acc[i];
                pi[i] = p[o + i];
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) pq4[i] = fadd_mul(pq4[i], pi[i], acc[i]);
        });
        chunk_acc<RT>(pq, (threadIdx.x & 31) % (RT / 4), [&](double s, int i) { return __dadd_rn(s, pq4[i]); });
    } else {
        bspmv_rows<RT>(a, p, cap, [&](int32_t row, const double (&acc)[RT]) {
#pragma unroll
            for (int v = 0; v < RT; ++v) {
                q[static_cast<int64_t>(row) * RT + v] = acc[v];
                pq[v] = fadd_mul(pq[v], p[static_cast<int64_t>(row) * RT + v], acc[v]);
            }
        });
    }
    if (project_later) return;
    block_sum_dyn<RT>(pq, RT, scratch, vals);
    if (grid_reduce_dyn(vals, RT, partials, &st->tick[1], tot)) {
        if (st->defer) {
            if (threadIdx.x < RT) st->dtot[threadIdx.x] = tot[threadIdx.x];
            return;
        }
        if (threadIdx.x < RT) fin_pq(st, tot, threadIdx.x);
    }
}

// ---- stencil-grid batched SpMV (natural-ordered N^3 grids with the 7- or 27-point pattern: C1-C4).
// The generic gather path reads each p row (RT values) from L2 once per matrix entry that
// references it -- 27 times on C3, ~86 GB per RT-24 SpMV: L2-bound (~6,300 B/cycle).  Here a CTA
// owns TX consecutive rows of one x-line; the p rows of the 9 (27-point) or 5 (7-point) x-segments
// they touch are staged once into shared memory by cp.async.bulk (contiguous: RT-interleaved rows),
// and every gather is a shared-memory read.  Each (row, chunk) sums its row's entries in stored
// order from 0.0 with separate roundings -- bitwise the generic kernel's q; (p, q) per rhs is a
// fixed-order block + grid sum (the same finaliser).
__global__ void k_grid_check(const int32_t* __restrict__ rs, const int32_t* __restrict__ ci, int32_t N, int st,
                             int* __restrict__ bad) {
    const int64_t n = static_cast<int64_t>(N) * N * N;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int x = static_cast<int>(i % N), y = static_cast<int>((i / N) % N), z = static_cast<int>(i / (int64_t(N) * N));
        int32_t e = rs[i];
        const int32_t end = rs[i + 1];
        bool ok = true;
        for (int dz = -1; dz <= 1 && ok; ++dz)
            for (int dy = -1; dy <= 1 && ok; ++dy)
                for (int dx = -1; dx <= 1 && ok; ++dx) {
                    const int nd = (dx != 0) + (dy != 0) + (dz != 0);
                    if (st == 7 && nd > 1) continue;
                    if (x + dx < 0 || x + dx >= N || y + dy < 0 || y + dy >= N || z + dz < 0 || z + dz >= N) continue;
                    const int64_t j = i + dx + static_cast<int64_t>(N) * dy + static_cast<int64_t>(N) * N * dz;
                    if (e >= end || ci[e] != j) ok = false;
                    ++e;
                }
        if (!ok || e != end) atomicExch(bad, 1);
    }
}

constexpr int kGridSpmvThreads = 256;

template <int RT, int ST>
__global__ void __launch_bounds__(kGridSpmvThreads) k_b_spmv_grid(SpmvArgs a, int32_t N, const double* __restrict__ p,
                                                                  double* __restrict__ q, BState* st, double* partials,
                                                                  int project_later) {
    constexpr int G = RT / 4;
    constexpr int TX = kGridSpmvThreads / G;       // rows per tile
    constexpr int NSEG = ST == 27 ? 9 : 5;
    constexpr int SEGR = TX + 2;                   // staged rows per segment (x0-1 .. x0+TX)
    extern __shared__ __align__(16) unsigned char gsm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(gsm);
    double* seg = reinterpret_cast<double*>(gsm + 16);
    __shared__ double scratch[RT * 32];
    __shared__ double vals[RT];
    __shared__ double tot[RT];
    if (st->nrun == 0) return;
    const int tid = threadIdx.x;
    const int tiles_per_line = (N + TX - 1) / TX;
    const int64_t lines = static_cast<int64_t>(N) * N;
    const int64_t ntiles = lines * tiles_per_line;
    const int64_t N2 = static_cast<int64_t>(N) * N;
    if (tid == 0) {
        mbar_init(bar);
        fence_mbar_init();
    }
    __syncthreads();
    unsigned phase = 0;
    double pq4[4] = {0.0, 0.0, 0.0, 0.0};
    const int c = tid % G;
    const int rloc = tid / G;  // row within the tile (< TX when tid < TX G)
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t line = t / tiles_per_line;
        const int x0 = static_cast<int>(t % tiles_per_line) * TX;
        const int y = static_cast<int>(line % N), z = static_cast<int>(line / N);
        const int xa = max(x0 - 1, 0), xb = min(x0 + TX, N - 1);  // staged x range [xa, xb]
        const int cnt = xb - xa + 1;
        // stage the segments (dy, dz): rows (xa..xb, y+dy, z+dz), RT values each
        if (tid == 0) {
            unsigned bytes = 0;
            for (int sidx = 0; sidx < NSEG; ++sidx) {
                int dy, dz;
                if (ST == 27) {
                    dz = sidx / 3 - 1;
                    dy = sidx % 3 - 1;
                } else {
                    const int o[5][2] = {{0, -1}, {-1, 0}, {0, 0}, {1, 0}, {0, 1}};  // (dy, dz)
                    dy = o[sidx][0];
                    dz = o[sidx][1];
                }
                if (y + dy < 0 || y + dy >= N || z + dz < 0 || z + dz >= N) continue;
                bytes += static_cast<unsigned>(cnt) * RT * 8u;
            }
            fence_proxy_async();  // the previous tile's generic reads of the segments precede these writes
            mbar_expect_tx(bar, bytes);
            for (int sidx = 0; sidx < NSEG; ++sidx) {
                int dy, dz;
                if (ST == 27) {
                    dz = sidx / 3 - 1;
                    dy = sidx % 3 - 1;
                } else {
                    const int o[5][2] = {{0, -1}, {-1, 0}, {0, 0}, {1, 0}, {0, 1}};
                    dy = o[sidx][0];
                    dz = o[sidx][1];
                }
                if (y + dy < 0 || y + dy >= N || z + dz < 0 || z + dz >= N) continue;
                const int64_t r0 = xa + static_cast<int64_t>(N) * (y + dy) + N2 * (z + dz);
                bulk_g2s(seg + static_cast<int64_t>(sidx) * SEGR * RT, p + r0 * RT, static_cast<unsigned>(cnt) * RT * 8u, bar);
            }
        }
        while (!mbar_try_wait(bar, phase)) {
        }
        phase ^= 1u;
        const int x = x0 + rloc;
        if (tid < TX * G && x < N) {
            const int64_t i = x + static_cast<int64_t>(N) * y + N2 * z;
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            const int32_t b = __ldg(a.rs + i), e = __ldg(a.rs + i + 1);
            for (int32_t k = b; k < e; ++k) {
                const int64_t j = __ldg(a.ci + k);
                const double av = __ldg(a.va + k);
                // j -> (dx, dy, dz) relative to i (each in -1..1, N >= 4: by comparisons, no
                // division) -> (segment, staged row); dxp = dx + 1 etc.
                int64_t d = j - i;
                const int dz = d < -(N2 >> 1) ? -1 : (d > (N2 >> 1) ? 1 : 0);
                d -= dz * N2;
                const int dy = d < -(N >> 1) ? -1 : (d > (N >> 1) ? 1 : 0);
                d -= static_cast<int64_t>(dy) * N;
                const int dzp = dz + 1, dyp = dy + 1, dxp = static_cast<int>(d) + 1;
                int sidx;
                if (ST == 27) {
                    sidx = dzp * 3 + dyp;
                } else {
                    sidx = dzp == 0 ? 0 : (dzp == 2 ? 4 : (dyp == 0 ? 1 : (dyp == 2 ? 3 : 2)));
                }
                const int xr = x + dxp - 1 - xa;
                const double* src = seg + (static_cast<int64_t>(sidx) * SEGR + xr) * RT + 4 * c;
                const double4 pv = *reinterpret_cast<const double4*>(src);
                acc[0] = fadd_mul(acc[0], av, pv.x);
                acc[1] = fadd_mul(acc[1], av, pv.y);
                acc[2] = fadd_mul(acc[2], av, pv.z);
                acc[3] = fadd_mul(acc[3], av, pv.w);
            }
            const int64_t o = i * RT + 4 * c;
            const double* pself = seg + (static_cast<int64_t>(ST == 27 ? 4 : 2) * SEGR + (x - xa)) * RT + 4 * c;
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                q[o + v] = acc[v];
                pq4[v] = fadd_mul(pq4[v], pself[v], acc[v]);
            }
        }
        __syncthreads();  // the staged segments are free for the next tile
    }
    if (project_later) return;
    double pq[RT];
#pragma unroll
    for (int v = 0; v < RT; ++v) pq[v] = 0.0;
    if (tid < TX * G) chunk_acc<RT>(pq, c, [&](double s, int v) { return __dadd_rn(s, pq4[v]); });
    block_sum_dyn<RT>(pq, RT, scratch, vals);
    if (grid_reduce_dyn(vals, RT, partials, &st->tick[1], tot)) {
        if (st->defer) {
            if (tid < RT) st->dtot[tid] = tot[tid];
            return;
        }
        if (tid < RT) fin_pq(st, tot, tid);
    }
}

template <int RT, int ST>
size_t grid_spmv_smem() {
    constexpr int TX = kGridSpmvThreads / (RT / 4);
    return 16 + static_cast<size_t>(ST == 27 ? 9 : 5) * (TX + 2) * RT * 8;
}

// the stencil of a matrix's pattern (cached): 7 / 27 for a natural-ordered N^3 box, else 0
static int grid_info(rcg_ctx* ctx, const rcg_matrix* a) {
    if (a->grid_st >= 0) return a->grid_st;
    a->grid_st = 0;
    // opt-in (RCG_GRID_SPMV=1): single-buffered staging measured slower than the generic gathers on
    // C3 at RT 24 (10.9 vs 9.1 ms: each tile waits for its 76 KB of segments)
    if (!(std::getenv("RCG_GRID_SPMV") && std::atoi(std::getenv("RCG_GRID_SPMV")) == 1)) return 0;
    const int64_t n = a->n;
    const int32_t N = static_cast<int32_t>(std::llround(std::cbrt(static_cast<double>(n))));
    if (N < 4 || static_cast<int64_t>(N) * N * N != n) return 0;
    int st = 0;
    if (a->nnz == 7 * n - 6LL * N * N) st = 7;
    else if (a->nnz == (3LL * N - 2) * (3LL * N - 2) * (3LL * N - 2)) st = 27;
    if (!st) return 0;
    int* bad = static_cast<int*>(dev_alloc_bytes(sizeof(int)));
    RCG_CK(cudaMemsetAsync(bad, 0, sizeof(int), ctx->stream));
    const int g = std::max(1, static_cast<int>(std::min<int64_t>((n + 255) / 256, ctx->num_sms * 8)));
    k_grid_check<<<g, 256, 0, ctx->stream>>>(a->rs, a->ci, N, st, bad);
    RCG_LAUNCHED(ctx);
    int h = 0;
    RCG_CK(cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    RCG_CK(cudaStreamSynchronize(ctx->stream));
    dev_free(bad);
    if (!h) {
        a->grid_st = st;
        a->gN = N;
    }
    return a->grid_st;
}

// f[j][k] = W_j . y_k for every (j, k).  Lane per row (each y row read as RT/2 16-byte loads,
// W_j[i] loads coalesced), JC columns x RT values in registers.  The m/JC column passes run as
// SIBLING CTAs over the same contiguous row range (consecutive block ids, so they are resident
// together and read the same y rows at about the same time: y comes from HBM about once, from L2
// for the siblings; W once).  Per output: thread partials, a fixed-order block sum, then the
// last CTA sums the row ranges in order.  Finaliser per rhs: u[:,k] = (W^T A W)^-1 f[:,k]
// (mode 1) and f.u (mode 2).  Host grid: X x P (BatchSolve::tgrid).
template <int RT>
__device__ __host__ constexpr int tallt_jc() {
    // columns per pass (m / JC sibling passes over the same rows): measured on C3 at RT 24, m 32:
    // JC 2 6.5 ms, JC 6 7.8 ms (3 CTAs per SM, y partly re-read from DRAM); RT 4 with 8 columns spilled
    return RT <= 8 ? 4 : 2;
}

template <int RT>
__global__ void __launch_bounds__(kElemThreads, RT <= 8 ? 4 : 6) k_b_tallt(const double* __restrict__ W, int64_t ldw, int m,
                                                            const double* __restrict__ y, int32_t n,
                                                            double* partials, const double* __restrict__ L,
                                                            double* __restrict__ u, int mode, BState* st,
                                                            int respect_done) {
    constexpr int JC = tallt_jc<RT>();
    constexpr int VW = RT % 4 == 0 ? 4 : 2;  // values per thread: G = RT/VW threads per row
    constexpr int G = RT / VW;
    __shared__ double scratch[kElemThreads * JC * (RT % 4 == 0 ? 4 : 2)];  // >= 2 x 6 x 128: fk / sol below
    __shared__ double tot[kMaxRedB];
    double (*fk)[128] = reinterpret_cast<double (*)[128]>(scratch);           // the finaliser's operands,
    double (*sol)[128] = reinterpret_cast<double (*)[128]>(scratch + 6 * 128);  // after the block sums
    __shared__ bool s_last;
    if (respect_done && st->nrun == 0) return;
    const int P = (m + JC - 1) / JC;
    const int X = gridDim.x / P;
    const int pc = blockIdx.x % P, x = blockIdx.x / P;
    const int j0 = pc * JC, mc = min(JC, m - j0);
    if (x < X) {
        const int32_t per = (n + X - 1) / X;
        const int32_t i0 = x * per, i1 = min(n, i0 + per);
        double acc[JC][VW];  // kElemThreads % G == 0: each thread keeps one chunk
#pragma unroll
        for (int jc = 0; jc < JC; ++jc)
#pragma unroll
            for (int v = 0; v < VW; ++v) acc[jc][v] = 0.0;
        const int64_t it1 = static_cast<int64_t>(i1) * G;
#pragma unroll kTalltUnroll
        for (int64_t it = static_cast<int64_t>(i0) * G + threadIdx.x; it < it1; it += kElemThreads) {
            const int64_t i = it / G;
            double yv[VW];
#pragma unroll
            for (int v = 0; v < VW / 2; ++v) {
                const double2 t = reinterpret_cast<const double2*>(y + it * VW)[v];
                yv[2 * v] = t.x;
                yv[2 * v + 1] = t.y;
            }
#pragma unroll
            for (int jc = 0; jc < JC; ++jc)
                if (jc < mc) {
                    const double wj = __ldg(W + (j0 + jc) * ldw + i);
#pragma unroll
                    for (int v = 0; v < VW; ++v) acc[jc][v] = fadd_mul(acc[jc][v], wj, yv[v]);
                }
        }
        {
            // block sum per output (jc, k): the threads of chunk c = k / VW in thread order (fixed),
            // through shared memory (a per-thread JC x RT array spills at RT <= 8, JC = 4)
#pragma unroll
            for (int jc = 0; jc < JC; ++jc)
#pragma unroll
                for (int v = 0; v < VW; ++v) scratch[threadIdx.x * (JC * VW) + jc * VW + v] = acc[jc][v];
            __syncthreads();
            for (int o = threadIdx.x; o < mc * RT; o += blockDim.x) {
                const int jc = o / RT, k = o % RT, cc = k / VW, v = k % VW;
                double sv = 0.0;
                for (int t = cc; t < kElemThreads; t += G) sv = __dadd_rn(sv, scratch[t * (JC * VW) + jc * VW + v]);
                partials[static_cast<int64_t>(j0 * RT + o) * X + x] = sv;
            }
        }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(&st->tick[2], 1u) == gridDim.x - 1u;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    {
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
        for (int o = wid; o < m * RT; o += nw) {
            double sv = 0.0;
            for (int xx = lane; xx < X; xx += 32) sv = __dadd_rn(sv, __ldcg(partials + static_cast<int64_t>(o) * X + xx));
            sv = warp_sum(sv);
            if (lane == 0) tot[o] = sv;
        }
        __syncthreads();
        if (threadIdx.x == 0) st->tick[2] = 0u;
    }
    if (st->defer) {
        for (int t = threadIdx.x; t < m * RT; t += blockDim.x) st->dtot[t] = tot[t];
        return;
    }
    fin_tallt<RT>(st, tot, L, m, u, mode, fk, sol);
}

// f[j][k] = W_j . y_k, register-blocked (RT a multiple of 4, m <= 128): the CTA stages a tile of
// kWtyRows rows of W (m columns) and of y (RT values per row) in shared memory once, and each
// thread accumulates a 4 (columns) x 4 (rhs) block of outputs over the tile rows of its row group
// -- 8 shared-memory loads per 16 multiply-adds, W and y read from HBM once.  (k_b_tallt's sibling
// passes re-read y m / 2 times and were bound by L1 / shared-memory traffic at RT 24: 6.5 ms on C3.)
// Determinism: each thread sums its rows in order (separate roundings), the row groups and the
// CTAs are combined in a fixed order; the finaliser is k_b_tallt's.
constexpr int kWtyThreads = 256;
constexpr int kWtyRows = 64;
constexpr int kWtyLd = kWtyRows + 2;  // padded W-tile row (16-byte multiple for the bulk copies); a thread's columns
                                     // are jb, jb + JB, ...: the warp's ~6 consecutive jb fall in distinct banks

template <int RT>
__global__ void __launch_bounds__(kWtyThreads) k_b_wty(const double* __restrict__ W, int64_t ldw, int m,
                                                        const double* __restrict__ y, int32_t n, double* partials,
                                                        const double* __restrict__ L, double* __restrict__ u, int mode,
                                                        BState* st, int respect_done) {
    constexpr int KB = RT / 4;  // rhs blocks of 4
    extern __shared__ __align__(16) double wsm[];  // two stages of: [m][kWtyLd] W tile, [kWtyRows][RT] y tile
    __shared__ double tot[kMaxRedB];
    __shared__ double fk[kWtyThreads / 32][128];  // fin_tallt: one row per warp
    __shared__ double sol[kWtyThreads / 32][128];
    __shared__ bool s_last;
    if (respect_done && st->nrun == 0) return;
    const int JB = (m + 3) / 4;
    const int nblk = JB * KB;                         // 4 x 4 output blocks
    const int groups = max(1, kWtyThreads / nblk);    // row groups
    const int tid = threadIdx.x;
    const int blk = tid % nblk, grp = tid / nblk;
    const bool active = grp < groups && nblk <= kWtyThreads;
    const int jb = blk / KB, k0 = (blk % KB) * 4;  // columns jb + a JB, a = 0..3
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    // Two stages filled by the TMA bulk engine: one warp requests the NEXT tile (m column segments
    // of 512 bytes and the contiguous y tile, completion on the stage's mbarrier) before the
    // current one is summed -- the synchronous version stalled every tile on its own loads (ncu:
    // 2.0 TB/s at RT 24).  The ragged last tile is filled by plain loads.
    const int64_t ntile = (static_cast<int64_t>(n) + kWtyRows - 1) / kWtyRows;
    const int64_t w_d = (static_cast<int64_t>(m) * kWtyLd + 3) & ~int64_t(3);
    const int64_t stage_d = w_d + static_cast<int64_t>(kWtyRows) * RT;
    __shared__ uint64_t bar[2];
    if (tid == 0) {
        mbar_init(&bar[0]);
        mbar_init(&bar[1]);
        fence_mbar_init();
    }
    __syncthreads();
    const int lane_i = tid & 31;
    auto is_full = [&](int64_t t) { return (t + 1) * kWtyRows <= static_cast<int64_t>(n); };
    auto request = [&](int64_t t, int sidx) {  // warp 0
        double* ws = wsm + sidx * stage_d;
        const int64_t i0 = t * kWtyRows;
        if (lane_i == 0) mbar_expect_tx(&bar[sidx], static_cast<unsigned>(8 * (m * kWtyRows + kWtyRows * RT)));
        __syncwarp();
        for (int j = lane_i; j < m; j += 32) bulk_g2s(ws + j * kWtyLd, W + j * ldw + i0, kWtyRows * 8, &bar[sidx]);
        if (lane_i == 0) bulk_g2s(ws + w_d, y + i0 * RT, kWtyRows * RT * 8, &bar[sidx]);
    };
    if (blockIdx.x < ntile && is_full(blockIdx.x) && tid < 32) request(blockIdx.x, 0);
    int it = 0;
    for (int64_t t = blockIdx.x; t < ntile; t += gridDim.x, ++it) {
        const int sidx = it & 1;
        const int64_t i0 = t * kWtyRows;
        const int rows = static_cast<int>(min(static_cast<int64_t>(kWtyRows), static_cast<int64_t>(n) - i0));
        const int64_t tn = t + gridDim.x;
        if (tn < ntile && is_full(tn) && tid < 32) {
            fence_proxy_async();
            request(tn, sidx ^ 1);
        }
        double* ws = wsm + sidx * stage_d;
        double* ysm = ws + w_d;
        if (is_full(t)) {
            while (!mbar_try_wait(&bar[sidx], (it >> 1) & 1)) {
            }
        } else {
            for (int e = tid; e < m * kWtyRows; e += kWtyThreads) {
                const int j = e / kWtyRows, r = e % kWtyRows;
                ws[j * kWtyLd + r] = r < rows ? __ldg(W + j * ldw + i0 + r) : 0.0;
            }
            for (int e = tid; e < kWtyRows * RT; e += kWtyThreads) ysm[e] = e < rows * RT ? __ldg(y + i0 * RT + e) : 0.0;
            __syncthreads();
        }
        if (active)
            for (int r = grp; r < rows; r += groups) {
                double wv[4];
#pragma unroll
                for (int a = 0; a < 4; ++a) wv[a] = jb + a * JB < m ? ws[(jb + a * JB) * kWtyLd + r] : 0.0;
                const double4 yv = *reinterpret_cast<const double4*>(ysm + r * RT + k0);
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    acc[a][0] = fadd_mul(acc[a][0], wv[a], yv.x);
                    acc[a][1] = fadd_mul(acc[a][1], wv[a], yv.y);
                    acc[a][2] = fadd_mul(acc[a][2], wv[a], yv.z);
                    acc[a][3] = fadd_mul(acc[a][3], wv[a], yv.w);
                }
            }
        __syncthreads();
    }
    // row groups in order -> the CTA's partial of every output (wsm reused: [groups][m * RT])
    if (active)
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b)
                if (jb + a * JB < m) wsm[static_cast<int64_t>(grp) * m * RT + (jb + a * JB) * RT + k0 + b] = acc[a][b];
    __syncthreads();
    const int X = gridDim.x;
    for (int o = tid; o < m * RT; o += kWtyThreads) {
        double sv = 0.0;
        for (int g = 0; g < groups; ++g) sv = __dadd_rn(sv, wsm[static_cast<int64_t>(g) * m * RT + o]);
        partials[static_cast<int64_t>(o) * X + blockIdx.x] = sv;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(&st->tick[2], 1u) == gridDim.x - 1u;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    {
        const int lane = tid & 31, wid = tid >> 5, nw = kWtyThreads >> 5;
        for (int o = wid; o < m * RT; o += nw) {
            double sv = 0.0;
            for (int xx = lane; xx < X; xx += 32) sv = __dadd_rn(sv, __ldcg(partials + static_cast<int64_t>(o) * X + xx));
            sv = warp_sum(sv);
            if (lane == 0) tot[o] = sv;
        }
        __syncthreads();
        if (tid == 0) st->tick[2] = 0u;
    }
    if (st->defer) {
        for (int t = tid; t < m * RT; t += kWtyThreads) st->dtot[t] = tot[t];
        return;
    }
    fin_tallt<RT>(st, tot, L, m, u, mode, fk, sol);
}

template <int RT>
size_t wty_smem(int m) {
    const int nblk = ((m + 3) / 4) * (RT / 4);
    const int groups = std::max(1, kWtyThreads / nblk);
    const size_t tiles = 2 * (((static_cast<size_t>(m) * kWtyLd + 3) & ~size_t(3)) + static_cast<size_t>(kWtyRows) * RT);
    return sizeof(double) * std::max(tiles, static_cast<size_t>(groups) * m * RT);
}

// The finalisers of the reducing kernels from allreduced totals (row slabs): which = 0 residual
// (arg: defer_check), 1 rho (arg: add_sc), 2 (p, q), 3 projected-residual check, 4 x / r update
// (arg: identity), 5 the m x RT projection coefficients (arg: tallt mode), 6 the projection
// coefficients of W^T q TOGETHER with (p, q) of the projected q (one allreduce of m RT + RT values,
// SURVEY 8(e)): with f = W^T q = (A W)^T p and u = (W^T A W)^-1 f, (p, q - A W u) = (p, q) - f . u.
// `off` is where the totals start in dtot (a deferred check's totals wait behind the next
// reduction's); `guard` repeats the producing kernel's early exit (nothing ran, nothing to finalise).
template <int RT>
__global__ void __launch_bounds__(kElemThreads) k_b_fin(BState* st, int which, int arg, int guard, const double* L, int m,
                                                        double* u, double* hist, int64_t hist_ld, int off) {
    __shared__ double tot[kMaxRedB + kRMax];
    __shared__ double fk[6][128];
    __shared__ double sol[6][128];
    if (guard && st->nrun == 0) return;
    const int cnt = which == 0 ? 2 * RT : (which == 5 ? m * RT : (which == 6 ? m * RT + RT : RT));
    for (int t = threadIdx.x; t < cnt; t += blockDim.x) tot[t] = st->dtot[off + t];
    __syncthreads();
    switch (which) {
        case 0:
            if (threadIdx.x < RT) fin_resid<RT>(st, tot, threadIdx.x, arg);
            break;
        case 1:
            if (threadIdx.x < RT) fin_rho(st, tot, threadIdx.x, arg);
            break;
        case 2:
            if (threadIdx.x < RT) fin_pq(st, tot, threadIdx.x);
            break;
        case 3:
            if (threadIdx.x < RT) fin_projcheck(st, tot, threadIdx.x);
            break;
        case 4:
            fin_xr<RT>(st, tot, hist, hist_ld, arg);
            break;
        case 6: {
            fin_tallt<RT>(st, tot, L, m, u, arg, fk, sol);
            __syncthreads();  // u (global, written by this block's warps) is visible past the barrier
            if (threadIdx.x < RT) {
                const int k = threadIdx.x;
                double fu = 0.0;
                for (int j = 0; j < m; ++j) fu = fadd_mul(fu, tot[j * RT + k], u[j * RT + k]);
                tot[m * RT + k] = __dsub_rn(tot[m * RT + k], fu);
                fin_pq(st, tot + m * RT, k);
            }
            break;
        }
        default:
            fin_tallt<RT>(st, tot, L, m, u, arg, fk, sol);
            break;
    }
}

// row slabs: move a reducing kernel's local totals behind the next reduction's, so that one
// allreduce carries both (dtot[src .. src + cnt) -> dtot[dst ..))
__global__ void k_b_stash(BState* st, int src, int dst, int cnt) {
    for (int t = threadIdx.x; t < cnt; t += blockDim.x) st->dtot[dst + t] = st->dtot[src + t];
}

// y -= sum_j u[j][k] C_j (running rhs) with (p, y) -> alpha (mode 0) or the projected initial
// residual check (mode 1).  Chunked like k_b_pupdate: a thread carries VW consecutive values of
// one row (coalesced 16-byte accesses, the block's chunk index fixed because kElemThreads is a
// multiple of every G), u staged in shared memory (read as broadcasts: the m-loop is instruction-
// bound at m = 32 otherwise); each value's update runs over j in order (subtract_combination).
template <int RT>
__global__ void __launch_bounds__(kElemThreads, 2) k_b_deflate(double* __restrict__ y, const double* __restrict__ Cm,
                                                            int64_t ldc, int m, const double* __restrict__ u,
                                                            const double* __restrict__ p, int32_t n, double* partials,
                                                            BState* st, int mode) {
    constexpr int VW = RT % 4 == 0 ? 4 : 2;
    constexpr int G = RT / VW;
    __shared__ double us[kMaxRedB];
    __shared__ double scratch[32 * RT];
    __shared__ double vals[RT];
    __shared__ double tot[RT];
    __shared__ int run[RT];
    if (st->nrun == 0 && mode == 0) return;
    for (int t = threadIdx.x; t < m * RT; t += blockDim.x) us[t] = u[t];
    if (threadIdx.x < RT) run[threadIdx.x] = mode == 1 || st->done[threadIdx.x] == kRunning;
    __syncthreads();
    const int c = threadIdx.x % G;  // fixed chunk: kElemThreads % G == 0, grid stride too
    const int k0 = c * VW;
    double acc[VW];
#pragma unroll
    for (int v = 0; v < VW; ++v) acc[v] = 0.0;
    // blocks of DR rows x one chunk per item: the coefficients u[j][chunk] of four columns are
    // loaded from shared memory once per block (not once per row) and the DR rows' C_j values are
    // one 32-byte load per column -- shared-memory traffic / DR (it bound the kernel at RT 24)
    constexpr int DR = 4;
    const int64_t nblk = (static_cast<int64_t>(n) + DR - 1) / DR;
    const int64_t items = nblk * G;
    for (int64_t it = blockIdx.x * static_cast<int64_t>(kElemThreads) + threadIdx.x; it < items;
         it += static_cast<int64_t>(gridDim.x) * kElemThreads) {
        const int64_t i0 = (it / G) * DR;
        const int nr = static_cast<int>(min(static_cast<int64_t>(DR), static_cast<int64_t>(n) - i0));
        double yv[DR][VW];
#pragma unroll
        for (int r = 0; r < DR; ++r)
            if (r < nr)
#pragma unroll
                for (int v = 0; v < VW; ++v) yv[r][v] = y[(i0 + r) * RT + k0 + v];
        for (int j0 = 0; j0 < m; j0 += 4) {  // four columns' loads in flight, then the updates in j order
            const int mm = min(4, m - j0);
            double cj[4][DR], uj[4][VW];
#pragma unroll
            for (int t = 0; t < 4; ++t)
                if (t < mm) {
                    const double* col = Cm + (j0 + t) * ldc + i0;
                    if (nr == DR && (ldc & 1) == 0) {
                        // even ldc (32-row padded blocks; a row slab's ld is its row count) and
                        // i0 % 4 == 0: two aligned 16-byte loads
                        const double2 c01 = __ldg(reinterpret_cast<const double2*>(col));
                        const double2 c23 = __ldg(reinterpret_cast<const double2*>(col) + 1);
                        cj[t][0] = c01.x, cj[t][1] = c01.y, cj[t][2] = c23.x, cj[t][3] = c23.y;
                    } else {
#pragma unroll
                        for (int r = 0; r < DR; ++r) cj[t][r] = r < nr ? __ldg(col + r) : 0.0;
                    }
#pragma unroll
                    for (int v = 0; v < VW; ++v) uj[t][v] = us[(j0 + t) * RT + k0 + v];
                }
#pragma unroll
            for (int t = 0; t < 4; ++t)
                if (t < mm)
#pragma unroll
                    for (int r = 0; r < DR; ++r)
#pragma unroll
                        for (int v = 0; v < VW; ++v) yv[r][v] = fsub_mul(yv[r][v], uj[t][v], cj[t][r]);
        }
#pragma unroll
        for (int r = 0; r < DR; ++r) {
            if (r >= nr) break;
            const int64_t e0 = (i0 + r) * RT + k0;
            double pv[VW];
            if (mode == 0)
#pragma unroll
                for (int v = 0; v < VW; ++v) pv[v] = p[e0 + v];
#pragma unroll
            for (int v = 0; v < VW; ++v)
                if (run[k0 + v]) {
                    y[e0 + v] = yv[r][v];
                    acc[v] = mode == 0 ? fadd_mul(acc[v], pv[v], yv[r][v]) : fadd_mul(acc[v], yv[r][v], yv[r][v]);
                }
        }
    }
    double full[RT];  // this thread's chunk, zeros elsewhere (adding 0.0 is exact)
#pragma unroll
    for (int t = 0; t < RT; ++t) full[t] = 0.0;
#pragma unroll
    for (int cc = 0; cc < G; ++cc)
        if (cc == c)
#pragma unroll
            for (int v = 0; v < VW; ++v) full[cc * VW + v] = acc[v];
    block_sum_dyn<RT>(full, RT, scratch, vals);
    if (grid_reduce_dyn(vals, RT, partials, &st->tick[3], tot)) {
        if (st->defer) {
            if (threadIdx.x < RT) st->dtot[threadIdx.x] = tot[threadIdx.x];
            return;
        }
        if (threadIdx.x < RT) {
            if (mode == 0)
                fin_pq(st, tot, threadIdx.x);
            else
                fin_projcheck(st, tot, threadIdx.x);
        }
    }
}

// k_b_deflate with the operands staged by the TMA bulk engine (RT 16 / 24, m <= 48).  The
// register version keeps only ~8 KB per SM in flight (a warp's 16-byte C_j loads hit 5-6 distinct
// addresses; 146 registers, 2 CTAs per SM: ncu 2.4 TB/s at RT 24); here a CTA walks 64-row tiles,
// one elected warp requests the NEXT tile -- m column segments of 512 bytes, the y tile and the p
// tile, one cp.async.bulk each, completion on the stage's mbarrier -- while the CTA updates the
// current one out of shared memory: 40 KB per CTA in flight at m = 32, RT = 24.  A thread owns 4
// consecutive rows x one 4-value chunk (C_j and u_j are one 32-byte shared load each per 16
// updates); every value's update runs over j in order (subtract_combination), bitwise k_b_deflate.
constexpr int kDtRows = 64;
template <int RT>
constexpr int dt_threads() { return kDtRows / 4 * (RT / 4); }
template <int RT>
size_t dt_smem(int m, bool with_p) {
    return sizeof(double) * (static_cast<size_t>(m) * RT + 2 * (static_cast<size_t>(m) * kDtRows + kDtRows * RT * (with_p ? 2 : 1))) + 16;
}

template <int RT>
__global__ void __launch_bounds__(dt_threads<RT>()) k_b_deflate_t(double* __restrict__ y, const double* __restrict__ Cm,
                                                                  int64_t ldc, int m, const double* __restrict__ u,
                                                                  const double* __restrict__ p, int32_t n,
                                                                  double* partials, BState* st, int mode) {
    constexpr int G = RT / 4;
    constexpr int TR = kDtRows;
    extern __shared__ __align__(128) unsigned char dsm[];
    __shared__ double scratch[32 * RT];
    __shared__ double vals[RT];
    __shared__ double tot[RT];
    __shared__ int run[RT];
    if (st->nrun == 0 && mode == 0) return;
    const int tid = threadIdx.x, lane = tid & 31;
    double* us = reinterpret_cast<double*>(dsm);
    const int64_t ss = static_cast<int64_t>(m) * TR + TR * RT * (p ? 2 : 1);  // doubles per stage
    double* stage0 = us + static_cast<int64_t>(m) * RT;
    uint64_t* bar = reinterpret_cast<uint64_t*>(stage0 + 2 * ss);
    if (tid == 0) {
        mbar_init(&bar[0]);
        mbar_init(&bar[1]);
        fence_mbar_init();
    }
    for (int t = tid; t < m * RT; t += blockDim.x) us[t] = u[t];
    if (tid < RT) run[tid] = mode == 1 || st->done[tid] == kRunning;
    __syncthreads();
    const int64_t ntile = (static_cast<int64_t>(n) + TR - 1) / TR;
    const unsigned tile_bytes = static_cast<unsigned>(sizeof(double) * ss);
    auto is_full = [&](int64_t t) { return (t + 1) * TR <= static_cast<int64_t>(n); };
    auto issue = [&](int64_t t, int sidx) {  // warp 0: lane j requests column j (+ y, p by lanes 0, 1)
        double* C = stage0 + sidx * ss;
        const int64_t i0 = t * TR;
        if (lane == 0) mbar_expect_tx(&bar[sidx], tile_bytes);
        __syncwarp();
        for (int j = lane; j < m; j += 32) bulk_g2s(C + j * TR, Cm + j * ldc + i0, TR * 8, &bar[sidx]);
        if (lane == 0) bulk_g2s(C + m * TR, y + i0 * RT, TR * RT * 8, &bar[sidx]);
        if (lane == 1 && p) bulk_g2s(C + m * TR + TR * RT, p + i0 * RT, TR * RT * 8, &bar[sidx]);
    };
    const int rb = tid / G, c = tid % G, k0 = c * 4, r0 = rb * 4;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    int64_t t = blockIdx.x;
    if (t < ntile && is_full(t) && tid < 32) issue(t, 0);
    for (int k = 0; t < ntile; t += gridDim.x, ++k) {
        const int sidx = k & 1;
        const int64_t tn = t + gridDim.x;
        if (tn < ntile && is_full(tn) && tid < 32) {
            fence_proxy_async();  // the stage's generic reads of two tiles ago before the async writes
            issue(tn, sidx ^ 1);
        }
        double* C = stage0 + sidx * ss;
        double* ys = C + m * TR;
        double* ps = ys + TR * RT;
        const int64_t i0 = t * TR;
        if (is_full(t)) {
            while (!mbar_try_wait(&bar[sidx], (k >> 1) & 1)) {
            }
        } else {  // the ragged last tile: plain loads, zero padding
            const int rows = static_cast<int>(static_cast<int64_t>(n) - i0);
            for (int e = tid; e < m * TR; e += blockDim.x) {
                const int j = e / TR, r = e % TR;
                C[e] = r < rows ? __ldg(Cm + j * ldc + i0 + r) : 0.0;
            }
            for (int e = tid; e < TR * RT; e += blockDim.x) {
                ys[e] = e < rows * RT ? y[i0 * RT + e] : 0.0;
                if (p) ps[e] = e < rows * RT ? p[i0 * RT + e] : 0.0;
            }
            __syncthreads();
        }
        double yv[4][4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const double4 t4 = *reinterpret_cast<const double4*>(ys + (r0 + r) * RT + k0);
            yv[r][0] = t4.x, yv[r][1] = t4.y, yv[r][2] = t4.z, yv[r][3] = t4.w;
        }
#pragma unroll 4
        for (int j = 0; j < m; ++j) {
            const double4 cj4 = *reinterpret_cast<const double4*>(C + j * TR + r0);
            const double4 uj4 = *reinterpret_cast<const double4*>(us + j * RT + k0);
            const double cj[4] = {cj4.x, cj4.y, cj4.z, cj4.w};
            const double uj[4] = {uj4.x, uj4.y, uj4.z, uj4.w};
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int v = 0; v < 4; ++v) yv[r][v] = fsub_mul(yv[r][v], uj[v], cj[r]);
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            if (i0 + r0 + r >= static_cast<int64_t>(n)) break;
            const int64_t e0 = (i0 + r0 + r) * RT + k0;
            const double4 o4 = *reinterpret_cast<const double4*>(ys + (r0 + r) * RT + k0);
            const double old[4] = {o4.x, o4.y, o4.z, o4.w};
            double pv[4] = {0.0, 0.0, 0.0, 0.0};
            if (mode == 0) {
                const double4 p4 = *reinterpret_cast<const double4*>(ps + (r0 + r) * RT + k0);
                pv[0] = p4.x, pv[1] = p4.y, pv[2] = p4.z, pv[3] = p4.w;
            }
            double out[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                out[v] = run[k0 + v] ? yv[r][v] : old[v];
                if (run[k0 + v])
                    acc[v] = mode == 0 ? fadd_mul(acc[v], pv[v], yv[r][v]) : fadd_mul(acc[v], yv[r][v], yv[r][v]);
            }
            *reinterpret_cast<double4*>(y + e0) = make_double4(out[0], out[1], out[2], out[3]);
        }
        __syncthreads();  // the stage is free for the tile after next
    }
    double full[RT];  // this thread's chunk, zeros elsewhere (adding 0.0 is exact)
#pragma unroll
    for (int q = 0; q < RT; ++q) full[q] = 0.0;
#pragma unroll
    for (int cc = 0; cc < G; ++cc)
        if (cc == c)
#pragma unroll
            for (int v = 0; v < 4; ++v) full[cc * 4 + v] = acc[v];
    block_sum_dyn<RT>(full, RT, scratch, vals);
    if (grid_reduce_dyn(vals, RT, partials, &st->tick[3], tot)) {
        if (st->defer) {
            if (threadIdx.x < RT) st->dtot[threadIdx.x] = tot[threadIdx.x];
            return;
        }
        if (threadIdx.x < RT) {
            if (mode == 0)
                fin_pq(st, tot, threadIdx.x);
            else
                fin_projcheck(st, tot, threadIdx.x);
        }
    }
}

// x += alpha p, r -= alpha q for running rhs; relres, history, convergence.  Element-parallel
// (coalesced), each thread on one rhs; per-rhs sums over the block's threads in a fixed order.
template <int RT>
__global__ void __launch_bounds__(kElemThreads) k_b_xr(double* __restrict__ x, double* __restrict__ r,
                                                       const double* __restrict__ p, const double* __restrict__ q,
                                                       int32_t n, double* partials, BState* st,
                                                       double* __restrict__ hist, int64_t hist_ld, int identity) {
    __shared__ double sred[kElemThreads];
    __shared__ double vals[RT];
    __shared__ double tot[RT];
    if (st->nrun == 0) return;
    const int kk = threadIdx.x % RT;
    const bool run_k = st->done[kk] == kRunning;
    const double alpha = st->alpha[kk];
    double acc = 0.0;
    if (run_k) {
        const int64_t total = static_cast<int64_t>(n) * RT;
        for (int64_t e = blockIdx.x * static_cast<int64_t>(kElemThreads) + threadIdx.x; e < total;
             e += static_cast<int64_t>(gridDim.x) * kElemThreads) {
            x[e] = fadd_mul(x[e], alpha, p[e]);
            const double ri = fsub_mul(r[e], alpha, q[e]);
            r[e] = ri;
            acc = fadd_mul(acc, ri, ri);
        }
    }
    sred[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x < RT) {
        double v = 0.0;
        for (int t = threadIdx.x; t < kElemThreads; t += RT) v = __dadd_rn(v, sred[t]);
        vals[threadIdx.x] = v;
    }
    __syncthreads();
    if (grid_reduce_dyn(vals, RT, partials, &st->tick[4], tot)) {
        if (st->defer) {
            if (threadIdx.x < RT) st->dtot[threadIdx.x] = tot[threadIdx.x];
            return;
        }
        fin_xr<RT>(st, tot, hist, hist_ld, identity);
    }
}

// zero-rhs solutions; deflated recombination x = P x + W (W^T A W)^-1 W^T b per rhs
template <int RT>
__global__ void k_b_finish_combine(double* __restrict__ x, const double* __restrict__ Cm, int64_t ldc, int m,
                                   const double* __restrict__ u, int32_t n, const BState* st, int mode) {
    const int64_t total = static_cast<int64_t>(n) * RT;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int k = static_cast<int>(e % RT);
        const int d = st->done[k];
        if (mode == 2) {  // zero rhs -> x = 0
            if (d == kZeroRhs) x[e] = 0.0;
            continue;
        }
        if (d == kBroken || d == kZeroRhs || d == kRunning) continue;
        const int64_t i = e / RT;
        if (mode == 0) {  // x -= W u (project_p)
            double v = x[e];
            for (int j = 0; j < m; ++j) v = fsub_mul(v, u[j * RT + k], __ldg(Cm + j * ldc + i));
            x[e] = v;
        } else {  // x += 0 + sum_j u_j W_j (direct_component)
            double t = 0.0;
            for (int j = 0; j < m; ++j) t = fadd_mul(t, u[j * RT + k], __ldg(Cm + j * ldc + i));
            x[e] = __dadd_rn(x[e], t);
        }
    }
}

// ------------------------------------------------------------------ compaction
// Running right-hand sides of a wider phase continue in a narrower one: vectors x, r, p, b and
// the per-rhs state (scalars, residual history, the subspace-correction coefficients u2) move
// to slots 0..cnt-1; the remaining slots are inert zero right-hand sides.
__global__ void k_b_carry_vec(const double* __restrict__ in, int rt_in, double* __restrict__ out, int rt_out,
                              SlotMap sel, int32_t n) {
    const int64_t total = static_cast<int64_t>(n) * rt_out;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / rt_out;
        const int k = static_cast<int>(e % rt_out);
        out[e] = k < sel.cnt ? in[i * rt_in + sel.slot[k]] : 0.0;
    }
}

__global__ void k_b_carry_state(const BState* __restrict__ a, BState* __restrict__ b, SlotMap sel, int rt_out,
                                const double* __restrict__ hist_a, double* __restrict__ hist_b, int64_t hist_ld,
                                const double* __restrict__ u2a, int rt_in, double* __restrict__ u2b, int m) {
    const int t = threadIdx.x;
    if (t == 0) {
        b->iter = a->iter;
        b->max_iter = a->max_iter;
        b->eps = a->eps;
        b->nrun = sel.cnt;
        for (int j = 0; j < 8; ++j) b->tick[j] = 0u;
        b->defer = a->defer;
        b->dtot = a->dtot;
    }
    if (t < rt_out) {
        if (t < sel.cnt) {
            const int s = sel.slot[t];
            b->done[t] = a->done[s];
            b->iters[t] = a->iters[s];
            b->status[t] = a->status[s];
            b->bnorm[t] = a->bnorm[s];
            b->rho[t] = a->rho[s];
            b->rho_prev[t] = a->rho_prev[s];
            b->beta[t] = a->beta[s];
            b->alpha[t] = a->alpha[s];
            b->pq[t] = a->pq[s];
            b->rr[t] = a->rr[s];
            b->relres[t] = a->relres[s];
            b->scal2[t] = a->scal2[s];
        } else {
            b->done[t] = kZeroRhs;
            b->iters[t] = 0;
            b->status[t] = 0;
            b->bnorm[t] = 0.0;
            b->rho[t] = b->rho_prev[t] = b->beta[t] = b->alpha[t] = b->pq[t] = b->rr[t] = b->relres[t] = 0.0;
            b->scal2[t] = 0.0;
        }
    }
    const int done_iters = a->iter - 1;
    for (int blk = 0; blk < 3; ++blk)  // relres, alpha, beta blocks
        for (int k = 0; k < sel.cnt; ++k)
            for (int i = t; i < done_iters; i += blockDim.x)
                hist_b[(blk * rt_out + k) * hist_ld + i] = hist_a[(blk * rt_in + sel.slot[k]) * hist_ld + i];
    for (int e = t; e < m * rt_out; e += blockDim.x) {
        const int j = e / rt_out, k = e % rt_out;
        u2b[e] = k < sel.cnt ? u2a[j * rt_in + sel.slot[k]] : 0.0;
    }
}

// x columns of the listed slots -> the caller's column-major X
__global__ void k_b_scatter_map(const double* __restrict__ in, int rt, SlotMap map, int64_t ldc,
                                double* __restrict__ cols, int32_t n) {
    const int64_t total = static_cast<int64_t>(n) * map.cnt;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int k = static_cast<int>(e % map.cnt);
        const int64_t i = e / map.cnt;
        cols[map.col[k] * ldc + i] = in[i * rt + map.slot[k]];
    }
}

// ------------------------------------------------------------------ host driver
// One solve of up to 16 right-hand sides, run in phases: a phase of width RT iterates until
// every slot is done or the running slots fit a narrower width (the converged ones stay frozen
// but still cost RT-wide passes), then retires its finished slots (deflated recombination,
// scatter to X, reports) and hands the running ones to the next, narrower phase.
struct BatchJob {
    rcg_ctx* ctx;
    const rcg_matrix* a;
    const rcg_prec* m;
    const rcg_basis* defl;
    int32_t n;
    int R;
    int max_iter;
    double eps;
    const double* b_cols;  // device, column-major (ld n)
    double* x_cols;        // device, column-major (ld n)
    rcg_solve_report* reps;
    double wall = 0.0;
    int broken = -1;
    int broken_status = 0;
    int phases = 0;
    BatchComm* comm = nullptr;  // row slabs (dist.cu): halo exchange + allreduced reductions
};

// RT: 2 for one or two right-hand sides, a multiple of 4 up to 16, else 24 (a multiple of the
// 4-value chunks and of kElemThreads' per-row thread groups)
static int pick_rt(int nrhs) { return nrhs <= 2 ? 2 : (nrhs <= 16 ? (nrhs + 3) / 4 * 4 : 24); }

template <int RT>
struct BatchSolve {
    BatchJob& job;
    rcg_ctx* ctx;
    const rcg_matrix* a;
    const rcg_prec* m;
    const rcg_basis* defl;
    int32_t n;
    int max_iter;
    double eps;
    bool ic = false, sc = false;
    const rcg_basis* scb = nullptr;
    BatchWs* w = nullptr;
    int sg = 1, pg = 1;
    int bcap = 256;  // batched SpMV stage capacity (entries per warp tile)
    int eg = 1;  // element-parallel grid (kElemThreads)
    int start_iter = 1;
    SlotMap map;  // slot k <-> original right-hand side map.col[k]

    explicit BatchSolve(BatchJob& j)
        : job(j), ctx(j.ctx), a(j.a), m(j.m), defl(j.defl), n(j.n), max_iter(j.max_iter), eps(j.eps) {}

    void setup(BatchWs*& slot) {
        ic = m->kind == RCG_PREC_IC || (m->kind == RCG_PREC_SC && m->ic);
        sc = m->kind == RCG_PREC_SC && m->sc && m->sc->k > 0;
        scb = sc ? m->sc : nullptr;
        int mm = 1;
        if (sc) mm = std::max(mm, scb->k);
        if (defl) mm = std::max(mm, defl->k);
        require(mm * RT <= kMaxRedB, "batch: basis columns x right-hand sides exceed the reduction capacity");
        require(mm <= 128, "batch: at most 128 basis columns");
        // row slabs: every interleaved vector carries the halo rows after the owned ones (p's are
        // filled by the exchange before each SpMV, x's before the initial residual)
        const int64_t nrt = (static_cast<int64_t>(n) + (job.comm ? job.comm->nhalo : 0)) * RT;
        // sweep tiles: the chunk-lane sweeps take RPW = 32 / (RT / 2) rows per warp tile (2 at RT 24)
        constexpr int kRpw = 32 / (RT / 2);
        int64_t ntiles = ic ? (std::max<int64_t>(std::max(m->ic->f_npos, m->ic->b_npos), n) + kRpw - 1) / kRpw : 1;
        const int64_t groups = (ntiles + kGroup - 1) / kGroup;
        const int64_t part = std::max<int64_t>(ntiles * RT, static_cast<int64_t>(kMaxRedB) * ctx->num_sms * 8);
        // history: relres, alpha, beta blocks of RT rows each (the CG coefficients feed the Lanczos estimate)
        w = &batch_ws(slot, nrt, 3 * static_cast<int64_t>(RT) * (max_iter + 1), static_cast<int64_t>(mm) * RT, part,
                      groups);
        sg = stream_grid(ctx, n);
        pg = spmv_grid(ctx, n);
        // The batched SpMV hides its RT-wide gathers with resident warps and L1: a matrix whose
        // widest tile needs a big stage (C3's 27-point rows: ~900 entries -> 1 CTA per SM, no L1,
        // 12 % of HBM) keeps a small stage (wider tiles read global memory through L1) instead.
        // RCG_BSPMV_CAP overrides.
        {
            static const int env_cap = [] {
                const char* e = std::getenv("RCG_BSPMV_CAP");
                return e ? std::atoi(e) : 0;
            }();
            // measured (C3 / C5, RT 12): cap 896 12.1 / 3.5 ms, 384 7.5 / 2.0 ms, 128 4.1 / 1.46 ms --
            // the L1 left to the gathers matters more than staging wide tiles
            bcap = env_cap > 0 ? env_cap : (a->cap <= 256 ? a->cap : 128);
        }
        if (bspmv_min_blocks(RT) > 2) {  // wider rows: one more resident CTA per SM (RT 12: 272 -> 210 us)
            const int blocks = ((n + 31) / 32 + kPipeWarps - 1) / kPipeWarps;
            pg = std::max(1, std::min(blocks, ctx->num_sms * (ctx->spmv_bps + bspmv_min_blocks(RT) - 2)));
        }
        eg = static_cast<int>(std::max<int64_t>(
            1, std::min<int64_t>((nrt + kElemThreads * 4 - 1) / (kElemThreads * 4), ctx->num_sms * 8)));
        static bool prepared = false;
        if (!prepared) {
            allow_smem(reinterpret_cast<const void*>(k_b_residual<RT>));
            allow_smem(reinterpret_cast<const void*>(k_b_spmv_pq<RT>));
            prepared = true;
        }
    }

    // first phase: right-hand sides 0..R-1 in slots 0..R-1
    void fresh() {
        map.cnt = job.R;
        for (int k = 0; k < job.R; ++k) map.slot[k] = map.col[k] = k;
        const int g = stream_grid(ctx, static_cast<int64_t>(n) * RT);
        k_b_gather<RT><<<g, kStreamThreads, 0, ctx->stream>>>(job.b_cols, job.R, n, w->b, n);
        RCG_LAUNCHED(ctx);
        k_b_gather<RT><<<g, kStreamThreads, 0, ctx->stream>>>(job.x_cols, job.R, n, w->x, n);
        RCG_LAUNCHED(ctx);
        initial();
        start_iter = 1;
    }

    // later phase: the running slots `sel` of a wider phase (state after a whole iteration)
    void resume(const BatchWs* from, int rt_from, const SlotMap& sel, int iter) {
        map.cnt = sel.cnt;
        for (int k = 0; k < sel.cnt; ++k) {
            map.slot[k] = k;
            map.col[k] = sel.col[k];
        }
        const int64_t nrt = static_cast<int64_t>(n) * RT;
        if (ic) {
            launch_fill_bits(ctx, w->y, nrt, kSentinelBits);
            launch_fill_bits(ctx, w->zs, nrt, kSentinelBits);
        }
        const int g = stream_grid(ctx, nrt);
        for (auto pr : {std::make_pair(from->b, w->b), std::make_pair(from->x, w->x), std::make_pair(from->r, w->r),
                        std::make_pair(from->p, w->p)}) {
            k_b_carry_vec<<<g, kStreamThreads, 0, ctx->stream>>>(pr.first, rt_from, pr.second, RT, sel, n);
            RCG_LAUNCHED(ctx);
        }
        k_b_carry_state<<<1, 256, 0, ctx->stream>>>(from->st, w->st, sel, RT, from->hist, w->hist, max_iter + 1,
                                                    from->u2, rt_from, w->u2, sc ? scb->k : 0);
        RCG_LAUNCHED(ctx);
        start_iter = iter;
    }

    // W^T y with the finaliser (u = (W^T A W)^-1 f, or f.u for mode 2): the register-blocked
    // k_b_wty where RT is a multiple of 4 (RCG_WTY=0: the sibling-pass k_b_tallt)
    void launch_wty(const double* Wm, int64_t ld, int mcols, const double* yv, const double* Lf, double* uo, int mode,
                    int respect_done) {
        static const int use = std::getenv("RCG_WTY") ? std::atoi(std::getenv("RCG_WTY")) : 1;
        if constexpr (RT % 4 == 0) {
            if (use && mcols >= 1 && mcols <= 128 && static_cast<int64_t>(mcols) * RT <= kMaxRedB && ld % 2 == 0) {
                static bool attr = false;
                if (!attr) {
                    RCG_CK(cudaFuncSetAttribute(k_b_wty<RT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
                    attr = true;
                }
                const size_t smem = wty_smem<RT>(mcols);
                const int64_t ntile = (static_cast<int64_t>(n) + kWtyRows - 1) / kWtyRows;
                const int per_sm = std::max(1, std::min(4, static_cast<int>((200 * 1024) / (smem + 20 * 1024))));
                const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ntile, ctx->num_sms * per_sm)));
                k_b_wty<RT><<<grid, kWtyThreads, smem, ctx->stream>>>(Wm, ld, mcols, yv, n, w->partials, Lf, uo, mode,
                                                                      w->st, respect_done);
                return;
            }
        }
        k_b_tallt<RT><<<tgrid(mcols), kElemThreads, 0, ctx->stream>>>(Wm, ld, mcols, yv, n, w->partials, Lf, uo, mode,
                                                                       w->st, respect_done);
    }

    // y -= C u (+ (p, y) or the projected-residual check): the TMA-staged kernel at RT 16 / 24
    // (RCG_DEFLATE_T=0: the register kernel)
    void launch_deflate(double* yv, const double* Cm, int64_t ldc, int mcols, const double* uv, const double* pv,
                        int mode) {
        static const int use = std::getenv("RCG_DEFLATE_T") ? std::atoi(std::getenv("RCG_DEFLATE_T")) : 1;
        if constexpr (RT == 16 || RT == 24) {
            if (use && mcols >= 1 && mcols <= 48 && ldc % 2 == 0 && n >= kDtRows) {
                static bool attr = false;
                if (!attr) {
                    RCG_CK(cudaFuncSetAttribute(k_b_deflate_t<RT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
                    attr = true;
                }
                const size_t smem = dt_smem<RT>(mcols, pv != nullptr);
                const int64_t ntile = (static_cast<int64_t>(n) + kDtRows - 1) / kDtRows;
                const int per_sm = std::max(1, std::min(3, static_cast<int>((220 * 1024) / (smem + 16 * 1024))));
                const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ntile, ctx->num_sms * per_sm)));
                k_b_deflate_t<RT><<<grid, dt_threads<RT>(), smem, ctx->stream>>>(yv, Cm, ldc, mcols, uv, pv, n, w->partials,
                                                                               w->st, mode);
                return;
            }
        }
        k_b_deflate<RT><<<eg, kElemThreads, 0, ctx->stream>>>(yv, Cm, ldc, mcols, uv, pv, n, w->partials, w->st, mode);
    }

    // k_b_tallt grid: X row ranges x P sibling column passes, one wave (4-6 CTAs per SM)
    int tgrid(int mcols) const {
        const int P = std::max(1, (mcols + tallt_jc<RT>() - 1) / tallt_jc<RT>());
        const int X = std::max(1, std::min((n + 255) / 256, ctx->num_sms * (RT <= 8 ? 4 : 6) / P));  // one wave
        return X * P;
    }  // (kElemThreads threads per CTA)

    SpmvArgs sargs() const {
        SpmvArgs s{};
        s.rs = a->rs;
        s.ci = a->ci;
        s.va = a->va;
        s.n = n;
        s.partials = w->partials;
        return s;
    }

    SweepArgs swargs(bool backward) {
        SweepArgs s = sweep_args(ctx, m->ic, backward);
        s.tickets = w->tickets + (backward ? 4 : 0);
        s.partials = w->partials;
        s.gpart = w->gpart;
        s.gcount = w->gcount;
        return s;
    }

    void initial() {
        BState h{};
        h.iter = 1;
        h.max_iter = max_iter;
        h.eps = eps;
        h.defer = job.comm ? 1 : 0;
        h.dtot = job.comm ? job.comm->dtot : nullptr;
        std::memcpy(ctx->host_pinned, &h, sizeof(h));
        RCG_CK(cudaMemcpyAsync(w->st, ctx->host_pinned, sizeof(BState), cudaMemcpyHostToDevice, ctx->stream));
        const int64_t nrt = static_cast<int64_t>(n) * RT;
        if (ic) {
            launch_fill_bits(ctx, w->y, nrt, kSentinelBits);
            launch_fill_bits(ctx, w->zs, nrt, kSentinelBits);
        }
        const bool dfl = defl && defl->k > 0;
        if (job.comm) job.comm->halo(ctx, w->x, RT);
        k_b_residual<RT><<<pg, kSpmvThreads, pipe_smem_bytes(bcap), ctx->stream>>>(sargs(), bcap, w->b, w->x, w->r, w->st,
                                                                          w->partials, dfl ? 1 : 0);
        RCG_LAUNCHED(ctx);
        reduce(0, 2 * RT, dfl ? 1 : 0, 0);
        if (dfl) {
            launch_wty(defl->w, defl->ld, defl->k, w->r, defl->l, w->u, 1, 0);
            RCG_LAUNCHED(ctx);
            reduce(5, defl->k * RT, 1, 0, defl->l, defl->k, w->u);
            launch_deflate(w->r, defl->aw, defl->ld, defl->k, w->u, nullptr, 1);
            RCG_LAUNCHED(ctx);
            reduce(3, RT, 0, 0);
        }
        if (sc) {
            launch_wty(scb->w, scb->ld, scb->k, w->r, scb->l, w->u2, 2, 0);
            RCG_LAUNCHED(ctx);
            reduce(5, scb->k * RT, 2, 0, scb->l, scb->k, w->u2);
        }
        k_b_count<<<1, 1, 0, ctx->stream>>>(w->st, RT);
        RCG_LAUNCHED(ctx);
    }

    void iteration() {
        const double* z = w->r;
        if (ic) {
            SweepArgs fa = swargs(false);
            fa.in = w->r;
            fa.out = w->y;
            launch_b_sweep(false, fa);
            SweepArgs ba = swargs(true);
            ba.in = w->y;
            ba.out = w->zs;
            ba.r = w->r;
            ba.add_sc = sc ? 1 : 0;
            launch_b_sweep(true, ba);
            if (pending_rr) {  // [rho | the previous iteration's (r, r)] in one allreduce: check, then rho
                pending_rr = false;
                job.comm->allreduce(ctx, 2 * RT);
                fin(4, 0, 1, RT);
                fin(1, 0, 1, 0);
            } else {
                reduce(1, RT, sc ? 1 : 0, 1);
            }
            z = w->zs;
        }
        require(ic || !sc, "batch: subspace correction needs the IC inner preconditioner");
        {
            KTimer t(ctx, 8, RT);
            k_b_pupdate<RT><<<sg, 256, 0, ctx->stream>>>(z, w->p, ic ? w->zs : nullptr, w->y, n, w->st,
                                                                    sc ? scb->w : nullptr, sc ? scb->ld : 0,
                                                                    sc ? scb->k : 0, w->u2);
            RCG_LAUNCHED(ctx);
        }
        const bool dfl = defl && defl->k > 0;
        const bool fuse = job.comm && fuse_enabled();
        if (job.comm) job.comm->halo(ctx, w->p, RT);
        {
            KTimer t(ctx, 5, RT);
            if (!launch_grid_spmv(dfl))
                k_b_spmv_pq<RT><<<pg, kSpmvThreads, pipe_smem_bytes(bcap), ctx->stream>>>(
                    sargs(), bcap, w->p, w->q, w->st, w->partials, dfl && !fuse ? 1 : 0);
            RCG_LAUNCHED(ctx);
        }
        if (!dfl) reduce(2, RT, 0, 1);
        if (dfl && fuse) {
            // the SpMV left the local (p, q) in dtot[0..RT): behind W^T q's m RT totals, one allreduce,
            // one finaliser (u, then alpha from (p, q) - f . u); the update's own (p, q) is not used
            const int mk = defl->k * RT;
            stash(0, mk, RT);
            {
                KTimer t(ctx, 9, RT);
                launch_wty(defl->w, defl->ld, defl->k, w->q, defl->l, w->u, 1, 1);
                RCG_LAUNCHED(ctx);
            }
            job.comm->allreduce(ctx, mk + RT);
            fin(6, 1, 1, 0, defl->l, defl->k, w->u);
            {
                KTimer t(ctx, 9, RT);
                launch_deflate(w->q, defl->aw, defl->ld, defl->k, w->u, w->p, 0);
                RCG_LAUNCHED(ctx);
            }
        } else if (dfl) {
            {
                KTimer t(ctx, 9, RT);
                launch_wty(defl->w, defl->ld, defl->k, w->q, defl->l, w->u, 1, 1);
                RCG_LAUNCHED(ctx);
            }
            reduce(5, defl->k * RT, 1, 1, defl->l, defl->k, w->u);
            {
                KTimer t(ctx, 9, RT);
                launch_deflate(w->q, defl->aw, defl->ld, defl->k, w->u, w->p, 0);
                RCG_LAUNCHED(ctx);
            }
            reduce(2, RT, 0, 1);
        }
        {
            KTimer t(ctx, 8, RT);
            k_b_xr<RT><<<eg, kElemThreads, 0, ctx->stream>>>(w->x, w->r, w->p, w->q, n, w->partials, w->st, w->hist,
                                                               max_iter + 1, (!ic && !sc) ? 1 : 0);
            RCG_LAUNCHED(ctx);
        }
        if (fuse && ic && !sc) {  // the check waits for the next iteration's (r, z) allreduce
            stash(0, RT, RT);
            pending_rr = true;
        } else if (fuse && sc) {
            // subspace correction: (r, r) travels with W^T r (subspace_correction.cpp:50-51) -- the
            // check first, then the coefficients, as unfused; W^T r of a just-finished solve is wasted
            const int mk = scb->k * RT;
            stash(0, mk, RT);
            {
                KTimer t(ctx, 9, RT);
                launch_wty(scb->w, scb->ld, scb->k, w->r, scb->l, w->u2, 2, 1);
                RCG_LAUNCHED(ctx);
            }
            job.comm->allreduce(ctx, mk + RT);
            fin(4, 0, 1, mk);
            fin(5, 2, 1, 0, scb->l, scb->k, w->u2);
            return;
        } else {
            reduce(4, RT, (!ic && !sc) ? 1 : 0, 1);
        }
        if (sc) {
            {
                KTimer t(ctx, 9, RT);
                launch_wty(scb->w, scb->ld, scb->k, w->r, scb->l, w->u2, 2, 1);
                RCG_LAUNCHED(ctx);
            }
            reduce(5, scb->k * RT, 2, 1, scb->l, scb->k, w->u2);
        }
    }

    // q = A p on a stencil grid through shared-memory staged segments (RT a multiple of 4)
    bool launch_grid_spmv(bool dfl) {
        if constexpr (RT % 4 != 0) {
            return false;
        } else {
            if (job.comm) return false;
            const int gst = grid_info(ctx, a);
            if (gst == 0) return false;
            static bool attr = false;
            if (!attr) {
                for (const void* k : {reinterpret_cast<const void*>(k_b_spmv_grid<RT, 27>),
                                      reinterpret_cast<const void*>(k_b_spmv_grid<RT, 7>)})
                    RCG_CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
                attr = true;
            }
            const size_t smem = gst == 27 ? grid_spmv_smem<RT, 27>() : grid_spmv_smem<RT, 7>();
            if (smem > 200 * 1024) return false;
            const int per_sm = std::max(1, static_cast<int>((220 * 1024) / (smem + 8 * 1024)));
            const int grid = ctx->num_sms * std::min(per_sm, 4);
            if (gst == 27)
                k_b_spmv_grid<RT, 27><<<grid, kGridSpmvThreads, smem, ctx->stream>>>(sargs(), a->gN, w->p, w->q, w->st,
                                                                                    w->partials, dfl ? 1 : 0);
            else
                k_b_spmv_grid<RT, 7><<<grid, kGridSpmvThreads, smem, ctx->stream>>>(sargs(), a->gN, w->p, w->q, w->st,
                                                                                   w->partials, dfl ? 1 : 0);
            return true;
        }
    }

    // row slabs: the last reducing kernel wrote its local totals (BState::defer): sum them over the
    // ranks and run its finaliser (k_b_fin); a no-op on one GPU, where the kernel finalised itself
    void reduce(int which, int count, int arg, int guard, const double* L = nullptr, int mm = 0, double* u = nullptr) {
        if (!job.comm) return;
        job.comm->allreduce(ctx, count);
        fin(which, arg, guard, 0, L, mm, u);
    }
    void fin(int which, int arg, int guard, int off, const double* L = nullptr, int mm = 0, double* u = nullptr) {
        k_b_fin<RT><<<1, kElemThreads, 0, ctx->stream>>>(w->st, which, arg, guard, L, mm, u, w->hist, max_iter + 1, off);
        RCG_LAUNCHED(ctx);
    }
    void stash(int src, int dst, int cnt) {
        k_b_stash<<<1, 32, 0, ctx->stream>>>(w->st, src, dst, cnt);
        RCG_LAUNCHED(ctx);
    }
    // row slabs, fused reductions (RCG_DIST_FUSE=0 keeps one allreduce per dot):
    // (p, q) travels with W^T q, and the convergence check's (r, r) waits for the next iteration's
    // (r, z) -- two allreduces per deflated iteration instead of four.  The deferred check is
    // flushed before the host reads the running count (run()).
    static bool fuse_enabled() {  // (read per call: the A/B test switches it inside one process)
        const char* e = std::getenv("RCG_DIST_FUSE");
        return !(e && std::atoi(e) == 0);
    }
    bool pending_rr = false;
    void flush_pending() {
        if (!pending_rr) return;
        pending_rr = false;
        stash(RT, 0, RT);
        job.comm->allreduce(ctx, RT);
        fin(4, 0, 1, 0);
    }

    void launch_b_sweep(bool backward, SweepArgs& s) {
        const rcg_ic* f = m->ic;
        // RCG_BSWEEP=0 selects the row-lane sweep (A/B only); default: chunk lanes
        static const int mode = std::getenv("RCG_BSWEEP") ? std::atoi(std::getenv("RCG_BSWEEP")) : 1;
        // residency: the single-sweep rule, except that the batched backward sweep keeps the
        // forward's CTAs (C3 RT 12: bwd 14.3 -> 8.7 ms) and rows of more than one dependency chunk
        // take 3 (C3 RT 12: fwd 5.4 -> 4.9, bwd 8.7 -> 7.8 ms)
        int bps0 = ctx->sweep_bps > 0 ? ctx->sweep_bps : sweep_ctas_per_sm(f, false, s.npos);
        if (ctx->sweep_bps <= 0 && f->n > 0 && static_cast<double>(f->nnz_l) / f->n > kDepChunkHost) bps0 = std::max(bps0, 3);
        s.backoff_ns = ctx->sweep_backoff_ns;
        KTimer t(ctx, backward ? 7 : 6, RT);
        // very wide levels (the multicolour orderings): one launch per level, no polling
        // (default shape rule of icsweep_lv.cu: >= 600K rows per level; mode 4 always).  Forced on
        // natural orderings at RT 8 it wins only on C4 (fwd 27.3 -> 20.8, bwd 37.7 -> 33.4 ms) and
        // loses on C5 (707 -> 842 us) and C3 (4.1 -> 17.3 ms)
        const std::vector<int32_t>& lp = f->h_lptr[backward ? 1 : 0];
        const int nlev = backward ? f->bwd_levels : f->fwd_levels;
        const bool level_ok = static_cast<int>(lp.size()) == nlev + 1 && nlev > 0;
        if (level_ok && (ctx->sweep_cluster == 4 || (ctx->sweep_cluster == 2 && s.npos / nlev >= 600000))) {
            const bool rho = backward && s.r;
            int64_t tile = 0;
            for (int l = 0; l < nlev; ++l) {
                const int32_t width = lp[l + 1] - lp[l];
                const int64_t items = static_cast<int64_t>(width) * (RT % 4 == 0 ? RT / 4 : RT / 2);
                const int g = static_cast<int>(std::max<int64_t>(
                    1, std::min<int64_t>((items + kElemThreads - 1) / kElemThreads, ctx->num_sms * 8)));
                if (backward)
                    k_b_level<true, RT><<<g, kElemThreads, 0, ctx->stream>>>(s, w->st, lp[l], width, w->tpart, tile);
                else
                    k_b_level<false, RT><<<g, kElemThreads, 0, ctx->stream>>>(s, w->st, lp[l], width, w->tpart, tile);
                RCG_LAUNCHED(ctx);
                tile += g;
            }
            if (rho) {
                const int gr = static_cast<int>(std::max<int64_t>(
                    1, std::min<int64_t>((tile * RT + kElemThreads * 4 - 1) / (kElemThreads * 4), ctx->num_sms * 8)));
                k_b_rho<RT><<<gr, kElemThreads, 0, ctx->stream>>>(w->tpart, tile, w->partials, w->st, s.add_sc);
                RCG_LAUNCHED(ctx);
            }
            return;
        }
        if (mode != 0 || job.comm) {  // (row slabs: rho always through k_b_rho's deferred finaliser)
            // chunk lanes: 16-byte chunks (measured faster than 32-byte), 4 parents per poll
            // chunk (register budget -> residency); 3x the single-sweep CTAs from RT = 12 on
            // (re-measured end of round 1, C2 fwd / bwd: RT 12 x1 992/1298, x2 632/788, x3 578/657,
            // x4 620/681 us; RT 4 x2 497/535, x3 506/559 us.  32-byte chunks (VW 4, half the
            // polling lanes) again slower: RT 12 700/828, RT 8 660/739, RT 16 668/744 us)
            // RT 24 with 16-byte chunks leaves 8 of 32 lanes idle (2 rows x 12 lanes per warp) and
            // writes 2.5x the rho tile partials; RCG_BSWEEP_VW=4 selects 32-byte chunks there (5 rows
            // x 6 lanes) -- A/B switch
            // measured on C3 at RT 24 (ms per launch, VW 2 / VW 4): forward 8.18 / 5.84, backward
            // 12.80 / 13.79 -- 32-byte chunks for the forward sweep only (RCG_BSWEEP_VW=2 / 4 forces)
            static const int vw_env = std::getenv("RCG_BSWEEP_VW") ? std::atoi(std::getenv("RCG_BSWEEP_VW")) : 0;
            const bool vw4 = RT == 24 && (vw_env == 4 || (vw_env == 0 && !backward));
            const int rpw = vw4 ? 32 / (RT / 4) : 32 / (RT / 2);
            static const int cmul_env = std::getenv("RCG_BSWEEP_CMUL") ? std::atoi(std::getenv("RCG_BSWEEP_CMUL")) : 0;
            const int cmul = cmul_env > 0 ? cmul_env : (RT >= 12 ? 3 : 2);
            const int ntiles = (s.npos + rpw * 4 - 1) / (rpw * 4);  // CTAs of 4 warp tiles
            const int grid = std::max(1, std::min(ntiles, ctx->num_sms * bps0 * cmul));
            const bool rho = backward && s.r;
            if (rho) s.partials = w->tpart;
            // (measured and dropped, C3 RT 24 fwd / bwd ms: 7 parents per chunk 6.9 / 14.4, 13 per
            // chunk -- 147 registers -- slower still; L1-cached first loads of the older parents
            // 7.4 / 16.4: stale sentinel sectors in L1 cost more re-polls than the hits save)
            auto go = [&](auto kern) { kern<<<grid, 128, 0, ctx->stream>>>(s, w->st); };
            bool launched = false;
            if constexpr (RT == 24) {
                if (vw4) {
                    launched = true;
                    backward ? go(k_b_sweepc<true, RT, 4, 4>) : go(k_b_sweepc<false, RT, 4, 4>);
                }
            }
            if (!launched) backward ? go(k_b_sweepc<true, RT, 2, 4>) : go(k_b_sweepc<false, RT, 2, 4>);
            RCG_LAUNCHED(ctx);
            if (rho) {
                const int64_t tiles = (s.npos + rpw - 1) / rpw;
                const int g = static_cast<int>(std::max<int64_t>(
                    1, std::min<int64_t>((tiles * RT + kElemThreads * 4 - 1) / (kElemThreads * 4), ctx->num_sms * 8)));
                k_b_rho<RT><<<g, kElemThreads, 0, ctx->stream>>>(w->tpart, tiles, w->partials, w->st, s.add_sc);
                RCG_LAUNCHED(ctx);
            }
            return;
        } else {
            const int ntiles = (s.npos + 127) / 128;  // in CTAs of 4 warp tiles
            const int grid = std::max(1, std::min(ntiles, ctx->num_sms * bps0));
            if (backward)
                k_b_sweep<true, RT><<<grid, 128, 0, ctx->stream>>>(s, w->st);
            else
                k_b_sweep<false, RT><<<grid, 128, 0, ctx->stream>>>(s, w->st);
        }
        RCG_LAUNCHED(ctx);
    }

    void finish() {
        k_b_finish_combine<RT><<<sg, kStreamThreads, 0, ctx->stream>>>(w->x, nullptr, 0, 0, nullptr, n, w->st, 2);
        RCG_LAUNCHED(ctx);
        if (defl && defl->k > 0) {  // x = P x + W (W^T A W)^-1 W^T b (pcg.cpp:152-157), finished slots
            launch_wty(defl->aw, defl->ld, defl->k, w->x, defl->l, w->u, 1, 0);
            RCG_LAUNCHED(ctx);
            reduce(5, defl->k * RT, 1, 0, defl->l, defl->k, w->u);
            k_b_finish_combine<RT><<<sg, kStreamThreads, 0, ctx->stream>>>(w->x, defl->w, defl->ld, defl->k, w->u, n,
                                                                           w->st, 0);
            RCG_LAUNCHED(ctx);
            launch_wty(defl->w, defl->ld, defl->k, w->b, defl->l, w->u, 1, 0);
            RCG_LAUNCHED(ctx);
            reduce(5, defl->k * RT, 1, 0, defl->l, defl->k, w->u);
            k_b_finish_combine<RT><<<sg, kStreamThreads, 0, ctx->stream>>>(w->x, defl->w, defl->ld, defl->k, w->u, n,
                                                                           w->st, 1);
            RCG_LAUNCHED(ctx);
        }
    }

    // iterate; returns early (allow_shrink) once the running slots fit a narrower phase
    void run(bool allow_shrink) {
        cudaEvent_t evs[2], t0, t1;
        RCG_CK(cudaEventCreateWithFlags(&evs[0], cudaEventDisableTiming));
        RCG_CK(cudaEventCreateWithFlags(&evs[1], cudaEventDisableTiming));
        RCG_CK(cudaEventCreate(&t0));
        RCG_CK(cudaEventCreate(&t1));
        RCG_CK(cudaEventRecord(t0, ctx->stream));
        volatile int* flags = reinterpret_cast<volatile int*>(ctx->host_pinned + 256);
        int enq = start_iter - 1, batch = 2, slot = 0, prev = 0;
        bool have_prev = false;
        while (enq < max_iter) {
            for (int j = 0; j < batch && enq < max_iter; ++j, ++enq) iteration();
            flush_pending();
            RCG_CK(cudaMemcpyAsync((void*)(flags + slot), &w->st->nrun, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
            RCG_CK(cudaEventRecord(evs[slot], ctx->stream));
            if (enq >= max_iter) break;
            if (have_prev) {
                RCG_CK(cudaEventSynchronize(evs[prev]));
                const int nr = flags[prev];
                if (nr == 0 || (allow_shrink && pick_rt(nr) < RT)) break;
            }
            have_prev = true;
            prev = slot;
            slot ^= 1;
            batch = std::min(batch * 2, 16);
        }
        RCG_CK(cudaEventRecord(t1, ctx->stream));
        RCG_CK(cudaEventSynchronize(t1));
        float ms = 0.f;
        RCG_CK(cudaEventElapsedTime(&ms, t0, t1));
        job.wall += ms * 1e-3;
        for (auto e : {evs[0], evs[1], t0, t1}) cudaEventDestroy(e);
    }

    // finish, scatter and report the slots that are done; returns the running ones (slot ->
    // original column) and their iteration
    SlotMap retire(int* iter) {
        finish();
        BState h{};
        RCG_CK(cudaMemcpyAsync(ctx->host_pinned + 1024, w->st, sizeof(BState), cudaMemcpyDeviceToHost, ctx->stream));
        RCG_CK(cudaStreamSynchronize(ctx->stream));
        std::memcpy(&h, ctx->host_pinned + 1024, sizeof(BState));
        SlotMap out, carry;
        for (int k = 0; k < map.cnt; ++k) {
            if (h.done[k] == kRunning) {
                carry.slot[carry.cnt] = k;
                carry.col[carry.cnt++] = map.col[k];
            } else {
                out.slot[out.cnt] = k;
                out.col[out.cnt++] = map.col[k];
            }
        }
        if (out.cnt > 0) {
            const int g = stream_grid(ctx, static_cast<int64_t>(n) * out.cnt);
            k_b_scatter_map<<<g, kStreamThreads, 0, ctx->stream>>>(w->x, RT, out, n, job.x_cols, n);
            RCG_LAUNCHED(ctx);
            std::vector<double> hist(static_cast<size_t>(max_iter + 1));
            for (int q = 0; q < out.cnt; ++q) {
                const int k = out.slot[q];
                rcg_solve_report& r = job.reps[out.col[q]];
                r.iterations = (h.done[k] == kZeroRhs) ? 0 : h.iters[k];
                r.converged = (h.done[k] == kConverged || h.done[k] == kZeroRhs) ? 1 : 0;
                const int cnt = std::min(r.iterations, r.cap);
                const int64_t hl = max_iter + 1;
                if (r.history && cnt > 0)
                    RCG_CK(cudaMemcpy(r.history, w->hist + k * hl, sizeof(double) * cnt, cudaMemcpyDeviceToHost));
                if (r.alphas && cnt > 0)
                    RCG_CK(cudaMemcpy(r.alphas, w->hist + (RT + k) * hl, sizeof(double) * cnt, cudaMemcpyDeviceToHost));
                if (r.betas && cnt > 0)
                    RCG_CK(cudaMemcpy(r.betas, w->hist + (2 * RT + k) * hl, sizeof(double) * cnt, cudaMemcpyDeviceToHost));
                if (h.done[k] == kBroken && (job.broken < 0 || out.col[q] < job.broken)) {
                    job.broken = out.col[q];
                    job.broken_status = h.status[k];
                }
            }
        }
        *iter = h.iter;
        return carry;
    }
};

static void run_phase(int rt, BatchJob& job, int wsi, const BatchWs* from, int rt_from, const SlotMap* sel, int iter);

template <int RT>
static void phase(BatchJob& job, int wsi, const BatchWs* from, int rt_from, const SlotMap* sel, int iter) {
    BatchSolve<RT> s(job);
    s.setup(wsi == 0 ? job.ctx->bws : job.ctx->bws2);
    if (from)
        s.resume(from, rt_from, *sel, iter);
    else
        s.fresh();
    ++job.phases;
    s.run(RT > 2);
    int it = 0;
    const SlotMap carry = s.retire(&it);
    if (carry.cnt > 0) run_phase(pick_rt(carry.cnt), job, wsi ^ 1, s.w, RT, &carry, it);
}

static void run_phase(int rt, BatchJob& job, int wsi, const BatchWs* from, int rt_from, const SlotMap* sel, int iter) {
    switch (rt) {
        case 2: phase<2>(job, wsi, from, rt_from, sel, iter); break;
        case 4: phase<4>(job, wsi, from, rt_from, sel, iter); break;
        case 8: phase<8>(job, wsi, from, rt_from, sel, iter); break;
        case 12: phase<12>(job, wsi, from, rt_from, sel, iter); break;
        case 16: phase<16>(job, wsi, from, rt_from, sel, iter); break;
        default: phase<24>(job, wsi, from, rt_from, sel, iter); break;
    }
}

}  // namespace rcg

using namespace rcg;

static int batch_entry(rcg_ctx* ctx, const rcg_matrix* a, const double* B, const rcg_prec* m, const rcg_basis* defl,
                       double* X, const rcg_solver_config* cfg, int nrhs, rcg_solve_report* reps) {
    NvtxRange range("batched solves");
    return guard([&] {
        require(ctx && a && reps && B && X, "batch solve: null argument");
        require(nrhs >= 1 && nrhs <= kRMax, "batch solve: nrhs must be in [1, 24]");
        check_cfg(cfg);
        check_prec(m, a->n);
        if (defl && defl->k > 0) require(defl->n == a->n, "deflated_pcg_solve: W row count does not match A");
        const int32_t n = a->n;
        Staged bs, xs;
        stage_in(ctx, B, static_cast<int64_t>(n) * nrhs, bs);
        stage_in(ctx, X, static_cast<int64_t>(n) * nrhs, xs);
        Staged xo;
        stage_out_begin(ctx, X, static_cast<int64_t>(n) * nrhs, xo);
        if (xo.dev != xs.dev && nrhs > 0)
            RCG_CK(cudaMemcpyAsync(xo.dev, xs.dev, sizeof(double) * n * nrhs, cudaMemcpyDeviceToDevice, ctx->stream));
        BatchJob job{ctx, a, m, defl, n, nrhs, cfg->max_iter, cfg->eps, bs.dev, xo.dev, reps};
        // RT: 2 for one or two right-hand sides, else a multiple of 4 (32-byte chunks: one
        // 256-bit access per chunk in the sweeps and spmv gathers)
        run_phase(pick_rt(nrhs), job, 0, nullptr, 0, nullptr, 1);
        stage_out_end(ctx, X, static_cast<int64_t>(n) * nrhs, xo);
        RCG_CK(cudaStreamSynchronize(ctx->stream));
        check_sweep_watchdog(ctx);
        // per right-hand side: the batch's loop time shared out, so sums over solves (the
        // sequence driver's avg_wall_time, driver.cpp:197-205) keep their per-solve meaning
        for (int k = 0; k < nrhs; ++k) reps[k].wall_time = job.wall / nrhs;
        if (job.broken >= 0) {
            const bool dfl = defl && defl->k > 0;
            throw Error(RCG_E_BREAKDOWN, std::string(dfl ? "deflated pcg" : "pcg") + ": breakdown in right-hand side " +
                                             std::to_string(job.broken) +
                                             (job.broken_status == kBrkRz ? " ((r, z) <= 0)" : " ((p, A p) <= 0)"));
        }
    });
}

namespace rcg {

// the batched solver over one row slab of a distributed system (dist.cu supplies the exchange
// and the allreduce); B / X hold nrhs vectors of the slab's nloc rows, device or host
void batch_solve_dist(rcg_ctx* ctx, const rcg_matrix* a, const rcg_prec* m, const rcg_basis* defl, BatchComm* comm,
                      const double* B, double* X, const rcg_solver_config* cfg, int nrhs, rcg_solve_report* reps) {
    require(ctx && a && reps && B && X && comm, "dist batch solve: null argument");
    require(nrhs >= 1 && nrhs <= kRMax, "batch solve: nrhs must be in [1, 24]");
    check_cfg(cfg);
    check_prec(m, a->n);
    const int32_t n = a->n;
    Staged bs, xs;
    stage_in(ctx, B, static_cast<int64_t>(n) * nrhs, bs);
    stage_in(ctx, X, static_cast<int64_t>(n) * nrhs, xs);
    Staged xo;
    stage_out_begin(ctx, X, static_cast<int64_t>(n) * nrhs, xo);
    if (xo.dev != xs.dev && nrhs > 0)
        RCG_CK(cudaMemcpyAsync(xo.dev, xs.dev, sizeof(double) * n * nrhs, cudaMemcpyDeviceToDevice, ctx->stream));
    BatchJob job{ctx, a, m, defl, n, nrhs, cfg->max_iter, cfg->eps, bs.dev, xo.dev, reps};
    job.comm = comm;
    run_phase(pick_rt(nrhs), job, 0, nullptr, 0, nullptr, 1);
    stage_out_end(ctx, X, static_cast<int64_t>(n) * nrhs, xo);
    RCG_CK(cudaStreamSynchronize(ctx->stream));
    check_sweep_watchdog(ctx);
    for (int k = 0; k < nrhs; ++k) reps[k].wall_time = job.wall / nrhs;
    if (job.broken >= 0) {
        const bool dfl = defl && defl->k > 0;
        throw Error(RCG_E_BREAKDOWN, std::string(dfl ? "deflated pcg" : "pcg") + ": breakdown in right-hand side " +
                                         std::to_string(job.broken) +
                                         (job.broken_status == kBrkRz ? " ((r, z) <= 0)" : " ((p, A p) <= 0)"));
    }
}

}  // namespace rcg

extern "C" {

int rcg_pcg_solve_batch(rcg_ctx* ctx, const rcg_matrix* a, const double* B, const rcg_prec* m, double* X,
                        const rcg_solver_config* cfg, int nrhs, rcg_solve_report* reps) {
    return batch_entry(ctx, a, B, m, nullptr, X, cfg, nrhs, reps);
}

int rcg_deflated_pcg_solve_batch(rcg_ctx* ctx, const rcg_matrix* a, const double* B, const rcg_prec* m,
                                 const rcg_basis* defl, double* X, const rcg_solver_config* cfg, int nrhs,
                                 rcg_solve_report* reps) {
    return batch_entry(ctx, a, B, m, defl, X, cfg, nrhs, reps);
}

}  // extern "C"
