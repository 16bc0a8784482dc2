// psweep.cu -- IC(0) sweeps as a pencil wavefront, for factors of natural-ordered box grids with
// the 7-point or the 27-point stencil pattern (C1-C4).
//
// Why.  The level-ordered sweep (icsweep.cu) pays one inter-SM publish -> observe round trip per
// DAG level plus each tile's chain of dependent loads (ticket -> perm -> row starts -> entries ->
// parents); on C3 that is 2-3 us per level over 1,786 levels.  On a stencil grid the DAG has a
// regular shape, so the schedule can be fixed in advance and almost every dependency kept on chip.
//
// Mapping.  A warp owns a UNIT = 32 consecutive y-rows of one z-plane (lane j <-> row y0 + j) and
// sweeps it along x in steps; lane j handles x = T - K j at step T (K = 2 for the 27-point stencil,
// 1 for the 7-point), so at every step each lane's row needs:
//   x-1 neighbour            -- the lane's own previous result (register)
//   (x-1..x+1, y-1) row      -- lane j-1's last K+1 results (warp shuffles; lane 0: HBM/L2)
//   (x-1..x+1, y-1..y+1, z-1)-- the z-1 plane, written by an earlier unit's warp: every lane loads
//                               ONE value of its own z-1 row per step, A steps ahead of use, and
//                               the 3 x 3 neighbourhood is assembled with shuffles (lanes 0 / 31:
//                               the y-block boundary rows, loaded the same way).
// Cross-warp values travel through the output vector with the sentinel protocol of icsweep.cu
// (each value its own ready flag; a value found unpublished at first use is re-polled).  The
// factor coefficients are pre-laid out per (unit, step) as one contiguous record [slot][lane]
// (plus the row's schedule position) and streamed into a per-warp shared-memory ring by
// cp.async.bulk, kStages steps ahead.  Units are taken from an atomic ticket in z-major order, so
// a unit only waits on units taken earlier (running or finished): deadlock-free with a resident
// grid.  The backward sweep is the same walk in mirrored coordinates (actual row n-1-f), whose
// slot order is the forward one reversed.
//
// Operator identity.  Each row is the reference loop (src/ic_preconditioner.cpp:130-143): forward
// s = r_i, s -= l_ik y_k in stored (ascending column) order; backward s = y_i / d_i,
// s -= u_ik z_k -- absent neighbours skipped -- so the output is bitwise k_sweep's.  The (r, z)
// products are written at the row's backward-schedule position and reduced in k_sweep's
// tile -> group -> total order (k_tile_partials + icsweep_lv.cu's k_level_groups / k_level_total),
// so rho and every iterate are bitwise identical whichever sweep kernel runs.
//
// Roofline: per sweep the records (8 S + 4 bytes per row and step slot: 108 B/row for the 27-point
// stencil) + in / out (+ d, r, the (r, z) product) -- HBM-bound once the wavefront is wide enough.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "internal.cuh"
#include "kernels.cuh"
#include "spmv_pipe.cuh"

namespace rcg {

constexpr int kPsWarps = 4;   // warps per CTA
constexpr int kPsStages = 4;  // coefficient records in flight per warp

template <int ST>
struct Sten;
template <>
struct Sten<27> {
    static constexpr int K = 2;   // lane skew in x
    static constexpr int S = 13;  // lower neighbours
    static constexpr int A = 6;   // z-1 load lead (steps)
    static constexpr int H = A + 4;
};
template <>
struct Sten<7> {
    static constexpr int K = 1;
    static constexpr int S = 3;
    static constexpr int A = 4;
    static constexpr int H = A + 1;
};

__host__ __device__ constexpr int ps_rec_bytes(int S) { return S * 32 * 8 + 32 * 4; }

struct PsArgs {
    const unsigned char* recs;  // [unit][step] records
    int32_t nx, ny, nz, nb;     // grid, y-blocks
    int32_t nt;                 // steps per unit
    int32_t units;
    int64_t n;
    const double* in;
    const double* d;            // backward
    const double* r;            // backward: (r, z) products when non-null
    double* out;
    double* cbuf;               // backward: r_i z_i at the row's schedule position
    int* tickets;               // [0] unit ticket, [1] exit count, [3] watchdog
    const DevState* st;
};

// bounded: a schedule fault sets the watchdog (check_sweep_watchdog raises) and every later
// poll of the launch gives up at once, so a fault is an error, never a hang
__device__ __forceinline__ double poll_value(const double* p, int* watchdog) {
    double v = ld_relaxed(p);
    unsigned spins = 0;
    while (is_sentinel(v)) {
        if (++spins > 64) __nanosleep(64);
        v = ld_relaxed(p);
        if ((spins & 1023u) == 0u && (spins >= (1u << 21) || *reinterpret_cast<volatile int*>(watchdog))) {
            atomicExch(watchdog, 1);
            return 0.0;
        }
    }
    return v;
}

template <int ST, bool BWD>
__global__ void __launch_bounds__(kPsWarps * 32) k_psweep(PsArgs a) {
    using P = Sten<ST>;
    constexpr int K = P::K, S = P::S, A = P::A, H = P::H;
    constexpr int REC = ps_rec_bytes(S);
    if (a.st->done) return;
    extern __shared__ __align__(16) unsigned char ps_smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned char* wbase = ps_smem + static_cast<size_t>(wid) * (16 * kPsStages + kPsStages * REC);
    uint64_t* bar = reinterpret_cast<uint64_t*>(wbase);
    unsigned char* ring = wbase + 16 * kPsStages;
    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < kPsStages; ++s) mbar_init(&bar[s]);
        fence_mbar_init();
    }
    __syncwarp();
    unsigned phase = 0u;  // parity bit per stage
    const int64_t nxy = static_cast<int64_t>(a.nx) * a.ny;
    const int64_t nlast = a.n - 1;
    // frame index -> actual row (the backward sweep walks the mirrored grid)
    auto act = [&](int64_t f) { return BWD ? nlast - f : f; };

    while (true) {
        int unit = 0;
        if (lane == 0) unit = atomicAdd(&a.tickets[0], 1);
        unit = __shfl_sync(0xffffffffu, unit, 0);
        if (unit >= a.units) break;
        const int z = unit / a.nb, b = unit % a.nb;
        const int y = b * 32 + lane;
        const bool yok = y < a.ny;
        const unsigned char* urec = a.recs + static_cast<int64_t>(unit) * a.nt * REC;
        // prologue: records of steps 0 .. kPsStages-2
        if (lane == 0) {
#pragma unroll
            for (int s = 0; s < kPsStages - 1; ++s)
                if (s < a.nt) {
                    fence_proxy_async();
                    mbar_expect_tx(&bar[s], REC);
                    bulk_g2s(ring + s * REC, urec + static_cast<int64_t>(s) * REC, REC, &bar[s]);
                }
        }
        // histories: own z-1 row (zh), y-block boundary rows (bA: lane 0 in-plane y0-1 / lane 31
        // z-1 row y0+32; bB: lane 0 z-1 row y0-1); zh[k] / bA[k] hold coordinate x + A - k
        double zh[H], bA[A + 2], bB[A + 2];
#pragma unroll
        for (int k = 0; k < H; ++k) zh[k] = 0.0;
#pragma unroll
        for (int k = 0; k < A + 2; ++k) bA[k] = bB[k] = 0.0;
        double h1 = 0.0, h2 = 0.0, h3 = 0.0;  // own results at x-1, x-2, x-3
        // frame bases of the rows this lane reads
        const int64_t f_row = static_cast<int64_t>(y) * a.nx + z * nxy;        // (0, y, z)
        const bool zm_ok = z > 0;
        const int64_t f_zm = f_row - nxy;                                      // (0, y, z-1)
        // lane 0: in-plane y0-1 (bA) and z-1 row y0-1 (bB); lane 31: z-1 row y0+32 (bA)
        const int yA = lane == 0 ? y - 1 : (ST == 27 && lane == 31 ? y + 1 : -1);
        const int zA = lane == 0 ? z : z - 1;
        const bool A_ok = yA >= 0 && yA < a.ny && zA >= 0 && (lane == 0 || lane == 31);
        const int64_t f_A = static_cast<int64_t>(yA) * a.nx + static_cast<int64_t>(zA) * nxy;
        const bool B_ok = ST == 27 && lane == 0 && y - 1 >= 0 && z > 0;
        const int64_t f_B = static_cast<int64_t>(y - 1) * a.nx + static_cast<int64_t>(z - 1) * nxy;
        int* wd = a.tickets + 3;
        const int x0 = -K * lane;

        for (int T = 0; T < a.nt; ++T) {
            const int x = x0 + T;
            // next record into the ring (stage of step T-1, freed by the __syncwarp below)
            if (lane == 0 && T + kPsStages - 1 < a.nt) {
                const int s = (T + kPsStages - 1) % kPsStages;
                fence_proxy_async();
                mbar_expect_tx(&bar[s], REC);
                bulk_g2s(ring + s * REC, urec + static_cast<int64_t>(T + kPsStages - 1) * REC, REC, &bar[s]);
            }
            // shift histories, issue the loads A steps ahead
            {
#pragma unroll
                for (int k = H - 1; k > 0; --k) zh[k] = zh[k - 1];
#pragma unroll
                for (int k = A + 1; k > 0; --k) {
                    bA[k] = bA[k - 1];
                    bB[k] = bB[k - 1];
                }
                const int xa = x + A;
                const bool xin = xa >= 0 && xa < a.nx;
                zh[0] = (xin && yok && zm_ok) ? ld_relaxed(a.out + act(f_zm + xa)) : 0.0;
                bA[0] = (xin && A_ok) ? ld_relaxed(a.out + act(f_A + xa)) : 0.0;
                if (ST == 27) bB[0] = (xin && B_ok) ? ld_relaxed(a.out + act(f_B + xa)) : 0.0;
            }
            // first use of the entries loaded A - (K+1) steps ago (27-point: zh[A-3] by lane j-1)
            {
                constexpr int kz = ST == 27 ? A - 3 : A;
                const int xz = x + A - kz;
                if (yok && zm_ok && xz >= 0 && xz < a.nx && is_sentinel(zh[kz]))
                    zh[kz] = poll_value(a.out + act(f_zm + xz), wd);
                constexpr int kb = ST == 27 ? A - 1 : A;
                const int xb = x + A - kb;
                if (A_ok && xb >= 0 && xb < a.nx && is_sentinel(bA[kb])) bA[kb] = poll_value(a.out + act(f_A + xb), wd);
                if (ST == 27 && B_ok && xb >= 0 && xb < a.nx && is_sentinel(bB[kb]))
                    bB[kb] = poll_value(a.out + act(f_B + xb), wd);
            }
            // this step's record
            const int st = T % kPsStages;
            while (!mbar_try_wait(&bar[st], (phase >> st) & 1u)) {
            }
            phase ^= 1u << st;
            const double* coef = reinterpret_cast<const double*>(ring + st * REC);
            const int32_t* cpos = reinterpret_cast<const int32_t*>(ring + st * REC + S * 32 * 8);
            const bool on = yok && x >= 0 && x < a.nx;
            const int64_t f = f_row + x;
            double s = 0.0;
            double rv = 0.0;
            if (on) {
                const int64_t i = act(f);
                s = BWD ? __ddiv_rn(__ldg(a.in + i), __ldg(a.d + i)) : __ldg(a.in + i);
                if (BWD && a.r) rv = __ldg(a.r + i);
            }
            // neighbours: slot values in forward numbering (see Sten), then the reference order
            if (ST == 27) {
                // z-1 plane: dy = -1 from lane j-1 (its x is x+2: k = A+3..A+1), dy = 0 own
                // (k = A+1..A-1), dy = +1 from lane j+1 (its x is x-2: k = A-1..A-3)
                double zm[9];
                zm[0] = __shfl_up_sync(0xffffffffu, zh[A + 3], 1);
                zm[1] = __shfl_up_sync(0xffffffffu, zh[A + 2], 1);
                zm[2] = __shfl_up_sync(0xffffffffu, zh[A + 1], 1);
                zm[3] = zh[A + 1];
                zm[4] = zh[A];
                zm[5] = zh[A - 1];
                zm[6] = __shfl_down_sync(0xffffffffu, zh[A - 1], 1);
                zm[7] = __shfl_down_sync(0xffffffffu, zh[A - 2], 1);
                zm[8] = __shfl_down_sync(0xffffffffu, zh[A - 3], 1);
                if (lane == 0) {
                    zm[0] = bB[A + 1];
                    zm[1] = bB[A];
                    zm[2] = bB[A - 1];
                }
                if (lane == 31) {
                    zm[6] = bA[A + 1];
                    zm[7] = bA[A];
                    zm[8] = bA[A - 1];
                }
                // in-plane y-1 row from lane j-1 (its results at x-1, x, x+1 = h3, h2, h1)
                double ym[3];
                ym[0] = __shfl_up_sync(0xffffffffu, h3, 1);
                ym[1] = __shfl_up_sync(0xffffffffu, h2, 1);
                ym[2] = __shfl_up_sync(0xffffffffu, h1, 1);
                if (lane == 0) {
                    ym[0] = bA[A + 1];
                    ym[1] = bA[A];
                    ym[2] = bA[A - 1];
                }
                if (on) {
                    const bool xl = x > 0, xr = x + 1 < a.nx, yl = y > 0, yr = y + 1 < a.ny;
                    bool ok[S];
                    double pv[S];
#pragma unroll
                    for (int q = 0; q < 9; ++q) {
                        const int dy = q / 3 - 1, dx = q % 3 - 1;
                        ok[q] = zm_ok && (dy < 0 ? yl : (dy > 0 ? yr : true)) && (dx < 0 ? xl : (dx > 0 ? xr : true));
                        pv[q] = zm[q];
                    }
#pragma unroll
                    for (int q = 0; q < 3; ++q) {
                        const int dx = q - 1;
                        ok[9 + q] = yl && (dx < 0 ? xl : (dx > 0 ? xr : true));
                        pv[9 + q] = ym[q];
                    }
                    ok[12] = xl;
                    pv[12] = h1;
#pragma unroll
                    for (int q = 0; q < S; ++q) {
                        const int sl = BWD ? S - 1 - q : q;
                        if (ok[sl]) s = fsub_mul(s, coef[sl * 32 + lane], pv[sl]);
                    }
                }
            } else {
                double yv = __shfl_up_sync(0xffffffffu, h1, 1);  // (x, y-1): lane j-1's previous result
                if (lane == 0) yv = bA[A];
                if (on) {
                    const bool ok0 = zm_ok, ok1 = y > 0, ok2 = x > 0;
                    if (!BWD) {
                        if (ok0) s = fsub_mul(s, coef[0 * 32 + lane], zh[A]);
                        if (ok1) s = fsub_mul(s, coef[1 * 32 + lane], yv);
                        if (ok2) s = fsub_mul(s, coef[2 * 32 + lane], h1);
                    } else {
                        if (ok2) s = fsub_mul(s, coef[2 * 32 + lane], h1);
                        if (ok1) s = fsub_mul(s, coef[1 * 32 + lane], yv);
                        if (ok0) s = fsub_mul(s, coef[0 * 32 + lane], zh[A]);
                    }
                }
            }
            if (on) {
                if (BWD && a.r) a.cbuf[cpos[lane]] = __dmul_rn(rv, s);  // k_sweep: r_i times the raw s
                s = publishable(s);
                st_relaxed(a.out + act(f), s);
            }
            h3 = h2;
            h2 = h1;
            h1 = s;
            __syncwarp();
        }
        // drain: every issued record was waited on (steps < nt), the ring is free for the next unit
    }
    if (lane == 0) {
        __threadfence();
        if (atomicAdd(&a.tickets[1], 1) == static_cast<int>(gridDim.x * kPsWarps) - 1) {
            a.tickets[0] = 0;
            a.tickets[1] = 0;
        }
    }
}

// Record builder: for every (unit, step, lane) with a row, the row's factor entries matched to
// the stencil slots (entries in stored order == ascending columns == the kernel's slot order),
// zeros elsewhere, and the row's position in the sweep's schedule.  A mismatch (an entry that
// is not a lower / upper stencil neighbour, a missing neighbour) sets *bad.
template <int ST, bool BWD>
__global__ void k_ps_build(unsigned char* __restrict__ recs, int32_t nx, int32_t ny, int32_t nz, int32_t nb,
                           int32_t nt, int32_t units, int64_t n, const int32_t* __restrict__ pos_of,
                           const int32_t* __restrict__ prs, const int32_t* __restrict__ pcol,
                           const double* __restrict__ pval, int* __restrict__ bad) {
    using P = Sten<ST>;
    constexpr int S = P::S, K = P::K;
    constexpr int REC = ps_rec_bytes(S);
    const int64_t total = static_cast<int64_t>(units) * nt * 32;
    const int64_t nxy = static_cast<int64_t>(nx) * ny;
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int lane = static_cast<int>(t % 32);
        const int64_t us = t / 32;
        const int T = static_cast<int>(us % nt);
        const int unit = static_cast<int>(us / nt);
        const int z = unit / nb, b = unit % nb;
        const int y = b * 32 + lane, x = T - K * lane;
        double* coef = reinterpret_cast<double*>(recs + us * REC);
        int32_t* cp = reinterpret_cast<int32_t*>(recs + us * REC + S * 32 * 8);
        for (int q = 0; q < S; ++q) coef[q * 32 + lane] = 0.0;
        cp[lane] = 0;
        if (y >= ny || x < 0 || x >= nx) continue;
        const int64_t f = x + static_cast<int64_t>(y) * nx + z * nxy;
        const int64_t i = BWD ? n - 1 - f : f;
        const int32_t pos = pos_of[i];
        cp[lane] = pos;
        int32_t e = prs[pos];
        const int32_t e_end = prs[pos + 1];
        for (int q = 0; q < S; ++q) {
            const int sl = BWD ? S - 1 - q : q;
            int dx, dy, dz;
            if (ST == 27) {
                if (sl < 9) {
                    dz = -1;
                    dy = sl / 3 - 1;
                    dx = sl % 3 - 1;
                } else if (sl < 12) {
                    dz = 0;
                    dy = -1;
                    dx = sl - 10;
                } else {
                    dz = 0;
                    dy = 0;
                    dx = -1;
                }
            } else {
                dz = sl == 0 ? -1 : 0;
                dy = sl == 1 ? -1 : 0;
                dx = sl == 2 ? -1 : 0;
            }
            if (x + dx < 0 || x + dx >= nx || y + dy < 0 || y + dy >= ny || z + dz < 0 || z + dz >= nz) continue;
            const int64_t fp = f + dx + static_cast<int64_t>(dy) * nx + dz * nxy;
            const int64_t col = BWD ? n - 1 - fp : fp;
            if (e >= e_end || pcol[e] != col) {
                atomicExch(bad, 1);
                break;
            }
            coef[sl * 32 + lane] = pval[e];
            ++e;
        }
        if (e != e_end) atomicExch(bad, 1);
    }
}

__global__ void k_ps_pos_of(const int32_t* __restrict__ perm, int32_t npos, int32_t* __restrict__ pos_of) {
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < npos;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t r = perm[p];
        if (r >= 0) pos_of[r] = static_cast<int32_t>(p);
    }
}

// (r, z) per 32-position tile of the backward schedule, warp_sum order of k_sweep's tile_reduce
__global__ void __launch_bounds__(256) k_tile_partials(const double* __restrict__ cbuf, int ntiles,
                                                       double* __restrict__ partials, const DevState* st) {
    if (st->done) return;
    const int lane = threadIdx.x & 31;
    for (int t = blockIdx.x * 8 + (threadIdx.x >> 5); t < ntiles; t += gridDim.x * 8) {
        const double v = warp_sum(cbuf[static_cast<int64_t>(t) * 32 + lane]);
        if (lane == 0) partials[t] = v;
    }
}

__global__ void __launch_bounds__(256) k_level_groups(const double* __restrict__ partials, double* __restrict__ gpart,
                                                      int ntiles, const DevState* st);  // icsweep_lv.cu
__global__ void k_level_total(const double* __restrict__ gpart, int ntiles, DevState* st, int add_sc);

// ------------------------------------------------------------------ host
struct PencilPlan {
    int st = 0;  // 0 off, 7 or 27
    int32_t nx = 0, ny = 0, nz = 0, nb = 0, nt = 0, units = 0;
    unsigned char* recs[2] = {nullptr, nullptr};
    double* cbuf = nullptr;  // backward-schedule positions (+ padding: zeros)
};

static size_t ps_smem_bytes(int st) { return static_cast<size_t>(kPsWarps) * (16 * kPsStages + kPsStages * ps_rec_bytes(st == 27 ? 13 : 3)); }

template <int ST, bool BWD>
static const void* ps_kernel() {
    return reinterpret_cast<const void*>(k_psweep<ST, BWD>);
}

void pencil_plan_free(rcg_ic* f) {
    if (!f->pencil) return;
    dev_free(f->pencil->recs[0]);
    dev_free(f->pencil->recs[1]);
    dev_free(f->pencil->cbuf);
    delete f->pencil;
    f->pencil = nullptr;
}

// Detect a natural-ordered nx x ny x nz box grid with the 7- or 27-point pattern (dims given, or
// a cube n = N^3) and build both directions' records.  Silently off when the pattern does not
// match (multicolour or block-Jacobi factors, kNN) or the records would not fit in HBM.
void pencil_plan_build(rcg_ctx* ctx, rcg_ic* f, int32_t nx, int32_t ny, int32_t nz) {
    pencil_plan_free(f);
    if (const char* e = std::getenv("RCG_PSWEEP"); e && std::atoi(e) == 0) return;
    const int64_t n = f->n;
    if (n <= 0) return;
    if (nx <= 0) {
        const int32_t N = static_cast<int32_t>(std::llround(std::cbrt(static_cast<double>(n))));
        if (static_cast<int64_t>(N) * N * N != n) return;
        nx = ny = nz = N;
    }
    if (static_cast<int64_t>(nx) * ny * nz != n) return;
    const double per_row = f->nnz_l / static_cast<double>(n);
    int st = 0;
    if (per_row > 2.0 && per_row <= 3.0) st = 7;
    else if (per_row > 10.0 && per_row <= 13.0) st = 27;
    if (!st) return;
    auto* p = new PencilPlan();
    p->st = st;
    p->nx = nx;
    p->ny = ny;
    p->nz = nz;
    p->nb = (ny + 31) / 32;
    p->nt = nx + (st == 27 ? 2 : 1) * 31;
    p->units = nz * p->nb;
    const int64_t rec = ps_rec_bytes(st == 27 ? 13 : 3);
    const int64_t bytes = static_cast<int64_t>(p->units) * p->nt * rec;
    int64_t ntiles_b = (f->b_npos + 31) / 32;
    size_t free_b = 0, total_b = 0;
    RCG_CK(cudaMemGetInfo(&free_b, &total_b));
    // leave room for the solve's workspaces / deflation blocks (records are an accelerator only)
    if (static_cast<double>(2 * bytes) > 0.35 * static_cast<double>(free_b)) {
        delete p;
        return;
    }
    int32_t* pos_of = nullptr;
    int* bad = nullptr;
    try {
        p->recs[0] = static_cast<unsigned char*>(dev_alloc_bytes(bytes));
        p->recs[1] = static_cast<unsigned char*>(dev_alloc_bytes(bytes));
        p->cbuf = dev_alloc(ntiles_b * 32);
        pos_of = static_cast<int32_t*>(dev_alloc_bytes(sizeof(int32_t) * n));
        bad = static_cast<int*>(dev_alloc_bytes(sizeof(int)));
        RCG_CK(cudaMemsetAsync(p->cbuf, 0, sizeof(double) * ntiles_b * 32, ctx->stream));
        RCG_CK(cudaMemsetAsync(bad, 0, sizeof(int), ctx->stream));
        const int g = std::max(1, std::min<int>(static_cast<int>((n + 255) / 256), ctx->num_sms * 8));
        const int gb = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((static_cast<int64_t>(p->units) * p->nt * 32 + 255) / 256,
                                                     ctx->num_sms * 16)));
        for (int dir = 0; dir < 2; ++dir) {
            const bool bwd = dir == 1;
            k_ps_pos_of<<<g, 256, 0, ctx->stream>>>(bwd ? f->b_perm : f->f_perm, bwd ? f->b_npos : f->f_npos, pos_of);
            RCG_LAUNCHED(ctx);
            const int32_t* prs = bwd ? f->b_prs : f->f_prs;
            const int32_t* pcol = bwd ? f->b_col : f->f_col;
            const double* pval = bwd ? f->b_val : f->f_val;
#define RCG_PS_BUILD(STV, B)                                                                                    \
    k_ps_build<STV, B><<<gb, 256, 0, ctx->stream>>>(p->recs[dir], nx, ny, nz, p->nb, p->nt, p->units, n, pos_of, \
                                                     prs, pcol, pval, bad)
            if (st == 27) {
                if (bwd) RCG_PS_BUILD(27, true);
                else RCG_PS_BUILD(27, false);
            } else {
                if (bwd) RCG_PS_BUILD(7, true);
                else RCG_PS_BUILD(7, false);
            }
#undef RCG_PS_BUILD
            RCG_LAUNCHED(ctx);
        }
        int hbad = 0;
        RCG_CK(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        RCG_CK(cudaStreamSynchronize(ctx->stream));
        dev_free(pos_of);
        dev_free(bad);
        pos_of = nullptr;
        bad = nullptr;
        f->pencil = p;
        if (hbad) pencil_plan_free(f);
    } catch (...) {
        dev_free(pos_of);
        dev_free(bad);
        f->pencil = p;
        pencil_plan_free(f);
        throw;
    }
}

bool pencil_available(const rcg_ctx* ctx, const rcg_ic* f) {
    return f->pencil != nullptr && (ctx->sweep_cluster == 2 || ctx->sweep_cluster == 5);
}

// warps per SM: about the width of the wavefront (units in flight beyond it only spin)
static int ps_warps_per_sm(const rcg_ctx* ctx, const PencilPlan& p) {
    if (const char* e = std::getenv("RCG_PSWEEP_WPS")) return std::max(1, std::atoi(e));
    const double levels = p.st == 27 ? (p.nx + 2.0 * p.ny + 4.0 * p.nz) : (1.0 * p.nx + p.ny + p.nz);
    const double active = p.units * static_cast<double>(p.nt) / levels;
    return std::max(2, std::min(16, static_cast<int>(std::ceil(1.25 * active / ctx->num_sms))));
}

void launch_pencil_sweep(rcg_ctx* ctx, const rcg_ic* f, bool backward, SweepArgs& a) {
    const PencilPlan& p = *f->pencil;
    static bool prepared = false;
    if (!prepared) {
        for (const void* k : {ps_kernel<27, false>(), ps_kernel<27, true>(), ps_kernel<7, false>(), ps_kernel<7, true>()}) {
            RCG_CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(ps_smem_bytes(27))));
        }
        prepared = true;
    }
    PsArgs q{};
    q.recs = p.recs[backward ? 1 : 0];
    q.nx = p.nx;
    q.ny = p.ny;
    q.nz = p.nz;
    q.nb = p.nb;
    q.nt = p.nt;
    q.units = p.units;
    q.n = f->n;
    q.in = a.in;
    q.d = a.d;
    q.r = a.r;
    q.out = a.out;
    q.cbuf = p.cbuf;
    q.tickets = a.tickets;
    q.st = a.st;
    const size_t smem = ps_smem_bytes(p.st);
    int occ = 0;
    const void* kern = p.st == 27 ? (backward ? ps_kernel<27, true>() : ps_kernel<27, false>())
                                  : (backward ? ps_kernel<7, true>() : ps_kernel<7, false>());
    RCG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kPsWarps * 32, smem));
    const int want_ctas_per_sm = std::max(1, (ps_warps_per_sm(ctx, p) + kPsWarps - 1) / kPsWarps);
    const int per_sm = std::max(1, std::min(occ, want_ctas_per_sm));
    const int grid = std::max(1, std::min((p.units + kPsWarps - 1) / kPsWarps, ctx->num_sms * per_sm));
    {
        KTimer t(ctx, backward ? 2 : 1);
        if (p.st == 27) {
            if (backward) k_psweep<27, true><<<grid, kPsWarps * 32, smem, ctx->stream>>>(q);
            else k_psweep<27, false><<<grid, kPsWarps * 32, smem, ctx->stream>>>(q);
        } else {
            if (backward) k_psweep<7, true><<<grid, kPsWarps * 32, smem, ctx->stream>>>(q);
            else k_psweep<7, false><<<grid, kPsWarps * 32, smem, ctx->stream>>>(q);
        }
        RCG_LAUNCHED(ctx);
        if (backward && a.r) {
            const int ntiles = static_cast<int>((f->b_npos + 31) / 32);
            const int gt = std::max(1, std::min((ntiles + 7) / 8, ctx->num_sms * 8));
            k_tile_partials<<<gt, 256, 0, ctx->stream>>>(p.cbuf, ntiles, a.partials, a.st);
            RCG_LAUNCHED(ctx);
            const int ngroups = (ntiles + kGroup - 1) / kGroup;
            k_level_groups<<<(ngroups + 7) / 8, 256, 0, ctx->stream>>>(a.partials, a.gpart, ntiles, a.st);
            RCG_LAUNCHED(ctx);
            k_level_total<<<1, 32, 0, ctx->stream>>>(a.gpart, ntiles, a.st, a.add_sc);
            RCG_LAUNCHED(ctx);
        }
    }
}

}  // namespace rcg

using namespace rcg;

extern "C" int rcg_ic_pencil(const rcg_ic* f, int* stencil) {
    return guard([&] {
        require(f && stencil, "rcg_ic_pencil: null argument");
        *stencil = f->pencil ? f->pencil->st : 0;
    });
}
