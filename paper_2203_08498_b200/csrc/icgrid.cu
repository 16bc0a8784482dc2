// icgrid.cu -- tiled IC(0) sweeps for matrices in the natural ordering of a 3D grid (C1-C4).
//
// The level-scheduled sweep (icsweep.cu) pays one inter-SM publish -> observe hop per DAG level
// (~1.1 us, 382 levels at 128^3).  On a grid, most of those dependencies can stay inside one
// SM: a CTA owns an (x, y) tile for all z, one thread per (x, y) column, and the threads walk
// their columns in steps of a level function L = wx x + wy y + wz z under which every factor
// entry's parent has a smaller L (checked for every entry on the host: (1,1,1) for the 7-point
// stencil, (1,2,4) for the 27-point one).  One step is a CTA barrier; in-tile parents come from
// a 2-plane shared-memory ring (column c holds its last two z values), only parents in another
// tile are polled in HBM (the same NaN-sentinel value-as-flag protocol as the level sweep).
// The cross-SM hops drop from one per level to one per tile boundary on the critical path.
// Row arithmetic is exactly the reference loop's (ic_preconditioner.cpp:130-143), so the
// result is bitwise that of the level sweep.
//
// Status (B200, C2 128^3): bitwise correct on every grid config, but slower than the
// level sweep (709 / 831 us vs 480 / 490 us with 32 x 8 tiles): a step costs ~950 cycles for the
// barrier + dependent shared-memory / FP64 chain alone and ~1,500 more for the cp.async staging,
// so ~400 steps do not beat ~400 hops.  Opt-in (rcg_ic_set_grid); off by default.
//
// Deadlock freedom: tiles are handed out in order of their first level.  If every cross-tile
// dependency points to an earlier tile (7-point), persistent CTAs over that order are safe;
// otherwise (27-point: parents at (x+1, y+1, z-1)) every tile must be resident at once, which
// rcg_ic_set_grid checks with the occupancy API (else the level sweep stays in use).
#include <algorithm>
#include <array>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "internal.cuh"
#include "kernels.cuh"

namespace rcg {

constexpr int kMaxSlots = 16;


struct GridArgs {
    int32_t nx, ny, nz;
    int tx, ty, wx, wy, wz, ntiles, nslots;
    int8_t sdx[kMaxSlots], sdy[kMaxSlots], sdz[kMaxSlots];  // slot -> parent offset (row - parent fwd, parent - row bwd)
    const double* coef;        // [slot][n]: the row's factor entry for stencil slot (ascending columns)
    const uint32_t* mask;      // [n]: slots present in the row
    const int32_t* tile_xy;    // ticket -> X | Y << 16 (ascending first level)
    const double* d;
    const double* in;
    double* out;
    const double* r;           // backward: (r, z) tile partials when non-null
    double* tpart;
    int* tickets;              // [0] tile ticket, [1] exit count, [3] watchdog
    DevState* st;
    long long* prof;           // RCG_GRID_PROF builds: cycle counters
};

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

template <int NS>
__host__ __device__ constexpr int grid_fields() { return 2 * NS + 3; }  // coef[NS], in, d, r, parent[NS]

// One thread per (x, y) column.  Each thread stages its own column's next rows -- mask,
// coefficients, input, pivot, residual and the values of the parents in other tiles -- into a
// double-buffered shared-memory chunk of Z rows with cp.async (no registers held, no waits
// until the chunk is reached); a staged parent that was still the sentinel is polled again.
// A step is then a CTA barrier plus shared-memory reads.
template <bool BWD, int NS, int Z>
__global__ void __launch_bounds__(512) k_sweep_grid(GridArgs a) {
    extern __shared__ double sm[];
    __shared__ int s_tile;
    __shared__ double red[32];
    if (a.st->done) return;
    constexpr int F = grid_fields<NS>();
    const int T = a.tx * a.ty;
    double* ring = sm;                                                   // [2][T]
    double* stage = ring + 2 * T;                                        // [2][Z][F][T]
    uint32_t* smask = reinterpret_cast<uint32_t*>(stage + 2 * Z * F * T);  // [2][Z][T]
    const int t = threadIdx.x;
    const int lx = t % a.tx, ly = t / a.tx;
    const int32_t nxy = a.nx * a.ny;
    const int sg = BWD ? 1 : -1;
    const int64_t slot_stride = static_cast<int64_t>(nxy) * a.nz;
    unsigned spins = 0;
    while (true) {
        __syncthreads();
        if (t == 0) s_tile = atomicAdd(&a.tickets[0], 1);
        __syncthreads();
        const int k = s_tile;
        if (k >= a.ntiles) break;
        const int packed = __ldg(a.tile_xy + (BWD ? a.ntiles - 1 - k : k));
        const int x0 = (packed & 0xffff) * a.tx, y0 = (packed >> 16) * a.ty;
        const int tw = min(a.tx, a.nx - x0), th = min(a.ty, a.ny - y0);
        const int x = x0 + lx, y = y0 + ly;
        const bool active = lx < tw && ly < th;
        const int lmin = a.wx * x0 + a.wy * y0;
        const int lmax = a.wx * (x0 + tw - 1) + a.wy * (y0 + th - 1) + a.wz * (a.nz - 1);
        const int base = a.wx * x + a.wy * y;
        unsigned ext = 0;  // slots whose parent column is outside this tile (or the domain)
#pragma unroll
        for (int q = 0; q < NS; ++q) {
            const int px = x + sg * a.sdx[q], py = y + sg * a.sdy[q];
            if (!(px >= x0 && px < x0 + tw && py >= y0 && py < y0 + th)) ext |= 1u << q;
        }
        // stage chunk c (rows zi = c Z .. c Z + Z - 1 in processing order) into buffer c & 1
        auto issue = [&](int c) {
            if (active)
                for (int r = 0; r < Z; ++r) {
                    const int zi = c * Z + r;
                    if (zi >= a.nz) break;
                    const int z = BWD ? a.nz - 1 - zi : zi;
                    const int32_t i = x + a.nx * y + nxy * z;
                    double* st = stage + ((static_cast<int64_t>(c & 1) * Z + r) * F) * T + t;
                    cp_async4(smask + (static_cast<int64_t>(c & 1) * Z + r) * T + t, a.mask + i);
#pragma unroll
                    for (int q = 0; q < NS; ++q) cp_async8(st + q * T, a.coef + q * slot_stride + i);
                    cp_async8(st + NS * T, a.in + i);
                    if (BWD) {
                        cp_async8(st + (NS + 1) * T, a.d + i);
                        if (a.r) cp_async8(st + (NS + 2) * T, a.r + i);
                    }
#pragma unroll
                    for (int q = 0; q < NS; ++q)
                        if ((ext >> q) & 1) {
                            const int px = x + sg * a.sdx[q], py = y + sg * a.sdy[q], pz = z + sg * a.sdz[q];
                            if (px >= 0 && px < a.nx && py >= 0 && py < a.ny && pz >= 0 && pz < a.nz)
                                cp_async8(st + (NS + 3 + q) * T, a.out + (px + a.nx * py + nxy * pz));
                        }
                }
            cp_async_commit();  // one group per chunk (possibly empty): wait_group 1 = "chunk c landed"
        };
        issue(0);
        issue(1);
        double contrib = 0.0;
#ifdef RCG_GRID_PROF
        const long long tstart = clock64();
#endif
        for (int step = 0; step <= lmax - lmin; ++step) {
            const int L = BWD ? lmax - step : lmin + step;
            const int rem = L - base;
            if (active && rem >= 0 && rem % a.wz == 0 && rem / a.wz < a.nz) {
                const int z = rem / a.wz;
                const int zi = BWD ? a.nz - 1 - z : z;
                const int c = zi / Z, r = zi - c * Z;
                if (r == 0) cp_async_wait1();
                const double* st = stage + ((static_cast<int64_t>(c & 1) * Z + r) * F) * T + t;
                const uint32_t m = smask[(static_cast<int64_t>(c & 1) * Z + r) * T + t];
                const int32_t i = x + a.nx * y + nxy * z;
                double sv = BWD ? __ddiv_rn(st[NS * T], st[(NS + 1) * T]) : st[NS * T];
#pragma unroll
                for (int q = 0; q < NS; ++q) {
                    if (!((m >> q) & 1)) continue;
                    const int px = x + sg * a.sdx[q], py = y + sg * a.sdy[q], pz = z + sg * a.sdz[q];
                    double pv;
                    if (!((ext >> q) & 1)) {
                        pv = ring[(pz & 1) * T + (py - y0) * a.tx + (px - x0)];
                    } else {
                        pv = st[(NS + 3 + q) * T];
                        if (is_sentinel(pv)) {
                            const int32_t j = px + a.nx * py + nxy * pz;
                            do {
                                if (++spins == (1u << 26)) {  // bounded: a schedule fault is an error
                                    atomicExch(&a.tickets[3], 1);
                                    pv = 0.0;
                                    break;
                                }
                                pv = ld_relaxed(a.out + j);
                            } while (is_sentinel(pv));
                        }
                    }
                    sv = fsub_mul(sv, st[q * T], pv);
                }
                st_relaxed(a.out + i, publishable(sv));
                ring[(z & 1) * T + ly * a.tx + lx] = sv;
                if (BWD && a.r) contrib = fadd_mul(contrib, st[(NS + 2) * T], sv);
                if (r == Z - 1) issue(c + 2);  // this buffer is free again
            }
            __syncthreads();
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
#ifdef RCG_GRID_PROF
        if (t == 0 && (k == 0 || k == a.ntiles - 1)) {
            a.prof[k == 0 ? 0 : 2] += clock64() - tstart;
            a.prof[k == 0 ? 1 : 3] += lmax - lmin + 1;
        }
#endif
        if (BWD && a.r) {  // this tile's (r, z) partial, fixed order
            double acc[1] = {contrib};
            block_sum<1>(acc, red);
            if (t == 0) a.tpart[BWD ? a.ntiles - 1 - k : k] = acc[0];
        }
    }
    if (t == 0) {
        __threadfence();
        if (atomicAdd(&a.tickets[1], 1) == static_cast<int>(gridDim.x) - 1) {
            a.tickets[0] = 0;
            a.tickets[1] = 0;
        }
    }
}

// (r, z) = sum of the tile partials in tile order; finaliser as the level sweep's (pcg.cpp:65-71)
__global__ void k_grid_rho(const double* __restrict__ tpart, int ntiles, DevState* st, int add_sc) {
    __shared__ double red[32];
    if (st->done) return;
    double acc[1] = {0.0};
    for (int q = threadIdx.x; q < ntiles; q += blockDim.x) acc[0] = __dadd_rn(acc[0], tpart[q]);
    block_sum<1>(acc, red);
    if (threadIdx.x == 0) {
        const double rho = add_sc ? acc[0] + st->scal[2] : acc[0];
        st->rho = rho;
        if (rho <= 0.0) {
            st->done = kBroken;
            st->status = kBrkRz;
        }
        st->beta = st->iter > 1 ? rho / st->rho_prev : 0.0;
    }
}

bool grid_sweep_available(const rcg_ic* f) { return f->grid.on; }

constexpr int kZ3 = 4, kZ13 = 2;  // staged rows per chunk (7-point / 27-point stencils)

template <int NS, int Z>
static size_t grid_smem(int threads) {
    return sizeof(double) * (2 + 2 * Z * grid_fields<NS>()) * threads + sizeof(uint32_t) * 2 * Z * threads;
}

template <bool BWD>
static void launch_grid(const GridArgs& a, int grid, int threads, cudaStream_t s) {
    if (a.nslots <= 3)
        k_sweep_grid<BWD, 3, kZ3><<<grid, threads, grid_smem<3, kZ3>(threads), s>>>(a);
    else if (a.nslots <= 13)
        k_sweep_grid<BWD, 13, kZ13><<<grid, threads, grid_smem<13, kZ13>(threads), s>>>(a);
    else
        k_sweep_grid<BWD, 16, kZ13><<<grid, threads, grid_smem<16, kZ13>(threads), s>>>(a);
}

void launch_grid_sweep(rcg_ctx* ctx, const rcg_ic* f, bool backward, SweepArgs& sa) {
    const GridSched& g = f->grid;
    GridArgs a{};
    a.nx = g.nx;
    a.ny = g.ny;
    a.nz = g.nz;
    a.tx = g.tx;
    a.ty = g.ty;
    a.wx = g.wx;
    a.wy = g.wy;
    a.wz = g.wz;
    a.ntiles = g.ntiles;
    const int dir = backward ? 1 : 0;
    a.nslots = g.nslots[dir];
    for (int q = 0; q < kMaxSlots; ++q) {
        a.sdx[q] = g.sdx[dir][q];
        a.sdy[q] = g.sdy[dir][q];
        a.sdz[q] = g.sdz[dir][q];
    }
    a.coef = g.coef[dir];
    a.mask = g.mask[dir];
    a.tile_xy = g.tile_xy;
    a.d = sa.d;
    a.in = sa.in;
    a.out = sa.out;
    a.r = sa.r;
    a.tpart = sa.partials;
    a.tickets = sa.tickets;
    a.st = sa.st;
#ifdef RCG_GRID_PROF
    static long long* prof = nullptr;
    if (!prof) {
        cudaMalloc(&prof, 64);
        cudaMemset(prof, 0, 64);
    }
    a.prof = prof;
    if (std::getenv("RCG_GRID_PROF_DUMP")) {
        long long h[4];
        cudaMemcpy(h, prof, 32, cudaMemcpyDeviceToHost);
        std::fprintf(stderr, "[grid prof] comp %lld load %lld bar %lld steps %lld\n", h[0], h[1], h[2], h[3]);
    }
#endif
    const int threads = g.tx * g.ty;
    const int grid = std::min(g.ntiles, g.max_ctas);
    KTimer t(ctx, backward ? 2 : 1);
    if (backward)
        launch_grid<true>(a, grid, threads, ctx->stream);
    else
        launch_grid<false>(a, grid, threads, ctx->stream);
    RCG_LAUNCHED(ctx);
    if (backward && sa.r) {
        k_grid_rho<<<1, 256, 0, ctx->stream>>>(sa.partials, g.ntiles, sa.st, sa.add_sc);
        RCG_LAUNCHED(ctx);
    }
}

template <bool BWD, int NS, int Z>
static int occupancy_one(int threads) {
    const void* fn = reinterpret_cast<const void*>(k_sweep_grid<BWD, NS, Z>);
    const size_t smem = grid_smem<NS, Z>(threads);
    int dev = 0, optin = 0;
    RCG_CK(cudaGetDevice(&dev));
    RCG_CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    if (smem > static_cast<size_t>(optin)) return 0;
    RCG_CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    int nb = 0;
    RCG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_sweep_grid<BWD, NS, Z>, threads, smem));
    return nb;
}

template <bool BWD>
static int occupancy(int threads, int nslots) {
    if (nslots <= 3) return occupancy_one<BWD, 3, kZ3>(threads);
    if (nslots <= 13) return occupancy_one<BWD, 13, kZ13>(threads);
    return occupancy_one<BWD, 16, kZ13>(threads);
}

static void free_grid(GridSched& g) {
    for (void* p : {(void*)g.tile_xy, (void*)g.coef[0], (void*)g.coef[1], (void*)g.mask[0], (void*)g.mask[1]})
        dev_free(p);
    g.tile_xy = nullptr;
    g.coef[0] = g.coef[1] = nullptr;
    g.mask[0] = g.mask[1] = nullptr;
    g.on = false;
}

// host: stencil slots of one triangle (forward L: parent = row - delta; backward U: parent =
// row + delta), ordered by ascending column; every row's entries must be distinct slots in
// ascending slot order (then applying the slots in order IS the reference's entry order)
static bool build_slots(const rcg_ic* f, bool upper, int32_t nx, int32_t ny, std::vector<int>& dxs,
                        std::vector<int>& dys, std::vector<int>& dzs, std::vector<uint32_t>& mask,
                        std::vector<double>& coef) {
    const int32_t n = f->n;
    const int64_t nxy = static_cast<int64_t>(nx) * ny;
    const std::vector<int32_t>& rs = upper ? f->h_urs : f->h_lrs;
    const std::vector<int32_t>& col = upper ? f->h_ucol : f->h_lcol;
    const std::vector<double>& val = upper ? f->h_uval : f->h_lval;
    auto coord = [&](int64_t i, int& x, int& y, int& z) {
        z = static_cast<int>(i / nxy);
        const int64_t r = i - z * nxy;
        y = static_cast<int>(r / nx);
        x = static_cast<int>(r - static_cast<int64_t>(y) * nx);
    };
    std::vector<std::array<int, 3>> deltas;
    for (int32_t i = 0; i < n; ++i)
        for (int32_t e = rs[i]; e < rs[i + 1]; ++e) {
            int x, y, z, px, py, pz;
            coord(i, x, y, z);
            coord(col[e], px, py, pz);
            const std::array<int, 3> dlt = upper ? std::array<int, 3>{px - x, py - y, pz - z}
                                                 : std::array<int, 3>{x - px, y - py, z - pz};
            if (std::find(deltas.begin(), deltas.end(), dlt) == deltas.end()) {
                if (deltas.size() == kMaxSlots) return false;
                deltas.push_back(dlt);
            }
        }
    auto off = [&](const std::array<int, 3>& d) { return d[0] + static_cast<int64_t>(nx) * d[1] + nxy * d[2]; };
    // ascending column: forward (parent = row - off) descending offset; backward ascending
    std::sort(deltas.begin(), deltas.end(),
              [&](const std::array<int, 3>& a, const std::array<int, 3>& b) { return upper ? off(a) < off(b) : off(a) > off(b); });
    for (size_t q = 0; q < deltas.size(); ++q)
        if (std::abs(deltas[q][0]) > 1 || std::abs(deltas[q][1]) > 1 || deltas[q][2] < 0 || deltas[q][2] > 1) return false;
    const size_t ns = deltas.size();
    mask.assign(n, 0);
    coef.assign(ns * static_cast<size_t>(n), 0.0);
    for (int32_t i = 0; i < n; ++i) {
        int last = -1;
        for (int32_t e = rs[i]; e < rs[i + 1]; ++e) {
            int x, y, z, px, py, pz;
            coord(i, x, y, z);
            coord(col[e], px, py, pz);
            const std::array<int, 3> dlt = upper ? std::array<int, 3>{px - x, py - y, pz - z}
                                                 : std::array<int, 3>{x - px, y - py, z - pz};
            const int q = static_cast<int>(std::find(deltas.begin(), deltas.end(), dlt) - deltas.begin());
            if (q <= last) return false;  // entry order must be slot order
            last = q;
            mask[i] |= 1u << q;
            coef[static_cast<size_t>(q) * n + i] = val[e];
        }
    }
    dxs.resize(ns);
    dys.resize(ns);
    dzs.resize(ns);
    for (size_t q = 0; q < ns; ++q) {
        dxs[q] = deltas[q][0];
        dys[q] = deltas[q][1];
        dzs[q] = deltas[q][2];
    }
    return true;
}

// host: choose the level function, check it against every factor entry (parents strictly
// earlier; the 2-plane ring never overwritten before its last in-tile reader), order the
// tiles, decide persistent vs co-resident, build the stencil layout, upload
static void grid_setup(rcg_ctx* ctx, rcg_ic* f, int32_t nx, int32_t ny, int32_t nz, int tx, int ty) {
    require(nx >= 1 && ny >= 1 && nz >= 1 && static_cast<int64_t>(nx) * ny * nz == f->n,
            "rcg_ic_set_grid: nx * ny * nz must equal the factor's n");
    require(tx >= 1 && ty >= 1 && tx * ty <= 512 && tx * ty % 32 == 0,
            "rcg_ic_set_grid: tile must hold a multiple of 32 columns, at most 512");
    require(nx < 65536 * tx && ny < 65536 * ty, "rcg_ic_set_grid: too many tiles");
    ensure_host_image(f);
    GridSched& g = f->grid;
    free_grid(g);
    std::vector<int> dx[2], dy[2], dz[2];
    std::vector<uint32_t> mask[2];
    std::vector<double> coef[2];
    for (int dir = 0; dir < 2; ++dir)
        require(build_slots(f, dir == 1, nx, ny, dx[dir], dy[dir], dz[dir], mask[dir], coef[dir]),
                "rcg_ic_set_grid: the factor's pattern is not a supported grid stencil in natural order");
    // level function: every forward slot's parent strictly earlier, and the 2-plane ring slot of
    // the parent's column not rewritten (plane pz + 2) before the row
    const int weights[2][3] = {{1, 1, 1}, {1, 2, 4}};
    int wsel = -1;
    for (int c = 0; c < 2 && wsel < 0; ++c) {
        bool ok = true;
        for (size_t q = 0; q < dx[0].size() && ok; ++q) {
            const int dl = weights[c][0] * dx[0][q] + weights[c][1] * dy[0][q] + weights[c][2] * dz[0][q];  // L(row) - L(parent)
            ok = dl > 0 && 2 * weights[c][2] > dl;
        }
        if (ok) wsel = c;
    }
    require(wsel >= 0, "rcg_ic_set_grid: no supported level function for this stencil");
    require(std::max(dx[0].size(), dx[1].size()) <= 3 || tx * ty <= 256,
            "rcg_ic_set_grid: tiles of a stencil with more than 3 lower entries hold at most 256 columns");
    g.nx = nx;
    g.ny = ny;
    g.nz = nz;
    g.tx = tx;
    g.ty = ty;
    g.wx = weights[wsel][0];
    g.wy = weights[wsel][1];
    g.wz = weights[wsel][2];
    for (int dir = 0; dir < 2; ++dir) {
        g.nslots[dir] = static_cast<int>(dx[dir].size());
        for (int q = 0; q < kMaxSlots; ++q) {
            g.sdx[dir][q] = q < g.nslots[dir] ? static_cast<int8_t>(dx[dir][q]) : 0;
            g.sdy[dir][q] = q < g.nslots[dir] ? static_cast<int8_t>(dy[dir][q]) : 0;
            g.sdz[dir][q] = q < g.nslots[dir] ? static_cast<int8_t>(dz[dir][q]) : 0;
        }
    }
    const int TX = (nx + tx - 1) / tx, TY = (ny + ty - 1) / ty;
    g.ntiles = TX * TY;
    std::vector<int> order(g.ntiles);
    for (int q = 0; q < g.ntiles; ++q) order[q] = q;
    auto lmin = [&](int q) { return g.wx * (q % TX) * tx + g.wy * (q / TX) * ty; };
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return lmin(a) < lmin(b); });
    std::vector<int> xy(g.ntiles);
    for (int k = 0; k < g.ntiles; ++k) xy[k] = (order[k] % TX) | ((order[k] / TX) << 16);
    // persistent CTAs are deadlock-free when every forward parent lies in this tile or in one
    // with a smaller first level (a tile neighbour at -x / -y only); else all tiles co-resident
    bool one_way = true;
    for (size_t q = 0; q < dx[0].size(); ++q)
        if (dx[0][q] < 0 || dy[0][q] < 0) one_way = false;  // parent at +x or +y of the row
    const int threads = tx * ty;
    const int resident = std::min(occupancy<true>(threads, g.nslots[1]), occupancy<false>(threads, g.nslots[0])) * ctx->num_sms;
    require(resident >= 1, "rcg_ic_set_grid: the tile does not fit on an SM");
    if (!one_way)
        require(g.ntiles <= resident, "rcg_ic_set_grid: tiles depend on each other both ways and do not all fit "
                                      "on the GPU at once (use larger tiles)");
    g.max_ctas = one_way ? resident : g.ntiles;
    g.tile_xy = static_cast<int32_t*>(dev_alloc_bytes(sizeof(int32_t) * g.ntiles));
    RCG_CK(cudaMemcpyAsync(g.tile_xy, xy.data(), sizeof(int32_t) * g.ntiles, cudaMemcpyHostToDevice, ctx->stream));
    for (int dir = 0; dir < 2; ++dir) {
        g.coef[dir] = dev_alloc(std::max<int64_t>(static_cast<int64_t>(coef[dir].size()), 1));
        g.mask[dir] = static_cast<uint32_t*>(dev_alloc_bytes(sizeof(uint32_t) * std::max<size_t>(mask[dir].size(), 1)));
        if (!coef[dir].empty())
            RCG_CK(cudaMemcpyAsync(g.coef[dir], coef[dir].data(), sizeof(double) * coef[dir].size(),
                                   cudaMemcpyHostToDevice, ctx->stream));
        RCG_CK(cudaMemcpyAsync(g.mask[dir], mask[dir].data(), sizeof(uint32_t) * mask[dir].size(),
                               cudaMemcpyHostToDevice, ctx->stream));
    }
    RCG_CK(cudaStreamSynchronize(ctx->stream));
    g.on = true;
}

}  // namespace rcg

using namespace rcg;

extern "C" int rcg_ic_set_grid(rcg_ctx* ctx, rcg_ic* f, int32_t nx, int32_t ny, int32_t nz, int tile_x, int tile_y) {
    return guard([&] {
        require(ctx && f, "rcg_ic_set_grid: null argument");
        if (tile_x == 0) {  // off: back to the level-scheduled sweeps
            f->grid.on = false;
            return;
        }
        grid_setup(ctx, f, nx, ny, nz, tile_x, tile_y);
    });
}
