// generators.cpp -- seeded synthetic inputs for the BASELINE.json configurations (the reference
// ships no generators; SURVEY.md section 8(d) fixes their definitions).  Host code: it runs
// once per problem and feeds the GPU path, the oracle harness and bench.py identically.
//
// All matrices are full-symmetric CSR in natural lexicographic order (x fastest), columns
// ascending, Dirichlet boundary eliminated.  Random numbers come from std::mt19937_64 (fully
// specified by the C++ standard) mapped like the reference's UniformPm1 (include/recycg/rng.hpp).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

#include "gen_math.h"
#include "host_error.h"

namespace rcg {
namespace {

inline double u01(std::mt19937_64& g) { return static_cast<double>(g() >> 11) * 0x1.0p-53; }

struct Csr {
    int32_t n = 0;
    std::vector<int32_t> rs, ci;
    std::vector<double> va;
};

// ---- C1: 7-point Laplacian, diagonal 6, off-diagonals -1
Csr poisson7(int32_t N) {
    Csr a;
    const int64_t n = static_cast<int64_t>(N) * N * N;
    require(n < (1LL << 31), "generator: grid too large for int32 rows");
    a.n = static_cast<int32_t>(n);
    a.rs.resize(n + 1);
    a.ci.reserve(7 * n);
    a.va.reserve(7 * n);
    const int64_t sy = N, sz = static_cast<int64_t>(N) * N;
    for (int z = 0; z < N; ++z)
        for (int y = 0; y < N; ++y)
            for (int x = 0; x < N; ++x) {
                const int64_t i = x + sy * y + sz * z;
                a.rs[i] = static_cast<int32_t>(a.ci.size());
                auto put = [&](int64_t j, double v) {
                    a.ci.push_back(static_cast<int32_t>(j));
                    a.va.push_back(v);
                };
                if (z > 0) put(i - sz, -1.0);
                if (y > 0) put(i - sy, -1.0);
                if (x > 0) put(i - 1, -1.0);
                put(i, 6.0);
                if (x < N - 1) put(i + 1, -1.0);
                if (y < N - 1) put(i + sy, -1.0);
                if (z < N - 1) put(i + sz, -1.0);
            }
    a.rs[n] = static_cast<int32_t>(a.ci.size());
    return a;
}

// ---- C2 / C4: 7-point with harmonic-mean edge coefficients 2 k_a k_b / (k_a + k_b); a
// Dirichlet neighbour contributes k_cell to the diagonal (unit coefficient gives C1 exactly).
// `count` disjoint cubes of edge `size` cells (one-cell gap, off the boundary) at seeded
// positions carry coefficient `contrast`.
}  // namespace

// inclusion origins of the FV contrast generator (shared with the device generator, gen_device.cu)
void fv7_inclusion_origins(int32_t N, int count, int size, uint64_t seed, std::vector<int>& ox, std::vector<int>& oy,
                           std::vector<int>& oz) {
    std::mt19937_64 g(seed);
    ox.clear();
    oy.clear();
    oz.clear();
    require(size >= 1 && size + 2 <= N, "generator: inclusion does not fit the grid");
    const int span = N - size - 1;  // origin in [1, span]
    int placed = 0;
    for (int attempt = 0; placed < count && attempt < 100000; ++attempt) {
        const int x0 = 1 + static_cast<int>(u01(g) * span);
        const int y0 = 1 + static_cast<int>(u01(g) * span);
        const int z0 = 1 + static_cast<int>(u01(g) * span);
        bool ok = true;
        for (int c = 0; c < placed && ok; ++c)
            ok = std::abs(x0 - ox[c]) > size || std::abs(y0 - oy[c]) > size || std::abs(z0 - oz[c]) > size;
        if (!ok) continue;
        ox.push_back(x0);
        oy.push_back(y0);
        oz.push_back(z0);
        ++placed;
    }
    require(placed == count, "generator: could not place the inclusions disjointly");
}

// C3's element coefficients exp(sigma N(0,1)), (N+1)^3 of them, element (ex, ey, ez) at
// ex + M (ey + M ez): one seeded mt19937_64 stream through Box-Muller (shared with gen_device.cu,
// which assembles the 27-point rows from them in HBM)
void q1_element_coefficients(int32_t N, double sigma, uint64_t seed, std::vector<double>& ke) {
    const int64_t M = static_cast<int64_t>(N) + 1;
    ke.assign(static_cast<size_t>(M * M * M), 0.0);
    std::mt19937_64 g(seed);
    const double two_pi = 6.283185307179586476925286766559;
    for (int64_t e = 0; e < M * M * M; e += 2) {
        const double a = u01(g), b = u01(g);
        const double r = std::sqrt(-2.0 * std::log(1.0 - a));
        ke[e] = std::exp(sigma * r * std::cos(two_pi * b));
        if (e + 1 < M * M * M) ke[e + 1] = std::exp(sigma * r * std::sin(two_pi * b));
    }
}

// C5's points: 3 npts uniform [0, 1) draws, point i = (P[3i], P[3i+1], P[3i+2]); and the edge
// count G of the bucket grid the exact kNN search uses (shared with gen_device.cu)
void knn_points(int32_t npts, uint64_t seed, std::vector<double>& P) {
    P.assign(3 * static_cast<size_t>(npts), 0.0);
    std::mt19937_64 g(seed);
    for (auto& v : P) v = u01(g);
}

int knn_grid_size(int32_t npts) { return std::max(1, static_cast<int>(std::cbrt(static_cast<double>(npts) / 2.0))); }

namespace {

Csr fv7_contrast(int32_t N, int count, int size, double contrast, uint64_t seed) {
    const int64_t n = static_cast<int64_t>(N) * N * N;
    require(n < (1LL << 31), "generator: grid too large for int32 rows");
    std::vector<float> kap(n, 1.0f);   // marker only; coefficient recomputed as double
    std::vector<uint8_t> inc(n, 0);
    std::vector<int> ox, oy, oz;
    fv7_inclusion_origins(N, count, size, seed, ox, oy, oz);
    const int64_t sy = N, sz = static_cast<int64_t>(N) * N;
    for (int c = 0; c < count; ++c)
        for (int z = oz[c]; z < oz[c] + size; ++z)
            for (int y = oy[c]; y < oy[c] + size; ++y)
                for (int x = ox[c]; x < ox[c] + size; ++x) inc[x + sy * y + sz * z] = 1;
    auto K = [&](int64_t i) { return inc[i] ? contrast : 1.0; };
    auto T = [&](int64_t i, int64_t j) {
        const double a = K(i), b = K(j);
        return 2.0 * a * b / (a + b);
    };
    Csr a;
    a.n = static_cast<int32_t>(n);
    a.rs.resize(n + 1);
    a.ci.reserve(7 * n);
    a.va.reserve(7 * n);
    for (int z = 0; z < N; ++z)
        for (int y = 0; y < N; ++y)
            for (int x = 0; x < N; ++x) {
                const int64_t i = x + sy * y + sz * z;
                a.rs[i] = static_cast<int32_t>(a.ci.size());
                const double ki = K(i);
                // neighbours in ascending column order; diagonal accumulated in a fixed order
                const int64_t nb[6] = {z > 0 ? i - sz : -1, y > 0 ? i - sy : -1, x > 0 ? i - 1 : -1,
                                       x < N - 1 ? i + 1 : -1, y < N - 1 ? i + sy : -1, z < N - 1 ? i + sz : -1};
                double diag = 0.0;
                double off[6];
                for (int d = 0; d < 6; ++d) {
                    off[d] = nb[d] >= 0 ? T(i, nb[d]) : ki;
                    diag += off[d];
                }
                for (int d = 0; d < 3; ++d)
                    if (nb[d] >= 0) {
                        a.ci.push_back(static_cast<int32_t>(nb[d]));
                        a.va.push_back(-off[d]);
                    }
                a.ci.push_back(static_cast<int32_t>(i));
                a.va.push_back(diag);
                for (int d = 3; d < 6; ++d)
                    if (nb[d] >= 0) {
                        a.ci.push_back(static_cast<int32_t>(nb[d]));
                        a.va.push_back(-off[d]);
                    }
            }
    a.rs[n] = static_cast<int32_t>(a.ci.size());
    (void)kap;
    return a;
}

// ---- C3: Q1 (trilinear hexahedron) stiffness, element coefficient exp(sigma N(0,1)).
// Unit-cube reference stiffness: 1/3 on the diagonal, 0 between nodes differing in one
// coordinate (kept as explicit zeros so the IC(0) pattern keeps them), -1/12 between nodes
// differing in two or three coordinates.  Elements are the (N+1)^3 cells of the node lattice
// including the eliminated boundary nodes; the scale factor h is dropped.
Csr q1_27pt(int32_t N, double sigma, uint64_t seed) {
    const int64_t n = static_cast<int64_t>(N) * N * N;
    require(n < (1LL << 31), "generator: grid too large for int32 rows");
    const int64_t M = N + 1;  // elements per axis
    std::vector<double> ke;
    q1_element_coefficients(N, sigma, seed, ke);
    auto E = [&](int64_t ex, int64_t ey, int64_t ez) { return ke[ex + M * (ey + M * ez)]; };
    Csr a;
    a.n = static_cast<int32_t>(n);
    a.rs.resize(n + 1);
    const int64_t nnz_est = (3LL * N - 2) * (3LL * N - 2) * (3LL * N - 2);
    require(nnz_est < (1LL << 31), "generator: nnz exceeds int32 CSR offsets");
    a.ci.resize(nnz_est);
    a.va.resize(nnz_est);
    // row lengths are known in closed form; fill rows in parallel
    std::vector<int64_t> start(n + 1, 0);
    auto cnt1 = [&](int c) { return (c > 0) + 1 + (c < N - 1); };
    for (int z = 0, i = 0; z < N; ++z)
        for (int y = 0; y < N; ++y)
            for (int x = 0; x < N; ++x, ++i) start[i + 1] = start[i] + cnt1(x) * cnt1(y) * cnt1(z);
    require(start[n] == nnz_est, "generator: Q1 nnz bookkeeping");
    const int64_t sy = N, sz = static_cast<int64_t>(N) * N;
    auto fill_plane = [&](int z) {
        for (int y = 0; y < N; ++y)
            for (int x = 0; x < N; ++x) {
                const int64_t i = x + sy * y + sz * z;
                int64_t p = start[i];
                for (int dz = -1; dz <= 1; ++dz) {
                    if (z + dz < 0 || z + dz >= N) continue;
                    for (int dy = -1; dy <= 1; ++dy) {
                        if (y + dy < 0 || y + dy >= N) continue;
                        for (int dx = -1; dx <= 1; ++dx) {
                            if (x + dx < 0 || x + dx >= N) continue;
                            const int nd = (dx != 0) + (dy != 0) + (dz != 0);
                            // elements containing both nodes: node coordinate c lies in elements
                            // c and c+1 (element e spans nodes e-1 .. e); ascending element order
                            const int exs = std::max(x, x + dx), exe = std::min(x, x + dx) + 1;
                            const int eys = std::max(y, y + dy), eye = std::min(y, y + dy) + 1;
                            const int ezs = std::max(z, z + dz), eze = std::min(z, z + dz) + 1;
                            double ksum = 0.0;
                            for (int ez = ezs; ez <= eze; ++ez)
                                for (int ey = eys; ey <= eye; ++ey)
                                    for (int ex = exs; ex <= exe; ++ex) ksum += E(ex, ey, ez);
                            double v;
                            if (nd == 0) v = ksum / 3.0;
                            else if (nd == 1) v = 0.0;
                            else v = -ksum / 12.0;
                            a.ci[p] = static_cast<int32_t>(i + dx + sy * dy + sz * dz);
                            a.va[p] = v;
                            ++p;
                        }
                    }
                }
            }
    };
    const unsigned hw = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    std::atomic<int> next{0};
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < hw; ++t)
        pool.emplace_back([&] {
            for (int z; (z = next.fetch_add(1)) < N;) fill_plane(z);
        });
    for (auto& th : pool) th.join();
    for (int64_t i = 0; i <= n; ++i) a.rs[i] = static_cast<int32_t>(start[i]);
    return a;
}

// sum of f(0..n-1): sequential within gm::kSumChunk-term chunks, then over the chunk sums
template <class F>
double chunked_sum(size_t n, F f) {
    double total = 0.0;
    for (size_t c0 = 0; c0 < n; c0 += gm::kSumChunk) {
        double s = 0.0;
        for (size_t t = c0; t < std::min(n, c0 + gm::kSumChunk); ++t) s += f(t);
        total += s;
    }
    return total;
}

// ---- C5: symmetric kNN graph Laplacian over uniform points in the unit cube.
// Edge (i,j) if j is among the k nearest of i or vice versa; w = exp(-d^2/h^2) with h the mean
// distance over all directed kNN pairs; L = D - W + 1e-6 * mean(degree) I.  Rows keep generation
// order.  Exact kNN by a uniform bucket grid and expanding shells (multi-threaded).  exp and the
// two global means use gen_math.h (portable exp, fixed chunk order), so the device generator
// (gen_device.cu) produces the same bits.
Csr knn_laplacian(int32_t npts, int k, uint64_t seed) {
    require(npts > k && k >= 1, "generator: kNN needs more points than neighbours");
    std::vector<double> P;
    knn_points(npts, seed, P);
    const int G = knn_grid_size(npts);
    const double cell = 1.0 / G;
    auto cidx = [&](double v) { return std::min(G - 1, static_cast<int>(v * G)); };
    std::vector<int32_t> cstart(static_cast<size_t>(G) * G * G + 1, 0), order(npts);
    for (int32_t i = 0; i < npts; ++i)
        cstart[cidx(P[3 * i]) + G * (cidx(P[3 * i + 1]) + G * cidx(P[3 * i + 2])) + 1]++;
    for (size_t c = 0; c + 1 < cstart.size(); ++c) cstart[c + 1] += cstart[c];
    {
        std::vector<int32_t> pos(cstart.begin(), cstart.end() - 1);
        for (int32_t i = 0; i < npts; ++i)
            order[pos[cidx(P[3 * i]) + G * (cidx(P[3 * i + 1]) + G * cidx(P[3 * i + 2]))]++] = i;
    }
    std::vector<int32_t> nbr(static_cast<size_t>(npts) * k);
    std::vector<double> nd2(static_cast<size_t>(npts) * k);
    auto search = [&](int32_t i) {
        const double px = P[3 * i], py = P[3 * i + 1], pz = P[3 * i + 2];
        const int cx = cidx(px), cy = cidx(py), cz = cidx(pz);
        std::vector<std::pair<double, int32_t>> best;  // max-heap of k best
        best.reserve(k + 1);
        for (int r = 0; r <= G; ++r) {
            for (int z = cz - r; z <= cz + r; ++z) {
                if (z < 0 || z >= G) continue;
                for (int y = cy - r; y <= cy + r; ++y) {
                    if (y < 0 || y >= G) continue;
                    for (int x = cx - r; x <= cx + r; ++x) {
                        if (x < 0 || x >= G) continue;
                        if (std::max({std::abs(x - cx), std::abs(y - cy), std::abs(z - cz)}) != r) continue;
                        const int c = x + G * (y + G * z);
                        for (int32_t p = cstart[c]; p < cstart[c + 1]; ++p) {
                            const int32_t j = order[p];
                            if (j == i) continue;
                            const double dx = P[3 * j] - px, dy = P[3 * j + 1] - py, dz = P[3 * j + 2] - pz;
                            const double d2 = dx * dx + dy * dy + dz * dz;
                            const std::pair<double, int32_t> cand{d2, j};
                            if (static_cast<int>(best.size()) < k) {
                                best.push_back(cand);
                                std::push_heap(best.begin(), best.end());
                            } else if (cand < best.front()) {
                                std::pop_heap(best.begin(), best.end());
                                best.back() = cand;
                                std::push_heap(best.begin(), best.end());
                            }
                        }
                    }
                }
            }
            // every point outside the searched shells is at least r*cell away (per axis)
            if (static_cast<int>(best.size()) == k) {
                const double reach = r * cell;
                if (best.front().first <= reach * reach) break;
            }
        }
        std::sort_heap(best.begin(), best.end());
        for (int t = 0; t < k; ++t) {
            nbr[static_cast<size_t>(i) * k + t] = best[t].second;
            nd2[static_cast<size_t>(i) * k + t] = best[t].first;
        }
    };
    const unsigned hw = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    {
        std::atomic<int32_t> next{0};
        std::vector<std::thread> pool;
        for (unsigned t = 0; t < hw; ++t)
            pool.emplace_back([&] {
                for (int32_t i; (i = next.fetch_add(1024)) < npts;)
                    for (int32_t j = i; j < std::min(npts, i + 1024); ++j) search(j);
            });
        for (auto& th : pool) th.join();
    }
    // h = mean kNN distance, summed in gm's fixed chunk order (the device generator's order)
    const double h = chunked_sum(nd2.size(), [&](size_t t) { return std::sqrt(nd2[t]); }) / static_cast<double>(nd2.size());
    // symmetric union: directed edges plus reversed, sorted and deduplicated per row
    std::vector<int64_t> deg(npts + 1, 0);
    for (int32_t i = 0; i < npts; ++i)
        for (int t = 0; t < k; ++t) {
            deg[i + 1]++;
            deg[nbr[static_cast<size_t>(i) * k + t] + 1]++;
        }
    for (int32_t i = 0; i < npts; ++i) deg[i + 1] += deg[i];
    std::vector<int32_t> adj(deg[npts]);
    {
        std::vector<int64_t> pos(deg.begin(), deg.end() - 1);
        for (int32_t i = 0; i < npts; ++i)
            for (int t = 0; t < k; ++t) {
                const int32_t j = nbr[static_cast<size_t>(i) * k + t];
                adj[pos[i]++] = j;
                adj[pos[j]++] = i;
            }
    }
    Csr a;
    a.n = npts;
    a.rs.assign(static_cast<size_t>(npts) + 1, 0);
    std::vector<std::vector<int32_t>> rows_unused;
    std::vector<int32_t> rowlen(npts);
    for (int32_t i = 0; i < npts; ++i) {
        std::sort(adj.begin() + deg[i], adj.begin() + deg[i + 1]);
        const auto e = std::unique(adj.begin() + deg[i], adj.begin() + deg[i + 1]);
        rowlen[i] = static_cast<int32_t>(e - (adj.begin() + deg[i]));
    }
    int64_t nnz = 0;
    for (int32_t i = 0; i < npts; ++i) nnz += rowlen[i] + 1;
    require(nnz < (1LL << 31), "generator: nnz exceeds int32 CSR offsets");
    a.ci.resize(nnz);
    a.va.resize(nnz);
    std::vector<double> degree(npts, 0.0);
    auto wt = [&](int32_t i, int32_t j) {
        const double dx = P[3 * j] - P[3 * i], dy = P[3 * j + 1] - P[3 * i + 1], dz = P[3 * j + 2] - P[3 * i + 2];
        // symmetric in (i, j): the squared distance is formed from |differences|
        const double d2 = dx * dx + dy * dy + dz * dz;
        return gm::exp(-d2 / (h * h));
    };
    for (int32_t i = 0; i < npts; ++i)
        for (int64_t p = deg[i]; p < deg[i] + rowlen[i]; ++p) degree[i] += wt(i, adj[p]);
    const double mdeg = chunked_sum(degree.size(), [&](size_t t) { return degree[t]; }) / npts;
    int64_t p = 0;
    for (int32_t i = 0; i < npts; ++i) {
        a.rs[i] = static_cast<int32_t>(p);
        bool diag_done = false;
        for (int64_t q = deg[i]; q < deg[i] + rowlen[i]; ++q) {
            const int32_t j = adj[q];
            if (!diag_done && j > i) {
                a.ci[p] = i;
                a.va[p++] = degree[i] + 1e-6 * mdeg;
                diag_done = true;
            }
            a.ci[p] = j;
            a.va[p++] = -wt(i, j);
        }
        if (!diag_done) {
            a.ci[p] = i;
            a.va[p++] = degree[i] + 1e-6 * mdeg;
        }
    }
    a.rs[npts] = static_cast<int32_t>(p);
    return a;
}

template <class T>
T* to_malloc(const std::vector<T>& v) {
    T* p = static_cast<T*>(std::malloc(sizeof(T) * std::max<size_t>(v.size(), 1)));
    if (!p) throw Error(RCG_E_CUDA, "host out of memory");
    if (!v.empty()) std::memcpy(p, v.data(), sizeof(T) * v.size());
    return p;
}

}  // namespace
}  // namespace rcg

using namespace rcg;

extern "C" {

int rcg_generate(const rcg_gen_params* p, int32_t* n, int64_t* nnz, int32_t** row_start, int32_t** col_idx,
                 double** values) {
    return guard([&] {
        Csr a;
        switch (p->kind) {
            case RCG_GEN_POISSON7:
                a = poisson7(p->grid);
                break;
            case RCG_GEN_FV7_CONTRAST:
                a = fv7_contrast(p->grid, p->inclusions, p->inclusion_size, p->contrast, p->seed);
                break;
            case RCG_GEN_Q1_27PT:
                a = q1_27pt(p->grid, p->sigma, p->seed);
                break;
            case RCG_GEN_KNN:
                a = knn_laplacian(p->grid, p->knn_k, p->seed);
                break;
            default:
                throw Error(RCG_E_INVALID, "generator: unknown kind");
        }
        *n = a.n;
        *nnz = static_cast<int64_t>(a.va.size());
        *row_start = to_malloc(a.rs);
        *col_idx = to_malloc(a.ci);
        *values = to_malloc(a.va);
    });
}

void rcg_uniform_pm1(uint64_t seed, uint64_t skip, int64_t n, double* out) {
    std::mt19937_64 g(seed);
    g.discard(skip);
    for (int64_t i = 0; i < n; ++i) out[i] = 2.0 * u01(g) - 1.0;
}

// N(0,1) values; value index v uses draws 2*(v/2) and 2*(v/2)+1 (cosine for even v, sine for odd)
void rcg_normal(uint64_t seed, uint64_t skip, int64_t n, double* out) {
    std::mt19937_64 g(seed);
    g.discard(2 * (skip / 2));
    const double two_pi = 6.283185307179586476925286766559;
    uint64_t v = 2 * (skip / 2);
    int64_t w = 0;
    while (w < n) {
        const double a = u01(g), b = u01(g);
        const double r = std::sqrt(-2.0 * std::log(1.0 - a));
        const double z0 = r * std::cos(two_pi * b), z1 = r * std::sin(two_pi * b);
        if (v >= skip) out[w++] = z0;
        if (w < n && v + 1 >= skip) out[w++] = z1;
        v += 2;
    }
}

void rcg_host_free(void* p) { std::free(p); }

// Greedy colouring in natural order (smallest colour unused by earlier neighbours): red-black
// for the 7-point stencil, 8 colours for the 27-point.  new_of_old[i] = position of row i after
// sorting by (colour, index).  Returns the colour count.
int rcg_multicolor_order(int32_t n, const int32_t* row_start, const int32_t* col_idx, int32_t* new_of_old,
                         int32_t* ncolors) {
    return guard([&] {
        std::vector<int32_t> color(n, -1);
        std::vector<int32_t> mark;
        int32_t nc = 0;
        for (int32_t i = 0; i < n; ++i) {
            for (int32_t p = row_start[i]; p < row_start[i + 1]; ++p) {
                const int32_t j = col_idx[p];
                if (j != i && color[j] >= 0) {
                    if (static_cast<int32_t>(mark.size()) <= color[j]) mark.resize(color[j] + 1, -1);
                    mark[color[j]] = i;
                }
            }
            int32_t c = 0;
            while (c < static_cast<int32_t>(mark.size()) && mark[c] == i) ++c;
            color[i] = c;
            nc = std::max(nc, c + 1);
        }
        std::vector<int64_t> start(nc + 1, 0);
        for (int32_t i = 0; i < n; ++i) start[color[i] + 1]++;
        for (int32_t c = 0; c < nc; ++c) start[c + 1] += start[c];
        for (int32_t i = 0; i < n; ++i) new_of_old[i] = static_cast<int32_t>(start[color[i]]++);
        *ncolors = nc;
    });
}

// B = P A P^T with B[new_of_old[i], new_of_old[j]] = A[i, j]; columns of each row ascending.
// Output arrays are malloc'ed (free with rcg_host_free).
int rcg_permute_symmetric(int32_t n, const int32_t* row_start, const int32_t* col_idx, const double* values,
                          const int32_t* new_of_old, int32_t** rs_out, int32_t** ci_out, double** va_out) {
    return guard([&] {
        std::vector<int32_t> old_of_new(n);
        for (int32_t i = 0; i < n; ++i) old_of_new[new_of_old[i]] = i;
        const int64_t nnz = row_start[n];
        std::vector<int32_t> rs(static_cast<size_t>(n) + 1, 0), ci(nnz);
        std::vector<double> va(nnz);
        for (int32_t r = 0; r < n; ++r) {
            const int32_t i = old_of_new[r];
            rs[r + 1] = rs[r] + (row_start[i + 1] - row_start[i]);
        }
        std::vector<std::pair<int32_t, double>> row;
        for (int32_t r = 0; r < n; ++r) {
            const int32_t i = old_of_new[r];
            row.clear();
            for (int32_t p = row_start[i]; p < row_start[i + 1]; ++p) row.emplace_back(new_of_old[col_idx[p]], values[p]);
            std::sort(row.begin(), row.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
            for (size_t t = 0; t < row.size(); ++t) {
                ci[rs[r] + t] = row[t].first;
                va[rs[r] + t] = row[t].second;
            }
        }
        *rs_out = to_malloc(rs);
        *ci_out = to_malloc(ci);
        *va_out = to_malloc(va);
    });
}

int rcg_level_depth(int32_t n, const int32_t* row_start, const int32_t* col_idx, int32_t* depth) {
    return guard([&] {
        std::vector<int32_t> lev(n, 0);
        int32_t d = 0;
        for (int32_t i = 0; i < n; ++i) {
            int32_t l = 0;
            for (int32_t p = row_start[i]; p < row_start[i + 1]; ++p)
                if (col_idx[p] < i) l = std::max(l, lev[col_idx[p]] + 1);
            lev[i] = l;
            d = std::max(d, l + 1);
        }
        *depth = d;
    });
}

}  // extern "C"
