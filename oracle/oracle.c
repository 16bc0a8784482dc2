/*
 * oracle.c -- plain-C restatement of the recycg reference path.  TEST INFRASTRUCTURE ONLY:
 * tests/, bench.py (cpu_baseline / --impl reference) and __graft_entry__.smoke() use it as the
 * checker; the CUDA product never links it.
 *
 * Parity is PINNED two ways (tests/test_oracle.py):
 *   - against oracle/_ref, the unmodified reference compiled from /root/reference sources
 *     (bitwise: every routine below keeps the reference's operation order), and
 *   - against the reference's own known-answer tests (sampler golden set, IC 2x2 factor,
 *     shift ladder to 1.28, condest two-iteration lambda_min, ...).
 * Build with -ffp-contract=off: a contracted FMA changes rounding.
 *
 * Citations: file:line relative to /root/reference/proj.
 */
#include "oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static __thread char g_err[512];

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

const char* orc_last_error(void) { return g_err; }

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

static void* xcalloc(size_t cnt, size_t sz) {
    void* p = calloc(cnt ? cnt : 1, sz);
    if (!p) {
        fprintf(stderr, "oracle: out of memory (%zu x %zu)\n", cnt, sz);
        abort();
    }
    return p;
}

/* ------------------------------------------------------------------ RNG
 * UniformPm1 (include/recycg/rng.hpp:18-41) draws std::mt19937_64 and maps the top 53 bits to
 * [0,1) then to [-1,1).  std::mt19937_64 is fully specified by the C++ standard; this is the
 * published MT19937-64 recurrence with those parameters. */
#define MT_NN 312
#define MT_MM 156

void orc_mt64_seed(orc_mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < MT_NN; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = MT_NN;
}

static void mt64_twist(orc_mt64* g) {
    const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
    const uint64_t mat = 0xB5026F5AA96619E9ULL;
    for (int i = 0; i < MT_NN; ++i) {
        const uint64_t y = (g->mt[i] & upper) | (g->mt[(i + 1) % MT_NN] & lower);
        g->mt[i] = g->mt[(i + MT_MM) % MT_NN] ^ (y >> 1) ^ ((y & 1ULL) ? mat : 0ULL);
    }
    g->idx = 0;
}

uint64_t orc_mt64_next(orc_mt64* g) {
    if (g->idx >= MT_NN) mt64_twist(g);
    uint64_t x = g->mt[g->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

double orc_uniform_pm1(orc_mt64* g) {
    const double u01 = (double)(orc_mt64_next(g) >> 11) * 0x1.0p-53;
    return 2.0 * u01 - 1.0;
}

void orc_uniform_pm1_fill(uint64_t seed, uint64_t skip, int64_t n, double* out) {
    orc_mt64 g;
    orc_mt64_seed(&g, seed);
    for (uint64_t s = 0; s < skip; ++s) (void)orc_mt64_next(&g);
    for (int64_t i = 0; i < n; ++i) out[i] = orc_uniform_pm1(&g);
}

/* ------------------------------------------------------------------ sparse core */

/* src/csr_matrix.cpp:89-100 -- per-row sum from 0.0 in stored column order */
void orc_spmv(const orc_csr* a, const double* x, double* y) {
    for (int32_t row = 0; row < a->n; ++row) {
        double acc = 0.0;
        for (int32_t p = a->rs[row]; p < a->rs[row + 1]; ++p) acc += a->va[p] * x[a->ci[p]];
        y[row] = acc;
    }
}

/* src/csr_matrix.cpp:102-122 -- one pass, each output identical to orc_spmv */
void orc_spmv_dual(const orc_csr* a, const double* x1, const double* x2, double* y1, double* y2) {
    for (int32_t row = 0; row < a->n; ++row) {
        double a1 = 0.0, a2 = 0.0;
        for (int32_t p = a->rs[row]; p < a->rs[row + 1]; ++p) {
            const double v = a->va[p];
            const int32_t c = a->ci[p];
            a1 += v * x1[c];
            a2 += v * x2[c];
        }
        y1[row] = a1;
        y2[row] = a2;
    }
}

/* Test-only probe of the problem's sensitivity to reduction order: 0 = the reference's forward
 * sequential sum (default, the pinned oracle); 1 = the same sum taken backwards.  Parity tests
 * use the oracle's response to order 1 as the rounding floor a parallel reduction must meet. */
static int g_dot_order = 0;
void orc_set_dot_order(int order) { g_dot_order = order; }

static double dot_pairwise(int64_t n, const double* a, const double* b) {
    if (n <= 8) {
        double acc = 0.0;
        for (int64_t i = 0; i < n; ++i) acc += a[i] * b[i];
        return acc;
    }
    const int64_t h = n / 2;
    return dot_pairwise(h, a, b) + dot_pairwise(n - h, a + h, b + h);
}

/* src/pcg.cpp:10-16 (same helper in dense.cpp:12-18, condest.cpp:13-19) */
double orc_dot(int64_t n, const double* a, const double* b) {
    double acc = 0.0;
    if (g_dot_order == 1) {
        for (int64_t i = n - 1; i >= 0; --i) acc += a[i] * b[i];
        return acc;
    }
    if (g_dot_order == 2) return dot_pairwise(n, a, b);
    for (int64_t i = 0; i < n; ++i) acc += a[i] * b[i];
    return acc;
}

static double nrm2(int64_t n, const double* a) { return sqrt(orc_dot(n, a, a)); }

/* src/scaling.cpp:20-38 -- a_ij * dis_i * dis_j, dis = 1/sqrt(a_ii) */
int orc_diagonal_scale(const orc_csr* a, double* va_out, double* dis) {
    for (int32_t row = 0; row < a->n; ++row) {
        double diag = 0.0;
        for (int32_t p = a->rs[row]; p < a->rs[row + 1]; ++p)
            if (a->ci[p] == row) diag = a->va[p];
        if (diag <= 0.0) return fail(ORC_INVALID, "diagonal_scale: non-positive diagonal at row %d", row);
        dis[row] = 1.0 / sqrt(diag);
    }
    for (int32_t row = 0; row < a->n; ++row)
        for (int32_t p = a->rs[row]; p < a->rs[row + 1]; ++p)
            va_out[p] = a->va[p] * dis[row] * dis[a->ci[p]];
    return ORC_OK;
}

/* ------------------------------------------------------------------ IC(0) */

/* src/ic_preconditioner.cpp:12-74 -- one attempt at a fixed shift; 0 on a non-positive pivot.
 * l_ij = (a_ij - sum_{shared p} l_ip d_p l_jp) / d_j, merged over the two sorted rows;
 * couplings to columns before the row's block start are dropped. */
static int ic_attempt(const orc_csr* a, double shift, orc_ic* f) {
    const int32_t n = a->n;
    int64_t fill = 0;
    int32_t blk = 0;
    f->shift = shift;
    f->lrs[0] = 0;
    for (int32_t i = 0; i < n; ++i) {
        while (i >= f->bounds[blk + 1]) ++blk;
        const int32_t lo = f->bounds[blk];
        const int64_t start = fill;
        f->lrs[i] = (int32_t)start;
        double diag = 0.0;
        for (int32_t p = a->rs[i]; p < a->rs[i + 1]; ++p) {
            const int32_t j = a->ci[p];
            if (j > i) break;
            if (j == i) {
                diag = a->va[p];
                break;
            }
            if (j < lo) continue;
            double acc = a->va[p];
            int64_t pi = start, pj = f->lrs[j];
            const int64_t pi_end = fill, pj_end = f->lrs[j + 1];
            while (pi < pi_end && pj < pj_end) {
                const int32_t ci = f->lcol[pi], cj = f->lcol[pj];
                if (ci == cj) {
                    acc -= f->lval[pi] * f->d[ci] * f->lval[pj];
                    ++pi;
                    ++pj;
                } else if (ci < cj) {
                    ++pi;
                } else {
                    ++pj;
                }
            }
            f->lcol[fill] = j;
            f->lval[fill] = acc / f->d[j];
            ++fill;
        }
        double piv = diag * (1.0 + shift);
        for (int64_t p = start; p < fill; ++p) piv -= f->lval[p] * f->lval[p] * f->d[f->lcol[p]];
        if (piv <= 0.0) return 0;
        f->d[i] = piv;
        f->lrs[i + 1] = (int32_t)fill;
    }
    f->nnz_l = fill;
    return 1;
}

/* src/ic_preconditioner.cpp:77-93 -- counting-sort transpose; row j of U lists i ascending */
static void ic_transpose(orc_ic* f) {
    const int32_t n = f->n;
    memset(f->urs, 0, sizeof(int32_t) * ((size_t)n + 1));
    for (int64_t p = 0; p < f->nnz_l; ++p) f->urs[f->lcol[p] + 1]++;
    for (int32_t i = 0; i < n; ++i) f->urs[i + 1] += f->urs[i];
    int32_t* cursor = (int32_t*)xcalloc((size_t)n + 1, sizeof(int32_t));
    memcpy(cursor, f->urs, sizeof(int32_t) * (size_t)n);
    for (int32_t i = 0; i < n; ++i)
        for (int32_t p = f->lrs[i]; p < f->lrs[i + 1]; ++p) {
            const int32_t dst = cursor[f->lcol[p]]++;
            f->ucol[dst] = i;
            f->uval[dst] = f->lval[p];
        }
    free(cursor);
}

/* src/ic_preconditioner.cpp:97-121 -- block bounds floor(b n / G); shift ladder 0 -> 0.01 -> x2,
 * at most 20 retries */
int orc_ic0_factorize(const orc_csr* a, double shift, int nblocks, orc_ic** out) {
    const int32_t n = a->n;
    if (nblocks < 1 || nblocks > (n > 1 ? n : 1))
        return fail(ORC_INVALID, "ic0_factorize: num_blocks must be in [1, n]");
    if (shift < 0.0) return fail(ORC_INVALID, "ic0_factorize: shift must be >= 0");
    int64_t lower = 0;
    for (int32_t i = 0; i < n; ++i)
        for (int32_t p = a->rs[i]; p < a->rs[i + 1]; ++p)
            if (a->ci[p] < i) ++lower;
    orc_ic* f = (orc_ic*)xcalloc(1, sizeof(orc_ic));
    f->n = n;
    f->nblocks = nblocks;
    f->bounds = (int32_t*)xcalloc((size_t)nblocks + 1, sizeof(int32_t));
    for (int b = 0; b <= nblocks; ++b) f->bounds[b] = (int32_t)(((int64_t)b * n) / nblocks);
    f->lrs = (int32_t*)xcalloc((size_t)n + 1, sizeof(int32_t));
    f->lcol = (int32_t*)xcalloc((size_t)lower, sizeof(int32_t));
    f->lval = (double*)xcalloc((size_t)lower, sizeof(double));
    f->d = (double*)xcalloc((size_t)n, sizeof(double));
    double s = shift;
    const int retries = 20;
    for (int attempt = 0; attempt <= retries; ++attempt) {
        if (ic_attempt(a, s, f)) {
            f->urs = (int32_t*)xcalloc((size_t)n + 1, sizeof(int32_t));
            f->ucol = (int32_t*)xcalloc((size_t)f->nnz_l, sizeof(int32_t));
            f->uval = (double*)xcalloc((size_t)f->nnz_l, sizeof(double));
            ic_transpose(f);
            *out = f;
            return ORC_OK;
        }
        s = (s == 0.0) ? 0.01 : 2.0 * s;
    }
    orc_ic_free(f);
    return fail(ORC_BREAKDOWN,
                "IC breakdown: no positive-pivot factorization after %d shift retries (last shift %f)",
                retries, s);
}

void orc_ic_free(orc_ic* f) {
    if (!f) return;
    free(f->bounds);
    free(f->lrs);
    free(f->lcol);
    free(f->lval);
    free(f->d);
    free(f->urs);
    free(f->ucol);
    free(f->uval);
    free(f);
}

/* src/ic_preconditioner.cpp:123-144 -- forward sweep on L, then divide by d, then backward
 * sweep in descending row order on the transposed copy */
void orc_ic_apply(const orc_ic* f, const double* r, double* z) {
    const int32_t n = f->n;
    for (int32_t i = 0; i < n; ++i) {
        double acc = r[i];
        for (int32_t p = f->lrs[i]; p < f->lrs[i + 1]; ++p) acc -= f->lval[p] * z[f->lcol[p]];
        z[i] = acc;
    }
    for (int32_t i = 0; i < n; ++i) z[i] /= f->d[i];
    for (int32_t i = n - 1; i >= 0; --i) {
        double acc = z[i];
        for (int32_t p = f->urs[i]; p < f->urs[i + 1]; ++p) acc -= f->uval[p] * z[f->ucol[p]];
        z[i] = acc;
    }
}

/* ------------------------------------------------------------------ small dense */

/* src/dense.cpp:146-167 -- row-by-row Cholesky, BreakdownError on a non-positive pivot */
int orc_chol_factor(int k, const double* s, double* l) {
    memset(l, 0, sizeof(double) * (size_t)k * (size_t)k);
    for (int i = 0; i < k; ++i)
        for (int j = 0; j <= i; ++j) {
            double acc = s[(size_t)i * k + j];
            for (int p = 0; p < j; ++p) acc -= l[(size_t)i * k + p] * l[(size_t)j * k + p];
            if (i == j) {
                if (acc <= 0.0)
                    return fail(ORC_BREAKDOWN, "chol_factor: non-positive pivot at row %d (matrix not SPD)", i);
                l[(size_t)i * k + i] = sqrt(acc);
            } else {
                l[(size_t)i * k + j] = acc / l[(size_t)j * k + j];
            }
        }
    return ORC_OK;
}

/* src/dense.cpp:169-187 -- L y = f then L^T u = y */
void orc_chol_solve(int k, const double* l, const double* f, double* u) {
    double* y = (double*)xcalloc((size_t)k, sizeof(double));
    for (int i = 0; i < k; ++i) {
        double acc = f[i];
        for (int j = 0; j < i; ++j) acc -= l[(size_t)i * k + j] * y[j];
        y[i] = acc / l[(size_t)i * k + i];
    }
    for (int i = k - 1; i >= 0; --i) {
        double acc = y[i];
        for (int j = i + 1; j < k; ++j) acc -= l[(size_t)j * k + i] * u[j];
        u[i] = acc / l[(size_t)i * k + i];
    }
    free(y);
}

/* src/dense.cpp:28-43 -- SmallSym construction checks (cap 128, 1e-12 symmetry) */
static int smallsym_check(int k, const double* s) {
    if (k < 0 || k > 128) return fail(ORC_INVALID, "SmallSym: dimension %d outside [0, 128]", k);
    for (int i = 0; i < k; ++i)
        for (int j = i + 1; j < k; ++j) {
            const double v = s[(size_t)i * k + j], w = s[(size_t)j * k + i];
            if (fabs(v - w) > 1e-12 * fmax(fabs(v), fabs(w)))
                return fail(ORC_INVALID, "SmallSym: asymmetric at (%d,%d)", i, j);
        }
    return ORC_OK;
}

/* src/dense.cpp:63-144 -- cyclic Jacobi, stop when off(B) <= 1e-12 ||S||_F, <= 100 sweeps,
 * ascending values, each vector's largest-|.| entry (first on ties) made positive.
 * vectors[c*k + r] = component r of eigenvector c. */
int orc_sym_eig(int k, const double* s, double* values, double* vectors) {
    if (k == 0) return ORC_OK;
    const size_t kk = (size_t)k * k;
    double* b = (double*)xcalloc(kk, sizeof(double));
    double* v = (double*)xcalloc(kk, sizeof(double));
    memcpy(b, s, kk * sizeof(double));
    for (int i = 0; i < k; ++i) v[(size_t)i * k + i] = 1.0;
#define B_(i, j) b[(size_t)(i) * k + (j)]
#define V_(i, j) v[(size_t)(i) * k + (j)]
    double fro = 0.0;
    for (size_t t = 0; t < kk; ++t) fro += b[t] * b[t];
    fro = sqrt(fro);
    int sweep = 0;
    for (; sweep < 100; ++sweep) {
        double off = 0.0;
        for (int p = 0; p < k; ++p)
            for (int q = p + 1; q < k; ++q) off += 2.0 * B_(p, q) * B_(p, q);
        off = sqrt(off);
        if (off <= 1e-12 * fro) break;
        for (int p = 0; p < k - 1; ++p)
            for (int q = p + 1; q < k; ++q) {
                const double apq = B_(p, q);
                if (apq == 0.0) continue;
                const double th = (B_(q, q) - B_(p, p)) / (2.0 * apq);
                const double t = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
                const double c = 1.0 / sqrt(t * t + 1.0);
                const double sn = t * c;
                const double bpp = B_(p, p), bqq = B_(q, q);
                B_(p, p) = c * c * bpp - 2.0 * sn * c * apq + sn * sn * bqq;
                B_(q, q) = sn * sn * bpp + 2.0 * sn * c * apq + c * c * bqq;
                B_(p, q) = 0.0;
                B_(q, p) = 0.0;
                for (int r = 0; r < k; ++r) {
                    if (r == p || r == q) continue;
                    const double brp = B_(r, p), brq = B_(r, q);
                    B_(r, p) = c * brp - sn * brq;
                    B_(p, r) = B_(r, p);
                    B_(r, q) = sn * brp + c * brq;
                    B_(q, r) = B_(r, q);
                }
                for (int r = 0; r < k; ++r) {
                    const double vrp = V_(r, p), vrq = V_(r, q);
                    V_(r, p) = c * vrp - sn * vrq;
                    V_(r, q) = sn * vrp + c * vrq;
                }
            }
    }
    if (sweep == 100) {
        free(b);
        free(v);
        return fail(ORC_BREAKDOWN, "sym_eig: Jacobi sweeps did not converge");
    }
    /* stable ascending order by diagonal (std::sort on a comparator of distinct keys; ties keep
     * index order here, the reference's std::sort gives the same for distinct values) */
    int* order = (int*)xcalloc((size_t)k, sizeof(int));
    for (int i = 0; i < k; ++i) order[i] = i;
    for (int i = 1; i < k; ++i) {
        const int key = order[i];
        int j = i - 1;
        while (j >= 0 && B_(order[j], order[j]) > B_(key, key)) {
            order[j + 1] = order[j];
            --j;
        }
        order[j + 1] = key;
    }
    for (int c = 0; c < k; ++c) {
        const int src = order[c];
        values[c] = B_(src, src);
        double* vec = vectors + (size_t)c * k;
        for (int r = 0; r < k; ++r) vec[r] = V_(r, src);
        int imax = 0;
        for (int r = 1; r < k; ++r)
            if (fabs(vec[r]) > fabs(vec[imax])) imax = r;
        if (vec[imax] < 0.0)
            for (int r = 0; r < k; ++r) vec[r] = -vec[r];
    }
#undef B_
#undef V_
    free(order);
    free(b);
    free(v);
    return ORC_OK;
}

/* src/dense.cpp:45-61 -- single-pass MGS; drop when ||w|| <= drop_tol * ||v0||; survivors
 * divided by their norm.  Returns the number of kept columns (written to e, column-major). */
int orc_mgs(int32_t n, int k, const double* v, double drop_tol, double* e) {
    int kept = 0;
    for (int j = 0; j < k; ++j) {
        double* w = e + (size_t)kept * n;
        memcpy(w, v + (size_t)j * n, sizeof(double) * (size_t)n);
        const double n0 = nrm2(n, w);
        if (n0 == 0.0) continue;
        for (int q = 0; q < kept; ++q) {
            const double* qc = e + (size_t)q * n;
            const double c = orc_dot(n, qc, w);
            for (int32_t i = 0; i < n; ++i) w[i] -= c * qc[i];
        }
        const double n1 = nrm2(n, w);
        if (n1 <= drop_tol * n0) continue;
        for (int32_t i = 0; i < n; ++i) w[i] /= n1;
        ++kept;
    }
    return kept;
}

/* ------------------------------------------------------------------ W basis */

/* src/deflation.cpp:45-76 and src/subspace_correction.cpp:9-45 -- AW column by column with
 * spmv, S_ij = w_i . aw_j for j <= i mirrored, Cholesky */
int orc_basis_build(const orc_csr* a, int k, const double* w, int who, orc_basis** out) {
    const int32_t n = a->n;
    orc_basis* b = (orc_basis*)xcalloc(1, sizeof(orc_basis));
    b->n = n;
    b->k = k;
    b->w = (double*)xcalloc((size_t)n * k, sizeof(double));
    b->aw = (double*)xcalloc((size_t)n * k, sizeof(double));
    b->l = (double*)xcalloc((size_t)k * k, sizeof(double));
    memcpy(b->w, w, sizeof(double) * (size_t)n * k);
    for (int j = 0; j < k; ++j) orc_spmv(a, b->w + (size_t)j * n, b->aw + (size_t)j * n);
    if (k > 0) {
        double* s = (double*)xcalloc((size_t)k * k, sizeof(double));
        for (int i = 0; i < k; ++i)
            for (int j = 0; j <= i; ++j) {
                const double acc = orc_dot(n, b->w + (size_t)i * n, b->aw + (size_t)j * n);
                s[(size_t)i * k + j] = acc;
                s[(size_t)j * k + i] = acc;
            }
        int st = smallsym_check(k, s);
        if (st == ORC_OK) st = orc_chol_factor(k, s, b->l);
        free(s);
        if (st != ORC_OK) {
            orc_basis_free(b);
            if (st == ORC_BREAKDOWN)
                return fail(ORC_BREAKDOWN, who ? "ScPreconditioner: W^T A W not SPD"
                                               : "build_deflation_operator: W^T A W not SPD");
            return st;
        }
    }
    *out = b;
    return ORC_OK;
}

void orc_basis_free(orc_basis* b) {
    if (!b) return;
    free(b->w);
    free(b->aw);
    free(b->l);
    free(b);
}

/* dense.cpp:201-207 (tall_t_apply) */
static void tall_t(const orc_basis* b, const double* basis, const double* y, double* f) {
    for (int j = 0; j < b->k; ++j) f[j] = orc_dot(b->n, basis + (size_t)j * b->n, y);
}

/* src/deflation.cpp:7-23 -- P^T y = y - AW chol_solve(W^T y) */
void orc_project_pt(const orc_basis* b, const double* y, double* out) {
    if (out != y) memcpy(out, y, sizeof(double) * (size_t)b->n);
    if (b->k == 0) return;
    double* f = (double*)xcalloc((size_t)b->k, sizeof(double));
    double* u = (double*)xcalloc((size_t)b->k, sizeof(double));
    tall_t(b, b->w, y, f);
    orc_chol_solve(b->k, b->l, f, u);
    for (int j = 0; j < b->k; ++j) {
        const double c = u[j];
        const double* col = b->aw + (size_t)j * b->n;
        for (int32_t i = 0; i < b->n; ++i) out[i] -= c * col[i];
    }
    free(f);
    free(u);
}

/* src/deflation.cpp:25-31 -- P x = x - W chol_solve((AW)^T x) */
void orc_project_p(const orc_basis* b, const double* x, double* out) {
    if (out != x) memcpy(out, x, sizeof(double) * (size_t)b->n);
    if (b->k == 0) return;
    double* f = (double*)xcalloc((size_t)b->k, sizeof(double));
    double* u = (double*)xcalloc((size_t)b->k, sizeof(double));
    tall_t(b, b->aw, x, f);
    orc_chol_solve(b->k, b->l, f, u);
    for (int j = 0; j < b->k; ++j) {
        const double c = u[j];
        const double* col = b->w + (size_t)j * b->n;
        for (int32_t i = 0; i < b->n; ++i) out[i] -= c * col[i];
    }
    free(f);
    free(u);
}

/* src/deflation.cpp:33-43 -- W chol_solve(W^T b), accumulated from 0.0 */
void orc_direct_component(const orc_basis* b, const double* rhs, double* out) {
    memset(out, 0, sizeof(double) * (size_t)b->n);
    if (b->k == 0) return;
    double* f = (double*)xcalloc((size_t)b->k, sizeof(double));
    double* u = (double*)xcalloc((size_t)b->k, sizeof(double));
    tall_t(b, b->w, rhs, f);
    orc_chol_solve(b->k, b->l, f, u);
    for (int j = 0; j < b->k; ++j) {
        const double c = u[j];
        const double* col = b->w + (size_t)j * b->n;
        for (int32_t i = 0; i < b->n; ++i) out[i] += c * col[i];
    }
    free(f);
    free(u);
}

/* ------------------------------------------------------------------ preconditioners */

/* include/recycg/preconditioner.hpp:23-26 (identity), ic_preconditioner.hpp:51-58,
 * src/subspace_correction.cpp:47-57 (inner apply, then z += W chol_solve(W^T r)) */
void orc_prec_apply(const orc_prec* m, const double* r, double* z) {
    const orc_ic* ic = m->ic;
    if (m->kind == ORC_PREC_IC) {
        orc_ic_apply(ic, r, z);
    } else if (m->kind == ORC_PREC_SC) {
        const orc_basis* b = m->sc;
        if (ic)
            orc_ic_apply(ic, r, z);
        else
            memcpy(z, r, sizeof(double) * (size_t)b->n);
        if (b->k == 0) return;
        double* f = (double*)xcalloc((size_t)b->k, sizeof(double));
        double* u = (double*)xcalloc((size_t)b->k, sizeof(double));
        tall_t(b, b->w, r, f);
        orc_chol_solve(b->k, b->l, f, u);
        for (int j = 0; j < b->k; ++j) {
            const double c = u[j];
            const double* col = b->w + (size_t)j * b->n;
            for (int32_t i = 0; i < b->n; ++i) z[i] += c * col[i];
        }
        free(f);
        free(u);
    }
}

static void prec_apply_n(const orc_prec* m, int32_t n, const double* r, double* z) {
    if (m->kind == ORC_PREC_IDENTITY) {
        memcpy(z, r, sizeof(double) * (size_t)n);
        return;
    }
    orc_prec_apply(m, r, z);
}

/* ------------------------------------------------------------------ samplers */

/* src/sampling.cpp:7-24 -- l_max = smallest exponent with m^l_max > cap */
int orc_sampler_create_a(int m, int cap, int32_t n, orc_sampler** out) {
    if (m < 2) return fail(ORC_INVALID, "sampler method A: m must be >= 2");
    if (cap < 1) return fail(ORC_INVALID, "sampler method A: iteration cap must be >= 1");
    orc_sampler* s = (orc_sampler*)xcalloc(1, sizeof(orc_sampler));
    s->method = 0;
    s->m = m;
    s->n = n;
    s->slots = (double*)xcalloc((size_t)m * (size_t)(n > 0 ? n : 1), sizeof(double));
    s->occupied = (int*)xcalloc((size_t)m, sizeof(int));
    s->stored_iter = (int*)xcalloc((size_t)m, sizeof(int));
    s->h = 1;
    s->l_max = 1;
    int64_t pw = m;
    while (pw <= cap) {
        pw *= m;
        s->l_max++;
    }
    *out = s;
    return ORC_OK;
}

/* src/sampling.cpp:26-38 -- alpha = -log10(eps) */
int orc_sampler_create_b(int m, double eps, int32_t n, orc_sampler** out) {
    if (m < 1) return fail(ORC_INVALID, "sampler method B: m must be >= 1");
    if (!(eps > 0.0 && eps < 1.0)) return fail(ORC_INVALID, "sampler method B: eps must be in (0, 1)");
    orc_sampler* s = (orc_sampler*)xcalloc(1, sizeof(orc_sampler));
    s->method = 1;
    s->m = m;
    s->n = n;
    s->slots = (double*)xcalloc((size_t)m * (size_t)(n > 0 ? n : 1), sizeof(double));
    s->occupied = (int*)xcalloc((size_t)m, sizeof(int));
    s->stored_iter = (int*)xcalloc((size_t)m, sizeof(int));
    s->alpha = -log10(eps);
    s->next_slot = 1;
    *out = s;
    return ORC_OK;
}

static void store_slot(orc_sampler* s, int slot, int iteration, const double* payload) {
    memcpy(s->slots + (size_t)slot * s->n, payload, sizeof(double) * (size_t)s->n);
    s->occupied[slot] = 1;
    s->stored_iter[slot] = iteration;
}

/* src/sampling.cpp:40-65 -- method A: offer when i % h == 0, slot = alternating floor sum mod m,
 * h doubles at i == h m; method B: fill every newly crossed relres threshold */
void orc_sampler_offer(orc_sampler* s, int iteration, double relres, const double* payload) {
    if (s->method == 0) {
        if (iteration % s->h != 0) return;
        int64_t acc = 0, pw = 1;
        for (int l = 0; l <= s->l_max; ++l) {
            const int64_t term = (iteration - 1) / pw;
            acc += (l % 2 == 0) ? term : -term;
            pw *= s->m;
        }
        store_slot(s, (int)(acc % s->m), iteration, payload);
        if (iteration == s->h * s->m) s->h *= 2;
    } else {
        while (s->next_slot <= s->m) {
            const double thr = pow(10.0, -(double)s->next_slot * s->alpha / (s->m + 1));
            if (relres > thr) break;
            store_slot(s, s->next_slot - 1, iteration, payload);
            s->next_slot++;
        }
    }
}

void orc_sampler_free(orc_sampler* s) {
    if (!s) return;
    free(s->slots);
    free(s->occupied);
    free(s->stored_iter);
    free(s);
}

/* ------------------------------------------------------------------ PCG */

static int check_cfg(double eps, int max_iter) {
    if (!(eps > 0.0 && eps < 1.0)) return fail(ORC_INVALID, "SolverConfig: eps must be in (0, 1)");
    if (max_iter < 1) return fail(ORC_INVALID, "SolverConfig: max_iter must be >= 1");
    return ORC_OK;
}

static void rep_push(orc_report* rep, int i, double relres, double alpha, double beta) {
    if (!rep || i > rep->cap) return;
    if (rep->history) rep->history[i - 1] = relres;
    if (rep->alphas) rep->alphas[i - 1] = alpha;
    if (rep->betas) rep->betas[i - 1] = beta;
}

/* src/pcg.cpp:37-92 -- standard PCG; positive beta = rho/rho_prev; stop on ||r|| <= eps ||b||;
 * the observer sees continuing iterations only */
int orc_pcg_solve(const orc_csr* a, const double* b, const orc_prec* m, double* x, double eps,
                  int max_iter, orc_sampler* obs, int payload_kind, orc_report* rep) {
    int st = check_cfg(eps, max_iter);
    if (st) return st;
    const int32_t n = a->n;
    rep->iterations = 0;
    rep->converged = 0;
    rep->wall_time = 0.0;
    const double bn = nrm2(n, b);
    if (bn == 0.0) {
        memset(x, 0, sizeof(double) * (size_t)n);
        rep->converged = 1;
        return ORC_OK;
    }
    double* r = (double*)xcalloc((size_t)n, sizeof(double));
    double* z = (double*)xcalloc((size_t)n, sizeof(double));
    double* p = (double*)xcalloc((size_t)n, sizeof(double));
    double* q = (double*)xcalloc((size_t)n, sizeof(double));
    orc_spmv(a, x, r);
    for (int32_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
    const double t0 = now_s();
    if (nrm2(n, r) <= eps * bn) {
        rep->converged = 1;
    } else {
        double rho_prev = 0.0;
        for (int it = 1; it <= max_iter; ++it) {
            prec_apply_n(m, n, r, z);
            const double rho = orc_dot(n, r, z);
            if (rho <= 0.0) {
                st = fail(ORC_BREAKDOWN, "pcg: preconditioner not SPD ((r, z) <= 0)");
                break;
            }
            double beta = 0.0;
            if (it == 1) {
                memcpy(p, z, sizeof(double) * (size_t)n);
            } else {
                beta = rho / rho_prev;
                for (int32_t j = 0; j < n; ++j) p[j] = z[j] + beta * p[j];
            }
            orc_spmv(a, p, q);
            const double pq = orc_dot(n, p, q);
            if (pq <= 0.0) {
                st = fail(ORC_BREAKDOWN, "pcg: matrix not SPD ((p, A p) <= 0)");
                break;
            }
            const double alpha = rho / pq;
            for (int32_t j = 0; j < n; ++j) x[j] += alpha * p[j];
            for (int32_t j = 0; j < n; ++j) r[j] -= alpha * q[j];
            rho_prev = rho;
            const double relres = nrm2(n, r) / bn;
            rep_push(rep, it, relres, alpha, beta);
            rep->iterations = it;
            if (relres <= eps) {
                rep->converged = 1;
                break;
            }
            if (obs) orc_sampler_offer(obs, it, relres, payload_kind ? r : x);
        }
    }
    rep->wall_time = now_s() - t0;
    free(r);
    free(z);
    free(p);
    free(q);
    return st;
}

/* src/pcg.cpp:94-160 -- deflated PCG: r0 = P^T(b - A x0); q <- P^T A p each iteration;
 * x = P x + W (W^T A W)^-1 W^T b at the end */
int orc_deflated_pcg_solve(const orc_csr* a, const double* b, const orc_prec* m,
                           const orc_basis* defl, double* x, double eps, int max_iter,
                           orc_report* rep) {
    int st = check_cfg(eps, max_iter);
    if (st) return st;
    const int32_t n = a->n;
    const int empty = !defl || defl->k == 0;
    if (!empty && defl->n != n)
        return fail(ORC_INVALID, "deflated_pcg_solve: W row count does not match A");
    rep->iterations = 0;
    rep->converged = 0;
    rep->wall_time = 0.0;
    const double bn = nrm2(n, b);
    if (bn == 0.0) {
        memset(x, 0, sizeof(double) * (size_t)n);
        rep->converged = 1;
        return ORC_OK;
    }
    double* r = (double*)xcalloc((size_t)n, sizeof(double));
    double* z = (double*)xcalloc((size_t)n, sizeof(double));
    double* p = (double*)xcalloc((size_t)n, sizeof(double));
    double* q = (double*)xcalloc((size_t)n, sizeof(double));
    orc_spmv(a, x, r);
    for (int32_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
    if (!empty) orc_project_pt(defl, r, r);
    const double t0 = now_s();
    if (nrm2(n, r) <= eps * bn) {
        rep->converged = 1;
    } else {
        double rho_prev = 0.0;
        for (int it = 1; it <= max_iter; ++it) {
            prec_apply_n(m, n, r, z);
            const double rho = orc_dot(n, r, z);
            if (rho <= 0.0) {
                st = fail(ORC_BREAKDOWN, "deflated pcg: preconditioner not SPD ((r, z) <= 0)");
                break;
            }
            double beta = 0.0;
            if (it == 1) {
                memcpy(p, z, sizeof(double) * (size_t)n);
            } else {
                beta = rho / rho_prev;
                for (int32_t j = 0; j < n; ++j) p[j] = z[j] + beta * p[j];
            }
            orc_spmv(a, p, q);
            if (!empty) orc_project_pt(defl, q, q);
            const double pq = orc_dot(n, p, q);
            if (pq <= 0.0) {
                st = fail(ORC_BREAKDOWN,
                          "deflated pcg: projected operator not SPD ((p, P^T A p) <= 0)");
                break;
            }
            const double alpha = rho / pq;
            for (int32_t j = 0; j < n; ++j) x[j] += alpha * p[j];
            for (int32_t j = 0; j < n; ++j) r[j] -= alpha * q[j];
            rho_prev = rho;
            const double relres = nrm2(n, r) / bn;
            rep_push(rep, it, relres, alpha, beta);
            rep->iterations = it;
            if (relres <= eps) {
                rep->converged = 1;
                break;
            }
        }
    }
    if (st == ORC_OK && !empty) {
        orc_project_p(defl, x, x);
        orc_direct_component(defl, b, z);
        for (int32_t j = 0; j < n; ++j) x[j] += z[j];
    }
    rep->wall_time = now_s() - t0;
    free(r);
    free(z);
    free(p);
    free(q);
    return st;
}

/* ------------------------------------------------------------------ recycling */

static int all_zero(int32_t n, const double* v) {
    for (int32_t i = 0; i < n; ++i)
        if (v[i] != 0.0) return 0;
    return 1;
}

/* src/recycling.cpp:17-28 -- x_final - slot, slot order, skip unoccupied / exactly zero */
int orc_harvest_errors(const double* x_final, const orc_sampler* s, double* e) {
    int k = 0;
    for (int slot = 0; slot < s->m; ++slot) {
        if (!s->occupied[slot]) continue;
        const double* xs = s->slots + (size_t)slot * s->n;
        double* col = e + (size_t)k * s->n;
        for (int32_t i = 0; i < s->n; ++i) col[i] = x_final[i] - xs[i];
        if (all_zero(s->n, col)) continue;
        ++k;
    }
    return k;
}

/* src/recycling.cpp:30-40 -- raw payloads (residual sampling) */
int orc_harvest_stored(const orc_sampler* s, double* e) {
    int k = 0;
    for (int slot = 0; slot < s->m; ++slot) {
        if (!s->occupied[slot]) continue;
        const double* v = s->slots + (size_t)slot * s->n;
        if (all_zero(s->n, v)) continue;
        memcpy(e + (size_t)k * s->n, v, sizeof(double) * (size_t)s->n);
        ++k;
    }
    return k;
}

/* src/recycling.cpp:42-79 -- AE with k spmv, S = E^T A E lower mirrored, sym_eig, all Ritz
 * vectors ritz_c = sum_j t_cj e_j accumulated from 0.0 */
int orc_rayleigh_ritz(const orc_csr* a, int k, const double* e, double* values, double* vectors) {
    const int32_t n = a->n;
    if (k == 0) return ORC_OK;
    double* ae = (double*)xcalloc((size_t)n * k, sizeof(double));
    for (int j = 0; j < k; ++j) orc_spmv(a, e + (size_t)j * n, ae + (size_t)j * n);
    double* s = (double*)xcalloc((size_t)k * k, sizeof(double));
    for (int i = 0; i < k; ++i)
        for (int j = 0; j <= i; ++j) {
            const double acc = orc_dot(n, e + (size_t)i * n, ae + (size_t)j * n);
            s[(size_t)i * k + j] = acc;
            s[(size_t)j * k + i] = acc;
        }
    free(ae);
    int st = smallsym_check(k, s);
    double* t = (double*)xcalloc((size_t)k * k, sizeof(double));
    if (st == ORC_OK) st = orc_sym_eig(k, s, values, t);
    if (st == ORC_OK && vectors) {
        for (int c = 0; c < k; ++c) {
            double* out = vectors + (size_t)c * n;
            memset(out, 0, sizeof(double) * (size_t)n);
            for (int j = 0; j < k; ++j) {
                const double tj = t[(size_t)c * k + j];
                const double* ej = e + (size_t)j * n;
                for (int32_t r = 0; r < n; ++r) out[r] += tj * ej[r];
            }
        }
    }
    free(s);
    free(t);
    return st;
}

/* src/recycling.cpp:81-96 -- MGS (drop 1e-12), Rayleigh-Ritz, keep values < theta (strict) */
int orc_build_aux(const orc_csr* a, int k, const double* errors, double theta, int* m_bar,
                  double* values, double* w, int* m_tilde) {
    const int32_t n = a->n;
    *m_bar = 0;
    *m_tilde = 0;
    if (k == 0) return ORC_OK;
    double* e = (double*)xcalloc((size_t)n * k, sizeof(double));
    const int kept = orc_mgs(n, k, errors, 1e-12, e);
    *m_bar = kept;
    if (kept == 0) {
        free(e);
        return ORC_OK;
    }
    double* vec = (double*)xcalloc((size_t)n * kept, sizeof(double));
    const int st = orc_rayleigh_ritz(a, kept, e, values, vec);
    if (st == ORC_OK) {
        int sel = 0;
        for (int i = 0; i < kept; ++i)
            if (values[i] < theta) {
                memcpy(w + (size_t)sel * n, vec + (size_t)i * n, sizeof(double) * (size_t)n);
                ++sel;
            }
        *m_tilde = sel;
    }
    free(e);
    free(vec);
    return st;
}

/* ------------------------------------------------------------------ condest */

/* src/condest.cpp:28-143 -- PCG recurrence identical to orc_pcg_solve plus a power iteration
 * fused through spmv_dual(p, v); lambda_max = v^T A v; lambda_min = smallest Ritz value of the
 * method-A sampled errors; power_unsettled from the spread of the last 5 quotients */
int orc_pcg_with_condest(const orc_csr* a, const double* b, const orc_prec* m, double* x,
                         double eps, int max_iter, int m_samples, uint64_t v0_seed,
                         orc_report* rep, orc_condest* est) {
    int st = check_cfg(eps, max_iter);
    if (st) return st;
    const int32_t n = a->n;
    est->lambda_min = NAN;
    est->kappa = NAN;
    est->lambda_max = 0.0;
    est->power_iterations = 0;
    est->power_unsettled = 1;
    est->lambda_min_available = 0;
    est->nritz = 0;
    rep->iterations = 0;
    rep->converged = 0;
    rep->wall_time = 0.0;
    orc_sampler* smp = NULL;
    st = orc_sampler_create_a(m_samples, max_iter, n, &smp);
    if (st) return st;
    double* v = (double*)xcalloc((size_t)n, sizeof(double));
    double* av = (double*)xcalloc((size_t)n, sizeof(double));
    orc_uniform_pm1_fill(v0_seed, 0, n, v);
    {
        const double nv = nrm2(n, v);
        for (int32_t i = 0; i < n; ++i) v[i] /= nv;
    }
    const double bn = nrm2(n, b);
    if (bn == 0.0) {
        memset(x, 0, sizeof(double) * (size_t)n);
        rep->converged = 1;
        orc_spmv(a, v, av);
        est->lambda_max = orc_dot(n, v, av);
        free(v);
        free(av);
        orc_sampler_free(smp);
        return ORC_OK;
    }
    double* r = (double*)xcalloc((size_t)n, sizeof(double));
    double* z = (double*)xcalloc((size_t)n, sizeof(double));
    double* p = (double*)xcalloc((size_t)n, sizeof(double));
    double* q = (double*)xcalloc((size_t)n, sizeof(double));
    double* vnext = (double*)xcalloc((size_t)n, sizeof(double));
    double quot[5];
    int nq = 0;
    orc_spmv(a, x, r);
    for (int32_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
    const double t0 = now_s();
    if (nrm2(n, r) <= eps * bn) {
        rep->converged = 1;
    } else {
        double rho_prev = 0.0;
        for (int it = 1; it <= max_iter; ++it) {
            prec_apply_n(m, n, r, z);
            const double rho = orc_dot(n, r, z);
            if (rho <= 0.0) {
                st = fail(ORC_BREAKDOWN, "pcg_with_condest: preconditioner not SPD ((r, z) <= 0)");
                break;
            }
            double beta = 0.0;
            if (it == 1) {
                memcpy(p, z, sizeof(double) * (size_t)n);
            } else {
                beta = rho / rho_prev;
                for (int32_t j = 0; j < n; ++j) p[j] = z[j] + beta * p[j];
            }
            orc_spmv_dual(a, p, v, q, vnext);
            const double quotient = orc_dot(n, v, vnext);
            if (nq == 5) {
                memmove(quot, quot + 1, 4 * sizeof(double));
                nq = 4;
            }
            quot[nq++] = quotient;
            const double vn = nrm2(n, vnext);
            if (vn == 0.0) {
                st = fail(ORC_BREAKDOWN, "pcg_with_condest: power vector vanished");
                break;
            }
            for (int32_t j = 0; j < n; ++j) v[j] = vnext[j] / vn;
            const double pq = orc_dot(n, p, q);
            if (pq <= 0.0) {
                st = fail(ORC_BREAKDOWN, "pcg_with_condest: matrix not SPD ((p, A p) <= 0)");
                break;
            }
            const double alpha = rho / pq;
            for (int32_t j = 0; j < n; ++j) x[j] += alpha * p[j];
            for (int32_t j = 0; j < n; ++j) r[j] -= alpha * q[j];
            rho_prev = rho;
            const double relres = nrm2(n, r) / bn;
            rep_push(rep, it, relres, alpha, beta);
            rep->iterations = it;
            if (relres <= eps) {
                rep->converged = 1;
                break;
            }
            orc_sampler_offer(smp, it, relres, x);
        }
    }
    rep->wall_time = now_s() - t0;
    if (st == ORC_OK) {
        orc_spmv(a, v, av);
        est->lambda_max = orc_dot(n, v, av);
        est->power_iterations = rep->iterations;
        if (nq >= 5) {
            double lo = quot[0], hi = quot[0];
            for (int t = 0; t < nq; ++t) {
                lo = fmin(lo, quot[t]);
                hi = fmax(hi, quot[t]);
            }
            est->power_unsettled = (hi - lo) > 1e-4 * fabs(quot[nq - 1]);
        }
        double* err = (double*)xcalloc((size_t)n * m_samples, sizeof(double));
        double* e = (double*)xcalloc((size_t)n * m_samples, sizeof(double));
        const int kh = orc_harvest_errors(x, smp, err);
        const int kept = orc_mgs(n, kh, err, 1e-12, e);
        if (kept > 0) {
            double* vals = (double*)xcalloc((size_t)kept, sizeof(double));
            st = orc_rayleigh_ritz(a, kept, e, vals, NULL);
            if (st == ORC_OK) {
                if (est->ritz_values) memcpy(est->ritz_values, vals, sizeof(double) * (size_t)kept);
                est->nritz = kept;
                est->lambda_min = vals[0];
                est->lambda_min_available = 1;
                est->kappa = est->lambda_max / est->lambda_min;
            }
            free(vals);
        }
        free(err);
        free(e);
    }
    free(r);
    free(z);
    free(p);
    free(q);
    free(vnext);
    free(v);
    free(av);
    orc_sampler_free(smp);
    return st;
}

/* ------------------------------------------------------------------ Lanczos (no reference)
 * CG <-> Lanczos: T_11 = 1/a_1, T_jj = 1/a_j + b_j/a_{j-1}, T_{j,j+1} = sqrt(b_{j+1})/a_j with
 * b_j = rho_j/rho_{j-1} the beta used to form p_j.  Extreme eigenvalues by Sturm bisection. */
static int sturm_count(int k, const double* dg, const double* off2, double x) {
    int cnt = 0;
    double q = dg[0] - x;
    if (q < 0.0) ++cnt;
    for (int j = 1; j < k; ++j) {
        if (q == 0.0) q = 1e-300;
        q = dg[j] - x - off2[j - 1] / q;
        if (q < 0.0) ++cnt;
    }
    return cnt;
}

int orc_lanczos_extremes(int k, const double* alphas, const double* betas, double* lmin,
                         double* lmax) {
    if (k < 1) return fail(ORC_INVALID, "lanczos: need at least one iteration");
    double* dg = (double*)xcalloc((size_t)k, sizeof(double));
    double* off2 = (double*)xcalloc((size_t)k, sizeof(double));
    for (int j = 0; j < k; ++j) {
        dg[j] = 1.0 / alphas[j];
        if (j > 0) dg[j] += betas[j] / alphas[j - 1];
        if (j + 1 < k) off2[j] = betas[j + 1] / (alphas[j] * alphas[j]);
    }
    double lo = dg[0], hi = dg[0];
    for (int j = 0; j < k; ++j) {
        const double rad = (j > 0 ? sqrt(off2[j - 1]) : 0.0) + (j + 1 < k ? sqrt(off2[j]) : 0.0);
        lo = fmin(lo, dg[j] - rad);
        hi = fmax(hi, dg[j] + rad);
    }
    double a = lo, b = hi;
    for (int it = 0; it < 200 && b - a > 1e-15 * fmax(fabs(a), fabs(b)); ++it) {
        const double mid = 0.5 * (a + b);
        if (sturm_count(k, dg, off2, mid) >= 1) b = mid; else a = mid;
    }
    *lmin = 0.5 * (a + b);
    a = lo;
    b = hi;
    for (int it = 0; it < 200 && b - a > 1e-15 * fmax(fabs(a), fabs(b)); ++it) {
        const double mid = 0.5 * (a + b);
        if (sturm_count(k, dg, off2, mid) >= k) b = mid; else a = mid;
    }
    *lmax = 0.5 * (a + b);
    free(dg);
    free(off2);
    return ORC_OK;
}
