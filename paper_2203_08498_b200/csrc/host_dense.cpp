// host_dense.cpp -- the k x k pieces that stay on the host (k <= 128): Cholesky of W^T A W,
// cyclic Jacobi for the Rayleigh-Ritz matrix, and the Lanczos-tridiagonal extremes.
// They are O(k^3) scalar work once per basis, not data-parallel; compiled without FP contraction.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <numeric>
#include <stdexcept>
#include <vector>

#include "internal.cuh"

namespace rcg {

// Row-by-row Cholesky (src/dense.cpp:146-167).  The reference rejects a pivot <= 0; the device
// Gram is a tree reduction, so an exactly dependent W can leave a rounding-size positive pivot.
// A pivot at or below 16 k eps max|S_ii| is therefore also rejected,
// which keeps the reference's "W^T A W not SPD" behaviour for rank-deficient bases.
bool chol_factor_host(int k, const std::vector<double>& s, std::vector<double>& l, int* bad_row) {
    l.assign(static_cast<size_t>(k) * k, 0.0);
    double dmax = 0.0;
    for (int i = 0; i < k; ++i) dmax = std::max(dmax, std::fabs(s[static_cast<size_t>(i) * k + i]));
    const double floor_piv = 16.0 * k * DBL_EPSILON * dmax;
    for (int i = 0; i < k; ++i)
        for (int j = 0; j <= i; ++j) {
            double acc = s[static_cast<size_t>(i) * k + j];
            for (int p = 0; p < j; ++p) acc -= l[static_cast<size_t>(i) * k + p] * l[static_cast<size_t>(j) * k + p];
            if (i == j) {
                if (acc <= 0.0 || acc <= floor_piv) {
                    if (bad_row) *bad_row = i;
                    return false;
                }
                l[static_cast<size_t>(i) * k + i] = std::sqrt(acc);
            } else {
                l[static_cast<size_t>(i) * k + j] = acc / l[static_cast<size_t>(j) * k + j];
            }
        }
    return true;
}

// L y = f, L^T u = y (src/dense.cpp:169-187)
void chol_solve_host(int k, const std::vector<double>& l, const double* f, double* u) {
    std::vector<double> y(k);
    for (int i = 0; i < k; ++i) {
        double acc = f[i];
        for (int j = 0; j < i; ++j) acc -= l[static_cast<size_t>(i) * k + j] * y[j];
        y[i] = acc / l[static_cast<size_t>(i) * k + i];
    }
    for (int i = k - 1; i >= 0; --i) {
        double acc = y[i];
        for (int j = i + 1; j < k; ++j) acc -= l[static_cast<size_t>(j) * k + i] * u[j];
        u[i] = acc / l[static_cast<size_t>(i) * k + i];
    }
}

// Cyclic Jacobi with the reference's rotation formulas, stopping rule (off <= 1e-12 ||S||_F,
// <= 100 sweeps), ascending order and sign convention (src/dense.cpp:63-144).
// vectors[c*k + r] = component r of eigenvector c.
void sym_eig_host(int k, const std::vector<double>& s, std::vector<double>& values, std::vector<double>& vectors) {
    values.assign(k, 0.0);
    vectors.assign(static_cast<size_t>(k) * k, 0.0);
    if (k == 0) return;
    std::vector<double> a = s, v(static_cast<size_t>(k) * k, 0.0);
    auto A = [&](int i, int j) -> double& { return a[static_cast<size_t>(i) * k + j]; };
    auto V = [&](int i, int j) -> double& { return v[static_cast<size_t>(i) * k + j]; };
    for (int i = 0; i < k; ++i) V(i, i) = 1.0;
    double fro = 0.0;
    for (double x : a) fro += x * x;
    fro = std::sqrt(fro);
    int sweep = 0;
    for (; sweep < 100; ++sweep) {
        double off = 0.0;
        for (int p = 0; p < k; ++p)
            for (int q = p + 1; q < k; ++q) off += 2.0 * A(p, q) * A(p, q);
        if (std::sqrt(off) <= 1e-12 * fro) break;
        for (int p = 0; p + 1 < k; ++p)
            for (int q = p + 1; q < k; ++q) {
                const double apq = A(p, q);
                if (apq == 0.0) continue;
                const double th = (A(q, q) - A(p, p)) / (2.0 * apq);
                const double t = (th >= 0.0 ? 1.0 : -1.0) / (std::fabs(th) + std::sqrt(th * th + 1.0));
                const double c = 1.0 / std::sqrt(t * t + 1.0);
                const double sn = t * c;
                const double app = A(p, p), aqq = A(q, q);
                A(p, p) = c * c * app - 2.0 * sn * c * apq + sn * sn * aqq;
                A(q, q) = sn * sn * app + 2.0 * sn * c * apq + c * c * aqq;
                A(p, q) = 0.0;
                A(q, p) = 0.0;
                for (int r = 0; r < k; ++r) {
                    if (r == p || r == q) continue;
                    const double arp = A(r, p), arq = A(r, q);
                    A(r, p) = c * arp - sn * arq;
                    A(p, r) = A(r, p);
                    A(r, q) = sn * arp + c * arq;
                    A(q, r) = A(r, q);
                }
                for (int r = 0; r < k; ++r) {
                    const double vrp = V(r, p), vrq = V(r, q);
                    V(r, p) = c * vrp - sn * vrq;
                    V(r, q) = sn * vrp + c * vrq;
                }
            }
    }
    if (sweep == 100) throw Error(RCG_E_BREAKDOWN, "sym_eig: Jacobi sweeps did not converge");
    std::vector<int> order(k);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int i, int j) { return A(i, i) < A(j, j); });
    for (int c = 0; c < k; ++c) {
        const int src = order[c];
        values[c] = A(src, src);
        double* vec = vectors.data() + static_cast<size_t>(c) * k;
        for (int r = 0; r < k; ++r) vec[r] = V(r, src);
        int imax = 0;
        for (int r = 1; r < k; ++r)
            if (std::fabs(vec[r]) > std::fabs(vec[imax])) imax = r;
        if (vec[imax] < 0.0)
            for (int r = 0; r < k; ++r) vec[r] = -vec[r];
    }
}

// Extreme eigenvalues of the CG Lanczos tridiagonal T (T_11 = 1/a_1, T_jj = 1/a_j + b_j/a_{j-1},
// T_{j,j+1} = sqrt(b_{j+1})/a_j) by Sturm-sequence bisection.
static int sturm_below(int k, const std::vector<double>& dg, const std::vector<double>& off2, double x) {
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

void lanczos_extremes_host(int k, const double* alphas, const double* betas, double* lmin, double* lmax) {
    std::vector<double> dg(k), off2(std::max(k, 1), 0.0);
    for (int j = 0; j < k; ++j) {
        dg[j] = 1.0 / alphas[j];
        if (j > 0) dg[j] += betas[j] / alphas[j - 1];
        if (j + 1 < k) off2[j] = betas[j + 1] / (alphas[j] * alphas[j]);
    }
    double lo = dg[0], hi = dg[0];
    for (int j = 0; j < k; ++j) {
        const double rad = (j > 0 ? std::sqrt(off2[j - 1]) : 0.0) + (j + 1 < k ? std::sqrt(off2[j]) : 0.0);
        lo = std::min(lo, dg[j] - rad);
        hi = std::max(hi, dg[j] + rad);
    }
    auto bisect = [&](int target) {
        double a = lo, b = hi;
        for (int it = 0; it < 200 && b - a > 1e-15 * std::max(std::fabs(a), std::fabs(b)); ++it) {
            const double mid = 0.5 * (a + b);
            if (sturm_below(k, dg, off2, mid) >= target) b = mid; else a = mid;
        }
        return 0.5 * (a + b);
    };
    *lmin = bisect(1);
    *lmax = bisect(k);
}

}  // namespace rcg
