// bridge_driver.cpp -- a program written against the reference's public C++ API only
// (proj/include/recycg; no bridge header): the run_sequence shape of driver.cpp:108-222.  The
// SAME source is linked twice (Makefile): against the whole reference library (CPU) and against
// the reference library with its hot-path modules replaced by the bridge (GPU).
// tests/test_bridge.py compares the two runs.
//
// usage: bridge_driver OUT_DIR [grid]
//            7-point Poisson: scaling, IC(0), solve 1 with the reference's own
//            error_sampling_observer, harvest_errors + build_aux_matrix, build_deflation_operator,
//            deflated solves, CG, pcg_with_condest, plus single calls of spmv_dual, ic_apply,
//            project_pt / project_p / direct_component, mgs_orthonormalize, rayleigh_ritz,
//            harvest_stored and ScPreconditioner::apply (their outputs are compared)
//        bridge_driver OUT_DIR --csr FILE --method sc|deflation --rhs K --samples M --keep KEEP
//            the sequence on a matrix read from FILE (int32 n, int64 nnz, row_start, col_idx,
//            values): solve 1 with the sampler, build_aux_matrix (theta = +inf, the KEEP smallest
//            Ritz vectors), then ScPreconditioner(IC(0), W) or build_deflation_operator(W) and
//            solves 2..K -- the C2 bench protocol through the reference API
//        bridge_driver --errors
//            the error contract: one "case: exception: message" line per misuse / breakdown case
//            (pcg.cpp:17-26 and :55-75)
// Writes OUT_DIR/report.json and OUT_DIR/<kind><k>.bin (solutions).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <chrono>
#include <cstdlib>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "recycg/condest.hpp"
#include "recycg/csr_matrix.hpp"
#include "recycg/deflation.hpp"
#include "recycg/ic_preconditioner.hpp"
#include "recycg/pcg.hpp"
#include "recycg/recycling.hpp"
#include "recycg/sampling.hpp"
#include "recycg/scaling.hpp"
#include "recycg/subspace_correction.hpp"

using namespace recycg;

namespace {

CsrMatrix poisson7(int g) {
    const index_t n = g * g * g;
    std::vector<index_t> rs{0}, ci;
    std::vector<double> va;
    for (int z = 0; z < g; ++z)
        for (int y = 0; y < g; ++y)
            for (int x = 0; x < g; ++x) {
                const index_t i = (z * g + y) * g + x;
                const index_t nb[7] = {z > 0 ? i - g * g : -1, y > 0 ? i - g : -1, x > 0 ? i - 1 : -1, i,
                                       x + 1 < g ? i + 1 : -1, y + 1 < g ? i + g : -1, z + 1 < g ? i + g * g : -1};
                for (index_t j : nb)
                    if (j >= 0) {
                        ci.push_back(j);
                        va.push_back(j == i ? 6.0 : -1.0);
                    }
                rs.push_back(static_cast<index_t>(ci.size()));
            }
    return CsrMatrix(n, std::move(rs), std::move(ci), std::move(va));
}

// b = A x_k with x_k from a splitmix64 stream mapped to [-1, 1)
bool g_perturb = false;  // the reference's own rounding-level spread (the parity bar's floor)

Vector rhs(const CsrMatrix& a, int k) {
    std::uint64_t s = 0x9E3779B97F4A7C15ull * static_cast<std::uint64_t>(k + 1);
    Vector x(static_cast<std::size_t>(a.n()));
    for (double& v : x) {
        std::uint64_t z = (s += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        v = static_cast<double>(z >> 11) * 0x1.0p-52 - 1.0;
    }
    Vector b;
    spmv(a, x, b);
    if (g_perturb) {  // --perturb: every entry moved by one unit in the last place (seeded signs)
        std::uint64_t t = 0xD1B54A32D192ED03ull * static_cast<std::uint64_t>(k + 7);
        for (double& v : b) {
            t ^= t << 13, t ^= t >> 7, t ^= t << 17;
            v *= 1.0 + ((t & 1) ? 0x1.0p-52 : -0x1.0p-52);
        }
    }
    return b;
}

void dump(const std::string& path, const Vector& x) {
    FILE* f = std::fopen(path.c_str(), "wb");
    if (!f || std::fwrite(x.data(), sizeof(double), x.size(), f) != x.size()) throw std::runtime_error("write " + path);
    std::fclose(f);
}

}  // namespace

// every failure the reference reports through exceptions, one line each
int error_cases() {
    const CsrMatrix a = poisson7(4);
    const IdentityPreconditioner id;
    const IcPreconditioner ic(ic0_factorize(a));
    auto run = [](const char* name, auto&& f) {
        try {
            f();
            std::printf("%s: no exception\n", name);
        } catch (const BreakdownError& e) {
            std::printf("%s: BreakdownError: %s\n", name, e.what());
        } catch (const std::invalid_argument& e) {
            std::printf("%s: invalid_argument: %s\n", name, e.what());
        } catch (const std::exception& e) {
            std::printf("%s: other: %s\n", name, e.what());
        }
    };
    const std::size_t n = static_cast<std::size_t>(a.n());
    SolverConfig cfg;
    run("eps_zero", [&] { Vector x(n, 0.0); cfg.eps = 0.0; pcg_solve(a, Vector(n, 1.0), ic, x, cfg); });
    cfg.eps = 1e-8;
    run("max_iter_zero", [&] { Vector x(n, 0.0); SolverConfig c = cfg; c.max_iter = 0; pcg_solve(a, Vector(n, 1.0), id, x, c); });
    run("size_b", [&] { Vector x(n, 0.0); pcg_solve(a, Vector(n - 1, 1.0), id, x, cfg); });
    run("size_x", [&] { Vector x(n + 1, 0.0); deflated_pcg_solve(a, Vector(n, 1.0), id, DeflationOperator{}, x, cfg); });
    run("condest_size", [&] { Vector x(n + 1, 0.0); pcg_with_condest(a, Vector(n, 1.0), id, x, cfg, 8, 42); });
    // A = [[1, 2], [2, 1]] (eigenvalues 3, -1), b = (1, -1): (p, A p) = -2 at the first iteration
    const CsrMatrix indef(2, {0, 2, 4}, {0, 1, 0, 1}, {1.0, 2.0, 2.0, 1.0});
    run("pap_breakdown", [&] { Vector x(2, 0.0); pcg_solve(indef, Vector{1.0, -1.0}, id, x, cfg); });
    run("deflated_pap_breakdown", [&] { Vector x(2, 0.0); deflated_pcg_solve(indef, Vector{1.0, -1.0}, id, DeflationOperator{}, x, cfg); });
    run("zero_rhs", [&] { Vector x(n, 0.0); const SolveReport r = pcg_solve(a, Vector(n, 0.0), ic, x, cfg);
                          std::printf("zero_rhs: iterations %d converged %d\n", r.iterations, r.converged ? 1 : 0); });
    return 0;
}

namespace {

std::string jnum(double v) {
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    return buf;
}

std::string jlist(const std::vector<double>& v) {
    std::string s = "[";
    for (std::size_t j = 0; j < v.size(); ++j) s += (j ? ", " : "") + jnum(v[j]);
    return s + "]";
}

struct Recorder {
    std::string out, js;
    bool first = true;
    void solve(const char* kind, int k, const SolveReport& r, const Vector& x) {
        js += std::string(first ? "" : ", ") + "{\"kind\": \"" + kind + "\", \"k\": " + std::to_string(k) +
              ", \"iterations\": " + std::to_string(r.iterations) + ", \"converged\": " +
              (r.converged ? "true" : "false") + ", \"history_len\": " + std::to_string(r.history.size()) +
              ", \"wall_time\": " + jnum(r.wall_time) + "}";
        first = false;
        dump(out + "/" + kind + std::to_string(k) + ".bin", x);
    }
};

CsrMatrix read_csr(const std::string& path) {
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw std::runtime_error("cannot open " + path);
    std::int32_t n = 0;
    std::int64_t nnz = 0;
    bool ok = std::fread(&n, sizeof n, 1, f) == 1 && std::fread(&nnz, sizeof nnz, 1, f) == 1;
    std::vector<index_t> rs(ok ? static_cast<std::size_t>(n) + 1 : 0), ci(ok ? static_cast<std::size_t>(nnz) : 0);
    std::vector<double> va(ci.size());
    ok = ok && std::fread(rs.data(), sizeof(index_t), rs.size(), f) == rs.size() &&
         std::fread(ci.data(), sizeof(index_t), ci.size(), f) == ci.size() &&
         std::fread(va.data(), sizeof(double), va.size(), f) == va.size();
    std::fclose(f);
    if (!ok) throw std::runtime_error("short read " + path);
    return CsrMatrix(n, std::move(rs), std::move(ci), std::move(va));
}

double seconds_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// run_sequence (driver.cpp:108-222) through the public API: the C2 bench protocol when FILE is
// the C2 matrix (10 RHS, 32 samples, SC with the 16 smallest Ritz vectors)
// W (k columns of n doubles) to / from a file: the shared-input protocol runs the accelerated
// solves of both builds on the same basis
void write_w(const std::string& path, const TallDense& w) {
    FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw std::runtime_error("cannot write " + path);
    for (const Vector& c : w.cols) std::fwrite(c.data(), sizeof(double), c.size(), f);
    std::fclose(f);
}

TallDense read_w(const std::string& path, index_t n) {
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw std::runtime_error("cannot open " + path);
    TallDense w(n);
    Vector c(static_cast<std::size_t>(n));
    while (std::fread(c.data(), sizeof(double), c.size(), f) == c.size()) w.cols.push_back(c);
    std::fclose(f);
    return w;
}

int sequence_mode(const std::string& out, const std::string& csr, const std::string& method, int n_rhs, int m,
                  int keep, const std::string& w_in) {
    using clock = std::chrono::steady_clock;
    const auto t_all = clock::now();
    const CsrMatrix a0 = read_csr(csr);
    auto t0 = clock::now();
    auto [a, scaling] = diagonal_scale(a0);
    auto inner = std::make_shared<IcPreconditioner>(ic0_factorize(a));
    const double t_setup = seconds_since(t0);
    SolverConfig cfg;
    cfg.eps = 1e-8;
    cfg.max_iter = 5000;
    cfg.record_history = true;
    Recorder rec{out, "{\"n\": " + std::to_string(a.n()) + ", \"solves\": ["};
    t0 = clock::now();
    SamplerState s = SamplerState::method_a(std::max(m, 2), cfg.max_iter);  // driver.cpp:142
    Vector x(static_cast<std::size_t>(a.n()), 0.0);
    rec.solve("iccg_sampled", 0, pcg_solve(a, scaling.scale_rhs(rhs(a0, 0)), *inner, x, cfg, error_sampling_observer(s)), x);
    const double t_solve1 = seconds_since(t0);
    t0 = clock::now();
    const AuxBasis aux = build_aux_matrix(a, harvest_errors(x, s), std::numeric_limits<double>::infinity());
    TallDense w(a.n());
    for (int j = 0; j < std::min<int>(keep, aux.w.k()); ++j) w.cols.push_back(aux.w.cols[static_cast<std::size_t>(j)]);
    write_w(out + "/w.bin", w);
    if (!w_in.empty()) w = read_w(w_in, a.n());  // shared-input protocol: the other build's basis
    std::unique_ptr<ScPreconditioner> sc;
    DeflationOperator defl;
    if (method == "sc")
        sc = std::make_unique<ScPreconditioner>(inner, a, w);
    else
        defl = build_deflation_operator(a, w);
    const double t_basis = seconds_since(t0);
    t0 = clock::now();
    for (int k = 1; k < n_rhs; ++k) {
        Vector xk(static_cast<std::size_t>(a.n()), 0.0);
        const Vector bk = scaling.scale_rhs(rhs(a0, k));
        dump(out + "/rhs" + std::to_string(k) + ".bin", bk);  // the parity floor (tests/test_bridge.py)
        if (sc)
            rec.solve("accelerated", k, pcg_solve(a, bk, *sc, xk, cfg), xk);
        else
            rec.solve("accelerated", k, deflated_pcg_solve(a, bk, *inner, defl, xk, cfg), xk);
    }
    const double t_acc = seconds_since(t0);
    rec.js += "], \"m_bar\": " + std::to_string(aux.m_bar) + ", \"m_tilde\": " + std::to_string(w.k()) +
              ", \"ritz\": " + jlist(aux.spectrum.values) + ", \"seconds\": {\"setup\": " + jnum(t_setup) +
              ", \"solve1\": " + jnum(t_solve1) + ", \"recycle_and_basis\": " + jnum(t_basis) +
              ", \"accelerated\": " + jnum(t_acc) + ", \"total\": " + jnum(seconds_since(t_all)) + "}}\n";
    FILE* f = std::fopen((out + "/report.json").c_str(), "w");
    if (!f) throw std::runtime_error("cannot write report.json");
    std::fputs(rec.js.c_str(), f);
    std::fclose(f);
    std::fputs(rec.js.c_str(), stdout);
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc >= 2 && std::string(argv[1]) == "--errors") return error_cases();
    if (argc < 2) {
        std::fprintf(stderr, "usage: %s OUT_DIR [grid] | OUT_DIR --csr FILE --method sc|deflation --rhs K "
                             "--samples M --keep KEEP [--w W.bin]\n", argv[0]);
        return 2;
    }
    const std::string out = argv[1];
    try {
        if (argc > 2 && std::string(argv[2]) == "--csr") {
            std::string csr, method = "sc", w_in;
            int n_rhs = 10, m = 32, keep = 16;
            for (int i = 2; i + 1 < argc; i += 2) {
                const std::string k = argv[i], v = argv[i + 1];
                if (k == "--csr") csr = v;
                else if (k == "--method") method = v;
                else if (k == "--rhs") n_rhs = std::atoi(v.c_str());
                else if (k == "--samples") m = std::atoi(v.c_str());
                else if (k == "--keep") keep = std::atoi(v.c_str());
                else if (k == "--w") w_in = v;
                else if (k == "--perturb") g_perturb = v == "1";
            }
            return sequence_mode(out, csr, method, n_rhs, m, keep, w_in);
        }
        const int grid = argc > 2 ? std::atoi(argv[2]) : 32;
        const int m = 16, cap = 5000, n_rhs = 4;
        const double theta = 0.05;
        const CsrMatrix a0 = poisson7(grid);
        auto [a, scaling] = diagonal_scale(a0);
        auto ic = std::make_shared<IcPreconditioner>(ic0_factorize(a));
        const IdentityPreconditioner id;
        SolverConfig cfg;
        cfg.eps = 1e-8;
        cfg.max_iter = cap;
        cfg.record_history = true;
        Recorder rec{out, "{\"n\": " + std::to_string(a.n()) + ", \"solves\": ["};

        // solve 1 with the reference's own error sampler (driver.cpp:150-160)
        SamplerState s = SamplerState::method_a(m, cap);
        Vector x(static_cast<std::size_t>(a.n()), 0.0);
        const Vector b0 = scaling.scale_rhs(rhs(a0, 0));
        rec.solve("iccg_sampled", 0, pcg_solve(a, b0, *ic, x, cfg, error_sampling_observer(s)), x);
        std::vector<double> occ, its;
        for (int j = 0; j < m; ++j) {
            occ.push_back(s.occupied(j) ? 1 : 0);
            its.push_back(s.occupied(j) ? s.stored_iteration(j) : 0);
        }
        // the recycling step (recycling.cpp:81-96) and the deflation operator
        const TallDense errors = harvest_errors(x, s);
        const AuxBasis aux = build_aux_matrix(a, errors, theta);
        const DeflationOperator defl = build_deflation_operator(a, aux.w);
        for (int k = 1; k < n_rhs; ++k) {
            Vector xk(static_cast<std::size_t>(a.n()), 0.0);
            rec.solve("deflated", k, deflated_pcg_solve(a, scaling.scale_rhs(rhs(a0, k)), *ic, defl, xk, cfg), xk);
        }
        Vector xc(static_cast<std::size_t>(a.n()), 0.0);
        rec.solve("cg", 1, pcg_solve(a, scaling.scale_rhs(rhs(a0, 1)), id, xc, cfg), xc);
        // subspace correction around IC(0) with the same W (subspace_correction.cpp:27-57)
        const ScPreconditioner sc(ic, a, aux.w);
        Vector xs(static_cast<std::size_t>(a.n()), 0.0);
        rec.solve("sc", 1, pcg_solve(a, scaling.scale_rhs(rhs(a0, 1)), sc, xs, cfg), xs);
        // pcg_with_condest (condest.cpp:28-143) with IC(0), 20 samples, seed 42
        Vector xe(static_cast<std::size_t>(a.n()), 0.0);
        const CondestResult ce = pcg_with_condest(a, scaling.scale_rhs(rhs(a0, 2)), *ic, xe, cfg, 20, 42);
        rec.solve("condest", 2, ce.solve, xe);
        // single calls of the other hot-path functions on fixed inputs
        const Vector v = rhs(a0, 7), u = rhs(a0, 8);
        Vector y1, y2, z, zs;
        spmv_dual(a, v, u, y1, y2);
        ic_apply(ic->factor(), v, z);
        sc.apply(v, zs);
        dump(out + "/op_spmv_dual1.bin", y1);
        dump(out + "/op_spmv_dual2.bin", y2);
        dump(out + "/op_ic_apply.bin", z);
        dump(out + "/op_sc_apply.bin", zs);
        dump(out + "/op_project_pt.bin", defl.project_pt(v));
        dump(out + "/op_project_p.bin", defl.project_p(v));
        dump(out + "/op_direct_component.bin", defl.direct_component(v));
        const TallDense q = mgs_orthonormalize(errors);
        const RitzSpectrum rr = rayleigh_ritz(a, q);
        for (int j = 0; j < std::min<int>(2, q.k()); ++j) dump(out + "/op_mgs" + std::to_string(j) + ".bin", q.cols[j]);
        const TallDense st = harvest_stored(s);
        rec.js += "], \"condest\": {\"lambda_max\": " + jnum(ce.estimate.lambda_max) + ", \"lambda_min\": " +
                  jnum(ce.estimate.lambda_min) + ", \"kappa\": " + jnum(ce.estimate.kappa) +
                  ", \"power_iterations\": " + std::to_string(ce.estimate.power_iterations) + "}, \"occupied\": " +
                  jlist(occ) + ", \"stored_iterations\": " + jlist(its) + ", \"m_bar\": " + std::to_string(aux.m_bar) +
                  ", \"m_tilde\": " + std::to_string(defl.k()) + ", \"ritz\": " + jlist(aux.spectrum.values) +
                  ", \"mgs_k\": " + std::to_string(q.k()) + ", \"rr_values\": " + jlist(rr.values) +
                  ", \"harvest_stored_k\": " + std::to_string(st.k()) + ", \"errors_k\": " + std::to_string(errors.k()) +
                  ", \"sc_chol_k\": " + std::to_string(sc.subspace_dim()) + "}\n";
        FILE* f = std::fopen((out + "/report.json").c_str(), "w");
        if (!f) throw std::runtime_error("cannot write report.json");
        std::fputs(rec.js.c_str(), f);
        std::fclose(f);
        std::fputs(rec.js.c_str(), stdout);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "bridge_driver: %s\n", e.what());
        return 1;
    }
    return 0;
}
