// bridge_driver.cpp -- a program written against the reference's public C++ API only
// (proj/include/recycg): the run_sequence shape of driver.cpp:108-222 on a 7-point Poisson
// matrix -- diagonal scaling, IC(0), solve 1 with the error sampler, the recycling step
// (harvest_errors + build_aux_matrix), build_deflation_operator, deflated solves 2..k, plus a
// plain CG solve.  The SAME source is linked twice (Makefile): against the whole reference
// library (CPU) and against the reference library with src/pcg.cpp replaced by
// recycg_b200_bridge.cpp (GPU).  tests/test_gpu_bridge.py compares the two runs.
//
// usage: bridge_driver OUT_DIR [grid]   (writes OUT_DIR/report.json and OUT_DIR/x<k>.bin)
//        bridge_driver --errors          (the error contract: one "case: exception: message" line
//                                         per misuse / breakdown case, pcg.cpp:17-26 and :55-75)
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
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
#include "recycg_b200.hpp"

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

int main(int argc, char** argv) {
    if (argc >= 2 && std::string(argv[1]) == "--errors") return error_cases();
    if (argc < 2) {
        std::fprintf(stderr, "usage: %s OUT_DIR [grid]\n", argv[0]);
        return 2;
    }
    const std::string out = argv[1];
    const int grid = argc > 2 ? std::atoi(argv[2]) : 32;
    const int m = 16, cap = 5000, n_rhs = 4;
    const double theta = 0.05;
    try {
        const CsrMatrix a0 = poisson7(grid);
        auto [a, scaling] = diagonal_scale(a0);
        const IcPreconditioner ic(ic0_factorize(a));
        const IdentityPreconditioner id;
        SolverConfig cfg;
        cfg.eps = 1e-8;
        cfg.max_iter = cap;
        cfg.record_history = true;

        std::string js = "{\"n\": " + std::to_string(a.n()) + ", \"solves\": [";
        auto record = [&](const char* kind, int k, const SolveReport& r, const Vector& x) {
            js += std::string(k || std::string(kind) != "iccg_sampled" ? ", " : "") + "{\"kind\": \"" + kind +
                  "\", \"k\": " + std::to_string(k) + ", \"iterations\": " + std::to_string(r.iterations) +
                  ", \"converged\": " + (r.converged ? "true" : "false") +
                  ", \"history_len\": " + std::to_string(r.history.size()) +
                  ", \"wall_time\": " + std::to_string(r.wall_time) + "}";
            dump(out + "/" + kind + std::to_string(k) + ".bin", x);
        };

        // solve 1 with the error sampler (driver.cpp:150-160)
        SamplerState s = SamplerState::method_a(m, cap);
        Vector x(static_cast<std::size_t>(a.n()), 0.0);
        const Vector b0 = scaling.scale_rhs(rhs(a0, 0));
        record("iccg_sampled", 0, pcg_solve(a, b0, ic, x, cfg, b200::error_sampling_observer_a(s, cap)), x);
        std::string occ = "[", its = "[";
        for (int j = 0; j < m; ++j) {
            occ += std::string(j ? ", " : "") + (s.occupied(j) ? "1" : "0");
            its += std::string(j ? ", " : "") + std::to_string(s.occupied(j) ? s.stored_iteration(j) : 0);
        }
        // the recycling step on the host (recycling.cpp:81-96) and the deflation operator
        const AuxBasis aux = build_aux_matrix(a, harvest_errors(x, s), theta);
        const DeflationOperator defl = build_deflation_operator(a, aux.w);
        for (int k = 1; k < n_rhs; ++k) {
            Vector xk(static_cast<std::size_t>(a.n()), 0.0);
            record("deflated", k, deflated_pcg_solve(a, scaling.scale_rhs(rhs(a0, k)), ic, defl, xk, cfg), xk);
        }
        Vector xc(static_cast<std::size_t>(a.n()), 0.0);
        record("cg", 1, pcg_solve(a, scaling.scale_rhs(rhs(a0, 1)), id, xc, cfg), xc);
        // pcg_with_condest (condest.cpp:28-143) with IC(0), 20 samples, seed 42
        Vector xe(static_cast<std::size_t>(a.n()), 0.0);
        const CondestResult ce = pcg_with_condest(a, scaling.scale_rhs(rhs(a0, 2)), ic, xe, cfg, 20, 42);
        record("condest", 2, ce.solve, xe);
        char cbuf[160];
        std::snprintf(cbuf, sizeof cbuf,
                      "\"condest\": {\"lambda_max\": %.17g, \"lambda_min\": %.17g, \"kappa\": %.17g, \"power_iterations\": %d}, ",
                      ce.estimate.lambda_max, ce.estimate.lambda_min, ce.estimate.kappa, ce.estimate.power_iterations);
        js += std::string("], ") + cbuf + "\"occupied\": " + occ + "], \"stored_iterations\": " + its + "], \"m_bar\": " +
              std::to_string(aux.m_bar) + ", \"m_tilde\": " + std::to_string(defl.k()) + ", \"ritz\": [";
        for (int j = 0; j < aux.spectrum.k(); ++j) {
            char buf[40];
            std::snprintf(buf, sizeof buf, "%s%.17g", j ? ", " : "", aux.spectrum.values[static_cast<std::size_t>(j)]);
            js += buf;
        }
        js += "]}\n";
        FILE* f = std::fopen((out + "/report.json").c_str(), "w");
        if (!f) throw std::runtime_error("cannot write report.json");
        std::fputs(js.c_str(), f);
        std::fclose(f);
        std::fputs(js.c_str(), stdout);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "bridge_driver: %s\n", e.what());
        return 1;
    }
    return 0;
}
