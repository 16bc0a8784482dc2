// ref_shim.cpp -- extern "C" handle layer over the UNMODIFIED reference library (TEST
// INFRASTRUCTURE ONLY).  oracle/Makefile compiles the reference's own hot-path sources from
// /root/reference/proj/src together with this file into oracle/_ref/librecycg_ref.so; nothing
// from the reference is copied into this repository.  tests/ use it to pin the C oracle
// (bitwise) and bench.py --impl reference uses it as the CPU arm.
//
// Exceptions map to status codes: 1 std::invalid_argument, 2 BreakdownError, 3 ParseError,
// 4 anything else; the message is kept per thread (ref_last_error).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "recycg/condest.hpp"
#include "recycg/csr_matrix.hpp"
#include "recycg/deflation.hpp"
#include "recycg/dense.hpp"
#include "recycg/ic_preconditioner.hpp"
#include "recycg/pcg.hpp"
#include "recycg/recycling.hpp"
#include "recycg/sampling.hpp"
#include "recycg/scaling.hpp"
#include "recycg/subspace_correction.hpp"

namespace rg = recycg;

namespace {
thread_local std::string g_msg;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_msg = e.what();
        return 1;
    } catch (const rg::BreakdownError& e) {
        g_msg = e.what();
        return 2;
    } catch (const rg::ParseError& e) {
        g_msg = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_msg = e.what();
        return 4;
    }
}

rg::TallDense tall_from(int32_t n, int k, const double* cols) {
    rg::TallDense t(n);
    for (int j = 0; j < k; ++j)
        t.push_col(rg::Vector(cols + static_cast<size_t>(j) * n, cols + static_cast<size_t>(j + 1) * n));
    return t;
}

void tall_to(const rg::TallDense& t, double* out) {
    for (int j = 0; j < t.k(); ++j)
        std::memcpy(out + static_cast<size_t>(j) * t.n, t.cols[j].data(), sizeof(double) * t.n);
}
}  // namespace

struct ref_report {
    int iterations;
    int converged;
    double wall_time;
    int cap;
    double* history;
    double* alphas;
    double* betas;
};

struct ref_condest_out {
    double lambda_max, lambda_min, kappa;
    int power_iterations, power_unsettled, lambda_min_available, nritz;
    double* ritz_values;
};

static void fill_report(const rg::SolveReport& r, ref_report* out) {
    out->iterations = r.iterations;
    out->converged = r.converged ? 1 : 0;
    out->wall_time = r.wall_time;
    if (out->history)
        for (size_t i = 0; i < r.history.size() && static_cast<int>(i) < out->cap; ++i)
            out->history[i] = r.history[i];
}

extern "C" {

const char* ref_last_error() { return g_msg.c_str(); }

// ---- matrices
void* ref_csr_create(int32_t n, const int32_t* rs, const int32_t* ci, const double* va, int* status) {
    rg::CsrMatrix* out = nullptr;
    *status = guarded([&] {
        const int32_t nnz = rs[n];
        out = new rg::CsrMatrix(n, std::vector<int32_t>(rs, rs + n + 1), std::vector<int32_t>(ci, ci + nnz),
                                std::vector<double>(va, va + nnz));
    });
    return out;
}
void ref_csr_free(void* a) { delete static_cast<rg::CsrMatrix*>(a); }

int ref_spmv(void* a, const double* x, double* y) {
    return guarded([&] {
        auto& m = *static_cast<rg::CsrMatrix*>(a);
        rg::Vector xv(x, x + m.n()), yv;
        rg::spmv(m, xv, yv);
        std::memcpy(y, yv.data(), sizeof(double) * yv.size());
    });
}

int ref_spmv_dual(void* a, const double* x1, const double* x2, double* y1, double* y2) {
    return guarded([&] {
        auto& m = *static_cast<rg::CsrMatrix*>(a);
        rg::Vector a1(x1, x1 + m.n()), a2(x2, x2 + m.n()), o1, o2;
        rg::spmv_dual(m, a1, a2, o1, o2);
        std::memcpy(y1, o1.data(), sizeof(double) * o1.size());
        std::memcpy(y2, o2.data(), sizeof(double) * o2.size());
    });
}

int ref_diagonal_scale(void* a, double* va_out, double* dis) {
    return guarded([&] {
        auto [s, sv] = rg::diagonal_scale(*static_cast<rg::CsrMatrix*>(a));
        std::memcpy(va_out, s.values().data(), sizeof(double) * s.values().size());
        std::memcpy(dis, sv.d_inv_sqrt.data(), sizeof(double) * sv.d_inv_sqrt.size());
    });
}

// ---- IC(0)
void* ref_ic0(void* a, double shift, int nblocks, int* status) {
    rg::IcFactor* f = nullptr;
    *status = guarded([&] { f = new rg::IcFactor(rg::ic0_factorize(*static_cast<rg::CsrMatrix*>(a), shift, nblocks)); });
    return f;
}
void ref_ic_free(void* f) { delete static_cast<rg::IcFactor*>(f); }
int64_t ref_ic_nnz(void* f) { return static_cast<int64_t>(static_cast<rg::IcFactor*>(f)->l_val.size()); }
double ref_ic_shift(void* f) { return static_cast<rg::IcFactor*>(f)->shift_used; }
void ref_ic_export(void* fp, int32_t* lrs, int32_t* lcol, double* lval, double* d, int32_t* urs,
                   int32_t* ucol, double* uval) {
    auto& f = *static_cast<rg::IcFactor*>(fp);
    std::memcpy(lrs, f.l_row_start.data(), sizeof(int32_t) * f.l_row_start.size());
    std::memcpy(lcol, f.l_col.data(), sizeof(int32_t) * f.l_col.size());
    std::memcpy(lval, f.l_val.data(), sizeof(double) * f.l_val.size());
    std::memcpy(d, f.d.data(), sizeof(double) * f.d.size());
    std::memcpy(urs, f.u_row_start.data(), sizeof(int32_t) * f.u_row_start.size());
    std::memcpy(ucol, f.u_col.data(), sizeof(int32_t) * f.u_col.size());
    std::memcpy(uval, f.u_val.data(), sizeof(double) * f.u_val.size());
}
int ref_ic_apply(void* fp, const double* r, double* z) {
    return guarded([&] {
        auto& f = *static_cast<rg::IcFactor*>(fp);
        rg::Vector rv(r, r + f.n), zv;
        rg::ic_apply(f, rv, zv);
        std::memcpy(z, zv.data(), sizeof(double) * zv.size());
    });
}

// ---- preconditioners (owned shared_ptr handles)
using PrecPtr = std::shared_ptr<const rg::Preconditioner>;
void* ref_prec_identity() { return new PrecPtr(std::make_shared<rg::IdentityPreconditioner>()); }
void* ref_prec_ic(void* f) {
    return new PrecPtr(std::make_shared<rg::IcPreconditioner>(*static_cast<rg::IcFactor*>(f)));
}
void* ref_prec_sc(void* inner, void* a, int k, const double* w, int* status) {
    PrecPtr* out = nullptr;
    *status = guarded([&] {
        auto& m = *static_cast<rg::CsrMatrix*>(a);
        out = new PrecPtr(std::make_shared<rg::ScPreconditioner>(*static_cast<PrecPtr*>(inner), m,
                                                                 tall_from(m.n(), k, w)));
    });
    return out;
}
void ref_prec_free(void* p) { delete static_cast<PrecPtr*>(p); }
int ref_prec_apply(void* p, int32_t n, const double* r, double* z) {
    return guarded([&] {
        rg::Vector rv(r, r + n), zv;
        (*static_cast<PrecPtr*>(p))->apply(rv, zv);
        std::memcpy(z, zv.data(), sizeof(double) * n);
    });
}

// ---- deflation
void* ref_deflation_build(void* a, int k, const double* w, int* status) {
    rg::DeflationOperator* op = nullptr;
    *status = guarded([&] {
        auto& m = *static_cast<rg::CsrMatrix*>(a);
        op = new rg::DeflationOperator(rg::build_deflation_operator(m, tall_from(m.n(), k, w)));
    });
    return op;
}
void ref_deflation_free(void* d) { delete static_cast<rg::DeflationOperator*>(d); }
int ref_project_pt(void* d, int32_t n, const double* y, double* out) {
    return guarded([&] {
        const auto v = static_cast<rg::DeflationOperator*>(d)->project_pt(rg::Vector(y, y + n));
        std::memcpy(out, v.data(), sizeof(double) * n);
    });
}

// ---- samplers
void* ref_sampler_a(int m, int cap, int* status) {
    rg::SamplerState* s = nullptr;
    *status = guarded([&] { s = new rg::SamplerState(rg::SamplerState::method_a(m, cap)); });
    return s;
}
void* ref_sampler_b(int m, double eps, int* status) {
    rg::SamplerState* s = nullptr;
    *status = guarded([&] { s = new rg::SamplerState(rg::SamplerState::method_b(m, eps)); });
    return s;
}
void ref_sampler_free(void* s) { delete static_cast<rg::SamplerState*>(s); }
void ref_sampler_offer(void* s, int it, double relres, int32_t n, const double* payload) {
    static_cast<rg::SamplerState*>(s)->offer(it, relres, rg::Vector(payload, payload + n));
}
int ref_sampler_occupied(void* s, int slot) { return static_cast<rg::SamplerState*>(s)->occupied(slot) ? 1 : 0; }
int ref_sampler_stored_iteration(void* s, int slot) {
    return static_cast<rg::SamplerState*>(s)->stored_iteration(slot);
}
void ref_sampler_slot(void* s, int slot, double* out) {
    const auto& v = static_cast<rg::SamplerState*>(s)->slot(slot);
    std::memcpy(out, v.data(), sizeof(double) * v.size());
}

// ---- solvers
int ref_pcg_solve(void* a, const double* b, void* prec, double* x, double eps, int max_iter,
                  void* sampler, int payload_kind, ref_report* rep) {
    return guarded([&] {
        auto& m = *static_cast<rg::CsrMatrix*>(a);
        const int32_t n = m.n();
        rg::Vector bv(b, b + n), xv(x, x + n);
        rg::SolverConfig cfg;
        cfg.eps = eps;
        cfg.max_iter = max_iter;
        cfg.record_history = rep->history != nullptr;
        rg::IterationObserver obs;
        if (sampler) {
            auto& s = *static_cast<rg::SamplerState*>(sampler);
            obs = payload_kind ? rg::residual_sampling_observer(s) : rg::error_sampling_observer(s);
        }
        const auto r = rg::pcg_solve(m, bv, **static_cast<PrecPtr*>(prec), xv, cfg, obs);
        std::memcpy(x, xv.data(), sizeof(double) * n);
        fill_report(r, rep);
    });
}

int ref_deflated_pcg_solve(void* a, const double* b, void* prec, void* defl, double* x, double eps,
                           int max_iter, ref_report* rep) {
    return guarded([&] {
        auto& m = *static_cast<rg::CsrMatrix*>(a);
        const int32_t n = m.n();
        rg::Vector bv(b, b + n), xv(x, x + n);
        rg::SolverConfig cfg;
        cfg.eps = eps;
        cfg.max_iter = max_iter;
        cfg.record_history = rep->history != nullptr;
        const rg::DeflationOperator empty;
        const rg::DeflationOperator& d = defl ? *static_cast<rg::DeflationOperator*>(defl) : empty;
        const auto r = rg::deflated_pcg_solve(m, bv, **static_cast<PrecPtr*>(prec), d, xv, cfg);
        std::memcpy(x, xv.data(), sizeof(double) * n);
        fill_report(r, rep);
    });
}

int ref_pcg_with_condest(void* a, const double* b, void* prec, double* x, double eps, int max_iter,
                         int m_samples, uint64_t seed, ref_report* rep, ref_condest_out* est) {
    return guarded([&] {
        auto& m = *static_cast<rg::CsrMatrix*>(a);
        const int32_t n = m.n();
        rg::Vector bv(b, b + n), xv(x, x + n);
        rg::SolverConfig cfg;
        cfg.eps = eps;
        cfg.max_iter = max_iter;
        cfg.record_history = rep->history != nullptr;
        const auto r = rg::pcg_with_condest(m, bv, **static_cast<PrecPtr*>(prec), xv, cfg, m_samples, seed);
        std::memcpy(x, xv.data(), sizeof(double) * n);
        fill_report(r.solve, rep);
        est->lambda_max = r.estimate.lambda_max;
        est->lambda_min = r.estimate.lambda_min;
        est->kappa = r.estimate.kappa;
        est->power_iterations = r.estimate.power_iterations;
        est->power_unsettled = r.estimate.power_unsettled ? 1 : 0;
        est->lambda_min_available = r.estimate.lambda_min_available ? 1 : 0;
        est->nritz = static_cast<int>(r.estimate.ritz_values.size());
        if (est->ritz_values)
            std::memcpy(est->ritz_values, r.estimate.ritz_values.data(), sizeof(double) * est->nritz);
    });
}

// ---- recycling and dense
int ref_harvest_errors(const double* x_final, int32_t n, void* sampler, double* e, int* k) {
    return guarded([&] {
        const auto t = rg::harvest_errors(rg::Vector(x_final, x_final + n), *static_cast<rg::SamplerState*>(sampler));
        tall_to(t, e);
        *k = t.k();
    });
}

int ref_build_aux(void* a, int k, const double* errors, double theta, int* m_bar, double* values, double* w,
                  int* m_tilde) {
    return guarded([&] {
        auto& m = *static_cast<rg::CsrMatrix*>(a);
        const auto basis = rg::build_aux_matrix(m, tall_from(m.n(), k, errors), theta);
        *m_bar = basis.m_bar;
        *m_tilde = basis.w.k();
        for (int i = 0; i < basis.spectrum.k(); ++i) values[i] = basis.spectrum.values[i];
        tall_to(basis.w, w);
    });
}

int ref_rayleigh_ritz(void* a, int k, const double* e, double* values, double* vectors) {
    return guarded([&] {
        auto& m = *static_cast<rg::CsrMatrix*>(a);
        const auto rs = rg::rayleigh_ritz(m, tall_from(m.n(), k, e));
        for (int i = 0; i < rs.k(); ++i) values[i] = rs.values[i];
        if (vectors) tall_to(rs.vectors, vectors);
    });
}

int ref_mgs(int32_t n, int k, const double* v, double drop_tol, double* e, int* kept) {
    return guarded([&] {
        const auto t = rg::mgs_orthonormalize(tall_from(n, k, v), drop_tol);
        tall_to(t, e);
        *kept = t.k();
    });
}

int ref_sym_eig(int k, const double* s, double* values, double* vectors) {
    return guarded([&] {
        const auto eig = rg::sym_eig(rg::SmallSym(k, std::vector<double>(s, s + static_cast<size_t>(k) * k)));
        for (int c = 0; c < k; ++c) {
            values[c] = eig.values[c];
            for (int r = 0; r < k; ++r) vectors[static_cast<size_t>(c) * k + r] = eig.vectors[c][r];
        }
    });
}

int ref_chol_factor(int k, const double* s, double* l) {
    return guarded([&] {
        const auto c = rg::chol_factor(rg::SmallSym(k, std::vector<double>(s, s + static_cast<size_t>(k) * k)));
        std::memcpy(l, c.l.data(), sizeof(double) * c.l.size());
    });
}

}  // extern "C"
