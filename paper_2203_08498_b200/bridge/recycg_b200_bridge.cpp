// recycg_b200_bridge.cpp -- definitions of the reference's hot-path declarations
// (proj/include/recycg/pcg.hpp:39-52: pcg_solve, deflated_pcg_solve; condest.hpp:46-48:
// pcg_with_condest) over librcg_b200.  Linked INSTEAD of src/pcg.cpp and src/condest.cpp into a
// build of the reference library; the rest of the reference is unchanged.  The solves run on the
// GPU (device-resident PCG loop, IC(0) sweeps on the reference's ordering, deflation
// projections); there is no CPU path here -- without a GPU every call throws std::runtime_error
// (RCG_E_CUDA).
//
// Conventions kept from the reference:
//  * argument checks and messages of pcg.cpp:17-26 / :98-99 (std::invalid_argument);
//  * status -> exception: RCG_E_INVALID -> std::invalid_argument, RCG_E_BREAKDOWN ->
//    BreakdownError (the reference's "(r, z) <= 0" / "(p, A p) <= 0" messages), RCG_E_PARSE ->
//    ParseError, RCG_E_CUDA -> std::runtime_error;
//  * preconditioners dispatched by dynamic type {IdentityPreconditioner, IcPreconditioner};
//    ScPreconditioner keeps its inner preconditioner private (subspace_correction.hpp:34), so it
//    cannot be mirrored on the device from outside and throws std::invalid_argument here;
//  * the observer: recycg::b200::SamplingObserver (recycg_b200.hpp) is run on the device and
//    replayed into the host SamplerState; any other non-empty observer throws
//    std::invalid_argument (the device loop does not call back per iteration);
//  * device images of CsrMatrix / IcFactor / DeflationOperator are cached by object identity
//    (the reference types are immutable after construction).
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "rcg_b200.h"
#include "recycg/condest.hpp"
#include "recycg/deflation.hpp"
#include "recycg/ic_preconditioner.hpp"
#include "recycg/pcg.hpp"
#include "recycg/sampling.hpp"
#include "recycg/subspace_correction.hpp"
#include "recycg_b200.hpp"

namespace recycg {
namespace {

void rethrow(int st) {
    if (st == RCG_OK) return;
    const std::string m = rcg_last_error();
    if (st == RCG_E_INVALID) throw std::invalid_argument(m);
    if (st == RCG_E_BREAKDOWN) throw BreakdownError(m);
    if (st == RCG_E_PARSE) throw ParseError(m);
    throw std::runtime_error("librcg_b200: " + m);
}

rcg_ctx* ctx() {
    static rcg_ctx* c = [] {
        rcg_ctx* p = nullptr;
        rethrow(rcg_ctx_create(0, &p));
        return p;
    }();
    return c;
}

// identity key: object address + its payload address + size (a destroyed object's address reused
// by another object of different contents would have to reuse the payload buffer as well)
using Key = std::tuple<const void*, const void*, std::size_t>;
struct Images {
    std::map<Key, rcg_matrix*> mats;
    std::map<Key, rcg_ic*> ics;
    std::map<Key, rcg_basis*> bases;
};
Images& images() {
    static Images im;
    return im;
}

rcg_matrix* device(const CsrMatrix& a) {
    const Key k{&a, a.values().data(), a.values().size()};
    auto& m = images().mats;
    auto it = m.find(k);
    if (it != m.end()) return it->second;
    rcg_matrix* d = nullptr;
    // validate = 0: a CsrMatrix is validated by its constructor (csr_matrix.cpp:36-87)
    rethrow(rcg_matrix_create(ctx(), a.n(), a.row_start().data(), a.col_idx().data(), a.values().data(), 0, &d));
    m.emplace(k, d);
    return d;
}

rcg_ic* device(const IcFactor& f) {
    const Key k{&f, f.l_val.data(), f.l_val.size()};
    auto& m = images().ics;
    auto it = m.find(k);
    if (it != m.end()) return it->second;
    rcg_ic* d = nullptr;
    rethrow(rcg_ic_create(ctx(), f.n, f.num_blocks(), f.block_bounds.data(), f.l_row_start.data(), f.l_col.data(),
                          f.l_val.data(), f.d.data(), f.u_row_start.data(), f.u_col.data(), f.u_val.data(),
                          f.shift_used, &d));
    m.emplace(k, d);
    return d;
}

// DeflationOperator (deflation.hpp:17-33): W uploaded column-major; AW and chol(W^T A W) are
// rebuilt on the device from W (build_deflation_operator, deflation.cpp:45-76)
rcg_basis* device(const CsrMatrix& a, const DeflationOperator& defl) {
    if (defl.empty()) return nullptr;
    const Key k{&defl, defl.w.cols[0].data(), static_cast<std::size_t>(defl.k())};
    auto& m = images().bases;
    auto it = m.find(k);
    if (it != m.end()) return it->second;
    const std::size_t n = static_cast<std::size_t>(defl.w.n);
    std::vector<double> cols(n * static_cast<std::size_t>(defl.k()));
    for (int j = 0; j < defl.k(); ++j) std::memcpy(cols.data() + j * n, defl.w.cols[j].data(), n * sizeof(double));
    rcg_tall* w = nullptr;
    rethrow(rcg_tall_create(ctx(), defl.w.n, defl.k(), cols.data(), &w));
    rcg_basis* b = nullptr;
    const int st = rcg_basis_create(ctx(), device(a), w, RCG_BASIS_DEFLATION, &b);
    rcg_tall_destroy(w);
    rethrow(st);
    m.emplace(k, b);
    return b;
}

rcg_prec prec_of(const Preconditioner& m) {
    if (dynamic_cast<const IdentityPreconditioner*>(&m)) return {RCG_PREC_IDENTITY, nullptr, nullptr};
    if (auto* ic = dynamic_cast<const IcPreconditioner*>(&m)) return {RCG_PREC_IC, device(ic->factor()), nullptr};
    if (dynamic_cast<const ScPreconditioner*>(&m))
        throw std::invalid_argument(
            "pcg_solve: ScPreconditioner's inner preconditioner is private (subspace_correction.hpp:34); "
            "expose it to run subspace correction on the GPU");
    throw std::invalid_argument("pcg_solve: preconditioner type has no GPU implementation");
}

// pcg.cpp:17-26
void check_inputs(const CsrMatrix& a, const Vector& b, const Vector& x, const SolverConfig& cfg) {
    if (!(cfg.eps > 0.0 && cfg.eps < 1.0)) throw std::invalid_argument("SolverConfig: eps must be in (0, 1)");
    if (cfg.max_iter < 1) throw std::invalid_argument("SolverConfig: max_iter must be >= 1");
    const std::size_t n = static_cast<std::size_t>(a.n());
    if (b.size() != n || x.size() != n) throw std::invalid_argument("pcg: vector size does not match matrix");
}

struct Sampler {
    rcg_sampler* h = nullptr;
    ~Sampler() {
        if (h) rcg_sampler_destroy(h);
    }
};

// Replay the device sampler's outcome into the host SamplerState through its public offer():
// offer every iteration the observer saw (pcg.cpp:88: 1..T-1 after convergence, 1..T at the
// cap) with its relres; iterations whose write is the slot's final one carry the device
// snapshot, every other iteration a placeholder (either not stored by the schedule or
// overwritten later).  The schedule is a function of (iteration, relres) only
// (sampling.cpp:7-72), so the host state ends exactly as the host solve would leave it.
void replay(SamplerState& s, const rcg_sampler* d, int offered, const std::vector<double>& hist, int n) {
    const int m = s.m();
    std::vector<int> occ(m), it(m);
    const int cnt = rcg_sampler_state(d, occ.data(), it.data());
    if (cnt < 0) rethrow(-cnt);
    std::map<int, int> final_write;  // iteration -> slot
    for (int j = 0; j < m; ++j)
        if (occ[j]) final_write[it[j]] = j;
    const Vector placeholder(static_cast<std::size_t>(n), 0.0);
    Vector snap(static_cast<std::size_t>(n));
    for (int i = 1; i <= offered; ++i) {
        auto f = final_write.find(i);
        if (f != final_write.end()) {
            rethrow(rcg_sampler_slot(ctx(), d, f->second, snap.data()));
            s.offer(i, hist[static_cast<std::size_t>(i - 1)], snap);
        } else {
            s.offer(i, hist[static_cast<std::size_t>(i - 1)], placeholder);
        }
    }
    for (int j = 0; j < m; ++j)
        if (static_cast<bool>(occ[j]) != s.occupied(j) || (occ[j] && it[j] != s.stored_iteration(j)))
            throw std::runtime_error("pcg_solve: device sampler and host SamplerState schedules disagree");
}

}  // namespace

namespace b200 {
void release_device_images() {
    auto& im = images();
    for (auto& kv : im.bases) rcg_basis_destroy(kv.second);
    for (auto& kv : im.ics) rcg_ic_destroy(kv.second);
    for (auto& kv : im.mats) rcg_matrix_destroy(kv.second);
    im = Images{};
}
}  // namespace b200

SolveReport pcg_solve(const CsrMatrix& a, const Vector& b, const Preconditioner& m, Vector& x,
                      const SolverConfig& cfg, const IterationObserver& observer) {
    check_inputs(a, b, x, cfg);
    const b200::SamplingObserver* so = observer ? observer.target<b200::SamplingObserver>() : nullptr;
    if (observer && !so)
        throw std::invalid_argument(
            "pcg_solve: this observer cannot run inside the device loop; use recycg::b200::"
            "error_sampling_observer_a/_b or residual_sampling_observer_a (recycg_b200.hpp)");
    const rcg_prec p = prec_of(m);
    Sampler smp;
    if (so) {
        if (so->s->stored_count() != 0)
            throw std::invalid_argument("pcg_solve: the sampler must be fresh (no stored snapshots)");
        const bool meth_b = so->s->method() == SamplingMethod::B;
        rethrow(rcg_sampler_create(ctx(), meth_b ? RCG_SAMPLER_B : RCG_SAMPLER_A, so->s->m(),
                                   meth_b ? 1 : so->iteration_cap, meth_b ? so->eps : 0.5, a.n(), &smp.h));
    }
    std::vector<double> hist(static_cast<std::size_t>(cfg.max_iter));
    rcg_solver_config c{cfg.eps, cfg.max_iter, 1};
    rcg_solve_report r{0, 0, 0.0, cfg.max_iter, hist.data(), nullptr, nullptr};
    rethrow(rcg_pcg_solve(ctx(), device(a), b.data(), &p, x.data(), &c, smp.h,
                          so && so->residual ? RCG_PAYLOAD_R : RCG_PAYLOAD_X, &r));
    SolveReport rep;
    rep.iterations = r.iterations;
    rep.converged = r.converged != 0;
    rep.wall_time = r.wall_time;
    if (cfg.record_history) rep.history.assign(hist.begin(), hist.begin() + r.iterations);
    if (so) replay(*so->s, smp.h, rep.converged ? r.iterations - 1 : r.iterations, hist, a.n());
    return rep;
}

SolveReport deflated_pcg_solve(const CsrMatrix& a, const Vector& b, const Preconditioner& m,
                               const DeflationOperator& defl, Vector& x, const SolverConfig& cfg) {
    check_inputs(a, b, x, cfg);
    if (!defl.empty() && defl.w.n != a.n())
        throw std::invalid_argument("deflated_pcg_solve: W row count does not match A");
    const rcg_prec p = prec_of(m);
    std::vector<double> hist(static_cast<std::size_t>(cfg.record_history ? cfg.max_iter : 0));
    rcg_solver_config c{cfg.eps, cfg.max_iter, cfg.record_history ? 1 : 0};
    rcg_solve_report r{0, 0, 0.0, static_cast<int>(hist.size()), hist.empty() ? nullptr : hist.data(), nullptr,
                       nullptr};
    rethrow(rcg_deflated_pcg_solve(ctx(), device(a), b.data(), &p, device(a, defl), x.data(), &c, &r));
    SolveReport rep;
    rep.iterations = r.iterations;
    rep.converged = r.converged != 0;
    rep.wall_time = r.wall_time;
    if (cfg.record_history) rep.history.assign(hist.begin(), hist.begin() + r.iterations);
    return rep;
}

// condest.cpp:28-143: the PCG iterate of pcg_solve plus the fused power iteration (lambda_max)
// and the method-A sampled Ritz values (lambda_min), all inside the device loop
CondestResult pcg_with_condest(const CsrMatrix& a, const Vector& b, const Preconditioner& m, Vector& x,
                               const SolverConfig& cfg, int m_samples, std::uint64_t v0_seed) {
    if (!(cfg.eps > 0.0 && cfg.eps < 1.0)) throw std::invalid_argument("SolverConfig: eps must be in (0, 1)");
    if (cfg.max_iter < 1) throw std::invalid_argument("SolverConfig: max_iter must be >= 1");
    const std::size_t n = static_cast<std::size_t>(a.n());
    if (b.size() != n || x.size() != n)
        throw std::invalid_argument("pcg_with_condest: vector size does not match matrix");
    const rcg_prec p = prec_of(m);
    std::vector<double> hist(static_cast<std::size_t>(cfg.record_history ? cfg.max_iter : 0));
    std::vector<double> ritz(static_cast<std::size_t>(m_samples > 0 ? m_samples : 1));
    rcg_solver_config c{cfg.eps, cfg.max_iter, cfg.record_history ? 1 : 0};
    rcg_solve_report r{0, 0, 0.0, static_cast<int>(hist.size()), hist.empty() ? nullptr : hist.data(), nullptr,
                       nullptr};
    rcg_cond_estimate e{};
    e.ritz_values = ritz.data();
    rethrow(rcg_pcg_with_condest(ctx(), device(a), b.data(), &p, x.data(), &c, m_samples, v0_seed, &r, &e));
    CondestResult out;
    out.solve.iterations = r.iterations;
    out.solve.converged = r.converged != 0;
    out.solve.wall_time = r.wall_time;
    if (cfg.record_history) out.solve.history.assign(hist.begin(), hist.begin() + r.iterations);
    out.estimate.lambda_max = e.lambda_max;
    out.estimate.lambda_min = e.lambda_min;
    out.estimate.kappa = e.kappa;
    out.estimate.power_iterations = e.power_iterations;
    out.estimate.power_unsettled = e.power_unsettled != 0;
    out.estimate.lambda_min_available = e.lambda_min_available != 0;
    out.estimate.ritz_values.assign(ritz.begin(), ritz.begin() + e.nritz);
    return out;
}

}  // namespace recycg
