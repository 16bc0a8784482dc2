// recycg_b200_bridge.cpp -- the reference's solver entry points over librcg_b200: pcg_solve and
// deflated_pcg_solve (proj/include/recycg/pcg.hpp:39-52, replacing src/pcg.cpp) and
// pcg_with_condest (condest.hpp:46-48, replacing src/condest.cpp).  Linked into a build of the
// reference library together with recycg_b200_ops.cpp (the other hot-path modules) and
// bridge_core.cpp; the rest of the reference is unchanged.  The solves run on the GPU
// (device-resident PCG loop, IC(0) sweeps on the reference's ordering, deflation projections,
// subspace correction); there is no CPU path -- without a GPU every call throws
// std::runtime_error (RCG_E_CUDA).
//
// Conventions kept from the reference:
//  * argument checks and messages of pcg.cpp:17-26 / :98-99 (std::invalid_argument);
//  * status -> exception mapping (bridge_core.hpp);
//  * preconditioners dispatched by dynamic type {IdentityPreconditioner, IcPreconditioner,
//    ScPreconditioner over an identity or IC(0) inner};
//  * the observer: the error / residual sampling observers of sampling.hpp:67-70 (the reference's
//    own factory functions, defined by recycg_b200_ops.cpp as a named functor) run on the device
//    inside the solve and are replayed into the host SamplerState; any other non-empty observer
//    throws std::invalid_argument (the device loop does not call back per iteration).
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "bridge_core.hpp"
#include "recycg/condest.hpp"
#include "recycg/deflation.hpp"
#include "recycg/ic_preconditioner.hpp"
#include "recycg/pcg.hpp"
#include "recycg/sampling.hpp"
#include "recycg/subspace_correction.hpp"
#include "recycg_b200.hpp"

namespace recycg {
namespace {

using namespace b200::detail;

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
            throw std::runtime_error(
                "pcg_solve: device sampler and host SamplerState schedules disagree (a method-A state made "
                "with an iteration cap below the solve's iteration count, or a method-B state made with "
                "another eps than the solve's)");
}

}  // namespace

SolveReport pcg_solve(const CsrMatrix& a, const Vector& b, const Preconditioner& m, Vector& x,
                      const SolverConfig& cfg, const IterationObserver& observer) {
    check_inputs(a, b, x, cfg);
    const b200::SamplingObserver* so = observer ? observer.target<b200::SamplingObserver>() : nullptr;
    if (observer && !so)
        throw std::invalid_argument(
            "pcg_solve: this observer cannot run inside the device loop; use error_sampling_observer / "
            "residual_sampling_observer (sampling.hpp:67-70)");
    const PrecRef p = prec_of(m);
    const MatrixRef ad = device(a);
    Sampler smp;
    if (so) {
        if (so->s->stored_count() != 0)
            throw std::invalid_argument("pcg_solve: the sampler must be fresh (no stored snapshots)");
        // the device schedule equals the host state's whenever the host's method-A cap is at
        // least the solve's iteration count (m^l_max > cap >= T: the extra alternating-sum terms
        // vanish) -- the driver makes it with cap = max_iter (driver.cpp:142); method B uses the
        // solve's eps (driver.cpp:143).  replay() verifies the outcome.
        const bool meth_b = so->s->method() == SamplingMethod::B;
        const int cap = so->iteration_cap > 0 ? so->iteration_cap : cfg.max_iter;
        const double eps = so->eps > 0.0 ? so->eps : cfg.eps;
        rethrow(rcg_sampler_create(ctx(), meth_b ? RCG_SAMPLER_B : RCG_SAMPLER_A, so->s->m(), meth_b ? 1 : cap,
                                   meth_b ? eps : 0.5, a.n(), &smp.h));
    }
    std::vector<double> hist(static_cast<std::size_t>(cfg.max_iter));
    rcg_solver_config c{cfg.eps, cfg.max_iter, 1};
    rcg_solve_report r{0, 0, 0.0, cfg.max_iter, hist.data(), nullptr, nullptr};
    rethrow(rcg_pcg_solve(ctx(), ad.get(), b.data(), &p.p, x.data(), &c, smp.h,
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
    const PrecRef p = prec_of(m);
    const MatrixRef ad = device(a);
    const BasisRef bd = device_basis(defl.w, defl.aw, defl.waw_chol, RCG_BASIS_DEFLATION);
    std::vector<double> hist(static_cast<std::size_t>(cfg.record_history ? cfg.max_iter : 0));
    rcg_solver_config c{cfg.eps, cfg.max_iter, cfg.record_history ? 1 : 0};
    rcg_solve_report r{0, 0, 0.0, static_cast<int>(hist.size()), hist.empty() ? nullptr : hist.data(), nullptr,
                       nullptr};
    rethrow(rcg_deflated_pcg_solve(ctx(), ad.get(), b.data(), &p.p, bd.get(), x.data(), &c, &r));
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
    const PrecRef p = prec_of(m);
    const MatrixRef ad = device(a);
    std::vector<double> hist(static_cast<std::size_t>(cfg.record_history ? cfg.max_iter : 0));
    std::vector<double> ritz(static_cast<std::size_t>(m_samples > 0 ? m_samples : 1));
    rcg_solver_config c{cfg.eps, cfg.max_iter, cfg.record_history ? 1 : 0};
    rcg_solve_report r{0, 0, 0.0, static_cast<int>(hist.size()), hist.empty() ? nullptr : hist.data(), nullptr,
                       nullptr};
    rcg_cond_estimate e{};
    e.ritz_values = ritz.data();
    rethrow(rcg_pcg_with_condest(ctx(), ad.get(), b.data(), &p.p, x.data(), &c, m_samples, v0_seed, &r, &e));
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
