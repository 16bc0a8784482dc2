// recycg_b200_ops.cpp -- the rest of the reference's hot-path declarations defined over
// librcg_b200, so a program written against proj/include/recycg runs every data-parallel step on
// the GPU.  Linked INSTEAD of these reference modules:
//   src/ic_preconditioner.cpp     ic0_factorize (device factorisation, bitwise the reference
//                                 factor), ic_apply (level-scheduled sweeps, bitwise)
//   src/sampling.cpp              SamplerState, error_sampling_observer, residual_sampling_observer
//   src/recycling.cpp             harvest_errors, harvest_stored, rayleigh_ritz, build_aux_matrix
//   src/deflation.cpp             build_deflation_operator, DeflationOperator::project_*
//   src/subspace_correction.cpp   ScPreconditioner (constructor, apply)
// and, inside the reference's own csr_matrix.cpp / dense.cpp (compiled with the reference
// definitions renamed -- bridge/Makefile), spmv / spmv_dual and mgs_orthonormalize.  Argument
// checks and exception messages follow the reference (file:line cited per function).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "bridge_core.hpp"
#include "recycg/csr_matrix.hpp"
#include "recycg/deflation.hpp"
#include "recycg/dense.hpp"
#include "recycg/ic_preconditioner.hpp"
#include "recycg/recycling.hpp"
#include "recycg/sampling.hpp"
#include "recycg/subspace_correction.hpp"
#include "recycg_b200.hpp"

namespace recycg {

using namespace b200::detail;

// ------------------------------------------------------------------ sparse core (csr_matrix.hpp:54-59)
void spmv(const CsrMatrix& a, const Vector& x, Vector& y) {
    if (x.size() != static_cast<std::size_t>(a.n())) throw std::invalid_argument("spmv: vector size does not match matrix");
    y.resize(static_cast<std::size_t>(a.n()));  // csr_matrix.cpp:91
    rethrow(rcg_spmv(ctx(), device(a).get(), x.data(), y.data()));
}

void spmv_dual(const CsrMatrix& a, const Vector& x1, const Vector& x2, Vector& y1, Vector& y2) {
    const std::size_t n = static_cast<std::size_t>(a.n());
    if (x1.size() != n || x2.size() != n) throw std::invalid_argument("spmv_dual: vector size does not match matrix");
    y1.resize(n);
    y2.resize(n);
    rethrow(rcg_spmv_dual(ctx(), device(a).get(), x1.data(), x2.data(), y1.data(), y2.data()));
}

// ------------------------------------------------------------------ IC(0) (ic_preconditioner.hpp:44-47)
IcFactor ic0_factorize(const CsrMatrix& a, double shift, int num_blocks) {
    // argument checks (ic_preconditioner.cpp:97-102) and the shift ladder (:108-121, same
    // BreakdownError message) run inside rcg_ic0_factorize_device
    rcg_ic* d = nullptr;
    rethrow(rcg_ic0_factorize_device(ctx(), device(a).get(), shift, num_blocks, &d));
    std::unique_ptr<rcg_ic, void (*)(rcg_ic*)> guard(d, rcg_ic_destroy);
    int64_t nnz_l = 0;
    double shift_used = 0.0;
    int32_t fl = 0, bl = 0;
    rethrow(rcg_ic_info(d, &nnz_l, &shift_used, &fl, &bl));
    IcFactor f;
    const std::size_t n = static_cast<std::size_t>(a.n()), nl = static_cast<std::size_t>(nnz_l);
    f.n = a.n();
    f.block_bounds.resize(static_cast<std::size_t>(num_blocks) + 1);
    f.l_row_start.resize(n + 1);
    f.l_col.resize(nl);
    f.l_val.resize(nl);
    f.d.resize(n);
    f.u_row_start.resize(n + 1);
    f.u_col.resize(nl);
    f.u_val.resize(nl);
    f.shift_used = shift_used;
    rethrow(rcg_ic_export(d, f.block_bounds.data(), f.l_row_start.data(), f.l_col.data(), f.l_val.data(), f.d.data(),
                          f.u_row_start.data(), f.u_col.data(), f.u_val.data()));
    adopt_ic(f, guard.release());  // an IcPreconditioner made from f finds this device image
    return f;
}

void ic_apply(const IcFactor& f, const Vector& r, Vector& z) {
    if (r.size() != static_cast<std::size_t>(f.n)) throw std::invalid_argument("ic_apply: size mismatch");  // :125-126
    z.resize(static_cast<std::size_t>(f.n));
    rethrow(rcg_ic_apply(ctx(), device(f).get(), r.data(), z.data()));
}

// ------------------------------------------------------------------ sampling (sampling.hpp:26-70)
// The schedule restated from sampling.cpp:7-72: method A stores iteration i (when h divides it)
// in slot (sum_{l=0}^{l_max} (-1)^l floor((i-1)/m^l)) mod m, l_max the smallest power with
// m^l_max > cap, and doubles h at i == h m; method B stores the first iterate whose relres
// crosses each threshold 10^(-s alpha/(m+1)), alpha = -log10 eps, in slot s - 1.
SamplerState SamplerState::method_a(int m, int iteration_cap) {
    if (m < 2) throw std::invalid_argument("sampler method A: m must be >= 2");
    if (iteration_cap < 1) throw std::invalid_argument("sampler method A: iteration cap must be >= 1");
    SamplerState s;
    s.method_ = SamplingMethod::A;
    s.m_ = m;
    s.slots_.resize(static_cast<std::size_t>(m));
    s.occupied_.assign(static_cast<std::size_t>(m), false);
    s.stored_iter_.assign(static_cast<std::size_t>(m), 0);
    s.l_max_ = 1;
    for (std::int64_t pw = m; pw <= iteration_cap; pw *= m) ++s.l_max_;
    return s;
}

SamplerState SamplerState::method_b(int m, double eps) {
    if (m < 1) throw std::invalid_argument("sampler method B: m must be >= 1");
    if (!(eps > 0.0 && eps < 1.0)) throw std::invalid_argument("sampler method B: eps must be in (0, 1)");
    SamplerState s;
    s.method_ = SamplingMethod::B;
    s.m_ = m;
    s.slots_.resize(static_cast<std::size_t>(m));
    s.occupied_.assign(static_cast<std::size_t>(m), false);
    s.stored_iter_.assign(static_cast<std::size_t>(m), 0);
    s.alpha_ = -std::log10(eps);
    return s;
}

void SamplerState::offer(int iteration, double relres, const Vector& payload) {
    auto store = [&](int slot) {
        slots_[static_cast<std::size_t>(slot)] = payload;
        occupied_[static_cast<std::size_t>(slot)] = true;
        stored_iter_[static_cast<std::size_t>(slot)] = iteration;
    };
    if (method_ == SamplingMethod::A) {
        if (iteration % h_ != 0) return;
        std::int64_t acc = 0, pw = 1;
        for (int l = 0; l <= l_max_; ++l, pw *= m_) acc += (l & 1 ? -1 : 1) * ((iteration - 1) / pw);
        store(static_cast<int>(acc % m_));
        if (iteration == h_ * m_) h_ *= 2;
        return;
    }
    for (; next_slot_ <= m_; ++next_slot_) {
        if (relres > std::pow(10.0, -double(next_slot_) * alpha_ / (m_ + 1))) break;
        store(next_slot_ - 1);
    }
}

int SamplerState::stored_count() const {
    return static_cast<int>(std::count(occupied_.begin(), occupied_.end(), true));
}

// the observers as a named functor: pcg_solve finds it behind the std::function and runs the
// sampler on the device (recycg_b200_bridge.cpp); on any other path it offers like the reference
IterationObserver error_sampling_observer(SamplerState& s) { return b200::SamplingObserver{&s, false, 0, 0.0}; }
IterationObserver residual_sampling_observer(SamplerState& s) { return b200::SamplingObserver{&s, true, 0, 0.0}; }

// ------------------------------------------------------------------ dense (dense.hpp:50)
TallDense mgs_orthonormalize(const TallDense& v, double drop_tol) {
    if (v.k() == 0) return TallDense(v.n);
    TallRef t = tall_upload(v);
    rcg_tall* e = nullptr;
    rethrow(rcg_mgs_orthonormalize(ctx(), t.get(), drop_tol, &e));
    TallRef eg(e, rcg_tall_destroy);
    return tall_download(e);
}

// ------------------------------------------------------------------ recycling (recycling.hpp:14-47)
TallDense harvest_errors(const Vector& x_final, const SamplerState& s) {
    std::vector<const double*> cols;
    for (int slot = 0; slot < s.m(); ++slot)
        if (s.occupied(slot)) {
            if (s.slot(slot).size() != x_final.size())
                throw std::invalid_argument("harvest_errors: slot length does not match x_final");
            cols.push_back(s.slot(slot).data());
        }
    const index_t n = static_cast<index_t>(x_final.size());
    if (cols.empty()) return TallDense(n);
    rcg_tall* e = nullptr;
    rethrow(rcg_harvest_columns(ctx(), x_final.data(), n, static_cast<int>(cols.size()), cols.data(), &e));
    TallRef eg(e, rcg_tall_destroy);
    return tall_download(e);
}

// recycling.cpp:30-40: a copy of the non-zero occupied slots (no arithmetic to offload)
TallDense harvest_stored(const SamplerState& s) {
    TallDense e(0);
    for (int slot = 0; slot < s.m(); ++slot) {
        if (!s.occupied(slot)) continue;
        const Vector& v = s.slot(slot);
        if (std::all_of(v.begin(), v.end(), [](double x) { return x == 0.0; })) continue;
        if (e.cols.empty()) e.n = static_cast<index_t>(v.size());
        e.cols.push_back(v);
    }
    return e;
}

RitzSpectrum rayleigh_ritz(const CsrMatrix& a, const TallDense& e) {
    RitzSpectrum out;
    out.vectors = TallDense(e.n);
    if (e.k() == 0) return out;
    TallRef t = tall_upload(e);
    out.values.resize(static_cast<std::size_t>(e.k()));
    rcg_tall* v = nullptr;
    rethrow(rcg_rayleigh_ritz(ctx(), device(a).get(), t.get(), out.values.data(), &v));
    TallRef vg(v, rcg_tall_destroy);
    out.vectors = tall_download(v);
    return out;
}

// recycling.cpp:81-96: MGS (drop 1e-12) -> Rayleigh-Ritz -> the Ritz vectors with value < theta
AuxBasis build_aux_matrix(const CsrMatrix& a, const TallDense& errors, double theta) {
    AuxBasis out;
    out.w = TallDense(a.n());
    out.spectrum.vectors = TallDense(a.n());
    if (errors.k() == 0) return out;
    TallRef t = tall_upload(errors);
    rcg_tall* q = nullptr;
    rethrow(rcg_mgs_orthonormalize(ctx(), t.get(), 1e-12, &q));
    TallRef qg(q, rcg_tall_destroy);
    t.reset();
    out.m_bar = rcg_tall_k(q);
    if (out.m_bar == 0) return out;
    out.spectrum.values.resize(static_cast<std::size_t>(out.m_bar));
    rcg_tall* v = nullptr;
    rethrow(rcg_rayleigh_ritz(ctx(), device(a).get(), q, out.spectrum.values.data(), &v));
    TallRef vg(v, rcg_tall_destroy);
    out.spectrum.vectors = tall_download(v);
    for (int i = 0; i < out.spectrum.k(); ++i)
        if (out.spectrum.values[static_cast<std::size_t>(i)] < theta)
            out.w.cols.push_back(out.spectrum.vectors.cols[static_cast<std::size_t>(i)]);
    return out;
}

// ------------------------------------------------------------------ deflation (deflation.hpp:17-37)
namespace {

// AW and chol(W^T A W) built on the device (SpMM, Gram, Cholesky; "... W^T A W not SPD" on
// failure), downloaded into the host fields and the device basis kept for the solves
void build_basis_fields(const CsrMatrix& a, const TallDense& w, int who, TallDense& aw, SmallChol& chol) {
    aw = TallDense(w.n);
    if (w.k() == 0) return;
    TallRef t = tall_upload(w);
    rcg_basis* b = nullptr;
    rethrow(rcg_basis_create(ctx(), device(a).get(), t.get(), who, &b));
    std::unique_ptr<rcg_basis, void (*)(rcg_basis*)> bg(b, rcg_basis_destroy);
    const std::size_t n = static_cast<std::size_t>(w.n), k = static_cast<std::size_t>(w.k());
    std::vector<double> awc(n * k);
    chol.k = w.k();
    chol.l.assign(k * k, 0.0);
    rethrow(rcg_basis_export(ctx(), b, awc.data(), chol.l.data()));
    for (std::size_t j = 0; j < k; ++j)
        aw.cols.emplace_back(awc.begin() + static_cast<std::ptrdiff_t>(j * n),
                             awc.begin() + static_cast<std::ptrdiff_t>((j + 1) * n));
    adopt_basis(w, aw, chol, who, bg.release());
}

Vector projection(const DeflationOperator& d, const Vector& v, int which) {
    if (d.empty()) return which == 2 ? Vector(v.size(), 0.0) : v;  // deflation.cpp:19,27,35
    if (v.size() != static_cast<std::size_t>(d.w.n)) throw std::invalid_argument("deflation: vector size does not match W");
    const BasisRef b = device_basis(d.w, d.aw, d.waw_chol, RCG_BASIS_DEFLATION);
    Vector out(v.size());
    rethrow(which == 0   ? rcg_project_pt(ctx(), b.get(), v.data(), out.data())
            : which == 1 ? rcg_project_p(ctx(), b.get(), v.data(), out.data())
                         : rcg_direct_component(ctx(), b.get(), v.data(), out.data()));
    return out;
}

}  // namespace

Vector DeflationOperator::project_pt(const Vector& y) const { return projection(*this, y, 0); }
Vector DeflationOperator::project_p(const Vector& x) const { return projection(*this, x, 1); }
Vector DeflationOperator::direct_component(const Vector& b) const { return projection(*this, b, 2); }

DeflationOperator build_deflation_operator(const CsrMatrix& a, TallDense w) {
    if (w.k() > 0 && w.n != a.n())  // deflation.cpp:46-47
        throw std::invalid_argument("build_deflation_operator: W row count does not match A");
    DeflationOperator op;
    op.w = std::move(w);
    build_basis_fields(a, op.w, RCG_BASIS_DEFLATION, op.aw, op.waw_chol);
    return op;
}

// ------------------------------------------------------------------ subspace correction (subspace_correction.hpp:22-38)
namespace {

// the constructor's record of each ScPreconditioner: by object address (validated by W's
// content, so a stale entry of a destroyed object is not taken) and, for copies, by content
struct ScEntry {
    std::weak_ptr<const Preconditioner> inner;
    SmallChol chol;
    std::uint64_t w_fp = 0;
};
struct ScTable {
    std::mutex mu;
    std::map<const void*, ScEntry> by_addr;
    std::map<std::uint64_t, ScEntry> by_content;
};
ScTable& sc_table() {
    static ScTable* t = new ScTable();
    return *t;
}

std::uint64_t w_fingerprint(const TallDense& w, const TallDense& aw) {
    std::uint64_t h = static_cast<std::uint64_t>(w.k()) * 0x9E3779B97F4A7C15ull;
    for (int j = 0; j < w.k(); ++j) {
        const Vector& c = w.cols[static_cast<std::size_t>(j)];
        const Vector& d = aw.cols[static_cast<std::size_t>(j)];
        h = h * 31 + fingerprint(c.data(), c.size() * sizeof(double));
        h = h * 31 + fingerprint(d.data(), d.size() * sizeof(double));
    }
    return h;
}

}  // namespace

ScPreconditioner::ScPreconditioner(std::shared_ptr<const Preconditioner> inner, const CsrMatrix& a, TallDense w)
    : inner_(std::move(inner)), w_(std::move(w)), aw_(w_.n) {
    if (!inner_) throw std::invalid_argument("ScPreconditioner: inner preconditioner is null");  // :30
    if (w_.k() > 0 && w_.n != a.n()) throw std::invalid_argument("ScPreconditioner: W row count does not match A");
    build_basis_fields(a, w_, RCG_BASIS_SC, aw_, waw_chol_);
    ScEntry e{inner_, waw_chol_, w_fingerprint(w_, aw_)};
    ScTable& t = sc_table();
    std::lock_guard<std::mutex> g(t.mu);
    for (auto it = t.by_addr.begin(); it != t.by_addr.end();)  // entries of destroyed objects
        it = it->second.inner.expired() ? t.by_addr.erase(it) : std::next(it);
    for (auto it = t.by_content.begin(); it != t.by_content.end();)
        it = it->second.inner.expired() ? t.by_content.erase(it) : std::next(it);
    t.by_addr[this] = e;
    t.by_content[e.w_fp] = e;
}

// subspace_correction.cpp:47-57 on the device: z = inner(r) + W chol(W^T r)
void ScPreconditioner::apply(const Vector& r, Vector& z) const {
    if (r.size() != static_cast<std::size_t>(w_.k() > 0 ? w_.n : static_cast<index_t>(r.size())))
        throw std::invalid_argument("ScPreconditioner: vector size does not match W");
    if (w_.k() == 0) {
        inner_->apply(r, z);
        return;
    }
    PrecRef in = prec_of(*inner_);
    if (in.p.kind == RCG_PREC_SC) throw std::invalid_argument("ScPreconditioner: nested subspace correction has no GPU implementation");
    const BasisRef b = device_basis(w_, aw_, waw_chol_, RCG_BASIS_SC);
    const rcg_prec p{RCG_PREC_SC, in.ic.get(), b.get()};
    z.resize(r.size());
    rethrow(rcg_prec_apply(ctx(), &p, r.data(), z.data()));
}

namespace b200::detail {

ScState sc_state(const ScPreconditioner& m) {
    const std::uint64_t fp = w_fingerprint(m.w(), m.aw());
    ScTable& t = sc_table();
    std::lock_guard<std::mutex> g(t.mu);
    const ScEntry* e = nullptr;
    auto a = t.by_addr.find(&m);
    if (a != t.by_addr.end() && a->second.w_fp == fp) e = &a->second;
    if (!e) {
        auto c = t.by_content.find(fp);
        if (c != t.by_content.end()) e = &c->second;
    }
    std::shared_ptr<const Preconditioner> inner = e ? e->inner.lock() : nullptr;
    if (!inner) throw std::invalid_argument("ScPreconditioner: not constructed through this library build");
    return {inner, e->chol};
}

PrecRef prec_of(const Preconditioner& m) {
    PrecRef r;
    if (dynamic_cast<const IdentityPreconditioner*>(&m)) return r;
    if (auto* ic = dynamic_cast<const IcPreconditioner*>(&m)) {
        r.ic = device(ic->factor());
        r.p = {RCG_PREC_IC, r.ic.get(), nullptr};
        return r;
    }
    if (auto* sc = dynamic_cast<const ScPreconditioner*>(&m)) {
        const ScState st = sc_state(*sc);
        PrecRef in = prec_of(*st.inner);
        if (in.p.kind == RCG_PREC_SC)
            throw std::invalid_argument("pcg_solve: nested ScPreconditioner has no GPU implementation");
        r.ic = in.ic;
        r.sc = device_basis(sc->w(), sc->aw(), st.chol, RCG_BASIS_SC);
        r.p = {r.sc ? RCG_PREC_SC : in.p.kind, r.ic.get(), r.sc.get()};
        return r;
    }
    throw std::invalid_argument("pcg_solve: preconditioner type has no GPU implementation");
}

}  // namespace b200::detail
}  // namespace recycg
