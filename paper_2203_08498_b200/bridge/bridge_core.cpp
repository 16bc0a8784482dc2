// bridge_core.cpp -- see bridge_core.hpp.
#include "bridge_core.hpp"

#include <algorithm>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <thread>

#include "recycg/types.hpp"

namespace recycg::b200::detail {

void rethrow(int st) {
    if (st == RCG_OK) return;
    const std::string m = rcg_last_error();
    if (st == RCG_E_INVALID) throw std::invalid_argument(m);
    if (st == RCG_E_BREAKDOWN) throw BreakdownError(m);
    if (st == RCG_E_PARSE) throw ParseError(m);
    throw std::runtime_error("librcg_b200: " + m);
}

namespace {

struct CtxHolder {
    rcg_ctx* c = nullptr;
    ~CtxHolder() {
        if (c) rcg_ctx_destroy(c);
    }
};

}  // namespace

rcg_ctx* ctx() {
    thread_local CtxHolder h;
    if (!h.c) rethrow(rcg_ctx_create(0, &h.c));
    return h.c;
}

// ------------------------------------------------------------------ fingerprints
namespace {

inline std::uint64_t mix(std::uint64_t w, std::uint64_t i) {
    std::uint64_t z = w ^ (i * 0x9E3779B97F4A7C15ull);
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 31;
    z *= 0x94D049BB133111EBull;
    return z ^ (z >> 29);
}

std::uint64_t hash_words(const unsigned char* p, std::size_t words, std::uint64_t first) {
    std::uint64_t acc = 0;
    for (std::size_t i = 0; i < words; ++i) {
        std::uint64_t w;
        std::memcpy(&w, p + 8 * i, 8);
        acc += mix(w, first + i);
    }
    return acc;
}

// one stream of arrays, word positions continuing across arrays
struct Stream {
    std::vector<std::pair<const void*, std::size_t>> parts;
    void add(const void* p, std::size_t bytes) { parts.emplace_back(p, bytes); }
};

std::uint64_t fingerprint_stream(const Stream& s) {
    std::size_t total = 0;
    for (auto& pr : s.parts) total += pr.second;
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const unsigned nt = total < (std::size_t(64) << 20) ? 1u : std::min(hw, 32u);
    std::uint64_t acc = 0, pos = 0;
    for (auto& pr : s.parts) {
        const auto* p = static_cast<const unsigned char*>(pr.first);
        const std::size_t words = pr.second / 8;
        if (nt == 1 || words < (std::size_t(1) << 20)) {
            acc += hash_words(p, words, pos);
        } else {
            std::vector<std::uint64_t> part(nt, 0);
            std::vector<std::thread> th;
            const std::size_t chunk = (words + nt - 1) / nt;
            for (unsigned t = 0; t < nt; ++t) {
                const std::size_t w0 = std::min(words, t * chunk), w1 = std::min(words, w0 + chunk);
                th.emplace_back([&, t, w0, w1] { part[t] = hash_words(p + 8 * w0, w1 - w0, pos + w0); });
            }
            for (auto& x : th) x.join();
            for (auto v : part) acc += v;
        }
        std::uint64_t tail = 0;  // the last bytes of an array not filling a word
        if (pr.second % 8) std::memcpy(&tail, p + 8 * words, pr.second % 8);
        acc += mix(tail ^ 0xA5A5A5A5A5A5A5A5ull, pos + words);
        pos += words + 1;
    }
    return acc ^ mix(total, 0x5EEDull);
}

}  // namespace

std::uint64_t fingerprint(const void* p, std::size_t bytes) {
    Stream s;
    s.add(p, bytes);
    return fingerprint_stream(s);
}

// ------------------------------------------------------------------ bounded content-keyed caches
namespace {

struct Key {
    std::uint64_t a = 0, b = 0, c = 0, d = 0;
    bool operator==(const Key& o) const { return a == o.a && b == o.b && c == o.c && d == o.d; }
};

template <class H>
struct Cache {
    struct Entry {
        Key key;
        std::shared_ptr<H> h;
        std::uint64_t tick;
    };
    std::size_t cap;
    std::vector<Entry> e;
    explicit Cache(std::size_t c) : cap(c) {}
    std::shared_ptr<H> find(const Key& k, std::uint64_t tick) {
        for (auto& x : e)
            if (x.key == k) {
                x.tick = tick;
                return x.h;
            }
        return nullptr;
    }
    std::shared_ptr<H> put(const Key& k, std::shared_ptr<H> h, std::uint64_t tick) {
        if (auto old = find(k, tick)) return old;  // another thread built it meanwhile
        e.push_back({k, std::move(h), tick});
        while (e.size() > cap) {
            auto lru = std::min_element(e.begin(), e.end(), [](const Entry& x, const Entry& y) { return x.tick < y.tick; });
            e.erase(lru);
        }
        return e.back().key == k ? e.back().h : find(k, tick);
    }
};

struct Images {
    std::mutex mu;
    std::uint64_t tick = 0;
    Cache<rcg_matrix> mats{4};
    Cache<rcg_ic> ics{4};
    Cache<rcg_basis> bases{8};
};

Images& images() {
    static Images* im = new Images();  // never destroyed: images may outlive static teardown order
    return *im;
}

Key matrix_key(const CsrMatrix& a) {
    Stream s;
    s.add(a.row_start().data(), a.row_start().size() * sizeof(index_t));
    s.add(a.col_idx().data(), a.col_idx().size() * sizeof(index_t));
    s.add(a.values().data(), a.values().size() * sizeof(double));
    return {static_cast<std::uint64_t>(a.n()), static_cast<std::uint64_t>(a.nnz()), fingerprint_stream(s), 1};
}

Key basis_key(const TallDense& w, const TallDense& aw, const SmallChol& chol, int who) {
    Stream s;
    for (const Vector& c : w.cols) s.add(c.data(), c.size() * sizeof(double));
    for (const Vector& c : aw.cols) s.add(c.data(), c.size() * sizeof(double));
    s.add(chol.l.data(), chol.l.size() * sizeof(double));
    return {static_cast<std::uint64_t>(w.n) | (static_cast<std::uint64_t>(w.k()) << 32), fingerprint_stream(s),
            static_cast<std::uint64_t>(chol.k), static_cast<std::uint64_t>(who) + 2};
}

template <class H, class Make>
std::shared_ptr<H> get_or_build(Cache<H>& cache, const Key& k, Make&& make) {
    Images& im = images();
    {
        std::lock_guard<std::mutex> g(im.mu);
        if (auto h = cache.find(k, ++im.tick)) return h;
    }
    std::shared_ptr<H> built = make();
    rethrow(rcg_ctx_synchronize(ctx()));  // usable from every thread's stream from here on
    std::lock_guard<std::mutex> g(im.mu);
    return cache.put(k, std::move(built), ++im.tick);
}

}  // namespace

MatrixRef device(const CsrMatrix& a) {
    return get_or_build(images().mats, matrix_key(a), [&] {
        rcg_matrix* d = nullptr;
        // validate = 0: a CsrMatrix is validated by its constructor (csr_matrix.cpp:36-87)
        rethrow(rcg_matrix_create(ctx(), a.n(), a.row_start().data(), a.col_idx().data(), a.values().data(), 0, &d));
        return MatrixRef(d, rcg_matrix_destroy);
    });
}

namespace {
Key ic_key(const IcFactor& f) {
    Stream s;
    s.add(f.block_bounds.data(), f.block_bounds.size() * sizeof(index_t));
    s.add(f.l_row_start.data(), f.l_row_start.size() * sizeof(index_t));
    s.add(f.l_col.data(), f.l_col.size() * sizeof(index_t));
    s.add(f.l_val.data(), f.l_val.size() * sizeof(double));
    s.add(f.d.data(), f.d.size() * sizeof(double));
    s.add(f.u_row_start.data(), f.u_row_start.size() * sizeof(index_t));
    s.add(f.u_col.data(), f.u_col.size() * sizeof(index_t));
    s.add(f.u_val.data(), f.u_val.size() * sizeof(double));
    s.add(&f.shift_used, sizeof(double));
    return {static_cast<std::uint64_t>(f.n), f.l_val.size(), fingerprint_stream(s), 7};
}
}  // namespace

IcRef device(const IcFactor& f) {
    return get_or_build(images().ics, ic_key(f), [&] {
        rcg_ic* d = nullptr;
        rethrow(rcg_ic_create(ctx(), f.n, f.num_blocks(), f.block_bounds.data(), f.l_row_start.data(), f.l_col.data(),
                              f.l_val.data(), f.d.data(), f.u_row_start.data(), f.u_col.data(), f.u_val.data(),
                              f.shift_used, &d));
        return IcRef(d, rcg_ic_destroy);
    });
}

TallRef tall_upload(const TallDense& t) {
    std::vector<const double*> cols(t.cols.size());
    for (std::size_t j = 0; j < cols.size(); ++j) {
        if (static_cast<index_t>(t.cols[j].size()) != t.n) throw std::invalid_argument("TallDense: column length mismatch");
        cols[j] = t.cols[j].data();
    }
    rcg_tall* d = nullptr;
    rethrow(rcg_tall_create_cols(ctx(), t.n, t.k(), cols.empty() ? nullptr : cols.data(), &d));
    return TallRef(d, rcg_tall_destroy);
}

TallDense tall_download(const rcg_tall* t) {
    const index_t n = rcg_tall_n(t);
    const int k = rcg_tall_k(t);
    TallDense out(n);
    if (k == 0) return out;
    std::vector<double> buf(static_cast<std::size_t>(n) * k);
    rethrow(rcg_tall_download(ctx(), t, buf.data()));
    for (int j = 0; j < k; ++j)
        out.cols.emplace_back(buf.begin() + static_cast<std::ptrdiff_t>(j) * n,
                              buf.begin() + static_cast<std::ptrdiff_t>(j + 1) * n);
    return out;
}

BasisRef device_basis(const TallDense& w, const TallDense& aw, const SmallChol& chol, int who) {
    if (w.k() == 0) return nullptr;
    if (aw.k() != w.k() || aw.n != w.n || chol.k != w.k() ||
        chol.l.size() != static_cast<std::size_t>(w.k()) * static_cast<std::size_t>(w.k()))
        throw std::invalid_argument("basis: W, AW and chol(W^T A W) dimensions disagree");
    return get_or_build(images().bases, basis_key(w, aw, chol, who), [&] {
        std::vector<const double*> wc, ac;
        for (int j = 0; j < w.k(); ++j) {
            if (static_cast<index_t>(w.cols[j].size()) != w.n || static_cast<index_t>(aw.cols[j].size()) != w.n)
                throw std::invalid_argument("TallDense: column length mismatch");
            wc.push_back(w.cols[j].data());
            ac.push_back(aw.cols[j].data());
        }
        rcg_basis* b = nullptr;
        rethrow(rcg_basis_create_from(ctx(), w.n, w.k(), wc.data(), ac.data(), chol.l.data(), who, &b));
        return BasisRef(b, rcg_basis_destroy);
    });
}

void adopt_basis(const TallDense& w, const TallDense& aw, const SmallChol& chol, int who, rcg_basis* b) {
    BasisRef ref(b, rcg_basis_destroy);
    if (w.k() == 0) return;
    const Key k = basis_key(w, aw, chol, who);
    rethrow(rcg_ctx_synchronize(ctx()));
    Images& im = images();
    std::lock_guard<std::mutex> g(im.mu);
    im.bases.put(k, std::move(ref), ++im.tick);
}

void adopt_ic(const IcFactor& f, rcg_ic* d) {
    IcRef ref(d, rcg_ic_destroy);
    const Key k = ic_key(f);
    rethrow(rcg_ctx_synchronize(ctx()));
    Images& im = images();
    std::lock_guard<std::mutex> g(im.mu);
    im.ics.put(k, std::move(ref), ++im.tick);
}

void release_all() {
    Images& im = images();
    std::lock_guard<std::mutex> g(im.mu);
    im.mats.e.clear();
    im.ics.e.clear();
    im.bases.e.clear();
}

}  // namespace recycg::b200::detail

namespace recycg::b200 {
void release_device_images() { detail::release_all(); }
}  // namespace recycg::b200
