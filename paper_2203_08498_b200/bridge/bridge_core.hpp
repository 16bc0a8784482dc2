// bridge_core.hpp -- shared plumbing of the C++ drop-in (recycg_b200_*.cpp): per-thread device
// contexts, status -> exception mapping, and the device images of the reference's immutable
// objects (CsrMatrix, IcFactor, TallDense bases) reused across calls.
//
// Image reuse is keyed by the host object's address and size AND validated by a content
// fingerprint of every array (a multi-threaded 64-bit hash, recomputed on every call): the
// reference API has no "release" step, so a freed object's address can come back holding
// different values -- a cache hit is only taken when the contents are the same.  Each cache is
// bounded (least recently used entries are dropped); a dropped image stays alive while a call
// that took it is still running (shared_ptr).
//
// Threading (distinct solves on shared A / M / D may run concurrently): every
// thread gets its own rcg_ctx (own CUDA stream, workspaces, pinned flags); the caches are
// guarded by one mutex, and images are read-only once built.
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "rcg_b200.h"
#include "recycg/csr_matrix.hpp"
#include "recycg/dense.hpp"
#include "recycg/ic_preconditioner.hpp"
#include "recycg/preconditioner.hpp"
#include "recycg/subspace_correction.hpp"

namespace recycg::b200::detail {

// RCG_E_INVALID -> std::invalid_argument, RCG_E_BREAKDOWN -> BreakdownError, RCG_E_PARSE ->
// ParseError, RCG_E_CUDA -> std::runtime_error (no GPU / CUDA fault: there is no CPU path)
void rethrow(int st);

// this thread's context on device 0 (created on first use, destroyed at thread exit)
rcg_ctx* ctx();

// order-independent 64-bit fingerprint of `bytes` bytes (position-mixed words, summed over
// worker threads for large arrays)
std::uint64_t fingerprint(const void* p, std::size_t bytes);

using MatrixRef = std::shared_ptr<rcg_matrix>;
using IcRef = std::shared_ptr<rcg_ic>;
using BasisRef = std::shared_ptr<rcg_basis>;
using TallRef = std::unique_ptr<rcg_tall, void (*)(rcg_tall*)>;

MatrixRef device(const CsrMatrix& a);
IcRef device(const IcFactor& f);
// the device image of a host basis exactly as its fields hold it -- W, AW and chol(W^T A W)
// (DeflationOperator's public fields; ScPreconditioner's w() / aw() and its factor) -- for
// deflation (RCG_BASIS_DEFLATION) or subspace correction (RCG_BASIS_SC); null for an empty W
BasisRef device_basis(const TallDense& w, const TallDense& aw, const SmallChol& chol, int who);
// adopt a basis just built on the device (build_deflation_operator / the ScPreconditioner
// constructor) under the fingerprint of the host fields downloaded from it, so the solves that
// follow find it without an upload
void adopt_basis(const TallDense& w, const TallDense& aw, const SmallChol& chol, int who, rcg_basis* b);

// ic0_factorize's device factor, cached under the content of the IcFactor exported from it
void adopt_ic(const IcFactor& f, rcg_ic* d);

// a Preconditioner's device form: identity, IC(0), or subspace correction over one of them
struct PrecRef {
    rcg_prec p{RCG_PREC_IDENTITY, nullptr, nullptr};
    IcRef ic;
    BasisRef sc;
};
PrecRef prec_of(const Preconditioner& m);

// what the bridge's ScPreconditioner constructor recorded (its inner preconditioner and
// chol(W^T A W) are private members, subspace_correction.hpp:34-37)
struct ScState {
    std::shared_ptr<const Preconditioner> inner;
    SmallChol chol;
};
ScState sc_state(const ScPreconditioner& m);

TallRef tall_upload(const TallDense& t);
TallDense tall_download(const rcg_tall* t);

// every cached image dropped (tests; images in use stay alive until their calls return)
void release_all();

}  // namespace recycg::b200::detail
