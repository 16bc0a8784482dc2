// recycg_b200.hpp -- the C++ side of the drop-in: the reference's own hot-path declarations
// (proj/include/recycg: pcg.hpp, condest.hpp, csr_matrix.hpp spmv / spmv_dual, ic_preconditioner.hpp,
// sampling.hpp, recycling.hpp, dense.hpp mgs_orthonormalize, deflation.hpp,
// subspace_correction.hpp) are DEFINED over librcg_b200 by recycg_b200_bridge.cpp and
// recycg_b200_ops.cpp, which replace those modules in a build of the reference library
// (bridge/Makefile).  A program written against the reference API needs no change: the
// reference's own error_sampling_observer(s) / residual_sampling_observer(s) return the named
// functor below, which pcg_solve finds behind the std::function (target<>), runs on the device
// inside the solve and replays into `s` through offer(), so `s` ends in the state the host solve
// would have left (same occupied slots, stored iterations and schedule counters).
#pragma once

#include "recycg/pcg.hpp"
#include "recycg/sampling.hpp"

namespace recycg::b200 {

struct SamplingObserver {
    SamplerState* s;
    bool residual;      // false: error sampling (payload x), true: residual sampling (payload r)
    int iteration_cap;  // method A: the cap given to SamplerState::method_a (0: the solve's max_iter)
    double eps;         // method B: the eps given to SamplerState::method_b (0: the solve's eps)
    void operator()(int iter, double relres, const Vector& x, const Vector& r) const {
        s->offer(iter, relres, residual ? r : x);
    }
};

// explicit variants naming the state's cap / eps (the reference factories use the solve's)
// error_sampling_observer(s) (sampling.hpp:67) for a method-A state made with method_a(m, cap)
inline IterationObserver error_sampling_observer_a(SamplerState& s, int iteration_cap) {
    return SamplingObserver{&s, false, iteration_cap, 0.0};
}
// ... and for a method-B state made with method_b(m, eps)
inline IterationObserver error_sampling_observer_b(SamplerState& s, double eps) {
    return SamplingObserver{&s, false, 0, eps};
}
// residual_sampling_observer(s) (sampling.hpp:70)
inline IterationObserver residual_sampling_observer_a(SamplerState& s, int iteration_cap) {
    return SamplingObserver{&s, true, iteration_cap, 0.0};
}

// drop the cached device images (matrices, factors, bases; optional -- the caches are bounded
// and every reuse is validated against the host object's contents)
void release_device_images();

}  // namespace recycg::b200
