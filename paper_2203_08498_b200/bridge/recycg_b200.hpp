// recycg_b200.hpp -- the C++ side of the drop-in: the reference's own solver declarations
// (proj/include/recycg/pcg.hpp:39-52) are DEFINED over librcg_b200 by recycg_b200_bridge.cpp,
// which replaces src/pcg.cpp in a build of the reference library.  Everything else of the
// reference (CsrMatrix, ic0_factorize, the recycling step, build_deflation_operator, the drivers)
// links unchanged.
//
// The one call-site change: the error-sampling observer.  The reference's
// error_sampling_observer(s) (src/sampling.cpp:74-78) returns a lambda, whose type no other
// translation unit can name, so pcg_solve cannot recognise it behind the std::function.  This
// header gives the same observer as a NAMED functor: on any CPU path it behaves exactly like the
// reference's (it calls s.offer(iter, relres, x or r)); the bridge's pcg_solve finds it with
// std::function::target<>, runs the sampler on the device inside the solve (rcg_sampler) and
// replays the outcome into `s` through its public offer(), so `s` ends in the state the host
// solve would have left (same occupied slots, stored iterations and schedule counters).
#pragma once

#include "recycg/pcg.hpp"
#include "recycg/sampling.hpp"

namespace recycg::b200 {

struct SamplingObserver {
    SamplerState* s;
    bool residual;      // false: error sampling (payload x), true: residual sampling (payload r)
    int iteration_cap;  // method A: the cap given to SamplerState::method_a
    double eps;         // method B: the eps given to SamplerState::method_b
    void operator()(int iter, double relres, const Vector& x, const Vector& r) const {
        s->offer(iter, relres, residual ? r : x);
    }
};

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

// drop the cached device images (matrices, factors, bases) -- call before freeing the host
// objects they were made from if their addresses may be reused for different contents
void release_device_images();

}  // namespace recycg::b200
