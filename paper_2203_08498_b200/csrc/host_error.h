// host_error.h -- host-only error plumbing shared by librcg_b200.so and the standalone host
// generator build (oracle/Makefile builds csrc/generators.cpp with g++ alone, so the reference
// arm of bench.py never maps librcg_b200.so).  Status codes map 1:1 to the reference exceptions.
#pragma once

#include <stdint.h>

#include <new>
#include <stdexcept>
#include <string>

#include "rcg_b200.h"

namespace rcg {

// ------------------------------------------------------------------ errors
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_error(const std::string& msg);
void clear_error();

template <class F>
int guard(F&& f) {
    try {
        clear_error();
        f();
        return RCG_OK;
    } catch (const Error& e) {
        set_error(e.what());
        return e.code;
    } catch (const std::bad_alloc&) {
        set_error("host out of memory");
        return RCG_E_CUDA;
    } catch (const std::exception& e) {
        set_error(e.what());
        return RCG_E_CUDA;
    }
}

inline void require(bool ok, const std::string& msg, int code = RCG_E_INVALID) {
    if (!ok) throw Error(code, msg);
}

}  // namespace rcg
