// gen_math.h -- arithmetic shared by the host generator (generators.cpp, also compiled by g++
// into oracle/libgen_host.so) and the device generator (gen_device.cu), so both produce the
// same bits.  Every operation is a single IEEE-754 double add / sub / mul / div / sqrt or an
// exact operation (floor, power-of-two scaling); nothing is left to a libm whose last bit differs
// between glibc and CUDA.  Host builds use -ffp-contract=off, device code the _rn intrinsics.
#pragma once

#include <cstdint>
#include <cstring>

#if defined(__CUDACC__)
#define RCG_GM_HD __host__ __device__ __forceinline__
#else
#define RCG_GM_HD inline
#endif

namespace rcg {
namespace gm {

#if defined(__CUDA_ARCH__)
RCG_GM_HD double mul(double a, double b) { return __dmul_rn(a, b); }
RCG_GM_HD double add(double a, double b) { return __dadd_rn(a, b); }
RCG_GM_HD double sub(double a, double b) { return __dsub_rn(a, b); }
RCG_GM_HD double bits_to_double(uint64_t u) { return __longlong_as_double(static_cast<long long>(u)); }
#else
RCG_GM_HD double mul(double a, double b) { return a * b; }
RCG_GM_HD double add(double a, double b) { return a + b; }
RCG_GM_HD double sub(double a, double b) { return a - b; }
RCG_GM_HD double bits_to_double(uint64_t u) {
    double d;
    std::memcpy(&d, &u, sizeof d);
    return d;
}
#endif

// 2^k for -1022 <= k <= 1023 (exact)
RCG_GM_HD double pow2(int k) { return bits_to_double(static_cast<uint64_t>(k + 1023) << 52); }

// exp(x): Cody-Waite reduction x = k ln2 + r (|r| <= ln2/2, the fdlibm split of ln2 so k ln2_hi
// is exact), a degree-13 Taylor polynomial in Horner form (truncation < 1e-17 relative), then an
// exact scaling by 2^k (two steps below the normal range: one rounding into the subnormals).
// Max error about 1 ulp against a correctly rounded exp -- a generator function, not libm.
RCG_GM_HD double exp(double x) {
    if (!(x > -745.2)) return 0.0;
    if (x > 709.7) return pow2(1023) * 2.0;  // +inf
    const double inv_ln2 = 1.4426950408889634074;
    const double ln2_hi = 6.93147180369123816490e-01;  // 0x3fe62e42fee00000
    const double ln2_lo = 1.90821492927058770002e-10;  // 0x3dea39ef35793c76
    double kd = add(mul(x, inv_ln2), 0.5);
#if defined(__CUDA_ARCH__)
    kd = ::floor(kd);
#else
    kd = __builtin_floor(kd);
#endif
    const int k = static_cast<int>(kd);
    const double r = sub(sub(x, mul(kd, ln2_hi)), mul(kd, ln2_lo));
    // 1/j! for j = 13 .. 2
    const double c[12] = {1.6059043836821614599e-10, 2.0876756987868098979e-09, 2.5052108385441718775e-08,
                          2.7557319223985890653e-07, 2.7557319223985890653e-06, 2.4801587301587301566e-05,
                          1.9841269841269841253e-04, 1.3888888888888888889e-03, 8.3333333333333333333e-03,
                          4.1666666666666666667e-02, 1.6666666666666666667e-01, 5.0000000000000000000e-01};
    double p = c[0];
    for (int j = 1; j < 12; ++j) p = add(mul(p, r), c[j]);
    p = add(mul(p, r), 1.0);
    p = add(mul(p, r), 1.0);
    if (k >= -1022) return k > 1023 ? mul(mul(p, pow2(1023)), pow2(k - 1023)) : mul(p, pow2(k));
    return mul(mul(p, pow2(k + 54)), pow2(-54));
}

// The fixed-order sum used for the generator's global means: sequential within chunks of
// kSumChunk terms (from 0.0), then sequential over the chunk sums -- a device kernel reproduces
// it with one thread per chunk.
constexpr int64_t kSumChunk = 4096;

}  // namespace gm
}  // namespace rcg
