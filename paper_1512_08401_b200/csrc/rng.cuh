// The reference's counter RNG on the device: the i-th draw of CounterRng(seed).next_normal()
// (`proj/src/rng.hpp:30-43`; splitmix64 counter stream, Box-Muller pairs (cos, sin)). The
// step estimate's start vector is CounterRng(0x5eed) over all n (`solver.cpp:74-77`).
#pragma once

#include <cstdint>

namespace wbx {

__device__ __forceinline__ uint64_t rng_at(uint64_t seed, uint64_t i) {
    uint64_t z = seed + 0x9e3779b97f4a7c15ull * (i + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ double rng_u01(uint64_t v) {
    return (static_cast<double>(v >> 11) + 0.5) * 0x1p-53;
}
__device__ __forceinline__ double rng_normal(uint64_t seed, uint64_t i) {
    const uint64_t m = i >> 1;
    const double u1 = rng_u01(rng_at(seed, 2 * m));
    const double u2 = rng_u01(rng_at(seed, 2 * m + 1));
    const double r = sqrt(-2.0 * log(u1));
    const double a = 2.0 * M_PI * u2;
    return (i & 1) ? r * sin(a) : r * cos(a);
}

}  // namespace wbx
