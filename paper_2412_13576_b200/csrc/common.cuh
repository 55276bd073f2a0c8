// Shared device helpers for the MAPLE sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace maple {

// splitmix64 finaliser (the start-sampling counter RNG, reading #2 in DESIGN.md §3).
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// U in [0, 1) for (seed, global start i, coordinate j): x = mix(seed ^ mix(i*n + j + 1)), U = (x>>11) 2^-53.
__device__ __forceinline__ double counter_uniform(uint64_t seed, int64_t i, int j, int n) {
    uint64_t key = (uint64_t)i * (uint64_t)n + (uint64_t)j + 1ULL;
    uint64_t x = splitmix64(seed ^ splitmix64(key));
    return (double)(x >> 11) * 0x1.0p-53;
}

// g0_j = (l_j - u_j) + U * (2 (u_j - l_j)) with explicit IEEE roundings (no FMA contraction), so the
// value is bit-identical to the fp64 oracle's (Alg. 3 line 4).
__device__ __forceinline__ double start_coord(double U, int lo, int hi) {
    return __dadd_rn((double)(lo - hi), __dmul_rn(U, (double)(2 * (hi - lo))));
}

// nearest integer, halves away from zero (reading #6); exact because z - trunc(z) is exact.
__device__ __forceinline__ int round_half_away(float z) {
    float t = truncf(z);
    float f = z - t;
    int r = (int)t;
    if (fabsf(f) >= 0.5f) r += (z > 0.f) ? 1 : -1;
    return r;
}

// round half away from zero in float (the same value as round_half_away; + 0 turns -0 into +0):
// trunc(z + copysign(1/2, z)) with the addition rounded toward zero. Below 2^24 every integer is representable,
// so rounding |z| + 1/2 toward zero never drops below floor(|z| + 1/2): the truncation is that floor (e.g.
// 0.49999997 + 0.5 -> 0.99999994 -> 0, where round-to-nearest would give 1.0); from 2^23 on z is an integer
// and the sum rounds back to it. Four instructions instead of seven.
__device__ __forceinline__ float round_half_away_f(float z) {
    const float h = __uint_as_float((__float_as_uint(z) & 0x80000000u) | 0x3F000000u);   // copysign(0.5, z)
    return truncf(__fadd_rz(z, h)) + 0.f;
}

__device__ __forceinline__ float fsign(float y) { return (float)((y > 0.f) - (y < 0.f)); }

__device__ __forceinline__ uint64_t mix64(uint64_t h) { return splitmix64(h); }

}  // namespace maple
