// philox.hpp -- counter-based RNG of the CUDA path (host + device).
//
// Philox4x32-10 (Salmon et al., SC'11) and the RNG contract of qtraj.h:
// key = (seed_lo32, seed_hi32), counter = (ordinal, purpose, traj_lo32,
// traj_hi32); u53(a, b) = ((a >> 5) * 2^26 + (b >> 6)) * 2^-53 in [0, 1).
// Alg. 2 line 3 draws one r per channel; the sampler draws one
// uniform per level.  This is the product's own implementation; the oracle
// implements the same contract separately (no shared code).
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define QT_HD __host__ __device__ __forceinline__
#else
#define QT_HD inline
#endif

namespace qt {

enum : uint32_t { kPurposeChannel = 1, kPurposeSample = 2, kPurposeReadout = 3 };

struct U32x4 { uint32_t v[4]; };

QT_HD void mulhilo32(uint32_t a, uint32_t b, uint32_t& hi, uint32_t& lo) {
#if defined(__CUDA_ARCH__)
    lo = a * b;
    hi = __umulhi(a, b);
#else
    uint64_t p = (uint64_t)a * (uint64_t)b;
    hi = (uint32_t)(p >> 32);
    lo = (uint32_t)p;
#endif
}

QT_HD U32x4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                          uint32_t k0, uint32_t k1) {
    const uint32_t kM0 = 0xD2511F53u, kM1 = 0xCD9E8D57u;
    const uint32_t kW0 = 0x9E3779B9u, kW1 = 0xBB67AE85u;
#pragma unroll
    for (int i = 0; i < 10; ++i) {
        uint32_t h0, l0, h1, l1;
        mulhilo32(kM0, c0, h0, l0);
        mulhilo32(kM1, c2, h1, l1);
        const uint32_t n0 = h1 ^ c1 ^ k0;
        const uint32_t n2 = h0 ^ c3 ^ k1;
        c0 = n0; c1 = l1; c2 = n2; c3 = l0;
        k0 += kW0; k1 += kW1;
    }
    U32x4 r;
    r.v[0] = c0; r.v[1] = c1; r.v[2] = c2; r.v[3] = c3;
    return r;
}

QT_HD double u53(uint32_t a, uint32_t b) {
    const uint64_t bits = ((uint64_t)(a >> 5) << 26) | (uint64_t)(b >> 6);
    return (double)bits * (1.0 / 9007199254740992.0);
}

// Uniform of (seed, ordinal, purpose, traj), half 0 -> (x0, x1), 1 -> (x2, x3).
QT_HD double draw(uint64_t seed, uint32_t ordinal, uint32_t purpose, uint64_t traj, int half) {
    U32x4 x = philox4x32_10(ordinal, purpose, (uint32_t)traj, (uint32_t)(traj >> 32),
                            (uint32_t)seed, (uint32_t)(seed >> 32));
    return half ? u53(x.v[2], x.v[3]) : u53(x.v[0], x.v[1]);
}

}  // namespace qt
