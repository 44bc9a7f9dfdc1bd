// Philox4x64-10 counter-based generator, as used by numpy.random.Philox
// (Random123 constants), and numpy's float32 uniform draw on top of it.
//
// numpy's Philox bit generator keeps a 256-bit counter that it increments
// *before* producing each block of four 64-bit words; a fresh generator has
// counter 0, so block b (0-based) of a stream is philox(counter = b + 1, key).
// random(dtype=float32) consumes 32-bit halves of consecutive 64-bit words
// (low half first) and maps u -> (u >> 8) * 2^-24.  The reference draws
// h then x from the same stream (harness.py:97-107), so float index f of a
// trial lives in 64-bit word f / 2 (half f % 2), i.e. block f / 8.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define WINO_HD __host__ __device__ __forceinline__
#else
#define WINO_HD inline
#endif

namespace wino {

WINO_HD void mulhilo64(uint64_t a, uint64_t b, uint64_t* hi, uint64_t* lo) {
#if defined(__CUDA_ARCH__)
    *lo = a * b;
    *hi = __umul64hi(a, b);
#else
    unsigned __int128 p = (unsigned __int128)a * b;
    *lo = (uint64_t)p;
    *hi = (uint64_t)(p >> 64);
#endif
}

// One Philox4x64 block with 10 rounds.
WINO_HD void philox4x64_10(const uint64_t ctr_in[4], uint64_t k0, uint64_t k1, uint64_t out[4]) {
    const uint64_t M0 = 0xD2E7470EE14C6C93ULL, M1 = 0xCA5A826395121157ULL;
    const uint64_t W0 = 0x9E3779B97F4A7C15ULL, W1 = 0xBB67AE8584CAA73BULL;
    uint64_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    for (int r = 0; r < 10; ++r) {
        if (r > 0) {
            k0 += W0;
            k1 += W1;
        }
        uint64_t hi0, lo0, hi1, lo1;
        mulhilo64(M0, c0, &hi0, &lo0);
        mulhilo64(M1, c2, &hi1, &lo1);
        const uint64_t n0 = hi1 ^ c1 ^ k0;
        const uint64_t n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
    }
    out[0] = c0;
    out[1] = c1;
    out[2] = c2;
    out[3] = c3;
}

// Eight consecutive float32 uniforms [0,1) of block `b` of the (seed, trial) stream.
WINO_HD void philox_block_floats(uint64_t seed, uint64_t trial, uint64_t b, float out[8]) {
    uint64_t ctr[4] = {b + 1, 0, 0, 0};
    if (ctr[0] == 0) ctr[1] = 1;  // carry (unreachable for realistic streams)
    uint64_t w[4];
    philox4x64_10(ctr, seed, trial, w);
    for (int i = 0; i < 4; ++i) {
        const uint32_t lo = (uint32_t)(w[i] & 0xffffffffu);
        const uint32_t hi = (uint32_t)(w[i] >> 32);
        out[2 * i] = (float)(lo >> 8) * (1.0f / 16777216.0f);
        out[2 * i + 1] = (float)(hi >> 8) * (1.0f / 16777216.0f);
    }
}

}  // namespace wino
