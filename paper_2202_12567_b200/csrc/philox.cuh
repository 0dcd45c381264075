// philox.cuh — Philox4x32-10 counter-based generator (Salmon et al., SC'11) for the CUDA path.
// Counter = (a, b, slice, tag), key = 64-bit seed (R7).  Random integers in [0, n)
// are (u * n) >> 32 and uniform reals (u >> 8) * 2^-24 (exact in fp32 and fp64).
#pragma once
#include <stdint.h>

namespace lmc {

__device__ __forceinline__ uint4 philox4(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint64_t seed)
{
    uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
        uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
        uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return make_uint4(c0, c1, c2, c3);
}

__device__ __forceinline__ uint32_t randint_u(uint32_t u, uint32_t n) { return (uint32_t)(((uint64_t)u * n) >> 32); }
__device__ __forceinline__ float unif_f(uint32_t u) { return (float)(u >> 8) * (1.0f / 16777216.0f); }

}  // namespace lmc
