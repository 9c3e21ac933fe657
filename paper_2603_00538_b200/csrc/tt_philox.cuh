// Philox4x32-10 counter-based generator (Salmon, Moraes, Dror, Shaw, SC'11).
// counter = (sample j, element lo32, element hi32, 0), key = (seed lo32, seed hi32);
// uniforms xi_c = (u_c + 0.5) * 2^-32 in (0, 1).  Host KAT: tests/test_oracle.py.
#pragma once
#include <stdint.h>

namespace tt {

__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) { k0 += W0; k1 += W1; }
        uint32_t hi0 = __umulhi(M0, c[0]), lo0 = M0 * c[0];
        uint32_t hi1 = __umulhi(M1, c[2]), lo1 = M1 * c[2];
        uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
    }
}

__device__ __forceinline__ void philox_uniforms(uint64_t seed, uint64_t elem, uint64_t sample,
                                                double* xi) {
    uint32_t c[4] = {(uint32_t)sample, (uint32_t)elem, (uint32_t)(elem >> 32), 0u};
    philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
#pragma unroll
    for (int i = 0; i < 3; ++i) xi[i] = ((double)c[i] + 0.5) * 2.3283064365386963e-10;
}

}  // namespace tt
