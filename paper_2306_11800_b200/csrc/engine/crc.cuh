// CRC-32/IEEE (reflected, poly 0xEDB88320) combine algebra, host + device.
// crc32 (codec.cpp:275-288) is linear: reg(A||B) = shift(reg(A), |B|) ^ reg(B)
// with shift(v, n bytes) = v * x^(8n) mod P, and
// crc(M) = reg0(M) ^ shift(0xFFFFFFFF, |M|) ^ 0xFFFFFFFF, reg0 = zero-init register.
#pragma once

#include <stdint.h>

namespace dqtg {

__host__ __device__ inline uint32_t crc_multmodp(uint32_t a, uint32_t b) {
    uint32_t m = 1u << 31, p = 0;
    for (;;) {
        if (a & m) {
            p ^= b;
            if ((a & (m - 1)) == 0) break;
        }
        m >>= 1;
        b = (b & 1) ? (b >> 1) ^ 0xedb88320u : b >> 1;
    }
    return p;
}

// x^(2^k) mod P for k = 0..31 (x^1 = bit 30 in the reflected representation)
struct CrcX2N {
    uint32_t t[32];
};

inline CrcX2N crc_x2n_table() {
    CrcX2N x;
    uint32_t p = 1u << 30;
    x.t[0] = p;
    for (int k = 1; k < 32; ++k) x.t[k] = p = crc_multmodp(p, p);
    return x;
}

// x^(n * 2^k) mod P
__host__ __device__ inline uint32_t crc_x2nmodp(const uint32_t* t, uint64_t n, unsigned k) {
    uint32_t p = 1u << 31;
    while (n) {
        if (n & 1) p = crc_multmodp(t[k & 31], p);
        n >>= 1;
        k++;
    }
    return p;
}

// register after feeding n zero bytes
__host__ __device__ inline uint32_t crc_shift(const uint32_t* t, uint32_t v, uint64_t nbytes) {
    return nbytes ? crc_multmodp(crc_x2nmodp(t, nbytes, 3), v) : v;
}

}  // namespace dqtg
