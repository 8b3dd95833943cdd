// philox.cuh — Philox4x32-10 (Salmon et al., SC'11) for the device draw.
// Independent of oracle/philox.py; both are pinned to the Random123 known-answer vectors.
// Keying (R11): key = seed, counter = (step, request_id);
// u = ((x1 << 32 | x0) >> 11) * 2^-53 in [0, 1).
#pragma once
#include <cstdint>

namespace smp {

__host__ __device__ inline void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += W0;
      k1 += W1;
    }
    const uint64_t p0 = (uint64_t)M0 * c[0];
    const uint64_t p1 = (uint64_t)M1 * c[2];
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
  }
}

__host__ __device__ inline double philox_uniform(uint64_t seed, uint64_t request, uint64_t step) {
  uint32_t c[4] = {(uint32_t)step, (uint32_t)(step >> 32), (uint32_t)request,
                   (uint32_t)(request >> 32)};
  philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  const uint64_t x = ((uint64_t)c[1] << 32) | c[0];
  return (double)(x >> 11) * 0x1.0p-53;
}

}  // namespace smp
