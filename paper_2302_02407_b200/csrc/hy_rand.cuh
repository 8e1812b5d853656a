// hy_rand.cuh -- Philox4x32-10 (Salmon et al., SC'11) and the samplers of
// DESIGN R-PRNG, usable on host and device (product implementation).
//   counter = (i, limb, obj_lo32, domain << 24 | obj_hi24), key = (seed_lo, seed_hi)
//   uniform mod q  : 128-bit word (w3:w2:w1:w0) mod q
//   CBD(21)        : popcount(w0 & 0x1FFFFF) - popcount(w1 & 0x1FFFFF), limb = 0
//   HWT secret     : partial Fisher-Yates, draw t -> j = t + (w1:w0) mod (N - t), sign = w2 & 1
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define HY_HD __host__ __device__ __forceinline__
#else
#define HY_HD inline
#endif

namespace hy {

enum : uint32_t { kDomSecret = 1, kDomEvkA = 2, kDomEvkE = 3, kDomEncA = 4, kDomEncE = 5 };

struct Philox4 {
  uint32_t v[4];
};

HY_HD uint32_t mulhi32(uint32_t a, uint32_t b) { return (uint32_t)(((uint64_t)a * b) >> 32); }

HY_HD Philox4 philox10(uint64_t seed, uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3) {
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
  for (int round = 0; round < 10; ++round) {
    uint32_t hi0 = mulhi32(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    uint32_t hi1 = mulhi32(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return Philox4{{c0, c1, c2, c3}};
}

HY_HD Philox4 draw(uint64_t seed, uint32_t dom, uint64_t obj, uint32_t limb, uint32_t i) {
  return philox10(seed, i, limb, (uint32_t)obj, (dom << 24) | (uint32_t)((obj >> 32) & 0xFFFFFFu));
}

// (w3:w2:w1:w0) mod q for q < 2^62 (Horner over 32-bit digits; keygen/encryption only)
HY_HD uint64_t uniform_mod(const Philox4& w, uint64_t q) {
  uint64_t r = 0;
#pragma unroll
  for (int d = 3; d >= 0; --d) {
    unsigned __int128 x = ((unsigned __int128)r << 32) | w.v[d];
    r = (uint64_t)(x % q);
  }
  return r;
}

HY_HD int32_t cbd21(const Philox4& w) {
#ifdef __CUDA_ARCH__
  return (int32_t)__popc(w.v[0] & 0x1FFFFFu) - (int32_t)__popc(w.v[1] & 0x1FFFFFu);
#else
  return (int32_t)__builtin_popcount(w.v[0] & 0x1FFFFFu) - (int32_t)__builtin_popcount(w.v[1] & 0x1FFFFFu);
#endif
}

}  // namespace hy
