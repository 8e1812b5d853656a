// hy_arith.cuh -- 64-bit modular arithmetic on the integer pipes (sm_100a).
//
// All moduli are < 2^62.  Shoup multiplication by a precomputed constant w
// (w' = floor(w * 2^64 / q)) is the workhorse of the NTT and of every
// basis-conversion constant; products of two variables (key-switch inner
// product, PMult) are accumulated in 128 bits and reduced once.
#pragma once
#include <stdint.h>

#include "hy_internal.h"

namespace hy {

__device__ __forceinline__ uint64_t csub(uint64_t x, uint64_t q) { return x >= q ? x - q : x; }

// x * w mod q, result in [0, 2q)  (Shoup)
__device__ __forceinline__ uint64_t shoup_lazy(uint64_t x, uint64_t w, uint64_t wsh, uint64_t q) {
  uint64_t qh = __umul64hi(x, wsh);
  return x * w - qh * q;
}
__device__ __forceinline__ uint64_t shoup(uint64_t x, uint64_t w, uint64_t wsh, uint64_t q) {
  return csub(shoup_lazy(x, w, wsh, q), q);
}

__device__ __forceinline__ uint64_t add_mod(uint64_t a, uint64_t b, uint64_t q) { return csub(a + b, q); }
__device__ __forceinline__ uint64_t sub_mod(uint64_t a, uint64_t b, uint64_t q) { return a >= b ? a - b : a + q - b; }

// 128-bit accumulator
struct U128 {
  uint64_t lo, hi;
};
__device__ __forceinline__ void mac(U128& acc, uint64_t a, uint64_t b) {
  uint64_t lo = a * b, hi = __umul64hi(a, b);
  acc.lo += lo;
  acc.hi += hi + (acc.lo < lo);
}

// (hi*2^64 + lo) mod q for hi < 2^64, using r64 = 2^64 mod q (Shoup) and Barrett mu = floor(2^64/q).
__device__ __forceinline__ uint64_t reduce128(U128 x, const PrimeConst& p) {
  uint64_t a = shoup_lazy(x.hi, p.r64, p.r64_sh, p.q);  // [0, 2q)
  uint64_t b = x.lo - __umul64hi(x.lo, p.mu) * p.q;      // [0, 2q)
  uint64_t s = a + b;                                    // [0, 4q) < 2^64
  s = csub(s, p.two_q);
  return csub(s, p.q);
}

// Barrett reduction of a 64-bit word
__device__ __forceinline__ uint64_t reduce64(uint64_t x, const PrimeConst& p) {
  uint64_t b = x - __umul64hi(x, p.mu) * p.q;
  return csub(b, p.q);
}

__device__ __forceinline__ uint64_t mul_mod(uint64_t a, uint64_t b, const PrimeConst& p) {
  U128 t{a * b, __umul64hi(a, b)};
  return reduce128(t, p);
}

__device__ __forceinline__ uint32_t bitrev32(uint32_t x, int bits) { return __brev(x) >> (32 - bits); }

}  // namespace hy
