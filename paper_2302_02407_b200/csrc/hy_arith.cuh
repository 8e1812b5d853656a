// hy_arith.cuh -- modular arithmetic of the product path (sm_100a).
//
// Every prime is < 2^48 (DESIGN R-PRIMES), so residues are exact doubles and the hot
// kernels (NTT, BConv, key-switch inner product, ModDown, PMult) run on B200's full-rate
// FP64 pipe with the six-operation fmulmod below (DESIGN R-FP64).  The 64-bit integer
// helpers (Shoup / Barrett / 128-bit accumulation) serve the cold paths: key generation,
// encryption, decryption and the 48-bit wire-format conversions.
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

// NTT-domain index permutation of the automorphism kappa_k: out[p] = in[perm(p)],
// 2 br(perm(p)) + 1 = (2 br(p) + 1) k mod 2N.  Used for ciphertext rotations and for PRot of
// plaintexts fused into their consumers as a gather.
__device__ __forceinline__ uint32_t aut_index(uint32_t p, uint64_t k, int logN) {
  uint32_t e = 2 * bitrev32(p, logN) + 1;
  // only the low logN + 1 bits of e k are needed, so a 32-bit product suffices (k < 2N <= 2^17)
  uint32_t e2 = (e * (uint32_t)k) & ((2u << logN) - 1);
  return bitrev32((e2 - 1) >> 1, logN);
}

// ---------------------------------------------------------------- FP64-pipe modular arithmetic
// Residues of primes q < 2^48 are exact doubles.  B200 issues FP64 FMA at full
// rate (64/clk/SM, measured 18.2 TFMA/s), so the NTT butterflies run on the FP64
// pipe instead of the half-rate 64-bit IMAD chains (tools/microbench/fp_modmul.cu:
// 1.66 vs 0.97 T modmul/s with full reduction).
constexpr double kTwo52 = 4503599627370496.0;   // 2^52
constexpr double kMagic = 6755399441055744.0;   // 1.5 * 2^52: (x + M) - M = rint(x) for |x| < 2^51

__device__ __forceinline__ double u2d(uint64_t v) {  // v < 2^52
  return __longlong_as_double((long long)(v | 0x4330000000000000ull)) - kTwo52;
}
__device__ __forceinline__ uint64_t d2u(double d) {  // d integer in [0, 2^52)
  return (uint64_t)__double_as_longlong(d + kTwo52) & 0xFFFFFFFFFFFFFull;
}
// b*w mod q as an integer-valued double r, for 0 <= w < q < 2^48 and |b * w / q| < 2^51 (the magic-rounding
// range; |b| < 2^51 suffices): h + l = b*w exactly (FMA error term), c = rint(fl(h * qinv)), r = (h - c q) + l,
// every step exact, and |r| <= q/2 + |b| q 2^-52 (c is off round(h/q) by at most |h/q| 2^-53 and |l| <= |h| 2^-53).
// For the 48-bit primes that is |r| <= (1/2 + beta/16) q for |b| <= beta q; DESIGN R-FP64 derives from it the
// growth bound of the unreduced forward passes (largest operand 6.62 q < 2^51, tests/test_fp64_bound_cpu.py).
__device__ __forceinline__ double fmulmod(double b, double w, double q, double qinv) {
  const double h = b * w;
  const double l = fma(b, w, -h);
  const double c = fma(h, qinv, kMagic) - kMagic;
  return fma(-c, q, h) + l;
}
// v - rint(v/q) q, in [-q/2 - 1, q/2 + 1] for |v| < 2^51
__device__ __forceinline__ double fred(double v, double q, double qinv) {
  const double c = fma(v, qinv, kMagic) - kMagic;
  return fma(-c, q, v);
}
// canonical residue in [0, q) for |v| < 2^51
__device__ __forceinline__ double fcanon(double v, double q, double qinv) {
  double r = fred(v, q, qinv);
  r = r < 0.0 ? r + q : r;
  return r >= q ? r - q : r;
}

// ---- packed evaluation keys (DESIGN "Evk layout"): every residue is < 2^48 (R-PRIMES), so a key word takes
// 6 bytes: word x of a limb at bytes [6x, 6x+6) little-endian, a limb is 6N bytes = 3N/4 uint64 (N >= 4),
// a 256-word row 1536 bytes.  Limb li of a key [dnum][2][n_q+n_p] starts at evk + li * 3N/4.
constexpr uint64_t kM48 = (1ull << 48) - 1;
__host__ __device__ __forceinline__ size_t evk_limb_words(size_t N) { return N / 4 * 3; }
__device__ __forceinline__ const uint64_t* evk_limb(const uint64_t* evk, size_t li, size_t N) {
  return evk + li * evk_limb_words(N);
}
// word x of a packed limb (streaming loads; the second only when the word straddles two uint64)
__device__ __forceinline__ uint64_t evk_word(const uint64_t* limb, uint32_t x) {
  const uint32_t o = 6 * x, a = o >> 3, sh = (o & 7) * 8;
  uint64_t w = __ldcs(limb + a) >> sh;
  if (sh > 16) w |= __ldcs(limb + a + 1) << (64 - sh);
  return w & kM48;
}
// words 4m..4m+3 from the three uint64 (24 bytes) that hold them
__device__ __forceinline__ void evk_unpack4(uint64_t p0, uint64_t p1, uint64_t p2, uint64_t& w0, uint64_t& w1,
                                            uint64_t& w2, uint64_t& w3) {
  w0 = p0 & kM48;
  w1 = (p0 >> 48) | ((p1 & 0xFFFFFFFFull) << 16);
  w2 = (p1 >> 32) | ((p2 & 0xFFFFull) << 32);
  w3 = p2 >> 16;
}
// store word x (three 2-byte stores: threads of neighbouring words never share a store address)
__device__ __forceinline__ void evk_store(uint64_t* limb, uint32_t x, uint64_t w) {
  uint16_t* p = reinterpret_cast<uint16_t*>(reinterpret_cast<uint8_t*>(limb) + 6ull * x);
  p[0] = (uint16_t)w;
  p[1] = (uint16_t)(w >> 16);
  p[2] = (uint16_t)(w >> 32);
}

// bulk async copies (TMA bulk engine: cp.async.bulk global -> shared, completion on an mbarrier)
namespace tma {
__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(saddr(b)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_row(void* dst, const void* src, uint64_t* b, uint32_t bytes = 2048) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   saddr(dst)),
               "l"(src), "r"(bytes), "r"(saddr(b))
               : "memory");
}
__device__ __forceinline__ void proxy_fence() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
}  // namespace tma

}  // namespace hy
