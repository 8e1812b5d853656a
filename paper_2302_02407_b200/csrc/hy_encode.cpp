// hy_encode.cpp -- CKKS encoding (client side, untimed: P:1030-1031).
//
// DESIGN R-ENCODE: for real slots z_0..z_{n-1} (slot j <-> zeta^{5^j},
// zeta = exp(i pi / N)), the plaintext coefficients are
//   m = round_half_away( scale * tau^{-1}(z) ),
// with |frac - 1/2| < 2^-40 treated as an exact tie.  tau^{-1} is evaluated by
// the "special" inverse FFT over the rotation group <5> (n/2 log n butterflies)
// in double-double arithmetic (~104-bit significand), so the computed value is
// within ~2^-55 of the exact one and the rounding equals the rounding of the
// exact value (the oracle computes the same value by a plain 2N-point DFT in
// binary128; the two share no code).
#include <quadmath.h>

#include <cmath>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include "../../include/hyphen.h"

namespace {

struct DD {
  double hi, lo;
};
inline DD two_sum(double a, double b) {
  double s = a + b, bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
inline DD quick_two_sum(double a, double b) {
  double s = a + b;
  return {s, b - (s - a)};
}
inline DD dd_add(DD a, DD b) {
  DD s = two_sum(a.hi, b.hi), t = two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = quick_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return quick_two_sum(s.hi, s.lo);
}
inline DD dd_neg(DD a) { return {-a.hi, -a.lo}; }
inline DD dd_mul(DD a, DD b) {
  double p = a.hi * b.hi;
  double e = std::fma(a.hi, b.hi, -p);
  e += a.hi * b.lo + a.lo * b.hi;
  return quick_two_sum(p, e);
}
struct CDD {
  DD re, im;
};
inline CDD c_add(CDD a, CDD b) { return {dd_add(a.re, b.re), dd_add(a.im, b.im)}; }
inline CDD c_sub(CDD a, CDD b) { return {dd_add(a.re, dd_neg(b.re)), dd_add(a.im, dd_neg(b.im))}; }
inline CDD c_mul(CDD a, CDD b) {
  return {dd_add(dd_mul(a.re, b.re), dd_neg(dd_mul(a.im, b.im))), dd_add(dd_mul(a.re, b.im), dd_mul(a.im, b.re))};
}

DD from_q(__float128 x) {
  double hi = (double)x;
  double lo = (double)(x - (__float128)hi);
  return {hi, lo};
}

// ksi^k = exp(2 pi i k / M), k in [0, M], and the rotation group 5^j mod M
struct Tables {
  std::vector<CDD> ksi;
  std::vector<uint64_t> rot;
};
std::mutex g_mu;
std::map<uint32_t, std::shared_ptr<Tables>> g_tables;

std::shared_ptr<Tables> tables(uint32_t log_n) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_tables.find(log_n);
  if (it != g_tables.end()) return it->second;
  auto t = std::make_shared<Tables>();
  const uint64_t N = 1ull << log_n, M = 2 * N, n = N / 2;
  t->ksi.resize(M + 1);
  for (uint64_t k = 0; k <= M; ++k) {
    const __float128 pi = acosq((__float128)-1);
    __float128 a = 2 * pi * (__float128)k / (__float128)M;
    t->ksi[k] = {from_q(cosq(a)), from_q(sinq(a))};
  }
  t->rot.resize(n);
  uint64_t g = 1;
  for (uint64_t j = 0; j < n; ++j) {
    t->rot[j] = g;
    g = (g * 5) % M;
  }
  g_tables[log_n] = t;
  return t;
}

}  // namespace

namespace hy {
// the encoder's tables for the device path (hy_encode_dev.cu): ksi^k, k in [0, 2N], as (re.hi, re.lo, im.hi,
// im.lo), and the rotation group 5^j mod 2N, j < N/2
void encode_tables(uint32_t log_n, std::vector<double>& ksi4, std::vector<uint32_t>& rot) {
  auto T = tables(log_n);
  ksi4.resize(4 * T->ksi.size());
  for (size_t k = 0; k < T->ksi.size(); ++k) {
    ksi4[4 * k] = T->ksi[k].re.hi;
    ksi4[4 * k + 1] = T->ksi[k].re.lo;
    ksi4[4 * k + 2] = T->ksi[k].im.hi;
    ksi4[4 * k + 3] = T->ksi[k].im.lo;
  }
  rot.assign(T->rot.begin(), T->rot.end());
}
}  // namespace hy

namespace {

int64_t round_dd(DD x) {
  double fl = std::floor(x.hi);
  DD r = dd_add({x.hi - fl, 0.0}, {x.lo, 0.0});
  double frac = r.hi + r.lo;
  if (frac < 0) {
    fl -= 1;
    frac += 1;
  } else if (frac >= 1) {
    fl += 1;
    frac -= 1;
  }
  const bool positive = x.hi > 0 || (x.hi == 0 && x.lo > 0);
  if (std::fabs(frac - 0.5) < 0x1p-40) return (int64_t)fl + (positive ? 1 : 0);
  return (int64_t)fl + (frac > 0.5 ? 1 : 0);
}

}  // namespace

extern "C" hy_status hy_encode_coeffs_complex(uint32_t log_n, const double* slots, const double* slots_im,
                                              uint32_t n_slots, uint64_t scale, int64_t* out) {
  if (!slots || !out || log_n < 2 || log_n > 17) return HY_E_ARG;
  const uint64_t N = 1ull << log_n, n = N / 2, M = 2 * N;
  if (n_slots > n) return HY_E_CAPACITY;
  auto T = tables(log_n);
  std::vector<CDD> v(n);
  for (uint64_t j = 0; j < n; ++j)
    v[j] = {{j < n_slots ? slots[j] : 0.0, 0.0}, {(j < n_slots && slots_im) ? slots_im[j] : 0.0, 0.0}};
  // special inverse FFT over the orbit of 5
  for (uint64_t len = n; len >= 2; len >>= 1) {
    const uint64_t lenh = len >> 1, lenq = len << 2, gap = M / lenq;
    for (uint64_t i = 0; i < n; i += len) {
      for (uint64_t j = 0; j < lenh; ++j) {
        const uint64_t idx = (lenq - (T->rot[j] % lenq)) * gap;
        CDD u = c_add(v[i + j], v[i + j + lenh]);
        CDD w = c_mul(c_sub(v[i + j], v[i + j + lenh]), T->ksi[idx]);
        v[i + j] = u;
        v[i + j + lenh] = w;
      }
    }
  }
  // bit reversal over n entries
  int bits = 0;
  while ((1ull << bits) < n) ++bits;
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t r = 0;
    for (int b = 0; b < bits; ++b) r |= ((i >> b) & 1ull) << (bits - 1 - b);
    if (r > i) std::swap(v[i], v[r]);
  }
  const double sh = (double)scale;
  const DD sc = {sh, (double)(int64_t)(scale - (uint64_t)sh)};
  const DD inv_n = {1.0 / (double)n, 0.0};
  for (uint64_t i = 0; i < n; ++i) {
    DD re = dd_mul(dd_mul(v[i].re, inv_n), sc);
    DD im = dd_mul(dd_mul(v[i].im, inv_n), sc);
    if (std::fabs(re.hi) >= 0x1p62 || std::fabs(im.hi) >= 0x1p62) return HY_E_CAPACITY;
    out[i] = round_dd(re);
    out[i + n] = round_dd(im);
  }
  return HY_OK;
}

extern "C" hy_status hy_encode_coeffs(uint32_t log_n, const double* slots, uint32_t n_slots, uint64_t scale,
                                      int64_t* out) {
  return hy_encode_coeffs_complex(log_n, slots, nullptr, n_slots, scale, out);
}

// CKKS decode (client side, untimed): the inverse of R-ENCODE.  The N real coefficients m_i
// form the complex vector v_i = (m_i + i m_{i+n}) / scale; the "special" forward FFT over <5> evaluates
// it at zeta^{5^j}, i.e. z_j = m(zeta^{5^j}) / scale (canonical embedding, slot j <-> zeta^{5^j}).
// Decode is a floating-point result (a tolerance, not bit-exactness, is its contract), so plain
// double arithmetic over the double-double tables' high parts is used.
extern "C" hy_status hy_decode_coeffs(uint32_t log_n, const double* coeffs, double scale, uint32_t n_slots,
                                      double* re, double* im) {
  if (!coeffs || !re || log_n < 2 || log_n > 17 || !(scale > 0)) return HY_E_ARG;
  const uint64_t N = 1ull << log_n, n = N / 2, M = 2 * N;
  if (n_slots > n) return HY_E_CAPACITY;
  auto T = tables(log_n);
  std::vector<double> vr(n), vi(n);
  const double inv = 1.0 / scale;
  for (uint64_t i = 0; i < n; ++i) {
    vr[i] = coeffs[i] * inv;
    vi[i] = coeffs[i + n] * inv;
  }
  int bits = 0;
  while ((1ull << bits) < n) ++bits;
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t r = 0;
    for (int b = 0; b < bits; ++b) r |= ((i >> b) & 1ull) << (bits - 1 - b);
    if (r > i) {
      std::swap(vr[i], vr[r]);
      std::swap(vi[i], vi[r]);
    }
  }
  for (uint64_t len = 2; len <= n; len <<= 1) {
    const uint64_t lenh = len >> 1, lenq = len << 2, gap = M / lenq;
    for (uint64_t i = 0; i < n; i += len) {
      for (uint64_t j = 0; j < lenh; ++j) {
        const CDD& w = T->ksi[(T->rot[j] % lenq) * gap];
        const double wr = w.re.hi, wi = w.im.hi;
        const double ar = vr[i + j + lenh], ai = vi[i + j + lenh];
        const double br = ar * wr - ai * wi, bi = ar * wi + ai * wr;
        const double ur = vr[i + j], ui = vi[i + j];
        vr[i + j] = ur + br;
        vi[i + j] = ui + bi;
        vr[i + j + lenh] = ur - br;
        vi[i + j + lenh] = ui - bi;
      }
    }
  }
  for (uint32_t j = 0; j < n_slots; ++j) {
    re[j] = vr[j];
    if (im) im[j] = vi[j];
  }
  return HY_OK;
}

namespace hy {
// Centred CRT of the n coefficient-domain limbs limbs[u][N] (moduli mods[0..n)) to doubles: the unique
// representative of x mod Q in (-Q/2, Q/2], found by Garner's mixed-radix algorithm with centred digits
// a_k in [-(q_k-1)/2, (q_k-1)/2] (the symmetric digit set covers exactly Q consecutive integers around 0),
// then evaluated in binary128 by Horner from the top digit and rounded to double.
void crt_centered_to_double(const uint64_t* limbs, uint32_t n, uint64_t N, const uint64_t* mods, double* out) {
  using u128 = unsigned __int128;
  // Mmod[k][j] = (q_0 ... q_{j-1}) mod q_k for j < k; inv[k] = (q_0 ... q_{k-1})^{-1} mod q_k
  std::vector<uint64_t> Mmod((size_t)n * n, 0), inv(n, 1);
  auto powmod = [](uint64_t b, uint64_t e, uint64_t q) {
    uint64_t r = 1;
    for (; e; e >>= 1, b = (uint64_t)((u128)b * b % q))
      if (e & 1) r = (uint64_t)((u128)r * b % q);
    return r;
  };
  for (uint32_t k = 0; k < n; ++k) {
    uint64_t m = 1 % mods[k];
    for (uint32_t j = 0; j < k; ++j) {
      Mmod[(size_t)k * n + j] = m;
      m = (uint64_t)((u128)m * (mods[j] % mods[k]) % mods[k]);
    }
    inv[k] = powmod(m, mods[k] - 2, mods[k]);
  }
  std::vector<int64_t> a(n);
  for (uint64_t x = 0; x < N; ++x) {
    for (uint32_t k = 0; k < n; ++k) {
      const uint64_t q = mods[k];
      u128 s = 0;
      for (uint32_t j = 0; j < k; ++j) {
        const uint64_t aj = a[j] < 0 ? q - (uint64_t)(-a[j]) % q : (uint64_t)a[j] % q;
        s = (s + (u128)aj * Mmod[(size_t)k * n + j]) % q;
      }
      const uint64_t xk = limbs[(size_t)k * N + x] % q;
      const uint64_t d = (uint64_t)(((u128)(xk + q - (uint64_t)s) % q) * inv[k] % q);
      a[k] = d > (q - 1) / 2 ? (int64_t)d - (int64_t)q : (int64_t)d;
    }
    __float128 v = 0;
    for (int k = (int)n - 1; k >= 0; --k) v = v * (__float128)mods[k] + (__float128)a[k];
    out[x] = (double)v;
  }
}
}  // namespace hy
