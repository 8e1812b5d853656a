/*
 * ckks_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of the RNS-CKKS
 * operations on HyPHEN's homomorphic-convolution hot path (arXiv 2302.02407).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header,
 * table or constant generator with the CUDA product path
 * (paper_2302_02407_b200/csrc); the two meet only through seeded inputs.
 *
 * Arithmetic: every modular product is (unsigned __int128)a*b % q.  No
 * Montgomery/Shoup/Barrett, no lazy reduction, no fusion.  Every function
 * cites the passage it follows; "DESIGN R#" names a reading of a point the
 * paper leaves silent (DESIGN.md section "Readings").
 *
 *   P:n = /root/reference/PAPER.md line n.
 *
 * Paper anchors:
 *   ring Z[X]/(X^N+1), slots, plaintext/ciphertext ............ P:96-100
 *   AddCt/AddPt/MulPt/Rescale/levels ......................... P:102-112
 *   CRot rotates LEFT by r; PRot ............................. P:120-126
 *   N=2^16, h=192 ............................................ P:1028
 *   Set_hyp L+1=24, dnum=6; Ctxt 10MB / Ptxt 5MB / Evk 168MB .. P:1207-1208
 *   hybrid key switching with dnum (Han-Ki) .................. P:1232-1239
 *
 * Parity: pinned (tests/test_oracle_*.py): Philox (Random123 KAT), primes
 * (Miller-Rabin + root order), NTT (direct evaluation, schoolbook product),
 * encode (mpmath direct evaluation, encode(decode(m)) = m), keygen/enc/dec
 * (dec(enc(m)) - m = e exactly), automorphism (coefficient map = slot roll),
 * ModUp/ModDown (big-int CRT identities), key switch (decrypt identity within
 * the closed-form bound), rescale (exact big-int rounding).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <quadmath.h>

typedef unsigned __int128 u128;
typedef __int128 i128;

#define ORC_MAXP 64

/* ------------------------------------------------------------------ */
/* Plain modular arithmetic                                            */
/* ------------------------------------------------------------------ */
static uint64_t mulmod(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)(((u128)a * b) % q); }
static uint64_t addmod(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)(((u128)a + b) % q); }
static uint64_t submod(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)(((u128)a + q - b) % q); }
static uint64_t powmod(uint64_t a, uint64_t e, uint64_t q) {
  uint64_t r = 1 % q;
  a %= q;
  while (e) { if (e & 1) r = mulmod(r, a, q); a = mulmod(a, a, q); e >>= 1; }
  return r;
}
static uint64_t invmod(uint64_t a, uint64_t q) { return powmod(a, q - 2, q); } /* q prime */
static uint64_t from_signed(int64_t v, uint64_t q) {
  i128 r = (i128)v % (i128)q;
  if (r < 0) r += q;
  return (uint64_t)r;
}

/* Deterministic Miller-Rabin for n < 2^64 (bases 2..37). */
int orc_is_prime(uint64_t n) {
  static const uint64_t B[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (n < 2) return 0;
  for (int i = 0; i < 12; ++i) { if (n == B[i]) return 1; if (n % B[i] == 0) return 0; }
  uint64_t d = n - 1; int s = 0;
  while ((d & 1) == 0) { d >>= 1; ++s; }
  for (int i = 0; i < 12; ++i) {
    uint64_t x = powmod(B[i], d, n);
    if (x == 1 || x == n - 1) continue;
    int comp = 1;
    for (int r = 1; r < s; ++r) { x = mulmod(x, x, n); if (x == n - 1) { comp = 0; break; } }
    if (comp) return 0;
  }
  return 1;
}

/* ------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon et al., SC'11; Random123 reference)           */
/* ------------------------------------------------------------------ */
void orc_philox4x32_10(const uint32_t key_in[2], const uint32_t ctr_in[4], uint32_t out[4]) {
  uint32_t k0 = key_in[0], k1 = key_in[1];
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* DESIGN R-PRNG: counter = (i, limb, obj_lo, domain<<24 | obj_hi24), key = seed. */
enum { DOM_SK = 1, DOM_EVK_A = 2, DOM_EVK_E = 3, DOM_ENC_A = 4, DOM_ENC_E = 5 };

static void draw(uint64_t seed, uint32_t dom, uint64_t obj, uint32_t limb, uint32_t i, uint32_t w[4]) {
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t ctr[4] = {i, limb, (uint32_t)obj, (dom << 24) | (uint32_t)((obj >> 32) & 0xFFFFFFu)};
  orc_philox4x32_10(key, ctr, w);
}
/* uniform mod q: the 128-bit word w3:w2:w1:w0 reduced mod q. */
static uint64_t draw_uniform(uint64_t seed, uint32_t dom, uint64_t obj, uint32_t limb, uint32_t i, uint64_t q) {
  uint32_t w[4];
  draw(seed, dom, obj, limb, i, w);
  u128 x = ((u128)w[3] << 96) | ((u128)w[2] << 64) | ((u128)w[1] << 32) | (u128)w[0];
  return (uint64_t)(x % q);
}
/* centred binomial, k = 21: popcount(w0 & (2^21-1)) - popcount(w1 & (2^21-1)). */
static int32_t draw_cbd(uint64_t seed, uint32_t dom, uint64_t obj, uint32_t i) {
  uint32_t w[4];
  draw(seed, dom, obj, 0, i, w);
  return (int32_t)__builtin_popcount(w[0] & 0x1FFFFFu) - (int32_t)__builtin_popcount(w[1] & 0x1FFFFFu);
}

/* ------------------------------------------------------------------ */
/* Context: primes, roots, NTT tables                                   */
/* ------------------------------------------------------------------ */
typedef struct {
  int logN, N, nq, np, dnum, alpha;
  uint64_t mod[ORC_MAXP];      /* chain: q_0..q_{nq-1}, p_0..p_{np-1} */
  uint64_t psi[ORC_MAXP];
  uint64_t *psi_rev[ORC_MAXP]; /* psi^{br(k)} */
  uint64_t *psi_inv_rev[ORC_MAXP];
} orc_ctx;

static uint32_t bitrev(uint32_t x, int bits) {
  uint32_t r = 0;
  for (int i = 0; i < bits; ++i) { r = (r << 1) | (x & 1); x >>= 1; }
  return r;
}

/* DESIGN R-PRIMES: in chain order, each prime is the largest unused prime
 * below 2^bits with p == 1 (mod 2N). */
static uint64_t next_prime_below(int bits, uint64_t twoN, const uint64_t* used, int nused) {
  uint64_t top = (bits == 64) ? ~(uint64_t)0 : (((uint64_t)1 << bits) - 1);
  uint64_t x = ((top - 1) / twoN) * twoN + 1;
  for (; x > twoN; x -= twoN) {
    int dup = 0;
    for (int i = 0; i < nused; ++i) if (used[i] == x) dup = 1;
    if (!dup && orc_is_prime(x)) return x;
  }
  return 0;
}

/* DESIGN R-NTT: psi = the smallest primitive 2N-th root of unity mod q. */
static uint64_t min_primitive_2n_root(uint64_t q, uint64_t twoN) {
  uint64_t N = twoN / 2;
  for (uint64_t g = 2; g < q; ++g) {
    uint64_t c = powmod(g, (q - 1) / twoN, q);
    if (powmod(c, N, q) != q - 1) continue;
    uint64_t best = c, x = c, c2 = mulmod(c, c, q);
    for (uint64_t e = 1; e < twoN; e += 2) { if (x < best) best = x; x = mulmod(x, c2, q); }
    return best;
  }
  return 0;
}

orc_ctx* orc_ctx_new(int logN, int nq, const int* qbits, int np, const int* pbits, int dnum) {
  if (nq + np > ORC_MAXP || logN < 2 || logN > 17 || dnum < 1) return NULL;
  orc_ctx* c = (orc_ctx*)calloc(1, sizeof(orc_ctx));
  c->logN = logN; c->N = 1 << logN; c->nq = nq; c->np = np; c->dnum = dnum;
  c->alpha = (nq + dnum - 1) / dnum;
  uint64_t twoN = 2 * (uint64_t)c->N;
  for (int i = 0; i < nq + np; ++i) {
    int b = i < nq ? qbits[i] : pbits[i - nq];
    c->mod[i] = next_prime_below(b, twoN, c->mod, i);
    if (!c->mod[i]) { free(c); return NULL; }
  }
  for (int i = 0; i < nq + np; ++i) {
    uint64_t q = c->mod[i];
    c->psi[i] = min_primitive_2n_root(q, twoN);
    uint64_t pinv = invmod(c->psi[i], q);
    c->psi_rev[i] = (uint64_t*)malloc(sizeof(uint64_t) * c->N);
    c->psi_inv_rev[i] = (uint64_t*)malloc(sizeof(uint64_t) * c->N);
    uint64_t* pw = (uint64_t*)malloc(sizeof(uint64_t) * c->N);
    uint64_t* pwi = (uint64_t*)malloc(sizeof(uint64_t) * c->N);
    pw[0] = 1; pwi[0] = 1;
    for (int k = 1; k < c->N; ++k) { pw[k] = mulmod(pw[k - 1], c->psi[i], q); pwi[k] = mulmod(pwi[k - 1], pinv, q); }
    for (int k = 0; k < c->N; ++k) {
      c->psi_rev[i][k] = pw[bitrev(k, logN)];
      c->psi_inv_rev[i][k] = pwi[bitrev(k, logN)];
    }
    free(pw); free(pwi);
  }
  return c;
}

void orc_ctx_free(orc_ctx* c) {
  if (!c) return;
  for (int i = 0; i < c->nq + c->np; ++i) { free(c->psi_rev[i]); free(c->psi_inv_rev[i]); }
  free(c);
}
void orc_ctx_moduli(const orc_ctx* c, uint64_t* out) { for (int i = 0; i < c->nq + c->np; ++i) out[i] = c->mod[i]; }
void orc_ctx_psi(const orc_ctx* c, uint64_t* out) { for (int i = 0; i < c->nq + c->np; ++i) out[i] = c->psi[i]; }
int orc_ctx_alpha(const orc_ctx* c) { return c->alpha; }

/* ------------------------------------------------------------------ */
/* NTT: textbook merged negacyclic Cooley-Tukey / Gentleman-Sande       */
/* DESIGN R-NTT: output index k holds a(psi^(2*br(k)+1)).               */
/* ------------------------------------------------------------------ */
void orc_ntt(const orc_ctx* c, int chain_idx, uint64_t* a) {
  const uint64_t q = c->mod[chain_idx];
  const uint64_t* W = c->psi_rev[chain_idx];
  int N = c->N, t = N;
  for (int m = 1; m < N; m *= 2) {
    t /= 2;
    for (int i = 0; i < m; ++i) {
      int j1 = 2 * i * t;
      uint64_t S = W[m + i];
      for (int j = j1; j < j1 + t; ++j) {
        uint64_t U = a[j], V = mulmod(a[j + t], S, q);
        a[j] = addmod(U, V, q);
        a[j + t] = submod(U, V, q);
      }
    }
  }
}

void orc_intt(const orc_ctx* c, int chain_idx, uint64_t* a) {
  const uint64_t q = c->mod[chain_idx];
  const uint64_t* W = c->psi_inv_rev[chain_idx];
  int N = c->N, t = 1;
  for (int m = N; m > 1; m /= 2) {
    int j1 = 0, h = m / 2;
    for (int i = 0; i < h; ++i) {
      uint64_t S = W[h + i];
      for (int j = j1; j < j1 + t; ++j) {
        uint64_t U = a[j], V = a[j + t];
        a[j] = addmod(U, V, q);
        a[j + t] = mulmod(submod(U, V, q), S, q);
      }
      j1 += 2 * t;
    }
    t *= 2;
  }
  uint64_t ninv = invmod((uint64_t)N % q, q);
  for (int j = 0; j < N; ++j) a[j] = mulmod(a[j], ninv, q);
}

/* Batched helpers over a contiguous [n][N] array whose limb u uses chain[u]. */
static void ntt_limbs(const orc_ctx* c, uint64_t* a, const int* chain, int n) {
#pragma omp parallel for schedule(dynamic)
  for (int u = 0; u < n; ++u) orc_ntt(c, chain[u], a + (size_t)u * c->N);
}
static void intt_limbs(const orc_ctx* c, uint64_t* a, const int* chain, int n) {
#pragma omp parallel for schedule(dynamic)
  for (int u = 0; u < n; ++u) orc_intt(c, chain[u], a + (size_t)u * c->N);
}

/* Chain index of extended-basis limb u at level l: q_0..q_l then p_0..p_{K-1}. */
static int ext_chain(const orc_ctx* c, int level, int u) { return u <= level ? u : c->nq + (u - level - 1); }

/* ------------------------------------------------------------------ */
/* Automorphism kappa_k: a(X) -> a(X^k), k odd             */
/* Coefficient domain: coefficient i moves to i*k mod 2N, negated when   */
/* that index is >= N (X^N = -1).                                        */
/* ------------------------------------------------------------------ */
void orc_automorph_coeff(const orc_ctx* c, int chain_idx, uint64_t k, const uint64_t* in, uint64_t* out) {
  const uint64_t q = c->mod[chain_idx];
  const uint64_t N = c->N, twoN = 2 * N;
  for (uint64_t i = 0; i < N; ++i) {
    uint64_t e = (i * k) % twoN;
    if (e < N) out[e] = in[i];
    else out[e - N] = in[i] == 0 ? 0 : q - in[i];
  }
}

/* NTT-domain automorphism done the obvious way: iNTT, coefficient map, NTT. */
static void automorph_ntt_limbs(const orc_ctx* c, const uint64_t* in, uint64_t* out, const int* chain, int n, uint64_t k) {
#pragma omp parallel for schedule(dynamic)
  for (int u = 0; u < n; ++u) {
    uint64_t* tmp = (uint64_t*)malloc(sizeof(uint64_t) * c->N);
    memcpy(tmp, in + (size_t)u * c->N, sizeof(uint64_t) * c->N);
    orc_intt(c, chain[u], tmp);
    orc_automorph_coeff(c, chain[u], k, tmp, out + (size_t)u * c->N);
    orc_ntt(c, chain[u], out + (size_t)u * c->N);
    free(tmp);
  }
}

/* Galois element of a left rotation by r slots: 5^r mod 2N, r taken mod N/2. */
uint64_t orc_galois_elt(const orc_ctx* c, int64_t r) {
  int64_t n = c->N / 2;
  int64_t rr = ((r % n) + n) % n;
  return powmod(5, (uint64_t)rr, 2 * (uint64_t)c->N);
}

/* ------------------------------------------------------------------ */
/* Secret key, errors (ternary, Hamming weight h)               */
/* ------------------------------------------------------------------ */
/* DESIGN R-SK: partial Fisher-Yates over Philox draws. */
void orc_sample_secret(const orc_ctx* c, uint64_t seed, int h, int8_t* s) {
  int N = c->N;
  uint32_t* idx = (uint32_t*)malloc(sizeof(uint32_t) * N);
  for (int i = 0; i < N; ++i) { idx[i] = i; s[i] = 0; }
  for (int t = 0; t < h; ++t) {
    uint32_t w[4];
    draw(seed, DOM_SK, 0, 0, (uint32_t)t, w);
    uint64_t u = ((uint64_t)w[1] << 32) | w[0];
    uint32_t j = (uint32_t)(t + u % (uint64_t)(N - t));
    uint32_t tmp = idx[t]; idx[t] = idx[j]; idx[j] = tmp;
    s[idx[t]] = (w[2] & 1) ? -1 : 1;
  }
  free(idx);
}

void orc_sample_cbd(uint64_t seed, uint32_t dom, uint64_t obj, int N, int32_t* e) {
  for (int i = 0; i < N; ++i) e[i] = draw_cbd(seed, dom, obj, (uint32_t)i);
}

/* small signed polynomial -> NTT-domain limb on chain index t */
static void small_to_ntt_i32(const orc_ctx* c, const int32_t* v, int t, uint64_t* out) {
  for (int i = 0; i < c->N; ++i) out[i] = from_signed(v[i], c->mod[t]);
  orc_ntt(c, t, out);
}
static void small_to_ntt_i8(const orc_ctx* c, const int8_t* v, int t, uint64_t* out) {
  for (int i = 0; i < c->N; ++i) out[i] = from_signed(v[i], c->mod[t]);
  orc_ntt(c, t, out);
}

/* ------------------------------------------------------------------ */
/* Rotation key for Galois element k (hybrid KS; DESIGN R-EVK)  */
/* evk layout [dnum][2][nq+np][N] NTT domain; [.][0]=b, [.][1]=a;       */
/* b_j = -a_j*s + e_j + g_j*kappa_k(s), g_j = P on q-limbs of digit j,  */
/* 0 on other q-limbs and on every p-limb.                              */
/* ------------------------------------------------------------------ */
void orc_keygen_rot(const orc_ctx* c, uint64_t sk_seed, int h, uint64_t ek_seed, uint64_t k, uint64_t* evk) {
  const int N = c->N, L1 = c->nq + c->np;
  int8_t* s = (int8_t*)malloc(N);
  orc_sample_secret(c, sk_seed, h, s);
  /* kappa_k(s) in the coefficient domain over the integers */
  int8_t* sk = (int8_t*)calloc(N, 1);
  for (uint64_t i = 0; i < (uint64_t)N; ++i) {
    uint64_t e = (i * k) % (2 * (uint64_t)N);
    if (e < (uint64_t)N) sk[e] = s[i]; else sk[e - N] = (int8_t)(-s[i]);
  }
#pragma omp parallel for schedule(dynamic)
  for (int jt = 0; jt < c->dnum * L1; ++jt) {
    int j = jt / L1, t = jt % L1;
    uint64_t q = c->mod[t];
    uint64_t obj = (k << 8) | (uint64_t)j;
    uint64_t* b = evk + ((size_t)(j * 2 + 0) * L1 + t) * N;
    uint64_t* a = evk + ((size_t)(j * 2 + 1) * L1 + t) * N;
    uint64_t* s_ntt = (uint64_t*)malloc(sizeof(uint64_t) * N);
    uint64_t* sk_ntt = (uint64_t*)malloc(sizeof(uint64_t) * N);
    uint64_t* e_ntt = (uint64_t*)malloc(sizeof(uint64_t) * N);
    int32_t* e = (int32_t*)malloc(sizeof(int32_t) * N);
    small_to_ntt_i8(c, s, t, s_ntt);
    small_to_ntt_i8(c, sk, t, sk_ntt);
    orc_sample_cbd(ek_seed, DOM_EVK_E, obj, N, e);
    small_to_ntt_i32(c, e, t, e_ntt);
    /* g_j mod chain prime t */
    uint64_t g = 0;
    if (t < c->nq && t >= j * c->alpha && t < (j + 1) * c->alpha) {
      g = 1;
      for (int kk = 0; kk < c->np; ++kk) g = mulmod(g, c->mod[c->nq + kk] % q, q);
    }
    for (int i = 0; i < N; ++i) {
      a[i] = draw_uniform(ek_seed, DOM_EVK_A, obj, (uint32_t)t, (uint32_t)i, q);
      uint64_t v = submod(e_ntt[i], mulmod(a[i], s_ntt[i], q), q);
      b[i] = addmod(v, mulmod(g, sk_ntt[i], q), q);
    }
    free(s_ntt); free(sk_ntt); free(e_ntt); free(e);
  }
  free(s); free(sk);
}

/* ------------------------------------------------------------------ */
/* Secret-key encryption / decryption (DESIGN R-ENC)              */
/* ct layout [2][level+1][N] NTT domain.                                */
/* ------------------------------------------------------------------ */
void orc_encrypt(const orc_ctx* c, uint64_t sk_seed, int h, uint64_t enc_seed, uint64_t ct_id,
                 const uint64_t* m, int level, uint64_t* ct) {
  const int N = c->N, n = level + 1;
  int8_t* s = (int8_t*)malloc(N);
  int32_t* e = (int32_t*)malloc(sizeof(int32_t) * N);
  orc_sample_secret(c, sk_seed, h, s);
  orc_sample_cbd(enc_seed, DOM_ENC_E, ct_id, N, e);
#pragma omp parallel for schedule(dynamic)
  for (int i = 0; i < n; ++i) {
    uint64_t q = c->mod[i];
    uint64_t* s_ntt = (uint64_t*)malloc(sizeof(uint64_t) * N);
    uint64_t* e_ntt = (uint64_t*)malloc(sizeof(uint64_t) * N);
    small_to_ntt_i8(c, s, i, s_ntt);
    small_to_ntt_i32(c, e, i, e_ntt);
    uint64_t* c0 = ct + (size_t)i * N;
    uint64_t* c1 = ct + ((size_t)n + i) * N;
    for (int x = 0; x < N; ++x) {
      c1[x] = draw_uniform(enc_seed, DOM_ENC_A, ct_id, (uint32_t)i, (uint32_t)x, q);
      c0[x] = addmod(submod(e_ntt[x], mulmod(c1[x], s_ntt[x], q), q), m[(size_t)i * N + x], q);
    }
    free(s_ntt); free(e_ntt);
  }
  free(s); free(e);
}

/* m = c0 + c1*s (NTT domain) */
void orc_decrypt(const orc_ctx* c, uint64_t sk_seed, int h, const uint64_t* ct, int level, uint64_t* m) {
  const int N = c->N, n = level + 1;
  int8_t* s = (int8_t*)malloc(N);
  orc_sample_secret(c, sk_seed, h, s);
#pragma omp parallel for schedule(dynamic)
  for (int i = 0; i < n; ++i) {
    uint64_t q = c->mod[i];
    uint64_t* s_ntt = (uint64_t*)malloc(sizeof(uint64_t) * N);
    small_to_ntt_i8(c, s, i, s_ntt);
    for (int x = 0; x < N; ++x)
      m[(size_t)i * N + x] = addmod(ct[(size_t)i * N + x], mulmod(ct[((size_t)n + i) * N + x], s_ntt[x], q), q);
    free(s_ntt);
  }
  free(s);
}

/* ------------------------------------------------------------------ */
/* CKKS encoding (DESIGN R-ENCODE)                            */
/* m_k = round( Delta/N * Re sum_{odd e} v[e] zeta^{-e k} ),            */
/* v[5^j mod 2N] = z_j, v[-5^j mod 2N] = conj(z_j), zeta = exp(i pi/N). */
/* Computed with a radix-2 complex FFT of length 2N in __float128;      */
/* rounding half away from zero, |frac-1/2| < 2^-40 counts as a tie.    */
/* ------------------------------------------------------------------ */
static void fft_q(__complex128* x, int n, int inverse) {
  /* iterative radix-2, bit-reversal permutation first; X[k] = sum x[j] e^{-+2 pi i jk/n} */
  int bits = 0; while ((1 << bits) < n) ++bits;
  for (int i = 0; i < n; ++i) { int j = (int)bitrev((uint32_t)i, bits); if (j > i) { __complex128 t = x[i]; x[i] = x[j]; x[j] = t; } }
  for (int len = 2; len <= n; len <<= 1) {
    for (int k = 0; k < len / 2; ++k) {
      __float128 ang = 2 * M_PIq * k / len;
      __complex128 w = cosq(ang) + (inverse ? 1 : -1) * sinq(ang) * 1.0iQ;
      for (int i = 0; i < n; i += len) {
        __complex128 u = x[i + k], v = x[i + k + len / 2] * w;
        x[i + k] = u + v;
        x[i + k + len / 2] = u - v;
      }
    }
  }
}

static int64_t round_tie_away(__float128 x) {
  __float128 f = floorq(x);
  __float128 frac = x - f;
  __float128 d = frac - 0.5Q;
  if (d < 0) d = -d;
  int64_t fl = (int64_t)f;
  if (d < 0x1p-40Q) return x > 0 ? fl + 1 : fl;
  return frac > 0.5Q ? fl + 1 : fl;
}

/* z_re/z_im: n_slots values (n_slots = N/2); z_im may be NULL. scale: exact integer Delta.
 * out: N signed integer coefficients. Returns 0, or -1 if some |m_k| >= 2^62. */
int orc_encode_coeffs(const orc_ctx* c, const double* z_re, const double* z_im, uint64_t scale, int64_t* out) {
  const int N = c->N, n = N / 2, twoN = 2 * N;
  __complex128* v = (__complex128*)calloc(twoN, sizeof(__complex128));
  uint64_t g = 1;
  for (int j = 0; j < n; ++j) {
    __float128 re = z_re[j], im = z_im ? z_im[j] : 0;
    v[g] = re + im * 1.0iQ;
    v[twoN - g] = re - im * 1.0iQ;
    g = (g * 5) % (uint64_t)twoN;
  }
  fft_q(v, twoN, 0);
  int rc = 0;
  for (int k = 0; k < N; ++k) {
    __float128 x = crealq(v[k]) * (__float128)scale / N;
    if (fabsq(x) >= 0x1p62Q) rc = -1;
    out[k] = round_tie_away(x);
  }
  free(v);
  return rc;
}

/* integer coefficients -> NTT-domain plaintext on chain limbs 0..level */
void orc_coeffs_to_pt(const orc_ctx* c, const int64_t* coef, int level, uint64_t* pt) {
#pragma omp parallel for
  for (int i = 0; i <= level; ++i) {
    for (int x = 0; x < c->N; ++x) pt[(size_t)i * c->N + x] = from_signed(coef[x], c->mod[i]);
    orc_ntt(c, i, pt + (size_t)i * c->N);
  }
}

/* ------------------------------------------------------------------ */
/* Key switching pieces (DESIGN R-MODUP / R-MODDOWN)       */
/* ------------------------------------------------------------------ */
static int n_digits(const orc_ctx* c, int level) { return (level + 1 + c->alpha - 1) / c->alpha; }
int orc_n_digits(const orc_ctx* c, int level) { return n_digits(c, level); }

/* ModUp of one polynomial given in the COEFFICIENT domain on q_0..q_level.
 * out: [beta][level+1+K][N] NTT domain.  Digit j = q-limbs [j*alpha, min((j+1)*alpha, level+1)).
 * Fast basis conversion without correction:
 *   y_i = [d_i * (D_j/q_i)^{-1}]_{q_i},  d~_j[t] = sum_i y_i * [(D_j/q_i) mod t]  mod t. */
void orc_modup_coeff(const orc_ctx* c, int level, const uint64_t* d, uint64_t* out) {
  const int N = c->N, K = c->np, E = level + 1 + K, beta = n_digits(c, level);
  int* chain = (int*)malloc(sizeof(int) * E);
  for (int u = 0; u < E; ++u) chain[u] = ext_chain(c, level, u);
  for (int j = 0; j < beta; ++j) {
    int lo = j * c->alpha, hi = (j + 1) * c->alpha; if (hi > level + 1) hi = level + 1;
    uint64_t* o = out + (size_t)j * E * N;
    /* constants */
    uint64_t hat_inv[ORC_MAXP];            /* (D_j/q_i)^{-1} mod q_i */
    for (int i = lo; i < hi; ++i) {
      uint64_t q = c->mod[i], v = 1;
      for (int i2 = lo; i2 < hi; ++i2) if (i2 != i) v = mulmod(v, c->mod[i2] % q, q);
      hat_inv[i] = invmod(v, q);
    }
#pragma omp parallel for schedule(dynamic)
    for (int u = 0; u < E; ++u) {
      int t = chain[u];
      uint64_t* ou = o + (size_t)u * N;
      if (u >= lo && u < hi) { memcpy(ou, d + (size_t)u * N, sizeof(uint64_t) * N); continue; }
      uint64_t mt = c->mod[t];
      uint64_t hat_mod_t[ORC_MAXP];        /* (D_j/q_i) mod t */
      for (int i = lo; i < hi; ++i) {
        uint64_t v = 1;
        for (int i2 = lo; i2 < hi; ++i2) if (i2 != i) v = mulmod(v, c->mod[i2] % mt, mt);
        hat_mod_t[i] = v;
      }
      for (int x = 0; x < N; ++x) {
        uint64_t acc = 0;
        for (int i = lo; i < hi; ++i) {
          uint64_t y = mulmod(d[(size_t)i * N + x], hat_inv[i], c->mod[i]);
          acc = addmod(acc, mulmod(y % mt, hat_mod_t[i], mt), mt);
        }
        ou[x] = acc;
      }
    }
    ntt_limbs(c, o, chain, E);
  }
  free(chain);
}

/* Inner product with the evaluation key: u_c[u] = sum_j ext[j][u] * evk[j][c][chain(u)] (NTT domain).
 * ext: [beta][E][N]; evk: [dnum][2][nq+np][N]; u_out: [2][E][N]. */
void orc_ks_inner_product(const orc_ctx* c, int level, const uint64_t* ext, const uint64_t* evk, uint64_t* u_out) {
  const int N = c->N, E = level + 1 + c->np, beta = n_digits(c, level), L1 = c->nq + c->np;
#pragma omp parallel for schedule(dynamic)
  for (int cu = 0; cu < 2 * E; ++cu) {
    int cc = cu / E, u = cu % E, t = ext_chain(c, level, u);
    uint64_t q = c->mod[t];
    uint64_t* o = u_out + ((size_t)cc * E + u) * N;
    for (int x = 0; x < N; ++x) {
      uint64_t acc = 0;
      for (int j = 0; j < beta; ++j)
        acc = addmod(acc, mulmod(ext[((size_t)j * E + u) * N + x], evk[((size_t)(j * 2 + cc) * L1 + t) * N + x], q), q);
      o[x] = acc;
    }
  }
}

/* ModDown of one polynomial u [E][N] (NTT domain, Q_l u P) -> out [level+1][N] (NTT domain):
 * z_k = [v_k * (P/p_k)^{-1}]_{p_k} with v = iNTT(u on P), taken as the centred remainder in (-p_k/2, p_k/2]
 * (DESIGN R-MODDOWN: then sum_k z_k (P/p_k) = [u]_P + e P with e symmetric about 0, |e| <= K/2, and the division by
 * P rounds without bias), out_i = (u_i - NTT_i( sum_k z_k * [(P/p_k) mod q_i] mod q_i )) * [P^{-1}]_{q_i}. */
void orc_moddown(const orc_ctx* c, int level, const uint64_t* u, uint64_t* out) {
  const int N = c->N, K = c->np, nq_l = level + 1;
  uint64_t* v = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)K * N);
  memcpy(v, u + (size_t)nq_l * N, sizeof(uint64_t) * (size_t)K * N);
  int pchain[ORC_MAXP];
  for (int k = 0; k < K; ++k) pchain[k] = c->nq + k;
  intt_limbs(c, v, pchain, K);
  /* z_k */
  for (int k = 0; k < K; ++k) {
    uint64_t pk = c->mod[c->nq + k], hat = 1;
    for (int k2 = 0; k2 < K; ++k2) if (k2 != k) hat = mulmod(hat, c->mod[c->nq + k2] % pk, pk);
    uint64_t hinv = invmod(hat, pk);
    for (int x = 0; x < N; ++x) v[(size_t)k * N + x] = mulmod(v[(size_t)k * N + x], hinv, pk);
  }
#pragma omp parallel for schedule(dynamic)
  for (int i = 0; i < nq_l; ++i) {
    uint64_t q = c->mod[i];
    uint64_t hat_mod_q[ORC_MAXP], Pmod = 1;
    for (int k = 0; k < K; ++k) {
      uint64_t h = 1;
      for (int k2 = 0; k2 < K; ++k2) if (k2 != k) h = mulmod(h, c->mod[c->nq + k2] % q, q);
      hat_mod_q[k] = h;
      Pmod = mulmod(Pmod, c->mod[c->nq + k] % q, q);
    }
    uint64_t Pinv = invmod(Pmod, q);
    uint64_t* w = (uint64_t*)malloc(sizeof(uint64_t) * N);
    for (int x = 0; x < N; ++x) {
      uint64_t acc = 0;
      for (int k = 0; k < K; ++k) {
        const uint64_t pk = c->mod[c->nq + k], z = v[(size_t)k * N + x];
        /* centred z: z - p_k when z > (p_k - 1)/2, reduced mod q */
        const uint64_t zq = z > (pk - 1) / 2 ? (q - (pk - z) % q) % q : z % q;
        acc = addmod(acc, mulmod(zq, hat_mod_q[k], q), q);
      }
      w[x] = acc;
    }
    orc_ntt(c, i, w);
    for (int x = 0; x < N; ++x) out[(size_t)i * N + x] = mulmod(submod(u[(size_t)i * N + x], w[x], q), Pinv, q);
    free(w);
  }
  free(v);
}

/* ------------------------------------------------------------------ */
/* HRot variants (DESIGN R-HROT)                              */
/* ------------------------------------------------------------------ */
static int* q_chain(int n) { int* ch = (int*)malloc(sizeof(int) * n); for (int i = 0; i < n; ++i) ch[i] = i; return ch; }

/* plain: ModUp(kappa(c1)) */
void orc_hrot(const orc_ctx* c, int level, const uint64_t* evk, uint64_t k, const uint64_t* ct, uint64_t* out) {
  const int N = c->N, n = level + 1, E = n + c->np, beta = n_digits(c, level);
  size_t pl = (size_t)n * N;
  if (k == 1) { memcpy(out, ct, sizeof(uint64_t) * 2 * pl); return; }
  int* ch = q_chain(n);
  uint64_t* rc = (uint64_t*)malloc(sizeof(uint64_t) * 2 * pl);
  automorph_ntt_limbs(c, ct, rc, ch, n, k);
  automorph_ntt_limbs(c, ct + pl, rc + pl, ch, n, k);
  uint64_t* d = (uint64_t*)malloc(sizeof(uint64_t) * pl);
  memcpy(d, rc + pl, sizeof(uint64_t) * pl);
  intt_limbs(c, d, ch, n);
  uint64_t* ext = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)beta * E * N);
  orc_modup_coeff(c, level, d, ext);
  uint64_t* u = (uint64_t*)malloc(sizeof(uint64_t) * 2 * (size_t)E * N);
  orc_ks_inner_product(c, level, ext, evk, u);
  orc_moddown(c, level, u, out);
  orc_moddown(c, level, u + (size_t)E * N, out + pl);
  for (int i = 0; i < n; ++i)
    for (int x = 0; x < N; ++x) out[(size_t)i * N + x] = addmod(out[(size_t)i * N + x], rc[(size_t)i * N + x], c->mod[i]);
  free(ch); free(rc); free(d); free(ext); free(u);
}

/* hoisted (Halevi-Shoup): one ModUp of c1, kappa applied to the extended digits per rotation. */
void orc_hrot_hoisted(const orc_ctx* c, int level, const uint64_t* const* evks, const uint64_t* ks, int nrot,
                      const uint64_t* ct, uint64_t* const* outs) {
  const int N = c->N, n = level + 1, E = n + c->np, beta = n_digits(c, level);
  size_t pl = (size_t)n * N;
  int* ch = q_chain(n);
  int* ech = (int*)malloc(sizeof(int) * E);
  for (int u = 0; u < E; ++u) ech[u] = ext_chain(c, level, u);
  uint64_t* d = (uint64_t*)malloc(sizeof(uint64_t) * pl);
  memcpy(d, ct + pl, sizeof(uint64_t) * pl);
  intt_limbs(c, d, ch, n);
  uint64_t* ext = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)beta * E * N);
  orc_modup_coeff(c, level, d, ext);
  uint64_t* ext_r = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)beta * E * N);
  uint64_t* u = (uint64_t*)malloc(sizeof(uint64_t) * 2 * (size_t)E * N);
  uint64_t* c0r = (uint64_t*)malloc(sizeof(uint64_t) * pl);
  for (int r = 0; r < nrot; ++r) {
    uint64_t k = ks[r];
    if (k == 1) { memcpy(outs[r], ct, sizeof(uint64_t) * 2 * pl); continue; }
    for (int j = 0; j < beta; ++j)
      automorph_ntt_limbs(c, ext + (size_t)j * E * N, ext_r + (size_t)j * E * N, ech, E, k);
    orc_ks_inner_product(c, level, ext_r, evks[r], u);
    orc_moddown(c, level, u, outs[r]);
    orc_moddown(c, level, u + (size_t)E * N, outs[r] + pl);
    automorph_ntt_limbs(c, ct, c0r, ch, n, k);
    for (int i = 0; i < n; ++i)
      for (int x = 0; x < N; ++x)
        outs[r][(size_t)i * N + x] = addmod(outs[r][(size_t)i * N + x], c0r[(size_t)i * N + x], c->mod[i]);
  }
  free(ch); free(ech); free(d); free(ext); free(ext_r); free(u); free(c0r);
}

/* lazy sum: sum_t HRot_{k_t}(x_t) with the inner products accumulated over Q_l u P and one ModDown.
 * Terms with k_t == 1 are added without key switching. */
void orc_hrot_sum(const orc_ctx* c, int level, const uint64_t* const* evks, const uint64_t* ks, int nterm,
                  const uint64_t* const* cts, uint64_t* out) {
  const int N = c->N, n = level + 1, E = n + c->np, beta = n_digits(c, level);
  size_t pl = (size_t)n * N;
  int* ch = q_chain(n);
  uint64_t* acc_u = (uint64_t*)calloc(2 * (size_t)E * N, sizeof(uint64_t));
  uint64_t* acc_c = (uint64_t*)calloc(2 * pl, sizeof(uint64_t));
  uint64_t* rc = (uint64_t*)malloc(sizeof(uint64_t) * 2 * pl);
  uint64_t* d = (uint64_t*)malloc(sizeof(uint64_t) * pl);
  uint64_t* ext = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)beta * E * N);
  uint64_t* u = (uint64_t*)malloc(sizeof(uint64_t) * 2 * (size_t)E * N);
  int any_ks = 0;
  for (int t = 0; t < nterm; ++t) {
    if (ks[t] == 1) {
      for (int i = 0; i < n; ++i)
        for (int x = 0; x < N; ++x) {
          acc_c[(size_t)i * N + x] = addmod(acc_c[(size_t)i * N + x], cts[t][(size_t)i * N + x], c->mod[i]);
          acc_c[pl + (size_t)i * N + x] = addmod(acc_c[pl + (size_t)i * N + x], cts[t][pl + (size_t)i * N + x], c->mod[i]);
        }
      continue;
    }
    any_ks = 1;
    automorph_ntt_limbs(c, cts[t], rc, ch, n, ks[t]);
    automorph_ntt_limbs(c, cts[t] + pl, rc + pl, ch, n, ks[t]);
    memcpy(d, rc + pl, sizeof(uint64_t) * pl);
    intt_limbs(c, d, ch, n);
    orc_modup_coeff(c, level, d, ext);
    orc_ks_inner_product(c, level, ext, evks[t], u);
    for (int cc = 0; cc < 2; ++cc)
      for (int uu = 0; uu < E; ++uu) {
        uint64_t q = c->mod[ext_chain(c, level, uu)];
        for (int x = 0; x < N; ++x) {
          size_t o = ((size_t)cc * E + uu) * N + x;
          acc_u[o] = addmod(acc_u[o], u[o], q);
        }
      }
    for (int i = 0; i < n; ++i)
      for (int x = 0; x < N; ++x)
        acc_c[(size_t)i * N + x] = addmod(acc_c[(size_t)i * N + x], rc[(size_t)i * N + x], c->mod[i]);
  }
  if (any_ks) {
    orc_moddown(c, level, acc_u, out);
    orc_moddown(c, level, acc_u + (size_t)E * N, out + pl);
  } else {
    memset(out, 0, sizeof(uint64_t) * 2 * pl);
  }
  for (size_t o = 0; o < 2 * pl; ++o) {
    int i = (int)((o % pl) / N);
    out[o] = addmod(out[o], acc_c[o], c->mod[i]);
  }
  free(ch); free(acc_u); free(acc_c); free(rc); free(d); free(ext); free(u);
}

/* ------------------------------------------------------------------ */
/* MulPt / AddCt / Rescale                                   */
/* ------------------------------------------------------------------ */
/* ct [2][level+1][N] times pt [level+1][N], limbwise (no auto-rescale). */
void orc_pmult(const orc_ctx* c, int level, const uint64_t* ct, const uint64_t* pt, uint64_t* out) {
  const int N = c->N, n = level + 1;
  for (int p = 0; p < 2; ++p)
    for (int i = 0; i < n; ++i)
      for (int x = 0; x < N; ++x) {
        size_t o = ((size_t)p * n + i) * N + x;
        out[o] = mulmod(ct[o], pt[(size_t)i * N + x], c->mod[i]);
      }
}

/* elementwise add of two [npoly][level+1][N] arrays */
void orc_add(const orc_ctx* c, int level, int npoly, const uint64_t* a, const uint64_t* b, uint64_t* out) {
  const int N = c->N, n = level + 1;
  for (int p = 0; p < npoly; ++p)
    for (int i = 0; i < n; ++i)
      for (int x = 0; x < N; ++x) {
        size_t o = ((size_t)p * n + i) * N + x;
        out[o] = addmod(a[o], b[o], c->mod[i]);
      }
}

/* Rescale (DESIGN R-RESCALE): v = iNTT(c_l), centred (v > (q_l-1)/2 -> v - q_l),
 * c'_i = (c_i - NTT_i([v]_{q_i})) * q_l^{-1} mod q_i, i < l.  out: [2][level][N]. */
void orc_rescale(const orc_ctx* c, int level, const uint64_t* ct, uint64_t* out) {
  const int N = c->N, n = level + 1;
  const uint64_t ql = c->mod[level];
  for (int p = 0; p < 2; ++p) {
    uint64_t* v = (uint64_t*)malloc(sizeof(uint64_t) * N);
    memcpy(v, ct + ((size_t)p * n + level) * N, sizeof(uint64_t) * N);
    orc_intt(c, level, v);
#pragma omp parallel for
    for (int i = 0; i < level; ++i) {
      uint64_t q = c->mod[i];
      uint64_t qinv = invmod(ql % q, q);
      uint64_t* w = (uint64_t*)malloc(sizeof(uint64_t) * N);
      for (int x = 0; x < N; ++x) {
        int64_t sv = v[x] > (ql - 1) / 2 ? (int64_t)v[x] - (int64_t)ql : (int64_t)v[x];
        w[x] = from_signed(sv, q);
      }
      orc_ntt(c, i, w);
      for (int x = 0; x < N; ++x)
        out[((size_t)p * level + i) * N + x] = mulmod(submod(ct[((size_t)p * n + i) * N + x], w[x], q), qinv, q);
      free(w);
    }
    free(v);
  }
}

/* ------------------------------------------------------------------ */
/* MulCt with relinearization (key switching P:1238-1241)    */
/* ------------------------------------------------------------------ */
/* Relinearization key (DESIGN R-RELIN): the hybrid key-switching key from s^2 to s,
 * b_j = -a_j*s + e_j + g_j*s^2 with the g_j of R-EVK, object id (0 << 8) | j (Galois element 0,
 * which no rotation uses).  Layout as orc_keygen_rot. */
void orc_keygen_relin(const orc_ctx* c, uint64_t sk_seed, int h, uint64_t ek_seed, uint64_t* evk) {
  const int N = c->N, L1 = c->nq + c->np;
  int8_t* s = (int8_t*)malloc(N);
  orc_sample_secret(c, sk_seed, h, s);
#pragma omp parallel for schedule(dynamic)
  for (int jt = 0; jt < c->dnum * L1; ++jt) {
    int j = jt / L1, t = jt % L1;
    uint64_t q = c->mod[t];
    uint64_t obj = (uint64_t)j;
    uint64_t* b = evk + ((size_t)(j * 2 + 0) * L1 + t) * N;
    uint64_t* a = evk + ((size_t)(j * 2 + 1) * L1 + t) * N;
    uint64_t* s_ntt = (uint64_t*)malloc(sizeof(uint64_t) * N);
    uint64_t* e_ntt = (uint64_t*)malloc(sizeof(uint64_t) * N);
    int32_t* e = (int32_t*)malloc(sizeof(int32_t) * N);
    small_to_ntt_i8(c, s, t, s_ntt);
    orc_sample_cbd(ek_seed, DOM_EVK_E, obj, N, e);
    small_to_ntt_i32(c, e, t, e_ntt);
    uint64_t g = 0;
    if (t < c->nq && t >= j * c->alpha && t < (j + 1) * c->alpha) {
      g = 1;
      for (int kk = 0; kk < c->np; ++kk) g = mulmod(g, c->mod[c->nq + kk] % q, q);
    }
    for (int i = 0; i < N; ++i) {
      a[i] = draw_uniform(ek_seed, DOM_EVK_A, obj, (uint32_t)t, (uint32_t)i, q);
      uint64_t v = submod(e_ntt[i], mulmod(a[i], s_ntt[i], q), q);
      /* s^2 in the NTT domain is the pointwise square (NTT multiplication = negacyclic product) */
      b[i] = addmod(v, mulmod(g, mulmod(s_ntt[i], s_ntt[i], q), q), q);
    }
    free(s_ntt); free(e_ntt); free(e);
  }
  free(s);
}

/* MulCt: the tensor product of a = (a0, a1) and b = (b0, b1) at level l,
 *   d0 = a0 b0, d1 = a0 b1 + a1 b0, d2 = a1 b1            (NTT domain, limbwise mod q_i),
 * so that d0 + d1 s + d2 s^2 = (a0 + a1 s)(b0 + b1 s); then d2 is key-switched from s^2 to s with the
 * relinearization key exactly as HRot's plain path switches kappa(c1) (iNTT, ModUp, IP, ModDown; no
 * automorphism):  out = (d0 + KS_0(d2), d1 + KS_1(d2)).  No rescale (the caller rescales). */
void orc_mulct(const orc_ctx* c, int level, const uint64_t* a, const uint64_t* b, const uint64_t* rlk, uint64_t* out) {
  const int N = c->N, n = level + 1, E = n + c->np, beta = n_digits(c, level);
  size_t pl = (size_t)n * N;
  uint64_t* d2 = (uint64_t*)malloc(sizeof(uint64_t) * pl);
  for (int i = 0; i < n; ++i) {
    uint64_t q = c->mod[i];
    for (int x = 0; x < N; ++x) {
      size_t o = (size_t)i * N + x;
      out[o] = mulmod(a[o], b[o], q);
      out[pl + o] = addmod(mulmod(a[o], b[pl + o], q), mulmod(a[pl + o], b[o], q), q);
      d2[o] = mulmod(a[pl + o], b[pl + o], q);
    }
  }
  int* ch = q_chain(n);
  intt_limbs(c, d2, ch, n);
  uint64_t* ext = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)beta * E * N);
  orc_modup_coeff(c, level, d2, ext);
  uint64_t* u = (uint64_t*)malloc(sizeof(uint64_t) * 2 * (size_t)E * N);
  orc_ks_inner_product(c, level, ext, rlk, u);
  uint64_t* ks = (uint64_t*)malloc(sizeof(uint64_t) * 2 * pl);
  orc_moddown(c, level, u, ks);
  orc_moddown(c, level, u + (size_t)E * N, ks + pl);
  for (size_t o = 0; o < 2 * pl; ++o) out[o] = addmod(out[o], ks[o], c->mod[(o % pl) / N]);
  free(ch); free(d2); free(ext); free(u); free(ks);
}
