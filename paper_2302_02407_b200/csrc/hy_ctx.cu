// hy_ctx.cu -- context creation: primes, roots, twiddle tables, basis-conversion
// constants, workspace and error plumbing (host side of the C ABI).
//
// Parameter readings:
//   R-PRIMES  chain order q_0..q_{nq-1}, p_0..p_{np-1}; each is the largest
//             unused prime below 2^bits with p == 1 (mod 2N).
//   R-NTT     psi = smallest primitive 2N-th root of unity mod p; forward NTT
//             output index k holds a(psi^(2 br(k) + 1)).
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "hy_internal.h"

using u128 = unsigned __int128;

namespace {
thread_local std::string g_err;

uint64_t mul_h(uint64_t a, uint64_t b, uint64_t m) { return (uint64_t)((u128)a * b % m); }
uint64_t pow_h(uint64_t b, uint64_t e, uint64_t m) {
  uint64_t r = 1 % m;
  b %= m;
  for (; e; e >>= 1, b = mul_h(b, b, m))
    if (e & 1) r = mul_h(r, b, m);
  return r;
}
uint64_t inv_h(uint64_t a, uint64_t m) {  // extended Euclid (m need not be prime)
  int64_t t = 0, nt = 1;
  uint64_t r = m, nr = a % m;
  while (nr) {
    uint64_t qq = r / nr;
    int64_t tt = t - (int64_t)qq * nt;
    t = nt;
    nt = tt;
    uint64_t rr = r - qq * nr;
    r = nr;
    nr = rr;
  }
  return t < 0 ? (uint64_t)(t + (int64_t)m) : (uint64_t)t;
}
uint64_t shoup_pre(uint64_t w, uint64_t q) { return (uint64_t)(((u128)w << 64) / q); }

// Miller-Rabin with the first twelve prime bases: deterministic below 3.3e24.
bool is_prime_h(uint64_t n) {
  if (n < 2) return false;
  const uint64_t bases[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  for (uint64_t b : bases) {
    if (n % b == 0) return n == b;
  }
  uint64_t d = n - 1;
  int r = 0;
  while (!(d & 1)) d >>= 1, ++r;
  for (uint64_t b : bases) {
    uint64_t x = pow_h(b, d, n);
    if (x == 1 || x == n - 1) continue;
    bool witness = true;
    for (int i = 1; i < r && witness; ++i) {
      x = mul_h(x, x, n);
      if (x == n - 1) witness = false;
    }
    if (witness) return false;
  }
  return true;
}

uint32_t brev(uint32_t x, int bits) {
  uint32_t r = 0;
  for (int i = 0; i < bits; ++i) r |= ((x >> i) & 1u) << (bits - 1 - i);
  return r;
}
}  // namespace

namespace hy {
hy_status fail(hy_status s, const std::string& msg) {
  g_err = msg;
  return s;
}
hy_status cuda_check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(HY_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return HY_OK;
}
}  // namespace hy

extern "C" const char* hy_last_error(void) { return g_err.c_str(); }

extern "C" hy_status hy_ctx_create(const hy_params* prm, int cuda_device, hy_ctx** out) {
  using namespace hy;
  if (!prm || !out || !prm->q_bits || !prm->p_bits) return fail(HY_E_ARG, "null argument");
  if (prm->log_n < 10 || prm->log_n > 16) return fail(HY_E_ARG, "log_n must be in [10,16]");
  if (prm->n_q < 1 || prm->n_q + prm->n_p > (uint32_t)kMaxChain || prm->dnum < 1)
    return fail(HY_E_ARG, "bad chain length / dnum");
  uint32_t alpha = (prm->n_q + prm->dnum - 1) / prm->dnum;
  if (alpha > 8 || prm->n_p > 8 || prm->n_p < 1) return fail(HY_E_ARG, "alpha and n_p must be in [1,8]");
  // hybrid key switching needs P >= every digit's product D_j (the KS noise bound, DESIGN R-KSBOUND): with
  // primes of at most 48 bits and digits of alpha primes that means K >= alpha special primes
  if (prm->n_p < alpha) return fail(HY_E_ARG, "n_p (K special primes) must be >= alpha = ceil(n_q/dnum)");
  if (prm->n_q + prm->n_p > (uint32_t)kMaxExt) return fail(HY_E_ARG, "chain too long");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= cuda_device) {
    cudaGetLastError();
    return fail(HY_E_NO_DEVICE, "no CUDA device (the product path has no CPU fallback)");
  }
  cudaSetDevice(cuda_device);

  hy_ctx* c = new hy_ctx();
  c->device = cuda_device;
  c->log_n = prm->log_n;
  c->N = 1u << prm->log_n;
  c->n_q = prm->n_q;
  c->n_p = prm->n_p;
  c->dnum = prm->dnum;
  c->alpha = alpha;
  c->h = prm->hamming_weight;
  const uint64_t twoN = 2ull * c->N;
  const uint32_t L = c->n_q + c->n_p;

  // primes (R-PRIMES)
  for (uint32_t t = 0; t < L; ++t) {
    uint32_t bits = t < c->n_q ? prm->q_bits[t] : prm->p_bits[t - c->n_q];
    if (bits < 20 || bits > 48) {  // the FP64-pipe NTT needs q < 2^48 (hy_ntt.cu)
      delete c;
      return fail(HY_E_ARG, "prime bit sizes must be in [20,48]");
    }
    uint64_t cand = (((1ull << bits) - 2) / twoN) * twoN + 1;
    for (;; cand -= twoN) {
      if (cand <= twoN) {
        delete c;
        return fail(HY_E_ARG, "ran out of primes");
      }
      bool used = false;
      for (uint64_t m : c->mod) used |= (m == cand);
      if (!used && is_prime_h(cand)) break;
    }
    c->mod.push_back(cand);
  }
  // roots (R-NTT): smallest element of the set of primitive 2N-th roots
  for (uint32_t t = 0; t < L; ++t) {
    uint64_t q = c->mod[t], root = 0;
    for (uint64_t g = 2; !root; ++g) {
      uint64_t x = pow_h(g, (q - 1) / twoN, q);
      if (pow_h(x, c->N, q) == q - 1) root = x;
    }
    uint64_t best = root, x = root, r2 = mul_h(root, root, q);
    for (uint64_t e = 3; e < twoN; e += 2) {
      x = mul_h(x, r2, q);
      if (x < best) best = x;
    }
    c->psi.push_back(best);
  }

  // twiddle tables + prime constants, one allocation
  const size_t tw_words = (size_t)L * c->N;
  std::vector<double> tw(tw_words), itw(tw_words);
  std::vector<PrimeConst> pc(L);
  std::vector<uint64_t> pw(c->N), ipw(c->N);
  for (uint32_t t = 0; t < L; ++t) {
    uint64_t q = c->mod[t], ps = c->psi[t], ips = inv_h(ps, q);
    pw[0] = ipw[0] = 1;
    for (uint32_t k = 1; k < c->N; ++k) {
      pw[k] = mul_h(pw[k - 1], ps, q);
      ipw[k] = mul_h(ipw[k - 1], ips, q);
    }
    for (uint32_t k = 0; k < c->N; ++k) {
      size_t o = (size_t)t * c->N + k;
      tw[o] = (double)pw[brev(k, c->log_n)];
      itw[o] = (double)ipw[brev(k, c->log_n)];
    }
    PrimeConst& p = pc[t];
    p.q = q;
    p.two_q = 2 * q;
    p.mu = (uint64_t)((((u128)1) << 64) / q);
    p.r64 = (uint64_t)((((u128)1) << 64) % q);
    p.r64_sh = shoup_pre(p.r64, q);
    p.n_inv = inv_h(c->N % q, q);
    p.n_inv_sh = shoup_pre(p.n_inv, q);
    p.qd = (double)q;
    p.qinv = 1.0 / (double)q;
    p.n_inv_d = (double)p.n_inv;
  }
  size_t bytes = 2 * tw_words * 8 + L * sizeof(PrimeConst);
  if (cudaMalloc(&c->d_tables, bytes) != cudaSuccess) {
    delete c;
    return cuda_check("cudaMalloc tables");
  }
  uint64_t* base = (uint64_t*)c->d_tables;
  cudaMemcpy(base, tw.data(), tw_words * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(base + tw_words, itw.data(), tw_words * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(base + 2 * tw_words, pc.data(), L * sizeof(PrimeConst), cudaMemcpyHostToDevice);
  c->dt.tw = reinterpret_cast<const double*>(base);
  c->dt.itw = reinterpret_cast<const double*>(base + tw_words);
  c->dt.pc = reinterpret_cast<const PrimeConst*>(base + 2 * tw_words);

  // basis-conversion constants per level
  const uint32_t K = c->n_p;
  c->h_modup.resize(c->n_q);
  c->h_moddown.resize(c->n_q);
  c->h_rescale.resize(c->n_q);
  for (uint32_t lvl = 0; lvl < c->n_q; ++lvl) {
    uint32_t beta = n_digits(c, lvl), E = lvl + 1 + K;
    auto& mu = c->h_modup[lvl];
    mu.assign(beta, ModUpConst{});
    for (uint32_t j = 0; j < beta; ++j) {
      ModUpConst& m = mu[j];
      m.lo = j * alpha;
      m.hi = std::min((j + 1) * alpha, lvl + 1);
      for (int i = m.lo; i < m.hi; ++i) {
        uint64_t qi = c->mod[i], prod = 1;
        for (int i2 = m.lo; i2 < m.hi; ++i2)
          if (i2 != i) prod = mul_h(prod, c->mod[i2] % qi, qi);
        m.hat_inv[i - m.lo] = inv_h(prod, qi);
        m.hat_inv_sh[i - m.lo] = shoup_pre(m.hat_inv[i - m.lo], qi);
        for (uint32_t u = 0; u < E; ++u) {
          uint64_t mt = c->mod[ext_chain(c, lvl, u)], v = 1;
          for (int i2 = m.lo; i2 < m.hi; ++i2)
            if (i2 != i) v = mul_h(v, c->mod[i2] % mt, mt);
          m.hat_mod[u][i - m.lo] = v;
        }
      }
    }
    ModDownConst& md = c->h_moddown[lvl];
    memset(&md, 0, sizeof(md));
    for (uint32_t k = 0; k < K; ++k) {
      uint64_t pk = c->mod[c->n_q + k], prod = 1;
      for (uint32_t k2 = 0; k2 < K; ++k2)
        if (k2 != k) prod = mul_h(prod, c->mod[c->n_q + k2] % pk, pk);
      md.phat_inv[k] = inv_h(prod, pk);
      md.phat_inv_sh[k] = shoup_pre(md.phat_inv[k], pk);
    }
    for (uint32_t i = 0; i <= lvl; ++i) {
      uint64_t qi = c->mod[i], P = 1;
      for (uint32_t k = 0; k < K; ++k) {
        uint64_t v = 1;
        for (uint32_t k2 = 0; k2 < K; ++k2)
          if (k2 != k) v = mul_h(v, c->mod[c->n_q + k2] % qi, qi);
        md.phat_mod[i][k] = v;
        P = mul_h(P, c->mod[c->n_q + k] % qi, qi);
      }
      md.p_inv[i] = inv_h(P, qi);
      md.p_inv_sh[i] = shoup_pre(md.p_inv[i], qi);
    }
    md.src0 = c->n_q;
    md.center = 1;  // R-MODDOWN: the centred remainder (zero-mean rounding; a floor-style lift biases every coefficient)
    RescaleConst& rc = c->h_rescale[lvl];
    memset(&rc, 0, sizeof(rc));
    for (uint32_t i = 0; i < lvl; ++i) {
      rc.ql_inv[i] = inv_h(c->mod[lvl] % c->mod[i], c->mod[i]);
      rc.ql_inv_sh[i] = shoup_pre(rc.ql_inv[i], c->mod[i]);
    }
  }
  c->d_modup.resize(c->n_q);
  c->d_moddown.resize(c->n_q);
  c->d_rescale.resize(c->n_q);
  c->d_rescale_md.assign(c->n_q, nullptr);
  for (uint32_t lvl = 1; lvl < c->n_q; ++lvl) {  // rescale = ModDown by P = q_lvl (K = 1), centred
    ModDownConst md;
    memset(&md, 0, sizeof(md));
    md.phat_inv[0] = 1;  // P / p_0 = 1
    for (uint32_t i = 0; i < lvl; ++i) {
      md.phat_mod[i][0] = 1 % c->mod[i];
      md.p_inv[i] = c->h_rescale[lvl].ql_inv[i];
      md.p_inv_sh[i] = c->h_rescale[lvl].ql_inv_sh[i];
    }
    md.src0 = lvl;
    md.center = 1;
    cudaMalloc(&c->d_rescale_md[lvl], sizeof(ModDownConst));
    cudaMemcpy(c->d_rescale_md[lvl], &md, sizeof(ModDownConst), cudaMemcpyHostToDevice);
  }
  for (uint32_t lvl = 0; lvl < c->n_q; ++lvl) {
    size_t b1 = sizeof(ModUpConst) * c->h_modup[lvl].size();
    cudaMalloc(&c->d_modup[lvl], b1);
    cudaMemcpy(c->d_modup[lvl], c->h_modup[lvl].data(), b1, cudaMemcpyHostToDevice);
    cudaMalloc(&c->d_moddown[lvl], sizeof(ModDownConst));
    cudaMemcpy(c->d_moddown[lvl], &c->h_moddown[lvl], sizeof(ModDownConst), cudaMemcpyHostToDevice);
    cudaMalloc(&c->d_rescale[lvl], sizeof(RescaleConst));
    cudaMemcpy(c->d_rescale[lvl], &c->h_rescale[lvl], sizeof(RescaleConst), cudaMemcpyHostToDevice);
  }
  hy_status s = cuda_check("ctx tables");
  if (s != HY_OK) {
    hy_ctx_destroy(c);
    return s;
  }
  *out = c;
  return HY_OK;
}

extern "C" void hy_ctx_destroy(hy_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  cudaFree(c->d_tables);
  if (c->d_enc) cudaFree(c->d_enc);
  for (auto p : c->d_modup) cudaFree(p);
  for (auto p : c->d_moddown) cudaFree(p);
  for (auto p : c->d_rescale) cudaFree(p);
  for (auto p : c->d_rescale_md) cudaFree(p);
  delete c;
}

extern "C" hy_status hy_ctx_moduli(const hy_ctx* c, uint64_t* out) {
  if (!c || !out) return hy::fail(HY_E_ARG, "null");
  for (size_t i = 0; i < c->mod.size(); ++i) out[i] = c->mod[i];
  return HY_OK;
}
extern "C" uint32_t hy_ctx_alpha(const hy_ctx* c) { return c ? c->alpha : 0; }
extern "C" uint32_t hy_ctx_n_digits(const hy_ctx* c, uint32_t level) { return c ? hy::n_digits(c, level) : 0; }
extern "C" uint64_t hy_ctx_launch_count(const hy_ctx* c) { return c ? c->launches : 0; }

extern "C" uint64_t hy_galois_elt(const hy_ctx* c, int64_t r) {
  int64_t n = c->N / 2;
  int64_t rr = ((r % n) + n) % n;
  return pow_h(5, (uint64_t)rr, 2ull * c->N);
}

// Workspace layout (words of N): see hy_keyswitch.cu ks_workspace().
extern "C" size_t hy_workspace_bytes(const hy_ctx* c, uint32_t max_level, uint32_t max_terms) {
  if (!c) return 0;
  if (max_level >= c->n_q) max_level = c->n_q - 1;
  // max_terms key switches per batched launch (capped at kG), plus one accumulator ciphertext;
  // at least enough for key generation (3 (n_q + n_p) limbs + small buffers)
  const size_t items = std::max<uint32_t>(1, std::min<uint32_t>(max_terms, (uint32_t)hy::kG));
  const size_t n = max_level + 1;
  const size_t ks = items * hy::ks_item_bytes(c, max_level) + 2 * n * (size_t)c->N * 8 + 4096;
  const size_t keygen = (3 * (size_t)(c->n_q + c->n_p) + 2) * c->N * 8 + 65536;
  return std::max(ks, keygen);
}

extern "C" hy_status hy_ctx_set_workspace(hy_ctx* c, void* d_ws, size_t bytes) {
  if (!c) return hy::fail(HY_E_ARG, "null ctx");
  c->ws = (uint8_t*)d_ws;
  c->ws_bytes = bytes;
  return HY_OK;
}

extern "C" hy_status hy_ctx_time_kernels(hy_ctx* c, uint32_t family_mask) {
  if (!c) return hy::fail(HY_E_ARG, "null ctx");
  c->time_mask = family_mask;
  c->timed.clear();
  c->ev_used = 0;
  return HY_OK;
}

extern "C" hy_status hy_ctx_kernel_times(hy_ctx* c, uint32_t family_mask, double* total_ms, uint64_t* n_launches,
                                        uint64_t* alg_bytes) {
  if (!c || !total_ms || !n_launches || !alg_bytes) return hy::fail(HY_E_ARG, "null");
  double tot = 0;
  uint64_t n = 0, by = 0;
  for (const auto& t : c->timed) {
    if (!(t.fam & family_mask)) continue;
    if (cudaEventSynchronize(t.b) != cudaSuccess) return hy::cuda_check("hy_ctx_kernel_times");
    float ms = 0;
    cudaEventElapsedTime(&ms, t.a, t.b);
    tot += ms;
    by += t.bytes;
    ++n;
  }
  *total_ms = tot;
  *n_launches = n;
  *alg_bytes = by;
  return HY_OK;
}
