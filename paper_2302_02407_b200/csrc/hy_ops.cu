// hy_ops.cu -- MulPt / MulFilter&Sum / AddCt / Rescale and the
// client-side key generation, encryption and decryption (
// DESIGN R-SK, R-EVK, R-ENC, R-PRNG), all as device kernels.
#include <vector>

#include "hy_arith.cuh"
#include "hy_rand.cuh"

namespace hy {
void launch_automorph(hy_ctx* c, const uint64_t* in, uint64_t* out, uint32_t n_limbs, uint64_t k, cudaStream_t s);

namespace {
constexpr int kT = 256;
constexpr int kMaxTerms = 64;

struct TermPtrs {
  const uint64_t* ct[kMaxTerms];
  const uint64_t* pt[kMaxTerms];
  uint64_t prot[kMaxTerms];  // Galois element of a PRot applied to pt (1 = none), fused as a gather
};

// out[p][i][x] (+)= sum_m ct_m[p][i][x] * pt_m[i][x] mod q_i.  grid (N/256, l+1, 2)
__global__ void k_pmult_acc(const __grid_constant__ TermPtrs tp, int nterm, uint64_t* __restrict__ out, DevTables dt, int level, int logN,
                            int accumulate) {
  const size_t N = (size_t)1 << logN;
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y, p = blockIdx.z;
  const size_t n = level + 1;
  const size_t o = ((size_t)p * n + i) * N + x;
  const PrimeConst& pc = dt.pc[i];
  U128 acc{0, 0};
  for (int m = 0; m < nterm; ++m) {
    const uint32_t xs = tp.prot[m] != 1 ? aut_index(x, tp.prot[m], logN) : x;
    mac(acc, tp.ct[m][o], tp.pt[m][(size_t)i * N + xs]);
  }
  uint64_t r = reduce128(acc, pc);
  if (accumulate) r = add_mod(r, out[o], pc.q);
  out[o] = r;
}

// out = a + b over [npoly][l+1][N].  grid (N/256, (l+1)*npoly)
__global__ void k_add(const uint64_t* __restrict__ a, const uint64_t* __restrict__ b, uint64_t* __restrict__ out,
                      DevTables dt, int nlimb, int logN) {
  const size_t N = (size_t)1 << logN;
  const size_t o = (size_t)blockIdx.y * N + blockIdx.x * blockDim.x + threadIdx.x;
  out[o] = add_mod(a[o], b[o], dt.pc[blockIdx.y % nlimb].q);
}

// Rescale step 2: w[p][i][x] = [centre(v[p][x])]_{q_i}, v = iNTT(c_p on q_l).  grid (N/256, l, 2)
__global__ void k_rescale_lift(const uint64_t* __restrict__ v, uint64_t* __restrict__ w, DevTables dt, int level,
                               int logN) {
  const size_t N = (size_t)1 << logN;
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y, p = blockIdx.z;
  const uint64_t ql = dt.pc[level].q, qi = dt.pc[i].q;
  uint64_t val = v[(size_t)p * N + x];
  uint64_t r;
  if (val > (ql - 1) / 2) {  // negative representative val - ql
    uint64_t m = reduce64(ql - val, dt.pc[i]);
    r = m ? qi - m : 0;
  } else {
    r = reduce64(val, dt.pc[i]);
  }
  w[((size_t)p * level + i) * N + x] = r;
}

// Rescale step 4: out[p][i] = (c[p][i] - w[p][i]) * q_l^{-1}.  grid (N/256, l, 2)
__global__ void k_rescale_final(const uint64_t* __restrict__ ct, const uint64_t* __restrict__ w,
                                const RescaleConst* rc, DevTables dt, int level, uint64_t* __restrict__ out,
                                int logN) {
  const size_t N = (size_t)1 << logN;
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y, p = blockIdx.z;
  const uint64_t q = dt.pc[i].q;
  uint64_t v = sub_mod(ct[((size_t)p * (level + 1) + i) * N + x], w[((size_t)p * level + i) * N + x], q);
  out[((size_t)p * level + i) * N + x] = shoup(v, rc->ql_inv[i], rc->ql_inv_sh[i], q);
}

// small signed values (int8 or int32 source) to residues on chain limbs [0, nlimb).  grid (N/256, nlimb)
template <class T>
__global__ void k_small_to_limbs(const T* __restrict__ v, uint64_t* __restrict__ out, const uint8_t* chain_map,
                                 DevTables dt, int logN) {
  const size_t N = (size_t)1 << logN;
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  const int t = chain_map ? chain_map[blockIdx.y] : blockIdx.y;
  const uint64_t q = dt.pc[t].q;
  const int64_t s = (int64_t)v[x];
  uint64_t r;
  if (s >= 0) {
    r = reduce64((uint64_t)s, dt.pc[t]);
  } else {
    const uint64_t m = reduce64((uint64_t)(-s), dt.pc[t]);
    r = m ? q - m : 0;
  }
  out[(size_t)blockIdx.y * N + x] = r;
}

// CBD(21) error polynomial (coefficient domain).  grid N/256
__global__ void k_sample_cbd(uint64_t seed, uint32_t dom, uint64_t obj, int32_t* __restrict__ e) {
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  e[x] = cbd21(draw(seed, dom, obj, 0, x));
}

// Rotation-key digit j: a = uniform (NTT domain) written to evk[j][1],
// b = -a*s + e + g_j*kappa(s) written to evk[j][0].  grid (N/256, n_q+n_p)
__global__ void k_evk_digit(uint64_t* __restrict__ evk, const uint64_t* __restrict__ s_ntt,
                            const uint64_t* __restrict__ sk_ntt, const uint64_t* __restrict__ e_ntt, uint64_t seed,
                            uint64_t obj, const uint64_t* __restrict__ gmod, int j, int L1, DevTables dt, int logN) {
  const size_t N = (size_t)1 << logN;
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  const int t = blockIdx.y;
  const PrimeConst& pc = dt.pc[t];
  const size_t o = (size_t)t * N + x;
  const uint64_t a = uniform_mod(draw(seed, kDomEvkA, obj, (uint32_t)t, x), pc.q);
  uint64_t b = sub_mod(e_ntt[o], mul_mod(a, s_ntt[o], pc), pc.q);
  if (gmod[t]) b = add_mod(b, mul_mod(gmod[t], sk_ntt[o], pc), pc.q);
  evk[((size_t)(j * 2 + 1) * L1 + t) * N + x] = a;
  evk[((size_t)(j * 2 + 0) * L1 + t) * N + x] = b;
}

// Encryption: c1 = a (uniform, NTT domain), c0 = -a*s + e + m.  grid (N/256, l+1)
__global__ void k_encrypt(const uint64_t* __restrict__ m, const uint64_t* __restrict__ s_ntt,
                          const uint64_t* __restrict__ e_ntt, uint64_t seed, uint64_t ct_id, uint64_t* __restrict__ ct,
                          DevTables dt, int level, int logN) {
  const size_t N = (size_t)1 << logN;
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  const PrimeConst& pc = dt.pc[i];
  const size_t o = (size_t)i * N + x;
  const uint64_t a = uniform_mod(draw(seed, kDomEncA, ct_id, (uint32_t)i, x), pc.q);
  uint64_t c0 = sub_mod(e_ntt[o], mul_mod(a, s_ntt[o], pc), pc.q);
  c0 = add_mod(c0, m[o], pc.q);
  ct[o] = c0;
  ct[(size_t)(level + 1) * N + o] = a;
}

// m = c0 + c1 * s.  grid (N/256, l+1)
__global__ void k_decrypt(const uint64_t* __restrict__ ct, const uint64_t* __restrict__ s_ntt,
                          uint64_t* __restrict__ m, DevTables dt, int level, int logN) {
  const size_t N = (size_t)1 << logN;
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  const PrimeConst& pc = dt.pc[i];
  const size_t o = (size_t)i * N + x;
  m[o] = add_mod(ct[o], mul_mod(ct[(size_t)(level + 1) * N + o], s_ntt[o], pc), pc.q);
}

// HWT secret (DESIGN R-SK), host side: partial Fisher-Yates over Philox draws.
void sample_secret(uint64_t seed, uint32_t N, uint32_t h, std::vector<int8_t>& s) {
  std::vector<uint32_t> idx(N);
  for (uint32_t i = 0; i < N; ++i) idx[i] = i;
  s.assign(N, 0);
  for (uint32_t t = 0; t < h && t < N; ++t) {
    Philox4 w = draw(seed, kDomSecret, 0, 0, t);
    uint64_t u = ((uint64_t)w.v[1] << 32) | w.v[0];
    uint32_t j = t + (uint32_t)(u % (N - t));
    std::swap(idx[t], idx[j]);
    s[idx[t]] = (w.v[2] & 1) ? -1 : 1;
  }
}

// s in the NTT domain on chain limbs 0..nlimb-1 (or a chain map), into out [nlimb][N].
hy_status secret_ntt(hy_ctx* c, uint64_t seed, uint32_t nlimb, uint64_t* out, int8_t* d_s, cudaStream_t s) {
  std::vector<int8_t> h_s;
  sample_secret(seed, c->N, c->h, h_s);
  cudaMemcpyAsync(d_s, h_s.data(), c->N, cudaMemcpyHostToDevice, s);
  cudaStreamSynchronize(s);  // h_s is a pageable temporary
  dim3 g(c->N / kT, nlimb);
  {
    KTimer kt(c, FAM_CLIENT, s);
    k_small_to_limbs<int8_t><<<g, kT, 0, s>>>(d_s, out, nullptr, c->dt, c->log_n);
  }
  std::vector<uint32_t> chain(nlimb);
  for (uint32_t i = 0; i < nlimb; ++i) chain[i] = i;
  ntt_contig(c, out, out, chain.data(), nlimb, false, s);
  return HY_OK;
}

}  // namespace
}  // namespace hy

using namespace hy;

namespace hy {
// out (+)= sum_i ct_i (.) PRot_{k_i}(pt_i)   (k_i = Galois element, 1 = no rotation)
hy_status pmult_acc_prot(hy_ctx* c, const uint64_t* const* cts, const uint64_t* const* pts, const uint64_t* ks,
                         uint32_t n, uint32_t level, uint64_t* out, int accumulate, void* stream) {
  if (!c || !cts || !pts || !out) return fail(HY_E_ARG, "null");
  if (level >= c->n_q) return fail(HY_E_ARG, "level out of range");
  if (n == 0 && !accumulate) return fail(HY_E_ARG, "empty product sum");
  cudaStream_t s = st(stream);
  for (uint32_t done = 0; done < n || (n == 0 && done == 0);) {
    uint32_t m = std::min<uint32_t>(n - done, kMaxTerms);
    if (m == 0) break;
    TermPtrs tp;
    for (uint32_t i = 0; i < m; ++i) {
      tp.ct[i] = cts[done + i];
      tp.pt[i] = pts[done + i];
      tp.prot[i] = ks ? ks[done + i] : 1;
      if (!tp.ct[i] || !tp.pt[i]) return fail(HY_E_ARG, "null term");
    }
    dim3 g(c->N / kT, level + 1, 2);
    KTimer kt(c, FAM_ELEM, s);
    kt.bytes = ((uint64_t)m * 3 * (level + 1) + 2ull * (level + 1) * ((accumulate || done > 0) ? 2 : 1)) * c->N * 8;
    k_pmult_acc<<<g, kT, 0, s>>>(tp, (int)m, out, c->dt, level, c->log_n, (accumulate || done > 0) ? 1 : 0);
    done += m;
  }
  return cuda_check("hy_pmult_acc");
}
}  // namespace hy

extern "C" hy_status hy_pmult_acc(hy_ctx* c, const uint64_t* const* cts, const uint64_t* const* pts, uint32_t n,
                                  uint32_t level, uint64_t* out, int accumulate, void* stream) {
  return hy::pmult_acc_prot(c, cts, pts, nullptr, n, level, out, accumulate, stream);
}

extern "C" hy_status hy_pmult(hy_ctx* c, const uint64_t* ct, const uint64_t* pt, uint32_t level, uint64_t* out,
                              void* stream) {
  const uint64_t* a[1] = {ct};
  const uint64_t* b[1] = {pt};
  return hy_pmult_acc(c, a, b, 1, level, out, 0, stream);
}

extern "C" hy_status hy_add(hy_ctx* c, const uint64_t* a, const uint64_t* b, uint32_t npoly, uint32_t level,
                            uint64_t* out, void* stream) {
  if (!c || !a || !b || !out) return fail(HY_E_ARG, "null");
  if (level >= c->n_q || npoly == 0) return fail(HY_E_ARG, "level/npoly out of range");
  dim3 g(c->N / kT, (level + 1) * npoly);
  KTimer kt(c, FAM_ELEM, st(stream));
  kt.bytes = 3ull * (level + 1) * npoly * c->N * 8;
  k_add<<<g, kT, 0, st(stream)>>>(a, b, out, c->dt, level + 1, c->log_n);
  return cuda_check("hy_add");
}

extern "C" hy_status hy_rescale(hy_ctx* c, const uint64_t* ct, uint32_t level, uint64_t* out, void* stream) {
  if (!c || !ct || !out) return fail(HY_E_ARG, "null");
  if (level >= c->n_q) return fail(HY_E_ARG, "level out of range");
  if (level == 0) return fail(HY_E_LEVEL_EXHAUSTED, "rescale at level 0");
  if (!c->ws) return fail(HY_E_WORKSPACE, "workspace not set");
  cudaStream_t s = st(stream);
  const size_t N = c->N, n = level + 1;
  Ws ws{c->ws, c->ws_bytes};
  uint64_t* v = ws.take<uint64_t>(2 * N);
  uint64_t* w = ws.take<uint64_t>(2 * level * N);
  if (!w) return fail(HY_E_WORKSPACE, "workspace too small");
  LimbBatch b;
  b.n = 2;
  for (int p = 0; p < 2; ++p) {
    b.src[p] = ct + ((size_t)p * n + level) * N;
    b.dst[p] = v + (size_t)p * N;
    b.chain[p] = (uint8_t)level;
  }
  launch_ntt(c, b, true, s);
  dim3 g(c->N / kT, level, 2);
  {
    KTimer kt(c, FAM_RESCALE, s);
    k_rescale_lift<<<g, kT, 0, s>>>(v, w, c->dt, level, c->log_n);
  }
  b.n = 0;
  for (int p = 0; p < 2; ++p)
    for (uint32_t i = 0; i < level; ++i) {
      uint64_t* q = w + ((size_t)p * level + i) * N;
      b.src[b.n] = q;
      b.dst[b.n] = q;
      b.chain[b.n] = (uint8_t)i;
      ++b.n;
    }
  launch_ntt(c, b, false, s);
  {
    KTimer kt(c, FAM_RESCALE, s);
    k_rescale_final<<<g, kT, 0, s>>>(ct, w, c->d_rescale[level], c->dt, level, out, c->log_n);
  }
  return cuda_check("hy_rescale");
}

extern "C" hy_status hy_keygen_galois(hy_ctx* c, uint64_t sk_seed, uint64_t ek_seed, uint64_t k, uint64_t* evk,
                                      void* stream) {
  if (!c || !evk) return fail(HY_E_ARG, "null");
  if (!(k & 1) || k >= 2ull * c->N) return fail(HY_E_ARG, "bad Galois element");
  if (!c->ws) return fail(HY_E_WORKSPACE, "workspace not set");
  cudaStream_t s = st(stream);
  const uint32_t L1 = c->n_q + c->n_p;
  const size_t N = c->N;
  Ws ws{c->ws, c->ws_bytes};
  uint64_t* s_ntt = ws.take<uint64_t>(L1 * N);
  uint64_t* sk_ntt = ws.take<uint64_t>(L1 * N);
  uint64_t* e_ntt = ws.take<uint64_t>(L1 * N);
  int32_t* e = ws.take<int32_t>(N);
  int8_t* d_s = ws.take<int8_t>(N);
  uint64_t* gm = ws.take<uint64_t>(kMaxChain);
  if (!gm) return fail(HY_E_WORKSPACE, "workspace too small for key generation");
  secret_ntt(c, sk_seed, L1, s_ntt, d_s, s);
  launch_automorph(c, s_ntt, sk_ntt, L1, k, s);  // kappa_k(s): NTT-domain permutation
  std::vector<uint32_t> chain(L1);
  for (uint32_t i = 0; i < L1; ++i) chain[i] = i;
  std::vector<uint64_t> g(L1);
  for (uint32_t j = 0; j < c->dnum; ++j) {
    const uint64_t obj = (k << 8) | j;
    dim3 gg(c->N / kT, L1);
    {
      KTimer kt(c, FAM_CLIENT, s, 2);
      k_sample_cbd<<<c->N / kT, kT, 0, s>>>(ek_seed, kDomEvkE, obj, e);
      k_small_to_limbs<int32_t><<<gg, kT, 0, s>>>(e, e_ntt, nullptr, c->dt, c->log_n);
    }
    ntt_contig(c, e_ntt, e_ntt, chain.data(), L1, false, s);
    // g_j = P on the q-limbs of digit j, 0 elsewhere (DESIGN R-EVK)
    for (uint32_t t = 0; t < L1; ++t) {
      g[t] = 0;
      if (t < c->n_q && t >= j * c->alpha && t < (j + 1) * c->alpha) {
        const uint64_t qt = c->mod[t];
        uint64_t v = 1;
        for (uint32_t kk = 0; kk < c->n_p; ++kk) v = (uint64_t)((unsigned __int128)v * (c->mod[c->n_q + kk] % qt) % qt);
        g[t] = v;
      }
    }
    cudaMemcpyAsync(gm, g.data(), L1 * 8, cudaMemcpyHostToDevice, s);
    {
      KTimer kt(c, FAM_CLIENT, s);
      k_evk_digit<<<gg, kT, 0, s>>>(evk, s_ntt, sk_ntt, e_ntt, ek_seed, obj, gm, (int)j, (int)L1, c->dt, c->log_n);
    }
    cudaStreamSynchronize(s);  // g is reused on the host
  }
  return cuda_check("hy_keygen_galois");
}

extern "C" hy_status hy_keygen_rot(hy_ctx* c, uint64_t sk_seed, uint64_t ek_seed, int32_t r, uint64_t* evk,
                                   void* stream) {
  if (!c) return fail(HY_E_ARG, "null");
  return hy_keygen_galois(c, sk_seed, ek_seed, hy_galois_elt(c, r), evk, stream);
}

extern "C" hy_status hy_encrypt(hy_ctx* c, uint64_t sk_seed, uint64_t enc_seed, uint64_t ct_id, const uint64_t* pt,
                                uint32_t level, uint64_t* ct, void* stream) {
  if (!c || !pt || !ct) return fail(HY_E_ARG, "null");
  if (level >= c->n_q) return fail(HY_E_ARG, "level out of range");
  if (!c->ws) return fail(HY_E_WORKSPACE, "workspace not set");
  cudaStream_t s = st(stream);
  const size_t N = c->N, n = level + 1;
  Ws ws{c->ws, c->ws_bytes};
  uint64_t* s_ntt = ws.take<uint64_t>(n * N);
  uint64_t* e_ntt = ws.take<uint64_t>(n * N);
  int32_t* e = ws.take<int32_t>(N);
  int8_t* d_s = ws.take<int8_t>(N);
  if (!d_s) return fail(HY_E_WORKSPACE, "workspace too small");
  secret_ntt(c, sk_seed, n, s_ntt, d_s, s);
  dim3 g(c->N / kT, n);
  {
    KTimer kt(c, FAM_CLIENT, s, 2);
    k_sample_cbd<<<c->N / kT, kT, 0, s>>>(enc_seed, kDomEncE, ct_id, e);
    k_small_to_limbs<int32_t><<<g, kT, 0, s>>>(e, e_ntt, nullptr, c->dt, c->log_n);
  }
  std::vector<uint32_t> chain(n);
  for (uint32_t i = 0; i < n; ++i) chain[i] = i;
  ntt_contig(c, e_ntt, e_ntt, chain.data(), n, false, s);
  KTimer kt(c, FAM_CLIENT, s);
  k_encrypt<<<g, kT, 0, s>>>(pt, s_ntt, e_ntt, enc_seed, ct_id, ct, c->dt, level, c->log_n);
  return cuda_check("hy_encrypt");
}

extern "C" hy_status hy_decrypt(hy_ctx* c, uint64_t sk_seed, const uint64_t* ct, uint32_t level, uint64_t* pt,
                                void* stream) {
  if (!c || !pt || !ct) return fail(HY_E_ARG, "null");
  if (level >= c->n_q) return fail(HY_E_ARG, "level out of range");
  if (!c->ws) return fail(HY_E_WORKSPACE, "workspace not set");
  cudaStream_t s = st(stream);
  const size_t N = c->N, n = level + 1;
  Ws ws{c->ws, c->ws_bytes};
  uint64_t* s_ntt = ws.take<uint64_t>(n * N);
  int8_t* d_s = ws.take<int8_t>(N);
  if (!d_s) return fail(HY_E_WORKSPACE, "workspace too small");
  secret_ntt(c, sk_seed, n, s_ntt, d_s, s);
  dim3 g(c->N / kT, n);
  KTimer kt(c, FAM_CLIENT, s);
  k_decrypt<<<g, kT, 0, s>>>(ct, s_ntt, pt, c->dt, level, c->log_n);
  return cuda_check("hy_decrypt");
}

extern "C" hy_status hy_pt_from_coeffs(hy_ctx* c, const int64_t* h_coeffs, uint32_t level, uint64_t* pt,
                                       void* stream) {
  if (!c || !h_coeffs || !pt) return fail(HY_E_ARG, "null");
  if (level >= c->n_q) return fail(HY_E_ARG, "level out of range");
  if (!c->ws) return fail(HY_E_WORKSPACE, "workspace not set");
  cudaStream_t s = st(stream);
  Ws ws{c->ws, c->ws_bytes};
  int64_t* d = ws.take<int64_t>(c->N);
  if (!d) return fail(HY_E_WORKSPACE, "workspace too small");
  cudaMemcpyAsync(d, h_coeffs, c->N * 8, cudaMemcpyHostToDevice, s);
  const uint32_t n = level + 1;
  dim3 g(c->N / kT, n);
  {
    KTimer kt(c, FAM_CLIENT, s);
    k_small_to_limbs<int64_t><<<g, kT, 0, s>>>(d, pt, nullptr, c->dt, c->log_n);
  }
  std::vector<uint32_t> chain(n);
  for (uint32_t i = 0; i < n; ++i) chain[i] = i;
  ntt_contig(c, pt, pt, chain.data(), n, false, s);
  cudaStreamSynchronize(s);  // h_coeffs may be pageable and reused by the caller
  return cuda_check("hy_pt_from_coeffs");
}

extern "C" hy_status hy_encode(hy_ctx* c, const double* h_slots, uint32_t n_slots, uint64_t scale, uint32_t level,
                               uint64_t* pt, void* stream) {
  if (!c) return fail(HY_E_ARG, "null");
  std::vector<int64_t> coeffs(c->N);
  hy_status s0 = hy_encode_coeffs(c->log_n, h_slots, n_slots, scale, coeffs.data());
  if (s0 != HY_OK) return s0;
  return hy_pt_from_coeffs(c, coeffs.data(), level, pt, stream);
}
