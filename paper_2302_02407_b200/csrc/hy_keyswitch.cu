// hy_keyswitch.cu -- automorphism, ModUp, key-switch inner product, ModDown and
// the three HRot variants (DESIGN R-HROT).
//
// HRot_r (left rotation by r) with Galois element k = 5^r mod 2N:
//   plain   : c' = kappa(c); d = iNTT(c'_1); ModUp(d) -> IP(evk_k) -> ModDown; out_0 += c'_0
//   hoisted : d = iNTT(c_1) once; ModUp once; per r the IP reads the extended
//             digits through the NTT-domain permutation of kappa_k (Halevi-Shoup)
//   lazy sum: per term plain ModUp + IP accumulated over Q_l u P; ONE ModDown.
// Data layout (HBM): ct [2][l+1][N], ext [beta][l+1+K][N], u [2][l+1+K][N], evk
// [dnum][2][n_q+n_p][N]; every limb is N contiguous uint64 (coalesced rows).
#include <algorithm>

#include "hy_arith.cuh"

namespace hy {

// NTT-domain index permutation of kappa_k: out[p] = in[perm(p)],
// 2 br(perm(p)) + 1 = (2 br(p) + 1) k mod 2N.
__device__ __forceinline__ uint32_t aut_index(uint32_t p, uint64_t k, int logN) {
  uint32_t e = 2 * bitrev32(p, logN) + 1;
  uint32_t e2 = (uint32_t)(((uint64_t)e * k) & ((2ull << logN) - 1));
  return bitrev32((e2 - 1) >> 1, logN);
}

namespace {

constexpr int kT = 256;

// IP operands: digit j's limb u is own[u] (the NTT-domain c1 the digits were
// cut from) when u belongs to digit j, else ext[j][u].
struct IPArgs {
  const uint64_t* ext;
  const uint64_t* own;  // may be null: then every limb comes from ext
};

// out[l][p] (+)= in[l][perm_k(p)]; limb l uses prime chain (l % limbs_per_poly).
__global__ void k_automorph(const uint64_t* __restrict__ in, uint64_t* __restrict__ out, uint64_t k, int logN,
                            int limbs_per_poly, int accumulate, DevTables dt) {
  const size_t N = (size_t)1 << logN;
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  const size_t off = (size_t)blockIdx.y * N;
  uint64_t v = in[off + aut_index(p, k, logN)];
  if (accumulate) v = add_mod(v, out[off + p], dt.pc[blockIdx.y % limbs_per_poly].q);
  out[off + p] = v;
}

// FP64 constants of one prime, staged in shared memory.
struct FConst {
  double q, qinv;
};

// ModUp basis conversion for digit j = blockIdx.y; one thread per coefficient x
// produces every non-own limb of the digit.  grid (N/256, beta).
// y_i = [d_i (D_j/q_i)^{-1}]_{q_i} in [0, q_i);  ext[j][u][x] = [sum_i y_i ((D_j/q_i) mod t_u)]_{t_u}.
// Every product is reduced on the FP64 pipe (fmulmod, |term| <= 1.5 t), the A terms are summed
// exactly and canonicalised once.  A = alpha (compile time); a partial last digit pads with 0.
template <int A>
__global__ void __launch_bounds__(256) k_modup_bconv(const uint64_t* __restrict__ d, uint64_t* __restrict__ ext,
                                                     const ModUpConst* mc, DevTables dt, int level, int n_q, int E,
                                                     int logN) {
  __shared__ double s_hat[kMaxExt][A];
  __shared__ FConst s_fc[kMaxExt];
  const size_t N = (size_t)1 << logN;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  const ModUpConst& m = mc[j];
  const int nsrc = m.hi - m.lo;
  for (int i = threadIdx.x; i < E * A; i += blockDim.x) {
    const int u = i / A, ii = i % A;
    s_hat[u][ii] = ii < nsrc ? (double)m.hat_mod[u][ii] : 0.0;
  }
  for (int u = threadIdx.x; u < E; u += blockDim.x) {
    const PrimeConst& pc = dt.pc[u <= level ? u : n_q + (u - level - 1)];
    s_fc[u] = FConst{pc.qd, pc.qinv};
  }
  double y[A];
#pragma unroll
  for (int i = 0; i < A; ++i) {
    if (i < nsrc) {
      const PrimeConst& pc = dt.pc[m.lo + i];
      y[i] = fcanon(fmulmod(u2d(d[(size_t)(m.lo + i) * N + x]), (double)m.hat_inv[i], pc.qd, pc.qinv), pc.qd,
                    pc.qinv);
    } else {
      y[i] = 0.0;
    }
  }
  __syncthreads();
  uint64_t* out = ext + (size_t)j * E * N + x;
  for (int u = 0; u < E; ++u) {
    if (u >= m.lo && u < m.hi) continue;
    const FConst f = s_fc[u];
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < A; ++i) acc += fmulmod(y[i], s_hat[u][i], f.q, f.qinv);
    out[(size_t)u * N] = d2u(fcanon(acc, f.q, f.qinv));
  }
}

// Key-switch inner product, B = beta digits (compile time).  grid (N/256, E).
// u[c][u][x] (+)= sum_j src_j[u][perm(x)] * evk[j][c][chain(u)][x], where src_j[u] is the digit's own
// limb of `own` (the NTT-domain c1 the digits were cut from) when u belongs to digit j, else ext[j][u].
// Products reduced on the FP64 pipe, summed exactly (|sum| <= 1.5 B t < 2^51), canonicalised once.
template <int B>
__global__ void __launch_bounds__(256) k_ks_ip(const uint64_t* __restrict__ ext, const uint64_t* __restrict__ own,
                                               const uint64_t* __restrict__ evk, uint64_t* __restrict__ uo,
                                               DevTables dt, int level, int n_q, int L1, int E, int alpha,
                                               uint64_t kperm, int logN, int accumulate) {
  const size_t N = (size_t)1 << logN;
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  const int u = blockIdx.y;
  const int t = u <= level ? u : n_q + (u - level - 1);
  const PrimeConst& p = dt.pc[t];
  const double q = p.qd, qinv = p.qinv;
  const uint32_t xs = kperm != 1 ? aut_index(x, kperm, logN) : x;
  const int own_digit = (own && u <= level) ? u / alpha : -1;
  uint64_t v[B], e0[B], e1[B];
#pragma unroll
  for (int j = 0; j < B; ++j) {
    const uint64_t* src = (j == own_digit) ? own + (size_t)u * N : ext + ((size_t)j * E + u) * N;
    v[j] = src[xs];
    const uint64_t* e = evk + ((size_t)(j * 2) * L1 + t) * N + x;
    e0[j] = __ldcs(e);
    e1[j] = __ldcs(e + (size_t)L1 * N);
  }
  double a0 = 0.0, a1 = 0.0;
#pragma unroll
  for (int j = 0; j < B; ++j) {
    const double vj = u2d(v[j]);
    a0 += fmulmod(vj, u2d(e0[j]), q, qinv);
    a1 += fmulmod(vj, u2d(e1[j]), q, qinv);
  }
  uint64_t* o0 = uo + (size_t)u * N + x;
  uint64_t* o1 = uo + ((size_t)E + u) * N + x;
  if (accumulate) {
    a0 += u2d(*o0);
    a1 += u2d(*o1);
  }
  *o0 = d2u(fcanon(a0, q, qinv));
  *o1 = d2u(fcanon(a1, q, qinv));
}

// ModDown basis conversion P -> Q_l, KP = K special primes (compile time).  grid (N/256, npoly);
// v = iNTT(u on P) [npoly][K][N];  z_k = [v_k (P/p_k)^{-1}]_{p_k} in [0, p_k);
// w[c][i] = [sum_k z_k ((P/p_k) mod q_i)]_{q_i}.
template <int KP>
__global__ void __launch_bounds__(256) k_moddown_bconv(const uint64_t* __restrict__ v, uint64_t* __restrict__ w,
                                                       const ModDownConst* md, DevTables dt, int level, int n_q,
                                                       int logN) {
  __shared__ double s_hat[kMaxChain][KP];
  __shared__ FConst s_fc[kMaxChain];
  const size_t N = (size_t)1 << logN;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  const int n = level + 1;
  for (int i = threadIdx.x; i < n * KP; i += blockDim.x) s_hat[i / KP][i % KP] = (double)md->phat_mod[i / KP][i % KP];
  for (int i = threadIdx.x; i < n; i += blockDim.x) s_fc[i] = FConst{dt.pc[i].qd, dt.pc[i].qinv};
  double z[KP];
#pragma unroll
  for (int k = 0; k < KP; ++k) {
    const PrimeConst& pc = dt.pc[n_q + k];
    z[k] = fcanon(fmulmod(u2d(v[((size_t)c * KP + k) * N + x]), (double)md->phat_inv[k], pc.qd, pc.qinv), pc.qd,
                  pc.qinv);
  }
  __syncthreads();
  uint64_t* out = w + (size_t)c * n * N + x;
  for (int i = 0; i < n; ++i) {
    const FConst f = s_fc[i];
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < KP; ++k) acc += fmulmod(z[k], s_hat[i][k], f.q, f.qinv);
    out[(size_t)i * N] = d2u(fcanon(acc, f.q, f.qinv));
  }
}

#define HY_DISPATCH_1_8(KERNEL, VAL, GRID, BLOCK, STREAM, ...)                      \
  switch (VAL) {                                                                     \
    case 1: KERNEL<1><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__); break;               \
    case 2: KERNEL<2><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__); break;               \
    case 3: KERNEL<3><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__); break;               \
    case 4: KERNEL<4><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__); break;               \
    case 5: KERNEL<5><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__); break;               \
    case 6: KERNEL<6><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__); break;               \
    case 7: KERNEL<7><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__); break;               \
    default: KERNEL<8><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__); break;              \
  }

// out[c][i] = (u[c][i] - w[c][i]) P^{-1} (+ add0[i][perm(x)] for c = 0) (+ add1[i][x] for c = 1)
//             (+ addct[c][i][x] for both polys).  out may alias addct (read before write, same x).
// grid (N/256, l+1, npoly)
__global__ void k_moddown_final(const uint64_t* __restrict__ u, int E, const uint64_t* __restrict__ w,
                                const ModDownConst* md, DevTables dt, int level, uint64_t* out,
                                const uint64_t* __restrict__ add0, uint64_t k0, const uint64_t* __restrict__ add1,
                                const uint64_t* addct, int logN) {
  const size_t N = (size_t)1 << logN;
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y, c = blockIdx.z;
  const uint64_t q = dt.pc[i].q;
  uint64_t val = sub_mod(u[((size_t)c * E + i) * N + x], w[((size_t)c * (level + 1) + i) * N + x], q);
  val = shoup(val, md->p_inv[i], md->p_inv_sh[i], q);
  if (c == 0 && add0) {
    const uint32_t xs = k0 != 1 ? aut_index(x, k0, logN) : x;
    val = add_mod(val, add0[(size_t)i * N + xs], q);
  }
  if (c == 1 && add1) val = add_mod(val, add1[(size_t)i * N + x], q);
  const size_t o = ((size_t)c * (level + 1) + i) * N + x;
  if (addct) val = add_mod(val, addct[o], q);
  out[o] = val;
}

// ---------------------------------------------------------------- host-side building blocks
struct KsBufs {
  uint64_t *rc, *d, *ext, *u, *v, *w, *acc;
};

hy_status carve(hy_ctx* c, uint32_t level, KsBufs& b) {
  if (!c->ws) return fail(HY_E_WORKSPACE, "workspace not set (hy_ctx_set_workspace)");
  const size_t N = c->N, n = level + 1, E = n + c->n_p, beta = n_digits(c, level);
  Ws ws{c->ws, c->ws_bytes};
  b.rc = ws.take<uint64_t>(2 * n * N);
  b.d = ws.take<uint64_t>(n * N);
  b.ext = ws.take<uint64_t>(beta * E * N);
  b.u = ws.take<uint64_t>(2 * E * N);
  b.v = ws.take<uint64_t>(2 * c->n_p * N);
  b.w = ws.take<uint64_t>(2 * n * N);
  b.acc = ws.take<uint64_t>(2 * n * N);
  if (!b.acc) return fail(HY_E_WORKSPACE, "workspace too small for this level");
  return HY_OK;
}

void automorph(hy_ctx* c, const uint64_t* in, uint64_t* out, uint32_t nlimbs, uint32_t per_poly, uint64_t k,
               bool accumulate, cudaStream_t s) {
  dim3 g(c->N / kT, nlimbs);
  KTimer kt(c, FAM_AUT, s);
  kt.bytes = (uint64_t)nlimbs * c->N * 8 * (accumulate ? 3 : 2);
  k_automorph<<<g, kT, 0, s>>>(in, out, k, c->log_n, per_poly, accumulate ? 1 : 0, c->dt);
}

// d: coefficient-domain [l+1][N] -> ext [beta][E][N] (non-own limbs, NTT domain)
void modup_core(hy_ctx* c, uint32_t level, const uint64_t* d, uint64_t* ext, cudaStream_t s) {
  const int n = level + 1, E = n + c->n_p, beta = n_digits(c, level);
  dim3 g(c->N / kT, beta);
  {
    KTimer kt(c, FAM_MODUP, s);
    kt.bytes = ((uint64_t)n + (uint64_t)beta * E - n) * c->N * 8;  // read d once, write non-own ext limbs
    HY_DISPATCH_1_8(k_modup_bconv, c->alpha, g, kT, s, d, ext, c->d_modup[level], c->dt, (int)level, (int)c->n_q, E,
                    (int)c->log_n);
  }
  LimbBatch b;
  b.n = 0;
  for (int j = 0; j < beta; ++j) {
    const auto& m = c->h_modup[level][j];
    for (int u = 0; u < E; ++u) {
      if (u >= m.lo && u < m.hi) continue;
      if (b.n == kMaxBatch) {
        launch_ntt(c, b, false, s);
        b.n = 0;
      }
      uint64_t* p = ext + ((size_t)j * E + u) * c->N;
      b.src[b.n] = p;
      b.dst[b.n] = p;
      b.chain[b.n] = (uint8_t)ext_chain(c, level, u);
      ++b.n;
    }
  }
  launch_ntt(c, b, false, s);
}

IPArgs ip_args(hy_ctx*, uint32_t, const uint64_t* ext, const uint64_t* own /* c1 NTT, or null */) {
  return IPArgs{ext, own};
}

void ip(hy_ctx* c, uint32_t level, const IPArgs& a, const uint64_t* evk, uint64_t* u, uint64_t kperm, bool acc,
        cudaStream_t s) {
  const int n = level + 1, E = n + c->n_p, beta = n_digits(c, level);
  dim3 g(c->N / kT, E);
  KTimer kt(c, FAM_IP, s);
  kt.bytes = ((uint64_t)beta * E * 3 + 2ull * E * (acc ? 2 : 1)) * c->N * 8;  // ext + 2 evk polys in, u out
  HY_DISPATCH_1_8(k_ks_ip, beta, g, kT, s, a.ext, a.own, evk, u, c->dt, (int)level, (int)c->n_q,
                  (int)(c->n_q + c->n_p), E, (int)c->alpha, kperm, (int)c->log_n, acc ? 1 : 0);
}

// u [npoly][E][N] (NTT) -> out [npoly][l+1][N]
void moddown_core(hy_ctx* c, uint32_t level, int npoly, const uint64_t* u, uint64_t* out, const uint64_t* add0,
                  uint64_t k0, const uint64_t* add1, uint64_t* v, uint64_t* w, cudaStream_t s,
                  const uint64_t* addct = nullptr) {
  const int n = level + 1, E = n + c->n_p, K = c->n_p;
  LimbBatch b;
  b.n = 0;
  for (int cc = 0; cc < npoly; ++cc)
    for (int k = 0; k < K; ++k) {
      b.src[b.n] = u + ((size_t)cc * E + n + k) * c->N;
      b.dst[b.n] = v + ((size_t)cc * K + k) * c->N;
      b.chain[b.n] = (uint8_t)(c->n_q + k);
      ++b.n;
    }
  launch_ntt(c, b, true, s);
  dim3 g(c->N / kT, npoly);
  {
    KTimer kt(c, FAM_MODDOWN, s);
    kt.bytes = ((uint64_t)npoly * K + (uint64_t)npoly * n) * c->N * 8;
    HY_DISPATCH_1_8(k_moddown_bconv, K, g, kT, s, v, w, c->d_moddown[level], c->dt, (int)level, (int)c->n_q,
                    (int)c->log_n);
  }
  b.n = 0;
  for (int cc = 0; cc < npoly; ++cc)
    for (int i = 0; i < n; ++i) {
      uint64_t* p = w + ((size_t)cc * n + i) * c->N;
      b.src[b.n] = p;
      b.dst[b.n] = p;
      b.chain[b.n] = (uint8_t)i;
      ++b.n;
    }
  launch_ntt(c, b, false, s);
  dim3 g2(c->N / kT, n, npoly);
  KTimer kt(c, FAM_MODDOWN, s);
  kt.bytes = ((uint64_t)npoly * n * (addct ? 4 : 3) + (add0 ? n : 0) + (add1 ? n : 0)) * c->N * 8;
  k_moddown_final<<<g2, kT, 0, s>>>(u, E, w, c->d_moddown[level], c->dt, level, out, add0, k0, add1, addct,
                                    c->log_n);
}

void intt_poly(hy_ctx* c, const uint64_t* in, uint64_t* out, uint32_t level, cudaStream_t s) {
  LimbBatch b;
  b.n = level + 1;
  for (uint32_t i = 0; i <= level; ++i) {
    b.src[i] = in + (size_t)i * c->N;
    b.dst[i] = out + (size_t)i * c->N;
    b.chain[i] = (uint8_t)i;
  }
  launch_ntt(c, b, true, s);
}

hy_status check_level(hy_ctx* c, uint32_t level) {
  if (!c) return fail(HY_E_ARG, "null ctx");
  if (level >= c->n_q) return fail(HY_E_ARG, "level out of range");
  return HY_OK;
}

}  // namespace

// out = HRot_r(ct) (+ addct).  out may alias addct (and ct, since ct is consumed into the
// workspace before the final write).
hy_status hrot_plain(hy_ctx* c, const uint64_t* evk, const uint64_t* ct, uint32_t level, int32_t r, uint64_t* out,
                     cudaStream_t s, const uint64_t* addct) {
  const uint64_t k = hy_galois_elt(c, r);
  const size_t n = level + 1, N = c->N;
  if (k == 1) {
    if (addct) {  // out = ct + addct
      if (out != addct) cudaMemcpyAsync(out, addct, 2 * n * N * 8, cudaMemcpyDeviceToDevice, s);
      automorph(c, ct, out, 2 * n, n, 1, true, s);
    } else if (out != ct) {
      cudaMemcpyAsync(out, ct, 2 * n * N * 8, cudaMemcpyDeviceToDevice, s);
    }
    return HY_OK;
  }
  if (!evk) return fail(HY_E_MISSING_KEY, "no evaluation key for rotation");
  KsBufs b;
  hy_status st = carve(c, level, b);
  if (st != HY_OK) return st;
  automorph(c, ct, b.rc, 2 * n, n, k, false, s);
  intt_poly(c, b.rc + n * N, b.d, level, s);
  modup_core(c, level, b.d, b.ext, s);
  IPArgs a = ip_args(c, level, b.ext, b.rc + n * N);
  ip(c, level, a, evk, b.u, 1, false, s);
  moddown_core(c, level, 2, b.u, out, b.rc, 1, nullptr, b.v, b.w, s, addct);
  return HY_OK;
}

namespace {
}  // namespace

void launch_automorph(hy_ctx* c, const uint64_t* in, uint64_t* out, uint32_t n_limbs, uint64_t k, cudaStream_t s) {
  automorph(c, in, out, n_limbs, n_limbs, k, false, s);
}

}  // namespace hy

using namespace hy;

extern "C" hy_status hy_automorph(hy_ctx* c, const uint64_t* in, uint64_t* out, uint32_t n_limbs, uint64_t k,
                                  void* stream) {
  if (!c || !in || !out) return fail(HY_E_ARG, "null");
  if (!(k & 1) || k >= 2ull * c->N) return fail(HY_E_ARG, "Galois element must be odd and < 2N");
  if (in == out) return fail(HY_E_ARG, "automorphism cannot run in place");
  automorph(c, in, out, n_limbs, 1, k, false, st(stream));
  return cuda_check("hy_automorph");
}

extern "C" hy_status hy_modup(hy_ctx* c, uint32_t level, const uint64_t* d, uint64_t* ext, void* stream) {
  hy_status s0 = check_level(c, level);
  if (s0 != HY_OK) return s0;
  if (!d || !ext) return fail(HY_E_ARG, "null");
  cudaStream_t s = st(stream);
  modup_core(c, level, d, ext, s);
  // own-digit limbs: NTT(d)
  const int E = level + 1 + c->n_p;
  LimbBatch b;
  b.n = 0;
  for (uint32_t j = 0; j < n_digits(c, level); ++j) {
    const auto& m = c->h_modup[level][j];
    for (int i = m.lo; i < m.hi; ++i) {
      b.src[b.n] = d + (size_t)i * c->N;
      b.dst[b.n] = ext + ((size_t)j * E + i) * c->N;
      b.chain[b.n] = (uint8_t)i;
      ++b.n;
    }
  }
  launch_ntt(c, b, false, s);
  return cuda_check("hy_modup");
}

extern "C" hy_status hy_ks_inner_product(hy_ctx* c, uint32_t level, const uint64_t* ext, const uint64_t* evk,
                                         uint64_t* u, void* stream) {
  hy_status s0 = check_level(c, level);
  if (s0 != HY_OK) return s0;
  if (!ext || !evk || !u) return fail(HY_E_ARG, "null");
  IPArgs a = ip_args(c, level, ext, nullptr);
  ip(c, level, a, evk, u, 1, false, st(stream));
  return cuda_check("hy_ks_inner_product");
}

extern "C" hy_status hy_moddown(hy_ctx* c, uint32_t level, const uint64_t* u, uint64_t* out, void* stream) {
  hy_status s0 = check_level(c, level);
  if (s0 != HY_OK) return s0;
  if (!u || !out) return fail(HY_E_ARG, "null");
  KsBufs b;
  hy_status st0 = carve(c, level, b);
  if (st0 != HY_OK) return st0;
  moddown_core(c, level, 1, u, out, nullptr, 1, nullptr, b.v, b.w, st(stream));
  return cuda_check("hy_moddown");
}

extern "C" hy_status hy_hrot(hy_ctx* c, const uint64_t* evk, const uint64_t* ct, uint32_t level, int32_t r,
                             uint64_t* out, void* stream) {
  hy_status s0 = check_level(c, level);
  if (s0 != HY_OK) return s0;
  if (!ct || !out) return fail(HY_E_ARG, "null");
  if (ct == out) return fail(HY_E_ARG, "hrot cannot run in place");
  s0 = hrot_plain(c, evk, ct, level, r, out, st(stream), nullptr);
  if (s0 != HY_OK) return s0;
  return cuda_check("hy_hrot");
}

extern "C" hy_status hy_hrot_batch(hy_ctx* c, const uint64_t* const* evks, const uint64_t* const* cts, uint32_t level,
                                   const int32_t* r, uint32_t n, uint64_t* const* outs, void* stream) {
  hy_status s0 = check_level(c, level);
  if (s0 != HY_OK) return s0;
  if (!evks || !cts || !r || !outs) return fail(HY_E_ARG, "null");
  for (uint32_t i = 0; i < n; ++i) {
    if (cts[i] == outs[i]) return fail(HY_E_ARG, "hrot cannot run in place");
    s0 = hrot_plain(c, evks[i], cts[i], level, r[i], outs[i], st(stream), nullptr);
    if (s0 != HY_OK) return s0;
  }
  return cuda_check("hy_hrot_batch");
}

extern "C" hy_status hy_hrot_hoisted(hy_ctx* c, const uint64_t* const* evks, const uint64_t* ct, uint32_t level,
                                     const int32_t* r, uint32_t n, uint64_t* const* outs, void* stream) {
  hy_status s0 = check_level(c, level);
  if (s0 != HY_OK) return s0;
  if (!evks || !ct || !r || !outs) return fail(HY_E_ARG, "null");
  cudaStream_t s = st(stream);
  const size_t nl = level + 1, N = c->N;
  KsBufs b;
  s0 = carve(c, level, b);
  if (s0 != HY_OK) return s0;
  bool need_ks = false;
  for (uint32_t i = 0; i < n; ++i) {
    if (outs[i] == ct) return fail(HY_E_ARG, "hrot cannot run in place");
    if (hy_galois_elt(c, r[i]) != 1) {
      need_ks = true;
      if (!evks[i]) return fail(HY_E_MISSING_KEY, "no evaluation key for rotation");
    }
  }
  if (need_ks) {
    intt_poly(c, ct + nl * N, b.d, level, s);
    modup_core(c, level, b.d, b.ext, s);
  }
  IPArgs a = ip_args(c, level, b.ext, ct + nl * N);
  for (uint32_t i = 0; i < n; ++i) {
    const uint64_t k = hy_galois_elt(c, r[i]);
    if (k == 1) {
      cudaMemcpyAsync(outs[i], ct, 2 * nl * N * 8, cudaMemcpyDeviceToDevice, s);
      continue;
    }
    ip(c, level, a, evks[i], b.u, k, false, s);
    moddown_core(c, level, 2, b.u, outs[i], ct, k, nullptr, b.v, b.w, s);
  }
  return cuda_check("hy_hrot_hoisted");
}

extern "C" hy_status hy_hrot_sum(hy_ctx* c, const uint64_t* const* evks, const uint64_t* const* cts, uint32_t level,
                                 const int32_t* r, uint32_t n, uint64_t* out, void* stream) {
  hy_status s0 = check_level(c, level);
  if (s0 != HY_OK) return s0;
  if (!evks || !cts || !r || !out || n == 0) return fail(HY_E_ARG, "null / empty");
  cudaStream_t s = st(stream);
  const size_t nl = level + 1, N = c->N;
  KsBufs b;
  s0 = carve(c, level, b);
  if (s0 != HY_OK) return s0;
  for (uint32_t t = 0; t < n; ++t) {
    if (cts[t] == out) return fail(HY_E_ARG, "output aliases an input");
    if (hy_galois_elt(c, r[t]) != 1 && !evks[t]) return fail(HY_E_MISSING_KEY, "no evaluation key for rotation");
  }
  uint64_t* acc0 = b.acc;          // sum of kappa(c0_t) and unrotated c0_t
  uint64_t* acc1 = b.acc + nl * N; // sum of unrotated c1_t
  cudaMemsetAsync(b.acc, 0, 2 * nl * N * 8, s);
  bool first = true, any1 = false;
  for (uint32_t t = 0; t < n; ++t) {
    const uint64_t k = hy_galois_elt(c, r[t]);
    if (k == 1) {
      automorph(c, cts[t], acc0, nl, nl, 1, true, s);
      automorph(c, cts[t] + nl * N, acc1, nl, nl, 1, true, s);
      any1 = true;
      continue;
    }
    automorph(c, cts[t], acc0, nl, nl, k, true, s);
    automorph(c, cts[t] + nl * N, b.rc, nl, nl, k, false, s);
    intt_poly(c, b.rc, b.d, level, s);
    modup_core(c, level, b.d, b.ext, s);
    IPArgs a = ip_args(c, level, b.ext, b.rc);
    ip(c, level, a, evks[t], b.u, 1, !first, s);
    first = false;
  }
  if (first) {  // no key switching at all: out = accumulated sum
    cudaMemcpyAsync(out, b.acc, 2 * nl * N * 8, cudaMemcpyDeviceToDevice, s);
  } else {
    moddown_core(c, level, 2, b.u, out, acc0, 1, any1 ? acc1 : nullptr, b.v, b.w, s);
  }
  return cuda_check("hy_hrot_sum");
}
