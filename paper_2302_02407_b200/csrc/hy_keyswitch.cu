// hy_keyswitch.cu -- automorphism, ModUp, key-switch inner product, ModDown and
// the three HRot variants (DESIGN R-HROT).
//
// HRot_r (left rotation by r) with Galois element k = 5^r mod 2N:
//   plain   : c' = kappa(c); d = iNTT(c'_1); ModUp(d) -> IP(evk_k) -> ModDown; out_0 += c'_0
//   hoisted : d = iNTT(c_1) once; ModUp once; per r the IP reads the extended
//             digits through the NTT-domain permutation of kappa_k (Halevi-Shoup)
//   lazy sum: per term plain ModUp + IP accumulated over Q_l u P; ONE ModDown.
//
// Batched engine: every stage runs on up to kG key switches per launch (items g),
// so a batch of rotations costs one launch per stage instead of one per rotation,
// and items that share an evaluation key (RaS of all output groups of a conv
// layer) stream that key from HBM once for the whole batch.
//
// Data layout (HBM): ct [2][l+1][N], ext [beta][l+1+K][N], u [2][l+1+K][N], evk (6-byte packed words)
// [dnum][2][n_q+n_p][N]; every limb is N contiguous uint64 (coalesced rows).
#include <algorithm>
#include <vector>

#include "hy_arith.cuh"

namespace hy {
namespace {

constexpr int kT = 256;
// kG (key switches per batched launch) lives in hy_internal.h

template <class T>
struct Arr {
  T p[kG];
};

// ---------------------------------------------------------------- automorphism
// item g: out_g[l][x] (+)= in_g[l][perm_{k_g}(x)]; limb l on prime l % per_poly.  grid (N/256, limbs, G)
// (Arr parameters are __grid_constant__: indexed by blockIdx / loop counters straight out of the
// parameter bank instead of being copied to a per-thread local-memory frame.)
__global__ void k_automorph(const __grid_constant__ Arr<const uint64_t*> in, const __grid_constant__ Arr<uint64_t*> out,
                            const __grid_constant__ Arr<uint64_t> k, int logN, int per_poly,
                            int accumulate, DevTables dt) {
  const size_t N = (size_t)1 << logN;
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  const int g = blockIdx.z;
  const size_t off = (size_t)blockIdx.y * N;
  uint64_t v = in.p[g][off + aut_index(x, k.p[g], logN)];
  if (accumulate) v = add_mod(v, out.p[g][off + x], dt.pc[blockIdx.y % per_poly].q);
  out.p[g][off + x] = v;
}

// out[l][x] (+)= sum_g in_g[l][perm_{k_g}(x)] (race-free reduction of G permuted polynomials).
// grid (N/256, limbs)
__global__ void k_automorph_sum(const __grid_constant__ Arr<const uint64_t*> in,
                                const __grid_constant__ Arr<uint64_t> k, int G, uint64_t* __restrict__ out,
                                int logN, int per_poly, DevTables dt) {
  const size_t N = (size_t)1 << logN;
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  const size_t off = (size_t)blockIdx.y * N;
  const uint64_t q = dt.pc[blockIdx.y % per_poly].q;
  uint64_t v = out[off + x];
  for (int g = 0; g < G; ++g) v = add_mod(v, in.p[g][off + aut_index(x, k.p[g], logN)], q);
  out[off + x] = v;
}

// MulCt tensor product of item g = blockIdx.z at limb i = blockIdx.y:
//   d0 = a0 b0 -> out[0], d1 = a0 b1 + a1 b0 -> out[1], d2 = a1 b1 -> d2 (all canonical, NTT domain).
// Every input word is read before the thread writes, so out may alias a or b.  grid (N/256, l+1, G)
__global__ void k_tensor(const __grid_constant__ Arr<const uint64_t*> a, const __grid_constant__ Arr<const uint64_t*> b,
                         const __grid_constant__ Arr<uint64_t*> out, const __grid_constant__ Arr<uint64_t*> d2,
                         int level, int logN, DevTables dt) {
  const size_t N = (size_t)1 << logN, pl = (size_t)(level + 1) * N;
  const int g = blockIdx.z, i = blockIdx.y;
  const size_t o = (size_t)i * N + blockIdx.x * blockDim.x + threadIdx.x;
  const PrimeConst& pc = dt.pc[i];
  const double q = pc.qd, qinv = pc.qinv;
  const double a0 = u2d(a.p[g][o]), a1 = u2d(a.p[g][pl + o]), b0 = u2d(b.p[g][o]), b1 = u2d(b.p[g][pl + o]);
  const double d0 = fmulmod(a0, b0, q, qinv);
  const double d1 = fmulmod(a0, b1, q, qinv) + fmulmod(a1, b0, q, qinv);
  const double dd = fmulmod(a1, b1, q, qinv);
  out.p[g][o] = d2u(fcanon(d0, q, qinv));
  out.p[g][pl + o] = d2u(fcanon(d1, q, qinv));
  d2.p[g][o] = d2u(fcanon(dd, q, qinv));
}

// FP64 constants of one prime, staged in shared memory.
struct FConst {
  double q, qinv;
};

// ---------------------------------------------------------------- ModUp basis conversion
// Item g = blockIdx.z, digit j = blockIdx.y; one thread per coefficient x produces every
// non-own limb of the digit.  grid (N/256, beta, G).
// y_i = [d_i (D_j/q_i)^{-1}]_{q_i} in [0, q_i);  ext[j][u][x] = [sum_i y_i ((D_j/q_i) mod t_u)]_{t_u}.
// Every product is reduced on the FP64 pipe (fmulmod, |term| <= 1.5 t), the A terms are summed
// exactly and canonicalised once.  A = alpha (compile time); a partial last digit pads with 0.
template <int A>
__global__ void __launch_bounds__(256) k_modup_bconv(const __grid_constant__ Arr<const uint64_t*> dd,
                                                     const __grid_constant__ Arr<uint64_t*> ee,
                                                     const ModUpConst* mc, DevTables dt, int level, int n_q, int E,
                                                     int logN) {
  __shared__ double s_hat[kMaxExt][A];
  __shared__ FConst s_fc[kMaxExt];
  const size_t N = (size_t)1 << logN;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  const uint64_t* d = dd.p[blockIdx.z];
  uint64_t* ext = ee.p[blockIdx.z];
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

// ---------------------------------------------------------------- key-switch inner product
// B = beta digits (compile time).
// u_g[c][u][x] (+)= sum_j src_g,j[u][perm_g(x)] * evk_g[j][c][chain(u)][x], where src_g,j[u] is the
// digit's own limb of own_g (the NTT-domain c1 the digits were cut from) when u belongs to digit j,
// else ext_g[j][u].
//   default: grid (G, N/256, E), one item per x-slice: the item index is the fastest grid dimension,
//            so when the items share their digits (hoisted: one ModUp, G Galois permutations) every
//            digit limb is fetched from HBM once per batch and then served from L2;
//   SHARED : grid (1, N/256, E), each thread loops over the items with evk_0 held in registers, so
//            the key is streamed from HBM once for the whole batch;
//   SUM    : grid (1, N/256, E), all items accumulate into u_0 (the lazy HRotSum), race-free because
//            one thread owns (u, x).
// Products reduced on the FP64 pipe and summed exactly (|sum| <= 1.5 B t < 2^53), canonicalised once
// per item (SUM: each item's sum is re-centred with fred before the cross-item sum).
template <int B, bool SHARED, bool SUM>
__global__ void __launch_bounds__(256) k_ks_ip(const __grid_constant__ Arr<const uint64_t*> ext,
                                               const __grid_constant__ Arr<const uint64_t*> own,
                                               const __grid_constant__ Arr<const uint64_t*> evk,
                                               const __grid_constant__ Arr<uint64_t*> uo,
                                               const __grid_constant__ Arr<uint64_t> kperm, int G, DevTables dt,
                                               int level, int n_q, int L1, int E, int alpha, int logN,
                                               int accumulate, int u0) {
  const size_t N = (size_t)1 << logN;
  const uint32_t x = blockIdx.y * blockDim.x + threadIdx.x;
  const int u = u0 + (int)blockIdx.z;
  const int t = u <= level ? u : n_q + (u - level - 1);
  const PrimeConst& p = dt.pc[t];
  const double q = p.qd, qinv = p.qinv;
  const int own_digit = u <= level ? u / alpha : -1;
  double e0[B], e1[B];
  if (SHARED) {
#pragma unroll
    for (int j = 0; j < B; ++j) {
      e0[j] = u2d(evk_word(evk_limb(evk.p[0], (size_t)(j * 2) * L1 + t, N), x));
      e1[j] = u2d(evk_word(evk_limb(evk.p[0], (size_t)(j * 2 + 1) * L1 + t, N), x));
    }
  }
  double s0 = 0.0, s1 = 0.0;
  const int g0 = (SHARED || SUM) ? 0 : (int)blockIdx.x;
  const int g1 = (SHARED || SUM) ? G : g0 + 1;
  for (int g = g0; g < g1; ++g) {
    const uint32_t xs = kperm.p[g] != 1 ? aut_index(x, kperm.p[g], logN) : x;
    uint64_t v[B];
#pragma unroll
    for (int j = 0; j < B; ++j) {
      const uint64_t* src = (j == own_digit && own.p[g]) ? own.p[g] + (size_t)u * N
                                                          : ext.p[g] + ((size_t)j * E + u) * N;
      v[j] = src[xs];
    }
    if (!SHARED) {
#pragma unroll
      for (int j = 0; j < B; ++j) {
        e0[j] = u2d(evk_word(evk_limb(evk.p[g], (size_t)(j * 2) * L1 + t, N), x));
        e1[j] = u2d(evk_word(evk_limb(evk.p[g], (size_t)(j * 2 + 1) * L1 + t, N), x));
      }
    }
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int j = 0; j < B; ++j) {
      const double vj = u2d(v[j]);
      a0 += fmulmod(vj, e0[j], q, qinv);
      a1 += fmulmod(vj, e1[j], q, qinv);
    }
    if (SUM) {
      s0 += fred(a0, q, qinv);
      s1 += fred(a1, q, qinv);
      if ((g & 31) == 31) {  // keep the running sum below 2^52 (exact) for batches of up to kG = 64
        s0 = fred(s0, q, qinv);
        s1 = fred(s1, q, qinv);
      }
      continue;
    }
    uint64_t* o0 = uo.p[g] + (size_t)u * N + x;
    uint64_t* o1 = uo.p[g] + ((size_t)E + u) * N + x;
    if (accumulate) {
      a0 += u2d(*o0);
      a1 += u2d(*o1);
    }
    *o0 = d2u(fcanon(a0, q, qinv));
    *o1 = d2u(fcanon(a1, q, qinv));
  }
  if (SUM) {
    uint64_t* o0 = uo.p[0] + (size_t)u * N + x;
    uint64_t* o1 = uo.p[0] + ((size_t)E + u) * N + x;
    if (accumulate) {
      s0 += u2d(*o0);
      s1 += u2d(*o1);
    }
    *o0 = d2u(fcanon(s0, q, qinv));
    *o1 = d2u(fcanon(s1, q, qinv));
  }
}

// ---------------------------------------------------------------- ModDown
// P -> Q_l basis conversion, KP = K special primes (compile time).  grid (N/256, npoly, G);
// v_g = iNTT(u_g on P) [npoly][K][N];  z_k = [v_k (P/p_k)^{-1}]_{p_k} in [0, p_k);
// w_g[c][i] = [sum_k z_k ((P/p_k) mod q_i)]_{q_i}.
template <int KP>
__global__ void __launch_bounds__(256) k_moddown_bconv(const __grid_constant__ Arr<const uint64_t*> vv,
                                                       const __grid_constant__ Arr<uint64_t*> ww,
                                                       const ModDownConst* md, DevTables dt, int level, int n_q,
                                                       int logN) {
  __shared__ double s_hat[kMaxChain][KP];
  __shared__ FConst s_fc[kMaxChain];
  const size_t N = (size_t)1 << logN;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  const uint64_t* v = vv.p[blockIdx.z];
  uint64_t* w = ww.p[blockIdx.z];
  const int n = level + 1;
  for (int i = threadIdx.x; i < n * KP; i += blockDim.x) s_hat[i / KP][i % KP] = (double)md->phat_mod[i / KP][i % KP];
  for (int i = threadIdx.x; i < n; i += blockDim.x) s_fc[i] = FConst{dt.pc[i].qd, dt.pc[i].qinv};
  double z[KP];
#pragma unroll
  for (int k = 0; k < KP; ++k) {
    const PrimeConst& pc = dt.pc[n_q + k];
    z[k] = fcanon(fmulmod(u2d(v[((size_t)c * KP + k) * N + x]), (double)md->phat_inv[k], pc.qd, pc.qinv), pc.qd,
                  pc.qinv);
    if (md->center && z[k] > 0.5 * (pc.qd - 1.0)) z[k] -= pc.qd;  // R-MODDOWN: centred remainder in (-p/2, p/2]
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

// out_g[c][i] = (u_g[c][i] - w_g[c][i]) P^{-1} (+ add0_g[i][perm_g(x)] for c = 0) (+ add1_g[i][x] for c = 1)
//               (+ addct_g[c][i][x]).  out_g may alias addct_g (read before write, same x).
// grid (N/256, l+1, npoly * G), blockIdx.z = g * npoly + c
struct FinalArgs {
  Arr<const uint64_t*> u, w, add0, add1, addct;
  Arr<uint64_t*> out;
  Arr<uint64_t> k0;
};
__global__ void k_moddown_final(const __grid_constant__ FinalArgs a, int npoly, int E, const ModDownConst* md,
                                DevTables dt, int level,
                                int logN) {
  const size_t N = (size_t)1 << logN;
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y, g = blockIdx.z / npoly, c = blockIdx.z % npoly;
  const uint64_t q = dt.pc[i].q;
  uint64_t val = sub_mod(a.u.p[g][((size_t)c * E + i) * N + x], a.w.p[g][((size_t)c * (level + 1) + i) * N + x], q);
  val = shoup(val, md->p_inv[i], md->p_inv_sh[i], q);
  if (c == 0 && a.add0.p[g]) {
    const uint32_t xs = a.k0.p[g] != 1 ? aut_index(x, a.k0.p[g], logN) : x;
    val = add_mod(val, a.add0.p[g][(size_t)i * N + xs], q);
  }
  if (c == 1 && a.add1.p[g]) val = add_mod(val, a.add1.p[g][(size_t)i * N + x], q);
  const size_t o = ((size_t)c * (level + 1) + i) * N + x;
  if (a.addct.p[g]) val = add_mod(val, a.addct.p[g][o], q);
  a.out.p[g][o] = val;
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

#define HY_DISPATCH_IP(SH, SM)                                                                              \
  switch (beta) {                                                                                           \
    case 1: k_ks_ip<1, SH, SM><<<g, kT, 0, s>>>(ARGS); break;                                                \
    case 2: k_ks_ip<2, SH, SM><<<g, kT, 0, s>>>(ARGS); break;                                                \
    case 3: k_ks_ip<3, SH, SM><<<g, kT, 0, s>>>(ARGS); break;                                                \
    case 4: k_ks_ip<4, SH, SM><<<g, kT, 0, s>>>(ARGS); break;                                                \
    case 5: k_ks_ip<5, SH, SM><<<g, kT, 0, s>>>(ARGS); break;                                                \
    case 6: k_ks_ip<6, SH, SM><<<g, kT, 0, s>>>(ARGS); break;                                                \
    case 7: k_ks_ip<7, SH, SM><<<g, kT, 0, s>>>(ARGS); break;                                                \
    default: k_ks_ip<8, SH, SM><<<g, kT, 0, s>>>(ARGS); break;                                               \
  }

// ---------------------------------------------------------------- host-side building blocks
// Per-item key-switch workspace.
struct KsItem {
  uint64_t *rc, *d, *ext, *u, *v, *w;
};

size_t item_words(const hy_ctx* c, uint32_t level) {
  const size_t n = level + 1, E = n + c->n_p, beta = n_digits(c, level);
  return (2 * n + n + beta * E + 2 * E + 2 * c->n_p + 2 * n) * c->N + 6 * 32;
}

// carve G item workspaces plus one [2][l+1][N] accumulator
hy_status carve(hy_ctx* c, uint32_t level, int G, KsItem* it, uint64_t** acc) {
  if (!c->ws) return fail(HY_E_WORKSPACE, "workspace not set (hy_ctx_set_workspace)");
  const size_t N = c->N, n = level + 1, E = n + c->n_p, beta = n_digits(c, level);
  Ws ws{c->ws, c->ws_bytes};
  for (int g = 0; g < G; ++g) {
    it[g].rc = ws.take<uint64_t>(2 * n * N);
    it[g].d = ws.take<uint64_t>(n * N);
    it[g].ext = ws.take<uint64_t>(beta * E * N);
    it[g].u = ws.take<uint64_t>(2 * E * N);
    it[g].v = ws.take<uint64_t>(2 * c->n_p * N);
    it[g].w = ws.take<uint64_t>(2 * n * N);
    if (!it[g].w) return fail(HY_E_WORKSPACE, "workspace too small for this level / batch");
  }
  if (acc) {
    *acc = ws.take<uint64_t>(2 * n * N);
    if (!*acc) return fail(HY_E_WORKSPACE, "workspace too small for this level / batch");
  }
  return HY_OK;
}

// how many items fit the workspace at this level (<= kG)
int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

int max_items(const hy_ctx* c, uint32_t level) {
  const size_t per = item_words(c, level) * 8 + 6 * 256;
  const size_t acc = 2 * (level + 1) * (size_t)c->N * 8 + 256;
  if (c->ws_bytes <= acc) return 0;
  static const int cap = std::max(1, std::min(kG, env_int("HY_KS_BATCH", kG)));
  return (int)std::min<size_t>(cap, (c->ws_bytes - acc) / per);
}

void automorph_batch(hy_ctx* c, int G, const uint64_t* const* in, uint64_t* const* out, const uint64_t* k,
                     uint32_t nlimbs, uint32_t per_poly, bool accumulate, cudaStream_t s) {
  if (G == 0) return;
  Arr<const uint64_t*> ai{};
  Arr<uint64_t*> ao{};
  Arr<uint64_t> ak{};
  for (int g = 0; g < G; ++g) {
    ai.p[g] = in[g];
    ao.p[g] = out[g];
    ak.p[g] = k[g];
  }
  dim3 grid(c->N / kT, nlimbs, G);
  KTimer kt(c, FAM_AUT, s);
  kt.bytes = (uint64_t)G * nlimbs * c->N * 8 * (accumulate ? 3 : 2);
  k_automorph<<<grid, kT, 0, s>>>(ai, ao, ak, c->log_n, per_poly, accumulate ? 1 : 0, c->dt);
}

void automorph(hy_ctx* c, const uint64_t* in, uint64_t* out, uint32_t nlimbs, uint32_t per_poly, uint64_t k,
               bool accumulate, cudaStream_t s) {
  automorph_batch(c, 1, &in, &out, &k, nlimbs, per_poly, accumulate, s);
}

// d_g: coefficient-domain [l+1][N] -> ext_g [beta][E][N] (non-own limbs, NTT domain).
// cols_only: stop after the NTT column pass (the row pass is fused into the IP, launch_ntt_rows_ip).
void modup_batch(hy_ctx* c, uint32_t level, int G, const uint64_t* const* d, uint64_t* const* ext, cudaStream_t s,
                 bool cols_only = false) {
  const int n = level + 1, E = n + c->n_p, beta = n_digits(c, level);
  Arr<const uint64_t*> ad{};
  Arr<uint64_t*> ae{};
  for (int g = 0; g < G; ++g) {
    ad.p[g] = d[g];
    ae.p[g] = ext[g];
  }
  dim3 grid(c->N / kT, beta, G);
  {
    KTimer kt(c, FAM_MODUP, s);
    kt.bytes = (uint64_t)G * ((uint64_t)n + (uint64_t)beta * E - n) * c->N * 8;
    HY_DISPATCH_1_8(k_modup_bconv, c->alpha, grid, kT, s, ad, ae, c->d_modup[level], c->dt, (int)level,
                    (int)c->n_q, E, (int)c->log_n);
  }
  LimbList L;
  for (int g = 0; g < G; ++g)
    for (int j = 0; j < beta; ++j) {
      const auto& m = c->h_modup[level][j];
      for (int u = 0; u < E; ++u) {
        if (u >= m.lo && u < m.hi) continue;
        uint64_t* p = ext[g] + ((size_t)j * E + u) * c->N;
        L.add(p, p, ext_chain(c, level, u));
      }
    }
  if (cols_only) ntt_cols_list(c, L, s);
  else ntt_list(c, L, false, s);
}

void intt_polys(hy_ctx* c, int G, const uint64_t* const* in, uint64_t* const* out, uint32_t level, cudaStream_t s);

// ModUp + IP of G items from the NTT-domain c1 (own): inverse row pass into d, then the fused
// iNTT-column / BConv / NTT-column kernel (N = 2^16; else iNTT + BConv + column pass), then the fused
// row pass / IP (hy_ntt.cu)
void modup_ip_fused(hy_ctx* c, uint32_t level, int G, uint64_t* const* d, uint64_t* const* ext,
                    const uint64_t* const* own, const uint64_t* const* evk, uint64_t* const* u, bool acc, bool sum,
                    cudaStream_t s, int u0 = 0, uint64_t* const* v = nullptr, bool rows_done = false,
                    const uint64_t* own_k = nullptr, int groups = 1) {
  if (modup_cols_ok(c)) {
    if (!rows_done) {  // rows_done: d already holds the inverse row pass (launch_ntt_rows_inv_aut)
      LimbList L;
      for (int g = 0; g < G; ++g)
        for (uint32_t i = 0; i <= level; ++i) L.add(own[g] + (size_t)i * c->N, d[g] + (size_t)i * c->N, i);
      rows_list(c, L, true, s);
    }
    ModUpColsArgs ma{};
    for (int g = 0; g < G; ++g) {
      ma.src[g] = d[g];
      ma.ext[g] = ext[g];
    }
    launch_modup_cols(c, ma, G, level, s);
  } else {
    intt_polys(c, G, own, d, level, s);
    modup_batch(c, level, G, d, ext, s, true);
  }
  RowsIpArgs ra{};
  for (int g = 0; g < G; ++g) {
    ra.ext[g] = ext[g];
    ra.own[g] = own[g];
    ra.evk[g] = evk[g];
    ra.u[g] = u[sum ? g / (G / groups) : g];  // sum: one u per group of G / groups items
    ra.v[g] = v ? v[g] : nullptr;
    ra.kx[g] = own_k ? own_k[g] : 1;  // own_k: the own digit is read from own_g through kappa (summed IP only)
  }
  launch_ntt_rows_ip(c, ra, G, level, sum, acc, s, u0, v != nullptr, false, groups);
}

// HY_FUSE_IP=0 / HY_FUSE_MD=0 run the unfused ModUp NTT + IP / ModDown NTT + epilogue (A/B measurements)
bool fuse_ip() {
  static const bool on = env_int("HY_FUSE_IP", 1) != 0;
  return on;
}
bool fuse_moddown() {
  static const bool on = env_int("HY_FUSE_MD", 1) != 0;
  return on;
}
// HY_SPLIT_MD=0: store every limb of the inner product and run ModDown afterwards (A/B measurements)
bool split_moddown() {
  static const bool on = env_int("HY_SPLIT_MD", 1) != 0 && env_int("HY_FUSE_IP", 1) != 0;
  return on;
}

// IP of G items.  shared: all items use evk[0]; sum: all items accumulate into u[0].  u0: first
// extended limb produced (l+1: the P limbs only, for the split ModDown).
void ip_batch(hy_ctx* c, uint32_t level, int G, const uint64_t* const* ext, const uint64_t* const* own,
              const uint64_t* const* evk, uint64_t* const* u, const uint64_t* kperm, bool acc, bool shared, bool sum,
              cudaStream_t s, int u0 = 0) {
  const int n = level + 1, E = n + c->n_p, beta = n_digits(c, level), nu = E - u0;
  Arr<const uint64_t*> ae{}, ao{}, ak{};
  Arr<uint64_t*> au{};
  Arr<uint64_t> ap{};
  for (int g = 0; g < G; ++g) {
    ae.p[g] = ext[g];
    ao.p[g] = own ? own[g] : nullptr;
    ak.p[g] = evk[shared ? 0 : g];
    au.p[g] = u[sum ? 0 : g];
    ap.p[g] = kperm ? kperm[g] : 1;
  }
  dim3 g((shared || sum) ? 1 : G, c->N / kT, nu);
  KTimer kt(c, FAM_IP, s);
  const uint64_t keys = shared ? 1 : G, outs = sum ? 1 : G;
  kt.bytes = ((uint64_t)G * beta * nu * 8 + keys * 2ull * beta * nu * 6 + outs * 2ull * nu * (acc ? 2 : 1) * 8) * c->N;
#define ARGS ae, ao, ak, au, ap, G, c->dt, (int)level, (int)c->n_q, (int)(c->n_q + c->n_p), E, (int)c->alpha, \
             (int)c->log_n, acc ? 1 : 0, u0
  if (shared && !sum) {
    HY_DISPATCH_IP(true, false)
  } else if (!shared && sum) {
    HY_DISPATCH_IP(false, true)
  } else if (shared && sum) {
    HY_DISPATCH_IP(true, true)
  } else {
    HY_DISPATCH_IP(false, false)
  }
#undef ARGS
}

// ModDown of G items: u_g [npoly][E][N] (NTT) -> out_g [npoly][l+1][N], with the final addends.
struct DownItem {
  const uint64_t* u;
  uint64_t* out;
  const uint64_t* add0;
  uint64_t k0;
  const uint64_t* add1;
  const uint64_t* addct;
  uint64_t *v, *w;  // scratch
};
void moddown_batch(hy_ctx* c, uint32_t level, int npoly, int G, const DownItem* it, cudaStream_t s) {
  const int n = level + 1, E = n + c->n_p, K = c->n_p;
  LimbList L;
  for (int g = 0; g < G; ++g)
    for (int cc = 0; cc < npoly; ++cc)
      for (int k = 0; k < K; ++k)
        L.add(it[g].u + ((size_t)cc * E + n + k) * c->N, it[g].v + ((size_t)cc * K + k) * c->N, c->n_q + k);
  ntt_list(c, L, true, s);
  Arr<const uint64_t*> av{};
  Arr<uint64_t*> aw{};
  for (int g = 0; g < G; ++g) {
    av.p[g] = it[g].v;
    aw.p[g] = it[g].w;
  }
  dim3 grid(c->N / kT, npoly, G);
  {
    KTimer kt(c, FAM_MODDOWN, s);
    kt.bytes = (uint64_t)G * ((uint64_t)npoly * K + (uint64_t)npoly * n) * c->N * 8;
    HY_DISPATCH_1_8(k_moddown_bconv, K, grid, kT, s, av, aw, c->d_moddown[level], c->dt, (int)level, (int)c->n_q,
                    (int)c->log_n);
  }
  LimbList L2;
  for (int g = 0; g < G; ++g)
    for (int cc = 0; cc < npoly; ++cc)
      for (int i = 0; i < n; ++i) {
        uint64_t* p = it[g].w + ((size_t)cc * n + i) * c->N;
        L2.add(p, p, i);
      }
  if (fuse_moddown()) {  // column pass, then the row pass fused with the epilogue
    ntt_cols_list(c, L2, s);
    RowsFinalArgs ra{};
    for (int g = 0; g < G; ++g) {
      ra.u[g] = it[g].u;
      ra.w[g] = it[g].w;
      ra.add0[g] = it[g].add0;
      ra.k0[g] = it[g].k0;
      ra.add1[g] = it[g].add1;
      ra.addct[g] = it[g].addct;
      ra.out[g] = it[g].out;
    }
    launch_ntt_rows_final(c, ra, G, npoly, level, s);
    return;
  }
  ntt_list(c, L2, false, s);
  FinalArgs a{};
  uint64_t extra = 0;
  for (int g = 0; g < G; ++g) {
    a.u.p[g] = it[g].u;
    a.w.p[g] = it[g].w;
    a.out.p[g] = it[g].out;
    a.add0.p[g] = it[g].add0;
    a.k0.p[g] = it[g].k0;
    a.add1.p[g] = it[g].add1;
    a.addct.p[g] = it[g].addct;
    extra += (it[g].add0 ? n : 0) + (it[g].add1 ? n : 0) + (it[g].addct ? (uint64_t)npoly * n : 0);
  }
  dim3 g2(c->N / kT, n, npoly * G);
  KTimer kt(c, FAM_MODDOWN, s);
  kt.bytes = ((uint64_t)G * npoly * n * 3 + extra) * c->N * 8;
  k_moddown_final<<<g2, kT, 0, s>>>(a, npoly, E, c->d_moddown[level], c->dt, (int)level, (int)c->log_n);
}

// Split ModDown, first half: the P limbs of u_g (computed first) -> iNTT -> P -> Q_l conversion -> forward
// column pass into w_g [2][l+1][N]; the second half is launch_rows_ip_final, which computes the Q limbs
// of the inner product and finishes (u - w) P^{-1} without storing them.
// v_ready: v already holds the P limbs after their inverse row pass (fused into the P-limb IP).
void moddown_p(hy_ctx* c, uint32_t level, int G, uint64_t* const* u, uint64_t* const* v, uint64_t* const* w,
               cudaStream_t s, bool v_ready = false) {
  const int n = level + 1, E = n + c->n_p, K = c->n_p;
  if (moddown_cols_ok(c)) {  // inverse row pass (unless fused upstream), then one fused column kernel
    if (!v_ready) {
      LimbList L;
      for (int g = 0; g < G; ++g)
        for (int cc = 0; cc < 2; ++cc)
          for (int k = 0; k < K; ++k)
            L.add(u[g] + ((size_t)cc * E + n + k) * c->N, v[g] + ((size_t)cc * K + k) * c->N, c->n_q + k);
      rows_list(c, L, true, s);
    }
    ModUpColsArgs ma{};
    for (int g = 0; g < G; ++g) {
      ma.src[g] = v[g];
      ma.ext[g] = w[g];
    }
    launch_moddown_cols(c, ma, G, level, s);
    return;
  }
  LimbList L;
  for (int g = 0; g < G; ++g)
    for (int cc = 0; cc < 2; ++cc)
      for (int k = 0; k < K; ++k)
        L.add(u[g] + ((size_t)cc * E + n + k) * c->N, v[g] + ((size_t)cc * K + k) * c->N, c->n_q + k);
  ntt_list(c, L, true, s);
  Arr<const uint64_t*> av{};
  Arr<uint64_t*> aw{};
  for (int g = 0; g < G; ++g) {
    av.p[g] = v[g];
    aw.p[g] = w[g];
  }
  dim3 grid(c->N / kT, 2, G);
  {
    KTimer kt(c, FAM_MODDOWN, s);
    kt.bytes = (uint64_t)G * ((uint64_t)2 * K + (uint64_t)2 * n) * c->N * 8;
    HY_DISPATCH_1_8(k_moddown_bconv, K, grid, kT, s, av, aw, c->d_moddown[level], c->dt, (int)level, (int)c->n_q,
                    (int)c->log_n);
  }
  LimbList L2;
  for (int g = 0; g < G; ++g)
    for (int cc = 0; cc < 2; ++cc)
      for (int i = 0; i < n; ++i) {
        uint64_t* p = w[g] + ((size_t)cc * n + i) * c->N;
        L2.add(p, p, i);
      }
  ntt_cols_list(c, L2, s);
}

void intt_polys(hy_ctx* c, int G, const uint64_t* const* in, uint64_t* const* out, uint32_t level, cudaStream_t s) {
  LimbList L;
  for (int g = 0; g < G; ++g)
    for (uint32_t i = 0; i <= level; ++i) L.add(in[g] + (size_t)i * c->N, out[g] + (size_t)i * c->N, i);
  ntt_list(c, L, true, s);
}

hy_status check_level(hy_ctx* c, uint32_t level) {
  if (!c) return fail(HY_E_ARG, "null ctx");
  if (level >= c->n_q) return fail(HY_E_ARG, "level out of range");
  return HY_OK;
}

}  // namespace

// Plain HRot of G ciphertexts: out_g = HRot_{r_g}(ct_g) (+ addct_g).  evk may repeat (shared key).
// out_g may alias ct_g and addct_g (ct_g is consumed into the workspace before the final write).
hy_status hrot_multi(hy_ctx* c, const uint64_t* const* evk, const uint64_t* const* ct, uint32_t level,
                     const int32_t* r, uint32_t n_items, uint64_t* const* out, const uint64_t* const* addct,
                     cudaStream_t s, const uint64_t* gal) {
  const size_t n = level + 1, N = c->N;
  // rotations by 0 first (copies / adds), then key switches in chunks
  std::vector<uint32_t> ks;
  for (uint32_t i = 0; i < n_items; ++i) {
    const uint64_t k = gal ? gal[i] : hy_galois_elt(c, r[i]);
    if (k != 1) {
      if (!evk[i]) return fail(HY_E_MISSING_KEY, "no evaluation key for rotation");
      ks.push_back(i);
      continue;
    }
    const uint64_t* a = addct ? addct[i] : nullptr;
    if (a) {  // out = ct + addct
      if (out[i] != a) cudaMemcpyAsync(out[i], a, 2 * n * N * 8, cudaMemcpyDeviceToDevice, s);
      automorph(c, ct[i], out[i], 2 * n, n, 1, true, s);
    } else if (out[i] != ct[i]) {
      cudaMemcpyAsync(out[i], ct[i], 2 * n * N * 8, cudaMemcpyDeviceToDevice, s);
    }
  }
  const int cap = max_items(c, level);
  if (!ks.empty() && cap == 0) return fail(HY_E_WORKSPACE, "workspace too small for this level");
  KsItem it[kG];
  for (size_t done = 0; done < ks.size();) {
    const int G = (int)std::min<size_t>(ks.size() - done, cap);
    hy_status st0 = carve(c, level, G, it, nullptr);
    if (st0 != HY_OK) return st0;
    const uint64_t* cin[kG];
    uint64_t* rc[kG];
    const uint64_t* rc1[kG];
    uint64_t* rc1w[kG];
    uint64_t* d[kG];
    uint64_t* ext[kG];
    uint64_t* u[kG];
    const uint64_t* keys[kG];
    uint64_t kk[kG];
    DownItem di[kG];
    bool shared = true, alias = false;
    for (int g = 0; g < G; ++g)  // an output overwriting any input c0 of the batch forbids the late gather
      for (int h = 0; h < G; ++h) alias |= out[ks[done + g]] == ct[ks[done + h]];
    for (int g = 0; g < G; ++g) {
      const uint32_t i = ks[done + g];
      cin[g] = ct[i];
      rc[g] = it[g].rc;
      rc1[g] = rc1w[g] = it[g].rc + n * N;
      d[g] = it[g].d;
      ext[g] = it[g].ext;
      u[g] = it[g].u;
      keys[g] = evk[i];
      kk[g] = gal ? gal[i] : hy_galois_elt(c, r[i]);
      shared &= evk[i] == evk[ks[done]];
      // kappa(c0) is gathered by the ModDown epilogue straight from ct (unless out aliases ct)
      di[g] = alias ? DownItem{it[g].u, out[i], it[g].rc, 1, nullptr, addct ? addct[i] : nullptr, it[g].v, it[g].w}
                    : DownItem{it[g].u, out[i], ct[i], kk[g], nullptr, addct ? addct[i] : nullptr, it[g].v, it[g].w};
      if (!alias) cin[g] = ct[i] + n * N;
    }
    // kappa fused into the inverse row pass and the own-digit reads (N = 2^16, no aliasing): kappa(c1) is never
    // stored; otherwise kappa(c1) (or the whole ct when an output aliases an input) is permuted into rc
    const bool fuse_aut = split_moddown() && !alias && modup_cols_ok(c);
    if (fuse_aut) {
      RowsAutArgs ra{};
      for (int g = 0; g < G; ++g) {
        ra.src[g] = ct[ks[done + g]] + n * N;
        ra.dst[g] = d[g];
        ra.k[g] = kk[g];
        rc1[g] = ct[ks[done + g]] + n * N;  // the own digits are read from c1 through kappa
      }
      launch_ntt_rows_inv_aut(c, ra, G, level, s);
    } else if (alias) {
      automorph_batch(c, G, cin, rc, kk, 2 * n, n, false, s);
    } else {
      automorph_batch(c, G, cin, rc1w, kk, n, n, false, s);
    }
    if (split_moddown()) {
      uint64_t* v[kG];
      uint64_t* w[kG];
      for (int g = 0; g < G; ++g) {
        v[g] = it[g].v;
        w[g] = it[g].w;
      }
      const bool vr = moddown_cols_ok(c);  // P-limb IP with the inverse row pass fused
      modup_ip_fused(c, level, G, d, ext, rc1, keys, u, false, false, s, (int)n, vr ? v : nullptr, fuse_aut);
      IpFinalArgs fa{};
      for (int g = 0; g < G; ++g) {
        fa.ext[g] = ext[g];
        fa.own[g] = rc1[g];
        fa.evk[g] = keys[g];
        fa.w[g] = w[g];
        fa.add0[g] = di[g].add0;
        fa.k0[g] = di[g].k0;
        fa.addct[g] = di[g].addct;
        fa.out[g] = di[g].out;
        fa.kx[g] = fuse_aut ? kk[g] : 1;  // own digits gathered from c1 through kappa
      }
      moddown_p(c, level, G, u, v, w, s, vr);
      launch_rows_ip_final(c, fa, G, level, false, s);
      done += G;
      continue;
    }
    if (fuse_ip()) {
      modup_ip_fused(c, level, G, d, ext, rc1, keys, u, false, false, s);
    } else {
      intt_polys(c, G, rc1, d, level, s);
      modup_batch(c, level, G, d, ext, s);
      ip_batch(c, level, G, ext, rc1, keys, u, nullptr, false, shared && G > 1, false, s);
    }
    moddown_batch(c, level, 2, G, di, s);
    done += G;
  }
  return HY_OK;
}

// MulCt + relinearization of G pairs: the tensor product, then d2 is key-switched from s^2 to
// s with the relinearization key through the split-ModDown engine of plain HRot (no automorphism): the
// P-limb IP, the ModDown column kernel, and the Q-limb IP fused with the epilogue, which adds (d0, d1)
// (held in out itself).  One key for every item: its rows stream from HBM once per batch.
hy_status mulct_multi(hy_ctx* c, const uint64_t* rlk, const uint64_t* const* a, const uint64_t* const* b,
                      uint32_t level, uint32_t n_items, uint64_t* const* out, cudaStream_t s) {
  const size_t n = level + 1, N = c->N;
  const int cap = max_items(c, level);
  if (n_items && cap == 0) return fail(HY_E_WORKSPACE, "workspace too small for this level");
  KsItem it[kG];
  for (size_t done = 0; done < n_items;) {
    const int G = (int)std::min<size_t>(n_items - done, cap);
    hy_status st0 = carve(c, level, G, it, nullptr);
    if (st0 != HY_OK) return st0;
    Arr<const uint64_t*> aa{}, bb{};
    Arr<uint64_t*> oo{}, dd{};
    uint64_t* d[kG];
    uint64_t* ext[kG];
    uint64_t* u[kG];
    uint64_t* v[kG];
    uint64_t* w[kG];
    const uint64_t* own[kG];
    const uint64_t* keys[kG];
    IpFinalArgs fa{};
    for (int g = 0; g < G; ++g) {
      aa.p[g] = a[done + g];
      bb.p[g] = b[done + g];
      oo.p[g] = out[done + g];
      dd.p[g] = it[g].rc + n * N;  // d2 takes the place of kappa(c1)
      own[g] = dd.p[g];
      d[g] = it[g].d;
      ext[g] = it[g].ext;
      u[g] = it[g].u;
      v[g] = it[g].v;
      w[g] = it[g].w;
      keys[g] = rlk;
      fa.ext[g] = ext[g];
      fa.own[g] = own[g];
      fa.evk[g] = rlk;
      fa.w[g] = w[g];
      fa.add0[g] = out[done + g];  // d0
      fa.k0[g] = 1;
      fa.add1[g] = out[done + g] + n * N;  // d1
      fa.out[g] = out[done + g];
      fa.kx[g] = 1;
    }
    {
      dim3 grid(c->N / kT, n, G);
      KTimer kt(c, FAM_ELEM, s);
      kt.bytes = (uint64_t)G * 7 * n * N * 8;
      k_tensor<<<grid, kT, 0, s>>>(aa, bb, oo, dd, (int)level, c->log_n, c->dt);
    }
    const bool vr = moddown_cols_ok(c);
    modup_ip_fused(c, level, G, d, ext, own, keys, u, false, false, s, (int)n, vr ? v : nullptr);
    moddown_p(c, level, G, u, v, w, s, vr);
    launch_rows_ip_final(c, fa, G, level, false, s);
    done += G;
  }
  return HY_OK;
}

hy_status hrot_plain(hy_ctx* c, const uint64_t* evk, const uint64_t* ct, uint32_t level, int32_t r, uint64_t* out,
                     cudaStream_t s, const uint64_t* addct) {
  return hrot_multi(c, &evk, &ct, level, &r, 1, &out, addct ? &addct : nullptr, s);
}

void launch_automorph(hy_ctx* c, const uint64_t* in, uint64_t* out, uint32_t n_limbs, uint64_t k, cudaStream_t s) {
  automorph(c, in, out, n_limbs, n_limbs, k, false, s);
}

size_t ks_item_bytes(const hy_ctx* c, uint32_t level) { return item_words(c, level) * 8 + 6 * 256; }

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

extern "C" hy_status hy_prot(hy_ctx* c, const uint64_t* pt, uint32_t level, int32_t r, uint64_t* out, void* stream) {
  if (!c || !pt || !out) return fail(HY_E_ARG, "null");
  if (level >= c->n_q) return fail(HY_E_ARG, "level out of range");
  if (pt == out) return fail(HY_E_ARG, "prot cannot run in place");
  const uint64_t k = hy_galois_elt(c, r);
  if (k == 1) {
    cudaMemcpyAsync(out, pt, (size_t)(level + 1) * c->N * 8, cudaMemcpyDeviceToDevice, st(stream));
  } else {
    automorph(c, pt, out, level + 1, 1, k, false, st(stream));
  }
  return cuda_check("hy_prot");
}

extern "C" hy_status hy_modup(hy_ctx* c, uint32_t level, const uint64_t* d, uint64_t* ext, void* stream) {
  hy_status s0 = check_level(c, level);
  if (s0 != HY_OK) return s0;
  if (!d || !ext) return fail(HY_E_ARG, "null");
  cudaStream_t s = st(stream);
  modup_batch(c, level, 1, &d, &ext, s);
  // own-digit limbs: NTT(d)
  const int E = level + 1 + c->n_p;
  LimbList L;
  for (uint32_t j = 0; j < n_digits(c, level); ++j) {
    const auto& m = c->h_modup[level][j];
    for (int i = m.lo; i < m.hi; ++i) L.add(d + (size_t)i * c->N, ext + ((size_t)j * E + i) * c->N, i);
  }
  ntt_list(c, L, false, s);
  return cuda_check("hy_modup");
}

extern "C" hy_status hy_ks_inner_product(hy_ctx* c, uint32_t level, const uint64_t* ext, const uint64_t* evk,
                                         uint64_t* u, void* stream) {
  hy_status s0 = check_level(c, level);
  if (s0 != HY_OK) return s0;
  if (!ext || !evk || !u) return fail(HY_E_ARG, "null");
  ip_batch(c, level, 1, &ext, nullptr, &evk, &u, nullptr, false, false, false, st(stream));
  return cuda_check("hy_ks_inner_product");
}

extern "C" hy_status hy_moddown(hy_ctx* c, uint32_t level, const uint64_t* u, uint64_t* out, void* stream) {
  hy_status s0 = check_level(c, level);
  if (s0 != HY_OK) return s0;
  if (!u || !out) return fail(HY_E_ARG, "null");
  KsItem it[1];
  s0 = carve(c, level, 1, it, nullptr);
  if (s0 != HY_OK) return s0;
  DownItem di{u, out, nullptr, 1, nullptr, nullptr, it[0].v, it[0].w};
  moddown_batch(c, level, 1, 1, &di, st(stream));
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
  // no output may overlap any input of the batch: items run in key-switch chunks and r = 0 items are copied
  // first, so an output over another item's input would corrupt it (include/hyphen.h)
  const size_t ctw = 2ull * (level + 1) * c->N;
  for (uint32_t i = 0; i < n; ++i) {
    if (!outs[i] || !cts[i]) return fail(HY_E_ARG, "null ciphertext");
    for (uint32_t j = 0; j < n; ++j)
      if (outs[i] < cts[j] + ctw && cts[j] < outs[i] + ctw)
        return fail(HY_E_ARG, i == j ? "hrot cannot run in place" : "an output overlaps another item's input");
  }
  s0 = hrot_multi(c, evks, cts, level, r, n, outs, nullptr, st(stream));
  if (s0 != HY_OK) return s0;
  return cuda_check("hy_hrot_batch");
}

extern "C" hy_status hy_hrot_galois(hy_ctx* c, const uint64_t* evk, const uint64_t* ct, uint32_t level, uint64_t k,
                                    uint64_t* out, void* stream) {
  hy_status s0 = check_level(c, level);
  if (s0 != HY_OK) return s0;
  if (!ct || !out) return fail(HY_E_ARG, "null");
  if (!(k & 1) || k >= 2ull * c->N) return fail(HY_E_ARG, "Galois element must be odd and < 2N");
  if (out == ct) return fail(HY_E_ARG, "the key switch cannot run in place");
  const int32_t r0 = 0;
  s0 = hrot_multi(c, &evk, &ct, level, &r0, 1, &out, nullptr, st(stream), &k);
  if (s0 != HY_OK) return s0;
  return cuda_check("hy_hrot_galois");
}

extern "C" hy_status hy_hrot_hoisted(hy_ctx* c, const uint64_t* const* evks, const uint64_t* ct, uint32_t level,
                                     const int32_t* r, uint32_t n, uint64_t* const* outs, void* stream) {
  hy_status s0 = check_level(c, level);
  if (s0 != HY_OK) return s0;
  if (!evks || !ct || !r || !outs) return fail(HY_E_ARG, "null");
  cudaStream_t s = st(stream);
  const size_t nl = level + 1, N = c->N;
  std::vector<uint32_t> ks;
  for (uint32_t i = 0; i < n; ++i) {
    if (outs[i] == ct) return fail(HY_E_ARG, "hrot cannot run in place");
    if (hy_galois_elt(c, r[i]) == 1) {
      cudaMemcpyAsync(outs[i], ct, 2 * nl * N * 8, cudaMemcpyDeviceToDevice, s);
      continue;
    }
    if (!evks[i]) return fail(HY_E_MISSING_KEY, "no evaluation key for rotation");
    ks.push_back(i);
  }
  if (ks.empty()) return cuda_check("hy_hrot_hoisted");
  const int cap = max_items(c, level);
  if (cap == 0) return fail(HY_E_WORKSPACE, "workspace too small for this level");
  KsItem it[kG];
  s0 = carve(c, level, cap, it, nullptr);
  if (s0 != HY_OK) return s0;
  // one ModUp of c1 into item 0's buffers, shared by every rotation
  const uint64_t* c1 = ct + nl * N;
  intt_polys(c, 1, &c1, &it[0].d, level, s);
  modup_batch(c, level, 1, (const uint64_t* const*)&it[0].d, &it[0].ext, s);
  for (size_t done = 0; done < ks.size();) {
    const int G = (int)std::min<size_t>(ks.size() - done, cap);
    const uint64_t* ext[kG];
    const uint64_t* own[kG];
    const uint64_t* keys[kG];
    uint64_t* u[kG];
    uint64_t kk[kG];
    DownItem di[kG];
    for (int g = 0; g < G; ++g) {
      const uint32_t i = ks[done + g];
      ext[g] = it[0].ext;
      own[g] = c1;
      keys[g] = evks[i];
      u[g] = it[g].u;
      kk[g] = hy_galois_elt(c, r[i]);
      di[g] = DownItem{it[g].u, outs[i], ct, kk[g], nullptr, nullptr, it[g].v, it[g].w};
    }
    if (split_moddown()) {  // P limbs of the IP, their conversion, then the Q limbs fused with the epilogue
      uint64_t* v[kG];
      uint64_t* w[kG];
      IpFinalArgs fa{};
      for (int g = 0; g < G; ++g) {
        v[g] = it[g].v;
        w[g] = it[g].w;
        fa.ext[g] = it[0].ext;
        fa.own[g] = c1;
        fa.evk[g] = keys[g];
        fa.w[g] = w[g];
        fa.add0[g] = ct;
        fa.k0[g] = kk[g];
        fa.out[g] = outs[ks[done + g]];
        fa.kx[g] = kk[g];
      }
      const bool vr = moddown_cols_ok(c);
      if (vr) {  // P-limb IP as a row kernel with the inverse row pass fused (v in the between-pass format)
        RowsIpArgs ra{};
        for (int g = 0; g < G; ++g) {
          ra.ext[g] = ext[g];
          ra.own[g] = c1;
          ra.evk[g] = keys[g];
          ra.u[g] = u[g];
          ra.v[g] = v[g];
          ra.kx[g] = kk[g];
        }
        launch_ntt_rows_ip(c, ra, G, level, false, false, s, (int)nl, true, true);
      } else {
        ip_batch(c, level, G, ext, own, keys, u, kk, false, false, false, s, (int)nl);
      }
      moddown_p(c, level, G, u, v, w, s, vr);
      launch_rows_ip_final(c, fa, G, level, true, s);
      done += G;
      continue;
    }
    ip_batch(c, level, G, ext, own, keys, u, kk, false, false, false, s);
    moddown_batch(c, level, 2, G, di, s);
    done += G;
  }
  return cuda_check("hy_hrot_hoisted");
}

namespace hy {

// The hoisted rotations of I ciphertexts by the same n amounts (CAConv Slide_f over the layer's inputs),
// batched: the I ModUps in one launch set, then all I x n (input, rotation) items' P-limb IP, ModDown columns and
// Q-limb IP + epilogue together; each item's operations are hy_hrot_hoisted's (bit-identical).  outs[i n + t] =
// HRot_{r_t}(cts[i]); every r_t must need a key switch.  HY_E_WORKSPACE: not batchable here (nothing launched),
// call hy_hrot_hoisted per input.
hy_status hrot_hoisted_multi(hy_ctx* c, const uint64_t* const* evks, const uint64_t* const* cts, uint32_t I,
                             uint32_t level, const int32_t* r, uint32_t n, uint64_t* const* outs, cudaStream_t s) {
  static const bool on = env_int("HY_HOIST_MULTI", 1) != 0;  // HY_HOIST_MULTI=0: hy_hrot_hoisted per input (A/B)
  if (!on || I < 2 || n == 0 || !split_moddown() || !moddown_cols_ok(c)) return HY_E_WORKSPACE;
  const size_t nl = level + 1, N = c->N;
  for (uint32_t t = 0; t < n; ++t) {
    if (hy_galois_elt(c, r[t]) == 1) return HY_E_WORKSPACE;
    if (!evks[t]) return fail(HY_E_MISSING_KEY, "no evaluation key for rotation");
  }
  for (size_t k = 0; k < (size_t)I * n; ++k)
    for (uint32_t i = 0; i < I; ++i)
      if (outs[k] == cts[i]) return HY_E_WORKSPACE;
  const int cap = max_items(c, level);
  const uint32_t ic = cap / (int)n;  // inputs per launch set
  if (ic < 2) return HY_E_WORKSPACE;
  if (I > ic) {
    for (uint32_t i0 = 0; i0 < I; i0 += ic) {
      const uint32_t in_ = std::min(ic, I - i0);
      hy_status st2 = in_ >= 2 ? hrot_hoisted_multi(c, evks, cts + i0, in_, level, r, n, outs + (size_t)i0 * n, s)
                               : HY_E_WORKSPACE;
      if (st2 == HY_E_WORKSPACE) st2 = hy_hrot_hoisted(c, evks, cts[i0], level, r, n, outs + (size_t)i0 * n, s);
      if (st2 != HY_OK) return st2;
    }
    return HY_OK;
  }
  KsItem it[kG];
  hy_status s0 = carve(c, level, cap, it, nullptr);
  if (s0 != HY_OK) return s0;
  // one ModUp per input into item i's d / ext (the rotation items use only their u / v / w)
  const uint64_t* c1[kG];
  uint64_t* dd[kG];
  uint64_t* ee[kG];
  for (uint32_t i = 0; i < I; ++i) {
    c1[i] = cts[i] + nl * N;
    dd[i] = it[i].d;
    ee[i] = it[i].ext;
  }
  intt_polys(c, (int)I, c1, dd, level, s);
  modup_batch(c, level, (int)I, (const uint64_t* const*)dd, ee, s);
  const int G = (int)(I * n);
  RowsIpArgs ra{};
  IpFinalArgs fa{};
  uint64_t* u[kG];
  uint64_t* v[kG];
  uint64_t* w[kG];
  for (int g = 0; g < G; ++g) {
    const uint32_t i = g / n, t = g % n;
    const uint64_t kk = hy_galois_elt(c, r[t]);
    u[g] = it[g].u;
    v[g] = it[g].v;
    w[g] = it[g].w;
    ra.ext[g] = ee[i];
    ra.own[g] = c1[i];
    ra.evk[g] = evks[t];
    ra.u[g] = u[g];
    ra.v[g] = v[g];
    ra.kx[g] = kk;
    fa.ext[g] = ee[i];
    fa.own[g] = c1[i];
    fa.evk[g] = evks[t];
    fa.w[g] = w[g];
    fa.add0[g] = cts[i];
    fa.k0[g] = kk;
    fa.out[g] = outs[g];
    fa.kx[g] = kk;
  }
  launch_ntt_rows_ip(c, ra, G, level, false, false, s, (int)nl, true, true);
  moddown_p(c, level, G, u, v, w, s, true);
  launch_rows_ip_final(c, fa, G, level, true, s);
  return HY_OK;
}

// The lazy HRotSum state of n terms (hy_hrot_sum before its ModDown, DESIGN R-HROT):
//   u   [2][l+1+K][N]  sum_t of the key-switch inner products IP_t(kappa_t(c1_t)) over Q_l u P (NTT, canonical;
//                      zero when no term needs a key switch)
//   acc [2][l+1][N]    (sum_t kappa_t(c0_t) incl. the r = 0 terms' c0, sum of the r = 0 terms' c1)
// it: cap carved key-switch items (their u / v / w are not used).  *any_ks: some term was key-switched.
hy_status hrot_sum_state(hy_ctx* c, const uint64_t* const* evks, const uint64_t* const* cts, uint32_t level,
                         const int32_t* r, uint32_t n, uint64_t* u, uint64_t* acc, KsItem* it, int cap, bool* any_ks,
                         cudaStream_t s) {
  const size_t nl = level + 1, N = c->N, E = nl + c->n_p;
  std::vector<uint32_t> ks, zero;
  for (uint32_t t = 0; t < n; ++t) {
    if (hy_galois_elt(c, r[t]) == 1) {
      zero.push_back(t);
    } else {
      if (!evks[t]) return fail(HY_E_MISSING_KEY, "no evaluation key for rotation");
      ks.push_back(t);
    }
  }
  uint64_t* acc0 = acc;           // sum of kappa(c0_t) (and unrotated c0_t)
  uint64_t* acc1 = acc + nl * N;  // sum of unrotated c1_t
  cudaMemsetAsync(acc, 0, 2 * nl * N * 8, s);
  // r = 0 terms: added without key switching
  for (uint32_t t : zero) {
    automorph(c, cts[t], acc0, nl, nl, 1, true, s);
    automorph(c, cts[t] + nl * N, acc1, nl, nl, 1, true, s);
  }
  bool first = true;
  for (size_t done = 0; done < ks.size();) {
    const int G = (int)std::min<size_t>(ks.size() - done, cap);
    const uint64_t* c0[kG];
    const uint64_t* c1[kG];
    uint64_t* rc1[kG];
    const uint64_t* rc1c[kG];
    uint64_t* d[kG];
    uint64_t* ext[kG];
    const uint64_t* keys[kG];
    uint64_t kk[kG];
    for (int g = 0; g < G; ++g) {
      const uint32_t t = ks[done + g];
      c0[g] = cts[t];
      c1[g] = cts[t] + nl * N;
      rc1[g] = it[g].rc;
      rc1c[g] = it[g].rc;
      d[g] = it[g].d;
      ext[g] = it[g].ext;
      keys[g] = evks[t];
      kk[g] = hy_galois_elt(c, r[t]);
    }
    // acc0 += sum_g kappa_g(c0_g), race-free in one kernel
    {
      Arr<const uint64_t*> ai{};
      Arr<uint64_t> ak{};
      for (int g = 0; g < G; ++g) {
        ai.p[g] = c0[g];
        ak.p[g] = kk[g];
      }
      dim3 grid(c->N / kT, nl);
      KTimer kt(c, FAM_AUT, s);
      kt.bytes = ((uint64_t)G + 2) * nl * N * 8;
      k_automorph_sum<<<grid, kT, 0, s>>>(ai, ak, G, acc0, c->log_n, (int)nl, c->dt);
    }
    if (fuse_ip() && modup_cols_ok(c) && sum_tma_on()) {
      // kappa fused into the inverse row pass of c1 and into the own-digit reads of the summed IP: kappa(c1) is
      // never stored
      RowsAutArgs ra{};
      for (int g = 0; g < G; ++g) {
        ra.src[g] = c1[g];
        ra.dst[g] = d[g];
        ra.k[g] = kk[g];
      }
      launch_ntt_rows_inv_aut(c, ra, G, level, s);
      modup_ip_fused(c, level, G, d, ext, c1, keys, &u, !first, true, s, 0, nullptr, true, kk);
    } else if (fuse_ip()) {
      automorph_batch(c, G, c1, rc1, kk, nl, nl, false, s);
      modup_ip_fused(c, level, G, d, ext, rc1c, keys, &u, !first, true, s);
    } else {
      automorph_batch(c, G, c1, rc1, kk, nl, nl, false, s);
      intt_polys(c, G, rc1c, d, level, s);
      modup_batch(c, level, G, d, ext, s);
      ip_batch(c, level, G, ext, rc1c, keys, &u, nullptr, !first, false, true, s);
    }
    first = false;
    done += G;
  }
  if (first) cudaMemsetAsync(u, 0, 2 * E * N * 8, s);
  *any_ks = !first;
  return HY_OK;
}

// hrot_sum_state into caller buffers (carves its own key-switch items)
hy_status hrot_sum_partial(hy_ctx* c, const uint64_t* const* evks, const uint64_t* const* cts, uint32_t level,
                           const int32_t* r, uint32_t n, uint64_t* u, uint64_t* acc, cudaStream_t s) {
  const int cap = max_items(c, level);
  if (cap == 0) return fail(HY_E_WORKSPACE, "workspace too small for this level");
  KsItem it[kG];
  hy_status s0 = carve(c, level, cap, it, nullptr);
  if (s0 != HY_OK) return s0;
  bool any = false;
  return hrot_sum_state(c, evks, cts, level, r, n, u, acc, it, cap, &any, s);
}

// out = ModDown(u) + acc (the lazy HRotSum's one ModDown); u, acc canonical.
hy_status hrot_sum_finish(hy_ctx* c, uint32_t level, const uint64_t* u, const uint64_t* acc, uint64_t* out,
                          cudaStream_t s) {
  if (max_items(c, level) == 0) return fail(HY_E_WORKSPACE, "workspace too small for this level");
  KsItem it[1];
  hy_status s0 = carve(c, level, 1, it, nullptr);
  if (s0 != HY_OK) return s0;
  const size_t nl = level + 1, N = c->N;
  DownItem di{u, out, acc, 1, acc + nl * N, nullptr, it[0].v, it[0].w};
  moddown_batch(c, level, 2, 1, &di, s);
  return HY_OK;
}

// The lazy HRotSums of O outputs over the same n rotations (RAConv_Reorder: every output sums its f^2 tap
// accumulators with the same tap amounts): out_o = sum_t HRot_{r_t}(cts[o n + t]).  Each output's terms
// are the same operations as hy_hrot_sum's (bit-identical), batched over the outputs: one inverse row pass, one
// ModUp column kernel and one grouped summed IP for all O x T key-switched terms, one ModDown for the O sums.
// Returns HY_E_WORKSPACE (nothing launched) when the O x T items or the O accumulators do not fit; callers then
// fall back to hy_hrot_sum per output.
hy_status hrot_sum_multi(hy_ctx* c, const uint64_t* const* evks, const uint64_t* const* cts, uint32_t level,
                         const int32_t* r, uint32_t n, uint32_t O, uint64_t* const* outs, cudaStream_t s) {
  static const bool on = env_int("HY_SUM_MULTI", 1) != 0;  // HY_SUM_MULTI=0: one hy_hrot_sum per output (A/B)
  if (!on || !(fuse_ip() && modup_cols_ok(c) && sum_tma_on())) return HY_E_WORKSPACE;
  const size_t nl = level + 1, N = c->N;
  std::vector<uint32_t> ks, zero;
  for (uint32_t t = 0; t < n; ++t) {
    if (hy_galois_elt(c, r[t]) == 1) {
      zero.push_back(t);
    } else {
      if (!evks[t]) return fail(HY_E_MISSING_KEY, "no evaluation key for rotation");
      ks.push_back(t);
    }
  }
  const int T = (int)ks.size();
  const int cap = max_items(c, level);
  if (T == 0 || cap < 4) return HY_E_WORKSPACE;
  const uint32_t oc = (uint32_t)std::min(cap / T, cap / 2);  // outputs per launch set
  if (oc < 2) return HY_E_WORKSPACE;
  if (O > oc) {  // chunks of oc outputs (stream-ordered: each chunk reuses the workspace after the previous one)
    for (uint32_t o0 = 0; o0 < O; o0 += oc) {
      const uint32_t on = std::min(oc, O - o0);
      hy_status st2 = on >= 2 ? hrot_sum_multi(c, evks, cts + (size_t)o0 * n, level, r, n, on, outs + o0, s)
                               : HY_E_WORKSPACE;
      if (st2 == HY_E_WORKSPACE) st2 = hy_hrot_sum(c, evks, cts + (size_t)o0 * n, level, r, n, outs[o0], s);
      if (st2 != HY_OK) return st2;
    }
    return HY_OK;
  }
  if (O < 2) return HY_E_WORKSPACE;
  const int G = (int)O * T;
  KsItem it[kG];
  hy_status s0 = carve(c, level, cap, it, nullptr);
  if (s0 != HY_OK) return s0;
  // accumulators: (sum_t kappa_t(c0_t) incl. the r = 0 terms' c0, sum of the r = 0 terms' c1) of output o in the
  // w buffer of item O + o (the summed IP uses only d / ext / u; ModDown's scratch is items 0 .. O - 1)
  std::vector<uint64_t*> acc(O), u(O);
  for (uint32_t o = 0; o < O; ++o) {
    acc[o] = it[O + o].w;
    u[o] = it[o].u;
  }
  uint64_t kk[kG];
  for (int t = 0; t < T; ++t) kk[t] = hy_galois_elt(c, r[ks[t]]);
  for (uint32_t o = 0; o < O; ++o) {
    const uint64_t* const* co = cts + (size_t)o * n;
    uint64_t* acc0 = acc[o];
    uint64_t* acc1 = acc[o] + nl * N;
    cudaMemsetAsync(acc[o], 0, 2 * nl * N * 8, s);
    for (uint32_t t : zero) {
      automorph(c, co[t], acc0, nl, nl, 1, true, s);
      automorph(c, co[t] + nl * N, acc1, nl, nl, 1, true, s);
    }
    Arr<const uint64_t*> ai{};
    Arr<uint64_t> ak{};
    for (int t = 0; t < T; ++t) {
      ai.p[t] = co[ks[t]];
      ak.p[t] = kk[t];
    }
    dim3 grid(c->N / kT, nl);
    KTimer kt(c, FAM_AUT, s);
    kt.bytes = ((uint64_t)T + 2) * nl * N * 8;
    k_automorph_sum<<<grid, kT, 0, s>>>(ai, ak, T, acc0, c->log_n, (int)nl, c->dt);
  }
  // item g = o T + t: c1 of output o's term ks[t]
  const uint64_t* c1[kG];
  uint64_t* d[kG];
  uint64_t* ext[kG];
  const uint64_t* keys[kG];
  uint64_t kg[kG];
  RowsAutArgs ra{};
  for (int g = 0; g < G; ++g) {
    const int o = g / T, t = g % T;
    c1[g] = cts[(size_t)o * n + ks[t]] + nl * N;
    d[g] = it[g].d;
    ext[g] = it[g].ext;
    keys[g] = evks[ks[t]];
    kg[g] = kk[t];
    ra.src[g] = c1[g];
    ra.dst[g] = d[g];
    ra.k[g] = kg[g];
  }
  launch_ntt_rows_inv_aut(c, ra, G, level, s);
  modup_ip_fused(c, level, G, d, ext, c1, keys, u.data(), false, true, s, 0, nullptr, true, kg, (int)O);
  std::vector<DownItem> di(O);
  for (uint32_t o = 0; o < O; ++o) di[o] = DownItem{u[o], outs[o], acc[o], 1, acc[o] + nl * N, nullptr, it[o].v, it[o].w};
  moddown_batch(c, level, 2, (int)O, di.data(), s);
  return HY_OK;
}

// x mod q_t in place for words < 2^64 (sums of canonical residues over ranks): [npoly][nlimb][N], limb i of
// every poly on chain index chain0[i]
__global__ void k_mod_reduce(uint64_t* __restrict__ x, const __grid_constant__ Arr<uint64_t> chain, int nlimb,
                             int logN, DevTables dt) {
  const size_t N = (size_t)1 << logN;
  const int i = blockIdx.y % nlimb;
  const size_t o = (size_t)blockIdx.y * N + blockIdx.x * blockDim.x + threadIdx.x;
  x[o] = reduce64(x[o], dt.pc[chain.p[i]]);
}

hy_status mod_reduce_ext(hy_ctx* c, uint32_t level, uint64_t* u, uint64_t* acc, cudaStream_t s) {
  const int nl = level + 1, E = nl + c->n_p;
  Arr<uint64_t> ch{};  // kG chain indices per launch: limbs are reduced in slices of at most kG
  for (int lo = 0; lo < E; lo += kG) {
    const int m = std::min(kG, E - lo);
    for (int i = 0; i < m; ++i) ch.p[i] = ext_chain(c, level, lo + i);
    for (int p = 0; p < 2; ++p) {
      dim3 g(c->N / kT, m);
      KTimer kt(c, FAM_ELEM, s);
      kt.bytes = 2ull * m * c->N * 8;
      k_mod_reduce<<<g, kT, 0, s>>>(u + ((size_t)p * E + lo) * c->N, ch, m, c->log_n, c->dt);
    }
  }
  for (int lo = 0; lo < nl; lo += kG) {
    const int m = std::min(kG, nl - lo);
    for (int i = 0; i < m; ++i) ch.p[i] = lo + i;
    for (int p = 0; p < 2; ++p) {
      dim3 g(c->N / kT, m);
      KTimer kt(c, FAM_ELEM, s);
      kt.bytes = 2ull * m * c->N * 8;
      k_mod_reduce<<<g, kT, 0, s>>>(acc + ((size_t)p * nl + lo) * c->N, ch, m, c->log_n, c->dt);
    }
  }
  return HY_OK;
}

}  // namespace hy

extern "C" hy_status hy_hrot_sum(hy_ctx* c, const uint64_t* const* evks, const uint64_t* const* cts, uint32_t level,
                                 const int32_t* r, uint32_t n, uint64_t* out, void* stream) {
  hy_status s0 = check_level(c, level);
  if (s0 != HY_OK) return s0;
  if (!evks || !cts || !r || !out || n == 0) return fail(HY_E_ARG, "null / empty");
  for (uint32_t t = 0; t < n; ++t)
    if (cts[t] == out) return fail(HY_E_ARG, "output aliases an input");
  cudaStream_t s = st(stream);
  const size_t nl = level + 1, N = c->N;
  const int cap = max_items(c, level);
  if (cap == 0) return fail(HY_E_WORKSPACE, "workspace too small for this level");
  KsItem it[kG];
  uint64_t* acc = nullptr;
  s0 = carve(c, level, cap, it, &acc);
  if (s0 != HY_OK) return s0;
  bool any_ks = false;
  s0 = hrot_sum_state(c, evks, cts, level, r, n, it[0].u, acc, it, cap, &any_ks, s);
  if (s0 != HY_OK) return s0;
  if (!any_ks) {  // no key switching at all: out = accumulated sum
    cudaMemcpyAsync(out, acc, 2 * nl * N * 8, cudaMemcpyDeviceToDevice, s);
  } else {
    DownItem di{it[0].u, out, acc, 1, acc + nl * N, nullptr, it[0].v, it[0].w};
    moddown_batch(c, level, 2, 1, &di, s);
  }
  return cuda_check("hy_hrot_sum");
}

extern "C" hy_status hy_mulct_batch(hy_ctx* c, const uint64_t* rlk, const uint64_t* const* a, const uint64_t* const* b,
                                    uint32_t level, uint32_t n, uint64_t* const* outs, void* stream) {
  hy_status s0 = check_level(c, level);
  if (s0 != HY_OK) return s0;
  if (!rlk || !a || !b || !outs) return fail(HY_E_ARG, "null");
  for (uint32_t i = 0; i < n; ++i) {
    if (!a[i] || !b[i] || !outs[i]) return fail(HY_E_ARG, "null ciphertext");
    for (uint32_t j = 0; j < n; ++j)  // an output may alias its own inputs only
      if (j != i && (outs[i] == a[j] || outs[i] == b[j])) return fail(HY_E_ARG, "output aliases another item's input");
  }
  s0 = mulct_multi(c, rlk, a, b, level, n, outs, st(stream));
  if (s0 != HY_OK) return s0;
  return cuda_check("hy_mulct_batch");
}

extern "C" hy_status hy_mulct(hy_ctx* c, const uint64_t* rlk, const uint64_t* a, const uint64_t* b, uint32_t level,
                              uint64_t* out, void* stream) {
  return hy_mulct_batch(c, rlk, &a, &b, level, 1, &out, stream);
}
