// hy_internal.h -- context layout and launcher declarations shared by the
// product's CUDA translation units.  Nothing here is visible through the C ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/hyphen.h"

namespace hy {

constexpr int kMaxChain = 64;   // n_q + n_p
constexpr int kMaxBatch = 256;  // limbs per batched NTT launch
constexpr int kMaxDigits = 16;
constexpr int kMaxExt = 48;     // l+1+K

// Per-prime constants (device resident, indexed by chain index).
struct PrimeConst {
  uint64_t q;
  uint64_t two_q;
  uint64_t mu;          // floor(2^64 / q)            (Barrett for 64-bit words)
  uint64_t r64;         // 2^64 mod q                 (128-bit reduction)
  uint64_t r64_sh;      // Shoup companion of r64
  uint64_t n_inv;       // N^{-1} mod q
  uint64_t n_inv_sh;
  double qd;            // q as a double (exact: q < 2^48)
  double qinv;          // 1/q rounded to double
  double n_inv_d;       // N^{-1} mod q as a double
};

// Basis-conversion constants for one (level, digit): ModUp  D_j -> other limbs.
struct ModUpConst {
  int lo, hi;                               // q-limb range of digit j
  uint64_t hat_inv[8], hat_inv_sh[8];      // (D_j/q_i)^{-1} mod q_i
  // (D_j/q_i) mod t for every ext limb u (u indexes Q_l u P), [u][i]
  uint64_t hat_mod[kMaxExt][8];
};

struct ModDownConst {
  uint64_t phat_inv[8], phat_inv_sh[8];    // (P/p_k)^{-1} mod p_k
  uint64_t phat_mod[kMaxChain][8];         // (P/p_k) mod q_i
  uint64_t p_inv[kMaxChain], p_inv_sh[kMaxChain];  // P^{-1} mod q_i
  // chain index of the first source limb (ModDown: n_q, the first special prime); center: lift the source
  // residue to (-p/2, p/2] before converting it (the fused rescale, a ModDown by P = q_l with the centred
  // remainder of R-RESCALE)
  uint32_t src0, center;
};

struct RescaleConst {  // for dropping q_l
  uint64_t ql_inv[kMaxChain], ql_inv_sh[kMaxChain];  // q_l^{-1} mod q_i
};

struct DevTables {
  const double* tw;        // [chain][N] psi^{br(k)} (exact doubles, q < 2^48)
  const double* itw;       // [chain][N] psi^{-br(k)}
  const PrimeConst* pc;    // [chain]
};

}  // namespace hy

struct hy_ctx {
  int device = 0;
  uint32_t log_n = 0, N = 0, n_q = 0, n_p = 0, dnum = 0, alpha = 0, h = 0;
  std::vector<uint64_t> mod;      // chain moduli
  std::vector<uint64_t> psi;
  hy::DevTables dt{};
  void* d_tables = nullptr;       // single allocation behind dt
  // per-level constant blocks (device), index = level
  std::vector<hy::ModUpConst*> d_modup;      // [level] -> device array [beta]
  std::vector<hy::ModDownConst*> d_moddown;  // [level]
  std::vector<hy::RescaleConst*> d_rescale;  // [level] (drop q_level)
  std::vector<hy::ModDownConst*> d_rescale_md;  // [level >= 1]: rescale as a centred ModDown by q_level
  // host copies (used to fill launch parameters)
  std::vector<std::vector<hy::ModUpConst>> h_modup;
  std::vector<hy::ModDownConst> h_moddown;
  std::vector<hy::RescaleConst> h_rescale;
  // workspace
  uint8_t* ws = nullptr;
  size_t ws_bytes = 0;
  uint64_t launches = 0;
  // per-kernel-family CUDA-event timing (hy_ctx_time_kernels)
  uint32_t time_mask = 0;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  struct TimedPair {
    uint32_t fam;
    cudaEvent_t a, b;
    uint64_t bytes;  // algorithmic bytes of the bracketed launch(es)
  };
  std::vector<TimedPair> timed;
  // device CKKS-encoding tables (hy_encode_dev.cu): ksi^k as complex double-double, then 5^j mod 2N (uint32)
  void* d_enc = nullptr;
  size_t enc_rot_off = 0;
};

namespace hy {

// error plumbing
hy_status fail(hy_status s, const std::string& msg);
hy_status cuda_check(const char* what);
inline cudaStream_t st(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline uint32_t n_digits(const hy_ctx* c, uint32_t level) { return (level + 1 + c->alpha - 1) / c->alpha; }
inline uint32_t ext_chain(const hy_ctx* c, uint32_t level, uint32_t u) {
  return u <= level ? u : c->n_q + (u - level - 1);
}

// A batch of limbs for one launch: src/dst pointer and chain index per limb.
struct LimbBatch {
  const uint64_t* src[kMaxBatch];
  uint64_t* dst[kMaxBatch];
  uint8_t chain[kMaxBatch];
  int n;
};

// NTT launchers (hy_ntt.cu)
void launch_ntt(hy_ctx* c, const LimbBatch& b, bool inverse, cudaStream_t s);

// Any number of limbs as (src, dst, chain) lists, launched in LimbBatch chunks (hy_ntt.cu)
struct LimbList {
  std::vector<uint64_t*> src, dst;
  std::vector<uint8_t> chain;
  void add(const uint64_t* a, uint64_t* b, uint32_t t) {
    src.push_back(const_cast<uint64_t*>(a));
    dst.push_back(b);
    chain.push_back((uint8_t)t);
  }
};
void ntt_list(hy_ctx* c, const LimbList& L, bool inverse, cudaStream_t s);  // both passes
void rows_list(hy_ctx* c, const LimbList& L, bool inverse, cudaStream_t s);  // row pass only
void ntt_cols_list(hy_ctx* c, const LimbList& L, cudaStream_t s);            // forward column pass only
// batched rescale / mask product (hy_ops.cu); rescale outputs must not alias inputs
hy_status rescale_multi(hy_ctx* c, const uint64_t* const* cts, uint32_t n, uint32_t level, uint64_t* const* outs,
                        cudaStream_t s);
hy_status pmult_many(hy_ctx* c, const uint64_t* const* cts, uint32_t n, const uint64_t* pt, uint32_t level,
                     uint64_t* const* outs, cudaStream_t s);
// forward pass A only (the column stages); the row stages are then run by launch_ntt_rows_ip
void launch_ntt_cols(hy_ctx* c, const LimbBatch& b, cudaStream_t s);

constexpr int kG = 64;  // key switches per batched launch (upper bound; HY_KS_BATCH and the workspace set the size)

// Fused ModUp NTT row pass + key-switch inner product (hy_ntt.cu), per item g:
//   u_g[c][u] (+)= sum_j NTT_rows(ext_g[j][u]) (.) evk_g[j][c][chain(u)]   (own digit: own_g[u] as is)
// ext_g[j][u] holds the column-pass output of the digit's non-own limbs.  sum: every item accumulates
// into u[0] (lazy HRotSum).  Items with the same evk pointer reuse the key rows through L2.
struct RowsIpArgs {
  const uint64_t* ext[kG];
  const uint64_t* own[kG];
  const uint64_t* evk[kG];
  uint64_t* u[kG];
  uint64_t* v[kG];   // inv_p: [2][K][N] P limbs after the inverse row pass (between-pass format)
  uint64_t kx[kG];   // hoist: Galois element each item reads the shared NTT-domain digits through
};
// u0: first extended limb produced (0: all of Q_l u P; l+1: the P limbs only, for the split ModDown)
// inv_p (with u0 = l+1): store the P limbs after their inverse row pass into v instead (split ModDown)
// hoist: ext holds the NTT-domain digits of one shared ModUp, read through kx_g (hoisted batch)
void launch_ntt_rows_ip(hy_ctx* c, const RowsIpArgs& a, int G, uint32_t level, bool sum, bool accumulate,
                        cudaStream_t s, int u0 = 0, bool inv_p = false, bool hoist = false, int groups = 1);

// Key-switch inner product on the Q_l limbs fused with the ModDown epilogue (hy_ntt.cu), per item g,
// limb i <= level, poly c:
//   out_g[c][i] = (sum_j D_j(ext_g, own_g)[i] (.) evk_g[j][c][i] - NTT_rows(w_g[c][i])) P^{-1}
//                 (+ add0_g[i][kappa_k0(x)] for c = 0) (+ add1_g[i] for c = 1) (+ addct_g[c][i])
// where D_j is the digit's limb i in the NTT domain: plain -- the row pass of the column-pass output
// ext_g[j][i] (own digit: own_g[i] as is); hoisted -- ext_g[j][i] / own_g[i] read through the Galois
// permutation kx_g (Halevi-Shoup).  w_g is the column-pass output of the P -> Q_l conversion of the
// P limbs of the same inner product, so the Q limbs of u are never stored.  out_g may alias addct_g.
struct IpFinalArgs {
  const uint64_t* ext[kG];
  const uint64_t* own[kG];
  const uint64_t* evk[kG];
  const uint64_t* w[kG];
  const uint64_t* add0[kG];
  const uint64_t* add1[kG];
  const uint64_t* addct[kG];
  uint64_t* out[kG];
  uint64_t k0[kG];
  uint64_t kx[kG];
};
void launch_rows_ip_final(hy_ctx* c, const IpFinalArgs& a, int G, uint32_t level, bool hoisted, cudaStream_t s);

// Fused ModDown NTT row pass + epilogue (hy_ntt.cu), per item g and poly c < npoly:
//   out_g[c][i] = (u_g[c][i] - NTT_rows(w_g[c][i])) P^{-1} (+ add0_g[i][kappa_k0(x)] for c = 0)
//                 (+ add1_g[i] for c = 1) (+ addct_g[c][i]),   i <= level
// w_g[c][i] holds the column-pass output of the P -> Q_l conversion.  out_g may alias addct_g.
struct RowsFinalArgs {
  const uint64_t* u[kG];
  const uint64_t* w[kG];
  const uint64_t* add0[kG];
  const uint64_t* add1[kG];
  const uint64_t* addct[kG];
  uint64_t* out[kG];
  uint64_t k0[kG];
};
void launch_ntt_rows_final(hy_ctx* c, const RowsFinalArgs& a, int G, int npoly, uint32_t level, cudaStream_t s);

// Fused ModUp column kernel (hy_ntt.cu), per item g, digit j and 16-column strip:
//   d_i = inverse column pass of src_g[i] (i in digit j; src_g = c1 after the inverse row pass),
//   y_i = [d_i (D_j/q_i)^{-1}]_{q_i},  ext_g[j][u] = forward column pass of [sum_i y_i (D_j/q_i)]_{t_u}
// for every non-own limb u; ext is left in the between-pass format for launch_ntt_rows_ip / rows.
struct ModUpColsArgs {
  const uint64_t* src[kG];
  uint64_t* ext[kG];
};
void launch_modup_cols(hy_ctx* c, const ModUpColsArgs& a, int G, uint32_t level, cudaStream_t s);
// Device CKKS encoding (DESIGN R-ENCODE, same rounding as hy_encode_coeffs) of P real slot vectors d_slots
// [P][N/2] at integer scales h_scales[P] into NTT-domain plaintexts out + p*stride on q_0..q_{nl-1}.
// Uses ws (P * 40 * N bytes + 256); synchronous.
hy_status encode_batch_device(hy_ctx* c, const double* d_slots, const uint64_t* h_scales, uint32_t P, uint32_t nl,
                              uint64_t* out, size_t stride, uint8_t* ws, size_t ws_bytes, cudaStream_t s);
bool modup_cols_ok(const hy_ctx* c);  // N = 2^16 and alpha <= 4
// The same fused column kernel for ModDown, per item g and poly c: inverse column pass of the K P limbs
// src_g[c][k] (after their inverse row pass), z_k = [v_k (P/p_k)^{-1}]_{p_k}, and for every q_i <= level
// ext_g[c][i] = forward column pass of [sum_k z_k ((P/p_k) mod q_i)] (between-pass format).
void launch_moddown_cols(hy_ctx* c, const ModUpColsArgs& a, int G, uint32_t level, cudaStream_t s);
// Fused rescale of G ciphertexts at `level` (N = 2^16): src_g = the two last limbs after their inverse row pass
// (between-pass format, [2][N]) -> w_g [2][level][N] (column kernel, centred lift to q_0..q_{level-1}); then
// out_g[c][i] = (ct_g[c][i] - NTT(w_g[c][i])) q_level^{-1} (row kernel).
void launch_rescale_cols(hy_ctx* c, const ModUpColsArgs& a, int G, uint32_t level, cudaStream_t s);
void launch_rescale_rows_final(hy_ctx* c, const RowsFinalArgs& a, int G, uint32_t level, cudaStream_t s);
bool moddown_cols_ok(const hy_ctx* c);  // N = 2^16 and K <= 4
// Inverse row pass of kappa_{k_g}(c1_g) read straight from c1_g (the automorphism fused as a row gather),
// [l+1][N] each, into dst_g in the between-pass format (for launch_modup_cols)
struct RowsAutArgs {
  const uint64_t* src[kG];
  uint64_t* dst[kG];
  uint64_t k[kG];
};
void launch_ntt_rows_inv_aut(hy_ctx* c, const RowsAutArgs& a, int G, uint32_t level, cudaStream_t s);
// the summed (lazy HRotSum) IP runs on the bulk-copy ring (HY_SUMTMA, default on); it can read the own digit
// through kappa, so the lazy path then fuses kappa into the inverse row pass
bool sum_tma_on();
// the hoisted rotations of I ciphertexts by the same n amounts, batched (hy_keyswitch.cu); HY_E_WORKSPACE: not
// batchable here (nothing launched), call hy_hrot_hoisted per input
hy_status hrot_hoisted_multi(hy_ctx* c, const uint64_t* const* evks, const uint64_t* const* cts, uint32_t I,
                             uint32_t level, const int32_t* r, uint32_t n, uint64_t* const* outs, cudaStream_t s);
// the lazy HRotSums of O outputs over the same n rotations, batched (hy_keyswitch.cu); HY_E_WORKSPACE: not
// batchable here (nothing launched), call hy_hrot_sum per output
hy_status hrot_sum_multi(hy_ctx* c, const uint64_t* const* evks, const uint64_t* const* cts, uint32_t level,
                         const int32_t* r, uint32_t n, uint32_t O, uint64_t* const* outs, cudaStream_t s);
// one NTT row pass (forward: reads the between-pass format; inverse: writes it)
void launch_ntt_rows(hy_ctx* c, const LimbBatch& b, bool inverse, cudaStream_t s);
// convenience: contiguous [n][N] arrays with chain indices
void ntt_contig(hy_ctx* c, const uint64_t* in, uint64_t* out, const uint32_t* chain, uint32_t n, bool inverse,
                cudaStream_t s);

// elementwise / keyswitch launchers (hy_ops.cu / hy_keyswitch.cu)
// out = HRot_r(ct) (+ addct); out may alias ct and addct (hy_keyswitch.cu)
hy_status hrot_plain(hy_ctx* c, const uint64_t* evk, const uint64_t* ct, uint32_t level, int32_t r, uint64_t* out,
                     cudaStream_t s, const uint64_t* addct);
// batched plain HRot: out_g = HRot_{r_g}(ct_g) (+ addct_g); identical evk pointers share one key stream
// gal (optional): the Galois elements of the items (then r is ignored) -- any automorphism, e.g. conjugation
hy_status hrot_multi(hy_ctx* c, const uint64_t* const* evk, const uint64_t* const* ct, uint32_t level,
                     const int32_t* r, uint32_t n_items, uint64_t* const* out, const uint64_t* const* addct,
                     cudaStream_t s, const uint64_t* gal = nullptr);
// Lazy HRotSum split at its ModDown (RAConv tap sharding, hy_conv.cu):
//   hrot_sum_partial: u [2][l+1+K][N] = sum of the terms' key-switch inner products (NTT, canonical; zero if no
//                     term is switched), acc [2][l+1][N] = (sum kappa_t(c0_t), sum of the r = 0 terms' c1)
//   mod_reduce_ext:   u, acc mod q in place (after an integer sum of partials over ranks)
//   hrot_sum_finish:  out = ModDown(u) + acc
hy_status hrot_sum_partial(hy_ctx* c, const uint64_t* const* evks, const uint64_t* const* cts, uint32_t level,
                           const int32_t* r, uint32_t n, uint64_t* u, uint64_t* acc, cudaStream_t s);
hy_status mod_reduce_ext(hy_ctx* c, uint32_t level, uint64_t* u, uint64_t* acc, cudaStream_t s);
hy_status hrot_sum_finish(hy_ctx* c, uint32_t level, const uint64_t* u, const uint64_t* acc, uint64_t* out,
                          cudaStream_t s);
// workspace bytes of one batched key-switch item at `level`
size_t ks_item_bytes(const hy_ctx* c, uint32_t level);
// out (+)= sum_i ct_i (.) PRot_{k_i}(pt_i), k_i Galois elements (1 = none), PRot fused as a gather (hy_ops.cu)
hy_status pmult_acc_prot(hy_ctx* c, const uint64_t* const* cts, const uint64_t* const* pts, const uint64_t* ks,
                         uint32_t n, uint32_t level, uint64_t* out, int accumulate, void* stream);
void launch_automorph(hy_ctx* c, const uint64_t* in, uint64_t* out, uint32_t n_limbs, uint64_t k, cudaStream_t s);
// dense MulFilter&Sum block (hy_ops.cu): out_m (+)= sum_j ct_j (.) PRot_{gal[m*J+j]}(pt_base[pt_idx[m*J+j]]),
// M <= 8 outputs, any J (chunks of 64 operands)
hy_status pmult_block(hy_ctx* c, const uint64_t* const* cts, uint32_t J, uint64_t* const* outs, uint32_t M,
                      const uint64_t* pt_base, const uint32_t* pt_idx, const uint64_t* gal, uint32_t level,
                      int accumulate, void* stream);

// Kernel families for live CUDA-event timing (values of HY_FAM_* in hyphen.h).
enum Family : uint32_t {
  FAM_NTT_A = 1, FAM_NTT_B = 2, FAM_MODUP = 4, FAM_IP = 8, FAM_MODDOWN = 16, FAM_AUT = 32, FAM_ELEM = 64,
  FAM_RESCALE = 128, FAM_CLIENT = 256, FAM_NTT_IP = 512
};

inline cudaEvent_t pooled_event(hy_ctx* c) {
  if (c->ev_used == c->ev_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->ev_pool.push_back(e);
  }
  return c->ev_pool[c->ev_used++];
}

// Counts one launch (or n) and, when the family is being timed, brackets it
// with CUDA events on the launching stream.
struct KTimer {
  hy_ctx* c;
  uint32_t fam;
  cudaStream_t s;
  cudaEvent_t a = nullptr, b = nullptr;
  uint64_t bytes = 0;  // algorithmic bytes (minimal reads + writes), set by the launcher
  KTimer(hy_ctx* c_, uint32_t fam_, cudaStream_t s_, uint32_t n = 1) : c(c_), fam(fam_), s(s_) {
    c->launches += n;
    if (c->time_mask & fam) {
      a = pooled_event(c);
      b = pooled_event(c);
      cudaEventRecord(a, s);
    }
  }
  ~KTimer() {
    if (b) {
      cudaEventRecord(b, s);
      c->timed.push_back({fam, a, b, bytes});
    }
  }
};

// workspace carving
struct Ws {
  uint8_t* p;
  size_t left;
  template <class T>
  T* take(size_t count) {
    size_t bytes = (count * sizeof(T) + 255) & ~size_t(255);
    if (bytes > left) return nullptr;
    T* r = reinterpret_cast<T*>(p);
    p += bytes;
    left -= bytes;
    return r;
  }
};

}  // namespace hy
