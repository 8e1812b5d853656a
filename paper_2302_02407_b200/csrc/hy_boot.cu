// hy_boot.cu -- the linear steps of CKKS bootstrapping (partial): ModRaise and the
// homomorphic diagonal linear transform (baby-step / giant-step) that CoeffToSlot and SlotToCoeff are made of.
// EvalMod (the polynomial approximation of the modular reduction) is not built.
//
// Linear transform (DESIGN R-LINTRANS): y = sum_{d in D} diag_d (.) Rot_d(x), diag_d[j] = M[j][(j + d) mod n], so
// y = M x on the slots.  With d = g bs + b (0 <= b < bs):
//     y = sum_g Rot_{g bs}( sum_b Rot_{-g bs}(diag_{g bs + b}) (.) Rot_b(x) ),
// evaluated as: the baby steps Rot_b(x) as one hoisted HRot batch (one ModUp), the inner sums as one dense
// MulFilter&Sum block per 8 giant steps (k_pmult_block / k_pmult_ring; a missing (g, b) pair multiplies a zero
// plaintext), the giant steps as one lazy HRotSum (one ModDown for all of them, Alg. P:727-733), then a rescale:
// the plaintexts are encoded at scale q_l, so the output returns to the input scale at level l - 1.
#include <algorithm>
#include <cstring>
#include <map>
#include <vector>

#include "hy_arith.cuh"

struct hy_lintrans {
  int64_t n = 0, bs = 1;
  std::vector<int64_t> diags;                 // canonical, ascending (the encode order)
  std::vector<int64_t> babies, giants;        // b values (incl. 0 if used), g values (g bs canonical)
  std::map<std::pair<int64_t, int64_t>, int64_t> pt_of;  // (g, b) -> plaintext index
  std::vector<int64_t> rots;                  // nonzero amounts needing keys, ascending
  int64_t n_pt() const { return (int64_t)diags.size() + 1; }  // + one zero plaintext (absent pairs)
};

namespace hy {
namespace {
// out[p][i][x] = centred(v[p][x]) mod q_i, v = the coefficient-domain limb 0 (mod q_0).  grid (N/256, l+1, 2)
__global__ void k_mod_raise_lift(const uint64_t* __restrict__ v, uint64_t* __restrict__ out, DevTables dt, int level,
                                 int logN) {
  const size_t N = (size_t)1 << logN;
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y, p = blockIdx.z;
  const uint64_t q0 = dt.pc[0].q, qi = dt.pc[i].q;
  const uint64_t val = v[(size_t)p * N + x];
  uint64_t r;
  if (val > (q0 - 1) / 2) {  // negative representative val - q0
    const uint64_t m = reduce64(q0 - val, dt.pc[i]);
    r = m ? qi - m : 0;
  } else {
    r = reduce64(val, dt.pc[i]);
  }
  out[((size_t)p * (level + 1) + i) * N + x] = r;
}
}  // namespace
}  // namespace hy

using namespace hy;

extern "C" hy_status hy_mod_raise(hy_ctx* c, const uint64_t* ct0, uint32_t level, uint64_t* out, void* stream) {
  if (!c || !ct0 || !out) return fail(HY_E_ARG, "null");
  if (level >= c->n_q) return fail(HY_E_ARG, "level out of range");
  if (out == ct0) return fail(HY_E_ARG, "mod_raise cannot run in place");
  if (!c->ws || c->ws_bytes < 2ull * c->N * 8) return fail(HY_E_WORKSPACE, "workspace too small");
  cudaStream_t s = st(stream);
  uint64_t* v = reinterpret_cast<uint64_t*>(c->ws);
  const uint32_t ch0[2] = {0, 0};
  ntt_contig(c, ct0, v, ch0, 2, true, s);  // c0, c1 limb 0 -> coefficient domain
  {
    KTimer kt(c, FAM_ELEM, s);
    kt.bytes = 2ull * (1 + level + 1) * c->N * 8;
    dim3 g(c->N / 256, level + 1, 2);
    k_mod_raise_lift<<<g, 256, 0, s>>>(v, out, c->dt, (int)level, (int)c->log_n);
  }
  std::vector<uint32_t> chain(2 * (level + 1));
  for (uint32_t p = 0; p < 2; ++p)
    for (uint32_t i = 0; i <= level; ++i) chain[p * (level + 1) + i] = i;
  ntt_contig(c, out, out, chain.data(), (uint32_t)chain.size(), false, s);
  return cuda_check("hy_mod_raise");
}

extern "C" hy_status hy_lintrans_create(uint32_t log_n, const int32_t* diags, uint32_t n_diag, uint32_t bs,
                                        hy_lintrans** out) {
  if (!out || !diags || !n_diag || log_n < 4 || log_n > 17 || bs == 0) return fail(HY_E_ARG, "null / shape");
  auto* p = new hy_lintrans();
  p->n = (1ll << log_n) / 2;
  if ((int64_t)bs > p->n) {
    delete p;
    return fail(HY_E_ARG, "baby-step size above the slot count");
  }
  p->bs = bs;
  for (uint32_t k = 0; k < n_diag; ++k) p->diags.push_back((((int64_t)diags[k] % p->n) + p->n) % p->n);
  std::sort(p->diags.begin(), p->diags.end());
  if (std::adjacent_find(p->diags.begin(), p->diags.end()) != p->diags.end()) {
    delete p;
    return fail(HY_E_ARG, "repeated diagonal");
  }
  for (size_t k = 0; k < p->diags.size(); ++k) {
    const int64_t d = p->diags[k], g = d / p->bs, b = d % p->bs;
    p->pt_of[{g, b}] = (int64_t)k;
    p->babies.push_back(b);
    p->giants.push_back(g);
  }
  for (auto* v : {&p->babies, &p->giants}) {
    std::sort(v->begin(), v->end());
    v->erase(std::unique(v->begin(), v->end()), v->end());
  }
  for (int64_t b : p->babies)
    if (b) p->rots.push_back(b);
  for (int64_t g : p->giants)
    if (g) p->rots.push_back((g * p->bs) % p->n);
  std::sort(p->rots.begin(), p->rots.end());
  p->rots.erase(std::unique(p->rots.begin(), p->rots.end()), p->rots.end());
  *out = p;
  return HY_OK;
}

extern "C" void hy_lintrans_destroy(hy_lintrans* p) { delete p; }

extern "C" hy_status hy_lintrans_query(const hy_lintrans* p, uint32_t* n_pt, uint32_t* n_baby, uint32_t* n_giant,
                                       uint32_t* n_rot, int32_t* rots) {
  if (!p) return fail(HY_E_ARG, "null");
  if (n_pt) *n_pt = (uint32_t)p->n_pt();
  if (n_baby) *n_baby = (uint32_t)p->babies.size();
  if (n_giant) *n_giant = (uint32_t)p->giants.size();
  if (n_rot) *n_rot = (uint32_t)p->rots.size();
  if (rots)
    for (size_t k = 0; k < p->rots.size(); ++k) rots[k] = (int32_t)p->rots[k];
  return HY_OK;
}

extern "C" size_t hy_lintrans_pt_words(const hy_ctx* c, const hy_lintrans* p, uint32_t level) {
  if (!c || !p) return 0;
  return (size_t)p->n_pt() * (level + 1) * c->N;
}

extern "C" size_t hy_lintrans_scratch_words(const hy_ctx* c, const hy_lintrans* p, uint32_t level) {
  if (!c || !p) return 0;
  // baby-step rotations + giant-step inner sums + the HRotSum output
  return (p->babies.size() + p->giants.size() + 1) * 2ull * (level + 1) * c->N;
}

extern "C" hy_status hy_lintrans_encode(hy_ctx* c, const hy_lintrans* p, const double* re, const double* im,
                                        uint32_t level, uint64_t* d_pts, void* stream) {
  if (!c || !p || !re || !d_pts) return fail(HY_E_ARG, "null");
  if (level >= c->n_q || level < 1) return fail(HY_E_LEVEL_EXHAUSTED, "level too low");
  if (p->n != (int64_t)c->N / 2) return fail(HY_E_PLAN, "plan ring size differs from the context's");
  const size_t n = (size_t)p->n, stride = (size_t)(level + 1) * c->N;
  std::vector<double> vr(n), vi(n);
  std::vector<int64_t> coef(c->N);
  for (size_t k = 0; k < p->diags.size(); ++k) {
    // Rot_{-g bs}(diag_d): v[j] = diag[j - g bs]
    const int64_t sh = (p->diags[k] / p->bs) * p->bs;
    for (size_t j = 0; j < n; ++j) {
      const size_t src = (size_t)((((int64_t)j - sh) % p->n + p->n) % p->n);
      vr[j] = re[k * n + src];
      vi[j] = im ? im[k * n + src] : 0.0;
    }
    hy_status st = hy_encode_coeffs_complex(c->log_n, vr.data(), vi.data(), (uint32_t)n, c->mod[level], coef.data());
    if (st == HY_OK) st = hy_pt_from_coeffs(c, coef.data(), level, d_pts + k * stride, stream);
    if (st != HY_OK) return st;
  }
  cudaMemsetAsync(d_pts + p->diags.size() * stride, 0, stride * 8, st(stream));  // the zero plaintext
  return cuda_check("hy_lintrans_encode");
}

extern "C" hy_status hy_lintrans_apply(hy_ctx* c, const hy_lintrans* p, const uint64_t* const* evks,
                                       const uint64_t* ct, uint32_t level, const uint64_t* pts, uint64_t* scratch,
                                       uint64_t* out, void* stream) {
  if (!c || !p || !evks || !ct || !pts || !scratch || !out) return fail(HY_E_ARG, "null");
  if (level >= c->n_q || level < 1) return fail(HY_E_LEVEL_EXHAUSTED, "level too low");
  if (p->n != (int64_t)c->N / 2) return fail(HY_E_PLAN, "plan ring size differs from the context's");
  cudaStream_t s = st(stream);
  const size_t ct_l = 2ull * (level + 1) * c->N;
  auto key = [&](int64_t r) -> const uint64_t* {
    const int64_t rr = ((r % p->n) + p->n) % p->n;
    auto it = std::lower_bound(p->rots.begin(), p->rots.end(), rr);
    return (it != p->rots.end() && *it == rr) ? evks[it - p->rots.begin()] : nullptr;
  };
  // baby steps: one hoisted batch
  const size_t B = p->babies.size(), G = p->giants.size();
  std::vector<const uint64_t*> rotx(B);
  std::vector<int32_t> rs;
  std::vector<const uint64_t*> ks;
  std::vector<uint64_t*> outs;
  for (size_t k = 0; k < B; ++k) {
    if (p->babies[k] == 0) {
      rotx[k] = ct;
      continue;
    }
    uint64_t* o = scratch + k * ct_l;
    rotx[k] = o;
    rs.push_back((int32_t)p->babies[k]);
    ks.push_back(key(p->babies[k]));
    outs.push_back(o);
  }
  hy_status stt = HY_OK;
  if (!rs.empty()) stt = hy_hrot_hoisted(c, ks.data(), ct, level, rs.data(), (uint32_t)rs.size(), outs.data(), stream);
  if (stt != HY_OK) return stt;
  // giant-step inner sums, dense blocks of <= 8 giant steps over every baby step
  uint64_t* inner = scratch + B * ct_l;
  std::vector<uint32_t> idx;
  std::vector<uint64_t> gal;
  for (size_t g0 = 0; g0 < G; g0 += 8) {
    const size_t M = std::min<size_t>(8, G - g0);
    idx.assign(M * B, (uint32_t)p->diags.size());  // absent pairs: the zero plaintext
    gal.assign(M * B, 1);
    std::vector<uint64_t*> o(M);
    for (size_t m = 0; m < M; ++m) {
      o[m] = inner + (g0 + m) * ct_l;
      for (size_t k = 0; k < B; ++k) {
        auto it = p->pt_of.find({p->giants[g0 + m], p->babies[k]});
        if (it != p->pt_of.end()) idx[m * B + k] = (uint32_t)it->second;
      }
    }
    stt = pmult_block(c, rotx.data(), (uint32_t)B, o.data(), (uint32_t)M, pts, idx.data(), gal.data(), level, 0,
                      stream);
    if (stt != HY_OK) return stt;
  }
  // giant steps: one lazy HRotSum, then the rescale
  std::vector<const uint64_t*> gin(G), gks(G);
  std::vector<int32_t> grs(G);
  for (size_t m = 0; m < G; ++m) {
    gin[m] = inner + m * ct_l;
    grs[m] = (int32_t)((p->giants[m] * p->bs) % p->n);
    gks[m] = grs[m] ? key(grs[m]) : nullptr;
  }
  uint64_t* sum = inner + G * ct_l;
  stt = hy_hrot_sum(c, gks.data(), gin.data(), level, grs.data(), (uint32_t)G, sum, stream);
  if (stt != HY_OK) return stt;
  stt = hy_rescale(c, sum, level, out, stream);
  if (stt != HY_OK) return stt;
  return cuda_check("hy_lintrans_apply");
}
