// hy_conv.cu -- HyPHEN convolution layers on the device: CAConv and
// RAConv_Reorder over 2D-gap packed ciphertexts, including
// stride-2 downsampling (Fig. 2(d)) -- the plan (rotation amounts, weight and mask
// slot vectors) is built on the host, every homomorphic step runs in the library's
// kernels (hoisted HRot, PMult-accumulate, lazy HRotSum, rescale, HRot+add).
//
// Slot layout (DESIGN.md R-LAYOUT): physical width W_p, gap g, cell kappa in [0, m d)
// with low->high digits (g_c, g_r, e_idx) at slot offsets (1, W_p, W_p^2); channel block
// size B = e W_p^2 (e = m d / g^2), c_n = n / B blocks.
//   CA(m, d): mu = kappa % m, rho = kappa / m; ciphertext i holds channel i c_n m + b m + mu.
//   RA(m, d): mu = kappa / d, rho = kappa % d; ciphertext i holds channel i m + mu in every block.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <vector>

#include "hy_internal.h"

namespace {

int lg2(uint64_t x) {
  int v = 0;
  while ((1ull << v) < x) ++v;
  return v;
}
bool pow2(uint64_t x) { return x && !(x & (x - 1)); }

struct Layout {
  bool ca;
  int64_t n, wp, g, m, d;
  int64_t S = 1;  // PRCR row segments (pi_CA' when ca && S > 1)
  int64_t I() const { return wp * wp; }
  int64_t F() const { return I() / S; }  // slots per row segment (fragment)
  int64_t e() const { return m * d / (g * g); }
  int64_t B() const { return e() * I(); }
  int64_t cn() const { return n / B(); }
  // slot distance of cell bit k
  int64_t stride(int k) const {
    const int lgg = lg2(g);
    if (k < lgg) return 1ll << k;
    if (k < 2 * lgg) return wp << (k - lgg);
    return I() << (k - 2 * lgg);
  }
  struct Pos {
    int64_t b, h, w, kappa;
  };
  Pos at(int64_t s) const {
    const int64_t b = s / B(), r = s % B();
    const int64_t ei = r / I(), pr = (r % I()) / wp, pc = r % wp;
    return {b, pr / g, pc / g, (pc % g) + g * ((pr % g) + g * ei)};
  }
  int64_t mu(int64_t kappa) const { return ca ? kappa % m : kappa / d; }
  int64_t rho(int64_t kappa) const { return ca ? kappa / m : kappa % d; }
  // pi_CA' (PRCR): member im of family k holds, at global row segment G = slot / F, rows of channel
  // k c_n S m + ((G + im) mod c_n S) m + mu -- fragments organised circularly
  int64_t channel(int64_t ct, const Pos& p, int64_t slot) const {
    if (!ca) return ct * m + mu(p.kappa);
    if (S > 1) {
      const int64_t fam = ct / S, im = ct % S, G = slot / F();
      return fam * cn() * S * m + ((G + im) % (cn() * S)) * m + mu(p.kappa);
    }
    return ct * cn() * m + p.b * m + mu(p.kappa);
  }
  int64_t cts_for(int64_t c) const {
    if (ca && S > 1) return S * ((c + cn() * S * m - 1) / (cn() * S * m));
    const int64_t per = ca ? cn() * m : m;
    return (c + per - 1) / per;
  }
};

}  // namespace

// A limited rotation-key set: the loaded amounts and, over Z_n, the breadth-first tree from 0
// whose edges are the loaded amounts (DESIGN R-KEYSET): the shortest decomposition of any amount into loaded ones,
// ties broken by discovery order (FIFO queue, amounts ascending).
struct hy_keyset {
  int64_t n = 0;
  std::vector<int64_t> loaded;          // ascending, canonical in (0, n)
  std::vector<int32_t> parent_amount;   // per node: the loaded amount of its tree edge (-1: root / unreached)
  std::vector<int32_t> parent;          // per node: its tree parent
  std::vector<int64_t> steps(int64_t r) const {  // application order; empty if unreachable (r != 0)
    std::vector<int64_t> out;
    int64_t v = ((r % n) + n) % n;
    while (v != 0) {
      if (parent_amount[v] < 0) return {};
      out.push_back(parent_amount[v]);
      v = parent[v];
    }
    std::reverse(out.begin(), out.end());
    return out;
  }
};

struct hy_conv_plan {
  hy_conv_spec s;
  int64_t n, pad, wo;
  Layout in, out;
  std::vector<int64_t> taps;
  int64_t n_in, n_groups, n_out;
  std::vector<int64_t> ras, ras_g, ir_g;
  bool has_mask = false, has_combine = false;
  bool has_bias = false;  // AddPt of a per-output-channel bias after the layer (DESIGN R-BIAS)
  int64_t combine = 0;
  std::vector<int64_t> rots;  // distinct nonzero rotation amounts mod n (key order)
  uint32_t counts[5] = {0, 0, 0, 0, 0};
  // limited key set (hy_conv_plan_set_keyset): amount -> its loaded steps, for every non-Slide amount that is not
  // loaded itself (empty map: every key the plan needs is loaded); eff_counts = counts with those rotations
  // counted once per step ("eff. total")
  std::map<int64_t, std::vector<int64_t>> decomp;
  uint32_t eff_counts[5] = {0, 0, 0, 0, 0};
  std::vector<int64_t> steps_of(int64_t r) const {
    const int64_t rr = ((r % n) + n) % n;
    auto it = decomp.find(rr);
    if (it != decomp.end()) return it->second;
    return {r};
  }
  int64_t S = 1;              // PRCR segments
  int64_t f2() const { return (int64_t)s.f * s.f; }
  // stored weight plaintexts: CA [group][input or family][tap]; RA [output or family][input][tap]
  int64_t n_w_in() const { return s.algo == HY_CONV_CA ? n_in / S : n_in; }
  int64_t n_w_grp() const { return s.algo == HY_CONV_CA ? n_groups : n_groups / S; }
  int64_t n_pt() const { return n_w_grp() * n_w_in() * f2(); }
  // device words of the weight buffer before the bias plaintexts: n_pt x [l+1][N], then the mask [l][N]
  size_t bias_offset(uint32_t level, size_t N) const {
    return ((size_t)n_pt() * (level + 1) + (has_mask ? level : 0)) * N;
  }
  uint32_t out_level(uint32_t level) const { return level - 1 - (has_mask ? 1 : 0); }
  // (stored plaintext index, PRot amount) of term (group/output grp, input ct i, tap t):
  // PRCR shares one plaintext per family, member im using PRot(P, r_t + im F) on the CA input
  // side and PRot(P, im F - r_t) on the RA output side (DESIGN R-PRCR)
  std::pair<int64_t, int64_t> term(int64_t grp, int64_t i, int64_t t) const {
    if (S == 1) return {(grp * n_in + i) * f2() + t, 0};
    if (s.algo == HY_CONV_CA) return {(grp * n_w_in() + i / S) * f2() + t, taps[t] + (i % S) * in.F()};
    return {((grp / S) * n_in + i) * f2() + t, (grp % S) * out.F() - taps[t]};
  }
};

namespace {

int64_t tap_amount(const hy_conv_plan& p, int j1, int j2) {
  return ((int64_t)j1 - p.pad) * p.s.gap * p.s.wp + ((int64_t)j2 - p.pad) * p.s.gap;
}

// weight slot vector of plaintext idx (or the mask when idx == n_pt)
void weight_slots(const hy_conv_plan& p, const double* K, int64_t idx, double* v) {
  const hy_conv_spec& s = p.s;
  const int64_t f2 = (int64_t)s.f * s.f;
  if (idx == p.n_pt()) {  // IR_g mask
    for (int64_t x = 0; x < p.n; ++x) {
      bool keep;
      if (s.algo == HY_CONV_CA && s.stride == 1) {
        const Layout::Pos q = p.in.at(x);
        keep = p.in.mu(q.kappa) == 0 && (p.S == 1 || (q.h < p.wo && q.w < p.wo));  // PRCR: valid outputs
      } else if (s.algo == HY_CONV_CA) {  // dsconv: new-cell bits [0, lg m), lg g, 2 lg g + 1 all zero
        const int64_t k2 = p.out.at(x).kappa;
        const int lgg = lg2(s.gap);
        keep = true;
        for (int k = 0; k < lg2(s.m); ++k) keep &= !((k2 >> k) & 1);
        keep &= !((k2 >> lgg) & 1) && !((k2 >> (2 * lgg + 1)) & 1);
      } else {
        const Layout::Pos q = p.out.at(x);
        keep = p.out.rho(q.kappa) == 0 && (p.S == 1 || (q.h < p.wo && q.w < p.wo));
      }
      v[x] = keep ? 1.0 : 0.0;
    }
    return;
  }
  const int64_t t = idx % f2, i = (idx / f2) % p.n_w_in(), grp = idx / f2 / p.n_w_in();
  const int j1 = (int)(t / s.f), j2 = (int)(t % s.f);
  auto K_at = [&](int64_t o, int64_t c) { return K[((o * s.ci + c) * s.f + j1) * s.f + j2]; };
  std::fill(v, v + p.n, 0.0);
  if (p.S > 1) {
    // PRCR: member-0 view, no pixel masks -- out-of-image sources read zero padding and invalid
    // outputs are zeroed by the mask step (DESIGN R-PRCR).  CA: grp = group, i = family;
    // RA: grp = output family, i = input ciphertext.
    for (int64_t x = 0; x < p.n; ++x) {
      const int64_t G = x / p.in.F();
      if (s.algo == HY_CONV_CA) {
        const Layout::Pos q = p.in.at(x);
        const int64_t mu = p.in.mu(q.kappa), rho = p.in.rho(q.kappa);
        const int64_t c = i * p.in.cn() * p.S * s.m + G * s.m + mu, o = grp * s.d + rho;
        if (c < s.ci && o < s.co) v[x] = K_at(o, c);
      } else {
        const Layout::Pos q = p.out.at(x);
        const int64_t mu = p.out.mu(q.kappa), rho = p.out.rho(q.kappa);
        const int64_t oc = grp * p.out.cn() * p.S * p.out.m + G * p.out.m + mu, c = i * s.m + rho;
        if (c < s.ci && oc < s.co) v[x] = K_at(oc, c);
      }
    }
    return;
  }
  if (s.algo == HY_CONV_CA) {
    for (int64_t x = 0; x < p.n; ++x) {
      const Layout::Pos q = p.in.at(x);
      const int64_t mu = p.in.mu(q.kappa), rho = p.in.rho(q.kappa);
      const int64_t c = i * p.in.cn() * s.m + q.b * s.m + mu;
      int64_t o;
      bool out_ok;
      if (s.stride == 1) {
        o = grp * s.d + rho;
        out_ok = q.h < p.wo && q.w < p.wo;
      } else {
        const int64_t lo = rho % s.gap, hi = rho / s.gap;
        o = (grp / 2) * (2 * (int64_t)s.d) + lo + (int64_t)s.gap * (grp & 1) + 2 * (int64_t)s.gap * hi;
        out_ok = !(q.h & 1) && !(q.w & 1) && q.h / 2 < p.wo && q.w / 2 < p.wo;
      }
      const int64_t sh = q.h + j1 - p.pad, sw = q.w + j2 - p.pad;
      if (out_ok && sh >= 0 && sh < s.w && sw >= 0 && sw < s.w && c < s.ci && o < s.co) v[x] = K_at(o, c);
    }
  } else {
    // RAConv: plain SISO weight W for output ct grp, then inversely rotated W' = Rot_{-r_t}(W) (Alg. 2)
    const int64_t r = p.taps[t];
    for (int64_t x = 0; x < p.n; ++x) {
      const Layout::Pos q = p.out.at(x);
      const int64_t mu = p.out.mu(q.kappa), rho = p.out.rho(q.kappa);
      const int64_t oc = grp * p.out.cn() * p.out.m + q.b * p.out.m + mu;
      const int64_t c = i * s.m + rho;
      const int64_t sh = q.h + j1 - p.pad, sw = q.w + j2 - p.pad;
      if (q.h < p.wo && q.w < p.wo && sh >= 0 && sh < s.w && sw >= 0 && sw < s.w && c < s.ci && oc < s.co)
        v[((x + r) % p.n + p.n) % p.n] = K_at(oc, c);  // W'[x + r] = W[x]
    }
  }
}

// bias slot vector of output ciphertext j: b[c] at every valid slot (pixel inside the wo x wo output, every
// replica) of output channel c in the layer's output format, 0 elsewhere -- the output format's packing of the
// image B[c][h][w] = b[c] (DESIGN R-BIAS), so AddPt of it adds the conv bias of Y = conv2d(X, K) + b
void bias_slots(const hy_conv_plan& p, const double* bias, int64_t j, double* v) {
  for (int64_t x = 0; x < p.n; ++x) {
    const Layout::Pos q = p.out.at(x);
    const int64_t c = p.out.channel(j, q, x);
    v[x] = (q.h < p.wo && q.w < p.wo && c < (int64_t)p.s.co) ? bias[c] : 0.0;
  }
}

// ------------------------------------------------------------------ device orchestration
struct Ctx {
  hy_ctx* c;
  const hy_conv_plan* p;
  const uint64_t* const* evks;
  cudaStream_t s;
  const uint64_t* key(int64_t r) const {
    const int64_t rr = ((r % p->n) + p->n) % p->n;
    auto it = std::lower_bound(p->rots.begin(), p->rots.end(), rr);
    return (it != p->rots.end() && *it == rr) ? evks[it - p->rots.begin()] : nullptr;
  }
};

// out_g = HRot_r(in_g) (+ addct_g) for all g at once -- one batched HRot per loaded step of r (an
// amount whose key is not loaded is synthesized from loaded ones, HRot_{a+b} = HRot_a o HRot_b); the intermediate
// steps ping-pong through tmp_a / tmp_b (G ciphertexts each, tmp_stride words apart), the last step adds addct.
// Same aliasing rules as hrot_multi (out may alias in and addct).
hy_status hrot_steps(const Ctx& x, int64_t r, uint32_t level, const std::vector<const uint64_t*>& in,
                     const std::vector<uint64_t*>& out, const std::vector<const uint64_t*>* addct, uint64_t* tmp_a,
                     uint64_t* tmp_b, size_t tmp_stride) {
  const size_t G = in.size();
  const std::vector<int64_t> steps = x.p->steps_of(r);
  if (steps.size() > 1 && (!tmp_a || !tmp_b)) return hy::fail(HY_E_WORKSPACE, "no scratch for a synthesized rotation");
  std::vector<const uint64_t*> cur(in);
  for (size_t k = 0; k < steps.size(); ++k) {
    const bool last = k + 1 == steps.size();
    std::vector<uint64_t*> dst(G);
    for (size_t g = 0; g < G; ++g) dst[g] = last ? out[g] : ((k & 1) ? tmp_b : tmp_a) + g * tmp_stride;
    std::vector<const uint64_t*> keys(G, x.key(steps[k]));
    std::vector<int32_t> rr(G, (int32_t)steps[k]);
    hy_status st = hy::hrot_multi(x.c, keys.data(), cur.data(), level, rr.data(), (uint32_t)G, dst.data(),
                                  last && addct ? addct->data() : nullptr, x.s);
    if (st != HY_OK) return st;
    cur.assign(dst.begin(), dst.end());
  }
  return HY_OK;
}

// x_g += HRot_r(x_g) for every r in rs, in order, for all ciphertexts x_g at once: each step is one
// batched HRot whose evaluation key is shared by every item (RaS / RaS_g / IR_g)
// tmp (optional): v.size() scratch ciphertexts (stride tmp_stride words): the steps ping-pong between v and tmp
// (out = in + HRot(in) never aliases its input, so the key switch reads c1 / c0 through kappa without first
// copying the permuted ciphertext), and an odd final position is copied back into v.  syn_a / syn_b (limited key
// sets): v.size() scratch ciphertexts each, syn_stride words apart, for the intermediate steps of synthesized
// rotations.
hy_status ras_all(const Ctx& x, const std::vector<uint64_t*>& v, uint32_t level, const std::vector<int64_t>& rs,
                  uint64_t* tmp = nullptr, size_t tmp_stride = 0, uint64_t* syn_a = nullptr,
                  uint64_t* syn_b = nullptr, size_t syn_stride = 0) {
  if (v.empty() || rs.empty()) return HY_OK;
  const size_t G = v.size(), bytes = 2ull * (level + 1) * x.c->N * 8;
  std::vector<uint64_t*> cur(v.begin(), v.end()), nxt(G);
  for (size_t g = 0; g < G; ++g) nxt[g] = tmp ? tmp + g * tmp_stride : v[g];
  for (int64_t r : rs) {
    std::vector<const uint64_t*> in_c(cur.begin(), cur.end());
    hy_status st = hrot_steps(x, r, level, in_c, nxt, &in_c, syn_a, syn_b, syn_stride);
    if (st != HY_OK) return st;
    if (tmp) std::swap(cur, nxt);
  }
  if (tmp && cur[0] != v[0])
    for (size_t g = 0; g < G; ++g) cudaMemcpyAsync(v[g], cur[g], bytes, cudaMemcpyDeviceToDevice, x.s);
  return HY_OK;
}

// out_g = Rescale(ct_g (.) mask) for all g, in blocks of `blk` through the temporaries tmp[0..blk-1] (one
// batched PMult and one batched rescale per block: the rescale's grids are too small to fill the GPU for a few
// ciphertexts at a low level)
hy_status mask_rescale(const Ctx& x, const std::vector<uint64_t*>& v, const uint64_t* mask, uint32_t level,
                       uint64_t* tmp, size_t tmp_stride, const std::vector<uint64_t*>& outs, size_t blk = 8) {
  for (size_t g0 = 0; g0 < v.size(); g0 += blk) {
    const size_t M = std::min<size_t>(blk, v.size() - g0);
    std::vector<const uint64_t*> in(v.begin() + g0, v.begin() + g0 + M);
    std::vector<uint64_t*> t(M);
    for (size_t m = 0; m < M; ++m) t[m] = tmp + m * tmp_stride;
    hy_status st = hy::pmult_many(x.c, in.data(), (uint32_t)M, mask, level, t.data(), x.s);
    if (st == HY_OK) {
      std::vector<const uint64_t*> tc(t.begin(), t.end());
      st = hy::rescale_multi(x.c, tc.data(), (uint32_t)M, level, outs.data() + g0, x.s);
    }
    if (st != HY_OK) return st;
  }
  return HY_OK;
}

}  // namespace

using namespace hy;

extern "C" hy_status hy_conv_plan_create(uint32_t log_n, const hy_conv_spec* spec, hy_conv_plan** out) {
  if (!spec || !out || log_n < 4 || log_n > 17) return fail(HY_E_ARG, "null / log_n");
  const hy_conv_spec& s = *spec;
  if (s.f % 2 == 0 || s.f == 0 || (s.stride != 1 && s.stride != 2) || !s.ci || !s.co || !s.w)
    return fail(HY_E_SHAPE, "conv spec: odd f, stride 1 or 2, nonzero sizes");
  if (!pow2(s.wp) || !pow2(s.gap) || !pow2(s.m) || !pow2(s.d)) return fail(HY_E_FORMAT, "W_p, g, m, d must be powers of two");
  if ((uint64_t)s.m * s.d % ((uint64_t)s.gap * s.gap)) return fail(HY_E_FORMAT, "m d must be a multiple of g^2");
  if ((uint64_t)s.w * s.gap > s.wp) return fail(HY_E_CAPACITY, "image does not fit the physical width");
  auto* p = new hy_conv_plan();
  p->s = s;
  p->n = (1ll << log_n) / 2;
  p->pad = (s.f - 1) / 2;
  p->wo = (s.w + s.stride - 1) / s.stride;
  const int64_t e = (int64_t)s.m * s.d / ((int64_t)s.gap * s.gap);
  if ((int64_t)s.wp * s.wp * e > p->n || p->n % ((int64_t)s.wp * s.wp * e)) {
    delete p;
    return fail(HY_E_CAPACITY, "channel block does not divide the slot count");
  }
  p->S = s.segments > 1 ? s.segments : 1;
  p->has_bias = s.bias != 0;
  if (p->S > 1) {  // PRCR preconditions (DESIGN R-PRCR)
    const char* why = nullptr;
    if (!pow2(p->S) || (s.wp / s.gap) % p->S) why = "PRCR: |S| must be a power of two dividing wp/gap";
    else if (e != 1) why = "PRCR: needs m d = g^2 (e = 1)";
    else if (s.stride != 1) why = "PRCR: stride 1 only";
    else if ((int64_t)s.wp / s.gap < (int64_t)s.w + p->pad) why = "PRCR: needs (f-1)/2 rows/columns of zero padding";
    if (why) {
      delete p;
      return fail(HY_E_FORMAT, why);
    }
  }
  if (s.algo == HY_CONV_CA) {
    p->in = Layout{true, p->n, s.wp, s.gap, s.m, s.d, p->S};
    if (s.stride == 1) {
      p->out = Layout{false, p->n, s.wp, s.gap, s.d, s.m};
    } else {
      if (s.m != s.gap) {
        delete p;
        return fail(HY_E_FORMAT, "stride-2 CAConv needs m == g (DESIGN R-DSCONV)");
      }
      p->out = Layout{false, p->n, s.wp, 2 * (int64_t)s.gap, 2 * (int64_t)s.d, 2 * (int64_t)s.m};
    }
    p->n_in = p->in.cts_for(s.ci);
    p->n_groups = (s.co + s.d - 1) / s.d;
    if (s.stride == 2) p->n_groups += p->n_groups % 2;
    for (int k = 0; k < lg2(p->in.cn()); ++k) p->ras.push_back(p->in.B() << k);
    for (int k = 0; k < lg2(s.m); ++k) p->ras_g.push_back(p->in.stride(k));
    if (s.stride == 1) {
      p->n_out = p->n_groups;
      p->has_mask = s.m > 1 || p->S > 1;  // PRCR also zeroes invalid output pixels in the mask step
      for (int k = 0; k < lg2(s.m); ++k) p->ir_g.push_back(-p->in.stride(k));
    } else {
      const int lgg = lg2(s.gap);
      p->n_out = p->n_groups / 2;
      p->has_mask = true;
      p->has_combine = true;
      p->combine = -p->out.stride(2 * lgg + 1);
      for (int k = 0; k <= lgg; ++k) p->ir_g.push_back(-p->out.stride(k));
    }
  } else {
    if (s.stride != 1) {
      delete p;
      return fail(HY_E_FORMAT, "RAConv is stride 1 (downsampling happens in CAConv)");
    }
    p->in = Layout{false, p->n, s.wp, s.gap, s.m, s.d, p->S};
    p->out = Layout{true, p->n, s.wp, s.gap, s.d, s.m, p->S};
    p->n_in = p->in.cts_for(s.ci);
    p->n_out = p->n_groups = p->out.cts_for(s.co);
    for (int k = 0; k < lg2(p->out.d); ++k) p->ras_g.push_back(p->out.stride(lg2(p->out.m) + k));
    p->has_mask = p->out.d > 1 || p->S > 1;
    for (int64_t r : p->ras_g) p->ir_g.push_back(-r);
  }
  for (uint32_t j1 = 0; j1 < s.f; ++j1)
    for (uint32_t j2 = 0; j2 < s.f; ++j2) p->taps.push_back(tap_amount(*p, j1, j2));
  std::vector<int64_t> all = p->taps;
  all.insert(all.end(), p->ras.begin(), p->ras.end());
  all.insert(all.end(), p->ras_g.begin(), p->ras_g.end());
  all.insert(all.end(), p->ir_g.begin(), p->ir_g.end());
  if (p->has_combine) all.push_back(p->combine);
  for (int64_t r : all) {
    const int64_t rr = ((r % p->n) + p->n) % p->n;
    if (rr) p->rots.push_back(rr);
  }
  std::sort(p->rots.begin(), p->rots.end());
  p->rots.erase(std::unique(p->rots.begin(), p->rots.end()), p->rots.end());
  int64_t nz_taps = 0;
  for (int64_t r : p->taps) nz_taps += (r % p->n) != 0;
  const bool ca = s.algo == HY_CONV_CA;
  p->counts[0] = (uint32_t)(nz_taps * (ca ? p->n_in : p->n_out));
  p->counts[1] = (uint32_t)(p->ras.size() * p->n_groups);
  p->counts[2] = (uint32_t)(p->ras_g.size() * p->n_groups);
  p->counts[3] = (uint32_t)(p->ir_g.size() * p->n_out + (p->has_combine ? p->n_out : 0));
  p->counts[4] = (uint32_t)(p->n_groups * p->n_in * p->f2());  // PMult terms (PRCR reuses plaintexts)
  memcpy(p->eff_counts, p->counts, sizeof(p->counts));
  *out = p;
  return HY_OK;
}

extern "C" void hy_conv_plan_destroy(hy_conv_plan* p) { delete p; }

// ------------------------------------------------------------------ limited key sets (DESIGN R-KEYSET)
extern "C" hy_status hy_keyset_create(uint32_t log_n, const int32_t* amounts, uint32_t n_amounts, hy_keyset** out) {
  if (!out || (!amounts && n_amounts) || log_n < 4 || log_n > 17) return fail(HY_E_ARG, "null / log_n");
  auto* k = new hy_keyset();
  k->n = (1ll << log_n) / 2;
  for (uint32_t i = 0; i < n_amounts; ++i) {
    const int64_t r = (((int64_t)amounts[i] % k->n) + k->n) % k->n;
    if (r) k->loaded.push_back(r);
  }
  std::sort(k->loaded.begin(), k->loaded.end());
  k->loaded.erase(std::unique(k->loaded.begin(), k->loaded.end()), k->loaded.end());
  // breadth-first search from 0 over Z_n, edges = the loaded amounts in ascending order, FIFO queue: the first
  // discovery of a node fixes its parent (the shortest decomposition, deterministic tie-break)
  k->parent.assign(k->n, -1);
  k->parent_amount.assign(k->n, -1);
  std::vector<int64_t> q;
  q.reserve(k->n);
  std::vector<char> seen(k->n, 0);
  seen[0] = 1;
  q.push_back(0);
  for (size_t h = 0; h < q.size(); ++h) {
    const int64_t u = q[h];
    for (int64_t a : k->loaded) {
      const int64_t v = (u + a) % k->n;
      if (seen[v]) continue;
      seen[v] = 1;
      k->parent[v] = (int32_t)u;
      k->parent_amount[v] = (int32_t)a;
      q.push_back(v);
    }
  }
  *out = k;
  return HY_OK;
}

extern "C" void hy_keyset_destroy(hy_keyset* k) { delete k; }

extern "C" hy_status hy_keyset_decompose(const hy_keyset* k, int32_t r, int32_t* steps, uint32_t max_steps,
                                         uint32_t* n_steps) {
  if (!k || !n_steps) return fail(HY_E_ARG, "null");
  const std::vector<int64_t> st = k->steps(r);
  if (st.empty() && (((int64_t)r % k->n) + k->n) % k->n) return fail(HY_E_MISSING_KEY, "amount not reachable");
  *n_steps = (uint32_t)st.size();
  if (steps) {
    if (st.size() > max_steps) return fail(HY_E_ARG, "steps buffer too small");
    for (size_t i = 0; i < st.size(); ++i) steps[i] = (int32_t)st[i];
  }
  return HY_OK;
}

extern "C" hy_status hy_conv_plan_set_keyset(hy_conv_plan* p, const hy_keyset* k) {
  if (!p) return fail(HY_E_ARG, "null plan");
  p->decomp.clear();
  // rebuild the key list from the plan's amounts: Slide taps must be loaded (they are hoisted: one ModUp shared
  // by the tap rotations); every other amount is used directly when loaded, else through its decomposition
  std::vector<int64_t> keys;
  auto canon = [&](int64_t r) { return ((r % p->n) + p->n) % p->n; };
  for (int64_t t : p->taps) {
    const int64_t rr = canon(t);
    if (!rr) continue;
    if (k && !std::binary_search(k->loaded.begin(), k->loaded.end(), rr))
      return fail(HY_E_MISSING_KEY, "a Slide (tap) amount is not in the key set");
    keys.push_back(rr);
  }
  std::vector<int64_t> other = p->ras;
  other.insert(other.end(), p->ras_g.begin(), p->ras_g.end());
  other.insert(other.end(), p->ir_g.begin(), p->ir_g.end());
  if (p->has_combine) other.push_back(p->combine);
  for (int64_t r : other) {
    const int64_t rr = canon(r);
    if (!rr) continue;
    if (!k || std::binary_search(k->loaded.begin(), k->loaded.end(), rr)) {
      keys.push_back(rr);
      continue;
    }
    if (k->n != p->n) return fail(HY_E_PLAN, "key set ring size differs from the plan's");
    const std::vector<int64_t> st = k->steps(rr);
    if (st.empty()) return fail(HY_E_MISSING_KEY, "an amount cannot be synthesized from the key set");
    p->decomp[rr] = st;
    keys.insert(keys.end(), st.begin(), st.end());
  }
  std::sort(keys.begin(), keys.end());
  keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
  p->rots = keys;
  // effective counts: each rotation counted once per step
  auto eff = [&](const std::vector<int64_t>& rs) {
    int64_t c = 0;
    for (int64_t r : rs) c += (int64_t)p->steps_of(r).size() * (canon(r) != 0);
    return c;
  };
  p->eff_counts[0] = p->counts[0];
  p->eff_counts[1] = (uint32_t)(eff(p->ras) * p->n_groups);
  p->eff_counts[2] = (uint32_t)(eff(p->ras_g) * p->n_groups);
  p->eff_counts[3] = (uint32_t)(eff(p->ir_g) * p->n_out + (p->has_combine ? eff({p->combine}) * p->n_out : 0));
  p->eff_counts[4] = p->counts[4];
  return HY_OK;
}

extern "C" hy_status hy_conv_plan_eff_counts(const hy_conv_plan* p, uint32_t* counts) {
  if (!p || !counts) return fail(HY_E_ARG, "null");
  memcpy(counts, p->eff_counts, sizeof(p->eff_counts));
  return HY_OK;
}

extern "C" hy_status hy_conv_plan_query(const hy_conv_plan* p, uint32_t* n_in, uint32_t* n_out, uint32_t* n_pt,
                                        uint32_t* has_mask, uint32_t* n_rot, int32_t* rots, uint32_t* counts) {
  if (!p) return fail(HY_E_ARG, "null plan");
  if (n_in) *n_in = (uint32_t)p->n_in;
  if (n_out) *n_out = (uint32_t)p->n_out;
  if (n_pt) *n_pt = (uint32_t)p->n_pt();
  if (has_mask) *has_mask = p->has_mask;
  if (n_rot) *n_rot = (uint32_t)p->rots.size();
  if (rots)
    for (size_t i = 0; i < p->rots.size(); ++i) rots[i] = (int32_t)p->rots[i];
  if (counts) memcpy(counts, p->counts, sizeof(p->counts));
  return HY_OK;
}

extern "C" hy_status hy_conv_weight_slots(const hy_conv_plan* p, const double* K, uint32_t idx, double* slots) {
  if (!p || !K || !slots) return fail(HY_E_ARG, "null");
  if ((int64_t)idx > p->n_pt() || ((int64_t)idx == p->n_pt() && !p->has_mask)) return fail(HY_E_ARG, "index");
  weight_slots(*p, K, idx, slots);
  return HY_OK;
}

extern "C" hy_status hy_conv_bias_slots(const hy_conv_plan* p, const double* bias, uint32_t out_index,
                                        double* slots) {
  if (!p || !bias || !slots) return fail(HY_E_ARG, "null");
  if ((int64_t)out_index >= p->n_out) return fail(HY_E_ARG, "output index");
  bias_slots(*p, bias, out_index, slots);
  return HY_OK;
}

extern "C" size_t hy_conv_weight_words(const hy_ctx* c, const hy_conv_plan* p, uint32_t level) {
  if (!c || !p || level < 1u + (p->has_mask ? 1u : 0u)) return 0;
  return p->bias_offset(level, c->N) + (p->has_bias ? (size_t)p->n_out * (p->out_level(level) + 1) * c->N : 0);
}

extern "C" size_t hy_conv_scratch_words(const hy_ctx* c, const hy_conv_plan* p, uint32_t level) {
  if (!c || !p) return 0;
  const size_t ct = 2ull * (level + 1) * c->N;
  const size_t f2 = (size_t)p->s.f * p->s.f;
  // CA: slid inputs + acc + (up to) two ciphertexts per SISO group (group sums, masked groups)
  // (8 = one block of MulFilter&Sum accumulators)
  // (+ n_groups ping-pong ciphertexts for the RaS / RaS_g / IR_g steps)
  // (+ 2 n_groups for the intermediate steps of synthesized rotations with a limited key set)
  // (the accumulators: one per group, at least 8, so that all groups are rescaled in one batched call)
  if (p->s.algo == HY_CONV_CA)
    return (p->n_in * f2 + std::max<size_t>(8, p->n_groups) + (p->decomp.empty() ? 3 : 5) * p->n_groups) * ct;
  return (std::max<size_t>(p->n_out * (f2 + 1), 6) + 8) * ct;     // tap accumulators + one sum per output
}

extern "C" hy_status hy_conv_encode_weights(hy_ctx* c, const hy_conv_plan* p, const double* K, const double* bias,
                                            uint64_t bias_scale, uint32_t level, uint64_t* d_pts, void* stream) {
  if (!c || !p || !K || !d_pts) return fail(HY_E_ARG, "null");
  if (level >= c->n_q || level < 1u + (p->has_mask ? 1u : 0u)) return fail(HY_E_LEVEL_EXHAUSTED, "level too low");
  if (p->n != (int64_t)c->N / 2) return fail(HY_E_PLAN, "plan ring size differs from the context's");
  if (p->has_bias && (!bias || bias_scale == 0)) return fail(HY_E_ARG, "the plan adds a bias: bias and its scale needed");
  if (!c->ws) return fail(HY_E_WORKSPACE, "workspace not set");
  // Slot vectors are built on the host (the plan's weight placement, OpenMP), uploaded in batches and
  // encoded on the device (hy_encode_dev.cu; the same rounding as hy_encode_coeffs, DESIGN R-ENCODE).
  // Weights at scale q_level, the mask at q_{level-1}: each rescale restores the ciphertext scale; the bias
  // plaintexts at the layer's output level and the output ciphertext scale bias_scale (DESIGN R-BIAS).
  cudaStream_t s = st(stream);
  const size_t n = (size_t)p->n, per = n * 8 + n * 32 + (size_t)c->N * 8 + 64;
  if (c->ws_bytes < 4096 + per) return fail(HY_E_WORKSPACE, "workspace too small for weight encoding");
  const int64_t B = std::min<int64_t>(64, (int64_t)((c->ws_bytes - 4096) / per));
  double* h_slots = nullptr;
  if (cudaMallocHost(&h_slots, (size_t)B * n * 8) != cudaSuccess) return fail(HY_E_CUDA, "pinned slot buffer");
  double* d_slots = reinterpret_cast<double*>(c->ws);
  uint8_t* ws_rest = c->ws + (((size_t)B * n * 8 + 255) & ~(size_t)255);
  const size_t rest_bytes = c->ws_bytes - (size_t)(ws_rest - c->ws);
  hy_status err = HY_OK;
  // one segment = cnt plaintexts of nl limbs at one scale, written stride words apart from dst
  auto segment = [&](int64_t cnt, uint32_t nl, uint64_t scale, uint64_t* dst, size_t stride, auto&& slots_of) {
    for (int64_t k0 = 0; k0 < cnt && err == HY_OK;) {
      const int64_t m = std::min<int64_t>(B, cnt - k0);
#pragma omp parallel for schedule(dynamic)
      for (int64_t k = 0; k < m; ++k) slots_of(k0 + k, h_slots + (size_t)k * n);
      cudaMemcpyAsync(d_slots, h_slots, (size_t)m * n * 8, cudaMemcpyHostToDevice, s);
      std::vector<uint64_t> sc((size_t)m, scale);
      err = encode_batch_device(c, d_slots, sc.data(), (uint32_t)m, nl, dst + (size_t)k0 * stride, stride, ws_rest,
                                rest_bytes, s);
      // the pinned slot buffer is rewritten by the next batch: wait for its upload
      cudaStreamSynchronize(s);
      k0 += m;
    }
  };
  const size_t stride = (size_t)(level + 1) * c->N;
  segment(p->n_pt(), level + 1, c->mod[level], d_pts, stride,
          [&](int64_t idx, double* v) { weight_slots(*p, K, idx, v); });
  if (p->has_mask)
    segment(1, level, c->mod[level - 1], d_pts + (size_t)p->n_pt() * stride, 0,
            [&](int64_t, double* v) { weight_slots(*p, K, p->n_pt(), v); });
  if (p->has_bias) {
    const uint32_t lo = p->out_level(level);
    segment(p->n_out, lo + 1, bias_scale, d_pts + p->bias_offset(level, c->N), (size_t)(lo + 1) * c->N,
            [&](int64_t j, double* v) { bias_slots(*p, bias, j, v); });
  }
  cudaFreeHost(h_slots);
  if (err != HY_OK) return err;
  return cuda_check("hy_conv_encode_weights");
}

namespace {

// RAConv after its lazy Slide_1&Sum_f: rescale, RaS_g, then (with a mask) the IR_g mask product + rescale
// and the IR_g rotations, batched over the outputs.  dst: per output, a ciphertext buffer at level - 1
// (the output itself without a mask); tmp: up to 8 temporaries of ct_l words.
// pp / pp_stride: no ping-pong ciphertexts for the RaS_g / IR_g steps (nullptr: in place).
hy_status ra_tail(const Ctx& x, std::vector<const uint64_t*>& sums, std::vector<uint64_t*>& dst, uint32_t level,
                  const uint64_t* mask, uint64_t* tmp, size_t ct_l, uint64_t* const* out, uint64_t* pp = nullptr,
                  size_t pp_stride = 0, uint64_t* sa = nullptr, uint64_t* sb = nullptr) {
  const hy_conv_plan* p = x.p;
  const size_t no = sums.size();
  hy_status stt = rescale_multi(x.c, sums.data(), (uint32_t)no, level, dst.data(), x.s);
  if (stt == HY_OK) stt = ras_all(x, dst, level - 1, p->ras_g, pp, pp_stride, sa, sb, pp_stride);
  if (stt == HY_OK && p->has_mask) {
    std::vector<uint64_t*> fin(out, out + no);
    stt = mask_rescale(x, dst, mask, level - 1, tmp, ct_l, fin);
    if (stt == HY_OK) stt = ras_all(x, fin, level - 2, p->ir_g, pp, pp_stride, sa, sb, pp_stride);
  }
  return stt;
}

// RAConv tap accumulators of output o for taps [tb, te): acc_t = sum_j x_j (.) W'_{o,j,t} (MulFilter&Sum_{c_i})
hy_status ra_taps(const Ctx& x, const uint64_t* const* in, uint32_t level, const uint64_t* wpt, uint32_t o,
                  size_t tb, size_t te, uint64_t* const* accs) {
  const hy_conv_plan* p = x.p;
  const size_t J = (size_t)p->n_in;
  // the taps' accumulators share the operands: blocks of up to 8 taps per MulFilter&Sum launch
  for (size_t t0 = tb; t0 < te; t0 += 8) {
    const size_t M = std::min<size_t>(8, te - t0);
    std::vector<uint32_t> bidx(M * J);
    std::vector<uint64_t> bgal(M * J);
    for (size_t m = 0; m < M; ++m)
      for (size_t i = 0; i < J; ++i) {
        const auto tm = p->term(o, (int64_t)i, (int64_t)(t0 + m));
        bidx[m * J + i] = (uint32_t)tm.first;
        bgal[m * J + i] = hy_galois_elt(x.c, tm.second);
      }
    hy_status st = pmult_block(x.c, in, (uint32_t)J, accs + (t0 - tb), (uint32_t)M, wpt, bidx.data(), bgal.data(),
                               level, 0, x.s);
    if (st != HY_OK) return st;
  }
  return HY_OK;
}

// pre_slid (CAConv only): a complete Slide_f result [n_in][f^2] ciphertexts (hy_caconv_slide layout); the Slide
// step is then skipped (multi-GPU Slide sharding) and `in` is not read
hy_status conv_core(hy_ctx* c, const hy_conv_plan* p, const uint64_t* const* evks, const uint64_t* const* in,
                    uint32_t level, const uint64_t* pts, uint64_t* scratch, uint32_t ob, uint32_t oe,
                    uint64_t* const* out, void* stream, const uint64_t* pre_slid = nullptr) {
  if (!c || !p || !evks || (!in && !pre_slid) || !pts || !scratch || !out) return fail(HY_E_ARG, "null");
  if (level >= c->n_q || level < 1u + (p->has_mask ? 1u : 0u)) return fail(HY_E_LEVEL_EXHAUSTED, "level too low");
  if (ob > oe || oe > p->n_out) return fail(HY_E_PLAN, "output range outside the plan");
  if (!pre_slid)
    for (int64_t i = 0; i < p->n_in; ++i)
      if (!in[i]) return fail(HY_E_ARG, "null input ciphertext");
  Ctx x{c, p, evks, st(stream)};
  const size_t N = c->N, f2 = (size_t)p->s.f * p->s.f;
  const size_t ct_l = 2 * (level + 1) * N;
  const uint64_t* wpt = pts;                                       // [n_pt][level+1][N]
  const uint64_t* mask = pts + (size_t)p->n_pt() * (level + 1) * N;  // [level][N]
  // MulFilter&Sum as dense blocks of <= 8 outputs: term (output m, operand j) -> stored plaintext index
  // and the Galois element of its PRot; each operand ciphertext is read once per block
  std::vector<uint32_t> bidx;
  std::vector<uint64_t> bgal;
  auto set_term = [&](size_t m, size_t J, size_t j, int64_t grp, int64_t i, int64_t t) {
    const auto tm = p->term(grp, i, t);
    bidx[m * J + j] = (uint32_t)tm.first;
    bgal[m * J + j] = hy_galois_elt(c, tm.second);
  };
  hy_status stt;
  if (p->s.algo == HY_CONV_CA) {
    // Slide_f: hoisted rotations of every input
    std::vector<std::vector<const uint64_t*>> slid(p->n_in, std::vector<const uint64_t*>(f2));
    uint64_t* sbuf = scratch;
    for (int64_t i = 0; i < p->n_in && pre_slid; ++i)
      for (size_t t = 0; t < f2; ++t) slid[i][t] = pre_slid + ((size_t)i * f2 + t) * ct_l;
    if (!pre_slid) {
      // every input rotates by the same tap amounts: one batched hoisted launch set for all inputs (round 2), else
      // one hy_hrot_hoisted per input
      std::vector<int32_t> rs;
      std::vector<const uint64_t*> ks;
      for (size_t t = 0; t < f2; ++t)
        if (p->taps[t] % p->n != 0) {
          rs.push_back((int32_t)p->taps[t]);
          ks.push_back(x.key(p->taps[t]));
        }
      std::vector<uint64_t*> outs;  // [input][rotation]
      for (int64_t i = 0; i < p->n_in; ++i)
        for (size_t t = 0; t < f2; ++t) {
          if (p->taps[t] % p->n == 0) {
            slid[i][t] = in[i];
            continue;
          }
          uint64_t* o = sbuf + ((size_t)i * f2 + t) * ct_l;
          slid[i][t] = o;
          outs.push_back(o);
        }
      if (!rs.empty()) {
        const uint32_t nr = (uint32_t)rs.size();
        stt = p->n_in >= 2 ? hrot_hoisted_multi(c, ks.data(), in, (uint32_t)p->n_in, level, rs.data(), nr,
                                                outs.data(), x.s)
                           : HY_E_WORKSPACE;
        if (stt == HY_E_WORKSPACE)
          for (int64_t i = 0; i < p->n_in; ++i) {
            stt = hy_hrot_hoisted(c, ks.data(), in[i], level, rs.data(), nr, outs.data() + (size_t)i * nr, stream);
            if (stt != HY_OK) return stt;
          }
        if (stt != HY_OK) return stt;
      }
    }
    // All SISO groups of the requested outputs advance together, so every RaS / RaS_g / IR_g step
    // is one batched HRot whose evaluation key is streamed once for all groups.
    const bool ds = p->s.stride == 2;
    std::vector<int64_t> grps;
    for (uint32_t j = ob; j < oe; ++j) {
      if (ds) {
        grps.push_back(2 * j);
        grps.push_back(2 * j + 1);
      } else {
        grps.push_back(j);
      }
    }
    const size_t G = grps.size();
    const size_t nacc = std::max<size_t>(8, G);
    uint64_t* acc = sbuf + (size_t)p->n_in * f2 * ct_l;          // one MulFilter&Sum accumulator per group
    uint64_t* gbuf = acc + nacc * ct_l;                           // G group ciphertexts (level - 1)
    const size_t ct_m = 2 * (size_t)level * N;
    std::vector<uint64_t*> gp(G);
    for (size_t g = 0; g < G; ++g)
      gp[g] = (!p->has_mask && !ds) ? out[g] : gbuf + g * ct_m;  // no mask: write the output directly
    // MulFilter&Sum_f over every (tap, input) operand, 8 groups per block, then rescale.  Operands are
    // tap-major so that a PRCR family's inputs (same stored plaintext) are adjacent.
    const size_t J = (size_t)p->n_in * f2;
    std::vector<const uint64_t*> ops(J);
    for (size_t t = 0; t < f2; ++t)
      for (int64_t i = 0; i < p->n_in; ++i) ops[t * p->n_in + i] = slid[i][t];
    for (size_t g0 = 0; g0 < G; g0 += 8) {
      const size_t M = std::min<size_t>(8, G - g0);
      bidx.assign(M * J, 0);
      bgal.assign(M * J, 1);
      std::vector<uint64_t*> accs(M);
      for (size_t m = 0; m < M; ++m) {
        accs[m] = acc + (g0 + m) * ct_l;
        for (size_t t = 0; t < f2; ++t)
          for (int64_t i = 0; i < p->n_in; ++i) set_term(m, J, t * p->n_in + i, grps[g0 + m], i, (int64_t)t);
      }
      stt = pmult_block(c, ops.data(), (uint32_t)J, accs.data(), (uint32_t)M, wpt, bidx.data(), bgal.data(), level,
                        0, stream);
      if (stt != HY_OK) return stt;
    }
    {  // every group's rescale in one batched call (r02t: R18 rescale family 3.15 -> ... ms per ds layer)
      std::vector<const uint64_t*> ac(G);
      for (size_t g = 0; g < G; ++g) ac[g] = acc + g * ct_l;
      stt = rescale_multi(c, ac.data(), (uint32_t)G, level, gp.data(), x.s);
      if (stt != HY_OK) return stt;
    }
    uint64_t* pp = gbuf + 2 * G * ct_m;  // G ping-pong ciphertexts (hy_conv_scratch_words)
    // limited key sets: 2 G more for the intermediate steps of synthesized rotations
    uint64_t* sa = p->decomp.empty() ? nullptr : pp + G * ct_m;
    uint64_t* sb = p->decomp.empty() ? nullptr : pp + 2 * G * ct_m;
    stt = ras_all(x, gp, level - 1, p->ras, pp, ct_m, sa, sb, ct_m);                        // RaS over C_a
    if (stt == HY_OK) stt = ras_all(x, gp, level - 1, p->ras_g, pp, ct_m, sa, sb, ct_m);    // RaS_g over C_g
    if (stt != HY_OK || (!p->has_mask && !ds)) return stt == HY_OK ? cuda_check("hy_caconv") : stt;
    // IR_g: mask (one level) ...
    std::vector<uint64_t*> masked(G);
    for (size_t g = 0; g < G; ++g) masked[g] = ds ? gbuf + (G + g) * ct_m : out[g];
    stt = mask_rescale(x, gp, mask, level - 1, acc, ct_l, masked, nacc);
    if (stt != HY_OK) return stt;
    std::vector<uint64_t*> fin(out, out + (oe - ob));
    if (ds) {  // ... merge the two groups of each output into the doubled gap (DESIGN R-DSCONV) ...
      const size_t J = oe - ob;
      std::vector<const uint64_t*> b(J), a(J);
      for (size_t j = 0; j < J; ++j) {
        a[j] = masked[2 * j];
        b[j] = masked[2 * j + 1];
      }
      stt = hrot_steps(x, p->combine, level - 2, b, fin, &a, sa, sb, ct_m);
      if (stt != HY_OK) return stt;
    }
    stt = ras_all(x, fin, level - 2, p->ir_g, pp, ct_m, sa, sb, ct_m);           // ... and replicate
    if (stt != HY_OK) return stt;
    return cuda_check("hy_caconv");
  }
  // RAConv_Reorder: MulFilter&Sum_{c_i} into f^2 accumulators, one lazy Slide_1&Sum_f, rescale, RaS_g, IR_g
  // accumulators [output][tap], filled as dense blocks of 8 outputs per tap: each input ciphertext is read
  // once per (tap, block), and a PRCR family's outputs (same stored plaintext) share a block
  uint64_t* accs = scratch;
  uint64_t* tmp = scratch + (size_t)(oe - ob) * f2 * ct_l;
  std::vector<const uint64_t*> keys(f2);
  std::vector<int32_t> rs(f2);
  for (size_t t = 0; t < f2; ++t) {
    rs[t] = (int32_t)p->taps[t];
    keys[t] = (p->taps[t] % p->n) ? x.key(p->taps[t]) : nullptr;
  }
  const size_t J = (size_t)p->n_in;
  if (oe - ob < 8) {  // fewer than 8 outputs (ResNet-20 RAConv: one): blocks of 8 (output, tap) accumulators,
    // which all read the same n_in operands, instead of one launch per tap with the few outputs
    std::vector<std::pair<uint32_t, size_t>> pr;  // (output, tap)
    for (uint32_t o = ob; o < oe; ++o)
      for (size_t t = 0; t < f2; ++t) pr.emplace_back(o, t);
    for (size_t k0 = 0; k0 < pr.size(); k0 += 8) {
      const size_t M = std::min<size_t>(8, pr.size() - k0);
      bidx.assign(M * J, 0);
      bgal.assign(M * J, 1);
      std::vector<uint64_t*> outs(M);
      for (size_t m = 0; m < M; ++m) {
        const uint32_t o = pr[k0 + m].first;
        const size_t t = pr[k0 + m].second;
        outs[m] = accs + ((o - ob) * f2 + t) * ct_l;
        for (size_t i = 0; i < J; ++i) set_term(m, J, i, o, (int64_t)i, (int64_t)t);
      }
      stt = pmult_block(c, in, (uint32_t)J, outs.data(), (uint32_t)M, wpt, bidx.data(), bgal.data(), level, 0,
                        stream);
      if (stt != HY_OK) return stt;
    }
  }
  for (size_t t = 0; t < f2 && oe - ob >= 8; ++t)
    for (uint32_t o0 = ob; o0 < oe; o0 += 8) {
      const size_t M = std::min<size_t>(8, oe - o0);
      bidx.assign(M * J, 0);
      bgal.assign(M * J, 1);
      std::vector<uint64_t*> outs(M);
      for (size_t m = 0; m < M; ++m) {
        outs[m] = accs + ((o0 + m - ob) * f2 + t) * ct_l;
        for (size_t i = 0; i < J; ++i) set_term(m, J, i, o0 + m, (int64_t)i, (int64_t)t);
      }
      stt = pmult_block(c, in, (uint32_t)J, outs.data(), (uint32_t)M, wpt, bidx.data(), bgal.data(), level, 0,
                        stream);
      if (stt != HY_OK) return stt;
    }
  // one lazy Slide_1&Sum_f per output (Alg. P:727-733), then every later step batched over the outputs
  const size_t no = oe - ob;
  std::vector<const uint64_t*> sums(no);
  std::vector<uint64_t*> dst(no);
  std::vector<const uint64_t*> tap_accs(no * f2);
  std::vector<uint64_t*> sum_out(no);
  for (uint32_t o = ob; o < oe; ++o) {
    uint64_t* oacc = accs + (size_t)(o - ob) * f2 * ct_l;
    for (size_t t = 0; t < f2; ++t) tap_accs[(o - ob) * f2 + t] = oacc + t * ct_l;
    sum_out[o - ob] = tmp + (size_t)(o - ob) * ct_l;
    sums[o - ob] = sum_out[o - ob];
    dst[o - ob] = p->has_mask ? oacc : out[o - ob];  // the output's consumed tap accumulators
  }
  // every output's lazy HRotSum in one batched launch set (round 2), else one hy_hrot_sum per output
  stt = no >= 2 ? hrot_sum_multi(c, keys.data(), tap_accs.data(), level, rs.data(), (uint32_t)f2, (uint32_t)no,
                                 sum_out.data(), x.s)
                : HY_E_WORKSPACE;
  if (stt == HY_E_WORKSPACE)
    for (size_t o = 0; o < no; ++o) {
      stt = hy_hrot_sum(c, keys.data(), tap_accs.data() + o * f2, level, rs.data(), (uint32_t)f2, sum_out[o], stream);
      if (stt != HY_OK) return stt;
    }
  if (stt != HY_OK) return stt;
  // ping-pong buffers: the second tap accumulator of every output (consumed by its HRotSum; f^2 >= 2)
  const bool ppok = f2 >= 2;
  // limited key sets: the third and fourth tap accumulators hold the intermediate steps (f^2 >= 4)
  const bool syn = !p->decomp.empty() && f2 >= 4;
  stt = ra_tail(x, sums, dst, level, mask, tmp, ct_l, out, ppok ? accs + ct_l : nullptr, f2 * ct_l,
                syn ? accs + 2 * ct_l : nullptr, syn ? accs + 3 * ct_l : nullptr);
  if (stt != HY_OK) return stt;
  return cuda_check("hy_raconv");
}

// the layer's bias (DESIGN R-BIAS): AddPt of bias plaintext o into c0 of output o, at the output level
hy_status add_bias(hy_ctx* c, const hy_conv_plan* p, uint32_t level, const uint64_t* pts, uint32_t ob, uint32_t oe,
                   uint64_t* const* out, void* stream) {
  if (!p->has_bias) return HY_OK;
  const uint32_t lo = p->out_level(level);
  const uint64_t* bias = pts + p->bias_offset(level, c->N);
  for (uint32_t o = ob; o < oe; ++o) {
    hy_status st = hy_add(c, out[o - ob], bias + (size_t)o * (lo + 1) * c->N, 1, lo, out[o - ob], stream);
    if (st != HY_OK) return st;
  }
  return HY_OK;
}

hy_status conv_run(hy_ctx* c, const hy_conv_plan* p, const uint64_t* const* evks, const uint64_t* const* in,
                   uint32_t level, const uint64_t* pts, uint64_t* scratch, uint32_t ob, uint32_t oe,
                   uint64_t* const* out, void* stream) {
  hy_status st = conv_core(c, p, evks, in, level, pts, scratch, ob, oe, out, stream);
  if (st != HY_OK) return st;
  return add_bias(c, p, level, pts, ob, oe, out, stream);
}

}  // namespace

extern "C" hy_status hy_caconv(hy_ctx* c, const hy_conv_plan* p, const uint64_t* const* evks,
                               const uint64_t* const* in, uint32_t level, const uint64_t* pts, uint64_t* scratch,
                               uint32_t out_begin, uint32_t out_end, uint64_t* const* out, void* stream) {
  if (p && p->s.algo != HY_CONV_CA) return fail(HY_E_PLAN, "plan is not a CAConv plan");
  return conv_run(c, p, evks, in, level, pts, scratch, out_begin, out_end, out, stream);
}

extern "C" hy_status hy_raconv(hy_ctx* c, const hy_conv_plan* p, const uint64_t* const* evks,
                               const uint64_t* const* in, uint32_t level, const uint64_t* pts, uint64_t* scratch,
                               uint32_t out_begin, uint32_t out_end, uint64_t* const* out, void* stream) {
  if (p && p->s.algo != HY_CONV_RA) return fail(HY_E_PLAN, "plan is not an RAConv plan");
  return conv_run(c, p, evks, in, level, pts, scratch, out_begin, out_end, out, stream);
}

extern "C" hy_status hy_caconv_slide(hy_ctx* c, const hy_conv_plan* p, const uint64_t* const* evks,
                                     const uint64_t* const* in, uint32_t level, uint32_t in_begin, uint32_t in_end,
                                     uint64_t* slid, void* stream) {
  if (!c || !p || !evks || !in || !slid) return fail(HY_E_ARG, "null");
  if (p->s.algo != HY_CONV_CA) return fail(HY_E_PLAN, "plan is not a CAConv plan");
  if (level >= c->n_q || level < 1u + (p->has_mask ? 1u : 0u)) return fail(HY_E_LEVEL_EXHAUSTED, "level too low");
  if (in_begin > in_end || in_end > p->n_in) return fail(HY_E_PLAN, "input range outside the plan");
  const size_t f2 = (size_t)p->s.f * p->s.f, ct_l = 2ull * (level + 1) * c->N;
  Ctx x{c, p, evks, st(stream)};
  std::vector<int32_t> rs;
  std::vector<const uint64_t*> ks;
  for (size_t t = 0; t < f2; ++t)
    if (p->taps[t] % p->n != 0) {
      rs.push_back((int32_t)p->taps[t]);
      ks.push_back(x.key(p->taps[t]));
    }
  std::vector<uint64_t*> outs;  // [input][rotation]
  for (uint32_t i = in_begin; i < in_end; ++i) {
    if (!in[i]) return fail(HY_E_ARG, "null input ciphertext");
    for (size_t t = 0; t < f2; ++t) {
      uint64_t* o = slid + ((size_t)(i - in_begin) * f2 + t) * ct_l;
      if (p->taps[t] % p->n == 0) {
        cudaMemcpyAsync(o, in[i], ct_l * 8, cudaMemcpyDeviceToDevice, x.s);
        continue;
      }
      outs.push_back(o);
    }
  }
  const uint32_t ni = in_end - in_begin, nr = (uint32_t)rs.size();
  if (nr && ni) {  // the inputs' hoisted Slides batched (as in hy_caconv), else one hy_hrot_hoisted per input
    hy_status stt = ni >= 2 ? hrot_hoisted_multi(c, ks.data(), in + in_begin, ni, level, rs.data(), nr, outs.data(), x.s)
                            : HY_E_WORKSPACE;
    if (stt == HY_E_WORKSPACE)
      for (uint32_t i = 0; i < ni; ++i) {
        stt = hy_hrot_hoisted(c, ks.data(), in[in_begin + i], level, rs.data(), nr, outs.data() + (size_t)i * nr,
                              stream);
        if (stt != HY_OK) return stt;
      }
    if (stt != HY_OK) return stt;
  }
  return cuda_check("hy_caconv_slide");
}

extern "C" hy_status hy_caconv_slid(hy_ctx* c, const hy_conv_plan* p, const uint64_t* const* evks,
                                    const uint64_t* slid, uint32_t level, const uint64_t* pts, uint64_t* scratch,
                                    uint32_t out_begin, uint32_t out_end, uint64_t* const* out, void* stream) {
  if (!slid) return fail(HY_E_ARG, "null slid buffer");
  if (p && p->s.algo != HY_CONV_CA) return fail(HY_E_PLAN, "plan is not a CAConv plan");
  hy_status st = conv_core(c, p, evks, nullptr, level, pts, scratch, out_begin, out_end, out, stream, slid);
  if (st != HY_OK) return st;
  return add_bias(c, p, level, pts, out_begin, out_end, out, stream);
}

extern "C" size_t hy_raconv_partial_words(const hy_ctx* c, uint32_t level) {
  if (!c) return 0;
  return (2ull * (level + 1 + c->n_p) + 2ull * (level + 1)) * c->N;
}

namespace {
hy_status ra_check(hy_ctx* c, const hy_conv_plan* p, uint32_t level, uint32_t o) {
  if (!c || !p) return fail(HY_E_ARG, "null");
  if (p->s.algo != HY_CONV_RA) return fail(HY_E_PLAN, "plan is not an RAConv plan");
  if (level >= c->n_q || level < 1u + (p->has_mask ? 1u : 0u)) return fail(HY_E_LEVEL_EXHAUSTED, "level too low");
  if (o >= p->n_out) return fail(HY_E_PLAN, "output index outside the plan");
  return HY_OK;
}
}  // namespace

extern "C" hy_status hy_raconv_partial(hy_ctx* c, const hy_conv_plan* p, const uint64_t* const* evks,
                                       const uint64_t* const* in, uint32_t level, const uint64_t* pts,
                                       uint64_t* scratch, uint32_t out_index, uint32_t tap_begin, uint32_t tap_end,
                                       uint64_t* state, void* stream) {
  hy_status stt = ra_check(c, p, level, out_index);
  if (stt != HY_OK) return stt;
  const size_t f2 = (size_t)p->s.f * p->s.f;
  if (!evks || !in || !pts || !scratch || !state) return fail(HY_E_ARG, "null");
  if (tap_begin > tap_end || tap_end > f2) return fail(HY_E_PLAN, "tap range outside the filter");
  for (int64_t i = 0; i < p->n_in; ++i)
    if (!in[i]) return fail(HY_E_ARG, "null input ciphertext");
  Ctx x{c, p, evks, st(stream)};
  const size_t N = c->N, nl = level + 1, ct_l = 2 * nl * N, nt = tap_end - tap_begin;
  uint64_t* u = state;
  uint64_t* acc = state + 2 * (nl + c->n_p) * N;
  if (nt == 0) {  // an empty shard contributes zero
    cudaMemsetAsync(state, 0, hy_raconv_partial_words(c, level) * 8, x.s);
    return cuda_check("hy_raconv_partial");
  }
  std::vector<uint64_t*> accs(nt);
  std::vector<const uint64_t*> accc(nt), keys(nt);
  std::vector<int32_t> rs(nt);
  for (size_t k = 0; k < nt; ++k) {
    const size_t t = tap_begin + k;
    accs[k] = scratch + k * ct_l;
    accc[k] = accs[k];
    rs[k] = (int32_t)p->taps[t];
    keys[k] = (p->taps[t] % p->n) ? x.key(p->taps[t]) : nullptr;
  }
  stt = ra_taps(x, in, level, pts, out_index, tap_begin, tap_end, accs.data());
  if (stt == HY_OK)
    stt = hrot_sum_partial(c, keys.data(), accc.data(), level, rs.data(), (uint32_t)nt, u, acc, x.s);
  if (stt != HY_OK) return stt;
  return cuda_check("hy_raconv_partial");
}

extern "C" hy_status hy_raconv_finish(hy_ctx* c, const hy_conv_plan* p, const uint64_t* const* evks, uint32_t level,
                                      const uint64_t* pts, uint64_t* state, uint64_t* scratch, uint32_t out_index,
                                      uint64_t* out, void* stream) {
  hy_status stt = ra_check(c, p, level, out_index);
  if (stt != HY_OK) return stt;
  if (!evks || !pts || !state || !scratch || !out) return fail(HY_E_ARG, "null");
  Ctx x{c, p, evks, st(stream)};
  const size_t N = c->N, nl = level + 1, ct_l = 2 * nl * N;
  uint64_t* u = state;
  uint64_t* acc = state + 2 * (nl + c->n_p) * N;
  const uint64_t* mask = pts + (size_t)p->n_pt() * nl * N;
  stt = mod_reduce_ext(c, level, u, acc, x.s);  // the partials were summed as integers
  uint64_t* sum = scratch;
  uint64_t* dstb = scratch + ct_l;
  uint64_t* tmp = scratch + 2 * ct_l;
  if (stt == HY_OK) stt = hrot_sum_finish(c, level, u, acc, sum, x.s);
  if (stt != HY_OK) return stt;
  std::vector<const uint64_t*> sums{sum};
  std::vector<uint64_t*> dst{p->has_mask ? dstb : out};
  stt = ra_tail(x, sums, dst, level, mask, tmp, ct_l, &out, scratch + 3 * ct_l, ct_l, scratch + 4 * ct_l,
                scratch + 5 * ct_l);
  if (stt == HY_OK) stt = add_bias(c, p, level, pts, out_index, out_index + 1, &out, stream);
  if (stt != HY_OK) return stt;
  return cuda_check("hy_raconv_finish");
}
