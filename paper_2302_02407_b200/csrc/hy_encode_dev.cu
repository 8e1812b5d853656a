// hy_encode_dev.cu -- CKKS encoding on the device, for the bulk weight plaintexts of the conv layers
// ("device encode for bulk weights"; untimed in the paper).
//
// The same computation as the host encoder (hy_encode.cpp, DESIGN R-ENCODE): real slots z_0..z_{n-1},
// the "special" inverse FFT over the rotation group <5> in double-double arithmetic, bit reversal, then
// m = round_half_away(scale * v / n) with |frac - 1/2| < 2^-40 taken as a tie.  The computed value is within
// ~2^-55 of the exact one, so its rounding is the rounding of the exact value (identical to the host's and to
// the oracle's binary128 DFT; bit-exactness is tested).
//
// Layout: a batch of P plaintexts, each n = N/2 complex double-double values (32 bytes: re.hi, re.lo, im.hi,
// im.lo) in the workspace.  The log2(n) stages are split like the NTT:
//   pass 1 (k_enc_cols): the stages with half-length >= 256 pair elements that differ only in the bits above
//     bit 7, so for a fixed low byte b the n/256 elements a*256 + b form an independent problem; a CTA holds
//     8 such columns (8 x n/256 values, 32 KB at N = 2^16) in shared memory for all those stages;
//   pass 2 (k_enc_rows): the last 8 stages work inside contiguous 256-element blocks; a CTA holds 2 blocks,
//     then applies the bit reversal, the scale and the rounding and writes the int64 coefficients
//     (re part at br(e), im part at br(e) + n).
// Twiddles ksi^k = exp(2 pi i k / 2N) (double-double, from binary128 on the host) and the rotation group
// 5^j mod 2N live in a per-context device table built on first use.
#include <algorithm>
#include <cstdint>
#include <vector>

#include "hy_arith.cuh"

namespace hy {
void encode_tables(uint32_t log_n, std::vector<double>& ksi4, std::vector<uint32_t>& rot);  // hy_encode.cpp

namespace {

struct DDd {
  double hi, lo;
};
__device__ __forceinline__ DDd two_sum(double a, double b) {
  const double s = a + b, bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ DDd quick_two_sum(double a, double b) {
  const double s = a + b;
  return {s, b - (s - a)};
}
__device__ __forceinline__ DDd dd_add(DDd a, DDd b) {
  DDd s = two_sum(a.hi, b.hi), t = two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = quick_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return quick_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ DDd dd_neg(DDd a) { return {-a.hi, -a.lo}; }
__device__ __forceinline__ DDd dd_mul(DDd a, DDd b) {
  const double p = a.hi * b.hi;
  double e = __fma_rn(a.hi, b.hi, -p);
  e += a.hi * b.lo + a.lo * b.hi;
  return quick_two_sum(p, e);
}
// complex double-double as double4 (re.hi, re.lo, im.hi, im.lo)
__device__ __forceinline__ DDd re_(const double4& v) { return {v.x, v.y}; }
__device__ __forceinline__ DDd im_(const double4& v) { return {v.z, v.w}; }
__device__ __forceinline__ double4 mk(DDd r, DDd i) { return make_double4(r.hi, r.lo, i.hi, i.lo); }
__device__ __forceinline__ double4 c_add(const double4& a, const double4& b) {
  return mk(dd_add(re_(a), re_(b)), dd_add(im_(a), im_(b)));
}
__device__ __forceinline__ double4 c_sub(const double4& a, const double4& b) {
  return mk(dd_add(re_(a), dd_neg(re_(b))), dd_add(im_(a), dd_neg(im_(b))));
}
__device__ __forceinline__ double4 c_mul(const double4& a, const double4& b) {
  return mk(dd_add(dd_mul(re_(a), re_(b)), dd_neg(dd_mul(im_(a), im_(b)))),
            dd_add(dd_mul(re_(a), im_(b)), dd_mul(im_(a), re_(b))));
}

// inverse special-FFT butterfly of element e (first of its pair, partner e + lenh) at stage len
__device__ __forceinline__ void enc_bfly(double4& x, double4& y, uint32_t e, uint32_t len, const double4* ksi,
                                         const uint32_t* rot, uint32_t M) {
  const uint32_t lenq = len << 2, gap = M / lenq;
  const uint32_t j = e & (len - 1);
  const uint32_t idx = (lenq - (rot[j] & (lenq - 1))) * gap;
  const double4 u = c_add(x, y);
  y = c_mul(c_sub(x, y), ksi[idx]);
  x = u;
}

// pass 1: grid (32 groups of 8 columns, P); CTA 256 threads; A = n/256 values per column
__global__ void __launch_bounds__(256) k_enc_cols(const double* __restrict__ slots, double4* __restrict__ v,
                                                  const double4* __restrict__ ksi, const uint32_t* __restrict__ rot,
                                                  int log_n_slots) {
  extern __shared__ double4 sv[];  // [A][8]
  const uint32_t n = 1u << log_n_slots, A = n >> 8, M = n << 2;
  const uint32_t b0 = blockIdx.x * 8, p = blockIdx.y;
  const double* z = slots + (size_t)p * n;
  for (uint32_t t = threadIdx.x; t < 8 * A; t += blockDim.x) {
    const uint32_t a = t >> 3, c = t & 7;
    sv[t] = make_double4(z[a * 256 + b0 + c], 0.0, 0.0, 0.0);
  }
  __syncthreads();
  for (uint32_t len = n; len >= 512; len >>= 1) {
    const uint32_t h = (len >> 1) >> 8;  // partner distance in a
    for (uint32_t t = threadIdx.x; t < 4 * A; t += blockDim.x) {  // 8 columns x A/2 pairs
      const uint32_t c = t & 7, pi = t >> 3;
      const uint32_t a = (pi / h) * 2 * h + (pi % h);
      double4 x = sv[a * 8 + c], y = sv[(a + h) * 8 + c];
      enc_bfly(x, y, a * 256 + b0 + c, len, ksi, rot, M);
      sv[a * 8 + c] = x;
      sv[(a + h) * 8 + c] = y;
    }
    __syncthreads();
  }
  double4* o = v + (size_t)p * n;
  for (uint32_t t = threadIdx.x; t < 8 * A; t += blockDim.x) {
    const uint32_t a = t >> 3, c = t & 7;
    o[a * 256 + b0 + c] = sv[t];
  }
}

__device__ __forceinline__ int64_t round_dd(DDd x) {
  double fl = floor(x.hi);
  const DDd r = dd_add({x.hi - fl, 0.0}, {x.lo, 0.0});
  double frac = r.hi + r.lo;
  if (frac < 0) {
    fl -= 1;
    frac += 1;
  } else if (frac >= 1) {
    fl += 1;
    frac -= 1;
  }
  const bool positive = x.hi > 0 || (x.hi == 0 && x.lo > 0);
  if (fabs(frac - 0.5) < 0x1p-40) return (int64_t)fl + (positive ? 1 : 0);
  return (int64_t)fl + (frac > 0.5 ? 1 : 0);
}

// pass 2: grid (n/512, P); CTA 256 threads = 2 blocks of 256 elements x 128 butterflies; then bit reversal,
// scale and rounding into coeffs [P][N] (int64).  Any |value| >= 2^62 sets *overflow.
__global__ void __launch_bounds__(256) k_enc_rows(const double4* __restrict__ v, int64_t* __restrict__ coeffs,
                                                  const double4* __restrict__ ksi, const uint32_t* __restrict__ rot,
                                                  const uint64_t* __restrict__ scales, int log_n_slots,
                                                  int* overflow) {
  __shared__ double4 sv[512];
  const uint32_t n = 1u << log_n_slots, M = n << 2, p = blockIdx.y;
  const uint32_t base = blockIdx.x * 512;
  const double4* src = v + (size_t)p * n + base;
  for (uint32_t t = threadIdx.x; t < 512; t += blockDim.x) sv[t] = src[t];
  __syncthreads();
  const uint32_t blk = threadIdx.x >> 7, bt = threadIdx.x & 127;
  for (uint32_t len = 256; len >= 2; len >>= 1) {
    const uint32_t h = len >> 1;
    const uint32_t e = (bt / h) * len + (bt % h);  // first element of the pair inside the block
    double4 x = sv[blk * 256 + e], y = sv[blk * 256 + e + h];
    enc_bfly(x, y, base + blk * 256 + e, len, ksi, rot, M);
    sv[blk * 256 + e] = x;
    sv[blk * 256 + e + h] = y;
    __syncthreads();
  }
  const uint64_t scale = scales[p];
  const double sh = (double)scale;
  const DDd sc = {sh, (double)(int64_t)(scale - (uint64_t)sh)};
  const DDd inv_n = {1.0 / (double)n, 0.0};
  int64_t* out = coeffs + (size_t)p * 2 * n;
  for (uint32_t t = threadIdx.x; t < 512; t += blockDim.x) {
    const uint32_t e = base + t;
    const uint32_t k = __brev(e) >> (32 - log_n_slots);
    const DDd re = dd_mul(dd_mul(re_(sv[t]), inv_n), sc), im = dd_mul(dd_mul(im_(sv[t]), inv_n), sc);
    if (fabs(re.hi) >= 0x1p62 || fabs(im.hi) >= 0x1p62) *overflow = 1;
    out[k] = round_dd(re);
    out[k + n] = round_dd(im);
  }
}

// signed coefficients [P][N] -> residues on q_0..q_{nl-1} of plaintext p at out + p * stride.
// grid (N/256, nl, P)
__global__ void k_coeffs_to_limbs(const int64_t* __restrict__ coeffs, uint64_t* __restrict__ out, size_t stride,
                                  DevTables dt, int logN) {
  const size_t N = (size_t)1 << logN;
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  const int t = blockIdx.y;
  const PrimeConst& pc = dt.pc[t];
  const int64_t s = coeffs[(size_t)blockIdx.z * N + x];
  const uint64_t m = reduce64(s >= 0 ? (uint64_t)s : (uint64_t)(-s), pc);
  out[(size_t)blockIdx.z * stride + (size_t)t * N + x] = s >= 0 ? m : (m ? pc.q - m : 0);
}

}  // namespace

// Encode P real slot vectors (device, [P][N/2] doubles) at the given integer scales (host array) into the
// NTT-domain plaintexts out + p * stride (limbs q_0..q_{nl-1}).  Workspace: P * (N/2 * 32 + N * 8) bytes + 256.
hy_status encode_batch_device(hy_ctx* c, const double* d_slots, const uint64_t* h_scales, uint32_t P, uint32_t nl,
                              uint64_t* out, size_t stride, uint8_t* ws, size_t ws_bytes, cudaStream_t s) {
  if (P == 0) return HY_OK;
  const uint32_t n = c->N / 2, logn = c->log_n - 1;
  if (n < 512) return fail(HY_E_ARG, "device encoding needs N >= 1024");
  if (!c->d_enc) {  // twiddles and the rotation group, built once per context
    std::vector<double> ksi4;
    std::vector<uint32_t> rot;
    encode_tables(c->log_n, ksi4, rot);
    const size_t kb = ksi4.size() * 8, rb = rot.size() * 4;
    if (cudaMalloc(&c->d_enc, kb + rb) != cudaSuccess) return fail(HY_E_CUDA, "encode tables");
    cudaMemcpy(c->d_enc, ksi4.data(), kb, cudaMemcpyHostToDevice);
    cudaMemcpy((uint8_t*)c->d_enc + kb, rot.data(), rb, cudaMemcpyHostToDevice);
    c->enc_rot_off = kb;
  }
  const double4* ksi = (const double4*)c->d_enc;
  const uint32_t* rot = (const uint32_t*)((const uint8_t*)c->d_enc + c->enc_rot_off);
  Ws w{ws, ws_bytes};
  double4* v = w.take<double4>((size_t)P * n);
  int64_t* coeffs = w.take<int64_t>((size_t)P * c->N);
  uint64_t* d_sc = w.take<uint64_t>(P);
  int* flag = w.take<int>(1);
  if (!flag) return fail(HY_E_WORKSPACE, "workspace too small for the encode batch");
  cudaMemcpyAsync(d_sc, h_scales, P * 8, cudaMemcpyHostToDevice, s);
  cudaMemsetAsync(flag, 0, sizeof(int), s);
  {
    KTimer kt(c, FAM_CLIENT, s, 3);
    const size_t smem = (size_t)8 * (n / 256) * sizeof(double4);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_enc_cols, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
      attr = true;
    }
    k_enc_cols<<<dim3(32, P), 256, smem, s>>>(d_slots, v, ksi, rot, (int)logn);
    k_enc_rows<<<dim3(n / 512, P), 256, 0, s>>>(v, coeffs, ksi, rot, d_sc, (int)logn, flag);
    k_coeffs_to_limbs<<<dim3(c->N / 256, nl, P), 256, 0, s>>>(coeffs, out, stride, c->dt, (int)c->log_n);
  }
  std::vector<uint32_t> chain(nl);
  for (uint32_t i = 0; i < nl; ++i) chain[i] = i;
  for (uint32_t p = 0; p < P; ++p) ntt_contig(c, out + p * stride, out + p * stride, chain.data(), nl, false, s);
  int h_flag = 0;
  cudaMemcpyAsync(&h_flag, flag, sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);  // h_scales / the caller's host slots may be reused
  if (h_flag) return fail(HY_E_CAPACITY, "encoded coefficient exceeds 2^62");
  return cuda_check("encode_batch_device");
}

}  // namespace hy

using namespace hy;

extern "C" hy_status hy_encode_batch(hy_ctx* c, const double* h_slots, uint32_t P, uint64_t scale, uint32_t level,
                                     uint64_t* d_pts, void* stream) {
  if (!c || !h_slots || !d_pts) return fail(HY_E_ARG, "null");
  if (level >= c->n_q) return fail(HY_E_ARG, "level out of range");
  if (!c->ws) return fail(HY_E_WORKSPACE, "workspace not set");
  cudaStream_t s = st(stream);
  const size_t n = c->N / 2, per = n * 8 + n * 32 + (size_t)c->N * 8 + 64, stride = (size_t)(level + 1) * c->N;
  const size_t B = std::min<size_t>({64, (size_t)P, c->ws_bytes > 4096 ? (c->ws_bytes - 4096) / per : 0});
  if (P && B < 1) return fail(HY_E_WORKSPACE, "workspace too small for encoding");
  double* d_slots = reinterpret_cast<double*>(c->ws);
  uint8_t* rest = c->ws + ((B * n * 8 + 255) & ~(size_t)255);
  const size_t rest_bytes = c->ws_bytes - (size_t)(rest - c->ws);
  for (uint32_t p0 = 0; p0 < P;) {
    const uint32_t cnt = (uint32_t)std::min<size_t>(B, P - p0);
    cudaMemcpyAsync(d_slots, h_slots + (size_t)p0 * n, (size_t)cnt * n * 8, cudaMemcpyHostToDevice, s);
    std::vector<uint64_t> sc(cnt, scale);
    hy_status e = encode_batch_device(c, d_slots, sc.data(), cnt, level + 1, d_pts + (size_t)p0 * stride, stride,
                                      rest, rest_bytes, s);
    if (e != HY_OK) return e;
    p0 += cnt;
  }
  return HY_OK;
}
