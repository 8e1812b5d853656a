// hy_ntt.cu -- batched negacyclic NTT / inverse NTT for N = 2^10 .. 2^16 on sm_100a.
//
// Transform (DESIGN R-NTT): merged-twiddle Cooley-Tukey forward with
// psi^{br(k)} twiddles, output in bit-reversed order (index k holds
// a(psi^(2 br(k)+1))); Gentleman-Sande inverse.  At the stage whose butterfly
// distance is t, the element x uses twiddle index (N + x) / (2t).
//
// Decomposition: N = R x 256 (R = N/256 rows of 256 contiguous words).
//   pass A: the log2(R) stages with t >= 256 -- R-point transforms down the
//           columns (x = r*256 + c);
//   pass B: the 8 stages with t < 256 -- 256-point transforms along each row.
// Forward = A then B; inverse = B then A (with the N^{-1} scaling fused in).
// Each 256-point transform lives in registers, 8 words per thread, and moves
// through shared memory twice (layouts L1 -> L2 -> L3) so that every stage is
// a register-local butterfly: L1 owns bits {7,6,5}, L2 {4,3,2}, L3 {1,0}.
// Arithmetic runs on the FP64 pipe (hy_arith.cuh fmulmod): residues are loaded
// as uint64, converted exactly to doubles, and stored back canonical in [0, q).
// Between the two passes the limb holds the raw bits of fred-reduced doubles
// (|v| <= q/2 + 1), so neither pass pays for canonicalisation / conversion there;
// only the fused row kernels below and the second pass read that format.
#include <algorithm>
#include <cstdlib>

#include "hy_arith.cuh"

namespace hy {
namespace {

// intermediate (between-pass) format: raw double bits
__device__ __forceinline__ double raw2d(uint64_t v) { return __longlong_as_double((long long)v); }
__device__ __forceinline__ uint64_t d2raw(double d) { return (uint64_t)__double_as_longlong(d); }

template <int LAY>
__device__ __forceinline__ int elem(int l, int k) {
  if (LAY == 1) return l + 32 * k;
  if (LAY == 2) return 32 * (l >> 2) + 4 * k + (l & 3);
  return 4 * (l + 32 * (k >> 2)) + (k & 3);
}
template <int LAY>
__device__ __forceinline__ int kbit(int s) {
  return LAY == 1 ? s - 5 : (LAY == 2 ? s - 2 : s);
}

// Run stages [s_lo, s_hi] (forward: descending, inverse: ascending) on the 8
// register values of one thread in layout LAY, on the FP64 pipe.  Twiddles come
// from a shared-memory "heap" table T[li], li = (256 + e) >> (s+1) in [1, 256).
//   forward (CT):  a' = a + b w, b' = a - b w   with |b w mod q| <= (1/2 + beta/16) q for |b| <= beta q
//                  (hy_arith.cuh fmulmod), no reduction inside a pass: 8 stages from |v| <= q take the
//                  operand bound to 6.62 q (from the between-pass format |v| <= q/2 + 1: 5.81 q), below
//                  fmulmod's 2^51 / q_max = 8 (DESIGN R-FP64, tests/test_fp64_bound_cpu.py);
//   inverse (GS):  a' = a + b, b' = (a - b) w; sums double per stage, so every
//                  register round ends with a reduction (fred) of all 8 values.
template <int LAY, bool FWD>
__device__ __forceinline__ void run_stages(double (&x)[8], int l, int s_hi, int s_lo, const double* __restrict__ T,
                                           double q, double qinv) {
#pragma unroll
  for (int it = 0; it <= s_hi - s_lo; ++it) {
    const int s = FWD ? s_hi - it : s_lo + it;
    const int kb = 1 << kbit<LAY>(s);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (k & kb) continue;
      const double w = T[(256 + elem<LAY>(l, k)) >> (s + 1)];
      const double a = x[k], b = x[k | kb];
      if (FWD) {
        const double t = fmulmod(b, w, q, qinv);
        x[k] = a + t;
        x[k | kb] = a - t;
      } else {
        x[k] = a + b;
        x[k | kb] = fmulmod(a - b, w, q, qinv);
      }
    }
  }
  if (!FWD) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fred(x[k], q, qinv);
  }
}

// Fill the twiddle heap of one 256-point transform: T[li] = W[((hb - 1) << m) + li],
// m = floor(log2 li).  hb = 1 for pass A (global index = li) and R + row for
// pass B (global index = (N + row*256 + e) >> (s+1)).  nthr threads cooperate.
__device__ __forceinline__ void load_twiddles(double* T, const double* __restrict__ W, uint32_t hb, int tid,
                                              int nthr) {
  for (int li = tid; li < 256; li += nthr) {
    if (li == 0) continue;
    const int m = 31 - __clz(li);
    T[li] = __ldg(W + ((hb - 1) << m) + (uint32_t)li);
  }
}
// One warp fills a row's heap: all 8 loads are issued before the first shared-memory store, so the
// warp waits for one L2 round trip instead of eight.
__device__ __forceinline__ void load_twiddles_warp(double* T, const double* __restrict__ W, uint32_t hb, int l) {
  double v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int li = l + 32 * k;
    const int m = 31 - __clz(li | 1);
    v[k] = li ? __ldg(W + ((hb - 1) << m) + (uint32_t)li) : 0.0;
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) T[l + 32 * k] = v[k];
}

// Shared-memory word of element e in a warp's 256-word transpose buffer: an XOR swizzle (a bijection
// on [0, 256)) under which every layout access of a half-warp (S[pidx(elem<L>(l, k))], L = 1, 2, 3)
// touches 16 distinct 8-byte banks (checked by brute force over all l, k, L).
__device__ __forceinline__ int pidx(int e) { return e ^ ((e >> 2) & 1) ^ (((e >> 4) & 7) << 1); }
// The same for an 8-column strip [256][8] (thread column c = tid & 7, lane l = tid >> 3): word of
// (element e, column c); rows e and e^1 / e^4 met by one half-warp land in opposite bank halves.
__device__ __forceinline__ int sidx8(int e, int c) { return 8 * (e ^ ((e >> 2) & 1)) + c; }

// ---------------------------------------------------------------- pass B (rows)
// CTA = 8 warps, one 256-word row per warp.  grid = (N/256/8, n_limbs)
template <bool FWD>
__global__ void __launch_bounds__(256) k_ntt_rows(LimbBatch b, DevTables dt, int logN) {
  __shared__ double sm[8][272];
  __shared__ double tws[8][256];
  const int limb = blockIdx.y, w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + w;
  const size_t N = (size_t)1 << logN;
  if (row >= (int)(N >> 8)) return;  // N = 2^10: 4 rows in an 8-warp CTA
  const int t = b.chain[limb];
  const PrimeConst& pc = dt.pc[t];
  const double q = pc.qd, qinv = pc.qinv;
  const double* W = (FWD ? dt.tw : dt.itw) + (size_t)t * N;
  const uint64_t* src = b.src[limb] + (size_t)row * 256;
  uint64_t* dst = b.dst[limb] + (size_t)row * 256;
  double* S = sm[w];
  double* T = tws[w];
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = FWD ? raw2d(src[elem<1>(l, k)]) : u2d(src[elem<1>(l, k)]);
  load_twiddles_warp(T, W, (uint32_t)(N >> 8) + (uint32_t)row, l);
  __syncwarp();
  if (FWD) {
    run_stages<1, true>(x, l, 7, 5, T, q, qinv);
#pragma unroll
    for (int k = 0; k < 8; ++k) S[pidx(elem<1>(l, k))] = x[k];
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = S[pidx(elem<2>(l, k))];
    run_stages<2, true>(x, l, 4, 2, T, q, qinv);
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 8; ++k) S[pidx(elem<2>(l, k))] = x[k];
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = S[pidx(elem<3>(l, k))];
    run_stages<3, true>(x, l, 1, 0, T, q, qinv);
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 8; ++k) S[pidx(elem<3>(l, k))] = fcanon(x[k], q, qinv);
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 8; ++k) dst[elem<1>(l, k)] = d2u(S[pidx(elem<1>(l, k))]);
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) S[pidx(elem<1>(l, k))] = x[k];
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = S[pidx(elem<3>(l, k))];
    run_stages<3, false>(x, l, 1, 0, T, q, qinv);
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 8; ++k) S[pidx(elem<3>(l, k))] = x[k];
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = S[pidx(elem<2>(l, k))];
    run_stages<2, false>(x, l, 4, 2, T, q, qinv);
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 8; ++k) S[pidx(elem<2>(l, k))] = x[k];
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = S[pidx(elem<1>(l, k))];
    run_stages<1, false>(x, l, 7, 5, T, q, qinv);
#pragma unroll
    for (int k = 0; k < 8; ++k) dst[elem<1>(l, k)] = d2raw(x[k]);
  }
}

// ---------------------------------------------------------------- pass B (rows), inverse, with the automorphism
// The inverse row pass of kappa_k(c1) read straight from c1 (plain HRot): the NTT-domain Galois permutation maps
// every 256-word row onto one source row (the high index bits of kappa depend only on high bits), so each warp
// gathers its row from one 2 KB source row (L1-resident) and kappa(c1) is never stored.  Item g = blockIdx.z,
// limb i = blockIdx.y (chain index i), grid (R/8, l+1, G).
__global__ void __launch_bounds__(256) k_ntt_rows_inv_aut(const __grid_constant__ RowsAutArgs a, DevTables dt,
                                                          int logN) {
  __shared__ double sm[8][272];
  __shared__ double tws[8][256];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + w, i = blockIdx.y, g = blockIdx.z;
  const size_t N = (size_t)1 << logN;
  if (row >= (int)(N >> 8)) return;
  const PrimeConst& pc = dt.pc[i];
  const double q = pc.qd, qinv = pc.qinv;
  const uint64_t* src = a.src[g] + (size_t)i * N;
  uint64_t* dst = a.dst[g] + (size_t)i * N + (size_t)row * 256;
  const uint64_t k = a.k[g];
  double* S = sm[w];
  double* T = tws[w];
  double x[8];
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    const uint32_t xi = (uint32_t)row * 256 + elem<1>(l, kk);
    x[kk] = u2d(src[k != 1 ? aut_index(xi, k, logN) : xi]);
  }
  load_twiddles_warp(T, dt.itw + (size_t)i * N, (uint32_t)(N >> 8) + (uint32_t)row, l);
  __syncwarp();
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) S[pidx(elem<1>(l, kk))] = x[kk];
  __syncwarp();
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) x[kk] = S[pidx(elem<3>(l, kk))];
  run_stages<3, false>(x, l, 1, 0, T, q, qinv);
  __syncwarp();
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) S[pidx(elem<3>(l, kk))] = x[kk];
  __syncwarp();
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) x[kk] = S[pidx(elem<2>(l, kk))];
  run_stages<2, false>(x, l, 4, 2, T, q, qinv);
  __syncwarp();
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) S[pidx(elem<2>(l, kk))] = x[kk];
  __syncwarp();
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) x[kk] = S[pidx(elem<1>(l, kk))];
  run_stages<1, false>(x, l, 7, 5, T, q, qinv);
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) dst[elem<1>(l, kk)] = d2raw(x[kk]);
}

// ---------------------------------------------------------------- pass A (columns), R = 256
// CTA = 512 threads: column c = tid & 15 of a 16-column strip, virtual lane l = tid >> 4.
// grid = (256/16, n_limbs)
template <bool FWD>
__global__ void __launch_bounds__(512) k_ntt_cols256(LimbBatch b, DevTables dt, int logN) {
  __shared__ double sm[16 * 273];
  __shared__ double T[256];
  const int limb = blockIdx.y, c = threadIdx.x & 15, l = threadIdx.x >> 4;
  const int col = blockIdx.x * 16 + c;
  const int t = b.chain[limb];
  const size_t N = (size_t)1 << logN;
  const PrimeConst& pc = dt.pc[t];
  const double q = pc.qd, qinv = pc.qinv;
  const double* W = (FWD ? dt.tw : dt.itw) + (size_t)t * N;
  const uint64_t* src = FWD ? b.src[limb] : b.dst[limb];  // inverse runs in place after pass B
  uint64_t* dst = b.dst[limb];
  double* S = sm + c * 273;
  double x[8];
  if (FWD) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = u2d(src[(size_t)elem<1>(l, k) * 256 + col]);
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = raw2d(src[(size_t)elem<3>(l, k) * 256 + col]);
  }
  load_twiddles(T, W, 1, threadIdx.x, blockDim.x);
  __syncthreads();
  if (FWD) {
    run_stages<1, true>(x, l, 7, 5, T, q, qinv);
#pragma unroll
    for (int k = 0; k < 8; ++k) S[elem<1>(l, k)] = x[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = S[elem<2>(l, k)];
    run_stages<2, true>(x, l, 4, 2, T, q, qinv);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 8; ++k) S[elem<2>(l, k)] = x[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = S[elem<3>(l, k)];
    run_stages<3, true>(x, l, 1, 0, T, q, qinv);
#pragma unroll
    for (int k = 0; k < 8; ++k) dst[(size_t)elem<3>(l, k) * 256 + col] = d2raw(fred(x[k], q, qinv));
  } else {
    run_stages<3, false>(x, l, 1, 0, T, q, qinv);
#pragma unroll
    for (int k = 0; k < 8; ++k) S[elem<3>(l, k)] = x[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = S[elem<2>(l, k)];
    run_stages<2, false>(x, l, 4, 2, T, q, qinv);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 8; ++k) S[elem<2>(l, k)] = x[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = S[elem<1>(l, k)];
    run_stages<1, false>(x, l, 7, 5, T, q, qinv);
#pragma unroll
    for (int k = 0; k < 8; ++k)
      dst[(size_t)elem<1>(l, k) * 256 + col] = d2u(fcanon(fmulmod(x[k], pc.n_inv_d, q, qinv), q, qinv));
  }
}

// ---------------------------------------------------------------- pass A, generic R < 256
// CTA = 256 threads on a strip of 16 columns x R rows held in shared memory (exact
// canonical arithmetic per butterfly: only used for N < 2^16).
template <bool FWD>
__global__ void __launch_bounds__(256) k_ntt_cols_small(LimbBatch b, DevTables dt, int logN) {
  __shared__ double sm[128 * 16];
  const int limb = blockIdx.y;
  const int logR = logN - 8, R = 1 << logR;
  const int t = b.chain[limb];
  const size_t N = (size_t)1 << logN;
  const PrimeConst& pc = dt.pc[t];
  const double q = pc.qd, qinv = pc.qinv;
  const double* W = (FWD ? dt.tw : dt.itw) + (size_t)t * N;
  const uint64_t* src = FWD ? b.src[limb] : b.dst[limb];
  uint64_t* dst = b.dst[limb];
  const int col0 = blockIdx.x * 16;
  for (int i = threadIdx.x; i < R * 16; i += blockDim.x) {
    int r = i >> 4, c = i & 15;
    sm[i] = FWD ? u2d(src[(size_t)r * 256 + col0 + c]) : raw2d(src[(size_t)r * 256 + col0 + c]);
  }
  __syncthreads();
  for (int it = 0; it < logR; ++it) {
    const int s = FWD ? logR - 1 - it : it;
    const int half = 1 << s;
    for (int bf = threadIdx.x; bf < (R / 2) * 16; bf += blockDim.x) {
      int c = bf & 15, j = bf >> 4;                       // butterfly j in [0, R/2)
      int r = ((j >> s) << (s + 1)) | (j & (half - 1));   // lower element row
      const double w = W[(uint32_t)(R + r) >> (s + 1)];
      const double a = sm[r * 16 + c], bb = sm[(r + half) * 16 + c];
      if (FWD) {
        const double tt = fmulmod(bb, w, q, qinv);
        sm[r * 16 + c] = fred(a + tt, q, qinv);
        sm[(r + half) * 16 + c] = fred(a - tt, q, qinv);
      } else {
        sm[r * 16 + c] = fred(a + bb, q, qinv);
        sm[(r + half) * 16 + c] = fmulmod(a - bb, w, q, qinv);
      }
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < R * 16; i += blockDim.x) {
    int r = i >> 4, c = i & 15;
    double v = sm[i];
    if (!FWD) v = fmulmod(v, pc.n_inv_d, q, qinv);
    dst[(size_t)r * 256 + col0 + c] = FWD ? d2raw(v) : d2u(fcanon(v, q, qinv));
  }
}

// ---------------------------------------------------------------- pass B fused with the key-switch IP
// The forward row stages of one 256-word row, layout L1 in -> layout L3 out (values |v| <= 5.81 q from the
// between-pass format, DESIGN R-FP64; not canonicalised), S = the warp's transpose buffer, T = the row's twiddle heap.
__device__ __forceinline__ void rows_forward_l3(double (&x)[8], int l, double* S, const double* T, double q,
                                                double qinv) {
  run_stages<1, true>(x, l, 7, 5, T, q, qinv);
#pragma unroll
  for (int k = 0; k < 8; ++k) S[pidx(elem<1>(l, k))] = x[k];
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = S[pidx(elem<2>(l, k))];
  run_stages<2, true>(x, l, 4, 2, T, q, qinv);
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 8; ++k) S[pidx(elem<2>(l, k))] = x[k];
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = S[pidx(elem<3>(l, k))];
  run_stages<3, true>(x, l, 1, 0, T, q, qinv);
  __syncwarp();
}

// The inverse row stages of one 256-word row from layout L3 (|v| <= q/2 + 1) to layout L1 (between-pass
// format, as k_ntt_rows<false> leaves it), S = the warp's transpose buffer, T = the row's inverse heap.
__device__ __forceinline__ void rows_inverse_from_l3(double (&x)[8], int l, double* S, const double* T, double q,
                                                     double qinv) {
  run_stages<3, false>(x, l, 1, 0, T, q, qinv);
#pragma unroll
  for (int k = 0; k < 8; ++k) S[pidx(elem<3>(l, k))] = x[k];
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = S[pidx(elem<2>(l, k))];
  run_stages<2, false>(x, l, 4, 2, T, q, qinv);
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 8; ++k) S[pidx(elem<2>(l, k))] = x[k];
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = S[pidx(elem<1>(l, k))];
  run_stages<1, false>(x, l, 7, 5, T, q, qinv);
}

// Layout L3 holds words 4(l + 32h) + m (m < 4) in x[4h + m]: two 32-byte runs per lane.
__device__ __forceinline__ void load_l3(const uint64_t* __restrict__ p, int l, ulonglong2 (&v)[4], bool stream) {
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const ulonglong2* a = reinterpret_cast<const ulonglong2*>(p + 4 * (l + 32 * h) + 2 * i);
      v[2 * h + i] = stream ? __ldcs(a) : *a;
    }
}
// The same layout from a packed key limb (hy_arith.cuh): the 4 words 4(l + 32h)..+3 of row `roff` are the
// 24 bytes at uint64 3(l + 32h) of the 192-uint64 packed row (streaming loads).
__device__ __forceinline__ void load_l3_evk(const uint64_t* __restrict__ limb, size_t roff, int l,
                                            ulonglong2 (&v)[4]) {
  const uint64_t* r = limb + roff / 4 * 3;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const uint64_t* p = r + 3 * (l + 32 * h);
    uint64_t w0, w1, w2, w3;
    evk_unpack4(__ldcs(p), __ldcs(p + 1), __ldcs(p + 2), w0, w1, w2, w3);
    v[2 * h] = make_ulonglong2(w0, w1);
    v[2 * h + 1] = make_ulonglong2(w2, w3);
  }
}
__device__ __forceinline__ double l3_word(const ulonglong2 (&v)[4], int k) {
  const ulonglong2 w = v[k >> 1];
  return u2d((k & 1) ? w.y : w.x);
}
__device__ __forceinline__ void store_l3(uint64_t* p, int l, const double (&x)[8], double q, double qinv,
                                         bool accumulate) {
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      ulonglong2* a = reinterpret_cast<ulonglong2*>(p + 4 * (l + 32 * h) + 2 * i);
      double lo = x[4 * h + 2 * i], hi = x[4 * h + 2 * i + 1];
      if (accumulate) {
        const ulonglong2 o = *a;
        lo += u2d(o.x);
        hi += u2d(o.y);
      }
      *a = make_ulonglong2(d2u(fcanon(lo, q, qinv)), d2u(fcanon(hi, q, qinv)));
    }
}

// One warp per (item g, extended limb u, row): for every digit j it runs the row stages of
// ext_g[j][u] (the column pass already done; the own digit's limb own_g[u] is already in the NTT
// domain) and multiplies the result, still in registers, by the evk rows of (j, c = 0, 1).  The B
// products per word are reduced with fmulmod (|.| <= 1.5 t) and summed exactly (< 2^53), then
// canonicalised once; the NTT'd digits never reach HBM.  The twiddle heap of (chain(u), row) is
// loaded once and serves all B digits.  grid (G or 1 (SUM), R/8, E), CTA = 8 warps = 8 rows; the
// item index is the fastest grid dimension so that items sharing a key hit its rows in L2.
// SUM: one warp loops over all G items and accumulates into u[0] (each item's sum re-centred with
// fred first), race-free because one warp owns (u, row).
// HOIST: the digits are the NTT-domain extended digits of one shared ModUp, read through the Galois permutation
// kx_g of each item (Halevi-Shoup; used for the P limbs of the hoisted batch, with inv_p).
template <int B, bool SUM, bool HOIST>
__global__ void __launch_bounds__(256, 2) k_ntt_rows_ip(const __grid_constant__ RowsIpArgs a, int G, DevTables dt,
                                                        int level, int n_q, int L1, int E, int alpha, int logN,
                                                        int accumulate, int u0, int inv_p) {
  __shared__ double sm[8][272];
  __shared__ double tws[8][256];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const size_t N = (size_t)1 << logN;
  const int R = (int)(N >> 8);
  const int row = blockIdx.y * 8 + w, u = u0 + (int)blockIdx.z;
  if (row >= R) return;  // N = 2^10: 4 rows in an 8-warp CTA (warp-level sync only below)
  const int t = u <= level ? u : n_q + (u - level - 1);
  const PrimeConst& pc = dt.pc[t];
  const double q = pc.qd, qinv = pc.qinv;
  const int own_digit = u <= level ? u / alpha : -1;
  double* S = sm[w];
  double* T = tws[w];
  load_twiddles_warp(T, dt.tw + (size_t)t * N, (uint32_t)R + (uint32_t)row, l);
  __syncwarp();
  const size_t roff = (size_t)row * 256;
  double s0[8], s1[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) s0[k] = s1[k] = 0.0;
  const int g0 = SUM ? 0 : (int)blockIdx.x, g1 = SUM ? G : g0 + 1;
  for (int g = g0; g < g1; ++g) {
    double a0[8], a1[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a0[k] = a1[k] = 0.0;
#pragma unroll 1
    for (int j = 0; j < B; ++j) {
      ulonglong2 k0[4], k1[4];
      load_l3_evk(evk_limb(a.evk[g], (size_t)(j * 2) * L1 + t, N), roff, l, k0);
      load_l3_evk(evk_limb(a.evk[g], (size_t)(j * 2 + 1) * L1 + t, N), roff, l, k1);
      double x[8];
      if (HOIST) {
        const uint64_t kx = a.kx[g];
        const uint64_t* src = j == own_digit ? a.own[g] + (size_t)u * N : a.ext[g] + ((size_t)j * E + u) * N;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t xi = (uint32_t)(roff + elem<3>(l, k));
          x[k] = u2d(src[kx != 1 ? aut_index(xi, kx, logN) : xi]);
        }
      } else if (j == own_digit) {
        ulonglong2 v[4];
        load_l3(a.own[g] + (size_t)u * N + roff, l, v, false);
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = l3_word(v, k);
      } else {
        const uint64_t* src = a.ext[g] + ((size_t)j * E + u) * N + roff;
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = raw2d(src[elem<1>(l, k)]);
        rows_forward_l3(x, l, S, T, q, qinv);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        a0[k] += fmulmod(x[k], l3_word(k0, k), q, qinv);
        a1[k] += fmulmod(x[k], l3_word(k1, k), q, qinv);
      }
    }
    if (SUM) {
      // |fred| <= q/2 + 1 < 2^47: re-centre every 32 items so the running sum stays below 2^52 (exact)
      const bool wrap = (g & 31) == 31;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        s0[k] += fred(a0[k], q, qinv);
        s1[k] += fred(a1[k], q, qinv);
        if (wrap) {
          s0[k] = fred(s0[k], q, qinv);
          s1[k] = fred(s1[k], q, qinv);
        }
      }
    } else if (inv_p) {
      // split ModDown: the P limb's inverse row pass straight from registers (layout L3), stored in the
      // between-pass format for the ModDown column kernel: v_g[c][u - (l+1)]
      __syncwarp();
      load_twiddles_warp(T, dt.itw + (size_t)t * N, (uint32_t)R + (uint32_t)row, l);
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        double x[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fred(c ? a1[k] : a0[k], q, qinv);
        __syncwarp();
        rows_inverse_from_l3(x, l, S, T, q, qinv);
        uint64_t* dst = a.v[g] + ((size_t)c * (E - level - 1) + (u - level - 1)) * N + roff;
#pragma unroll
        for (int k = 0; k < 8; ++k) dst[elem<1>(l, k)] = d2raw(x[k]);
      }
    } else {
      store_l3(a.u[g] + (size_t)u * N + roff, l, a0, q, qinv, accumulate);
      store_l3(a.u[g] + ((size_t)E + u) * N + roff, l, a1, q, qinv, accumulate);
    }
  }
  if (SUM) {
    store_l3(a.u[0] + (size_t)u * N + roff, l, s0, q, qinv, accumulate);
    store_l3(a.u[0] + ((size_t)E + u) * N + roff, l, s1, q, qinv, accumulate);
  }
}

// ---------------------------------------------------------------- pass B fused with the ModDown epilogue
// One warp per (item g, poly c, limb i <= level, row): the row stages of w_g[c][i] (column pass done),
// then in layout L3: (u - w) P^{-1} (fmulmod, |u - w| <= q + 5.81 q) plus the optional addends, canonicalised
// once.  grid (R/8, l+1, npoly * G), blockIdx.z = g * npoly + c.
__global__ void __launch_bounds__(256) k_ntt_rows_final(const __grid_constant__ RowsFinalArgs a, int npoly, int E,
                                                        const ModDownConst* md, DevTables dt, int level, int logN) {
  __shared__ double sm[8][272];
  __shared__ double tws[8][256];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const size_t N = (size_t)1 << logN;
  const int R = (int)(N >> 8);
  const int row = blockIdx.x * 8 + w, i = blockIdx.y;
  const int g = blockIdx.z / npoly, c = blockIdx.z % npoly;
  if (row >= R) return;
  const PrimeConst& pc = dt.pc[i];
  const double q = pc.qd, qinv = pc.qinv;
  double* S = sm[w];
  double* T = tws[w];
  load_twiddles_warp(T, dt.tw + (size_t)i * N, (uint32_t)R + (uint32_t)row, l);
  const size_t roff = (size_t)row * 256;
  const uint64_t* src = a.w[g] + ((size_t)c * (level + 1) + i) * N + roff;
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = raw2d(src[elem<1>(l, k)]);
  __syncwarp();
  rows_forward_l3(x, l, S, T, q, qinv);
  ulonglong2 uv[4];
  load_l3(a.u[g] + ((size_t)c * E + i) * N + roff, l, uv, false);
  const double pinv = (double)md->p_inv[i];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = fmulmod(l3_word(uv, k) - x[k], pinv, q, qinv);
  if (c == 0 && a.add0[g]) {
    const uint64_t* a0 = a.add0[g] + (size_t)i * N;
    const uint64_t k0 = a.k0[g];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t xi = (uint32_t)(roff + elem<3>(l, k));
      x[k] += u2d(a0[k0 != 1 ? aut_index(xi, k0, logN) : xi]);
    }
  }
  if (c == 1 && a.add1[g]) {
    ulonglong2 v[4];
    load_l3(a.add1[g] + (size_t)i * N + roff, l, v, false);
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] += l3_word(v, k);
  }
  uint64_t* o = a.out[g] + ((size_t)c * (level + 1) + i) * N + roff;
  if (a.addct[g]) {
    ulonglong2 v[4];
    load_l3(a.addct[g] + ((size_t)c * (level + 1) + i) * N + roff, l, v, false);
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] += l3_word(v, k);
  }
  store_l3(o, l, x, q, qinv, false);
}

// ---------------------------------------------------------------- Q-limb IP fused with the ModDown epilogue
// One warp per (item g, limb i <= level, row), both polys: the inner product of the digits' row i with the
// evk rows (plain: row pass of the column-pass output; hoisted: NTT-domain digits gathered through kx_g),
// kept in registers; then for c = 0, 1 the row pass of the conversion w_g[c][i] and
// out = (fred(acc_c) - w) P^{-1} (+ addends), canonicalised once.  |fred(acc) - w| <= q/2 + 1 + 5.81 q.
// grid (G, R/8, l+1): the item index is the fastest grid dimension (hoisted items share their digits).
template <int B, bool HOIST>
__global__ void __launch_bounds__(256, 2) k_rows_ip_final(const __grid_constant__ IpFinalArgs a, DevTables dt,
                                                          const ModDownConst* md, int level, int L1, int E,
                                                          int alpha, int logN) {
  __shared__ double sm[8][272];
  __shared__ double tws[8][256];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const size_t N = (size_t)1 << logN;
  const int R = (int)(N >> 8);
  const int g = blockIdx.x, row = blockIdx.y * 8 + w, i = blockIdx.z;
  if (row >= R) return;  // N = 2^10: 4 rows in an 8-warp CTA (warp-level sync only below)
  const PrimeConst& pc = dt.pc[i];
  const double q = pc.qd, qinv = pc.qinv;
  const int own_digit = i / alpha;
  double* S = sm[w];
  double* T = tws[w];
  load_twiddles_warp(T, dt.tw + (size_t)i * N, (uint32_t)R + (uint32_t)row, l);
  __syncwarp();
  const size_t roff = (size_t)row * 256;
  // gathered positions: hoisted -- every digit; plain -- the own digit, read from c1 through kappa_kx
  uint32_t gi[8];
  const uint64_t kx = a.kx[g];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t xi = (uint32_t)(roff + elem<3>(l, k));
    gi[k] = kx != 1 ? aut_index(xi, kx, logN) : xi;
  }
  double a0[8], a1[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a0[k] = a1[k] = 0.0;
#pragma unroll 1
  for (int j = 0; j < B; ++j) {
    ulonglong2 k0[4], k1[4];
    load_l3_evk(evk_limb(a.evk[g], (size_t)(j * 2) * L1 + i, N), roff, l, k0);
    load_l3_evk(evk_limb(a.evk[g], (size_t)(j * 2 + 1) * L1 + i, N), roff, l, k1);
    double x[8];
    if (HOIST) {
      const uint64_t* src = j == own_digit ? a.own[g] + (size_t)i * N : a.ext[g] + ((size_t)j * E + i) * N;
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = u2d(src[gi[k]]);
    } else if (j == own_digit) {
      const uint64_t* src = a.own[g] + (size_t)i * N;
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = u2d(src[gi[k]]);
    } else {
      const uint64_t* src = a.ext[g] + ((size_t)j * E + i) * N + roff;
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = raw2d(src[elem<1>(l, k)]);
      rows_forward_l3(x, l, S, T, q, qinv);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      a0[k] += fmulmod(x[k], l3_word(k0, k), q, qinv);
      a1[k] += fmulmod(x[k], l3_word(k1, k), q, qinv);
    }
  }
  const double pinv = (double)md->p_inv[i];
#pragma unroll 1
  for (int c = 0; c < 2; ++c) {
    const uint64_t* src = a.w[g] + ((size_t)c * (level + 1) + i) * N + roff;
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = raw2d(src[elem<1>(l, k)]);
    __syncwarp();
    rows_forward_l3(x, l, S, T, q, qinv);
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fmulmod(fred(c ? a1[k] : a0[k], q, qinv) - x[k], pinv, q, qinv);
    if (c == 0 && a.add0[g]) {
      const uint64_t* p0 = a.add0[g] + (size_t)i * N;
      const uint64_t k0 = a.k0[g];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t xi = (uint32_t)(roff + elem<3>(l, k));
        x[k] += u2d(p0[k0 != 1 ? aut_index(xi, k0, logN) : xi]);
      }
    }
    if (c == 1 && a.add1[g]) {
      ulonglong2 v[4];
      load_l3(a.add1[g] + (size_t)i * N + roff, l, v, false);
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] += l3_word(v, k);
    }
    const size_t o = ((size_t)c * (level + 1) + i) * N + roff;
    if (a.addct[g]) {
      ulonglong2 v[4];
      load_l3(a.addct[g] + o, l, v, false);
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] += l3_word(v, k);
    }
    store_l3(a.out[g] + o, l, x, q, qinv, false);
  }
}

// ---------------------------------------------------------------- the same, rows staged by bulk async copies
// (TMA bulk engine, cp.async.bulk + mbarrier): every 2 KB row a warp consumes -- the two evk rows and the
// digit row of each digit, then the two conversion rows w_g[0][i], w_g[1][i] and the c0 row of the gather --
// is copied global -> shared by one lane one step ahead (two stages per warp), so the row loads of digit
// j + 1 are in flight while digit j is transformed and multiplied, without staging registers.  The digit
// row's stage buffer doubles as the warp's transpose buffer once it is in registers.  Hoisted: the Galois
// permutation maps a 256-word row onto one row (the high index bits of kappa depend only on high bits), so
// the source row is copied whole and gathered from shared memory.

// per warp: twiddle heap + NST stages x (e0, e1, x) rows, and NST mbarriers
__host__ __device__ constexpr int rows_warp_words(int nst) { return 256 * (1 + 3 * nst); }
constexpr size_t rows_tma_smem(int nst) { return 8 * ((size_t)rows_warp_words(nst) * 8 + 8 * nst); }

// (item g, row block by, Q limb i) of the Q-limb kernel; dsm = rows_tma_smem(NST) bytes of dynamic smem
// PL (P-limb mode, split ModDown): i = the special prime k; the B digit iterations only (no own digit), then the
// inverse row pass of the two products stored into a.out[g] + (c K + k) N in the between-pass format (the input
// of the ModDown column kernel).  Otherwise i = the Q limb and the ModDown epilogue follows.
template <int B, bool HOIST, int NST, bool PL = false>
__device__ __forceinline__ void rows_ip_final_tma_body(const IpFinalArgs& a, const DevTables& dt,
                                                       const ModDownConst* md, int level, int L1, int E, int alpha,
                                                       int logN, double* dsm, int g, int by, int ii) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const size_t N = (size_t)1 << logN;
  const int R = (int)(N >> 8);
  const int row = by * 8 + w;
  if (row >= R) return;  // N = 2^10: 4 rows in an 8-warp CTA (warp-level sync only below)
  double* T = dsm + (size_t)w * rows_warp_words(NST);  // stage s at T + 256 + 768 s: e0, e1, digit (x) rows
  uint64_t* mbar = reinterpret_cast<uint64_t*>(dsm + 8 * rows_warp_words(NST)) + NST * w;
  const int K = E - level - 1;
  const int i = PL ? L1 - K + ii : ii;      // chain index of the limb (Q: the limb itself)
  const int ui = PL ? level + 1 + ii : ii;  // its index among the extended limbs
  constexpr int LAST = PL ? B - 1 : B;      // last iteration (Q: the epilogue)
  const PrimeConst& pc = dt.pc[i];
  const double q = pc.qd, qinv = pc.qinv;
  const int own_digit = PL ? -1 : i / alpha;
  const size_t roff = (size_t)row * 256;
  // source rows of the permuted reads (hoisted digits; the c0 gather)
  // kx: hoisted -- every digit is read through kappa_kx; plain -- the own digit (c1 itself, kappa fused here)
  const uint32_t rowx = a.kx[g] != 1 ? aut_index((uint32_t)roff, a.kx[g], logN) >> 8 : (uint32_t)row;
  const uint64_t k0 = a.add0[g] ? a.k0[g] : 1;
  const uint32_t row0 = k0 != 1 ? aut_index((uint32_t)roff, k0, logN) >> 8 : (uint32_t)row;
  // iteration j < B: digit j; j == B: the ModDown epilogue (w rows and the c0 row)
  auto issue = [&](int j) {
    double* b = T + 256 + 768 * (j % NST);
    uint64_t* mb = mbar + j % NST;
    if (j < B) {
      // packed key rows: 1536 bytes each (hy_arith.cuh), at the start of their 2048-byte stage slots
      const uint64_t* e0 = evk_limb(a.evk[g], (size_t)(j * 2) * L1 + i, N) + roff / 4 * 3;
      const uint64_t* e1 = evk_limb(a.evk[g], (size_t)(j * 2 + 1) * L1 + i, N) + roff / 4 * 3;
      const uint64_t* xs = (j == own_digit ? a.own[g] + (size_t)i * N : a.ext[g] + ((size_t)j * E + ui) * N) +
                           ((HOIST || j == own_digit) ? (size_t)rowx * 256 : roff);
      tma::mbar_expect(mb, 2 * 1536 + 2048);
      tma::bulk_row(b, e0, mb, 1536);
      tma::bulk_row(b + 256, e1, mb, 1536);
      tma::bulk_row(b + 512, xs, mb);
    } else {
      const bool c0 = a.add0[g] != nullptr;
      tma::mbar_expect(mb, (c0 ? 3 : 2) * 2048);
      tma::bulk_row(b, a.w[g] + (size_t)i * N + roff, mb);
      tma::bulk_row(b + 256, a.w[g] + ((size_t)(level + 1) + i) * N + roff, mb);
      if (c0) tma::bulk_row(b + 512, a.add0[g] + (size_t)i * N + (size_t)row0 * 256, mb);
    }
  };
  // hoisted: in-row positions of the 8 gathered words, packed 4 per register
  uint32_t gpk[2] = {0, 0};
  {
    const uint64_t kx = a.kx[g];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t xi = (uint32_t)(roff + elem<3>(l, k));
      gpk[k >> 2] |= ((kx != 1 ? aut_index(xi, kx, logN) : xi) & 255u) << (8 * (k & 3));
    }
  }
  if (l == 0) {
    for (int t = 0; t < NST; ++t) tma::mbar_init(mbar + t);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int t = 0; t < NST - 1 && t <= LAST; ++t) issue(t);
  }
  load_twiddles_warp(T, dt.tw + (size_t)i * N, (uint32_t)R + (uint32_t)row, l);
  __syncwarp();
  double a0[8], a1[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a0[k] = a1[k] = 0.0;
#pragma unroll 1
  for (int j = 0; j <= LAST; ++j) {
    if (l == 0 && j + NST - 1 <= LAST) issue(j + NST - 1);  // its stage was released at the end of j - 1
    double* b = T + 256 + 768 * (j % NST);
    tma::mbar_wait(mbar + j % NST, (uint32_t)(j / NST) & 1);
    if (j < B) {
      double x[8];
      const uint64_t* xb = reinterpret_cast<const uint64_t*>(b + 512);
      if (HOIST || j == own_digit) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = u2d(xb[(gpk[k >> 2] >> (8 * (k & 3))) & 255]);
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = raw2d(xb[elem<1>(l, k)]);
        __syncwarp();
        rows_forward_l3(x, l, b + 512, T, q, qinv);  // the row buffer is now the transpose buffer
      }
      // the packed evk rows in layout L3: elements 4h..4h+3 = words 4(l + 32h)..+3 = the 24 bytes at
      // uint64 3(l + 32h) (8-byte reads at a 24-byte lane stride: conflict-free per half-warp)
      const uint64_t* e0 = reinterpret_cast<const uint64_t*>(b);
      const uint64_t* e1 = reinterpret_cast<const uint64_t*>(b + 256);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int o = 3 * (l + 32 * h);
        uint64_t v0[4], v1[4];
        evk_unpack4(e0[o], e0[o + 1], e0[o + 2], v0[0], v0[1], v0[2], v0[3]);
        evk_unpack4(e1[o], e1[o + 1], e1[o + 2], v1[0], v1[1], v1[2], v1[3]);
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          a0[4 * h + m] += fmulmod(x[4 * h + m], u2d(v0[m]), q, qinv);
          a1[4 * h + m] += fmulmod(x[4 * h + m], u2d(v1[m]), q, qinv);
        }
      }
    } else {
      const double pinv = (double)md->p_inv[i];
      const uint64_t* c0b = reinterpret_cast<const uint64_t*>(b + 512);
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        const uint64_t* wb = reinterpret_cast<const uint64_t*>(b + 256 * c);
        double x[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = raw2d(wb[elem<1>(l, k)]);
        __syncwarp();
        rows_forward_l3(x, l, b + 256 * c, T, q, qinv);  // w_c's own buffer as the transpose buffer
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fmulmod(fred(c ? a1[k] : a0[k], q, qinv) - x[k], pinv, q, qinv);
        if (c == 0 && a.add0[g]) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint32_t xi = (uint32_t)(roff + elem<3>(l, k));
            x[k] += u2d(c0b[(k0 != 1 ? aut_index(xi, k0, logN) : xi) & 255]);
          }
        }
        if (c == 1 && a.add1[g]) {
          ulonglong2 v[4];
          load_l3(a.add1[g] + (size_t)i * N + roff, l, v, false);
#pragma unroll
          for (int k = 0; k < 8; ++k) x[k] += l3_word(v, k);
        }
        const size_t o = ((size_t)c * (level + 1) + i) * N + roff;
        if (a.addct[g]) {
          ulonglong2 v[4];
          load_l3(a.addct[g] + o, l, v, false);
#pragma unroll
          for (int k = 0; k < 8; ++k) x[k] += l3_word(v, k);
        }
        store_l3(a.out[g] + o, l, x, q, qinv, false);
      }
    }
    // release the stage: every lane's generic accesses before the next bulk write into it (issued at j + 1 only when
    // j + NST <= LAST; the last iterations skip the fence, whose MEMBAR would wait for the epilogue's global stores)
    if (j + NST <= LAST) {
      tma::proxy_fence();
      __syncwarp();
    }
  }
  if constexpr (PL) {
    // the P limb's inverse row pass straight from registers (layout L3), stage 0's buffer as transpose space
    __syncwarp();
    load_twiddles_warp(T, dt.itw + (size_t)i * N, (uint32_t)R + (uint32_t)row, l);
    __syncwarp();
    double* S = T + 256;
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      double x[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fred(c ? a1[k] : a0[k], q, qinv);
      __syncwarp();
      rows_inverse_from_l3(x, l, S, T, q, qinv);
      uint64_t* dst = a.out[g] + ((size_t)c * K + ii) * N + roff;
#pragma unroll
      for (int k = 0; k < 8; ++k) dst[elem<1>(l, k)] = d2raw(x[k]);
    }
  }
}

template <int B, bool HOIST, int NST>
__global__ void __launch_bounds__(256, 2) k_rows_ip_final_tma(const __grid_constant__ IpFinalArgs a, DevTables dt,
                                                              const ModDownConst* md, int level, int L1, int E,
                                                              int alpha, int logN) {
  extern __shared__ __align__(128) double dsm[];
  rows_ip_final_tma_body<B, HOIST, NST>(a, dt, md, level, L1, E, alpha, logN, dsm, blockIdx.x, blockIdx.y,
                                        blockIdx.z);
}

// Lazy HRotSum inner product on the bulk-copy ring: u = sum over the G items and their B digits, every
// extended limb.  One warp per (row, limb u) walks the G x B (item, digit) rows through its NST-stage ring
// (keys packed, digits in the column-pass format, the own digit's limb from own_g = kappa_g(c1) in the NTT
// domain); the running sums are re-centred at every item boundary (|a| <= q/2 + 1 + 1.5 B q < 2^52, exact).
// a.out[0] = u [2][E][N] (accumulate: added to it).  grid (1, R/8, E)
template <int B>
__global__ void __launch_bounds__(256, 2) k_rows_ip_sum_tma(const __grid_constant__ IpFinalArgs a, int G,
                                                            DevTables dt, int level, int L1, int E, int alpha,
                                                            int logN, int accumulate) {
  constexpr int NST = 2;
  extern __shared__ __align__(128) double dsm[];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const size_t N = (size_t)1 << logN;
  const int R = (int)(N >> 8);
  const int row = blockIdx.y * 8 + w, u = blockIdx.z;
  if (row >= R) return;
  double* T = dsm + (size_t)w * rows_warp_words(NST);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(dsm + 8 * rows_warp_words(NST)) + NST * w;
  const int K = E - level - 1;
  const int t = u <= level ? u : L1 - K + (u - level - 1);
  const int own_digit = u <= level ? u / alpha : -1;
  const PrimeConst& pc = dt.pc[t];
  const double q = pc.qd, qinv = pc.qinv;
  const size_t roff = (size_t)row * 256;
  const int last = G * B - 1;
  const int gb = blockIdx.x * G;  // grouped (round 2): output blockIdx.x sums items gb .. gb + G - 1
  auto issue = [&](int it) {
    const int g = gb + it / B, j = it % B;
    double* b = T + 256 + 768 * (it % NST);
    uint64_t* mb = mbar + it % NST;
    const uint64_t* e0 = evk_limb(a.evk[g], (size_t)(j * 2) * L1 + t, N) + roff / 4 * 3;
    const uint64_t* e1 = evk_limb(a.evk[g], (size_t)(j * 2 + 1) * L1 + t, N) + roff / 4 * 3;
    // the own digit's limb: own_g itself, through kappa_{kx_g} (one source row) when kx_g != 1
    const uint64_t kx = a.kx[g];
    const size_t srow = (j == own_digit && kx != 1) ? (size_t)(aut_index((uint32_t)roff, kx, logN) >> 8) * 256 : roff;
    const uint64_t* xs = (j == own_digit ? a.own[g] + (size_t)u * N : a.ext[g] + ((size_t)j * E + u) * N) + srow;
    tma::mbar_expect(mb, 2 * 1536 + 2048);
    tma::bulk_row(b, e0, mb, 1536);
    tma::bulk_row(b + 256, e1, mb, 1536);
    tma::bulk_row(b + 512, xs, mb);
  };
  if (l == 0) {
    for (int s = 0; s < NST; ++s) tma::mbar_init(mbar + s);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < NST - 1 && s <= last; ++s) issue(s);
  }
  load_twiddles_warp(T, dt.tw + (size_t)t * N, (uint32_t)R + (uint32_t)row, l);
  __syncwarp();
  double a0[8], a1[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a0[k] = a1[k] = 0.0;
#pragma unroll 1
  for (int it = 0; it <= last; ++it) {
    if (l == 0 && it + NST - 1 <= last) issue(it + NST - 1);
    const int j = it % B;
    double* b = T + 256 + 768 * (it % NST);
    tma::mbar_wait(mbar + it % NST, (uint32_t)(it / NST) & 1);
    double x[8];
    const uint64_t* xb = reinterpret_cast<const uint64_t*>(b + 512);
    if (j == own_digit) {
      const uint64_t kx = a.kx[gb + it / B];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t xi = (uint32_t)(roff + elem<3>(l, k));
        x[k] = u2d(xb[(kx != 1 ? aut_index(xi, kx, logN) : xi) & 255]);
      }
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = raw2d(xb[elem<1>(l, k)]);
      __syncwarp();
      rows_forward_l3(x, l, b + 512, T, q, qinv);
    }
    const uint64_t* e0 = reinterpret_cast<const uint64_t*>(b);
    const uint64_t* e1 = reinterpret_cast<const uint64_t*>(b + 256);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int o = 3 * (l + 32 * h);
      uint64_t v0[4], v1[4];
      evk_unpack4(e0[o], e0[o + 1], e0[o + 2], v0[0], v0[1], v0[2], v0[3]);
      evk_unpack4(e1[o], e1[o + 1], e1[o + 2], v1[0], v1[1], v1[2], v1[3]);
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        a0[4 * h + m] += fmulmod(x[4 * h + m], u2d(v0[m]), q, qinv);
        a1[4 * h + m] += fmulmod(x[4 * h + m], u2d(v1[m]), q, qinv);
      }
    }
    if (j == B - 1) {  // item boundary: re-centre
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        a0[k] = fred(a0[k], q, qinv);
        a1[k] = fred(a1[k], q, qinv);
      }
    }
    if (it + NST <= last) {  // the stage is refilled at it + 1 (see rows_ip_final_tma_body)
      tma::proxy_fence();
      __syncwarp();
    }
  }
  store_l3(a.out[blockIdx.x] + (size_t)u * N + roff, l, a0, q, qinv, accumulate);
  store_l3(a.out[blockIdx.x] + ((size_t)E + u) * N + roff, l, a1, q, qinv, accumulate);
}

// P limbs of the IP (split ModDown) on the same bulk-copy ring: grid (G, R/8, K); a.out[g] = v_g [2][K][N]
template <int B, bool HOIST>
__global__ void __launch_bounds__(256, 2) k_rows_ip_p_tma(const __grid_constant__ IpFinalArgs a, DevTables dt,
                                                          int level, int L1, int E, int alpha, int logN) {
  extern __shared__ __align__(128) double dsm[];
  rows_ip_final_tma_body<B, HOIST, 2, true>(a, dt, nullptr, level, L1, E, alpha, logN, dsm, blockIdx.x, blockIdx.y,
                                            blockIdx.z);
}

// ---------------------------------------------------------------- iNTT column pass + fast BConv + NTT column pass
// CTA = 256 threads on one 8-column strip (thread: column c = tid & 7, lane l = tid >> 3; the
// k_ntt_cols256 scheme at half width, so that two CTAs of 126-register threads share an SM and one
// CTA's barriers are covered by the other's work) of item g = blockIdx.z and group blockIdx.y.
//   ModUp (DOWN = false), group = digit j: sources = the digit's A limbs of c1 (after the inverse row
//     pass), y_i = [d_i (D_j/q_i)^{-1}]_{q_i}; targets = every limb u of Q_l u P outside the digit,
//     x = [sum_i y_i ((D_j/q_i) mod t_u)]; out = ext_g[j][u].
//   ModDown (DOWN = true), group = poly c: sources = the K P-limbs of the inner product u_g[c] (after the
//     inverse row pass), z_k = [v_k (P/p_k)^{-1}]_{p_k}; targets = the l+1 limbs q_i,
//     x = [sum_k z_k ((P/p_k) mod q_i)]; out = w_g[c][i].
// Phase i < A: inverse column stages of source i, ending in layout L1 with the source word (canonical:
// the fast BConv lifts it as an integer) kept in registers; N^{-1} is folded into its constant.  Then one
// phase per target: x = fred(sum_i fmulmod(y_i, hat_i)) (|x| <= t/2 + 1) goes straight into the forward
// column stages and is stored fred-reduced (between-pass format, for the fused row kernels).  The
// coefficient-domain sources and the un-transformed conversion never reach HBM.  The next phase's
// twiddle heap is fetched into a register during the current phase (double-buffered T).
// shared memory of one column CTA: the 8-column strip, the double-buffered twiddle heap, the BConv constants
template <int A>
__host__ __device__ constexpr int cols_smem_words() { return 8 * 256 + 2 * 256 + kMaxExt * A; }

// YS (round 2): the source words y_1 .. y_{A-1} live in shared memory ([A-1][8][256] doubles after the strip, the
// twiddles and the constants) instead of registers, so the kernel fits 3 CTAs (24 warps) per SM
template <int A>
__host__ __device__ constexpr int cols_ys_words() { return (A - 1) * 8 * 256; }

// (strip bx, group j, item g); sm = cols_smem_words<A>() (+ cols_ys_words<A>() with YS) doubles of shared memory
template <int A, bool DOWN, bool YS = false>
__device__ __forceinline__ void bconv_cols_body(const ModUpColsArgs& a, const ModUpConst* mc, const ModDownConst* md,
                                                const DevTables& dt, int level, int n_q, int E, int logN,
                                                double* sm, int bx, int j, int g) {
  double* T = sm + 8 * 256;       // [2][256]
  double* s_hat = T + 2 * 256;    // [kMaxExt][A]
  const int c = threadIdx.x & 7, l = threadIdx.x >> 3, tid = threadIdx.x;
  const int col = bx * 8 + c;
  const size_t N = (size_t)1 << logN;
  const int n = level + 1;
  int lo = 0, nsrc = A, nph = A + n;  // DOWN: K sources, l+1 targets
  if constexpr (!DOWN) {
    lo = mc[j].lo;
    nsrc = mc[j].hi - mc[j].lo;
    nph = E;  // nsrc inverse phases + (E - nsrc) targets
  }
  for (int i = tid; i < (DOWN ? n : E) * A; i += blockDim.x) {
    const int u = i / A, ii = i % A;
    if constexpr (DOWN) s_hat[u * A + ii] = (double)md->phat_mod[u][ii];
    else s_hat[u * A + ii] = ii < nsrc ? (double)mc[j].hat_mod[u][ii] : 0.0;
  }
  // target phase p >= nsrc -> target index (ModUp: the (p - nsrc)-th ext limb outside [lo, hi))
  auto target = [&](int p) {
    const int k = p - nsrc;
    return (DOWN || k < lo) ? k : k + nsrc;
  };
  auto src_chain = [&](int p) { return DOWN ? (int)md->src0 + p : lo + p; };
  auto tgt_chain = [&](int u) { return (DOWN || u <= level) ? u : n_q + (u - level - 1); };
  auto table = [&](int p) -> const double* {
    if (p < nsrc) return dt.itw + (size_t)src_chain(p) * N;
    return dt.tw + (size_t)tgt_chain(target(p)) * N;
  };
  if (tid > 0 && tid < 256) T[tid] = table(0)[tid];
  constexpr int AR = YS ? 1 : A;  // sources held in registers
  double y[AR][8];
  double* ysm = sm + cols_smem_words<A>();  // YS: [A-1][8][256], word (i, k) of thread tid at ysm[(i*8+k)*256+tid]
#pragma unroll
  for (int i = 0; i < AR; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) y[i][k] = 0.0;
  if constexpr (YS) {
    for (int w = tid; w < cols_ys_words<A>(); w += blockDim.x) ysm[w] = 0.0;
  }
  __syncthreads();
  for (int p = 0; p < nph; ++p) {
    const double tw_next = (p + 1 < nph && tid > 0 && tid < 256) ? table(p + 1)[tid] : 0.0;
    const double* Tp = T + 256 * (p & 1);
    double x[8];
    if (p < nsrc) {  // inverse column pass of source p
      const PrimeConst& pc = dt.pc[src_chain(p)];
      const double q = pc.qd, qinv = pc.qinv;
      const uint64_t* src = a.src[g] + (size_t)(DOWN ? j * A + p : lo + p) * N + col;
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = raw2d(src[(size_t)elem<3>(l, k) * 256]);
      run_stages<3, false>(x, l, 1, 0, Tp, q, qinv);
#pragma unroll
      for (int k = 0; k < 8; ++k) sm[sidx8(elem<3>(l, k), c)] = x[k];
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = sm[sidx8(elem<2>(l, k), c)];
      run_stages<2, false>(x, l, 4, 2, Tp, q, qinv);
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 8; ++k) sm[sidx8(elem<2>(l, k), c)] = x[k];
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = sm[sidx8(elem<1>(l, k), c)];
      run_stages<1, false>(x, l, 7, 5, Tp, q, qinv);
      const double hinv = DOWN ? (double)md->phat_inv[p] : (double)mc[j].hat_inv[p];
      const double cst = fcanon(fmulmod(pc.n_inv_d, hinv, q, qinv), q, qinv);
      const bool center = DOWN && md->center;  // rescale: the centred remainder in (-q/2, q/2] (R-RESCALE)
      const double half = 0.5 * (q - 1.0);
#pragma unroll
      for (int i = 0; i < A; ++i)
        if (i == p) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const double v = fcanon(fmulmod(x[k], cst, q, qinv), q, qinv);
            const double yv = center && v > half ? v - q : v;
            if (i < AR) y[i < AR ? i : 0][k] = yv;
            else ysm[((i - 1) * 8 + k) * 256 + tid] = yv;
          }
        }
    } else {  // BConv to target u, then the forward column pass
      const int u = target(p);
      const PrimeConst& pc = dt.pc[tgt_chain(u)];
      const double q = pc.qd, qinv = pc.qinv;
      double h[A];
#pragma unroll
      for (int i = 0; i < A; ++i) h[i] = s_hat[u * A + i];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i < A; ++i)
          acc += fmulmod(i < AR ? y[i < AR ? i : 0][k] : ysm[((i - 1) * 8 + k) * 256 + tid], h[i], q, qinv);
        x[k] = fred(acc, q, qinv);
      }
      run_stages<1, true>(x, l, 7, 5, Tp, q, qinv);
#pragma unroll
      for (int k = 0; k < 8; ++k) sm[sidx8(elem<1>(l, k), c)] = x[k];
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = sm[sidx8(elem<2>(l, k), c)];
      run_stages<2, true>(x, l, 4, 2, Tp, q, qinv);
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 8; ++k) sm[sidx8(elem<2>(l, k), c)] = x[k];
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = sm[sidx8(elem<3>(l, k), c)];
      run_stages<3, true>(x, l, 1, 0, Tp, q, qinv);
      uint64_t* dst = a.ext[g] + (size_t)(DOWN ? j * n + u : j * E + u) * N + col;
#pragma unroll
      for (int k = 0; k < 8; ++k) dst[(size_t)elem<3>(l, k) * 256] = d2raw(fred(x[k], q, qinv));
    }
    if (tid > 0 && tid < 256) T[256 * ((p + 1) & 1) + tid] = tw_next;
    __syncthreads();
  }
}

template <int A, bool DOWN>
__global__ void __launch_bounds__(256, 2) k_bconv_cols(const __grid_constant__ ModUpColsArgs a,
                                                       const ModUpConst* mc, const ModDownConst* md, DevTables dt,
                                                       int level, int n_q, int E, int logN) {
  __shared__ double sm[cols_smem_words<A>()];
  bconv_cols_body<A, DOWN>(a, mc, md, dt, level, n_q, E, logN, sm, blockIdx.x, blockIdx.y, blockIdx.z);
}

// the YS variant: 3 CTAs per SM (<= 85 registers), dynamic shared memory
template <int A, bool DOWN>
__global__ void __launch_bounds__(256, 3) k_bconv_cols_ys(const __grid_constant__ ModUpColsArgs a,
                                                          const ModUpConst* mc, const ModDownConst* md, DevTables dt,
                                                          int level, int n_q, int E, int logN) {
  extern __shared__ __align__(16) double dsm_cols[];
  bconv_cols_body<A, DOWN, true>(a, mc, md, dt, level, n_q, E, logN, dsm_cols, blockIdx.x, blockIdx.y, blockIdx.z);
}
template <int A>
constexpr size_t cols_ys_smem() { return (size_t)(cols_smem_words<A>() + cols_ys_words<A>()) * 8; }
bool cols_ys_on() {
  static const bool on = getenv("HY_COLS_YS") != nullptr && atoi(getenv("HY_COLS_YS")) != 0;  // A/B only: slower (r02h)
  return on;
}
template <int A, bool DOWN>
void launch_cols_ys(dim3 grid, cudaStream_t s, const ModUpColsArgs& a, const ModUpConst* mc, const ModDownConst* md,
                    const DevTables& dt, int lv, int nq, int E, int lg) {
  static bool at = false;
  if (!at) {
    cudaFuncSetAttribute(k_bconv_cols_ys<A, DOWN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cols_ys_smem<A>());
    at = true;
  }
  k_bconv_cols_ys<A, DOWN><<<grid, 256, cols_ys_smem<A>(), s>>>(a, mc, md, dt, lv, nq, E, lg);
}

}  // namespace

bool modup_cols_ok(const hy_ctx* c) { return c->N == 65536 && c->alpha <= 4; }
bool moddown_cols_ok(const hy_ctx* c) { return c->N == 65536 && c->n_p <= 4; }

void launch_ntt_rows(hy_ctx* c, const LimbBatch& b, bool inverse, cudaStream_t s) {
  if (b.n == 0) return;
  const int R = (int)c->N / 256;
  dim3 gB(R / 8 > 0 ? R / 8 : 1, b.n);
  KTimer kt(c, FAM_NTT_B, s);
  kt.bytes = 2ull * b.n * c->N * 8;
  if (inverse) k_ntt_rows<false><<<gB, 256, 0, s>>>(b, c->dt, (int)c->log_n);
  else k_ntt_rows<true><<<gB, 256, 0, s>>>(b, c->dt, (int)c->log_n);
}

void launch_ntt_rows_inv_aut(hy_ctx* c, const RowsAutArgs& a, int G, uint32_t level, cudaStream_t s) {
  if (G <= 0) return;
  const int R = (int)c->N / 256;
  dim3 grid(R / 8 > 0 ? R / 8 : 1, level + 1, G);
  KTimer kt(c, FAM_NTT_B, s);
  kt.bytes = 2ull * G * (level + 1) * c->N * 8;
  k_ntt_rows_inv_aut<<<grid, 256, 0, s>>>(a, c->dt, (int)c->log_n);
}

void launch_modup_cols(hy_ctx* c, const ModUpColsArgs& a, int G, uint32_t level, cudaStream_t s) {
  if (G <= 0) return;
  const int n = (int)level + 1, E = n + (int)c->n_p, beta = (int)n_digits(c, level);
  dim3 grid(32, beta, G);
  KTimer kt(c, FAM_MODUP, s);
  // algorithmic bytes: the l+1 limbs of c1 in, beta x (E - alpha) limbs out (the last digit may be short)
  uint64_t outs = 0;
  for (int j = 0; j < beta; ++j) outs += E - (c->h_modup[level][j].hi - c->h_modup[level][j].lo);
  kt.bytes = (uint64_t)G * (n + outs) * c->N * 8;
  const ModUpConst* mc = c->d_modup[level];
  const int nq = (int)c->n_q, lg = (int)c->log_n, lv = (int)level;
  switch (c->alpha) {
    case 1: k_bconv_cols<1, false><<<grid, 256, 0, s>>>(a, mc, nullptr, c->dt, lv, nq, E, lg); break;
    case 2: k_bconv_cols<2, false><<<grid, 256, 0, s>>>(a, mc, nullptr, c->dt, lv, nq, E, lg); break;
    case 3: k_bconv_cols<3, false><<<grid, 256, 0, s>>>(a, mc, nullptr, c->dt, lv, nq, E, lg); break;
    case 4:
      if (cols_ys_on()) launch_cols_ys<4, false>(grid, s, a, mc, nullptr, c->dt, lv, nq, E, lg);
      else k_bconv_cols<4, false><<<grid, 256, 0, s>>>(a, mc, nullptr, c->dt, lv, nq, E, lg);
      break;
    default: break;  // callers check modup_cols_ok
  }
}

void launch_moddown_cols(hy_ctx* c, const ModUpColsArgs& a, int G, uint32_t level, cudaStream_t s) {
  if (G <= 0) return;
  const int n = (int)level + 1, E = n + (int)c->n_p;
  dim3 grid(32, 2, G);
  KTimer kt(c, FAM_MODDOWN, s);
  // algorithmic bytes: the 2K P limbs in, the 2(l+1) conversion limbs out
  kt.bytes = (uint64_t)G * 2 * (c->n_p + n) * c->N * 8;
  const ModDownConst* md = c->d_moddown[level];
  const int nq = (int)c->n_q, lg = (int)c->log_n, lv = (int)level;
  switch (c->n_p) {
    case 1: k_bconv_cols<1, true><<<grid, 256, 0, s>>>(a, nullptr, md, c->dt, lv, nq, E, lg); break;
    case 2: k_bconv_cols<2, true><<<grid, 256, 0, s>>>(a, nullptr, md, c->dt, lv, nq, E, lg); break;
    case 3: k_bconv_cols<3, true><<<grid, 256, 0, s>>>(a, nullptr, md, c->dt, lv, nq, E, lg); break;
    case 4:
      if (cols_ys_on()) launch_cols_ys<4, true>(grid, s, a, nullptr, md, c->dt, lv, nq, E, lg);
      else k_bconv_cols<4, true><<<grid, 256, 0, s>>>(a, nullptr, md, c->dt, lv, nq, E, lg);
      break;
    default: break;  // callers check moddown_cols_ok
  }
}

void launch_rescale_cols(hy_ctx* c, const ModUpColsArgs& a, int G, uint32_t level, cudaStream_t s) {
  if (G <= 0) return;
  dim3 grid(32, 2, G);
  KTimer kt(c, FAM_RESCALE, s);
  // algorithmic bytes: the 2 dropped limbs in, the 2 level conversion limbs out
  kt.bytes = (uint64_t)G * 2 * (1 + level) * c->N * 8;
  // a ModDown by P = q_level: one source (chain level), targets q_0..q_{level-1}, i.e. the DOWN kernel at level-1
  k_bconv_cols<1, true><<<grid, 256, 0, s>>>(a, nullptr, c->d_rescale_md[level], c->dt, (int)level - 1,
                                              (int)c->n_q, (int)level + 1, (int)c->log_n);
}

void launch_rescale_rows_final(hy_ctx* c, const RowsFinalArgs& a, int G, uint32_t level, cudaStream_t s) {
  if (G <= 0) return;
  const int R = (int)(c->N / 256);
  dim3 grid(R / 8 > 0 ? R / 8 : 1, level, 2 * G);
  KTimer kt(c, FAM_RESCALE, s);
  // the input ciphertext's first level limbs and w in, the output written
  kt.bytes = (uint64_t)G * 2 * 3 * level * c->N * 8;
  k_ntt_rows_final<<<grid, 256, 0, s>>>(a, 2, (int)level + 1, c->d_rescale_md[level], c->dt, (int)level - 1,
                                        (int)c->log_n);
}

void launch_ntt_rows_final(hy_ctx* c, const RowsFinalArgs& a, int G, int npoly, uint32_t level, cudaStream_t s) {
  if (G <= 0) return;
  const int n = (int)level + 1, E = n + (int)c->n_p, R = (int)(c->N / 256);
  uint64_t extra = 0;
  for (int g = 0; g < G; ++g)
    extra += (a.add0[g] ? n : 0) + (a.add1[g] ? n : 0) + (a.addct[g] ? (uint64_t)npoly * n : 0);
  dim3 grid(R / 8 > 0 ? R / 8 : 1, n, npoly * G);
  KTimer kt(c, FAM_MODDOWN, s);
  // w (column-pass output) and u in, out written, plus the addends
  kt.bytes = ((uint64_t)G * npoly * n * 3 + extra) * c->N * 8;
  k_ntt_rows_final<<<grid, 256, 0, s>>>(a, npoly, E, c->d_moddown[level], c->dt, (int)level, (int)c->log_n);
}

void launch_ntt_cols(hy_ctx* c, const LimbBatch& b, cudaStream_t s) {
  if (b.n == 0) return;
  const int logN = (int)c->log_n;
  dim3 gA(256 / 16, b.n);
  KTimer kt(c, FAM_NTT_A, s);
  kt.bytes = 2ull * b.n * c->N * 8;
  if (c->N == 65536) k_ntt_cols256<true><<<gA, 512, 0, s>>>(b, c->dt, logN);
  else k_ntt_cols_small<true><<<gA, 256, 0, s>>>(b, c->dt, logN);
}

bool sum_tma_on() {
  static const bool on = getenv("HY_SUMTMA") == nullptr || atoi(getenv("HY_SUMTMA")) != 0;
  return on;
}

void launch_ntt_rows_ip(hy_ctx* c, const RowsIpArgs& a, int G, uint32_t level, bool sum, bool accumulate,
                        cudaStream_t s, int u0, bool inv_p, bool hoist, int groups) {
  if (G <= 0) return;
  const int n = (int)level + 1, E = n + (int)c->n_p, beta = (int)n_digits(c, level), R = (int)(c->N / 256);
  const int nu = E - u0;  // extended limbs produced
  int keys = 0;
  for (int g = 0; g < G; ++g) {
    bool seen = false;
    for (int h = 0; h < g; ++h) seen |= a.evk[h] == a.evk[g];
    keys += seen ? 0 : 1;
  }
  dim3 grid(sum ? 1 : G, R / 8 > 0 ? R / 8 : 1, nu);
  KTimer kt(c, FAM_NTT_IP, s);
  // HY_SUMTMA (default on): the lazy HRotSum IP (all limbs summed over the items) on the bulk-copy ring
  if (sum_tma_on() && sum && !hoist && !inv_p && u0 == 0) {
    IpFinalArgs fa{};
    for (int g = 0; g < G; ++g) {
      fa.ext[g] = a.ext[g];
      fa.own[g] = a.own[g];
      fa.evk[g] = a.evk[g];
      fa.kx[g] = a.kx[g] ? a.kx[g] : 1;
    }
    const int per = G / groups;  // items per output (grouped lazy sums)
    for (int o = 0; o < groups; ++o) fa.out[o] = a.u[o * per];
    grid.x = groups;
    const size_t smem = rows_tma_smem(2);
    const int L1s = (int)(c->n_q + c->n_p), lv = (int)level, al = (int)c->alpha, lg = (int)c->log_n;
#define HY_ST(BB)                                                                                              \
  case BB: {                                                                                                   \
    static bool at = false;                                                                                    \
    if (!at) {                                                                                                 \
      cudaFuncSetAttribute(k_rows_ip_sum_tma<BB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);     \
      at = true;                                                                                               \
    }                                                                                                          \
    k_rows_ip_sum_tma<BB><<<grid, 256, smem, s>>>(fa, per, c->dt, lv, L1s, E, al, lg, accumulate ? 1 : 0);    \
  } break;
    switch (beta) {
      HY_ST(1)
      HY_ST(2)
      HY_ST(3)
      HY_ST(4)
      HY_ST(5)
      HY_ST(6)
      HY_ST(7)
      default:
        HY_ST(8)
    }
#undef HY_ST
    return;
  }
  // HY_PTMA (default on): the split-ModDown P limbs on the bulk-copy ring of the Q-limb kernel
  static const bool ptma = getenv("HY_PTMA") == nullptr || atoi(getenv("HY_PTMA")) != 0;
  if (ptma && !sum && !accumulate && inv_p && u0 == n) {
    IpFinalArgs fa{};
    for (int g = 0; g < G; ++g) {
      fa.ext[g] = a.ext[g];
      fa.own[g] = a.own[g];
      fa.evk[g] = a.evk[g];
      fa.out[g] = a.v[g];
      fa.k0[g] = 1;
      fa.kx[g] = hoist ? a.kx[g] : 1;
    }
    const size_t smem = rows_tma_smem(2);
    const int L1p = (int)(c->n_q + c->n_p), lv = (int)level, al = (int)c->alpha, lg = (int)c->log_n;
    kt.bytes = ((uint64_t)(hoist ? 1 : G) * beta * nu * 8 + (uint64_t)keys * 2 * beta * nu * 6 +
                (uint64_t)G * 2 * nu * 8) * c->N;
#define HY_PT(BB)                                                                                              \
  case BB:                                                                                                     \
    if (hoist) {                                                                                               \
      static bool at = false;                                                                                  \
      if (!at) {                                                                                               \
        cudaFuncSetAttribute(k_rows_ip_p_tma<BB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        at = true;                                                                                             \
      }                                                                                                        \
      k_rows_ip_p_tma<BB, true><<<grid, 256, smem, s>>>(fa, c->dt, lv, L1p, E, al, lg);                        \
    } else {                                                                                                   \
      static bool at = false;                                                                                  \
      if (!at) {                                                                                               \
        cudaFuncSetAttribute(k_rows_ip_p_tma<BB, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,           \
                             (int)smem);                                                                       \
        at = true;                                                                                             \
      }                                                                                                        \
      k_rows_ip_p_tma<BB, false><<<grid, 256, smem, s>>>(fa, c->dt, lv, L1p, E, al, lg);                       \
    }                                                                                                          \
    break;
    switch (beta) {
      HY_PT(1)
      HY_PT(2)
      HY_PT(3)
      HY_PT(4)
      HY_PT(5)
      HY_PT(6)
      HY_PT(7)
      default:
        HY_PT(8)
    }
#undef HY_PT
    return;
  }
  // algorithmic bytes: every digit limb in once, each distinct key once, the outputs (read back too
  // when accumulating)
  const uint64_t outs = sum ? 1 : G;
  kt.bytes = ((uint64_t)G * beta * nu * 8 + (uint64_t)keys * 2 * beta * nu * 6 + outs * 2 * nu * (accumulate ? 2 : 1) * 8) *
             c->N;  // key words packed in 6 bytes
  const int L1 = (int)(c->n_q + c->n_p);
#define HY_RIP(BB)                                                                                             \
  case BB:                                                                                                     \
    if (sum)                                                                                                   \
      k_ntt_rows_ip<BB, true, false><<<grid, 256, 0, s>>>(a, G, c->dt, (int)level, (int)c->n_q, L1, E,         \
                                                          (int)c->alpha, (int)c->log_n, accumulate ? 1 : 0, u0, \
                                                          inv_p);                                              \
    else if (hoist)                                                                                            \
      k_ntt_rows_ip<BB, false, true><<<grid, 256, 0, s>>>(a, G, c->dt, (int)level, (int)c->n_q, L1, E,         \
                                                          (int)c->alpha, (int)c->log_n, accumulate ? 1 : 0, u0, \
                                                          inv_p);                                              \
    else                                                                                                       \
      k_ntt_rows_ip<BB, false, false><<<grid, 256, 0, s>>>(a, G, c->dt, (int)level, (int)c->n_q, L1, E,        \
                                                           (int)c->alpha, (int)c->log_n, accumulate ? 1 : 0,    \
                                                           u0, inv_p);                                         \
    break;
  switch (beta) {
    HY_RIP(1)
    HY_RIP(2)
    HY_RIP(3)
    HY_RIP(4)
    HY_RIP(5)
    HY_RIP(6)
    HY_RIP(7)
    default:
      HY_RIP(8)
  }
#undef HY_RIP
}

void launch_rows_ip_final(hy_ctx* c, const IpFinalArgs& a, int G, uint32_t level, bool hoisted, cudaStream_t s) {
  if (G <= 0) return;
  const int n = (int)level + 1, E = n + (int)c->n_p, beta = (int)n_digits(c, level), R = (int)(c->N / 256);
  int keys = 0;
  for (int g = 0; g < G; ++g) {
    bool seen = false;
    for (int h = 0; h < g; ++h) seen |= a.evk[h] == a.evk[g];
    keys += seen ? 0 : 1;
  }
  uint64_t extra = 0;
  for (int g = 0; g < G; ++g) extra += (a.add0[g] ? n : 0) + (a.add1[g] ? n : 0) + (a.addct[g] ? 2 * n : 0);
  dim3 grid(G, R / 8 > 0 ? R / 8 : 1, n);
  KTimer kt(c, FAM_NTT_IP, s);
  // algorithmic bytes: the digits' Q limbs in (hoisted: shared, once), each distinct key's Q rows once,
  // the conversion w in, the output written, the addends
  const uint64_t digits = (hoisted ? 1 : (uint64_t)G) * beta * n;
  kt.bytes = ((digits + (uint64_t)G * 4 * n + extra) * 8 + (uint64_t)keys * 2 * beta * n * 6) * c->N;  // packed key
  const int L1 = (int)(c->n_q + c->n_p), lv = (int)level, al = (int)c->alpha, lg = (int)c->log_n;
  const ModDownConst* md = c->d_moddown[level];
  // HY_TMA=0: register loads instead of the bulk-copy staged rows (A/B; staged: +0.2 % plain, +3 % hoisted)
  static const bool use_tma = getenv("HY_TMA") == nullptr || atoi(getenv("HY_TMA")) != 0;
  // HY_TMA_STAGES: depth of the per-warp bulk-copy ring (2: two CTAs per SM; 3 or 4: one CTA per SM)
  static const int nst = getenv("HY_TMA_STAGES") ? atoi(getenv("HY_TMA_STAGES")) : 2;
#define HY_TMA_LAUNCH(BB, HH, NS)                                                                             \
  {                                                                                                           \
    static bool attr = false;                                                                                 \
    if (!attr) {                                                                                              \
      cudaFuncSetAttribute(k_rows_ip_final_tma<BB, HH, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize,      \
                           (int)rows_tma_smem(NS));                                                           \
      attr = true;                                                                                            \
    }                                                                                                         \
    k_rows_ip_final_tma<BB, HH, NS><<<grid, 256, rows_tma_smem(NS), s>>>(a, c->dt, md, lv, L1, E, al, lg);    \
  }
#define HY_TMA_NST(BB, HH)                   \
  if (nst <= 2) HY_TMA_LAUNCH(BB, HH, 2)     \
  else if (nst == 3) HY_TMA_LAUNCH(BB, HH, 3) \
  else HY_TMA_LAUNCH(BB, HH, 4)
#define HY_RIF(BB)                                                                                            \
  case BB:                                                                                                    \
    if (use_tma) {                                                                                            \
      if (hoisted) HY_TMA_NST(BB, true)                                                                       \
      else HY_TMA_NST(BB, false)                                                                              \
    } else if (hoisted) {                                                                                     \
      k_rows_ip_final<BB, true><<<grid, 256, 0, s>>>(a, c->dt, md, lv, L1, E, al, lg);                        \
    } else {                                                                                                  \
      k_rows_ip_final<BB, false><<<grid, 256, 0, s>>>(a, c->dt, md, lv, L1, E, al, lg);                       \
    }                                                                                                         \
    break;
  switch (beta) {
    HY_RIF(1)
    HY_RIF(2)
    HY_RIF(3)
    HY_RIF(4)
    HY_RIF(5)
    HY_RIF(6)
    HY_RIF(7)
    default:
      HY_RIF(8)
  }
#undef HY_RIF
#undef HY_TMA_NST
#undef HY_TMA_LAUNCH
}

void launch_ntt(hy_ctx* c, const LimbBatch& b, bool inverse, cudaStream_t s) {
  if (b.n == 0) return;
  const int logN = (int)c->log_n;
  const int R = (int)c->N / 256;
  dim3 gB(R / 8 > 0 ? R / 8 : 1, b.n), gA(256 / 16, b.n);
  const uint64_t pass_bytes = 2ull * b.n * c->N * 8;  // read + write every limb once
  if (!inverse) {
    {
      KTimer kt(c, FAM_NTT_A, s);
      kt.bytes = pass_bytes;
      if (R == 256) k_ntt_cols256<true><<<gA, 512, 0, s>>>(b, c->dt, logN);
      else k_ntt_cols_small<true><<<gA, 256, 0, s>>>(b, c->dt, logN);
    }
    // pass B runs in place on dst
    LimbBatch b2 = b;
    for (int i = 0; i < b.n; ++i) b2.src[i] = b.dst[i];
    KTimer kt(c, FAM_NTT_B, s);
    kt.bytes = pass_bytes;
    k_ntt_rows<true><<<gB, 256, 0, s>>>(b2, c->dt, logN);
  } else {
    {
      KTimer kt(c, FAM_NTT_B, s);
      kt.bytes = pass_bytes;
      k_ntt_rows<false><<<gB, 256, 0, s>>>(b, c->dt, logN);
    }
    KTimer kt(c, FAM_NTT_A, s);
    kt.bytes = pass_bytes;
    if (R == 256) k_ntt_cols256<false><<<gA, 512, 0, s>>>(b, c->dt, logN);
    else k_ntt_cols_small<false><<<gA, 256, 0, s>>>(b, c->dt, logN);
  }
}

namespace {
enum class Pass { Both, Rows, Cols };
void run_list(hy_ctx* c, const LimbList& L, bool inverse, Pass pass, cudaStream_t s) {
  LimbBatch b;
  for (size_t done = 0; done < L.src.size();) {
    const size_t m = std::min<size_t>(L.src.size() - done, kMaxBatch);
    b.n = (int)m;
    for (size_t i = 0; i < m; ++i) {
      b.src[i] = L.src[done + i];
      b.dst[i] = L.dst[done + i];
      b.chain[i] = L.chain[done + i];
    }
    if (pass == Pass::Both) launch_ntt(c, b, inverse, s);
    else if (pass == Pass::Rows) launch_ntt_rows(c, b, inverse, s);
    else launch_ntt_cols(c, b, s);
    done += m;
  }
}
}  // namespace

void ntt_list(hy_ctx* c, const LimbList& L, bool inverse, cudaStream_t s) { run_list(c, L, inverse, Pass::Both, s); }
void rows_list(hy_ctx* c, const LimbList& L, bool inverse, cudaStream_t s) { run_list(c, L, inverse, Pass::Rows, s); }
void ntt_cols_list(hy_ctx* c, const LimbList& L, cudaStream_t s) { run_list(c, L, false, Pass::Cols, s); }

void ntt_contig(hy_ctx* c, const uint64_t* in, uint64_t* out, const uint32_t* chain, uint32_t n, bool inverse,
                cudaStream_t s) {
  LimbBatch b;
  for (uint32_t done = 0; done < n;) {
    uint32_t m = std::min<uint32_t>(n - done, kMaxBatch);
    b.n = (int)m;
    for (uint32_t i = 0; i < m; ++i) {
      b.src[i] = in + (size_t)(done + i) * c->N;
      b.dst[i] = out + (size_t)(done + i) * c->N;
      b.chain[i] = (uint8_t)chain[done + i];
    }
    launch_ntt(c, b, inverse, s);
    done += m;
  }
}

}  // namespace hy

extern "C" hy_status hy_ntt(hy_ctx* c, const uint64_t* d_in, uint64_t* d_out, const uint32_t* chain,
                            uint32_t n_limbs, int inverse, void* stream) {
  if (!c || !d_in || !d_out || !chain) return hy::fail(HY_E_ARG, "null argument");
  for (uint32_t i = 0; i < n_limbs; ++i)
    if (chain[i] >= c->n_q + c->n_p) return hy::fail(HY_E_ARG, "chain index out of range");
  hy::ntt_contig(c, d_in, d_out, chain, n_limbs, inverse != 0, hy::st(stream));
  return hy::cuda_check("hy_ntt");
}
