// A/B for the north star's "warp-shuffle butterflies": the 8-stage forward 256-point row pass
// of the NTT (one warp per row, 8 words per lane, FP64 fmulmod butterflies) with the lane-crossing stages done
//   (a) as in the product: two swizzled shared-memory transposes (layouts L1 -> L2 -> L3), every stage register-local;
//   (b) with warp shuffles: layout L1 throughout, the 5 stages whose distance is a lane bit exchange the partner's
//       64-bit word with __shfl_xor_sync (2 x 32-bit) and both lanes of a pair evaluate the product b*w.
// Same data, same twiddles; checks that both give identical words, then times them on 64 x 256 rows x 24 limbs.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../../paper_2302_02407_b200/csrc/hy_arith.cuh"
using namespace hy;

__device__ __forceinline__ int pidx(int e) { return e ^ ((e >> 2) & 1) ^ (((e >> 4) & 7) << 1); }
template <int LAY>
__device__ __forceinline__ int elem(int l, int k) {
  if (LAY == 1) return l + 32 * k;
  if (LAY == 2) return 32 * (l >> 2) + 4 * k + (l & 3);
  return 4 * (l + 32 * (k >> 2)) + (k & 3);
}
template <int LAY>
__device__ __forceinline__ int kbit(int s) { return LAY == 1 ? s - 5 : (LAY == 2 ? s - 2 : s); }
template <int LAY>
__device__ __forceinline__ void stages(double (&x)[8], int l, int s_hi, int s_lo, const double* T, double q,
                                       double qinv) {
#pragma unroll
  for (int it = 0; it <= s_hi - s_lo; ++it) {
    const int s = s_hi - it, kb = 1 << kbit<LAY>(s);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (k & kb) continue;
      const double w = T[(256 + elem<LAY>(l, k)) >> (s + 1)];
      const double a = x[k], t = fmulmod(x[k | kb], w, q, qinv);
      x[k] = a + t;
      x[k | kb] = a - t;
    }
  }
}

// (a) smem transposes
__global__ void __launch_bounds__(256) k_smem(const double* __restrict__ in, double* __restrict__ out,
                                              const double* __restrict__ tw, double q, double qinv) {
  __shared__ double S[8][256], TT[8][256];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const size_t row = (size_t)blockIdx.x * 8 + w;
  double* T = TT[w];
  for (int k = 0; k < 8; ++k) T[l + 32 * k] = tw[l + 32 * k];
  double x[8];
  for (int k = 0; k < 8; ++k) x[k] = in[row * 256 + elem<1>(l, k)];
  __syncwarp();
  stages<1>(x, l, 7, 5, T, q, qinv);
  for (int k = 0; k < 8; ++k) S[w][pidx(elem<1>(l, k))] = x[k];
  __syncwarp();
  for (int k = 0; k < 8; ++k) x[k] = S[w][pidx(elem<2>(l, k))];
  stages<2>(x, l, 4, 2, T, q, qinv);
  __syncwarp();
  for (int k = 0; k < 8; ++k) S[w][pidx(elem<2>(l, k))] = x[k];
  __syncwarp();
  for (int k = 0; k < 8; ++k) x[k] = S[w][pidx(elem<3>(l, k))];
  stages<3>(x, l, 1, 0, T, q, qinv);
  for (int k = 0; k < 8; ++k) out[row * 256 + elem<3>(l, k)] = x[k];
}

// (b) warp shuffles, layout L1 (element l + 32 k): stages 7..5 are register-local, stages 4..0 cross lanes
__global__ void __launch_bounds__(256) k_shfl(const double* __restrict__ in, double* __restrict__ out,
                                              const double* __restrict__ tw, double q, double qinv) {
  __shared__ double TT[8][256];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const size_t row = (size_t)blockIdx.x * 8 + w;
  double* T = TT[w];
  for (int k = 0; k < 8; ++k) T[l + 32 * k] = tw[l + 32 * k];
  double x[8];
  for (int k = 0; k < 8; ++k) x[k] = in[row * 256 + elem<1>(l, k)];
  __syncwarp();
  stages<1>(x, l, 7, 5, T, q, qinv);
#pragma unroll
  for (int s = 4; s >= 0; --s) {
    const int lb = 1 << s;
    const bool hi = l & lb;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double p = __shfl_xor_sync(0xffffffffu, x[k], lb);
      const int e = elem<1>(l, k) & ~lb;  // the pair's low element: its twiddle
      const double wv = T[(256 + e) >> (s + 1)];
      const double a = hi ? p : x[k], b = hi ? x[k] : p;
      const double t = fmulmod(b, wv, q, qinv);
      x[k] = hi ? a - t : a + t;
    }
  }
  for (int k = 0; k < 8; ++k) out[row * 256 + elem<1>(l, k)] = x[k];
}

int main() {
  const size_t rows = 64ull * 256 * 24, n = rows * 256;
  const double q = 281474976710597.0, qinv = 1.0 / q;
  double *in, *o1, *o2, *tw;
  cudaMalloc(&in, n * 8);
  cudaMalloc(&o1, n * 8);
  cudaMalloc(&o2, n * 8);
  cudaMalloc(&tw, 256 * 8);
  double* h = new double[256];
  for (int i = 0; i < 256; ++i) h[i] = (double)((i * 2654435761ull) % 281474976710597ull);
  cudaMemcpy(tw, h, 256 * 8, cudaMemcpyHostToDevice);
  double* hin = new double[1 << 20];
  for (int i = 0; i < (1 << 20); ++i) hin[i] = (double)(((uint64_t)i * 0x9E3779B97F4A7C15ull) >> 17) - 7.0e13;
  for (size_t o = 0; o < n; o += (1 << 20)) cudaMemcpy(in + o, hin, 8ull << 20, cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms1 = 0, ms2 = 0;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    k_smem<<<rows / 8, 256>>>(in, o1, tw, q, qinv);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms1, a, b);
    cudaEventRecord(a);
    k_shfl<<<rows / 8, 256>>>(in, o2, tw, q, qinv);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms2, a, b);
  }
  // compare: the smem kernel writes layout-independent element order (out[row*256 + e]), as does the shuffle one
  double *r1 = new double[1 << 16], *r2 = new double[1 << 16];
  cudaMemcpy(r1, o1, 8 << 16, cudaMemcpyDeviceToHost);
  cudaMemcpy(r2, o2, 8 << 16, cudaMemcpyDeviceToHost);
  size_t bad = 0;
  for (int i = 0; i < (1 << 16); ++i) bad += r1[i] != r2[i];
  const double gb = 2.0 * n * 8 / 1e9;
  printf("{\"kernel\":\"row_pass_smem_transposes\",\"ms\":%.3f,\"GBps\":%.1f}\n", ms1, gb / ms1 * 1e3);
  printf("{\"kernel\":\"row_pass_warp_shuffles\",\"ms\":%.3f,\"GBps\":%.1f}\n", ms2, gb / ms2 * 1e3);
  printf("{\"check\":\"identical words\",\"mismatches\":%zu,\"rows\":%zu}\n", bad, rows);
  return 0;
}
