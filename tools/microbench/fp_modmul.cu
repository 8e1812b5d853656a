// FP64-pipe vs integer-pipe 64-bit modular multiplication by a constant (NTT twiddle
// pattern) on sm_100a.  Primes < 2^50.  Validates results against __int128 on a sample.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int CH = 8;
__device__ __forceinline__ double u2d(uint64_t v) { return __longlong_as_double((long long)(v | 0x4330000000000000ull)) - 4503599627370496.0; }
__device__ __forceinline__ uint64_t d2u(double d) { return (uint64_t)__double_as_longlong(d + 4503599627370496.0) & 0xFFFFFFFFFFFFFull; }
// r = x*w mod q, x in [0, 2q), result in [0, q): Harvey-style double-precision product
__device__ __forceinline__ double fmul_mod(double x, double w, double wq, double q) {
  const double M = 6755399441055744.0;  // 1.5 * 2^52: rint by addition
  double h = x * w;
  double l = fma(x, w, -h);
  double c = fma(x, wq, M) - M;
  double d = fma(-c, q, h);
  double r = d + l;
  r = r < 0 ? r + q : r;
  r = r >= q ? r - q : r;
  return r;
}
__global__ void k_fp(uint64_t* out, int iters, double w, double wq, double q) {
  double x[CH];
  for (int c = 0; c < CH; ++c) x[c] = (double)(threadIdx.x * 977 + c * 7777);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fmul_mod(x[c], w, wq, q);
  }
  uint64_t s = 0;
  for (int c = 0; c < CH; ++c) s ^= d2u(x[c]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__device__ __forceinline__ uint64_t shoup(uint64_t x, uint64_t w, uint64_t wp, uint64_t q) {
  uint64_t r = x * w - __umul64hi(x, wp) * q;
  return r >= q ? r - q : r;
}
__global__ void k_int(uint64_t* out, int iters, uint64_t w, uint64_t wp, uint64_t q) {
  uint64_t x[CH];
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 977 + c * 7777;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = shoup(x[c], w, wp, q);
  }
  uint64_t s = 0;
  for (int c = 0; c < CH; ++c) s ^= x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// conversion round trips through the bit trick
__global__ void k_conv(uint64_t* out, int iters, uint64_t q) {
  uint64_t x[CH];
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 977 + c * 7777;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = d2u(u2d(x[c]) + 1.0);
  }
  uint64_t s = 0;
  for (int c = 0; c < CH; ++c) s ^= x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_check(uint64_t* bad, uint64_t w, double wq, uint64_t q, uint64_t seed) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t x = (i * 0x9E3779B97F4A7C15ull + seed) % (2 * q);
  double r = fmul_mod(u2d(x), u2d(w), wq, (double)q);
  uint64_t want = (uint64_t)((unsigned __int128)x * w % q);
  if (d2u(r) != want) atomicAdd((unsigned long long*)bad, 1ull);
}
int main() {
  const uint64_t q = 1125899906826241ull;  // a prime < 2^50 with q = 1 mod 2^17 (value irrelevant for rate)
  const uint64_t w = 987654321012345ull % q;
  const uint64_t wp = (uint64_t)(((unsigned __int128)w << 64) / q);
  const double wq = (double)w / (double)q;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int T = 256, B = sms * 8, it = 4096;
  uint64_t* out; cudaMalloc(&out, (size_t)T * B * 8);
  uint64_t* bad; cudaMalloc(&bad, 8); cudaMemset(bad, 0, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  double tot = (double)T * B * it * CH;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); k_fp<<<B, T>>>(out, it, (double)w, wq, (double)q); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); if (rep) printf("{\"kernel\":\"fp64_modmul\",\"T_per_s\":%.3f}\n", tot / ms / 1e9);
    cudaEventRecord(e0); k_int<<<B, T>>>(out, it, w, wp, q); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); if (rep) printf("{\"kernel\":\"int_shoup_modmul\",\"T_per_s\":%.3f}\n", tot / ms / 1e9);
    cudaEventRecord(e0); k_conv<<<B, T>>>(out, it, q); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); if (rep) printf("{\"kernel\":\"u64_f64_roundtrip\",\"T_per_s\":%.3f}\n", tot / ms / 1e9);
  }
  for (int s = 0; s < 16; ++s) k_check<<<4096, 256>>>(bad, w, wq, q, s * 12345);
  uint64_t nb; cudaMemcpy(&nb, bad, 8, cudaMemcpyDeviceToHost);
  printf("{\"check\":\"fp64_modmul vs int128\",\"samples\":%d,\"mismatches\":%llu}\n", 16 * 4096 * 256, (unsigned long long)nb);
  return 0;
}
