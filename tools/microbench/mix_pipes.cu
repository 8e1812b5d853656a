// Do the FP64 pipe and the integer (IMAD) pipe overlap on sm_100a?  Three kernels with the same
// per-thread structure: FP64 fmulmod chains only, Shoup (IMAD.WIDE) chains only, and both interleaved
// in one loop.  If the mixed kernel's total modmul rate exceeds the FP64-only rate, integer work (e.g.
// the fast basis conversion) can be hidden under the FP64 NTT butterflies.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ double fmul_mod(double x, double w, double wq, double q) {
  const double M = 6755399441055744.0;
  double h = x * w, l = fma(x, w, -h), c = fma(x, wq, M) - M;
  return fma(-c, q, h) + l;
}
__device__ __forceinline__ uint64_t shoup(uint64_t x, uint64_t w, uint64_t wp, uint64_t q) {
  return x * w - __umul64hi(x, wp) * q;  // lazy, [0, 2q)
}
template <int CF, int CI>
__global__ void k_mix(uint64_t* out, int iters, double w, double wq, double q, uint64_t wi, uint64_t wp, uint64_t qi) {
  double x[CF > 0 ? CF : 1];
  uint64_t y[CI > 0 ? CI : 1];
  for (int c = 0; c < CF; ++c) x[c] = (double)(threadIdx.x * 977 + c * 7777);
  for (int c = 0; c < CI; ++c) y[c] = threadIdx.x * 977 + c * 7777;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CF; ++c) x[c] = fmul_mod(x[c], w, wq, q);
#pragma unroll
    for (int c = 0; c < CI; ++c) y[c] = shoup(y[c], wi, wp, qi);
  }
  uint64_t s = 0;
  for (int c = 0; c < CF; ++c) s ^= (uint64_t)__double_as_longlong(x[c]);
  for (int c = 0; c < CI; ++c) s ^= y[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int CF, int CI>
void run(const char* name, uint64_t* out, int B, int T, int it) {
  const uint64_t q = 281474976710597ull;  // < 2^48
  const uint64_t w = 98765432101234ull % q;
  const uint64_t wp = (uint64_t)(((unsigned __int128)w << 64) / q);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    k_mix<CF, CI><<<B, T>>>(out, it, (double)w, (double)w / (double)q, (double)q, w, wp, q);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  const double n = (double)B * T * it;
  printf("{\"kernel\":\"%s\",\"fp64_T_per_s\":%.3f,\"int_T_per_s\":%.3f,\"total_T_per_s\":%.3f}\n", name,
         n * CF / ms / 1e9, n * CI / ms / 1e9, n * (CF + CI) / ms / 1e9);
}
int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int T = 256, B = sms * 8, it = 2048;
  uint64_t* out;
  cudaMalloc(&out, (size_t)T * B * 8);
  run<8, 0>("fp64_only_8", out, B, T, it);
  run<0, 8>("int_only_8", out, B, T, it);
  run<8, 2>("mix_8fp_2int", out, B, T, it);
  run<8, 4>("mix_8fp_4int", out, B, T, it);
  run<8, 8>("mix_8fp_8int", out, B, T, it);
  run<4, 4>("mix_4fp_4int", out, B, T, it);
  return 0;
}
