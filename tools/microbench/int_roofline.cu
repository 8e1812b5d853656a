// Integer-pipe roofline microbenchmark for sm_100a.
// Measures: 32-bit IMAD rate, 64-bit Shoup modmul rate, 64-bit Montgomery
// modmul rate, FP64 FMA rate, and prints device properties.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int CHAINS = 8;

__global__ void k_imad(uint32_t* out, int iters, uint32_t a) {
  uint32_t x[CHAINS];
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = x[c] * a + c;  // IMAD
  }
  uint32_t s = 0;
  for (int c = 0; c < CHAINS; ++c) s ^= x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ uint64_t shoup_mul(uint64_t x, uint64_t w, uint64_t wp, uint64_t q) {
  uint64_t hi = __umul64hi(x, wp);
  uint64_t r = x * w - hi * q;
  return r;  // in [0, 2q)
}

__global__ void k_shoup(uint64_t* out, int iters, uint64_t w, uint64_t wp, uint64_t q) {
  uint64_t x[CHAINS];
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x + c * 7777;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = shoup_mul(x[c], w, wp, q);
  }
  uint64_t s = 0;
  for (int c = 0; c < CHAINS; ++c) s ^= x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ uint64_t mont_mul(uint64_t a, uint64_t b, uint64_t q, uint64_t qinv_neg) {
  uint64_t lo = a * b, hi = __umul64hi(a, b);
  uint64_t m = lo * qinv_neg;
  uint64_t mh = __umul64hi(m, q);
  // (a*b + m*q)/2^64 = hi + mh + carry(lo + m*q_lo != 0)
  uint64_t r = hi + mh + (lo != 0);
  return r;  // < 2q
}

__global__ void k_mont(uint64_t* out, int iters, uint64_t b, uint64_t q, uint64_t qn) {
  uint64_t x[CHAINS];
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x + c * 7777;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = mont_mul(x[c], b, q, qn);
  }
  uint64_t s = 0;
  for (int c = 0; c < CHAINS; ++c) s ^= x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dfma(double* out, int iters, double a) {
  double x[CHAINS];
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, 0.5);
  }
  double s = 0;
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_copy(const ulonglong2* __restrict__ a, ulonglong2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) b[i] = a[i];
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"name\":\"%s\",\"sms\":%d,\"smem_per_sm\":%zu,\"smem_optin\":%zu,\"l2\":%d,\"regs_per_sm\":%d,\"clock_khz\":%d,\"cc\":\"%d.%d\",\"mem_gb\":%.1f}\n",
         p.name, p.multiProcessorCount, p.sharedMemPerMultiprocessor, p.sharedMemPerBlockOptin, p.l2CacheSize,
         p.regsPerMultiprocessor, clk, p.major, p.minor, p.totalGlobalMem / 1e9);
  const int sms = p.multiProcessorCount;
  const int threads = 256, blocks = sms * 8;
  const int iters = 4096;
  void* out; CK(cudaMalloc(&out, (size_t)threads * blocks * 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  const uint64_t q = 0x0FFFFFFFFFE00001ULL;  // placeholder odd 60-bit modulus (rate test only)
  const uint64_t w = 123456789012345ULL % q;
  const uint64_t wp = (uint64_t)(((unsigned __int128)w << 64) / q);
  uint64_t qinv = 1; for (int i = 0; i < 6; ++i) qinv *= 2 - q * qinv;  // q^-1 mod 2^64
  const uint64_t qn = (uint64_t)0 - qinv;
  for (int rep = 0; rep < 2; ++rep) {
    double tot = (double)threads * blocks * iters * CHAINS;
    cudaEventRecord(e0); k_imad<<<blocks, threads>>>((uint32_t*)out, iters, 12345u); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    if (rep) printf("{\"kernel\":\"imad32\",\"ms\":%.3f,\"Tops\":%.3f}\n", ms, tot / ms / 1e9);
    cudaEventRecord(e0); k_shoup<<<blocks, threads>>>((uint64_t*)out, iters, w, wp, q); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    if (rep) printf("{\"kernel\":\"shoup64\",\"ms\":%.3f,\"Tmodmul_per_s\":%.3f}\n", ms, tot / ms / 1e9);
    cudaEventRecord(e0); k_mont<<<blocks, threads>>>((uint64_t*)out, iters, w, q, qn); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    if (rep) printf("{\"kernel\":\"mont64\",\"ms\":%.3f,\"Tmodmul_per_s\":%.3f}\n", ms, tot / ms / 1e9);
    cudaEventRecord(e0); k_dfma<<<blocks, threads>>>((double*)out, iters, 0.999); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    if (rep) printf("{\"kernel\":\"dfma\",\"ms\":%.3f,\"Tflop_fma_per_s\":%.3f}\n", ms, tot / ms / 1e9);
  }
  size_t bytes = (size_t)1 << 31;
  void *a, *b; CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes));
  cudaMemset(a, 1, bytes);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0); k_copy<<<sms * 16, 512>>>((ulonglong2*)a, (ulonglong2*)b, bytes / 16); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    if (rep == 2) printf("{\"kernel\":\"copy\",\"ms\":%.3f,\"GBps\":%.1f}\n", ms, 2.0 * bytes / ms / 1e6);
  }
  return 0;
}
