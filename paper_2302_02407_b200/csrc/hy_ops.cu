// hy_ops.cu -- MulPt / MulFilter&Sum / AddCt / Rescale and the
// client-side key generation, encryption and decryption (
// DESIGN R-SK, R-EVK, R-ENC, R-PRNG), all as device kernels.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "hy_arith.cuh"
#include "hy_rand.cuh"

namespace hy {
void launch_automorph(hy_ctx* c, const uint64_t* in, uint64_t* out, uint32_t n_limbs, uint64_t k, cudaStream_t s);

namespace {
constexpr int kT = 256;
constexpr int kMaxTerms = 64;

constexpr int kPbJ = 128, kPbM = 8;  // up to 128 operands per launch: a 3x3 block of 8 inputs (72) in one
struct PBlock {
  const uint64_t* ct[kPbJ];
  uint64_t* out[kPbM];
  const uint64_t* pt_base;        // stored weight plaintexts [..][l+1][N]
  uint32_t pt_idx[kPbM][kPbJ];    // plaintext index of term (m, j)
  uint32_t prot[kPbM][kPbJ];      // Galois element of its PRot (1 = none)
};

struct TermPtrs {
  const uint64_t* ct[kMaxTerms];
  const uint64_t* pt[kMaxTerms];
  uint64_t prot[kMaxTerms];  // Galois element of a PRot applied to pt (1 = none), fused as a gather
};

// Blocked MulFilter&Sum: M outputs x J ciphertext operands, dense,
//   out_m[p][i][x] (+)= sum_j ct_j[p][i][x] * PRot_{k_mj}(pt_{mj})[i][x]
// Each thread owns (x, limb i) for both polys and all M outputs: ct_j is read once per block of M outputs
// (instead of once per term) and each gathered weight word serves both polys.  Products on the FP64 pipe
// (fmulmod, |r| <= 1.5 q for canonical operands), summed exactly in a double and re-centred with fred
// every 4 operands (|acc| < 6.5 q), canonicalised once per output word.  grid (N/256, l+1)
// KM (round 2): how the PRot Galois elements of a block vary -- 0: per term; 1: per operand only (CAConv PRCR: the
// shift r_t + im F depends on the input member, not the output), the gather index computed once per operand for
// all M terms; 2: per output only (RAConv PRCR: im F - r_t depends on the output member), the M gather indices
// computed once per launch.  Products are re-centred every 8 operands (8 x 0.57 q + q/2 < 2^51: exact).
template <int M, int KM>
__global__ void __launch_bounds__(256) k_pmult_block(const __grid_constant__ PBlock b, int J, DevTables dt, int level,
                                                     int logN, int accumulate) {
  const size_t N = (size_t)1 << logN;
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  const size_t n = level + 1;
  const PrimeConst& pc = dt.pc[i];
  const double q = pc.qd, qinv = pc.qinv;
  double acc[M][2];
#pragma unroll
  for (int m = 0; m < M; ++m) acc[m][0] = acc[m][1] = 0.0;
  uint32_t xm[KM == 2 ? M : 1];
  if constexpr (KM == 2) {
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const uint32_t k = b.prot[m][0];
      xm[m] = (uint32_t)i * (uint32_t)N + (k != 1 ? aut_index(x, k, logN) : x);
    }
  }
  const uint64_t* ct_lo = nullptr;
  // unrolled by 2 so that the loads of two operands are in flight together (r02r A/B on the ResNet-18 PRCR layers:
  // unroll 1 / 2 / 4 / 8 -> L1_ra MulFilter&Sum 3.03 / 2.91 / 3.14 / 3.61 ms, L1_ca 5.02 / 5.02 / 5.12 / 5.14 ms)
#pragma unroll 2
  for (int j = 0; j < J; ++j) {
    ct_lo = b.ct[j] + (size_t)i * N + x;
    const double c0 = u2d(__ldcs(ct_lo)), c1 = u2d(__ldcs(ct_lo + n * N));
    uint32_t xj = 0;
    if constexpr (KM == 1) {
      const uint32_t k = b.prot[0][j];
      xj = (uint32_t)i * (uint32_t)N + (k != 1 ? aut_index(x, k, logN) : x);
    }
#pragma unroll
    for (int m = 0; m < M; ++m) {
      uint32_t off;
      if constexpr (KM == 0) {
        const uint32_t k = b.prot[m][j];
        off = (uint32_t)i * (uint32_t)N + (k != 1 ? aut_index(x, k, logN) : x);
      } else if constexpr (KM == 1) {
        off = xj;
      } else {
        off = xm[m];
      }
      const double w = u2d(b.pt_base[(size_t)b.pt_idx[m][j] * n * N + off]);
      acc[m][0] += fmulmod(c0, w, q, qinv);
      acc[m][1] += fmulmod(c1, w, q, qinv);
    }
    if ((j & 7) == 7) {
#pragma unroll
      for (int m = 0; m < M; ++m) {
        acc[m][0] = fred(acc[m][0], q, qinv);
        acc[m][1] = fred(acc[m][1], q, qinv);
      }
    }
  }
#pragma unroll
  for (int m = 0; m < M; ++m)
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      uint64_t* o = b.out[m] + ((size_t)p * n + i) * N + x;
      double v = acc[m][p];
      if (accumulate) v += u2d(*o);
      *o = d2u(fcanon(v, q, qinv));
    }
}

// The same block with the PRot gathers staged through shared memory (PRCR reuses one stored weight
// plaintext per family through PRot).  In the NTT domain the Galois permutation maps every 256-word row onto ONE
// source row (its high index bits depend only on the row, hy_arith.cuh aut_index), so a CTA = one row x of limb i
// loads, per operand j, the M source rows of its terms with coalesced 2 KB reads (instead of M scattered 8-byte
// gathers per thread, one 32-byte sector each) into a double-buffered shared tile, then gathers from shared memory.
// The next operand's ciphertext words and weight rows are loaded into registers while the current one is
// multiplied.  grid (N/256, l+1), CTA = 256 threads (one row).
template <int M>
__global__ void __launch_bounds__(256) k_pmult_rows(const __grid_constant__ PBlock b, int J, DevTables dt, int level,
                                                    int logN, int accumulate) {
  __shared__ double W[2][M][256];
  const size_t N = (size_t)1 << logN;
  const int t = threadIdx.x;
  const uint32_t r = blockIdx.x, x = r * 256 + t;
  const int i = blockIdx.y;
  const size_t n = level + 1;
  const PrimeConst& pc = dt.pc[i];
  const double q = pc.qd, qinv = pc.qinv;
  double acc[M][2];
#pragma unroll
  for (int m = 0; m < M; ++m) acc[m][0] = acc[m][1] = 0.0;
  uint64_t pw[M], p0, p1;
  auto load = [&](int j) {
    p0 = __ldcs(b.ct[j] + (size_t)i * N + x);
    p1 = __ldcs(b.ct[j] + (n + i) * N + x);
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const uint32_t k = b.prot[m][j];
      const uint32_t sr = k != 1 ? aut_index(r * 256u, k, logN) >> 8 : r;
      pw[m] = b.pt_base[((size_t)b.pt_idx[m][j] * n + i) * N + (size_t)sr * 256 + t];
    }
  };
  load(0);
#pragma unroll
  for (int m = 0; m < M; ++m) W[0][m][t] = u2d(pw[m]);
  double c0 = u2d(p0), c1 = u2d(p1);
  __syncthreads();
  for (int j = 0; j < J; ++j) {
    const int buf = j & 1;
    if (j + 1 < J) load(j + 1);
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const uint32_t k = b.prot[m][j];
      const uint32_t pos = k != 1 ? aut_index(x, k, logN) & 255u : (uint32_t)t;
      const double w = W[buf][m][pos];
      acc[m][0] += fmulmod(c0, w, q, qinv);
      acc[m][1] += fmulmod(c1, w, q, qinv);
    }
    if ((j & 3) == 3) {
#pragma unroll
      for (int m = 0; m < M; ++m) {
        acc[m][0] = fred(acc[m][0], q, qinv);
        acc[m][1] = fred(acc[m][1], q, qinv);
      }
    }
    if (j + 1 < J) {
#pragma unroll
      for (int m = 0; m < M; ++m) W[buf ^ 1][m][t] = u2d(pw[m]);
      c0 = u2d(p0);
      c1 = u2d(p1);
    }
    __syncthreads();
  }
#pragma unroll
  for (int m = 0; m < M; ++m)
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      uint64_t* o = b.out[m] + ((size_t)p * n + i) * N + x;
      double v = acc[m][p];
      if (accumulate) v += u2d(*o);
      *o = d2u(fcanon(v, q, qinv));
    }
}

// The same with every row moved by the TMA bulk engine: per operand j one stage of the NST-deep shared ring holds
// the operand's c0 and c1 rows and the M source rows of its weight terms (2 KB each, cp.async.bulk issued by one
// thread, completion on the stage's mbarrier), so NST - 1 operands are in flight while one is multiplied -- the
// PRCR stream re-reads each stored weight row once per family member from L2 and needs that memory parallelism.
constexpr int kPbStages = 4;
template <int M>
constexpr size_t pmult_ring_smem() { return (size_t)kPbStages * (M + 2) * 2048 + 8 * kPbStages; }
template <int M, int NS = kPbStages>
constexpr size_t pmult_ring_ws_smem() { return (size_t)NS * (M + 2) * 2048 + 16 * NS; }
template <int M>
__global__ void __launch_bounds__(256) k_pmult_ring(const __grid_constant__ PBlock b, int J, DevTables dt, int level,
                                                    int logN, int accumulate) {
  extern __shared__ __align__(128) double ring[];  // [NST][M + 2][256] then the NST mbarriers
  uint64_t* mbar = reinterpret_cast<uint64_t*>(ring + (size_t)kPbStages * (M + 2) * 256);
  const size_t N = (size_t)1 << logN;
  const int t = threadIdx.x;
  const uint32_t r = blockIdx.x, x = r * 256 + t;
  const int i = blockIdx.y;
  const size_t n = level + 1;
  const PrimeConst& pc = dt.pc[i];
  const double q = pc.qd, qinv = pc.qinv;
  auto issue = [&](int j) {  // thread 0
    const int st = j % kPbStages;
    uint64_t* dst = reinterpret_cast<uint64_t*>(ring + (size_t)st * (M + 2) * 256);
    tma::mbar_expect(mbar + st, (M + 2) * 2048);
    tma::bulk_row(dst, b.ct[j] + (size_t)i * N + (size_t)r * 256, mbar + st);
    tma::bulk_row(dst + 256, b.ct[j] + (n + i) * N + (size_t)r * 256, mbar + st);
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const uint32_t k = b.prot[m][j];
      const uint32_t sr = k != 1 ? aut_index(r * 256u, k, logN) >> 8 : r;
      tma::bulk_row(dst + 256 * (2 + m), b.pt_base + ((size_t)b.pt_idx[m][j] * n + i) * N + (size_t)sr * 256,
                    mbar + st);
    }
  };
  if (t == 0) {
    for (int st = 0; st < kPbStages; ++st) tma::mbar_init(mbar + st);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int j = 0; j < kPbStages - 1 && j < J; ++j) issue(j);
  }
  __syncthreads();
  double acc[M][2];
#pragma unroll
  for (int m = 0; m < M; ++m) acc[m][0] = acc[m][1] = 0.0;
  for (int j = 0; j < J; ++j) {
    const int st = j % kPbStages;
    if (t == 0 && j + kPbStages - 1 < J) issue(j + kPbStages - 1);  // its stage was released at the end of j - 1
    tma::mbar_wait(mbar + st, (uint32_t)(j / kPbStages) & 1);
    const uint64_t* S = reinterpret_cast<const uint64_t*>(ring + (size_t)st * (M + 2) * 256);
    const double c0 = u2d(S[t]), c1 = u2d(S[256 + t]);
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const uint32_t k = b.prot[m][j];
      const uint32_t pos = k != 1 ? aut_index(x, k, logN) & 255u : (uint32_t)t;
      const double w = u2d(S[256 * (2 + m) + pos]);
      acc[m][0] += fmulmod(c0, w, q, qinv);
      acc[m][1] += fmulmod(c1, w, q, qinv);
    }
    if ((j & 3) == 3) {
#pragma unroll
      for (int m = 0; m < M; ++m) {
        acc[m][0] = fred(acc[m][0], q, qinv);
        acc[m][1] = fred(acc[m][1], q, qinv);
      }
    }
    tma::proxy_fence();  // this thread's reads of the stage precede the next bulk write into it
    __syncthreads();
  }
#pragma unroll
  for (int m = 0; m < M; ++m)
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      uint64_t* o = b.out[m] + ((size_t)p * n + i) * N + x;
      double v = acc[m][p];
      if (accumulate) v += u2d(*o);
      *o = d2u(fcanon(v, q, qinv));
    }
}

// The same ring with a producer warp (round 2): warps 0-7 consume (one thread per word, as above), warp 8 only
// refills the ring.  A stage is released by one arrival per consumer warp on its "empty" mbarrier, so the consumer
// warps never wait for each other (no CTA barrier per operand); the producer waits for the 8 arrivals before it
// reuses a stage.  Same arithmetic, term order and output as k_pmult_ring.
template <int M, int NS = kPbStages>
__global__ void __launch_bounds__(288) k_pmult_ring_ws(const __grid_constant__ PBlock b, int J, DevTables dt,
                                                       int level, int logN, int accumulate) {
  extern __shared__ __align__(128) double ring[];  // [NST][M + 2][256], then NST full and NST empty mbarriers
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)NS * (M + 2) * 256);
  uint64_t* empty = full + NS;
  const size_t N = (size_t)1 << logN;
  const int t = threadIdx.x;
  const uint32_t r = blockIdx.x;
  const int i = blockIdx.y;
  const size_t n = level + 1;
  if (t == 0) {
    for (int st = 0; st < NS; ++st) {
      tma::mbar_init(full + st);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(tma::saddr(empty + st)) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (t >= 256) {  // producer warp
    if (t == 256) {
      for (int j = 0; j < J; ++j) {
        const int st = j % NS;
        if (j >= NS) tma::mbar_wait(empty + st, (uint32_t)(j / NS - 1) & 1);
        uint64_t* dst = reinterpret_cast<uint64_t*>(ring + (size_t)st * (M + 2) * 256);
        tma::mbar_expect(full + st, (M + 2) * 2048);
        tma::bulk_row(dst, b.ct[j] + (size_t)i * N + (size_t)r * 256, full + st);
        tma::bulk_row(dst + 256, b.ct[j] + (n + i) * N + (size_t)r * 256, full + st);
#pragma unroll
        for (int m = 0; m < M; ++m) {
          const uint32_t k = b.prot[m][j];
          const uint32_t sr = k != 1 ? aut_index(r * 256u, k, logN) >> 8 : r;
          tma::bulk_row(dst + 256 * (2 + m), b.pt_base + ((size_t)b.pt_idx[m][j] * n + i) * N + (size_t)sr * 256,
                        full + st);
        }
      }
    }
    return;
  }
  const uint32_t x = r * 256 + t;
  const PrimeConst& pc = dt.pc[i];
  const double q = pc.qd, qinv = pc.qinv;
  double acc[M][2];
#pragma unroll
  for (int m = 0; m < M; ++m) acc[m][0] = acc[m][1] = 0.0;
  for (int j = 0; j < J; ++j) {
    const int st = j % NS;
    tma::mbar_wait(full + st, (uint32_t)(j / NS) & 1);
    const uint64_t* S = reinterpret_cast<const uint64_t*>(ring + (size_t)st * (M + 2) * 256);
    const double c0 = u2d(S[t]), c1 = u2d(S[256 + t]);
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const uint32_t k = b.prot[m][j];
      const uint32_t pos = k != 1 ? aut_index(x, k, logN) & 255u : (uint32_t)t;
      const double w = u2d(S[256 * (2 + m) + pos]);
      acc[m][0] += fmulmod(c0, w, q, qinv);
      acc[m][1] += fmulmod(c1, w, q, qinv);
    }
    if ((j & 3) == 3) {
#pragma unroll
      for (int m = 0; m < M; ++m) {
        acc[m][0] = fred(acc[m][0], q, qinv);
        acc[m][1] = fred(acc[m][1], q, qinv);
      }
    }
    if (j + NS < J) {  // the stage is refilled for j + NST: release it (one arrival per warp)
      tma::proxy_fence();
      __syncwarp();
      if ((t & 31) == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tma::saddr(empty + st)) : "memory");
    }
  }
#pragma unroll
  for (int m = 0; m < M; ++m)
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      uint64_t* o = b.out[m] + ((size_t)p * n + i) * N + x;
      double v = acc[m][p];
      if (accumulate) v += u2d(*o);
      *o = d2u(fcanon(v, q, qinv));
    }
}

// out[p][i][x] (+)= sum_m ct_m[p][i][x] * pt_m[i][x] mod q_i.  grid (N/256, l+1, 2)
__global__ void k_pmult_acc(const __grid_constant__ TermPtrs tp, int nterm, uint64_t* __restrict__ out, DevTables dt, int level, int logN,
                            int accumulate) {
  const size_t N = (size_t)1 << logN;
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y, p = blockIdx.z;
  const size_t n = level + 1;
  const size_t o = ((size_t)p * n + i) * N + x;
  const PrimeConst& pc = dt.pc[i];
  U128 acc{0, 0};
  for (int m = 0; m < nterm; ++m) {
    const uint32_t xs = tp.prot[m] != 1 ? aut_index(x, tp.prot[m], logN) : x;
    mac(acc, tp.ct[m][o], tp.pt[m][(size_t)i * N + xs]);
  }
  uint64_t r = reduce128(acc, pc);
  if (accumulate) r = add_mod(r, out[o], pc.q);
  out[o] = r;
}

// out = a + b over [npoly][l+1][N].  grid (N/256, (l+1)*npoly)
__global__ void k_add(const uint64_t* __restrict__ a, const uint64_t* __restrict__ b, uint64_t* __restrict__ out,
                      DevTables dt, int nlimb, int logN) {
  const size_t N = (size_t)1 << logN;
  const size_t o = (size_t)blockIdx.y * N + blockIdx.x * blockDim.x + threadIdx.x;
  out[o] = add_mod(a[o], b[o], dt.pc[blockIdx.y % nlimb].q);
}

// Batched rescale / mask product over up to kG items (pointer arrays as __grid_constant__ parameters).
struct ItemPtrs {
  const uint64_t* in[kG];
  uint64_t* out[kG];
  uint64_t* v[kG];  // rescale scratch: iNTT of the dropped limb [2][N]
  uint64_t* w[kG];  // rescale scratch: its lift [2][l][N]
};
// w_g[p][i] = [centre(v_g[p])]_{q_i}.  grid (N/256, l, 2 G), blockIdx.z = 2 g + p
__global__ void k_rescale_lift_multi(const __grid_constant__ ItemPtrs a, DevTables dt, int level, int logN) {
  const size_t N = (size_t)1 << logN;
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y, g = blockIdx.z >> 1, p = blockIdx.z & 1;
  const uint64_t ql = dt.pc[level].q, qi = dt.pc[i].q;
  const uint64_t val = a.v[g][(size_t)p * N + x];
  uint64_t r;
  if (val > (ql - 1) / 2) {  // negative representative val - ql
    const uint64_t m = reduce64(ql - val, dt.pc[i]);
    r = m ? qi - m : 0;
  } else {
    r = reduce64(val, dt.pc[i]);
  }
  a.w[g][((size_t)p * level + i) * N + x] = r;
}
// out_g[p][i] = (in_g[p][i] - w_g[p][i]) q_l^{-1}.  grid (N/256, l, 2 G)
__global__ void k_rescale_final_multi(const __grid_constant__ ItemPtrs a, const RescaleConst* rc, DevTables dt,
                                      int level, int logN) {
  const size_t N = (size_t)1 << logN;
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y, g = blockIdx.z >> 1, p = blockIdx.z & 1;
  const uint64_t q = dt.pc[i].q;
  const uint64_t v = sub_mod(a.in[g][((size_t)p * (level + 1) + i) * N + x], a.w[g][((size_t)p * level + i) * N + x], q);
  a.out[g][((size_t)p * level + i) * N + x] = shoup(v, rc->ql_inv[i], rc->ql_inv_sh[i], q);
}
// out_g = in_g (.) pt (one plaintext for every item; the IR_g mask).  grid (N/256, l+1, 2 G)
__global__ void k_pmult_many(const __grid_constant__ ItemPtrs a, const uint64_t* __restrict__ pt, DevTables dt,
                             int level, int logN) {
  const size_t N = (size_t)1 << logN;
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y, g = blockIdx.z >> 1, p = blockIdx.z & 1;
  const PrimeConst& pc = dt.pc[i];
  const size_t o = ((size_t)p * (level + 1) + i) * N + x;
  a.out[g][o] = d2u(fcanon(fmulmod(u2d(a.in[g][o]), u2d(pt[(size_t)i * N + x]), pc.qd, pc.qinv), pc.qd, pc.qinv));
}

// small signed values (int8 or int32 source) to residues on chain limbs [0, nlimb).  grid (N/256, nlimb)
template <class T>
__global__ void k_small_to_limbs(const T* __restrict__ v, uint64_t* __restrict__ out, const uint8_t* chain_map,
                                 DevTables dt, int logN) {
  const size_t N = (size_t)1 << logN;
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  const int t = chain_map ? chain_map[blockIdx.y] : blockIdx.y;
  const uint64_t q = dt.pc[t].q;
  const int64_t s = (int64_t)v[x];
  uint64_t r;
  if (s >= 0) {
    r = reduce64((uint64_t)s, dt.pc[t]);
  } else {
    const uint64_t m = reduce64((uint64_t)(-s), dt.pc[t]);
    r = m ? q - m : 0;
  }
  out[(size_t)blockIdx.y * N + x] = r;
}

// CBD(21) error polynomial (coefficient domain).  grid N/256
__global__ void k_sample_cbd(uint64_t seed, uint32_t dom, uint64_t obj, int32_t* __restrict__ e) {
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  e[x] = cbd21(draw(seed, dom, obj, 0, x));
}

// Rotation-key digit j: a = uniform (NTT domain) written to evk[j][1],
// b = -a*s + e + g_j*kappa(s) written to evk[j][0].  grid (N/256, n_q+n_p)
__global__ void k_evk_digit(uint64_t* __restrict__ evk, const uint64_t* __restrict__ s_ntt,
                            const uint64_t* __restrict__ sk_ntt, const uint64_t* __restrict__ e_ntt, uint64_t seed,
                            uint64_t obj, const uint64_t* __restrict__ gmod, int j, int L1, DevTables dt, int logN) {
  const size_t N = (size_t)1 << logN;
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  const int t = blockIdx.y;
  const PrimeConst& pc = dt.pc[t];
  const size_t o = (size_t)t * N + x;
  const uint64_t a = uniform_mod(draw(seed, kDomEvkA, obj, (uint32_t)t, x), pc.q);
  uint64_t b = sub_mod(e_ntt[o], mul_mod(a, s_ntt[o], pc), pc.q);
  if (gmod[t]) b = add_mod(b, mul_mod(gmod[t], sk_ntt[o], pc), pc.q);
  evk_store(evk + ((size_t)(j * 2 + 1) * L1 + t) * evk_limb_words(N), x, a);  // packed (hy_arith.cuh)
  evk_store(evk + ((size_t)(j * 2 + 0) * L1 + t) * evk_limb_words(N), x, b);
}

// Generic 48-bit packing of n4 groups of 4 words (hy_pack48 / hy_unpack48): group m = words 4m..4m+3 <->
// the 3 uint64 (24 bytes) at 3m, the layout of the packed keys.  One thread per group.
__global__ void k_pack48(const uint64_t* __restrict__ in, uint64_t* __restrict__ out, size_t n4) {
  const size_t m = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n4) return;
  const ulonglong2 a = reinterpret_cast<const ulonglong2*>(in)[2 * m];
  const ulonglong2 b = reinterpret_cast<const ulonglong2*>(in)[2 * m + 1];
  out[3 * m] = (a.x & kM48) | (a.y << 48);
  out[3 * m + 1] = ((a.y & kM48) >> 16) | (b.x << 32);
  out[3 * m + 2] = ((b.x & kM48) >> 32) | (b.y << 16);
}
__global__ void k_unpack48(const uint64_t* __restrict__ in, uint64_t* __restrict__ out, size_t n4) {
  const size_t m = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n4) return;
  uint64_t w0, w1, w2, w3;
  evk_unpack4(in[3 * m], in[3 * m + 1], in[3 * m + 2], w0, w1, w2, w3);
  reinterpret_cast<ulonglong2*>(out)[2 * m] = make_ulonglong2(w0, w1);
  reinterpret_cast<ulonglong2*>(out)[2 * m + 1] = make_ulonglong2(w2, w3);
}

// Packed key <-> one uint64 per word (hy_evk_pack / hy_evk_unpack).  grid (N/256, n_limbs)
__global__ void k_evk_pack(const uint64_t* __restrict__ in, uint64_t* __restrict__ out, int logN) {
  const size_t N = (size_t)1 << logN;
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  evk_store(out + blockIdx.y * evk_limb_words(N), x, in[blockIdx.y * N + x]);
}
__global__ void k_evk_unpack(const uint64_t* __restrict__ in, uint64_t* __restrict__ out, int logN) {
  const size_t N = (size_t)1 << logN;
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  out[blockIdx.y * N + x] = evk_word(in + blockIdx.y * evk_limb_words(N), x);
}

// Encryption: c1 = a (uniform, NTT domain), c0 = -a*s + e + m.  grid (N/256, l+1)
__global__ void k_encrypt(const uint64_t* __restrict__ m, const uint64_t* __restrict__ s_ntt,
                          const uint64_t* __restrict__ e_ntt, uint64_t seed, uint64_t ct_id, uint64_t* __restrict__ ct,
                          DevTables dt, int level, int logN) {
  const size_t N = (size_t)1 << logN;
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  const PrimeConst& pc = dt.pc[i];
  const size_t o = (size_t)i * N + x;
  const uint64_t a = uniform_mod(draw(seed, kDomEncA, ct_id, (uint32_t)i, x), pc.q);
  uint64_t c0 = sub_mod(e_ntt[o], mul_mod(a, s_ntt[o], pc), pc.q);
  c0 = add_mod(c0, m[o], pc.q);
  ct[o] = c0;
  ct[(size_t)(level + 1) * N + o] = a;
}

// m = c0 + c1 * s.  grid (N/256, l+1)
__global__ void k_decrypt(const uint64_t* __restrict__ ct, const uint64_t* __restrict__ s_ntt,
                          uint64_t* __restrict__ m, DevTables dt, int level, int logN) {
  const size_t N = (size_t)1 << logN;
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  const PrimeConst& pc = dt.pc[i];
  const size_t o = (size_t)i * N + x;
  m[o] = add_mod(ct[o], mul_mod(ct[(size_t)(level + 1) * N + o], s_ntt[o], pc), pc.q);
}

// HWT secret (DESIGN R-SK), host side: partial Fisher-Yates over Philox draws.
void sample_secret(uint64_t seed, uint32_t N, uint32_t h, std::vector<int8_t>& s) {
  std::vector<uint32_t> idx(N);
  for (uint32_t i = 0; i < N; ++i) idx[i] = i;
  s.assign(N, 0);
  for (uint32_t t = 0; t < h && t < N; ++t) {
    Philox4 w = draw(seed, kDomSecret, 0, 0, t);
    uint64_t u = ((uint64_t)w.v[1] << 32) | w.v[0];
    uint32_t j = t + (uint32_t)(u % (N - t));
    std::swap(idx[t], idx[j]);
    s[idx[t]] = (w.v[2] & 1) ? -1 : 1;
  }
}

// s in the NTT domain on chain limbs 0..nlimb-1 (or a chain map), into out [nlimb][N].
hy_status secret_ntt(hy_ctx* c, uint64_t seed, uint32_t nlimb, uint64_t* out, int8_t* d_s, cudaStream_t s) {
  std::vector<int8_t> h_s;
  sample_secret(seed, c->N, c->h, h_s);
  cudaMemcpyAsync(d_s, h_s.data(), c->N, cudaMemcpyHostToDevice, s);
  cudaStreamSynchronize(s);  // h_s is a pageable temporary
  dim3 g(c->N / kT, nlimb);
  {
    KTimer kt(c, FAM_CLIENT, s);
    k_small_to_limbs<int8_t><<<g, kT, 0, s>>>(d_s, out, nullptr, c->dt, c->log_n);
  }
  std::vector<uint32_t> chain(nlimb);
  for (uint32_t i = 0; i < nlimb; ++i) chain[i] = i;
  ntt_contig(c, out, out, chain.data(), nlimb, false, s);
  return HY_OK;
}

}  // namespace
}  // namespace hy

using namespace hy;

namespace hy {
// out (+)= sum_i ct_i (.) PRot_{k_i}(pt_i)   (k_i = Galois element, 1 = no rotation)
hy_status pmult_acc_prot(hy_ctx* c, const uint64_t* const* cts, const uint64_t* const* pts, const uint64_t* ks,
                         uint32_t n, uint32_t level, uint64_t* out, int accumulate, void* stream) {
  if (!c || !cts || !pts || !out) return fail(HY_E_ARG, "null");
  if (level >= c->n_q) return fail(HY_E_ARG, "level out of range");
  if (n == 0 && !accumulate) return fail(HY_E_ARG, "empty product sum");
  cudaStream_t s = st(stream);
  for (uint32_t done = 0; done < n || (n == 0 && done == 0);) {
    uint32_t m = std::min<uint32_t>(n - done, kMaxTerms);
    if (m == 0) break;
    TermPtrs tp;
    for (uint32_t i = 0; i < m; ++i) {
      tp.ct[i] = cts[done + i];
      tp.pt[i] = pts[done + i];
      tp.prot[i] = ks ? ks[done + i] : 1;
      if (!tp.ct[i] || !tp.pt[i]) return fail(HY_E_ARG, "null term");
    }
    dim3 g(c->N / kT, level + 1, 2);
    KTimer kt(c, FAM_ELEM, s);
    kt.bytes = ((uint64_t)m * 3 * (level + 1) + 2ull * (level + 1) * ((accumulate || done > 0) ? 2 : 1)) * c->N * 8;
    k_pmult_acc<<<g, kT, 0, s>>>(tp, (int)m, out, c->dt, level, c->log_n, (accumulate || done > 0) ? 1 : 0);
    done += m;
  }
  return cuda_check("hy_pmult_acc");
}

// Dense block: out_m (+)= sum_j ct_j (.) PRot_{gal[m*J+j]}(pt_base[pt_idx[m*J+j]]), m < M, j < J
hy_status pmult_block(hy_ctx* c, const uint64_t* const* cts, uint32_t J, uint64_t* const* outs, uint32_t M,
                      const uint64_t* pt_base, const uint32_t* pt_idx, const uint64_t* gal, uint32_t level,
                      int accumulate, void* stream) {
  if (!c || !cts || !outs || !pt_base || !pt_idx || !gal) return fail(HY_E_ARG, "null");
  if (level >= c->n_q) return fail(HY_E_ARG, "level out of range");
  if (M == 0 || M > (uint32_t)kPbM || J == 0) return fail(HY_E_ARG, "block shape");
  cudaStream_t s = st(stream);
  for (uint32_t done = 0; done < J;) {
    // operands per launch (HY_PMB_J A/B: 64 splits a 72-operand 3x3 block of 8 inputs into 64 + 8)
    static const uint32_t jcap = getenv("HY_PMB_J") ? (uint32_t)std::max(1, std::min(kPbJ, atoi(getenv("HY_PMB_J"))))
                                                    : (uint32_t)kPbJ;
    const uint32_t jn = std::min<uint32_t>(J - done, jcap);
    PBlock b;
    b.pt_base = pt_base;
    for (uint32_t j = 0; j < jn; ++j) b.ct[j] = cts[done + j];
    for (uint32_t m = 0; m < M; ++m) {
      b.out[m] = outs[m];
      for (uint32_t j = 0; j < jn; ++j) {
        b.pt_idx[m][j] = pt_idx[(size_t)m * J + done + j];
        b.prot[m][j] = (uint32_t)gal[(size_t)m * J + done + j];
      }
    }
    const int acc = (accumulate || done > 0) ? 1 : 0;
    dim3 g(c->N / kT, level + 1);
    KTimer kt(c, FAM_ELEM, s);
    // cts (2 polys) once, every term's weight limb once, outputs written (and read when accumulating)
    kt.bytes = ((uint64_t)jn * 2 + (uint64_t)M * jn + (uint64_t)M * 2 * (acc ? 2 : 1)) * (level + 1) * c->N * 8;
    // HY_PMB_ROWS=0: the per-thread gather kernel (A/B)
    // Kernel choice (r02 A/B): blocks without PRot gathers (every non-PRCR layer) stream their
    // operand and weight rows through the bulk-copy ring (R18 L2_ds MulFilter&Sum 19.5 -> 14.7 ms); PRCR blocks keep
    // the per-thread gather kernel, whose L1-served gathers beat staging rows for the 8-fold reuse of each stored
    // weight row (R18 L1_ca 5.8 ms vs 9.2 ms staged).  HY_PMB_ROWS forces 2 (ring), 1 (register-prefetch rows) or
    // 0 (per-thread gathers).
    bool any_prot = false;
    for (uint32_t m = 0; m < M; ++m)
      for (uint32_t j = 0; j < jn; ++j) any_prot |= b.prot[m][j] != 1;
    static const int forced = getenv("HY_PMB_ROWS") ? atoi(getenv("HY_PMB_ROWS")) : -1;
    const int rows = forced >= 0 ? forced : (any_prot ? 0 : 2);
    if (rows == 2) {
      // HY_PMB_WS=0: the ring without the producer warp (one CTA barrier per operand)
      static const bool ws = getenv("HY_PMB_WS") == nullptr || atoi(getenv("HY_PMB_WS")) != 0;
#define HY_PR(MM)                                                                                                 \
  case MM: {                                                                                                    \
    static bool at = false;                                                                                     \
    if (!at) {                                                                                                  \
      cudaFuncSetAttribute(k_pmult_ring<MM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pmult_ring_smem<MM>()); \
      cudaFuncSetAttribute(k_pmult_ring_ws<MM>, cudaFuncAttributeMaxDynamicSharedMemorySize,                   \
                           (int)pmult_ring_ws_smem<MM>());                                                      \
      at = true;                                                                                                \
    }                                                                                                           \
    if (ws) k_pmult_ring_ws<MM><<<g, kT + 32, pmult_ring_ws_smem<MM>(), s>>>(b, (int)jn, c->dt, level, c->log_n, acc); \
    else k_pmult_ring<MM><<<g, kT, pmult_ring_smem<MM>(), s>>>(b, (int)jn, c->dt, level, c->log_n, acc);        \
  } break;
      switch (M) {
        HY_PR(1)
        HY_PR(2)
        HY_PR(3)
        HY_PR(4)
        HY_PR(5)
        HY_PR(6)
        HY_PR(7)
        default:
          HY_PR(8)
      }
#undef HY_PR
      done += jn;
      continue;
    }
    if (rows == 1) {
      switch (M) {
        case 1: k_pmult_rows<1><<<g, kT, 0, s>>>(b, (int)jn, c->dt, level, c->log_n, acc); break;
        case 2: k_pmult_rows<2><<<g, kT, 0, s>>>(b, (int)jn, c->dt, level, c->log_n, acc); break;
        case 3: k_pmult_rows<3><<<g, kT, 0, s>>>(b, (int)jn, c->dt, level, c->log_n, acc); break;
        case 4: k_pmult_rows<4><<<g, kT, 0, s>>>(b, (int)jn, c->dt, level, c->log_n, acc); break;
        case 5: k_pmult_rows<5><<<g, kT, 0, s>>>(b, (int)jn, c->dt, level, c->log_n, acc); break;
        case 6: k_pmult_rows<6><<<g, kT, 0, s>>>(b, (int)jn, c->dt, level, c->log_n, acc); break;
        case 7: k_pmult_rows<7><<<g, kT, 0, s>>>(b, (int)jn, c->dt, level, c->log_n, acc); break;
        default: k_pmult_rows<8><<<g, kT, 0, s>>>(b, (int)jn, c->dt, level, c->log_n, acc); break;
      }
      done += jn;
      continue;
    }
    // the PRot structure of the block (KM, see k_pmult_block)
    bool per_j = true, per_m = true;
    for (uint32_t m = 0; m < M; ++m)
      for (uint32_t j = 0; j < jn; ++j) {
        per_j &= b.prot[m][j] == b.prot[0][j];
        per_m &= b.prot[m][j] == b.prot[m][0];
      }
    const int km = per_j ? 1 : (per_m ? 2 : 0);
#define HY_PB(MM)                                                                                 \
  case MM:                                                                                        \
    if (km == 1) k_pmult_block<MM, 1><<<g, kT, 0, s>>>(b, (int)jn, c->dt, level, c->log_n, acc);  \
    else if (km == 2) k_pmult_block<MM, 2><<<g, kT, 0, s>>>(b, (int)jn, c->dt, level, c->log_n, acc); \
    else k_pmult_block<MM, 0><<<g, kT, 0, s>>>(b, (int)jn, c->dt, level, c->log_n, acc);           \
    break;
    switch (M) {
      HY_PB(1)
      HY_PB(2)
      HY_PB(3)
      HY_PB(4)
      HY_PB(5)
      HY_PB(6)
      HY_PB(7)
      default:
        HY_PB(8)
    }
#undef HY_PB
    done += jn;
  }
  return cuda_check("pmult_block");
}
}  // namespace hy

extern "C" hy_status hy_pmult_acc(hy_ctx* c, const uint64_t* const* cts, const uint64_t* const* pts, uint32_t n,
                                  uint32_t level, uint64_t* out, int accumulate, void* stream) {
  return hy::pmult_acc_prot(c, cts, pts, nullptr, n, level, out, accumulate, stream);
}

extern "C" hy_status hy_pmult(hy_ctx* c, const uint64_t* ct, const uint64_t* pt, uint32_t level, uint64_t* out,
                              void* stream) {
  const uint64_t* a[1] = {ct};
  const uint64_t* b[1] = {pt};
  return hy_pmult_acc(c, a, b, 1, level, out, 0, stream);
}

extern "C" hy_status hy_pmult_batch(hy_ctx* c, const uint64_t* const* cts, uint32_t n, const uint64_t* pt,
                                    uint32_t level, uint64_t* const* outs, void* stream) {
  if (!c || !pt || (n && (!cts || !outs))) return fail(HY_E_ARG, "null");
  for (uint32_t i = 0; i < n; ++i)
    for (uint32_t j = 0; j < n; ++j)
      if (i != j && outs[i] == cts[j]) return fail(HY_E_ARG, "an output aliases another item's input");
  return pmult_many(c, cts, n, pt, level, outs, st(stream));
}

extern "C" hy_status hy_add(hy_ctx* c, const uint64_t* a, const uint64_t* b, uint32_t npoly, uint32_t level,
                            uint64_t* out, void* stream) {
  if (!c || !a || !b || !out) return fail(HY_E_ARG, "null");
  if (level >= c->n_q || npoly == 0) return fail(HY_E_ARG, "level/npoly out of range");
  dim3 g(c->N / kT, (level + 1) * npoly);
  KTimer kt(c, FAM_ELEM, st(stream));
  kt.bytes = 3ull * (level + 1) * npoly * c->N * 8;
  k_add<<<g, kT, 0, st(stream)>>>(a, b, out, c->dt, level + 1, c->log_n);
  return cuda_check("hy_add");
}

// out = a - b mod q over [npoly][l+1][N].  grid (N/256, (l+1)*npoly)
namespace hy {
namespace {
__global__ void k_sub(const uint64_t* __restrict__ a, const uint64_t* __restrict__ b, uint64_t* __restrict__ out,
                      DevTables dt, int nlimb) {
  const size_t N = (size_t)gridDim.x * blockDim.x;
  const size_t o = (size_t)blockIdx.y * N + blockIdx.x * blockDim.x + threadIdx.x;
  out[o] = sub_mod(a[o], b[o], dt.pc[blockIdx.y % nlimb].q);
}
}  // namespace
}  // namespace hy

extern "C" hy_status hy_sub(hy_ctx* c, const uint64_t* a, const uint64_t* b, uint32_t npoly, uint32_t level,
                            uint64_t* out, void* stream) {
  if (!c || !a || !b || !out) return fail(HY_E_ARG, "null");
  if (level >= c->n_q || npoly == 0) return fail(HY_E_ARG, "level/npoly out of range");
  dim3 g(c->N / kT, (level + 1) * npoly);
  KTimer kt(c, FAM_ELEM, st(stream));
  kt.bytes = 3ull * (level + 1) * npoly * c->N * 8;
  k_sub<<<g, kT, 0, st(stream)>>>(a, b, out, c->dt, level + 1);
  return cuda_check("hy_sub");
}

extern "C" hy_status hy_level_down(hy_ctx* c, const uint64_t* ct, uint32_t level, uint32_t new_level,
                                   uint64_t* out, void* stream) {
  if (!c || !ct || !out) return fail(HY_E_ARG, "null");
  if (level >= c->n_q) return fail(HY_E_ARG, "level out of range");
  if (new_level > level) return fail(HY_E_LEVEL_MISMATCH, "level_down cannot raise the level");
  if (ct == out && new_level != level) return fail(HY_E_ARG, "level_down cannot run in place");
  if (ct == out) return HY_OK;
  const size_t N = c->N;
  // the first new_level+1 limbs of each polynomial: Q_l -> Q_l' is a reduction of every coefficient, which in
  // the RNS is dropping the limbs above new_level (scale unchanged)
  cudaMemcpy2DAsync(out, (new_level + 1) * N * 8, ct, (size_t)(level + 1) * N * 8, (new_level + 1) * N * 8, 2,
                    cudaMemcpyDeviceToDevice, st(stream));
  return cuda_check("hy_level_down");
}

namespace hy {
// Rescale of n ciphertexts at `level` (DESIGN R-RESCALE), batched kG per launch set:
// iNTT of every dropped limb, centred lift, NTT of the lifts, (c - w) q_l^{-1}.  out_g must not alias in_g.
hy_status rescale_multi(hy_ctx* c, const uint64_t* const* cts, uint32_t n, uint32_t level, uint64_t* const* outs,
                        cudaStream_t s) {
  if (!c || (n && (!cts || !outs))) return fail(HY_E_ARG, "null");
  if (level >= c->n_q) return fail(HY_E_ARG, "level out of range");
  if (level == 0) return fail(HY_E_LEVEL_EXHAUSTED, "rescale at level 0");
  if (!c->ws) return fail(HY_E_WORKSPACE, "workspace not set");
  const size_t N = c->N, nl = level + 1;
  // items per launch set: kG, and what the workspace holds (v [2][N] + w [2][level][N] per item, plus alignment)
  const size_t per_item = (2 * N + 2 * (size_t)level * N) * 8 + 512;
  const uint32_t cap = (uint32_t)std::max<size_t>(1, std::min<size_t>(kG, c->ws_bytes / per_item));
  static const bool fused = getenv("HY_FUSE_RESCALE") == nullptr || atoi(getenv("HY_FUSE_RESCALE")) != 0;
  if (fused && moddown_cols_ok(c)) {
    // a ModDown by P = q_level with the centred remainder: inverse row pass of the two dropped limbs, one
    // column kernel (inverse column pass, centred lift, forward column pass of the level targets), one row
    // kernel ((c_i - t_i) q_level^{-1}); the lifted limbs never make an HBM round trip through separate passes
    for (uint32_t done = 0; done < n;) {
      const int G = (int)std::min<uint32_t>(n - done, cap);
      Ws ws{c->ws, c->ws_bytes};
      LimbList L;
      ModUpColsArgs ma{};
      RowsFinalArgs fa{};
      for (int g = 0; g < G; ++g) {
        const uint64_t* in = cts[done + g];
        uint64_t* out = outs[done + g];
        if (!in || !out) return fail(HY_E_ARG, "null ciphertext");
        if (in == out) return fail(HY_E_ARG, "rescale cannot run in place");
        uint64_t* v = ws.take<uint64_t>(2 * N);
        uint64_t* w = ws.take<uint64_t>(2 * level * N);
        if (!w) return fail(HY_E_WORKSPACE, "workspace too small");
        for (int p = 0; p < 2; ++p) L.add(in + ((size_t)p * nl + level) * N, v + (size_t)p * N, level);
        ma.src[g] = v;
        ma.ext[g] = w;
        fa.u[g] = in;
        fa.w[g] = w;
        fa.out[g] = out;
        fa.k0[g] = 1;
      }
      rows_list(c, L, true, s);
      launch_rescale_cols(c, ma, G, level, s);
      launch_rescale_rows_final(c, fa, G, level, s);
      done += G;
    }
    return cuda_check("rescale");
  }
  for (uint32_t done = 0; done < n;) {
    const int G = (int)std::min<uint32_t>(n - done, cap);
    Ws ws{c->ws, c->ws_bytes};
    ItemPtrs a{};
    LimbBatch b;
    b.n = 0;
    for (int g = 0; g < G; ++g) {
      a.in[g] = cts[done + g];
      a.out[g] = outs[done + g];
      if (!a.in[g] || !a.out[g]) return fail(HY_E_ARG, "null ciphertext");
      if (a.in[g] == a.out[g]) return fail(HY_E_ARG, "rescale cannot run in place");
      a.v[g] = ws.take<uint64_t>(2 * N);
      a.w[g] = ws.take<uint64_t>(2 * level * N);
      if (!a.w[g]) return fail(HY_E_WORKSPACE, "workspace too small");
      for (int p = 0; p < 2; ++p) {
        b.src[b.n] = a.in[g] + ((size_t)p * nl + level) * N;
        b.dst[b.n] = a.v[g] + (size_t)p * N;
        b.chain[b.n++] = (uint8_t)level;
      }
    }
    launch_ntt(c, b, true, s);
    dim3 g3(c->N / kT, level, 2 * G);
    {
      KTimer kt(c, FAM_RESCALE, s);
      kt.bytes = (uint64_t)G * (2 + 2 * level) * N * 8;
      k_rescale_lift_multi<<<g3, kT, 0, s>>>(a, c->dt, level, c->log_n);
    }
    LimbList L;
    for (int g = 0; g < G; ++g)
      for (int p = 0; p < 2; ++p)
        for (uint32_t i = 0; i < level; ++i) {
          uint64_t* q = a.w[g] + ((size_t)p * level + i) * N;
          L.add(q, q, i);
        }
    ntt_list(c, L, false, s);
    {
      KTimer kt(c, FAM_RESCALE, s);
      kt.bytes = (uint64_t)G * 2 * (nl + 2 * level) * N * 8;
      k_rescale_final_multi<<<g3, kT, 0, s>>>(a, c->d_rescale[level], c->dt, level, c->log_n);
    }
    done += G;
  }
  return cuda_check("rescale");
}

// out_g = ct_g (.) pt for n ciphertexts (one plaintext), batched kG per launch
hy_status pmult_many(hy_ctx* c, const uint64_t* const* cts, uint32_t n, const uint64_t* pt, uint32_t level,
                     uint64_t* const* outs, cudaStream_t s) {
  if (!c || !pt || (n && (!cts || !outs))) return fail(HY_E_ARG, "null");
  if (level >= c->n_q) return fail(HY_E_ARG, "level out of range");
  for (uint32_t done = 0; done < n;) {
    const int G = (int)std::min<uint32_t>(n - done, kG);
    ItemPtrs a{};
    for (int g = 0; g < G; ++g) {
      a.in[g] = cts[done + g];
      a.out[g] = outs[done + g];
    }
    dim3 g3(c->N / kT, level + 1, 2 * G);
    KTimer kt(c, FAM_ELEM, s);
    kt.bytes = (uint64_t)(level + 1) * c->N * 8 * (4 * G + 1);
    k_pmult_many<<<g3, kT, 0, s>>>(a, pt, c->dt, level, c->log_n);
    done += G;
  }
  return cuda_check("pmult_many");
}
}  // namespace hy

extern "C" hy_status hy_rescale(hy_ctx* c, const uint64_t* ct, uint32_t level, uint64_t* out, void* stream) {
  if (!c || !ct || !out) return fail(HY_E_ARG, "null");
  return rescale_multi(c, &ct, 1, level, &out, st(stream));
}

extern "C" hy_status hy_rescale_batch(hy_ctx* c, const uint64_t* const* cts, uint32_t n, uint32_t level,
                                      uint64_t* const* outs, void* stream) {
  if (!c || (n && (!cts || !outs))) return fail(HY_E_ARG, "null");
  for (uint32_t i = 0; i < n; ++i)
    for (uint32_t j = 0; j < n; ++j)
      if (outs[i] == cts[j]) return fail(HY_E_ARG, "rescale output aliases an input");
  return rescale_multi(c, cts, n, level, outs, st(stream));
}

namespace hy {
namespace {
// s^2 in the NTT domain: the pointwise square of NTT(s) (NTT multiplication = negacyclic product)
__global__ void k_square_limbs(const uint64_t* __restrict__ s_ntt, uint64_t* __restrict__ out, DevTables dt,
                               int logN) {
  const size_t N = (size_t)1 << logN;
  const size_t o = (size_t)blockIdx.y * N + blockIdx.x * blockDim.x + threadIdx.x;
  out[o] = mul_mod(s_ntt[o], s_ntt[o], dt.pc[blockIdx.y]);
}

// Key-switching key to the secret s from kappa_k(s) (k odd: rotation key, DESIGN R-EVK) or from s^2 (k = 0:
// relinearization key, DESIGN R-RELIN); object ids (k << 8) | j.
hy_status keygen_ks(hy_ctx* c, uint64_t sk_seed, uint64_t ek_seed, uint64_t k, uint64_t* evk, void* stream) {
  if (!c || !evk) return fail(HY_E_ARG, "null");
  if (k != 0 && (!(k & 1) || k >= 2ull * c->N)) return fail(HY_E_ARG, "bad Galois element");
  if (!c->ws) return fail(HY_E_WORKSPACE, "workspace not set");
  cudaStream_t s = st(stream);
  const uint32_t L1 = c->n_q + c->n_p;
  const size_t N = c->N;
  Ws ws{c->ws, c->ws_bytes};
  uint64_t* s_ntt = ws.take<uint64_t>(L1 * N);
  uint64_t* sk_ntt = ws.take<uint64_t>(L1 * N);
  uint64_t* e_ntt = ws.take<uint64_t>(L1 * N);
  int32_t* e = ws.take<int32_t>(N);
  int8_t* d_s = ws.take<int8_t>(N);
  uint64_t* gm = ws.take<uint64_t>(kMaxChain);
  if (!gm) return fail(HY_E_WORKSPACE, "workspace too small for key generation");
  secret_ntt(c, sk_seed, L1, s_ntt, d_s, s);
  if (k == 0) {
    KTimer kt(c, FAM_CLIENT, s);
    k_square_limbs<<<dim3(c->N / kT, L1), kT, 0, s>>>(s_ntt, sk_ntt, c->dt, c->log_n);
  } else {
    launch_automorph(c, s_ntt, sk_ntt, L1, k, s);  // kappa_k(s): NTT-domain permutation
  }
  std::vector<uint32_t> chain(L1);
  for (uint32_t i = 0; i < L1; ++i) chain[i] = i;
  std::vector<uint64_t> g(L1);
  for (uint32_t j = 0; j < c->dnum; ++j) {
    const uint64_t obj = (k << 8) | j;
    dim3 gg(c->N / kT, L1);
    {
      KTimer kt(c, FAM_CLIENT, s, 2);
      k_sample_cbd<<<c->N / kT, kT, 0, s>>>(ek_seed, kDomEvkE, obj, e);
      k_small_to_limbs<int32_t><<<gg, kT, 0, s>>>(e, e_ntt, nullptr, c->dt, c->log_n);
    }
    ntt_contig(c, e_ntt, e_ntt, chain.data(), L1, false, s);
    // g_j = P on the q-limbs of digit j, 0 elsewhere (DESIGN R-EVK)
    for (uint32_t t = 0; t < L1; ++t) {
      g[t] = 0;
      if (t < c->n_q && t >= j * c->alpha && t < (j + 1) * c->alpha) {
        const uint64_t qt = c->mod[t];
        uint64_t v = 1;
        for (uint32_t kk = 0; kk < c->n_p; ++kk) v = (uint64_t)((unsigned __int128)v * (c->mod[c->n_q + kk] % qt) % qt);
        g[t] = v;
      }
    }
    cudaMemcpyAsync(gm, g.data(), L1 * 8, cudaMemcpyHostToDevice, s);
    {
      KTimer kt(c, FAM_CLIENT, s);
      k_evk_digit<<<gg, kT, 0, s>>>(evk, s_ntt, sk_ntt, e_ntt, ek_seed, obj, gm, (int)j, (int)L1, c->dt, c->log_n);
    }
    cudaStreamSynchronize(s);  // g is reused on the host
  }
  return cuda_check("hy_keygen");
}
}  // namespace
}  // namespace hy

extern "C" hy_status hy_keygen_galois(hy_ctx* c, uint64_t sk_seed, uint64_t ek_seed, uint64_t k, uint64_t* evk,
                                      void* stream) {
  if (k == 0) return fail(HY_E_ARG, "bad Galois element");
  return keygen_ks(c, sk_seed, ek_seed, k, evk, stream);
}

extern "C" hy_status hy_keygen_relin(hy_ctx* c, uint64_t sk_seed, uint64_t ek_seed, uint64_t* rlk, void* stream) {
  return keygen_ks(c, sk_seed, ek_seed, 0, rlk, stream);
}

extern "C" hy_status hy_keygen_rot(hy_ctx* c, uint64_t sk_seed, uint64_t ek_seed, int32_t r, uint64_t* evk,
                                   void* stream) {
  if (!c) return fail(HY_E_ARG, "null");
  return hy_keygen_galois(c, sk_seed, ek_seed, hy_galois_elt(c, r), evk, stream);
}

extern "C" hy_status hy_encrypt(hy_ctx* c, uint64_t sk_seed, uint64_t enc_seed, uint64_t ct_id, const uint64_t* pt,
                                uint32_t level, uint64_t* ct, void* stream) {
  if (!c || !pt || !ct) return fail(HY_E_ARG, "null");
  if (level >= c->n_q) return fail(HY_E_ARG, "level out of range");
  if (!c->ws) return fail(HY_E_WORKSPACE, "workspace not set");
  cudaStream_t s = st(stream);
  const size_t N = c->N, n = level + 1;
  Ws ws{c->ws, c->ws_bytes};
  uint64_t* s_ntt = ws.take<uint64_t>(n * N);
  uint64_t* e_ntt = ws.take<uint64_t>(n * N);
  int32_t* e = ws.take<int32_t>(N);
  int8_t* d_s = ws.take<int8_t>(N);
  if (!d_s) return fail(HY_E_WORKSPACE, "workspace too small");
  secret_ntt(c, sk_seed, n, s_ntt, d_s, s);
  dim3 g(c->N / kT, n);
  {
    KTimer kt(c, FAM_CLIENT, s, 2);
    k_sample_cbd<<<c->N / kT, kT, 0, s>>>(enc_seed, kDomEncE, ct_id, e);
    k_small_to_limbs<int32_t><<<g, kT, 0, s>>>(e, e_ntt, nullptr, c->dt, c->log_n);
  }
  std::vector<uint32_t> chain(n);
  for (uint32_t i = 0; i < n; ++i) chain[i] = i;
  ntt_contig(c, e_ntt, e_ntt, chain.data(), n, false, s);
  KTimer kt(c, FAM_CLIENT, s);
  k_encrypt<<<g, kT, 0, s>>>(pt, s_ntt, e_ntt, enc_seed, ct_id, ct, c->dt, level, c->log_n);
  return cuda_check("hy_encrypt");
}

extern "C" hy_status hy_decrypt(hy_ctx* c, uint64_t sk_seed, const uint64_t* ct, uint32_t level, uint64_t* pt,
                                void* stream) {
  if (!c || !pt || !ct) return fail(HY_E_ARG, "null");
  if (level >= c->n_q) return fail(HY_E_ARG, "level out of range");
  if (!c->ws) return fail(HY_E_WORKSPACE, "workspace not set");
  cudaStream_t s = st(stream);
  const size_t N = c->N, n = level + 1;
  Ws ws{c->ws, c->ws_bytes};
  uint64_t* s_ntt = ws.take<uint64_t>(n * N);
  int8_t* d_s = ws.take<int8_t>(N);
  if (!d_s) return fail(HY_E_WORKSPACE, "workspace too small");
  secret_ntt(c, sk_seed, n, s_ntt, d_s, s);
  dim3 g(c->N / kT, n);
  KTimer kt(c, FAM_CLIENT, s);
  k_decrypt<<<g, kT, 0, s>>>(ct, s_ntt, pt, c->dt, level, c->log_n);
  return cuda_check("hy_decrypt");
}

extern "C" hy_status hy_pt_from_coeffs(hy_ctx* c, const int64_t* h_coeffs, uint32_t level, uint64_t* pt,
                                       void* stream) {
  if (!c || !h_coeffs || !pt) return fail(HY_E_ARG, "null");
  if (level >= c->n_q) return fail(HY_E_ARG, "level out of range");
  if (!c->ws) return fail(HY_E_WORKSPACE, "workspace not set");
  cudaStream_t s = st(stream);
  Ws ws{c->ws, c->ws_bytes};
  int64_t* d = ws.take<int64_t>(c->N);
  if (!d) return fail(HY_E_WORKSPACE, "workspace too small");
  cudaMemcpyAsync(d, h_coeffs, c->N * 8, cudaMemcpyHostToDevice, s);
  const uint32_t n = level + 1;
  dim3 g(c->N / kT, n);
  {
    KTimer kt(c, FAM_CLIENT, s);
    k_small_to_limbs<int64_t><<<g, kT, 0, s>>>(d, pt, nullptr, c->dt, c->log_n);
  }
  std::vector<uint32_t> chain(n);
  for (uint32_t i = 0; i < n; ++i) chain[i] = i;
  ntt_contig(c, pt, pt, chain.data(), n, false, s);
  cudaStreamSynchronize(s);  // h_coeffs may be pageable and reused by the caller
  return cuda_check("hy_pt_from_coeffs");
}

extern "C" hy_status hy_encode(hy_ctx* c, const double* h_slots, uint32_t n_slots, uint64_t scale, uint32_t level,
                               uint64_t* pt, void* stream) {
  if (!c) return fail(HY_E_ARG, "null");
  std::vector<int64_t> coeffs(c->N);
  hy_status s0 = hy_encode_coeffs(c->log_n, h_slots, n_slots, scale, coeffs.data());
  if (s0 != HY_OK) return s0;
  return hy_pt_from_coeffs(c, coeffs.data(), level, pt, stream);
}

namespace hy {
void crt_centered_to_double(const uint64_t* limbs, uint32_t n, uint64_t N, const uint64_t* mods, double* out);
}

extern "C" hy_status hy_decode(hy_ctx* c, const uint64_t* pt, uint32_t level, double scale, uint32_t n_slots,
                               double* h_re, double* h_im, void* stream) {
  if (!c || !pt || !h_re) return fail(HY_E_ARG, "null");
  if (level >= c->n_q) return fail(HY_E_ARG, "level out of range");
  if (n_slots > c->N / 2) return fail(HY_E_CAPACITY, "more slots than N/2");
  if (!(scale > 0)) return fail(HY_E_ARG, "scale must be positive");
  if (!c->ws) return fail(HY_E_WORKSPACE, "workspace not set");
  cudaStream_t s = st(stream);
  const uint32_t n = level + 1;
  Ws ws{c->ws, c->ws_bytes};
  uint64_t* coeff = ws.take<uint64_t>((size_t)n * c->N);
  if (!coeff) return fail(HY_E_WORKSPACE, "workspace too small");
  std::vector<uint32_t> chain(n);
  for (uint32_t i = 0; i < n; ++i) chain[i] = i;
  ntt_contig(c, pt, coeff, chain.data(), n, true, s);
  std::vector<uint64_t> h((size_t)n * c->N);
  cudaMemcpyAsync(h.data(), coeff, h.size() * 8, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  hy_status e = cuda_check("hy_decode");
  if (e != HY_OK) return e;
  std::vector<double> m(c->N);
  crt_centered_to_double(h.data(), n, c->N, c->mod.data(), m.data());
  e = hy_decode_coeffs(c->log_n, m.data(), scale, n_slots, h_re, h_im);
  return e == HY_OK ? HY_OK : fail(e, "hy_decode_coeffs");
}

extern "C" size_t hy_evk_words(const hy_ctx* c) {
  return c ? (size_t)c->dnum * 2 * (c->n_q + c->n_p) * evk_limb_words(c->N) : 0;
}

extern "C" hy_status hy_evk_pack(hy_ctx* c, const uint64_t* d_in, uint64_t* d_out, void* stream) {
  if (!c || !d_in || !d_out) return fail(HY_E_ARG, "null");
  const uint32_t L = c->dnum * 2 * (c->n_q + c->n_p);
  KTimer kt(c, FAM_CLIENT, st(stream));
  k_evk_pack<<<dim3(c->N / kT, L), kT, 0, st(stream)>>>(d_in, d_out, (int)c->log_n);
  return cuda_check("hy_evk_pack");
}

extern "C" hy_status hy_evk_unpack(hy_ctx* c, const uint64_t* d_in, uint64_t* d_out, void* stream) {
  if (!c || !d_in || !d_out) return fail(HY_E_ARG, "null");
  const uint32_t L = c->dnum * 2 * (c->n_q + c->n_p);
  KTimer kt(c, FAM_CLIENT, st(stream));
  k_evk_unpack<<<dim3(c->N / kT, L), kT, 0, st(stream)>>>(d_in, d_out, (int)c->log_n);
  return cuda_check("hy_evk_unpack");
}

extern "C" hy_status hy_pack48(hy_ctx* c, const uint64_t* d_in, uint64_t* d_out, size_t n_words, void* stream) {
  if (!c || !d_in || !d_out) return fail(HY_E_ARG, "null");
  if (n_words % 4) return fail(HY_E_ARG, "n_words must be a multiple of 4");
  const size_t n4 = n_words / 4;
  if (!n4) return HY_OK;
  KTimer kt(c, FAM_ELEM, st(stream));
  kt.bytes = n_words * 14;
  k_pack48<<<(unsigned)((n4 + 255) / 256), 256, 0, st(stream)>>>(d_in, d_out, n4);
  return cuda_check("hy_pack48");
}

extern "C" hy_status hy_unpack48(hy_ctx* c, const uint64_t* d_in, uint64_t* d_out, size_t n_words, void* stream) {
  if (!c || !d_in || !d_out) return fail(HY_E_ARG, "null");
  if (n_words % 4) return fail(HY_E_ARG, "n_words must be a multiple of 4");
  const size_t n4 = n_words / 4;
  if (!n4) return HY_OK;
  KTimer kt(c, FAM_ELEM, st(stream));
  kt.bytes = n_words * 14;
  k_unpack48<<<(unsigned)((n4 + 255) / 256), 256, 0, st(stream)>>>(d_in, d_out, n4);
  return cuda_check("hy_unpack48");
}

// ---------------------------------------------------------------- AddPt, sizes, coefficient wire format
extern "C" hy_status hy_add_pt(hy_ctx* c, const uint64_t* ct, double ct_scale, const uint64_t* pt, double pt_scale,
                               uint32_t level, uint64_t* out, void* stream) {
  if (!c || !ct || !pt || !out) return fail(HY_E_ARG, "null");
  if (level >= c->n_q) return fail(HY_E_ARG, "level out of range");
  if (!(ct_scale > 0.0) || !(pt_scale > 0.0) || std::fabs(ct_scale - pt_scale) > ct_scale * 0x1p-30)
    return fail(HY_E_SCALE_MISMATCH, "AddPt: ciphertext and plaintext scales differ");
  const size_t limb = (size_t)(level + 1) * c->N;
  if (out != ct)  // c1 unchanged
    cudaMemcpyAsync(out + limb, ct + limb, limb * 8, cudaMemcpyDeviceToDevice, st(stream));
  return hy_add(c, ct, pt, 1, level, out, stream);
}

extern "C" size_t hy_ct_bytes(const hy_ctx* c, uint32_t level) {
  return (!c || level >= c->n_q) ? 0 : 2ull * (level + 1) * c->N * 8;
}

extern "C" size_t hy_pt_bytes(const hy_ctx* c, uint32_t level, int with_p) {
  return (!c || level >= c->n_q) ? 0 : (size_t)(level + 1 + (with_p ? c->n_p : 0)) * c->N * 8;
}

extern "C" hy_status hy_export_coeff(hy_ctx* c, const uint64_t* d_ntt, const uint32_t* chain, uint32_t n_limbs,
                                     uint64_t* h_coeff, void* stream) {
  if (!c || !d_ntt || !chain || !h_coeff) return fail(HY_E_ARG, "null");
  for (uint32_t u = 0; u < n_limbs; ++u)
    if (chain[u] >= c->n_q + c->n_p) return fail(HY_E_ARG, "chain index out of range");
  if (!c->ws) return fail(HY_E_WORKSPACE, "workspace not set");
  const size_t N = c->N, per = std::min<size_t>(c->ws_bytes / (N * 8), (size_t)kMaxBatch);
  if (per == 0) return fail(HY_E_WORKSPACE, "workspace smaller than one limb");
  cudaStream_t s = st(stream);
  uint64_t* buf = reinterpret_cast<uint64_t*>(c->ws);
  for (uint32_t u0 = 0; u0 < n_limbs; u0 += (uint32_t)per) {
    const uint32_t m = std::min<uint32_t>((uint32_t)per, n_limbs - u0);
    ntt_contig(c, d_ntt + (size_t)u0 * N, buf, chain + u0, m, true, s);
    cudaMemcpyAsync(h_coeff + (size_t)u0 * N, buf, (size_t)m * N * 8, cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) return cuda_check("hy_export_coeff");
  }
  return cuda_check("hy_export_coeff");
}

extern "C" hy_status hy_import_coeff(hy_ctx* c, const uint64_t* h_coeff, const uint32_t* chain, uint32_t n_limbs,
                                     uint64_t* d_ntt, void* stream) {
  if (!c || !d_ntt || !chain || !h_coeff) return fail(HY_E_ARG, "null");
  const size_t N = c->N;
  for (uint32_t u = 0; u < n_limbs; ++u) {
    if (chain[u] >= c->n_q + c->n_p) return fail(HY_E_ARG, "chain index out of range");
    const uint64_t q = c->mod[chain[u]];
    for (size_t x = 0; x < N; ++x)
      if (h_coeff[(size_t)u * N + x] >= q) return fail(HY_E_ARG, "coefficient not reduced mod its prime");
  }
  cudaStream_t s = st(stream);
  cudaMemcpyAsync(d_ntt, h_coeff, (size_t)n_limbs * N * 8, cudaMemcpyHostToDevice, s);
  ntt_contig(c, d_ntt, d_ntt, chain, n_limbs, false, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return cuda_check("hy_import_coeff");  // host buffer released
  return cuda_check("hy_import_coeff");
}
