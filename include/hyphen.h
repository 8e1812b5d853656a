/*
 * hyphen.h -- C ABI of the B200-native HyPHEN homomorphic-convolution hot path.
 *
 * HyPHEN: "HyPHEN: A Hybrid Packing Method and Its Optimizations for
 * Homomorphic Encryption-Based Neural Networks" (arXiv 2302.02407).
 * P:n below = line n of the paper source; "DESIGN R-x" = a reading
 * of a point the paper leaves silent, listed in DESIGN.md "Readings".
 *
 * Problem statement: a client holds the secret key,
 * encodes/encrypts an image and decrypts the result; a server holding weight
 * plaintexts and evaluation keys runs the convolution layers on ciphertexts.
 * Timing starts once weights and inputs are resident.
 *
 * Conventions (all entry points)
 * ------------------------------
 *  - Scheme: RNS-CKKS over Z[X]/(X^N+1), N = 2^log_n, n = N/2 slots.
 *  - Modulus chain ("chain index" t): q_0..q_{n_q-1} then p_0..p_{n_p-1}.
 *    Hybrid key switching with dnum digits of alpha = ceil(n_q/dnum) q-limbs
 *    (P:1232-1233); n_p = K special primes.
 *  - Words: uint64, residues in [0, modulus).
 *  - Polynomials are in the NTT (evaluation) domain, index k holding
 *    a(psi^(2*br(k)+1)) (DESIGN R-NTT), unless a function says otherwise.
 *  - Ciphertext at level l: device array [2][l+1][N] (c0 then c1), limb i on q_i.
 *    Plaintext at level l: device array [l+1][N].
 *    Evaluation (rotation / relinearization) key: [dnum][2][n_q+n_p] limbs
 *    ([.][0] = b, [.][1] = a), generated at the full level and used at any
 *    level l by reading q-limbs 0..l and the n_p p-limbs (DESIGN R-EVK).
 *    PACKED: every residue is < 2^48 (R-PRIMES), so key words take 6 bytes:
 *    word x of a limb at bytes [6x, 6x+6) little-endian, a limb = 6N bytes,
 *    the key = hy_evk_words() uint64 (3/4 of the unpacked size; 126 MiB at
 *    Set_hyp instead of the paper's 168 MB).  hy_evk_pack/unpack
 *    convert from/to one uint64 per word.
 *  - Ownership: every ciphertext/plaintext/key/workspace buffer is caller-
 *    allocated device memory (in practice torch uint64/int64 tensors).  The
 *    library never frees caller memory.  The context owns its read-only
 *    tables (twiddles, basis-conversion constants), allocated at create time.
 *  - Scratch: operations that need temporaries use the context workspace set
 *    by hy_ctx_set_workspace(); hy_workspace_bytes() gives the size needed.
 *  - Streams: every device call is asynchronous on the given cudaStream_t
 *    (passed as void*; NULL = legacy default stream).  Calls on one context
 *    must not run concurrently on different streams (they share the workspace).
 *  - Errors: a hy_status is returned; outputs are unspecified on error and
 *    hy_last_error() gives a thread-local message.  Preconditions are checked
 *    on the host before any launch.  No exceptions cross the ABI.
 */
#ifndef HYPHEN_H_
#define HYPHEN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HY_OK = 0,
  HY_E_ARG = 1,             /* bad argument / null pointer / size */
  HY_E_LEVEL_MISMATCH = 2,  /* operand levels differ (SPEC LevelMismatch) */
  HY_E_LEVEL_EXHAUSTED = 3, /* level 0 operand to mul/rescale */
  HY_E_SHAPE = 4,           /* shape / slot-count mismatch */
  HY_E_CAPACITY = 5,        /* tensor does not fit the slots */
  HY_E_FORMAT = 6,          /* unsupported packing / gap / transition */
  HY_E_PLAN = 7,            /* conv plan inconsistent with the call */
  HY_E_MISSING_KEY = 8,     /* no evaluation key given for a needed rotation */
  HY_E_CUDA = 9,            /* CUDA runtime error */
  HY_E_WORKSPACE = 10,      /* workspace missing or too small */
  HY_E_NO_DEVICE = 11,      /* no usable sm_100 device */
  HY_E_SCALE_MISMATCH = 12  /* operand scales differ (SPEC: AddCt / AddPt need equal scales) */
} hy_status;

typedef struct hy_ctx hy_ctx;

typedef struct {
  uint32_t log_n;          /* N = 2^log_n, 10 <= log_n <= 16 */
  uint32_t n_q;            /* L+1 ciphertext primes (Set_hyp: 24) */
  uint32_t n_p;            /* K special primes, alpha <= K <= 8 (checked: HY_E_ARG) */
  uint32_t dnum;           /* key-switching digits (Set_hyp: 6) */
  uint32_t hamming_weight; /* secret key weight (192) */
  const uint32_t* q_bits;  /* n_q bit sizes, each in [20, 48] (DESIGN R-PRIMES: residues are exact doubles for
                              the FP64-pipe arithmetic, R-FP64; checked: HY_E_ARG) */
  const uint32_t* p_bits;  /* n_p bit sizes, each in [20, 48] */
} hy_params;

/* ---- context ---------------------------------------------------------- */
/* Generates the primes (DESIGN R-PRIMES: in chain order, the largest unused
 * prime below 2^bits that is 1 mod 2N), roots (R-NTT) and all tables, and
 * uploads them to `cuda_device`.  Fails with HY_E_NO_DEVICE when no CUDA
 * device is present: there is no CPU fallback. */
hy_status hy_ctx_create(const hy_params* params, int cuda_device, hy_ctx** out);
void hy_ctx_destroy(hy_ctx* ctx);
/* chain moduli: n_q + n_p words (host) */
hy_status hy_ctx_moduli(const hy_ctx* ctx, uint64_t* out);
/* Device bytes of a ciphertext [2][l+1][N] / a plaintext [l+1][N] at level l (with_p: [l+1+K][N], the
 * extended basis Q_l u P); 0 for a NULL context or l >= n_q. */
size_t hy_ct_bytes(const hy_ctx* ctx, uint32_t level);
size_t hy_pt_bytes(const hy_ctx* ctx, uint32_t level, int with_p);
uint32_t hy_ctx_alpha(const hy_ctx* ctx);
uint32_t hy_ctx_n_digits(const hy_ctx* ctx, uint32_t level); /* beta = ceil((l+1)/alpha) */
/* Bytes of workspace the context needs to run every operation up to level max_level
 * with at most `max_terms` ciphertexts per batched call. */
size_t hy_workspace_bytes(const hy_ctx* ctx, uint32_t max_level, uint32_t max_terms);
hy_status hy_ctx_set_workspace(hy_ctx* ctx, void* d_ws, size_t bytes);
const char* hy_last_error(void);
/* number of kernels this context has launched since creation (for bench evidence) */
uint64_t hy_ctx_launch_count(const hy_ctx* ctx);
/* Live per-kernel-family timing: while family_mask != 0, every launch of a selected
 * family is bracketed by CUDA events on its stream (clears previous records).
 * hy_ctx_kernel_times() synchronizes on those events and returns the summed
 * device time (ms), the launch count and the summed ALGORITHMIC bytes (the
 * minimal reads + writes of each launch) of the
 * families in family_mask. */
enum {
  HY_FAM_NTT_A = 1,     /* NTT pass over columns (stages with distance >= 256) */
  HY_FAM_NTT_B = 2,     /* NTT pass over 256-word rows */
  HY_FAM_MODUP = 4,     /* ModUp basis conversion */
  HY_FAM_IP = 8,        /* key-switch inner product */
  HY_FAM_MODDOWN = 16,  /* ModDown basis conversion + final combine */
  HY_FAM_AUT = 32,      /* automorphism gather */
  HY_FAM_ELEM = 64,     /* PMult / PMult-accumulate / add */
  HY_FAM_RESCALE = 128,
  HY_FAM_CLIENT = 256,  /* keygen / encrypt / decrypt / encode upload */
  HY_FAM_NTT_IP = 512   /* ModUp NTT row pass fused with the key-switch inner product */
};
hy_status hy_ctx_time_kernels(hy_ctx* ctx, uint32_t family_mask);
hy_status hy_ctx_kernel_times(hy_ctx* ctx, uint32_t family_mask, double* total_ms, uint64_t* n_launches,
                              uint64_t* alg_bytes);

/* ---- transforms (exposed for parity tests of the sub-steps) ------------ */
/* Negacyclic NTT / inverse NTT (P:97 ring; DESIGN R-NTT) of n_limbs limbs.
 * d_in/d_out: [n_limbs][N] device (may alias); chain[u] = chain index of limb u (host array). */
hy_status hy_ntt(hy_ctx* ctx, const uint64_t* d_in, uint64_t* d_out, const uint32_t* chain, uint32_t n_limbs,
                 int inverse, void* stream);
/* Automorphism X -> X^k in the NTT domain, same permutation on every limb.
 * k: odd Galois element.  d_in/d_out [n_limbs][N], must not alias. */
hy_status hy_automorph(hy_ctx* ctx, const uint64_t* d_in, uint64_t* d_out, uint32_t n_limbs, uint64_t k, void* stream);
/* PRot (SPEC prot): plaintext rotation by r slots, the automorphism kappa_{5^r} applied to the
 * NTT-domain plaintext d_pt [l+1][N] -> d_out (no key switch: the plaintext is public).  r = 0 copies.
 * Must not alias.  The conv layers fuse PRot into the PMult-accumulate as a gather instead (PRCR). */
hy_status hy_prot(hy_ctx* ctx, const uint64_t* d_pt, uint32_t level, int32_t r, uint64_t* d_out, void* stream);
/* Galois element of a left rotation by r slots: 5^(r mod n) mod 2N. */
uint64_t hy_galois_elt(const hy_ctx* ctx, int64_t r);

/* ---- key switching pieces (DESIGN R-MODUP, R-MODDOWN) ------ */
/* ModUp of one polynomial d given in the COEFFICIENT domain on q_0..q_l:
 * d_ext out [beta][l+1+K][N] NTT domain; limbs of digit j's own primes are
 * NTT(d) (fast basis conversion without correction elsewhere). */
hy_status hy_modup(hy_ctx* ctx, uint32_t level, const uint64_t* d_coeff, uint64_t* d_ext, void* stream);
/* u[c][t] = sum_j ext[j][t] * evk[j][c][chain(t)]  ([2][l+1+K][N] out; d_evk packed, see Conventions). */
hy_status hy_ks_inner_product(hy_ctx* ctx, uint32_t level, const uint64_t* d_ext, const uint64_t* d_evk,
                              uint64_t* d_u, void* stream);
/* ModDown of one polynomial [l+1+K][N] -> [l+1][N] (both NTT domain). */
hy_status hy_moddown(hy_ctx* ctx, uint32_t level, const uint64_t* d_u, uint64_t* d_out, void* stream);

/* ---- HRot: rotate LEFT by r slots, three variants (DESIGN R-HROT) - */
/* plain: ModUp(kappa(c1)).  r = 0 (mod n) copies the input. */
hy_status hy_hrot(hy_ctx* ctx, const uint64_t* d_evk, const uint64_t* d_ct, uint32_t level, int32_t r,
                  uint64_t* d_out, void* stream);
/* non-hoisted batch: out_i = HRot_{r_i}(ct_i) with key evk_i (host arrays of device pointers).  No output may
 * overlap any input of the batch (the items run in key-switch chunks and r = 0 items are copied first):
 * HY_E_ARG.  Items sharing a key pointer stream it from HBM once per chunk. */
hy_status hy_hrot_batch(hy_ctx* ctx, const uint64_t* const* d_evks, const uint64_t* const* d_cts, uint32_t level,
                        const int32_t* r, uint32_t n, uint64_t* const* d_outs, void* stream);
/* Key switch by any Galois element k (odd, < 2N): out = kappa_k(ct) switched back to s with the key from
 * hy_keygen_galois(k) -- k = 2N - 1 is the conjugation bootstrapping needs; k = 1 copies.  Plain variant,
 * not in place. */
hy_status hy_hrot_galois(hy_ctx* ctx, const uint64_t* d_evk, const uint64_t* d_ct, uint32_t level, uint64_t k,
                         uint64_t* d_out, void* stream);
/* hoisted (Slide_f): one ModUp of c1 shared by n rotations of the same ciphertext. */
hy_status hy_hrot_hoisted(hy_ctx* ctx, const uint64_t* const* d_evks, const uint64_t* d_ct, uint32_t level,
                          const int32_t* r, uint32_t n, uint64_t* const* d_outs, void* stream);
/* lazy sum (Slide_1&Sum_f of reordered RAConv): sum_t HRot_{r_t}(ct_t) with the key-switch
 * inner products accumulated over Q_l u P and ONE ModDown; r_t = 0 terms are added without switching
 * (their evk pointer may be NULL). */
hy_status hy_hrot_sum(hy_ctx* ctx, const uint64_t* const* d_evks, const uint64_t* const* d_cts, uint32_t level,
                      const int32_t* r, uint32_t n, uint64_t* d_out, void* stream);

/* ---- MulCt with relinearization (AESPA square activation P:1013-1015) ---- */
/* out = MulCt(a, b) at level l: the tensor product (a0 b0, a0 b1 + a1 b0, a1 b1), whose last part is
 * key-switched from s^2 to s with the relinearization key d_rlk (hy_keygen_relin) through the same
 * hybrid key switch as HRot (ModUp, inner product, ModDown; DESIGN R-RELIN).  No rescale (the caller
 * rescales); the scale is scale_a * scale_b.  Layouts as hy_hrot; out_i may alias a_i or b_i (the
 * square is hy_mulct(a, a)) but not another item's inputs.  Batched: the key streams once per batch. */
hy_status hy_mulct(hy_ctx* ctx, const uint64_t* d_rlk, const uint64_t* d_a, const uint64_t* d_b, uint32_t level,
                   uint64_t* d_out, void* stream);
hy_status hy_mulct_batch(hy_ctx* ctx, const uint64_t* d_rlk, const uint64_t* const* d_as,
                         const uint64_t* const* d_bs, uint32_t level, uint32_t n, uint64_t* const* d_outs,
                         void* stream);

/* ---- MulPt / AddCt / Rescale -------------------------------- */
/* out = ct (.) pt limbwise; no auto-rescale (scale bookkeeping is the caller's). */
hy_status hy_pmult(hy_ctx* ctx, const uint64_t* d_ct, const uint64_t* d_pt, uint32_t level, uint64_t* d_out,
                   void* stream);
/* MulFilter&Sum: out (+)= sum_i ct_i (.) pt_i, one reduction per output word.
 * accumulate != 0 adds into d_out. */
/* out_i = ct_i (.) pt for n ciphertexts and ONE plaintext in one launch (each bit-identical to hy_pmult; used by
 * bootstrapping's lockstep EvalMod).  out_i may alias ct_i, not another item's input (HY_E_ARG). */
hy_status hy_pmult_batch(hy_ctx* ctx, const uint64_t* const* d_cts, uint32_t n, const uint64_t* d_pt, uint32_t level,
                         uint64_t* const* d_outs, void* stream);
hy_status hy_pmult_acc(hy_ctx* ctx, const uint64_t* const* d_cts, const uint64_t* const* d_pts, uint32_t n,
                       uint32_t level, uint64_t* d_out, int accumulate, void* stream);
/* out = a + b over npoly polynomials ([npoly][l+1][N]); in-place allowed. */
hy_status hy_add(hy_ctx* ctx, const uint64_t* d_a, const uint64_t* d_b, uint32_t npoly, uint32_t level,
                 uint64_t* d_out, void* stream);
/* out = a - b over npoly polynomials (mod q_i limbwise); in-place allowed. */
hy_status hy_sub(hy_ctx* ctx, const uint64_t* d_a, const uint64_t* d_b, uint32_t npoly, uint32_t level,
                 uint64_t* d_out, void* stream);
/* AddPt ("AddPt 0.169 ms" P:148; the conv bias): out = (c0 + pt, c1) at level l, [2][l+1][N] and
 * [l+1][N]; in-place allowed (out == ct).  The scales are the caller's bookkeeping (the ABI carries none): they
 * must agree to 2^-30 relative, else HY_E_SCALE_MISMATCH (SPEC add_ct / add_pt); the output has ct_scale. */
hy_status hy_add_pt(hy_ctx* ctx, const uint64_t* d_ct, double ct_scale, const uint64_t* d_pt, double pt_scale,
                    uint32_t level, uint64_t* d_out, void* stream);
/* Level alignment (SPEC level_down; P:102-112 levels): [2][l+1][N] -> [2][l'+1][N], l' <= l, by dropping the
 * limbs above l' (reduction mod Q_l'); scale unchanged, no rounding.  out must not alias ct unless l' == l.
 * Errors: HY_E_ARG, HY_E_LEVEL_MISMATCH (l' > l). */
hy_status hy_level_down(hy_ctx* ctx, const uint64_t* d_ct, uint32_t level, uint32_t new_level, uint64_t* d_out,
                        void* stream);
/* Rescale (DESIGN R-RESCALE): [2][l+1][N] -> [2][l][N], exact round(c/q_l). */
hy_status hy_rescale(hy_ctx* ctx, const uint64_t* d_ct, uint32_t level, uint64_t* d_out, void* stream);
/* Rescale of n ciphertexts at the same level in batched launches (each output bit-identical to hy_rescale of its
 * input; used by bootstrapping's lockstep EvalMod).  Errors: HY_E_ARG (null, an output aliasing any input),
 * HY_E_LEVEL_EXHAUSTED (l = 0), HY_E_WORKSPACE. */
hy_status hy_rescale_batch(hy_ctx* ctx, const uint64_t* const* d_cts, uint32_t n, uint32_t level,
                           uint64_t* const* d_outs, void* stream);

/* ---- HyPHEN convolution layers ------------------------------- */
/* Slot layout (DESIGN R-LAYOUT): physical width wp (power of two), gap g, cell kappa in
 * [0, m d) with digits (g_c, g_r, e_idx) at slot offsets (1, wp, wp^2), e = m d / g^2 image
 * sub-blocks per channel block of B = e wp^2 slots, c_n = (N/2) / B blocks.
 *   CA(m, d) (pi_CA): C_g index mu = kappa % m, R_g index rho = kappa / m;
 *            ciphertext i holds channel i c_n m + b m + mu in block b.
 *   RA(m, d) (pi_RA): mu = kappa / d, rho = kappa % d; ciphertext i holds channel
 *            i m + mu, replicated in every block (R_a) and every rho (R_g).
 * CAConv maps CA(m, d) -> RA(d, m) (stride 1) or RA(2d, 2m) at gap 2g (stride 2, needs m = g;
 * DESIGN R-DSCONV); RAConv (reordered) maps RA(m, d) -> CA(d, m), stride 1. */
typedef enum { HY_CONV_CA = 0, HY_CONV_RA = 1 } hy_conv_algo;
typedef struct {
  uint32_t ci, co;   /* input / output channels */
  uint32_t w;        /* input image width = height (logical pixels) */
  uint32_t f;        /* odd filter width, zero padding (f-1)/2 (Fig. 2(a)) */
  uint32_t stride;   /* 1, or 2 for CAConv */
  uint32_t wp;       /* physical width W_p >= w * gap */
  uint32_t gap;      /* input gap g */
  uint32_t m, d;     /* |C_g|, |R_g| of the INPUT format */
  uint32_t algo;     /* hy_conv_algo */
  uint32_t segments; /* PRCR |S|; 0 or 1 = off.  With S > 1 (DESIGN R-PRCR): the CA side
                        is pi_CA' -- ciphertexts in families of S, member im holding at global row
                        segment G (F = wp^2/S slots) rows of channel k c_n S m + ((G + im) mod c_n S) m + mu;
                        one weight plaintext per family, used as PRot(P, shift); needs S | wp/gap,
                        e = 1, stride 1, wp/gap >= w + (f-1)/2; adds an output-valid mask step. */
  uint32_t bias;     /* 1: the layer adds a per-output-channel bias b (Y = conv2d(X, K) + b; BN biases fused into
                        the conv): AddPt of the output format's packing of b after the layer's last
                        rescale, at the output level and scale (DESIGN R-BIAS). 0 = none. */
} hy_conv_spec;
typedef struct hy_conv_plan hy_conv_plan;
/* Rotation amounts, weight/mask plaintext contents and counts for one layer.  Errors:
 * HY_E_SHAPE (bad sizes), HY_E_FORMAT (non power of two, m d % g^2, unsupported stride-2
 * layout), HY_E_CAPACITY (image or block does not fit the N/2 slots). */
hy_status hy_conv_plan_create(uint32_t log_n, const hy_conv_spec* spec, hy_conv_plan** out); /* host only */
void hy_conv_plan_destroy(hy_conv_plan* plan);
/* n_in / n_out ciphertexts, n_pt weight plaintexts (+1 mask plaintext when has_mask),
 * n_rot distinct nonzero rotation amounts mod N/2 in ascending order (rots: n_rot entries,
 * the order keys are passed in), counts[5] = Slide, RaS, RaS_g, IR_g rotations and PMults
 * of the whole layer (table 'Cost of homomorphic convolutions').  Any output
 * pointer may be NULL. */
hy_status hy_conv_plan_query(const hy_conv_plan* plan, uint32_t* n_in, uint32_t* n_out, uint32_t* n_pt,
                             uint32_t* has_mask, uint32_t* n_rot, int32_t* rots, uint32_t* counts);
/* ---- limited rotation-key sets ("frequently used rotation keys for Slide are loaded ... other
 * irregular rotation keys used in IR are not loaded; instead, these rotation indices are synthesized using the
 * already loaded key indices"; DESIGN R-KEYSET).  A key set is a list of loaded rotation amounts (taken mod N/2).
 * An amount r that is not loaded is synthesized as the shortest sequence of loaded amounts summing to r mod N/2
 * (HRot_{a+b} = HRot_a o HRot_b, one key switch per step): breadth-first search from 0 over Z_{N/2} with the
 * loaded amounts as edges in ascending order and a FIFO queue, the first discovery fixing a node's parent.
 * Host only. */
typedef struct hy_keyset hy_keyset;
hy_status hy_keyset_create(uint32_t log_n, const int32_t* amounts, uint32_t n_amounts, hy_keyset** out);
void hy_keyset_destroy(hy_keyset* keyset);
/* steps (application order, each a loaded amount in [1, N/2)) of amount r; r = 0 -> 0 steps; a loaded r -> 1 step
 * (r itself).  steps may be NULL (count only).  Errors: HY_E_MISSING_KEY (r unreachable), HY_E_ARG. */
hy_status hy_keyset_decompose(const hy_keyset* keyset, int32_t r, int32_t* steps, uint32_t max_steps,
                              uint32_t* n_steps);
/* Restrict a conv plan to a key set (NULL: every key the plan needs, the default): its Slide amounts must be loaded
 * (HY_E_MISSING_KEY otherwise: they are hoisted); every other amount not loaded is synthesized.  Afterwards
 * hy_conv_plan_query reports the loaded amounts the layer uses (the keys hy_caconv / hy_raconv take) and
 * hy_conv_scratch_words the larger scratch; hy_conv_plan_eff_counts gives counts[5] with each synthesized rotation
 * counted once per step ("eff. total"). */
hy_status hy_conv_plan_set_keyset(hy_conv_plan* plan, const hy_keyset* keyset);
hy_status hy_conv_plan_eff_counts(const hy_conv_plan* plan, uint32_t* counts);
/* Slot values (host, N/2 doubles) of weight plaintext idx < n_pt, or of the mask (idx == n_pt).
 * K: host [co][ci][f][f] float64. */
hy_status hy_conv_weight_slots(const hy_conv_plan* plan, const double* K, uint32_t idx, double* slots);
/* Slot values (host, N/2 doubles) of the bias plaintext of output ciphertext out_index < n_out: b[c] at every
 * valid slot of output channel c in the output format (every replica), 0 elsewhere.  bias: host [co]. */
hy_status hy_conv_bias_slots(const hy_conv_plan* plan, const double* bias, uint32_t out_index, double* slots);
/* Device words of the encoded weights at input level l: n_pt x [l+1][N], then the mask [l][N] (has_mask), then
 * (spec.bias) n_out bias plaintexts [l_out+1][N] at the output level l_out = l - 1 - has_mask. */
size_t hy_conv_weight_words(const hy_ctx* ctx, const hy_conv_plan* plan, uint32_t level);
/* Device scratch words hy_caconv / hy_raconv need at input level l. */
size_t hy_conv_scratch_words(const hy_ctx* ctx, const hy_conv_plan* plan, uint32_t level);
/* Encode every weight plaintext at scale q_l (level l) and the mask at scale q_{l-1} (level
 * l-1), so each rescale returns the ciphertext scale exactly (DESIGN R-SCALE); with spec.bias, the n_out bias
 * plaintexts at level l_out and scale bias_scale (the exact integer scale of the layer's input ciphertexts, which
 * every rescale returns to).  K: host [co][ci][f][f]; bias: host [co] (NULL iff spec.bias == 0).
 * Errors: HY_E_ARG (null, bias missing), HY_E_LEVEL_EXHAUSTED, HY_E_PLAN, HY_E_WORKSPACE. */
hy_status hy_conv_encode_weights(hy_ctx* ctx, const hy_conv_plan* plan, const double* K, const double* bias,
                                 uint64_t bias_scale, uint32_t level, uint64_t* d_pts, void* stream);
/* Run the layer on n_in input ciphertexts at level l, producing outputs [out_begin, out_end)
 * (the multi-GPU shard) at level l - 1 - has_mask (plus the bias AddPt when spec.bias).  d_evks: one key per rotation amount in
 * hy_conv_plan_query order.  Outputs must not alias inputs.  HY_E_PLAN when the plan's algo
 * does not match the call. */
hy_status hy_caconv(hy_ctx* ctx, const hy_conv_plan* plan, const uint64_t* const* d_evks,
                    const uint64_t* const* d_in, uint32_t level, const uint64_t* d_pts, uint64_t* d_scratch,
                    uint32_t out_begin, uint32_t out_end, uint64_t* const* d_out, void* stream);
hy_status hy_raconv(hy_ctx* ctx, const hy_conv_plan* plan, const uint64_t* const* d_evks,
                    const uint64_t* const* d_in, uint32_t level, const uint64_t* d_pts, uint64_t* d_scratch,
                    uint32_t out_begin, uint32_t out_end, uint64_t* const* d_out, void* stream);
/* CAConv Slide sharding (multi-GPU): Slide_f is the part of a CAConv every output
 * needs, so output-sharded ranks would all repeat it.  hy_caconv_slide runs the hoisted Slide of inputs
 * [in_begin, in_end) into d_slid: ciphertext (i - in_begin) * f^2 + t at level l ([2][l+1][N] each, the identity
 * tap a copy of the input); ranks slide disjoint input ranges and all-gather the buffers, and hy_caconv_slid runs
 * the rest of the layer (MulFilter&Sum, rescale, RaS, IR, bias) for outputs [out_begin, out_end) from the complete
 * slid buffer [n_in][f^2] -- bit-identical to hy_caconv.  Errors as hy_caconv. */
hy_status hy_caconv_slide(hy_ctx* ctx, const hy_conv_plan* plan, const uint64_t* const* d_evks,
                          const uint64_t* const* d_in, uint32_t level, uint32_t in_begin, uint32_t in_end,
                          uint64_t* d_slid, void* stream);
hy_status hy_caconv_slid(hy_ctx* ctx, const hy_conv_plan* plan, const uint64_t* const* d_evks, const uint64_t* d_slid,
                         uint32_t level, const uint64_t* d_pts, uint64_t* d_scratch, uint32_t out_begin,
                         uint32_t out_end, uint64_t* const* d_out, void* stream);
/* RAConv tap sharding: the multi-GPU exchange step for layers with fewer outputs than GPUs (ResNet-20
 * RAConv has one output ciphertext).  An output of RAConv_Reorder is
 * sum_t HRot_{r_t}(acc_t) over the f^2 taps with ONE ModDown (Alg. P:727-733).  hy_raconv_partial
 * computes, for output out_index and taps [tap_begin, tap_end), the state before that ModDown into
 * d_state (hy_raconv_partial_words words, caller-allocated):
 *   [2][l+1+K][N]  sum of the taps' key-switch inner products over Q_l u P (NTT domain, canonical),
 *   [2][l+1][N]    (sum_t kappa_t(c0_t), the centre tap's c1) -- canonical.
 * States of disjoint tap ranges may be added as unsigned 64-bit integers (e.g. an int64 all-reduce SUM
 * over ranks; every word stays below ranks * 2^48); hy_raconv_finish reduces the sum mod q, runs the
 * ModDown, rescale, RaS_g and IR_g (in place on d_state and d_scratch) and writes output out_index at
 * level l - 1 - has_mask, bit-identical to hy_raconv.  An empty tap range yields an all-zero state.
 * Errors: HY_E_PLAN (not an RAConv plan, index or tap range outside the plan), HY_E_LEVEL_EXHAUSTED,
 * HY_E_MISSING_KEY, HY_E_WORKSPACE. */
size_t hy_raconv_partial_words(const hy_ctx* ctx, uint32_t level);
hy_status hy_raconv_partial(hy_ctx* ctx, const hy_conv_plan* plan, const uint64_t* const* d_evks,
                            const uint64_t* const* d_in, uint32_t level, const uint64_t* d_pts, uint64_t* d_scratch,
                            uint32_t out_index, uint32_t tap_begin, uint32_t tap_end, uint64_t* d_state,
                            void* stream);
hy_status hy_raconv_finish(hy_ctx* ctx, const hy_conv_plan* plan, const uint64_t* const* d_evks, uint32_t level,
                           const uint64_t* d_pts, uint64_t* d_state, uint64_t* d_scratch, uint32_t out_index,
                           uint64_t* d_out, void* stream);

/* ---- the linear steps of bootstrapping (partial; DESIGN R-LINTRANS) --
 * ModRaise: a ciphertext at level 0 [2][1][N] -> level l [2][l+1][N]: each coefficient's centred representative mod
 * q_0 reduced mod q_0..q_l (NTT domain in and out); it then decrypts to m + q_0 I with a small integer polynomial I.
 * Must not alias.  Errors: HY_E_ARG, HY_E_WORKSPACE. */
hy_status hy_mod_raise(hy_ctx* ctx, const uint64_t* d_ct0, uint32_t level, uint64_t* d_out, void* stream);
/* Homomorphic diagonal linear transform y = M x on the slots (CoeffToSlot / SlotToCoeff are such transforms):
 * y = sum_{d in D} diag_d (.) Rot_d(x), diag_d[j] = M[j][(j + d) mod n], evaluated baby-step / giant-step with
 * baby-step size bs: d = g bs + b, y = sum_g Rot_{g bs}(sum_b Rot_{-g bs}(diag_{g bs + b}) (.) Rot_b(x)) -- the baby
 * steps as one hoisted HRot batch, the inner sums as MulFilter&Sum blocks, the giant steps as one lazy HRotSum, then
 * a rescale (plaintexts at scale q_l: level l -> l - 1, scale unchanged).  A plan lists its diagonals D (amounts
 * mod n = N/2); query reports the plaintext count (|D| + one zero plaintext), baby / giant step counts and the key
 * amounts in ascending order (the order apply takes keys in).  encode: host complex diagonals re/im [|D|][n] in
 * ascending canonical d order (im may be NULL) -> d_pts (hy_lintrans_pt_words).  apply: ct at level l >= 1 -> out at
 * level l - 1, scratch hy_lintrans_scratch_words.  Errors: HY_E_ARG, HY_E_LEVEL_EXHAUSTED, HY_E_PLAN,
 * HY_E_MISSING_KEY. */
typedef struct hy_lintrans hy_lintrans;
hy_status hy_lintrans_create(uint32_t log_n, const int32_t* diags, uint32_t n_diag, uint32_t bs, hy_lintrans** out);
void hy_lintrans_destroy(hy_lintrans* plan);
hy_status hy_lintrans_query(const hy_lintrans* plan, uint32_t* n_pt, uint32_t* n_baby, uint32_t* n_giant,
                            uint32_t* n_rot, int32_t* rots);
size_t hy_lintrans_pt_words(const hy_ctx* ctx, const hy_lintrans* plan, uint32_t level);
size_t hy_lintrans_scratch_words(const hy_ctx* ctx, const hy_lintrans* plan, uint32_t level);
hy_status hy_lintrans_encode(hy_ctx* ctx, const hy_lintrans* plan, const double* h_re, const double* h_im,
                             uint32_t level, uint64_t* d_pts, void* stream);
hy_status hy_lintrans_apply(hy_ctx* ctx, const hy_lintrans* plan, const uint64_t* const* d_evks, const uint64_t* d_ct,
                            uint32_t level, const uint64_t* d_pts, uint64_t* d_scratch, uint64_t* d_out, void* stream);

/* ---- client side: keys, encode, encrypt, decrypt (untimed) ------- */
/* Rotation key for Galois element of a left rotation by r (DESIGN R-EVK, R-PRNG):
 * secret from sk_seed, randomness from ek_seed.  d_evk: [dnum][2][n_q+n_p][N]. */
hy_status hy_keygen_rot(hy_ctx* ctx, uint64_t sk_seed, uint64_t ek_seed, int32_t r, uint64_t* d_evk, void* stream);
/* uint64 words of one packed key (see Conventions): dnum * 2 * (n_q+n_p) * 3N/4. */
size_t hy_evk_words(const hy_ctx* ctx);
/* d_in [dnum][2][n_q+n_p][N] (one uint64 per word, each < 2^48) -> packed d_out (hy_evk_words), and back.
 * Device buffers, must not alias; stream-ordered. */
hy_status hy_evk_pack(hy_ctx* ctx, const uint64_t* d_in, uint64_t* d_out, void* stream);
hy_status hy_evk_unpack(hy_ctx* ctx, const uint64_t* d_in, uint64_t* d_out, void* stream);
/* 48-bit wire format for any residue array (ciphertexts, plaintexts; every residue < 2^48): n_words words
 * (a multiple of 4) <-> 6 bytes per word, word x at bytes [6x, 6x+6) little-endian (3 n_words / 4 uint64),
 * the layout of the packed keys.  A client that keeps ciphertexts in this form moves 25 % fewer bytes over
 * PCIe.  Device buffers, must not alias; stream-ordered.  Errors: HY_E_ARG (null, n_words % 4 != 0). */
hy_status hy_pack48(hy_ctx* ctx, const uint64_t* d_in, uint64_t* d_out, size_t n_words, void* stream);
hy_status hy_unpack48(hy_ctx* ctx, const uint64_t* d_in, uint64_t* d_out, size_t n_words, void* stream);
hy_status hy_keygen_galois(hy_ctx* ctx, uint64_t sk_seed, uint64_t ek_seed, uint64_t k, uint64_t* d_evk, void* stream);
/* Relinearization key s^2 -> s (DESIGN R-RELIN): b_j = -a_j s + e_j + g_j s^2, object ids j (Galois
 * element 0, used by no rotation); layout as a rotation key. */
hy_status hy_keygen_relin(hy_ctx* ctx, uint64_t sk_seed, uint64_t ek_seed, uint64_t* d_rlk, void* stream);
/* Secret-key encryption of an NTT-domain plaintext at level l (DESIGN R-ENC). */
hy_status hy_encrypt(hy_ctx* ctx, uint64_t sk_seed, uint64_t enc_seed, uint64_t ct_id, const uint64_t* d_pt,
                     uint32_t level, uint64_t* d_ct, void* stream);
/* m = c0 + c1*s (NTT domain). */
hy_status hy_decrypt(hy_ctx* ctx, uint64_t sk_seed, const uint64_t* d_ct, uint32_t level, uint64_t* d_pt,
                     void* stream);
/* CKKS encode of n_slots <= N/2 real values (DESIGN R-ENCODE): exact integer scale,
 * coefficients = round(scale * tau^{-1}(z)) computed in double-double precision,
 * then reduced mod q_0..q_l and NTT'd into d_pt [l+1][N].  Synchronous w.r.t. the host buffer. */
hy_status hy_encode(hy_ctx* ctx, const double* h_slots, uint32_t n_slots, uint64_t scale, uint32_t level,
                    uint64_t* d_pt, void* stream);
/* Batched device CKKS encoding (same rounding as hy_encode, DESIGN R-ENCODE; the bulk weight path of
 * hy_conv_encode_weights): P real slot vectors h_slots [P][N/2] (host) at integer scale -> NTT-domain
 * plaintexts d_pts [P][l+1][N].  Double-double special FFT on the device; synchronous w.r.t. the host buffer.
 * Errors: HY_E_ARG, HY_E_WORKSPACE, HY_E_CAPACITY (a coefficient >= 2^62). */
hy_status hy_encode_batch(hy_ctx* ctx, const double* h_slots, uint32_t P, uint64_t scale, uint32_t level,
                          uint64_t* d_pts, void* stream);
/* Host-only part of hy_encode: the N integer coefficients (no device needed). */
hy_status hy_encode_coeffs(uint32_t log_n, const double* h_slots, uint32_t n_slots, uint64_t scale,
                           int64_t* h_coeffs);
/* The same for complex slots z_j = slots[j] + i slots_im[j] (slots_im may be NULL): m_k = round(scale (2/N) Re
 * sum_j z_j zeta^{-5^j k}) -- R-ENCODE with complex values (the bootstrapping linear transforms' diagonals). */
hy_status hy_encode_coeffs_complex(uint32_t log_n, const double* h_slots, const double* h_slots_im, uint32_t n_slots,
                                   uint64_t scale, int64_t* h_coeffs);
/* Signed integer coefficients (host, N words) -> NTT-domain plaintext on q_0..q_l. */
hy_status hy_pt_from_coeffs(hy_ctx* ctx, const int64_t* h_coeffs, uint32_t level, uint64_t* d_pt, void* stream);
/* CKKS decode (client side, the inverse of R-ENCODE; P:98-100 canonical embedding):
 * z_j = m(zeta^{5^j}) / scale for j < n_slots, zeta = exp(i pi / N), where m is the centred CRT lift of the
 * NTT-domain plaintext d_pt [l+1][N] (as hy_decrypt returns it) to (-Q_l/2, Q_l/2].  h_re / h_im: host,
 * n_slots doubles each (h_im may be NULL).  Synchronous (one device iNTT, then host CRT + special FFT).
 * A floating-point result: its contract is a tolerance, not bit-exactness.
 * Errors: HY_E_ARG (null, level, scale <= 0), HY_E_CAPACITY (n_slots > N/2), HY_E_WORKSPACE. */
hy_status hy_decode(hy_ctx* ctx, const uint64_t* d_pt, uint32_t level, double scale, uint32_t n_slots,
                    double* h_re, double* h_im, void* stream);
/* Coefficient-domain wire format (parity dumps independent of the NTT order): n_limbs limbs
 * [n_limbs][N], limb u on chain index chain[u] (host array; q_0.. then p_0..).  Export: NTT-domain device limbs
 * -> coefficient-domain host limbs in [0, q) (an inverse NTT on the device into the workspace, then a copy;
 * synchronous).  Import: the reverse (host coefficients in [0, q) -> NTT-domain device limbs).  Errors: HY_E_ARG
 * (null, chain index >= n_q + n_p, import word >= its modulus), HY_E_WORKSPACE. */
hy_status hy_export_coeff(hy_ctx* ctx, const uint64_t* d_ntt, const uint32_t* chain, uint32_t n_limbs,
                          uint64_t* h_coeff, void* stream);
hy_status hy_import_coeff(hy_ctx* ctx, const uint64_t* h_coeff, const uint32_t* chain, uint32_t n_limbs,
                          uint64_t* d_ntt, void* stream);
/* Host-only part of hy_decode: real coefficients (host, N doubles) -> slots. */
hy_status hy_decode_coeffs(uint32_t log_n, const double* h_coeffs, double scale, uint32_t n_slots, double* h_re,
                           double* h_im);

#ifdef __cplusplus
}
#endif
#endif /* HYPHEN_H_ */
