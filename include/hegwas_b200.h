/*
 * hegwas_b200.h -- C-ABI of the B200 (sm_100a) evaluator for the power-of-two-modulus
 * approximate HE scheme of arXiv 1902.04303 (reference package `hegwas`).
 *
 * Every entry point takes plain device pointers, sizes and a cudaStream_t passed as
 * void*.  No torch types cross this boundary.  The Python host layer
 * (paper_1902_04303_b200/) binds these with ctypes; a maintainer of the reference would
 * bind the same symbols.
 *
 * Polynomial layout ("limb-major"): a ring element of Z_{2^bits}[x]/(x^N+1) is stored as
 * W = ceil(bits/32) arrays of N uint32 words, word w of coefficient j at p[w*N + j]
 * (little-endian radix 2^32).  Canonical representatives are in [0, 2^bits) with the
 * top word masked, exactly like ring.RingElement (reference ring.py:68-85).
 *
 * An operand descriptor (hg_operand) additionally says how to read the value:
 *   signed_rep = 0 : unsigned integer of `bits` bits (canonical residue),
 *   signed_rep = 1 : two's complement integer of `bits` bits (centered representative).
 * Products mod 2^k do not depend on the representative when k <= bits of the operand
 * (SURVEY §8a R3), so the host picks the narrowest legal view.
 *
 * Status codes: 0 = HG_OK, otherwise an HG_E* value; hg_last_error() returns a
 * thread-local message.  The library never silently falls back to the CPU.
 */
#ifndef HEGWAS_B200_H
#define HEGWAS_B200_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HG_OK 0
#define HG_EINVAL 1      /* bad argument (maps to ParameterError on the Python side) */
#define HG_ENOMEM 2      /* device allocation failed */
#define HG_ECUDA 3       /* CUDA runtime error */
#define HG_ERANGE 4      /* product too wide for the NTT prime basis */

typedef struct hg_ctx hg_ctx;
typedef struct hg_key hg_key;

typedef struct hg_operand {
    const uint32_t* words;  /* device pointer, [W][N] */
    int32_t bits;           /* value width (W = ceil(bits/32) words are read) */
    int32_t signed_rep;     /* 0 unsigned, 1 two's complement */
} hg_operand;

/* ---- library / context ------------------------------------------------------------ */
const char* hg_last_error(void);
int hg_version(void);
/* Context for ring degree N = 2^log_n (2 <= log_n <= 17): NTT prime basis
 * (30-bit primes p = 1 mod 2^18), twiddles, base-conversion tables.  Replaces the
 * implicit CPython/gmpy2 big-int engine behind ring.negacyclic_mul (ring.py:61-65). */
int hg_ctx_create(int log_n, int device, hg_ctx** out);
int hg_ctx_destroy(hg_ctx* ctx);
/* Largest exact product width (bits) the prime basis supports. */
int hg_ctx_max_product_bits(const hg_ctx* ctx);
int hg_ctx_num_primes(const hg_ctx* ctx);
/* Copy the prime list (host array of length hg_ctx_num_primes). */
int hg_ctx_primes(const hg_ctx* ctx, uint32_t* out);
int hg_sync(hg_ctx* ctx, void* stream);

/* ---- elementwise ring ops (ring.py:114-196) ---------------------------------------- */
/* out = a + b mod 2^bits                                     RingElement.add  ring.py:114 */
int hg_poly_add(hg_ctx* ctx, uint32_t* out, const uint32_t* a, const uint32_t* b,
                int bits, void* stream);
/* out = a - b mod 2^bits                                     RingElement.sub  ring.py:123 */
int hg_poly_sub(hg_ctx* ctx, uint32_t* out, const uint32_t* a, const uint32_t* b,
                int bits, void* stream);
/* out = sum_k terms[k] mod 2^bits; `terms` is a HOST array of `count` device pointers.
 * One pass over the terms (the sum of matrix.py's Sum_i mult(...) loops, e.g. cp_rep_matmul
 * matrix.py:173-193, instead of count-1 pairwise adds); exact, so order-independent.    */
int hg_poly_sum(hg_ctx* ctx, uint32_t* out, const uint32_t* const* terms, int count, int bits,
                void* stream);
/* out = -a mod 2^bits                                        RingElement.neg  ring.py:132 */
int hg_poly_neg(hg_ctx* ctx, uint32_t* out, const uint32_t* a, int bits, void* stream);
/* out = a * k mod 2^bits; k given as (k mod 2^bits) in kw host words (kw <= W)
 *                                                     RingElement.scalar_mul  ring.py:136 */
int hg_poly_scalar_mul(hg_ctx* ctx, uint32_t* out, const uint32_t* a, int bits,
                       const uint32_t* k_words_host, int kw, void* stream);
/* out (out_bits) = a mod 2^out_bits, a has in_bits >= out_bits  RingElement.reduce_to  ring.py:168 */
int hg_poly_reduce_to(hg_ctx* ctx, uint32_t* out, int out_bits, const uint32_t* a,
                      int in_bits, void* stream);
/* out (out_bits) = centered(a) mod 2^out_bits (sign-extend)  lift_centered_to  ring.py:177 */
int hg_poly_lift_centered(hg_ctx* ctx, uint32_t* out, int out_bits, const uint32_t* a,
                          int in_bits, void* stream);
/* out (out_bits) = ((a + 2^(shift-1)) >> shift) mod 2^out_bits   divide_round  ring.py:184 */
int hg_poly_divide_round(hg_ctx* ctx, uint32_t* out, int out_bits, const uint32_t* a,
                         int in_bits, int shift, void* stream);
/* out = a(x^k) mod (x^N+1), k odd                       RingElement.automorphism  ring.py:152 */
int hg_poly_automorphism(hg_ctx* ctx, uint32_t* out, const uint32_t* a, int bits,
                         int64_t k, void* stream);

/* out[i] = float(centered(a_i) >> s) as Python's float(int) rounds it (nearest, ties to even),
 * s = bitlen(max_i |centered(a_i)|) - 500 if that exceeds 960 else 0; aux is a device int[2]
 * that receives (max bit length, s).  The coefficient -> float64 step of decode
 * (encoding.py:93-105, 108-115; the caller applies the multiplier 2^min(s,300)).         */
int hg_poly_to_double(hg_ctx* ctx, double* out, int* aux, const uint32_t* a, int bits,
                      void* stream);

/* ---- exact negacyclic product ------------------------------------------------------ */
/* out (out_bits) = (a * b) mod 2^out_bits, exact negacyclic convolution of the two
 * operand values.  Replaces RingElement.mul / mul_mod (ring.py:140-150), i.e.
 * negacyclic_mul + mask (ring.py:46-65).                                               */
int hg_poly_mul(hg_ctx* ctx, uint32_t* out, int out_bits, hg_operand a, hg_operand b,
                void* stream);
/* Same, for the ciphertext tensor of ckks.mult (ckks.py:176-178):
 *   d0 = a0*b0, d1 = a0*b1 + a1*b0, d2 = a1*b1   (all mod 2^out_bits).               */
int hg_poly_tensor(hg_ctx* ctx, uint32_t* d0, uint32_t* d1, uint32_t* d2, int out_bits,
                   hg_operand a0, hg_operand a1, hg_operand b0, hg_operand b1, void* stream);

/* ---- key switching (ckks._keyswitch, ckks.py:187-194) ------------------------------ */
/* Prepare a switching key (b, a) (device, key_bits each) for inputs at `level`:
 * reduce to level+big_l bits, convert to the NTT/RNS domain and keep it resident. */
int hg_key_prepare(hg_ctx* ctx, const uint32_t* kb, const uint32_t* ka, int key_bits,
                   int level, int big_l, void* stream, hg_key** out);
int hg_key_destroy(hg_key* key);
/* Stream-ordered destroy: the key's device memory is reused only after the work queued on
 * `stream` so far has completed (no host synchronisation, unlike hg_key_destroy). */
int hg_key_release(hg_key* key, void* stream);
size_t hg_key_device_bytes(const hg_key* key);
/* (out0, out1) = (round(x*kb / 2^L), round(x*ka / 2^L)) mod 2^level, x canonical
 * (level bits).  If automorph_k != 1, x is first mapped by x -> x(X^k) (fused
 * _apply_automorphism, ckks.py:247-253).                                                */
int hg_keyswitch(hg_ctx* ctx, const hg_key* key, const uint32_t* x, int64_t automorph_k,
                 uint32_t* out0, uint32_t* out1, void* stream);

/* ---- fused scheme ops --------------------------------------------------------------- */
/* HeEngine.mult (ckks.py:310-313): tensor, relinearise with evk prepared at `level`,
 * add, rescale by rescale_bits.  Inputs canonical at `level`; outputs at
 * level - rescale_bits.  (rescale_bits = 0 skips the rescale.)                         */
int hg_ct_mult(hg_ctx* ctx, const hg_key* evk, const uint32_t* a0, const uint32_t* a1,
               const uint32_t* b0, const uint32_t* b1, int level, int rescale_bits,
               uint32_t* out0, uint32_t* out1, void* stream);
/* Resident left operand for repeated products (the 245 duplicated projector columns of the
 * per-batch loop, gwas.py:310/325): forward-NTT residues of (c0, c1) at `level`, kept in HBM. */
typedef struct hg_ctprep hg_ctprep;
int hg_ct_prepare(hg_ctx* ctx, const uint32_t* c0, const uint32_t* c1, int level, void* stream,
                  hg_ctprep** out);
/* `count` independent hg_ct_mult_prepared products (a[i] (x) b_i -> out_i), up to four per group of
 * launches so rows of a prime share twiddle loads and the persistent kernels get twice the
 * work per launch; outputs identical to hg_ct_mult_prepared's.  Replaces the per-term
 * HeEngine.mult of cp_rep_matmul (matrix.py:173-193) over the 245 duplicated projector
 * columns. */
int hg_ct_mult_prepared_batch(hg_ctx* ctx, const hg_key* evk, int count, const hg_ctprep* const* a,
                              const uint32_t* const* b0s, const uint32_t* const* b1s, int level,
                              int rescale_bits, uint32_t* const* out0s, uint32_t* const* out1s,
                              void* stream);
/* `count` independent hg_ct_mult products (a_i (x) b_i, relinearised, rescaled by
 * rescale_bits), up to four per group of launches; outputs identical to hg_ct_mult's.  Replaces the
 * per-term HeEngine.mult of cp_matvec (matrix.py:99-106) and other independent products. */
int hg_ct_mult_batch(hg_ctx* ctx, const hg_key* evk, int count, const uint32_t* const* a0s,
                     const uint32_t* const* a1s, const uint32_t* const* b0s, const uint32_t* const* b1s,
                     int level, int rescale_bits, uint32_t* const* out0s, uint32_t* const* out1s,
                     void* stream);
/* As hg_ct_prepare, with the NTT basis widened for a sum of `terms` such products
 * (hg_ct_inner_prepared). */
int hg_ct_prepare_sum(hg_ctx* ctx, const uint32_t* c0, const uint32_t* c1, int level, int terms,
                      void* stream, hg_ctprep** out);
/* nq inner products over nb ciphertexts: out[q] = rescale(relinearise(sum_b a[q*nb+b] (x) b_b)),
 * i.e. sum_b HeEngine.mult without a relinearisation/rescale per term: the tensors are summed
 * exactly in the NTT domain (every b's forward residues computed once for all q), then one
 * inverse NTT, CRT and key switch (+ rescale by rescale_bits) per q.  The a operands must be
 * prepared at `level` with hg_ct_prepare_sum(..., terms >= nb).  No reference counterpart
 * (config-4 weighted sums, paper_1902_04303_b200/gwas_scale.py). */
int hg_ct_inner_prepared(hg_ctx* ctx, const hg_key* evk, int nq, int nb, const hg_ctprep* const* a,
                         const uint32_t* const* b0s, const uint32_t* const* b1s, int level,
                         int rescale_bits, uint32_t* const* out0s, uint32_t* const* out1s, void* stream);
int hg_ctprep_destroy(hg_ctprep* prep);
int hg_ctprep_release(hg_ctprep* prep, void* stream);   /* stream-ordered, as hg_key_release */
size_t hg_ctprep_device_bytes(const hg_ctprep* prep);
/* hg_ct_mult with the left operand prepared (same output, bit for bit). */
int hg_ct_mult_prepared(hg_ctx* ctx, const hg_key* evk, const hg_ctprep* a, const uint32_t* b0,
                        const uint32_t* b1, int level, int rescale_bits, uint32_t* out0,
                        uint32_t* out1, void* stream);
/* _apply_automorphism (ckks.py:247-253): out = (phi_k(c0) + e0, e1), (e0, e1) =
 * keyswitch(phi_k(c1)).  Used by rotate (ckks.py:256-273) and conjugate (:276-279). */
int hg_ct_automorph(hg_ctx* ctx, const hg_key* key, const uint32_t* c0, const uint32_t* c1,
                    int level, int64_t k, uint32_t* out0, uint32_t* out1, void* stream);
/* `count` independent hg_ct_automorph calls with one key, exponent and level (host arrays of
 * device pointers; outputs must not alias inputs): up to 4 rotations share each group of
 * launches.  Used for the rotate-and-add ladders of many independent ciphertexts (matrix.py
 * replicate / duplicate).  Results are identical to the one-by-one calls.            */
int hg_ct_automorph_batch(hg_ctx* ctx, const hg_key* key, int count, const uint32_t* const* c0s,
                          const uint32_t* const* c1s, int level, int64_t k,
                          uint32_t* const* out0s, uint32_t* const* out1s, void* stream);
/* As hg_ct_automorph_batch, accumulating: out_i = c_i + phi_k(c_i) key-switched -- one step of
 * the rotate-and-sum ladders (c += rot(c, 2^j), matrix.py:79-170) in one call, identical to the
 * rotation followed by the ciphertext add. */
int hg_ct_rotate_add_batch(hg_ctx* ctx, const hg_key* key, int count, const uint32_t* const* c0s,
                           const uint32_t* const* c1s, int level, int64_t k, uint32_t* const* out0s,
                           uint32_t* const* out1s, void* stream);

/* ---- plaintext products and batched ciphertext ops (arrays of device pointers in host
 * arrays; outputs must not alias inputs) --------------------------------------------------
 * HeEngine.mult_plain = mult_plain then rescale by the plaintext's scale (hegwas ckks.py:147-163,
 * 197-224, 315-317) with the rescale fused into the CRT window.
 * hg_ct_mult_plain_many: ONE ciphertext (c0, c1 at `level`) times `count` plaintexts ms[i]
 *   (replicate's masks, matrix.py:79-96; ccp_to_cp's column ranges, :196-209) -> (out0s[i], out1s[i]).
 * hg_ct_mult_plain_batch: `count` ciphertexts times ONE plaintext m. */
int hg_ct_mult_plain_many(hg_ctx* ctx, const uint32_t* c0, const uint32_t* c1, int level, int count,
                          const hg_operand* ms, int rescale_bits, uint32_t* const* out0s,
                          uint32_t* const* out1s, void* stream);
int hg_ct_mult_plain_batch(hg_ctx* ctx, int count, const uint32_t* const* c0s, const uint32_t* const* c1s,
                           int level, hg_operand m, int rescale_bits, uint32_t* const* out0s,
                           uint32_t* const* out1s, void* stream);
/* rescale (ckks.py:197-224) of `count` ciphertexts at `level` by `bits`: outputs at level - bits. */
int hg_ct_rescale_batch(hg_ctx* ctx, int count, const uint32_t* const* c0s, const uint32_t* const* c1s,
                        int level, int bits, uint32_t* const* out0s, uint32_t* const* out1s, void* stream);
/* add / sub (ckks.py:108-125) of `count` aligned ciphertext pairs (subtract != 0: a - b). */
int hg_ct_add_batch(hg_ctx* ctx, int count, const uint32_t* const* a0s, const uint32_t* const* a1s,
                    const uint32_t* const* b0s, const uint32_t* const* b1s, int bits, int subtract,
                    uint32_t* const* out0s, uint32_t* const* out1s, void* stream);
/* HeEngine.mult_const (ckks.py:351-356): times the constant plaintext k (|k| < 2^32, the single
 * coefficient of encode_constant, encoding.py:82-90), then rescale by `shift`, in one pass. */
int hg_ct_mult_const_rescale_batch(hg_ctx* ctx, int count, const uint32_t* const* c0s,
                                   const uint32_t* const* c1s, int level, int64_t k, int shift,
                                   uint32_t* const* out0s, uint32_t* const* out1s, void* stream);

/* ---- microbenchmarks / measurement ------------------------------------------------ */
/* Batched forward+inverse negacyclic NTT over `count` length-N rows of residues
 * (prime i % num_primes for row i); data is [count][N] uint32 on device.            */
int hg_ntt_forward(hg_ctx* ctx, uint32_t* data, int count, int prime_offset, void* stream);
int hg_ntt_inverse(hg_ctx* ctx, uint32_t* data, int count, int prime_offset, void* stream);
/* NTT kernel variant: 0 = two passes (strided tiles, contiguous chunks), 1 = log_n 17 on 8-CTA
   clusters exchanging through distributed shared memory, 2 = log_n 17 both passes in one launch
   on 8-CTA clusters with the intermediate through L2 (other sizes: two passes).  Same output
   words; 0 is the default (measured fastest). */
int hg_set_ntt_variant(hg_ctx* ctx, int variant);
/* Integer-pipe peak microbenchmark: runs the NTT butterfly modmul sequence register-
 * resident on all SMs; returns butterflies executed (host) for `iters`.              */
int hg_bench_modmul(hg_ctx* ctx, int iters, uint32_t* sink, double* ops_out, void* stream);
/* Base-conversion MAC probe: the exact fold-every-4 32x32->64 multiply-accumulate of the
 * ModUp/CRT kernels, register resident; returns MACs executed.                       */
int hg_bench_mac(hg_ctx* ctx, int iters, uint32_t* sink, double* ops_out, void* stream);
/* Number of kernel launches issued by this library since context creation. */
long long hg_launch_count(const hg_ctx* ctx);
/* Live kernel timing: when enabled, CUDA events bracket every launch of the
 * instrumented kernel classes (0 = CRT, 1 = ModUp, 2 = NTT, 3 = pointwise,
 * 4 = elementwise) on the launching stream.  hg_kernel_stats synchronises the recorded
 * events and returns, for one class, the summed device milliseconds, the number of
 * launches and the algorithmic work (MACs for CRT/ModUp, butterflies for NTT, bytes
 * for pointwise/elementwise).  Enabling resets the counters.  `enabled`: 0 = off,
 * 1 = every class, otherwise (mask << 1) with bit k of mask selecting class k (so a
 * timed region can bracket only the class whose roofline it reports).                */
int hg_set_kernel_timing(hg_ctx* ctx, int enabled);
/* Host-side replay of CPython's random.Random (MT19937) for the reference's encryption
 * samplers (ring.py:212-235): `state` is getstate()'s 624 words + position, advanced in place.
 * hg_rng_ternary: n x getrandbits(2) -> {+1, 0, 0, -1}.  hg_rng_gaussian: rounded
 * gauss(0, sigma) draws, |x| > 6 sigma redrawn; the Box-Muller spare goes in/out through
 * gauss_next / has_next.  Bit-identical to the Python samplers (tests/test_host.py). */
int hg_rng_ternary(uint32_t* state, int n, int8_t* out);
int hg_rng_gaussian(uint32_t* state, double* gauss_next, int* has_next, int n, double sigma,
                    int32_t* out);
int hg_kernel_stats(hg_ctx* ctx, int kind, double* ms, long long* launches, double* work);
/* Device arena for the library's long-lived objects (prepared switching keys and
 * prepared operands): reserve one more slab of `bytes` up front, so a job's first uses
 * carve keys out of it instead of growing device memory piece by piece.  Replaces the
 * capacity sizing of the reference's CiphertextCache (cache.py:78-97) for the objects
 * that stay resident.  `stream` is unused (the slab is not stream-ordered).
 * hg_pool_bytes: reserved bytes (in_use = 0) or bytes held by live objects (in_use = 1). */
int hg_pool_reserve(hg_ctx* ctx, size_t bytes, void* stream);
size_t hg_pool_bytes(const hg_ctx* ctx, int in_use);
/* Return the arena slabs that hold no live object to the device; returns the bytes freed. */
size_t hg_pool_trim(hg_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* HEGWAS_B200_H */
