/*
 * hegpu.h -- C ABI of the B200-native CKKS engine (libhegpu.so, sm_100a).
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `hebert` (/root/reference/pkg/src/hebert).  Two groups of entry points:
 *
 *  1. Host-array kernel table (hegpu_k_*): exactly the ten functions of the
 *     reference kernel seam `hebert._kernels` (_kernels.py:319-328, numpy twins
 *     :352-361), same arguments and ownership (C-contiguous uint64 arrays owned
 *     by the caller; *_inplace mutate their first argument, the others write a
 *     caller-provided output).  They copy to the GPU, run the device kernels and
 *     copy back; they exist for parity and for callers that bind the kernel
 *     table directly.
 *
 *  2. Device-resident entry points (hegpu_*): operate on device pointers to
 *     limb-major RNS polynomials.  A "poly group" is n_polys polynomials of k
 *     limbs each, poly p at ptr + p*stride (stride in uint64 elements), limb l
 *     at +l*N.  Limb l of every poly in the group uses the ring prime with
 *     global index primes[l] (chain primes are 0..n_chain-1, special primes
 *     follow).  All calls are stream-ordered on `stream` (a cudaStream_t, NULL
 *     = legacy default stream) and never synchronise unless stated.
 *
 * Every function returns 0 on success or a nonzero HEGPU_E_* code; the message
 * of the last failure on the calling thread is hegpu_last_error().  The Python
 * shim maps codes onto the reference error taxonomy (errors.py:4-75):
 * HEGPU_E_ARG -> CryptoError, HEGPU_E_CUDA -> CryptoError (with the CUDA text),
 * HEGPU_E_NOMEM -> CryptoError.
 */
#ifndef HEGPU_H_
#define HEGPU_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HEGPU_OK 0
#define HEGPU_E_ARG 1
#define HEGPU_E_CUDA 2
#define HEGPU_E_NOMEM 3

#define HEGPU_MAX_PRIMES 64

typedef struct hegpu_ring* hegpu_ring_t;

/* -------------------------------------------------------------------------
 * library / ring context
 * ---------------------------------------------------------------------- */

/* Library version string. */
const char* hegpu_version(void);
/* Message of the last failed call on this thread ("" if none). */
const char* hegpu_last_error(void);
/* Number of visible CUDA devices (0 if none); never fails. */
int hegpu_device_count(void);

/* Total kernel launches issued by this library since load (for accounting). */
long long hegpu_launch_count(void);
/* Measured 64-bit Shoup modular-multiplication throughput of this GPU
 * (modmul/s, 8 independent chains per thread, all SMs); synchronous. */
int hegpu_bench_modmul_peak(int iters, double* modmul_per_s);
/* The same for the FP64-pipe modmul the engine uses for primes < 2^46
 * (exact double arithmetic, 6 FP64 ops per product); synchronous. */
int hegpu_bench_fp_modmul_peak(int iters, double* modmul_per_s);
/* Enable (1) / disable (0) per-launch CUDA-event timing; clears records. */
int hegpu_profile_enable(int on);
/* Synchronise the device, then report and clear, per kernel class, the
 * accumulated device time (ms), launch count, algorithmic bytes (inputs read
 * once + outputs written once) and modular multiplications.  Classes:
 * 0 ntt, 1 elementwise, 2 lift, 3 automorphism, 4 tensor, 5 basis conversion,
 * 6 key-switch inner product, 7 diagonal multiply-accumulate, 8 encrypt. */
int hegpu_profile_read(double* ms, long long* counts, double* bytes, double* modmuls,
                       int n_classes);

/* Build a ring context: NTT tables for every prime (psi = the first base in
 * [2, 10^4) whose (q-1)/2N power has order 2N -- ring.py:69-78; tables in
 * bit-reversed order -- ring.py:94-108) plus Montgomery/Shoup constants, on
 * the current CUDA device.  Replaces RingParams/PrimeTables/StackedTables
 * precompute (ring.py:81-177).  Primes must be < 2^62, = 1 mod 2N. */
int hegpu_ring_create(int log_n, const uint64_t* chain, int n_chain,
                      const uint64_t* special, int n_special, hegpu_ring_t* out);
int hegpu_ring_destroy(hegpu_ring_t ring);
/* Copy the device twiddle tables of global prime p to host: 4N words,
 * interleaved (psi_rev[i], shoup(psi_rev[i])) pairs for i < N, then
 * (ipsi_rev[i], shoup(ipsi_rev[i])); natural form, bit-reversed order. */
int hegpu_ring_get_tables(hegpu_ring_t ring, int p, uint64_t* host_out4n);

/* -------------------------------------------------------------------------
 * device-resident polynomial kernels (ring.py:287-482)
 * ---------------------------------------------------------------------- */

/* Negacyclic NTT.  inverse=0: natural -> bit-reversed evaluation order
 * (CT DIT, _kernels.py:144-171); inverse=1: GS DIF back to natural order
 * times N^-1 (_kernels.py:173-204).  in may equal out. */
int hegpu_ntt(hegpu_ring_t ring, int inverse, const uint64_t* in, int64_t in_stride,
              uint64_t* out, int64_t out_stride, int n_polys, int k,
              const int32_t* primes, void* stream);

#define HEGPU_OP_ADD 0  /* a + b          (addmod_rows, _kernels.py:229-240)   */
#define HEGPU_OP_SUB 1  /* a - b          (submod_rows, _kernels.py:242-253)   */
#define HEGPU_OP_MUL 2  /* a * b          (elementwise_mulmod, :288-298)       */
#define HEGPU_OP_MONT 3 /* a * b * R^-1   (elementwise_mont, :206-215)         */
#define HEGPU_OP_NEG 4  /* -a             (ring.neg_mod, ring.py:54-57)        */
#define HEGPU_OP_SCALAR 5 /* a * c[l], c natural per limb (poly_scalar_mul)    */
#define HEGPU_OP_ROWMONT 6 /* a * c[l] * R^-1 (rowwise_mont, :217-227)         */
#define HEGPU_OP_FMA 7  /* out = out + a * b (fma_inplace, :255-269)           */
#define HEGPU_OP_COPY 8 /* out = a                                             */
#define HEGPU_OP_ADDC 9 /* a + c[l], c natural per limb (constant add_plain)   */
#define HEGPU_OP_REDUCE 10 /* a mod q for any 64-bit a (after a wrapping NCCL sum) */
#define HEGPU_OP_AXPYC 11 /* b + a * c[l], c natural per limb                  */

/* Elementwise op over a poly group.  b may be NULL for unary ops; consts is a
 * host array of k per-limb scalars for SCALAR / ROWMONT. */
int hegpu_elementwise(hegpu_ring_t ring, int op, const uint64_t* a, int64_t a_stride,
                      const uint64_t* b, int64_t b_stride, uint64_t* out,
                      int64_t out_stride, int n_polys, int k, const int32_t* primes,
                      const uint64_t* consts, void* stream);

/* out[l] = np.mod(src, q_l) for signed int64 coefficients (limbs_from_signed,
 * ring.py:381-387).  src poly p at src + p*src_stride. */
int hegpu_lift_signed(hegpu_ring_t ring, const int64_t* src, int64_t src_stride,
                      uint64_t* out, int64_t out_stride, int n_polys, int k,
                      const int32_t* primes, void* stream);

/* Centered lift of one limb (prime src_prime, coefficient form) into k limbs:
 * v > q/2 -> v - q, then mod q_l (rescale/ModRaise lift, ops.py:170-173,
 * bootstrap.py:266-270). */
int hegpu_lift_centered(hegpu_ring_t ring, const uint64_t* src, int64_t src_stride,
                        int src_prime, uint64_t* out, int64_t out_stride, int n_polys,
                        int k, const int32_t* primes, void* stream);

/* Full-slot bootstrap diagonals, generated and encoded on the device: for
 * i < n_diags the slot vector of diagonal d[i] of the CoeffToSlot (kind 0,
 * bootstrap.py:174-184) or SlotToCoeff (kind 1, bootstrap.py:187-197) map of
 * output/input half `half`, times `fold`, rolled by g0[i] and conjugated when
 * conj[i] (the BSGS plaintexts of bootstrap.py:219-236), encoded at `scale`
 * like encoding.encode (encoding.py:62-97): out[i*N + k] = rounded int64
 * coefficient k.  d, g0, conj are host arrays; scratch is a device buffer of
 * min(n_diags, 256) * N * 16 bytes.  Coefficients >= 2^62 in magnitude set a
 * sticky flag read (and cleared) by hegpu_encode_overflow (synchronizes). */
int hegpu_encode_diags(hegpu_ring_t ring, int kind, int half, double fold, double scale,
                       int n_diags, const int32_t* d, const int32_t* g0, const uint8_t* conj,
                       void* scratch, int64_t* out, void* stream);
int hegpu_encode_overflow(hegpu_ring_t ring, int* flag);

/* numpy Generator(PCG64).integers(0, bounds[l], size=n, dtype=uint64) for
 * l = 0..k-1 in order (the per-limb uniform sampling of ring.sample_poly,
 * ring.py:494-498, and keygen, keys.py:133-151, 204-206), drawn on the device
 * from the generator state (state, inc as 128-bit halves) into out + l *
 * out_stride.  Bounds must exceed 2^32.  *consumed = 64-bit draws used
 * (k*n plus rejections); the caller advances its generator by that much.
 * Synchronizes the stream. */
int hegpu_pcg64_uniform(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                        const uint64_t* bounds, int k, int n, uint64_t* out,
                        int64_t out_stride, long long* consumed, void* stream);

/* Encryption randomness of an UNSEEDED encryption (replaces the host draws of
 * ops.py:87-100 when the reference would seed numpy from OS entropy): out
 * rows 0, 1, 2 (each n int64) = v ternary on {-1,0,1}, e0, e1 = rint of
 * N(0, sigma^2), expanded on the device from the 64-bit `seed` (the caller's
 * OS entropy) by Philox4x32-10.  Seeded encryptions keep the host numpy
 * stream for bit-exact parity. */
int hegpu_sample_encrypt(int64_t* out, int n, uint64_t seed, double sigma, void* stream);

/* Forward NTT of signed int64 coefficient rows into k eval-form limbs: the
 * lift of poly_from_signed (ring.py:381-393) fused into the NTT's first pass.
 * src poly p at src + p*src_stride, out poly p at out + p*out_stride. */
int hegpu_ntt_from_signed(hegpu_ring_t ring, const int64_t* src, int64_t src_stride,
                          uint64_t* out, int64_t out_stride, int n_polys, int k,
                          const int32_t* primes, void* stream);

/* X -> X^g.  eval_form=1: slot permutation on bit-reversed evaluation form
 * (poly_automorphism_eval, ring.py:471-482); eval_form=0: signed coefficient
 * permutation (poly_automorphism, ring.py:426-437).  in != out. */
int hegpu_automorphism(hegpu_ring_t ring, int eval_form, uint64_t g, const uint64_t* in,
                       int64_t in_stride, uint64_t* out, int64_t out_stride,
                       int n_polys, int k, const int32_t* primes, void* stream);

/* CKKS tensor product (ops.py:355-357): d0 = a0 b0, d1 = a0 b1 + a1 b0,
 * d2 = a1 b1 over chain limbs 0..k-1.  Each operand is a poly group with its
 * own stride. */
int hegpu_tensor(hegpu_ring_t ring, const uint64_t* a0, const uint64_t* a1, int64_t a_stride,
                 const uint64_t* b0, const uint64_t* b1, int64_t b_stride, uint64_t* d0,
                 uint64_t* d1, uint64_t* d2, int64_t d_stride, int n_polys, int k,
                 void* stream);

/* hegpu_tensor with a periodic first operand: product p uses a at index
 * p % a_period (one batch of a against n_polys / a_period stacked batches
 * of b, e.g. one giant power against every node of a polynomial level). */
int hegpu_tensor_periodic(hegpu_ring_t ring, const uint64_t* a0, const uint64_t* a1,
                          int64_t a_stride, int a_period, const uint64_t* b0, const uint64_t* b1,
                          int64_t b_stride, uint64_t* d0, uint64_t* d1, uint64_t* d2,
                          int64_t d_stride, int n_polys, int k, void* stream);

/* -------------------------------------------------------------------------
 * fused CKKS kernels (ckks/ops.py, ckks/keys.py, bootstrap.py)
 * ---------------------------------------------------------------------- */

/* Hybrid key switch (ks_apply, keys.py:278-339), batched over n_batch
 * ciphertext components that share one switching key (the key is streamed
 * once per batch).  d: eval-form polys at `level` (level+1 chain limbs).
 * key_b/key_a: host arrays of n_digits device pointers, each digit a
 * (key_rows, N) eval-form poly over chain primes then special primes
 * (key_rows = n_chain + n_special).  alpha = digit size (params.py:48-51).
 * out_b / out_a: eval-form results at `level`.  accumulate bit 0 / bit 1: add
 * the result into out_b / out_a instead of overwriting (fuses the
 * "d0 + KS(d2).b" of mult and rotate into the ModDown epilogue).  Bit-exact
 * with the reference. */
int hegpu_ks_apply(hegpu_ring_t ring, int level, int alpha, const uint64_t* d,
                   int64_t d_stride, int n_batch, const uint64_t* const* key_b,
                   const uint64_t* const* key_a, int n_digits, uint64_t* out_b,
                   uint64_t* out_a, int64_t out_stride, int accumulate, void* stream);

/* Key switch fused with the following rescale (relinearize-then-rescale of
 * mult, ops.py:346-367): for each batch element b,
 *   out.c{0,1} = round((P * in.c{0,1} + KS(d).{b,a}) / (P * q_level))
 * at level-1, by ONE ModDown from the basis {q_level} + P.  Decrypts like
 * hegpu_ks_apply(accumulate=3) followed by hegpu_rescale (same message and
 * scale); limbs differ by the conversion rounding.  in.c0 at in +
 * b*in_stride, c1 at + in_c1_off (level+1 limbs, may be clobbered); out
 * likewise with `level` limbs.  Needs level >= 1. */
int hegpu_ks_apply_rescale(hegpu_ring_t ring, int level, int alpha, const uint64_t* d,
                           int64_t d_stride, int n_batch, const uint64_t* const* key_b,
                           const uint64_t* const* key_a, int n_digits, uint64_t* in,
                           int64_t in_stride, int64_t in_c1_off, uint64_t* out,
                           int64_t out_stride, int64_t out_c1_off, void* stream);

/* Hoisted rotations of one (batched) ciphertext by n_rot Galois elements
 * (the bootstrap baby steps, bootstrap.py:214-217): ModUp of c1 once, then
 * per rotation r a digit permutation, the inner product with rotation key r
 * (key_b/key_a: host arrays of n_rot*n_digits device pointers, rotation-major)
 * and ModDown; outs[r] (host array of device pointers) receives the packed
 * rotated ciphertexts (c0 at outs[r] + b*cs, c1 at +c1_off).  Input c0 at
 * c + b*cs, c1 at c + b*cs + c1_off.  Decrypts like the unhoisted rotation;
 * limbs are not bit-identical to it (the digit lift commutes with the
 * automorphism only up to a multiple of the digit modulus).
 * pq_out = 1 (double hoisting): no ModDown; outs[r] receives the P-scaled
 * extended-basis rotation (n_batch, 2, level+1+K, N) = (P sigma(c0) + kb, ka),
 * and the outputs must be packed rotation-major (outs[r] = outs[0] +
 * r*n_batch*2*(level+1+K)*N). */
int hegpu_ks_hoisted(hegpu_ring_t ring, int level, int alpha, const uint64_t* c, int64_t cs,
                     int64_t c1_off, int n_batch, int n_rot, const uint64_t* galois,
                     const uint64_t* const* key_b, const uint64_t* const* key_a, int n_digits,
                     uint64_t* const* outs, int pq_out, void* stream);

/* Hoisted rotation sum: out = ct + sum_{r < n_rot} rot_r(ct), rot_r = X ->
 * X^galois[r] then a key switch with key r (key_b/key_a: host arrays of
 * n_rot*n_digits device pointers, rotation-major).  One ModUp of c1, n_rot
 * digit permutations + inner products accumulated in the extended basis, one
 * ModDown (the reference's rotate-and-sum loops run one full key switch per
 * rotation, logreg.py:202-229).  Decrypts like the sequential sum; limbs
 * differ.  c: n_batch packed ciphertexts (c0 at c + b*cs, c1 at + c1_off);
 * out likewise with out_stride / out_c1_off; out must not alias c. */
int hegpu_ks_rotsum(hegpu_ring_t ring, int level, int alpha, const uint64_t* c, int64_t cs,
                    int64_t c1_off, int n_batch, int n_rot, const uint64_t* galois,
                    const uint64_t* const* key_b, const uint64_t* const* key_a, int n_digits,
                    uint64_t* out, int64_t out_stride, int64_t out_c1_off, void* stream);

/* Giant steps of a BSGS linear transform with one lazy ModDown:
 * out = partial[0] + sum_{g=1}^{n_giants-1} rot_g(partial[g]) where rot_g is
 * X -> X^galois[g] followed by a key switch with key g (key_b/key_a: host
 * arrays of n_giants*n_digits device pointers, giant-major; entries of giant
 * 0 unused).  partials: packed (n_batch, 2, level+1, N) ciphertexts at
 * partials + g*gstride; out: packed (n_batch, 2, level+1, N).  The inner
 * products accumulate in the extended basis and are brought down once
 * (bootstrap.py:243-245 rotates and adds per giant); decrypts identically,
 * limbs differ.  rescale = 1: the final ModDown also divides by q_level
 * (the transform's rescale, bootstrap.py:247) and out is packed
 * (n_batch, 2, level, N) at level - 1.  pq_in = 1 (with rescale = 1): the
 * partials are P-scaled extended-basis ciphertexts (n_batch, 2, level+1+K, N)
 * from double-hoisted babies; only each giant's c1 is brought down for its
 * key switch, one final ModDown by q_level * P remains; partials are
 * clobbered.  N >= 2^12.  pq_in = 2: as 1, but out receives the
 * extended-basis sum (n_batch, 2, level+1+K, N) BEFORE the final ModDown
 * (a transform split across ranks modular-all-reduces these first, then
 * calls hegpu_moddown_rescale_ext). */
int hegpu_bsgs_giants(hegpu_ring_t ring, int level, int alpha, const uint64_t* partials,
                      int64_t gstride, int n_batch, int n_giants, const uint64_t* galois,
                      const uint64_t* const* key_b, const uint64_t* const* key_a, int n_digits,
                      uint64_t* out, int rescale, int pq_in, void* stream);

/* Scratch allocator hook.  The library's temporary device buffers
 * (stream-ordered, freed before the call returns in stream order) come from
 * alloc/free when set -- e.g. a framework's caching allocator, so one pool
 * serves both -- and from cudaMallocAsync/cudaFreeAsync when both are NULL.
 * alloc(bytes, stream) returns NULL on failure (-> HEGPU_E_NOMEM). */
typedef void* (*hegpu_alloc_fn)(size_t bytes, void* stream);
typedef void (*hegpu_free_fn)(void* ptr, size_t bytes, void* stream);
int hegpu_set_allocator(hegpu_alloc_fn alloc, hegpu_free_fn free_fn);

/* ModDown of P-scaled extended-basis ciphertexts by q_level * P (the final
 * step of a double-hoisted transform, bootstrap.py:243-247 + keys.py:330-338):
 * in (n_batch, 2, level+1+K, N) eval form (clobbered) -> out (n_batch, 2,
 * level, N) at level - 1.  N >= 2^12. */
int hegpu_moddown_rescale_ext(hegpu_ring_t ring, int level, int alpha, uint64_t* in,
                              int n_batch, uint64_t* out, void* stream);

/* Rescale by q_level (_poly_rescale, ops.py:164-189): in has level+1 chain
 * limbs (eval form), out gets `level` limbs.  in may equal out. */
int hegpu_rescale(hegpu_ring_t ring, int level, const uint64_t* in, int64_t in_stride,
                  uint64_t* out, int64_t out_stride, int n_polys, void* stream);

/* ModRaise (_mod_raise, bootstrap.py:260-275): eval-form level-0 polys ->
 * centered lift to chain limbs 0..to_level, eval form. */
int hegpu_mod_raise(hegpu_ring_t ring, const uint64_t* in, int64_t in_stride,
                    uint64_t* out, int64_t out_stride, int n_polys, int to_level,
                    void* stream);

/* Public-key encryption combine (encrypt, ops.py:102-116): given eval-form
 * v, e0, e1, m (k limbs each) and pk (b, a) sliced to k limbs:
 * c0 = v*b + e0 + m, c1 = v*a + e1.  m may be NULL (zero). */
int hegpu_encrypt_combine(hegpu_ring_t ring, const uint64_t* v, const uint64_t* e0,
                          const uint64_t* e1, const uint64_t* m, const uint64_t* pk_b,
                          const uint64_t* pk_a, uint64_t* c0, uint64_t* c1, int k,
                          void* stream);

/* Plaintext-diagonal multiply-accumulate for the BSGS linear transforms
 * (_apply_diag_transform, bootstrap.py:200-247): for each of n_terms terms t
 * and each of n_batch ciphertexts b,
 *   out_b.c0 (+)= pt[t] * ct[t]_b.c0,   out_b.c1 (+)= pt[t] * ct[t]_b.c1,
 * where ct[t]_b.c0 is at ct_ptrs[t] + b*ct_bstride, c1 at +ct_c1_off, and
 * out_b.c0 at out + b*out_bstride, c1 at +out_c1_off; k chain limbs.  Each
 * plaintext diagonal is read once per batch.  accumulate=0 overwrites out.
 * ct_ptrs / pt_ptrs are host arrays of device pointers. */
int hegpu_diag_mac(hegpu_ring_t ring, const uint64_t* const* ct_ptrs, int64_t ct_c1_off,
                   int64_t ct_bstride, const uint64_t* const* pt_ptrs, int n_terms,
                   int n_batch, uint64_t* out, int64_t out_c1_off, int64_t out_bstride, int k,
                   int accumulate, void* stream);

/* All-giants BSGS multiply-accumulate (one launch per linear transform):
 * for every giant g < n_giants and batch element b < n_batch,
 *   out[g]_b.c{0,1} = sum_{t < n_terms} pt[idx[g][t]] * baby[t]_b.c{0,1}
 * with baby[t]_b.c0 at babies[t] + b*bstride, c1 at +c1_off (host array of
 * n_terms <= 128 device pointers); diagonal i at pt_base + i*pt_stride;
 * pt_idx a DEVICE int32 array [n_giants][n_terms] (-1 = zero diagonal);
 * out[g]_b.c0 at out + g*out_gstride + b*bstride, c1 at +c1_off.  Every
 * diagonal, baby and output crosses HBM once.
 * pt_log_run = r in [0, 5]: the diagonals are run-compressed, k limbs of
 * N >> r words each, and coefficient x of limb l reads word (l*N + x) >> r.
 * Evaluation vectors of polynomials in X^(2^r) have this form in the
 * bit-reversed NTT order (slot vectors periodic with period N / 2^(r+1)).
 * The last n_special_rows of the k limbs are the special primes (babies in
 * the extended basis Q_level + P of double-hoisted transforms), else 0. */
int hegpu_bsgs(hegpu_ring_t ring, const uint64_t* const* babies, int n_terms, int64_t c1_off,
               int64_t bstride, int n_batch, const uint64_t* pt_base, int64_t pt_stride,
               int pt_log_run, const int32_t* pt_idx, int n_giants, uint64_t* out,
               int64_t out_gstride, int k, int n_special_rows, void* stream);

/* -------------------------------------------------------------------------
 * host-array kernel table: drop-in for hebert._kernels (_kernels.py:319-328)
 * shapes are (k, n) row-major uint64; vectors are length k
 * ---------------------------------------------------------------------- */
int hegpu_k_ntt_forward_inplace(uint64_t* a, int k, int n, const uint64_t* psi_rev,
                                const uint64_t* q, const uint64_t* qinv);
int hegpu_k_ntt_inverse_inplace(uint64_t* a, int k, int n, const uint64_t* ipsi_rev,
                                const uint64_t* ninv, const uint64_t* q,
                                const uint64_t* qinv);
int hegpu_k_elementwise_mont(const uint64_t* a, const uint64_t* b, uint64_t* out, int k,
                             int n, const uint64_t* q, const uint64_t* qinv);
int hegpu_k_elementwise_mulmod(const uint64_t* a, const uint64_t* b, uint64_t* out, int k,
                               int n, const uint64_t* q, const uint64_t* qinv,
                               const uint64_t* r2);
int hegpu_k_rowwise_mont(const uint64_t* a, const uint64_t* c, uint64_t* out, int k, int n,
                         const uint64_t* q, const uint64_t* qinv);
int hegpu_k_addmod_rows(const uint64_t* a, const uint64_t* b, uint64_t* out, int k, int n,
                        const uint64_t* q);
int hegpu_k_submod_rows(const uint64_t* a, const uint64_t* b, uint64_t* out, int k, int n,
                        const uint64_t* q);
/* hat (l, n), punc (l, kt) Montgomery form, out (kt, n) */
int hegpu_k_base_convert(const uint64_t* hat, int l, int n, const uint64_t* punc, int kt,
                         const uint64_t* q_to, const uint64_t* qinv_to, uint64_t* out);
int hegpu_k_fma_inplace(uint64_t* acc, const uint64_t* a, const uint64_t* b, int k, int n,
                        const uint64_t* q, const uint64_t* qinv, const uint64_t* r2);
/* key (key_rows, n); rows int64[k] */
int hegpu_k_fma_gather_inplace(uint64_t* acc, const uint64_t* a, const uint64_t* key,
                               int key_rows, const int64_t* rows, int k, int n,
                               const uint64_t* q, const uint64_t* qinv,
                               const uint64_t* r2);

#ifdef __cplusplus
}
#endif
#endif /* HEGPU_H_ */
