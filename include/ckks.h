/*
 * include/ckks.h -- C ABI of libckks, the B200-native (sm_100a) RNS-CKKS hot path of
 * PrivFT (arXiv 1908.06972).  Plain C: pointers and sizes only, no torch types.
 *
 * Citations: P:NNN = /root/reference/PAPER.md line NNN (section / equation / algorithm);
 * S:NNN = SPEC.md.  Readings A1..A32 = DESIGN.md "Readings".
 *
 * DATA LAYOUT.  A ckks_buf is a view over CALLER-OWNED DEVICE memory holding `count`
 * plaintexts (n_polys = 1) or ciphertexts (n_polys = 2) laid out
 *        data[count][n_polys][capacity][N]   (uint64 residues)
 * Only the first `level` limbs of each polynomial are active; limb i is the residue
 * polynomial modulo q_i (q_0 > q_1 > ... ).  Resident data is in the library's
 * NTT domain (bit-reversed evaluation order, canonical residues in [0, q_i)); the
 * BOUNDARY form used by ckks_import_coeffs / ckks_export_coeffs is the coefficient
 * domain, canonical, same layout.  All ops act on every element of the batch.
 *
 * OWNERSHIP.  The context owns its prime tables, twiddles, keys and scratch (device
 * memory it allocates itself).  The caller owns every ckks_buf; outputs must be
 * allocated with capacity >= result level and count equal to the inputs'.  `out` may
 * alias an input of the same op.
 *
 * RANDOMNESS.  The library never samples: secret key, key and encryption randomness
 * are caller-supplied device arrays (seeded generators live outside the library).
 *
 * ERRORS.  Every call returns ckks_status and never aborts.  Argument checks are
 * synchronous.  Kernels are stream-ordered on the context stream; asynchronous CUDA
 * errors surface as CKKS_E_CUDA from the next call (message: ckks_last_error).
 * A context is single-threaded.
 */
#ifndef CKKS_H
#define CKKS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    CKKS_OK = 0,
    CKKS_E_INVALID_ARG = -1,
    CKKS_E_LEVEL_MISMATCH = -2,   /* ops on different levels (A30)            */
    CKKS_E_SCALE_MISMATCH = -3,   /* add with non-identical scales (A13)             */
    CKKS_E_LEVEL_EXHAUSTED = -4,  /* rescale at level 1                             */
    CKKS_E_MISSING_KEY = -5,      /* relin / Galois / secret key not present        */
    CKKS_E_PRIME_EXHAUSTED = -6,  /* not enough primes = 1 mod 2N below 2^bits        */
    CKKS_E_ENCODE_OVERFLOW = -7,  /* encoded coefficient does not fit int64         */
    CKKS_E_CUDA = -8,
    CKKS_E_OOM = -9,
    CKKS_E_UNSUPPORTED = -10
} ckks_status;

typedef struct ckks_ctx ckks_ctx;
typedef struct ckks_privft_model ckks_privft_model;

typedef struct {
    uint64_t *data;     /* DEVICE pointer: [count][n_polys][capacity][N] uint64          */
    uint32_t count;     /* batch size (>= 1)                                            */
    uint32_t n_polys;   /* 1 = plaintext, 2 = ciphertext                                */
    uint32_t level;     /* active limbs l, 1 <= l <= L                                  */
    uint32_t capacity;  /* limb stride per polynomial, >= level                        */
    double scale;       /* Delta, tracked exactly in IEEE double (A13)                  */
} ckks_buf;

/* SETUP (Sec. 3.4) and the prime chain (reading A5).
 * Primes: when `primes` is NULL the chain is scanned: one descending scan per bit size
 * over q = 1 mod 2N (deterministic Miller-Rabin); the special prime P is drawn first
 * from the special_bits scan (K of them), then q_0, q_1, ... in order from limb_bits[i]'s
 * scan.  Otherwise primes[0..L-1] = q_i and primes[L..L+K-1] = p_k.  Every prime must be
 * < 2^61.  P = p_0 ... p_{K-1}. */
typedef struct {
    uint32_t log_n;             /* N = 2^log_n, 10 <= log_n <= 16                       */
    uint32_t n_limbs;           /* L                                                     */
    const uint32_t *limb_bits;  /* [L] bit size of each q_i (ignored if primes != NULL)  */
    uint32_t special_bits;      /* bit size of P (one special prime, A6)                 */
    const uint64_t *primes;     /* optional explicit [L+K] chain (host)                  */
    double scale;               /* default Delta = 2^rho                         */
    uint32_t n_special;         /* K special primes (0 -> 1).  K = 1 and digit_limbs = 1  */
    uint32_t digit_limbs;       /* alpha (0 -> 1) is the per-limb key switch of A6; else */
                                /* hybrid key switching: alpha-limb      */
                                /* digits + fast base conversion, alpha, K <= 16          */
} ckks_params;

/* ---- context ------------------------------------------------------------------ */
ckks_status ckks_ctx_create(const ckks_params *params, int device, void *cuda_stream, ckks_ctx **out);
ckks_status ckks_ctx_destroy(ckks_ctx *ctx);
ckks_status ckks_set_stream(ckks_ctx *ctx, void *cuda_stream);
/* primes_out: [L+K] host (q_0..q_{L-1}, p_0..p_{K-1}); any pointer may be NULL. */
ckks_status ckks_ctx_info(const ckks_ctx *ctx, uint32_t *log_n, uint32_t *n_limbs, uint64_t *primes_out);
const char *ckks_last_error(const ckks_ctx *ctx);
/* Number of kernel launches issued by this context since creation (instrumentation). */
uint64_t ckks_launch_count(const ckks_ctx *ctx);
/* Per-kernel timing: when enabled, every launch is bracketed by CUDA events on the
 * context stream.  ckks_profile_read synchronises on them and returns, for up to `cap`
 * kernel names (strings owned by the context, valid until the next read), the total
 * milliseconds, launch counts and algorithmic work work[5k..5k+4] = (radix-2 butterflies on
 * the integer pipe, 64-bit modular multiply(-accumulate)s on the integer pipe, ideal HBM
 * bytes, radix-2 butterflies on the FP64 pipe, modular multiply-accumulates on the FP64
 * pipe); `work` holds 5 * cap doubles; *n receives the number of names; reset != 0 clears
 * the totals. */
ckks_status ckks_profile_enable(ckks_ctx *ctx, int on);
ckks_status ckks_profile_read(ckks_ctx *ctx, const char **names, double *ms, uint64_t *counts, double *work,
                              uint32_t cap, uint32_t *n, int reset);

/* ---- keys (P:139 KEYGEN, P:149 relinearisation, P:163 / P:431 rotation keys) ----
 * All randomness is caller-supplied DEVICE memory:
 *   s  : int64 [N], entries in {0,1}  (binary secret, reading A2)
 *   a  : uint64, uniform residues;  e : int64 small errors (sigma = 3.2)
 * Public key  : a [L][N], e [N];        b = -a s + e
 * Switch keys : a [dnum][L+K][N], e [dnum][N], dnum = ceil(L / alpha); for digit d,
 *               limb i in {q_0..q_{L-1}, p_0..p_{K-1}}:
 *               b_{d,i} = -a_{d,i} s + e_d + [i in digit d] (P mod q_i) s_from (A6, A9)
 *               s_from = s^2 (relinearisation) or phi_kappa(s) (rotation by `step`,
 *               kappa = 5^step mod 2N, negative step -> 5^{-|step|}, A10).       */
ckks_status ckks_set_secret(ckks_ctx *ctx, const int64_t *s_dev);
ckks_status ckks_keygen_public(ckks_ctx *ctx, const uint64_t *a_dev, const int64_t *e_dev);
ckks_status ckks_keygen_relin(ckks_ctx *ctx, const uint64_t *a_dev, const int64_t *e_dev);
ckks_status ckks_keygen_galois(ckks_ctx *ctx, int32_t step, const uint64_t *a_dev, const int64_t *e_dev);
/* Import a switching key already in COEFFICIENT form, layout [dnum][2 (b|a)][L+K][N]
 * (device).  kind 0 = relinearisation (step ignored), 1 = Galois for `step`. */
ckks_status ckks_import_switch_key(ckks_ctx *ctx, int kind, int32_t step, const uint64_t *key_coeff_dev);
/* Galois element for a rotation step (A10). */
uint64_t ckks_galois_elt(const ckks_ctx *ctx, int32_t step);

/* ---- boundary form ----------------------------------------------------------- */
/* src/dst: DEVICE [count][n_polys][level][N] coefficient-form canonical residues
 * (packed: stride = level).  Import applies the forward NTT; export the inverse.   */
ckks_status ckks_import_coeffs(ckks_ctx *ctx, const uint64_t *src_dev, ckks_buf *dst);
ckks_status ckks_export_coeffs(ckks_ctx *ctx, const ckks_buf *src, uint64_t *dst_dev);
/* ---- persistence / client-server transport ("the client sends ... encrypted", P:465
 * "123 ciphertexts") ------------------------------------------------------------
 * Serialised form, little-endian HOST bytes: a 64-byte header
 *   "CKKSBUF1" | u32 version (1) | u32 log_n | u32 count | u32 n_polys | u32 level | u32 0 |
 *   f64 scale | u64 chain hash (FNV-1a over the level's primes q_0..q_{level-1}) | 16 zero bytes
 * followed by [count][n_polys][level][N] u64 COEFFICIENT-form canonical residues.
 * ckks_export: host_bytes == NULL -> *len = bytes needed, CKKS_OK; cap too small ->
 *   CKKS_E_INVALID_ARG (with *len = bytes needed).  Synchronous: returns when the bytes are written.
 * ckks_import_info: validates the header (magic, version, ring, chain hash, length) and reports
 *   the shape; ckks_import: dst must be caller-allocated with count >= the stored count and
 *   capacity >= level; it receives count / n_polys / level / scale.  Residues >= q_i, a foreign
 *   chain or a truncated buffer -> CKKS_E_INVALID_ARG, nothing written. */
ckks_status ckks_export(ckks_ctx *ctx, const ckks_buf *src, void *host_bytes, size_t cap, size_t *len);
ckks_status ckks_import_info(ckks_ctx *ctx, const void *host_bytes, size_t len, uint32_t *count,
                             uint32_t *n_polys, uint32_t *level, double *scale);
ckks_status ckks_import(ckks_ctx *ctx, const void *host_bytes, size_t len, ckks_buf *dst);
/* Evaluation keys (and the public key, when set) for the server side (the server never
 * needs s): header "CKKSKEY1" | u32 version | u32 log_n | u32 L | u32 K | u32 alpha | u32 n_keys |
 * u64 chain hash (all L+K primes) | 24 zero bytes, then per key a 16-byte record
 *   u32 kind (0 relinearisation, 1 Galois, 2 public) | u32 0 | u64 Galois element kappa (0)
 * and its COEFFICIENT-form words: switching keys [dnum][2][L+K][N] (the layout
 * ckks_import_switch_key takes), the public key [2 (b|a)][L][N].  Same size-query / capacity
 * rules as ckks_export.  ckks_import_keys installs every key it carries (replacing keys of the
 * same kind / kappa); a header for another ring, chain, alpha or K -> CKKS_E_INVALID_ARG. */
ckks_status ckks_export_keys(ckks_ctx *ctx, void *host_bytes, size_t cap, size_t *len);
ckks_status ckks_import_keys(ckks_ctx *ctx, const void *host_bytes, size_t len);
/* Raw batched negacyclic NTT (row a1): data DEVICE [count][level][N], limb i mod q_i,
 * in place.  inverse = 0: coefficient -> NTT domain;  1: NTT -> coefficient. */
ckks_status ckks_ntt(ckks_ctx *ctx, uint64_t *data_dev, uint32_t count, uint32_t level, int inverse);

/* ---- encode / decode (host FP, reading A12) ------------------------
 * re/im: HOST arrays of n_slots <= N/2 doubles (im may be NULL); slots past n_slots are
 * zero.  pt must have count == 1, n_polys == 1.  Coefficients are llround()ed (A28). */
ckks_status ckks_encode(ckks_ctx *ctx, const double *re, const double *im, size_t n_slots, double scale,
                        uint32_t level, ckks_buf *pt);
ckks_status ckks_decode(ckks_ctx *ctx, const ckks_buf *pt, double *re_out, double *im_out, size_t n_slots);

/* ---- batched GPU encode / decode -------------
 * The same maps as ckks_encode / ckks_decode, for pt->count plaintexts at once, entirely
 * in sm_100a kernels (codec.cu): a four-step fp64 FFT with the slot scatter, rounding and
 * RNS residues (encode) or the centred CRT lift and slot gather (decode) fused into it.
 * z_dev: DEVICE, [pt->count][n_slots] complex values as interleaved (re, im) doubles,
 * n_slots <= N/2 (slots past n_slots encode as zero / are not written).
 * Encode: pt (n_polys 1, capacity >= level) receives NTT-form residues at `level`;
 *   pt->level/scale are set.  A coefficient that overflows int64 is encoded as 0
 *   and raises a sticky device flag read by ckks_encode_overflowed.  Coefficients are
 *   rounded half away from zero (A28); they agree with the host encode to +-1.
 * Decode: needs |m_k| < 2^127 for every coefficient of the plaintext (reading A33),
 *   true for any message that decodes to finite slots.
 * Both are stream-ordered and asynchronous (no host sync). */
ckks_status ckks_encode_batch(ckks_ctx *ctx, const double *z_dev, size_t n_slots, double scale, uint32_t level,
                              ckks_buf *pt);
ckks_status ckks_decode_batch(ckks_ctx *ctx, const ckks_buf *pt, double *z_dev, size_t n_slots);
/* Synchronises the stream; *flag = 1 if any ckks_encode_batch since the last call
 * overflowed, then clears the flag. */
ckks_status ckks_encode_overflowed(ckks_ctx *ctx, int *flag);

/* ---- encrypt / decrypt (reading A1) -------------------------------
 * u_dev: int64 [count][N] binary; e0_dev, e1_dev: int64 [count][N].
 * c0 = b u + mu + e0, c1 = a u + e1.   Decrypt: mu = c0 + c1 s (needs the secret). */
ckks_status ckks_encrypt(ckks_ctx *ctx, const ckks_buf *pt, const int64_t *u_dev, const int64_t *e0_dev,
                         const int64_t *e1_dev, ckks_buf *ct);
ckks_status ckks_decrypt(ckks_ctx *ctx, const ckks_buf *ct, ckks_buf *pt);

/* ---- homomorphic ops (Sec. 3.4) ---------------------------------------- */
ckks_status ckks_add(ckks_ctx *ctx, const ckks_buf *a, const ckks_buf *b, ckks_buf *out);          /* HADD  */
ckks_status ckks_sub(ckks_ctx *ctx, const ckks_buf *a, const ckks_buf *b, ckks_buf *out);
ckks_status ckks_add_plain(ckks_ctx *ctx, const ckks_buf *ct, const ckks_buf *pt, ckks_buf *out); /* HADDPLAIN */
/* HMULPLAIN: pt may have count 1 (broadcast over the batch) or count == ct->count. */
ckks_status ckks_mul_plain(ckks_ctx *ctx, const ckks_buf *ct, const ckks_buf *pt, ckks_buf *out);
/* multiply by the constant polynomial llround(value * const_scale); scale *= const_scale (A15) */
ckks_status ckks_mul_const(ckks_ctx *ctx, const ckks_buf *ct, double value, double const_scale, ckks_buf *out);
/* add the constant llround(value * ct->scale) to c0 */
ckks_status ckks_add_const(ckks_ctx *ctx, const ckks_buf *ct, double value, ckks_buf *out);
/* HMUL + relinearisation, no rescale. */
ckks_status ckks_mul_relin(ckks_ctx *ctx, const ckks_buf *a, const ckks_buf *b, ckks_buf *out);
/* HMult + relinearisation + RESCALE in one call (the BASELINE metric op, P:149 + P:157):
 * bit-identical to ckks_mul_relin followed by ckks_rescale (out at level l - 1, scale
 * scale_a scale_b / q_{l-1}).  With per-limb digits (alpha = K = 1) the key switch's ModDown
 * and the RESCALE run as ONE floor by P q_{l-1} (reading A7: floor(floor(x / P) / q) =
 * floor(x / (P q))), saving one broadcast NTT pass; with hybrid key switching (alpha or K > 1)
 * the ModDown conversion and the RESCALE share one conversion and one broadcast NTT, exact by
 * linearity of the NTT (reading H2).  Errors as ckks_mul_relin; level 1 ->
 * CKKS_E_LEVEL_EXHAUSTED. */
ckks_status ckks_mul_relin_rescale(ckks_ctx *ctx, const ckks_buf *a, const ckks_buf *b, ckks_buf *out);
/* RESCALE, Eq. (1) / Alg "RNS RESCALE": floor (A4); level - 1; scale /= q_{l-1}. */
ckks_status ckks_rescale(ckks_ctx *ctx, const ckks_buf *ct, ckks_buf *out);
/* ROTATE: left by `steps` slots; NAF over +-2^i keys (A10, A31). */
ckks_status ckks_rotate(ckks_ctx *ctx, const ckks_buf *ct, int32_t steps, ckks_buf *out);
/* Alg "TotalSum" (reading A11): for i < log2(N/2): ct += rotate(ct, 2^i). */
ckks_status ckks_total_sum(ckks_ctx *ctx, const ckks_buf *ct, ckks_buf *out);

/* ---- multi-GPU building block --------------------------------------
 * gathered: DEVICE [R][count][n_polys][capacity][N] (R copies laid out like `out`);
 * out = sum over R mod q_i (NCCL cannot reduce modulo q_i). */
ckks_status ckks_modadd_gathered(ckks_ctx *ctx, const uint64_t *gathered_dev, uint32_t R, ckks_buf *out);

/* ---- fused peer-memory modular all-reduce (P:309 data parallelism,
 * north star "NCCL has no modular reduction") -------------------------------------------
 * One process per GPU of one node, R <= 8 ranks.  Each rank exports the device buffers it
 * will reduce with ckks_ipc_export (CUDA IPC; handle = CKKS_IPC_HANDLE_BYTES opaque bytes +
 * the pointer's offset inside its allocation), ships handle and offset to its peers (the
 * caller's transport, e.g. torch.distributed all_gather_object), and maps each peer's buffer
 * once with ckks_ipc_open (release with ckks_ipc_close).
 * ckks_p2p_modsum: in_ptrs / out_ptrs are HOST arrays of R DEVICE pointers in rank order
 * (this rank's own buffers at index `rank`, the peers' mapped ones elsewhere), every buffer
 * laid out like `shape` ([count][n_polys][capacity][N], `level` limbs used).  This rank sums
 * its share of the count*n_polys*level limb rows over all R inputs mod q_i and stores the
 * result into all R outputs, in one kernel (P2P loads + stores over NVLink).  After EVERY rank
 * has run it, every out_ptrs[r] holds the full sum.  in == out (in place) is allowed: each
 * element is read and written by the same rank only.  Synchronisation is the caller's: all
 * inputs complete on all ranks before any rank's call starts (e.g. stream sync + barrier),
 * outputs complete after all ranks' streams have passed it (stream sync + barrier). */
#define CKKS_IPC_HANDLE_BYTES 64
ckks_status ckks_ipc_export(ckks_ctx *ctx, const void *dev_ptr, void *handle_out, uint64_t *offset_out);
ckks_status ckks_ipc_open(ckks_ctx *ctx, const void *handle, uint64_t offset, void **dev_ptr_out);
ckks_status ckks_ipc_close(ckks_ctx *ctx, void *dev_ptr);
ckks_status ckks_p2p_modsum(ckks_ctx *ctx, uint64_t *const *in_ptrs, uint64_t *const *out_ptrs, uint32_t R,
                            uint32_t rank, const ckks_buf *shape);

/* ---- limb-sharded key switching (north star: "RNS limbs shard across
 * GPUs with an NCCL all-gather over NVLink before base conversion") ----------------------
 * Rank r of R owns limbs [lo, hi) = [r w, min((r+1) w, l)), w = ceil(l / R), of every
 * polynomial of a batch at level l.  A SHARD buffer holds only those limbs (local limb k =
 * global limb lo + k; `level` = hi - lo).  One key switch is:
 *  (1) ckks_shard_ks_digits  -> D_own [count][w][N]: coefficient-form digits of the owned
 *      limbs of the polynomial being switched.  kind 0 (relinearisation): also the
 *      tensor product of shards a, b: out <- (d0, d1); d2 is kept in the context (per lo) until (3).
 *      kind 1 (rotation by `step`): phi_kappa(c1(a)) (b, out unused).
 *  (2) the CALLER all-gathers D_own over ranks into D_all [R][count][w][N] (NCCL, int64 view).
 *  (3) ckks_shard_ks_finish  -> out (shard): base + ModDown(sum_j ModUp(d_j) * ksk_j) for the
 *      owned targets; the special prime's accumulator is computed redundantly on each rank.
 *      kind 0: base = (d0, d1) already in out;  kind 1: base = (phi(c0(a)), 0).
 * Bit-identical to ckks_mul_relin / one ckks_rotate digit on the unsharded batch.
 * Per-limb digits only (alpha = K = 1; otherwise CKKS_E_UNSUPPORTED).
 * Sharded RESCALE (Eq. 1): the owner of limb l-1 computes X [count][2][N] (coefficient form of
 * that limb) with ckks_shard_rescale_last; the caller broadcasts X; every rank applies
 * ckks_shard_rescale_apply to its limbs < l-1. */
ckks_status ckks_shard_ks_digits(ckks_ctx *ctx, int kind, int32_t step, const ckks_buf *a, const ckks_buf *b,
                                 uint32_t lo, uint32_t l, uint32_t w, ckks_buf *out, uint64_t *D_own_dev);
ckks_status ckks_shard_ks_finish(ckks_ctx *ctx, int kind, int32_t step, const uint64_t *D_all_dev, uint32_t R,
                                 uint32_t w, const ckks_buf *a, uint32_t lo, uint32_t l, ckks_buf *out);
/* Digit-pipelined form of (2)+(3) (row f3): instead of waiting for the whole all-gather, the
 * caller hands over each rank's digit shard as soon as it has arrived:
 *  (3a) ckks_shard_ks_window(r): ModUp + inner product of digits [r w, min(r w + w, l)) -- rank
 *       r's shard D_win [count][w][N] -- for the owned targets and P, added (mod q_t) to the
 *       accumulators the context keeps per lo; first != 0 starts a new key switch.  Windows may
 *       come in any order (the sum mod q_t is order-free); each exactly once.
 *  (3b) ckks_shard_ks_combine: ModDown of the accumulators into out, as ckks_shard_ks_finish.
 * Bit-identical to ckks_shard_ks_finish.  Stream-ordered: D_win must be complete on the
 * context stream (e.g. the caller waits on the window's broadcast / all-gather event). */
ckks_status ckks_shard_ks_window(ckks_ctx *ctx, int kind, int32_t step, const uint64_t *D_win_dev, uint32_t r,
                                 uint32_t w, const ckks_buf *a, uint32_t lo, uint32_t l, int first);
ckks_status ckks_shard_ks_combine(ckks_ctx *ctx, int kind, int32_t step, const ckks_buf *a, uint32_t lo,
                                  uint32_t l, ckks_buf *out);
ckks_status ckks_shard_rescale_last(ckks_ctx *ctx, const ckks_buf *ct, uint32_t lo, uint32_t l, uint64_t *X_dev);
ckks_status ckks_shard_rescale_apply(ckks_ctx *ctx, const uint64_t *X_dev, const ckks_buf *ct, uint32_t lo,
                                     uint32_t l, ckks_buf *out);

/* ---- PrivFT encrypted inference -----------
 * Model: H is m x n (embedding), O is n x c (output layer).  Packing (P:205,
 * A16, A17): P^H_{j,k} has slot i = H[k t + i][j] (level L, default scale); P^O_j has
 * slot i = O[j][i] for i < c (level L-2).  H_host, O_host: row-major doubles (host).
 * ckks_privft_model_wrap instead adopts caller-owned, already-encoded device buffers
 * (H_pts: count n*K, ordered [j][k], level L; O_pts: count n, level L-2); the caller
 * keeps them alive until ckks_privft_model_destroy. */
ckks_status ckks_privft_model_create(ckks_ctx *ctx, const double *H_host, const double *O_host, uint32_t m,
                                     uint32_t n, uint32_t c, ckks_privft_model **out);
ckks_status ckks_privft_model_wrap(ckks_ctx *ctx, const ckks_buf *H_pts, const ckks_buf *O_pts, uint32_t m,
                                   uint32_t n, uint32_t c, ckks_privft_model **out);
ckks_status ckks_privft_model_destroy(ckks_privft_model *model);
#define CKKS_PRIVFT_POLY_SOFTMAX 1u
/* bag: ciphertexts, count = batch * K ([b][k] order), level L, all with the same scale.
 * w_host: [batch] token counts (plaintext).  scores: count = batch, capacity >=
 * L-3 (L-4 with POLY_SOFTMAX).  Sequence (A14-A20):
 *   a_j = sum_k HMULPLAIN(ct_k, P^H_{j,k}); rescale; TotalSum;
 *   h_j = rescale(a_j * llround(Delta / w));  s = rescale(sum_j HMULPLAIN(h_j, P^O_j));
 *   POLY_SOFTMAX: g = rescale(s*s + 4 s) + 2, scale *= 8   (= s^2/8 + s/2 + 1/4) */
/* The v.H step alone ("a_j = sum_k HMULPLAIN(ct_k, P^H_{j,k})"; row a8): out (count
 * batch * n ciphertexts, capacity >= L) receives, at level L and scale bag.scale * H.scale,
 * out[b*n + j] = sum_k bag[b*K + k] (x) P^H_{j,k} -- no rescale.  Same kernels as the first step
 * of ckks_privft_infer (tensor-core byte-plane chunk-dot unless CKKS_CHUNKDOT_TC=0 at model
 * creation). */
ckks_status ckks_privft_chunkdot(ckks_ctx *ctx, const ckks_privft_model *model, const ckks_buf *bag, uint32_t batch,
                                 ckks_buf *out);
ckks_status ckks_privft_infer(ckks_ctx *ctx, const ckks_privft_model *model, const ckks_buf *bag,
                              const uint32_t *w_host, uint32_t batch, uint32_t flags, ckks_buf *scores);
/* The same inference from and to HOST memory (the client/server boundary of P:203-215):
 *   bag_host   : [batch * K][2][L][N] uint64, NTT form, canonical (a ckks_buf with capacity L),
 *                all at scale bag_scale; page-locked memory lets the upload run asynchronously.
 *   scores_host: receives [batch][2][lo][N] uint64 (NTT form), lo = L-4 with POLY_SOFTMAX
 *                else L-3; *scores_scale / *scores_level (optional) receive its scale / level.
 * Stream-ordered and ASYNCHRONOUS: the call returns after enqueueing; the host buffers must
 * stay valid and scores_host is complete only after ckks_sync(ctx).  The upload runs on a
 * context-owned copy stream into one of two device staging buffers (alternating per call),
 * so consecutive calls overlap the next batch's upload with this batch's compute, and a
 * batch of >= 2 queries runs as two halves (the second half uploads while the first
 * computes); compute,
 * the result download and every kernel stay on the context stream.  Errors as
 * ckks_privft_infer, plus CKKS_E_OOM for the staging buffers. */
ckks_status ckks_privft_infer_host(ckks_ctx *ctx, const ckks_privft_model *model, const uint64_t *bag_host,
                                   double bag_scale, const uint32_t *w_host, uint32_t batch, uint32_t flags,
                                   uint64_t *scores_host, double *scores_scale, uint32_t *scores_level);
/* Block the host until every call enqueued on the context stream has completed. */
ckks_status ckks_sync(ckks_ctx *ctx);

/* ---- PrivFT encrypted training step (Alg "GDMiniBatchTraining" P:312-332,
 * P:307 "HMUL is used instead of HMULPLAIN ... a number of mask and shift operations") ----
 * Encrypted model: H count n, H_j slot i = H[i][j] (vertical packing, one chunk:
 * m <= N/2); O count n, O_j slot i = O[j][i] for i < c (horizontal).  Minibatch: bags count
 * E (one chunk each, level l0 = model level >= 10), w_host[E] token counts, y_host[E] labels
 * (plaintext to the server).  Per example (readings T1-T6 in DESIGN.md):
 *   a_j = TotalSum(rescale(HMUL(v, H_j))); h_j = rescale(a_j * llround(Delta / w))
 *   s = rescale(relin(sum_j h_j (x) O_j));  g = rescale(s^2 + 4 s) + 2, scale *= 8
 *   e = rescale(HMULPLAIN(g - onehot(y), mask_{<c}))
 *   GO_j += rescale(HMUL(h_j, e));  GH_j += rescale(rescale(HMUL(v, TotalSum(rescale(HMUL(O_j, e))))) / w)
 * ckks_privft_train_grad -> GH (count n, level l0-8) and GO (count n, level l0-6), summed over
 * the minibatch; ranks holding different examples sum them with an all-gather +
 * ckks_modadd_gathered.  ckks_privft_train_update -> H - eta GH, O - eta GO, both at level
 * l0 - 9 (nine levels per minibatch); the product eta*G is brought onto the model's
 * scale by the constant's scale (T5). */
/* neg_onehot: count E plaintexts, slot y_e = -1 (else 0), encoded at level l0-4 with the scale
 * of g (returned by ckks_privft_train_plan); mask: count 1, slots < c = 1, level l0-4, any scale
 * (the class mask of the "mask and shift operations"). */
ckks_status ckks_privft_train_plan(const ckks_ctx *ctx, const ckks_buf *H, const ckks_buf *O, const ckks_buf *bags,
                                   double *g_scale, uint32_t *g_level);
ckks_status ckks_privft_train_grad(ckks_ctx *ctx, const ckks_buf *H, const ckks_buf *O, const ckks_buf *bags,
                                   const uint32_t *w_host, const uint32_t *y_host, uint32_t n_classes,
                                   const ckks_buf *neg_onehot, const ckks_buf *mask, ckks_buf *GH, ckks_buf *GO);
ckks_status ckks_privft_train_update(ckks_ctx *ctx, const ckks_buf *H, const ckks_buf *O, const ckks_buf *GH,
                                     const ckks_buf *GO, double eta, ckks_buf *H_out, ckks_buf *O_out);

#ifdef __cplusplus
}
#endif
#endif /* CKKS_H */
