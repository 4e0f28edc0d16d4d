// internal.h -- declarations shared by the kernel launchers (kernels.cu) and the host
// orchestration (ckks.cu).  Not part of the public ABI (see include/ckks.h).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "ntt.cuh"

// Address of (flat polynomial p, limb i): base + ((p * cap + i) << log_n).
struct PolyMap {
    u64 *base;
    u32 cap;
};

// Which prime each limb of a polynomial uses:
//   limb i < lq  -> prime (qoff + i);   limb i >= lq -> prime (sp + i - lq)   (special primes)
struct LimbSet {
    u32 n;     // limbs per polynomial processed
    u32 lq;    // how many of them are ciphertext primes
    u32 qoff;  // index of the first ciphertext prime
    u32 sp;    // table index of the first special prime (= L)
};

// Division by a runtime divisor d via a precomputed multiplier (Granlund-Montgomery):
// x / d = (umulhi(x, m) + x) >> s for every 32-bit x.  m == 0 (not prepared on the host)
// falls back to the hardware-less integer division sequence.
struct FDiv {
    u32 d = 1, m = 0, s = 0;
    __host__ __device__ __forceinline__ u32 div(u32 x) const
    {
#ifdef __CUDA_ARCH__
        if (m) return (u32)(((unsigned long long)__umulhi(x, m) + x) >> s);
#endif
        return x / d;
    }
    __host__ __device__ __forceinline__ u32 mod(u32 x) const { return x - div(x) * d; }
};
inline FDiv make_fdiv(u32 d)
{
    FDiv f;
    f.d = d;
    u32 s = 0;
    while ((1ull << s) < d) ++s;
    f.s = s;
    f.m = (u32)((((1ull << 32) * ((1ull << s) - d)) / d) + 1);
    return f;
}

// Optional per-kernel CUDA-event timing (ckks_profile_*): when enabled, every launch is
// bracketed by events on the launching stream and durations accumulate per kernel name.
struct Prof;
// algorithmic work of one launch: radix-2 butterflies on the integer pipe, 64x64-bit modular
// MACs/products, bytes, and radix-2 butterflies on the FP64 pipe (ntt.cuh FP64 mode)
struct Work {
    double bfly, mac, bytes, fbfly = 0, fmac = 0;  // fmac: modular MACs on the FP64 pipe
};
struct ProfTotal {
    double ms = 0, bfly = 0, mac = 0, bytes = 0, fbfly = 0, fmac = 0;
    unsigned long long launches = 0;
};
void prof_begin(Prof *p, cudaStream_t st, const char *name, Work w);
void prof_end(Prof *p, cudaStream_t st);

Prof *prof_create();
void prof_destroy(Prof *p);
void prof_enable(Prof *p, bool on);
void prof_collect(Prof *p);
void prof_reset(Prof *p);
#include <map>
#include <string>
const std::map<std::string, ProfTotal> &prof_totals(Prof *p);

struct Launch {
    const Tables *tb;
    cudaStream_t st;
    unsigned long long *counter;  // kernel launch counter
    Prof *prof;                   // nullptr or a profiler (enabled state checked inside)
    const u64 *hprimes;           // host copy of the prime table (index as tb->mod)
    cudaStream_t aux = nullptr;   // second stream: integer-pipe work concurrent with FP64-pipe work
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    u64 *split = nullptr;         // scratch for digit-split key-switch launches (mac_launch)
    size_t split_words = 0;
    u32 n_sm = 148;               // cudaDevAttrMultiProcessorCount of the context's device
    bool key_compact = false;     // switching-key limbs of FP64-mode primes (all < 2^40) stored compact
};

// enqueue one kernel launch with optional profiling events and the launch counter
#define KLAUNCH(L, NAME, WORK, ...)                   \
    do {                                              \
        prof_begin((L).prof, (L).st, NAME, WORK);     \
        __VA_ARGS__;                          \
        prof_end((L).prof, (L).st);           \
        ++*(L).counter;                       \
    } while (0)

// ---- NTT family (ntt.cuh geometry) -------------------------------------------------
// forward: coefficient -> NTT (bit-reversed), canonical output; src/dst may alias.
void launch_ntt_fwd(const Launch &L, PolyMap src, PolyMap dst, u32 npolys, LimbSet ls);
// inverse: NTT -> coefficient; if perm != nullptr the input is read as src[perm[k]]
// (NTT-domain Galois automorphism fused into the load).  dst may alias src iff perm == nullptr.
void launch_ntt_inv(const Launch &L, PolyMap src, PolyMap dst, u32 npolys, LimbSet ls, const u32 *perm);

// Broadcast NTT + subtract/multiply epilogue (rescale, Eq. 1; ModDown, A7):
//   for p < npolys, i < nt:  y = NTT_{q_i}( X[p] mod q_i )
//   out[p][i] = [base[p][i]] + (x[p][i] - y) * C_i   (mod q_i)
// X: coefficient-form limb per polynomial at X + p*x_stride*N (residues mod prime x_prime).
// base (optional, base.base == nullptr -> none) is read through base_perm when given and
// only for even p (c0) when base_c0_only.  scratch: npolys * nt * N words.
// Targets are global limb indices toff .. toff+nt-1 (x, out, base, consts and primes all
// indexed globally; scratch locally).
// Fused ModDown + rescale (T != nullptr, reading A7): X is z = [P d + acc]_{q_{l-1}} (coefficient form)
// and T the second CRT digit, so y = NTT_{q_i}([X + q_{l-1} T]_{q_i}) with qlc[i] = (q_{l-1} mod q_i);
// out = (x - y) C_i + base bconsts_i.
void launch_bcast_submul(const Launch &L, const u64 *X, u32 x_stride, u32 x_prime, u32 npolys, u32 nt, u32 toff,
                         u64 *scratch, PolyMap x, PolyMap out, const ulonglong2 *consts, PolyMap base,
                         const u32 *base_perm, bool base_c0_only, PolyMap acc = PolyMap{nullptr, 0},
                         const u64 *T = nullptr, const ulonglong2 *qlc = nullptr, const ulonglong2 *bconsts = nullptr,
                         const double2 *qlcf = nullptr);
// fused ModDown + rescale tail (two launches): z[p] = INTT(P d[p][l-1] + acc[p][l-1] mod q_{l-1}),
// T[p] = (INTT(acc[p][P]) - z[p]) q_{l-1}^{-1} mod P; acc's P limb (index acc_cap - 1) is overwritten
void launch_fr_tail(const Launch &L, const u64 *d, u32 d_cap, u64 *acc, u32 acc_cap, u64 *z, u64 *T, u32 np,
                    u32 lm1, u32 sp, ulonglong2 pm, ulonglong2 qinv);

// Key switch, per-limb digits (alpha = 1), one special prime (readings A6-A9):
//   D   : [cnt][l][N] coefficient-form digits (canonical mod q_j)
//   I   : scratch [cnt][T][l][N]   phase-1 (column) outputs of NTT_{q_t}(D_j mod q_t)
//   din : NTT-form input polynomial (digit j == t is taken from it directly): PolyMap with
//         one poly per ciphertext, read through perm when perm != nullptr
//   key : [Lk][2][Lk+1][N] NTT form;  ext: [cnt][2][l+1][N] output accumulators
// Targets t0 .. t0+T-1 (t == l means the special prime).
// D: digit j of ciphertext c (chunk-local) at ((j / dw) * dcnt + c0 + c) * dw + j % dw limbs.
// INTT of the l digits of cnt polynomials (src, Galois gather `perm`) fused with the ModUp
// column phase for targets t0..t0+T-1 (I layout as launch_ks_modup_cols with dw = l); Dtmp
// ([cnt][l][N]) holds the row-phase intermediate.  The coefficient-form digits are not stored.
// launch_ntt_inv (source limb, ls.n = 1 per polynomial; row phase into tmp, which may be src)
// fused with launch_bcast_submul's column phase: same result as the two calls in sequence.
void launch_inv_bcast_submul(const Launch &L, PolyMap src, PolyMap tmp, LimbSet ls, u32 npolys, u32 nt, u32 toff,
                             u64 *scratch, PolyMap x, PolyMap out, const ulonglong2 *consts, PolyMap base,
                             const u32 *base_perm, bool base_c0_only, PolyMap acc, bool rows_done = false);
void launch_inv_modup(const Launch &L, PolyMap src, u64 *Dtmp, u32 cnt, u32 l, const u32 *perm, u32 t0, u32 T,
                      u64 *I, u32 sp, bool rows_done = false);
// Compact switching-key rows (the FP64 inner product reads 5 of every 8 key bytes): each row
// (digit, b|a, limb) of a listed limb (q < 2^40) becomes a u32 plane of the low words followed by
// a u8 plane of the high bytes inside its own N-word slot; inverse = expand back.  tmp: scratch of
// nrows * N words (one limb's rows at a time).
void launch_key_compact(const Launch &L, u64 *key, const u32 *limbs_host, u32 nl, u32 nrows, u32 Lk1, bool inverse,
                        u64 *tmp);
// HMULT tensor product + the relinearisation digits' inverse row phase (k_tensor_inv_rows):
// out = (a0 b0, a0 b1 + a1 b0), d2 = a1 b1 (NTT form), dr = row phase of INTT(d2) ([cnt][l][N])
void launch_tensor_inv_rows(const Launch &L, PolyMap a, PolyMap b, PolyMap out, PolyMap d2, PolyMap dr, u32 nct,
                            u32 l);
// the inverse NTT's column phase alone, in place (data holds the row-phase output)
void launch_ntt_inv_cols(const Launch &L, PolyMap data, u32 npolys, LimbSet ls);
// jw0 / nj: only digits [jw0, jw0 + nj) (nj = 0: all l) -- the pipelined limb-sharded key switch
void launch_ks_modup_cols(const Launch &L, const u64 *D, u32 dw, u32 dcnt, u32 c0, u32 l, u32 cnt, u32 t0, u32 T,
                          u64 *I, u32 sp, u32 jw0 = 0, u32 nj = 0);
// p_inv_rows: apply the INTT row phase to the special-prime target's output rows (ModDown
// fusion); returns whether it was applied (integer classes without digit split only).
// jw0 / jw1: digit window (jw1 = 0: all); accum: ext += the window's sum (mod q_t) instead of =
bool launch_ks_mac(const Launch &L, const u64 *I, PolyMap din, const u32 *perm, const u64 *key, u32 Lk, u32 l,
                   u32 cnt, u32 t0, u32 T, u64 *ext, u32 sp, bool p_inv_rows = false, u32 jw0 = 0, u32 jw1 = 0,
                   bool accum = false, u32 lay_t0 = 0, u32 lay_T = 0);  // lay_T: I holds targets [lay_t0, +lay_T)

// ---- elementwise (limb-wise modular arithmetic) ---------------------------
// All act on npolys polynomials x l limbs (limb i mod prime qoff + i).
enum ElemOp { EL_ADD = 0, EL_SUB = 1 };
void launch_addsub(const Launch &L, PolyMap a, PolyMap b, PolyMap out, u32 npolys, u32 l, int op);
// out[p] = a[p] * b[p / b_div] (HMULPLAIN with b_div = polys per ciphertext -> plaintext broadcast)
void launch_mul_poly(const Launch &L, PolyMap a, PolyMap b, u32 b_div, u32 b_mod, PolyMap out, u32 npolys, u32 l);
// out[p] = a[p] + b[p / b_div] for p % a_stride == 0 only (c0 + pt), other polys copied
void launch_add_plain(const Launch &L, PolyMap ct, PolyMap pt, u32 pt_bcast, PolyMap out, u32 nct, u32 l);
// out[p] = a[p] * c_i  (consts[i] = (c_i, shoup))
void launch_mul_scalar(const Launch &L, PolyMap a, PolyMap out, u32 npolys, u32 l, const ulonglong2 *consts);
// c0 of every ciphertext += c_i
void launch_add_scalar_c0(const Launch &L, PolyMap ct, PolyMap out, u32 nct, u32 l, const u64 *consts);
// HMUL tensor: (d0, d1) -> out polys 0,1 of each ct; d2 -> d2map (one poly per ct)
// pairing: output p uses a[(p / adiv) % amod] and b[(p / bdiv) % bmod] (mod 0 = no wrap)
void launch_tensor(const Launch &L, PolyMap a, PolyMap b, PolyMap out, PolyMap d2, u32 nct, u32 l, u32 adiv = 1,
                   u32 amod = 0, u32 bdiv = 1, u32 bmod = 0);
// int64 small polynomials -> residues of every limb in ls:  out[p][i] = e[p] mod prime(i)
void launch_from_signed(const Launch &L, const int64_t *e, PolyMap out, u32 npolys, LimbSet ls);
// generic copy of limbs
void launch_copy(const Launch &L, PolyMap src, PolyMap dst, u32 npolys, u32 l);
// dst[p][i][k] = src[p][i][perm[k]] over npolys x l limbs (NTT-domain automorphism)
void launch_permute(const Launch &L, PolyMap src, PolyMap dst, u32 npolys, u32 l, const u32 *perm);
// switching-key assembly in NTT form (A9, f2): for digit j < dnum, limb i < Lk+K:
//   b = -a*s + e_j + [i in digit j] (P mod q_i) sfrom ;   key[j][0][i] = b, key[j][1][i] = a
// a, e already NTT form: a [dnum][Lk+K][N], e [dnum][Lk+K][N]; s, sfrom [Lk+K][N]
void launch_keygen_b(const Launch &L, const u64 *a, const u64 *e, const u64 *s, const u64 *sfrom,
                     const u64 *pmod, u64 *key, u32 Lk, u32 K, u32 alpha, u32 dnum);
// out = a*s + b mod q (per limb), polynomials: a, b [l][N] ; used by decrypt / pk
void launch_mul_add(const Launch &L, PolyMap a, PolyMap s, u32 s_bcast, PolyMap b, PolyMap out, u32 npolys, u32 l,
                    int negate_prod);
// out = sum over R gathered copies (stride per copy = stride_words) mod q
void launch_modadd_gathered(const Launch &L, const u64 *g, size_t stride_words, u32 R, PolyMap out, u32 npolys,
                            u32 l);

// PrivFT chunk-dot: for b < B, jj < J (outputs), poly in {0,1}:
//   out[b*J + jj] = sum_{k<K} ct[b*K + k] (x) pt[jj*K + k]      (pointwise, NTT domain, mod q_i)
// ct: ciphertexts (2 polys, stride ct_cap), pt: plaintexts (1 poly, stride pt_cap),
// out: ciphertexts (stride out_cap); all at level l.
void launch_chunkdot(const Launch &L, const u64 *ct, u32 ct_cap, const u64 *pt, u32 pt_cap, u64 *out, u32 out_cap,
                     u32 B, u32 J, u32 K, u32 l);
// per-ciphertext scalar multiply: out[c] = ct[c] * consts[c * l + i] (consts: (value, shoup))
void launch_mul_scalar_per_ct(const Launch &L, PolyMap a, PolyMap out, u32 nct, u32 l, const ulonglong2 *consts);

// ---- hybrid key switching -------------------------------------------------
// ModUp: X[c][d][s] = NTT_{m_s}(conv_{D_d}(D[c])) for every extended slot s outside digit d
// (s < l: q_s, s = l + k: p_k); yinv [beta][alpha], conv [beta][alpha][ne].
// cols_only: leave the slots after the NTT column phase (lazy doubles) for launch_hyb_ip_fused
void launch_hyb_modup(const Launch &L, const u64 *D, u64 *X, const ulonglong2 *yinv, const u64 *conv, u32 cnt, u32 l,
                      u32 Lq, u32 K, u32 alpha, u32 beta, u32 ne, bool cols_only = false);
// the inner product on the k_ks_mac pipeline (hybrid mode): row phase of every digit's slot NTT +
// FP64 multiply-accumulate with the key, the accumulators in registers; requires hyb_fused_ip_ok
bool hyb_fused_ip_ok(const Launch &L, u32 l, u32 Lq, u32 K);
// zrs != nullptr (fused ModDown + rescale): targets l-1 .. l+K-1 leave with the INTT row phase
// applied, target l-1 after z = P zbase_{l-1} + acc_{l-1} (zrs: the launch_hyb_moddown_rs constants)
void launch_hyb_ip_fused(const Launch &L, const u64 *X, PolyMap din, const u32 *perm, const u64 *key, u64 *ext, u32 cnt,
                         u32 l, u32 Lq, u32 K, u32 alpha, u32 beta, u32 ne, PolyMap zbase = PolyMap{nullptr, 0},
                         const ulonglong2 *zrs = nullptr);
// inner product over digits: ext [cnt][2][ne][N]; digit-own slots taken from din (via perm)
void launch_hyb_ip(const Launch &L, const u64 *X, PolyMap din, const u32 *perm, const u64 *key, u64 *ext, u32 cnt,
                   u32 l, u32 Lq, u32 K, u32 alpha, u32 beta, u32 ne);
// ModDown: INTT of the special slots, fast base conversion to q_0..q_{l-1}, NTT, then
// out_i = [base_i] + (acc_i - conv_i) P^{-1}   (Y: scratch [npolys][l][N])
void launch_hyb_moddown(const Launch &L, u64 *ext, u64 *Y, const ulonglong2 *pyinv, const u64 *conv, u32 npolys, u32 l,
                        u32 Lq, u32 K, u32 ne, PolyMap out, PolyMap base, const u32 *base_perm, bool base_c0_only,
                        const ulonglong2 *pinv, PolyMap acc = PolyMap{nullptr, 0});

// Fused hybrid ModDown + RESCALE (reading A7 for K > 1; bit-exact with the two steps by
// linearity of the NTT): with h = base + (acc - NTT(Y)) P^{-1} the sequential ModDown result and
// g = INTT(h_{l-1}) = (INTT(P base_{l-1} + acc_{l-1}) - Y_{l-1}) P^{-1} mod q_{l-1} its last limb,
//   out_i = base_i q_{l-1}^{-1} + (acc_i - NTT(Y_i + [P]_{q_i} g)) (P q_{l-1})^{-1}    (i < l-1)
// rs: [3][l] Shoup pairs: [0][i] = (P q_{l-1})^{-1} mod q_i, [1][i] = q_{l-1}^{-1} mod q_i,
// [2][i] = (P mod q_i, -) for i < l-1; [0][l-1] = P mod q_{l-1}, [1][l-1] = P^{-1} mod q_{l-1}.
// base: (d0, d1) of the HMULT tensor, unpermuted; Y: scratch [npolys][l-1][N].
void launch_hyb_moddown_rs(const Launch &L, u64 *ext, u64 *Y, const ulonglong2 *pyinv, const u64 *conv, u32 npolys,
                           u32 l, u32 Lq, u32 K, u32 ne, PolyMap out, PolyMap base, const ulonglong2 *rs,
                           bool rows_done = false);

// out[q][k] = sum_{r<R} g[r*rs + q*qs][k]  (q < nout_ct ciphertexts of np polys, l limbs)
void launch_sum_strided(const Launch &L, PolyMap g, PolyMap out, u32 nout_ct, u32 np, u32 l, u32 R, u32 rs, u32 qs);

// ---- batched GPU encode / decode (codec.cu) -------------------------------
struct CodecTabs {
    const double2 *w;    // [N]  e^{-2 pi i m / N}
    const double2 *tw;   // [N]  e^{-i pi k / N}
    const u32 *slot;     // [N]  j | conj << 31 : which slot feeds FFT bin s (see codec.cu)
};
// per-limb constants of the centred CRT lift at one level (reading A33)
struct CrtConst {
    u64 qh_lo, qh_hi;     // (Q / q_i) mod 2^128
    u64 qhinv, qhinv_s;   // (Q / q_i)^{-1} mod q_i, Shoup companion
    double inv_q;         // 1 / q_i
    double pad_;
};
// z [cnt][n_slots] complex (device) -> out [cnt][l] COEFFICIENT form residues (caller NTTs);
// Y: scratch [cnt][N] double2; overflow: device flag set on an int64-overflowing coefficient.
void launch_encode(const Launch &L, const CodecTabs &tb, const double2 *z, u32 n_slots, double scale, u32 cnt,
                   double2 *Y, PolyMap out, u32 l, int *overflow);
// coef [cnt][l][N] coefficient form -> z [cnt][n_slots] complex (device)
void launch_decode(const Launch &L, const CodecTabs &tb, const u64 *coef, u32 l, const CrtConst *crt, u64 Q_lo,
                   u64 Q_hi, u32 cnt, double2 *Y, double2 *z, u32 n_slots, double scale);

// ---- fused peer-memory modular all-reduce (p2p.cu) ------------------------
#define CKKS_MAX_PEERS 8
// rank's contiguous share [row0, row0 + nrows) of `rows` limb rows (sizes differ by <= 1)
void p2p_slice(u32 rows, u32 R, u32 rank, u32 *row0, u32 *nrows);
// in[r], out[r]: rank r's buffer (mapped into this process), layout [npolys][cap][N], level limbs
void launch_p2p_modsum(const Launch &L, const u64 *const *in, u64 *const *out, u32 R, u32 rank, u32 npolys, u32 level,
                       u32 cap);

// ---- PrivFT v.H chunk-dot on the tensor cores (chunkdot_tc.cu) ------------------------------
u32 chunkdot_tc_planes(u64 q);  // byte planes of residues mod q
// u32 words of the H fragment layout for limbs 0..l-1
size_t chunkdot_tc_words(const u64 *hprimes, u32 l, u32 J, u32 K, u32 log_n);
bool chunkdot_tc_supported(const u64 *hprimes, u32 l, u32 B, u32 K);
// H: [J*K] plaintexts (stride h_cap) -> Hf (mma B-fragment byte planes, chunkdot_tc.cu)
void launch_chunkdot_prep_h(const Launch &L, const u64 *H, u32 h_cap, u32 *Hf, u32 l, u32 J, u32 K);
// out[b*J + j] = sum_k ct[b*K + k] (x) H[j*K + k]  over limbs 0..l-1 (same result as launch_chunkdot)
void launch_chunkdot_tc(const Launch &L, const u64 *ct, u32 ct_cap, const u32 *Hf, u64 *out, u32 out_cap, u32 B,
                        u32 J, u32 K, u32 l);

// ---- alpha = 1 key switch fused on thread-block clusters (ks_cluster.cu) ---------------------
bool ks_cluster_supported(const Launch &L);   // this N has a cluster configuration resident
size_t ks_cluster_part_words(const Launch &L);  // partial-sum scratch (words)
// same contract as launch_ks_modup_cols + launch_ks_mac for the FP64-mode targets listed in tmap
// (t <= l, t == l is P), writing ext [cnt][2][l+1][N]; key limbs of those targets in MAC layout.
void launch_ks_cluster(const Launch &L, cudaStream_t st, const u64 *D, u32 dw, u32 dcnt, u32 dc0, PolyMap din,
                       const u32 *perm, const u64 *key, u32 Lk, u32 l, u32 cnt, const u32 *tmap_dev,
                       const u32 *tmap_host, u32 nT, u64 *ext, double *part, u32 *ctr, u32 sp);
// switching key [2 nkeyrows][Lk1][N]: the listed limbs to (inverse: from) the MAC layout
void launch_key_mac_layout(const Launch &L, u64 *key, const u32 *limbs, u32 nl, u32 nkeyrows, u32 Lk1, bool inverse);
bool prof_on(const Prof *p);
