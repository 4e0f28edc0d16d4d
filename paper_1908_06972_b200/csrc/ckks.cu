// ckks.cu -- libckks C ABI (include/ckks.h): context, tables, keys, and the host
// orchestration of the sm_100a kernels in kernels.cu.
//
// Every arithmetic step of the hot path runs in the kernels; this file validates
// arguments, sizes scratch, enqueues launches on the context stream and keeps the
// scale/level bookkeeping (reading A13).
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "ckks.h"
#include "hostmath.h"
#include "internal.h"

// NVTX ranges per composer stage and per op (header-only nvtx3: inert without a profiler)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

namespace {
struct DevBuf {
    void *p = nullptr;
    size_t bytes = 0;
};
}  // namespace

struct FrLevel {
    ulonglong2 *c1 = nullptr;   // [L+K]: (P q_{l-1})^{-1} mod q_i
    ulonglong2 *qlc = nullptr;  // [L+K]: q_{l-1} mod q_i
    double2 *qlcf = nullptr;    // [L+K][2]: (c, c/q_i), (2^31 c mod q_i, .../q_i), c = q_{l-1} mod q_i (FP64 limbs)
    ulonglong2 pm_last{}, qinv_p{};  // P mod q_{l-1};  q_{l-1}^{-1} mod P (Shoup companions)
};

struct ckks_ctx {
    int device = 0;
    cudaStream_t st = nullptr;
    u32 log_n = 0, N = 0, L = 0;
    u32 K = 1, alpha = 1, dnum = 0;  // special primes, limbs per key-switch digit, digits
    std::vector<u64> primes;  // q_0..q_{L-1}, p_0..p_{K-1}
    double scale = 0;
    // device tables
    ModC *d_mod = nullptr;
    ulonglong2 *d_psi = nullptr, *d_ipsi = nullptr, *d_ninv = nullptr;
    double2 *d_psif = nullptr, *d_ipsif = nullptr;  // FP64-mode twiddles (ntt.cuh)
    ulonglong2 *d_rinv = nullptr;  // [(L+K)][(L+K)]: row l, entry k = q_{l-1}^{-1} mod q_k
    ulonglong2 *d_pinv = nullptr;  // [L+K]: P^{-1} mod q_i  (P = p_0 ... p_{K-1})
    u64 *d_pmod = nullptr;         // [L+K]: P mod q_i (0 for the special limbs)
    ulonglong2 *d_pyinv = nullptr; // [K]: (P/p_k)^{-1} mod p_k          (hybrid ModDown)
    u64 *d_pconv = nullptr;        // [K][L]: (P/p_k) mod q_i            (hybrid ModDown)
    struct HybLevel {
        ulonglong2 *yinv = nullptr;  // [beta][alpha]
        u64 *conv = nullptr;         // [beta][alpha][ne]
        ulonglong2 *rs = nullptr;    // [3][l] fused ModDown + rescale constants (launch_hyb_moddown_rs)
    };
    std::map<u32, HybLevel> hyb;     // per level: hybrid ModUp constants
    std::map<u32, FrLevel> fr;       // per level: fused ModDown + rescale constants
    // batched GPU codec (f4): FFT twiddles, twist, slot map; per-level CRT constants
    double2 *d_fft_w = nullptr, *d_fft_tw = nullptr;
    u32 *d_slot = nullptr;
    int *d_enc_overflow = nullptr;
    struct CrtLevel {
        CrtConst *c = nullptr;
        u64 Q_lo = 0, Q_hi = 0;
    };
    std::map<u32, CrtLevel> crt;
    std::map<void *, void *> ipc;  // mapped peer pointer -> base of its IPC mapping
    Tables tb{};
    // keys (NTT form)
    u64 *sk = nullptr;   // [L+K][N]
    u64 *pk = nullptr;   // [2][L][N]  (b, a)
    u64 *rlk = nullptr;  // [dnum][2][L+K][N]
    std::map<u64, u64 *> gk;
    std::map<u64, u32 *> perms;
    // cluster key switch (ks_cluster.cu): on for alpha = K = 1 at N >= 2^12; the FP64-mode limbs
    // of every switching key are then held in its MAC layout (as doubles)
    bool ksc = false;
    u32 *d_kc_limbs = nullptr;        // FP64-mode key limbs (indices into L+K)
    u32 n_kc_limbs = 0;
    std::map<u64, u32 *> kc_tmaps;    // (l, t_lo, t_hi) -> FP64-mode target list
    u32 *d_kc_ctr = nullptr;          // segment completion counters (zero between launches)
    size_t kc_ctr_n = 0;
    std::map<std::string, DevBuf> bufs;  // named scratch
    std::string err;
    unsigned long long launches = 0;
    Prof *prof = nullptr;
    std::vector<std::string> prof_names;
    cudaStream_t aux = nullptr;  // concurrent integer-pipe work (see mac_impl)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // host-buffer inference (ckks_privft_infer_host): upload stream, two bag staging buffers
    cudaStream_t up = nullptr;
    cudaEvent_t up_done[2][2] = {}, stage_free[2][2] = {};  // [staging buffer][batch half]
    u32 stage_next = 0;
    u32 n_sm = 148;
    // compact switching keys (launch_key_compact): the FP64-mode limbs (all < 2^40) of every key
    bool kcomp = false;
    std::vector<u32> kcomp_limbs;
    Launch lc()
    {
        Launch l{&tb, st, &launches, prof, primes.data(), aux, ev_fork, ev_join};
        l.n_sm = n_sm;
        l.key_compact = kcomp;
        return l;
    }
};

struct ckks_privft_model {
    ckks_ctx *ctx = nullptr;
    ckks_buf H{}, O{};
    bool owned = false;
    u32 m = 0, n = 0, c = 0, K = 0;
    u32 *Hf = nullptr;  // H in tensor-core fragment byte planes (chunkdot_tc.cu); nullptr: CUDA-core chunk-dot
};

namespace {

ckks_status fail(ckks_ctx *c, ckks_status s, const std::string &msg)
{
    if (c) c->err = msg;
    return s;
}

#define CUDA_TRY(ctx, call)                                                                  \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess) return fail(ctx, CKKS_E_CUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
    } while (0)

ckks_status check_launch(ckks_ctx *c)
{
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(c, CKKS_E_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
    return CKKS_OK;
}

// named, grow-only scratch buffer (cudaFree synchronises before reuse of old memory)
u64 *need(ckks_ctx *c, const char *name, size_t words)
{
    DevBuf &b = c->bufs[name];
    const size_t bytes = words * sizeof(u64);
    if (b.bytes < bytes) {
        if (b.p) cudaFree(b.p);
        b.p = nullptr;
        b.bytes = 0;
        if (cudaMalloc(&b.p, bytes) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        b.bytes = bytes;
    }
    return static_cast<u64 *>(b.p);
}

bool valid_buf(const ckks_ctx *c, const ckks_buf *b, u32 n_polys)
{
    return b && b->data && b->count >= 1 && b->n_polys == n_polys && b->level >= 1 && b->level <= c->L &&
           b->capacity >= b->level;
}

PolyMap pm(const ckks_buf *b) { return PolyMap{b->data, b->capacity}; }
// c0 / c1 of every ciphertext as a one-poly-per-ciphertext map
PolyMap pm_c(const ckks_buf *b, u32 which, u32 N)
{
    return PolyMap{b->data + (size_t)which * b->capacity * N, 2 * b->capacity};
}
LimbSet qlimbs(const ckks_ctx *c, u32 l) { return LimbSet{l, l, 0, c->L}; }
LimbSet extlimbs(const ckks_ctx *c) { return LimbSet{c->L + c->K, c->L, 0, c->L}; }
size_t key_words(const ckks_ctx *c) { return (size_t)c->dnum * 2 * (c->L + c->K) * c->N; }

long long llround_checked(double x, bool &ok)
{
    ok = std::isfinite(x) && std::fabs(x) < 9.2e18;
    return ok ? std::llround(x) : 0;
}

u64 residue_of(long long v, u64 q)
{
    if (v >= 0) return (u64)v % q;
    u64 r = (u64)(-(v + 1)) % q;  // -(v+1) >= 0 avoids overflow at LLONG_MIN
    return q - 1 - r;
}

const u32 *get_perm(ckks_ctx *c, u64 kappa)
{
    auto it = c->perms.find(kappa);
    if (it != c->perms.end()) return it->second;
    std::vector<u32> h(c->N);
    const u64 two_n = 2ull * c->N;
    for (u32 k = 0; k < c->N; ++k) {
        u64 e = (2ull * hm::bitrev(k, c->log_n) + 1) * kappa % two_n;  // odd
        h[k] = hm::bitrev((u32)((e - 1) / 2), c->log_n);
    }
    u32 *d = nullptr;
    if (cudaMalloc(&d, c->N * sizeof(u32)) != cudaSuccess) return nullptr;
    cudaMemcpy(d, h.data(), c->N * sizeof(u32), cudaMemcpyHostToDevice);
    c->perms[kappa] = d;
    return d;
}

u64 galois_elt(const ckks_ctx *c, int32_t step)
{
    const u64 two_n = 2ull * c->N;
    u64 k = hm::powmod(5, (u64)std::llabs((long long)step), two_n);
    if (step < 0) {
        // inverse of an odd number mod 2N: 5 has order N/2, so 5^{-s} = 5^{N/2 - s mod N/2}
        const u64 ord = c->N / 2;
        k = hm::powmod(5, (ord - ((u64)std::llabs((long long)step) % ord)) % ord, two_n);
    }
    return k;
}

// NAF digits of s in [0, t), increasing |2^i|; the digit of magnitude t is the identity (A10, A31)
std::vector<int32_t> rotation_steps(const ckks_ctx *c, int32_t steps)
{
    const long long t = c->N / 2;
    long long s = ((long long)steps % t + t) % t;
    std::vector<int32_t> out;
    for (int i = 0; s > 0; ++i, s >>= 1) {
        if (s & 1) {
            int d = 2 - (int)(s & 3);
            s -= d;
            if ((1ll << i) < t) out.push_back(d * (1 << i));
        }
    }
    return out;
}

// key-switch scratch budget per chunk (words); CKKS_KS_BUDGET_MB overrides (read per call
// so tests can force multi-chunk launch sequences)
size_t ks_budget_words()
{
    const char *e = std::getenv("CKKS_KS_BUDGET_MB");
    // 2 GiB default: re-measured after the fused column kernels (C4 326 -> 322 ms/step vs 1 GiB;
    // 4 GiB no further gain, 768 MiB 335 ms)
    const size_t mb = e ? std::strtoull(e, nullptr, 10) : 2048;
    return (mb ? mb : 2048) << 17;
}

// Coefficient-form key-switch digits supplied by the caller (limb-sharded path): digit j
// of ciphertext c at ((j / dw) * dcnt + c) * dw + j % dw limbs from D.  D == nullptr: the
// digits are computed here (INTT of din).
struct KsDigits {
    const u64 *D;
    u32 dw, dcnt;
};

// The broadcast (ModDown / rescale) with the source limb's INTT column phase fused in: on when
// the fused column launch keeps >= 16 CTAs per SM (CKKS_INV_BCAST=0/1 forces off / on).
// Both fused column kernels loop over every target inside one CTA: worth it when the launch
// keeps >= 16 CTAs per SM, or >= 4 with at most 6 targets per CTA (measured over N = 2^12..2^16:
// batched C1 / C4 HMult -6 %, C2 neutral, 2^15 x 4 and a single 2^16 ciphertext slower).
bool fused_cols_on(size_t ctas, u32 targets, u32 n_sm)
{
    return ctas >= (size_t)n_sm * 16 || (targets <= 6 && ctas >= (size_t)n_sm * 4);
}

bool inv_bcast_on(const ckks_ctx *c, u32 npolys, u32 nt)
{
    const char *e = std::getenv("CKKS_INV_BCAST");
    if (e) return e[0] == '1';
    return fused_cols_on((size_t)npolys * ((size_t)1 << (c->log_n - c->log_n / 2)) / 16, nt, c->n_sm);
}

ckks_status keyswitch_cluster(ckks_ctx *c, PolyMap din, const u32 *perm, u32 cnt, u32 l, const u64 *key, u32 t_lo,
                              u32 t_hi, KsDigits dg, PolyMap out, PolyMap base, const u32 *base_perm,
                              bool base_c0_only, PolyMap acc);

// fused ModDown + rescale constants at level l (alpha = K = 1; cached per level)
const FrLevel *fr_level(ckks_ctx *c, u32 l)
{
    auto it = c->fr.find(l);
    if (it != c->fr.end()) return &it->second;
    const u64 P = c->primes[c->L], ql = c->primes[l - 1];
    std::vector<ulonglong2> c1(c->L + c->K, make_ulonglong2(0, 0)), qlc(c->L + c->K, make_ulonglong2(0, 0));
    for (u32 i = 0; i + 1 < l; ++i) {
        const u64 q = c->primes[i];
        const u64 v = hm::invmod(hm::mulmod(P % q, ql % q, q), q);  // (P q_{l-1})^{-1} mod q_i
        c1[i] = make_ulonglong2(v, hm::shoup(v, q));
        qlc[i] = make_ulonglong2(ql % q, hm::shoup(ql % q, q));
    }
    std::vector<double2> qlcf(2 * (c->L + c->K), make_double2(0, 0));
    for (u32 i = 0; i + 1 < l; ++i) {
        const u64 q = c->primes[i];
        if (q >= c->tb.f64_qmax) continue;
        const u64 c0 = ql % q, c1 = hm::mulmod(c0, (1ull << 31) % q, q);
        qlcf[2 * i] = make_double2((double)c0, (double)c0 / (double)q);
        qlcf[2 * i + 1] = make_double2((double)c1, (double)c1 / (double)q);
    }
    FrLevel f;
    const u64 pm = P % ql, qi = hm::invmod(ql % P, P);
    f.pm_last = make_ulonglong2(pm, hm::shoup(pm, ql));
    f.qinv_p = make_ulonglong2(qi, hm::shoup(qi, P));
    if (cudaMalloc(&f.c1, c1.size() * sizeof(ulonglong2)) != cudaSuccess ||
        cudaMalloc(&f.qlc, qlc.size() * sizeof(ulonglong2)) != cudaSuccess ||
        cudaMalloc(&f.qlcf, qlcf.size() * sizeof(double2)) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    cudaMemcpy(f.c1, c1.data(), c1.size() * sizeof(ulonglong2), cudaMemcpyHostToDevice);
    cudaMemcpy(f.qlc, qlc.data(), qlc.size() * sizeof(ulonglong2), cudaMemcpyHostToDevice);
    cudaMemcpy(f.qlcf, qlcf.data(), qlcf.size() * sizeof(double2), cudaMemcpyHostToDevice);
    return &(c->fr[l] = f);
}

// ---- key switch for target limbs [t_lo, t_hi) plus P -----------------------------------------
// out_t = base_t + ModDown(sum_j ModUp(d_j) * ksk_j)_t  (readings A6-A9), chunked over
// ciphertexts and target groups so the phase-1 intermediates stay within the budget.
// fuse_rescale (relinearisation only: full target range, base = out = the tensor's (d0, d1),
// no base_perm / acc): ModDown and the following RESCALE in one broadcast pass (reading A7),
// out receives level l - 1.
// rows_done: [cnt][l][N] already holding the row phase of INTT(din) (launch_tensor_inv_rows); the
// column phase then runs in place there and those buffers become the digits.
ckks_status keyswitch_range(ckks_ctx *c, PolyMap din, const u32 *perm, u32 cnt, u32 l, const u64 *key, u32 t_lo,
                            u32 t_hi, KsDigits dg, PolyMap out, PolyMap base, const u32 *base_perm,
                            bool base_c0_only, PolyMap acc = PolyMap{nullptr, 0}, bool fuse_rescale = false,
                            u64 *rows_done = nullptr)
{
    if (c->ksc && !fuse_rescale)
        return keyswitch_cluster(c, din, perm, cnt, l, key, t_lo, t_hi, dg, out, base, base_perm, base_c0_only, acc);
    const FrLevel *fr = fuse_rescale ? fr_level(c, l) : nullptr;
    if (fuse_rescale && !fr) return fail(c, CKKS_E_OOM, "fused rescale constants");
    Launch L = c->lc();
    L.split_words = (size_t)256 << c->log_n;
    L.split = need(c, "ks_split", L.split_words);
    if (!L.split) L.split_words = 0;
    const size_t n = c->N;
    // phase-1 intermediates per chunk (words).  The path is ALU-bound, so a slab that
    // spills from L2 costs one extra HBM write+read that overlaps the arithmetic; a larger
    // chunk buys parallelism (more targets per ks_mac launch) and fewer launches.
    const size_t budget = ks_budget_words();
    const u32 ntg = t_hi - t_lo + 1;        // target limbs incl. P
    const size_t per = (size_t)l * n;       // one (ciphertext, target) slab of I
    u32 T = (u32)std::max<size_t>(1, std::min<size_t>(ntg, budget / per));
    u32 cc = (u32)std::max<size_t>(1, std::min<size_t>(cnt, budget / (per * T)));
    const size_t dwords = (dg.D || rows_done) ? 0 : (size_t)cc * l * n;
    const size_t words = dwords + (size_t)cc * T * l * n + (size_t)cc * 2 * (l + 1) * n +
                         (size_t)cc * 2 * (t_hi - t_lo) * n;
    u64 *s = need(c, "ks", words);
    if (!s) return fail(c, CKKS_E_OOM, "key-switch scratch");
    u64 *D = s, *I = D + dwords, *ext = I + (size_t)cc * T * l * n, *S = ext + (size_t)cc * 2 * (l + 1) * n;
    const u32 end = (t_hi == l) ? l + 1 : t_hi;  // P is contiguous with a full target range
    for (u32 c0 = 0; c0 < cnt; c0 += cc) {
        const u32 nc = std::min(cc, cnt - c0);
        PolyMap dch{din.base + (size_t)c0 * din.cap * n, din.cap};
        const u64 *Dp = dg.D;
        u32 dw = dg.dw, dcnt = dg.dcnt, dc0 = c0;
        // digits' INTT fused with the ModUp column phase (one target group covering every target)
        const char *ime = std::getenv("CKKS_INV_MODUP");
        // (each CTA then loops over every target: only when the launch still has >= 16 CTAs per SM,
        // e.g. C4's 819-ciphertext chunks; a single C3 ciphertext keeps the per-target launch)
        const size_t inv_ctas = (size_t)nc * l * ((size_t)1 << (c->log_n - c->log_n / 2)) / 16;
        bool inv_modup = !Dp && end == l + 1 && t_lo == 0 && T >= ntg && !(ime && ime[0] == '0') &&
                         (fused_cols_on(inv_ctas, l + 1, c->n_sm) || (ime && ime[0] == '1'));
        const bool want_pinv = !fuse_rescale && inv_bcast_on(c, 2 * nc, t_hi - t_lo);
        bool p_rows = false;  // the inner product left the P limb's INTT row phase applied
        u64 *rd = rows_done ? rows_done + (size_t)c0 * l * n : nullptr;
        if (inv_modup) {
            launch_inv_modup(L, dch, rd ? rd : D, nc, l, perm, 0, l + 1, I, c->L, rd != nullptr);
            p_rows = launch_ks_mac(L, I, dch, perm, key, c->L, l, nc, 0, l + 1, ext, c->L, want_pinv);
        } else if (rd) {
            launch_ntt_inv_cols(L, PolyMap{rd, l}, nc, qlimbs(c, l));
            Dp = rd;
            dw = l;
            dcnt = nc;
            dc0 = 0;
        } else if (!Dp) {
            launch_ntt_inv(L, dch, PolyMap{D, l}, nc, qlimbs(c, l), perm);
            Dp = D;
            dw = l;
            dcnt = nc;
            dc0 = 0;
        }
        auto run = [&](u32 t0, u32 tn) {
            launch_ks_modup_cols(L, Dp, dw, dcnt, dc0, l, nc, t0, tn, I, c->L);
            launch_ks_mac(L, I, dch, perm, key, c->L, l, nc, t0, tn, ext, c->L);
        };
        if (!inv_modup) {
            for (u32 t0 = t_lo; t0 < end; t0 += T) run(t0, std::min(T, end - t0));
            if (end != l + 1) run(l, 1);
        }
        // ModDown (A7): INTT of the P limb, then out_i = base + (acc_i - NTT_i([acc]_P)) P^{-1}
        PolyMap och{out.base + (size_t)c0 * 2 * out.cap * n, out.cap};
        PolyMap bch = base.base ? PolyMap{base.base + (size_t)c0 * 2 * base.cap * n, base.cap} : base;
        PolyMap ach = acc.base ? PolyMap{acc.base + (size_t)c0 * 2 * acc.cap * n, acc.cap} : acc;
        if (fuse_rescale) {
            // x = P d + acc over {q_0..q_{l-1}, P}; y = [x]_{P q_{l-1}} from its two residues
            // z = [x]_{q_{l-1}} and acc_P (CRT: y = z + q_{l-1} T, T = (acc_P - z) q_{l-1}^{-1} mod P);
            // out_i = (acc_i - y) (P q_{l-1})^{-1} + d_i q_{l-1}^{-1}  mod q_i,  i < l - 1
            u64 *Z = need(c, "fr_z", (size_t)2 * nc * n), *Tt = need(c, "fr_t", (size_t)2 * nc * n);
            if (!Z || !Tt) return fail(c, CKKS_E_OOM, "fused rescale scratch");
            launch_fr_tail(L, bch.base, bch.cap, ext, l + 1, Z, Tt, 2 * nc, l - 1, c->L, fr->pm_last, fr->qinv_p);
            launch_bcast_submul(L, Z, 1, l - 1, 2 * nc, l - 1, 0, S, PolyMap{ext, l + 1}, och, fr->c1, bch, nullptr,
                                false, PolyMap{nullptr, 0}, Tt, fr->qlc, c->d_rinv + (size_t)l * (c->L + c->K), fr->qlcf);
            continue;
        }
        if (inv_bcast_on(c, 2 * nc, t_hi - t_lo)) {  // INTT column phase of the P limb fused with the broadcast
            PolyMap pl{ext + (size_t)l * n, l + 1};
            launch_inv_bcast_submul(L, pl, pl, LimbSet{1, 0, 0, c->L}, 2 * nc, t_hi - t_lo, t_lo, S,
                                    PolyMap{ext, l + 1}, och, c->d_pinv, bch, base_perm, base_c0_only, ach, p_rows);
        } else {
            PolyMap pl{ext + (size_t)l * n, l + 1};
            launch_ntt_inv(L, pl, pl, 2 * nc, LimbSet{1, 0, 0, c->L}, nullptr);
            launch_bcast_submul(L, ext + (size_t)l * n, l + 1, c->L, 2 * nc, t_hi - t_lo, t_lo, S,
                                PolyMap{ext, l + 1}, och, c->d_pinv, bch, base_perm, base_c0_only, ach);
        }
    }
    return check_launch(c);
}

// ---- cluster key switch (ks_cluster.cu) -------------------------------------------------------
// FP64-mode targets of [t_lo, t_hi) plus P go to the fused cluster kernel; integer-mode targets
// (60-bit primes) keep the ModUp-column + inner-product pair, on the second stream so the
// IMAD-pipe work shares the SMs with the FP64-pipe kernel.
bool kc_is_f64(const ckks_ctx *c, u32 prime) { return c->primes[prime] < c->tb.f64_qmax; }

const u32 *kc_tmap(ckks_ctx *c, u32 l, u32 t_lo, u32 t_hi, std::vector<u32> &host)
{
    host.clear();
    for (u32 t = t_lo; t < t_hi; ++t)
        if (kc_is_f64(c, t)) host.push_back(t);
    if (kc_is_f64(c, c->L)) host.push_back(l);
    const u64 key = ((u64)l << 40) | ((u64)t_lo << 20) | t_hi;
    auto it = c->kc_tmaps.find(key);
    if (it != c->kc_tmaps.end()) return it->second;
    u32 *d = nullptr;
    if (host.empty()) return nullptr;
    if (cudaMalloc(&d, host.size() * sizeof(u32)) != cudaSuccess) return nullptr;
    cudaMemcpy(d, host.data(), host.size() * sizeof(u32), cudaMemcpyHostToDevice);
    return c->kc_tmaps[key] = d;
}

// make a freshly installed switching key's FP64-mode limbs MAC-layout doubles (cluster path) or
// compact (launch_key_compact: the FP64 inner product reads 5 of every 8 key bytes)
void kc_key_installed(ckks_ctx *c, u64 *key)
{
    if (c->ksc && key) launch_key_mac_layout(c->lc(), key, c->d_kc_limbs, c->n_kc_limbs, 2 * c->dnum, c->L + c->K,
                                             false);
    if (c->kcomp && key) {
        u64 *tmp = need(c, "kcomp_tmp", (size_t)2 * c->dnum * c->N);
        if (tmp)
            launch_key_compact(c->lc(), key, c->kcomp_limbs.data(), (u32)c->kcomp_limbs.size(), 2 * c->dnum,
                               c->L + c->K, false, tmp);
    }
}

ckks_status keyswitch_cluster(ckks_ctx *c, PolyMap din, const u32 *perm, u32 cnt, u32 l, const u64 *key, u32 t_lo,
                              u32 t_hi, KsDigits dg, PolyMap out, PolyMap base, const u32 *base_perm,
                              bool base_c0_only, PolyMap acc)
{
    Launch L = c->lc();
    L.split_words = (size_t)256 << c->log_n;
    L.split = need(c, "ks_split", L.split_words);
    if (!L.split) L.split_words = 0;
    const size_t n = c->N;
    std::vector<u32> fT;
    const u32 *tmap = kc_tmap(c, l, t_lo, t_hi, fT);
    if (!fT.empty() && !tmap) return fail(c, CKKS_E_OOM, "cluster target map");
    // integer-mode target runs (contiguous in the target index t, P as t = l)
    std::vector<std::pair<u32, u32>> iruns;
    u32 n_int = 0;
    for (u32 t = t_lo; t < t_hi; ++t) {
        if (kc_is_f64(c, t)) continue;
        ++n_int;
        if (!iruns.empty() && iruns.back().first + iruns.back().second == t)
            ++iruns.back().second;
        else
            iruns.push_back({t, 1});
    }
    if (!kc_is_f64(c, c->L)) {  // P (target index l)
        ++n_int;
        if (!iruns.empty() && iruns.back().first + iruns.back().second == l)
            ++iruns.back().second;
        else
            iruns.push_back({l, 1});
    }
    const size_t budget = ks_budget_words();
    const size_t per_ct = (dg.D ? 0 : (size_t)l * n) + (size_t)n_int * l * n + (size_t)2 * (l + 1) * n +
                          (size_t)2 * (t_hi - t_lo) * n;
    const u32 cc = (u32)std::max<size_t>(1, std::min<size_t>(cnt, budget / per_ct));
    const size_t dwords = dg.D ? 0 : (size_t)cc * l * n;
    u64 *s = need(c, "ks", per_ct * cc);
    double *part = reinterpret_cast<double *>(need(c, "kc_part", ks_cluster_part_words(L)));
    const size_t nctr = (size_t)cc * std::max<size_t>(fT.size(), 1) * (n >> 12);
    if (c->kc_ctr_n < nctr) {
        if (c->d_kc_ctr) cudaFree(c->d_kc_ctr);
        c->d_kc_ctr = nullptr;
        c->kc_ctr_n = 0;
        if (cudaMalloc(&c->d_kc_ctr, nctr * sizeof(u32)) != cudaSuccess) {
            cudaGetLastError();
            return fail(c, CKKS_E_OOM, "cluster counters");
        }
        c->kc_ctr_n = nctr;
        CUDA_TRY(c, cudaMemsetAsync(c->d_kc_ctr, 0, nctr * sizeof(u32), c->st));
    }
    if (!s || !part) return fail(c, CKKS_E_OOM, "key-switch scratch");
    u64 *D = s, *I = D + dwords, *ext = I + (size_t)cc * n_int * l * n, *S = ext + (size_t)cc * 2 * (l + 1) * n;
    for (u32 c0 = 0; c0 < cnt; c0 += cc) {
        const u32 nc = std::min(cc, cnt - c0);
        PolyMap dch{din.base + (size_t)c0 * din.cap * n, din.cap};
        const u64 *Dp = dg.D;
        u32 dw = dg.dw, dcnt = dg.dcnt, dc0 = c0;
        if (!Dp) {
            launch_ntt_inv(L, dch, PolyMap{D, l}, nc, qlimbs(c, l), perm);
            Dp = D;
            dw = l;
            dcnt = nc;
            dc0 = 0;
        }
        const bool fork = !iruns.empty() && !fT.empty() && L.aux && !(c->prof && prof_on(c->prof));
        if (fork) {
            CUDA_TRY(c, cudaEventRecord(L.ev_fork, L.st));
            CUDA_TRY(c, cudaStreamWaitEvent(L.aux, L.ev_fork, 0));
        }
        Launch Li = L;
        if (fork) Li.st = L.aux;
        u64 *Ib = I;
        for (auto &r : iruns) {  // integer targets: ModUp columns -> slab -> inner product
            launch_ks_modup_cols(Li, Dp, dw, dcnt, dc0, l, nc, r.first, r.second, Ib, c->L);
            launch_ks_mac(Li, Ib, dch, perm, key, c->L, l, nc, r.first, r.second, ext, c->L);
            Ib += (size_t)nc * r.second * l * n;
        }
        launch_ks_cluster(L, L.st, Dp, dw, dcnt, dc0, dch, perm, key, c->L, l, nc, tmap, fT.data(), (u32)fT.size(),
                          ext, part, c->d_kc_ctr, c->L);
        if (fork) {
            CUDA_TRY(c, cudaEventRecord(L.ev_join, L.aux));
            CUDA_TRY(c, cudaStreamWaitEvent(L.st, L.ev_join, 0));
        }
        // ModDown (A7): INTT of the P limb, then out_i = base + (acc_i - NTT_i([acc]_P)) P^{-1}
        PolyMap och{out.base + (size_t)c0 * 2 * out.cap * n, out.cap};
        PolyMap bch = base.base ? PolyMap{base.base + (size_t)c0 * 2 * base.cap * n, base.cap} : base;
        PolyMap ach = acc.base ? PolyMap{acc.base + (size_t)c0 * 2 * acc.cap * n, acc.cap} : acc;
        PolyMap pl{ext + (size_t)l * n, l + 1};
        if (inv_bcast_on(c, 2 * nc, t_hi - t_lo)) {
            launch_inv_bcast_submul(L, pl, pl, LimbSet{1, 0, 0, c->L}, 2 * nc, t_hi - t_lo, t_lo, S,
                                    PolyMap{ext, l + 1}, och, c->d_pinv, bch, base_perm, base_c0_only, ach, false);
        } else {
            launch_ntt_inv(L, pl, pl, 2 * nc, LimbSet{1, 0, 0, c->L}, nullptr);
            launch_bcast_submul(L, ext + (size_t)l * n, l + 1, c->L, 2 * nc, t_hi - t_lo, t_lo, S,
                                PolyMap{ext, l + 1}, och, c->d_pinv, bch, base_perm, base_c0_only, ach);
        }
    }
    return check_launch(c);
}

// hybrid ModUp constants for level l (computed once per level, cached)
const ckks_ctx::HybLevel *hyb_level(ckks_ctx *c, u32 l)
{
    auto it = c->hyb.find(l);
    if (it != c->hyb.end()) return &it->second;
    const u32 a = c->alpha, beta = (l + a - 1) / a, ne = l + c->K;
    std::vector<ulonglong2> yinv((size_t)beta * a, make_ulonglong2(0, 0));
    std::vector<u64> conv((size_t)beta * a * ne, 0);
    auto slot_mod = [&](u32 s) { return s < l ? c->primes[s] : c->primes[c->L + (s - l)]; };
    for (u32 d = 0; d < beta; ++d) {
        const u32 lo = d * a, hi = std::min(lo + a, l);
        for (u32 i = lo; i < hi; ++i) {
            const u64 qi = c->primes[i];
            u64 r = 1;  // (Q_D / q_i) mod q_i
            for (u32 j = lo; j < hi; ++j)
                if (j != i) r = hm::mulmod(r, c->primes[j] % qi, qi);
            const u64 v = hm::invmod(r, qi);
            yinv[(size_t)d * a + (i - lo)] = make_ulonglong2(v, hm::shoup(v, qi));
            for (u32 s = 0; s < ne; ++s) {
                const u64 m = slot_mod(s);
                u64 t = 1 % m;  // (Q_D / q_i) mod m_s
                for (u32 j = lo; j < hi; ++j)
                    if (j != i) t = hm::mulmod(t, c->primes[j] % m, m);
                conv[((size_t)d * a + (i - lo)) * ne + s] = t;
            }
        }
    }
    // fused ModDown + rescale (reading A7 with K special primes; internal.h launch_hyb_moddown_rs)
    std::vector<ulonglong2> rs((size_t)3 * l, make_ulonglong2(0, 0));
    {
        auto pmod = [&](u64 q) {  // P mod q
            u64 r = 1 % q;
            for (u32 k = 0; k < c->K; ++k) r = hm::mulmod(r, c->primes[c->L + k] % q, q);
            return r;
        };
        const u64 ql = c->primes[l - 1];
        for (u32 i = 0; i + 1 < l; ++i) {
            const u64 q = c->primes[i], pm = pmod(q);
            const u64 v = hm::invmod(hm::mulmod(pm, ql % q, q), q), w = hm::invmod(ql % q, q);
            rs[i] = make_ulonglong2(v, hm::shoup(v, q));
            rs[l + i] = make_ulonglong2(w, hm::shoup(w, q));
            rs[2 * l + i] = make_ulonglong2(pm, hm::shoup(pm, q));
        }
        if (l >= 2) {
            const u64 pm = pmod(ql), pi = hm::invmod(pm, ql);
            rs[l - 1] = make_ulonglong2(pm, hm::shoup(pm, ql));
            rs[2 * l - 1] = make_ulonglong2(pi, hm::shoup(pi, ql));
        }
    }
    ckks_ctx::HybLevel h;
    if (cudaMalloc(&h.yinv, yinv.size() * sizeof(ulonglong2)) != cudaSuccess ||
        cudaMalloc(&h.conv, conv.size() * sizeof(u64)) != cudaSuccess ||
        cudaMalloc(&h.rs, rs.size() * sizeof(ulonglong2)) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    cudaMemcpy(h.yinv, yinv.data(), yinv.size() * sizeof(ulonglong2), cudaMemcpyHostToDevice);
    cudaMemcpy(h.conv, conv.data(), conv.size() * sizeof(u64), cudaMemcpyHostToDevice);
    cudaMemcpy(h.rs, rs.data(), rs.size() * sizeof(ulonglong2), cudaMemcpyHostToDevice);
    return &(c->hyb[l] = h);
}

// Hybrid key switching: INTT(d) -> fast base conversion ModUp of each
// alpha-limb digit + NTT -> inner product over digits -> ModDown by the K special primes.
ckks_status keyswitch_hybrid(ckks_ctx *c, PolyMap din, const u32 *perm, u32 cnt, u32 l, const u64 *key, PolyMap out,
                             PolyMap base, const u32 *base_perm, bool base_c0_only, PolyMap acc,
                             u64 *rows_done = nullptr, bool fuse_rescale = false)
{
    const Launch L = c->lc();
    const size_t n = c->N;
    const u32 beta = (l + c->alpha - 1) / c->alpha, ne = l + c->K;
    const ckks_ctx::HybLevel *hl = hyb_level(c, l);
    if (!hl) return fail(c, CKKS_E_OOM, "hybrid constants");
    const bool fused_ip = hyb_fused_ip_ok(L, l, c->L, c->K);
    const size_t per = ((size_t)l + (size_t)beta * ne + 2 * ne + 2 * l) * n;
    const u32 cc = (u32)std::max<size_t>(1, std::min<size_t>(cnt, ks_budget_words() / per));
    u64 *s = need(c, "ks", per * cc);
    if (!s) return fail(c, CKKS_E_OOM, "key-switch scratch");
    u64 *D = s, *X = D + (size_t)cc * l * n, *ext = X + (size_t)cc * beta * ne * n, *Y = ext + (size_t)cc * 2 * ne * n;
    for (u32 c0 = 0; c0 < cnt; c0 += cc) {
        const u32 nc = std::min(cc, cnt - c0);
        PolyMap dch{din.base + (size_t)c0 * din.cap * n, din.cap};
        u64 *Dc = D;
        if (rows_done) {  // the tensor kernel applied the row phase: columns in place
            Dc = rows_done + (size_t)c0 * l * n;
            launch_ntt_inv_cols(L, PolyMap{Dc, l}, nc, qlimbs(c, l));
        } else {
            launch_ntt_inv(L, dch, PolyMap{D, l}, nc, qlimbs(c, l), perm);
        }
        PolyMap och{out.base + (size_t)c0 * 2 * out.cap * n, out.cap};
        PolyMap bch = base.base ? PolyMap{base.base + (size_t)c0 * 2 * base.cap * n, base.cap} : base;
        PolyMap ach = acc.base ? PolyMap{acc.base + (size_t)c0 * 2 * acc.cap * n, acc.cap} : acc;
        if (fused_ip) {  // row phase + inner product in one kernel (X never holds the NTT form)
            launch_hyb_modup(L, Dc, X, hl->yinv, hl->conv, nc, l, c->L, c->K, c->alpha, beta, ne, true);
            launch_hyb_ip_fused(L, X, dch, perm, key, ext, nc, l, c->L, c->K, c->alpha, beta, ne, bch,
                                fuse_rescale ? hl->rs : nullptr);
        } else {
            launch_hyb_modup(L, Dc, X, hl->yinv, hl->conv, nc, l, c->L, c->K, c->alpha, beta, ne);
            launch_hyb_ip(L, X, dch, perm, key, ext, nc, l, c->L, c->K, c->alpha, beta, ne);
        }
        if (fuse_rescale)  // out at level l-1: ModDown and RESCALE in one tail (base = the tensor's d0, d1)
            launch_hyb_moddown_rs(L, ext, Y, c->d_pyinv, c->d_pconv, 2 * nc, l, c->L, c->K, ne, och, bch, hl->rs,
                                  fused_ip);
        else
            launch_hyb_moddown(L, ext, Y, c->d_pyinv, c->d_pconv, 2 * nc, l, c->L, c->K, ne, och, bch, base_perm,
                               base_c0_only, c->d_pinv, ach);
    }
    return check_launch(c);
}

// out = [acc] + base + KS(din)   (acc: optional extra addend at the output index)
ckks_status keyswitch(ckks_ctx *c, PolyMap din, const u32 *perm, u32 cnt, u32 l, const u64 *key, PolyMap out,
                      PolyMap base, const u32 *base_perm, bool base_c0_only, PolyMap acc = PolyMap{nullptr, 0},
                      u64 *rows_done = nullptr)
{
    if (c->alpha > 1 || c->K > 1)
        return keyswitch_hybrid(c, din, perm, cnt, l, key, out, base, base_perm, base_c0_only, acc, rows_done);
    return keyswitch_range(c, din, perm, cnt, l, key, 0, l, KsDigits{nullptr, 0, 0}, out, base, base_perm,
                           base_c0_only, acc, false, rows_done);
}

// HMULT tensor product into out (d0, d1) and d2; with the relinearisation digits' INTT row phase
// fused in (k_tensor_inv_rows) when the plain pairing is used: returns the row-phase buffer, or
// nullptr when the tensor ran alone (CKKS_TENSOR_ROWS=0 for A/B)
u64 *tensor_for_relin(ckks_ctx *c, const ckks_buf *a, const ckks_buf *b, ckks_buf *out, u64 *d2, u32 cnt, u32 l)
{
    const char *e = std::getenv("CKKS_TENSOR_ROWS");
    u64 *dr = (e && e[0] == '0') ? nullptr : need(c, "d2_rows", (size_t)cnt * l * c->N);
    if (!dr) {
        launch_tensor(c->lc(), pm(a), pm(b), pm(out), PolyMap{d2, l}, cnt, l);
        return nullptr;
    }
    launch_tensor_inv_rows(c->lc(), pm(a), pm(b), pm(out), PolyMap{d2, l}, PolyMap{dr, l}, cnt, l);
    return dr;
}

ckks_status rescale_impl(ckks_ctx *c, const ckks_buf *ct, ckks_buf *out)
{
    const u32 l = ct->level, cnt = ct->count;
    const size_t n = c->N;
    u64 *X = need(c, "rs", (size_t)2 * cnt * n + (size_t)2 * cnt * (l - 1) * n);
    if (!X) return fail(c, CKKS_E_OOM, "rescale scratch");
    u64 *S = X + (size_t)2 * cnt * n;
    const Launch L = c->lc();
    if (inv_bcast_on(c, 2 * cnt, l - 1)) {
        launch_inv_bcast_submul(L, PolyMap{ct->data + (size_t)(l - 1) * n, ct->capacity}, PolyMap{X, 1},
                                LimbSet{1, 1, l - 1, c->L}, 2 * cnt, l - 1, 0, S, pm(ct), pm(out),
                                c->d_rinv + (size_t)l * (c->L + c->K), PolyMap{nullptr, 0}, nullptr, false,
                                PolyMap{nullptr, 0});
    } else {
        launch_ntt_inv(L, PolyMap{ct->data + (size_t)(l - 1) * n, ct->capacity}, PolyMap{X, 1}, 2 * cnt,
                       LimbSet{1, 1, l - 1, c->L}, nullptr);
        launch_bcast_submul(L, X, 1, l - 1, 2 * cnt, l - 1, 0, S, pm(ct), pm(out),
                            c->d_rinv + (size_t)l * (c->L + c->K), PolyMap{nullptr, 0}, nullptr, false);
    }
    out->level = l - 1;
    out->scale = ct->scale / (double)c->primes[l - 1];
    out->count = cnt;
    out->n_polys = 2;
    return check_launch(c);
}

// one Galois automorphism + key switch from `cur` into `dst` (dst != cur);
// accumulate: dst = cur + rotate(cur)  (TotalSum step fused into the ModDown epilogue)
ckks_status galois_step(ckks_ctx *c, const ckks_buf *cur, int32_t step, ckks_buf *dst, bool accumulate = false)
{
    const u64 kappa = galois_elt(c, step);
    auto it = c->gk.find(kappa);
    if (it == c->gk.end()) return fail(c, CKKS_E_MISSING_KEY, "missing Galois key for step " + std::to_string(step));
    const u32 *perm = get_perm(c, kappa);
    if (!perm) return fail(c, CKKS_E_OOM, "perm");
    ckks_status s = keyswitch(c, pm_c(cur, 1, c->N), perm, cur->count, cur->level, it->second, pm(dst), pm(cur), perm,
                              true, accumulate ? pm(cur) : PolyMap{nullptr, 0});
    dst->level = cur->level;
    dst->scale = cur->scale;
    dst->count = cur->count;
    dst->n_polys = 2;
    return s;
}

ckks_buf tmp_ct(ckks_ctx *c, const char *name, const ckks_buf *like)
{
    ckks_buf t = *like;
    t.capacity = like->level;
    t.data = need(c, name, (size_t)like->count * 2 * like->level * c->N);
    return t;
}

void copy_ct(ckks_ctx *c, const ckks_buf *src, ckks_buf *dst)
{
    if (src->data != dst->data) launch_copy(c->lc(), pm(src), pm(dst), src->count * src->n_polys, src->level);
    dst->level = src->level;
    dst->scale = src->scale;
    dst->count = src->count;
    dst->n_polys = src->n_polys;
}

ckks_status rotate_impl(ckks_ctx *c, const ckks_buf *ct, int32_t steps, ckks_buf *out)
{
    std::vector<int32_t> digits = rotation_steps(c, steps);
    for (int32_t d : digits)
        if (!c->gk.count(galois_elt(c, d)))
            return fail(c, CKKS_E_MISSING_KEY, "missing Galois key for step " + std::to_string(d));
    if (digits.empty()) {
        copy_ct(c, ct, out);
        return check_launch(c);
    }
    ckks_buf a = tmp_ct(c, "rotA", ct), b = tmp_ct(c, "rotB", ct);
    if (!a.data || !b.data) return fail(c, CKKS_E_OOM, "rotation scratch");
    const ckks_buf *cur = ct;
    for (size_t k = 0; k < digits.size(); ++k) {
        ckks_buf *dst;
        if (k + 1 == digits.size() && out->data != cur->data)
            dst = out;
        else
            dst = (cur->data == a.data) ? &b : &a;
        ckks_status s = galois_step(c, cur, digits[k], dst);
        if (s != CKKS_OK) return s;
        cur = dst;
    }
    if (cur != out) copy_ct(c, cur, out);
    return check_launch(c);
}

ckks_status upload_consts(ckks_ctx *c, const std::vector<ulonglong2> &h, const char *name, ulonglong2 **d)
{
    u64 *p = need(c, name, h.size() * 2);
    if (!p) return fail(c, CKKS_E_OOM, "const table");
    CUDA_TRY(c, cudaMemcpyAsync(p, h.data(), h.size() * sizeof(ulonglong2), cudaMemcpyHostToDevice, c->st));
    *d = reinterpret_cast<ulonglong2 *>(p);
    return CKKS_OK;
}

}  // namespace

// ======================================================================================
extern "C" {

ckks_status ckks_ctx_create(const ckks_params *params, int device, void *cuda_stream, ckks_ctx **out)
{
    if (!params || !out) return CKKS_E_INVALID_ARG;
    *out = nullptr;
    if (params->log_n < 10 || params->log_n > 16 || params->n_limbs < 1 || params->n_limbs > 60 ||
        !(params->scale > 0))
        return CKKS_E_INVALID_ARG;
    if (cudaSetDevice(device) != cudaSuccess) return CKKS_E_CUDA;
    ckks_ctx *c = new ckks_ctx();
    c->device = device;
    c->st = (cudaStream_t)cuda_stream;
    c->log_n = params->log_n;
    c->N = 1u << params->log_n;
    c->L = params->n_limbs;
    c->K = params->n_special ? params->n_special : 1;
    c->alpha = params->digit_limbs ? params->digit_limbs : 1;
    c->dnum = (c->L + c->alpha - 1) / c->alpha;
    c->scale = params->scale;
    if (c->K > 16 || c->alpha > 16) {
        delete c;
        return CKKS_E_UNSUPPORTED;
    }
    std::string err;
    if (params->primes) {
        c->primes.assign(params->primes, params->primes + c->L + c->K);
        for (u64 p : c->primes)
            if (!hm::is_prime(p) || (p - 1) % (2ull * c->N)) {
                delete c;
                return CKKS_E_INVALID_ARG;
            }
    } else {
        if (!params->limb_bits) {
            delete c;
            return CKKS_E_INVALID_ARG;
        }
        if (!hm::prime_chain(c->log_n, c->L, params->limb_bits, params->special_bits, c->K, c->primes, err)) {
            delete c;
            return CKKS_E_PRIME_EXHAUSTED;
        }
    }
    for (u64 p : c->primes)
        if (p >= (1ull << 61)) {  // lazy [0,4q) and 128-bit inner-product accumulation bounds
            delete c;
            return CKKS_E_UNSUPPORTED;
        }
    {  // distinct primes: the rescale / ModDown inverses (q_{l-1}^{-1}, P^{-1} mod q_i) need them
        std::vector<u64> sorted(c->primes);
        std::sort(sorted.begin(), sorted.end());
        if (std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end()) {
            delete c;
            return CKKS_E_INVALID_ARG;
        }
    }
    const u32 np = c->L + c->K, N = c->N;
    std::vector<ModC> mods(np);
    std::vector<ulonglong2> psi((size_t)np * N), ipsi((size_t)np * N), ninv(np);
    std::vector<double2> psif((size_t)np * N, make_double2(0, 0)), ipsif((size_t)np * N, make_double2(0, 0));
    const char *f64env = std::getenv("CKKS_NTT_F64");
    const u64 f64_qmax = (f64env && f64env[0] == '0') ? 0 : F64_Q_MAX;
    for (u32 i = 0; i < np; ++i) {
        const u64 q = c->primes[i];
        const u64 r64 = (u64)((((hm::u128)1) << 64) % q);
        mods[i] = ModC{q, r64, hm::shoup(r64, q), (u64)(~0ull / q)};
        const u64 g = hm::primitive_2n_root(q, c->log_n), gi = hm::invmod(g, q);
        std::vector<u64> pw(N), ipw(N);
        pw[0] = ipw[0] = 1;
        for (u32 k = 1; k < N; ++k) {
            pw[k] = hm::mulmod(pw[k - 1], g, q);
            ipw[k] = hm::mulmod(ipw[k - 1], gi, q);
        }
        for (u32 k = 0; k < N; ++k) {
            const u64 w = pw[hm::bitrev(k, c->log_n)], wi = ipw[hm::bitrev(k, c->log_n)];
            psi[(size_t)i * N + k] = make_ulonglong2(w, hm::shoup(w, q));
            ipsi[(size_t)i * N + k] = make_ulonglong2(wi, hm::shoup(wi, q));
            if (q < F64_Q_MAX) {  // FP64-mode twiddles (w, w/q); entry 0 (unused by the stages) = (q, 1/q)
                const double qd = (double)q;
                psif[(size_t)i * N + k] = k ? make_double2((double)w, (double)w / qd) : make_double2(qd, 1.0 / qd);
                ipsif[(size_t)i * N + k] = k ? make_double2((double)wi, (double)wi / qd) : make_double2(qd, 1.0 / qd);
            }
        }
        const u64 ni = hm::invmod(N % q, q);
        ninv[i] = make_ulonglong2(ni, hm::shoup(ni, q));
    }
    std::vector<ulonglong2> rinv((size_t)np * np, make_ulonglong2(0, 0)), pinv(np, make_ulonglong2(0, 0));
    std::vector<u64> pmod(np, 0);
    for (u32 l = 2; l <= c->L; ++l)
        for (u32 k = 0; k + 1 < l; ++k) {
            const u64 q = c->primes[k], v = hm::invmod(c->primes[l - 1] % q, q);
            rinv[(size_t)l * np + k] = make_ulonglong2(v, hm::shoup(v, q));
        }
    for (u32 i = 0; i < c->L; ++i) {  // P = p_0 ... p_{K-1}
        const u64 q = c->primes[i];
        u64 pm = 1;
        for (u32 k = 0; k < c->K; ++k) pm = hm::mulmod(pm, c->primes[c->L + k] % q, q);
        const u64 v = hm::invmod(pm, q);
        pinv[i] = make_ulonglong2(v, hm::shoup(v, q));
        pmod[i] = pm;
    }
    std::vector<ulonglong2> pyinv(c->K);
    std::vector<u64> pconv((size_t)c->K * c->L);
    for (u32 k = 0; k < c->K; ++k) {
        const u64 pk = c->primes[c->L + k];
        u64 r = 1;
        for (u32 j = 0; j < c->K; ++j)
            if (j != k) r = hm::mulmod(r, c->primes[c->L + j] % pk, pk);
        const u64 v = hm::invmod(r, pk);
        pyinv[k] = make_ulonglong2(v, hm::shoup(v, pk));
        for (u32 i = 0; i < c->L; ++i) {
            const u64 q = c->primes[i];
            u64 t = 1;
            for (u32 j = 0; j < c->K; ++j)
                if (j != k) t = hm::mulmod(t, c->primes[c->L + j] % q, q);
            pconv[(size_t)k * c->L + i] = t;
        }
    }
    auto up = [&](void **d, const void *h, size_t bytes) -> bool {
        return cudaMalloc(d, bytes) == cudaSuccess && cudaMemcpy(*d, h, bytes, cudaMemcpyHostToDevice) == cudaSuccess;
    };
    bool ok = up((void **)&c->d_mod, mods.data(), np * sizeof(ModC)) &&
              up((void **)&c->d_psi, psi.data(), psi.size() * sizeof(ulonglong2)) &&
              up((void **)&c->d_ipsi, ipsi.data(), ipsi.size() * sizeof(ulonglong2)) &&
              up((void **)&c->d_psif, psif.data(), psif.size() * sizeof(double2)) &&
              up((void **)&c->d_ipsif, ipsif.data(), ipsif.size() * sizeof(double2)) &&
              up((void **)&c->d_ninv, ninv.data(), ninv.size() * sizeof(ulonglong2)) &&
              up((void **)&c->d_rinv, rinv.data(), rinv.size() * sizeof(ulonglong2)) &&
              up((void **)&c->d_pinv, pinv.data(), pinv.size() * sizeof(ulonglong2)) &&
              up((void **)&c->d_pmod, pmod.data(), pmod.size() * sizeof(u64)) &&
              up((void **)&c->d_pyinv, pyinv.data(), pyinv.size() * sizeof(ulonglong2)) &&
              up((void **)&c->d_pconv, pconv.data(), pconv.size() * sizeof(u64));
    if (!ok) {
        cudaGetLastError();
        ckks_ctx_destroy(c);
        return CKKS_E_CUDA;
    }
    c->tb = Tables{c->d_mod, c->d_psi, c->d_ipsi, c->d_ninv, c->d_psif, c->d_ipsif, f64_qmax, c->log_n};
    // integer- and FP64-class inner-product runs on two streams (their CTAs share the SMs: the
    // integer class is IMAD-pipe bound, the FP64 class FP64/shared-memory bound).  On by default
    // since the shared-memory key-switch pipeline: C3 HMult 704 -> 696 us, C4 neutral;
    // CKKS_DUAL_STREAM=0 disables it.
    const char *dual = std::getenv("CKKS_DUAL_STREAM");
    if (!(dual && dual[0] == '0') &&
        (cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking) != cudaSuccess ||
         cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
         cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess)) {
        cudaGetLastError();  // single-stream operation: release whatever was created
        if (c->aux) cudaStreamDestroy(c->aux);
        if (c->ev_fork) cudaEventDestroy(c->ev_fork);
        if (c->ev_join) cudaEventDestroy(c->ev_join);
        c->aux = nullptr;
        c->ev_fork = c->ev_join = nullptr;
    }
    int nsm = 0;
    if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device) == cudaSuccess && nsm > 0)
        c->n_sm = (u32)nsm;
    cudaGetLastError();
    {  // cluster key switch: opt-in (CKKS_KS_CLUSTER=1).  Bit-exact, but measured at parity with
       // the two-kernel path (N = 2^14, 2^15) or slower (C3: 7 resident 16-CTA clusters = 112 SMs;
       // C4: the 60-bit targets stay on the two-kernel path and cannot share the SMs), DESIGN 7.
        const char *kce = std::getenv("CKKS_KS_CLUSTER");
        std::vector<u32> fl;
        for (u32 i = 0; i < c->L + c->K; ++i)
            if (c->primes[i] < f64_qmax) fl.push_back(i);
        if ((kce && kce[0] == '1') && c->alpha == 1 && c->K == 1 && c->log_n >= 12 && !fl.empty() &&
            ks_cluster_supported(c->lc())) {
            if (cudaMalloc(&c->d_kc_limbs, fl.size() * sizeof(u32)) == cudaSuccess &&
                cudaMemcpy(c->d_kc_limbs, fl.data(), fl.size() * sizeof(u32), cudaMemcpyHostToDevice) == cudaSuccess) {
                c->ksc = true;
                c->n_kc_limbs = (u32)fl.size();
            }
        }
        cudaGetLastError();
    }
    {  // compact keys: every FP64-mode limb below 2^40 and the key rows read only by k_ks_mac CLS 5
       // and export -- alpha = K = 1, or hybrid keys whose every limb is FP64-mode (the inner product
       // then always runs on k_ks_mac, hyb_fused_ip_ok); CKKS_KEY_COMPACT=0 disables
        const char *e = std::getenv("CKKS_KEY_COMPACT");
        const char *fe = std::getenv("CKKS_HYB_FUSED_IP");
        bool hyb_ok = c->log_n >= 12 && c->L + c->K <= 64 && !(fe && fe[0] == '0');
        for (u32 i = 0; hyb_ok && i < c->L + c->K; ++i) hyb_ok = c->primes[i] < f64_qmax;
        bool ok = !c->ksc && ((c->alpha == 1 && c->K == 1) || hyb_ok) && !(e && e[0] == '0');
        std::vector<u32> kl;
        for (u32 i = 0; ok && i < c->L + c->K; ++i) {
            if (c->primes[i] >= f64_qmax) continue;
            if (c->primes[i] >= (1ull << 40)) ok = false;
            kl.push_back(i);
        }
        if (ok && !kl.empty()) {
            c->kcomp = true;
            c->kcomp_limbs = kl;
        }
    }
    c->prof = prof_create();
    *out = c;
    return CKKS_OK;
}

ckks_status ckks_ctx_destroy(ckks_ctx *c)
{
    if (!c) return CKKS_E_INVALID_ARG;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->st);
    for (void *p : {(void *)c->d_mod, (void *)c->d_psi, (void *)c->d_ipsi, (void *)c->d_psif, (void *)c->d_ipsif,
                    (void *)c->d_ninv, (void *)c->d_rinv,
                    (void *)c->d_pinv, (void *)c->d_pmod, (void *)c->sk, (void *)c->pk, (void *)c->rlk,
                    (void *)c->d_pyinv, (void *)c->d_pconv, (void *)c->d_fft_w, (void *)c->d_fft_tw,
                    (void *)c->d_slot, (void *)c->d_enc_overflow})
        if (p) cudaFree(p);
    for (auto &kv : c->crt) cudaFree(kv.second.c);
    for (auto &kv : c->kc_tmaps) cudaFree(kv.second);
    for (auto &kv : c->fr) cudaFree(kv.second.c1), cudaFree(kv.second.qlc), cudaFree(kv.second.qlcf);
    if (c->d_kc_limbs) cudaFree(c->d_kc_limbs);
    if (c->d_kc_ctr) cudaFree(c->d_kc_ctr);
    if (c->aux) cudaStreamDestroy(c->aux);
    if (c->up) cudaStreamSynchronize(c->up), cudaStreamDestroy(c->up);
    for (int i = 0; i < 2; ++i)
        for (int h = 0; h < 2; ++h) {
            if (c->up_done[i][h]) cudaEventDestroy(c->up_done[i][h]);
            if (c->stage_free[i][h]) cudaEventDestroy(c->stage_free[i][h]);
        }
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    for (auto &kv : c->ipc) cudaIpcCloseMemHandle(kv.second);
    for (auto &kv : c->gk) cudaFree(kv.second);
    for (auto &kv : c->perms) cudaFree(kv.second);
    for (auto &kv : c->hyb) {
        cudaFree(kv.second.yinv);
        cudaFree(kv.second.conv);
        cudaFree(kv.second.rs);
    }
    for (auto &kv : c->bufs)
        if (kv.second.p) cudaFree(kv.second.p);
    prof_destroy(c->prof);
    delete c;
    return CKKS_OK;
}

ckks_status ckks_set_stream(ckks_ctx *c, void *s)
{
    if (!c) return CKKS_E_INVALID_ARG;
    c->st = (cudaStream_t)s;
    return CKKS_OK;
}

ckks_status ckks_ctx_info(const ckks_ctx *c, uint32_t *log_n, uint32_t *n_limbs, uint64_t *primes_out)
{
    if (!c) return CKKS_E_INVALID_ARG;
    if (log_n) *log_n = c->log_n;
    if (n_limbs) *n_limbs = c->L;
    if (primes_out) std::memcpy(primes_out, c->primes.data(), (c->L + c->K) * sizeof(u64));
    return CKKS_OK;
}

ckks_status ckks_profile_enable(ckks_ctx *c, int on)
{
    if (!c) return CKKS_E_INVALID_ARG;
    prof_enable(c->prof, on != 0);
    return CKKS_OK;
}

ckks_status ckks_profile_read(ckks_ctx *c, const char **names, double *ms, uint64_t *counts, double *work,
                              uint32_t cap, uint32_t *n, int reset)
{
    if (!c) return CKKS_E_INVALID_ARG;
    prof_collect(c->prof);
    const auto &tot = prof_totals(c->prof);
    c->prof_names.clear();
    uint32_t k = 0;
    for (auto &kv : tot) c->prof_names.push_back(kv.first);
    for (auto &kv : tot) {
        if (k < cap) {
            if (names) names[k] = c->prof_names[k].c_str();
            if (ms) ms[k] = kv.second.ms;
            if (counts) counts[k] = kv.second.launches;
            if (work) {
                work[5 * k] = kv.second.bfly;
                work[5 * k + 1] = kv.second.mac;
                work[5 * k + 2] = kv.second.bytes;
                work[5 * k + 3] = kv.second.fbfly;
                work[5 * k + 4] = kv.second.fmac;
            }
        }
        ++k;
    }
    if (n) *n = k;
    if (reset) prof_reset(c->prof);
    return CKKS_OK;
}

const char *ckks_last_error(const ckks_ctx *c) { return c ? c->err.c_str() : "null context"; }
uint64_t ckks_launch_count(const ckks_ctx *c) { return c ? c->launches : 0; }
uint64_t ckks_galois_elt(const ckks_ctx *c, int32_t step) { return c ? galois_elt(c, step) : 0; }

// ---- keys ---------------------------------------------------------------------------
ckks_status ckks_set_secret(ckks_ctx *c, const int64_t *s_dev)
{
    if (!c || !s_dev) return CKKS_E_INVALID_ARG;
    const u32 LK = c->L + c->K;
    if (!c->sk) CUDA_TRY(c, cudaMalloc(&c->sk, (size_t)LK * c->N * sizeof(u64)));
    const Launch L = c->lc();
    launch_from_signed(L, s_dev, PolyMap{c->sk, LK}, 1, extlimbs(c));
    launch_ntt_fwd(L, PolyMap{c->sk, LK}, PolyMap{c->sk, LK}, 1, extlimbs(c));
    return check_launch(c);
}

ckks_status ckks_keygen_public(ckks_ctx *c, const uint64_t *a_dev, const int64_t *e_dev)
{
    if (!c || !a_dev || !e_dev) return CKKS_E_INVALID_ARG;
    if (!c->sk) return fail(c, CKKS_E_MISSING_KEY, "secret key not set");
    const size_t n = c->N, L_ = c->L;
    if (!c->pk) CUDA_TRY(c, cudaMalloc(&c->pk, 2 * L_ * n * sizeof(u64)));
    const Launch L = c->lc();
    CUDA_TRY(c, cudaMemcpyAsync(c->pk + L_ * n, a_dev, L_ * n * sizeof(u64), cudaMemcpyDeviceToDevice, c->st));
    launch_ntt_fwd(L, PolyMap{c->pk + L_ * n, c->L}, PolyMap{c->pk + L_ * n, c->L}, 1, qlimbs(c, c->L));
    launch_from_signed(L, e_dev, PolyMap{c->pk, c->L}, 1, qlimbs(c, c->L));
    launch_ntt_fwd(L, PolyMap{c->pk, c->L}, PolyMap{c->pk, c->L}, 1, qlimbs(c, c->L));
    launch_mul_add(L, PolyMap{c->pk + L_ * n, c->L}, PolyMap{c->sk, c->L + c->K}, 1, PolyMap{c->pk, c->L},
                   PolyMap{c->pk, c->L}, 1, c->L, 1);
    return check_launch(c);
}

static ckks_status make_switch_key(ckks_ctx *c, const u64 *sfrom, const uint64_t *a_dev, const int64_t *e_dev,
                                   u64 **key)
{
    const u32 LK = c->L + c->K;
    const size_t kw = key_words(c) / 2;  // one of (b, a)
    u64 *A = need(c, "kgA", 2 * kw);
    if (!A) return fail(c, CKKS_E_OOM, "keygen scratch");
    u64 *E = A + kw;
    if (!*key) CUDA_TRY(c, cudaMalloc(key, 2 * kw * sizeof(u64)));
    const Launch L = c->lc();
    CUDA_TRY(c, cudaMemcpyAsync(A, a_dev, kw * sizeof(u64), cudaMemcpyDeviceToDevice, c->st));
    launch_ntt_fwd(L, PolyMap{A, LK}, PolyMap{A, LK}, c->dnum, extlimbs(c));
    launch_from_signed(L, e_dev, PolyMap{E, LK}, c->dnum, extlimbs(c));
    launch_ntt_fwd(L, PolyMap{E, LK}, PolyMap{E, LK}, c->dnum, extlimbs(c));
    launch_keygen_b(L, A, E, c->sk, sfrom, c->d_pmod, *key, c->L, c->K, c->alpha, c->dnum);
    kc_key_installed(c, *key);
    return check_launch(c);
}

ckks_status ckks_keygen_relin(ckks_ctx *c, const uint64_t *a_dev, const int64_t *e_dev)
{
    if (!c || !a_dev || !e_dev) return CKKS_E_INVALID_ARG;
    if (!c->sk) return fail(c, CKKS_E_MISSING_KEY, "secret key not set");
    const u32 LK = c->L + c->K;
    u64 *s2 = need(c, "kgS", (size_t)LK * c->N);
    if (!s2) return fail(c, CKKS_E_OOM, "keygen scratch");
    PolyMap skm{c->sk, LK};
    launch_mul_poly(c->lc(), skm, skm, 1, 0, PolyMap{s2, LK}, 1, LK);
    return make_switch_key(c, s2, a_dev, e_dev, &c->rlk);
}

ckks_status ckks_keygen_galois(ckks_ctx *c, int32_t step, const uint64_t *a_dev, const int64_t *e_dev)
{
    if (!c || !a_dev || !e_dev) return CKKS_E_INVALID_ARG;
    if (!c->sk) return fail(c, CKKS_E_MISSING_KEY, "secret key not set");
    const u64 kappa = galois_elt(c, step);
    const u32 *perm = get_perm(c, kappa);
    const u32 LK = c->L + c->K;
    u64 *sf = need(c, "kgS", (size_t)LK * c->N);
    if (!perm || !sf) return fail(c, CKKS_E_OOM, "keygen scratch");
    launch_permute(c->lc(), PolyMap{c->sk, LK}, PolyMap{sf, LK}, 1, LK, perm);
    u64 *key = c->gk.count(kappa) ? c->gk[kappa] : nullptr;
    ckks_status s = make_switch_key(c, sf, a_dev, e_dev, &key);
    if (key) c->gk[kappa] = key;
    return s;
}

static ckks_status install_switch_key(ckks_ctx *c, int kind, u64 kappa, const uint64_t *key_coeff_dev)
{
    const size_t kw = key_words(c);
    u64 *key = nullptr;
    if (kind == 0)
        key = c->rlk;
    else if (c->gk.count(kappa))
        key = c->gk[kappa];
    if (!key) CUDA_TRY(c, cudaMalloc(&key, kw * sizeof(u64)));
    if (kind == 0)
        c->rlk = key;
    else {
        c->gk[kappa] = key;
        if (!get_perm(c, kappa)) return fail(c, CKKS_E_OOM, "perm");
    }
    CUDA_TRY(c, cudaMemcpyAsync(key, key_coeff_dev, kw * sizeof(u64), cudaMemcpyDeviceToDevice, c->st));
    launch_ntt_fwd(c->lc(), PolyMap{key, c->L + c->K}, PolyMap{key, c->L + c->K}, 2 * c->dnum, extlimbs(c));
    kc_key_installed(c, key);
    return check_launch(c);
}

ckks_status ckks_import_switch_key(ckks_ctx *c, int kind, int32_t step, const uint64_t *key_coeff_dev)
{
    if (!c || !key_coeff_dev || (kind != 0 && kind != 1)) return CKKS_E_INVALID_ARG;
    return install_switch_key(c, kind, kind == 1 ? galois_elt(c, step) : 0, key_coeff_dev);
}

// ---- boundary form ----------------------------------------------------------------------
ckks_status ckks_import_coeffs(ckks_ctx *c, const uint64_t *src, ckks_buf *dst)
{
    if (!c || !src || !dst || !dst->data || dst->count < 1 || dst->n_polys < 1 || dst->n_polys > 2 ||
        dst->level < 1 || dst->level > c->L || dst->capacity < dst->level)
        return CKKS_E_INVALID_ARG;
    launch_ntt_fwd(c->lc(), PolyMap{const_cast<u64 *>(src), dst->level}, pm(dst), dst->count * dst->n_polys,
                   qlimbs(c, dst->level));
    return check_launch(c);
}

ckks_status ckks_export_coeffs(ckks_ctx *c, const ckks_buf *src, uint64_t *dst)
{
    if (!c || !dst || !src || !src->data || src->count < 1 || src->n_polys < 1 || src->n_polys > 2 ||
        src->level < 1 || src->level > c->L || src->capacity < src->level)
        return CKKS_E_INVALID_ARG;
    launch_ntt_inv(c->lc(), pm(src), PolyMap{dst, src->level}, src->count * src->n_polys, qlimbs(c, src->level),
                   nullptr);
    return check_launch(c);
}

// ---- persistence: host bytes (coefficient form) ------------------------------------------------
namespace {
constexpr size_t SER_HDR = 64;
u64 chain_hash(const u64 *p, u32 n)
{
    u64 h = 1469598103934665603ull;  // FNV-1a over the little-endian bytes of the primes
    for (u32 i = 0; i < n; ++i)
        for (int b = 0; b < 8; ++b) {
            h ^= (p[i] >> (8 * b)) & 0xff;
            h *= 1099511628211ull;
        }
    return h;
}
struct BufHdr {
    char magic[8];
    uint32_t version, log_n, count, n_polys, level, zero;
    double scale;
    uint64_t chain;
    uint64_t pad[2];
};
static_assert(sizeof(BufHdr) == SER_HDR, "header size");
struct KeyHdr {
    char magic[8];
    uint32_t version, log_n, L, K, alpha, n_keys;
    uint64_t chain;
    uint64_t pad[3];
};
static_assert(sizeof(KeyHdr) == SER_HDR, "key header size");
struct KeyRec {
    uint32_t kind, zero;
    uint64_t kappa;
};

ckks_status parse_buf_hdr(ckks_ctx *c, const void *bytes, size_t len, BufHdr &h)
{
    if (!bytes || len < SER_HDR) return fail(c, CKKS_E_INVALID_ARG, "import: truncated header");
    std::memcpy(&h, bytes, SER_HDR);
    if (std::memcmp(h.magic, "CKKSBUF1", 8) || h.version != 1) return fail(c, CKKS_E_INVALID_ARG, "import: not a ckks buffer");
    if (h.log_n != c->log_n || h.level < 1 || h.level > c->L || h.n_polys < 1 || h.n_polys > 2 || h.count < 1)
        return fail(c, CKKS_E_INVALID_ARG, "import: ring / level / shape mismatch");
    if (h.chain != chain_hash(c->primes.data(), h.level)) return fail(c, CKKS_E_INVALID_ARG, "import: foreign prime chain");
    const size_t words = (size_t)h.count * h.n_polys * h.level * c->N;
    if (len != SER_HDR + words * 8) return fail(c, CKKS_E_INVALID_ARG, "import: length mismatch");
    return CKKS_OK;
}

// words [rows][limbs][N] of residues: every limb i below its prime primes[i]
bool canonical(const u64 *w, size_t rows, u32 limbs, u32 N, const u64 *primes)
{
    for (size_t r = 0; r < rows; ++r)
        for (u32 i = 0; i < limbs; ++i) {
            const u64 *x = w + (r * limbs + i) * N, q = primes[i];
            for (u32 k = 0; k < N; ++k)
                if (x[k] >= q) return false;
        }
    return true;
}
}  // namespace

ckks_status ckks_export(ckks_ctx *c, const ckks_buf *src, void *host_bytes, size_t cap, size_t *len)
{
    if (!c || !src || !src->data || !len || src->count < 1 || src->n_polys < 1 || src->n_polys > 2 || src->level < 1 ||
        src->level > c->L || src->capacity < src->level)
        return CKKS_E_INVALID_ARG;
    const size_t words = (size_t)src->count * src->n_polys * src->level * c->N;
    *len = SER_HDR + words * 8;
    if (!host_bytes) return CKKS_OK;
    if (cap < *len) return fail(c, CKKS_E_INVALID_ARG, "export: capacity");
    u64 *d = need(c, "ser", words);
    if (!d) return fail(c, CKKS_E_OOM, "export scratch");
    launch_ntt_inv(c->lc(), pm(src), PolyMap{d, src->level}, src->count * src->n_polys, qlimbs(c, src->level), nullptr);
    BufHdr h{};
    std::memcpy(h.magic, "CKKSBUF1", 8);
    h.version = 1;
    h.log_n = c->log_n;
    h.count = src->count;
    h.n_polys = src->n_polys;
    h.level = src->level;
    h.scale = src->scale;
    h.chain = chain_hash(c->primes.data(), src->level);
    std::memcpy(host_bytes, &h, SER_HDR);
    CUDA_TRY(c, cudaMemcpyAsync(static_cast<char *>(host_bytes) + SER_HDR, d, words * 8, cudaMemcpyDeviceToHost, c->st));
    CUDA_TRY(c, cudaStreamSynchronize(c->st));
    return check_launch(c);
}

ckks_status ckks_import_info(ckks_ctx *c, const void *host_bytes, size_t len, uint32_t *count, uint32_t *n_polys,
                             uint32_t *level, double *scale)
{
    if (!c) return CKKS_E_INVALID_ARG;
    BufHdr h;
    ckks_status s = parse_buf_hdr(c, host_bytes, len, h);
    if (s != CKKS_OK) return s;
    if (count) *count = h.count;
    if (n_polys) *n_polys = h.n_polys;
    if (level) *level = h.level;
    if (scale) *scale = h.scale;
    return CKKS_OK;
}

ckks_status ckks_import(ckks_ctx *c, const void *host_bytes, size_t len, ckks_buf *dst)
{
    if (!c || !dst || !dst->data) return CKKS_E_INVALID_ARG;
    BufHdr h;
    ckks_status s = parse_buf_hdr(c, host_bytes, len, h);
    if (s != CKKS_OK) return s;
    if (dst->count < h.count || dst->capacity < h.level) return fail(c, CKKS_E_INVALID_ARG, "import: destination too small");
    const u64 *w = reinterpret_cast<const u64 *>(static_cast<const char *>(host_bytes) + SER_HDR);
    if (!canonical(w, (size_t)h.count * h.n_polys, h.level, c->N, c->primes.data()))
        return fail(c, CKKS_E_INVALID_ARG, "import: residue not below its prime");
    const size_t words = (size_t)h.count * h.n_polys * h.level * c->N;
    u64 *d = need(c, "ser", words);
    if (!d) return fail(c, CKKS_E_OOM, "import scratch");
    CUDA_TRY(c, cudaMemcpyAsync(d, w, words * 8, cudaMemcpyHostToDevice, c->st));
    dst->count = h.count;
    dst->n_polys = h.n_polys;
    dst->level = h.level;
    dst->scale = h.scale;
    launch_ntt_fwd(c->lc(), PolyMap{d, h.level}, pm(dst), h.count * h.n_polys, qlimbs(c, h.level));
    CUDA_TRY(c, cudaStreamSynchronize(c->st));
    return check_launch(c);
}

ckks_status ckks_export_keys(ckks_ctx *c, void *host_bytes, size_t cap, size_t *len)
{
    if (!c || !len) return CKKS_E_INVALID_ARG;
    const size_t kw = key_words(c), pw = (size_t)2 * c->L * c->N;
    std::vector<std::pair<KeyRec, const u64 *>> keys;
    if (c->pk) keys.push_back({KeyRec{2, 0, 0}, c->pk});
    if (c->rlk) keys.push_back({KeyRec{0, 0, 0}, c->rlk});
    for (auto &kv : c->gk) keys.push_back({KeyRec{1, 0, kv.first}, kv.second});
    size_t total = SER_HDR;
    for (auto &k : keys) total += sizeof(KeyRec) + 8 * (k.first.kind == 2 ? pw : kw);
    *len = total;
    if (!host_bytes) return CKKS_OK;
    if (cap < total) return fail(c, CKKS_E_INVALID_ARG, "export_keys: capacity");
    u64 *d = need(c, "ser", std::max(kw, pw));
    if (!d) return fail(c, CKKS_E_OOM, "export scratch");
    KeyHdr h{};
    std::memcpy(h.magic, "CKKSKEY1", 8);
    h.version = 1;
    h.log_n = c->log_n;
    h.L = c->L;
    h.K = c->K;
    h.alpha = c->alpha;
    h.n_keys = (uint32_t)keys.size();
    h.chain = chain_hash(c->primes.data(), c->L + c->K);
    char *o = static_cast<char *>(host_bytes);
    std::memcpy(o, &h, SER_HDR);
    o += SER_HDR;
    const Launch L = c->lc();
    for (auto &k : keys) {
        std::memcpy(o, &k.first, sizeof(KeyRec));
        o += sizeof(KeyRec);
        const size_t w = k.first.kind == 2 ? pw : kw;
        CUDA_TRY(c, cudaMemcpyAsync(d, k.second, w * 8, cudaMemcpyDeviceToDevice, c->st));
        if (k.first.kind == 2) {
            launch_ntt_inv(L, PolyMap{d, c->L}, PolyMap{d, c->L}, 2, qlimbs(c, c->L), nullptr);
        } else {
            if (c->ksc) launch_key_mac_layout(L, d, c->d_kc_limbs, c->n_kc_limbs, 2 * c->dnum, c->L + c->K, true);
            if (c->kcomp) {
                u64 *tmp = need(c, "kcomp_tmp", (size_t)2 * c->dnum * c->N);
                if (!tmp) return fail(c, CKKS_E_OOM, "export scratch");
                launch_key_compact(L, d, c->kcomp_limbs.data(), (u32)c->kcomp_limbs.size(), 2 * c->dnum, c->L + c->K,
                                   true, tmp);
            }
            launch_ntt_inv(L, PolyMap{d, c->L + c->K}, PolyMap{d, c->L + c->K}, 2 * c->dnum, extlimbs(c), nullptr);
        }
        CUDA_TRY(c, cudaMemcpyAsync(o, d, w * 8, cudaMemcpyDeviceToHost, c->st));
        CUDA_TRY(c, cudaStreamSynchronize(c->st));
        o += w * 8;
    }
    return check_launch(c);
}

ckks_status ckks_import_keys(ckks_ctx *c, const void *host_bytes, size_t len)
{
    if (!c || !host_bytes || len < SER_HDR) return CKKS_E_INVALID_ARG;
    KeyHdr h;
    std::memcpy(&h, host_bytes, SER_HDR);
    if (std::memcmp(h.magic, "CKKSKEY1", 8) || h.version != 1) return fail(c, CKKS_E_INVALID_ARG, "import_keys: not a key file");
    if (h.log_n != c->log_n || h.L != c->L || h.K != c->K || h.alpha != c->alpha ||
        h.chain != chain_hash(c->primes.data(), c->L + c->K))
        return fail(c, CKKS_E_INVALID_ARG, "import_keys: keys of another parameter set");
    const size_t kw = key_words(c), pw = (size_t)2 * c->L * c->N;
    // validate the whole file before installing anything
    std::vector<u64> ext(c->primes.begin(), c->primes.end());
    const char *p = static_cast<const char *>(host_bytes) + SER_HDR, *end = static_cast<const char *>(host_bytes) + len;
    for (uint32_t i = 0; i < h.n_keys; ++i) {
        if (end - p < (ptrdiff_t)sizeof(KeyRec)) return fail(c, CKKS_E_INVALID_ARG, "import_keys: truncated");
        KeyRec r;
        std::memcpy(&r, p, sizeof(KeyRec));
        p += sizeof(KeyRec);
        if (r.kind > 2 || (r.kind == 1 && (r.kappa % 2 == 0 || r.kappa >= 2ull * c->N)))
            return fail(c, CKKS_E_INVALID_ARG, "import_keys: bad record");
        const size_t w = r.kind == 2 ? pw : kw;
        if ((size_t)(end - p) < w * 8) return fail(c, CKKS_E_INVALID_ARG, "import_keys: truncated");
        const u64 *x = reinterpret_cast<const u64 *>(p);
        if (!(r.kind == 2 ? canonical(x, 2, c->L, c->N, ext.data()) : canonical(x, 2 * c->dnum, c->L + c->K, c->N, ext.data())))
            return fail(c, CKKS_E_INVALID_ARG, "import_keys: residue not below its prime");
        p += w * 8;
    }
    if (p != end) return fail(c, CKKS_E_INVALID_ARG, "import_keys: length mismatch");
    u64 *d = need(c, "ser", std::max(kw, pw));
    if (!d) return fail(c, CKKS_E_OOM, "import scratch");
    p = static_cast<const char *>(host_bytes) + SER_HDR;
    for (uint32_t i = 0; i < h.n_keys; ++i) {
        KeyRec r;
        std::memcpy(&r, p, sizeof(KeyRec));
        p += sizeof(KeyRec);
        const size_t w = r.kind == 2 ? pw : kw;
        CUDA_TRY(c, cudaMemcpyAsync(d, p, w * 8, cudaMemcpyHostToDevice, c->st));
        ckks_status s;
        if (r.kind == 2) {
            if (!c->pk) CUDA_TRY(c, cudaMalloc(&c->pk, pw * sizeof(u64)));
            launch_ntt_fwd(c->lc(), PolyMap{d, c->L}, PolyMap{c->pk, c->L}, 2, qlimbs(c, c->L));
            s = check_launch(c);
        } else {
            s = install_switch_key(c, (int)r.kind, r.kappa, d);
        }
        if (s != CKKS_OK) return s;
        CUDA_TRY(c, cudaStreamSynchronize(c->st));
        p += w * 8;
    }
    return CKKS_OK;
}

ckks_status ckks_ntt(ckks_ctx *c, uint64_t *data, uint32_t count, uint32_t level, int inverse)
{
    if (!c || !data || count < 1 || level < 1 || level > c->L + c->K) return CKKS_E_INVALID_ARG;
    PolyMap m{data, level};
    LimbSet ls = level <= c->L ? qlimbs(c, level) : extlimbs(c);
    if (inverse)
        launch_ntt_inv(c->lc(), m, m, count, ls, nullptr);
    else
        launch_ntt_fwd(c->lc(), m, m, count, ls);
    return check_launch(c);
}

// ---- encode / decode --------------------------------------------------------------------
ckks_status ckks_encode(ckks_ctx *c, const double *re, const double *im, size_t n_slots, double scale,
                        uint32_t level, ckks_buf *pt)
{
    if (!c || (!re && n_slots) || !pt || !pt->data || pt->count != 1 || pt->n_polys != 1 || level < 1 ||
        level > c->L || pt->capacity < level || !(scale > 0))
        return CKKS_E_INVALID_ARG;
    if (n_slots > c->N / 2) return fail(c, CKKS_E_INVALID_ARG, "overlong vector (S:170)");
    std::vector<std::complex<double>> z(n_slots);
    for (size_t j = 0; j < n_slots; ++j) z[j] = std::complex<double>(re[j], im ? im[j] : 0.0);
    std::vector<double> coef;
    hm::encode(z.data(), n_slots, scale, c->log_n, coef);
    std::vector<int64_t> ic(c->N);
    for (u32 k = 0; k < c->N; ++k) {
        bool ok;
        ic[k] = llround_checked(coef[k], ok);
        if (!ok) return fail(c, CKKS_E_ENCODE_OVERFLOW, "encoded coefficient overflows int64");
    }
    u64 *tmp = need(c, "encode", c->N);
    if (!tmp) return fail(c, CKKS_E_OOM, "encode scratch");
    CUDA_TRY(c, cudaMemcpyAsync(tmp, ic.data(), c->N * sizeof(int64_t), cudaMemcpyHostToDevice, c->st));
    launch_from_signed(c->lc(), reinterpret_cast<const int64_t *>(tmp), pm(pt), 1, qlimbs(c, level));
    launch_ntt_fwd(c->lc(), pm(pt), pm(pt), 1, qlimbs(c, level));
    CUDA_TRY(c, cudaStreamSynchronize(c->st));
    pt->level = level;
    pt->scale = scale;
    return check_launch(c);
}

ckks_status ckks_decode(ckks_ctx *c, const ckks_buf *pt, double *re_out, double *im_out, size_t n_slots)
{
    if (!c || !valid_buf(c, pt, 1) || pt->count != 1 || n_slots > c->N / 2) return CKKS_E_INVALID_ARG;
    const u32 l = pt->level;
    u64 *tmp = need(c, "decode", (size_t)l * c->N);
    if (!tmp) return fail(c, CKKS_E_OOM, "decode scratch");
    launch_ntt_inv(c->lc(), pm(pt), PolyMap{tmp, l}, 1, qlimbs(c, l), nullptr);
    std::vector<u64> h((size_t)l * c->N);
    CUDA_TRY(c, cudaMemcpyAsync(h.data(), tmp, h.size() * sizeof(u64), cudaMemcpyDeviceToHost, c->st));
    CUDA_TRY(c, cudaStreamSynchronize(c->st));
    hm::Crt crt;
    crt.init(std::vector<u64>(c->primes.begin(), c->primes.begin() + l));
    std::vector<double> coef(c->N);
    for (u32 k = 0; k < c->N; ++k) coef[k] = crt.centred(h.data() + k, c->N);
    std::vector<std::complex<double>> z;
    hm::decode(coef, pt->scale, c->log_n, z);
    for (size_t j = 0; j < n_slots; ++j) {
        if (re_out) re_out[j] = z[j].real();
        if (im_out) im_out[j] = z[j].imag();
    }
    return CKKS_OK;
}

// ---- batched GPU encode / decode (f4) --------------------------------------------------------
namespace {
ckks_status codec_tables(ckks_ctx *c)
{
    if (c->d_fft_w) return CKKS_OK;
    const u32 n = c->N;
    std::vector<double2> w(n), tw(n);
    for (u32 m = 0; m < n; ++m) {
        const double a = -2.0 * M_PI * (double)m / (double)n, b = -M_PI * (double)m / (double)n;
        w[m] = make_double2(std::cos(a), std::sin(a));
        tw[m] = make_double2(std::cos(b), std::sin(b));
    }
    // slot j < N/2 feeds bins (r_j - 1)/2 and N - 1 - (r_j - 1)/2 (conjugate), r_j = 5^j mod 2N
    std::vector<u32> slot(n, 0xffffffffu);
    u64 r = 1;
    for (u32 j = 0; j < n / 2; ++j) {
        const u32 s = (u32)((r - 1) / 2);
        slot[s] = j;
        slot[n - 1 - s] = j | 0x80000000u;
        r = (r * 5) % (2 * (u64)n);
    }
    for (u32 v : slot)
        if (v == 0xffffffffu) return fail(c, CKKS_E_UNSUPPORTED, "slot map is not a bijection");
    auto up = [&](void **d, const void *h, size_t bytes) -> bool {
        return cudaMalloc(d, bytes) == cudaSuccess && cudaMemcpy(*d, h, bytes, cudaMemcpyHostToDevice) == cudaSuccess;
    };
    if (!up((void **)&c->d_fft_w, w.data(), n * sizeof(double2)) ||
        !up((void **)&c->d_fft_tw, tw.data(), n * sizeof(double2)) ||
        !up((void **)&c->d_slot, slot.data(), n * sizeof(u32)) ||
        cudaMalloc((void **)&c->d_enc_overflow, sizeof(int)) != cudaSuccess ||
        cudaMemset(c->d_enc_overflow, 0, sizeof(int)) != cudaSuccess) {
        cudaGetLastError();
        return fail(c, CKKS_E_OOM, "codec tables");
    }
    return CKKS_OK;
}

// centred-CRT constants at level l (reading A33): (Q/q_i) mod 2^128 by wrapping u128
// products, (Q/q_i)^{-1} mod q_i, 1/q_i, and Q mod 2^128.
const ckks_ctx::CrtLevel *crt_level(ckks_ctx *c, u32 l)
{
    auto it = c->crt.find(l);
    if (it != c->crt.end()) return &it->second;
    std::vector<CrtConst> h(l);
    unsigned __int128 Q = 1;
    for (u32 i = 0; i < l; ++i) Q *= c->primes[i];
    for (u32 i = 0; i < l; ++i) {
        const u64 q = c->primes[i];
        unsigned __int128 qh = 1;
        u64 qh_mod = 1;
        for (u32 j = 0; j < l; ++j)
            if (j != i) {
                qh *= c->primes[j];
                qh_mod = hm::mulmod(qh_mod, c->primes[j] % q, q);
            }
        const u64 inv = hm::invmod(qh_mod, q);
        h[i] = CrtConst{(u64)qh, (u64)(qh >> 64), inv, hm::shoup(inv, q), 1.0 / (double)q, 0.0};
    }
    ckks_ctx::CrtLevel lv;
    lv.Q_lo = (u64)Q;
    lv.Q_hi = (u64)(Q >> 64);
    if (cudaMalloc((void **)&lv.c, l * sizeof(CrtConst)) != cudaSuccess ||
        cudaMemcpy(lv.c, h.data(), l * sizeof(CrtConst), cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return &(c->crt[l] = lv);
}

CodecTabs codec_of(const ckks_ctx *c) { return CodecTabs{c->d_fft_w, c->d_fft_tw, c->d_slot}; }
}  // namespace

ckks_status ckks_encode_batch(ckks_ctx *c, const double *z, size_t n_slots, double scale, uint32_t level,
                              ckks_buf *pt)
{
    if (!c || (!z && n_slots) || !pt || !pt->data || pt->count < 1 || pt->n_polys != 1 || level < 1 ||
        level > c->L || pt->capacity < level || !(scale > 0) || !std::isfinite(scale))
        return CKKS_E_INVALID_ARG;
    if (n_slots > c->N / 2) return fail(c, CKKS_E_INVALID_ARG, "overlong vector (S:170)");
    if (ckks_status s = codec_tables(c)) return s;
    double2 *Y = reinterpret_cast<double2 *>(need(c, "codecY", (size_t)2 * pt->count * c->N));
    if (!Y) return fail(c, CKKS_E_OOM, "encode scratch");
    const Launch L = c->lc();
    launch_encode(L, codec_of(c), reinterpret_cast<const double2 *>(z), (u32)n_slots, scale, pt->count, Y, pm(pt),
                  level, c->d_enc_overflow);
    launch_ntt_fwd(L, pm(pt), pm(pt), pt->count, qlimbs(c, level));
    pt->level = level;
    pt->scale = scale;
    return check_launch(c);
}

ckks_status ckks_decode_batch(ckks_ctx *c, const ckks_buf *pt, double *z, size_t n_slots)
{
    if (!c || !valid_buf(c, pt, 1) || (!z && n_slots) || n_slots > c->N / 2) return CKKS_E_INVALID_ARG;
    if (ckks_status s = codec_tables(c)) return s;
    const u32 l = pt->level, cnt = pt->count;
    const ckks_ctx::CrtLevel *cl = crt_level(c, l);
    if (!cl) return fail(c, CKKS_E_OOM, "CRT constants");
    u64 *C = need(c, "decodeC", (size_t)cnt * l * c->N);
    double2 *Y = reinterpret_cast<double2 *>(need(c, "codecY", (size_t)2 * cnt * c->N));
    if (!C || !Y) return fail(c, CKKS_E_OOM, "decode scratch");
    const Launch L = c->lc();
    launch_ntt_inv(L, pm(pt), PolyMap{C, l}, cnt, qlimbs(c, l), nullptr);
    launch_decode(L, codec_of(c), C, l, cl->c, cl->Q_lo, cl->Q_hi, cnt, Y, reinterpret_cast<double2 *>(z),
                  (u32)n_slots, pt->scale);
    return check_launch(c);
}

ckks_status ckks_encode_overflowed(ckks_ctx *c, int *flag)
{
    if (!c || !flag) return CKKS_E_INVALID_ARG;
    *flag = 0;
    if (!c->d_enc_overflow) return CKKS_OK;
    CUDA_TRY(c, cudaMemcpyAsync(flag, c->d_enc_overflow, sizeof(int), cudaMemcpyDeviceToHost, c->st));
    CUDA_TRY(c, cudaStreamSynchronize(c->st));
    CUDA_TRY(c, cudaMemsetAsync(c->d_enc_overflow, 0, sizeof(int), c->st));
    return CKKS_OK;
}

// ---- fused peer-memory modular all-reduce (f3) ---------------------------------------------
static_assert(sizeof(cudaIpcMemHandle_t) == CKKS_IPC_HANDLE_BYTES, "IPC handle size");

ckks_status ckks_ipc_export(ckks_ctx *c, const void *p, void *handle_out, uint64_t *offset_out)
{
    if (!c || !p || !handle_out || !offset_out) return CKKS_E_INVALID_ARG;
    CUDA_TRY(c, cudaSetDevice(c->device));
    // base of the allocation holding p (torch's caching allocator sub-allocates segments)
    using GetRange = int (*)(unsigned long long *, size_t *, unsigned long long);
    static GetRange get_range = nullptr;
    if (!get_range) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        CUDA_TRY(c, cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
        if (!fn || q != cudaDriverEntryPointSuccess) return fail(c, CKKS_E_CUDA, "cuMemGetAddressRange unavailable");
        get_range = reinterpret_cast<GetRange>(fn);
    }
    unsigned long long base = 0;
    size_t size = 0;
    if (get_range(&base, &size, (unsigned long long)(uintptr_t)p) != 0)
        return fail(c, CKKS_E_INVALID_ARG, "pointer is not device memory");
    cudaIpcMemHandle_t h;
    CUDA_TRY(c, cudaIpcGetMemHandle(&h, (void *)(uintptr_t)base));
    std::memcpy(handle_out, &h, sizeof(h));
    *offset_out = (uint64_t)((uintptr_t)p - base);
    return CKKS_OK;
}

ckks_status ckks_ipc_open(ckks_ctx *c, const void *handle, uint64_t offset, void **out)
{
    if (!c || !handle || !out) return CKKS_E_INVALID_ARG;
    CUDA_TRY(c, cudaSetDevice(c->device));
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    void *base = nullptr;
    CUDA_TRY(c, cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    *out = static_cast<char *>(base) + offset;
    c->ipc[*out] = base;
    return CKKS_OK;
}

ckks_status ckks_ipc_close(ckks_ctx *c, void *p)
{
    if (!c) return CKKS_E_INVALID_ARG;
    auto it = c->ipc.find(p);
    if (it == c->ipc.end()) return fail(c, CKKS_E_INVALID_ARG, "not a pointer returned by ckks_ipc_open");
    void *base = it->second;
    c->ipc.erase(it);
    for (auto &kv : c->ipc)
        if (kv.second == base) return CKKS_OK;  // another view of the same mapping stays open
    CUDA_TRY(c, cudaIpcCloseMemHandle(base));
    return CKKS_OK;
}

ckks_status ckks_p2p_modsum(ckks_ctx *c, uint64_t *const *in, uint64_t *const *out, uint32_t R, uint32_t rank,
                            const ckks_buf *shape)
{
    if (!c || !in || !out || R < 1 || R > CKKS_MAX_PEERS || rank >= R || !shape || shape->count < 1 ||
        shape->n_polys < 1 || shape->level < 1 || shape->level > c->L || shape->capacity < shape->level)
        return CKKS_E_INVALID_ARG;
    for (u32 r = 0; r < R; ++r)
        if (!in[r] || !out[r]) return CKKS_E_INVALID_ARG;
    launch_p2p_modsum(c->lc(), in, out, R, rank, shape->count * shape->n_polys, shape->level, shape->capacity);
    return check_launch(c);
}

// ---- encrypt / decrypt ----------------------------------------------------------------------
ckks_status ckks_encrypt(ckks_ctx *c, const ckks_buf *pt, const int64_t *u, const int64_t *e0, const int64_t *e1,
                         ckks_buf *ct)
{
    if (!c || !valid_buf(c, pt, 1) || !u || !e0 || !e1 || !ct || !ct->data || ct->capacity < pt->level ||
        ct->count != pt->count)
        return CKKS_E_INVALID_ARG;
    if (!c->pk) return fail(c, CKKS_E_MISSING_KEY, "public key not set");
    const u32 l = pt->level, cnt = pt->count;
    const size_t n = c->N, w = (size_t)cnt * l * n;
    u64 *U = need(c, "enc", 3 * w);
    if (!U) return fail(c, CKKS_E_OOM, "encrypt scratch");
    u64 *E0 = U + w, *E1 = E0 + w;
    const Launch L = c->lc();
    const int64_t *src[3] = {u, e0, e1};
    u64 *dst[3] = {U, E0, E1};
    for (int k = 0; k < 3; ++k) {
        launch_from_signed(L, src[k], PolyMap{dst[k], l}, cnt, qlimbs(c, l));
        launch_ntt_fwd(L, PolyMap{dst[k], l}, PolyMap{dst[k], l}, cnt, qlimbs(c, l));
    }
    ct->n_polys = 2;
    ct->count = cnt;
    PolyMap c0 = pm_c(ct, 0, c->N), c1 = pm_c(ct, 1, c->N);
    launch_mul_add(L, PolyMap{U, l}, PolyMap{c->pk, c->L}, 1, PolyMap{E0, l}, c0, cnt, l, 0);  // b u + e0
    launch_addsub(L, c0, pm(pt), c0, cnt, l, EL_ADD);                                          // + mu
    launch_mul_add(L, PolyMap{U, l}, PolyMap{c->pk + c->L * n, c->L}, 1, PolyMap{E1, l}, c1, cnt, l, 0);  // a u + e1
    ct->level = l;
    ct->scale = pt->scale;
    return check_launch(c);
}

ckks_status ckks_decrypt(ckks_ctx *c, const ckks_buf *ct, ckks_buf *pt)
{
    if (!c || !valid_buf(c, ct, 2) || !pt || !pt->data || pt->capacity < ct->level) return CKKS_E_INVALID_ARG;
    if (!c->sk) return fail(c, CKKS_E_MISSING_KEY, "secret key not set");
    launch_mul_add(c->lc(), pm_c(ct, 1, c->N), PolyMap{c->sk, c->L + c->K}, 1, pm_c(ct, 0, c->N), pm(pt), ct->count,
                   ct->level, 0);
    pt->n_polys = 1;
    pt->count = ct->count;
    pt->level = ct->level;
    pt->scale = ct->scale;
    return check_launch(c);
}

// ---- homomorphic ops ------------------------------------------------------------------------
static ckks_status addsub(ckks_ctx *c, const ckks_buf *a, const ckks_buf *b, ckks_buf *out, int op)
{
    if (!c || !valid_buf(c, a, 2) || !valid_buf(c, b, 2) || !out || !out->data || out->capacity < a->level ||
        a->count != b->count)
        return CKKS_E_INVALID_ARG;
    if (a->level != b->level) return fail(c, CKKS_E_LEVEL_MISMATCH, "level mismatch");
    if (a->scale != b->scale) return fail(c, CKKS_E_SCALE_MISMATCH, "scale mismatch");
    launch_addsub(c->lc(), pm(a), pm(b), pm(out), a->count * 2, a->level, op);
    out->n_polys = 2;
    out->count = a->count;
    out->level = a->level;
    out->scale = a->scale;
    return check_launch(c);
}

ckks_status ckks_add(ckks_ctx *c, const ckks_buf *a, const ckks_buf *b, ckks_buf *out) { return addsub(c, a, b, out, EL_ADD); }
ckks_status ckks_sub(ckks_ctx *c, const ckks_buf *a, const ckks_buf *b, ckks_buf *out) { return addsub(c, a, b, out, EL_SUB); }

ckks_status ckks_add_plain(ckks_ctx *c, const ckks_buf *ct, const ckks_buf *pt, ckks_buf *out)
{
    if (!c || !valid_buf(c, ct, 2) || !valid_buf(c, pt, 1) || !out || !out->data || out->capacity < ct->level ||
        (pt->count != 1 && pt->count != ct->count))
        return CKKS_E_INVALID_ARG;
    if (ct->level != pt->level) return fail(c, CKKS_E_LEVEL_MISMATCH, "level mismatch");
    if (ct->scale != pt->scale) return fail(c, CKKS_E_SCALE_MISMATCH, "scale mismatch");
    launch_add_plain(c->lc(), pm(ct), pm(pt), pt->count == 1 ? 1 : 0, pm(out), ct->count, ct->level);
    out->n_polys = 2;
    out->count = ct->count;
    out->level = ct->level;
    out->scale = ct->scale;
    return check_launch(c);
}

ckks_status ckks_mul_plain(ckks_ctx *c, const ckks_buf *ct, const ckks_buf *pt, ckks_buf *out)
{
    if (!c || !valid_buf(c, ct, 2) || !valid_buf(c, pt, 1) || !out || !out->data || out->capacity < ct->level ||
        (pt->count != 1 && pt->count != ct->count))
        return CKKS_E_INVALID_ARG;
    if (ct->level != pt->level) return fail(c, CKKS_E_LEVEL_MISMATCH, "level mismatch");
    launch_mul_poly(c->lc(), pm(ct), pm(pt), 2, pt->count == 1 ? 1 : 0, pm(out), 2 * ct->count, ct->level);
    out->n_polys = 2;
    out->count = ct->count;
    out->level = ct->level;
    out->scale = ct->scale * pt->scale;
    return check_launch(c);
}

ckks_status ckks_mul_const(ckks_ctx *c, const ckks_buf *ct, double value, double const_scale, ckks_buf *out)
{
    if (!c || !valid_buf(c, ct, 2) || !out || !out->data || out->capacity < ct->level || !(const_scale > 0))
        return CKKS_E_INVALID_ARG;
    bool ok;
    const long long v = llround_checked(value * const_scale, ok);
    if (!ok) return fail(c, CKKS_E_ENCODE_OVERFLOW, "constant overflows int64");
    std::vector<ulonglong2> h(ct->level);
    for (u32 i = 0; i < ct->level; ++i) {
        const u64 q = c->primes[i], r = residue_of(v, q);
        h[i] = make_ulonglong2(r, hm::shoup(r, q));
    }
    ulonglong2 *d;
    ckks_status s = upload_consts(c, h, "const", &d);
    if (s != CKKS_OK) return s;
    launch_mul_scalar(c->lc(), pm(ct), pm(out), 2 * ct->count, ct->level, d);
    out->n_polys = 2;
    out->count = ct->count;
    out->level = ct->level;
    out->scale = ct->scale * const_scale;
    return check_launch(c);
}

ckks_status ckks_add_const(ckks_ctx *c, const ckks_buf *ct, double value, ckks_buf *out)
{
    if (!c || !valid_buf(c, ct, 2) || !out || !out->data || out->capacity < ct->level) return CKKS_E_INVALID_ARG;
    bool ok;
    const long long v = llround_checked(value * ct->scale, ok);
    if (!ok) return fail(c, CKKS_E_ENCODE_OVERFLOW, "constant overflows int64");
    std::vector<ulonglong2> h((ct->level + 1) / 2);
    std::vector<u64> r(ct->level + (ct->level & 1), 0);
    for (u32 i = 0; i < ct->level; ++i) r[i] = residue_of(v, c->primes[i]);
    std::memcpy(h.data(), r.data(), r.size() * sizeof(u64));
    ulonglong2 *d;
    ckks_status s = upload_consts(c, h, "const", &d);
    if (s != CKKS_OK) return s;
    launch_add_scalar_c0(c->lc(), pm(ct), pm(out), ct->count, ct->level, reinterpret_cast<const u64 *>(d));
    out->n_polys = 2;
    out->count = ct->count;
    out->level = ct->level;
    out->scale = ct->scale;
    return check_launch(c);
}

ckks_status ckks_mul_relin(ckks_ctx *c, const ckks_buf *a, const ckks_buf *b, ckks_buf *out)
{
    NvtxRange nv_("mul_relin");
    if (!c || !valid_buf(c, a, 2) || !valid_buf(c, b, 2) || !out || !out->data || out->capacity < a->level ||
        a->count != b->count)
        return CKKS_E_INVALID_ARG;
    if (a->level != b->level) return fail(c, CKKS_E_LEVEL_MISMATCH, "level mismatch");
    if (!c->rlk) return fail(c, CKKS_E_MISSING_KEY, "relinearisation key not set");
    const u32 l = a->level, cnt = a->count;
    u64 *d2 = need(c, "d2", (size_t)cnt * l * c->N);
    if (!d2) return fail(c, CKKS_E_OOM, "tensor scratch");
    const double sc = a->scale * b->scale;
    u64 *dr = tensor_for_relin(c, a, b, out, d2, cnt, l);
    ckks_status s = keyswitch(c, PolyMap{d2, l}, nullptr, cnt, l, c->rlk, pm(out), pm(out), nullptr, false,
                              PolyMap{nullptr, 0}, dr);
    out->n_polys = 2;
    out->count = cnt;
    out->level = l;
    out->scale = sc;
    return s;
}

ckks_status ckks_mul_relin_rescale(ckks_ctx *c, const ckks_buf *a, const ckks_buf *b, ckks_buf *out)
{
    NvtxRange nv_("mul_relin_rescale");
    if (!c || !valid_buf(c, a, 2) || !valid_buf(c, b, 2) || !out || !out->data || out->capacity < a->level ||
        a->count != b->count)
        return CKKS_E_INVALID_ARG;
    if (a->level != b->level) return fail(c, CKKS_E_LEVEL_MISMATCH, "level mismatch");
    if (a->level < 2) return fail(c, CKKS_E_LEVEL_EXHAUSTED, "rescale at level 1");
    if (!c->rlk) return fail(c, CKKS_E_MISSING_KEY, "relinearisation key not set");
    const u32 l = a->level, cnt = a->count;
    if ((c->alpha > 1 || c->K > 1) && std::getenv("CKKS_HYB_RS") && std::getenv("CKKS_HYB_RS")[0] == '0') {
        ckks_status s = ckks_mul_relin(c, a, b, out);  // two steps (A/B and tests)
        return s != CKKS_OK ? s : ckks_rescale(c, out, out);
    }
    u64 *d2 = need(c, "d2", (size_t)cnt * l * c->N);
    if (!d2) return fail(c, CKKS_E_OOM, "tensor scratch");
    const double sc = a->scale * b->scale / (double)c->primes[l - 1];
    u64 *dr = tensor_for_relin(c, a, b, out, d2, cnt, l);
    if (c->alpha > 1 || c->K > 1) {  // hybrid: ModDown by the K special primes and RESCALE in one tail
        ckks_status s = keyswitch_hybrid(c, PolyMap{d2, l}, nullptr, cnt, l, c->rlk, pm(out), pm(out), nullptr, false,
                                         PolyMap{nullptr, 0}, dr, true);
        out->n_polys = 2;
        out->count = cnt;
        out->level = l - 1;
        out->scale = sc;
        return s;
    }
    ckks_status s = keyswitch_range(c, PolyMap{d2, l}, nullptr, cnt, l, c->rlk, 0, l, KsDigits{nullptr, 0, 0}, pm(out),
                                    pm(out), nullptr, false, PolyMap{nullptr, 0}, true, dr);
    out->n_polys = 2;
    out->count = cnt;
    out->level = l - 1;
    out->scale = sc;
    return s;
}

ckks_status ckks_rescale(ckks_ctx *c, const ckks_buf *ct, ckks_buf *out)
{
    NvtxRange nv_("rescale");
    if (!c || !valid_buf(c, ct, 2) || !out || !out->data || out->capacity + 1 < ct->level) return CKKS_E_INVALID_ARG;
    if (ct->level < 2) return fail(c, CKKS_E_LEVEL_EXHAUSTED, "rescale at level 1 (S:206)");
    return rescale_impl(c, ct, out);
}

ckks_status ckks_rotate(ckks_ctx *c, const ckks_buf *ct, int32_t steps, ckks_buf *out)
{
    NvtxRange nv_("rotate");
    if (!c || !valid_buf(c, ct, 2) || !out || !out->data || out->capacity < ct->level) return CKKS_E_INVALID_ARG;
    return rotate_impl(c, ct, steps, out);
}

ckks_status ckks_total_sum(ckks_ctx *c, const ckks_buf *ct, ckks_buf *out)
{
    NvtxRange nv_("total_sum");
    if (!c || !valid_buf(c, ct, 2) || !out || !out->data || out->capacity < ct->level) return CKKS_E_INVALID_ARG;
    for (u32 i = 0; i + 1 < c->log_n; ++i)
        if (!c->gk.count(galois_elt(c, 1 << i)))
            return fail(c, CKKS_E_MISSING_KEY, "missing Galois key for step " + std::to_string(1 << i));
    copy_ct(c, ct, out);
    ckks_buf t = tmp_ct(c, "tsum", ct);
    if (!t.data) return fail(c, CKKS_E_OOM, "total-sum scratch");
    ckks_buf *cur = out, *nxt = &t;  // ping-pong: nxt = cur + rotate(cur, 2^i)
    for (u32 i = 0; i + 1 < c->log_n; ++i) {  // reading A11: i = 0 .. log2(N/2) - 1
        ckks_status s = galois_step(c, cur, 1 << i, nxt, true);
        if (s != CKKS_OK) return s;
        std::swap(cur, nxt);
    }
    if (cur != out) copy_ct(c, cur, out);
    return check_launch(c);
}

ckks_status ckks_modadd_gathered(ckks_ctx *c, const uint64_t *g, uint32_t R, ckks_buf *out)
{
    if (!c || !g || R < 1 || !out || !out->data || out->count < 1 || out->level < 1 || out->level > c->L ||
        out->capacity < out->level)
        return CKKS_E_INVALID_ARG;
    const size_t stride = (size_t)out->count * out->n_polys * out->capacity * c->N;
    launch_modadd_gathered(c->lc(), g, stride, R, pm(out), out->count * out->n_polys, out->level);
    return check_launch(c);
}

// ---- limb-sharded key switching ------------------------------------------------
static bool shard_ok(const ckks_ctx *c, const ckks_buf *b, uint32_t lo, uint32_t l, uint32_t np)
{
    return b && b->data && b->count >= 1 && b->n_polys == np && l >= 1 && l <= c->L && lo < l &&
           b->level == std::min<u32>(l - lo, b->level) && b->level >= 1 && lo + b->level <= l &&
           b->capacity >= b->level;
}
// global-limb-indexed view of a shard holding limbs [lo, lo + level): limb i at local i - lo
static PolyMap shard_pm(const ckks_buf *b, uint32_t lo, uint32_t which_c = 2, u32 N = 0)
{
    u64 *base = b->data + (which_c < 2 ? (size_t)which_c * b->capacity * N : 0);
    const u32 cap = which_c < 2 ? 2 * b->capacity : b->capacity;
    return PolyMap{base - (size_t)lo * N, cap};
}

ckks_status ckks_shard_ks_digits(ckks_ctx *c, int kind, int32_t step, const ckks_buf *a, const ckks_buf *b,
                                 uint32_t lo, uint32_t l, uint32_t w, ckks_buf *out, uint64_t *D_own)
{
    if (!c || !shard_ok(c, a, lo, l, 2) || !D_own || w < a->level || (kind != 0 && kind != 1))
        return CKKS_E_INVALID_ARG;
    if (c->alpha > 1 || c->K > 1) return fail(c, CKKS_E_UNSUPPORTED, "sharded key switch needs alpha = K = 1");
    const u32 nl = a->level, cnt = a->count;
    const size_t n = c->N;
    if (kind == 0) {
        if (!shard_ok(c, b, lo, l, 2) || b->level != nl || b->count != cnt || !out || !out->data ||
            out->capacity < nl)
            return CKKS_E_INVALID_ARG;
        if (!c->rlk) return fail(c, CKKS_E_MISSING_KEY, "relinearisation key not set");
        u64 *d2 = need(c, ("shd2_" + std::to_string(lo)).c_str(), (size_t)cnt * nl * n);
        if (!d2) return fail(c, CKKS_E_OOM, "shard scratch");
        Tables ts = c->tb;  // elementwise kernels index moduli by local limb: shift the tables
        ts.mod = c->d_mod + lo;
        ts.psi = c->tb.psi + ((size_t)lo << c->log_n);
        ts.ipsi = c->tb.ipsi + ((size_t)lo << c->log_n);
        ts.psif = c->tb.psif + ((size_t)lo << c->log_n);
        ts.ipsif = c->tb.ipsif + ((size_t)lo << c->log_n);
        ts.ninv = c->tb.ninv + lo;
        Launch Ls{&ts, c->st, &c->launches, c->prof, c->primes.data() + lo};
        launch_tensor(Ls, pm(a), pm(b), pm(out), PolyMap{d2, nl}, cnt, nl);
        launch_ntt_inv(c->lc(), PolyMap{d2, nl}, PolyMap{D_own, w}, cnt, LimbSet{nl, nl, lo, c->L}, nullptr);
        out->n_polys = 2;
        out->count = cnt;
        out->level = nl;
        out->scale = a->scale * b->scale;
    } else {
        const u64 kappa = galois_elt(c, step);
        if (!c->gk.count(kappa)) return fail(c, CKKS_E_MISSING_KEY, "missing Galois key");
        const u32 *perm = get_perm(c, kappa);
        if (!perm) return fail(c, CKKS_E_OOM, "perm");
        launch_ntt_inv(c->lc(), pm_c(a, 1, c->N), PolyMap{D_own, w}, cnt, LimbSet{nl, nl, lo, c->L}, perm);
    }
    return check_launch(c);
}

ckks_status ckks_shard_ks_finish(ckks_ctx *c, int kind, int32_t step, const uint64_t *D_all, uint32_t R, uint32_t w,
                                 const ckks_buf *a, uint32_t lo, uint32_t l, ckks_buf *out)
{
    if (!c || !shard_ok(c, a, lo, l, 2) || !D_all || R < 1 || (size_t)R * w < l || !out || !out->data ||
        out->capacity < a->level || (kind != 0 && kind != 1))
        return CKKS_E_INVALID_ARG;
    if (c->alpha > 1 || c->K > 1) return fail(c, CKKS_E_UNSUPPORTED, "sharded key switch needs alpha = K = 1");
    const u32 nl = a->level, cnt = a->count;
    const size_t n = c->N;
    const KsDigits dg{D_all, w, cnt};
    PolyMap o = shard_pm(out, lo, 2, c->N);
    ckks_status s;
    if (kind == 0) {
        if (!c->rlk) return fail(c, CKKS_E_MISSING_KEY, "relinearisation key not set");
        u64 *d2 = need(c, ("shd2_" + std::to_string(lo)).c_str(), (size_t)cnt * nl * n);  // kept by ckks_shard_ks_digits
        s = keyswitch_range(c, PolyMap{d2 - (size_t)lo * n, nl}, nullptr, cnt, l, c->rlk, lo, lo + nl, dg, o, o,
                            nullptr, false);
    } else {
        const u64 kappa = galois_elt(c, step);
        auto it = c->gk.find(kappa);
        if (it == c->gk.end()) return fail(c, CKKS_E_MISSING_KEY, "missing Galois key");
        const u32 *perm = get_perm(c, kappa);
        s = keyswitch_range(c, shard_pm(a, lo, 1, c->N), perm, cnt, l, it->second, lo, lo + nl, dg, o,
                            shard_pm(a, lo, 2, c->N), perm, true);
        out->scale = a->scale;
    }
    out->n_polys = 2;
    out->count = cnt;
    out->level = nl;
    return s;
}

// digit window [jw0, jw1) of a limb-sharded key switch: ModUp + inner product for the owned
// targets [t_lo, t_hi) and P, into (first) or added to (later windows) ext [cnt][2][l+1][N]
static ckks_status ks_window(ckks_ctx *c, PolyMap din, const u32 *perm, u32 cnt, u32 l, const u64 *key, u32 t_lo,
                             u32 t_hi, const u64 *D, u32 dw, u32 jw0, u32 jw1, u64 *ext, bool first)
{
    Launch L = c->lc();
    const size_t n = c->N;
    const u32 T = t_hi - t_lo + 1;
    u64 *I = need(c, "shwI", (size_t)cnt * T * l * n);
    if (!I) return fail(c, CKKS_E_OOM, "window scratch");
    auto run = [&](u32 t0, u32 tn) {
        launch_ks_modup_cols(L, D, dw, cnt, 0, l, cnt, t0, tn, I, c->L, jw0, jw1 - jw0);
        launch_ks_mac(L, I, din, perm, key, c->L, l, cnt, t0, tn, ext, c->L, false, jw0, jw1, !first);
    };
    if (t_hi == l) {
        run(t_lo, t_hi - t_lo + 1);  // P (target index l) contiguous with the owned targets
    } else {
        if (t_hi > t_lo) run(t_lo, t_hi - t_lo);
        run(l, 1);
    }
    return check_launch(c);
}

ckks_status ckks_shard_ks_window(ckks_ctx *c, int kind, int32_t step, const uint64_t *D_win, uint32_t r, uint32_t w,
                                 const ckks_buf *a, uint32_t lo, uint32_t l, int first)
{
    if (!c || !shard_ok(c, a, lo, l, 2) || !D_win || w < a->level || (kind != 0 && kind != 1))
        return CKKS_E_INVALID_ARG;
    if (c->alpha > 1 || c->K > 1) return fail(c, CKKS_E_UNSUPPORTED, "sharded key switch needs alpha = K = 1");
    const u32 nl = a->level, cnt = a->count;
    const size_t n = c->N;
    const u32 jw0 = r * w, jw1 = std::min(l, r * w + w);
    if (jw0 >= l) return CKKS_OK;  // rank r holds no digits at this level
    u64 *ext = need(c, ("shext_" + std::to_string(lo)).c_str(), (size_t)cnt * 2 * (l + 1) * n);
    if (!ext) return fail(c, CKKS_E_OOM, "shard accumulators");
    const u64 *D = D_win - (size_t)r * cnt * w * n;  // digit j at ((j / w) cnt + c) w + j % w
    if (kind == 0) {
        if (!c->rlk) return fail(c, CKKS_E_MISSING_KEY, "relinearisation key not set");
        u64 *d2 = need(c, ("shd2_" + std::to_string(lo)).c_str(), (size_t)cnt * nl * n);  // kept by ckks_shard_ks_digits
        return ks_window(c, PolyMap{d2 - (size_t)lo * n, nl}, nullptr, cnt, l, c->rlk, lo, lo + nl, D, w, jw0, jw1,
                         ext, first != 0);
    }
    const u64 kappa = galois_elt(c, step);
    auto it = c->gk.find(kappa);
    if (it == c->gk.end()) return fail(c, CKKS_E_MISSING_KEY, "missing Galois key");
    const u32 *perm = get_perm(c, kappa);
    if (!perm) return fail(c, CKKS_E_OOM, "perm");
    return ks_window(c, shard_pm(a, lo, 1, c->N), perm, cnt, l, it->second, lo, lo + nl, D, w, jw0, jw1, ext,
                     first != 0);
}

ckks_status ckks_shard_ks_combine(ckks_ctx *c, int kind, int32_t step, const ckks_buf *a, uint32_t lo, uint32_t l,
                                  ckks_buf *out)
{
    if (!c || !shard_ok(c, a, lo, l, 2) || !out || !out->data || out->capacity < a->level || (kind != 0 && kind != 1))
        return CKKS_E_INVALID_ARG;
    const u32 nl = a->level, cnt = a->count;
    const size_t n = c->N;
    u64 *ext = need(c, ("shext_" + std::to_string(lo)).c_str(), (size_t)cnt * 2 * (l + 1) * n);
    u64 *S = need(c, ("shS_" + std::to_string(lo)).c_str(), (size_t)cnt * 2 * nl * n);
    if (!ext || !S) return fail(c, CKKS_E_OOM, "shard scratch");
    PolyMap o = shard_pm(out, lo, 2, c->N);
    const u32 *perm = nullptr;
    PolyMap base = o;
    bool c0_only = false;
    if (kind == 1) {
        const u64 kappa = galois_elt(c, step);
        if (!c->gk.count(kappa)) return fail(c, CKKS_E_MISSING_KEY, "missing Galois key");
        perm = get_perm(c, kappa);
        base = shard_pm(a, lo, 2, c->N);
        c0_only = true;
        out->scale = a->scale;
    }
    // ModDown (A7): INTT of the P limb, then out_i = base + (acc_i - NTT_i([acc]_P)) P^{-1}
    const Launch L = c->lc();
    PolyMap pl{ext + (size_t)l * n, l + 1};
    launch_ntt_inv(L, pl, pl, 2 * cnt, LimbSet{1, 0, 0, c->L}, nullptr);
    launch_bcast_submul(L, ext + (size_t)l * n, l + 1, c->L, 2 * cnt, nl, lo, S, PolyMap{ext, l + 1}, o, c->d_pinv,
                        base, perm, c0_only);
    out->n_polys = 2;
    out->count = cnt;
    out->level = nl;
    return check_launch(c);
}

ckks_status ckks_shard_rescale_last(ckks_ctx *c, const ckks_buf *ct, uint32_t lo, uint32_t l, uint64_t *X)
{
    if (!c || !shard_ok(c, ct, lo, l, 2) || !X || lo + ct->level != l || l < 2) return CKKS_E_INVALID_ARG;
    launch_ntt_inv(c->lc(), PolyMap{ct->data + (size_t)(l - 1 - lo) * c->N, ct->capacity}, PolyMap{X, 1},
                   2 * ct->count, LimbSet{1, 1, l - 1, c->L}, nullptr);
    return check_launch(c);
}

ckks_status ckks_shard_rescale_apply(ckks_ctx *c, const uint64_t *X, const ckks_buf *ct, uint32_t lo, uint32_t l,
                                     ckks_buf *out)
{
    if (!c || !shard_ok(c, ct, lo, l, 2) || !X || l < 2 || !out || !out->data) return CKKS_E_INVALID_ARG;
    const u32 hi = std::min<u32>(lo + ct->level, l - 1), cnt = ct->count;
    const u32 nt = hi > lo ? hi - lo : 0;
    if (nt && out->capacity < nt) return CKKS_E_INVALID_ARG;
    u64 *S = need(c, "rs", (size_t)2 * cnt * std::max<u32>(nt, 1) * c->N);
    if (!S) return fail(c, CKKS_E_OOM, "rescale scratch");
    launch_bcast_submul(c->lc(), X, 1, l - 1, 2 * cnt, nt, lo, S, shard_pm(ct, lo, 2, c->N),
                        shard_pm(out, lo, 2, c->N), c->d_rinv + (size_t)l * (c->L + c->K), PolyMap{nullptr, 0}, nullptr,
                        false);
    out->n_polys = 2;
    out->count = cnt;
    out->level = nt;
    out->scale = ct->scale / (double)c->primes[l - 1];
    return check_launch(c);
}

// ---- PrivFT encrypted training step ------------------------------------------
namespace {
// out[p] = relin(a[(p / adiv) % amod] (x) b[(p / bdiv) % bmod])   (HMUL)
ckks_status mul_relin_paired(ckks_ctx *c, const ckks_buf *a, const ckks_buf *b, ckks_buf *out, u32 cnt, u32 l,
                             u32 adiv, u32 amod, u32 bdiv, u32 bmod)
{
    u64 *d2 = need(c, "d2", (size_t)cnt * l * c->N);
    if (!d2) return fail(c, CKKS_E_OOM, "tensor scratch");
    launch_tensor(c->lc(), pm(a), pm(b), pm(out), PolyMap{d2, l}, cnt, l, adiv, amod, bdiv, bmod);
    const double sc = a->scale * b->scale;
    ckks_status s = keyswitch(c, PolyMap{d2, l}, nullptr, cnt, l, c->rlk, pm(out), pm(out), nullptr, false);
    out->n_polys = 2;
    out->count = cnt;
    out->level = l;
    out->scale = sc;
    return s;
}

ckks_buf scratch_ct(ckks_ctx *c, const char *name, u32 count, u32 n_polys, u32 cap)
{
    ckks_buf b{need(c, name, (size_t)count * n_polys * cap * c->N), count, n_polys, cap, cap, 1.0};
    return b;
}

ckks_buf dropped(const ckks_buf *b, u32 level)
{
    ckks_buf v = *b;
    v.level = level;
    return v;
}

ckks_status mul_const_per_ct(ckks_ctx *c, ckks_buf *ct, const std::vector<double> &vals, u32 per, double cscale)
{
    // constant for ciphertext p is llround(vals[p % per] * cscale)
    std::vector<ulonglong2> h((size_t)ct->count * ct->level);
    for (u32 p = 0; p < ct->count; ++p) {
        bool ok;
        const long long v = llround_checked(vals[p % per] * cscale, ok);
        if (!ok) return fail(c, CKKS_E_ENCODE_OVERFLOW, "constant overflows int64");
        for (u32 i = 0; i < ct->level; ++i) {
            const u64 q = c->primes[i], r = residue_of(v, q);
            h[(size_t)p * ct->level + i] = make_ulonglong2(r, hm::shoup(r, q));
        }
    }
    ulonglong2 *d;
    ckks_status s = upload_consts(c, h, "tr_const", &d);
    if (s != CKKS_OK) return s;
    launch_mul_scalar_per_ct(c->lc(), pm(ct), pm(ct), ct->count, ct->level, d);
    ct->scale *= cscale;
    return check_launch(c);
}
}  // namespace

// scale bookkeeping of the forward pass (A13): level and scale of g, where the caller must
// encode -onehot(y) (so that it adds to g exactly) and the class mask
static double train_g_scale(const ckks_ctx *c, double sv, double sH, double sO, u32 l0)
{
    const double sa = sv * sH / (double)c->primes[l0 - 1];           // rescale(v H)
    const double sh = sa * c->scale / (double)c->primes[l0 - 2];     // rescale(a / w)
    const double ss = sh * sO / (double)c->primes[l0 - 3];           // rescale(sum h O)
    return ss * ss / (double)c->primes[l0 - 4] * 8.0;                // rescale(s^2 + 4s), * 8
}

ckks_status ckks_privft_train_plan(const ckks_ctx *c, const ckks_buf *H, const ckks_buf *O, const ckks_buf *bags,
                                   double *g_scale, uint32_t *g_level)
{
    if (!c || !H || !O || !bags || H->level < 10) return CKKS_E_INVALID_ARG;
    if (g_scale) *g_scale = train_g_scale(c, bags->scale, H->scale, O->scale, H->level);
    if (g_level) *g_level = H->level - 4;
    return CKKS_OK;
}

ckks_status ckks_privft_train_grad(ckks_ctx *c, const ckks_buf *H, const ckks_buf *O, const ckks_buf *bags,
                                   const uint32_t *w, const uint32_t *y, uint32_t cls, const ckks_buf *neg_onehot,
                                   const ckks_buf *mask, ckks_buf *GH, ckks_buf *GO)
{
    if (!c || !valid_buf(c, H, 2) || !valid_buf(c, O, 2) || !valid_buf(c, bags, 2) || !w || !y || !GH || !GO ||
        !GH->data || !GO->data || cls < 1 || cls > c->N / 2 || !valid_buf(c, neg_onehot, 1) || !valid_buf(c, mask, 1))
        return CKKS_E_INVALID_ARG;
    const u32 n = H->count, E = bags->count, l0 = H->level, N = c->N, t = N / 2;
    if (O->count != n || O->level != l0 || bags->level != l0 || l0 < 10)
        return fail(c, CKKS_E_LEVEL_EXHAUSTED, "training needs model and bags at one level >= 10 (9 per step)");
    if (GH->capacity < l0 - 8 || GO->capacity < l0 - 6 || GH->count != n || GO->count != n)
        return CKKS_E_INVALID_ARG;
    if (!c->rlk) return fail(c, CKKS_E_MISSING_KEY, "relinearisation key not set");
    for (u32 e = 0; e < E; ++e)
        if (!w[e] || y[e] >= cls) return CKKS_E_INVALID_ARG;
    if (neg_onehot->count != E || mask->count != 1 || neg_onehot->level != l0 - 4 || mask->level != l0 - 4 ||
        neg_onehot->scale != train_g_scale(c, bags->scale, H->scale, O->scale, l0))
        return fail(c, CKKS_E_SCALE_MISMATCH, "-onehot / mask must be encoded at level l0-4, scale of g "
                                              "(ckks_privft_train_plan)");
    const u32 P = E * n;  // work items p = j * E + e  (column-major: j outer)
    std::vector<double> winv(E);
    for (u32 e = 0; e < E; ++e) winv[e] = 1.0 / (double)w[e];
    ckks_status s;
    // 1-3: a = TotalSum(rescale(v_e (x) H_j)); h = rescale(a / w_e)
    ckks_buf A = scratch_ct(c, "tr_A", P, 2, l0);
    if (!A.data) return fail(c, CKKS_E_OOM, "training scratch");
    if ((s = mul_relin_paired(c, bags, H, &A, P, l0, 1, E, E, 0)) != CKKS_OK) return s;
    if ((s = rescale_impl(c, &A, &A)) != CKKS_OK) return s;
    if ((s = ckks_total_sum(c, &A, &A)) != CKKS_OK) return s;
    if ((s = mul_const_per_ct(c, &A, winv, E, c->scale)) != CKKS_OK) return s;
    if ((s = rescale_impl(c, &A, &A)) != CKKS_OK) return s;  // h: level l0-2
    // 4: s_e = rescale(relin(sum_j h_{j,e} (x) O_j))  -- lazy relinearisation (T3)
    ckks_buf Od = dropped(O, A.level);
    ckks_buf T = scratch_ct(c, "tr_T", P, 2, A.level);
    u64 *d2 = need(c, "tr_d2", (size_t)P * A.level * N);
    ckks_buf S = scratch_ct(c, "tr_S", E, 2, l0);
    u64 *d2s = need(c, "tr_d2s", (size_t)E * A.level * N);
    if (!T.data || !d2 || !S.data || !d2s) return fail(c, CKKS_E_OOM, "training scratch");
    const u32 lh = A.level;
    launch_tensor(c->lc(), pm(&A), pm(&Od), pm(&T), PolyMap{d2, lh}, P, lh, 1, 0, E, 0);
    launch_sum_strided(c->lc(), pm(&T), pm(&S), E, 2, lh, n, E, 1);
    launch_sum_strided(c->lc(), PolyMap{d2, lh}, PolyMap{d2s, lh}, E, 1, lh, n, E, 1);
    if ((s = keyswitch(c, PolyMap{d2s, lh}, nullptr, E, lh, c->rlk, pm(&S), pm(&S), nullptr, false)) != CKKS_OK)
        return s;
    S.level = lh;
    S.scale = A.scale * O->scale;
    if ((s = rescale_impl(c, &S, &S)) != CKKS_OK) return s;  // level l0-3
    // 5: g = rescale(s^2 + 4 s) + 2, scale *= 8
    ckks_buf G = scratch_ct(c, "tr_G", E, 2, l0), L4 = scratch_ct(c, "tr_L4", E, 2, l0);
    if (!G.data || !L4.data) return fail(c, CKKS_E_OOM, "training scratch");
    if ((s = ckks_mul_relin(c, &S, &S, &G)) != CKKS_OK) return s;
    if ((s = ckks_mul_const(c, &S, 4.0, S.scale, &L4)) != CKKS_OK) return s;
    if ((s = ckks_add(c, &G, &L4, &G)) != CKKS_OK) return s;
    if ((s = rescale_impl(c, &G, &G)) != CKKS_OK) return s;
    if ((s = ckks_add_const(c, &G, 2.0, &G)) != CKKS_OK) return s;
    G.scale *= 8.0;  // level l0-4
    // 6: e = rescale(HMULPLAIN(g - onehot(y), mask_{<c}))  (plaintexts encoded by the caller)
    (void)t;
    if ((s = ckks_add_plain(c, &G, neg_onehot, &G)) != CKKS_OK) return s;
    if ((s = ckks_mul_plain(c, &G, mask, &G)) != CKKS_OK) return s;
    if ((s = rescale_impl(c, &G, &G)) != CKKS_OK) return s;  // e: level l0-5
    const u32 le = G.level;
    // 7: gO_{j,e} = rescale(relin(h_{j,e} (x) e_e));  GO_j = sum_e gO_{j,e}
    ckks_buf Ad = dropped(&A, le);
    ckks_buf GOp = scratch_ct(c, "tr_GO", P, 2, le);
    if (!GOp.data) return fail(c, CKKS_E_OOM, "training scratch");
    if ((s = mul_relin_paired(c, &Ad, &G, &GOp, P, le, 1, 0, 1, E)) != CKKS_OK) return s;
    if ((s = rescale_impl(c, &GOp, &GOp)) != CKKS_OK) return s;  // level l0-6
    launch_sum_strided(c->lc(), pm(&GOp), pm(GO), n, 2, GOp.level, E, 1, E);
    GO->n_polys = 2;
    GO->level = GOp.level;
    GO->scale = GOp.scale;
    // 8: gh_{j,e} = TotalSum(rescale(relin(O_j (x) e_e)))
    ckks_buf Oe = dropped(O, le);
    ckks_buf U = scratch_ct(c, "tr_U", P, 2, le);
    if (!U.data) return fail(c, CKKS_E_OOM, "training scratch");
    if ((s = mul_relin_paired(c, &Oe, &G, &U, P, le, E, 0, 1, E)) != CKKS_OK) return s;
    if ((s = rescale_impl(c, &U, &U)) != CKKS_OK) return s;
    if ((s = ckks_total_sum(c, &U, &U)) != CKKS_OK) return s;  // level l0-6
    // 9: gH_{j,e} = rescale(rescale(relin(v_e (x) gh_{j,e})) / w_e);  GH_j = sum_e gH_{j,e}
    ckks_buf Vd = dropped(bags, U.level);
    ckks_buf GHp = scratch_ct(c, "tr_GH", P, 2, U.level);
    if (!GHp.data) return fail(c, CKKS_E_OOM, "training scratch");
    if ((s = mul_relin_paired(c, &Vd, &U, &GHp, P, U.level, 1, E, 1, 0)) != CKKS_OK) return s;
    if ((s = rescale_impl(c, &GHp, &GHp)) != CKKS_OK) return s;
    if ((s = mul_const_per_ct(c, &GHp, winv, E, c->scale)) != CKKS_OK) return s;
    if ((s = rescale_impl(c, &GHp, &GHp)) != CKKS_OK) return s;  // level l0-8
    launch_sum_strided(c->lc(), pm(&GHp), pm(GH), n, 2, GHp.level, E, 1, E);
    GH->n_polys = 2;
    GH->level = GHp.level;
    GH->scale = GHp.scale;
    return check_launch(c);
}

ckks_status ckks_privft_train_update(ckks_ctx *c, const ckks_buf *H, const ckks_buf *O, const ckks_buf *GH,
                                     const ckks_buf *GO, double eta, ckks_buf *H_out, ckks_buf *O_out)
{
    if (!c || !valid_buf(c, H, 2) || !valid_buf(c, O, 2) || !valid_buf(c, GH, 2) || !valid_buf(c, GO, 2) || !H_out ||
        !O_out || !H_out->data || !O_out->data)
        return CKKS_E_INVALID_ARG;
    const u32 n = H->count, l0 = H->level, lf = l0 - 9;
    if (l0 < 10 || O->level != l0 || GH->level != l0 - 8 || GO->level != l0 - 6 || GH->count != n ||
        GO->count != n || O->count != n || H_out->capacity < lf || O_out->capacity < lf)
        return CKKS_E_INVALID_ARG;
    ckks_status s;
    // d = rescale(G * (-eta)) with the constant's scale chosen to land on the model's scale (T5)
    auto step = [&](const ckks_buf *M, const ckks_buf *Gr, ckks_buf *out, const char *nm) -> ckks_status {
        ckks_buf D = scratch_ct(c, nm, n, 2, Gr->level);
        if (!D.data) return fail(c, CKKS_E_OOM, "training scratch");
        const double cs = M->scale * (double)c->primes[Gr->level - 1] / Gr->scale;
        ckks_status r = ckks_mul_const(c, Gr, -eta, cs, &D);
        if (r != CKKS_OK) return r;
        if ((r = rescale_impl(c, &D, &D)) != CKKS_OK) return r;
        D.scale = M->scale;
        // limb-wise: adding then dropping to lf == dropping both operands to lf first
        ckks_buf Md = dropped(M, lf), Dd = dropped(&D, lf);
        return ckks_add(c, &Md, &Dd, out);
    };
    if ((s = step(H, GH, H_out, "tr_DH")) != CKKS_OK) return s;
    if ((s = step(O, GO, O_out, "tr_DO")) != CKKS_OK) return s;
    O_out->level = lf;  // model left at a common level l0 - 9 (nine levels per minibatch)
    H_out->level = lf;
    return check_launch(c);
}

// ---- PrivFT ----------------------------------------------------------------------------------
namespace {
// Re-lay H once into the tensor-core operand layout of the v.H chunk-dot (a snapshot of H at
// model creation).  Skipped (CUDA-core chunk-dot) when CKKS_CHUNKDOT_TC=0, K > 4096, or no memory.
void model_tc_layout(ckks_ctx *c, ckks_privft_model *md)
{
    const char *env = std::getenv("CKKS_CHUNKDOT_TC");
    if ((env && env[0] == '0') || !chunkdot_tc_supported(c->primes.data(), c->L, 1, md->K)) return;
    const size_t words = chunkdot_tc_words(c->primes.data(), c->L, md->n, md->K, c->log_n);
    if (cudaMalloc((void **)&md->Hf, words * sizeof(u32)) != cudaSuccess) {
        cudaGetLastError();
        md->Hf = nullptr;
        return;
    }
    launch_chunkdot_prep_h(c->lc(), md->H.data, md->H.capacity, md->Hf, c->L, md->n, md->K);
}
}  // namespace

ckks_status ckks_privft_model_wrap(ckks_ctx *c, const ckks_buf *H, const ckks_buf *O, uint32_t m, uint32_t n,
                                   uint32_t cls, ckks_privft_model **out)
{
    if (!c || !out || !valid_buf(c, H, 1) || !valid_buf(c, O, 1) || n < 1 || cls < 1 || cls > c->N / 2 || m < 1)
        return CKKS_E_INVALID_ARG;
    const u32 t = c->N / 2, K = (m + t - 1) / t;
    if (H->count != n * K || O->count != n || H->level != c->L || c->L < 4 || O->level != c->L - 2)
        return fail(c, CKKS_E_INVALID_ARG, "model packing shape/level");
    ckks_privft_model *md = new ckks_privft_model();
    md->ctx = c;
    md->H = *H;
    md->O = *O;
    md->m = m;
    md->n = n;
    md->c = cls;
    md->K = K;
    model_tc_layout(c, md);
    *out = md;
    return CKKS_OK;
}

ckks_status ckks_privft_model_create(ckks_ctx *c, const double *Hh, const double *Oh, uint32_t m, uint32_t n,
                                     uint32_t cls, ckks_privft_model **out)
{
    if (!c || !Hh || !Oh || !out || n < 1 || m < 1 || cls < 1 || cls > c->N / 2 || c->L < 4)
        return CKKS_E_INVALID_ARG;
    const u32 t = c->N / 2, K = (m + t - 1) / t, L = c->L;
    const size_t n_ = c->N;
    u64 *hp = nullptr, *op = nullptr;
    CUDA_TRY(c, cudaMalloc(&hp, (size_t)n * K * L * n_ * sizeof(u64)));
    if (cudaMalloc(&op, (size_t)n * (L - 2) * n_ * sizeof(u64)) != cudaSuccess) {
        cudaFree(hp);
        return fail(c, CKKS_E_OOM, "model");
    }
    std::vector<double> col(t);
    for (u32 j = 0; j < n; ++j)
        for (u32 k = 0; k < K; ++k) {  // P^H_{j,k}: slot i = H[k t + i][j]  (A17)
            for (u32 i = 0; i < t; ++i) {
                const size_t r = (size_t)k * t + i;
                col[i] = r < m ? Hh[r * n + j] : 0.0;
            }
            ckks_buf pt{hp + ((size_t)j * K + k) * L * n_, 1, 1, L, L, 0};
            ckks_status s = ckks_encode(c, col.data(), nullptr, t, c->scale, L, &pt);
            if (s != CKKS_OK) return s;
        }
    for (u32 j = 0; j < n; ++j) {  // P^O_j: slot i = O[j][i], i < c  (A16)
        std::vector<double> row(Oh + (size_t)j * cls, Oh + (size_t)(j + 1) * cls);
        ckks_buf pt{op + (size_t)j * (L - 2) * n_, 1, 1, L - 2, L - 2, 0};
        ckks_status s = ckks_encode(c, row.data(), nullptr, cls, c->scale, L - 2, &pt);
        if (s != CKKS_OK) return s;
    }
    ckks_privft_model *md = new ckks_privft_model();
    md->ctx = c;
    md->H = ckks_buf{hp, n * K, 1, L, L, c->scale};
    md->O = ckks_buf{op, n, 1, L - 2, L - 2, c->scale};
    md->owned = true;
    md->m = m;
    md->n = n;
    md->c = cls;
    md->K = K;
    model_tc_layout(c, md);
    *out = md;
    return CKKS_OK;
}

ckks_status ckks_privft_model_destroy(ckks_privft_model *md)
{
    if (!md) return CKKS_E_INVALID_ARG;
    if (md->owned) {
        cudaFree(md->H.data);
        cudaFree(md->O.data);
    }
    if (md->Hf) cudaFree(md->Hf);
    delete md;
    return CKKS_OK;
}

namespace {
void chunkdot_vh(ckks_ctx *c, const ckks_privft_model *md, const ckks_buf *bag, u32 batch, u64 *out, u32 out_cap)
{
    const u32 L = c->L;
    // tensor-core path: queries in sub-batches small enough for its shared-memory tile (a batch of
    // 256 queries at C4 needs 590 KB of A planes at once; 64 fit)
    const char *se = std::getenv("CKKS_CHUNKDOT_SB");  // cap on the sub-batch (tests: ragged sub-batches)
    u32 sb = se ? std::max<u32>(1, std::min<u32>(batch, (u32)std::atoi(se))) : batch;
    while (md->Hf && sb > 1 && !chunkdot_tc_supported(c->primes.data(), L, sb, md->K)) sb = (sb + 1) / 2;
    if (md->Hf && chunkdot_tc_supported(c->primes.data(), L, sb, md->K)) {
        const size_t n = c->N;
        for (u32 b0 = 0; b0 < batch; b0 += sb) {
            const u32 nb = std::min(sb, batch - b0);
            launch_chunkdot_tc(c->lc(), bag->data + (size_t)b0 * md->K * 2 * bag->capacity * n, bag->capacity, md->Hf,
                               out + (size_t)b0 * md->n * 2 * out_cap * n, out_cap, nb, md->n, md->K, L);
        }
    } else
        launch_chunkdot(c->lc(), bag->data, bag->capacity, md->H.data, md->H.capacity, out, out_cap, batch, md->n,
                        md->K, L);
}
}  // namespace

ckks_status ckks_privft_chunkdot(ckks_ctx *c, const ckks_privft_model *md, const ckks_buf *bag, uint32_t batch,
                                 ckks_buf *out)
{
    if (!c || !md || md->ctx != c || !valid_buf(c, bag, 2) || batch < 1 || !out || !out->data || out->n_polys != 2 ||
        out->count != batch * md->n || out->capacity < c->L)
        return CKKS_E_INVALID_ARG;
    if (bag->count != batch * md->K || bag->level != c->L) return fail(c, CKKS_E_INVALID_ARG, "bag shape/level");
    chunkdot_vh(c, md, bag, batch, out->data, out->capacity);
    out->level = c->L;
    out->scale = bag->scale * md->H.scale;
    return check_launch(c);
}

namespace {
ckks_status privft_infer_impl(ckks_ctx *c, const ckks_privft_model *md, const ckks_buf *bag, const uint32_t *w,
                              uint32_t batch, uint32_t flags, ckks_buf *scores, cudaEvent_t bag_consumed);
}

ckks_status ckks_privft_infer(ckks_ctx *c, const ckks_privft_model *md, const ckks_buf *bag, const uint32_t *w,
                              uint32_t batch, uint32_t flags, ckks_buf *scores)
{
    return privft_infer_impl(c, md, bag, w, batch, flags, scores, nullptr);
}

// Host-buffer inference: the bag upload runs on the context's upload stream into one of two
// staging buffers (alternating per call) and the main stream waits only for it, so a
// sequence of calls overlaps call k+1's upload with call k's compute (the upload waits for
// the chunk-dot that last read its staging buffer, the only reader of the bag).
ckks_status ckks_privft_infer_host(ckks_ctx *c, const ckks_privft_model *md, const uint64_t *bag_host,
                                   double bag_scale, const uint32_t *w, uint32_t batch, uint32_t flags,
                                   uint64_t *scores_host, double *scores_scale, uint32_t *scores_level)
{
    if (!c || !md || md->ctx != c || !bag_host || !w || batch < 1 || !scores_host) return CKKS_E_INVALID_ARG;
    const u32 L = c->L;
    const bool poly = flags & CKKS_PRIVFT_POLY_SOFTMAX;
    if (poly && L < 5) return fail(c, CKKS_E_LEVEL_EXHAUSTED, "level budget");
    if (!c->up) {
        if (cudaStreamCreateWithFlags(&c->up, cudaStreamNonBlocking) != cudaSuccess) return fail(c, CKKS_E_CUDA, "stream");
        for (int i = 0; i < 2; ++i)
            for (int h = 0; h < 2; ++h)
                if (cudaEventCreateWithFlags(&c->up_done[i][h], cudaEventDisableTiming) != cudaSuccess ||
                    cudaEventCreateWithFlags(&c->stage_free[i][h], cudaEventDisableTiming) != cudaSuccess)
                    return fail(c, CKKS_E_CUDA, "events");
    }
    for (u32 b = 0; b < batch; ++b)
        if (w[b] == 0) return CKKS_E_INVALID_ARG;
    const u32 i = c->stage_next;
    c->stage_next ^= 1;
    const size_t per_q = (size_t)md->K * 2 * L * c->N;  // one query's bag, words
    const size_t words = (size_t)batch * per_q;
    u64 *stage = need(c, i ? "pf_stage1" : "pf_stage0", words);
    const u32 lo = poly ? L - 4 : L - 3;
    const size_t sc_q = (size_t)2 * (L - 3) * c->N;
    u64 *sc = need(c, "pf_scores", (size_t)batch * sc_q);
    if (!stage || !sc) return fail(c, CKKS_E_OOM, "host-inference staging");
    // both halves' previous readers of this staging buffer (two calls ago) are done
    CUDA_TRY(c, cudaStreamWaitEvent(c->up, c->stage_free[i][0], 0));
    CUDA_TRY(c, cudaStreamWaitEvent(c->up, c->stage_free[i][1], 0));
    // the batch runs in two halves: the second half uploads while the first computes, so even
    // a lone call exposes only half of its upload
    const u32 nh = batch >= 2 ? 2 : 1;
    ckks_buf out{sc, batch, 2, lo, L - 3, 1.0};
    for (u32 h = 0; h < nh; ++h) {
        const u32 b0 = h * batch / nh, b1 = (h + 1) * batch / nh, nb = b1 - b0;
        CUDA_TRY(c, cudaMemcpyAsync(stage + b0 * per_q, bag_host + b0 * per_q, nb * per_q * 8,
                                    cudaMemcpyHostToDevice, c->up));
        CUDA_TRY(c, cudaEventRecord(c->up_done[i][h], c->up));
    }
    for (u32 h = 0; h < nh; ++h) {
        const u32 b0 = h * batch / nh, b1 = (h + 1) * batch / nh, nb = b1 - b0;
        CUDA_TRY(c, cudaStreamWaitEvent(c->st, c->up_done[i][h], 0));
        ckks_buf bag{stage + b0 * per_q, nb * md->K, 2, L, L, bag_scale};
        ckks_buf oh{sc + b0 * sc_q, nb, 2, lo, L - 3, 1.0};
        ckks_status s = privft_infer_impl(c, md, &bag, w + b0, nb, flags, &oh, c->stage_free[i][h]);
        if (s != CKKS_OK) return s;
        out.level = oh.level;
        out.scale = oh.scale;
    }
    if (nh == 1) CUDA_TRY(c, cudaEventRecord(c->stage_free[i][1], c->st));
    // result limbs [b][2][lo][N] (dense) to the host, on the main stream
    CUDA_TRY(c, cudaMemcpy2DAsync(scores_host, (size_t)lo * c->N * 8, sc, (size_t)(L - 3) * c->N * 8,
                                  (size_t)lo * c->N * 8, (size_t)batch * 2, cudaMemcpyDeviceToHost, c->st));
    if (scores_scale) *scores_scale = out.scale;
    if (scores_level) *scores_level = out.level;
    return check_launch(c);
}

ckks_status ckks_sync(ckks_ctx *c)
{
    if (!c) return CKKS_E_INVALID_ARG;
    if (cudaStreamSynchronize(c->st) != cudaSuccess) return fail(c, CKKS_E_CUDA, cudaGetErrorString(cudaGetLastError()));
    return CKKS_OK;
}

namespace {
ckks_status privft_infer_impl(ckks_ctx *c, const ckks_privft_model *md, const ckks_buf *bag, const uint32_t *w,
                              uint32_t batch, uint32_t flags, ckks_buf *scores, cudaEvent_t bag_consumed)
{
    if (!c || !md || md->ctx != c || !valid_buf(c, bag, 2) || !w || batch < 1 || !scores || !scores->data)
        return CKKS_E_INVALID_ARG;
    const u32 L = c->L, K = md->K, n = md->n;
    const bool poly = flags & CKKS_PRIVFT_POLY_SOFTMAX;
    if (bag->count != batch * K || bag->level != L) return fail(c, CKKS_E_INVALID_ARG, "bag shape/level");
    if (scores->capacity < L - 3 || (poly && L < 5)) return fail(c, CKKS_E_LEVEL_EXHAUSTED, "level budget");
    for (u32 b = 0; b < batch; ++b)
        if (w[b] == 0) return CKKS_E_INVALID_ARG;
    const size_t nn = c->N;
    const Launch Lc = c->lc();
    NvtxRange r_all("privft_infer");
    // a_j = sum_k HMULPLAIN(ct_k, P^H_{j,k})
    ckks_buf A{need(c, "pf_a", (size_t)batch * n * 2 * L * nn), batch * n, 2, L, L, bag->scale * md->H.scale};
    if (!A.data) return fail(c, CKKS_E_OOM, "privft scratch");
    {
        NvtxRange r("privft.chunkdot_vH");
        chunkdot_vh(c, md, bag, batch, A.data, L);
    }
    if (bag_consumed) CUDA_TRY(c, cudaEventRecord(bag_consumed, c->st));
    ckks_status s;
    {
        NvtxRange r("privft.rescale_a");
        s = rescale_impl(c, &A, &A);  // (A14) rescale before TotalSum
    }
    if (s != CKKS_OK) return s;
    {
        NvtxRange r("privft.total_sum");
        s = ckks_total_sum(c, &A, &A);  // Alg "TotalSum"
    }
    if (s != CKKS_OK) return s;
    NvtxRange r_tail("privft.scale_output_softmax");
    // h_j = rescale(a_j * llround(Delta / w))   (A15)
    std::vector<ulonglong2> hc((size_t)batch * n * A.level);
    for (u32 b = 0; b < batch; ++b) {
        bool ok;
        const long long v = llround_checked(c->scale / (double)w[b], ok);
        for (u32 j = 0; j < n; ++j)
            for (u32 i = 0; i < A.level; ++i) {
                const u64 q = c->primes[i], r = residue_of(v, q);
                hc[((size_t)b * n + j) * A.level + i] = make_ulonglong2(r, hm::shoup(r, q));
            }
    }
    ulonglong2 *dc;
    s = upload_consts(c, hc, "pf_const", &dc);
    if (s != CKKS_OK) return s;
    launch_mul_scalar_per_ct(Lc, pm(&A), pm(&A), A.count, A.level, dc);
    A.scale *= c->scale;
    s = rescale_impl(c, &A, &A);
    if (s != CKKS_OK) return s;
    // s = sum_j HMULPLAIN(h_j, P^O_j)
    if (md->O.level != A.level) return fail(c, CKKS_E_LEVEL_MISMATCH, "O level");
    ckks_buf S{need(c, "pf_s", (size_t)batch * 2 * A.level * nn), batch, 2, A.level, A.level, A.scale * md->O.scale};
    if (!S.data) return fail(c, CKKS_E_OOM, "privft scratch");
    launch_chunkdot(Lc, A.data, A.capacity, md->O.data, md->O.capacity, S.data, S.capacity, batch, 1, n, A.level);
    s = rescale_impl(c, &S, scores);
    if (s != CKKS_OK || !poly) return s;
    // poly softmax: g = rescale(s*s + 4 s) + 2, scale *= 8   (A19)
    ckks_buf sq = tmp_ct(c, "pf_sq", scores), lin = tmp_ct(c, "pf_lin", scores);
    if (!sq.data || !lin.data) return fail(c, CKKS_E_OOM, "privft scratch");
    if ((s = ckks_mul_relin(c, scores, scores, &sq)) != CKKS_OK) return s;
    if ((s = ckks_mul_const(c, scores, 4.0, scores->scale, &lin)) != CKKS_OK) return s;
    if ((s = ckks_add(c, &sq, &lin, &sq)) != CKKS_OK) return s;
    if ((s = rescale_impl(c, &sq, scores)) != CKKS_OK) return s;
    if ((s = ckks_add_const(c, scores, 2.0, scores)) != CKKS_OK) return s;
    scores->scale *= 8.0;
    return CKKS_OK;
}
}  // namespace

}  // extern "C"
