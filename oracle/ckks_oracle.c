/*
 * oracle/ckks_oracle.c -- PLAIN, SLOW, OBVIOUSLY-CORRECT CPU RNS-CKKS ARITHMETIC.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  The product path
 * (paper_1908_06972_b200/) never links, imports or executes anything under oracle/,
 * and this file shares no code, header, table or constant generator with it.
 *
 * Conventions
 *   - residues are uint64_t in canonical range [0, q);
 *   - every product is formed in unsigned __int128 and reduced with '%';
 *   - no lazy reduction, no Montgomery/Barrett/Shoup, no blocking or fusion;
 *   - polynomials are held in COEFFICIENT form, layout [limb][N] (limb-major);
 *   - the only transform is the textbook negacyclic NTT used inside poly_mul.
 *
 * Citations: "P:NNN" = /root/reference/PAPER.md line NNN (section / equation /
 * algorithm named beside it).  Readings of ambiguous passages are listed in
 * DESIGN.md section "Readings" (they follow SURVEY.md Appendix A, ids A1..A32).
 *
 * Pins (tests/test_oracle_*.py, run with -m "not gpu") tie every function here to
 * something other than itself: Python big-integer brute force, schoolbook
 * negacyclic convolution, direct O(N^2) evaluation of the NTT definition, the
 * worked examples of SPEC/PAPER under tests/golden/, and exact algebraic
 * identities (decrypt of the 3-part product, pre-ModDown key-switch identity).
 */
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef uint64_t u64;
typedef unsigned __int128 u128;

/* ---------------------------------------------------------------- scalars -- */

static u64 mulmod(u64 a, u64 b, u64 q) { return (u64)(((u128)a * b) % q); }
static u64 addmod(u64 a, u64 b, u64 q) { return (u64)(((u128)a + b) % q); }
/* a - b mod q for a, b already in [0, q) */
static u64 submod(u64 a, u64 b, u64 q) { return (u64)(((u128)a + q - b) % q); }

u64 or_powmod(u64 b, u64 e, u64 q)
{
    u64 r = 1 % q;
    b %= q;
    while (e) {
        if (e & 1) r = mulmod(r, b, q);
        b = mulmod(b, b, q);
        e >>= 1;
    }
    return r;
}

/* q prime: a^(q-2) (Fermat) */
u64 or_invmod(u64 a, u64 q) { return or_powmod(a % q, q - 2, q); }

/* Deterministic Miller-Rabin, bases 2..37 (exact below 3.3e24 > 2^64).
 * Prime chain of word-sized primes: P:136 (Sec. 3.4 "p_i's are small prime integers"). */
int or_is_prime(u64 n)
{
    static const u64 bases[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return 0;
    for (int i = 0; i < 12; ++i) {
        if (n == bases[i]) return 1;
        if (n % bases[i] == 0) return 0;
    }
    u64 d = n - 1;
    int s = 0;
    while ((d & 1) == 0) { d >>= 1; ++s; }
    for (int i = 0; i < 12; ++i) {
        u64 x = or_powmod(bases[i], d, n);
        if (x == 1 || x == n - 1) continue;
        int witness = 1;
        for (int r = 1; r < s; ++r) {
            x = mulmod(x, x, n);
            if (x == n - 1) { witness = 0; break; }
        }
        if (witness) return 0;
    }
    return 1;
}

/* Descending scan over q < 2^bits with q = 1 mod 2N (NTT-friendly), skipping the
 * first `skip` hits and returning the next `count`.  Returns the number found.
 * Reading A5 / SURVEY O1: chain = deterministic descending scan, P drawn first. */
int or_prime_scan(uint32_t log_n, uint32_t bits, uint32_t skip, uint32_t count, u64 *out)
{
    u64 two_n = (u64)2 << log_n;
    u64 top = (bits >= 64) ? ~(u64)0 : (((u64)1 << bits) - 1); /* largest value < 2^bits */
    if (top < 1) return 0;
    u64 x = ((top - 1) / two_n) * two_n + 1;                     /* largest x <= top, x = 1 mod 2N */
    uint32_t found = 0, seen = 0;
    while (found < count) {
        if (or_is_prime(x)) {
            if (seen >= skip) out[found++] = x;
            ++seen;
        }
        if (x <= two_n) break;
        x -= two_n;
    }
    return (int)found;
}

/* psi = the minimal primitive 2N-th root of unity mod q (reading A27).
 * A primitive 2N-th root is any g with g^N = -1 (N a power of two); all of them
 * are the odd powers of one such g.  We return the smallest one. */
u64 or_min_psi(u64 q, uint32_t log_n)
{
    u64 n = (u64)1 << log_n, two_n = 2 * n;
    if ((q - 1) % two_n) return 0;
    u64 g = 0;
    for (u64 x = 2; x < q; ++x) {
        u64 c = or_powmod(x, (q - 1) / two_n, q);
        if (or_powmod(c, n, q) == q - 1) { g = c; break; }
    }
    if (!g) return 0;
    u64 g2 = mulmod(g, g, q), cur = g, best = g;
    for (u64 k = 1; k < n; ++k) { /* odd powers g^(2k+1) */
        cur = mulmod(cur, g2, q);
        if (cur < best) best = cur;
    }
    return best;
}

/* ---------------------------------------------------------------- NTT ----- */
/* Negacyclic NTT (textbook): A_k = sum_j a_j psi^{(2k+1) j} mod q, natural order.
 * Computed as twist a_j <- a_j psi^j followed by the cyclic radix-2 DIT FFT over
 * Z_q with omega = psi^2 (bit-reversal then butterflies).  Pinned against the
 * direct O(N^2) sum in tests/test_oracle_ring.py.  Stand-in for the paper's DGT
 * (Sec. 5.1), see SPEC design decision S:99. */
static void bitrev_permute(u64 *a, u64 n)
{
    for (u64 i = 1, j = 0; i < n; ++i) {
        u64 bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) { u64 t = a[i]; a[i] = a[j]; a[j] = t; }
    }
}

static void cyclic_fft(u64 *a, u64 n, u64 omega, u64 q)
{
    bitrev_permute(a, n);
    for (u64 len = 2; len <= n; len <<= 1) {
        u64 wlen = or_powmod(omega, n / len, q);
        for (u64 i = 0; i < n; i += len) {
            u64 w = 1;
            for (u64 j = 0; j < len / 2; ++j) {
                u64 u = a[i + j];
                u64 v = mulmod(a[i + j + len / 2], w, q);
                a[i + j] = addmod(u, v, q);
                a[i + j + len / 2] = submod(u, v, q);
                w = mulmod(w, wlen, q);
            }
        }
    }
}

void or_ntt_fwd(u64 *a, uint32_t log_n, u64 q, u64 psi)
{
    u64 n = (u64)1 << log_n, p = 1;
    for (u64 j = 0; j < n; ++j) { a[j] = mulmod(a[j], p, q); p = mulmod(p, psi, q); }
    cyclic_fft(a, n, mulmod(psi, psi, q), q);
}

void or_ntt_inv(u64 *a, uint32_t log_n, u64 q, u64 psi)
{
    u64 n = (u64)1 << log_n;
    u64 psi_inv = or_invmod(psi, q);
    cyclic_fft(a, n, mulmod(psi_inv, psi_inv, q), q);
    u64 n_inv = or_invmod(n % q, q), p = 1;
    for (u64 j = 0; j < n; ++j) {
        a[j] = mulmod(mulmod(a[j], n_inv, q), p, q);
        p = mulmod(p, psi_inv, q);
    }
}

/* -------------------------------------------------------- ring R_q ops ---- */
/* All ops below act on `nl` limbs of length N = 2^log_n, limb i modulo mods[i]. */

/* out = a * b in Z_q[X]/(X^N+1), per limb (negacyclic convolution). */
void or_poly_mul(const u64 *a, const u64 *b, u64 *out, const u64 *mods, uint32_t nl, uint32_t log_n)
{
    u64 n = (u64)1 << log_n;
    #pragma omp parallel for schedule(dynamic, 1)
    for (uint32_t i = 0; i < nl; ++i) {
        u64 q = mods[i], psi = or_min_psi(q, log_n);
        u64 *x = (u64 *)malloc(n * sizeof(u64)), *y = (u64 *)malloc(n * sizeof(u64));
        memcpy(x, a + i * n, n * sizeof(u64));
        memcpy(y, b + i * n, n * sizeof(u64));
        or_ntt_fwd(x, log_n, q, psi);
        or_ntt_fwd(y, log_n, q, psi);
        for (u64 k = 0; k < n; ++k) x[k] = mulmod(x[k], y[k], q);
        or_ntt_inv(x, log_n, q, psi);
        memcpy(out + i * n, x, n * sizeof(u64));
        free(x); free(y);
    }
}

/* HADD: out = a + b; HADDPLAIN is the same on c0 only. */
void or_poly_add(const u64 *a, const u64 *b, u64 *out, const u64 *mods, uint32_t nl, uint32_t log_n)
{
    u64 n = (u64)1 << log_n;
    for (uint32_t i = 0; i < nl; ++i)
        for (u64 k = 0; k < n; ++k) out[i * n + k] = addmod(a[i * n + k], b[i * n + k], mods[i]);
}

void or_poly_sub(const u64 *a, const u64 *b, u64 *out, const u64 *mods, uint32_t nl, uint32_t log_n)
{
    u64 n = (u64)1 << log_n;
    for (uint32_t i = 0; i < nl; ++i)
        for (u64 k = 0; k < n; ++k) out[i * n + k] = submod(a[i * n + k], b[i * n + k], mods[i]);
}

void or_poly_neg(const u64 *a, u64 *out, const u64 *mods, uint32_t nl, uint32_t log_n)
{
    u64 n = (u64)1 << log_n;
    for (uint32_t i = 0; i < nl; ++i)
        for (u64 k = 0; k < n; ++k) out[i * n + k] = submod(0, a[i * n + k], mods[i]);
}

/* out = c_i * a, c_i a scalar per limb (the constant polynomial). */
void or_poly_scalar_mul(const u64 *a, const u64 *c, u64 *out, const u64 *mods, uint32_t nl, uint32_t log_n)
{
    u64 n = (u64)1 << log_n;
    for (uint32_t i = 0; i < nl; ++i)
        for (u64 k = 0; k < n; ++k) out[i * n + k] = mulmod(a[i * n + k], c[i], mods[i]);
}

/* Reduce a signed small integer polynomial e (|e_k| < 2^62) into every limb. */
void or_poly_from_signed(const int64_t *e, u64 *out, const u64 *mods, uint32_t nl, uint32_t log_n)
{
    u64 n = (u64)1 << log_n;
    for (uint32_t i = 0; i < nl; ++i)
        for (u64 k = 0; k < n; ++k) {
            int64_t v = e[k];
            u64 q = mods[i];
            out[i * n + k] = v >= 0 ? ((u64)v) % q : submod(0, ((u64)(-v)) % q, q);
        }
}

/* Galois automorphism phi_kappa: a(X) -> a(X^kappa) in Z_q[X]/(X^N+1), kappa odd
 * ("X -> X^kappa"): X^j maps to X^{j kappa mod 2N}, with a sign
 * flip when j kappa mod 2N >= N because X^N = -1. */
void or_automorphism(const u64 *a, u64 *out, const u64 *mods, uint32_t nl, uint32_t log_n, u64 kappa)
{
    u64 n = (u64)1 << log_n, two_n = 2 * n;
    for (uint32_t i = 0; i < nl; ++i) {
        u64 q = mods[i];
        for (u64 j = 0; j < n; ++j) {
            u64 e = (u64)(((u128)j * kappa) % two_n);
            u64 v = a[i * n + j];
            if (e < n) out[i * n + e] = v;
            else out[i * n + (e - n)] = submod(0, v, q);
        }
    }
}

/* RESCALE, Eq. (1) and Alg "RNS RESCALE by a single RNS modulus":
 * c'_k = (c_k - [c]_{q_{l-1}}) * q_{l-1}^{-1} mod q_k for k < l-1 (floor; reading A4).
 * c: [l][N] one polynomial, out: [l-1][N]. */
void or_rescale_poly(const u64 *c, u64 *out, const u64 *mods, uint32_t l, uint32_t log_n)
{
    u64 n = (u64)1 << log_n;
    u64 ql = mods[l - 1];
    for (uint32_t k = 0; k + 1 < l; ++k) {
        u64 q = mods[k];
        u64 inv = or_invmod(ql % q, q);
        for (u64 j = 0; j < n; ++j) {
            u64 last = c[(u64)(l - 1) * n + j] % q; /* [c]_{q_{l-1}} in [0, q_{l-1}), then mod q_k */
            out[k * n + j] = mulmod(submod(c[k * n + j], last, q), inv, q);
        }
    }
}

/* Key switch KS(d; ksk) with per-limb digits (alpha = 1) and one special prime P
 * (readings A6-A9; P:149 relinearization, P:163 footnote, "one rotation key
 * contains l ciphertexts").
 *   d     : [l][N]   coefficient form, limb i mod q_i, at level l
 *   key   : [Lk][2][Lk+1][N]  digit j, (b|a), limb i in {q_0..q_{Lk-1}, P}, coefficient form
 *   mods  : Lk+1 moduli q_0..q_{Lk-1}, P
 *   out0/1: [l][N]
 * Steps:
 *   ModUp   d~_j = d_j (unsigned representative in [0,q_j), A8) taken mod every target
 *   inner   acc_m = sum_j d~_j * ksk_{j,m}   for m in {q_0..q_{l-1}, P}
 *   ModDown out_i = (acc_i - [acc]_P) * P^{-1} mod q_i  (floor by P, A7)
 */
void or_keyswitch(const u64 *d, uint32_t l, const u64 *key, uint32_t key_levels,
                  const u64 *mods, uint32_t log_n, u64 *out0, u64 *out1)
{
    u64 n = (u64)1 << log_n;
    uint32_t lk1 = key_levels + 1;
    u64 *acc = (u64 *)calloc((size_t)2 * (l + 1) * n, sizeof(u64)); /* [2][l+1][N] */
    #pragma omp parallel for schedule(dynamic, 1)
    for (uint32_t m = 0; m <= l; ++m) {                 /* target limb, m == l is P */
        uint32_t key_limb = (m == l) ? key_levels : m;
        u64 qm = mods[key_limb];
        u64 *dt = (u64 *)malloc(n * sizeof(u64));
        u64 *prod = (u64 *)malloc(n * sizeof(u64));
        for (uint32_t j = 0; j < l; ++j) {             /* digit */
            for (u64 k = 0; k < n; ++k) dt[k] = d[(u64)j * n + k] % qm;
            for (int part = 0; part < 2; ++part) {
                const u64 *kp = key + (((u64)j * 2 + part) * lk1 + key_limb) * n;
                or_poly_mul(dt, kp, prod, &qm, 1, log_n);
                u64 *ac = acc + ((u64)part * (l + 1) + m) * n;
                for (u64 k = 0; k < n; ++k) ac[k] = addmod(ac[k], prod[k], qm);
            }
        }
        free(dt); free(prod);
    }
    u64 P = mods[key_levels];
    for (int part = 0; part < 2; ++part) {
        u64 *o = part ? out1 : out0;
        const u64 *accp = acc + ((u64)part * (l + 1) + l) * n;
        for (uint32_t i = 0; i < l; ++i) {
            u64 q = mods[i];
            u64 pinv = or_invmod(P % q, q);
            const u64 *ai = acc + ((u64)part * (l + 1) + i) * n;
            for (u64 k = 0; k < n; ++k)
                o[(u64)i * n + k] = mulmod(submod(ai[k], accp[k] % q, q), pinv, q);
        }
    }
    free(acc);
}

/* ---------------------------------------------------------------------------------------
 * Hybrid key switching (north star "ModUp fast base conversion"):
 * digits of alpha limbs, K special primes p_0..p_{K-1}, P = prod p_k.  Reduces to
 * or_keyswitch exactly when alpha = K = 1.
 *
 * Fast base conversion (HPS): x given by residues x_i mod q_i, i in a set D (Q_D = prod):
 *   conv_D(x) mod m = sum_{i in D} [ x_i (Q_D/q_i)^{-1} ]_{q_i} * (Q_D/q_i)   mod m
 * which equals x + u Q_D for some integer 0 <= u < |D| (pinned in tests).
 *
 *   d    : [l][N] coefficient form at level l
 *   key  : [dnum][2][L+K][N]  dnum = ceil(L/alpha); limb i < L mod q_i, limb L+k mod p_k
 *   mods : L+K moduli q_0..q_{L-1}, p_0..p_{K-1}
 * Steps (digit d covers limbs D_d = [d alpha, min(d alpha + alpha, l))):
 *   ModUp   x~_{d,t} = d_t for t in D_d, else conv_{D_d}(d) mod m_t, t in {q_0..q_{l-1}, p_k}
 *   inner   acc_t = sum_d x~_{d,t} * ksk_{d,t}
 *   ModDown y = conv_{P}(acc restricted to p_0..p_{K-1}) mod q_i;
 *           out_i = (acc_i - y_i) * P^{-1} mod q_i
 * --------------------------------------------------------------------------------------- */
static u64 prod_mod(const u64 *m, const uint32_t *idx, uint32_t n, uint32_t skip, u64 mod)
{
    u64 r = 1 % mod;
    for (uint32_t a = 0; a < n; ++a)
        if (a != skip) r = mulmod(r, m[idx[a]] % mod, mod);
    return r;
}

/* out[t][N] (t indexes `tgt`) = conv_{src}(x) mod mods[tgt[t]]; x: rows x[a] for src[a] */
static void fast_bconv(const u64 *const *x, const uint32_t *src, uint32_t ns, const uint32_t *tgt, uint32_t nt,
                       const u64 *mods, u64 n, u64 *out)
{
    u64 *yinv = (u64 *)malloc(ns * sizeof(u64));
    for (uint32_t a = 0; a < ns; ++a) {
        u64 qa = mods[src[a]];
        yinv[a] = or_invmod(prod_mod(mods, src, ns, a, qa), qa); /* (Q_D/q_a)^{-1} mod q_a */
    }
    #pragma omp parallel for schedule(static)
    for (uint32_t t = 0; t < nt; ++t) {
        u64 mt = mods[tgt[t]];
        for (u64 k = 0; k < n; ++k) {
            u64 acc = 0;
            for (uint32_t a = 0; a < ns; ++a) {
                u64 qa = mods[src[a]];
                u64 y = mulmod(x[a][k], yinv[a], qa);                 /* [x_a (Q_D/q_a)^{-1}]_{q_a} */
                acc = addmod(acc, mulmod(y % mt, prod_mod(mods, src, ns, a, mt), mt), mt);
            }
            out[(u64)t * n + k] = acc;
        }
    }
    free(yinv);
}

void or_fast_bconv(const u64 *x, const uint32_t *src, uint32_t ns, const uint32_t *tgt, uint32_t nt,
                   const u64 *mods, uint32_t log_n, u64 *out)
{
    u64 n = (u64)1 << log_n;
    const u64 **rows = (const u64 **)malloc(ns * sizeof(u64 *));
    for (uint32_t a = 0; a < ns; ++a) rows[a] = x + (u64)a * n;
    fast_bconv(rows, src, ns, tgt, nt, mods, n, out);
    free(rows);
}

void or_keyswitch_hybrid(const u64 *d, uint32_t l, const u64 *key, uint32_t L, uint32_t K, uint32_t alpha,
                         const u64 *mods, uint32_t log_n, u64 *out0, u64 *out1)
{
    u64 n = (u64)1 << log_n;
    uint32_t LK = L + K, ne = l + K;             /* extended basis at level l */
    uint32_t beta = (l + alpha - 1) / alpha;
    uint32_t *ext = (uint32_t *)malloc(ne * sizeof(uint32_t));
    for (uint32_t t = 0; t < l; ++t) ext[t] = t;
    for (uint32_t k = 0; k < K; ++k) ext[l + k] = L + k;
    u64 *acc = (u64 *)calloc((size_t)2 * ne * n, sizeof(u64));   /* [2][ne][N] */
    u64 *xt = (u64 *)malloc((size_t)ne * n * sizeof(u64));         /* x~_d over ext */
    uint32_t *src = (uint32_t *)malloc(alpha * sizeof(uint32_t));
    uint32_t *tgt = (uint32_t *)malloc(ne * sizeof(uint32_t));
    for (uint32_t dg = 0; dg < beta; ++dg) {
        uint32_t lo = dg * alpha, hi = lo + alpha < l ? lo + alpha : l, ns = hi - lo, nt = 0;
        for (uint32_t a = 0; a < ns; ++a) src[a] = lo + a;
        for (uint32_t t = 0; t < ne; ++t)
            if (!(t >= lo && t < hi)) tgt[nt++] = t;
        /* ModUp */
        u64 *conv = (u64 *)malloc((size_t)nt * n * sizeof(u64));
        {
            uint32_t *tg = (uint32_t *)malloc(nt * sizeof(uint32_t));
            for (uint32_t a = 0; a < nt; ++a) tg[a] = ext[tgt[a]];
            or_fast_bconv(d + (u64)lo * n, src, ns, tg, nt, mods, log_n, conv);
            free(tg);
        }
        for (uint32_t a = 0, c = 0; a < ne; ++a) {
            if (a >= lo && a < hi) memcpy(xt + (u64)a * n, d + (u64)a * n, n * sizeof(u64));
            else memcpy(xt + (u64)a * n, conv + (u64)(c++) * n, n * sizeof(u64));
        }
        free(conv);
        /* inner product with key digit dg (targets independent) */
        #pragma omp parallel for schedule(dynamic, 1)
        for (uint32_t t = 0; t < ne; ++t) {
            u64 mt = mods[ext[t]];
            u64 *prod = (u64 *)malloc(n * sizeof(u64));
            for (int part = 0; part < 2; ++part) {
                const u64 *kp = key + (((u64)dg * 2 + part) * LK + ext[t]) * n;
                or_poly_mul(xt + (u64)t * n, kp, prod, &mt, 1, log_n);
                u64 *ac = acc + ((u64)part * ne + t) * n;
                for (u64 k = 0; k < n; ++k) ac[k] = addmod(ac[k], prod[k], mt);
            }
            free(prod);
        }
    }
    /* ModDown */
    uint32_t *psrc = (uint32_t *)malloc(K * sizeof(uint32_t));
    uint32_t *qtgt = (uint32_t *)malloc(l * sizeof(uint32_t));
    for (uint32_t k = 0; k < K; ++k) psrc[k] = L + k;
    for (uint32_t i = 0; i < l; ++i) qtgt[i] = i;
    u64 *y = (u64 *)malloc((size_t)l * n * sizeof(u64));
    for (int part = 0; part < 2; ++part) {
        u64 *o = part ? out1 : out0;
        or_fast_bconv(acc + ((u64)part * ne + l) * n, psrc, K, qtgt, l, mods, log_n, y);
        for (uint32_t i = 0; i < l; ++i) {
            u64 q = mods[i], pm = 1;
            for (uint32_t k = 0; k < K; ++k) pm = mulmod(pm, mods[L + k] % q, q);
            u64 pinv = or_invmod(pm, q);
            const u64 *ai = acc + ((u64)part * ne + i) * n;
            for (u64 k = 0; k < n; ++k) o[(u64)i * n + k] = mulmod(submod(ai[k], y[(u64)i * n + k], q), pinv, q);
        }
    }
    free(y); free(psrc); free(qtgt); free(src); free(tgt); free(xt); free(acc); free(ext);
}

/* Threads of the OpenMP loops above (timing / process plumbing only: a forked worker sets 1,
 * since libgomp's thread pool does not survive fork()). */
void or_set_threads(int n) { omp_set_num_threads(n > 0 ? n : 1); }
