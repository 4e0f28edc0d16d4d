// ks_cluster.cu -- the alpha = 1 key switch's ModUp + NTT + inner product fused on
// thread-block clusters (readings A6-A9).
//
// For target prime q_t (an FP64-mode prime, q_t < 2^42) and digit j the key switch needs
//     NTT_t(d_j mod q_t) (.) ksk_{j,t}        summed over j < l        (d_j: coefficient form)
// The earlier two-kernel split (column phase -> HBM slab I -> row phase + MAC) moved every
// intermediate NTT through HBM (472 MB per C3 HMult).  Here one CLUSTER of CL = N / 4096 CTAs
// holds a whole limb: CTA cb owns coefficient block [cb 4096, (cb+1) 4096) of the NTT output
// and the matching inner-product accumulators (registers) for the whole digit loop, so the
// NTT intermediates never leave the chip:
//   phase 1  the S1 = log2 CL top Cooley-Tukey stages (index bits 11+S1 .. 12) on the CTA's
//            columns: CL segments of d_j (TMA bulk copies from L2), ModUp reduction in the
//            load, then each value goes straight into its owner's shared memory with an
//            asynchronous remote store (st.async, counted on the owner's mbarrier);
//   phase 2  the 12 stages of the local block as four radix-8 rounds (index bits 11..9, 8..6,
//            5..3, 2..0) with three shared-memory exchanges, 512 threads x 8 values, XOR-swizzled
//            so that every round's accesses are bank-conflict free;
//   MAC      acc_{b,a} += v * ksk  against the key block (TMA bulk copy, issued one digit
//            ahead), the key kept in HBM in this kernel's register order ("MAC layout").
// Phase 1 of the next digit is issued before phase 2 of the current one, so the DSMEM
// transfer overlaps the arithmetic (landing buffers double-buffered; a relaxed cluster barrier
// per digit orders their reuse).  Arithmetic: exact integers in doubles on the FP64 pipe
// (ntt.cuh FP64 mode), the modular product an FMA two-product with the quotient rounded from
// the high part; values stay lazy and signed (|v| < 17 q) through the transform, every MAC
// term is reduced (|term| < 0.6 q) and the accumulator (|acc| < 0.6 l q < 2^48) is
// canonicalised once.
//
// Work balance: units (ciphertext c, target t, digit j) are split into G equal contiguous
// ranges, one per resident cluster; a (c, t) segment cut between clusters is summed by the
// last CTA to finish it (partials in scratch, counters per (segment, block)).  Bit-identical
// to launch_ks_modup_cols + launch_ks_mac (the sum mod q_t is the same exact value).
#include <cooperative_groups.h>

#include <algorithm>

#include "internal.h"

namespace {

constexpr int KC_T = 512;                    // threads per CTA, 8 values each
constexpr int KC_B = 4096;                   // coefficients per CTA
constexpr int KC_TW = 7 + 56;                // shared twiddles: round A (7) + round B (56)
constexpr size_t KC_SMEM = (size_t)KC_B * 8        // dbuf (u64 digits, TMA)
                           + (size_t)2 * KC_B * 8  // kbuf (key b | a, TMA)
                           + (size_t)3 * KC_B * 8  // landing[2] (st.async) + exchange
                           + (size_t)(KC_TW + 16) * 8 + 64;

__device__ __forceinline__ u32 smem_u32(const void *p) { return (u32)__cvta_generic_to_shared(p); }

// ---- PTX wrappers: mbarrier, TMA bulk copy, cluster barrier, DSMEM ------------------------
__device__ __forceinline__ void mbar_init(u64 *bar, u32 count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(u64 *bar, u32 bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(u64 *bar, u32 parity)
{
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "KC_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra KC_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// wait for data written into this CTA by its cluster peers (st.async complete_tx)
__device__ __forceinline__ void mbar_wait_cluster(u64 *bar, u32 parity)
{
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "KC_WAITC_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra KC_WAITC_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_1d(void *dst, const void *src, u32 bytes, u64 *bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// the relaxed cluster barrier only orders the landing buffers' reuse (reads done before the next
// remote writes); data visibility comes from the st.async transaction counts
__device__ __forceinline__ void cluster_arrive_relaxed()
{
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ u32 cluster_rank()
{
    u32 r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ u32 dsmem_addr(u32 local, u32 rank)
{
    u32 r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
    return r;
}
// asynchronous remote store: 8 bytes into a peer's shared memory, counted on the peer's mbarrier
__device__ __forceinline__ void st_async(u32 addr, double v, u32 bar)
{
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(addr), "d"(v),
                 "r"(bar)
                 : "memory");
}

// y * w mod q as a signed representative (|r| < 0.53 q + 2^-53 |y| q) for |y| < 2^46, 0 <= w < q <
// 2^42: y w = h + lo exactly; c = round(h / q) (within one of the true quotient); h - c q is an
// integer below 2^41 (exact FMA) and adding lo is exact.
__device__ __forceinline__ double kc_mulmod(double y, double w, double q, double qinv)
{
    const double h = y * w;
    const double lo = fma(y, w, -h);
    const double c = fma(h, qinv, F64_C) - F64_C;
    return fma(-c, q, h) + lo;
}

// First NS stages of a radix-8 Cooley-Tukey round: v[r] holds the element whose 3 round bits
// are r (bit 2 = most significant); stage k pairs register bit 2-k with twiddle tw(k, r >> (3-k)).
template <int NS, class TW>
__device__ __forceinline__ void kc_ct8(double v[8], const TW &tw, double q, double qinv)
{
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        const int bit = 2 - k;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            if (r & (1 << bit)) continue;
            const double t = kc_mulmod(v[r | (1 << bit)], tw(k, r >> (bit + 1)), q, qinv);
            const double x = v[r];
            v[r] = x + t;
            v[r | (1 << bit)] = x - t;
        }
    }
}

struct KcArgs {
    const u64 *D;           // coefficient-form digits: digit j of ciphertext c at
    u32 dw, dcnt, dc0;      //   D + (((j / dw) dcnt + dc0 + c) dw + j % dw) N
    PolyMap din;            // NTT-form input (one poly per ciphertext), diagonal digit j == t
    const u32 *perm;        // NTT-domain Galois gather of din (nullptr: none)
    const double *key;      // [Lk][2][Lk+1][N]; FP64-mode limbs in MAC layout, as doubles
    u32 Lk, l, sp;          // key levels, active level, table index of P
    u64 *ext;               // [cnt][2][l+1][N] accumulators (NTT form, canonical)
    double *part;           // [G][2 slots][2 polys][N] partial sums of cut segments
    u32 *ctr;               // [cnt nT][CL] completion counters (zero between launches)
    const u32 *tmap;        // the nT FP64-mode targets (t <= l; t == l is P)
    u32 nT;
    u64 wide;               // bit j: digit source prime q_j >= 2^42 (reduced in integer first)
    u64 U;                  // units = cnt nT l
    u32 G;                  // clusters
};

__device__ __forceinline__ u64 kc_u0(u64 g, u64 U, u32 G) { return g * U / G; }
__device__ __forceinline__ u32 kc_cluster_of(u64 u, u64 U, u32 G) { return (u32)(((u + 1) * G - 1) / U); }

// bank-conflict-free placement of a 12-bit local index for all four round layouts (half-warp
// lanes vary index bits {0..3}, {0..3}, {0,1,2,6} and {3..6}): bits 0..2 ^= bits 4..6, bit 3 ^= bit 6
__device__ __forceinline__ int kc_sw(int x) { return x ^ ((x >> 4) & 7) ^ (((x >> 6) & 1) << 3); }

// unit iterator: unit u = (c nT + ti) l + j, advanced without divisions
struct KcUnit {
    u64 u;
    u32 c, ti, j, t;
    __device__ __forceinline__ void set(const KcArgs &a, u64 uu)
    {
        u = uu;
        const u64 seg = uu / a.l;
        j = (u32)(uu - seg * a.l);
        c = (u32)(seg / a.nT);
        ti = (u32)(seg - (u64)c * a.nT);
        t = __ldg(a.tmap + ti);
    }
    __device__ __forceinline__ void next(const KcArgs &a)
    {
        ++u;
        if (++j == a.l) {
            j = 0;
            if (++ti == a.nT) {
                ti = 0;
                ++c;
            }
            t = __ldg(a.tmap + ti);
        }
    }
    __device__ __forceinline__ bool diag() const { return j == t; }
};

template <int S1>
__global__ void __launch_bounds__(KC_T, 1) k_ks_cluster(KcArgs a, Tables tb)
{
    constexpr int CL = 1 << S1, SEG = KC_B / CL;  // SEG: elements per phase-1 segment
    constexpr int MM = S1 <= 3 ? 8 / CL : 1;
    extern __shared__ __align__(128) unsigned char kc_smem[];
    u64 *dbuf = reinterpret_cast<u64 *>(kc_smem);
    double *kbuf = reinterpret_cast<double *>(dbuf + KC_B);
    double *land = kbuf + 2 * KC_B;  // [2][KC_B]
    double *exch = land + 2 * KC_B;
    double *twS = exch + KC_B;       // round A (7) + round B (56) of the phase-2 target
    double *twP = twS + KC_TW;       // phase-1 stages of the phase-1 target (15)
    u64 *bars = reinterpret_cast<u64 *>(twP + 16);  // [0] digits, [1] key, [2..3] landing
    u32 *flag = reinterpret_cast<u32 *>(bars + 4);

    const int lt = threadIdx.x;
    const u32 cb = CL > 1 ? cluster_rank() : 0;
    const u32 g = blockIdx.x / CL;
    const u32 log_n = tb.log_n;
    const size_t nn = (size_t)1 << log_n;
    const u64 u0 = kc_u0(g, a.U, a.G), u1 = kc_u0(g + 1, a.U, a.G);
    if (u0 >= u1) return;  // (uniform per cluster)
    if (lt == 0) {
        for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cluster_arrive();  // peers' landing barriers are initialised before any remote store
    cluster_wait();

    // TMA issue (one thread): the digit's CL column segments of this block / the key block
    auto issue_d = [&](const KcUnit &x) {
        const u64 *src = a.D + (((size_t)(x.j / a.dw) * a.dcnt + a.dc0 + x.c) * a.dw + x.j % a.dw) * nn +
                         (size_t)cb * SEG;
        mbar_expect_tx(&bars[0], KC_B * 8);
#pragma unroll
        for (int h = 0; h < CL; ++h) tma_1d(dbuf + h * SEG, src + (size_t)h * KC_B, SEG * 8, &bars[0]);
    };
    auto issue_k = [&](const KcUnit &x) {
        const u32 kl = x.t < a.l ? x.t : a.Lk;
        const double *kb = a.key + ((size_t)(2 * x.j) * (a.Lk + 1) + kl) * nn + (size_t)cb * KC_B;
        mbar_expect_tx(&bars[1], 2 * KC_B * 8);
        tma_1d(kbuf, kb, KC_B * 8, &bars[1]);
        tma_1d(kbuf + KC_B, kb + (size_t)(a.Lk + 1) * nn, KC_B * 8, &bars[1]);
    };
    const double2 *psif = tb.psif;
    auto tw_of = [&](u32 t) { return psif + ((size_t)(t < a.l ? t : a.sp) << log_n); };

    u32 dpar = 0, kpar = 0, lpar = 0;  // mbarrier phase parities (lpar: bit b = landing b)
    KcUnit dq;                          // the unit whose digits the dbuf TMA carries next
    auto adv_nd = [&](KcUnit &x) {      // to the next non-diagonal unit (or u1)
        while (x.u < u1 && x.diag()) x.next(a);
    };
    u32 p1_t = 0xffffffffu;             // target whose phase-1 twiddles / modulus are loaded
    double p1_q = 0, p1_qi = 0;
    ModC p1_m{};
    // phase 1 of unit x into landing buffer `buf` of every CTA of the cluster; ends with the
    // block barrier after which dbuf, kbuf and exch are free (prefetches issued there)
    const int h3 = S1 == 4 ? (lt & 1) : 0;     // phase-1 ownership: (h bit 3,) column m0
    const int m0 = S1 == 4 ? (lt >> 1) : lt;
    auto phase1 = [&](const KcUnit &x, bool have, int buf, const KcUnit *knext) {
        const bool run = have && !x.diag();
        double v[8];
        if (run) {
            if (x.t != p1_t) {  // new phase-1 target: its stage twiddles and modulus
                const double2 *tw = tw_of(x.t);
                if (lt < (1 << S1) - 1) twP[lt] = tw[lt + 1].x;
                const double2 qq = __ldg(tw);
                p1_q = qq.x;
                p1_qi = qq.y;
                p1_m = load_mod(tb.mod, x.t < a.l ? x.t : a.sp);
                p1_t = x.t;
            }
            if (S1 > 0 && lt == 0) mbar_expect_tx(&bars[2 + buf], KC_B * 8);  // this block arrives from all peers
            mbar_wait(&bars[0], dpar);
            dpar ^= 1;
            const bool wide = x.j < 64 && ((a.wide >> x.j) & 1);
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const int h = S1 == 4 ? (h3 << 3) | r : r / MM, mm = S1 == 4 ? 0 : r % MM;
                const u64 y = dbuf[h * SEG + mm * KC_T + m0];
                v[r] = u2d(wide ? reduce64(y, p1_m.q, p1_m.bar) : y);
            }
        }
        __syncthreads();  // dbuf, kbuf (previous MAC) and exch (previous round D) consumed
        if (lt == 0) {
            if (run) {
                dq.next(a);
                adv_nd(dq);
                if (dq.u < u1) issue_d(dq);
            }
            if (knext) issue_k(*knext);
        }
        if (!run) return;
        if constexpr (S1 == 4) {
            // stage 0 (h bit 3) across the lane pair, then stages 1..3 on the register bits
            const double w = twP[0];
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const double o = __shfl_xor_sync(0xffffffffu, v[r], 1);
                const double lo = h3 ? o : v[r], hi = h3 ? v[r] : o;
                const double tt = kc_mulmod(hi, w, p1_q, p1_qi);
                v[r] = h3 ? lo - tt : lo + tt;
            }
            kc_ct8<3>(v, [&](int k, int e) { return twP[(2 << k) - 1 + (h3 << k) + e]; }, p1_q, p1_qi);
        } else if constexpr (S1 > 0) {
            kc_ct8<S1>(v, [&](int k, int e) { return twP[(1 << k) - 1 + e]; }, p1_q, p1_qi);
        }
        // value (h, m) belongs to CTA h at local index cb SEG + m
        const u32 lbase = smem_u32(land + buf * KC_B), bbase = smem_u32(&bars[2 + buf]);
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int h = S1 == 4 ? (h3 << 3) | r : r / MM, mm = S1 == 4 ? 0 : r % MM;
            const u32 pos = (u32)kc_sw((int)cb * SEG + mm * KC_T + m0);
            if constexpr (S1 == 0)  // a one-CTA "cluster": plain stores, ordered by the next barrier
                land[buf * KC_B + pos] = v[r];
            else
                st_async(dsmem_addr(lbase + 8u * pos, h), v[r], dsmem_addr(bbase, h));
        }
    };

    double acc0[8], acc1[8], twC[7], twD[7];
    double q = 0, qinv = 0;
    // per segment: round-A/B twiddles (shared) and round-C/D twiddles (registers) of (t, cb)
    auto load_tw = [&](u32 t) {
        const double2 *tw = tw_of(t);
        const double2 qq = __ldg(tw);
        q = qq.x;
        qinv = qq.y;
        for (int i = lt; i < KC_TW; i += KC_T) {
            double w;
            if (i < 7) {  // round A: stage k entry e
                const int k = 31 - __clz(i + 1), e = i + 1 - (1 << k);
                w = tw[(1u << (S1 + k)) + (cb << k) + e].x;
            } else {  // round B: stage k, (a << k) + e
                const int x = i - 7;
                const int k = x < 8 ? 0 : x < 24 ? 1 : 2;
                const int y = x - 8 * ((1 << k) - 1);
                w = tw[(1u << (S1 + 3 + k)) + (cb << (3 + k)) + y].x;
            }
            twS[i] = w;
        }
        const u32 hiC = (u32)lt >> 3;
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
            for (int e = 0; e < (1 << k); ++e) {
                twC[(1 << k) - 1 + e] = __ldg(&tw[(1u << (S1 + 6 + k)) + (cb << (6 + k)) + (hiC << k) + e].x);
                twD[(1 << k) - 1 + e] = __ldg(&tw[(1u << (S1 + 9 + k)) + (cb << (9 + k)) + ((u32)lt << k) + e].x);
            }
#pragma unroll
        for (int r = 0; r < 8; ++r) acc0[r] = acc1[r] = 0.0;
    };

    KcUnit cur, nxt;
    cur.set(a, u0);
    nxt = cur;
    nxt.next(a);
    load_tw(cur.t);
    if (lt == 0) {
        dq = cur;
        adv_nd(dq);
        if (dq.u < u1) issue_d(dq);
    } else {
        dq = cur;
    }
    phase1(cur, true, 0, nullptr);
    cluster_arrive_relaxed();
    const int aB = lt >> 6, bB = lt & 63;   // round B: thread bits 11..9 and 5..0
    const int hC = lt >> 3, lC = lt & 7;    // round C: thread bits 11..6 and 2..0
    u32 k = 0;
    for (; cur.u < u1; cur = nxt, nxt.next(a), ++k) {
        cluster_wait();  // every CTA finished reading landing[(k+1)&1] (unit k-1)
        // (its barrier also releases kbuf: the key of THIS unit is issued there, one phase 1 +
        // phase 2 ahead of the inner product that reads it)
        phase1(nxt, nxt.u < u1, (k + 1) & 1, &cur);
        // ---- phase 2 of unit cur ----
        double v[8];
        if (cur.diag()) {  // diagonal digit: din's own NTT-form limb, round-D positions
            const u64 *dp = a.din.base + (((size_t)cur.c * a.din.cap + cur.t) << log_n);
            const u32 i0 = cb * KC_B + ((u32)lt << 3);
#pragma unroll
            for (int r = 0; r < 8; ++r) v[r] = u2d(__ldg(dp + (a.perm ? __ldg(a.perm + i0 + r) : i0 + r)));
        } else {
            const int b = k & 1;
            if constexpr (S1 > 0) {
                mbar_wait_cluster(&bars[2 + b], (lpar >> b) & 1);
                lpar ^= 1u << b;
            }
            const double *lb = land + b * KC_B;
#pragma unroll
            for (int r = 0; r < 8; ++r) v[r] = lb[kc_sw((r << 9) | lt)];
            kc_ct8<3>(v, [&](int kk, int e) { return twS[(1 << kk) - 1 + e]; }, q, qinv);
#pragma unroll
            for (int r = 0; r < 8; ++r) exch[kc_sw((r << 9) | lt)] = v[r];
            __syncthreads();
#pragma unroll
            for (int r = 0; r < 8; ++r) v[r] = exch[kc_sw((aB << 9) | (r << 6) | bB)];
            kc_ct8<3>(v, [&](int kk, int e) { return twS[7 + 8 * ((1 << kk) - 1) + (aB << kk) + e]; }, q, qinv);
#pragma unroll
            for (int r = 0; r < 8; ++r) exch[kc_sw((aB << 9) | (r << 6) | bB)] = v[r];
            __syncthreads();
#pragma unroll
            for (int r = 0; r < 8; ++r) v[r] = exch[kc_sw((hC << 6) | (r << 3) | lC)];
            kc_ct8<3>(v, [&](int kk, int e) { return twC[(1 << kk) - 1 + e]; }, q, qinv);
#pragma unroll
            for (int r = 0; r < 8; ++r) exch[kc_sw((hC << 6) | (r << 3) | lC)] = v[r];
            __syncthreads();
#pragma unroll
            for (int r = 0; r < 8; ++r) v[r] = exch[kc_sw((lt << 3) | r)];
            kc_ct8<3>(v, [&](int kk, int e) { return twD[(1 << kk) - 1 + e]; }, q, qinv);
        }
        // ---- inner product with ksk_{j,t} (MAC layout: element lt*8 + r at r*512 + lt) ----
        mbar_wait(&bars[1], kpar);
        kpar ^= 1;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            acc0[r] += kc_mulmod(v[r], kbuf[r * KC_T + lt], q, qinv);
            acc1[r] += kc_mulmod(v[r], kbuf[KC_B + r * KC_T + lt], q, qinv);
        }
        // ---- end of a (c, t) segment: store or combine ----
        if (cur.j + 1 == a.l || cur.u + 1 == u1) {
            const u64 segi = cur.u / a.l, su0 = segi * a.l, su1 = su0 + a.l;
            const u32 glo = kc_cluster_of(su0, a.U, a.G), ghi = kc_cluster_of(su1 - 1, a.U, a.G);
            const size_t ob = (size_t)cb * KC_B + ((u32)lt << 3);
            u64 *e0 = a.ext + (((size_t)cur.c * 2 * (a.l + 1) + cur.t) << log_n) + ob;
            u64 *e1 = e0 + ((size_t)(a.l + 1) << log_n);
            bool write = glo == ghi;
            if (!write) {
                const u32 slot = (su0 <= u0) ? 0 : 1;
                double *p0 = a.part + ((size_t)(g * 2 + slot) * 2) * nn + ob;
                double *p1 = p0 + nn;
#pragma unroll
                for (int r = 0; r < 8; r += 2) {
                    *reinterpret_cast<double2 *>(p0 + r) = make_double2(acc0[r], acc0[r + 1]);
                    *reinterpret_cast<double2 *>(p1 + r) = make_double2(acc1[r], acc1[r + 1]);
                }
                __threadfence();
                __syncthreads();
                if (lt == 0) {
                    u32 *cp = a.ctr + segi * CL + cb;
                    const u32 old = atomicAdd(cp, 1u);
                    const bool last = old == ghi - glo;
                    if (last) *cp = 0;  // every part has arrived: reset for the next launch
                    *flag = last;
                }
                __syncthreads();
                write = *flag;
                if (write) {
                    __threadfence();
                    for (u32 go = glo; go <= ghi; ++go) {
                        if (go == g) continue;
                        const u32 so = (su0 <= kc_u0(go, a.U, a.G)) ? 0 : 1;
                        const double *q0 = a.part + ((size_t)(go * 2 + so) * 2) * nn + ob;
                        const double *q1 = q0 + nn;
#pragma unroll
                        for (int r = 0; r < 8; r += 2) {
                            const double2 x = __ldcg(reinterpret_cast<const double2 *>(q0 + r));
                            const double2 y = __ldcg(reinterpret_cast<const double2 *>(q1 + r));
                            acc0[r] += x.x;
                            acc0[r + 1] += x.y;
                            acc1[r] += y.x;
                            acc1[r + 1] += y.y;
                        }
                    }
                }
            }
            if (write) {
#pragma unroll
                for (int r = 0; r < 8; r += 2) {
                    *reinterpret_cast<ulonglong2 *>(e0 + r) =
                        make_ulonglong2(f64_canon(acc0[r], q, qinv), f64_canon(acc0[r + 1], q, qinv));
                    *reinterpret_cast<ulonglong2 *>(e1 + r) =
                        make_ulonglong2(f64_canon(acc1[r], q, qinv), f64_canon(acc1[r + 1], q, qinv));
                }
            }
            // next segment's tables: twS is read only in rounds A/B (all done: the barrier after
            // round C's stores), and the next round A follows the next phase-1 barrier
            if (nxt.u < u1) load_tw(nxt.t);
        }
        cluster_arrive_relaxed();
    }
    cluster_wait();  // no CTA leaves while a peer may still address its shared memory
}

// key limb -> MAC layout (in place, per 4096 block): element lt*8 + r moves to r*512 + lt, as a double
__global__ void __launch_bounds__(256) k_key_mac_layout(u64 *key, const u32 *limbs, u32 nl, u32 Lk1, u32 log_n,
                                                        int inverse)
{
    __shared__ u64 s[KC_B];
    const u32 blocks = 1u << (log_n - 12);
    const u32 b = blockIdx.x % blocks, rest = blockIdx.x / blocks;
    const u32 li = rest % nl, dp = rest / nl;  // dp = digit * 2 + poly
    u64 *p = key + (((size_t)dp * Lk1 + __ldg(limbs + li)) << log_n) + (size_t)b * KC_B;
    for (int i = threadIdx.x; i < KC_B; i += 256) s[i] = p[i];
    __syncthreads();
    for (int i = threadIdx.x; i < KC_B; i += 256) {
        const int r = i >> 9, l = i & 511;  // MAC position i = r*512 + l  <->  standard l*8 + r
        if (!inverse)
            p[i] = (u64)__double_as_longlong(u2d(s[l * 8 + r]));
        else
            p[l * 8 + r] = d2u(__longlong_as_double((long long)s[i]));
    }
}

template <int S1>
bool kc_prepare(int dev, int &clusters)
{
    static int cached[17] = {0};
    static bool done[17] = {false};
    if (!done[S1]) {
        done[S1] = true;
        auto *k = k_ks_cluster<S1>;
        if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)KC_SMEM) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        if ((1 << S1) > 8 && cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 1u << S1;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(1u << S1);
        cfg.blockDim = dim3(KC_T);
        cfg.dynamicSmemBytes = KC_SMEM;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, k, &cfg) != cudaSuccess) {
            cudaGetLastError();
            n = 0;
        }
        cached[S1] = n;
        (void)dev;
    }
    clusters = cached[S1];
    return clusters > 0;
}

template <int S1>
void kc_launch(const Launch &L, const KcArgs &a, cudaStream_t st, Work w)
{
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 1u << S1;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(a.G << S1);
    cfg.blockDim = dim3(KC_T);
    cfg.dynamicSmemBytes = KC_SMEM;
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    Launch Ls = L;
    Ls.st = st;
    KLAUNCH(Ls, "ks_cluster", w, (cudaLaunchKernelEx(&cfg, k_ks_cluster<S1>, a, *L.tb)));
}

}  // namespace

bool ks_cluster_supported(const Launch &L)
{
    int n = 0;
    switch (L.tb->log_n) {
    case 12: return kc_prepare<0>(0, n);
    case 13: return kc_prepare<1>(0, n);
    case 14: return kc_prepare<2>(0, n);
    case 15: return kc_prepare<3>(0, n);
    case 16: return kc_prepare<4>(0, n);
    default: return false;
    }
}

size_t ks_cluster_part_words(const Launch &L)
{
    int n = 0;
    switch (L.tb->log_n) {
    case 12: kc_prepare<0>(0, n); break;
    case 13: kc_prepare<1>(0, n); break;
    case 14: kc_prepare<2>(0, n); break;
    case 15: kc_prepare<3>(0, n); break;
    case 16: kc_prepare<4>(0, n); break;
    default: break;
    }
    return (size_t)std::max(n, 1) * 4 << L.tb->log_n;
}

void launch_key_mac_layout(const Launch &L, u64 *key, const u32 *limbs, u32 nl, u32 nkeyrows, u32 Lk1, bool inverse)
{
    if (!nl || !nkeyrows) return;
    const u32 blocks = (1u << (L.tb->log_n - 12)) * nl * nkeyrows;
    KLAUNCH(L, "key_mac_layout", (Work{0, 0, 16.0 * nl * nkeyrows * (1u << L.tb->log_n)}),
            (k_key_mac_layout<<<blocks, 256, 0, L.st>>>(key, limbs, nl, Lk1, L.tb->log_n, inverse ? 1 : 0)));
}

void launch_ks_cluster(const Launch &L, cudaStream_t st, const u64 *D, u32 dw, u32 dcnt, u32 dc0, PolyMap din,
                       const u32 *perm, const u64 *key, u32 Lk, u32 l, u32 cnt, const u32 *tmap_dev,
                       const u32 *tmap_host, u32 nT, u64 *ext, double *part, u32 *ctr, u32 sp)
{
    if (!cnt || !nT) return;
    const u32 log_n = L.tb->log_n, S1 = log_n - 12;
    int maxc = 0;
    switch (S1) {
    case 0: kc_prepare<0>(0, maxc); break;
    case 1: kc_prepare<1>(0, maxc); break;
    case 2: kc_prepare<2>(0, maxc); break;
    case 3: kc_prepare<3>(0, maxc); break;
    case 4: kc_prepare<4>(0, maxc); break;
    default: return;
    }
    KcArgs a{};
    a.D = D;
    a.dw = dw;
    a.dcnt = dcnt;
    a.dc0 = dc0;
    a.din = din;
    a.perm = perm;
    a.key = reinterpret_cast<const double *>(key);
    a.Lk = Lk;
    a.l = l;
    a.sp = sp;
    a.ext = ext;
    a.part = part;
    a.ctr = ctr;
    a.tmap = tmap_dev;
    a.nT = nT;
    a.U = (u64)cnt * nT * l;
    a.wide = 0;
    for (u32 j = 0; j < l && j < 64; ++j)
        if (L.hprimes[j] >= F64_Q_MAX) a.wide |= 1ull << j;
    a.G = (u32)std::min<u64>((u64)std::max(maxc, 1), a.U);
    // work: per non-diagonal unit one limb NTT on the FP64 pipe; 2 MACs per coefficient per unit
    u32 ndiag = 0;
    for (u32 i = 0; i < nT; ++i) ndiag += tmap_host[i] < l ? 1 : 0;
    const double n_ = (double)(1u << log_n);
    const double ntts = (double)cnt * ((double)nT * l - ndiag);
    Work w{0, 0, 0, 0, 0};
    w.fbfly = ntts * n_ / 2 * log_n;
    w.fmac = 2.0 * (double)a.U * n_;
    // bytes: digits (read per target from L2; counted once), key once per launch, output
    w.bytes = 8.0 * n_ * ((double)cnt * l + 2.0 * nT * l + 2.0 * cnt * nT);
    switch (S1) {
    case 0: kc_launch<0>(L, a, st, w); break;
    case 1: kc_launch<1>(L, a, st, w); break;
    case 2: kc_launch<2>(L, a, st, w); break;
    case 3: kc_launch<3>(L, a, st, w); break;
    case 4: kc_launch<4>(L, a, st, w); break;
    default: break;
    }
}
