// ntt.cuh -- batched negacyclic NTT/INTT building blocks for sm_100a.
//
// Transform: forward Cooley-Tukey with merged psi twiddles (Longa-Naehrig), output in
// bit-reversed order:  out[k] = sum_j a_j psi^{(2 brv(k) + 1) j}  mod q;  inverse is
// Gentleman-Sande with psi^{-1} and N^{-1}.  Global stage g (0 <= g < log N) pairs
// indices differing in bit (log N - 1 - g) and uses twiddle table entry 2^g + (index >> (log N - g)).
//
// Decomposition N = N1 x N2 (N1 = 2^B1 "column" length, N2 = 2^B2 "row" length,
// B1 = floor(log N / 2)).  Stages 0..B1-1 only mix elements of one column (stride N2);
// stages B1..logN-1 only mix elements of one row (contiguous).  Each phase is one
// kernel; a tile (column or row, 2^B elements) is processed by 2^B/8 threads holding
// 8 values each in registers: radix-8 rounds of 3 stages (Harvey lazy butterflies,
// Shoup twiddles), with shared-memory exchanges between rounds.  Rows are handled by
// <= 1 warp each (warp-synchronous exchanges, no block barriers); column tiles are 16
// adjacent columns per CTA so every global access is a 128-byte coalesced segment.
//
// Value ranges: for q >= 2^48 forward lazy in [0, 4q), inverse in [0, 2q) (Harvey); for
// q < 2^48 no corrections at all inside the transform (bounds grow by 2q per forward stage,
// double per inverse stage, both < 2^64 for log N <= 16).  Canonicalised at the end.
//
// FP64 mode (q < tb.f64_qmax = 2^42, every 30/40-bit limb): the tile transform runs on the
// FP64 pipe, which the integer kernels leave idle and which retires ~2.5x more butterflies
// per second on B200 than the 64-bit Shoup butterfly (bench/fp64_bfly.cu).  Residues are
// exact integers in doubles; the modular product is an FMA two-product with an FMA-rounded
// quotient (f64_mulmod below), exact for |y| < 2^50, w < q < 2^42; values are signed and
// lazy (|v| < 16q inside a round) and leave the tile canonical in [0, q).
#pragma once
#include "modarith.cuh"

struct Tables {
    const ModC *mod;         // [nprimes]
    const ulonglong2 *psi;   // [nprimes][N]  (psi^{brv(k)}, Shoup companion)
    const ulonglong2 *ipsi;  // [nprimes][N]  (psi^{-brv(k)}, Shoup companion)
    const ulonglong2 *ninv;  // [nprimes]     (N^{-1} mod q, Shoup companion)
    const double2 *psif;     // [nprimes][N]  (w, w/q) as doubles for FP64-mode primes; entry 0 = (q, 1/q)
    const double2 *ipsif;    // [nprimes][N]  same for psi^{-1}
    u64 f64_qmax;            // primes below this use the FP64 tile transform (0 = never)
    u32 log_n;
};

// ---- FP64-pipe modular arithmetic (exact integers held in doubles) -----------------
constexpr double F64_C = 6755399441055744.0;  // 1.5 * 2^52: fma(x, y, C) - C = nearest integer of x*y
constexpr double F64_2P52 = 4503599627370496.0;
__device__ __forceinline__ double u2d(u64 x)  // exact for x < 2^52
{
    return __longlong_as_double((long long)(x | 0x4330000000000000ull)) - F64_2P52;
}
__device__ __forceinline__ u64 d2u(double v)  // integer 0 <= v < 2^52
{
    return (u64)__double_as_longlong(v + F64_2P52) ^ 0x4330000000000000ull;
}
// y * w mod q as a signed representative, |r| < 1.5q.  y*w = h + l exactly (two-product);
// c = round(y * w/q) within +-1 (|y| < 2^50); r = (h - c q) + l, every step exact.
__device__ __forceinline__ double f64_mulmod(double y, double w, double wq, double q)
{
    const double h = y * w;
    const double l = fma(y, w, -h);
    const double c = fma(y, wq, F64_C) - F64_C;
    return fma(-c, q, h) + l;
}
// signed representative with |r| <= q/2 + 1 (|v| < 2^50)
__device__ __forceinline__ double f64_red(double v, double q, double qinv)
{
    const double c = fma(v, qinv, F64_C) - F64_C;
    return fma(-c, q, v);
}
__device__ __forceinline__ u64 f64_canon(double v, double q, double qinv)
{
    const double r = f64_red(v, q, qinv);
    return d2u(r < 0.0 ? r + q : r);
}

// local index of element i (0..7) of thread lt when the thread owns the 3-bit block at bit p
__device__ __forceinline__ int lidx(int lt, int i, int p)
{
    return ((lt >> p) << (p + 3)) | (i << p) | (lt & ((1 << p) - 1));
}

// Shared-memory twiddle caches (the key-switch inner product keeps its rows' row-phase twiddles):
// within stage s's segment, entry p lives at p ^ ((p >> 3) & 7) for s >= 3, so the threads of a
// row reading their 2 or 4 consecutive entries (32 / 64 bytes apart) hit distinct bank groups
// (natural layout: 2- and 4-way conflicts, ncu profiles/ncu_r2_c3_k_ks_mac.txt)
__host__ __device__ __forceinline__ u32 tw_cache_swz(u32 p, int s) { return s >= 3 ? p ^ ((p >> 3) & 7) : p; }

// ---- forward CT stages on bit positions QHI..QLO (descending) of a B-bit tile -------
// LAZY (q < 2^48): no conditional subtraction at all -- each stage adds < 2q to the bound
// (x + t, x - t + 2q with t in [0, 2q)), so after log N <= 16 stages values stay < 33q < 2^64;
// Shoup's product is valid for any input < 2^64.  Canonicalised once at the end (reduce64).
template <int B, int POWN, int QHI, int QLO, bool LAZY = false, bool SMEM_TW = false>
__device__ __forceinline__ void ct_stages(u64 v[8], int lt, int k, u32 hi, const ulonglong2 *tw, u64 q)
{
    const u64 q2 = q << 1;
#pragma unroll
    for (int qq = QHI; qq >= QLO; --qq) {
        const int s = B - 1 - qq;
        const int rel = qq - POWN;
        const int bit = 1 << rel;
        const u32 base = (1u << (k + s)) + (hi << s) + ((u32)(lt >> POWN) << (2 - rel));
#pragma unroll
        for (int g = 0; g < (8 >> (rel + 1)); ++g) {
            const ulonglong2 w = SMEM_TW ? tw[(1u << (k + s)) + tw_cache_swz(base - (1u << (k + s)) + g, s)]
                                         : __ldg(tw + base + g);
#pragma unroll
            for (int j = 0; j < bit; ++j) {
                const int i0 = (g << (rel + 1)) | j, i1 = i0 | bit;
                const u64 x = LAZY ? v[i0] : csub(v[i0], q2);
                const u64 t = shoup_lazy(v[i1], w.x, w.y, q);
                v[i0] = x + t;
                v[i1] = x - t + q2;
            }
        }
    }
}

// ---- inverse GS stages on bit positions QLO..QHI (ascending) ------------------------
// LAZY (q < 2^48): after a applied stages every value is < 2^a q; u = x + y needs no
// correction (< 2^(a+1) q) and the difference is offset by 2^a q instead of 2q, so after
// log N <= 16 stages values stay < 2^16 q < 2^64.  `applied` = stages applied before this
// tile phase (0 for the row phase, B2 for the column phase).
template <int B, int POWN, int QLO, int QHI, bool LAZY = false>
__device__ __forceinline__ void gs_stages(u64 v[8], int lt, int k, u32 hi, const ulonglong2 *itw, u64 q,
                                          int applied = 0)
{
    const u64 q2 = q << 1;
#pragma unroll
    for (int qq = QLO; qq <= QHI; ++qq) {
        const int s = B - 1 - qq;
        const int rel = qq - POWN;
        const int bit = 1 << rel;
        const u32 base = (1u << (k + s)) + (hi << s) + ((u32)(lt >> POWN) << (2 - rel));
#pragma unroll
        for (int g = 0; g < (8 >> (rel + 1)); ++g) {
            const ulonglong2 w = __ldg(itw + base + g);
#pragma unroll
            for (int j = 0; j < bit; ++j) {
                const int i0 = (g << (rel + 1)) | j, i1 = i0 | bit;
                const u64 x = v[i0], y = v[i1];
                if (LAZY) {
                    const u64 off = q << (applied + qq);  // > every y at this stage
                    v[i0] = x + y;
                    v[i1] = shoup_lazy(x - y + off, w.x, w.y, q);
                } else {
                    v[i0] = csub(x + y, q2);
                    v[i1] = shoup_lazy(x - y + q2, w.x, w.y, q);
                }
            }
        }
    }
}

// ---- FP64-mode stages (same index geometry as ct_stages / gs_stages) ---------------
template <int B, int POWN, int QHI, int QLO, bool SMEM_TW = false>
__device__ __forceinline__ void ct_stages_f64(double v[8], int lt, int k, u32 hi, const double2 *tw, double q)
{
#pragma unroll
    for (int qq = QHI; qq >= QLO; --qq) {
        const int s = B - 1 - qq;
        const int rel = qq - POWN;
        const int bit = 1 << rel;
        const u32 base = (1u << (k + s)) + (hi << s) + ((u32)(lt >> POWN) << (2 - rel));
#pragma unroll
        for (int g = 0; g < (8 >> (rel + 1)); ++g) {
            const double2 w = SMEM_TW ? tw[(1u << (k + s)) + tw_cache_swz(base - (1u << (k + s)) + g, s)]
                                      : __ldg(tw + base + g);
#pragma unroll
            for (int j = 0; j < bit; ++j) {
                const int i0 = (g << (rel + 1)) | j, i1 = i0 | bit;
                const double t = f64_mulmod(v[i1], w.x, w.y, q);
                const double x = v[i0];
                v[i0] = x + t;
                v[i1] = x - t;
            }
        }
    }
}
// the sum side doubles per stage: reduced at the round's last stage (|v| < 12q inside)
template <int B, int POWN, int QLO, int QHI>
__device__ __forceinline__ void gs_stages_f64(double v[8], int lt, int k, u32 hi, const double2 *itw, double q,
                                              double qinv)
{
#pragma unroll
    for (int qq = QLO; qq <= QHI; ++qq) {
        const int s = B - 1 - qq;
        const int rel = qq - POWN;
        const int bit = 1 << rel;
        const u32 base = (1u << (k + s)) + (hi << s) + ((u32)(lt >> POWN) << (2 - rel));
#pragma unroll
        for (int g = 0; g < (8 >> (rel + 1)); ++g) {
            const double2 w = __ldg(itw + base + g);
#pragma unroll
            for (int j = 0; j < bit; ++j) {
                const int i0 = (g << (rel + 1)) | j, i1 = i0 | bit;
                const double x = v[i0], y = v[i1];
                v[i0] = (qq == QHI) ? f64_red(x + y, q, qinv) : x + y;
                v[i1] = f64_mulmod(x - y, w.x, w.y, q);
            }
        }
    }
}

// Round geometry.  CT round r covers bits [max(B-3r-3,0), B-3r); GS round r covers
// [3r, min(3r+3, B)).  The thread always owns a full 3-bit block (POWN..POWN+2).
template <int B, int R>
struct CtRound {
    static constexpr int PHI = B - 3 * R;
    static constexpr int QHI = PHI - 1;
    static constexpr int QLO = (PHI - 3 > 0) ? PHI - 3 : 0;
    static constexpr int POWN = QLO;
};
template <int B, int R>
struct GsRound {
    static constexpr int QLO = 3 * R;
    static constexpr int QHI = (3 * R + 2 < B - 1) ? 3 * R + 2 : B - 1;
    static constexpr int POWN = (3 * R + 3 <= B) ? 3 * R : B - 3;
};
template <int B>
struct NRounds {
    static constexpr int value = (B + 2) / 3;
};

// Exchange policies: store the 8 values under ownership `from`, reload under `to`.
// Row tiles: one tile per <= 32 threads -> warp-synchronous; padded 1 word per 16.
struct RowEx {
    u64 *s;
    __device__ __forceinline__ static int pad(int x) { return x + (x >> 4); }
    template <class T>
    __device__ __forceinline__ void operator()(T v[8], int lt, int from, int to) const
    {
        T *st = reinterpret_cast<T *>(s);
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 8; ++i) st[pad(lidx(lt, i, from))] = v[i];
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = st[pad(lidx(lt, i, to))];
    }
};
// Column tiles: C columns interleaved, layout s[li * C + col]; block-synchronous.
template <int C>
struct ColEx {
    u64 *s;
    int col;
    template <class T>
    __device__ __forceinline__ void operator()(T v[8], int lt, int from, int to) const
    {
        T *st = reinterpret_cast<T *>(s);
        __syncthreads();
#pragma unroll
        for (int i = 0; i < 8; ++i) st[lidx(lt, i, from) * C + col] = v[i];
        __syncthreads();
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = st[lidx(lt, i, to) * C + col];
    }
};

template <int B, int R, bool LAZY, class Ex, bool SMEM_TW = false>
__device__ __forceinline__ void fwd_rounds_t(u64 v[8], const Ex &ex, int lt, int k, u32 hi, const ulonglong2 *tw,
                                             u64 q)
{
    if constexpr (R < NRounds<B>::value) {
        if constexpr (R > 0) ex(v, lt, CtRound<B, R - 1>::POWN, CtRound<B, R>::POWN);
        ct_stages<B, CtRound<B, R>::POWN, CtRound<B, R>::QHI, CtRound<B, R>::QLO, LAZY, SMEM_TW>(v, lt, k, hi, tw, q);
        fwd_rounds_t<B, R + 1, LAZY, Ex, SMEM_TW>(v, ex, lt, k, hi, tw, q);
    }
}

template <int B, int R, bool LAZY, class Ex>
__device__ __forceinline__ void inv_rounds_t(u64 v[8], const Ex &ex, int lt, int k, u32 hi, const ulonglong2 *itw,
                                             u64 q, int applied)
{
    if constexpr (R < NRounds<B>::value) {
        if constexpr (R > 0) ex(v, lt, GsRound<B, R - 1>::POWN, GsRound<B, R>::POWN);
        gs_stages<B, GsRound<B, R>::POWN, GsRound<B, R>::QLO, GsRound<B, R>::QHI, LAZY>(v, lt, k, hi, itw, q,
                                                                                      applied);
        inv_rounds_t<B, R + 1, LAZY>(v, ex, lt, k, hi, itw, q, applied);
    }
}

constexpr u64 LAZY_Q_MAX = 1ull << 48;
constexpr u64 F64_Q_MAX = 1ull << 42;

// Lazy forward phase for a wide prime (q >= 2^48): a phase of B <= 7 stages started from a
// CANONICAL input stays below (2B + 1) q < 2^64 without any correction (each lazy stage adds
// < 2q), so the Harvey conditional subtraction (6 instructions per butterfly) is dropped and
// the phase ends with one reduce64 per value.  Holds for every 60-bit prime when B <= 7 (the
// N <= 2^14 phases); the N = 2^16 phases (B = 8) keep Harvey for q > 2^64 / 17.
template <int B>
__host__ __device__ __forceinline__ bool lazy_wide(u64 q)
{
#ifdef CKKS_NO_LAZY_WIDE
    return false;
#else
    return B <= 7 && q >= LAZY_Q_MAX && q <= ~0ull / (2 * B + 1);
#endif
}

template <int B, int R, class Ex, bool SMEM_TW = false>
__device__ __forceinline__ void fwd_rounds_f64(double v[8], const Ex &ex, int lt, int k, u32 hi, const double2 *twf,
                                               double q)
{
    if constexpr (R < NRounds<B>::value) {
        if constexpr (R > 0) ex(v, lt, CtRound<B, R - 1>::POWN, CtRound<B, R>::POWN);
        ct_stages_f64<B, CtRound<B, R>::POWN, CtRound<B, R>::QHI, CtRound<B, R>::QLO, SMEM_TW>(v, lt, k, hi, twf, q);
        fwd_rounds_f64<B, R + 1, Ex, SMEM_TW>(v, ex, lt, k, hi, twf, q);
    }
}
template <int B, int R, class Ex>
__device__ __forceinline__ void inv_rounds_f64(double v[8], const Ex &ex, int lt, int k, u32 hi, const double2 *itwf,
                                               double q, double qinv)
{
    if constexpr (R < NRounds<B>::value) {
        if constexpr (R > 0) ex(v, lt, GsRound<B, R - 1>::POWN, GsRound<B, R>::POWN);
        gs_stages_f64<B, GsRound<B, R>::POWN, GsRound<B, R>::QLO, GsRound<B, R>::QHI>(v, lt, k, hi, itwf, q, qinv);
        inv_rounds_f64<B, R + 1>(v, ex, lt, k, hi, itwf, q, qinv);
    }
}
// FP64-mode tile transforms on u64 I/O: inputs < 2^52, outputs canonical [0, q)
template <int B, class Ex>
__device__ __forceinline__ void fwd_tile_f64(u64 v[8], const Ex &ex, int lt, int k, u32 hi, const double2 *twf)
{
    const double2 qq = __ldg(twf);  // entry 0: (q, 1/q)
    double d[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) d[i] = u2d(v[i]);
    fwd_rounds_f64<B, 0>(d, ex, lt, k, hi, twf, qq.x);
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = f64_canon(d[i], qq.x, qq.y);
}
// ... leaving the lazy signed doubles as raw bit patterns (|v| < 2^42 + 1.5 B q for inputs < 2^42):
// the ModUp slabs the key-switch inner product reads back as doubles (no canonicalisation, no
// integer conversion on either side)
template <int B, class Ex>
__device__ __forceinline__ void fwd_tile_f64_raw(u64 v[8], const Ex &ex, int lt, int k, u32 hi, const double2 *twf)
{
    const double2 qq = __ldg(twf);
    double d[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) d[i] = u2d(v[i]);
    fwd_rounds_f64<B, 0>(d, ex, lt, k, hi, twf, qq.x);
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = (u64)__double_as_longlong(d[i]);
}
template <int B, class Ex>
__device__ __forceinline__ void inv_tile_f64(u64 v[8], const Ex &ex, int lt, int k, u32 hi, const double2 *itwf)
{
    const double2 qq = __ldg(itwf);
    double d[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) d[i] = u2d(v[i]);
    inv_rounds_f64<B, 0>(d, ex, lt, k, hi, itwf, qq.x, qq.y);
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = f64_canon(d[i], qq.x, qq.y);
}

// Forward tile transform; values leave lazy: < 4q (q >= 2^48) or < (2 log N + 1) q (q < 2^48),
// canonical in FP64 mode (q < tb.f64_qmax: pass twf != nullptr and f64 = true).
template <int B, int R, class Ex>
__device__ __forceinline__ void fwd_rounds(u64 v[8], const Ex &ex, int lt, int k, u32 hi, const ulonglong2 *tw,
                                           u64 q, const double2 *twf = nullptr, bool f64 = false)
{
    if (f64)
        fwd_tile_f64<B>(v, ex, lt, k, hi, twf);
    else if (q < LAZY_Q_MAX || lazy_wide<B>(q))
        fwd_rounds_t<B, R, true>(v, ex, lt, k, hi, tw, q);
    else
        fwd_rounds_t<B, R, false>(v, ex, lt, k, hi, tw, q);
}

// Inverse tile transform; `applied` GS stages were applied before this phase.
// Values leave lazy: < 2q (q >= 2^48) or < 2^(applied + B) q (q < 2^48).
template <int B, int R, class Ex>
__device__ __forceinline__ void inv_rounds(u64 v[8], const Ex &ex, int lt, int k, u32 hi, const ulonglong2 *itw,
                                           u64 q, int applied, const double2 *itwf = nullptr, bool f64 = false)
{
    if (f64)
        inv_tile_f64<B>(v, ex, lt, k, hi, itwf);
    else if (q < LAZY_Q_MAX)
        inv_rounds_t<B, R, true>(v, ex, lt, k, hi, itw, q, applied);
    else
        inv_rounds_t<B, R, false>(v, ex, lt, k, hi, itw, q, applied);
}

// canonical residue of a forward-lazy value after a B-stage phase (already canonical in FP64 mode)
template <int B>
__device__ __forceinline__ u64 fwd_canon(u64 x, const ModC &m, bool f64 = false)
{
    return f64 ? x : (m.q < LAZY_Q_MAX || lazy_wide<B>(m.q)) ? reduce64(x, m.q, m.bar) : csub(csub(x, 2 * m.q), m.q);
}
__device__ __forceinline__ bool use_f64(const Tables &tb, u64 q) { return q < tb.f64_qmax; }

// First/last ownership of each phase (used for the global I/O patterns):
//   forward:  first POWN = B-3 (li = (i << (B-3)) | lt),  last POWN = 0 (li = 8 lt + i)
//   inverse:  first POWN = 0   (li = 8 lt + i),           last POWN = B-3
template <int B>
struct Phase {
    static constexpr int THR = (1 << B) / 8;
    static constexpr int FWD_FIRST = CtRound<B, 0>::POWN;
    static constexpr int FWD_LAST = CtRound<B, NRounds<B>::value - 1>::POWN;
    static constexpr int INV_FIRST = GsRound<B, 0>::POWN;
    static constexpr int INV_LAST = GsRound<B, NRounds<B>::value - 1>::POWN;
    static_assert(FWD_FIRST == B - 3 && FWD_LAST == 0 && INV_FIRST == 0 && INV_LAST == B - 3, "geometry");
};
