// modarith.cuh -- 64-bit modular arithmetic on the sm_100a integer pipes.
//
// Residues are u64 with primes q < 2^62 (checked at context creation), so lazy values
// in [0, 4q) fit a machine word.  Constant multiplications use Shoup's precomputed
// quotient (one mul.hi + two mul.lo); data x data products are formed in 128 bits
// (mad.lo.cc / madc.hi) and reduced by reduce128(), which handles ANY 128-bit input:
//   x = hi 2^64 + lo,  hi 2^64 = hi * (2^64 mod q)  (Shoup, result in [0, 2q))
//                      lo      = lo - floor(lo * floor(2^64/q) / 2^64) q    in [0, 2q)
// so sums of many products can be accumulated lazily in 128 bits (limb-wise modular
// multiply-add of the inner product) and reduced once.
#pragma once
#include <cstdint>

typedef uint64_t u64;
typedef unsigned int u32;

struct ModC {
    u64 q;     // prime
    u64 r64;   // 2^64 mod q
    u64 r64s;  // Shoup companion of r64: floor(r64 * 2^64 / q)
    u64 bar;   // floor(2^64 / q)  (= Shoup companion of 1)
};

__device__ __forceinline__ u64 csub(u64 x, u64 m) { return x >= m ? x - m : x; }

// x * w mod q in [0, 2q) for any x < 2^64, w < q, ws = floor(w 2^64 / q).
__device__ __forceinline__ u64 shoup_lazy(u64 x, u64 w, u64 ws, u64 q)
{
    return x * w - __umul64hi(x, ws) * q;
}

__device__ __forceinline__ u64 shoup(u64 x, u64 w, u64 ws, u64 q) { return csub(shoup_lazy(x, w, ws, q), q); }

// exact x mod q for any x < 2^64
__device__ __forceinline__ u64 reduce64(u64 x, u64 q, u64 bar)
{
    return csub(x - __umul64hi(x, bar) * q, q);
}

// (lo, hi) += a * b  (128-bit accumulate)
__device__ __forceinline__ void mac128(u64 &lo, u64 &hi, u64 a, u64 b)
{
    asm("mad.lo.cc.u64 %0, %2, %3, %0;\n\t"
        "madc.hi.u64 %1, %2, %3, %1;"
        : "+l"(lo), "+l"(hi)
        : "l"(a), "l"(b));
}

__device__ __forceinline__ u64 reduce128(u64 lo, u64 hi, const ModC &m)
{
    u64 t1 = shoup_lazy(hi, m.r64, m.r64s, m.q);
    u64 t2 = lo - __umul64hi(lo, m.bar) * m.q;
    u64 r = t1 + t2;  // < 4q < 2^64
    r = csub(r, 2 * m.q);
    return csub(r, m.q);
}

__device__ __forceinline__ u64 mulmod(u64 a, u64 b, const ModC &m)
{
    return reduce128(a * b, __umul64hi(a, b), m);
}

__device__ __forceinline__ u64 addmod(u64 a, u64 b, u64 q) { return csub(a + b, q); }
__device__ __forceinline__ u64 submod(u64 a, u64 b, u64 q) { return csub(a + q - b, q); }

__device__ __forceinline__ ModC load_mod(const ModC *mods, u32 i)
{
    ModC m;
    const ulonglong2 *p = reinterpret_cast<const ulonglong2 *>(mods + i);
    ulonglong2 a = __ldg(p), b = __ldg(p + 1);
    m.q = a.x; m.r64 = a.y; m.r64s = b.x; m.bar = b.y;
    return m;
}

// ---- multiply-accumulate of many 64x64-bit products -----------------------------------------
// Acc128: generic 128-bit accumulator (mad.lo.cc / madc.hi), any residues < 2^64.
struct Acc128 {
    u64 lo = 0, hi = 0;
    __device__ __forceinline__ void mac(u64 a, u64 b) { mac128(lo, hi, a, b); }
    __device__ __forceinline__ u64 reduce(const ModC &m) const { return reduce128(lo, hi, m); }
    __device__ __forceinline__ void fold(const ModC &m) { lo = reduce(m); hi = 0; }
};
// How many products of residues mod q (each <= (q-1)^2 < 2^(2b), b = bits(q)) an Acc128 that
// already holds a value < q can absorb without wrapping 2^128: 2^(128-2b) - 1 terms
// (255 for a 60-bit prime; 2^(128-2b) - 1 >= 15 for every q < 2^62).
__host__ __device__ __forceinline__ u32 acc128_fold_terms(u64 q)
{
    int b = 0;
    while (b < 64 && (q >> b)) ++b;
    const int e = 128 - 2 * b;
    return e >= 32 ? 0xffffffffu : (u32)((1ull << e) - 1);
}

// Acc40: residues a, b < 2^40 (40-bit primes), at most MAX_TERMS = 2^15 terms (the middle word
// c gains < 2^41 + 2^48 per term and must stay below 2^64).  With a = a0 + a1 2^32,
// b = b0 + b1 2^32 (a1, b1 < 2^8):  a b = a0 b0 + (a0 b1 + a1 b0) 2^32 + a1 b1 2^64.
//   s0 (96 bits) += a0 b0          -- one IMAD.WIDE.U32 + add-with-carry on the ALU pipe
//   c  (64 bits) += a0 b1 + a1 b0  -- two IMAD.WIDE.U32 with 64-bit addend (< 2^41 per term)
//   c_hi         += a1 b1          -- one 32-bit IMAD (the 2^64 term, as 2^32 * c_hi)
// i.e. 3 wide + 1 narrow multiplies instead of the generic 4-wide 64x64 product + carries.
struct Acc40 {
    static constexpr u32 MAX_TERMS = 1u << 15;
    u64 s0 = 0, c = 0;
    u32 s0h = 0;
    __device__ __forceinline__ void mac(u64 a, u64 b)
    {
        const u32 a0 = (u32)a, a1 = (u32)(a >> 32), b0 = (u32)b, b1 = (u32)(b >> 32);
        const u64 p = (u64)a0 * b0;
        asm("add.cc.u64 %0, %0, %2;\n\taddc.u32 %1, %1, 0;" : "+l"(s0), "+r"(s0h) : "l"(p));
        c += (u64)a0 * b1;
        c += (u64)a1 * b0;
        c += (u64)(a1 * b1) << 32;
    }
    __device__ __forceinline__ u64 reduce(const ModC &m) const
    {
        // value = s0h 2^64 + s0 + c 2^32
        u64 lo = s0, hi = s0h;
        const u64 cl = c << 32, ch = c >> 32;
        asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;" : "+l"(lo), "+l"(hi) : "l"(cl), "l"(ch));
        return reduce128(lo, hi, m);
    }
    __device__ __forceinline__ void fold(const ModC &m)
    {
        s0 = reduce(m);
        c = 0;
        s0h = 0;
    }
};
