// bcast13.cu -- the broadcast step of ModDown and RESCALE fused into one kernel for N = 2^13
// (the PrivFT inference ring).
//
// Both steps compute, for every target limb t of a polynomial,
//     out_t = [base_t] + [acc_t] + (x_t - NTT_t([X]_{q_t})) * C_t   with X = INTT_s(src)
// (ModDown, reading A7: src = the special-prime limb of the inner-product accumulator, C_t =
// P^{-1} mod q_t; RESCALE, Eq. (1): src = the ciphertext's last limb, C_t = q_{l-1}^{-1}).
// The generic path runs this as four launches (inverse rows, inverse columns, broadcast
// columns, rows + epilogue) with two HBM round trips of intermediates.  At N = 2^13 a limb is
// 64 KB, so one CTA of 1024 threads holds it: the inverse transform of src runs once, X stays
// in shared memory, and each target's forward transform + epilogue follows in place (all 13
// stages per tile, ntt.cuh radix-8 rounds with block-wide exchanges).  The inverse leaves
// thread lt holding X at positions (i << 10) | lt, which is exactly the forward transform's
// first ownership, and the forward output (8 lt + i) gives 64 contiguous bytes per thread for
// the epilogue's loads and stores.  Results are identical to the generic path.
//
// Opt-in (CKKS_BCAST13=1): measured 152 ms/step at C4 against 112 ms for the four kernels it
// replaces -- one 1024-thread CTA per SM (64-register cap, spills) with 20 block barriers per
// polynomial leaves the pipes idle more than the saved intermediate traffic buys back.
#include <cstdlib>

#include "internal.h"

namespace {

constexpr int B13 = 13, N13 = 1 << B13, T13 = N13 / 8;  // 1024 threads, 8 values each
constexpr int PAD13 = N13 + N13 / 16;

__device__ __forceinline__ const u64 *limb_ptr(const PolyMap &m, u32 p, u32 i, u32 log_n)
{
    return m.base + (((size_t)p * m.cap + i) << log_n);
}
__device__ __forceinline__ u64 *limb_ptr_w(const PolyMap &m, u32 p, u32 i, u32 log_n)
{
    return m.base + (((size_t)p * m.cap + i) << log_n);
}

// block-wide exchange: values stored under ownership `from`, reloaded under `to`
struct BlockEx13 {
    u64 *s;
    __device__ __forceinline__ static int pad(int x) { return x + (x >> 4); }
    template <class T>
    __device__ __forceinline__ void operator()(T v[8], int lt, int from, int to) const
    {
        T *st = reinterpret_cast<T *>(s);
        __syncthreads();
#pragma unroll
        for (int i = 0; i < 8; ++i) st[pad(lidx(lt, i, from))] = v[i];
        __syncthreads();
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = st[pad(lidx(lt, i, to))];
    }
};

struct Bcast13Args {
    const u64 *src;  // NTT-form limb of poly p at src + ((p * src_stride) << 13)
    u32 src_stride, src_prime;
    u32 nt, toff;    // targets toff .. toff + nt - 1 (prime index = limb index)
    PolyMap x, out, base, acc;
    const u32 *base_perm;
    int base_c0_only;
    const ulonglong2 *consts;  // per target prime index: (C_t, Shoup companion)
};

__global__ void __launch_bounds__(T13, 1) k_bcast13(Bcast13Args a, Tables tb)
{
    extern __shared__ __align__(16) u64 sm13b[];  // [PAD13] exchange | [N13] X (coefficient form)
    u64 *Xs = sm13b + PAD13;
    const u32 p = blockIdx.x;
    const int lt = threadIdx.x;
    const BlockEx13 ex{sm13b};
    {  // X = INTT_s(src): thread lt loads its 8 contiguous NTT-domain words
        const ModC ms = load_mod(tb.mod, a.src_prime);
        const u64 *sp = a.src + (((size_t)p * a.src_stride) << B13) + 8 * lt;
        u64 v[8];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            const ulonglong2 w = *reinterpret_cast<const ulonglong2 *>(sp + 2 * h);
            v[2 * h] = w.x;
            v[2 * h + 1] = w.y;
        }
        inv_rounds<B13, 0>(v, ex, lt, 0, 0u, tb.ipsi + ((size_t)a.src_prime << B13), ms.q, 0,
                           tb.ipsif + ((size_t)a.src_prime << B13), use_f64(tb, ms.q));
        const ulonglong2 ni = __ldg(tb.ninv + a.src_prime);
#pragma unroll
        for (int i = 0; i < 8; ++i) Xs[(i << 10) | lt] = shoup(v[i], ni.x, ni.y, ms.q);  // own slots only
    }
    const bool base_here = a.base.base != nullptr && (!a.base_c0_only || (p & 1) == 0);
    for (u32 tt = 0; tt < a.nt; ++tt) {
        const u32 t = a.toff + tt;
        const ModC m = load_mod(tb.mod, t);
        const bool f64 = use_f64(tb, m.q);
        u64 y[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) y[i] = reduce64(Xs[(i << 10) | lt], m.q, m.bar);
        fwd_rounds<B13, 0>(y, ex, lt, 0, 0u, tb.psi + ((size_t)t << B13), m.q, tb.psif + ((size_t)t << B13), f64);
        const u32 e0 = 8 * lt;  // epilogue: this thread's 8 contiguous NTT-domain words
        const ulonglong2 cst = __ldg(a.consts + t);
        const u64 *xp = limb_ptr(a.x, p, t, B13) + e0;
        u64 o[8];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            const ulonglong2 w = *reinterpret_cast<const ulonglong2 *>(xp + 2 * h);
            o[2 * h] = shoup(w.x + m.q - fwd_canon<B13>(y[2 * h], m, f64), cst.x, cst.y, m.q);
            o[2 * h + 1] = shoup(w.y + m.q - fwd_canon<B13>(y[2 * h + 1], m, f64), cst.x, cst.y, m.q);
        }
        if (base_here) {
            const u64 *bp = limb_ptr(a.base, p, t, B13);
            if (a.base_perm) {
#pragma unroll
                for (int i = 0; i < 8; ++i) o[i] = addmod(o[i], bp[__ldg(a.base_perm + e0 + i)], m.q);
            } else {
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const ulonglong2 w = *reinterpret_cast<const ulonglong2 *>(bp + e0 + 2 * h);
                    o[2 * h] = addmod(o[2 * h], w.x, m.q);
                    o[2 * h + 1] = addmod(o[2 * h + 1], w.y, m.q);
                }
            }
        }
        if (a.acc.base != nullptr) {
            const u64 *ap = limb_ptr(a.acc, p, t, B13) + e0;
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                const ulonglong2 w = *reinterpret_cast<const ulonglong2 *>(ap + 2 * h);
                o[2 * h] = addmod(o[2 * h], w.x, m.q);
                o[2 * h + 1] = addmod(o[2 * h + 1], w.y, m.q);
            }
        }
        u64 *op = limb_ptr_w(a.out, p, t, B13) + e0;
#pragma unroll
        for (int h = 0; h < 4; ++h) reinterpret_cast<ulonglong2 *>(op)[h] = make_ulonglong2(o[2 * h], o[2 * h + 1]);
    }
}

}  // namespace

bool bcast13_ok(const Launch &L)
{
    const char *e = std::getenv("CKKS_BCAST13");
    return L.tb->log_n == B13 && e && e[0] == '1';
}

void launch_bcast13(const Launch &L, const u64 *src, u32 src_stride, u32 src_prime, u32 npolys, u32 nt, u32 toff,
                    PolyMap x, PolyMap out, const ulonglong2 *consts, PolyMap base, const u32 *base_perm,
                    bool base_c0_only, PolyMap acc)
{
    if (!npolys || !nt) return;
    static bool attr = false;
    const size_t smem = (size_t)(PAD13 + N13) * sizeof(u64);
    if (!attr) {
        cudaFuncSetAttribute(k_bcast13, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    const Bcast13Args a{src, src_stride, src_prime, nt, toff, x, out, base, acc, base_perm, base_c0_only ? 1 : 0, consts};
    double f = 0;
    for (u32 t = toff; t < toff + nt; ++t) f += (L.hprimes[t] < L.tb->f64_qmax) ? 1 : 0;
    const double nh = (double)npolys * (N13 / 2) * B13;
    const bool sf64 = L.hprimes[src_prime] < L.tb->f64_qmax;
    Work w{nh * ((sf64 ? 0 : 1) + (nt - f)), (double)npolys * nt * N13, 8.0 * N13 * npolys * (1 + 4.0 * nt),
           nh * ((sf64 ? 1 : 0) + f)};
    KLAUNCH(L, "bcast13", w, (k_bcast13<<<npolys, T13, smem, L.st>>>(a, *L.tb)));
}
