// ks_fused.cu -- key-switch ModUp + inner product fused in one kernel for N = 2^13 (the PrivFT
// inference configuration), FP64-mode targets (q_t < 2^42).
//
// The generic path (kernels.cu) runs ModUp's forward NTT of every digit in two kernels
// (column phase -> L2/HBM intermediate I -> row phase inside ks_mac).  At N = 2^13 a whole
// limb is 64 KB, so one CTA of 1024 threads holds it: per (ciphertext, target t) the CTA
// loops over the digits j, lifts D_j mod q_t, runs all 13 NTT stages in registers and one
// shared-memory buffer (radix-8 rounds of ntt.cuh's FP64 stages, block-wide exchanges), and
// multiply-accumulates with the key rows in shared memory -- no intermediate leaves the SM.
// Digit j == t is the ciphertext's own NTT-form limb (with the Galois gather for rotations).
// Result: ext[c][0|1][t] = sum_j NTT_t(D_j) * key_{j,b|a,t}, canonical; identical to ks_mac.
#include <cstdlib>

#include "internal.h"

namespace {

constexpr int F13_LOGN = 13, F13_N = 1 << F13_LOGN, F13_THREADS = F13_N / 8;
constexpr int F13_PAD = F13_N + F13_N / 16;

// block-wide exchange: the 8 values of each thread stored under ownership `from`, reloaded under `to`
struct BlockEx {
    double *s;
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

// y * w mod q for two data operands (no precomputed w/q): |y| < 2^47, w < q < 2^42, |r| < 1.5q
__device__ __forceinline__ double f64_mulmod_dd(double y, double w, double q, double qinv)
{
    const double h = y * w;
    const double l = fma(y, w, -h);
    const double c = fma(h, qinv, F64_C) - F64_C;
    return fma(-c, q, h) + l;
}

struct FusedArgs {
    const u64 *D;  // digits (coefficient form), layout as TaskModUpCol
    PolyMap din;   // NTT-form polynomial being switched (one per ciphertext)
    const u32 *perm;
    const u64 *key;
    u64 *ext;
    u32 Lk, l, t0, T, sp, dw, dcnt, c0;
};

__global__ void __launch_bounds__(F13_THREADS, 1) k_ks_fused13(FusedArgs a, Tables tb)
{
    extern __shared__ double sm13[];  // [F13_PAD] exchange | [F13_N] acc b | [F13_N] acc a
    double *sx = sm13, *accb = sm13 + F13_PAD, *acca = accb + F13_N;
    const u32 cr = blockIdx.x, tl = cr % a.T, c = cr / a.T, t = a.t0 + tl;
    const u32 prime = (t < a.l) ? t : a.sp, klimb = (t < a.l) ? t : a.Lk;
    const int lt = threadIdx.x;
    const double2 *twf = tb.psif + ((size_t)prime << F13_LOGN);
    const double2 qq = __ldg(twf);
    const double q = qq.x, qinv = qq.y;
    const ModC m = load_mod(tb.mod, prime);
    const BlockEx ex{sx};
    // accumulators element-major (acc[i][lt]) so each access is one conflict-free row
#pragma unroll
    for (int i = 0; i < 8; ++i) accb[i * F13_THREADS + lt] = acca[i * F13_THREADS + lt] = 0.0;
    for (u32 j = 0; j < a.l; ++j) {
        double v[8];
        if (j == t) {
            const u64 *dp = a.din.base + (((size_t)c * a.din.cap + t) << F13_LOGN);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const u32 li = 8 * lt + i;
                v[i] = u2d(a.perm ? dp[__ldg(a.perm + li)] : dp[li]);
            }
        } else {
            const u64 *src = a.D + ((((size_t)(j / a.dw) * a.dcnt + a.c0 + c) * a.dw + j % a.dw) << F13_LOGN);
            const bool red = !use_f64(tb, tb.mod[j].q);  // 60-bit source: reduce mod q_t first
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const u64 x = src[(i << (F13_LOGN - 3)) | lt];
                v[i] = u2d(red ? reduce64(x, m.q, m.bar) : x);
            }
            fwd_rounds_f64<F13_LOGN, 0>(v, ex, lt, 0, 0u, twf, q);  // leaves li = 8 lt + i
        }
        const u64 *kb = a.key + (((size_t)(2 * j) * (a.Lk + 1) + klimb) << F13_LOGN) + 8 * lt;
        const u64 *ka = kb + ((size_t)(a.Lk + 1) << F13_LOGN);
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            const ulonglong2 xb = __ldg(reinterpret_cast<const ulonglong2 *>(kb) + h);
            const ulonglong2 xa = __ldg(reinterpret_cast<const ulonglong2 *>(ka) + h);
            accb[(2 * h) * F13_THREADS + lt] += f64_mulmod_dd(v[2 * h], u2d(xb.x), q, qinv);
            accb[(2 * h + 1) * F13_THREADS + lt] += f64_mulmod_dd(v[2 * h + 1], u2d(xb.y), q, qinv);
            acca[(2 * h) * F13_THREADS + lt] += f64_mulmod_dd(v[2 * h], u2d(xa.x), q, qinv);
            acca[(2 * h + 1) * F13_THREADS + lt] += f64_mulmod_dd(v[2 * h + 1], u2d(xa.y), q, qinv);
        }
    }
    u64 *e0 = a.ext + (((size_t)c * 2 * (a.l + 1) + t) << F13_LOGN) + 8 * lt;
    u64 *e1 = e0 + ((size_t)(a.l + 1) << F13_LOGN);
#pragma unroll
    for (int h = 0; h < 4; ++h) {
        const int i0 = 2 * h * F13_THREADS + lt, i1 = i0 + F13_THREADS;
        reinterpret_cast<ulonglong2 *>(e0)[h] = make_ulonglong2(f64_canon(accb[i0], q, qinv), f64_canon(accb[i1], q, qinv));
        reinterpret_cast<ulonglong2 *>(e1)[h] = make_ulonglong2(f64_canon(acca[i0], q, qinv), f64_canon(acca[i1], q, qinv));
    }
}

}  // namespace

bool ks_fused_ok(const Launch &L, u32 prime)
{
    // opt-in (CKKS_KS_FUSED=1): one 1024-thread CTA per SM leaves the load and barrier latency
    // exposed -- measured 123 ms/step vs 97 ms for the two-kernel path on the same targets
    const char *e = std::getenv("CKKS_KS_FUSED");
    return e && e[0] == '1' && L.tb->log_n == F13_LOGN && L.hprimes[prime] < L.tb->f64_qmax;
}

void launch_ks_fused(const Launch &L, const u64 *D, u32 dw, u32 dcnt, u32 c0, PolyMap din, const u32 *perm,
                     const u64 *key, u32 Lk, u32 l, u32 cnt, u32 t0, u32 T, u64 *ext, u32 sp)
{
    static bool attr = false;
    const size_t smem = (size_t)(F13_PAD + 2 * F13_N) * sizeof(double);
    if (!attr) {
        cudaFuncSetAttribute(k_ks_fused13, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    const FusedArgs a{D, din, perm, key, ext, Lk, l, t0, T, sp, dw, dcnt, c0};
    u32 diag = 0;
    for (u32 tl = 0; tl < T; ++tl) diag += (t0 + tl < l) ? 1 : 0;
    const double n = (double)F13_N, ntts = (double)cnt * ((double)T * l - diag);
    const double bytes = 8.0 * n * ((double)cnt * T * l + 2.0 * T * l + 2.0 * cnt * T);
    KLAUNCH(L, "ks_fused", (Work{0, 2.0 * cnt * T * l * n, bytes, ntts * n / 2 * F13_LOGN}),
            (k_ks_fused13<<<cnt * T, F13_THREADS, smem, L.st>>>(a, *L.tb)));
}
