// codec.cu -- batched GPU encode / decode (PAPER.md P:140 ENCODE,
// P:143 DECODE, "the client encodes and encrypts").
//
// The canonical embedding is one length-N complex DFT per plaintext (fp64), run as a
// four-step FFT N = N1 * N2 with N1 = 2^floor(log_n/2), N2 = N / N1 (both <= 256):
//   pass A: N2 column FFTs of length N1 over x[N2*n1 + n2], times W_N^{n2*k1}  -> Y[k1][n2]
//   pass B: N1 row FFTs of length N2 over Y[k1][.]                           -> X[k1 + N1*k2]
// Each CTA owns 16 lines (16 x 16 B = one 256-B segment per element row) staged in
// shared memory; every global access is coalesced.  The method's own steps are fused into
// the pass boundaries so each plaintext crosses HBM the minimum number of times:
//   encode: slot scatter B[(r_j-1)/2] = Delta z_j, B[N-1-(r_j-1)/2] = conj(...)  -> pass A load
//           m_k = round(Re(X_k e^{-i pi k/N}) / N), residues mod q_0..q_{l-1}      -> pass B store
//   decode: CRT lift to the centred integer (exact mod 2^128, reading A33), times e^{+i pi k/N}
//                                                                                  -> pass A load
//           slot gather z_j = X_{(r_j-1)/2} / Delta                                -> pass B store
// The NTT <-> coefficient conversions run in the existing NTT kernels (ckks.cu).
#include <cmath>

#include "internal.h"

namespace {

constexpr int FFT_LINES = 16;
constexpr int FFT_THREADS = 256;

__device__ __forceinline__ double2 cmul(double2 a, double2 b)
{
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

// W_N^m for the transform's sign (table holds e^{-2 pi i m / N})
__device__ __forceinline__ double2 wpow(const double2 *w, u32 m, u32 log_n, int sign)
{
    const double2 v = w[m & ((1u << log_n) - 1)];
    return sign > 0 ? make_double2(v.x, -v.y) : v;
}

// One pass of the four-step FFT.  PASS_A: line = column n2, element = n1, and the
// output is twiddled by W_N^{n2 k1}.  Element (line, e) is read from index
//   PASS_A: (e << (log_n - log_m)) + line      PASS_B: (line << log_m) + e
// and result (line, k) is written to index (k << (log_n - log_m)) + line in both passes.
template <bool PASS_A, class Ld, class St>
__global__ void __launch_bounds__(FFT_THREADS) k_fft_pass(Ld ld, St st, const double2 *w, u32 log_n, u32 log_m,
                                                         int sign, u32 groups)
{
    extern __shared__ double2 sm[];  // [FFT_LINES][M + 1] (one pad element per line: no bank aliasing)
    const u32 M = 1u << log_m, ld_m = M + 1, sh = log_n - log_m;
    const u32 b = blockIdx.x / groups, line0 = (blockIdx.x % groups) * FFT_LINES;
    const u32 per = (u32)FFT_LINES << log_m;
    for (u32 idx = threadIdx.x; idx < per; idx += FFT_THREADS) {
        u32 t, e;
        if (PASS_A) {
            t = idx & (FFT_LINES - 1);
            e = idx >> 4;
        } else {
            t = idx >> log_m;
            e = idx & (M - 1);
        }
        const u32 line = line0 + t;
        const u32 k = PASS_A ? ((e << sh) + line) : ((line << log_m) + e);
        sm[t * ld_m + (__brev(e) >> (32 - log_m))] = ld(b, k);  // bit-reversed: iterative DIT below
    }
    __syncthreads();
    for (u32 lh = 0; lh < log_m; ++lh) {
        const u32 h = 1u << lh;
        for (u32 idx = threadIdx.x; idx < per / 2; idx += FFT_THREADS) {
            const u32 t = idx >> (log_m - 1), j = idx & (M / 2 - 1);
            const u32 kk = j & (h - 1), i0 = ((j - kk) << 1) + kk;
            double2 *p = sm + t * ld_m;
            const double2 u = p[i0], v = cmul(p[i0 + h], wpow(w, kk << (log_n - lh - 1), log_n, sign));
            p[i0] = make_double2(u.x + v.x, u.y + v.y);
            p[i0 + h] = make_double2(u.x - v.x, u.y - v.y);
        }
        __syncthreads();
    }
    for (u32 idx = threadIdx.x; idx < per; idx += FFT_THREADS) {
        const u32 t = idx & (FFT_LINES - 1), k = idx >> 4, line = line0 + t;
        double2 v = sm[t * ld_m + k];
        if (PASS_A) v = cmul(v, wpow(w, line * k, log_n, sign));
        st(b, (k << sh) + line, v);
    }
}

struct YLd {
    const double2 *y;
    u32 log_n;
    __device__ double2 operator()(u32 b, u32 k) const { return y[((size_t)b << log_n) + k]; }
};
struct YSt {
    double2 *y;
    u32 log_n;
    __device__ void operator()(u32 b, u32 k, double2 v) const { y[((size_t)b << log_n) + k] = v; }
};

// slot[s] = j | (conj << 31): s = (r_j - 1)/2 (conj 0) or s = N - 1 - (r_j - 1)/2 (conj 1)
struct EncLd {
    const double2 *z;
    const u32 *slot;
    u32 n_slots;
    double scale;
    __device__ double2 operator()(u32 b, u32 s) const
    {
        const u32 v = __ldg(slot + s), j = v & 0x7fffffffu;
        if (j >= n_slots) return make_double2(0.0, 0.0);
        const double2 x = z[(size_t)b * n_slots + j];
        return make_double2(x.x * scale, (v >> 31) ? -x.y * scale : x.y * scale);
    }
};

// m_k = round_half_away(Re(X_k tw_k) / N) -> residues of the l limbs (reading A28)
struct EncSt {
    u64 *out;
    const double2 *tw;
    const ModC *mod;
    int *overflow;
    u32 cap, l, log_n;
    double inv_n;
    __device__ void operator()(u32 b, u32 k, double2 X) const
    {
        const double2 t = __ldg(tw + k);
        double m = fma(X.x, t.x, -X.y * t.y) * inv_n;
        if (!(fabs(m) < 9.2e18)) {  // int64 overflow: flag it, encode 0
            atomicOr(overflow, 1);
            m = 0.0;
        }
        const long long x = llround(m);
        const u64 ax = (u64)(x < 0 ? -x : x);
        u64 *o = out + (((size_t)b * cap) << log_n) + k;
        for (u32 i = 0; i < l; ++i) {
            const ModC q = mod[i];
            const u64 r = reduce64(ax, q.q, q.bar);
            o[(size_t)i << log_n] = (x < 0 && r) ? q.q - r : r;
        }
    }
};

// centred CRT lift of coefficient k (reading A33):
//   y_i = [c_i (Q/q_i)^{-1}]_{q_i},  u = rint(sum y_i / q_i),  x = sum y_i (Q/q_i) - u Q,
// with the sum taken exactly mod 2^128 (|x| < 2^127 for every decodable message), then
// b_k = x * e^{+i pi k/N}.
struct DecLd {
    const u64 *coef;  // [cnt][l][N] coefficient form
    const CrtConst *crt;
    const ModC *mod;
    const double2 *tw;
    u64 Q_lo, Q_hi;
    u32 l, log_n;
    __device__ double2 operator()(u32 b, u32 k) const
    {
        u64 lo = 0, hi = 0;
        double f = 0.0;
        const u64 *c = coef + (((size_t)b * l) << log_n) + k;
        for (u32 i = 0; i < l; ++i) {
            const CrtConst cc = crt[i];
            const u64 y = shoup(c[(size_t)i << log_n], cc.qhinv, cc.qhinv_s, mod[i].q);
            f = fma((double)y, cc.inv_q, f);
            const u64 plo = y * cc.qh_lo, phi = __umul64hi(y, cc.qh_lo) + y * cc.qh_hi;
            lo += plo;
            hi += phi + (lo < plo ? 1 : 0);
        }
        const u64 u = (u64)rint(f);
        const u64 ulo = u * Q_lo, uhi = __umul64hi(u, Q_lo) + u * Q_hi;
        const u64 nlo = lo - ulo;
        hi = hi - uhi - (lo < ulo ? 1 : 0);
        lo = nlo;
        double x;
        if ((long long)hi < 0) {
            lo = ~lo + 1;
            hi = ~hi + (lo == 0 ? 1 : 0);
            x = -fma((double)hi, 18446744073709551616.0, (double)lo);
        } else {
            x = fma((double)hi, 18446744073709551616.0, (double)lo);
        }
        const double2 t = __ldg(tw + k);
        return make_double2(x * t.x, -x * t.y);
    }
};

struct DecSt {
    double2 *z;
    const u32 *slot;
    u32 n_slots;
    double inv_scale;
    __device__ void operator()(u32 b, u32 s, double2 X) const
    {
        const u32 v = __ldg(slot + s);
        if (v >> 31) return;
        if (v < n_slots) z[(size_t)b * n_slots + v] = make_double2(X.x * inv_scale, X.y * inv_scale);
    }
};

template <bool PASS_A, class Ld, class St>
void fft_pass(const Launch &L, const char *name, double bytes, const Ld &ld, const St &st, const double2 *w,
              u32 log_m, int sign, u32 cnt)
{
    const u32 log_n = L.tb->log_n;
    const u32 groups = (1u << (log_n - log_m)) / FFT_LINES;
    const size_t smem = (size_t)FFT_LINES * ((1u << log_m) + 1) * sizeof(double2);
    static bool attr = false;  // per instantiation
    if (!attr) {
        cudaFuncSetAttribute(k_fft_pass<PASS_A, Ld, St>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(FFT_LINES * 257 * sizeof(double2)));
        attr = true;
    }
    KLAUNCH(L, name, (Work{0, 0, bytes}),
            (k_fft_pass<PASS_A, Ld, St><<<cnt * groups, FFT_THREADS, smem, L.st>>>(ld, st, w, log_n, log_m, sign,
                                                                                   groups)));
}

}  // namespace

void launch_encode(const Launch &L, const CodecTabs &tb, const double2 *z, u32 n_slots, double scale, u32 cnt,
                   double2 *Y, PolyMap out, u32 l, int *overflow)
{
    const u32 log_n = L.tb->log_n, b1 = log_n / 2;
    const double n = (double)(1u << log_n);
    fft_pass<true>(L, "encode_fft_a", cnt * (16.0 * n_slots + 16.0 * n), EncLd{z, tb.slot, n_slots, scale},
                   YSt{Y, log_n}, tb.w, b1, -1, cnt);
    fft_pass<false>(L, "encode_fft_b", cnt * n * (16.0 + 8.0 * l), YLd{Y, log_n},
                    EncSt{out.base, tb.tw, L.tb->mod, overflow, out.cap, l, log_n, 1.0 / n}, tb.w, log_n - b1, -1,
                    cnt);
}

void launch_decode(const Launch &L, const CodecTabs &tb, const u64 *coef, u32 l, const CrtConst *crt, u64 Q_lo,
                   u64 Q_hi, u32 cnt, double2 *Y, double2 *z, u32 n_slots, double scale)
{
    const u32 log_n = L.tb->log_n, b1 = log_n / 2;
    const double n = (double)(1u << log_n);
    fft_pass<true>(L, "decode_fft_a", cnt * n * (8.0 * l + 16.0), DecLd{coef, crt, L.tb->mod, tb.tw, Q_lo, Q_hi, l, log_n},
                   YSt{Y, log_n}, tb.w, b1, +1, cnt);
    fft_pass<false>(L, "decode_fft_b", cnt * (16.0 * n + 16.0 * n_slots), YLd{Y, log_n},
                    DecSt{z, tb.slot, n_slots, 1.0 / scale}, tb.w, log_n - b1, +1, cnt);
}
