// int_peak.cu -- measured integer roofline for the hot path's arithmetic on this B200.
//
// MEASURED_PEAKS.json carries HBM and bf16 tensor peaks only; the NTT-bearing kernels are
// bound by 64-bit modular arithmetic on the integer pipes.  This measures, with no memory
// traffic at all, the throughput of exactly the two primitives the kernels are built from:
//   * the Harvey/Shoup lazy butterfly (ntt.cuh ct_stages): x' = x mod 2q, t = W*y - hi(W'*y)*q,
//     (x'+t, x'-t+2q)  -- 64-bit, 2 mul.lo + 1 mul.hi + compare/select/add
//   * the 128-bit multiply-accumulate of the key-switch inner product (mad.lo.cc/madc.hi)
// plus a raw 32-bit IMAD rate for reference, and the FP64-pipe butterfly the NTT uses for
// q < 2^42 (ntt.cuh FP64 mode).  Each thread keeps 8 independent chains in
// registers; grids fill all 148 SMs.  The figures are the "peak" of bench.py's ALU roofline.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

typedef uint64_t u64;

__global__ void __launch_bounds__(256) k_bfly(u64 *out, u64 q, u64 w, u64 ws, int iters)
{
    u64 v[8];
    for (int i = 0; i < 8; ++i) v[i] = (threadIdx.x * 8 + i + blockIdx.x) % q;
    const u64 q2 = 2 * q;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int s = 0; s < 3; ++s) {
            const int bit = 1 << s;
#pragma unroll
            for (int i = 0; i < 8; ++i)
                if (!(i & bit)) {
                    u64 x = v[i] >= q2 ? v[i] - q2 : v[i];
                    u64 t = v[i | bit] * w - __umul64hi(v[i | bit], ws) * q;
                    v[i] = x + t;
                    v[i | bit] = x - t + q2;
                }
        }
    }
    u64 acc = 0;
    for (int i = 0; i < 8; ++i) acc ^= v[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// the FP64-pipe butterfly of ntt.cuh's FP64 mode (q < 2^42): exact FMA two-product modular
// product, lazy signed values (see bench/fp64_bfly.cu for its exactness check)
__device__ __forceinline__ double mulmod_f64(double y, double w, double wq, double q)
{
    const double C = 6755399441055744.0;
    const double h = y * w;
    const double l = fma(y, w, -h);
    const double c = fma(y, wq, C) - C;
    return fma(-c, q, h) + l;
}

__global__ void __launch_bounds__(256) k_bfly_f64(double *out, double q, double w, double wq, double qinv, int iters)
{
    double v[8];
    for (int i = 0; i < 8; ++i) v[i] = (double)((threadIdx.x * 8 + i + blockIdx.x) % 1000003);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int s = 0; s < 3; ++s) {
            const int bit = 1 << s;
#pragma unroll
            for (int i = 0; i < 8; ++i)
                if (!(i & bit)) {
                    const double t = mulmod_f64(v[i | bit], w, wq, q);
                    const double x = v[i];
                    v[i] = x + t;
                    v[i | bit] = x - t;
                }
        }
        if ((it & 7) == 7) {
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = fma(-rint(v[i] * qinv), q, v[i]);
        }
    }
    double acc = 0;
    for (int i = 0; i < 8; ++i) acc += v[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// the FP64-pipe modular multiply-accumulate of kernels.cu's FP64 inner product (ks_mac CLS 5):
// acc += v k - round(v k / q) q, exact two-product, 7 FP64 operations per MAC
__global__ void __launch_bounds__(256) k_fmac(double *out, double q, double qinv, int iters)
{
    const double C = 6755399441055744.0;
    double v[8], acc[8];
    for (int i = 0; i < 8; ++i) {
        v[i] = (double)((threadIdx.x * 8 + i + blockIdx.x) % 1000003);
        acc[i] = 0.0;
    }
    double k = 987654321.0 + blockIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const double h = v[i] * k;
            const double l = fma(v[i], k, -h);
            const double c = fma(h, qinv, C) - C;
            acc[i] += fma(-c, q, h) + l;
        }
        k += 1.0;
        if ((it & 63) == 63) {
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] = fma(-rint(acc[i] * qinv), q, acc[i]);
        }
    }
    double a = 0;
    for (int i = 0; i < 8; ++i) a += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = a;
}

__global__ void __launch_bounds__(256) k_mac(u64 *out, u64 a0, int iters)
{
    u64 lo[8], hi[8], a[8];
    for (int i = 0; i < 8; ++i) {
        lo[i] = hi[i] = 0;
        a[i] = a0 + threadIdx.x * 8 + i;
    }
    u64 b = a0 ^ blockIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mad.lo.cc.u64 %0, %2, %3, %0;\n\tmadc.hi.u64 %1, %2, %3, %1;"
                         : "+l"(lo[i]), "+l"(hi[i])
                         : "l"(a[i]), "l"(b));
        b += 0x9e3779b97f4a7c15ull;
    }
    u64 acc = 0;
    for (int i = 0; i < 8; ++i) acc ^= lo[i] ^ hi[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void __launch_bounds__(256) k_imad(unsigned *out, unsigned a, int iters)
{
    unsigned v[8];
    for (int i = 0; i < 8; ++i) v[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = v[i] * a + (unsigned)i;
    }
    unsigned acc = 0;
    for (int i = 0; i < 8; ++i) acc ^= v[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <class F>
static double time_ms(F f)
{
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();  // warm-up
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a);
        f();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return best;
}

// out[0] = butterflies/s (64-bit Shoup, integer pipe), out[1] = 128-bit MACs/s,
// out[2] = 32-bit IMADs/s, out[3] = SMs, out[4] = butterflies/s on the FP64 pipe (q < 2^42),
// out[5] = modular multiply-accumulates/s on the FP64 pipe
extern "C" int int_peak(double *out)
{
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int blocks = sms * 8, threads = 256, iters = 4096;
    u64 *buf;
    if (cudaMalloc(&buf, (size_t)blocks * threads * 8) != cudaSuccess) return -1;
    const u64 q = 1099510054913ull, w = 123456789ull, ws = (u64)(((unsigned __int128)w << 64) / q);
    double ms = time_ms([&] { k_bfly<<<blocks, threads>>>(buf, q, w, ws, iters); });
    out[0] = (double)blocks * threads * iters * 12.0 / (ms * 1e-3);
    ms = time_ms([&] { k_mac<<<blocks, threads>>>(buf, 0x123456789abcdefull, iters); });
    out[1] = (double)blocks * threads * iters * 8.0 / (ms * 1e-3);
    ms = time_ms([&] { k_imad<<<blocks, threads>>>((unsigned *)buf, 2654435761u, iters * 4); });
    out[2] = (double)blocks * threads * iters * 4 * 8.0 / (ms * 1e-3);
    out[3] = sms;
    {
        const double qd = (double)q;
        ms = time_ms([&] { k_bfly_f64<<<blocks, threads>>>((double *)buf, qd, (double)w, (double)w / qd, 1.0 / qd, iters); });
        out[4] = (double)blocks * threads * iters * 12.0 / (ms * 1e-3);
        ms = time_ms([&] { k_fmac<<<blocks, threads>>>((double *)buf, qd, 1.0 / qd, iters); });
        out[5] = (double)blocks * threads * iters * 8.0 / (ms * 1e-3);
    }
    cudaFree(buf);
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

int main()
{
    double o[6];
    if (int_peak(o)) return 1;
    printf("{\"bfly_per_s\": %.4e, \"mac128_per_s\": %.4e, \"imad32_per_s\": %.4e, \"sms\": %d, "
           "\"fbfly_per_s\": %.4e, \"fmac_per_s\": %.4e}\n", o[0], o[1], o[2], (int)o[3], o[4], o[5]);
    return 0;
}
