// fp64_bfly.cu -- microbenchmark: NTT butterflies on the FP64 pipe vs the integer pipe.
//
// For q < 2^50 a modular product is exact in IEEE double with an FMA two-product:
//   h = y*w, l = fma(y, w, -h)              (y*w = h + l exactly)
//   c = fma(y, w', C) - C,  w' = w/q        (nearest integer to y*w/q; C = 1.5 * 2^52)
//   r = fma(-c, q, h) + l                   (exact integer, |r| < q)
// so a lazy butterfly (x + r, x - r) is 8 FP64 instructions with no compare/select; values
// grow by < q per stage and stay exact far below 2^53.  This measures its throughput
// against the 64-bit Shoup butterfly (int_peak.cu's k_bfly) and a mix of both in one warp.
// Standalone: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_bfly fp64_bfly.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

typedef uint64_t u64;

__device__ __forceinline__ double mulmod_f64(double y, double w, double wq, double q)
{
    const double C = 6755399441055744.0;  // 1.5 * 2^52
    const double h = y * w;
    const double l = fma(y, w, -h);
    const double c = fma(y, wq, C) - C;
    return fma(-c, q, h) + l;
}

__global__ void __launch_bounds__(256) k_bfly_int(u64 *out, u64 q, u64 w, u64 ws, int iters)
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

// 3 radix-2 stages per iteration on 8 register values; values re-centred once per iteration
// (in a real NTT: once per kernel) to keep the microbenchmark's growth bounded.
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

// one warp in two runs the integer butterfly, the other the FP64 one (pipes in parallel)
__global__ void __launch_bounds__(256) k_bfly_mix(u64 *out, u64 q, u64 w, u64 ws, double wq, double qinv, int iters)
{
    if ((threadIdx.x >> 5) & 1) {
        double v[8];
        const double qd = (double)q, wd = (double)w;
        for (int i = 0; i < 8; ++i) v[i] = (double)((threadIdx.x * 8 + i + blockIdx.x) % 1000003);
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int s = 0; s < 3; ++s) {
                const int bit = 1 << s;
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    if (!(i & bit)) {
                        const double t = mulmod_f64(v[i | bit], wd, wq, qd);
                        const double x = v[i];
                        v[i] = x + t;
                        v[i | bit] = x - t;
                    }
            }
            if ((it & 7) == 7) {
#pragma unroll
                for (int i = 0; i < 8; ++i) v[i] = fma(-rint(v[i] * qinv), qd, v[i]);
            }
        }
        double acc = 0;
        for (int i = 0; i < 8; ++i) acc += v[i];
        out[blockIdx.x * blockDim.x + threadIdx.x] = (u64)acc;
    } else {
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
}

// exactness check of mulmod_f64 against __int128 on random operands (|y| < 64 q, w < q)
__global__ void k_check(int *bad, u64 q, u64 seed, int n)
{
    const double qd = (double)q;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        u64 s = seed ^ (0x9e3779b97f4a7c15ull * (u64)(i + 1));
        s ^= s >> 31;
        s *= 0xbf58476d1ce4e5b9ull;
        s ^= s >> 27;
        const u64 w = s % q;
        s *= 0x94d049bb133111ebull;
        s ^= s >> 29;
        const long long y = (long long)(s % (64 * q)) - 32 * (long long)q;
        const double r = mulmod_f64((double)y, (double)w, (double)w / qd, qd);
        __int128 e = ((__int128)y * (__int128)w) % (__int128)q;
        if (e < 0) e += q;
        long long rr = (long long)r;
        if (!(r > -qd && r < qd) || r != (double)rr) {
            atomicAdd(bad, 1);
            continue;
        }
        long long m = rr % (long long)q;
        if (m < 0) m += q;
        if ((__int128)m != e) atomicAdd(bad, 1);
    }
}

template <class F>
static double time_ms(F f)
{
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
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
    return best;
}

int main()
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, threads = 256, iters = 4096;
    u64 *buf;
    cudaMalloc(&buf, (size_t)blocks * threads * 8);
    int *bad;
    cudaMalloc(&bad, sizeof(int));
    const u64 qs[3] = {1099510054913ull, (1ull << 49) - 16383 /* not prime; arithmetic only */, 1152921504606830593ull};
    for (int k = 0; k < 2; ++k) {
        cudaMemset(bad, 0, sizeof(int));
        k_check<<<sms * 4, 256>>>(bad, qs[k], 1234 + k, 1 << 24);
        int h = 0;
        cudaMemcpy(&h, bad, sizeof(int), cudaMemcpyDeviceToHost);
        printf("mulmod_f64 exactness q=%llu (%d bits): %d bad of %d\n", (unsigned long long)qs[k],
               (int)std::log2((double)qs[k]) + 1, h, 1 << 24);
    }
    const u64 q = qs[0], w = 123456789ull, ws = (u64)(((unsigned __int128)w << 64) / q);
    const double qd = (double)q, wq = (double)w / qd, qinv = 1.0 / qd;
    const double nb = (double)blocks * threads * iters * 12.0;
    double ms = time_ms([&] { k_bfly_int<<<blocks, threads>>>(buf, q, w, ws, iters); });
    printf("int64 Shoup butterfly : %8.1f Gbfly/s\n", nb / (ms * 1e-3) / 1e9);
    ms = time_ms([&] { k_bfly_f64<<<blocks, threads>>>((double *)buf, qd, (double)w, wq, qinv, iters); });
    printf("fp64 FMA butterfly    : %8.1f Gbfly/s\n", nb / (ms * 1e-3) / 1e9);
    ms = time_ms([&] { k_bfly_mix<<<blocks, threads>>>(buf, q, w, ws, wq, qinv, iters); });
    printf("half/half mix         : %8.1f Gbfly/s\n", nb / (ms * 1e-3) / 1e9);
    cudaError_t e = cudaGetLastError();
    printf("cuda: %s\n", cudaGetErrorString(e));
    return 0;
}
