// mma_peak.cu -- microbenchmark: legacy mma.sync tensor-core throughput on sm_100a for the
// integer (u8 x u8 -> s32) and fp16 shapes, register-resident fragments, all SMs.
// Standalone: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_peak mma_peak.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) k_imma(int *out, int iters)
{
    unsigned a[4], b[2];
    int c[4][4] = {};
    for (int i = 0; i < 4; ++i) a[i] = 0x01020304u * (threadIdx.x + i);
    for (int i = 0; i < 2; ++i) b[i] = 0x05060708u + threadIdx.x * i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
            asm volatile(
                "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                "{%0,%1,%2,%3};\n"
                : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3])
                : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
    int s = 0;
    for (int j = 0; j < 4; ++j)
        for (int i = 0; i < 4; ++i) s ^= c[j][i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) k_hmma(float *out, int iters)
{
    unsigned a[4], b[2];
    float c[4][4] = {};
    for (int i = 0; i < 4; ++i) a[i] = 0x3c003c00u;
    for (int i = 0; i < 2; ++i) b[i] = 0x3c003c00u;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
            asm volatile(
                "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                "{%0,%1,%2,%3};\n"
                : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
    float s = 0;
    for (int j = 0; j < 4; ++j)
        for (int i = 0; i < 4; ++i) s += c[j][i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
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
    const int blocks = sms * 4, threads = 256, iters = 4096;
    int *buf;
    cudaMalloc(&buf, (size_t)blocks * threads * 4);
    const double warps = (double)blocks * threads / 32;
    double ms = time_ms([&] { k_imma<<<blocks, threads>>>(buf, iters); });
    printf("mma.sync m16n8k32 u8 : %8.1f TOPS (int8 ops, 2 per MAC)\n",
           warps * iters * 4 * (16.0 * 8 * 32 * 2) / (ms * 1e-3) / 1e12);
    ms = time_ms([&] { k_hmma<<<blocks, threads>>>((float *)buf, iters); });
    printf("mma.sync m16n8k16 f16: %8.1f TFLOPS\n", warps * iters * 4 * (16.0 * 8 * 16 * 2) / (ms * 1e-3) / 1e12);
    printf("cuda: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
