// FP32 FMA issue rates on this GPU: FFMA with a register / uniform-register
// operand and packed FFMA2, 8 independent chains per thread, 8 warps per SMSP.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long d;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__global__ void k_reg(float* out, float s, int iters) {
    float a[8], m = s + threadIdx.x * 1e-7f;
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = j;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], m, a[(j + 1) & 7]);
    float r = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) r += a[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
__global__ void k_uni(float* out, float s, int iters) {
    float a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = j + threadIdx.x;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], s, a[(j + 1) & 7]);
    float r = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) r += a[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
__global__ void k_f2(float* out, float s, int iters) {
    unsigned long long a[8], m;
    {
        float2 t = make_float2(s, s);
        m = *reinterpret_cast<unsigned long long*>(&t);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        float2 t = make_float2(j + threadIdx.x, j);
        a[j] = *reinterpret_cast<unsigned long long*>(&t);
    }
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = fma2(a[j], m, a[(j + 1) & 7]);
    float r = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        float2 t = *reinterpret_cast<float2*>(&a[j]);
        r += t.x + t.y;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int threads = 1024, blocks = sms * 2, iters = 20000;
    float* out;
    cudaMalloc(&out, sizeof(float) * threads * blocks);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char* names[3] = {"ffma_reg", "ffma_uniform", "ffma2_packed"};
    for (int v = 0; v < 3; ++v) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (v == 0) k_reg<<<blocks, threads>>>(out, 1.0000001f, iters);
            if (v == 1) k_uni<<<blocks, threads>>>(out, 1.0000001f, iters);
            if (v == 2) k_f2<<<blocks, threads>>>(out, 1.0000001f, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double fmas = (double)blocks * threads * iters * 8 * (v == 2 ? 2 : 1);
        printf("{\"kernel\": \"%s\", \"ms\": %.3f, \"TFMA_per_s\": %.2f, \"fma_per_clk_per_sm_at_1965\": %.1f}\n", names[v], ms,
               fmas / ms / 1e9, fmas / (ms * 1e-3) / sms / 1.965e9);
    }
    return 0;
}
