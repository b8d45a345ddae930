// Microbenchmark: cost of LDG.128 (L1-resident data) when only some lanes of
// a warp are predicated on, and FFMA vs FFMA2 issue throughput.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void ldg_pred(const float4 *__restrict__ buf, int mask_bits, int pattern, int iters, float *out) {
    const int lane = threadIdx.x & 31;
    float4 acc = make_float4(0, 0, 0, 0);
    unsigned seed = threadIdx.x * 2654435761u + blockIdx.x;
    int off = (threadIdx.x * 7) & 255;
    for (int it = 0; it < iters; it++) {
        seed = seed * 1664525u + 1013904223u;
        bool on;
        if (pattern == 0) on = ((seed >> 16) & 1023) < (unsigned)mask_bits;       // random, prob mask_bits/1024
        else if (pattern == 1) on = lane < mask_bits;                             // first k lanes
        else on = ((lane & 7) == 0) && ((lane >> 3) < mask_bits);                 // one lane per quarter
#pragma unroll
        for (int u = 0; u < 16; u++) {
            if (on) {
                float4 v = __ldg(buf + ((off + u * 17 + it) & 1023));
                acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
            }
        }
    }
    if (acc.x == 1234.5f) out[0] = acc.y + acc.z + acc.w;
}

__global__ void ffma1(float *out, int iters) {
    float a[8], b = threadIdx.x * 1e-3f, c = 0.999f;
    for (int i = 0; i < 8; i++) a[i] = i;
    for (int it = 0; it < iters; it++)
#pragma unroll
        for (int i = 0; i < 8; i++) a[i] = fmaf(a[i], c, b);
    float s = 0; for (int i = 0; i < 8; i++) s += a[i];
    if (s == 1234.5f) out[0] = s;
}

__global__ void ffma2(float *out, int iters) {
    float2 a[4], b = make_float2(threadIdx.x * 1e-3f, threadIdx.x * 1e-3f), c = make_float2(0.999f, 0.999f);
    for (int i = 0; i < 4; i++) a[i] = make_float2(i, i + 1);
    for (int it = 0; it < iters; it++)
#pragma unroll
        for (int i = 0; i < 4; i++) a[i] = __ffma2_rn(a[i], c, b);
    float s = 0; for (int i = 0; i < 4; i++) s += a[i].x + a[i].y;
    if (s == 1234.5f) out[0] = s;
}

int main() {
    float4 *buf; float *out;
    cudaMalloc(&buf, 1024 * sizeof(float4)); cudaMemset(buf, 0, 1024 * sizeof(float4));
    cudaMalloc(&out, 64);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int blocks = 148 * 8, threads = 256, iters = 256;
    auto run = [&](int mb, int pat) {
        ldg_pred<<<blocks, threads>>>(buf, mb, pat, iters, out);
        cudaEventRecord(e0);
        ldg_pred<<<blocks, threads>>>(buf, mb, pat, iters, out);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double warp_ldg = (double)blocks * threads / 32 * iters * 16;
        printf("pattern %d param %4d : %.3f ms, %.2f SM-cycles per warp-LDG.128 (@1.95GHz)\n", pat, mb, ms,
               ms * 1e-3 * 1.95e9 * 148 / warp_ldg);
    };
    for (int mb : {1024, 768, 512, 256, 128, 64, 16, 0}) run(mb, 0);
    for (int k : {32, 24, 16, 8, 4, 1}) run(k, 1);
    for (int k : {4, 2, 1}) run(k, 2);
    float ms;
    ffma1<<<blocks, threads>>>(out, 4096); cudaEventRecord(e0); ffma1<<<blocks, threads>>>(out, 4096);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA : %.1f TFLOP/s\n", 2.0 * blocks * threads * 4096 * 8 / (ms * 1e-3) / 1e12);
    ffma2<<<blocks, threads>>>(out, 4096); cudaEventRecord(e0); ffma2<<<blocks, threads>>>(out, 4096);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA2: %.1f TFLOP/s\n", 2.0 * blocks * threads * 4096 * 8 / (ms * 1e-3) / 1e12);
    return 0;
}
