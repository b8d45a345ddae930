// FP32 FMA throughput probe: the denominator of the K2 roofline (the ray
// march is FMA-issue bound; MEASURED_PEAKS.json carries only
// HBM and bf16 tensor peaks).
#include <algorithm>

#include "afam_internal.h"

namespace afam {

__global__ void __launch_bounds__(256) fma_probe_kernel(float *out, int iters) {
    float a[8];
#pragma unroll
    for (int k = 0; k < 8; k++) a[k] = threadIdx.x * 1e-3f + k;
    const float b = 0.999999f, c = 1e-7f;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int r = 0; r < 16; r++)
#pragma unroll
            for (int k = 0; k < 8; k++) a[k] = fmaf(a[k], b, c);
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; k++) s += a[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

}  // namespace afam

extern "C" int afam_bench_fma(float *out, int32_t iters, float *ms, double *flops, void *stream) {
    AFAM_CHECK(out && ms && flops && iters > 0, AFAM_E_VALUE, "bad afam_bench_fma arguments");
    cudaStream_t st = (cudaStream_t)stream;
    int dev = 0, sms = 148;
    AFAM_CUDA(cudaGetDevice(&dev));
    AFAM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int blocks = std::min(sms * 8, 148 * 8);
    cudaEvent_t e0, e1;
    AFAM_CUDA(cudaEventCreate(&e0));
    AFAM_CUDA(cudaEventCreate(&e1));
    afam::fma_probe_kernel<<<blocks, 256, 0, st>>>(out, 16);  // warm
    AFAM_CUDA(cudaEventRecord(e0, st));
    afam::fma_probe_kernel<<<blocks, 256, 0, st>>>(out, iters);
    AFAM_CUDA(cudaEventRecord(e1, st));
    AFAM_CUDA(cudaEventSynchronize(e1));
    AFAM_CUDA(cudaEventElapsedTime(ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *flops = 2.0 * 16 * 8 * (double)iters * blocks * 256;
    return AFAM_OK;
}
