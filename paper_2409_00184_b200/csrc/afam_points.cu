// K1: batched point decode (value [+ gradient]) from device-resident slots.
//
// Replaces MicroModel.values_at / gradients_at (reference model.py:64-87)
// and bspline.evaluate_points[_with_gradient] (bspline.py:206-229).  One
// thread per point; well-conditioned slots evaluate in float32, slots
// flagged AFAM_SLOT_FP64 (ill-conditioned fits) in float64.
#include "afam_eval.cuh"

namespace afam {

template <typename T, bool GRAD>
__device__ __forceinline__ T eval_dispatch(const BlockDesc &d, const T (&u)[3], T g[3]) {
    switch (d.deg) {
        case 1: return eval_uncached<1, T, GRAD>(d, u, g);
        case 2: return eval_uncached<2, T, GRAD>(d, u, g);
        default: return eval_uncached<3, T, GRAD>(d, u, g);
    }
}

template <bool GRAD>
__global__ void __launch_bounds__(256) eval_points_kernel(const BlockDesc *__restrict__ descs,
                                                          const int32_t *__restrict__ slots, int32_t slot,
                                                          const double *__restrict__ pts, int64_t n,
                                                          float *__restrict__ val, float *__restrict__ grad,
                                                          uint32_t flags) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t sl = slots ? __ldg(slots + i) : slot;
    const BlockDesc d = load_desc(descs + sl);
    const bool param = flags & AFAM_EVAL_PARAM;
    double p[3];
#pragma unroll
    for (int a = 0; a < 3; a++) p[a] = __ldg(pts + 3 * i + a);
    float v;
    float gf[3] = {0.f, 0.f, 0.f};
    if (d.flags & AFAM_SLOT_FP64) {
        double u[3], g[3];
#pragma unroll
        for (int a = 0; a < 3; a++)  // model.py:64-68 params_for (exact division) + bspline.py:194 clip
            u[a] = clamp01(param ? p[a] : __ddiv_rn(p[a] - d.lo[a], d.span[a]));
        double vv = eval_dispatch<double, GRAD>(d, u, g);
        v = (float)vv;
        if (GRAD)
#pragma unroll
            for (int a = 0; a < 3; a++) gf[a] = (float)(param ? g[a] : g[a] / d.span[a]);  // model.py:79
    } else {
        float u[3], g[3];
#pragma unroll
        for (int a = 0; a < 3; a++) u[a] = (float)clamp01(param ? p[a] : (p[a] - d.lo[a]) * d.inv_span[a]);
        v = eval_dispatch<float, GRAD>(d, u, g);
        if (GRAD)
#pragma unroll
            for (int a = 0; a < 3; a++) gf[a] = param ? g[a] : (float)((double)g[a] * d.inv_span[a]);
    }
    val[i] = v;
    if (GRAD) {
        grad[3 * i] = gf[0];
        grad[3 * i + 1] = gf[1];
        grad[3 * i + 2] = gf[2];
    }
}

}  // namespace afam

using namespace afam;

extern "C" int afam_eval_points(afam_store *s, const int32_t *slots, int32_t slot, const double *pts, int64_t n,
                                float *val, float *grad, uint32_t flags, void *stream) {
    AFAM_CHECK(s, AFAM_E_VALUE, "store is NULL");
    AFAM_CHECK(n >= 0, AFAM_E_VALUE, "negative point count");
    if (n == 0) return AFAM_OK;
    AFAM_CHECK(pts && val, AFAM_E_VALUE, "pts/val is NULL");
    cudaStream_t st = (cudaStream_t)stream;
    AFAM_CUDA(cudaSetDevice(s->device));
    if (!slots) {
        AFAM_CHECK(slot >= 0 && slot < s->nslots && s->host[slot].valid, AFAM_E_VALUE, "slot %d is empty", slot);
        AFAM_CUDA(cudaStreamWaitEvent(st, s->host[slot].ready, 0));
    } else {
        // every referenced slot must be uploaded; callers pass resident slots only
        for (int32_t k = 0; k < s->nslots; k++)
            if (s->host[k].valid) AFAM_CUDA(cudaStreamWaitEvent(st, s->host[k].ready, 0));
    }
    const int threads = 256;
    const int64_t blocks = (n + threads - 1) / threads;
    if (grad)
        eval_points_kernel<true><<<(unsigned)blocks, threads, 0, st>>>(s->d_desc, slots, slot, pts, n, val, grad, flags);
    else
        eval_points_kernel<false><<<(unsigned)blocks, threads, 0, st>>>(s->d_desc, slots, slot, pts, n, val, grad, flags);
    AFAM_CUDA(cudaGetLastError());
    return AFAM_OK;
}
