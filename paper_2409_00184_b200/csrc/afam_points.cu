// K1: batched point decode (value [+ gradient]) from device-resident slots.
//
// Replaces MicroModel.values_at / gradients_at (reference model.py:64-87)
// and bspline.evaluate_points[_with_gradient] (bspline.py:206-229).  One
// thread per point.  Parameters u = clip((p-lo)/(hi-lo), 0, 1) are formed in
// float64 with the reference's division and the knot span is chosen in
// float64 (bit-exact span selection); well-conditioned slots then evaluate
// the basis and contraction in float32, slots flagged AFAM_SLOT_FP64
// (ill-conditioned fits) in float64.  Output is float32, or float64 with
// AFAM_EVAL_OUT_F64 (ill-conditioned models take values far outside the
// data range between lattice points, where float32 storage alone would
// break the 1e-5 absolute gate).
#include "afam_eval.cuh"

namespace afam {

template <typename T, bool GRAD>
__device__ __forceinline__ T eval_dispatch(const BlockDesc &d, const double (&u)[3], T g[3]) {
    switch (d.deg) {
        case 1: return eval_uncached<1, T, GRAD>(d, u, g);
        case 2: return eval_uncached<2, T, GRAD>(d, u, g);
        default: return eval_uncached<3, T, GRAD>(d, u, g);
    }
}

template <bool GRAD, typename OT>
__global__ void __launch_bounds__(256) eval_points_kernel(const BlockDesc *__restrict__ descs,
                                                          const int32_t *__restrict__ slots, int32_t slot,
                                                          const double *__restrict__ pts, int64_t n,
                                                          OT *__restrict__ val, OT *__restrict__ grad,
                                                          uint32_t flags) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t sl = slots ? __ldg(slots + i) : slot;
    const BlockDesc d = load_desc(descs + sl);
    const bool param = flags & AFAM_EVAL_PARAM;
    double u[3];
#pragma unroll
    for (int a = 0; a < 3; a++) {
        const double p = __ldg(pts + 3 * i + a);
        // model.py:64-68 params_for, then the second clip of bspline.py:194
        u[a] = clamp01(param ? p : __ddiv_rn(__dsub_rn(p, d.lo[a]), d.span[a]));
    }
    double v, g[3] = {0.0, 0.0, 0.0};
    if (d.flags & AFAM_SLOT_FP64) {
        v = eval_dispatch<double, GRAD>(d, u, g);
    } else {
        float gf[3];
        v = eval_dispatch<float, GRAD>(d, u, gf);
        if (GRAD)
#pragma unroll
            for (int a = 0; a < 3; a++) g[a] = gf[a];
    }
    val[i] = (OT)v;
    if (GRAD) {
#pragma unroll
        for (int a = 0; a < 3; a++) grad[3 * i + a] = (OT)(param ? g[a] : g[a] / d.span[a]);  // model.py:79
    }
}

template <typename OT>
static void launch(const BlockDesc *descs, const int32_t *slots, int32_t slot, const double *pts, int64_t n,
                   void *val, void *grad, uint32_t flags, cudaStream_t st) {
    const int threads = 256;
    const unsigned blocks = (unsigned)((n + threads - 1) / threads);
    if (grad)
        eval_points_kernel<true, OT><<<blocks, threads, 0, st>>>(descs, slots, slot, pts, n, (OT *)val, (OT *)grad,
                                                                 flags);
    else
        eval_points_kernel<false, OT><<<blocks, threads, 0, st>>>(descs, slots, slot, pts, n, (OT *)val, nullptr,
                                                                  flags);
}

}  // namespace afam

using namespace afam;

extern "C" int afam_eval_points(afam_store *s, const int32_t *slots, int32_t slot, const double *pts, int64_t n,
                                void *val, void *grad, uint32_t flags, void *stream) {
    AFAM_CHECK(s, AFAM_E_VALUE, "store is NULL");
    AFAM_CHECK(n >= 0, AFAM_E_VALUE, "negative point count");
    if (n == 0) return AFAM_OK;
    AFAM_CHECK(pts && val, AFAM_E_VALUE, "pts/val is NULL");
    cudaStream_t st = (cudaStream_t)stream;
    AFAM_CUDA(cudaSetDevice(s->device));
    {
        std::lock_guard<std::mutex> lk(s->mu);
        if (!slots) {
            AFAM_CHECK(slot >= 0 && slot < s->nslots && s->host[slot].valid, AFAM_E_VALUE, "slot %d is empty", slot);
            AFAM_CHECK(!s->host[slot].ds, AFAM_E_VALUE, "slot %d holds a DS block (no spline to evaluate)", slot);
            AFAM_CUDA(cudaStreamWaitEvent(st, s->host[slot].ready, 0));
        } else {
            // the caller passes resident slots only; order after every upload still in flight
            for (int32_t k = 0; k < s->nslots; k++) {
                SlotHost &h = s->host[k];
                if (!h.valid || !h.pending) continue;
                if (cudaEventQuery(h.ready) == cudaSuccess) h.pending = false;
                else AFAM_CUDA(cudaStreamWaitEvent(st, h.ready, 0));
            }
        }
    }
    if (flags & AFAM_EVAL_OUT_F64) launch<double>(s->d_desc, slots, slot, pts, n, val, grad, flags, st);
    else launch<float>(s->d_desc, slots, slot, pts, n, val, grad, flags, st);
    AFAM_CUDA(cudaGetLastError());
    return AFAM_OK;
}
