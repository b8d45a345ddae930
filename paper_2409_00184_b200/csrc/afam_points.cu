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

// HD: the store holds blocks of degrees above AFAM_FAST_DEGREE (float64 from
// the knots, eval_any).  A separate instantiation: its call frame alone made
// the common kernel spill (0 -> 128 bytes, -28% on the 2^24-point batches).
template <typename T, bool GRAD, bool HD>
__device__ __forceinline__ T eval_dispatch(const BlockDesc &d, const double (&u)[3], T g[3]) {
    switch (d.deg) {
        case 1: return eval_uncached<1, T, GRAD>(d, u, g);
        case 2: return eval_uncached<2, T, GRAD>(d, u, g);
        case 3: return eval_uncached<3, T, GRAD>(d, u, g);
        default: {  // degrees above AFAM_FAST_DEGREE: float64 from the knots
            if constexpr (HD) {
                double gd[3];
                const double v = eval_any(d, u, GRAD ? gd : nullptr);
                if constexpr (GRAD)
                    for (int a = 0; a < 3; a++) g[a] = (T)gd[a];
                return (T)v;
            } else {
                return eval_uncached<3, T, GRAD>(d, u, g);  // not reached: the host picks HD for such stores
            }
        }
    }
}

// DS baseline blocks (AFAM_SLOT_DS, reference downsample.py:101-138):
// trilinear interpolation at continuous lattice indices x (_trilinear:
// base = clip(floor(x), 0, max(top - 1, 0)), neighbours min(base + 1, top)),
// in float64 from the float32 grid g of dims (nx, ny, nz), x fastest.
__device__ __forceinline__ double ds_trilinear(const float *__restrict__ g, const int (&dims)[3],
                                               const double (&x)[3]) {
    int b0[3], b1[3];
    double f[3];
#pragma unroll
    for (int a = 0; a < 3; a++) {
        const int top = dims[a] - 1;
        const int b = min(max((int)floor(x[a]), 0), max(top - 1, 0));
        b0[a] = b;
        b1[a] = min(b + 1, top);
        f[a] = x[a] - (double)b;
    }
    auto at = [&](int i, int j, int k) { return (double)__ldg(g + ((size_t)k * dims[1] + j) * dims[0] + i); };
    // the reference's order: x, then y, then z, each as a (1 - f) + b f
    const double c00 = at(b0[0], b0[1], b0[2]) * (1.0 - f[0]) + at(b1[0], b0[1], b0[2]) * f[0];
    const double c10 = at(b0[0], b1[1], b0[2]) * (1.0 - f[0]) + at(b1[0], b1[1], b0[2]) * f[0];
    const double c01 = at(b0[0], b0[1], b1[2]) * (1.0 - f[0]) + at(b1[0], b0[1], b1[2]) * f[0];
    const double c11 = at(b0[0], b1[1], b1[2]) * (1.0 - f[0]) + at(b1[0], b1[1], b1[2]) * f[0];
    const double c0 = c00 * (1.0 - f[1]) + c10 * f[1];
    const double c1 = c01 * (1.0 - f[1]) + c11 * f[1];
    return c0 * (1.0 - f[2]) + c1 * f[2];
}

template <bool GRAD, typename OT>
__device__ __forceinline__ void eval_ds(const BlockDesc &d, const double *__restrict__ pts, int64_t i, int64_t o,
                                        OT *val, OT *grad) {
    const int g = d.deg;  // ghost width
    const int n[3] = {d.ds_n[0], d.ds_n[1], d.ds_n[2]};
    const int nr[3] = {n[0] + 2 * g, n[1] + 2 * g, n[2] + 2 * g};
    double x[3], xg[3];
#pragma unroll
    for (int a = 0; a < 3; a++) {  // _continuous_index: clip((p - lo) / span, 0, 1) * (n - 1)
        const double p = __ldg(pts + 3 * i + a);
        x[a] = clamp01(__ddiv_rn(__dsub_rn(p, d.lo[a]), d.span[a])) * (double)(n[a] - 1);
        xg[a] = x[a] + (double)g;
    }
    val[o] = (OT)ds_trilinear(d.ctrl, nr, xg);
    if (GRAD) {
        const size_t plane = (size_t)n[0] * n[1] * n[2];
        const float *grids = reinterpret_cast<const float *>(d.ctrl4);
#pragma unroll
        for (int a = 0; a < 3; a++)  // central-difference grids x (n - 1) / span (downsample.py:118-128)
            grad[3 * o + a] = (OT)(ds_trilinear(grids + a * plane, n, x) * ((double)(n[a] - 1) / d.span[a]));
    }
}

template <bool GRAD, typename OT, bool HD>
__device__ __forceinline__ void eval_points_body(const BlockDesc *__restrict__ descs,
                                                 const int32_t *__restrict__ slots, int32_t slot,
                                                 const double *__restrict__ pts, int64_t n, OT *__restrict__ val,
                                                 OT *__restrict__ grad, uint32_t flags,
                                                 const int32_t *__restrict__ order, const int32_t *__restrict__ keep,
                                                 OT *__restrict__ tval, OT *__restrict__ tgrad) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= n) return;
    // order: the batch bucketed by slot (slot_scatter_kernel), so the lanes
    // of a warp gather from one block's control points (L1/L2 reuse); a
    // batch that already comes in runs of one slot keeps its order (*keep)
    const bool bucketed = order && !*keep;
    const int64_t i = bucketed ? (int64_t)__ldg(order + j) : j;
    // bucketed batches write their results in bucket order (coalesced);
    // unpermute_kernel moves them to the caller's order
    const int64_t o = bucketed ? j : i;
    if (bucketed) {
        val = tval;
        grad = tgrad;
    }
    const int32_t sl = slots ? __ldg(slots + i) : slot;
    const BlockDesc d = load_desc(descs + sl);
    if (d.flags & AFAM_SLOT_DS) {  // world points only (DS blocks have no parameter space)
        eval_ds<GRAD, OT>(d, pts, i, o, val, grad);
        return;
    }
    const bool param = flags & AFAM_EVAL_PARAM;
    double u[3];
#pragma unroll
    for (int a = 0; a < 3; a++) {
        const double p = __ldg(pts + 3 * i + a);
        // model.py:64-68 params_for, then the second clip of bspline.py:194
        u[a] = clamp01(param ? p : __ddiv_rn(__dsub_rn(p, d.lo[a]), d.span[a]));
    }
    double v, g[3] = {0.0, 0.0, 0.0};
    if ((d.flags & AFAM_SLOT_FP64) || d.deg > AFAM_FAST_DEGREE) {  // float64 (high degrees: eval_any)
        v = eval_dispatch<double, GRAD, HD>(d, u, g);
    } else {
        float gf[3];
        v = eval_dispatch<float, GRAD, HD>(d, u, gf);
        if (GRAD)
#pragma unroll
            for (int a = 0; a < 3; a++) g[a] = gf[a];
    }
    val[o] = (OT)v;
    if (GRAD) {
#pragma unroll
        for (int a = 0; a < 3; a++) grad[3 * o + a] = (OT)(param ? g[a] : g[a] / d.span[a]);  // model.py:79
    }
}

// value-only: 64 registers, 4 CTAs of 256 per SM; value + gradient held to
// 80 registers (3 CTAs per SM: at 86 it dropped to 2 and ran 15% slower)
template <typename OT, bool HD>
__global__ void __launch_bounds__(256) eval_points_kernel(const BlockDesc *__restrict__ descs,
                                                          const int32_t *__restrict__ slots, int32_t slot,
                                                          const double *__restrict__ pts, int64_t n,
                                                          OT *__restrict__ val, uint32_t flags,
                                                          const int32_t *__restrict__ order,
                                                          const int32_t *__restrict__ keep, OT *__restrict__ tval) {
    eval_points_body<false, OT, HD>(descs, slots, slot, pts, n, val, nullptr, flags, order, keep, tval, nullptr);
}

template <typename OT, bool HD>
__global__ void __launch_bounds__(256, 3) eval_points_grad_kernel(const BlockDesc *__restrict__ descs,
                                                                  const int32_t *__restrict__ slots, int32_t slot,
                                                                  const double *__restrict__ pts, int64_t n,
                                                                  OT *__restrict__ val, OT *__restrict__ grad,
                                                                  uint32_t flags, const int32_t *__restrict__ order,
                                                                  const int32_t *__restrict__ keep,
                                                                  OT *__restrict__ tval, OT *__restrict__ tgrad) {
    eval_points_body<true, OT, HD>(descs, slots, slot, pts, n, val, grad, flags, order, keep, tval, tgrad);
}

template <typename OT, bool HD>
static void launch_hd(const BlockDesc *descs, const int32_t *slots, int32_t slot, const double *pts, int64_t n,
                      void *val, void *grad, uint32_t flags, const int32_t *order, const int32_t *keep, void *tval,
                      void *tgrad, cudaStream_t st) {
    const int threads = 256;
    const unsigned blocks = (unsigned)((n + threads - 1) / threads);
    if (grad)
        eval_points_grad_kernel<OT, HD><<<blocks, threads, 0, st>>>(descs, slots, slot, pts, n, (OT *)val,
                                                                    (OT *)grad, flags, order, keep, (OT *)tval,
                                                                    (OT *)tgrad);
    else
        eval_points_kernel<OT, HD><<<blocks, threads, 0, st>>>(descs, slots, slot, pts, n, (OT *)val, flags, order,
                                                               keep, (OT *)tval);
}

template <typename OT>
static void launch(const BlockDesc *descs, const int32_t *slots, int32_t slot, const double *pts, int64_t n,
                   void *val, void *grad, uint32_t flags, const int32_t *order, const int32_t *keep, void *tval,
                   void *tgrad, cudaStream_t st, bool hd) {
    if (hd) launch_hd<OT, true>(descs, slots, slot, pts, n, val, grad, flags, order, keep, tval, tgrad, st);
    else launch_hd<OT, false>(descs, slots, slot, pts, n, val, grad, flags, order, keep, tval, tgrad, st);
}

// ---- bucketing a per-point slot batch by slot (counting sort, three passes)
// A random batch (points of many blocks interleaved) gathers each point's
// (p+1)^3 control points from a different block: 4 x 64-byte x-quad runs
// per point, each straddling DRAM bursts.  Bucketed, the lanes of a warp
// read one block's control points and L1/L2 serve the overlap.
constexpr int kBucketChunk = 8192;  // points per CTA (count and scatter passes)
constexpr int kBucketThreads = 512;
constexpr int kBucketMaxSlots = 16383;  // per-CTA shared histogram: nslots + 1 int32

__device__ __forceinline__ int bucket_of(int32_t sl, int nslots) { return (sl >= 0 && sl < nslots) ? sl : nslots; }

__global__ void __launch_bounds__(kBucketThreads) slot_count_kernel(const int32_t *__restrict__ slots, int64_t n,
                                                                    int nslots, int32_t *__restrict__ count,
                                                                    unsigned long long *__restrict__ runs) {
    extern __shared__ int32_t h[];
    for (int i = threadIdx.x; i <= nslots; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const int64_t b = (int64_t)blockIdx.x * kBucketChunk, e = min(n, b + kBucketChunk);
    unsigned breaks = 0;  // i with slots[i] != slots[i-1]: how far the batch already is from bucketed
    for (int64_t i = b + threadIdx.x; i < e; i += blockDim.x) {
        const int32_t sl = __ldg(slots + i);
        atomicAdd(&h[bucket_of(sl, nslots)], 1);
        breaks += (i > 0 && __ldg(slots + i - 1) != sl) ? 1u : 0u;
    }
    breaks = __reduce_add_sync(0xffffffffu, breaks);
    if ((threadIdx.x & 31) == 0 && breaks) atomicAdd(runs, (unsigned long long)breaks);
    __syncthreads();
    for (int i = threadIdx.x; i <= nslots; i += blockDim.x)
        if (h[i]) atomicAdd(&count[i], h[i]);
}

// exclusive scan of count[0..nb) into offs (one CTA of 1024 threads, tiles with a carry)
__global__ void __launch_bounds__(1024) slot_scan_kernel(const int32_t *__restrict__ count, int nb,
                                                         int32_t *__restrict__ offs,
                                                         const unsigned long long *__restrict__ runs, int64_t n,
                                                         int32_t *__restrict__ keep) {
    __shared__ int32_t wsum[32];
    __shared__ int32_t carry;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // runs of one slot averaging >= 256 points (8 warps): gathers are
    // already coherent, keep the caller's order (no scatter, no unpermute)
    if (threadIdx.x == 0) *keep = (*runs + 1) * 256 <= (unsigned long long)n ? 1 : 0;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < nb; base += 1024) {
        const int i = base + threadIdx.x;
        const int32_t v = i < nb ? count[i] : 0;
        int32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        if (warp == 0) {
            int32_t w = wsum[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += y;
            }
            wsum[lane] = w;
        }
        __syncthreads();
        const int32_t incl = x + (warp ? wsum[warp - 1] : 0);
        if (i < nb) offs[i] = carry + incl - v;
        __syncthreads();
        if (threadIdx.x == 1023) carry += incl;
        __syncthreads();
    }
}

// order[pos] = i with pos in slot i's bucket: per CTA a shared histogram,
// one global reservation per (CTA, slot), then shared cursors
__global__ void __launch_bounds__(kBucketThreads) slot_scatter_kernel(const int32_t *__restrict__ slots, int64_t n,
                                                                      int nslots, int32_t *__restrict__ cursor,
                                                                      int32_t *__restrict__ order,
                                                                      int32_t *__restrict__ inv,
                                                                      const int32_t *__restrict__ keep) {
    if (*keep) return;
    extern __shared__ int32_t h[];
    for (int i = threadIdx.x; i <= nslots; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const int64_t b = (int64_t)blockIdx.x * kBucketChunk, e = min(n, b + kBucketChunk);
    for (int64_t i = b + threadIdx.x; i < e; i += blockDim.x) atomicAdd(&h[bucket_of(__ldg(slots + i), nslots)], 1);
    __syncthreads();
    for (int i = threadIdx.x; i <= nslots; i += blockDim.x)
        if (h[i]) h[i] = atomicAdd(&cursor[i], h[i]);
    __syncthreads();
    for (int64_t i = b + threadIdx.x; i < e; i += blockDim.x) {
        const int pos = atomicAdd(&h[bucket_of(__ldg(slots + i), nslots)], 1);
        order[pos] = (int32_t)i;
        inv[i] = pos;
    }
}

// out[i] = tmp[inv[i]]: results back to the caller's order (coalesced
// writes, 16-byte random reads instead of scattered partial-sector writes)
template <typename OT>
__global__ void __launch_bounds__(256) unpermute_kernel(const int32_t *__restrict__ inv, int64_t n,
                                                        const OT *__restrict__ tval, const OT *__restrict__ tgrad,
                                                        OT *__restrict__ val, OT *__restrict__ grad,
                                                        const int32_t *__restrict__ keep) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n || *keep) return;
    const int64_t j = __ldg(inv + i);
    val[i] = tval[j];
    if (grad) {
        grad[3 * i] = tgrad[3 * j];
        grad[3 * i + 1] = tgrad[3 * j + 1];
        grad[3 * i + 2] = tgrad[3 * j + 2];
    }
}

// AFAM_EVAL_BUCKET=0 disables the bucketing (A/B)
static bool bucket_enabled() {
    static const bool v = [] {
        const char *e = getenv("AFAM_EVAL_BUCKET");
        return !(e && atoi(e) == 0);
    }();
    return v;
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
    bool hd = false;  // blocks of degrees above AFAM_FAST_DEGREE may be evaluated: the HD kernel
    {
        std::lock_guard<std::mutex> lk(s->mu);
        if (!slots) {
            hd = s->host[slot].valid && !s->host[slot].ds && s->host[slot].deg > AFAM_FAST_DEGREE;
            AFAM_CHECK(slot >= 0 && slot < s->nslots && s->host[slot].valid, AFAM_E_VALUE, "slot %d is empty", slot);
            AFAM_CHECK(!s->host[slot].ds || !(flags & AFAM_EVAL_PARAM), AFAM_E_VALUE,
                       "slot %d holds a DS block: parameter-space evaluation needs a spline", slot);
            AFAM_CUDA(cudaStreamWaitEvent(st, s->host[slot].ready, 0));
        } else {
            // the caller passes resident slots only; order after every upload still in flight
            bool any_ds = false;
            for (int32_t k = 0; k < s->nslots; k++) {
                SlotHost &h = s->host[k];
                any_ds = any_ds || (h.valid && h.ds);
                hd = hd || (h.valid && !h.ds && h.deg > AFAM_FAST_DEGREE);
                if (!h.valid || !h.pending) continue;
                if (cudaEventQuery(h.ready) == cudaSuccess) h.pending = false;
                else AFAM_CUDA(cudaStreamWaitEvent(st, h.ready, 0));
            }
            if ((flags & AFAM_EVAL_PARAM) && any_ds) {
                // parameter-space points need splines: the single-slot rule for
                // the per-point slots too (read back only when DS slots exist)
                std::vector<int32_t> hs((size_t)n);
                AFAM_CUDA(cudaMemcpyAsync(hs.data(), slots, (size_t)n * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
                AFAM_CUDA(cudaStreamSynchronize(st));
                for (int64_t i = 0; i < n; i++) {
                    const int32_t k = hs[(size_t)i];
                    AFAM_CHECK(!(k >= 0 && k < s->nslots && s->host[k].valid && s->host[k].ds), AFAM_E_VALUE,
                               "slot %d holds a DS block: parameter-space evaluation needs a spline", k);
                }
            }
        }
    }
    int32_t *order = nullptr, *count = nullptr, *inv = nullptr, *keep = nullptr;
    unsigned long long *runs = nullptr;
    void *tmp = nullptr;
    const size_t osz = (flags & AFAM_EVAL_OUT_F64) ? sizeof(double) : sizeof(float);
    if (slots && n >= (1 << 16) && n < INT32_MAX && s->nslots <= kBucketMaxSlots && bucket_enabled()) {
        const int nb = s->nslots + 1;
        const size_t hsm = (size_t)nb * sizeof(int32_t);
        const unsigned grid = (unsigned)((n + kBucketChunk - 1) / kBucketChunk);
        AFAM_CUDA(cudaMallocAsync(&order, (size_t)n * sizeof(int32_t), st));
        AFAM_CUDA(cudaMallocAsync(&inv, (size_t)n * sizeof(int32_t), st));
        AFAM_CUDA(cudaMallocAsync(&tmp, (size_t)n * osz * (grad ? 4 : 1), st));
        // count[nb] | offsets[nb] | keep (int32, padded) | runs (u64)
        AFAM_CUDA(cudaMallocAsync(&count, 2 * hsm + 32, st));
        AFAM_CUDA(cudaMemsetAsync(count, 0, 2 * hsm + 32, st));
        keep = count + 2 * nb;
        runs = reinterpret_cast<unsigned long long *>(reinterpret_cast<char *>(count) + ((2 * hsm + 8 + 7) & ~7ull));
        static bool configured = false;
        if (!configured) {
            AFAM_CUDA(cudaFuncSetAttribute(slot_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
            AFAM_CUDA(cudaFuncSetAttribute(slot_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
            configured = true;
        }
        slot_count_kernel<<<grid, kBucketThreads, hsm, st>>>(slots, n, s->nslots, count, runs);
        slot_scan_kernel<<<1, 1024, 0, st>>>(count, nb, count + nb, runs, n, keep);
        slot_scatter_kernel<<<grid, kBucketThreads, hsm, st>>>(slots, n, s->nslots, count + nb, order, inv, keep);
    }
    void *ev = order ? tmp : nullptr;
    void *eg = order && grad ? (void *)((char *)tmp + (size_t)n * osz) : nullptr;
    if (flags & AFAM_EVAL_OUT_F64)
        launch<double>(s->d_desc, slots, slot, pts, n, val, grad, flags, order, keep, ev, eg, st, hd);
    else
        launch<float>(s->d_desc, slots, slot, pts, n, val, grad, flags, order, keep, ev, eg, st, hd);
    AFAM_CUDA(cudaGetLastError());
    if (order) {
        const unsigned g2 = (unsigned)((n + 255) / 256);
        if (flags & AFAM_EVAL_OUT_F64)
            unpermute_kernel<double><<<g2, 256, 0, st>>>(inv, n, (const double *)ev, (const double *)eg,
                                                         (double *)val, (double *)grad, keep);
        else
            unpermute_kernel<float><<<g2, 256, 0, st>>>(inv, n, (const float *)ev, (const float *)eg, (float *)val,
                                                        (float *)grad, keep);
        AFAM_CUDA(cudaGetLastError());
        AFAM_CUDA(cudaFreeAsync(order, st));
        AFAM_CUDA(cudaFreeAsync(inv, st));
        AFAM_CUDA(cudaFreeAsync(tmp, st));
        AFAM_CUDA(cudaFreeAsync(count, st));
    }
    // later uploads into the slots read here wait for this launch (the
    // per-point slot ids are device data: every valid slot is marked)
    ThreadCtx *tc = thread_ctx(s->device);
    AFAM_CHECK(tc, AFAM_E_CUDA, "per-thread state unavailable");
    AFAM_CUDA(cudaEventRecord(tc->read, st));
    if (!slots) {
        mark_readers(s, &slot, 1, tc->read);
    } else {
        std::lock_guard<std::mutex> lk(s->mu);
        for (int32_t k = 0; k < s->nslots; k++)
            if (s->host[k].valid) s->host[k].reader = tc->read;
    }
    return AFAM_OK;
}
