// Device store of micro-models (K4): slot arena, .mfa ingest, per-span tables.
//
// Replaces the read side of store.load_model / model.deserialize
// (reference store.py:43-47, model.py:121-148) with an HBM-resident slot
// arena.  The .mfa payload is misaligned (knots at byte 1, control points
// at byte 1+12(ncp+d), FORMAT.md:24-30), so the raw file image is copied
// H2D verbatim and realigned on device by unpack_ctrl_kernel /
// build_tables_kernel; no host-side repacking.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cerrno>
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "afam_internal.h"

namespace afam {

static thread_local std::string g_err;

void set_error(const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
}

int cuda_fail(cudaError_t e, const char *what) {
    set_error("CUDA error %s (%s) in %s", cudaGetErrorName(e), cudaGetErrorString(e), what);
    return AFAM_E_CUDA;
}

// One ThreadCtx per (thread, device), created on first use (the caller has
// selected `device`) and kept for the life of the process.
ThreadCtx *thread_ctx(int device) {
    static thread_local std::map<int, ThreadCtx *> ctx;
    auto it = ctx.find(device);
    if (it != ctx.end()) return it->second;
    ThreadCtx *c = new ThreadCtx();
    bool ok = cudaEventCreateWithFlags(&c->read, cudaEventDisableTiming) == cudaSuccess;
    for (int r = 0; r < ThreadCtx::kRing; r++)
        ok = ok && cudaEventCreate(&c->k0[r]) == cudaSuccess && cudaEventCreate(&c->k1[r]) == cudaSuccess &&
             cudaEventCreateWithFlags(&c->ev_pack[r], cudaEventDisableTiming) == cudaSuccess;
    if (!ok) {
        set_error("cannot create the per-thread render events");
        return nullptr;
    }
    ctx[device] = c;
    return c;
}

static __device__ __forceinline__ float load_le_f32(const uint8_t *p) {
    uint32_t v = (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
    return __uint_as_float(v);
}

// One thread per padded control point: gather the little-endian float32 at
// byte offset src_off + 4*(ix + ncp*(iy + ncp*iz)) (x fastest, FORMAT.md:57-61)
// into the row-pitched layout ctrl[(iz*ncp + iy)*pitch + ix]; padding is 0.
// Also reduces max |c| into *maxabs (float bits are ordered for c >= 0).
__global__ void unpack_ctrl_kernel(const uint8_t *__restrict__ raw, uint64_t src_off, int ncp, int pitch,
                                   float *__restrict__ ctrl, unsigned int *maxabs) {
    const int64_t total = (int64_t)ncp * ncp * pitch;
    float m = 0.f;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int ix = (int)(i % pitch);
        int64_t row = i / pitch;  // iz*ncp + iy
        float v = 0.f;
        if (ix < ncp) {
            v = load_le_f32(raw + src_off + 4 * ((uint64_t)row * ncp + ix));
            m = fmaxf(m, fabsf(v));
        }
        ctrl[i] = v;
    }
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(maxabs, __float_as_uint(m));
}

// x-quad layout for the ray march, y innermost: ctrl4[(iz*ncp+ix)*ncp+iy] =
// c[ix..ix+3][iy][iz] (0 past ncp-1).  A (p+1)^3 gather is p+1 runs of p+1
// consecutive 16-byte rows (one address per z plane).
__global__ void unpack_quad_kernel(const uint8_t *__restrict__ raw, uint64_t src_off, int ncp,
                                   float4 *__restrict__ ctrl4) {
    const int64_t total = (int64_t)ncp * ncp * ncp;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int iy = (int)(i % ncp);
        const int ix = (int)((i / ncp) % ncp);
        const int64_t iz = i / ((int64_t)ncp * ncp);
        const uint8_t *row = raw + src_off + 4 * (uint64_t)((iz * ncp + iy) * ncp);  // x-fastest source row
        float v[4];
#pragma unroll
        for (int k = 0; k < 4; k++) v[k] = (ix + k < ncp) ? load_le_f32(row + 4 * (ix + k)) : 0.f;
        ctrl4[i] = make_float4(v[0], v[1], v[2], v[3]);
    }
}

// Value range of every knot cell: for cell (kx, ky, kz) the min and max of
// the (p+1)^3 control points that weight its samples, widened by
// max|c| * 2^-14.  The basis functions of a cell are non-negative and sum to
// one, so any value the ray march computes in the cell lies in that range
// (its float32 rounding is ~1e-6 max|c|, 60x inside the margin); a frame
// whose transfer function has zero opacity on the whole range skips the
// cell's samples without decoding them (render2_kernel, sample_fast2).
// One 64-thread CTA per aligned 4x4x4 cell group: the group's (4+p)^3
// control points staged in shared memory, one cell per thread, then the
// group's union (the second level, at crange + nspan^3).
__global__ void __launch_bounds__(64) cell_range_kernel(const float *__restrict__ ctrl, int ncp, int pitch, int deg,
                                                        const unsigned int *maxabs, float2 *__restrict__ crange) {
    const int nspan = ncp - deg, ns4 = (nspan + 3) / 4, W = 4 + deg;
    const int g = blockIdx.x;
    const int Y = g % ns4, X = (g / ns4) % ns4, Z = g / (ns4 * ns4);
    __shared__ float s[7 * 7 * 7];  // [z][y][x], W <= 7
    for (int i = threadIdx.x; i < W * W * W; i += 64) {
        const int x = i % W, y = (i / W) % W, z = i / (W * W);
        const int ix = 4 * X + x, iy = 4 * Y + y, iz = 4 * Z + z;
        s[i] = (ix < ncp && iy < ncp && iz < ncp) ? ctrl[((size_t)iz * ncp + iy) * pitch + ix] : 0.f;
    }
    __syncthreads();
    const float eps = __uint_as_float(*maxabs) * 0x1p-14f;
    const int tx = threadIdx.x & 3, ty = (threadIdx.x >> 2) & 3, tz = threadIdx.x >> 4;
    const int kx = 4 * X + tx, ky = 4 * Y + ty, kz = 4 * Z + tz;
    float lo = INFINITY, hi = -INFINITY;
    if (kx < nspan && ky < nspan && kz < nspan) {
        for (int cz = 0; cz <= deg; cz++)
            for (int by = 0; by <= deg; by++)
                for (int bx = 0; bx <= deg; bx++) {
                    const float v = s[((tz + cz) * W + ty + by) * W + tx + bx];
                    lo = fminf(lo, v);
                    hi = fmaxf(hi, v);
                }
        lo -= eps;
        hi += eps;
        crange[((size_t)kz * nspan + kx) * nspan + ky] = make_float2(lo, hi);
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    __shared__ float2 w[2];
    if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = make_float2(lo, hi);
    __syncthreads();
    if (threadIdx.x == 0)
        crange[(size_t)nspan * nspan * nspan + g] = make_float2(fminf(w[0].x, w[1].x), fmaxf(w[0].y, w[1].y));
}

// Knots + per-span basis tables + the slot descriptor.  knot_off: byte
// offset of the knots; has_t0 = 0 for .mfa images (t0 = 0 implicit,
// FORMAT.md:44-55), 1 for full vectors.
__global__ void build_tables_kernel(const uint8_t *__restrict__ raw, uint64_t knot_off, int has_t0, int ncp,
                                    int deg, float *__restrict__ knots, float *__restrict__ tab32,
                                    double *__restrict__ tab64, BlockDesc *desc, BlockDesc proto,
                                    const unsigned int *maxabs, float fp64_limit) {
    const int nk = ncp + deg + 1;
    const int nspan = ncp - deg;
    const int ts = tab_stride(deg);
    auto knot = [&](int a, int k) -> float {
        if (has_t0) return load_le_f32(raw + knot_off + 4 * (uint64_t)(a * nk + k));
        if (k == 0) return 0.f;
        return load_le_f32(raw + knot_off + 4 * (uint64_t)(a * (nk - 1) + (k - 1)));
    };
    __shared__ int uniform;
    if (threadIdx.x == 0) uniform = 1;
    __syncthreads();
    for (int i = threadIdx.x; i < 3 * nk; i += blockDim.x) {
        const int k = i % nk;
        const float t = knot(i / nk, k);
        knots[i] = t;
        // bspline.clamped_knots(ncp, deg).astype(float32) (bspline.py:29-38, model.py:98)
        const float want = k <= deg ? 0.f : (k >= ncp ? 1.f : (float)((double)(k - deg) / (double)nspan));
        if (__float_as_uint(t) != __float_as_uint(want)) atomicAnd(&uniform, 0);
    }
    // per-span tables for the fast degrees only (higher degrees evaluate from
    // the knots, afam_eval.cuh eval_any)
    for (int i = threadIdx.x; i < (deg <= AFAM_FAST_DEGREE ? 3 * nspan : 0); i += blockDim.x) {
        const int a = i / nspan, s = deg + i % nspan;
        double W[2 * AFAM_FAST_DEGREE];
        for (int k = 0; k < 2 * deg; k++) {
            int idx = s - deg + 1 + k;
            W[k] = (idx >= 0 && idx < nk) ? (double)knot(a, idx) : 0.0;
        }
        float *e32 = tab32 + (size_t)i * ts;
        double *e64 = tab64 + (size_t)i * ts;
        for (int k = 0; k < 2 * deg; k++) { e32[k] = (float)W[k]; e64[k] = W[k]; }
        int o = 2 * deg;
        for (int j = 1; j <= deg; j++)
            for (int r = 0; r < j; r++, o++) {
                // t[s+r+1] - t[s+1-j+r] = W[deg+r] - W[deg-j+r]
                double den = W[deg + r] - W[deg - j + r];
                double inv = den != 0.0 ? 1.0 / den : 0.0;
                e32[o] = (float)inv;
                e64[o] = inv;
            }
        for (; o < ts; o++) { e32[o] = 0.f; e64[o] = 0.0; }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        BlockDesc d = proto;
        d.max_abs = __uint_as_float(*maxabs);
        d.flags = AFAM_SLOT_VALID | (d.max_abs > fp64_limit ? AFAM_SLOT_FP64 : 0u) | (uniform ? kFlagUniform : 0u);
        *desc = d;
    }
}

}  // namespace afam

using namespace afam;

extern "C" {

const char *afam_last_error(void) { return g_err.c_str(); }
int afam_version(void) { return 1; }

int afam_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

static size_t serialized_size(int64_t ncp, int64_t deg) { return 1 + (size_t)((ncp + deg) * 3 + ncp * ncp * ncp) * 4; }
static int pitch_for(int ncp) { return (ncp + 3) & ~3; }

int afam_store_create(afam_store **out, int device, int32_t slots, int32_t max_ncp, double fp64_ctrl_limit) {
    AFAM_CHECK(out, AFAM_E_VALUE, "afam_store_create: out is NULL");
    AFAM_CHECK(slots >= 1, AFAM_E_VALUE, "cache capacity must be at least 1 slot");
    AFAM_CHECK(max_ncp >= 2 && max_ncp <= 1024, AFAM_E_VALUE, "max_ncp %d out of range", max_ncp);
    AFAM_CUDA(cudaSetDevice(device));
    afam_store *s = new afam_store();
    s->device = device;
    s->nslots = slots;
    s->max_ncp = max_ncp;
    s->fp64_limit = fp64_ctrl_limit > 0 ? fp64_ctrl_limit : 4.0;
    const size_t P = (size_t)pitch_for(max_ncp);
    // raw staging must also hold a decoded (full-knot) upload: 3*(ncp+4) + ncp^3 floats
    s->raw_bytes = std::max(serialized_size(max_ncp, AFAM_MAX_DEGREE),
                            (size_t)(3 * (max_ncp + AFAM_MAX_DEGREE + 1) + (size_t)max_ncp * max_ncp * max_ncp) * 4 + 64);
    s->ctrl_floats = P * max_ncp * max_ncp;
    s->ctrl4_elems = (size_t)max_ncp * max_ncp * max_ncp;
    s->knot_floats = 3 * (size_t)(max_ncp + AFAM_MAX_DEGREE + 1);
    s->tab_elems = 3 * (size_t)max_ncp * kTabStrideMax;
    const size_t ns4 = (size_t)(max_ncp + 3) / 4;
    s->crange_elems = (size_t)max_ncp * max_ncp * max_ncp + ns4 * ns4 * ns4;
    s->slot_bytes = s->crange_off() + afam_store::align256(s->crange_elems * 8);
    cudaError_t e = cudaMalloc(&s->arena, s->slot_bytes * (size_t)slots);
    if (e != cudaSuccess) {
        delete s;
        if (e == cudaErrorMemoryAllocation) {
            set_error("device store of %d slots x %zu bytes does not fit in device memory", slots,
                      (size_t)0);
            return AFAM_E_CAPACITY;
        }
        return cuda_fail(e, "cudaMalloc(arena)");
    }
    AFAM_CUDA(cudaMalloc(&s->d_desc, sizeof(BlockDesc) * slots));
    AFAM_CUDA(cudaMemset(s->d_desc, 0, sizeof(BlockDesc) * slots));
    AFAM_CUDA(cudaMalloc(&s->d_maxabs, sizeof(float) * slots));
    AFAM_CUDA(cudaHostAlloc((void **)&s->h_maxabs, sizeof(float) * slots, cudaHostAllocDefault));
    s->host.resize(slots);
    for (auto &h : s->host) AFAM_CUDA(cudaEventCreateWithFlags(&h.ready, cudaEventDisableTiming));
    {
        // the per-call argument buffers come from the device's stream-ordered
        // pool (cudaMallocAsync); keep its memory mapped across
        // synchronizations, or every frame would re-map it (ms per call)
        cudaMemPool_t pool;
        AFAM_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t keep = UINT64_MAX;
        AFAM_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    }
    *out = s;
    return AFAM_OK;
}

int afam_store_destroy(afam_store *s) {
    if (!s) return AFAM_OK;
    cudaSetDevice(s->device);
    cudaDeviceSynchronize();
    for (auto &h : s->host)
        if (h.ready) cudaEventDestroy(h.ready);
    for (int b = 0; b < afam_store::kFileRing; b++) {
        if (s->h_file[b]) cudaFreeHost(s->h_file[b]);
        if (s->ev_file[b]) cudaEventDestroy(s->ev_file[b]);
    }
    for (auto &kv : s->ops) {
        cudaFree(kv.second.b32);
        cudaFree(kv.second.b64);
        cudaFree(kv.second.col0);
        if (kv.second.tc_b) cudaFree(kv.second.tc_b);
    }
    for (auto &kv : s->fit_ops) {
        cudaFree(kv.second.fit);
        cudaFree(kv.second.dec);
        cudaFree(kv.second.fitT);
        cudaFree(kv.second.decT);
    }
    cudaFree(s->arena);
    cudaFree(s->d_desc);
    cudaFree(s->d_maxabs);
    if (s->h_maxabs) cudaFreeHost(s->h_maxabs);
    delete s;
    return AFAM_OK;
}

int afam_store_slots(const afam_store *s, int32_t *slots, int32_t *max_ncp) {
    AFAM_CHECK(s, AFAM_E_VALUE, "store is NULL");
    if (slots) *slots = s->nslots;
    if (max_ncp) *max_ncp = s->max_ncp;
    return AFAM_OK;
}

// Shared tail of both put paths: raw region already holds the bytes (queued on stream).
// The device's kFlagUniform test (build_tables_kernel) on the host: every
// stored knot equals float32((k - deg) / nspan) clamped to [0, 1], bitwise.
static bool uniform_knot(float t, int k, int ncp, int deg) {
    const float want = k <= deg ? 0.f : (k >= ncp ? 1.f : (float)((double)(k - deg) / (double)(ncp - deg)));
    uint32_t x, y;
    memcpy(&x, &t, 4);
    memcpy(&y, &want, 4);
    return x == y;
}

// .mfa image: knots t1.. per axis after the degree byte (t0 = 0 implicit, FORMAT.md:44-55)
static bool mfa_uniform(const uint8_t *bytes, int ncp, int deg) {
    const int stored = ncp + deg;
    for (int a = 0; a < 3; a++)
        for (int k = 1; k <= stored; k++) {
            float t;
            memcpy(&t, bytes + 1 + 4 * ((size_t)a * stored + (k - 1)), 4);
            if (!uniform_knot(t, k, ncp, deg)) return false;
        }
    return true;
}

// full knot vectors [3][ncp + deg + 1]
static bool knots_uniform(const float *knots, int ncp, int deg) {
    const int nk = ncp + deg + 1;
    for (int a = 0; a < 3; a++)
        for (int k = 0; k < nk; k++)
            if (!uniform_knot(knots[(size_t)a * nk + k], k, ncp, deg)) return false;
    return true;
}

// host_maxabs: max |c| when the caller scanned the control points on the host, else < 0
// host_uniform: the knots are known (on the host) to be the clamped uniform ones
static int launch_unpack(afam_store *s, int32_t slot, int deg, int ncp, uint64_t knot_off, int has_t0,
                         uint64_t ctrl_off, const double extent[6], cudaStream_t st, float host_maxabs,
                         bool host_uniform = false) {
    BlockDesc proto{};
    proto.ctrl = s->ctrl_ptr(slot);
    proto.ctrl4 = s->ctrl4_ptr(slot);
    proto.tab32 = s->tab32_ptr(slot);
    proto.tab64 = s->tab64_ptr(slot);
    proto.knots = s->knot_ptr(slot);
    proto.crange = deg <= AFAM_FAST_DEGREE ? s->crange_ptr(slot) : nullptr;
    for (int a = 0; a < 3; a++) {
        proto.lo[a] = extent[2 * a];
        proto.span[a] = extent[2 * a + 1] - extent[2 * a];
        proto.inv_span[a] = 1.0 / proto.span[a];
        proto.lo_f[a] = (float)proto.lo[a];
        proto.inv_span_f[a] = (float)proto.inv_span[a];
    }
    proto.ncp = ncp;
    proto.deg = deg;
    proto.pitch = pitch_for(ncp);
    proto.nk = ncp + deg + 1;
    proto.nspan = ncp - deg;
    AFAM_CUDA(cudaMemsetAsync(s->d_maxabs + slot, 0, sizeof(float), st));
    const int64_t total = (int64_t)ncp * ncp * proto.pitch;
    int grid = (int)std::min<int64_t>((total + 255) / 256, 1184);
    unpack_ctrl_kernel<<<grid, 256, 0, st>>>(s->raw_ptr(slot), ctrl_off, ncp, proto.pitch, s->ctrl_ptr(slot),
                                             (unsigned int *)(s->d_maxabs + slot));
    const int64_t total4 = (int64_t)ncp * ncp * ncp;
    unpack_quad_kernel<<<(int)std::min<int64_t>((total4 + 255) / 256, 1184), 256, 0, st>>>(
        s->raw_ptr(slot), ctrl_off, ncp, s->ctrl4_ptr(slot));
    if (deg <= AFAM_FAST_DEGREE) {
        const int ns4 = (ncp - deg + 3) / 4;
        cell_range_kernel<<<ns4 * ns4 * ns4, 64, 0, st>>>(s->ctrl_ptr(slot), ncp, proto.pitch, deg,
                                                          (const unsigned int *)(s->d_maxabs + slot),
                                                          s->crange_ptr(slot));
    }
    build_tables_kernel<<<1, 256, 0, st>>>(s->raw_ptr(slot), knot_off, has_t0, ncp, deg, s->knot_ptr(slot),
                                           s->tab32_ptr(slot), s->tab64_ptr(slot), s->d_desc + slot, proto,
                                           (const unsigned int *)(s->d_maxabs + slot), (float)s->fp64_limit);
    AFAM_CUDA(cudaGetLastError());
    SlotHost &h = s->host[slot];
    // the device's value lands in h_maxabs when the upload completes; a host
    // scan gives it now.  Either way it only selects afam_render's kernel
    // (both kernels decode every slot kind correctly), never a result.
    AFAM_CUDA(cudaMemcpyAsync(s->h_maxabs + slot, s->d_maxabs + slot, sizeof(float), cudaMemcpyDeviceToHost, st));
    h.maxabs_known = host_maxabs >= 0.f;
    if (h.maxabs_known) s->h_maxabs[slot] = host_maxabs;
    h.uniform = host_uniform;
    h.valid = true;
    h.pending = true;
    h.ncp = ncp;
    h.deg = deg;
    h.ds = false;
    for (int a = 0; a < 3; a++) { h.lo[a] = extent[2 * a]; h.hi[a] = extent[2 * a + 1]; }
    AFAM_CUDA(cudaEventRecord(h.ready, st));
    return AFAM_OK;
}

// DS gradient grids (reference downsample.py:83-105, DsBlock._gradient_grids):
// at every interior lattice point, per axis, (s[idx+1] - s[idx-1]) / 2 with
// the indices clipped to the ghosted array, in float64, stored float32.
__global__ void ds_gradient_kernel(const float *__restrict__ samp, int gx, int gy, int gz, int ghost, int nx, int ny,
                                   int nz, float *__restrict__ grid) {
    const int64_t total = (int64_t)nx * ny * nz;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(e % nx), j = (int)((e / nx) % ny), k = (int)(e / ((int64_t)nx * ny));
        const int I = i + ghost, J = j + ghost, K = k + ghost;
        auto at = [&](int a, int b, int c) { return (double)samp[((int64_t)c * gy + b) * gx + a]; };
        grid[e] = (float)((at(min(I + 1, gx - 1), J, K) - at(max(I - 1, 0), J, K)) / 2.0);
        grid[total + e] = (float)((at(I, min(J + 1, gy - 1), K) - at(I, max(J - 1, 0), K)) / 2.0);
        grid[2 * total + e] = (float)((at(I, J, min(K + 1, gz - 1)) - at(I, J, max(K - 1, 0))) / 2.0);
    }
}

static int check_put(afam_store *s, int32_t slot, int deg, int ncp, const double *extent) {
    AFAM_CHECK(s, AFAM_E_VALUE, "store is NULL");
    AFAM_CHECK(slot >= 0 && slot < s->nslots, AFAM_E_VALUE, "slot %d outside [0, %d)", slot, s->nslots);
    AFAM_CHECK(ncp <= s->max_ncp, AFAM_E_CAPACITY, "ncp %d exceeds the store's max_ncp %d", ncp, s->max_ncp);
    AFAM_CHECK(deg >= 1 && deg <= AFAM_MAX_DEGREE, AFAM_E_VALUE,
               "degree %d is not supported by the device path (1..%d)", deg, AFAM_MAX_DEGREE);
    AFAM_CHECK(extent, AFAM_E_VALUE, "extent is NULL");
    for (int a = 0; a < 3; a++)
        AFAM_CHECK(extent[2 * a + 1] > extent[2 * a], AFAM_E_VALUE, "degenerate extent");
    return AFAM_OK;
}

// model.py MicroModel: non-finite control points are a ValueError.  Host
// scan of the little-endian float32 payload by exponent bits (vectorizes).
// Also returns max |c| (for finite floats the magnitude order is the order of
// the bit patterns without the sign), the value the device derives in
// unpack_ctrl_kernel: afam_render picks its kernel from it before the upload
// has finished.
// (AVX2 clone where the host has it: 29 vs 78 us for a 65^3 block -- this
// scan is half the host time of a cache miss on the replay's frame thread)
__attribute__((target_clones("avx2", "default")))
static bool all_finite_le_f32(const uint8_t *p, size_t count, float *maxabs = nullptr) {
    uint32_t bad = 0, mx = 0;
    for (size_t i = 0; i < count; i++) {
        uint32_t u;
        memcpy(&u, p + 4 * i, 4);
        bad |= (uint32_t)((u & 0x7f800000u) == 0x7f800000u);
        mx = std::max(mx, u & 0x7fffffffu);
    }
    if (maxabs) memcpy(maxabs, &mx, 4);
    return bad == 0;
}

int afam_store_put_mfa(afam_store *s, int32_t slot, const uint8_t *bytes, uint64_t nbytes, int32_t ncp,
                       const double extent[6], void *stream) {
    AFAM_CHECK(bytes && nbytes >= 1, AFAM_E_FORMAT, "empty micro-model byte string");
    const int deg = bytes[0];
    // model.py:123-133
    AFAM_CHECK(deg < ncp, AFAM_E_FORMAT, "degree byte %d >= ncp %d", deg, ncp);
    const size_t expected = serialized_size(ncp, deg);
    AFAM_CHECK(nbytes == expected, AFAM_E_FORMAT,
               "micro-model length mismatch: expected %zu bytes for ncp=%d, degree=%d, found %llu", expected,
               ncp, deg, (unsigned long long)nbytes);
    // model.py MicroModel: non-finite control points are a ValueError
    float mx;
    AFAM_CHECK(all_finite_le_f32(bytes + 1 + 12ull * (ncp + deg), (size_t)ncp * ncp * ncp, &mx), AFAM_E_VALUE,
               "non-finite control points");
    int rc = check_put(s, slot, deg, ncp, extent);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    std::lock_guard<std::mutex> lk(s->mu);
    AFAM_CUDA(cudaSetDevice(s->device));
    // the previous upload into this slot (possibly on another stream) must be done
    AFAM_CUDA(cudaStreamWaitEvent(st, s->host[slot].ready, 0));
    AFAM_CUDA(wait_readers(s, slot, st));
    AFAM_CUDA(cudaMemcpyAsync(s->raw_ptr(slot), bytes, nbytes, cudaMemcpyHostToDevice, st));
    return launch_unpack(s, slot, deg, ncp, 1, 0, 1 + 12ull * (ncp + deg), extent, st, mx,
                         mfa_uniform(bytes, ncp, deg));
}


int afam_mfa_check(const uint8_t *bytes, uint64_t nbytes, int32_t ncp, int32_t *degree) {
    AFAM_CHECK(bytes && nbytes >= 1, AFAM_E_FORMAT, "empty micro-model byte string");
    const int deg = bytes[0];
    AFAM_CHECK(deg < ncp, AFAM_E_FORMAT, "degree byte %d >= ncp %d", deg, ncp);
    const size_t expected = serialized_size(ncp, deg);
    AFAM_CHECK(nbytes == expected, AFAM_E_FORMAT,
               "micro-model length mismatch: expected %zu bytes for ncp=%d, degree=%d, found %llu", expected,
               ncp, deg, (unsigned long long)nbytes);
    AFAM_CHECK(all_finite_le_f32(bytes + 1 + 12ull * (ncp + deg), (size_t)ncp * ncp * ncp), AFAM_E_VALUE,
               "non-finite control points");
    if (degree) *degree = deg;
    return AFAM_OK;
}

int afam_store_put_mfa_device(afam_store *s, int32_t slot, const uint8_t *dbytes, uint64_t nbytes, int32_t degree,
                              int32_t ncp, const double extent[6], void *stream) {
    AFAM_CHECK(dbytes, AFAM_E_VALUE, "NULL device image");
    AFAM_CHECK(degree >= 1 && degree < ncp && nbytes == serialized_size(ncp, degree), AFAM_E_FORMAT,
               "device .mfa image: %llu bytes for ncp=%d, degree=%d", (unsigned long long)nbytes, ncp, degree);
    int rc = check_put(s, slot, degree, ncp, extent);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    std::lock_guard<std::mutex> lk(s->mu);
    AFAM_CUDA(cudaSetDevice(s->device));
    AFAM_CUDA(cudaStreamWaitEvent(st, s->host[slot].ready, 0));
    AFAM_CUDA(wait_readers(s, slot, st));
    AFAM_CUDA(cudaMemcpyAsync(s->raw_ptr(slot), dbytes, nbytes, cudaMemcpyDeviceToDevice, st));
    return launch_unpack(s, slot, degree, ncp, 1, 0, 1 + 12ull * (ncp + degree), extent, st, -1.f);
}

int afam_store_put_file(afam_store *s, int32_t slot, const char *path, int32_t ncp, const double extent[6],
                        int32_t *degree, void *stream) {
    AFAM_CHECK(s && path, AFAM_E_VALUE, "NULL argument to afam_store_put_file");
    int rc = check_put(s, slot, 1, ncp, extent);
    if (rc) return rc;
    AFAM_CUDA(cudaSetDevice(s->device));
    int b;
    {
        std::lock_guard<std::mutex> lk(s->file_ring_mu);
        b = s->file_next;
        s->file_next = (s->file_next + 1) % afam_store::kFileRing;
    }
    std::lock_guard<std::mutex> blk(s->file_mu[b]);
    if (!s->h_file[b]) {
        AFAM_CUDA(cudaHostAlloc((void **)&s->h_file[b], s->raw_bytes, cudaHostAllocDefault));
        AFAM_CUDA(cudaEventCreateWithFlags(&s->ev_file[b], cudaEventDisableTiming));
    } else {
        AFAM_CUDA(cudaEventSynchronize(s->ev_file[b]));  // the buffer's previous H2D copy is done
    }
    // store.load_model_bytes (store.py:33-41): a missing file is a FormatError
    const int fd = open(path, O_RDONLY);
    AFAM_CHECK(fd >= 0, AFAM_E_FORMAT, "missing model file %s", path);
    struct stat sb;
    if (fstat(fd, &sb) != 0) {
        close(fd);
        AFAM_CHECK(false, AFAM_E_FORMAT, "cannot stat model file %s", path);
    }
    const uint64_t nbytes = (uint64_t)sb.st_size;
    if (nbytes < 1 || nbytes > s->raw_bytes) {
        close(fd);
        AFAM_CHECK(nbytes >= 1, AFAM_E_FORMAT, "empty micro-model byte string");
        // longer than any model of this store's max ncp: length mismatch below
    }
    const size_t want = std::min<size_t>(nbytes, s->raw_bytes);
    size_t got = 0;
    while (got < want) {
        const ssize_t r = read(fd, s->h_file[b] + got, want - got);
        if (r < 0 && errno == EINTR) continue;
        if (r <= 0) break;
        got += (size_t)r;
    }
    close(fd);
    AFAM_CHECK(got == want, AFAM_E_FORMAT, "short read of model file %s", path);
    const uint8_t *bytes = s->h_file[b];
    const int deg = bytes[0];
    // model.py:123-133
    AFAM_CHECK(deg < ncp, AFAM_E_FORMAT, "degree byte %d >= ncp %d", deg, ncp);
    const size_t expected = serialized_size(ncp, deg);
    AFAM_CHECK(nbytes == expected, AFAM_E_FORMAT,
               "micro-model length mismatch: expected %zu bytes for ncp=%d, degree=%d, found %llu", expected, ncp,
               deg, (unsigned long long)nbytes);
    const uint64_t coff = 1 + 12ull * (ncp + deg);
    float mx;
    AFAM_CHECK(all_finite_le_f32(bytes + coff, (size_t)ncp * ncp * ncp, &mx), AFAM_E_VALUE, "non-finite control points");
    rc = check_put(s, slot, deg, ncp, extent);
    if (rc) return rc;
    if (degree) *degree = deg;
    cudaStream_t st = (cudaStream_t)stream;
    std::lock_guard<std::mutex> lk(s->mu);
    AFAM_CUDA(cudaStreamWaitEvent(st, s->host[slot].ready, 0));
    AFAM_CUDA(wait_readers(s, slot, st));
    AFAM_CUDA(cudaMemcpyAsync(s->raw_ptr(slot), bytes, nbytes, cudaMemcpyHostToDevice, st));
    AFAM_CUDA(cudaEventRecord(s->ev_file[b], st));
    return launch_unpack(s, slot, deg, ncp, 1, 0, coff, extent, st, mx, mfa_uniform(bytes, ncp, deg));
}

int afam_store_put_ds(afam_store *s, int32_t slot, const uint8_t *bytes, uint64_t nbytes, const double extent[6],
                      void *stream) {
    AFAM_CHECK(s, AFAM_E_VALUE, "store is NULL");
    AFAM_CHECK(slot >= 0 && slot < s->nslots, AFAM_E_VALUE, "slot %d outside [0, %d)", slot, s->nslots);
    AFAM_CHECK(bytes && nbytes >= 16, AFAM_E_FORMAT, "truncated block file: header missing");
    uint32_t hd[4];
    memcpy(hd, bytes, 16);
    const uint64_t expected = 16 + (uint64_t)hd[0] * hd[1] * hd[2] * 4;
    AFAM_CHECK(nbytes == expected, AFAM_E_FORMAT,
               "block length mismatch: expected %llu bytes for dims (%u,%u,%u), found %llu",
               (unsigned long long)expected, hd[0], hd[1], hd[2], (unsigned long long)nbytes);
    const int g = (int)hd[3];
    AFAM_CHECK(g == 0 || g == 1, AFAM_E_VALUE, "ghost width must be 0 or 1");
    for (int a = 0; a < 3; a++)
        AFAM_CHECK((int64_t)hd[a] > 2 * g + 1, AFAM_E_VALUE, "sample array (%u, %u, %u) too small for ghost %d", hd[0],
                   hd[1], hd[2], g);
    AFAM_CHECK(extent, AFAM_E_VALUE, "extent is NULL");
    for (int a = 0; a < 3; a++)
        AFAM_CHECK(extent[2 * a + 1] > extent[2 * a], AFAM_E_VALUE, "degenerate extent");
    const int nx = (int)hd[0] - 2 * g, ny = (int)hd[1] - 2 * g, nz = (int)hd[2] - 2 * g;
    AFAM_CHECK(nbytes <= s->raw_bytes && (uint64_t)3 * nx * ny * nz <= 4 * s->ctrl4_elems, AFAM_E_CAPACITY,
               "DS block (%u, %u, %u) exceeds the store's slot size (max_ncp %d)", hd[0], hd[1], hd[2], s->max_ncp);
    cudaStream_t st = (cudaStream_t)stream;
    std::lock_guard<std::mutex> lk(s->mu);
    AFAM_CUDA(cudaSetDevice(s->device));
    AFAM_CUDA(cudaStreamWaitEvent(st, s->host[slot].ready, 0));
    AFAM_CUDA(wait_readers(s, slot, st));
    AFAM_CUDA(cudaMemcpyAsync(s->raw_ptr(slot), bytes, nbytes, cudaMemcpyHostToDevice, st));
    const float *samp = reinterpret_cast<const float *>(s->raw_ptr(slot) + 16);
    float *grid = reinterpret_cast<float *>(s->ctrl4_ptr(slot));
    const int64_t total = (int64_t)nx * ny * nz;
    ds_gradient_kernel<<<(int)std::min<int64_t>((total + 255) / 256, 1184), 256, 0, st>>>(
        samp, (int)hd[0], (int)hd[1], (int)hd[2], g, nx, ny, nz, grid);
    BlockDesc d{};
    d.ctrl = samp;
    d.ctrl4 = reinterpret_cast<const float4 *>(grid);
    for (int a = 0; a < 3; a++) {
        d.lo[a] = extent[2 * a];
        d.span[a] = extent[2 * a + 1] - extent[2 * a];
        d.inv_span[a] = 1.0 / d.span[a];
        d.lo_f[a] = (float)d.lo[a];
        d.inv_span_f[a] = (float)d.inv_span[a];
    }
    d.deg = g;
    d.ds_n[0] = nx;
    d.ds_n[1] = ny;
    d.ds_n[2] = nz;
    d.ncp = std::max(nx, std::max(ny, nz));
    d.flags = AFAM_SLOT_VALID | AFAM_SLOT_DS;
    // the descriptor goes up by value on the same stream (pinned staging not needed for 144 B:
    // cudaMemcpyAsync from this stack copy completes before the call returns for pageable memory)
    AFAM_CUDA(cudaMemcpyAsync(s->d_desc + slot, &d, sizeof(d), cudaMemcpyHostToDevice, st));
    AFAM_CUDA(cudaGetLastError());
    SlotHost &h = s->host[slot];
    h.valid = true;
    h.pending = true;
    h.ncp = d.ncp;
    h.deg = g;
    h.ds = true;
    h.uniform = false;
    for (int a = 0; a < 3; a++) { h.lo[a] = extent[2 * a]; h.hi[a] = extent[2 * a + 1]; }
    AFAM_CUDA(cudaEventRecord(h.ready, st));
    return AFAM_OK;
}

int afam_store_put(afam_store *s, int32_t slot, int32_t degree, int32_t ncp, const float *knots,
                   const float *ctrl, const double extent[6], void *stream) {
    int rc = check_put(s, slot, degree, ncp, extent);
    if (rc) return rc;
    AFAM_CHECK(knots && ctrl, AFAM_E_VALUE, "knots/ctrl is NULL");
    cudaStream_t st = (cudaStream_t)stream;
    std::lock_guard<std::mutex> lk(s->mu);
    AFAM_CUDA(cudaSetDevice(s->device));
    const size_t kb = sizeof(float) * 3 * (size_t)(ncp + degree + 1);
    const size_t cb = sizeof(float) * (size_t)ncp * ncp * ncp;
    const uint64_t koff = 0, coff = (kb + 15) & ~(size_t)15;
    AFAM_CUDA(cudaStreamWaitEvent(st, s->host[slot].ready, 0));
    AFAM_CUDA(wait_readers(s, slot, st));
    AFAM_CUDA(cudaMemcpyAsync(s->raw_ptr(slot) + koff, knots, kb, cudaMemcpyHostToDevice, st));
    AFAM_CUDA(cudaMemcpyAsync(s->raw_ptr(slot) + coff, ctrl, cb, cudaMemcpyHostToDevice, st));
    float mx = -1.f;  // max |c| when finite (a non-finite value leaves it to the device)
    if (!all_finite_le_f32(reinterpret_cast<const uint8_t *>(ctrl), (size_t)ncp * ncp * ncp, &mx)) mx = -1.f;
    return launch_unpack(s, slot, degree, ncp, koff, 1, coff, extent, st, mx, knots_uniform(knots, ncp, degree));
}

int afam_store_evict(afam_store *s, int32_t slot) {
    AFAM_CHECK(s, AFAM_E_VALUE, "store is NULL");
    AFAM_CHECK(slot >= 0 && slot < s->nslots, AFAM_E_VALUE, "slot %d outside [0, %d)", slot, s->nslots);
    std::lock_guard<std::mutex> lk(s->mu);
    s->host[slot].valid = false;
    return AFAM_OK;
}

int afam_store_info(afam_store *s, int32_t slot, int32_t *ncp, int32_t *degree, uint32_t *flags,
                    float *max_abs_ctrl) {
    AFAM_CHECK(s, AFAM_E_VALUE, "store is NULL");
    AFAM_CHECK(slot >= 0 && slot < s->nslots, AFAM_E_VALUE, "slot %d outside [0, %d)", slot, s->nslots);
    AFAM_CUDA(cudaSetDevice(s->device));
    SlotHost &h = s->host[slot];
    AFAM_CHECK(h.valid, AFAM_E_VALUE, "slot %d is empty", slot);
    AFAM_CUDA(cudaEventSynchronize(h.ready));
    BlockDesc d;
    AFAM_CUDA(cudaMemcpy(&d, s->d_desc + slot, sizeof(d), cudaMemcpyDeviceToHost));
    if (ncp) *ncp = d.ncp;
    if (degree) *degree = d.deg;
    if (flags) *flags = d.flags;
    if (max_abs_ctrl) *max_abs_ctrl = d.max_abs;
    return AFAM_OK;
}

int afam_store_read(afam_store *s, int32_t slot, float *ctrl, float *knots) {
    AFAM_CHECK(s, AFAM_E_VALUE, "store is NULL");
    AFAM_CHECK(slot >= 0 && slot < s->nslots, AFAM_E_VALUE, "slot %d outside [0, %d)", slot, s->nslots);
    SlotHost &h = s->host[slot];
    AFAM_CHECK(h.valid, AFAM_E_VALUE, "slot %d is empty", slot);
    AFAM_CHECK(!h.ds, AFAM_E_VALUE, "slot %d holds a DS block", slot);
    AFAM_CUDA(cudaSetDevice(s->device));
    AFAM_CUDA(cudaEventSynchronize(h.ready));
    const int ncp = h.ncp, P = pitch_for(ncp);
    if (ctrl) {
        // strip the row padding: rows of ncp floats at pitch P
        AFAM_CUDA(cudaMemcpy2D(ctrl, sizeof(float) * ncp, s->ctrl_ptr(slot), sizeof(float) * P,
                               sizeof(float) * ncp, (size_t)ncp * ncp, cudaMemcpyDeviceToHost));
    }
    if (knots)
        AFAM_CUDA(cudaMemcpy(knots, s->knot_ptr(slot), sizeof(float) * 3 * (ncp + h.deg + 1),
                             cudaMemcpyDeviceToHost));
    return AFAM_OK;
}

}  // extern "C"
