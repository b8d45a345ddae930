// Internal definitions shared by the libafam translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/afam.h"

namespace afam {

// Per-span basis table entry (built by the K4 unpack kernel, read by K1/K2).
// For degree p and span s the entry holds
//   W[k]   = t[s-p+1+k],                     k = 0 .. 2p-1   (knot window)
//   inv    = 1/(t[s+r+1] - t[s+1-j+r])       j = 1..p, r = 0..j-1 (row-major)
// i.e. every Cox-de Boor denominator of bspline.py:62-68 and the two
// derivative denominators of bspline.py:91-93 (the j = p row), so basis
// values and derivatives need no division on the hot path.
__host__ __device__ constexpr int tab_stride(int p) {
    return ((2 * p + p * (p + 1) / 2) + 3) / 4 * 4;  // p=1:4 p=2:8 p=3:12
}
constexpr int kTabStrideMax = 12;  // tab_stride(AFAM_FAST_DEGREE); higher degrees have no tables

// Device-resident descriptor of one slot (one micro-model).
struct alignas(16) BlockDesc {
    const float *ctrl;    // ncp x ncp rows of `pitch` floats: ctrl[(iz*ncp+iy)*pitch+ix]
    const float4 *ctrl4;  // x-quad layout: ctrl4[(iz*ncp+ix)*ncp+iy] = c[ix..ix+3][iy][iz] (0 past ncp-1)
    const float *tab32;   // [3][nspan][tab_stride(deg)] float
    const double *tab64;  // [3][nspan][tab_stride(deg)] double
    const float *knots;   // [3][nk] float (full clamped vectors)
    const float2 *crange; // [nspan^3] per knot cell (kz*nspan+kx)*nspan+ky: [min, max] of its (p+1)^3
                          // control points widened by max|c| * 2^-14 (degrees <= AFAM_FAST_DEGREE),
                          // then [ns4^3] (ns4 = ceil(nspan/4)) the same over aligned 4x4x4 cell groups
    double lo[3];         // extent low corner
    double span[3];       // hi - lo
    double inv_span[3];   // 1 / (hi - lo)
    float lo_f[3];        // lo as float32 (block extents are dyadic: exact)
    float inv_span_f[3];  // 1/(hi-lo) as float32
    int32_t ncp, deg, pitch, nk;
    int32_t nspan;        // ncp - deg
    uint32_t flags;       // AFAM_SLOT_* | kFlagUniform
    float max_abs;
    int32_t ds_n[3];      // AFAM_SLOT_DS: interior lattice dims (ghost width in `deg`,
                          // raw samples at `ctrl`, gradient grids [3][nz][ny][nx] at `ctrl4`)
};

// Internal desc flag: all three knot vectors are the clamped uniform ones
// (stored knot k == float32((k-deg)/nspan)), so interior spans use the
// closed-form uniform B-spline basis.
constexpr uint32_t kFlagUniform = 0x100u;

// Host mirror of a slot.
struct SlotHost {
    bool valid = false;
    bool pending = false;  // upload possibly still in flight (ready not yet observed)
    int32_t ncp = 0, deg = 0;
    bool ds = false;       // down-sampled raw block (AFAM_SLOT_DS)
    bool maxabs_known = false;  // afam_store::h_maxabs[slot] set on the host at put time (else after `ready`)
    bool uniform = false;       // host-checked: the knots are the clamped uniform ones (kFlagUniform)
    double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    cudaEvent_t ready = nullptr;  // recorded after the upload kernels
    cudaEvent_t reader = nullptr; // the last kernel reading the slot (a ThreadCtx event): uploads wait on it
};

// Per (calling thread, device) state of the frame path: the timing bracket
// of this thread's last afam_render, its pinned argument staging, and the
// event its point-query / decode launches record.  Two threads rendering
// from one store never share these (no lock, no overwritten kernel time).
// Never destroyed: slots may still name `k1` / `read` as their reader.
struct ThreadCtx {
    // afam_render keeps a ring of kRing frames per thread (a caller may
    // launch frame i+1 before collecting frame i): call n uses entry n % kRing
    static constexpr int kRing = 2;
    cudaEvent_t k0[kRing] = {}, k1[kRing] = {};  // bracket the call's kernels (timing, slot readers)
    unsigned char *pack[kRing] = {};              // pinned staging of the call's argument upload
    size_t pack_cap[kRing] = {};
    cudaEvent_t ev_pack[kRing] = {};              // the last upload out of pack[r]
    uint64_t nrender = 0;                         // afam_render calls made by this thread on this device
    cudaEvent_t read = nullptr;                   // recorded after afam_eval_points / afam_decode_grid launches
};
ThreadCtx *thread_ctx(int device);  // afam_store.cu

struct DecodeOp {  // banded collocation matrix of bspline.py:98-125 for (ncp, deg, m)
    float *b32 = nullptr;   // [m][4]
    double *b64 = nullptr;  // [m][4]
    int32_t *col0 = nullptr;// [m] first nonzero column (span - deg)
    // tensor-core decode (afam_decode.cu, m == 65, ncp <= 72): the first m-1
    // rows of B dense over K = kp columns (kp = ncp rounded up to 8), split
    // into tf32 hi and lo parts, in the K-major no-swizzle operand layout
    float *tc_b = nullptr;  // [2][kp/4][m-1][4]: hi panels, then lo panels
    int32_t tc_kp = 0;      // 0: the tensor-core path does not apply
    // register-tiled decode (afam_decode.cu, decode_fx_kernel): m == 65,
    // deg + 1 <= ncp <= 65 and the u = 1 row selecting the last control
    // point exactly
    bool fx_ok = false;
    bool any = false;       // degree above AFAM_FAST_DEGREE: decode_any_kernel over b64
};

// Banded rows of the collocation matrix of bspline.py:98-125 for (ncp, deg,
// m): params linspace(0, 1, m), fresh float64 clamped uniform knots; row i
// holds N[col0[i] .. col0[i] + deg] at b[i * band_stride(deg) + j] (afam_decode.cu).
inline int band_stride(int deg) { return deg + 1 > 4 ? deg + 1 : 4; }
void host_band(int ncp, int deg, int m, std::vector<double> &b, std::vector<int32_t> &col0);

struct FitOp {  // endpoint-pinned least-squares fit operator (bspline.py:109-159), device
    double *fit = nullptr;   // [ncp][m]: coefficients = fit @ samples along one axis
    double *dec = nullptr;   // [m][ncp]: dense collocation matrix (decode along one axis)
    double *fitT = nullptr;  // [m][ncp rounded up to 4]: fit transposed, zero-padded (tiled kernel)
    double *decT = nullptr;  // [ncp][m rounded up to 4]: dec transposed, zero-padded
};

}  // namespace afam

struct afam_store {
    int device = 0;
    int32_t nslots = 0, max_ncp = 0;
    double fp64_limit = 4.0;
    size_t raw_bytes = 0, ctrl_floats = 0, ctrl4_elems = 0, knot_floats = 0, tab_elems = 0, slot_bytes = 0;
    size_t crange_elems = 0;
    char *arena = nullptr;               // nslots * slot_bytes device bytes
    afam::BlockDesc *d_desc = nullptr;   // nslots descriptors (device)
    float *d_maxabs = nullptr;           // nslots (device)
    float *h_maxabs = nullptr;           // nslots (pinned host): copied back after each upload, valid once
                                         // the slot's `ready` event completed (afam_render: float64 kernel?)
    std::vector<afam::SlotHost> host;
    // afam_store_put_file: ring of pinned staging buffers (file -> pinned -> H2D)
    static constexpr int kFileRing = 4;
    unsigned char *h_file[kFileRing] = {nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t ev_file[kFileRing] = {nullptr, nullptr, nullptr, nullptr};
    int file_next = 0;
    std::mutex file_mu[kFileRing];
    std::mutex file_ring_mu;
    std::mutex mu;
    std::map<std::tuple<int, int, int>, afam::DecodeOp> ops;
    std::map<std::tuple<int, int, int>, afam::FitOp> fit_ops;  // (ncp, deg, m)

    char *slot_base(int32_t slot) const { return arena + (size_t)slot * slot_bytes; }
    uint8_t *raw_ptr(int32_t slot) const { return (uint8_t *)slot_base(slot); }
    float *ctrl_ptr(int32_t slot) const { return (float *)(slot_base(slot) + raw_off()); }
    float4 *ctrl4_ptr(int32_t slot) const { return (float4 *)(slot_base(slot) + ctrl4_off()); }
    float *knot_ptr(int32_t slot) const { return (float *)(slot_base(slot) + knot_off()); }
    float *tab32_ptr(int32_t slot) const { return (float *)(slot_base(slot) + tab32_off()); }
    double *tab64_ptr(int32_t slot) const { return (double *)(slot_base(slot) + tab64_off()); }
    float2 *crange_ptr(int32_t slot) const { return (float2 *)(slot_base(slot) + crange_off()); }
    static size_t align256(size_t v) { return (v + 255) & ~(size_t)255; }
    size_t raw_off() const { return align256(raw_bytes); }
    size_t ctrl4_off() const { return raw_off() + align256(ctrl_floats * 4); }
    size_t knot_off() const { return ctrl4_off() + align256(ctrl4_elems * 16); }
    size_t tab32_off() const { return knot_off() + align256(knot_floats * 4); }
    size_t tab64_off() const { return tab32_off() + align256(tab_elems * 4); }
    size_t crange_off() const { return tab64_off() + align256(tab_elems * 8); }
};

struct afam_manifest {
    int32_t levels = 0;
    std::vector<int32_t> bpa;
    std::vector<std::vector<double>> extents;  // per level, bpa^3*6
};

namespace afam {
void set_error(const char *fmt, ...);
int cuda_fail(cudaError_t e, const char *what);

// Order `st` after the slot's upload; uploads already observed complete cost
// one flag test (caller holds s->mu).
inline cudaError_t wait_slot(afam_store *s, int32_t slot, cudaStream_t st) {
    SlotHost &h = s->host[slot];
    if (!h.pending) return cudaSuccess;
    if (cudaEventQuery(h.ready) == cudaSuccess) {
        h.pending = false;
        return cudaSuccess;
    }
    return cudaStreamWaitEvent(st, h.ready, 0);
}

// Order an upload into `slot` on `st` after the kernels still reading the
// slot's previous contents (caller holds s->mu).
inline cudaError_t wait_readers(afam_store *s, int32_t slot, cudaStream_t st) {
    cudaEvent_t r = s->host[slot].reader;
    return r ? cudaStreamWaitEvent(st, r, 0) : cudaSuccess;
}

// Name `ev` (recorded after the launches that read these slots) as their
// last reader.
inline void mark_readers(afam_store *s, const int32_t *slots, int32_t n, cudaEvent_t ev) {
    std::lock_guard<std::mutex> lk(s->mu);
    for (int32_t b = 0; b < n; b++)
        if (slots[b] >= 0 && slots[b] < s->nslots) s->host[slots[b]].reader = ev;
}
}  // namespace afam

#define AFAM_CUDA(call)                                                         \
    do {                                                                        \
        cudaError_t e_ = (call);                                                \
        if (e_ != cudaSuccess) return afam::cuda_fail(e_, #call);               \
    } while (0)

#define AFAM_CHECK(cond, code, ...)                                             \
    do {                                                                        \
        if (!(cond)) {                                                          \
            afam::set_error(__VA_ARGS__);                                       \
            return code;                                                        \
        }                                                                       \
    } while (0)
