// K3: regular-grid decode of whole micro-blocks.
//
// Replaces MicroModel.decode_grid (reference model.py:89-93) ->
// bspline.decode_tensor_product (bspline.py:162-172), which applies the
// dense collocation matrix B (m x ncp, bspline.py:98-125, built from FRESH
// float64 uniform knots and params linspace(0,1,m)) along x, then y, then z
// as three float64 GEMMs.  B has only deg+1 non-zeros per row, so this
// kernel applies it in banded form: one CTA per (block, z-chunk), the three
// contractions staged through shared memory (z -> S1[n^2], y -> S2[n*m],
// x -> out), control points read once from HBM/L2 and the output written
// coalesced (x fastest).  Ill-conditioned slots (AFAM_SLOT_FP64) run the
// same schedule in float64.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "afam_internal.h"
#include "afam_umma.cuh"

namespace afam {

struct DecodeJob {
    int32_t slot;
    int32_t tc_kp;  // tensor-core path: K extent (ncp rounded up to 8); 0 = CUDA-core path
    int32_t fx;     // 1: float32 slots take decode_fx_kernel (register-tiled, m == 65)
    int32_t any;    // 1: degree above AFAM_FAST_DEGREE -> decode_any_kernel (b64: [m][deg+1] band)
    const int32_t *col0;
    const float *b32;
    const double *b64;
    const float *tc_b;
};

constexpr int kDecodeChunk = 65;     // output planes per CTA (a whole 65^3 block)
constexpr int kDecodeThreads = 416;  // 13 warps: 65 rows = 5 per warp
constexpr int kRing = AFAM_FAST_DEGREE + 1;  // plane slots: one window of p+1 planes

// ---- TMA bulk copy + mbarrier (PTX; SASS UBLKCP / SYNCS) ----
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

// 1-D bulk global -> shared copy completing on `bar` (16-byte aligned, size % 16 == 0)
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

constexpr int kMainGroups = 4;  // x-stage columns held per lane: up to 128 (longer rows use the tail path)

__device__ __forceinline__ void st4(float *p, const float (&v)[4]) {
    *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
}
__device__ __forceinline__ void st4(double *p, const double (&v)[4]) {
    reinterpret_cast<double2 *>(p)[0] = make_double2(v[0], v[1]);
    reinterpret_cast<double2 *>(p)[1] = make_double2(v[2], v[3]);
}
__device__ __forceinline__ void ld4(const float *p, float (&v)[4]) {
    const float4 t = *reinterpret_cast<const float4 *>(p);
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
}
__device__ __forceinline__ void ld4(const double *p, double (&v)[4]) {
    const double2 a = reinterpret_cast<const double2 *>(p)[0], b = reinterpret_cast<const double2 *>(p)[1];
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}

// acc[0..3] += w * v[0..3]: paired FMAs (FFMA2) in float32, scalar in float64
__device__ __forceinline__ void fma4(float w, float4 v, float (&acc)[4]) {
    const float2 lo = __ffma2_rn(make_float2(w, w), make_float2(v.x, v.y), make_float2(acc[0], acc[1]));
    const float2 hi = __ffma2_rn(make_float2(w, w), make_float2(v.z, v.w), make_float2(acc[2], acc[3]));
    acc[0] = lo.x; acc[1] = lo.y; acc[2] = hi.x; acc[3] = hi.y;
}
__device__ __forceinline__ void fma4(double w, float4 v, double (&acc)[4]) {
    acc[0] = fma(w, (double)v.x, acc[0]);
    acc[1] = fma(w, (double)v.y, acc[1]);
    acc[2] = fma(w, (double)v.z, acc[2]);
    acc[3] = fma(w, (double)v.w, acc[3]);
}
__device__ __forceinline__ void fma4(float w, const float *p, float (&acc)[4]) {
    fma4(w, *reinterpret_cast<const float4 *>(p), acc);
}
__device__ __forceinline__ void fma4(double w, const double *p, double (&acc)[4]) {
    double v[4];
    ld4(p, v);
#pragma unroll
    for (int e = 0; e < 4; e++) acc[e] = fma(w, v[e], acc[e]);
}

// Three smem-staged banded contractions per output plane, register-blocked:
// z and y items are 4 consecutive x (16-byte smem traffic), the x stage
// keeps each lane's Bx rows in registers for every row j.
template <int P, typename T>
__device__ __forceinline__ void decode_planes(const BlockDesc &d, const int32_t *__restrict__ col0g,
                                              const T *__restrict__ Bg, int m, int k0, int k1,
                                              float *__restrict__ out, unsigned char *smem) {
    constexpr int Q = P + 1;
    const int n = d.ncp, pitch = d.pitch, nq = pitch >> 2;
    T *S1 = reinterpret_cast<T *>(smem);  // [n][pitch]
    T *S2 = S1 + (size_t)n * pitch;       // [m][pitch]
    T *B = S2 + (size_t)m * pitch;        // [m][4]
    int *c0 = reinterpret_cast<int *>(B + (size_t)m * 4);
    for (int i = threadIdx.x; i < m * 4; i += blockDim.x) B[i] = Bg[i];
    for (int i = threadIdx.x; i < m; i += blockDim.x) c0[i] = col0g[i];
    __syncthreads();
    const float *__restrict__ C = d.ctrl;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    const int tid = threadIdx.x, nth = blockDim.x;
    const size_t zstride = (size_t)n * pitch;
    // z / y items: thread = (row group g_, x quad q_); groups * nq <= nth threads work
    const int groups = nth / nq, q_ = tid % nq, g_ = tid / nq, gstride = groups * pitch;
    const int ngroups = min(m / 32, kMainGroups), mainw = 32 * ngroups, tailw = m - mainw;
    const float inv_tail = tailw > 0 ? 1.f / (float)tailw : 0.f;
    T bx[kMainGroups][Q];
    int xi[kMainGroups];
#pragma unroll
    for (int t = 0; t < kMainGroups; t++) {
        const int i = min(lane + 32 * t, m - 1);
        xi[t] = c0[i];
#pragma unroll
        for (int a = 0; a < Q; a++) bx[t][a] = B[i * 4 + a];
    }
    // z-planes of control points stream through a ring of kRing smem slots by
    // TMA bulk copies (cp.async.bulk, one mbarrier per slot). The ring holds
    // one window of p+1 planes; the next output plane's new planes are issued
    // as soon as the Z stage has consumed the current window, so their HBM
    // latency hides behind the Y and X stages.
    // ring offset from the shared base (integer math keeps the shared address
    // space visible to the compiler: LDS with 32-bit addressing, not generic loads)
    const size_t ring_off = ((size_t)(reinterpret_cast<unsigned char *>(c0 + m) - smem) + 15) & ~(size_t)15;
    float *ring = reinterpret_cast<float *>(smem + ring_off);
    uint64_t *bar = reinterpret_cast<uint64_t *>(ring + (size_t)kRing * zstride);
    const uint32_t plane_bytes = (uint32_t)(zstride * sizeof(float));
    if (threadIdx.x == 0) {
        for (int r = 0; r < kRing; r++) mbar_init(bar + r, 1);
        fence_mbar_init();
    }
    __syncthreads();
    // planes are loaded in order from zbase, each exactly once: plane z is the
    // ((z - zbase) / kRing)-th load into slot (z - zbase) % kRing (its mbarrier phase)
    const int zbase = c0[k0];
    const int zlast = min(n - 1, c0[k1 - 1] + P);
    int issued = zbase - 1;  // highest plane whose load was issued (thread 0)
    // issue the loads of planes (issued, zmax]; a slot is recycled only after
    // every thread passed the barrier behind the z stage that last read it
    auto issue_upto = [&](int zmax) {
        fence_proxy_async();  // earlier generic reads of recycled slots before the async writes
        for (int z = issued + 1; z <= zmax; z++) {
            uint64_t *bz_ = bar + ((z - zbase) % kRing);
            mbar_arrive_expect_tx(bz_, plane_bytes);
            tma_load_1d(ring + (size_t)((z - zbase) % kRing) * zstride, C + (size_t)z * zstride, plane_bytes, bz_);
        }
        issued = max(issued, zmax);
    };
    if (threadIdx.x == 0) issue_upto(min(zlast, zbase + P));
    for (int k = k0; k < k1; k++) {
        const int z0 = c0[k];
        T bz[P + 1];
#pragma unroll
        for (int c = 0; c < P + 1; c++) bz[c] = B[k * 4 + c];
        const float *planes[P + 1];
#pragma unroll
        for (int c = 0; c < P + 1; c++) {
            const int zr = z0 + c - zbase;
            mbar_wait(bar + (zr % kRing), (uint32_t)((zr / kRing) & 1));
            planes[c] = ring + (size_t)(zr % kRing) * zstride;
        }
        // z contraction, 4 consecutive x per item: S1[b][a..a+3] = sum_c Bz[k,c] C[a.., b, z0+c];
        // thread (group g, quad q) takes rows b = g, g + groups, ... (no per-item division)
        if (g_ < groups)
            for (int off = g_ * pitch + 4 * q_; off < n * pitch; off += gstride) {
                T acc[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
                for (int c = 0; c < Q; c++) fma4(bz[c], *reinterpret_cast<const float4 *>(planes[c] + off), acc);
                st4(S1 + off, acc);
            }
        __syncthreads();
        // the ring planes below the next window are free now: fetch the next
        // window while the y and x stages run (kRing = P+1 slots suffice)
        if (threadIdx.x == 0 && k + 1 < k1) issue_upto(min(zlast, c0[k + 1] + P));
        // y contraction: S2[j][a..a+3] = sum_b By[j,b] S1[y0_j+b][a..a+3]
        if (g_ < groups)
            for (int j = g_; j < m; j += groups) {
                const T *s1 = S1 + c0[j] * pitch + 4 * q_;
                T acc[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
                for (int bb = 0; bb < Q; bb++) fma4(B[j * 4 + bb], s1 + bb * pitch, acc);
                st4(S2 + j * pitch + 4 * q_, acc);
            }
        __syncthreads();
        // x contraction + coalesced store out[i + m*j + m*m*k]: full-warp columns
        // i = lane + 32t with their Bx rows in registers, then the m % 32 tail
        float *outk = out + (size_t)k * m * m;
        if constexpr (sizeof(T) == 4) {
            if (ngroups == 2) {  // m in [64, 95]: both column groups in one paired FMA chain (FFMA2)
                for (int j = warp; j < m; j += nwarp) {
                    const float *s2 = reinterpret_cast<const float *>(S2) + (size_t)j * pitch;
                    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
                    for (int a = 0; a < Q; a++)
                        acc = __ffma2_rn(make_float2(bx[0][a], bx[1][a]), make_float2(s2[xi[0] + a], s2[xi[1] + a]),
                                         acc);
                    float *orow = outk + (size_t)j * m;
                    orow[lane] = acc.x;
                    orow[lane + 32] = acc.y;
                }
            }
        }
        for (int j = warp; j < m; j += nwarp) {
            if (sizeof(T) == 4 && ngroups == 2) break;  // done above
            const T *s2 = S2 + (size_t)j * pitch;
            float *orow = outk + (size_t)j * m;
#pragma unroll
            for (int t = 0; t < kMainGroups; t++) {
                if (t < ngroups) {
                    T acc = T(0);
#pragma unroll
                    for (int a = 0; a < Q; a++) acc = fma(bx[t][a], s2[xi[t] + a], acc);
                    orow[lane + 32 * t] = (float)acc;
                }
            }
        }
        for (int item = tid; item < m * tailw; item += nth) {
            const int j = (int)(((float)item + 0.5f) * inv_tail), i = mainw + (item - j * tailw);
            const T *s2 = S2 + (size_t)j * pitch + c0[i];
            T acc = T(0);
#pragma unroll
            for (int a = 0; a < Q; a++) acc = fma(B[i * 4 + a], s2[a], acc);
            outk[(size_t)j * m + i] = (float)acc;
        }
        __syncthreads();
    }
    // drain: planes loaded but never read (z0 jumping by more than one when m < nspan)
    // must land before the CTA's shared memory is released
    if (threadIdx.x == 0)
        for (int z = max(zbase, issued - kRing + 1); z <= issued; z++)
            mbar_wait(bar + ((z - zbase) % kRing), (uint32_t)(((z - zbase) / kRing) & 1));
}

// One instantiation per arithmetic type so the float kernel is not sized
// (registers, shared memory) for the float64 path; a CTA whose block has the
// other precision exits at once.
template <typename T>
__global__ void __launch_bounds__(kDecodeThreads) decode_grid_kernel(const BlockDesc *__restrict__ descs,
                                                                      const DecodeJob *__restrict__ jobs, int m,
                                                                      float *__restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem[];
    const DecodeJob jb = jobs[blockIdx.y];
    const BlockDesc d = descs[jb.slot];
    constexpr bool kF64 = sizeof(T) == 8;
    if (jb.any) return;  // decode_any_kernel
    if (((d.flags & AFAM_SLOT_FP64) != 0) != kF64) return;
    if (!kF64 && jb.tc_kp > 0) return;  // decoded by decode_tc_kernel
    if (!kF64 && jb.fx) return;         // decoded by decode_fx_kernel
    const int k0 = blockIdx.x * kDecodeChunk;
    const int k1 = min(m, k0 + kDecodeChunk);
    float *o = out + (size_t)blockIdx.y * m * m * m;
    const T *b;
    if constexpr (kF64) b = jb.b64; else b = jb.b32;
    switch (d.deg) {
        case 1: decode_planes<1, T>(d, jb.col0, b, m, k0, k1, o, smem); break;
        case 2: decode_planes<2, T>(d, jb.col0, b, m, k0, k1, o, smem); break;
        default: decode_planes<3, T>(d, jb.col0, b, m, k0, k1, o, smem); break;
    }
}


// ---------------------------------------------------------------------------
// Register-tiled grid decode (float32 slots, m == 65, ncp <= 65): the
// default CUDA-core path.  One CTA per block, the control-point z-planes
// streaming through a ring of kFxRing shared slots by TMA bulk copies;
// per input plane zc, in one pass and with one CTA barrier:
//   x stage: X[r][x] = sum_a Bx[x][a] C[zc][r][x0(x)+a] for every control row
//     r and lattice column x < 64 -- thread (row set, x quad q) reads the
//     12-float aligned window of its quad (3 LDS.128) and applies a dense
//     4 x 12 weight block held in registers (zeros off the band), one
//     16-byte store into the double-buffered X plane;
//   y stage: Y[y][x] = sum_b By[y][b] X[y0(y)+b][x] -- thread (q, g) owns
//     lattice rows y = 4g..4g+3 and columns x = q, q+16, q+32, q+48 (lanes
//     read consecutive words: conflict-free), a dense 4 x 7 window of By in
//     registers; the 16 results go into a register ring of the last 4 planes;
//   z stage: every output plane k whose last support plane is zc
//     (col0[k] + p == zc) is sum_c Bz[k][c] Y_{col0[k]+c}, read from the
//     register ring, and stored (16 lanes write 16 consecutive x).
// The lattice's last row/column (u = 1) selects the last control index
// exactly (checked on the host), so X[.][64] is the control column ncp-1 and
// Y[64][.] the X row ncp-1: threads 0..128 carry one such value each
// (threads 0..15 also take the x stage's control row 64).  Control points are read once from HBM (TMA), the
// output written once; x and y run out of registers and one X plane.
#ifndef AFAM_FX_RING
#define AFAM_FX_RING 4
#endif
constexpr int kFxRing = AFAM_FX_RING;  // TMA plane slots (-DAFAM_FX_RING for A/B)
constexpr int kFxXPitch = 68;    // X plane row pitch (floats)
constexpr int kFxXRows = 72;     // X plane rows (the y windows over-read up to row ncp + 4, zeros)
constexpr int kFxPad = 16;       // zero floats after each ring slot (x windows over-read the last row)


// SMW: the x / y weight windows live in shared memory instead of registers
// and the plane ring has 3 slots, so two CTAs fit on an SM (<= 128 registers,
// <= 113 KB of shared memory each): 16 warps instead of 8 to hide the
// latency-bound plane loop.
template <int P, int YPT, bool SMW>
__device__ __forceinline__ void fx_decode_block(const BlockDesc &d, const int32_t *__restrict__ c0g,
                                                const float *__restrict__ Bg, float *__restrict__ out,
                                                unsigned char *smem) {
    constexpr int Q = P + 1;
    constexpr int RING = SMW ? 3 : kFxRing;
    constexpr int M = 65;
    const int n = d.ncp, pitch = d.pitch;
    const int sstride = n * pitch + kFxPad;
    float *ring = reinterpret_cast<float *>(smem);
    float *xb = ring + RING * sstride;
    float *Bs = xb + 2 * kFxXRows * kFxXPitch;
    int *c0 = reinterpret_cast<int *>(Bs + M * 4);
    float *xcol = reinterpret_cast<float *>(c0 + 68);  // 2 x 72: X[.][64] = control column n-1, contiguous
    float4 *wxs = reinterpret_cast<float4 *>(xcol + 2 * 72);  // SMW: [10][16] x weights, (w0..w3)[e] per quad
    float4 *wys = wxs + (SMW ? 10 * 16 : 0);                  // SMW: [YW][NG] y weights, (wy[0..3])[e] per group
    uint64_t *bar = reinterpret_cast<uint64_t *>(wys + (SMW ? (YPT + 3) * (16 * 64 / YPT / 16) : 0));
    const int tid = threadIdx.x;

    for (int i = tid; i < M * 4; i += blockDim.x) Bs[i] = Bg[i];
    for (int i = tid; i < M; i += blockDim.x) c0[i] = c0g[i];
    for (int i = tid; i < RING * kFxPad; i += blockDim.x)
        ring[(i / kFxPad) * sstride + n * pitch + (i % kFxPad)] = 0.f;
    for (int i = tid; i < 2 * (kFxXRows - n) * kFxXPitch; i += blockDim.x) {
        const int b = i / ((kFxXRows - n) * kFxXPitch), o = i % ((kFxXRows - n) * kFxXPitch);
        xb[b * kFxXRows * kFxXPitch + n * kFxXPitch + o] = 0.f;
    }
    if (tid == 0) {
        for (int r = 0; r < RING; r++) mbar_init(bar + r, 1);
        fence_mbar_init();
    }
    __syncthreads();
    const float *__restrict__ C = d.ctrl;
    const uint32_t plane_bytes = (uint32_t)((size_t)n * pitch * sizeof(float));
    if (tid == 0) {
        fence_proxy_async();
        for (int z = 0; z < min(n, RING); z++) {
            mbar_arrive_expect_tx(bar + z, plane_bytes);
            tma_load_1d(ring + (size_t)z * sstride, C + (size_t)z * n * pitch, plane_bytes, bar + z);
        }
    }

    // x stage weights: quad q (lattice columns 4q..4q+3) over the aligned
    // 12-float window starting at cw (dense, zeros off the band)
    // YPT lattice rows per thread: 16 x lanes x (64 / YPT) row groups
    constexpr int NT = 16 * 64 / YPT, NG = NT / 16, YW = YPT + 3;
    const int q = tid & 15, g = tid >> 4;
    const int cw = c0[4 * q] & ~3;
    auto wx_at = [&](int xi, int e) {
        const int x = 4 * q + xi, a = e - (c0[x] - cw);
        return (a >= 0 && a < Q) ? Bs[x * 4 + a] : 0.f;
    };
    // y stage weights: rows 4g..4g+3 over the 7-row window starting at r0
    const int r0 = c0[YPT * g];
    auto wy_at = [&](int yi, int e) {
        const int y = YPT * g + yi, b = e - (c0[y] - r0);
        return (b >= 0 && b < Q) ? Bs[y * 4 + b] : 0.f;
    };
    float wx[SMW ? 1 : 4][SMW ? 1 : 10];
    float wy[SMW ? 1 : YPT][SMW ? 1 : YW];
    if constexpr (SMW) {
        if (g == 0)
            for (int e = 0; e < 10; e++) wxs[e * 16 + q] = make_float4(wx_at(0, e), wx_at(1, e), wx_at(2, e), wx_at(3, e));
        if (q == 0)
            for (int e = 0; e < YW; e++)
                wys[e * NG + g] = make_float4(wy_at(0, e), YPT > 1 ? wy_at(1, e) : 0.f, YPT > 2 ? wy_at(2, e) : 0.f,
                                              YPT > 3 ? wy_at(3, e) : 0.f);
        __syncthreads();  // the weight windows before plane 0's x stage reads them
    } else {
#pragma unroll
        for (int xi = 0; xi < 4; xi++)
#pragma unroll
            for (int e = 0; e < 10; e++) wx[xi][e] = wx_at(xi, e);
#pragma unroll
        for (int yi = 0; yi < YPT; yi++)
#pragma unroll
            for (int e = 0; e < YW; e++) wy[yi][e] = wy_at(yi, e);
    }
    float yr[4][YPT][4];  // [plane slot][yi][s]: Y of the last 4 planes, columns q + 16 s
    float er[4];        // threads 0..128: the lattice column x = 64 / row y = 64 value of the last 4 planes
    int knext = 0;

    // x stage of plane z into X plane z & 1 (ring slot z & 3)
    auto xstage = [&](int z) {
        mbar_wait(bar + (z % RING), (uint32_t)((z / RING) & 1));
        const float *Cp = ring + (z % RING) * sstride;
        float *X = xb + (z & 1) * kFxXRows * kFxXPitch;
                // ---- x stage: rows g + 16 i two at a time (four independent FFMA2
                // chains), threads 0..15 also take control row 64; window
                // entries 10, 11 never carry weight (offsets <= 3 + 3, p <= 3)
#pragma unroll
                for (int i = 0; i < 64 / NG; i += 2) {
                    const int ra = g + NG * i, rb = ra + NG;
                    const float4 *sa = reinterpret_cast<const float4 *>(Cp + min(ra, n - 1) * pitch + cw);
                    const float4 *sb = reinterpret_cast<const float4 *>(Cp + min(rb, n - 1) * pitch + cw);
                    const float4 a0 = sa[0], a1 = sa[1], a2 = sa[2], b0 = sb[0], b1 = sb[1], b2 = sb[2];
                    const float va[10] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w, a2.x, a2.y};
                    const float vb[10] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w, b2.x, b2.y};
                    // even / odd taps in separate chains: eight independent FFMA2 chains of 5
                    float2 pa01 = make_float2(0.f, 0.f), pa23 = pa01, pb01 = pa01, pb23 = pa01;
                    float2 qa01 = pa01, qa23 = pa01, qb01 = pa01, qb23 = pa01;
#pragma unroll
                    for (int e = 0; e < 10; e += 2) {
                        float4 w0, w1;  // (wx[0..3][e]), (wx[0..3][e + 1])
                        if constexpr (SMW) {
                            w0 = wxs[e * 16 + q];
                            w1 = wxs[(e + 1) * 16 + q];
                        } else {
                            w0 = make_float4(wx[0][e], wx[1][e], wx[2][e], wx[3][e]);
                            w1 = make_float4(wx[0][e + 1], wx[1][e + 1], wx[2][e + 1], wx[3][e + 1]);
                        }
                        pa01 = __ffma2_rn(make_float2(w0.x, w0.y), make_float2(va[e], va[e]), pa01);
                        pa23 = __ffma2_rn(make_float2(w0.z, w0.w), make_float2(va[e], va[e]), pa23);
                        pb01 = __ffma2_rn(make_float2(w0.x, w0.y), make_float2(vb[e], vb[e]), pb01);
                        pb23 = __ffma2_rn(make_float2(w0.z, w0.w), make_float2(vb[e], vb[e]), pb23);
                        qa01 = __ffma2_rn(make_float2(w1.x, w1.y), make_float2(va[e + 1], va[e + 1]), qa01);
                        qa23 = __ffma2_rn(make_float2(w1.z, w1.w), make_float2(va[e + 1], va[e + 1]), qa23);
                        qb01 = __ffma2_rn(make_float2(w1.x, w1.y), make_float2(vb[e + 1], vb[e + 1]), qb01);
                        qb23 = __ffma2_rn(make_float2(w1.z, w1.w), make_float2(vb[e + 1], vb[e + 1]), qb23);
                    }
                    pa01 = __fadd2_rn(pa01, qa01);
                    pa23 = __fadd2_rn(pa23, qa23);
                    pb01 = __fadd2_rn(pb01, qb01);
                    pb23 = __fadd2_rn(pb23, qb23);
                    if (ra < n) *reinterpret_cast<float4 *>(X + ra * kFxXPitch + 4 * q) = make_float4(pa01.x, pa01.y, pa23.x, pa23.y);
                    if (rb < n) *reinterpret_cast<float4 *>(X + rb * kFxXPitch + 4 * q) = make_float4(pb01.x, pb01.y, pb23.x, pb23.y);
                }
                if (g == NG - 1 && n > 64) {  // control row 64 (the last row group: the edge values sit on warps 0..4)
                    const float4 *src = reinterpret_cast<const float4 *>(Cp + 64 * pitch + cw);
                    const float4 v0 = src[0], v1 = src[1], v2 = src[2];
                    const float w[10] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w, v2.x, v2.y};
                    float2 a01 = make_float2(0.f, 0.f), a23 = make_float2(0.f, 0.f);
#pragma unroll
                    for (int e = 0; e < 10; e++) {
                        const float4 we = SMW ? wxs[e * 16 + q] : make_float4(wx[0][e], wx[1][e], wx[2][e], wx[3][e]);
                        a01 = __ffma2_rn(make_float2(we.x, we.y), make_float2(w[e], w[e]), a01);
                        a23 = __ffma2_rn(make_float2(we.z, we.w), make_float2(w[e], w[e]), a23);
                    }
                    *reinterpret_cast<float4 *>(X + 64 * kFxXPitch + 4 * q) = make_float4(a01.x, a01.y, a23.x, a23.y);
                }
                if (tid < n) xcol[(z & 1) * 72 + tid] = Cp[tid * pitch + n - 1];  // u = 1 column: control column n-1
    };
    // software pipeline over the planes, one barrier per plane: the x stage
    // of plane zc + 1 runs beside the y / z stages of plane zc (different X
    // buffers), so each warp has two independent instruction streams
    xstage(0);
    __syncthreads();
    if (tid == 0 && RING < n) {  // slot 0 is free: plane 0's x stage is done
        fence_proxy_async();
        mbar_arrive_expect_tx(bar, plane_bytes);
        tma_load_1d(ring, C + (size_t)RING * n * pitch, plane_bytes, bar);
    }
    for (int z0 = 0; z0 < n; z0 += 4) {
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const int zc = z0 + u;
            if (zc >= n) break;
            if (zc + 1 < n) xstage(zc + 1);
            const float *X = xb + (u & 1) * kFxXRows * kFxXPitch;
            // ---- y stage (into the register ring)
#pragma unroll
            for (int yi = 0; yi < YPT; yi++)
#pragma unroll
                for (int s = 0; s < 4; s++) yr[u][yi][s] = 0.f;
#pragma unroll
            for (int e = 0; e < YW; e++) {
                const float *xr = X + (r0 + e) * kFxXPitch + q;
                const float v[4] = {xr[0], xr[16], xr[32], xr[48]};
                float we[YPT];
                if constexpr (SMW) {
                    const float4 w4 = wys[e * NG + g];
                    const float wa[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
                    for (int yi = 0; yi < YPT; yi++) we[yi] = wa[yi];
                } else {
#pragma unroll
                    for (int yi = 0; yi < YPT; yi++) we[yi] = wy[yi][e];
                }
#pragma unroll
                for (int yi = 0; yi < YPT; yi++) {
                    float2 lo = make_float2(yr[u][yi][0], yr[u][yi][1]), hi = make_float2(yr[u][yi][2], yr[u][yi][3]);
                    lo = __ffma2_rn(make_float2(we[yi], we[yi]), make_float2(v[0], v[1]), lo);
                    hi = __ffma2_rn(make_float2(we[yi], we[yi]), make_float2(v[2], v[3]), hi);
                    yr[u][yi][0] = lo.x; yr[u][yi][1] = lo.y; yr[u][yi][2] = hi.x; yr[u][yi][3] = hi.y;
                }
            }
            // lattice column x = 64 (threads 0..64: y = tid) and row y = 64 (threads 65..128: x = tid - 65)
            if (tid <= 64) {
                float acc = 0.f;
                if (tid == 64) {
                    acc = xcol[(u & 1) * 72 + n - 1];
                } else {
#pragma unroll
                    for (int b = 0; b < Q; b++) acc = fmaf(Bs[tid * 4 + b], xcol[(u & 1) * 72 + c0[tid] + b], acc);
                }
                er[u] = acc;
            } else if (tid < 129) {
                er[u] = X[(n - 1) * kFxXPitch + tid - 65];
            }
            // ---- z stage: output planes whose support ends at zc
            while (knext < M && c0[knext] + P == zc) {
                const int k = knext++;
                float wz[Q];
#pragma unroll
                for (int c = 0; c < Q; c++) wz[c] = Bs[k * 4 + c];
                float *ok = out + (size_t)k * M * M;
#pragma unroll
                for (int yi = 0; yi < YPT; yi++) {
                    float2 lo = make_float2(0.f, 0.f), hi = make_float2(0.f, 0.f);
#pragma unroll
                    for (int c = 0; c < Q; c++) {
                        const int sl = (u - P + c) & 3;
                        lo = __ffma2_rn(make_float2(wz[c], wz[c]), make_float2(yr[sl][yi][0], yr[sl][yi][1]), lo);
                        hi = __ffma2_rn(make_float2(wz[c], wz[c]), make_float2(yr[sl][yi][2], yr[sl][yi][3]), hi);
                    }
                    float *orow = ok + (YPT * g + yi) * M + q;
                    orow[0] = lo.x;
                    orow[16] = lo.y;
                    orow[32] = hi.x;
                    orow[48] = hi.y;
                }
                if (tid < 129) {
                    float acc = 0.f;
#pragma unroll
                    for (int c = 0; c < Q; c++) acc = fmaf(wz[c], er[(u - P + c) & 3], acc);
                    ok[tid <= 64 ? tid * M + 64 : 64 * M + tid - 65] = acc;
                }
            }
            __syncthreads();
            // plane zc + 1's slot is free (its x stage is done): fetch plane zc + 1 + kFxRing
            if (tid == 0 && zc + 1 + RING < n) {
                const int sl = (zc + 1) % RING;
                fence_proxy_async();
                mbar_arrive_expect_tx(bar + sl, plane_bytes);
                tma_load_1d(ring + (size_t)sl * sstride, C + (size_t)(zc + 1 + RING) * n * pitch, plane_bytes,
                            bar + sl);
            }
        }
    }
}

template <int YPT, bool SMW>
__global__ void __launch_bounds__(16 * 64 / YPT, SMW ? 2 : 1) decode_fx_kernel(const BlockDesc *__restrict__ descs,
                                                                                const DecodeJob *__restrict__ jobs,
                                                                                float *__restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem[];
    const DecodeJob jb = jobs[blockIdx.x];
    if (!jb.fx) return;
    const BlockDesc d = descs[jb.slot];
    if (d.flags & AFAM_SLOT_FP64) return;  // float64 slots: decode_grid_kernel<double>
    float *o = out + (size_t)blockIdx.x * 65 * 65 * 65;
    switch (d.deg) {
        case 1: fx_decode_block<1, YPT, SMW>(d, jb.col0, jb.b32, o, smem); break;
        case 2: fx_decode_block<2, YPT, SMW>(d, jb.col0, jb.b32, o, smem); break;
        default: fx_decode_block<3, YPT, SMW>(d, jb.col0, jb.b32, o, smem); break;
    }
}

// ---------------------------------------------------------------------------
// Tensor-core grid decode (m == 65, float32 slots).  Per output plane k:
//   z stage (CUDA cores): S1[y][x] = sum_c Bz[k][c] C[z0+c][y][x] over the
//     TMA plane ring (as above);
//   y stage (CUDA cores): S2[j][x] = sum_b By[j][b] S1[y0_j+b][x] for
//     j < 64, split into tf32 hi/lo and stored as the A operand (64 rows,
//     K = x, K-major no-swizzle panels);
//   x stage (tcgen05, kind::tf32, 3xTF32): D[j][i] = sum_x S2[j][x] Bx[i][x]
//     for i < 64 -- one 64x64 accumulator in TMEM per plane, K = ncp
//     rounded up to 8, D += A_hi B_hi + A_lo B_hi + A_hi B_lo;
//   the last lattice row and column (u = 1) select the last control index
//   exactly (B row m-1 = e_{ncp-1}, checked on the host), so out[k][j][64]
//   = S2[j][ncp-1] and out[k][64][i] = x-contraction of S1[ncp-1] come from
//   the CUDA-core stages.
// Warp-specialised pipeline over the planes: 12 producer warps (z and y
// stages, A operand), one MMA warp (a single thread issues the tcgen05.mma
// chain of a plane and commits it to an mbarrier), 4 epilogue warps (TMEM ->
// shared staging -> 16-byte global stores).  A operands, TMEM accumulators
// and the u = 1 row/column buffers are double-buffered; mbarriers hand each
// buffer between the roles (A_full: producers -> MMA; D_full: MMA ->
// epilogue and producers (A free); E_done: epilogue -> MMA (TMEM free) and
// producers (row/column buffers free)).
constexpr int kTcProducerWarps = 12;
constexpr int kTcMmaWarp = kTcProducerWarps;
constexpr int kTcEpiWarp0 = kTcProducerWarps + 1;
constexpr int kTcThreads = 32 * (kTcProducerWarps + 1 + 4);  // 544
constexpr int kTcRows = 64;      // tensor-core rows / columns per plane (m - 1)
constexpr int kTcKmax = 72;      // ncp <= 72

struct TcSmem {  // byte offsets of the dynamic shared memory carve-up
    size_t bs, a, ring, s1, stage, band, col0, xlast, row64, bar, tmem, total;
};

__host__ __device__ inline size_t tc_align(size_t v, size_t a) { return (v + a - 1) / a * a; }

__host__ __device__ inline TcSmem tc_smem(int n, int kp, int m) {
    const int pitch = (n + 3) & ~3;
    TcSmem o;
    size_t off = 0;
    o.bs = off;    off += 2 * (size_t)kTcRows * kp * 4;         // basis hi, lo
    o.a = off;     off += 2 * 2 * (size_t)kTcRows * kp * 4;     // 2 buffers x (hi, lo)
    o.ring = off;  off += (size_t)kRing * n * pitch * 4;        // TMA plane ring
    o.s1 = off;    off += (size_t)n * pitch * 4;
    o.stage = off; off += tc_align((size_t)m * m * 4 + 16, 16); // output plane (+ alignment shift)
    o.band = off;  off += (size_t)m * 4 * 4;
    o.col0 = off;  off += tc_align((size_t)m * 4, 16);
    o.xlast = off; off += 2 * kTcRows * 4;
    o.row64 = off; off += tc_align(2 * (size_t)m * 4, 16);
    o.bar = off;   off += (kRing + 6) * 8;
    o.tmem = off;  off += 16;
    o.total = off;
    return o;
}

__device__ __forceinline__ void named_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int P>
__device__ __forceinline__ void tc_decode_block(const BlockDesc &d, const DecodeJob &jb, int m, float *__restrict__ out,
                                                size_t out_off, unsigned char *smem) {
    constexpr int Q = P + 1;
    const int n = d.ncp, pitch = d.pitch, nq = pitch >> 2, kp = jb.tc_kp, kq = kp >> 2;
    const TcSmem L = tc_smem(n, kp, m);
    float *Bs = reinterpret_cast<float *>(smem + L.bs);
    float *Abuf = reinterpret_cast<float *>(smem + L.a);
    float *ring = reinterpret_cast<float *>(smem + L.ring);
    float *S1 = reinterpret_cast<float *>(smem + L.s1);
    float *stage = reinterpret_cast<float *>(smem + L.stage);
    float *B = reinterpret_cast<float *>(smem + L.band);
    int *c0 = reinterpret_cast<int *>(smem + L.col0);
    float *xlast = reinterpret_cast<float *>(smem + L.xlast);
    float *row64 = reinterpret_cast<float *>(smem + L.row64);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + L.bar);
    uint64_t *ring_bar = bar, *a_full = bar + kRing, *d_full = a_full + 2, *e_done = d_full + 2;
    uint32_t *tmem_base = reinterpret_cast<uint32_t *>(smem + L.tmem);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const size_t abytes = (size_t)kTcRows * kp * 4;  // one operand panel set (hi or lo)

    {  // basis operand (hi, lo) and the banded rows for the CUDA-core stages
        const float4 *src = reinterpret_cast<const float4 *>(jb.tc_b);
        float4 *dst = reinterpret_cast<float4 *>(Bs);
        for (int i = tid; i < 2 * kTcRows * kq; i += blockDim.x) dst[i] = src[i];
        for (int i = tid; i < m * 4; i += blockDim.x) B[i] = jb.b32[i];
        for (int i = tid; i < m; i += blockDim.x) c0[i] = jb.col0[i];
    }
    if (tid == 0) {
        for (int r = 0; r < kRing + 6; r++) mbar_init(bar + r, 1);
        fence_mbar_init();
    }
    if (warp == 0) umma::tmem_alloc(tmem_base, 128);
    umma::fence_async_smem();
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tbase = *tmem_base;

    if (warp < kTcProducerWarps) {
        // ---------------- producers: z and y stages on the CUDA cores
        constexpr int NP = 32 * kTcProducerWarps;
        const float *__restrict__ C = d.ctrl;
        const size_t zstride = (size_t)n * pitch;
        const uint32_t plane_bytes = (uint32_t)(zstride * sizeof(float));
        const int zbase = c0[0];
        const int zlast = min(n - 1, c0[m - 1] + P);
        int issued = zbase - 1;
        auto issue_upto = [&](int zmax) {
            fence_proxy_async();
            for (int z = issued + 1; z <= zmax; z++) {
                uint64_t *bz_ = ring_bar + ((z - zbase) % kRing);
                mbar_arrive_expect_tx(bz_, plane_bytes);
                tma_load_1d(ring + (size_t)((z - zbase) % kRing) * zstride, C + (size_t)z * zstride, plane_bytes,
                            bz_);
            }
            issued = max(issued, zmax);
        };
        if (tid == 0) issue_upto(min(zlast, zbase + P));
        const float inv_nq = 1.f / (float)nq;
        for (int k = 0; k < m; k++) {
            const int b = k & 1, u = k >> 1;
            const int z0 = c0[k];
            float bz[Q];
#pragma unroll
            for (int c = 0; c < Q; c++) bz[c] = B[k * 4 + c];
            const float *planes[Q];
#pragma unroll
            for (int c = 0; c < Q; c++) {
                const int zr = z0 + c - zbase;
                mbar_wait(ring_bar + (zr % kRing), (uint32_t)((zr / kRing) & 1));
                planes[c] = ring + (size_t)(zr % kRing) * zstride;
            }
            // z stage: S1[y][x..x+3]
            for (int item = tid; item < n * nq; item += NP) {
                const int y = (int)(((float)item + 0.5f) * inv_nq), q = item - y * nq;
                float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int c = 0; c < Q; c++)
                    fma4(bz[c], *reinterpret_cast<const float4 *>(planes[c] + (size_t)y * pitch + 4 * q), acc);
                st4(S1 + (size_t)y * pitch + 4 * q, acc);
            }
            named_sync(1, NP);
            if (tid == 0 && k + 1 < m) issue_upto(min(zlast, c0[k + 1] + P));
            if (k >= 2) {  // buffer b: MMAs of plane k-2 done (A free), its epilogue done (row/col free)
                mbar_wait(d_full + b, (uint32_t)((u - 1) & 1));
                mbar_wait(e_done + b, (uint32_t)((u - 1) & 1));
            }
            // y stage into the A operand (rows j < 64, K = x; zero past ncp)
            float *Ah = Abuf + (size_t)b * 2 * kTcRows * kp, *Al = Ah + (size_t)kTcRows * kp;
            for (int item = tid; item < kTcRows * kq; item += NP) {
                const int q = item >> 6, j = item & (kTcRows - 1);
                float acc[4] = {0.f, 0.f, 0.f, 0.f};
                if (q < nq) {
                    const float *s1 = S1 + (size_t)c0[j] * pitch + 4 * q;
#pragma unroll
                    for (int bb = 0; bb < Q; bb++) fma4(B[j * 4 + bb], s1 + (size_t)bb * pitch, acc);
                    if (q == (n - 1) >> 2) xlast[b * kTcRows + j] = acc[(n - 1) & 3];
                }
                float hi[4], lo[4];
#pragma unroll
                for (int e = 0; e < 4; e++) umma::split_tf32(acc[e], hi[e], lo[e]);
                st4(Ah + (size_t)item * 4, hi);
                st4(Al + (size_t)item * 4, lo);
            }
            for (int i = tid; i < m; i += NP) {  // out[k][m-1][i]: x stage of S1[ncp-1] (= S2[m-1])
                const float *s = S1 + (size_t)(n - 1) * pitch + c0[i];
                float acc = 0.f;
#pragma unroll
                for (int a = 0; a < Q; a++) acc = fmaf(B[i * 4 + a], s[a], acc);
                row64[b * m + i] = acc;
            }
            umma::fence_async_smem();
            named_sync(1, NP);
            if (tid == 0) mbar_arrive(a_full + b);
        }
        // drain ring loads that were issued but never read
        if (tid == 0)
            for (int z = max(zbase, issued - kRing + 1); z <= issued; z++)
                mbar_wait(ring_bar + ((z - zbase) % kRing), (uint32_t)(((z - zbase) / kRing) & 1));
    } else if (warp == kTcMmaWarp) {
        // ---------------- MMA issue: x stage on the tensor core (3xTF32)
        if (lane == 0) {
            constexpr uint32_t idesc = umma::idesc_tf32(kTcRows, kTcRows);
            const uint32_t lbo = kTcRows * 16;
            const uint32_t bh = umma::smem_addr(Bs), bl = bh + (uint32_t)abytes;
            const uint64_t dbh0 = umma::desc_kmajor(bh, lbo, 128), dbl0 = umma::desc_kmajor(bl, lbo, 128);
            for (int k = 0; k < m; k++) {
                const int b = k & 1, u = k >> 1;
                mbar_wait(a_full + b, (uint32_t)(u & 1));
                if (k >= 2) mbar_wait(e_done + b, (uint32_t)((u - 1) & 1));  // TMEM buffer b drained
                umma::fence_after_sync();
                const uint32_t ah = umma::smem_addr(Abuf + (size_t)b * 2 * kTcRows * kp);
                const uint64_t dah0 = umma::desc_kmajor(ah, lbo, 128);
                const uint64_t dal0 = umma::desc_kmajor(ah + (uint32_t)abytes, lbo, 128);
                const uint32_t d_tmem = tbase + (uint32_t)(b * kTcRows);
                for (int ks = 0; ks < kp / 8; ks++) {
                    const uint64_t off = (uint64_t)((ks * 2 * lbo) >> 4);  // start-address field, 16-B units
                    umma::mma_tf32(d_tmem, dal0 + off, dbh0 + off, idesc, ks > 0);
                    umma::mma_tf32(d_tmem, dah0 + off, dbl0 + off, idesc, true);
                    umma::mma_tf32(d_tmem, dah0 + off, dbh0 + off, idesc, true);
                }
                umma::commit(d_full + b);
            }
        }
        __syncwarp();
    } else {
        // ---------------- epilogue: TMEM -> staging -> 16-byte global stores
        constexpr int NE = 128;
        const int et = tid - 32 * kTcEpiWarp0, sp = warp & 3;  // TMEM sub-partition of this warp
        for (int k = 0; k < m; k++) {
            const int b = k & 1, u = k >> 1;
            const size_t g0 = out_off + (size_t)k * m * m;
            const int r = (int)(g0 & 3);  // staging shift: stage[r + e] <-> out[g0 + e], 16-B aligned copies
            mbar_wait(d_full + b, (uint32_t)(u & 1));
            umma::fence_after_sync();
#pragma unroll
            for (int cg = 0; cg < 4; cg++) {  // M = 64 accumulator: row j in TMEM lane (j % 16) + 32 (j / 16)
                float v[16];
                umma::tmem_ld16(tbase + ((uint32_t)(32 * sp) << 16) + (uint32_t)(b * kTcRows + 16 * cg), v);
                if (lane < 16) {
                    float *row = stage + r + (size_t)(16 * sp + lane) * m + 16 * cg;
#pragma unroll
                    for (int c = 0; c < 16; c++) row[c] = v[c];
                }
            }
            for (int j = et; j < kTcRows; j += NE) stage[r + (size_t)j * m + kTcRows] = xlast[b * kTcRows + j];
            for (int i = et; i < m; i += NE) stage[r + (size_t)kTcRows * m + i] = row64[b * m + i];
            umma::fence_before_sync();
            named_sync(2, NE);
            if (et == 0) mbar_arrive(e_done + b);
            float *o = out + g0;
            const int total = m * m, h = (4 - r) & 3;
            for (int e = et; e < h; e += NE) o[e] = stage[r + e];
            const int nv = (total - h) >> 2;
            for (int v = et; v < nv; v += NE)
                reinterpret_cast<float4 *>(o + h)[v] = reinterpret_cast<const float4 *>(stage + r + h)[v];
            for (int e = h + 4 * nv + et; e < total; e += NE) o[e] = stage[r + e];
            named_sync(2, NE);  // staging free for the next plane
        }
    }
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    if (warp == 0) umma::tmem_dealloc(tbase, 128);
}

__global__ void __launch_bounds__(kTcThreads, 1) decode_tc_kernel(const BlockDesc *__restrict__ descs,
                                                                 const DecodeJob *__restrict__ jobs, int m,
                                                                 float *__restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem[];
    const DecodeJob jb = jobs[blockIdx.x];
    if (jb.tc_kp == 0) return;  // no tensor-core operator: CUDA-core path
    const BlockDesc d = descs[jb.slot];
    if (d.flags & AFAM_SLOT_FP64) return;  // ill-conditioned: float64 CUDA-core path
    const size_t off = (size_t)blockIdx.x * m * m * m;
    switch (d.deg) {
        case 1: tc_decode_block<1>(d, jb, m, out, off, smem); break;
        case 2: tc_decode_block<2>(d, jb, m, out, off, smem); break;
        default: tc_decode_block<3>(d, jb, m, out, off, smem); break;
    }
}

// Degrees above AFAM_FAST_DEGREE (any slot flags): the separable decode of
// bspline.py:162-172 evaluated per lattice point in float64, out[k][j][i] =
// sum_c Bz[k][c] sum_b By[j][b] sum_a Bx[i][a] C[x0+a][y0+b][z0+c] with the
// banded float64 collocation rows of host_band (stride deg + 1).  One thread
// per output; a correctness path (such degrees are rare), not a tuned one.
__global__ void decode_any_kernel(const BlockDesc *__restrict__ descs, const DecodeJob *__restrict__ jobs, int m,
                                  float *__restrict__ out) {
    const DecodeJob jb = jobs[blockIdx.y];
    if (!jb.any) return;
    const BlockDesc d = descs[jb.slot];
    const int p = d.deg, Q = p + 1;
    const int64_t mm = (int64_t)m * m, total = mm * m;
    float *o = out + (size_t)blockIdx.y * total;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(e % m), j = (int)((e / m) % m), k = (int)(e / mm);
        const double *bx = jb.b64 + (size_t)i * Q, *by = jb.b64 + (size_t)j * Q, *bz = jb.b64 + (size_t)k * Q;
        const int x0 = __ldg(jb.col0 + i), y0 = __ldg(jb.col0 + j), z0 = __ldg(jb.col0 + k);
        double v = 0.0;
        for (int c = 0; c < Q; c++) {
            double ay = 0.0;
            for (int b = 0; b < Q; b++) {
                const float *row = d.ctrl + ((size_t)(z0 + c) * d.ncp + (y0 + b)) * d.pitch + x0;
                double ax = 0.0;
                for (int a = 0; a < Q; a++) ax = fma(__ldg(bx + a), (double)__ldg(row + a), ax);
                ay = fma(__ldg(by + b), ax, ay);
            }
            v = fma(__ldg(bz + c), ay, v);
        }
        o[e] = (float)v;
    }
}

// Host: the banded rows of bspline._axis_operator's B for (ncp, deg, m):
// params linspace(0, 1, m), clamped uniform float64 knots
// (bspline.py:29-38, :98-125), Cox-de Boor with the reference's divisors.
void host_band(int ncp, int deg, int m, std::vector<double> &b, std::vector<int32_t> &col0) {
    const int nk = ncp + deg + 1;
    std::vector<double> kv(nk);
    for (int i = 0; i <= deg; i++) kv[i] = 0.0;
    for (int i = 1; i < ncp - deg; i++) kv[deg + i] = (double)i / (double)(ncp - deg);
    for (int i = 0; i <= deg; i++) kv[ncp + i] = 1.0;
    const int bs = band_stride(deg);
    b.assign((size_t)m * bs, 0.0);
    col0.assign(m, 0);
    const double step = m > 1 ? 1.0 / (double)(m - 1) : 0.0;
    for (int i = 0; i < m; i++) {
        double u = (double)i * step;
        if (m > 1 && i == m - 1) u = 1.0;
        int s = (int)(std::upper_bound(kv.begin(), kv.end(), u) - kv.begin()) - 1;
        s = std::min(std::max(s, deg), ncp - 1);
        double N[AFAM_MAX_DEGREE + 1], left[AFAM_MAX_DEGREE + 1], right[AFAM_MAX_DEGREE + 1];
        N[0] = 1.0;
        for (int j = 1; j <= deg; j++) {
            left[j] = u - kv[s + 1 - j];
            right[j] = kv[s + j] - u;
            double saved = 0.0;
            for (int r = 0; r < j; r++) {
                double tmp = N[r] / (right[r + 1] + left[j - r]);
                N[r] = saved + right[r + 1] * tmp;
                saved = left[j - r] * tmp;
            }
            N[j] = saved;
        }
        col0[i] = s - deg;
        for (int j = 0; j <= deg; j++) b[(size_t)i * bs + j] = N[j];
    }
}

}  // namespace afam

using namespace afam;

// AFAM_DECODE_AUTO picks the tensor-core decode only with AFAM_DECODE_TC=1
// in the environment: the banded CUDA-core kernel is faster on B200 (the
// dense 3xTF32 operands move more shared-memory bytes per plane than the
// banded x stage, K3).
static bool tc_default() {
    static const bool v = [] {
        const char *e = getenv("AFAM_DECODE_TC");
        return e && atoi(e) != 0;
    }();
    return v;
}

// AFAM_DECODE_FX=0: the banded smem-staged kernel for float32 slots instead
// of the register-tiled one (A/B checks)
static bool fx_disabled() {
    static const bool v = [] {
        const char *e = getenv("AFAM_DECODE_FX");
        return e && atoi(e) == 0;
    }();
    return v;
}

// lattice rows per thread of the register-tiled decode (AFAM_DECODE_FX_YPT=2|4 A/B)
static int fx_ypt() {
    static const int v = [] {
        const char *e = getenv("AFAM_DECODE_FX_YPT");
        return (e && atoi(e) == 2) ? 2 : 4;
    }();
    return v;
}

// AFAM_DECODE_FX_SMW=1: the two-CTAs-per-SM variant (measured slower: 2.42 vs
// 2.13 ms on config 5 -- 16 warps raise issue only from 31% to 34%, the
// plane loop is bound by the L1/shared-memory pipe, which the weight loads
// load further)
static bool fx_smw() {
    static const bool v = [] {
        const char *e = getenv("AFAM_DECODE_FX_SMW");
        return e && atoi(e) != 0;
    }();
    return v;
}

static int get_op(afam_store *s, int ncp, int deg, int m, DecodeOp **op) {
    auto key = std::make_tuple(ncp, deg, m);
    auto it = s->ops.find(key);
    if (it == s->ops.end()) {
        std::vector<double> b;
        std::vector<int32_t> c0;
        host_band(ncp, deg, m, b, c0);
        std::vector<float> b32(b.begin(), b.end());
        DecodeOp o;
        // tensor-core operator: m == 65, ncp <= 72, and the u = 1 row selecting
        // the last control point exactly (what lets the CUDA-core stages supply
        // lattice row/column m-1)
        o.any = deg > AFAM_FAST_DEGREE;
        if (!o.any && m == kTcRows + 1 && ncp <= kTcKmax) {
            // (in float32, as the CUDA-core kernels apply it: Cox-de Boor can
            // give 1 - 1e-16 at u = 1, which rounds to 1.0f)
            bool last_ok = c0[m - 1] + deg == ncp - 1 && (float)b[(size_t)(m - 1) * 4 + deg] == 1.0f;
            for (int a = 0; a < deg; a++) last_ok = last_ok && (float)b[(size_t)(m - 1) * 4 + a] == 0.0f;
            if (last_ok) {
                const int kp = (ncp + 7) & ~7;
                std::vector<float> tb((size_t)2 * kTcRows * kp, 0.f);
                for (int i = 0; i < kTcRows; i++)
                    for (int a = 0; a <= deg; a++) {
                        const int x = c0[i] + a;
                        const double v = b[(size_t)i * 4 + a];
                        float hi = (float)v;
                        uint32_t bits;
                        memcpy(&bits, &hi, 4);
                        bits &= 0xFFFFE000u;
                        memcpy(&hi, &bits, 4);
                        const float lo = (float)(v - (double)hi);
                        const size_t e = ((size_t)(x / 4) * kTcRows + i) * 4 + x % 4;
                        tb[e] = hi;
                        tb[(size_t)kTcRows * kp + e] = lo;
                    }
                AFAM_CUDA(cudaMalloc(&o.tc_b, tb.size() * sizeof(float)));
                AFAM_CUDA(cudaMemcpy(o.tc_b, tb.data(), tb.size() * sizeof(float), cudaMemcpyHostToDevice));
                o.tc_kp = kp;
            }
        }
        if (!o.any) {  // register-tiled decode: m == 65, deg + 1 <= ncp <= 65 (lattice steps advance the span by <= 1),
           // the u = 1 row e_{ncp-1} in float32
            bool ok = m == 65 && ncp <= 65 && ncp >= deg + 1 && c0[m - 1] + deg == ncp - 1 &&
                      (float)b[(size_t)(m - 1) * 4 + deg] == 1.0f;
            for (int a = 0; a < deg; a++) ok = ok && (float)b[(size_t)(m - 1) * 4 + a] == 0.0f;
            o.fx_ok = ok;
        }
        AFAM_CUDA(cudaMalloc(&o.b32, b32.size() * sizeof(float)));
        AFAM_CUDA(cudaMalloc(&o.b64, b.size() * sizeof(double)));
        AFAM_CUDA(cudaMalloc(&o.col0, c0.size() * sizeof(int32_t)));
        AFAM_CUDA(cudaMemcpy(o.b32, b32.data(), b32.size() * sizeof(float), cudaMemcpyHostToDevice));
        AFAM_CUDA(cudaMemcpy(o.b64, b.data(), b.size() * sizeof(double), cudaMemcpyHostToDevice));
        AFAM_CUDA(cudaMemcpy(o.col0, c0.data(), c0.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
        it = s->ops.emplace(key, o).first;
    }
    *op = &it->second;
    return AFAM_OK;
}

extern "C" int afam_decode_grid(afam_store *s, const int32_t *slots, int32_t nblk, int32_t m, float *out,
                                void *stream) {
    return afam_decode_grid_ex(s, slots, nblk, m, out, AFAM_DECODE_AUTO, nullptr, stream);
}

extern "C" int afam_decode_grid_ex(afam_store *s, const int32_t *slots, int32_t nblk, int32_t m, float *out,
                                   int32_t path, int32_t *ntc_out, void *stream) {
    AFAM_CHECK(path >= AFAM_DECODE_AUTO && path <= AFAM_DECODE_TENSOR_CORES, AFAM_E_VALUE, "unknown decode path %d",
               path);
    const bool use_tc = path == AFAM_DECODE_TENSOR_CORES || (path == AFAM_DECODE_AUTO && tc_default());
    if (ntc_out) *ntc_out = 0;
    AFAM_CHECK(s, AFAM_E_VALUE, "store is NULL");
    AFAM_CHECK(nblk >= 0, AFAM_E_VALUE, "negative block count");
    if (nblk == 0) return AFAM_OK;
    AFAM_CHECK(slots && out, AFAM_E_VALUE, "slots/out is NULL");
    AFAM_CHECK(m >= 2 && m <= 4096, AFAM_E_VALUE, "decode dims %d out of range", m);
    AFAM_CHECK(nblk <= 65535, AFAM_E_VALUE, "at most 65535 blocks per decode call");
    cudaStream_t st = (cudaStream_t)stream;
    AFAM_CUDA(cudaSetDevice(s->device));
    std::vector<DecodeJob> jobs(nblk);
    int maxn = 0, ntc = 0, maxkp = 0, maxn_tc = 0, nfx = 0, nany = 0;
    size_t maxfx = 0;  // largest ncp * pitch among the register-tiled jobs
    {
        std::lock_guard<std::mutex> lk(s->mu);
        for (int b = 0; b < nblk; b++) {
            const int32_t sl = slots[b];
            AFAM_CHECK(sl >= 0 && sl < s->nslots && s->host[sl].valid, AFAM_E_VALUE, "slot %d is empty", sl);
            AFAM_CHECK(!s->host[sl].ds, AFAM_E_VALUE, "slot %d holds a DS block (no spline to decode)", sl);
            const SlotHost &h = s->host[sl];
            DecodeOp *op = nullptr;
            int rc = get_op(s, h.ncp, h.deg, m, &op);
            if (rc) return rc;
            jobs[b].slot = sl;
            jobs[b].col0 = op->col0;
            jobs[b].b32 = op->b32;
            jobs[b].b64 = op->b64;
            jobs[b].tc_b = op->tc_b;
            jobs[b].tc_kp = use_tc ? op->tc_kp : 0;  // float64 slots (device flag) stay on the CUDA-core kernel
            jobs[b].fx = (!jobs[b].tc_kp && op->fx_ok && !fx_disabled()) ? 1 : 0;
            jobs[b].any = op->any ? 1 : 0;
            nany += jobs[b].any;
            if (jobs[b].fx) {
                nfx++;
                maxfx = std::max(maxfx, (size_t)h.ncp * (size_t)((h.ncp + 3) & ~3));
            }
            if (jobs[b].tc_kp) {
                ntc++;
                maxkp = std::max(maxkp, (int)jobs[b].tc_kp);
                maxn_tc = std::max(maxn_tc, (int)h.ncp);
            }
            maxn = std::max(maxn, (int)h.ncp);
            AFAM_CUDA(wait_slot(s, sl, st));
        }
    }
    // S1 + S2 + B in T + col0 (padded to 4) + plane ring + mbarriers
    const size_t maxpitch = (size_t)((maxn + 3) & ~3);
    auto smem_for = [&](size_t tsz) {
        return ((size_t)maxn * maxpitch + (size_t)m * maxpitch + (size_t)m * 4) * tsz + (size_t)((m + 3) & ~3) * 4 +
               (size_t)kRing * maxn * maxpitch * sizeof(float) + kRing * sizeof(uint64_t) + 16;
    };
    DecodeJob *d_jobs = nullptr;
    AFAM_CUDA(cudaMallocAsync(&d_jobs, sizeof(DecodeJob) * nblk, st));
    AFAM_CUDA(cudaMemcpyAsync(d_jobs, jobs.data(), sizeof(DecodeJob) * nblk, cudaMemcpyHostToDevice, st));
    const dim3 grid((m + kDecodeChunk - 1) / kDecodeChunk, nblk);
    if (ntc_out) *ntc_out = ntc;
    if (ntc > 0) {
        const size_t smem = tc_smem(maxn_tc, maxkp, m).total;
        AFAM_CHECK(smem <= 227 * 1024, AFAM_E_VALUE, "tensor-core decode needs %zu B of shared memory", smem);
        AFAM_CUDA(cudaFuncSetAttribute(decode_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        decode_tc_kernel<<<nblk, kTcThreads, smem, st>>>(s->d_desc, d_jobs, m, out);
    }
    if (nfx > 0) {
        // the SMW variant (weights in shared memory, 3-slot ring: 2 CTAs per SM) with AFAM_DECODE_FX_SMW=1
        const bool smw = fx_ypt() == 4 && fx_smw();
        const int ring = smw ? 3 : kFxRing;
        const size_t smem =
            ((size_t)ring * (maxfx + kFxPad) + 2 * (size_t)kFxXRows * kFxXPitch + 65 * 4 + 68 + 2 * 72) * 4 +
            (smw ? (10 * 16 + 7 * 16) * 16 : 0) + ring * 8;
        AFAM_CHECK(smem <= 227 * 1024, AFAM_E_VALUE, "register-tiled decode needs %zu B of shared memory", smem);
        if (smw) {
            AFAM_CUDA(cudaFuncSetAttribute(decode_fx_kernel<4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem));
            AFAM_CUDA(cudaFuncSetAttribute(decode_fx_kernel<4, true>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                           cudaSharedmemCarveoutMaxShared));  // room for two CTAs per SM
            decode_fx_kernel<4, true><<<nblk, 256, smem, st>>>(s->d_desc, d_jobs, out);
        } else if (fx_ypt() == 4) {
            AFAM_CUDA(cudaFuncSetAttribute(decode_fx_kernel<4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem));
            decode_fx_kernel<4, false><<<nblk, 256, smem, st>>>(s->d_desc, d_jobs, out);
        } else {
            AFAM_CUDA(cudaFuncSetAttribute(decode_fx_kernel<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem));
            decode_fx_kernel<2, false><<<nblk, 512, smem, st>>>(s->d_desc, d_jobs, out);
        }
    }
    if (nany > 0) decode_any_kernel<<<dim3(64, nblk), 256, 0, st>>>(s->d_desc, d_jobs, m, out);
    if (ntc + nfx + nany < nblk) {
        const size_t smem = smem_for(sizeof(float));
        AFAM_CHECK(smem <= 227 * 1024, AFAM_E_VALUE, "decode of ncp=%d onto m=%d needs %zu B of shared memory", maxn,
                   m, smem);
        AFAM_CUDA(cudaFuncSetAttribute(decode_grid_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
        decode_grid_kernel<float><<<grid, kDecodeThreads, smem, st>>>(s->d_desc, d_jobs, m, out);
    }
    {
        const size_t smem = smem_for(sizeof(double));
        AFAM_CHECK(smem <= 227 * 1024, AFAM_E_VALUE, "decode of ncp=%d onto m=%d needs %zu B of shared memory", maxn,
                   m, smem);
        AFAM_CUDA(cudaFuncSetAttribute(decode_grid_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
        decode_grid_kernel<double><<<grid, kDecodeThreads, smem, st>>>(s->d_desc, d_jobs, m, out);
    }
    AFAM_CUDA(cudaGetLastError());
    AFAM_CUDA(cudaFreeAsync(d_jobs, st));
    ThreadCtx *tc = thread_ctx(s->device);
    AFAM_CHECK(tc, AFAM_E_CUDA, "per-thread state unavailable");
    AFAM_CUDA(cudaEventRecord(tc->read, st));
    mark_readers(s, slots, nblk, tc->read);  // later uploads into these slots wait for the decode
    return AFAM_OK;
}
