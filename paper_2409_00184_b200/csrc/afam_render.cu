// K2: fused ray march -- owner lookup, B-spline value+gradient decode,
// transfer function, Blinn-Phong shading, front-to-back compositing, early
// termination and uint8 quantisation in one kernel.
//
// Replaces render.render (reference render.py:398-466) including
// _ray_grid (:323-337), _ray_box_span (:340-354), _BlockIndex (:357-380),
// _shade (:383-395) and TransferFunction.color_at/opacity_at (:117-124).
//
// Numerics.  Block/LOD selection must match the reference bit-exactly, so
// ray setup, the sample position t = t_enter + (k+0.5)*sd, pos = clip(o +
// t*d) and the finest-cell index are float64 with the reference's op order
// and no FMA contraction (__dadd_rn/__dmul_rn/...).  The knot span is also
// chosen in float64 against the stored float32 knots.  Decoding is float32
// (float64 for slots flagged AFAM_SLOT_FP64); TF, shading and compositing
// are float32 (parity gate: PSNR >= 60 dB).
//
// Schedule.  One thread per ray; a warp is an 8x4 pixel tile and a CTA a
// 16x8 tile, so a warp's samples almost always share the owner block
// (SURVEY.md sec. 7 coherence measurement).  Interior knot spans of
// clamped-uniform models use the closed-form uniform B-spline basis (no
// table, no division); the 2p boundary spans per axis read the per-span
// table.  The (p+1)^3 control points of the current spans stay in
// registers as (p+1)^2 float4 rows of the x-quad layout and are re-gathered
// (one 16-byte load per row) only when a span or the owner block changes.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <vector>

#include "afam_eval.cuh"

#include <chrono>
#include <cstdio>
#include <cstdlib>

// AFAM_HOST_TIMING=1: per-call host phase times of afam_render on stderr.
struct HostTimer {
    static bool on() {
        static const bool v = [] {
            const char *e = getenv("AFAM_HOST_TIMING");
            return e && atoi(e) != 0;
        }();
        return v;
    }
    std::chrono::steady_clock::time_point t[8];
    int n = 0;
    HostTimer() { if (on()) t[n++] = std::chrono::steady_clock::now(); }
    void mark() { if (on() && n < 8) t[n++] = std::chrono::steady_clock::now(); }
    void report(const char *what) const {
        if (!on()) return;
        fprintf(stderr, "[%s]", what);
        for (int i = 1; i < n; i++)
            fprintf(stderr, " %.3f", std::chrono::duration<double, std::milli>(t[i] - t[i - 1]).count());
        fprintf(stderr, " ms\n");
    }
};

namespace afam {

constexpr int kTfBuckets = 512;

// The breakpoint arrays (val, slope, bp: nbp entries each, any number of TF
// control points) follow the table in the frame's argument upload; the
// pointers are set to their device copies when the upload is packed.
struct TfTable {
    float4 c0[kTfBuckets];    // rgb at the bucket start; .w NaN: a color breakpoint lies in the bucket
    float4 dc[kTfBuckets];    // rgb increment across the bucket
    float2 alpha[kTfBuckets]; // (alpha at the bucket start, increment); .y NaN: an opacity breakpoint lies in it
    int32_t lut[kTfBuckets];  // last breakpoint <= bucket start (-1: none)
    const float4 *val;        // (r, g, b, alpha) at breakpoint j
    const float4 *slope;      // d/dv on [bp[j], bp[j+1]); 0 past the last breakpoint
    const float *bp;          // sorted union of color and opacity control scalars
    int32_t nbp;
    float lo, scale;          // bucket coordinate = (v - lo) * scale over the TF domain
    float op_lo, op_hi;       // opacity support (see build_tf_table)
};

struct alignas(16) RenderArgs {
    double origin[3], f[3], r[3], u[3];
    double tan_x, tan_y;
    double sd, o_max;
    double near_;
    int32_t width, height, band_rows, nparts, part, rows;
    int32_t cells, nb;
    float power, ambient, diffuse, specular, shininess;
    int32_t power_one;  // power == 1
    float dom_lo, dom_hi;
    float o_max_f;      // largest float32 <= o_max: (float)A <= o_max_f iff (double)A <= o_max
    uint32_t flags;
    float tf_lo, tf_scale;  // TfTable lo / scale, as launch arguments (constant bank, no per-sample load)
    float op_lo, op_hi;     // TF opacity support: the kernel's alpha_tf is exactly 0 unless op_lo < v < op_hi
    // the support pulled back through the domain clamp: clamp(v) <= op_lo iff
    // v <= clr_lo, clamp(v) >= op_hi iff v >= clr_hi (transparent-cell test)
    float clr_lo, clr_hi;
};

// TransferFunction.color_at / opacity_at (render.py:117-124): every
// channel is np.interp over its own control points; on the sorted union of
// all control scalars each channel is linear, so one segment search serves
// r, g, b and alpha.  Values at the breakpoints are the float64 np.interp
// values rounded to float32.  The hot path reads the per-bucket lines
// (tf_alpha / tf_color below); this search serves buckets holding a breakpoint.
__device__ __forceinline__ float4 tf_eval(const TfTable &T, float v) {
    int bi = __float2int_rz((v - T.lo) * T.scale);
    bi = min(max(bi, 0), kTfBuckets - 1);
    int j = T.lut[bi];
    while (j + 1 < T.nbp && v >= T.bp[j + 1]) ++j;
    while (j >= 0 && v < T.bp[j]) --j;
    if (j < 0) return T.val[0];
    const float4 a = T.val[j], s = T.slope[j];
    const float dx = v - T.bp[j];
    return make_float4(fmaf(s.x, dx, a.x), fmaf(s.y, dx, a.y), fmaf(s.z, dx, a.z), fmaf(s.w, dx, a.w));
}

// Global frame row of local row lr for (band_rows, nparts, part).
__device__ __forceinline__ int frame_row(const RenderArgs &A, int lr) {
    const int b = lr / A.band_rows;
    return (b * A.nparts + A.part) * A.band_rows + lr % A.band_rows;
}

// The owner block's fields used per sample (kept in registers).
struct BlockLite {
    const float4 *ctrl4;
    const float *tab32;
    const float *knots;
    double lo[3], scale[3];  // scale = nspan / (hi - lo): world offset -> span coordinate
    float inv_span_f[3], nspan_f;
    int32_t ncp, nspan, deg;
    uint32_t flags;
};

__device__ __forceinline__ void load_lite(const BlockDesc *__restrict__ p, BlockLite &b) {
    b.ctrl4 = (const float4 *)__ldg((const unsigned long long *)&p->ctrl4);
    b.tab32 = (const float *)__ldg((const unsigned long long *)&p->tab32);
    b.knots = (const float *)__ldg((const unsigned long long *)&p->knots);
    b.ncp = __ldg(&p->ncp);
    b.nspan = __ldg(&p->nspan);
    b.nspan_f = (float)b.nspan;
    b.deg = __ldg(&p->deg);
    b.flags = __ldg(&p->flags);
#pragma unroll
    for (int a = 0; a < 3; a++) {
        b.lo[a] = __ldg(&p->lo[a]);
        b.scale[a] = __ldg(&p->inv_span[a]) * (double)b.nspan;
        b.inv_span_f[a] = __ldg(&p->inv_span_f[a]);
    }
}

// Knot span + basis for one axis.  The span is the reference's
// searchsorted(float32 knots, u64, 'right') - 1 (bspline.py:41-47): for
// uniform models floor(u*nspan) except within 1e-4 of a knot, where the
// stored knots decide.
template <int P>
__device__ __forceinline__ int axis_basis(const BlockLite &b, const BlockDesc *__restrict__ dp, int a, double p,
                                          float (&N)[P + 1], float (&E)[P]) {
    // fast path: interior span of a uniform model, not within 1e-4 spans of a knot
    // no clamp needed here: a sample a hair outside [0, nspan] (rounding at a
    // block face) lands within 1e-4 of an end knot and takes the exact path
    // (span coordinate in float32 once the float64 offset is formed: for
    // nspan <= 128 its rounding, < 4e-6 of a span, is far inside the 1e-4
    // exactness margin and ~1e-7 in value)
    const double dpos = p - b.lo[a];
    const float tq = (float)(dpos * b.scale[a]);
    const int k = min((int)floorf(tq), b.nspan - 1);
    const float fr = tq - (float)k;
    int s = P + k;
    const bool uni = (b.flags & kFlagUniform) && b.nspan <= 128;
    if (uni && fr >= 1e-4f && fr <= 1.f - 1e-4f && s >= 2 * P - 1 && s <= b.ncp - P) {
        uniform_basis<P>(fr, b.nspan_f, N, E);
        return s;
    }
    // exact path: reference parameter (model.py:67) and span search against the stored knots
    const double u64 = clamp01(dpos * __ldg(&dp->inv_span[a]));
    s = find_span(b.knots + a * (b.ncp + P + 1), b.ncp, P, b.nspan, u64);
    if (uni && s >= 2 * P - 1 && s <= b.ncp - P) {
        uniform_basis<P>((float)(u64 * (double)b.nspan - (double)(s - P)), b.nspan_f, N, E);
    } else {
        Tab<float> t;
        load_entry<P>(b.tab32 + ((size_t)a * b.nspan + (s - P)) * tab_stride(P), t);
        basis_eval<P, float>(t, (float)u64, N, E);
    }
    return s;
}

template <int P>
__device__ __forceinline__ float q4(const float4 &v) {
    return P == 0 ? v.x : (P == 1 ? v.y : (P == 2 ? v.z : v.w));
}

template <int K>
__device__ __forceinline__ float comp(const float4 &v) {
    if constexpr (K == 0) return v.x;
    else if constexpr (K == 1) return v.y;
    else if constexpr (K == 2) return v.z;
    else return v.w;
}

template <int P, int AX, typename T>
__device__ __forceinline__ void row_contract(const float4 &r, const T (&Nx)[P + 1], const T (&Ex)[P], T &acc,
                                             T &dacc) {
    if constexpr (AX <= P) {
        acc = fma(Nx[AX], (T)comp<AX>(r), acc);
        if constexpr (AX < P) dacc = fma(Ex[AX], (T)comp<AX + 1>(r) - (T)comp<AX>(r), dacc);
        row_contract<P, AX + 1, T>(r, Nx, Ex, acc, dacc);
    }
}

// contract_grad (afam_eval.cuh) on x-quad rows c4[cz*Q+by].
template <int P, typename T>
__device__ __forceinline__ void contract_quad(const float4 (&c4)[16], const T (&Nx)[P + 1], const T (&Ex)[P],
                                              const T (&Ny)[P + 1], const T (&Ey)[P], const T (&Nz)[P + 1],
                                              const T (&Ez)[P], T &v, T (&g)[3]) {
    constexpr int Q = P + 1;
    T ry[Q], rdxy[Q], rdy[Q];
#pragma unroll
    for (int cz = 0; cz < Q; cz++) {
        T rx[Q], rdx[Q];
#pragma unroll
        for (int by = 0; by < Q; by++) {
            T acc = T(0), dacc = T(0);
            row_contract<P, 0, T>(c4[cz * Q + by], Nx, Ex, acc, dacc);
            rx[by] = acc;
            rdx[by] = dacc;
        }
        T ay = T(0), adxy = T(0), ady = T(0);
#pragma unroll
        for (int by = 0; by < Q; by++) {
            ay = fma(Ny[by], rx[by], ay);
            adxy = fma(Ny[by], rdx[by], adxy);
        }
#pragma unroll
        for (int k = 0; k < P; k++) ady = fma(Ey[k], rx[k + 1] - rx[k], ady);
        ry[cz] = ay; rdxy[cz] = adxy; rdy[cz] = ady;
    }
    T vv = T(0), gx = T(0), gy = T(0), gz = T(0);
#pragma unroll
    for (int cz = 0; cz < Q; cz++) {
        vv = fma(Nz[cz], ry[cz], vv);
        gx = fma(Nz[cz], rdxy[cz], gx);
        gy = fma(Nz[cz], rdy[cz], gy);
    }
#pragma unroll
    for (int k = 0; k < P; k++) gz = fma(Ez[k], ry[k + 1] - ry[k], gz);
    v = vv; g[0] = gx; g[1] = gy; g[2] = gz;
}

// Keep the gathered rows across samples (re-gather only on span/owner
// change).  Off by default: at LOD-1 span widths a lane changes span on most
// steps, so the cache mostly costs 64 registers of occupancy.
#ifndef AFAM_GATHER_CACHE
#define AFAM_GATHER_CACHE 0
#endif
constexpr bool kGatherCache = AFAM_GATHER_CACHE;

struct GatherCache {
    int32_t slot, x0, y0, z0;
    float4 c4[16];
};

// bspline.py:175-181 gather: (p+1)^2 rows of the x-quad layout, skipped
// when the owner slot and the three spans are unchanged since the last sample.
template <int P>
__device__ __forceinline__ void gather_quad(const BlockLite &b, int32_t slot, GatherCache &G, int x0, int y0, int z0) {
    constexpr int Q = P + 1;
    if (!kGatherCache || slot != G.slot || x0 != G.x0 || y0 != G.y0 || z0 != G.z0) {
        const float4 *base = b.ctrl4 + ((size_t)z0 * b.ncp + x0) * b.ncp + y0;
        const size_t plane = (size_t)b.ncp * b.ncp;
#pragma unroll
        for (int cz = 0; cz < Q; cz++) {
            const float4 *p = base + cz * plane;
#pragma unroll
            for (int by = 0; by < Q; by++) G.c4[cz * Q + by] = __ldg(p + by);
        }
        if (kGatherCache) {
            G.slot = slot;
            G.x0 = x0;
            G.y0 = y0;
            G.z0 = z0;
        }
    }
}

// Value first (separable x -> y -> z with the N weights, keeping the x and
// y partial sums), then the transfer function; the gradient (difference
// form, reusing the partial sums for d/dy and d/dz) only for samples the TF
// makes non-transparent.  A sample with alpha_tf = 0 has a_s = 0 and adds
// nothing to C or A (render.py:451-455), so skipping its gradient and
// shading leaves the frame bit-identical.
template <int P>
__device__ __forceinline__ void decode_f32(const BlockLite &b, const BlockDesc *__restrict__ dp, int32_t slot,
                                           GatherCache &G, const double (&pos)[3], const TfTable &tf, float dom_lo,
                                           float dom_hi, float &v, float4 &tfv, float (&g)[3]) {
    constexpr int Q = P + 1;
    float Nx[Q], Ex[P], Ny[Q], Ey[P], Nz[Q], Ez[P];
    // model.py:64-68 params_for: u = clip((p - lo)/span, 0, 1), float64
    const int sx = axis_basis<P>(b, dp, 0, pos[0], Nx, Ex);
    const int sy = axis_basis<P>(b, dp, 1, pos[1], Ny, Ey);
    const int sz = axis_basis<P>(b, dp, 2, pos[2], Nz, Ez);
    gather_quad<P>(b, slot, G, sx - P, sy - P, sz - P);
    // value pass; d/dy and d/dz come almost free from its partial sums
    float ry[Q], gy = 0.f;
#pragma unroll
    for (int cz = 0; cz < Q; cz++) {
        float rx[Q];
        float ay = 0.f;
#pragma unroll
        for (int by = 0; by < Q; by++) {
            const float4 &r = G.c4[cz * Q + by];
            float acc = Nx[0] * comp<0>(r);
            acc = fmaf(Nx[1], comp<1>(r), acc);
            if constexpr (P >= 2) acc = fmaf(Nx[2], comp<2>(r), acc);
            if constexpr (P >= 3) acc = fmaf(Nx[3], comp<3>(r), acc);
            rx[by] = acc;
            ay = fmaf(Ny[by], acc, ay);
        }
        float ady = 0.f;
#pragma unroll
        for (int k = 0; k < P; k++) ady = fmaf(Ey[k], rx[k + 1] - rx[k], ady);
        gy = fmaf(Nz[cz], ady, gy);
        ry[cz] = ay;
    }
    float vv = 0.f, gz = 0.f;
#pragma unroll
    for (int cz = 0; cz < Q; cz++) vv = fmaf(Nz[cz], ry[cz], vv);
#pragma unroll
    for (int k = 0; k < P; k++) gz = fmaf(Ez[k], ry[k + 1] - ry[k], gz);
    v = vv;
    tfv = tf_eval(tf, fminf(fmaxf(vv, dom_lo), dom_hi));  // TransferFunction (render.py:117-124)
    if (!(tfv.w > 0.f)) {
        g[0] = g[1] = g[2] = 0.f;
        return;
    }
    // d/dx: differences along the x-quad rows, re-read from L1 so the rows
    // need not stay in registers across the TF lookup
    float gx = 0.f;
    const float4 *base = b.ctrl4 + ((size_t)(sz - P) * b.ncp + (sx - P)) * b.ncp + (sy - P);
    const size_t plane = (size_t)b.ncp * b.ncp;
#pragma unroll
    for (int cz = 0; cz < Q; cz++) {
        float adxy = 0.f;
#pragma unroll
        for (int by = 0; by < Q; by++) {
            const float4 r = kGatherCache ? G.c4[cz * Q + by] : __ldg(base + cz * plane + by);
            float dacc = Ex[0] * (comp<1>(r) - comp<0>(r));
            if constexpr (P >= 2) dacc = fmaf(Ex[1], comp<2>(r) - comp<1>(r), dacc);
            if constexpr (P >= 3) dacc = fmaf(Ex[2], comp<3>(r) - comp<2>(r), dacc);
            adxy = fmaf(Ny[by], dacc, adxy);
        }
        gx = fmaf(Nz[cz], adxy, gx);
    }
    // model.py:79 gradient / span
    g[0] = gx * b.inv_span_f[0];
    g[1] = gy * b.inv_span_f[1];
    g[2] = gz * b.inv_span_f[2];
}

// Ill-conditioned slots: the same schedule with float64 parameters (the
// reference's division), float64 basis from the float64 table and float64
// accumulation; control points are float32 in the file, so the float4 rows
// are shared with the float32 path.
template <int P>
__device__ __noinline__ void grad_f64(const float4 *__restrict__ base, size_t plane, const double (&N)[3][P + 1],
                                      const double (&E)[3][P], double (&gg)[3]) {
    constexpr int Q = P + 1;
    float4 c4[16];
#pragma unroll
    for (int cz = 0; cz < Q; cz++)
#pragma unroll
        for (int by = 0; by < Q; by++) c4[cz * Q + by] = __ldg(base + cz * plane + by);
    double vv;
    contract_quad<P, double>(c4, N[0], E[0], N[1], E[1], N[2], E[2], vv, gg);
}

template <int P>
__device__ __forceinline__ void decode_f64(const BlockLite &b, const BlockDesc *__restrict__ dp, int32_t slot,
                                           GatherCache &G, const double (&pos)[3], const TfTable &tf, float dom_lo,
                                           float dom_hi, float &v, float4 &tfv, float (&g)[3]) {
    constexpr int Q = P + 1;
    double N[3][Q], E[3][P], span[3];
    int s[3];
    const double *tab64 = (const double *)__ldg((const unsigned long long *)&dp->tab64);
#pragma unroll
    for (int a = 0; a < 3; a++) {
        span[a] = __ldg(&dp->span[a]);
        const double u = clamp01(__ddiv_rn(__dsub_rn(pos[a], b.lo[a]), span[a]));
        s[a] = find_span(b.knots + a * (b.ncp + P + 1), b.ncp, P, b.nspan, u);
        Tab<double> t;
        load_entry<P>(tab64 + ((size_t)a * b.nspan + (s[a] - P)) * tab_stride(P), t);
        basis_eval<P, double>(t, u, N[a], E[a]);
    }
    gather_quad<P>(b, slot, G, s[0] - P, s[1] - P, s[2] - P);
    // value pass in float64 (x -> y -> z), then the TF: the gradient only
    // for samples it makes visible (alpha_tf = 0 adds nothing to C or A,
    // render.py:451-455, so the frame is unchanged)
    double vv = 0.0;
#pragma unroll
    for (int cz = 0; cz < Q; cz++) {
        double ay = 0.0;
#pragma unroll
        for (int by = 0; by < Q; by++) {
            double acc = 0.0, dacc = 0.0;
            row_contract<P, 0, double>(G.c4[cz * Q + by], N[0], E[0], acc, dacc);
            ay = fma(N[1][by], acc, ay);
        }
        vv = fma(N[2][cz], ay, vv);
    }
    v = (float)vv;
    tfv = tf_eval(tf, fminf(fmaxf(v, dom_lo), dom_hi));
    if (!(tfv.w > 0.f)) {
        g[0] = g[1] = g[2] = 0.f;
        return;
    }
    // the gradient in its own frame (re-reading the rows through L1): kept
    // out of line so the value pass's float64 conversions are not held live
    // across it (a fused value + gradient pass spilled ~1 KB per thread)
    double gg[3];
    grad_f64<P>(b.ctrl4 + ((size_t)(s[2] - P) * b.ncp + (s[0] - P)) * b.ncp + (s[1] - P), (size_t)b.ncp * b.ncp,
                N, E, gg);
#pragma unroll
    for (int a = 0; a < 3; a++) g[a] = (float)(gg[a] / span[a]);
}

// ---------------------------------------------------------------------------
// K2 march.  The reference's per-sample geometry (render.py:422-428,
// :377-380) is float64; the kernel evaluates it exactly (same op order, no
// contraction) only where its result could differ from a cheap float32
// prediction:
//  - the sample count comes from one exact search per ray (t_k is monotone
//    in k, so the alive samples are the prefix k < kend);
//  - the finest cell is evaluated exactly at the first sample and then only
//    at the first sample that could lie within 1e-6 cells of (or across) a
//    face of the current cell (knext, from the per-axis cell-coordinate
//    rate; exact_geometry); every sample in between keeps the owner;
//  - within a block the span coordinate is tq0 + (k - k0)*dtq from the exact
//    position at block entry k0 (error < 2e-5 spans).
// Owner selection therefore stays bit-exact while the common sample runs
// without float64 arithmetic.

struct RayState {  // per-thread, in local memory: read/written on the exact paths only
    double d[3];
    double te;
    float4 tfv;       // sample_exact results
    float g[3];
    int32_t pad;
};

struct March {
    int32_t k, kend;
    float kf;                      // (float)k, exact below 2^24
    float C0, C1, C2, Aacc;
    int32_t knext;                 // next sample whose finest cell is evaluated exactly
    float tq0[3], dtq[3], k0f;     // span-coordinate prediction within the current block
    int32_t own;
    uint32_t nshade;
    uint64_t h;
};

// The owner block's fields the fast path reads per sample.
// Internal render flag (AFAM_RENDER_FORCE_EXACT=1 in the environment): every
// sample on the exact path, for A/B checks of the fast path.
constexpr uint32_t kRenderForceExact = 0x100u;

struct BlockFast {
    const float4 *ctrl4;
    const float2 *rng;  // per-cell value ranges (BlockDesc::crange)
    int32_t ncp, nspan;
    int32_t plane;  // ncp^2: x-quad rows per z plane
    uint32_t nint;  // interior spans (k in [p-1, nspan-p]): max(nspan - 2p + 2, 0)
};

// Per-thread state the sample loop reads rarely (shading, boundary spans,
// counters of the rare paths), kept in shared memory so the registers go to
// the cached cell and the per-sample state.
struct alignas(16) ThreadCold {
    float4 vdir;         // ray direction (float32), for shading
    float4 ginv;         // 1/span per axis of the owner block (model.py:79)
    const float *tab32;  // owner block's per-span basis tables
    uint32_t ns64, nexact, ncell;
    uint32_t nclear;  // DEBUG kernels: samples in transparent cells
};

// render.py:422-428 sample position, float64 in the reference op order, and
// its finest cell (render.py:377-380).  Also returns knext, the first later
// sample whose cell could differ: along each axis the cell coordinate
// sc = ((q+1)/2)*cells moves by sd*d*cells/2 per sample, so every sample
// before knext lies at least 1e-6 cells inside the current cell's faces --
// far beyond the float64 rounding of the reference's expression (~1e-14) --
// and keeps this owner; knext itself is evaluated exactly again.
__device__ __forceinline__ void exact_geometry(const RenderArgs &A, const RayState &R, const int16_t *own_grid,
                                               int64_t k, int32_t kend, double (&p)[3], int32_t &own,
                                               int32_t &knext) {
    const double t = __dadd_rn(R.te, __dmul_rn((double)k + 0.5, A.sd));
    const double cellsd = (double)A.cells;
    int cidx = 0;
    double steps = 1e18;
#pragma unroll
    for (int a = 0; a < 3; a++) {
        double q = __dadd_rn(A.origin[a], __dmul_rn(t, R.d[a]));
        q = q < -1.0 ? -1.0 : (q > 1.0 ? 1.0 : q);  // np.clip (q is never NaN here)
        p[a] = q;
        const double sc = __dmul_rn(__dmul_rn(__dadd_rn(q, 1.0), 0.5), cellsd);
        int ci = __double2int_rz(sc);
        ci = min(max(ci, 0), A.cells - 1);
        cidx = cidx * A.cells + ci;
        const double v = A.sd * R.d[a] * (0.5 * cellsd);  // cell coordinate per sample
        const double dist = v > 0.0 ? (double)(ci + 1) - sc : sc - (double)ci;
        if (v != 0.0) steps = fmin(steps, (dist - 1e-6) / fabs(v));
    }
    own = own_grid[cidx];
    const double kn = (double)k + fmax(1.0, ceil(steps));
    knext = kn < (double)kend ? (int32_t)kn : kend;
}

__device__ __forceinline__ void exact_pos(const RenderArgs &A, const RayState &R, int64_t k, double (&p)[3]) {
    const double t = __dadd_rn(R.te, __dmul_rn((double)k + 0.5, A.sd));
#pragma unroll
    for (int a = 0; a < 3; a++) {
        const double q = __dadd_rn(A.origin[a], __dmul_rn(t, R.d[a]));
        p[a] = q < -1.0 ? -1.0 : (q > 1.0 ? 1.0 : q);
    }
}

// Paired float32 arithmetic (FFMA2/FMUL2/FADD2: two lanes of float math per
// issue slot; the scalar weight is a broadcast operand).
__device__ __forceinline__ float2 lo2(const float4 &v) { return make_float2(v.x, v.y); }
__device__ __forceinline__ float2 hi2(const float4 &v) { return make_float2(v.z, v.w); }
__device__ __forceinline__ float2 fma2s(float s, float2 x, float2 acc) { return __ffma2_rn(make_float2(s, s), x, acc); }
__device__ __forceinline__ float2 mul2s(float s, float2 x) { return __fmul2_rn(make_float2(s, s), x); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }

__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }

// uniform_N (afam_eval.cuh) for two axes at once: the same operations in the
// same order on float2 lanes, so each lane is bit-identical to uniform_N.
template <int P>
__device__ __forceinline__ void uniform_N2(float2 x, float2 (&N)[P + 1]) {
    const float2 m = __ffma2_rn(x, f2(-1.f), f2(1.f));  // 1 - x
    if (P == 1) {
        N[0] = m;
        N[1] = x;
    } else if (P == 2) {
        const float2 x2 = __fmul2_rn(x, x);
        N[0] = __fmul2_rn(__fmul2_rn(f2(0.5f), m), m);
        N[1] = __fadd2_rn(__ffma2_rn(f2(-1.f), x2, x), f2(0.5f));
        N[2] = __fmul2_rn(f2(0.5f), x2);
    } else {
        const float2 x2 = __fmul2_rn(x, x), x3 = __fmul2_rn(x2, x), m2 = __fmul2_rn(m, m);
        const float s6 = 1.f / 6.f;
        N[0] = __fmul2_rn(__fmul2_rn(f2(s6), m2), m);
        N[1] = __ffma2_rn(f2(0.5f), x3, __ffma2_rn(f2(-1.f), x2, f2(2.f / 3.f)));
        N[2] = __ffma2_rn(f2(-0.5f), x3, __ffma2_rn(f2(0.5f), x2, __ffma2_rn(f2(0.5f), x, f2(s6))));
        N[3] = __fmul2_rn(f2(s6), x3);
    }
}

// Per-axis basis of the fast path from the predicted span coordinate tq:
// span k = floor(tq) (clamped), fraction fr.  Interior spans of a
// clamped-uniform model use the closed form, the 2(p-1) boundary spans the
// per-span table.  Returns false (P = 1 only) within 1e-4 of a knot, where
// the gradient is discontinuous and the exact span must be searched.
// Per-axis span of the fast path from the predicted span coordinate tq:
// span k = floor(tq) (clamped), fraction fr; false (P = 1 only) within 1e-4
// of a knot, where the gradient is discontinuous and the exact span must be
// searched ...
template <int P>
__device__ __forceinline__ bool axis_span(const BlockFast &b, float tq, int &k, float &fr) {
    k = min(max(__float2int_rd(tq), 0), b.nspan - 1);
    fr = tq - (float)k;
    return !(P == 1 && !(fabsf(fr - 0.5f) < 0.5f - 1e-4f));
}

// ... interior spans of a clamped-uniform model use the closed form, the
// 2(p-1) boundary spans the per-span table
template <int P>
__device__ __forceinline__ bool span_interior(const BlockFast &b, int k) {
    return (uint32_t)(k - (P - 1)) < b.nint;  // k in [p-1, nspan-p]; none when nspan < 2p - 1
}

// Closed form of the cubic clamped-uniform basis on the two spans at either
// end (nspan >= 6): in the span's local coordinate f the knots are
// 0,0,0,0,1,2,3,4,... (span 0, 1) and the mirror image at the other end, so
// every block shares these polynomials (power basis, ascending; E_q is the
// difference-form weight sum_{i>q} dN_i/df).  Checked against exact
// rational Cox-de Boor in DESIGN.md's derivation script.
// The coefficients are immediates of the FFMAs (both classes evaluated,
// then selected): no dynamically indexed constant-bank loads per sample.
__device__ __forceinline__ float horner3(float c0, float c1, float c2, float c3, float f) {
    return fmaf(fmaf(fmaf(c3, f, c2), f, c1), f, c0);
}

__device__ __forceinline__ void bnd_N(int cls, float f, float (&n)[4]) {
    const float a0 = horner3(1.f, -3.f, 3.f, -1.f, f), b0 = horner3(0.25f, -0.75f, 0.75f, -0.25f, f);
    const float a1 = horner3(0.f, 3.f, -4.5f, 1.75f, f), b1 = horner3(7.f / 12.f, 0.25f, -1.25f, 7.f / 12.f, f);
    const float a2 = horner3(0.f, 0.f, 1.5f, -11.f / 12.f, f), b2 = horner3(1.f / 6.f, 0.5f, 0.5f, -0.5f, f);
    n[0] = cls ? b0 : a0;
    n[1] = cls ? b1 : a1;
    n[2] = cls ? b2 : a2;
    n[3] = horner3(0.f, 0.f, 0.f, 1.f / 6.f, f);
}

__device__ __forceinline__ float horner2(float c0, float c1, float c2, float f) { return fmaf(fmaf(c2, f, c1), f, c0); }

__device__ __forceinline__ void bnd_E(int cls, float f, float nsf, float (&e)[3]) {
    const float a0 = horner2(3.f, -6.f, 3.f, f), b0 = horner2(0.75f, -1.5f, 0.75f, f);
    const float a1 = horner2(0.f, 3.f, -2.25f, f), b1 = horner2(0.5f, 1.f, -1.f, f);
    e[0] = nsf * (cls ? b0 : a0);
    e[1] = nsf * (cls ? b1 : a1);
    e[2] = nsf * horner2(0.f, 0.f, 0.5f, f);
}

// span class of a cubic boundary span k (not interior): 0/1 from the left
// end, mirrored from the right end
__device__ __forceinline__ void bnd_class(const BlockFast &b, int k, int &cls, bool &mirror) {
    mirror = k > 1;
    cls = mirror ? b.nspan - 1 - k : k;
}

template <int P>
__device__ __forceinline__ void axis_table_N(const BlockFast &b, const ThreadCold &C, int a, int k, float tq,
                                             float (&N)[P + 1]) {
    if constexpr (P == 3) {
        if (b.nspan >= 6) {
            int cls;
            bool mirror;
            bnd_class(b, k, cls, mirror);
            const float fr = tq - (float)k;
            const float f = mirror ? 1.f - fr : fr;
            float n[4];
            bnd_N(cls, f, n);
#pragma unroll
            for (int i = 0; i < 4; i++) N[i] = mirror ? n[3 - i] : n[i];
            return;
        }
    }
    Tab<float> t;
    load_entry<P>(C.tab32 + ((size_t)a * b.nspan + k) * tab_stride(P), t);
    basis_vals_only<P, float>(t, clamp01(tq / (float)b.nspan), N);
}

template <int P>
__device__ __forceinline__ void axis_fast_E(const BlockFast &b, const ThreadCold &C, int a, int k, float fr,
                                            float (&E)[P]) {
    const float nsf = (float)b.nspan;
    if (span_interior<P>(b, k)) {
        uniform_E<P>(fr, nsf, E);
    } else if (P == 3 && b.nspan >= 6) {
        int cls;
        bool mirror;
        bnd_class(b, k, cls, mirror);
        const float f = mirror ? 1.f - fr : fr;
        float e[3];
        bnd_E(cls, f, nsf, e);
#pragma unroll
        for (int q = 0; q < P; q++) E[q] = mirror ? e[2 - q] : e[q];
    } else {
        Tab<float> t;
        float N[P + 1];
        load_entry<P>(C.tab32 + ((size_t)a * b.nspan + k) * tab_stride(P), t);
        basis_eval<P, float>(t, clamp01(((float)k + fr) / nsf), N, E);
    }
}

// TF opacity of a decoded value from the per-bucket lines (render.py:117-124
// np.interp); NaN-marked buckets hold a breakpoint and take the segment search.
// Shared memory: the TF opacity lines and the per-thread cold state are
// static arrays (fixed shared-window offsets, no per-sample base
// arithmetic); the dynamic part holds only the owner grid.
__shared__ float2 s_tf_alpha[kTfBuckets];
__shared__ ThreadCold s_cold[128];

// A fresh shared-memory read at every use (volatile): the compiler would
// otherwise hoist the loop-invariant loads into registers and keep them live
// across the sample loop, which is exactly what keeping them in shared
// memory is meant to avoid.
template <typename T>
__device__ __forceinline__ T vld(const T &x) {
    return *(const volatile T *)&x;
}

// K2's warp tile (both kernels): kWarpW x (32 / kWarpW) pixels, CTA tile kCtaW x
// (128 / kCtaW) (-DAFAM_WARP_W / -DAFAM_CTA_W for A/B).  Measured on config 3
// (ms per frame): 4x8 warps in 8x16 CTAs 1.965, 4x8 in 16x8 1.97, 2x16 in
// 8x16 1.99, 4x8 in 4x32 2.01, 8x4 in 16x8 2.07, 8x4 in 8x16 2.06, 16x2 in
// 16x8 2.22.
#ifndef AFAM_WARP_W
#define AFAM_WARP_W 4
#endif
constexpr int kWarpW = AFAM_WARP_W;
#ifndef AFAM_CTA_W
#define AFAM_CTA_W 8
#endif
constexpr int kCtaW = AFAM_CTA_W;  // render2_kernel's CTA tile: kCtaW x (128 / kCtaW) pixels

struct FastCold {  // render2_kernel's per-thread rarely-read state
    BlockFast b;                 // the owner block's fields read at cell changes
    int32_t kend;                // alive samples of the ray
    int32_t cur_own, slot, deg;  // owner index, its slot and degree
};
__shared__ FastCold s_fast[128];
extern __shared__ __align__(16) unsigned char afam_render_smem[];
constexpr size_t kSmemGridOff = 0;

__device__ __forceinline__ float tf_alpha(const RenderArgs &A, const TfTable &T, float v, int &bi, float &bf) {
    const float tb = (v - A.tf_lo) * A.tf_scale;
    bi = min(max(__float2int_rz(tb), 0), kTfBuckets - 1);
    bf = tb - (float)bi;
    // opacity lines staged in shared memory (the per-sample critical path)
    const float2 l = s_tf_alpha[bi];
    float a = fmaf(bf, l.y, l.x);
    if (isnan(a)) a = tf_eval(T, v).w;
    return a;
}

__device__ __forceinline__ float4 tf_color(const TfTable &T, float v, int bi, float bf, float atf) {
    const float4 c = __ldg(&T.c0[bi]), dc = __ldg(&T.dc[bi]);
    if (isnan(c.w)) {
        float4 r = tf_eval(T, v);
        r.w = atf;
        return r;
    }
    return make_float4(fmaf(bf, dc.x, c.x), fmaf(bf, dc.y, c.y), fmaf(bf, dc.z, c.z), atf);
}

// Shading and compositing of one sample (render.py:383-395, :451-455).
// MUFU approximations without the denormal-range fix-ups rsqrtf/exp2f add:
// gn2 > 1e-24 is always normal, and ndotl^shininess below 2^-126 only ever
// adds < 1e-38 to a colour that is quantised to 1/255.
__device__ __forceinline__ float rsqrt_ftz(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float lg2_ftz(float x) {
    float r;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float ex2_ftz(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ void composite(const RenderArgs &A, const float4 vdir, float4 tfv, const float (&g)[3],
                                          March &M) {
    const float atf = tfv.w;
    const float as = A.power_one ? 1.f - (1.f - atf) : 1.f - __powf(1.f - atf, A.power);
    const float gn2 = fmaf(g[2], g[2], fmaf(g[1], g[1], g[0] * g[0]));
    float ndotl = 0.f;
    if (gn2 > 1e-24f) {
        const float ig = rsqrt_ftz(gn2);
        ndotl = fabsf(g[0] * vdir.x + g[1] * vdir.y + g[2] * vdir.z) * ig;
    }
    const float dif = A.diffuse * ndotl;
    // ndotl**shininess via exp2(shininess * log2(ndotl)) (MUFU.LG2 + MUFU.EX2)
    const float spec = A.specular * (ndotl > 0.f ? ex2_ftz(A.shininess * lg2_ftz(ndotl))
                                                 : (A.shininess == 0.f ? 1.f : 0.f));
    const float lit = A.ambient + dif;
    const float w = (1.f - M.Aacc) * as;
    M.C0 = fmaf(w, __saturatef(fmaf(tfv.x, lit, spec)), M.C0);
    M.C1 = fmaf(w, __saturatef(fmaf(tfv.y, lit, spec)), M.C1);
    M.C2 = fmaf(w, __saturatef(fmaf(tfv.z, lit, spec)), M.C2);
    M.Aacc += w;
}

// The (p+1)^3 control points of the current cell, kept in registers across
// samples as (p+1)^2 x-quad rows (row cz*Q+by = c[x0..x0+3][y0+by][z0+cz],
// bspline.py:175-181).  A lane re-gathers only when its owner block or one of
// its three knot spans changed (~1 sample in 4 at LOD-2 span widths), and the
// L1 data path serves only the lanes that reload.
struct CellCache {
    int32_t key;  // x-quad row index of the cached cell's (0, 0) row in the owner block; -1: empty
    float4 c[16];
};

template <int P>
__device__ __forceinline__ void cell_gather(const BlockFast &b, int kx, int ky, int kz, CellCache &G) {
    constexpr int Q = P + 1;
    const int32_t id = (kz * b.ncp + kx) * b.ncp + ky;  // < 72^3: 32-bit index math on the hit path
    if (id != G.key) {
        const float4 *base = b.ctrl4 + id;
#pragma unroll
        for (int cz = 0; cz < Q; cz++)
#pragma unroll
            for (int by = 0; by < Q; by++) G.c[cz * Q + by] = __ldg(base + cz * b.plane + by);
        G.key = id;
    }
}

// sum_a W[a] X[a] over the x-quad components (x fastest, a = 0..P)
template <int P>
__device__ __forceinline__ float dot_x(const float (&W)[P + 1], float2 lo, float2 hi) {
    float s = W[0] * lo.x;
    s = fmaf(W[1], lo.y, s);
    if constexpr (P >= 2) s = fmaf(W[2], hi.x, s);
    if constexpr (P >= 3) s = fmaf(W[3], hi.y, s);
    return s;
}

// sum_q E[q] (X[q+1] - X[q]) over the x-quad components: d/dx in difference form
template <int P>
__device__ __forceinline__ float ddot_x(const float (&E)[P], float2 lo, float2 hi) {
    float s = E[0] * (lo.y - lo.x);
    if constexpr (P >= 2) s = fmaf(E[1], hi.x - lo.y, s);
    if constexpr (P >= 3) s = fmaf(E[2], hi.y - hi.x, s);
    return s;
}

// One sample of a clamped-uniform float32 block from the predicted span
// coordinates.  Value: y, then z, then x (bspline.py:214 einsum, separable),
// on x-quad halves with paired FMAs; then the TF opacity.  Only samples the
// TF makes non-transparent take the gradient (bspline.py:224-228) and the
// colour: d/dx from the z-contracted quad, d/dz from the kept y partials,
// d/dy from a z-first pass over the cached cell -- all in difference form
// (sum E_q (c_{q+1} - c_q)), so a patch that is flat along an axis gives an
// exactly zero derivative, as the reference's float64 gradient effectively
// does.  Returns false when the exact path must decode the sample.
template <int P>
__device__ __forceinline__ bool sample_fast(const RenderArgs &A, const TfTable &tf, const BlockFast &b,
                                            const float (&tq)[3], const ThreadCold &C, CellCache &G, March &M) {
    constexpr int Q = P + 1;
    int kx, ky, kz;
    float fx, fy, fz, Nx[Q], Ny[Q], Nz[Q];
    if (!axis_span<P>(b, tq[0], kx, fx) || !axis_span<P>(b, tq[1], ky, fy) || !axis_span<P>(b, tq[2], kz, fz))
        return false;
    cell_gather<P>(b, kx, ky, kz, G);
    {  // x and y closed forms paired, z alone; boundary spans from the table
        float2 Nxy[Q];
        uniform_N2<P>(make_float2(fx, fy), Nxy);
#pragma unroll
        for (int i = 0; i < Q; i++) {
            Nx[i] = Nxy[i].x;
            Ny[i] = Nxy[i].y;
        }
        const bool inx = span_interior<P>(b, kx), iny = span_interior<P>(b, ky), inz = span_interior<P>(b, kz);
        if (inx & iny & inz) {  // the common case: one branch
            uniform_N<P>(fz, Nz);
        } else {
            if (!inx) axis_table_N<P>(b, C, 0, kx, tq[0], Nx);
            if (!iny) axis_table_N<P>(b, C, 1, ky, tq[1], Ny);
            if (inz) uniform_N<P>(fz, Nz);
            else axis_table_N<P>(b, C, 2, kz, tq[2], Nz);
        }
    }
    // Y[cz] = sum_by Ny[by] c[cz][by] (x-quad), Z = sum_cz Nz[cz] Y[cz]
    float2 Ylo[Q], Yhi[Q], Zlo, Zhi;
#pragma unroll
    for (int cz = 0; cz < Q; cz++) {
        Ylo[cz] = mul2s(Ny[0], lo2(G.c[cz * Q]));
        Yhi[cz] = mul2s(Ny[0], hi2(G.c[cz * Q]));
#pragma unroll
        for (int by = 1; by < Q; by++) {
            Ylo[cz] = fma2s(Ny[by], lo2(G.c[cz * Q + by]), Ylo[cz]);
            Yhi[cz] = fma2s(Ny[by], hi2(G.c[cz * Q + by]), Yhi[cz]);
        }
    }
    Zlo = mul2s(Nz[0], Ylo[0]);
    Zhi = mul2s(Nz[0], Yhi[0]);
#pragma unroll
    for (int cz = 1; cz < Q; cz++) {
        Zlo = fma2s(Nz[cz], Ylo[cz], Zlo);
        Zhi = fma2s(Nz[cz], Yhi[cz], Zhi);
    }
    const float v = dot_x<P>(Nx, Zlo, Zhi);
    int bi;
    float bf;
    const float vc = fminf(fmaxf(v, A.dom_lo), A.dom_hi);
    const float atf = tf_alpha(A, tf, vc, bi, bf);
    if (!(atf > 0.f)) return true;  // a_s = 0: the sample changes neither C nor A
    ++M.nshade;
    float Ex[P], Ey[P], Ez[P];
    axis_fast_E<P>(b, C, 0, kx, fx, Ex);
    axis_fast_E<P>(b, C, 1, ky, fy, Ey);
    axis_fast_E<P>(b, C, 2, kz, fz, Ez);
    const float gx = ddot_x<P>(Ex, Zlo, Zhi);
    // d/dz: sum_q Ez[q] (Y[q+1] - Y[q]), then x
    float2 Dlo = mul2s(Ez[0], sub2(Ylo[1], Ylo[0])), Dhi = mul2s(Ez[0], sub2(Yhi[1], Yhi[0]));
#pragma unroll
    for (int q = 1; q < P; q++) {
        Dlo = fma2s(Ez[q], sub2(Ylo[q + 1], Ylo[q]), Dlo);
        Dhi = fma2s(Ez[q], sub2(Yhi[q + 1], Yhi[q]), Dhi);
    }
    const float gz = dot_x<P>(Nx, Dlo, Dhi);
    // d/dy: W[by] = sum_cz Nz[cz] c[cz][by]; sum_q Ey[q] (W[q+1] - W[q]), then x
    float2 Wlo[Q], Whi[Q];
#pragma unroll
    for (int by = 0; by < Q; by++) {
        Wlo[by] = mul2s(Nz[0], lo2(G.c[by]));
        Whi[by] = mul2s(Nz[0], hi2(G.c[by]));
#pragma unroll
        for (int cz = 1; cz < Q; cz++) {
            Wlo[by] = fma2s(Nz[cz], lo2(G.c[cz * Q + by]), Wlo[by]);
            Whi[by] = fma2s(Nz[cz], hi2(G.c[cz * Q + by]), Whi[by]);
        }
    }
    Dlo = mul2s(Ey[0], sub2(Wlo[1], Wlo[0]));
    Dhi = mul2s(Ey[0], sub2(Whi[1], Whi[0]));
#pragma unroll
    for (int q = 1; q < P; q++) {
        Dlo = fma2s(Ey[q], sub2(Wlo[q + 1], Wlo[q]), Dlo);
        Dhi = fma2s(Ey[q], sub2(Whi[q + 1], Whi[q]), Dhi);
    }
    const float gy = dot_x<P>(Nx, Dlo, Dhi);
    // model.py:79 gradient / span
    const float4 gi = C.ginv;
    const float g[3] = {gx * gi.x, gy * gi.y, gz * gi.z};
    composite(A, C.vdir, tf_color(tf, vc, bi, bf, atf), g, M);
    return true;
}

// ---------------------------------------------------------------------------
// Down-sampled (DS) baseline blocks (reference downsample.py, DsBlock):
// values by trilinear interpolation of the raw (ghosted) samples, gradients
// by trilinear interpolation of the clipped-index central-difference grids
// (built at upload), both at the continuous interior-lattice index
// u * (n - 1), u = clip((p - lo) / span, 0, 1) (downsample.py:107-129).
struct DsFast {
    const float *samp;  // (nx+2g)(ny+2g)(nz+2g), x fastest
    const float *grid;  // [3][nz][ny][nx]
    int32_t n[3], g;
};

// downsample._trilinear (downsample.py:131-146) on a dims[0] x dims[1] x
// dims[2] grid (x fastest) at continuous index x, float32, same op order.
__device__ __forceinline__ float ds_trilinear(const float *__restrict__ grid, const int (&dims)[3],
                                              const float (&x)[3]) {
    int i0[3], i1[3];
    float f[3];
#pragma unroll
    for (int a = 0; a < 3; a++) {
        const int top = dims[a] - 1;
        const int b = min(max(__float2int_rd(x[a]), 0), max(top - 1, 0));
        f[a] = x[a] - (float)b;
        i0[a] = b;
        i1[a] = min(b + 1, top);
    }
    const size_t sy = (size_t)dims[0], sz = (size_t)dims[0] * dims[1];
    auto at = [&](int i, int j, int k) { return __ldg(grid + (size_t)k * sz + (size_t)j * sy + i); };
    const float gx = 1.f - f[0], gy = 1.f - f[1], gz = 1.f - f[2];
    const float c00 = at(i0[0], i0[1], i0[2]) * gx + at(i1[0], i0[1], i0[2]) * f[0];
    const float c10 = at(i0[0], i1[1], i0[2]) * gx + at(i1[0], i1[1], i0[2]) * f[0];
    const float c01 = at(i0[0], i0[1], i1[2]) * gx + at(i1[0], i0[1], i1[2]) * f[0];
    const float c11 = at(i0[0], i1[1], i1[2]) * gx + at(i1[0], i1[1], i1[2]) * f[0];
    const float c0 = c00 * gy + c10 * f[1];
    const float c1 = c01 * gy + c11 * f[1];
    return c0 * gz + c1 * f[2];
}

// One DS sample from the predicted continuous interior index tq.
__device__ __forceinline__ void sample_ds(const RenderArgs &A, const TfTable &tf, const DsFast &b,
                                          const float (&tq)[3], const ThreadCold &C, March &M) {
    float xi[3], xs[3];
    int ds[3], dn[3];
#pragma unroll
    for (int a = 0; a < 3; a++) {
        xi[a] = fminf(fmaxf(tq[a], 0.f), (float)(b.n[a] - 1));
        xs[a] = xi[a] + (float)b.g;
        dn[a] = b.n[a];
        ds[a] = b.n[a] + 2 * b.g;
    }
    const float v = ds_trilinear(b.samp, ds, xs);
    int bi;
    float bf;
    const float vc = fminf(fmaxf(v, A.dom_lo), A.dom_hi);
    const float atf = tf_alpha(A, tf, vc, bi, bf);
    if (!(atf > 0.f)) return;
    ++M.nshade;
    const size_t plane = (size_t)dn[0] * dn[1] * dn[2];
    const float4 gi = C.ginv;  // (n - 1) / span per axis
    const float g[3] = {ds_trilinear(b.grid, dn, xi) * gi.x, ds_trilinear(b.grid + plane, dn, xi) * gi.y,
                        ds_trilinear(b.grid + 2 * plane, dn, xi) * gi.z};
    composite(A, C.vdir, tf_color(tf, vc, bi, bf, atf), g, M);
}

// One sample on the exact path: float64 position, the reference's span
// search; float32 (non-uniform knots, P = 1 near a knot) or float64
// (ill-conditioned slot) arithmetic.  Out of line (rare), so its registers
// do not weigh on the fast loop; arguments and results go through shared
// memory (GA: the launch arguments in global memory, tf: the block's shared
// TF table, R: this ray).
// Returns 1 when the slot is float64.
template <int P>
__device__ __noinline__ int sample_exact(const RenderArgs *GA, const TfTable *tf, RayState *R,
                                         const BlockDesc *__restrict__ dp,
                                         int32_t slot, int32_t k) {
    double pos[3];
    exact_pos(*GA, *R, k, pos);
    BlockLite b;
    load_lite(dp, b);
    GatherCache G;
    G.slot = -1;
    float v, g[3];
    float4 tfv;
    const bool f64 = b.flags & AFAM_SLOT_FP64;
    if (f64) {
        decode_f64<P>(b, dp, slot, G, pos, *tf, GA->dom_lo, GA->dom_hi, v, tfv, g);
    } else {
        decode_f32<P>(b, dp, slot, G, pos, *tf, GA->dom_lo, GA->dom_hi, v, tfv, g);
    }
    R->tfv = tfv;
    R->g[0] = g[0];
    R->g[1] = g[1];
    R->g[2] = g[2];
    return f64 ? 1 : 0;
}

// Degrees above AFAM_FAST_DEGREE: float64 evaluation from the knots
// (afam_eval.cuh eval_any, the reference's Cox-de Boor with its divisions),
// parameters with the reference's division (model.py:64-68); always a
// float64 sample.  Compiled only into the render2_kernel instantiations the
// host selects for frames holding such blocks (HI), so the common kernels
// carry no trace of its frame.
__device__ __noinline__ int sample_exact_any(const RenderArgs *GA, const TfTable *tf, RayState *R,
                                             const BlockDesc *__restrict__ dp, int32_t k) {
    double pos[3];
    exact_pos(*GA, *R, k, pos);
    const BlockDesc d = load_desc(dp);
    double u[3], gg[3];
#pragma unroll
    for (int a = 0; a < 3; a++) u[a] = clamp01(__ddiv_rn(__dsub_rn(pos[a], d.lo[a]), d.span[a]));
    const double v = eval_any(d, u, gg);
    const float4 tfv = tf_eval(*tf, fminf(fmaxf((float)v, GA->dom_lo), GA->dom_hi));
    R->tfv = tfv;
#pragma unroll
    for (int a = 0; a < 3; a++) R->g[a] = tfv.w > 0.f ? (float)(gg[a] / d.span[a]) : 0.f;
    return 1;
}

template <bool DEBUG, bool SMEM_GRID, int FD, int MINB>
__global__ void __launch_bounds__(128, MINB) render_kernel(const BlockDesc *__restrict__ descs,
                                                        const int16_t *__restrict__ grid,
                                                        const int32_t *__restrict__ idx2slot, const RenderArgs A,
                                                        const RenderArgs *__restrict__ GA,
                                                        const TfTable *__restrict__ gtf, uint8_t *__restrict__ rgba,
                                                        afam_render_stats *stats, int32_t *__restrict__ nsamp,
                                                        uint64_t *__restrict__ ohash) {
    extern __shared__ __align__(16) unsigned char smem[];
    // the TF tables stay in global memory (one L1-resident copy per SM, read
    // through the read-only path), shared memory holds only the owner grid,
    // so L1 keeps the most room for control-point rows; GA: the launch
    // arguments in global memory, for the out-of-line exact path
    const TfTable &tf = *gtf;
    ThreadCold &C = s_cold[threadIdx.x];
    int16_t *sgrid = reinterpret_cast<int16_t *>(smem + kSmemGridOff);
    for (int i = threadIdx.x; i < kTfBuckets; i += blockDim.x) s_tf_alpha[i] = gtf->alpha[i];
    if (SMEM_GRID)
        for (int i = threadIdx.x; i < A.cells * A.cells * A.cells; i += blockDim.x) sgrid[i] = grid[i];
    __syncthreads();
    const int16_t *own_grid = SMEM_GRID ? sgrid : grid;
    RayState R;  // local memory: touched on the exact paths only

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int WPR = kCtaW / kWarpW;  // the render2_kernel tiles
    const int j = blockIdx.x * kCtaW + (warp % WPR) * kWarpW + (lane % kWarpW);
    const int lr = blockIdx.y * (128 / kCtaW) + (warp / WPR) * (32 / kWarpW) + lane / kWarpW;
    const bool inside = j < A.width && lr < A.rows;
    const int i = inside ? frame_row(A, lr) : 0;

    // _ray_grid (render.py:332-337): exact op order, no contraction
    const double xs = __dsub_rn(__dmul_rn(__ddiv_rn((double)j, (double)A.width), 2.0), 1.0);
    const double ys = __dsub_rn(1.0, __dmul_rn(__ddiv_rn((double)i, (double)A.height), 2.0));
    const double px = __dmul_rn(xs, A.tan_x), py = __dmul_rn(ys, A.tan_y);
    double d[3];
#pragma unroll
    for (int a = 0; a < 3; a++) d[a] = __dadd_rn(__dadd_rn(A.f[a], __dmul_rn(px, A.r[a])), __dmul_rn(py, A.u[a]));
    const double nrm =
        __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(d[0], d[0]), __dmul_rn(d[1], d[1])), __dmul_rn(d[2], d[2])));
#pragma unroll
    for (int a = 0; a < 3; a++) d[a] = __ddiv_rn(d[a], nrm);
    // _ray_box_span (render.py:340-354)
    double te = -INFINITY, tx = INFINITY;
#pragma unroll
    for (int a = 0; a < 3; a++) {
        const double inv = __drcp_rn(d[a]);
        const double ta = __dmul_rn(__dsub_rn(-1.0, A.origin[a]), inv);
        const double tb = __dmul_rn(__dsub_rn(1.0, A.origin[a]), inv);
        double lo = fmin(ta, tb), hi = fmax(ta, tb);
        if (isnan(lo)) lo = -INFINITY;
        if (isnan(hi)) hi = INFINITY;
        te = fmax(te, lo);
        tx = fmin(tx, hi);
    }
    te = fmax(te, A.near_);
    const bool active = inside && te < tx;
#pragma unroll
    for (int a = 0; a < 3; a++) R.d[a] = d[a];
    R.te = te;

    C.vdir = make_float4((float)d[0], (float)d[1], (float)d[2], 0.f);
    C.ns64 = C.nexact = C.ncell = C.nclear = 0;
    March M;
    M.k = 0;
    M.kend = 0;
    M.kf = 0.f;
    M.C0 = M.C1 = M.C2 = M.Aacc = 0.f;
    M.nshade = 0;
    M.h = 1469598103934665603ULL;
    M.own = -1;

    if (active) {
        // alive samples: t_k = te + (k + 0.5) sd < tx, a prefix of k (render.py:423)
        auto tk = [&](int64_t k) { return __dadd_rn(te, __dmul_rn((double)k + 0.5, A.sd)); };
        int64_t ke = (int64_t)fmax(ceil((tx - te) / A.sd - 0.5), 0.0);
        while (ke > 0 && !(tk(ke - 1) < tx)) --ke;
        while (tk(ke) < tx) ++ke;
        M.kend = (int32_t)min(ke, (int64_t)INT32_MAX);
        // the float32 sample index kf and span prediction need k < 2^24
        const bool k24 = ke < (1 << 24);
        {
            double p[3];
            exact_geometry(A, R, own_grid, 0, M.kend, p, M.own, M.knext);
        }
        int32_t cur_own = -1, slot = -1, deg = 0;
        BlockFast b;
        bool fast = false;
        CellCache G;
        G.key = -1;
        DsFast dsb;
        while (M.k < M.kend) {
            if (M.own < 0) break;  // render.py:430-436 (reported after the loop)
            if (M.own != cur_own) {
                cur_own = M.own;
                slot = __ldg(idx2slot + cur_own);
                const BlockDesc *dp = descs + slot;
                if constexpr (FD == 0) {  // DS blocks (AFAM_SLOT_DS)
                    dsb.samp = (const float *)__ldg((const unsigned long long *)&dp->ctrl);
                    dsb.grid = (const float *)__ldg((const unsigned long long *)&dp->ctrl4);
                    dsb.g = __ldg(&dp->deg);
                    double p[3];
                    exact_pos(A, R, M.k, p);
                    float gs[3];
#pragma unroll
                    for (int a = 0; a < 3; a++) {
                        dsb.n[a] = __ldg(&dp->ds_n[a]);
                        const double sc = __ldg(&dp->inv_span[a]) * (double)(dsb.n[a] - 1);
                        M.tq0[a] = (float)((p[a] - __ldg(&dp->lo[a])) * sc);
                        M.dtq[a] = (float)(A.sd * R.d[a] * sc);
                        gs[a] = (float)sc;
                    }
                    C.ginv = make_float4(gs[0], gs[1], gs[2], 0.f);
                    M.k0f = M.kf;
                    fast = true;
                } else {
                b.ctrl4 = (const float4 *)__ldg((const unsigned long long *)&dp->ctrl4);
                C.tab32 = (const float *)__ldg((const unsigned long long *)&dp->tab32);
                b.ncp = __ldg(&dp->ncp);
                b.nspan = __ldg(&dp->nspan);
                b.plane = b.ncp * b.ncp;
                b.nint = (uint32_t)max(b.nspan - 2 * (FD > 0 ? FD : 1) + 2, 0);
                G.key = -1;
                deg = __ldg(&dp->deg);
                const uint32_t flags = __ldg(&dp->flags);
                fast = deg == FD && (flags & kFlagUniform) && !(flags & AFAM_SLOT_FP64) && (deg > 1 || b.nspan <= 128) &&
                       k24 && !(A.flags & kRenderForceExact);
                // span-coordinate prediction from the exact entry position
                double p[3];
                exact_pos(A, R, M.k, p);
#pragma unroll
                for (int a = 0; a < 3; a++) {
                    const double sc = __ldg(&dp->inv_span[a]) * (double)b.nspan;
                    M.tq0[a] = (float)((p[a] - __ldg(&dp->lo[a])) * sc);
                    M.dtq[a] = (float)(A.sd * R.d[a] * sc);
                }
                C.ginv = make_float4(__ldg(&dp->inv_span_f[0]), __ldg(&dp->inv_span_f[1]),
                                     __ldg(&dp->inv_span_f[2]), 0.f);
                M.k0f = M.kf;
                }
            }
            // one sample per iteration (a flat loop keeps the lanes of a warp
            // in step across their different block runs)
            if (DEBUG) M.h = (M.h ^ (uint64_t)(uint32_t)cur_own) * 1099511628211ULL;
            bool ok = false;
            if constexpr (FD == 0) {
                const float dk = M.kf - M.k0f;
                const float tq[3] = {fmaf(dk, M.dtq[0], M.tq0[0]), fmaf(dk, M.dtq[1], M.tq0[1]),
                                     fmaf(dk, M.dtq[2], M.tq0[2])};
                sample_ds(A, tf, dsb, tq, C, M);
                ok = true;
            } else if (fast) {
                const float dk = M.kf - M.k0f;
                const float tq[3] = {fmaf(dk, M.dtq[0], M.tq0[0]), fmaf(dk, M.dtq[1], M.tq0[1]),
                                     fmaf(dk, M.dtq[2], M.tq0[2])};
                ok = sample_fast<(FD > 0 ? FD : 1)>(A, tf, b, tq, C, G, M);
            }
            if (!ok) {
                const BlockDesc *dpx = descs + slot;
                int f64;
                if (deg == 3) f64 = sample_exact<3>(GA, &tf, &R, dpx, slot, M.k);
                else if (deg == 2) f64 = sample_exact<2>(GA, &tf, &R, dpx, slot, M.k);
                else f64 = sample_exact<1>(GA, &tf, &R, dpx, slot, M.k);  // (the host routes degrees > 3 to render2_kernel)
                C.ns64 += f64;
                ++C.nexact;
                const float4 tfv = R.tfv;
                if (tfv.w > 0.f) {
                    ++M.nshade;
                    const float g[3] = {R.g[0], R.g[1], R.g[2]};
                    composite(A, C.vdir, tfv, g, M);
                }
            }
            // render.py:423 alive test before the next sample
            ++M.k;
            M.kf += 1.f;
            if (M.k >= M.kend || !(M.Aacc <= A.o_max_f)) break;
            if (M.k >= M.knext) {
                double p[3];
                ++C.ncell;
                exact_geometry(A, R, own_grid, M.k, M.kend, p, M.own, M.knext);
            }
        }
    }
    const uint32_t ns = (uint32_t)M.k;
    if (inside) {
        // render.py:458-461 quantise (round half to even)
        uchar4 px4;
        px4.x = (unsigned char)min(max(__float2int_rn(M.C0 * 255.f), 0), 255);
        px4.y = (unsigned char)min(max(__float2int_rn(M.C1 * 255.f), 0), 255);
        px4.z = (unsigned char)min(max(__float2int_rn(M.C2 * 255.f), 0), 255);
        px4.w = (unsigned char)min(max(__float2int_rn(M.Aacc * 255.f), 0), 255);
        const int64_t local = (int64_t)lr * A.width + j;
        // full-frame output: this part's rows at their frame rows (a peer GPU's frame over NVLink)
        const int64_t dst = (A.flags & AFAM_RENDER_FULL_FRAME) ? (int64_t)i * A.width + j : local;
        reinterpret_cast<uchar4 *>(rgba)[dst] = px4;
        if (DEBUG) {
            nsamp[local] = (int32_t)ns;
            ohash[local] = M.h;
        }
    }
    // per-warp reductions of the counters
    const uint32_t wsum = __reduce_add_sync(0xffffffffu, ns);
    const uint32_t wsum64 = __reduce_add_sync(0xffffffffu, C.ns64);
    const uint32_t wshade = __reduce_add_sync(0xffffffffu, M.nshade);
    const uint32_t wexact = __reduce_add_sync(0xffffffffu, C.nexact);
    const uint32_t wcell = __reduce_add_sync(0xffffffffu, C.ncell);
    // the march stopped at a sample without a resident owner: (step, full-frame ray id)
    int64_t wmiss = M.own < 0 && M.k < M.kend ? ((int64_t)M.k << 32) | ((int64_t)i * A.width + j) : INT64_MAX;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const int64_t other = __shfl_xor_sync(0xffffffffu, wmiss, o);
        wmiss = other < wmiss ? other : wmiss;
    }
    if (lane == 0) {
        if (wsum) atomicAdd((unsigned long long *)&stats->samples, (unsigned long long)wsum);
        if (wsum64) atomicAdd((unsigned long long *)&stats->fp64_samples, (unsigned long long)wsum64);
        if (wshade) atomicAdd((unsigned long long *)&stats->shaded_samples, (unsigned long long)wshade);
        if (wexact) atomicAdd((unsigned long long *)&stats->exact_samples, (unsigned long long)wexact);
        if (wcell) atomicAdd((unsigned long long *)&stats->exact_cells, (unsigned long long)wcell);
        if (wmiss != INT64_MAX) atomicMin((long long *)&stats->missing_key, (long long)wmiss);
    }
}

// ---------------------------------------------------------------------------
// K2, restructured sample loop (render2_kernel): the same numerics as
// render_kernel's fast path (identical span coordinates, bases, contraction
// order and compositing, so the frames are bit-identical), with the work
// that is constant within a knot cell hoisted out of the per-sample path:
//  - the lane's current cell is kept as its lower corner (float span
//    coordinates); a sample stays in the cell iff its three fractions
//    tq - corner lie in [0, 1) (three unsigned compares on the float bits),
//    so the span, clamp, cell key and interior test are recomputed only on
//    a cell change (about one sample in four at LOD-2 span widths);
//  - which axes sit on interior spans (closed-form uniform basis) is a
//    per-cell bit mask;
//  - the owner change, the next exact-geometry sample and the end of the
//    ray are one per-sample compare against the segment end
//    min(knext, kend).
// The cell's x-quad rows cz*Q+by (bspline.py:175-181): the first NR in
// registers, the last SR in this thread's column of a shared array
// (s[k * 128]), so SR trades registers (occupancy) for LDS traffic.
template <int P, int SR>
struct FastCell {
    static constexpr int NR = (P + 1) * (P + 1) - SR;
    float4 c[NR > 0 ? NR : 1];
    float4 *s;                    // this thread's shared rows (stride 128)
    float cx, cy, cz;             // the cell's lower corner in span coordinates
    uint32_t lim;                 // float bits of the cell's width: 1 (a knot cell) or 4 (a transparent
                                  // 4x4x4 group, AFAM_CELL_GROUP)
    int32_t key;                  // x-quad row index of the (0, 0) row in the owner block; -1: none
    uint32_t inner;               // bit a: axis a on an interior span
    __device__ __forceinline__ float4 get(int i) const { return i < NR ? c[i] : s[(i - NR) * 128]; }
    __device__ __forceinline__ void set(int i, float4 v) {
        if (i < NR) c[i] = v;
        else s[(i - NR) * 128] = v;
    }
};

__device__ __forceinline__ bool in_unit(float f) {  // 0 <= f < 1 (also rejects -0.0 and NaN)
    return __float_as_uint(f) < 0x3f800000u;
}
__device__ __forceinline__ bool in_lim(float f, uint32_t lim) {  // 0 <= f < lim (lim: float bits)
    return __float_as_uint(f) < lim;
}
constexpr uint32_t kLim1 = 0x3f800000u, kLim4 = 0x40800000u;

// Re-derive the cell of predicted span coordinates tq (render_kernel's
// axis_span: floor, clamped to the block's spans) and re-gather its rows
// when the cell key changed.
template <int P>
__device__ __forceinline__ BlockFast fast_block(const BlockFast &sb) {  // sb in shared memory
    BlockFast b;
    b.ctrl4 = vld(sb.ctrl4);
    b.rng = vld(sb.rng);
    b.ncp = vld(sb.ncp);
    b.nspan = vld(sb.nspan);
    b.plane = vld(sb.plane);
    b.nint = vld(sb.nint);
    return b;
}

#ifndef AFAM_CELL_GROUP
#define AFAM_CELL_GROUP 1  // transparent 4x4x4 cell groups passed as one cell (float32 fast path)
#endif
#ifndef AFAM_CELL_SKIP
#define AFAM_CELL_SKIP 1  // skip the samples of cells the TF makes transparent (BlockDesc::crange)
#endif

// Bit 3 of FastCell::inner: every value the cell can produce is outside the
// TF's opacity support, so its samples are transparent without decoding
// (the per-sample test of sample_fast2 would return on each of them) and
// its rows are not gathered.
constexpr uint32_t kCellClear = 8u;

template <int P, int SR, int SKIP = 0>
__device__ __forceinline__ void fast_cell_update_k(const BlockFast &b, int kx, int ky, int kz, FastCell<P, SR> &G,
                                                   const RenderArgs *A = nullptr) {
    constexpr int Q = P + 1;
    G.cx = (float)kx;
    G.cy = (float)ky;
    G.cz = (float)kz;
    G.inner = (span_interior<P>(b, kx) ? 1u : 0u) | (span_interior<P>(b, ky) ? 2u : 0u) |
              (span_interior<P>(b, kz) ? 4u : 0u);
    G.lim = kLim1;
    if constexpr (SKIP != 0 && AFAM_CELL_SKIP) {
        // the clamp of render.py's value to the TF domain is monotone: the
        // clamped range bounds every clamped sample value
        auto clear = [&](float2 r) { return !(r.y > A->clr_lo) || !(r.x < A->clr_hi); };
        const int ns = b.nspan;
        const float2 r = __ldg(b.rng + (kz * ns + kx) * ns + ky);
        if (SKIP == 2 && AFAM_CELL_GROUP) {
            // the cell's aligned 4x4x4 group (loaded beside the cell's own
            // range): when the whole group is transparent the lane treats it
            // as one cell of width 4 -- any sample whose span coordinates lie
            // in it falls in one of its cells (the clamp to the block's spans
            // keeps the group's cells), so it is transparent too
            const int n4 = (ns + 3) >> 2;
            const float2 r4 = __ldg(b.rng + ns * ns * ns + ((kz >> 2) * n4 + (kx >> 2)) * n4 + (ky >> 2));
            if (clear(r4)) {
                G.cx = (float)(kx & ~3);
                G.cy = (float)(ky & ~3);
                G.cz = (float)(kz & ~3);
                G.lim = kLim4;
                G.inner |= kCellClear;
                return;
            }
        }
        if (clear(r)) {
            G.inner |= kCellClear;
            return;  // the rows of G.key stay valid for that key
        }
    }
    const int32_t id = (kz * b.ncp + kx) * b.ncp + ky;
    if (id != G.key) {
        const float4 *base = b.ctrl4 + id;
#pragma unroll
        for (int cz = 0; cz < Q; cz++)
#pragma unroll
            for (int by = 0; by < Q; by++) G.set(cz * Q + by, __ldg(base + cz * b.plane + by));
        G.key = id;
    }
}

template <int P, int SR>
__device__ __forceinline__ void fast_cell_update(const BlockFast &sb, float tqx, float tqy, float tqz,
                                                 FastCell<P, SR> &G, const RenderArgs &A) {
    const BlockFast b = fast_block<P>(sb);
    const int kx = min(max(__float2int_rd(tqx), 0), b.nspan - 1);
    const int ky = min(max(__float2int_rd(tqy), 0), b.nspan - 1);
    const int kz = min(max(__float2int_rd(tqz), 0), b.nspan - 1);
    fast_cell_update_k<P, SR, 2>(b, kx, ky, kz, G, &A);
}

// One sample of a clamped-uniform float32 block (render_kernel's
// sample_fast, same arithmetic).  Returns false when the exact path must
// decode it (P = 1 within 1e-4 of a knot).
template <int P, int SR>
__device__ __forceinline__ bool sample_fast2(const RenderArgs &A, const TfTable &tf, const BlockFast &sb, float tqx,
                                             float tqy, float tqz, const ThreadCold &C, FastCell<P, SR> &G,
                                             March &M) {
    constexpr int Q = P + 1;
    float fx = tqx - G.cx, fy = tqy - G.cy, fz = tqz - G.cz;
    if (!(in_lim(fx, G.lim) & in_lim(fy, G.lim) & in_lim(fz, G.lim))) {
        fast_cell_update<P, SR>(sb, tqx, tqy, tqz, G, A);
        fx = tqx - G.cx;
        fy = tqy - G.cy;
        fz = tqz - G.cz;
    }
    if (AFAM_CELL_SKIP && (G.inner & kCellClear)) return true;  // transparent: changes neither C nor A
    if constexpr (P == 1) {
        if (!(fabsf(fx - 0.5f) < 0.5f - 1e-4f) || !(fabsf(fy - 0.5f) < 0.5f - 1e-4f) ||
            !(fabsf(fz - 0.5f) < 0.5f - 1e-4f))
            return false;
    }
    float Nx[Q], Ny[Q], Nz[Q];
    {
        float2 Nxy[Q];
        uniform_N2<P>(make_float2(fx, fy), Nxy);
#pragma unroll
        for (int i = 0; i < Q; i++) {
            Nx[i] = Nxy[i].x;
            Ny[i] = Nxy[i].y;
        }
        if (G.inner == 7u) {
            uniform_N<P>(fz, Nz);
        } else {
            const BlockFast b = fast_block<P>(sb);
            if (!(G.inner & 1u)) axis_table_N<P>(b, C, 0, (int)G.cx, tqx, Nx);
            if (!(G.inner & 2u)) axis_table_N<P>(b, C, 1, (int)G.cy, tqy, Ny);
            if (G.inner & 4u) uniform_N<P>(fz, Nz);
            else axis_table_N<P>(b, C, 2, (int)G.cz, tqz, Nz);
        }
    }
    float2 Ylo[Q], Yhi[Q], Zlo, Zhi;
#pragma unroll
    for (int cz = 0; cz < Q; cz++) {
        Ylo[cz] = mul2s(Ny[0], lo2(G.get(cz * Q)));
        Yhi[cz] = mul2s(Ny[0], hi2(G.get(cz * Q)));
#pragma unroll
        for (int by = 1; by < Q; by++) {
            Ylo[cz] = fma2s(Ny[by], lo2(G.get(cz * Q + by)), Ylo[cz]);
            Yhi[cz] = fma2s(Ny[by], hi2(G.get(cz * Q + by)), Yhi[cz]);
        }
    }
    if constexpr (P == 3) {  // pairwise trees: depth 3 instead of 4-long chains
        Zlo = __fadd2_rn(fma2s(Nz[1], Ylo[1], mul2s(Nz[0], Ylo[0])), fma2s(Nz[3], Ylo[3], mul2s(Nz[2], Ylo[2])));
        Zhi = __fadd2_rn(fma2s(Nz[1], Yhi[1], mul2s(Nz[0], Yhi[0])), fma2s(Nz[3], Yhi[3], mul2s(Nz[2], Yhi[2])));
    } else {
        Zlo = mul2s(Nz[0], Ylo[0]);
        Zhi = mul2s(Nz[0], Yhi[0]);
#pragma unroll
        for (int cz = 1; cz < Q; cz++) {
            Zlo = fma2s(Nz[cz], Ylo[cz], Zlo);
            Zhi = fma2s(Nz[cz], Yhi[cz], Zhi);
        }
    }
    float v;
    if constexpr (P == 3) {
        const float2 t = __ffma2_rn(Zhi, make_float2(Nx[2], Nx[3]), __fmul2_rn(Zlo, make_float2(Nx[0], Nx[1])));
        v = t.x + t.y;
    } else {
        v = dot_x<P>(Nx, Zlo, Zhi);
    }
    int bi;
    float bf;
    // outside the TF's opacity support alpha_tf is exactly 0: no lookup
    // (clr_lo/clr_hi: the support pulled back through the domain clamp)
    if (!(v > A.clr_lo) || !(v < A.clr_hi)) return true;
    const float vc = fminf(fmaxf(v, A.dom_lo), A.dom_hi);
    const float atf = tf_alpha(A, tf, vc, bi, bf);
    if (!(atf > 0.f)) return true;  // a_s = 0: the sample changes neither C nor A
    ++M.nshade;
    float Ex[P], Ey[P], Ez[P];
    if (G.inner == 7u) {
        const float nsf = (float)vld(sb.nspan);
        uniform_E<P>(fx, nsf, Ex);
        uniform_E<P>(fy, nsf, Ey);
        uniform_E<P>(fz, nsf, Ez);
    } else {
        const BlockFast b = fast_block<P>(sb);
        axis_fast_E<P>(b, C, 0, (int)G.cx, fx, Ex);
        axis_fast_E<P>(b, C, 1, (int)G.cy, fy, Ey);
        axis_fast_E<P>(b, C, 2, (int)G.cz, fz, Ez);
    }
    const float gx = ddot_x<P>(Ex, Zlo, Zhi);
    float2 Dlo = mul2s(Ez[0], sub2(Ylo[1], Ylo[0])), Dhi = mul2s(Ez[0], sub2(Yhi[1], Yhi[0]));
#pragma unroll
    for (int q = 1; q < P; q++) {
        Dlo = fma2s(Ez[q], sub2(Ylo[q + 1], Ylo[q]), Dlo);
        Dhi = fma2s(Ez[q], sub2(Yhi[q + 1], Yhi[q]), Dhi);
    }
    const float gz = dot_x<P>(Nx, Dlo, Dhi);
    float2 Wlo[Q], Whi[Q];
#pragma unroll
    for (int by = 0; by < Q; by++) {
        Wlo[by] = mul2s(Nz[0], lo2(G.get(by)));
        Whi[by] = mul2s(Nz[0], hi2(G.get(by)));
#pragma unroll
        for (int cz = 1; cz < Q; cz++) {
            Wlo[by] = fma2s(Nz[cz], lo2(G.get(cz * Q + by)), Wlo[by]);
            Whi[by] = fma2s(Nz[cz], hi2(G.get(cz * Q + by)), Whi[by]);
        }
    }
    Dlo = mul2s(Ey[0], sub2(Wlo[1], Wlo[0]));
    Dhi = mul2s(Ey[0], sub2(Whi[1], Whi[0]));
#pragma unroll
    for (int q = 1; q < P; q++) {
        Dlo = fma2s(Ey[q], sub2(Wlo[q + 1], Wlo[q]), Dlo);
        Dhi = fma2s(Ey[q], sub2(Whi[q + 1], Whi[q]), Dhi);
    }
    const float gy = dot_x<P>(Nx, Dlo, Dhi);
    const float4 gi = C.ginv;
    const float g[3] = {gx * gi.x, gy * gi.y, gz * gi.z};
    composite(A, C.vdir, tf_color(tf, vc, bi, bf, atf), g, M);
    return true;
}

// ---------------------------------------------------------------------------
// Float64 fast path (render2_kernel<..., F64>, frames holding ill-conditioned
// slots: endpoint-pinned fits whose large cancelling
// coefficients need float64 basis and accumulation): the float32 fast
// path's schedule -- the owner block's cell rows cached in registers across
// samples, the span coordinate predicted from the exact block-entry position
// (tq0 + (k - k0) dtq, now in float64), closed-form uniform bases on interior
// spans (the float64 Cox-de Boor table on the boundary spans), contraction
// and gradient in float64 -- instead of the exact path's per-sample float64
// position, division, span search, table loads and uncached gather.
// -DAFAM_F64_VALUE_FIRST=1: value-first float64 samples in the all-fast kernel
// (measured: 3.15 vs 3.11 ms on config 2 -- the saved DFMAs of transparent
// samples are eaten by 228 bytes of spills)
#ifndef AFAM_F64_VALUE_FIRST
#define AFAM_F64_VALUE_FIRST 0
#endif
constexpr bool F64_VF = AFAM_F64_VALUE_FIRST != 0;

struct Pred64 {  // per thread, shared memory: the float64 span prediction of the current owner
    double tq0[3], dtq[3];
    const double *tab64;
};
__shared__ Pred64 s_pred64[128];

// uniform_basis (afam_eval.cuh) in float64
template <int P>
__device__ __forceinline__ void uniform_NE_f64(double x, double ns, double (&N)[P + 1], double (&E)[P]) {
    const double m = 1.0 - x;
    if (P == 1) {
        N[0] = m;
        N[1] = x;
        E[0] = ns;
    } else if (P == 2) {
        const double x2 = x * x;
        N[0] = 0.5 * m * m;
        N[1] = fma(-1.0, x2, x) + 0.5;
        N[2] = 0.5 * x2;
        E[0] = ns * m;
        E[1] = ns * x;
    } else {
        const double x2 = x * x, x3 = x2 * x, m2 = m * m, s6 = 1.0 / 6.0;
        N[0] = s6 * m2 * m;
        N[1] = fma(0.5, x3, fma(-1.0, x2, 2.0 / 3.0));
        N[2] = fma(-0.5, x3, fma(0.5, x2, fma(0.5, x, s6)));
        N[3] = s6 * x3;
        const double hn = 0.5 * ns;
        E[0] = hn * m2;
        E[1] = ns * (fma(-1.0, x2, x) + 0.5);
        E[2] = hn * x2;
    }
}

// VF: value first, the derivative weights and the gradient contraction only
// for samples the TF makes visible
template <int P, int SR, bool VF>
__device__ __forceinline__ bool sample_fast64(const RenderArgs &A, const TfTable &tf, const BlockFast &sb,
                                              const Pred64 &PD, float dk, ThreadCold &C, FastCell<P, SR> &G,
                                              March &M) {
    constexpr int Q = P + 1;
    const double dkd = (double)dk;
    double tq[3], f[3];
#pragma unroll
    for (int a = 0; a < 3; a++) tq[a] = fma(dkd, vld(PD.dtq[a]), vld(PD.tq0[a]));
    f[0] = tq[0] - (double)G.cx;
    f[1] = tq[1] - (double)G.cy;
    f[2] = tq[2] - (double)G.cz;
    auto in01 = [](double v) { return v >= 0.0 && v < 1.0; };
    if (!(in01(f[0]) & in01(f[1]) & in01(f[2]))) {
        const BlockFast b = fast_block<P>(sb);
        int k[3];
#pragma unroll
        for (int a = 0; a < 3; a++) k[a] = min(max((int)floor(tq[a]), 0), b.nspan - 1);
        fast_cell_update_k<P, SR, 1>(b, k[0], k[1], k[2], G, &A);
#pragma unroll
        for (int a = 0; a < 3; a++) f[a] = tq[a] - (double)k[a];
    }
    if constexpr (P == 1) {  // the gradient jumps at a knot: the exact path decides there
#pragma unroll
        for (int a = 0; a < 3; a++)
            if (!(fabs(f[a] - 0.5) < 0.5 - 1e-4)) return false;
    }
    // transparent cell (the float64 value rounds into the cell's widened range)
    if (AFAM_CELL_SKIP && (G.inner & kCellClear)) {
        ++C.ns64;
        return true;
    }
    // basis values now, the derivative weights only for visible samples
    auto basis = [&](int a, double (&Na)[Q], double (&Ea)[P]) {
        const int nspan = vld(sb.nspan);
        if (G.inner & (1u << a)) {
            uniform_NE_f64<P>(f[a], (double)nspan, Na, Ea);
        } else {  // boundary span: float64 Cox-de Boor from the span's table entry
            const int k = (int)(a == 0 ? G.cx : (a == 1 ? G.cy : G.cz));
            Tab<double> t;
            load_entry<P>(vld(PD.tab64) + ((size_t)a * nspan + k) * tab_stride(P), t);
            basis_eval<P, double>(t, clamp01(tq[a] / (double)nspan), Na, Ea);
        }
    };
    double N[3][Q];
    double E[3][P];
    double v, g[3];
    if constexpr (VF) {
#pragma unroll
        for (int a = 0; a < 3; a++) {
            double Ed[P];
            basis(a, N[a], Ed);
        }
        v = 0.0;
#pragma unroll
        for (int cz = 0; cz < Q; cz++) {
            double ay = 0.0;
#pragma unroll
            for (int by = 0; by < Q; by++) {
                const float4 r = G.get(cz * Q + by);
                double acc = N[0][0] * (double)r.x;
                acc = fma(N[0][1], (double)r.y, acc);
                if constexpr (P >= 2) acc = fma(N[0][2], (double)r.z, acc);
                if constexpr (P >= 3) acc = fma(N[0][3], (double)r.w, acc);
                ay = fma(N[1][by], acc, ay);
            }
            v = fma(N[2][cz], ay, v);
        }
    } else {
#pragma unroll
        for (int a = 0; a < 3; a++) basis(a, N[a], E[a]);
        float4 c4[16];
#pragma unroll
        for (int i = 0; i < Q * Q; i++) c4[i] = G.get(i);
        contract_quad<P, double>(c4, N[0], E[0], N[1], E[1], N[2], E[2], v, g);
    }
    ++C.ns64;
    if (!((float)v > A.clr_lo) || !((float)v < A.clr_hi)) return true;
    const float vc = fminf(fmaxf((float)v, A.dom_lo), A.dom_hi);
    int bi;
    float bf;
    const float atf = tf_alpha(A, tf, vc, bi, bf);
    if (!(atf > 0.f)) return true;
    ++M.nshade;
    if constexpr (VF) {
#pragma unroll
        for (int a = 0; a < 3; a++) basis(a, N[a], E[a]);
        float4 c4[16];
#pragma unroll
        for (int i = 0; i < Q * Q; i++) c4[i] = G.get(i);
        double vv;
        contract_quad<P, double>(c4, N[0], E[0], N[1], E[1], N[2], E[2], vv, g);
    }
    const float4 gi = C.ginv;
    const float gs[3] = {(float)g[0] * gi.x, (float)g[1] * gi.y, (float)g[2] * gi.z};  // model.py:79
    composite(A, C.vdir, tf_color(tf, vc, bi, bf, atf), gs, M);
    return true;
}

// AF ("all fast"): the host checked that every resident block takes the
// fast path (degree P, clamped-uniform knots, float32 slot, rays shorter
// than 2^24 samples, no forced exact path), so the per-sample fast / exact
// dispatch is compiled out.
template <bool DEBUG, bool SMEM_GRID, int P, int MINB, int SR, bool HI, bool F64, bool AF>
__global__ void __launch_bounds__(128, MINB) render2_kernel(const BlockDesc *__restrict__ descs,
                                                         const int16_t *__restrict__ grid,
                                                         const int32_t *__restrict__ idx2slot, const RenderArgs A,
                                                         const RenderArgs *__restrict__ GA,
                                                         const TfTable *__restrict__ gtf, uint8_t *__restrict__ rgba,
                                                         afam_render_stats *stats, int32_t *__restrict__ nsamp,
                                                         uint64_t *__restrict__ ohash) {
    extern __shared__ __align__(16) unsigned char smem[];
    const TfTable &tf = *gtf;
    ThreadCold &C = s_cold[threadIdx.x];
    int16_t *sgrid = reinterpret_cast<int16_t *>(smem + kSmemGridOff);
    for (int i = threadIdx.x; i < kTfBuckets; i += blockDim.x) s_tf_alpha[i] = gtf->alpha[i];
    if (SMEM_GRID)
        for (int i = threadIdx.x; i < A.cells * A.cells * A.cells; i += blockDim.x) sgrid[i] = grid[i];
    __syncthreads();
    const int16_t *own_grid = SMEM_GRID ? sgrid : grid;
    RayState R;
    // state the sample loop reads only at cell changes and segment ends
    // (owner block fields, ray end, next exact sample) lives in shared
    // memory, so the registers hold the cached cell and the per-sample state
    FastCold &F = s_fast[threadIdx.x];

    // this thread's pixel: column j, local row lr, frame row i (recomputed
    // after the march instead of held in registers across it)
    auto pixel = [&](int &j, int &lr, int &i) {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        constexpr int W = kWarpW, WPR = kCtaW / kWarpW;  // warp tile W x (32 / W), WPR warps per CTA row
        j = blockIdx.x * kCtaW + (warp % WPR) * W + (lane % W);
        lr = blockIdx.y * (128 / kCtaW) + (warp / WPR) * (32 / W) + lane / W;
        const bool in = j < A.width && lr < A.rows;
        i = in ? frame_row(A, lr) : 0;
        return in;
    };
    int j, lr, i;
    bool inside = pixel(j, lr, i);

    // _ray_grid (render.py:332-337): exact op order, no contraction
    const double xs = __dsub_rn(__dmul_rn(__ddiv_rn((double)j, (double)A.width), 2.0), 1.0);
    const double ys = __dsub_rn(1.0, __dmul_rn(__ddiv_rn((double)i, (double)A.height), 2.0));
    const double px = __dmul_rn(xs, A.tan_x), py = __dmul_rn(ys, A.tan_y);
    double d[3];
#pragma unroll
    for (int a = 0; a < 3; a++) d[a] = __dadd_rn(__dadd_rn(A.f[a], __dmul_rn(px, A.r[a])), __dmul_rn(py, A.u[a]));
    const double nrm =
        __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(d[0], d[0]), __dmul_rn(d[1], d[1])), __dmul_rn(d[2], d[2])));
#pragma unroll
    for (int a = 0; a < 3; a++) d[a] = __ddiv_rn(d[a], nrm);
    // _ray_box_span (render.py:340-354)
    double te = -INFINITY, tx = INFINITY;
#pragma unroll
    for (int a = 0; a < 3; a++) {
        const double inv = __drcp_rn(d[a]);
        const double ta = __dmul_rn(__dsub_rn(-1.0, A.origin[a]), inv);
        const double tb = __dmul_rn(__dsub_rn(1.0, A.origin[a]), inv);
        double lo = fmin(ta, tb), hi = fmax(ta, tb);
        if (isnan(lo)) lo = -INFINITY;
        if (isnan(hi)) hi = INFINITY;
        te = fmax(te, lo);
        tx = fmin(tx, hi);
    }
    te = fmax(te, A.near_);
    const bool active = inside && te < tx;
#pragma unroll
    for (int a = 0; a < 3; a++) R.d[a] = d[a];
    R.te = te;

    C.vdir = make_float4((float)d[0], (float)d[1], (float)d[2], 0.f);
    C.ns64 = C.nexact = C.ncell = C.nclear = 0;
    March M;
    M.k = 0;
    F.kend = 0;
    M.C0 = M.C1 = M.C2 = M.Aacc = 0.f;
    M.nshade = 0;
    M.h = 1469598103934665603ULL;
    M.own = -1;

    if (active) {
        // alive samples: t_k = te + (k + 0.5) sd < tx, a prefix of k (render.py:423)
        auto tk = [&](int64_t k) { return __dadd_rn(te, __dmul_rn((double)k + 0.5, A.sd)); };
        int64_t ke = (int64_t)fmax(ceil((tx - te) / A.sd - 0.5), 0.0);
        while (ke > 0 && !(tk(ke - 1) < tx)) --ke;
        while (tk(ke) < tx) ++ke;
        F.kend = (int32_t)min(ke, (int64_t)INT32_MAX);
        const bool k24 = ke < (1 << 24);  // the float32 sample offset dk needs k < 2^24
        int32_t seg_end = 0;              // next sample that needs the exact geometry (or kend)
        F.cur_own = -1;
        F.slot = -1;
        F.deg = 0;
        BlockFast &b = F.b;
        bool fast = false;
        bool is64 = false;  // F64: the owner is an ill-conditioned (float64) slot
        __shared__ float4 s_cellrows[SR > 0 ? SR : 1][128];
        FastCell<P, SR> G;
        G.s = &s_cellrows[0][threadIdx.x];
        G.key = -1;
        G.cx = G.cy = G.cz = -1e30f;
        G.inner = 0;
        G.lim = kLim1;
        float dk = 0.f;  // M.k - (sample at which tq0 was taken), exact below 2^24
        for (;;) {
            if (M.k >= seg_end) {  // rare: exact finest cell, owner change, end of ray
                if (M.k >= vld(F.kend)) break;
                double p[3];
                ++C.ncell;
                int32_t own, knext;
                exact_geometry(A, R, own_grid, M.k, vld(F.kend), p, own, knext);
                seg_end = knext;
                M.own = own;
                if (own < 0) break;  // render.py:430-436 (reported after the loop)
                if (own != vld(F.cur_own)) {
                    F.cur_own = own;
                    const int32_t slot = __ldg(idx2slot + own);
                    F.slot = slot;
                    const BlockDesc *dp = descs + slot;
                    b.ctrl4 = (const float4 *)__ldg((const unsigned long long *)&dp->ctrl4);
                    b.rng = (const float2 *)__ldg((const unsigned long long *)&dp->crange);
                    C.tab32 = (const float *)__ldg((const unsigned long long *)&dp->tab32);
                    b.ncp = __ldg(&dp->ncp);
                    b.nspan = __ldg(&dp->nspan);
                    b.plane = b.ncp * b.ncp;
                    b.nint = (uint32_t)max(b.nspan - 2 * P + 2, 0);
                    G.key = -1;
                    G.cx = G.cy = G.cz = -1e30f;
                    const int32_t deg = __ldg(&dp->deg);
                    F.deg = deg;
                    const uint32_t flags = __ldg(&dp->flags);
                    fast = deg == P && (flags & kFlagUniform) && (F64 || !(flags & AFAM_SLOT_FP64)) &&
                           (deg > 1 || b.nspan <= 128) && k24 && !(A.flags & kRenderForceExact);
                    if constexpr (F64) is64 = (flags & AFAM_SLOT_FP64) != 0;
                    // span-coordinate prediction from the exact entry position
#pragma unroll
                    for (int a = 0; a < 3; a++) {
                        const double sc = __ldg(&dp->inv_span[a]) * (double)b.nspan;
                        M.tq0[a] = (float)((p[a] - __ldg(&dp->lo[a])) * sc);
                        M.dtq[a] = (float)(A.sd * R.d[a] * sc);
                        if constexpr (F64) {
                            if (is64) {
                                s_pred64[threadIdx.x].tq0[a] = (p[a] - __ldg(&dp->lo[a])) * sc;
                                s_pred64[threadIdx.x].dtq[a] = A.sd * R.d[a] * sc;
                            }
                        }
                    }
                    if constexpr (F64)
                        if (is64) s_pred64[threadIdx.x].tab64 = (const double *)__ldg((const unsigned long long *)&dp->tab64);
                    C.ginv = make_float4(__ldg(&dp->inv_span_f[0]), __ldg(&dp->inv_span_f[1]),
                                         __ldg(&dp->inv_span_f[2]), 0.f);
                    dk = 0.f;
                }
            }
            if (DEBUG) M.h = (M.h ^ (uint64_t)(uint32_t)vld(F.cur_own)) * 1099511628211ULL;
            bool ok = false;
            if (AF || fast) {
                if (F64 && is64) {
                    ok = sample_fast64<P, SR, AF && F64_VF>(A, tf, b, s_pred64[threadIdx.x], dk, C, G, M);
                } else {
                    const float tqx = fmaf(dk, M.dtq[0], M.tq0[0]);
                    const float tqy = fmaf(dk, M.dtq[1], M.tq0[1]);
                    const float tqz = fmaf(dk, M.dtq[2], M.tq0[2]);
                    ok = sample_fast2<P, SR>(A, tf, b, tqx, tqy, tqz, C, G, M);
                }
            }
            if (DEBUG && (AF || fast) && ok && (G.inner & kCellClear)) ++C.nclear;
            if (!ok) {
                const int32_t slot = vld(F.slot), deg = vld(F.deg);
                const BlockDesc *dpx = descs + slot;
                int f64;
                if (deg == 3) f64 = sample_exact<3>(GA, &tf, &R, dpx, slot, M.k);
                else if (deg == 2) f64 = sample_exact<2>(GA, &tf, &R, dpx, slot, M.k);
                else if (!HI || deg == 1) f64 = sample_exact<1>(GA, &tf, &R, dpx, slot, M.k);
                else f64 = sample_exact_any(GA, &tf, &R, dpx, M.k);  // degrees above AFAM_FAST_DEGREE
                C.ns64 += f64;
                ++C.nexact;
                const float4 tfv = R.tfv;
                if (tfv.w > 0.f) {
                    ++M.nshade;
                    const float g[3] = {R.g[0], R.g[1], R.g[2]};
                    composite(A, C.vdir, tfv, g, M);
                }
            }
            // render.py:423 alive test before the next sample
            ++M.k;
            dk += 1.f;
            if (!(M.Aacc <= A.o_max_f)) break;
        }
    }
    const uint32_t ns = (uint32_t)M.k;
    M.kend = F.kend;
    inside = pixel(j, lr, i);
    const int lane = threadIdx.x & 31;
    if (inside) {
        // render.py:458-461 quantise (round half to even)
        uchar4 px4;
        px4.x = (unsigned char)min(max(__float2int_rn(M.C0 * 255.f), 0), 255);
        px4.y = (unsigned char)min(max(__float2int_rn(M.C1 * 255.f), 0), 255);
        px4.z = (unsigned char)min(max(__float2int_rn(M.C2 * 255.f), 0), 255);
        px4.w = (unsigned char)min(max(__float2int_rn(M.Aacc * 255.f), 0), 255);
        const int64_t local = (int64_t)lr * A.width + j;
        const int64_t dst = (A.flags & AFAM_RENDER_FULL_FRAME) ? (int64_t)i * A.width + j : local;
        reinterpret_cast<uchar4 *>(rgba)[dst] = px4;
        if (DEBUG) {
            nsamp[local] = (int32_t)ns;
            ohash[local] = M.h;
        }
    }
    const uint32_t wsum = __reduce_add_sync(0xffffffffu, ns);
    const uint32_t wsum64 = __reduce_add_sync(0xffffffffu, C.ns64);
    const uint32_t wshade = __reduce_add_sync(0xffffffffu, M.nshade);
    const uint32_t wexact = __reduce_add_sync(0xffffffffu, C.nexact);
    const uint32_t wcell = __reduce_add_sync(0xffffffffu, C.ncell);
    const uint32_t wclear = DEBUG ? __reduce_add_sync(0xffffffffu, C.nclear) : 0u;
    int64_t wmiss = M.own < 0 && M.k < M.kend ? ((int64_t)M.k << 32) | ((int64_t)i * A.width + j) : INT64_MAX;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const int64_t other = __shfl_xor_sync(0xffffffffu, wmiss, o);
        wmiss = other < wmiss ? other : wmiss;
    }
    if (lane == 0) {
        if (wsum) atomicAdd((unsigned long long *)&stats->samples, (unsigned long long)wsum);
        if (wsum64) atomicAdd((unsigned long long *)&stats->fp64_samples, (unsigned long long)wsum64);
        if (wshade) atomicAdd((unsigned long long *)&stats->shaded_samples, (unsigned long long)wshade);
        if (wexact) atomicAdd((unsigned long long *)&stats->exact_samples, (unsigned long long)wexact);
        if (wcell) atomicAdd((unsigned long long *)&stats->exact_cells, (unsigned long long)wcell);
        if (wclear) atomicAdd((unsigned long long *)&stats->clear_samples, (unsigned long long)wclear);
        if (wmiss != INT64_MAX) atomicMin((long long *)&stats->missing_key, (long long)wmiss);
    }
}

__global__ void init_stats_kernel(afam_render_stats *s) {
    s->samples = 0;
    s->fp64_samples = 0;
    s->missing_key = INT64_MAX;
    s->shaded_samples = 0;
    s->exact_samples = 0;
    s->exact_cells = 0;
    s->clear_samples = 0;
}

__global__ void finish_stats_kernel(afam_render_stats *s) {
    if (s->missing_key == INT64_MAX) s->missing_key = -1;
}

// np.interp(x, xs, ys) (numpy compiled_base.c) in float64 on the host, over
// n points of `stride` doubles (scalar first), value column `col`.
static double host_interp(double x, const double *pts, int n, int stride, int col) {
    auto X = [&](int k) { return pts[(size_t)k * stride]; };
    auto Y = [&](int k) { return pts[(size_t)k * stride + col]; };
    if (n == 1 || x <= X(0)) return Y(0);
    if (x >= X(n - 1)) return Y(n - 1);
    int j;  // the last k with X(k) <= x (binary search)
    {
        int lo = 0, hi = n - 1;  // X(lo) <= x < X(hi)
        while (hi - lo > 1) {
            const int mid = (lo + hi) / 2;
            if (X(mid) <= x) lo = mid;
            else hi = mid;
        }
        j = lo;
    }
    if (X(j) == x) return Y(j);
    const double slope = (Y(j + 1) - Y(j)) / (X(j + 1) - X(j));
    return slope * (x - X(j)) + Y(j);
}

// The TF's control points: the inline arrays, or the caller's when given.
static const double *tf_color_pts(const afam_frame *F) { return F->color_pts ? F->color_pts : &F->color[0][0]; }
static const double *tf_opacity_pts(const afam_frame *F) {
    return F->opacity_pts ? F->opacity_pts : &F->opacity[0][0];
}

// Host half of the TF table: the device table plus its breakpoint arrays.
struct TfHost {
    TfTable T;
    std::vector<float4> val, slope;
    std::vector<float> bp;
};

static void build_tf_table(const afam_frame *F, TfHost &H) {
    TfTable &T = H.T;
    const double *cp = tf_color_pts(F), *op = tf_opacity_pts(F);
    std::vector<double> xs, xc, xo;
    for (int k = 0; k < F->ncolor; k++) xc.push_back(cp[4 * k]);
    for (int k = 0; k < F->nopacity; k++) xo.push_back(op[2 * k]);
    xs = xc;
    xs.insert(xs.end(), xo.begin(), xo.end());
    std::sort(xs.begin(), xs.end());
    xs.erase(std::unique(xs.begin(), xs.end()), xs.end());
    T.nbp = (int)xs.size();
    auto eval = [&](double x, int c) {
        return c < 3 ? host_interp(x, cp, F->ncolor, 4, 1 + c) : host_interp(x, op, F->nopacity, 2, 1);
    };
    H.val.assign(T.nbp, make_float4(0.f, 0.f, 0.f, 0.f));
    H.slope.assign(T.nbp, make_float4(0.f, 0.f, 0.f, 0.f));
    H.bp.assign(T.nbp, 0.f);
    for (int j = 0; j < T.nbp; j++) {
        H.bp[j] = (float)xs[j];
        float v[4], s[4];
        for (int c = 0; c < 4; c++) {
            v[c] = (float)eval(xs[j], c);
            s[c] = j + 1 < T.nbp ? (float)((eval(xs[j + 1], c) - eval(xs[j], c)) / (xs[j + 1] - xs[j])) : 0.f;
        }
        H.val[j] = make_float4(v[0], v[1], v[2], v[3]);
        H.slope[j] = make_float4(s[0], s[1], s[2], s[3]);
    }
    // Opacity support: below the breakpoint preceding the first nonzero
    // opacity point (and above the one following the last) every breakpoint
    // value and slope of the opacity channel is 0, and so is every clean
    // bucket line there, so alpha_tf is exactly 0 for v <= op_lo and
    // v >= op_hi (float32, the kernel's comparisons); buckets straddling
    // them hold a breakpoint and take the exact segment search.
    {
        const int n = F->nopacity;
        int k1 = -1, k2 = -1;
        for (int k = 0; k < n; k++)
            if (op[2 * k + 1] != 0.0) {
                if (k1 < 0) k1 = k;
                k2 = k;
            }
        const float inf = std::numeric_limits<float>::infinity();
        if (k1 < 0) {  // fully transparent TF
            T.op_lo = inf;
            T.op_hi = -inf;
        } else {
            T.op_lo = k1 > 0 && (float)op[2 * k1] > (float)op[2 * (k1 - 1)] ? (float)op[2 * (k1 - 1)] : -inf;
            T.op_hi = k2 + 1 < n && (float)op[2 * (k2 + 1)] > (float)op[2 * k2] ? (float)op[2 * (k2 + 1)] : inf;
        }
    }
    const double lo = F->domain_lo, hi = F->domain_hi;
    const bool ok = hi > lo;
    T.lo = (float)lo;
    T.scale = ok ? (float)(kTfBuckets / (hi - lo)) : 0.f;
    const double w = ok ? (hi - lo) / kTfBuckets : 0.0, margin = 0.01 * w;
    const float qnan = std::numeric_limits<float>::quiet_NaN();
    // a bucket is "clean" for a channel group when none of that group's
    // control scalars lies within it (plus a margin for the float32 bucket
    // coordinate): np.interp is then one linear function across the bucket
    auto clean = [&](const std::vector<double> &pts, double x0, double x1) {
        for (double q : pts)
            if (q > x0 - margin && q < x1 + margin) return false;
        return ok;
    };
    for (int i = 0; i < kTfBuckets; i++) {
        const double x0 = lo + w * i, x1 = lo + w * (i + 1);
        int j = -1;
        while (j + 1 < T.nbp && xs[j + 1] <= x0) ++j;
        T.lut[i] = j;
        if (clean(xo, x0, x1)) {
            const double a0 = eval(x0, 3), a1 = eval(x1, 3);
            T.alpha[i] = make_float2((float)a0, (float)(a1 - a0));
        } else {
            T.alpha[i] = make_float2(0.f, qnan);
        }
        if (clean(xc, x0, x1)) {
            double c0[3], c1[3];
            for (int c = 0; c < 3; c++) {
                c0[c] = eval(x0, c);
                c1[c] = eval(x1, c);
            }
            T.c0[i] = make_float4((float)c0[0], (float)c0[1], (float)c0[2], 0.f);
            T.dc[i] = make_float4((float)(c1[0] - c0[0]), (float)(c1[1] - c0[1]), (float)(c1[2] - c0[2]), 0.f);
        } else {
            T.c0[i] = make_float4(0.f, 0.f, 0.f, qnan);
            T.dc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
}

// render.py:357-375 _BlockIndex over the given (sorted) slots.
static int build_owner_grid(afam_store *s, const int32_t *slots, int32_t nb, int32_t &cells,
                            std::vector<int16_t> &grid) {
    std::vector<int> bpa(nb);
    cells = 1;
    for (int b = 0; b < nb; b++) {
        AFAM_CHECK(slots[b] >= 0 && slots[b] < s->nslots && s->host[slots[b]].valid, AFAM_E_VALUE,
                   "slot %d is empty", slots[b]);
        const SlotHost &h = s->host[slots[b]];
        const double w = h.hi[0] - h.lo[0];
        bpa[b] = (int)std::nearbyint(2.0 / w);  // int(round(2/width)), half-to-even
        if (b == 0 || bpa[b] > cells) cells = bpa[b];
    }
    AFAM_CHECK(cells >= 1 && cells <= 1024, AFAM_E_VALUE, "finest-cell grid of %d^3 cells is unsupported", cells);
    grid.assign((size_t)cells * cells * cells, (int16_t)-1);
    for (int b = 0; b < nb; b++) {
        const SlotHost &h = s->host[slots[b]];
        const int width = cells / std::max(1, bpa[b]);
        int lo[3];
        for (int a = 0; a < 3; a++) lo[a] = (int)std::nearbyint((h.lo[a] - -1.0) / 2.0 * (double)cells);
        for (int x = std::max(0, lo[0]); x < std::min(cells, lo[0] + width); x++)
            for (int y = std::max(0, lo[1]); y < std::min(cells, lo[1] + width); y++)
                for (int z = std::max(0, lo[2]); z < std::min(cells, lo[2] + width); z++)
                    grid[((size_t)x * cells + y) * cells + z] = (int16_t)b;
    }
    return AFAM_OK;
}

constexpr int kSmemGridMaxCells = 24;  // 24^3 int16 = 27 KB

// CTAs per SM the register allocation is sized for (launch bounds), per
// fast-path degree: the cubic path keeps the cell's 64 control points in
// registers.  AFAM_RENDER_MINB=2|3|4 overrides it for the cubic kernel.
static int render_minb() {
    static int v = [] {
        const char *e = getenv("AFAM_RENDER_MINB");
        const int m = e ? atoi(e) : 0;
        return (m == 2 || m == 4) ? m : 3;
    }();
    return v;
}

// A/B override of the p = 2 fast path's CTAs per SM (AFAM_RENDER_MINB2=3|4|5)
static int render_minb2() {
    static int v = [] {
        const char *e = getenv("AFAM_RENDER_MINB2");
        const int m = e ? atoi(e) : 0;
        return (m == 3 || m == 5) ? m : 4;
    }();
    return v;
}

struct LaunchArgs {
    dim3 grid;
    size_t smem;
    cudaStream_t st;
    const BlockDesc *descs;
    const int16_t *owner;
    const int32_t *idx;
    const RenderArgs *gargs;
    const TfTable *gtf;
    uint8_t *rgba;
    afam_render_stats *stats;
    int32_t *nsamp;
    uint64_t *ohash;
};

template <bool DEBUG, bool SMEM, int FD, int MINB>
static void launch_render_v(const LaunchArgs &L, const RenderArgs &A) {
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(render_kernel<DEBUG, SMEM, FD, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             64 * 1024);
        configured = true;
    }
    render_kernel<DEBUG, SMEM, FD, MINB><<<L.grid, 128, L.smem, L.st>>>(L.descs, L.owner, L.idx, A, L.gargs, L.gtf,
                                                                        L.rgba, L.stats, L.nsamp, L.ohash);
}

template <bool DEBUG, bool SMEM, int P, int MINB, int SR = 0, bool HI = false, bool F64 = false, bool AF = false>
static void launch_render2_v(const LaunchArgs &L, const RenderArgs &A) {
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(render2_kernel<DEBUG, SMEM, P, MINB, SR, HI, F64, AF>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        configured = true;
    }
    render2_kernel<DEBUG, SMEM, P, MINB, SR, HI, F64, AF><<<L.grid, 128, L.smem, L.st>>>(L.descs, L.owner, L.idx, A, L.gargs,
                                                                             L.gtf, L.rgba, L.stats, L.nsamp,
                                                                             L.ohash);
}

// AFAM_RENDER_V1=1: the round-1 sample loop (render_kernel) for spline
// blocks, for A/B checks of render2_kernel.
static bool render_v1() {
    static const bool v = [] {
        const char *e = getenv("AFAM_RENDER_V1");
        return e && atoi(e) != 0;
    }();
    return v;
}

// CTAs per SM of render2_kernel's cubic instantiation (AFAM_RENDER2_MINB=3|4|5 A/B).
static int render2_minb() {
    static int v = [] {
        const char *e = getenv("AFAM_RENDER2_MINB");
        const int m = e ? atoi(e) : 0;
        return (m == 4 || m == 5 || m == 48 || m == 44) ? m : 3;
    }();
    return v;
}

// AFAM_RENDER_NO_F64=1: float64 slots on the exact path (A/B of the float64 fast path)
static bool render_no_f64() {
    static const bool v = [] {
        const char *e = getenv("AFAM_RENDER_NO_F64");
        return e && atoi(e) != 0;
    }();
    return v;
}

// CTAs per SM of the all-fast float64 instantiation (AFAM_RENDER_F64_MINB=2|3 A/B)
static int render_f64_minb() {
    static const int v = [] {
        const char *e = getenv("AFAM_RENDER_F64_MINB");
        return (e && atoi(e) == 2) ? 2 : 3;
    }();
    return v;
}

// fd: the degree the fast path is compiled for (blocks of other degrees take
// the exact path); debug and non-shared-grid launches use the default bounds.
template <bool DEBUG, bool SMEM>
static void launch_render(const LaunchArgs &L, const RenderArgs &A, int fd, bool hi, bool f64, bool allfast,
                          bool allfast64) {
    if (fd == 0) return launch_render_v<DEBUG, SMEM, 0, 4>(L, A);  // DS blocks
    if (allfast && SMEM && !render_v1() && render2_minb() == 4 && fd == 3)  // A/B: 4 CTAs/SM (128 registers)
        return launch_render2_v<DEBUG, SMEM, 3, 4, 0, false, false, true>(L, A);
    if (allfast && SMEM && !render_v1() && render2_minb() == 3) {
        if (fd == 3) return launch_render2_v<DEBUG, SMEM, 3, 3, 0, false, false, true>(L, A);
        if (fd == 2) return launch_render2_v<DEBUG, SMEM, 2, 4, 0, false, false, true>(L, A);
    }
    if (hi) {  // blocks of degrees above AFAM_FAST_DEGREE present
        if (fd == 1) return launch_render2_v<DEBUG, SMEM, 1, 4, 0, true>(L, A);
        if (fd == 2) return launch_render2_v<DEBUG, SMEM, 2, 4, 0, true>(L, A);
        return launch_render2_v<DEBUG, SMEM, 3, 3, 0, true>(L, A);
    }
    if (f64 && allfast64 && !render_no_f64() && SMEM) {  // ... every block on a fast path (float32 or float64)
        if (fd == 3) {
            if (render_f64_minb() == 2) return launch_render2_v<DEBUG, SMEM, 3, 2, 0, false, true, true>(L, A);
            return launch_render2_v<DEBUG, SMEM, 3, 3, 0, false, true, true>(L, A);
        }
    }
    if (f64 && !render_no_f64()) {  // ill-conditioned (float64) slots present: the float64 fast path
        if (fd == 2) return launch_render2_v<DEBUG, SMEM, 2, 3, 0, false, true>(L, A);
        if (fd == 3) return launch_render2_v<DEBUG, SMEM, 3, 2, 0, false, true>(L, A);
    }
    if (!render_v1()) {
        if (fd == 1) return launch_render2_v<DEBUG, SMEM, 1, 4>(L, A);
        if (fd == 2) return launch_render2_v<DEBUG, SMEM, 2, 4>(L, A);
        if (DEBUG || !SMEM) return launch_render2_v<DEBUG, SMEM, 3, 3>(L, A);
        switch (render2_minb()) {
            case 4: return launch_render2_v<DEBUG, SMEM, 3, 4>(L, A);
            case 5: return launch_render2_v<DEBUG, SMEM, 3, 5>(L, A);
            case 48: return launch_render2_v<DEBUG, SMEM, 3, 4, 8>(L, A);   // 8 rows in shared memory
            case 44: return launch_render2_v<DEBUG, SMEM, 3, 4, 4>(L, A);   // 4 rows in shared memory
            default: return launch_render2_v<DEBUG, SMEM, 3, 3>(L, A);
        }
    }
    if (fd == 1) return launch_render_v<DEBUG, SMEM, 1, 4>(L, A);
    if (fd == 2) {
        if (!DEBUG && SMEM && render_minb2() == 3) return launch_render_v<DEBUG, SMEM, 2, 3>(L, A);
        if (!DEBUG && SMEM && render_minb2() == 5) return launch_render_v<DEBUG, SMEM, 2, 5>(L, A);
        return launch_render_v<DEBUG, SMEM, 2, 4>(L, A);
    }
    if (DEBUG || !SMEM) return launch_render_v<DEBUG, SMEM, 3, 3>(L, A);
    switch (render_minb()) {
        case 2: launch_render_v<DEBUG, SMEM, 3, 2>(L, A); break;
        case 4: launch_render_v<DEBUG, SMEM, 3, 4>(L, A); break;
        default: launch_render_v<DEBUG, SMEM, 3, 3>(L, A); break;
    }
}

}  // namespace afam

using namespace afam;

extern "C" int32_t afam_frame_rows(int32_t height, int32_t band_rows, int32_t nparts, int32_t part) {
    if (band_rows < 1 || nparts < 1 || part < 0 || part >= nparts) return 0;
    const int32_t nbands = (height + band_rows - 1) / band_rows;
    int32_t rows = 0;
    for (int32_t b = part; b < nbands; b += nparts) rows += std::min(band_rows, height - b * band_rows);
    return rows;
}

extern "C" int afam_owner_grid(afam_store *s, const int32_t *slots, int32_t nblocks, int32_t *cells, int32_t *grid,
                               int32_t cap) {
    AFAM_CHECK(s && cells, AFAM_E_VALUE, "store/cells is NULL");
    std::vector<int16_t> g;
    int32_t c = 1;
    int rc;
    {
        std::lock_guard<std::mutex> lk(s->mu);
        rc = build_owner_grid(s, slots, nblocks, c, g);
    }
    if (rc) return rc;
    *cells = c;
    if (grid) {
        AFAM_CHECK((int64_t)c * c * c <= cap, AFAM_E_CAPACITY, "owner grid needs %d^3 entries", c);
        for (size_t k = 0; k < g.size(); k++) grid[k] = g[k];
    }
    return AFAM_OK;
}

extern "C" int afam_render(afam_store *s, const afam_frame *F, const int32_t *slots, int32_t nblocks,
                           uint8_t *rgba, afam_render_stats *stats, int32_t *nsamp, uint64_t *ohash, void *stream) {
    AFAM_CHECK(s && F && rgba && stats, AFAM_E_VALUE, "NULL argument to afam_render");
    AFAM_CHECK(F->width >= 1 && F->height >= 1, AFAM_E_VALUE, "frame dimensions must be positive");
    AFAM_CHECK(F->sample_distance > 0, AFAM_E_VALUE, "sample distance must be positive");
    AFAM_CHECK(F->o_max > 0 && F->o_max <= 1, AFAM_E_VALUE, "o_max must be in (0, 1]");
    AFAM_CHECK(F->ncolor >= 1 && F->nopacity >= 1, AFAM_E_VALUE, "transfer function needs control points");
    AFAM_CHECK((F->ncolor <= AFAM_MAX_TF_POINTS || F->color_pts) &&
                   (F->nopacity <= AFAM_MAX_TF_POINTS || F->opacity_pts),
               AFAM_E_VALUE, "more than %d inline transfer-function points (pass color_pts / opacity_pts)",
               AFAM_MAX_TF_POINTS);
    AFAM_CHECK(nblocks >= 0 && nblocks < 32768, AFAM_E_VALUE, "too many resident blocks (%d)", nblocks);
    const bool debug = F->flags & AFAM_RENDER_DEBUG;
    AFAM_CHECK(!debug || (nsamp && ohash), AFAM_E_VALUE, "debug buffers missing");
    const int band_rows = F->band_rows > 0 ? F->band_rows : F->height;
    const int nparts = F->nparts > 0 ? F->nparts : 1;
    AFAM_CHECK(F->part >= 0 && F->part < nparts, AFAM_E_VALUE, "part %d outside [0, %d)", F->part, nparts);
    cudaStream_t st = (cudaStream_t)stream;
    HostTimer ht;
    AFAM_CUDA(cudaSetDevice(s->device));
    ht.mark();

    RenderArgs A;
    memset(&A, 0, sizeof(A));
    for (int a = 0; a < 3; a++) {
        A.origin[a] = F->origin[a];
        A.f[a] = F->f[a];
        A.r[a] = F->r[a];
        A.u[a] = F->u[a];
    }
    A.tan_x = F->tan_x;
    A.tan_y = F->tan_y;
    A.sd = F->sample_distance;
    A.o_max = F->o_max;
    A.near_ = F->near_;
    A.width = F->width;
    A.height = F->height;
    A.band_rows = band_rows;
    A.nparts = nparts;
    A.part = F->part;
    A.rows = afam_frame_rows(F->height, band_rows, nparts, F->part);
    A.power = (float)F->power;
    A.power_one = F->power == 1.0;
    A.ambient = (float)F->ambient;
    A.diffuse = (float)F->diffuse;
    A.specular = (float)F->specular;
    A.shininess = (float)F->shininess;
    A.dom_lo = (float)F->domain_lo;
    A.dom_hi = (float)F->domain_hi;
    {
        float of = (float)F->o_max;
        if ((double)of > F->o_max) of = std::nextafter(of, -INFINITY);
        A.o_max_f = of;
    }
    A.flags = F->flags & (AFAM_RENDER_DEBUG | AFAM_RENDER_FULL_FRAME);
    A.tf_lo = 0.f;  // set from the TF table below
    A.tf_scale = 0.f;
    {
        static const bool force_exact = [] {
            const char *e = getenv("AFAM_RENDER_FORCE_EXACT");
            return e && atoi(e) != 0;
        }();
        if (force_exact) A.flags |= kRenderForceExact;
    }
    // the TF table depends only on the TF's control points and domain: a
    // per-thread copy is rebuilt only when they change (replay renders every
    // frame with the same TF)
    struct TfCache {
        bool valid = false;
        std::vector<double> key;
        TfHost table;
    };
    static thread_local TfCache tfc;
    std::vector<double> key;
    {
        const double *cp = tf_color_pts(F), *op = tf_opacity_pts(F);
        key.reserve(4 + 4 * (size_t)F->ncolor + 2 * (size_t)F->nopacity);
        key.push_back(F->ncolor);
        key.push_back(F->nopacity);
        key.insert(key.end(), cp, cp + 4 * (size_t)F->ncolor);
        key.insert(key.end(), op, op + 2 * (size_t)F->nopacity);
        key.push_back(F->domain_lo);
        key.push_back(F->domain_hi);
    }
    if (!tfc.valid || key.size() != tfc.key.size() ||
        memcmp(key.data(), tfc.key.data(), key.size() * sizeof(double)) != 0) {
        memset(&tfc.table.T, 0, sizeof(tfc.table.T));
        build_tf_table(F, tfc.table);
        tfc.key.swap(key);
        tfc.valid = true;
    }
    const TfHost &tfh = tfc.table;
    const TfTable &tf = tfh.T;
    A.tf_lo = tf.lo;
    A.tf_scale = tf.scale;
    A.op_lo = tf.op_lo;
    A.op_hi = tf.op_hi;
    {
        const float inf = std::numeric_limits<float>::infinity();
        // clamp(x) = min(max(x, dom_lo), dom_hi) is monotone: for dom_lo <= op_lo < dom_hi,
        // clamp(x) <= op_lo iff x <= op_lo; above that range always, below it never
        A.clr_lo = A.op_lo >= A.dom_hi ? inf : (A.op_lo < A.dom_lo ? -inf : A.op_lo);
        A.clr_hi = A.op_hi <= A.dom_lo ? -inf : (A.op_hi > A.dom_hi ? inf : A.op_hi);
    }
    ht.mark();

    std::vector<int16_t> grid;
    int32_t cells = 1;
    int fd = 3;  // fast-path degree: the most common degree among the blocks
    bool hi = false, any64 = false, allfast = true, allfast64 = true;
    {
        std::lock_guard<std::mutex> lk(s->mu);
        int rc = build_owner_grid(s, slots, nblocks, cells, grid);
        if (rc) return rc;
        for (int b = 0; b < nblocks; b++) {
            AFAM_CUDA(wait_slot(s, slots[b], st));
            // float64 slot (max|c| over the limit, afam_store.cu build_tables_kernel)? unknown
            // while its upload is in flight: then the float64-capable kernel
            const SlotHost &h = s->host[slots[b]];
            const bool f64slot = (h.pending && !h.maxabs_known) || s->h_maxabs[slots[b]] > (float)s->fp64_limit;
            if (!h.ds && f64slot) any64 = true;
            allfast = allfast && !h.ds && !f64slot && h.uniform;
            allfast64 = allfast64 && !h.ds && h.uniform;
        }
        int cnt[4] = {0, 0, 0, 0}, nds = 0;
        hi = false;
        for (int b = 0; b < nblocks; b++) {
            if (s->host[slots[b]].ds) {
                ++nds;
                continue;
            }
            const int dg = s->host[slots[b]].deg;
            if (dg >= 1 && dg <= AFAM_FAST_DEGREE) cnt[dg]++;
            else hi = true;  // higher degrees: render2_kernel<..., HI> (sample_exact_any)
        }
        AFAM_CHECK(nds == 0 || nds == nblocks, AFAM_E_VALUE,
                   "resident blocks mix spline models and DS blocks (%d of %d DS)", nds, nblocks);
        fd = nds ? 0 : (cnt[3] >= cnt[2] && cnt[3] >= cnt[1] ? 3 : (cnt[2] >= cnt[1] ? 2 : 1));
        // every block on the fast path of degree fd (render2_kernel<..., AF>)?
        for (int b = 0; b < nblocks && (allfast || allfast64); b++) {
            allfast = allfast && s->host[slots[b]].deg == fd;
            allfast64 = allfast64 && s->host[slots[b]].deg == fd;
        }
        // the float32 sample offset needs rays shorter than 2^24 samples: the
        // cube's diagonal (2 sqrt 3) over the sample distance
        allfast = allfast && !hi && fd >= 2 && F->sample_distance > 3.5 / 16777216.0 && !(A.flags & kRenderForceExact);
        allfast64 = allfast64 && !hi && fd >= 2 && F->sample_distance > 3.5 / 16777216.0 &&
                    !(A.flags & kRenderForceExact);
    }
    ht.mark();
    A.cells = cells;
    A.nb = nblocks;
    // one upload: [RenderArgs | TfTable | TF breakpoints (val, slope, bp) |
    // owner grid | slot of each owner index]
    auto al = [](size_t v) { return (v + 255) & ~(size_t)255; };
    const size_t gbytes = grid.size() * sizeof(int16_t);
    const size_t nbp = (size_t)std::max(tf.nbp, 1);
    const size_t off_tf = al(sizeof(RenderArgs)), off_bp = off_tf + al(sizeof(TfTable));
    const size_t off_grid = off_bp + al(nbp * (2 * sizeof(float4) + sizeof(float)));
    const size_t off_idx = off_grid + al(gbytes);
    const size_t total = off_idx + std::max<size_t>(1, (size_t)nblocks) * sizeof(int32_t);
    // staged in this thread's pinned buffer, so the H2D copy is asynchronous
    // (a pageable source would block until the stream drains); the thread's
    // previous frame's copy out of it is fenced by ev_pack
    ThreadCtx *tc = thread_ctx(s->device);
    AFAM_CHECK(tc, AFAM_E_CUDA, "per-thread render state unavailable");
    ht.mark();
    const int ring = (int)(tc->nrender % ThreadCtx::kRing);
    if (tc->pack_cap[ring] < total) {
        AFAM_CUDA(cudaEventSynchronize(tc->ev_pack[ring]));
        if (tc->pack[ring]) AFAM_CUDA(cudaFreeHost(tc->pack[ring]));
        tc->pack[ring] = nullptr;
        tc->pack_cap[ring] = 0;
        AFAM_CUDA(cudaHostAlloc((void **)&tc->pack[ring], total + (64 << 10), cudaHostAllocDefault));
        tc->pack_cap[ring] = total + (64 << 10);
    } else {
        AFAM_CUDA(cudaEventSynchronize(tc->ev_pack[ring]));
    }
    unsigned char *pack = tc->pack[ring];
    unsigned char *d_pack = nullptr;
    AFAM_CUDA(cudaMallocAsync(&d_pack, total, st));
    memset(pack, 0, total);
    memcpy(pack, &A, sizeof(A));
    {
        TfTable t = tf;
        t.val = (const float4 *)(d_pack + off_bp);
        t.slope = t.val + nbp;
        t.bp = (const float *)(t.slope + nbp);
        memcpy(pack + off_tf, &t, sizeof(t));
        const size_t n = tfh.bp.size();
        memcpy(pack + off_bp, tfh.val.data(), n * sizeof(float4));
        memcpy(pack + off_bp + nbp * sizeof(float4), tfh.slope.data(), n * sizeof(float4));
        memcpy(pack + off_bp + 2 * nbp * sizeof(float4), tfh.bp.data(), n * sizeof(float));
    }
    memcpy(pack + off_grid, grid.data(), gbytes);
    if (nblocks) memcpy(pack + off_idx, slots, (size_t)nblocks * sizeof(int32_t));
    AFAM_CUDA(cudaMemcpyAsync(d_pack, pack, total, cudaMemcpyHostToDevice, st));
    AFAM_CUDA(cudaEventRecord(tc->ev_pack[ring], st));
    ht.mark();
    AFAM_CUDA(cudaEventRecord(tc->k0[ring], st));
    init_stats_kernel<<<1, 1, 0, st>>>(stats);
    if (A.rows > 0) {
        LaunchArgs L;
        L.grid = dim3((A.width + kCtaW - 1) / kCtaW, (A.rows + 128 / kCtaW - 1) / (128 / kCtaW));
        const bool sg = cells <= kSmemGridMaxCells;
        L.smem = kSmemGridOff + (sg ? gbytes : 0);
        L.st = st;
        L.descs = s->d_desc;
        L.owner = (const int16_t *)(d_pack + off_grid);
        L.idx = (const int32_t *)(d_pack + off_idx);
        L.gargs = (const RenderArgs *)d_pack;
        L.gtf = (const TfTable *)(d_pack + off_tf);
        L.rgba = rgba;
        L.stats = stats;
        L.nsamp = nsamp;
        L.ohash = ohash;
        if (debug) {
            if (sg) launch_render<true, true>(L, A, fd, hi, any64, allfast, allfast64);
            else launch_render<true, false>(L, A, fd, hi, any64, allfast, allfast64);
        } else {
            if (sg) launch_render<false, true>(L, A, fd, hi, any64, allfast, allfast64);
            else launch_render<false, false>(L, A, fd, hi, any64, allfast, allfast64);
        }
    }
    finish_stats_kernel<<<1, 1, 0, st>>>(stats);
    AFAM_CUDA(cudaEventRecord(tc->k1[ring], st));
    AFAM_CUDA(cudaGetLastError());
    mark_readers(s, slots, nblocks, tc->k1[ring]);  // uploads into these slots now wait for this frame
    tc->nrender++;
    AFAM_CUDA(cudaFreeAsync(d_pack, st));
    ht.mark();
    ht.report("afam_render: setdevice, args+tf, grid+waits, pack lock, pack+upload, launches");
    return AFAM_OK;
}

extern "C" int afam_ipc_get_handle(const void *dev_ptr, uint8_t *handle) {
    AFAM_CHECK(dev_ptr && handle, AFAM_E_VALUE, "NULL argument to afam_ipc_get_handle");
    cudaIpcMemHandle_t h;
    AFAM_CUDA(cudaIpcGetMemHandle(&h, const_cast<void *>(dev_ptr)));
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    memcpy(handle, &h, sizeof(h));
    return AFAM_OK;
}

extern "C" int afam_ipc_open(const uint8_t *handle, int32_t device, void **dev_ptr) {
    AFAM_CHECK(handle && dev_ptr, AFAM_E_VALUE, "NULL argument to afam_ipc_open");
    AFAM_CUDA(cudaSetDevice(device));
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    AFAM_CUDA(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return AFAM_OK;
}

extern "C" int afam_device_alloc(int32_t device, uint64_t bytes, void **dev_ptr) {
    AFAM_CHECK(dev_ptr && bytes > 0, AFAM_E_VALUE, "bad argument to afam_device_alloc");
    AFAM_CUDA(cudaSetDevice(device));
    AFAM_CUDA(cudaMalloc(dev_ptr, bytes));
    return AFAM_OK;
}

extern "C" int afam_device_free(void *dev_ptr) {
    if (dev_ptr) AFAM_CUDA(cudaFree(dev_ptr));
    return AFAM_OK;
}

extern "C" int afam_copy_to_host(void *host, const void *dev_ptr, uint64_t bytes) {
    AFAM_CHECK(host && dev_ptr, AFAM_E_VALUE, "NULL argument to afam_copy_to_host");
    AFAM_CUDA(cudaMemcpy(host, dev_ptr, bytes, cudaMemcpyDeviceToHost));
    return AFAM_OK;
}

extern "C" int afam_ipc_close(void *dev_ptr) {
    AFAM_CHECK(dev_ptr, AFAM_E_VALUE, "NULL argument to afam_ipc_close");
    AFAM_CUDA(cudaIpcCloseMemHandle(dev_ptr));
    return AFAM_OK;
}

extern "C" int afam_render_elapsed(afam_store *s, float *ms) {
    AFAM_CHECK(s && ms, AFAM_E_VALUE, "NULL argument to afam_render_elapsed");
    AFAM_CUDA(cudaSetDevice(s->device));
    ThreadCtx *tc = thread_ctx(s->device);
    AFAM_CHECK(tc, AFAM_E_CUDA, "per-thread render state unavailable");
    AFAM_CHECK(tc->nrender > 0, AFAM_E_VALUE, "no afam_render call on this thread");
    return afam_render_elapsed_seq(s, tc->nrender - 1, ms);
}

extern "C" int afam_render_seq(afam_store *s, uint64_t *count) {
    AFAM_CHECK(s && count, AFAM_E_VALUE, "NULL argument to afam_render_seq");
    ThreadCtx *tc = thread_ctx(s->device);
    AFAM_CHECK(tc, AFAM_E_CUDA, "per-thread render state unavailable");
    *count = tc->nrender;
    return AFAM_OK;
}

extern "C" int afam_render_elapsed_seq(afam_store *s, uint64_t seq, float *ms) {
    AFAM_CHECK(s && ms, AFAM_E_VALUE, "NULL argument to afam_render_elapsed_seq");
    AFAM_CUDA(cudaSetDevice(s->device));
    ThreadCtx *tc = thread_ctx(s->device);
    AFAM_CHECK(tc, AFAM_E_CUDA, "per-thread render state unavailable");
    AFAM_CHECK(seq < tc->nrender && tc->nrender - seq <= (uint64_t)ThreadCtx::kRing, AFAM_E_VALUE,
               "afam_render call %llu of this thread is not among its last %d", (unsigned long long)seq,
               ThreadCtx::kRing);
    const int r = (int)(seq % ThreadCtx::kRing);
    AFAM_CUDA(cudaEventSynchronize(tc->k1[r]));
    AFAM_CUDA(cudaEventElapsedTime(ms, tc->k0[r], tc->k1[r]));
    return AFAM_OK;
}
