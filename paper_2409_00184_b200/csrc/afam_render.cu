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
#include <vector>

#include "afam_eval.cuh"

namespace afam {

constexpr int kTfMaxBp = 2 * AFAM_MAX_TF_POINTS;
constexpr int kTfLut = 256;

struct TfTable {
    float4 val[kTfMaxBp];    // (r, g, b, alpha) at breakpoint j
    float4 slope[kTfMaxBp];  // d/dv on [bp[j], bp[j+1]); 0 past the last breakpoint
    float bp[kTfMaxBp];      // sorted union of color and opacity control scalars
    int32_t nbp;
    float lut_lo, lut_scale; // bucket = (v - lut_lo) * lut_scale over the TF domain
    int8_t lut[kTfLut];      // last breakpoint <= bucket start (-1: none)
    uint8_t clean[kTfLut];   // 1: no breakpoint within (a margin of) the bucket, lut is the segment
};

struct RenderArgs {
    double origin[3], f[3], r[3], u[3];
    double tan_x, tan_y;
    double sd, o_max;
    double near_;
    int32_t width, height, band_rows, nparts, part, rows;
    int32_t cells, nb;
    float power, ambient, diffuse, specular, shininess;
    int32_t power_one;  // power == 1
    float dom_lo, dom_hi;
    TfTable tf;
    uint32_t flags;
};

// TransferFunction.color_at / opacity_at (render.py:117-124): every
// channel is np.interp over its own control points; on the sorted union of
// all control scalars each channel is linear, so one segment search serves
// r, g, b and alpha.  Values at the breakpoints are the float64 np.interp
// values rounded to float32.
__device__ __forceinline__ float4 tf_eval(const TfTable &T, float v) {
    int bi = (int)((v - T.lut_lo) * T.lut_scale);
    bi = min(max(bi, 0), kTfLut - 1);
    int j = T.lut[bi];
    if (!T.clean[bi]) {
        while (j + 1 < T.nbp && v >= T.bp[j + 1]) ++j;
        while (j >= 0 && v < T.bp[j]) --j;
    }
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
__device__ __forceinline__ void decode_f64(const BlockLite &b, const BlockDesc *__restrict__ dp, int32_t slot,
                                           GatherCache &G, const double (&pos)[3], float &v, float (&g)[3]) {
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
    double vv, gg[3];
    contract_quad<P, double>(G.c4, N[0], E[0], N[1], E[1], N[2], E[2], vv, gg);
    v = (float)vv;
#pragma unroll
    for (int a = 0; a < 3; a++) g[a] = (float)(gg[a] / span[a]);
}

template <bool DEBUG, bool SMEM_GRID, int MINB>
__global__ void __launch_bounds__(128, MINB) render_kernel(const BlockDesc *__restrict__ descs,
                                                        const int16_t *__restrict__ grid,
                                                        const int32_t *__restrict__ idx2slot, const RenderArgs A,
                                                        uint8_t *__restrict__ rgba, afam_render_stats *stats,
                                                        int32_t *__restrict__ nsamp, uint64_t *__restrict__ ohash) {
    extern __shared__ __align__(16) unsigned char smem[];
    TfTable &tf = *reinterpret_cast<TfTable *>(smem);
    int16_t *sgrid = reinterpret_cast<int16_t *>(smem + sizeof(TfTable));
    {
        const int *src = reinterpret_cast<const int *>(&A.tf);
        int *dst = reinterpret_cast<int *>(&tf);
        for (int i = threadIdx.x; i < (int)(sizeof(TfTable) / 4); i += blockDim.x) dst[i] = src[i];
    }
    if (SMEM_GRID)
        for (int i = threadIdx.x; i < A.cells * A.cells * A.cells; i += blockDim.x) sgrid[i] = grid[i];
    __syncthreads();
    const int16_t *own_grid = SMEM_GRID ? sgrid : grid;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int j = blockIdx.x * 16 + (warp & 1) * 8 + (lane & 7);
    const int lr = blockIdx.y * 8 + (warp >> 1) * 4 + (lane >> 3);
    const bool inside = j < A.width && lr < A.rows;
    const int i = inside ? frame_row(A, lr) : 0;
    const int64_t ray = (int64_t)i * A.width + j;  // full-frame ray id (render.py:407)

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

    const float vdir[3] = {(float)d[0], (float)d[1], (float)d[2]};
    const double cellsd = (double)A.cells;
    const float o_max = (float)A.o_max;
    const bool o_max_exact = (double)o_max == A.o_max;
    float C0 = 0.f, C1 = 0.f, C2 = 0.f, Aacc = 0.f;
    uint32_t ns = 0, ns64 = 0, nshade = 0;
    uint64_t h = 1469598103934665603ULL;
    int64_t miss = INT64_MAX;

    int32_t cur_own = -1, cur_slot = -1;
    BlockLite b;
    b.deg = 0;
    b.flags = 0;
    GatherCache G;
    G.slot = -1;

    // sample k's position and finest-cell owner (render.py:422-428, :377-380):
    // float64, reference op order, no contraction
    auto geometry = [&](int64_t k, double &t, double (&pos)[3], int &own) {
        t = __dadd_rn(te, __dmul_rn((double)k + 0.5, A.sd));
        int cidx = 0;
#pragma unroll
        for (int a = 0; a < 3; a++) {
            double p = __dadd_rn(A.origin[a], __dmul_rn(t, d[a]));
            p = p < -1.0 ? -1.0 : (p > 1.0 ? 1.0 : p);  // np.clip (p is never NaN here)
            pos[a] = p;
            const double sc = __dmul_rn(__dmul_rn(__dadd_rn(p, 1.0), 0.5), cellsd);
            int ci = __double2int_rz(sc);
            ci = min(max(ci, 0), A.cells - 1);
            cidx = cidx * A.cells + ci;
        }
        own = own_grid[cidx];
    };

    if (active) {
        for (int64_t k = 0;; k++) {
            double t, pos[3];
            int own;
            geometry(k, t, pos, own);
            // render.py:423 alive test, before sample k
            if (!(t < tx && (o_max_exact ? Aacc <= o_max : (double)Aacc <= A.o_max))) break;
            if (own < 0) {  // render.py:430-436
                miss = ((int64_t)k << 32) | ray;
                break;
            }
            if (own != cur_own) {
                cur_own = own;
                cur_slot = __ldg(idx2slot + own);
                load_lite(descs + cur_slot, b);
            }
            float v, g[3];
            float4 tfv;
            if (b.flags & AFAM_SLOT_FP64) {
                ++ns64;
                if (b.deg == 3) decode_f64<3>(b, descs + cur_slot, cur_slot, G, pos, v, g);
                else if (b.deg == 2) decode_f64<2>(b, descs + cur_slot, cur_slot, G, pos, v, g);
                else decode_f64<1>(b, descs + cur_slot, cur_slot, G, pos, v, g);
                tfv = tf_eval(tf, fminf(fmaxf(v, A.dom_lo), A.dom_hi));
            } else {
                if (b.deg == 3) decode_f32<3>(b, descs + cur_slot, cur_slot, G, pos, tf, A.dom_lo, A.dom_hi, v, tfv, g);
                else if (b.deg == 2)
                    decode_f32<2>(b, descs + cur_slot, cur_slot, G, pos, tf, A.dom_lo, A.dom_hi, v, tfv, g);
                else decode_f32<1>(b, descs + cur_slot, cur_slot, G, pos, tf, A.dom_lo, A.dom_hi, v, tfv, g);
            }
            ++ns;
            if (DEBUG) h = (h ^ (uint64_t)(uint32_t)own) * 1099511628211ULL;
            const float atf = tfv.w;
            if (!(atf > 0.f)) continue;  // a_s = 0: the sample changes neither C nor A
            ++nshade;
            const float col[3] = {tfv.x, tfv.y, tfv.z};
            // render.py:451 opacity correction
            const float as = A.power_one ? 1.f - (1.f - atf) : 1.f - __powf(1.f - atf, A.power);
            // _shade (render.py:383-395)
            const float gn2 = fmaf(g[2], g[2], fmaf(g[1], g[1], g[0] * g[0]));
            float ndotl = 0.f;
            if (gn2 > 1e-24f) {
                const float ig = rsqrtf(gn2);
                ndotl = fabsf(g[0] * vdir[0] + g[1] * vdir[1] + g[2] * vdir[2]) * ig;
            }
            const float dif = A.diffuse * ndotl;
            // ndotl**shininess via exp2(shininess * log2(ndotl)) (MUFU.LG2 + MUFU.EX2)
            const float spec = A.specular * (ndotl > 0.f ? exp2f(A.shininess * __log2f(ndotl))
                                                         : (A.shininess == 0.f ? 1.f : 0.f));
            const float lit = A.ambient + dif;
            // render.py:453-455 front-to-back composite
            const float w = (1.f - Aacc) * as;
            C0 = fmaf(w, __saturatef(fmaf(col[0], lit, spec)), C0);
            C1 = fmaf(w, __saturatef(fmaf(col[1], lit, spec)), C1);
            C2 = fmaf(w, __saturatef(fmaf(col[2], lit, spec)), C2);
            Aacc += w;
        }
    }
    if (inside) {
        // render.py:458-461 quantise (round half to even)
        uchar4 px4;
        px4.x = (unsigned char)min(max(__float2int_rn(C0 * 255.f), 0), 255);
        px4.y = (unsigned char)min(max(__float2int_rn(C1 * 255.f), 0), 255);
        px4.z = (unsigned char)min(max(__float2int_rn(C2 * 255.f), 0), 255);
        px4.w = (unsigned char)min(max(__float2int_rn(Aacc * 255.f), 0), 255);
        const int64_t local = (int64_t)lr * A.width + j;
        reinterpret_cast<uchar4 *>(rgba)[local] = px4;
        if (DEBUG) {
            nsamp[local] = (int32_t)ns;
            ohash[local] = h;
        }
    }
    // per-warp reductions of the counters
    const uint32_t wsum = __reduce_add_sync(0xffffffffu, ns);
    const uint32_t wsum64 = __reduce_add_sync(0xffffffffu, ns64);
    const uint32_t wshade = __reduce_add_sync(0xffffffffu, nshade);
    int64_t wmiss = miss;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const int64_t other = __shfl_xor_sync(0xffffffffu, wmiss, o);
        wmiss = other < wmiss ? other : wmiss;
    }
    if (lane == 0) {
        if (wsum) atomicAdd((unsigned long long *)&stats->samples, (unsigned long long)wsum);
        if (wsum64) atomicAdd((unsigned long long *)&stats->fp64_samples, (unsigned long long)wsum64);
        if (wshade) atomicAdd((unsigned long long *)&stats->shaded_samples, (unsigned long long)wshade);
        if (wmiss != INT64_MAX) atomicMin((long long *)&stats->missing_key, (long long)wmiss);
    }
}

__global__ void init_stats_kernel(afam_render_stats *s) {
    s->samples = 0;
    s->fp64_samples = 0;
    s->missing_key = INT64_MAX;
    s->shaded_samples = 0;
}

__global__ void finish_stats_kernel(afam_render_stats *s) {
    if (s->missing_key == INT64_MAX) s->missing_key = -1;
}

// np.interp(x, xs, ys) (numpy compiled_base.c) in float64 on the host.
static double host_interp(double x, const double (*pts)[4], const double (*opts)[2], int n, int col, bool color) {
    auto X = [&](int k) { return color ? pts[k][0] : opts[k][0]; };
    auto Y = [&](int k) { return color ? pts[k][col] : opts[k][1]; };
    if (n == 1 || x <= X(0)) return Y(0);
    if (x >= X(n - 1)) return Y(n - 1);
    int j = 0;
    while (j + 1 < n && X(j + 1) <= x) ++j;
    if (X(j) == x) return Y(j);
    const double slope = (Y(j + 1) - Y(j)) / (X(j + 1) - X(j));
    return slope * (x - X(j)) + Y(j);
}

static void build_tf_table(const afam_frame *F, TfTable &T) {
    std::vector<double> xs;
    for (int k = 0; k < F->ncolor; k++) xs.push_back(F->color[k][0]);
    for (int k = 0; k < F->nopacity; k++) xs.push_back(F->opacity[k][0]);
    std::sort(xs.begin(), xs.end());
    xs.erase(std::unique(xs.begin(), xs.end()), xs.end());
    T.nbp = (int)xs.size();
    auto eval = [&](double x, int c) {
        return c < 3 ? host_interp(x, F->color, F->opacity, F->ncolor, 1 + c, true)
                     : host_interp(x, F->color, F->opacity, F->nopacity, 1, false);
    };
    for (int j = 0; j < T.nbp; j++) {
        T.bp[j] = (float)xs[j];
        float v[4], s[4];
        for (int c = 0; c < 4; c++) {
            v[c] = (float)eval(xs[j], c);
            s[c] = j + 1 < T.nbp ? (float)((eval(xs[j + 1], c) - eval(xs[j], c)) / (xs[j + 1] - xs[j])) : 0.f;
        }
        T.val[j] = make_float4(v[0], v[1], v[2], v[3]);
        T.slope[j] = make_float4(s[0], s[1], s[2], s[3]);
    }
    const double lo = F->domain_lo, hi = F->domain_hi;
    T.lut_lo = (float)lo;
    T.lut_scale = (float)(kTfLut / (hi - lo));
    const double w = (hi - lo) / kTfLut, margin = 0.01 * w;
    for (int i = 0; i < kTfLut; i++) {
        const double x = lo + (hi - lo) * i / kTfLut;
        int j = -1;
        while (j + 1 < T.nbp && xs[j + 1] <= x) ++j;
        T.lut[i] = (int8_t)j;
        bool clean = true;  // no breakpoint near the bucket: the bucket index alone decides the segment
        for (int q = 0; q < T.nbp; q++)
            if (xs[q] > x - margin && xs[q] < x + w + margin) clean = false;
        T.clean[i] = clean;
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

// Resident CTAs per SM the kernel is compiled for (register budget
// 65536/(128*MINB)); AFAM_RENDER_MINB=2|3|4 selects the variant (default 4:
// 128 registers, 16 warps/SM, measured fastest on B200).
static int render_minb() {
    static int v = [] {
        const char *e = getenv("AFAM_RENDER_MINB");
        const int m = e ? atoi(e) : 0;
        return (m == 3 || m == 5 || m == 6) ? m : 4;
    }();
    return v;
}

template <bool DEBUG, bool SMEM, int MINB>
static void launch_render_v(dim3 g, size_t smem, cudaStream_t st, const BlockDesc *descs, const int16_t *grid,
                            const int32_t *idx, const RenderArgs &A, uint8_t *rgba, afam_render_stats *stats,
                            int32_t *nsamp, uint64_t *ohash) {
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(render_kernel<DEBUG, SMEM, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        configured = true;
    }
    render_kernel<DEBUG, SMEM, MINB><<<g, 128, smem, st>>>(descs, grid, idx, A, rgba, stats, nsamp, ohash);
}

template <bool DEBUG, bool SMEM>
static void launch_render(dim3 g, size_t smem, cudaStream_t st, const BlockDesc *descs, const int16_t *grid,
                          const int32_t *idx, const RenderArgs &A, uint8_t *rgba, afam_render_stats *stats,
                          int32_t *nsamp, uint64_t *ohash) {
    if (render_minb() == 5)
        launch_render_v<DEBUG, SMEM, 5>(g, smem, st, descs, grid, idx, A, rgba, stats, nsamp, ohash);
    else if (render_minb() == 6)
        launch_render_v<DEBUG, SMEM, 6>(g, smem, st, descs, grid, idx, A, rgba, stats, nsamp, ohash);
    else if (render_minb() == 4)
        launch_render_v<DEBUG, SMEM, 4>(g, smem, st, descs, grid, idx, A, rgba, stats, nsamp, ohash);
    else
        launch_render_v<DEBUG, SMEM, 3>(g, smem, st, descs, grid, idx, A, rgba, stats, nsamp, ohash);
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
    AFAM_CHECK(F->ncolor >= 1 && F->ncolor <= AFAM_MAX_TF_POINTS && F->nopacity >= 1 &&
                   F->nopacity <= AFAM_MAX_TF_POINTS,
               AFAM_E_VALUE, "transfer function needs 1..%d control points", AFAM_MAX_TF_POINTS);
    AFAM_CHECK(nblocks >= 0 && nblocks < 32768, AFAM_E_VALUE, "too many resident blocks (%d)", nblocks);
    const bool debug = F->flags & AFAM_RENDER_DEBUG;
    AFAM_CHECK(!debug || (nsamp && ohash), AFAM_E_VALUE, "debug buffers missing");
    const int band_rows = F->band_rows > 0 ? F->band_rows : F->height;
    const int nparts = F->nparts > 0 ? F->nparts : 1;
    AFAM_CHECK(F->part >= 0 && F->part < nparts, AFAM_E_VALUE, "part %d outside [0, %d)", F->part, nparts);
    cudaStream_t st = (cudaStream_t)stream;
    AFAM_CUDA(cudaSetDevice(s->device));

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
    build_tf_table(F, A.tf);
    A.flags = F->flags;

    std::vector<int16_t> grid;
    int32_t cells = 1;
    {
        std::lock_guard<std::mutex> lk(s->mu);
        int rc = build_owner_grid(s, slots, nblocks, cells, grid);
        if (rc) return rc;
        for (int b = 0; b < nblocks; b++) AFAM_CUDA(wait_slot(s, slots[b], st));
    }
    A.cells = cells;
    A.nb = nblocks;
    int16_t *d_grid = nullptr;
    int32_t *d_idx = nullptr;
    const size_t gbytes = grid.size() * sizeof(int16_t);
    const size_t ibytes = std::max<size_t>(1, (size_t)nblocks) * sizeof(int32_t);
    AFAM_CUDA(cudaMallocAsync(&d_grid, gbytes, st));
    AFAM_CUDA(cudaMallocAsync(&d_idx, ibytes, st));
    AFAM_CUDA(cudaMemcpyAsync(d_grid, grid.data(), gbytes, cudaMemcpyHostToDevice, st));
    if (nblocks) AFAM_CUDA(cudaMemcpyAsync(d_idx, slots, (size_t)nblocks * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    AFAM_CUDA(cudaEventRecord(s->ev_k0, st));
    init_stats_kernel<<<1, 1, 0, st>>>(stats);
    if (A.rows > 0) {
        dim3 g((A.width + 15) / 16, (A.rows + 7) / 8);
        const bool sg = cells <= kSmemGridMaxCells;
        const size_t smem = sizeof(TfTable) + (sg ? gbytes : 0);
        if (debug) {
            if (sg) launch_render<true, true>(g, smem, st, s->d_desc, d_grid, d_idx, A, rgba, stats, nsamp, ohash);
            else launch_render<true, false>(g, smem, st, s->d_desc, d_grid, d_idx, A, rgba, stats, nsamp, ohash);
        } else {
            if (sg) launch_render<false, true>(g, smem, st, s->d_desc, d_grid, d_idx, A, rgba, stats, nsamp, ohash);
            else launch_render<false, false>(g, smem, st, s->d_desc, d_grid, d_idx, A, rgba, stats, nsamp, ohash);
        }
    }
    finish_stats_kernel<<<1, 1, 0, st>>>(stats);
    AFAM_CUDA(cudaEventRecord(s->ev_k1, st));
    AFAM_CUDA(cudaGetLastError());
    AFAM_CUDA(cudaFreeAsync(d_grid, st));
    AFAM_CUDA(cudaFreeAsync(d_idx, st));
    return AFAM_OK;
}

extern "C" int afam_render_elapsed(afam_store *s, float *ms) {
    AFAM_CHECK(s && ms, AFAM_E_VALUE, "NULL argument to afam_render_elapsed");
    AFAM_CUDA(cudaSetDevice(s->device));
    AFAM_CUDA(cudaEventSynchronize(s->ev_k1));
    AFAM_CUDA(cudaEventElapsedTime(ms, s->ev_k0, s->ev_k1));
    return AFAM_OK;
}
