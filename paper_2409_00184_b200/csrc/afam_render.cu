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
// and no FMA contraction (__dadd_rn/__dmul_rn/...).  Decoding is float32
// (float64 for slots flagged AFAM_SLOT_FP64); TF, shading and compositing
// are float32 (parity gate: PSNR >= 60 dB).
//
// Schedule.  One thread per ray; a warp is an 8x4 pixel tile and a CTA a
// 16x8 tile, so a warp's samples almost always share the owner block
// (SURVEY.md sec. 7 coherence measurement).  Along a ray the (p+1)^3
// control points and the three per-axis span tables stay in registers and
// are re-gathered only when the ray crosses into a new knot span or block.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "afam_eval.cuh"

namespace afam {

struct RenderArgs {
    double origin[3], f[3], r[3], u[3];
    double tan_x, tan_y;
    double sd, o_max;
    double near_;
    int32_t width, height, band_rows, nparts, part, rows;
    int32_t cells, nb;
    float power, ambient, diffuse, specular, shininess;
    int32_t shin_int;   // shininess as a small non-negative integer, else -1
    int32_t power_one;  // power == 1
    int32_t ncolor, nopac;
    float dom_lo, dom_hi;
    float cx[AFAM_MAX_TF_POINTS], cv[3][AFAM_MAX_TF_POINTS], cs[3][AFAM_MAX_TF_POINTS];
    float ox[AFAM_MAX_TF_POINTS], ov[AFAM_MAX_TF_POINTS], os[AFAM_MAX_TF_POINTS];
    uint32_t flags;
};

// np.interp(v, xs, ys) (numpy compiled_base.c) for v already clipped to the
// TF domain; slopes precomputed on the host in float64.
__device__ __forceinline__ int tf_segment(const float *xs, int n, float v) {
    int j = 0;
    for (int k = 1; k < n - 1; k++) j = (v >= xs[k]) ? k : j;
    return j;
}

__device__ __forceinline__ float tf_lerp(const float *xs, const float *ys, const float *sl, int n, int j, float v) {
    if (n == 1 || v < xs[0]) return ys[0];
    if (v >= xs[n - 1]) return ys[n - 1];
    return fmaf(sl[j], v - xs[j], ys[j]);
}

__device__ __forceinline__ float powi(float x, int e) {
    float r = 1.f;
    while (e) {
        if (e & 1) r *= x;
        x *= x;
        e >>= 1;
    }
    return r;
}

// Global frame row of local row lr for (band_rows, nparts, part).
__device__ __forceinline__ int frame_row(const RenderArgs &A, int lr) {
    const int b = lr / A.band_rows;
    return (b * A.nparts + A.part) * A.band_rows + lr % A.band_rows;
}

// Per-thread decode state: cached block descriptor, span tables and the
// (P+1)^3 control points of the current spans.
struct MarchCache {
    int32_t slot;
    int32_t s[3];
    float c[64];
};

template <int P>
__device__ __forceinline__ void decode_f32(const BlockDesc &d, MarchCache &mc, Tab<float> (&te)[3],
                                           const double (&pos)[3], float &v, float (&g)[3], bool fresh) {
    float u[3];
    int s[3];
    bool span_changed = fresh;
#pragma unroll
    for (int a = 0; a < 3; a++) {
        // model.py:64-68 params_for: u = clip((p - lo)/span, 0, 1); span chosen in float64
        const double u64 = clamp01((pos[a] - d.lo[a]) * d.inv_span[a]);
        u[a] = (float)u64;
        s[a] = find_span(d.knots + a * d.nk, d.ncp, P, d.nspan, u64);
        if (fresh || s[a] != mc.s[a]) {
            load_entry<P>(d.tab32 + ((size_t)a * d.nspan + (s[a] - P)) * tab_stride(P), te[a]);
            mc.s[a] = s[a];
            span_changed = true;
        }
    }
    if (span_changed) gather<P>(d.ctrl, d.ncp, d.pitch, s[0] - P, s[1] - P, s[2] - P, mc.c);
    float Nx[P + 1], Dx[P], Ny[P + 1], Dy[P], Nz[P + 1], Dz[P];
    basis_eval<P, float>(te[0], u[0], Nx, Dx);
    basis_eval<P, float>(te[1], u[1], Ny, Dy);
    basis_eval<P, float>(te[2], u[2], Nz, Dz);
    float gg[3];
    contract_grad<P, float, float>(mc.c, Nx, Dx, Ny, Dy, Nz, Dz, v, gg);
    // model.py:79 gradient / span
#pragma unroll
    for (int a = 0; a < 3; a++) g[a] = gg[a] * (float)d.inv_span[a];
}

template <int P>
__device__ __forceinline__ void decode_f64(const BlockDesc &d, const double (&pos)[3], float &v, float (&g)[3]) {
    double u[3], gg[3];
#pragma unroll
    for (int a = 0; a < 3; a++) u[a] = clamp01(__ddiv_rn(__dsub_rn(pos[a], d.lo[a]), d.span[a]));
    double vv = eval_uncached<P, double, true>(d, u, gg);
    v = (float)vv;
#pragma unroll
    for (int a = 0; a < 3; a++) g[a] = (float)(gg[a] / d.span[a]);
}

__global__ void __launch_bounds__(128) render_kernel(const BlockDesc *__restrict__ descs,
                                                     const int16_t *__restrict__ grid,
                                                     const int32_t *__restrict__ idx2slot, const RenderArgs A,
                                                     uint8_t *__restrict__ rgba, afam_render_stats *stats,
                                                     int32_t *__restrict__ nsamp, uint64_t *__restrict__ ohash) {
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
    const double nrm = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(d[0], d[0]), __dmul_rn(d[1], d[1])), __dmul_rn(d[2], d[2])));
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
    float C0 = 0.f, C1 = 0.f, C2 = 0.f, Aacc = 0.f;
    uint32_t ns = 0, ns64 = 0;
    uint64_t h = 1469598103934665603ULL;
    int64_t miss = INT64_MAX;

    MarchCache mc;
    mc.slot = -1;
    BlockDesc desc;
    desc.deg = 0;
    desc.flags = 0;
    Tab<float> tabs[3];

    if (active) {
        for (int64_t k = 0;; k++) {
            // render.py:422-423
            const double t = __dadd_rn(te, __dmul_rn((double)k + 0.5, A.sd));
            if (!(t < tx && (double)Aacc <= A.o_max)) break;
            // render.py:427-428, :378-379
            double pos[3];
            int cidx = 0;
#pragma unroll
            for (int a = 0; a < 3; a++) {
                double p = __dadd_rn(A.origin[a], __dmul_rn(t, d[a]));
                p = fmin(fmax(p, -1.0), 1.0);
                pos[a] = p;
                const double sc = __dmul_rn(__dmul_rn(__dadd_rn(p, 1.0), 0.5), cellsd);
                int ci = __double2int_rz(sc);
                ci = min(max(ci, 0), A.cells - 1);
                cidx = cidx * A.cells + ci;
            }
            const int own = __ldg(grid + cidx);
            if (own < 0) {  // render.py:430-436
                miss = ((int64_t)k << 32) | ray;
                break;
            }
            const int32_t slot = __ldg(idx2slot + own);
            bool fresh = false;
            if (slot != mc.slot) {
                desc = load_desc(descs + slot);
                mc.slot = slot;
                fresh = true;
            }
            float v, g[3];
            if (desc.flags & AFAM_SLOT_FP64) {
                ++ns64;
                if (desc.deg == 3) decode_f64<3>(desc, pos, v, g);
                else if (desc.deg == 2) decode_f64<2>(desc, pos, v, g);
                else decode_f64<1>(desc, pos, v, g);
            } else {
                if (desc.deg == 3) decode_f32<3>(desc, mc, tabs, pos, v, g, fresh);
                else if (desc.deg == 2) decode_f32<2>(desc, mc, tabs, pos, v, g, fresh);
                else decode_f32<1>(desc, mc, tabs, pos, v, g, fresh);
            }
            ++ns;
            if (A.flags & AFAM_RENDER_DEBUG) h = (h ^ (uint64_t)(uint32_t)own) * 1099511628211ULL;

            // TransferFunction (render.py:117-124)
            const float vc = fminf(fmaxf(v, A.dom_lo), A.dom_hi);
            const int jo = tf_segment(A.ox, A.nopac, vc);
            const float atf = tf_lerp(A.ox, A.ov, A.os, A.nopac, jo, vc);
            const int jc = tf_segment(A.cx, A.ncolor, vc);
            float col[3];
#pragma unroll
            for (int c = 0; c < 3; c++) col[c] = tf_lerp(A.cx, A.cv[c], A.cs[c], A.ncolor, jc, vc);
            // render.py:451 opacity correction
            const float as = A.power_one ? 1.f - (1.f - atf) : 1.f - __powf(1.f - atf, A.power);
            // _shade (render.py:383-395)
            const float gn = sqrtf(fmaf(g[2], g[2], fmaf(g[1], g[1], g[0] * g[0])));
            float ndotl = 0.f;
            if (gn > 1e-12f) {
                const float ig = 1.f / gn;
                ndotl = fabsf(-(g[0] * ig * vdir[0] + g[1] * ig * vdir[1] + g[2] * ig * vdir[2]));
            }
            const float dif = A.diffuse * ndotl;
            const float spec = A.specular * (A.shin_int >= 0 ? powi(ndotl, A.shin_int)
                                                             : (ndotl > 0.f ? __powf(ndotl, A.shininess) : 0.f));
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
        if (A.flags & AFAM_RENDER_DEBUG) {
            nsamp[local] = (int32_t)ns;
            ohash[local] = h;
        }
    }
    // per-warp reductions of the counters
    uint32_t wsum = __reduce_add_sync(0xffffffffu, ns);
    uint32_t wsum64 = __reduce_add_sync(0xffffffffu, ns64);
    int64_t wmiss = miss;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        int64_t other = __shfl_xor_sync(0xffffffffu, wmiss, o);
        wmiss = other < wmiss ? other : wmiss;
    }
    if (lane == 0) {
        if (wsum) atomicAdd((unsigned long long *)&stats->samples, (unsigned long long)wsum);
        if (wsum64) atomicAdd((unsigned long long *)&stats->fp64_samples, (unsigned long long)wsum64);
        if (wmiss != INT64_MAX) atomicMin((long long *)&stats->missing_key, (long long)wmiss);
    }
}

__global__ void init_stats_kernel(afam_render_stats *s) {
    s->samples = 0;
    s->fp64_samples = 0;
    s->missing_key = INT64_MAX;
    s->pad = 0;
}

__global__ void finish_stats_kernel(afam_render_stats *s) {
    if (s->missing_key == INT64_MAX) s->missing_key = -1;
}

// render.py:357-375 _BlockIndex over the given (sorted) slots.
static int build_owner_grid(afam_store *s, const int32_t *slots, int32_t nb, int32_t &cells,
                            std::vector<int16_t> &grid) {
    std::vector<int> bpa(nb);
    cells = 1;
    for (int b = 0; b < nb; b++) {
        const SlotHost &h = s->host[slots[b]];
        AFAM_CHECK(slots[b] >= 0 && slots[b] < s->nslots && h.valid, AFAM_E_VALUE, "slot %d is empty", slots[b]);
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
    AFAM_CHECK(!(F->flags & AFAM_RENDER_DEBUG) || (nsamp && ohash), AFAM_E_VALUE, "debug buffers missing");
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
    A.shin_int = (F->shininess >= 0 && F->shininess <= 1024 && F->shininess == std::floor(F->shininess))
                     ? (int)F->shininess : -1;
    A.ncolor = F->ncolor;
    A.nopac = F->nopacity;
    A.dom_lo = (float)F->domain_lo;
    A.dom_hi = (float)F->domain_hi;
    for (int k = 0; k < F->ncolor; k++) {
        A.cx[k] = (float)F->color[k][0];
        for (int c = 0; c < 3; c++) {
            A.cv[c][k] = (float)F->color[k][1 + c];
            A.cs[c][k] = k + 1 < F->ncolor ? (float)((F->color[k + 1][1 + c] - F->color[k][1 + c]) /
                                                     (F->color[k + 1][0] - F->color[k][0]))
                                           : 0.f;
        }
    }
    for (int k = 0; k < F->nopacity; k++) {
        A.ox[k] = (float)F->opacity[k][0];
        A.ov[k] = (float)F->opacity[k][1];
        A.os[k] = k + 1 < F->nopacity
                      ? (float)((F->opacity[k + 1][1] - F->opacity[k][1]) / (F->opacity[k + 1][0] - F->opacity[k][0]))
                      : 0.f;
    }
    A.flags = F->flags;

    std::vector<int16_t> grid;
    int32_t cells = 1;
    {
        std::lock_guard<std::mutex> lk(s->mu);
        int rc = build_owner_grid(s, slots, nblocks, cells, grid);
        if (rc) return rc;
        for (int b = 0; b < nblocks; b++) AFAM_CUDA(cudaStreamWaitEvent(st, s->host[slots[b]].ready, 0));
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
    init_stats_kernel<<<1, 1, 0, st>>>(stats);
    if (A.rows > 0) {
        dim3 g((A.width + 15) / 16, (A.rows + 7) / 8);
        render_kernel<<<g, 128, 0, st>>>(s->d_desc, d_grid, d_idx, A, rgba, stats, nsamp, ohash);
    }
    finish_stats_kernel<<<1, 1, 0, st>>>(stats);
    AFAM_CUDA(cudaGetLastError());
    AFAM_CUDA(cudaFreeAsync(d_grid, st));
    AFAM_CUDA(cudaFreeAsync(d_idx, st));
    return AFAM_OK;
}
