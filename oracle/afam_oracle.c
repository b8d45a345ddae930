/*
 * afam_oracle.c -- CPU float64 restatement of the reference decode-and-render
 * path (splinecast, arXiv 2409.00184).  TEST INFRASTRUCTURE ONLY.
 *
 * This file is the parity checker.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load it; the product
 * (paper_2409_00184_b200/) never links or calls it.
 *
 * Every function restates one reference function and cites it as
 * file:line into /root/reference/pkg/src/splinecast/.  Arithmetic is IEEE
 * float64, compiled with -ffp-contract=off so every '*' and '+' rounds
 * separately exactly like numpy's element-wise ufuncs.  Where the reference
 * goes through a 1-D BLAS ddot (np.linalg.norm of a vector, `a @ b` of
 * vectors) we use the FMA chain that OpenBLAS' ddot produces on this host
 * (SURVEY.md Appendix A); that is the only fused arithmetic in this file.
 *
 * Parity of this restatement is pinned by tests/test_oracle_golden.py
 * against fixtures produced by the unmodified reference
 * (tests/golden/gen_golden.py).
 *
 * Layouts: control points are x-fastest (flat index ix + n*(iy + n*iz)),
 * the .mfa file order (FORMAT.md:57-61).  Knot vectors are the full clamped
 * vectors, float32 values upcast to float64 (model.py:27-31, bspline.py:193).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define AFO_MAXQ 16 /* degree <= 15 */

/* OpenBLAS ddot(n=3) as an FMA chain (measured). */
static inline double ddot3(const double *a, const double *b) {
    return fma(a[2], b[2], fma(a[1], b[1], a[0] * b[0]));
}

/* bspline.py:41-47  searchsorted(knots, u, 'right') - 1, clipped to [d, ncp-1]. */
int afo_find_span(const double *kv, int nk, int ncp, int deg, double u) {
    /* number of knots <= u (side='right') */
    int lo = 0, hi = nk;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (kv[mid] <= u) lo = mid + 1; else hi = mid;
    }
    int s = lo - 1;
    if (s < deg) s = deg;
    if (s > ncp - 1) s = ncp - 1;
    return s;
}

/* bspline.py:50-70  Cox-de Boor left/right recurrence; N[j] = N_{span-deg+j,deg}(u). */
void afo_basis(const double *kv, int deg, int span, double u, double *N) {
    double left[AFO_MAXQ], right[AFO_MAXQ];
    for (int j = 0; j <= deg; j++) N[j] = 0.0;
    N[0] = 1.0;
    for (int j = 1; j <= deg; j++) {
        left[j] = u - kv[span + 1 - j];
        right[j] = kv[span + j] - u;
        double saved = 0.0;
        for (int r = 0; r < j; r++) {
            double tmp = N[r] / (right[r + 1] + left[j - r]);
            N[r] = saved + right[r + 1] * tmp;
            saved = left[j - r] * tmp;
        }
        N[j] = saved;
    }
}

/* bspline.py:73-95  values plus first derivatives by degree reduction. */
void afo_basis_ders(const double *kv, int deg, int span, double u, double *N, double *dN) {
    afo_basis(kv, deg, span, u, N);
    for (int j = 0; j <= deg; j++) dN[j] = 0.0;
    if (deg == 0) return;
    double low[AFO_MAXQ];
    afo_basis(kv, deg - 1, span, u, low);
    for (int j = 0; j <= deg; j++) {
        int i = span - deg + j;
        double term = 0.0;
        if (j > 0) term = low[j - 1] / (kv[i + deg] - kv[i]);
        if (j < deg) term = term - low[j] / (kv[i + deg + 1] - kv[i + 1]);
        dN[j] = (double)deg * term;
    }
}

static inline double clip01(double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }

/*
 * bspline.py:184-229 (evaluate_points / evaluate_points_with_gradient) for one
 * parameter triple u (already in [0,1] or clipped here, bspline.py:194).
 * Returns value; grad (parameter space) when non-NULL.
 */
static double eval_one(const float *C, int ncp, int deg, const double *kx, const double *ky,
                       const double *kz, int nk, const double *u, double *grad) {
    double N[3][AFO_MAXQ], D[3][AFO_MAXQ];
    int s[3];
    const double *kv[3] = {kx, ky, kz};
    for (int a = 0; a < 3; a++) {
        double ua = clip01(u[a]);
        s[a] = afo_find_span(kv[a], nk, ncp, deg, ua);
        if (grad) afo_basis_ders(kv[a], deg, s[a], ua, N[a], D[a]);
        else afo_basis(kv[a], deg, s[a], ua, N[a]);
    }
    const int q = deg + 1;
    const int x0 = s[0] - deg, y0 = s[1] - deg, z0 = s[2] - deg;
    double v = 0.0, gx = 0.0, gy = 0.0, gz = 0.0;
    /* bspline.py:175-181 gather + :214/:224-228 einsum contractions */
    for (int a = 0; a < q; a++)
        for (int b = 0; b < q; b++)
            for (int c = 0; c < q; c++) {
                double cp = (double)C[(size_t)(x0 + a) + (size_t)ncp * ((size_t)(y0 + b) + (size_t)ncp * (size_t)(z0 + c))];
                v += cp * N[0][a] * N[1][b] * N[2][c];
                if (grad) {
                    gx += cp * D[0][a] * N[1][b] * N[2][c];
                    gy += cp * N[0][a] * D[1][b] * N[2][c];
                    gz += cp * N[0][a] * N[1][b] * D[2][c];
                }
            }
    if (grad) { grad[0] = gx; grad[1] = gy; grad[2] = gz; }
    return v;
}

/*
 * bspline.py:206-229.  knots: (3, nk) float64 (nk = ncp+deg+1); NULL means the
 * default clamped uniform vector (bspline.py:188-190, :29-38).
 */
void afo_eval_points(const float *coeff, int ncp, int deg, const double *knots, int64_t n,
                     const double *u, double *val, double *grad) {
    int nk = ncp + deg + 1;
    double *own = NULL;
    if (!knots) {
        own = (double *)malloc(sizeof(double) * 3 * nk);
        for (int a = 0; a < 3; a++) {
            for (int i = 0; i <= deg; i++) own[a * nk + i] = 0.0;
            for (int i = 1; i < ncp - deg; i++) own[a * nk + deg + i] = (double)i / (double)(ncp - deg);
            for (int i = 0; i <= deg; i++) own[a * nk + ncp + i] = 1.0;
        }
        knots = own;
    }
    for (int64_t i = 0; i < n; i++) {
        double g[3];
        double v = eval_one(coeff, ncp, deg, knots, knots + nk, knots + 2 * nk, nk, u + 3 * i, grad ? g : NULL);
        if (val) val[i] = v;
        if (grad) { grad[3 * i] = g[0]; grad[3 * i + 1] = g[1]; grad[3 * i + 2] = g[2]; }
    }
    free(own);
}

/*
 * bspline.py:98-125 collocation matrix row for params = linspace(0,1,m) with
 * FRESH float64 clamped knots (bspline.py:118-120), then bspline.py:162-172
 * decode: contract axis 0 (x), then 1 (y), then 2 (z).  out is x-fastest
 * (m, m, m): out[i + m*(j + m*k)].
 */
void afo_decode_grid(const float *coeff, int ncp, int deg, int m, double *out) {
    int nk = ncp + deg + 1;
    double *kv = (double *)malloc(sizeof(double) * nk);
    for (int i = 0; i <= deg; i++) kv[i] = 0.0;
    for (int i = 1; i < ncp - deg; i++) kv[deg + i] = (double)i / (double)(ncp - deg);
    for (int i = 0; i <= deg; i++) kv[ncp + i] = 1.0;
    /* dense B (m x ncp) */
    double *B = (double *)calloc((size_t)m * ncp, sizeof(double));
    for (int i = 0; i < m; i++) {
        /* np.linspace(0, 1, m): step = 1/(m-1); value i*step, last exactly 1 */
        double p;
        if (m == 1) p = 0.0;
        else {
            double step = 1.0 / (double)(m - 1);
            p = (double)i * step;
            if (i == m - 1) p = 1.0;
        }
        int s = afo_find_span(kv, nk, ncp, deg, p);
        double N[AFO_MAXQ];
        afo_basis(kv, deg, s, p, N);
        for (int j = 0; j <= deg; j++) B[(size_t)i * ncp + (s - deg + j)] = N[j];
    }
    size_t n = (size_t)ncp;
    /* T1[i,b,c] = sum_a B[i,a] C[a,b,c]  (x-fastest storage of each stage) */
    double *T1 = (double *)calloc((size_t)m * n * n, sizeof(double));
    for (size_t c = 0; c < n; c++)
        for (size_t b = 0; b < n; b++)
            for (int i = 0; i < m; i++) {
                double acc = 0.0;
                for (size_t a = 0; a < n; a++)
                    acc += B[(size_t)i * n + a] * (double)coeff[a + n * (b + n * c)];
                T1[(size_t)i + (size_t)m * (b + n * c)] = acc;
            }
    double *T2 = (double *)calloc((size_t)m * m * n, sizeof(double));
    for (size_t c = 0; c < n; c++)
        for (int j = 0; j < m; j++)
            for (int i = 0; i < m; i++) {
                double acc = 0.0;
                for (size_t b = 0; b < n; b++)
                    acc += B[(size_t)j * n + b] * T1[(size_t)i + (size_t)m * (b + n * c)];
                T2[(size_t)i + (size_t)m * ((size_t)j + (size_t)m * c)] = acc;
            }
    for (int k = 0; k < m; k++)
        for (int j = 0; j < m; j++)
            for (int i = 0; i < m; i++) {
                double acc = 0.0;
                for (size_t c = 0; c < n; c++)
                    acc += B[(size_t)k * n + c] * T2[(size_t)i + (size_t)m * ((size_t)j + (size_t)m * c)];
                out[(size_t)i + (size_t)m * ((size_t)j + (size_t)m * (size_t)k)] = acc;
            }
    free(T2); free(T1); free(B); free(kv);
}

/* ------------------------------------------------------------------------ */
/* Visibility: render.py:249-320                                             */
/* ------------------------------------------------------------------------ */

/* render.py:249-261  lod = searchsorted(bands, d, 'right') + 1 */
int afo_lod_for_distance(double d, int levels, const double *ranges, int nranges) {
    int cnt = 0;
    if (ranges) {
        for (int i = 0; i < nranges; i++) if (ranges[i] <= d) cnt++;
    } else {
        for (int k = 1; k < levels; k++) {
            double band = ((double)k * 4.0) / 5.0; /* render.py:253 arange(1,L)*4.0/5.0 */
            if (band <= d) cnt++;
        }
    }
    return cnt + 1;
}

typedef struct {
    int levels;
    const int *bpa;        /* bpa[lod-1] blocks per axis */
    const double *const *extents; /* extents[lod-1]: bpa^3 * 6 doubles, (i*bpa+j)*bpa+k, [lo0,hi0,lo1,hi1,lo2,hi2] */
    const double *pos;
    const double *ranges;
    int nranges;
    int *out;              /* (lod, i, j, k) quadruples */
    int nout, cap;
} vis_ctx;

static void vis_walk(vis_ctx *v, int lod, int i, int j, int k) {
    int b = v->bpa[lod - 1];
    const double *e = v->extents[lod - 1] + 6 * (((size_t)i * b + j) * b + k);
    double diff[3];
    for (int a = 0; a < 3; a++) {
        double cen = (e[2 * a] + e[2 * a + 1]) / 2.0; /* extent.mean(axis=1), render.py:306 */
        diff[a] = cen - v->pos[a];
    }
    double d = sqrt(ddot3(diff, diff)); /* np.linalg.norm(1-D) -> ddot, render.py:307 */
    if (lod > 1 && afo_lod_for_distance(d, v->levels, v->ranges, v->nranges) < lod) {
        for (int a = 0; a < 2; a++)
            for (int bb = 0; bb < 2; bb++)
                for (int c = 0; c < 2; c++) vis_walk(v, lod - 1, 2 * i + a, 2 * j + bb, 2 * k + c);
        return;
    }
    if (v->nout < v->cap) {
        int *o = v->out + 4 * v->nout;
        o[0] = lod; o[1] = i; o[2] = j; o[3] = k;
    }
    v->nout++;
}

static int cmp_addr(const void *a, const void *b) {
    const int *x = (const int *)a, *y = (const int *)b;
    for (int i = 0; i < 4; i++) if (x[i] != y[i]) return x[i] < y[i] ? -1 : 1;
    return 0;
}

/*
 * render.py:281-320.  f, r, u: the PointOfView.basis() triad (render.py:68-73);
 * tan_y = math.tan(math.radians(fov)/2) computed by the caller (render.py:267).
 * Returns the number of visible blocks (sorted (lod,i,j,k) in out), or -1 if
 * cap is too small.
 */
int afo_select_visible(int levels, const int *bpa, const double *const *extents, const double *pos,
                       const double *f, const double *r, const double *u, double tan_y, double aspect,
                       double near_, const double *ranges, int nranges, int *out, int cap) {
    int total = 0;
    for (int l = 0; l < levels; l++) total += bpa[l] * bpa[l] * bpa[l];
    int *tmp = (int *)malloc(sizeof(int) * 4 * (size_t)total);
    vis_ctx v = {levels, bpa, extents, pos, ranges, nranges, tmp, 0, total};
    int c = bpa[levels - 1];
    for (int i = 0; i < c; i++)
        for (int j = 0; j < c; j++)
            for (int k = 0; k < c; k++) vis_walk(&v, levels, i, j, k);
    /* render.py:264-272 frustum planes */
    double tan_x = tan_y * aspect;
    double pn[5][3], po[5];
    for (int a = 0; a < 3; a++) pn[0][a] = f[a];
    po[0] = ddot3(f, pos) + near_;
    for (int a = 0; a < 3; a++) {
        pn[1][a] = tan_x * f[a] + r[a];
        pn[2][a] = tan_x * f[a] - r[a];
        pn[3][a] = tan_y * f[a] + u[a];
        pn[4][a] = tan_y * f[a] - u[a];
    }
    for (int p = 1; p < 5; p++) po[p] = ddot3(pn[p], pos);
    int nvis = 0;
    for (int e = 0; e < v.nout; e++) {
        int *ad = tmp + 4 * e;
        int b = bpa[ad[0] - 1];
        const double *ex = extents[ad[0] - 1] + 6 * (((size_t)ad[1] * b + ad[2]) * b + ad[3]);
        int outside = 0;
        for (int p = 0; p < 5 && !outside; p++) {
            double reach[3];
            for (int a = 0; a < 3; a++) reach[a] = pn[p][a] >= 0.0 ? ex[2 * a + 1] : ex[2 * a];
            if (ddot3(reach, pn[p]) < po[p]) outside = 1; /* render.py:275-278 */
        }
        if (!outside) {
            memmove(tmp + 4 * nvis, ad, 4 * sizeof(int));
            nvis++;
        }
    }
    qsort(tmp, nvis, 4 * sizeof(int), cmp_addr);
    int ret = nvis;
    if (nvis > cap) ret = -1;
    else memcpy(out, tmp, sizeof(int) * 4 * nvis);
    free(tmp);
    return ret;
}

/* ------------------------------------------------------------------------ */
/* Ray casting: render.py:323-466                                            */
/* ------------------------------------------------------------------------ */

typedef struct {
    const float *ctrl;     /* x-fastest ncp^3 */
    const double *knots;   /* (3, ncp+deg+1) float64 (upcast float32) */
    double lo[3], hi[3];   /* extent */
    int ncp, deg;
} afo_block;

typedef struct {
    /* camera (render.py:68-73, :329-331) */
    double origin[3], f[3], r[3], u[3];
    double tan_x, tan_y;
    int width, height;
    int row0, row1;        /* render rows [row0, row1) of the full frame */
    /* RenderParams (render.py:168-192) */
    double sd, power, o_max, near_;
    double ambient, diffuse, specular, shininess;
    /* TransferFunction (render.py:93-124) */
    const double *color_pts; int ncolor;   /* (ncolor, 4) */
    const double *opac_pts; int nopac;     /* (nopac, 2) */
    double dom_lo, dom_hi;
} afo_frame;

/* np.interp(x, xp, fp) for sorted xp (numpy compiled_base.c semantics). */
static double np_interp(double x, const double *pts, int n, int stride, int col) {
    double x0 = pts[0];
    if (n == 1) return pts[col];
    if (x < x0) return pts[col];
    double xl = pts[(size_t)(n - 1) * stride];
    if (x > xl) return pts[(size_t)(n - 1) * stride + col];
    if (x == xl) return pts[(size_t)(n - 1) * stride + col];
    /* j with xp[j] <= x < xp[j+1] */
    int lo = 0, hi = n - 1;
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (pts[(size_t)mid * stride] <= x) lo = mid; else hi = mid;
    }
    double xj = pts[(size_t)lo * stride], xj1 = pts[(size_t)(lo + 1) * stride];
    double yj = pts[(size_t)lo * stride + col], yj1 = pts[(size_t)(lo + 1) * stride + col];
    double slope = (yj1 - yj) / (xj1 - xj);
    double res = slope * (x - xj) + yj;
    if (isnan(res)) {
        res = slope * (x - xj1) + yj1;
        if (isnan(res) && yj == yj1) res = yj;
    }
    return res;
}

/* render.py:357-380 owner grid: cells = max round(2/width); fill [rint((lo+1)/2*cells), +cells/bpa). */
int afo_owner_grid(const afo_block *blocks, int nb, int *grid_out /* cells^3 or NULL */, int cap_cells) {
    int cells = 1;
    int *bpa = (int *)malloc(sizeof(int) * (nb > 0 ? nb : 1));
    for (int b = 0; b < nb; b++) {
        double w = blocks[b].hi[0] - blocks[b].lo[0];
        bpa[b] = (int)nearbyint(2.0 / w);
        if (b == 0 || bpa[b] > cells) cells = bpa[b];
    }
    if (nb == 0) cells = 1;
    if (grid_out && cells <= cap_cells) {
        size_t nc = (size_t)cells * cells * cells;
        for (size_t i = 0; i < nc; i++) grid_out[i] = -1;
        for (int b = 0; b < nb; b++) {
            int width = cells / bpa[b];
            int lo[3];
            for (int a = 0; a < 3; a++) lo[a] = (int)nearbyint((blocks[b].lo[a] + 1.0) / 2.0 * (double)cells);
            for (int i = lo[0]; i < lo[0] + width && i < cells; i++)
                for (int j = lo[1]; j < lo[1] + width && j < cells; j++)
                    for (int k = lo[2]; k < lo[2] + width && k < cells; k++)
                        grid_out[((size_t)i * cells + j) * cells + k] = b;
        }
    }
    free(bpa);
    return cells;
}

typedef struct {
    int64_t samples;       /* total decoded samples */
    int64_t missing_key;   /* (step << 32) | ray of the first missing sample, or -1 */
} afo_stats;

/*
 * render.py:398-466 restated per ray (the lock-step loop only batches
 * independent rays).  rgba: (row1-row0, width, 4) uint8.  Optional per-ray
 * debug outputs: nsamp[ray], ohash[ray] (FNV-1a over owner indices).
 * blocks must be in sorted address order (render.py:361).
 */
int afo_render(const afo_frame *F, const afo_block *blocks, int nb, uint8_t *rgba, int32_t *nsamp,
               uint64_t *ohash, afo_stats *stats, int nthreads) {
    int cells = afo_owner_grid(blocks, nb, NULL, 0);
    size_t nc = (size_t)cells * cells * cells;
    int *grid = (int *)malloc(sizeof(int) * nc);
    afo_owner_grid(blocks, nb, grid, cells);
    const int W = F->width, H = F->height;
    const int nrows = F->row1 - F->row0;
    const int64_t nrays = (int64_t)nrows * W;
    int64_t total = 0;
    int64_t miss = INT64_MAX;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : total) reduction(min : miss)
#endif
    for (int64_t ray = 0; ray < nrays; ray++) {
        int i = F->row0 + (int)(ray / W), j = (int)(ray % W);
        /* render.py:332-337 (exact op order, unfused) */
        double xs = ((double)j / (double)W) * 2.0 - 1.0;
        double ys = 1.0 - ((double)i / (double)H) * 2.0;
        double px = xs * F->tan_x, py = ys * F->tan_y;
        double d[3];
        for (int a = 0; a < 3; a++) d[a] = (F->f[a] + px * F->r[a]) + py * F->u[a];
        double nrm = sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
        for (int a = 0; a < 3; a++) d[a] = d[a] / nrm;
        /* render.py:340-354 slab test */
        double te = -INFINITY, tx = INFINITY;
        for (int a = 0; a < 3; a++) {
            double inv = 1.0 / d[a];
            double ta = (-1.0 - F->origin[a]) * inv;
            double tb = (1.0 - F->origin[a]) * inv;
            double tlo = fmin(ta, tb), thi = fmax(ta, tb);
            if (isnan(tlo)) tlo = -INFINITY;
            if (isnan(thi)) thi = INFINITY;
            if (tlo > te) te = tlo;
            if (thi < tx) tx = thi;
        }
        if (te < F->near_) te = F->near_;
        double C[3] = {0, 0, 0}, A = 0.0;
        int32_t ns = 0;
        uint64_t h = 1469598103934665603ULL;
        if (te < tx) {
            for (int64_t step = 0;; step++) {
                double t = te + ((double)step + 0.5) * F->sd;   /* render.py:422 */
                if (!(t < tx && A <= F->o_max)) break;           /* render.py:423 */
                double p[3];
                int cell[3];
                for (int a = 0; a < 3; a++) {
                    double v = F->origin[a] + t * d[a];          /* render.py:427 */
                    v = v < -1.0 ? -1.0 : (v > 1.0 ? 1.0 : v);   /* render.py:428 */
                    p[a] = v;
                    double sc = (v - (-1.0)) / (1.0 - (-1.0)) * (double)cells; /* render.py:378 */
                    int ci = (int)sc;                            /* astype(intp): trunc */
                    if (ci < 0) ci = 0;
                    if (ci > cells - 1) ci = cells - 1;
                    cell[a] = ci;
                }
                int own = grid[((size_t)cell[0] * cells + cell[1]) * cells + cell[2]];
                if (own < 0) {                                   /* render.py:430-436 */
                    int64_t key = (step << 32) | (int64_t)ray;
                    if (key < miss) miss = key;
                    break;
                }
                h = (h ^ (uint64_t)(uint32_t)own) * 1099511628211ULL;
                ns++;
                const afo_block *B = &blocks[own];
                /* model.py:64-68 params_for, then model.py:81-87 value / gradient */
                double uu[3], span[3];
                for (int a = 0; a < 3; a++) {
                    span[a] = B->hi[a] - B->lo[a];
                    uu[a] = clip01((p[a] - B->lo[a]) / span[a]);
                }
                int nk = B->ncp + B->deg + 1;
                double g[3];
                double val = eval_one(B->ctrl, B->ncp, B->deg, B->knots, B->knots + nk, B->knots + 2 * nk, nk, uu, g);
                for (int a = 0; a < 3; a++) g[a] = g[a] / span[a]; /* model.py:79 */
                /* render.py:117-124 TF */
                double v = val < F->dom_lo ? F->dom_lo : (val > F->dom_hi ? F->dom_hi : val);
                double atf = np_interp(v, F->opac_pts, F->nopac, 2, 1);
                double col[3];
                for (int c = 0; c < 3; c++) col[c] = np_interp(v, F->color_pts, F->ncolor, 4, 1 + c);
                double as = 1.0 - pow(1.0 - atf, F->power);      /* render.py:451 */
                /* render.py:383-395 shading */
                double gn = sqrt((g[0] * g[0] + g[1] * g[1]) + g[2] * g[2]);
                double ndotl = 0.0;
                if (gn > 1e-12) {
                    double s = (g[0] / gn) * (-d[0]) + (g[1] / gn) * (-d[1]) + (g[2] / gn) * (-d[2]);
                    ndotl = fabs(s);
                }
                double dif = F->diffuse * ndotl;
                double spec = F->specular * pow(ndotl, F->shininess);
                double rem = 1.0 - A;                            /* render.py:453-455 */
                double w = rem * as;
                for (int c = 0; c < 3; c++) {
                    double sh = col[c] * (F->ambient + dif) + spec;
                    sh = sh < 0.0 ? 0.0 : (sh > 1.0 ? 1.0 : sh);
                    C[c] += w * sh;
                }
                A += rem * as;
            }
        }
        total += ns;
        if (nsamp) nsamp[ray] = ns;
        if (ohash) ohash[ray] = h;
        /* render.py:458-461 quantise */
        double q[4] = {C[0], C[1], C[2], A};
        for (int c = 0; c < 4; c++) {
            double x = nearbyint(q[c] * 255.0);
            x = x < 0.0 ? 0.0 : (x > 255.0 ? 255.0 : x);
            rgba[(size_t)ray * 4 + c] = (uint8_t)x;
        }
    }
    free(grid);
    if (stats) {
        stats->samples = total;
        stats->missing_key = miss == INT64_MAX ? -1 : miss;
    }
    return miss == INT64_MAX ? 0 : 1;
}

int afo_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
