// Device-side B-spline evaluation shared by K1 (points) and K2 (ray march).
//
// Restates, in registers, reference bspline.py:41-95 (span search and the
// Cox-de Boor value/derivative recurrences) and bspline.py:175-229 (gather
// of the (p+1)^3 control points and the tensor-product contraction), using
// the per-span tables built by the store (afam_internal.h: tab_stride) so
// the hot path has no divisions.
#pragma once

#include "afam_internal.h"

namespace afam {

template <typename T>
__device__ __forceinline__ T clamp01(T v) {
    return v < T(0) ? T(0) : (v > T(1) ? T(1) : v);
}

// searchsorted(knots, u, 'right') - 1 clipped to [deg, ncp-1]
// (bspline.py:41-47): start from the uniform-knot guess and walk to the
// exact span using the stored knots, so any (non-uniform) knot vector works.
// The comparison is float64 against the float32 knots upcast, exactly as
// the reference compares its float64 parameters (bspline.py:193-195), so
// the span (and the one-sided derivative at a knot) matches bit-for-bit.
__device__ __forceinline__ int find_span(const float *__restrict__ kv, int ncp, int deg, int nspan, double u) {
    int s = deg + min(max((int)(u * (double)nspan), 0), nspan - 1);
    while (s > deg && u < (double)__ldg(kv + s)) --s;
    while (s < ncp - 1 && u >= (double)__ldg(kv + s + 1)) ++s;
    return s;
}

// Register copy of one table entry; only the first tab_stride(P) values are used.
template <typename T>
using Tab = T[kTabStrideMax];

template <int P>
__device__ __forceinline__ void load_entry(const float *__restrict__ p, Tab<float> &t) {
    const float4 *q = reinterpret_cast<const float4 *>(p);
#pragma unroll
    for (int i = 0; i < tab_stride(P) / 4; i++) {
        float4 v = __ldg(q + i);
        t[4 * i] = v.x; t[4 * i + 1] = v.y; t[4 * i + 2] = v.z; t[4 * i + 3] = v.w;
    }
}

template <int P>
__device__ __forceinline__ void load_entry(const double *__restrict__ p, Tab<double> &t) {
    const double2 *q = reinterpret_cast<const double2 *>(p);
#pragma unroll
    for (int i = 0; i < tab_stride(P) / 2; i++) {
        double2 v = __ldg(q + i);
        t[2 * i] = v.x; t[2 * i + 1] = v.y;
    }
}

// Cox-de Boor (bspline.py:50-70) and the degree-reduction derivative
// (bspline.py:73-95) from one table entry: window W = t[s-p+1 .. s+p],
// inv[j][r] = 1/(t[s+r+1] - t[s+1-j+r]).
//
// The derivative is returned in difference form: with L the degree p-1
// bases, sum_j c_j N'_j = sum_{k<p} E[k] (c_{k+1} - c_k) where
// E[k] = p * L[k] / (t[s+k+1] - t[s+k+1-p]) -- the same identity as the
// reference's N'_j, regrouped so a locally constant patch has an exactly
// zero gradient (the reference's float64 gradient there is ~1e-17, below
// its 1e-12 "lit" threshold in _shade, render.py:386; a float32
// sum_j c_j N'_j would leave ~1e-8 noise and light flat regions).
template <int P, typename T>
__device__ __forceinline__ void basis_eval(const Tab<T> &t, T u, T (&N)[P + 1], T (&E)[P]) {
    const T *W = t;
    const T *inv = t + 2 * P;
    T left[P + 1], right[P + 1], L[P];
    N[0] = T(1);
    int o = 0;
#pragma unroll
    for (int j = 1; j <= P; j++) {
        left[j] = u - W[P - j];
        right[j] = W[P - 1 + j] - u;
        T saved = T(0);
#pragma unroll
        for (int r = 0; r < j; r++) {
            T tmp = N[r] * inv[o + r];
            N[r] = saved + right[r + 1] * tmp;
            saved = left[j - r] * tmp;
        }
        N[j] = saved;
        o += j;
        if (j == P - 1) {
#pragma unroll
            for (int k = 0; k < P; k++) L[k] = N[k];
        }
    }
    if (P == 1) L[0] = T(1);
    const T *invP = inv + P * (P - 1) / 2;
#pragma unroll
    for (int k = 0; k < P; k++) E[k] = T(P) * L[k] * invP[k];
}

template <int P, typename T>
__device__ __forceinline__ void basis_vals_only(const Tab<T> &t, T u, T (&N)[P + 1]) {
    const T *W = t;
    const T *inv = t + 2 * P;
    T left[P + 1], right[P + 1];
    N[0] = T(1);
    int o = 0;
#pragma unroll
    for (int j = 1; j <= P; j++) {
        left[j] = u - W[P - j];
        right[j] = W[P - 1 + j] - u;
        T saved = T(0);
#pragma unroll
        for (int r = 0; r < j; r++) {
            T tmp = N[r] * inv[o + r];
            N[r] = saved + right[r + 1] * tmp;
            saved = left[j - r] * tmp;
        }
        N[j] = saved;
        o += j;
    }
}

// Separable contraction of the (P+1)^3 control points c[(cz*Q+by)*Q+ax]
// (bspline.py:214, :224-228): x first, then y, then z.  Value uses the
// N weights; each gradient component applies the difference weights E of
// basis_eval to forward differences along its own axis.
template <int P, typename T, typename CT>
__device__ __forceinline__ void contract_grad(const CT (&c)[64], const T (&Nx)[P + 1], const T (&Ex)[P],
                                              const T (&Ny)[P + 1], const T (&Ey)[P], const T (&Nz)[P + 1],
                                              const T (&Ez)[P], T &v, T g[3]) {
    constexpr int Q = P + 1;
    T ry[Q], rdxy[Q], rdy[Q];
#pragma unroll
    for (int cz = 0; cz < Q; cz++) {
        T rx[Q], rdx[Q];
#pragma unroll
        for (int by = 0; by < Q; by++) {
            T cv[Q];
#pragma unroll
            for (int ax = 0; ax < Q; ax++) cv[ax] = (T)c[(cz * Q + by) * Q + ax];
            T acc = T(0), dacc = T(0);
#pragma unroll
            for (int ax = 0; ax < Q; ax++) acc = fma(Nx[ax], cv[ax], acc);
#pragma unroll
            for (int k = 0; k < P; k++) dacc = fma(Ex[k], cv[k + 1] - cv[k], dacc);
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

template <int P, typename T, typename CT>
__device__ __forceinline__ T contract_val(const CT (&c)[64], const T (&Nx)[P + 1],
                                          const T (&Ny)[P + 1], const T (&Nz)[P + 1]) {
    constexpr int Q = P + 1;
    T vv = T(0);
#pragma unroll
    for (int cz = 0; cz < Q; cz++) {
        T ay = T(0);
#pragma unroll
        for (int by = 0; by < Q; by++) {
            T rx = T(0);
#pragma unroll
            for (int ax = 0; ax < Q; ax++) rx = fma(Nx[ax], (T)c[(cz * Q + by) * Q + ax], rx);
            ay = fma(Ny[by], rx, ay);
        }
        vv = fma(Nz[cz], ay, vv);
    }
    return vv;
}

// Gather the (P+1)^3 control points at corner (x0,y0,z0) (bspline.py:175-181).
template <int P>
__device__ __forceinline__ void gather(const float *__restrict__ ctrl, int ncp, int pitch, int x0, int y0, int z0,
                                       float (&c)[64]) {
    constexpr int Q = P + 1;
#pragma unroll
    for (int cz = 0; cz < Q; cz++)
#pragma unroll
        for (int by = 0; by < Q; by++) {
            const float *row = ctrl + ((size_t)(z0 + cz) * ncp + (y0 + by)) * pitch + x0;
#pragma unroll
            for (int ax = 0; ax < Q; ax++) c[(cz * Q + by) * Q + ax] = __ldg(row + ax);
        }
}

// Same gather from the x-quad layout (ctrl4[(iz*ncp+ix)*ncp+iy] =
// c[ix..ix+3][iy][iz]): one 16-byte load per (iy, iz) row.
template <int P>
__device__ __forceinline__ void gather_quad_rows(const float4 *__restrict__ ctrl4, int ncp, int x0, int y0, int z0,
                                                 float (&c)[64]) {
    constexpr int Q = P + 1;
    const float4 *base = ctrl4 + ((size_t)z0 * ncp + x0) * ncp + y0;
    const size_t plane = (size_t)ncp * ncp;
#pragma unroll
    for (int cz = 0; cz < Q; cz++)
#pragma unroll
        for (int by = 0; by < Q; by++) {
            const float4 r = __ldg(base + cz * plane + by);
            const float rr[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
            for (int ax = 0; ax < Q; ax++) c[(cz * Q + by) * Q + ax] = rr[ax];
        }
}

// One full evaluation (no caching): parameters u in [0,1]^3 -> value and
// parameter-space gradient (bspline.py:217-229).
// Uniform B-spline basis on an interior span, local coordinate x in [0,1):
// the Cox-de Boor values for equally spaced knots, and the difference-form
// derivative weights E[k] = nspan * L[k] (L: degree p-1 basis), cf. basis_eval.
template <int P>
__device__ __forceinline__ void uniform_basis(float x, float ns, float (&N)[P + 1], float (&E)[P]) {
    const float m = 1.f - x;
    if (P == 1) {
        N[0] = m;
        N[1] = x;
        E[0] = ns;
    } else if (P == 2) {
        const float x2 = x * x;
        N[0] = 0.5f * m * m;
        N[1] = fmaf(-1.f, x2, x) + 0.5f;
        N[2] = 0.5f * x2;
        E[0] = ns * m;
        E[1] = ns * x;
    } else {
        const float x2 = x * x, x3 = x2 * x, m2 = m * m;
        const float s6 = 1.f / 6.f;
        N[0] = s6 * m2 * m;
        N[1] = fmaf(0.5f, x3, fmaf(-1.f, x2, 2.f / 3.f));
        N[2] = fmaf(-0.5f, x3, fmaf(0.5f, x2, fmaf(0.5f, x, s6)));
        N[3] = s6 * x3;
        const float hn = 0.5f * ns;
        E[0] = hn * m2;
        E[1] = ns * (fmaf(-1.f, x2, x) + 0.5f);
        E[2] = hn * x2;
    }
}

// uniform_basis split into the values and the derivative weights, so the
// ray march evaluates E only for samples it shades.
template <int P>
__device__ __forceinline__ void uniform_N(float x, float (&N)[P + 1]) {
    const float m = 1.f - x;
    if (P == 1) {
        N[0] = m;
        N[1] = x;
    } else if (P == 2) {
        const float x2 = x * x;
        N[0] = 0.5f * m * m;
        N[1] = fmaf(-1.f, x2, x) + 0.5f;
        N[2] = 0.5f * x2;
    } else {
        const float x2 = x * x, x3 = x2 * x, m2 = m * m;
        const float s6 = 1.f / 6.f;
        N[0] = s6 * m2 * m;
        N[1] = fmaf(0.5f, x3, fmaf(-1.f, x2, 2.f / 3.f));
        N[2] = fmaf(-0.5f, x3, fmaf(0.5f, x2, fmaf(0.5f, x, s6)));
        N[3] = s6 * x3;
    }
}

template <int P>
__device__ __forceinline__ void uniform_E(float x, float ns, float (&E)[P]) {
    const float m = 1.f - x;
    if (P == 1) {
        E[0] = ns;
    } else if (P == 2) {
        E[0] = ns * m;
        E[1] = ns * x;
    } else {
        const float x2 = x * x, hn = 0.5f * ns;
        E[0] = hn * (m * m);
        E[1] = ns * (fmaf(-1.f, x2, x) + 0.5f);
        E[2] = hn * x2;
    }
}

// Span + basis (values and difference-form derivative weights) of one axis
// at parameter u64 (float64, already clipped).  float32 evaluation of a
// clamped-uniform model takes the closed form on interior spans away from
// knots (no knot or table loads); everything else searches the stored knots
// and uses the per-span table.
template <int P, typename T>
__device__ __forceinline__ int axis_eval(const BlockDesc &d, int a, double u64, T (&N)[P + 1], T (&E)[P]) {
    if constexpr (sizeof(T) == 4) {
        if ((d.flags & kFlagUniform) && d.nspan <= 128) {
            const float tq = (float)(u64 * (double)d.nspan);
            const int k = min((int)floorf(tq), d.nspan - 1);
            const float fr = tq - (float)k;
            const int s = P + k;
            if (fr >= 1e-4f && fr <= 1.f - 1e-4f && s >= 2 * P - 1 && s <= d.ncp - P) {
                uniform_basis<P>(fr, (float)d.nspan, N, E);
                return s;
            }
        }
    }
    const int s = find_span(d.knots + a * d.nk, d.ncp, P, d.nspan, u64);
    Tab<T> t;
    const size_t off = ((size_t)a * d.nspan + (s - P)) * tab_stride(P);
    if constexpr (sizeof(T) == 4) load_entry<P>(d.tab32 + off, t);
    else load_entry<P>(d.tab64 + off, t);
    basis_eval<P, T>(t, (T)u64, N, E);
    return s;
}

template <int P, typename T, bool GRAD>
__device__ __forceinline__ T eval_uncached(const BlockDesc &d, const double (&u64)[3], T g[3]) {
    T Nx[P + 1], Dx[P], Ny[P + 1], Dy[P], Nz[P + 1], Dz[P];
    const int sx = axis_eval<P, T>(d, 0, u64[0], Nx, Dx);
    const int sy = axis_eval<P, T>(d, 1, u64[1], Ny, Dy);
    const int sz = axis_eval<P, T>(d, 2, u64[2], Nz, Dz);
    float c[64];
    gather_quad_rows<P>(d.ctrl4, d.ncp, sx - P, sy - P, sz - P, c);
    if constexpr (GRAD) {
        T v;
        contract_grad<P, T, float>(c, Nx, Dx, Ny, Dy, Nz, Dz, v, g);
        return v;
    } else {
        return contract_val<P, T, float>(c, Nx, Ny, Nz);
    }
}

// ---------------------------------------------------------------------------
// Any degree (AFAM_FAST_DEGREE < p <= AFAM_MAX_DEGREE; also valid for p <= 3):
// float64 straight from the stored float32 knots upcast and the pitched
// control points, with the reference's divisions -- bspline.py:50-70
// (basis_values), :73-95 (basis_values_and_derivatives: the degree p-1
// bases on the same span, N'_j = p (L_{j-1}/(t_{i+p}-t_i) -
// L_j/(t_{i+p+1}-t_{i+1}))), :175-229 (gather + contraction).  No per-span
// tables: slots of these degrees carry none.
constexpr int kAnyQ = AFAM_MAX_DEGREE + 1;

static __device__ inline void cox_de_boor_any(const float *__restrict__ kv, int p, int s, double u, double *N) {
    double left[kAnyQ], right[kAnyQ];
    N[0] = 1.0;
    for (int j = 1; j <= p; j++) {
        left[j] = u - (double)__ldg(kv + s + 1 - j);
        right[j] = (double)__ldg(kv + s + j) - u;
        double saved = 0.0;
        for (int r = 0; r < j; r++) {
            const double tmp = N[r] / (right[r + 1] + left[j - r]);
            N[r] = saved + right[r + 1] * tmp;
            saved = left[j - r] * tmp;
        }
        N[j] = saved;
    }
}

// Span, p+1 basis values and (with D) their derivatives on one axis.
static __device__ inline int axis_any(const float *__restrict__ kv, int ncp, int p, double u, double *N, double *D) {
    const int s = find_span(kv, ncp, p, ncp - p, u);
    cox_de_boor_any(kv, p, s, u, N);
    if (D) {
        double L[kAnyQ];
        cox_de_boor_any(kv, p - 1, s, u, L);  // N_{s-p+1 .. s, p-1}
        for (int j = 0; j <= p; j++) {
            const int i = s - p + j;
            double term = 0.0;
            if (j > 0) term = L[j - 1] / ((double)__ldg(kv + i + p) - (double)__ldg(kv + i));
            if (j < p) term = term - L[j] / ((double)__ldg(kv + i + p + 1) - (double)__ldg(kv + i + 1));
            D[j] = (double)p * term;
        }
    }
    return s;
}

// Value (and parameter-space gradient when g != nullptr) at u in [0,1]^3.
static __device__ __noinline__ double eval_any(const BlockDesc &d, const double (&u)[3], double *g) {
    const int p = d.deg, Q = p + 1;
    double N[3][kAnyQ], D[3][kAnyQ];
    int s[3];
    for (int a = 0; a < 3; a++) s[a] = axis_any(d.knots + a * d.nk, d.ncp, p, u[a], N[a], g ? D[a] : nullptr);
    double v = 0.0, gx = 0.0, gy = 0.0, gz = 0.0;
    for (int cz = 0; cz < Q; cz++) {
        double ry = 0.0, rdx = 0.0, rdy = 0.0;
        for (int by = 0; by < Q; by++) {
            const float *row = d.ctrl + ((size_t)(s[2] - p + cz) * d.ncp + (s[1] - p + by)) * d.pitch + (s[0] - p);
            double rx = 0.0, dx = 0.0;
            for (int ax = 0; ax < Q; ax++) {
                const double c = (double)__ldg(row + ax);
                rx = fma(N[0][ax], c, rx);
                if (g) dx = fma(D[0][ax], c, dx);
            }
            ry = fma(N[1][by], rx, ry);
            if (g) {
                rdx = fma(N[1][by], dx, rdx);
                rdy = fma(D[1][by], rx, rdy);
            }
        }
        v = fma(N[2][cz], ry, v);
        if (g) {
            gx = fma(N[2][cz], rdx, gx);
            gy = fma(N[2][cz], rdy, gy);
            gz = fma(D[2][cz], ry, gz);
        }
    }
    if (g) {
        g[0] = gx;
        g[1] = gy;
        g[2] = gz;
    }
    return v;
}

__device__ __forceinline__ BlockDesc load_desc(const BlockDesc *__restrict__ p) {
    BlockDesc d;
    const int4 *src = reinterpret_cast<const int4 *>(p);
    int4 *dst = reinterpret_cast<int4 *>(&d);
#pragma unroll
    for (int i = 0; i < (int)(sizeof(BlockDesc) / 16); i++) dst[i] = __ldg(src + i);
    return d;
}

}  // namespace afam
