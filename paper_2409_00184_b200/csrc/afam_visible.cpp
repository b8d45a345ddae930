// Native visible-set selection (host C++), bit-exact with the reference.
//
// Replaces render.select_visible / lod_for_distance / _frustum_planes /
// _box_outside_plane (reference render.py:249-320), which take ~8.7 ms per
// frame in Python on the 4,680-block config-3 manifest.
// Bit-exactness rules: element-wise numpy arithmetic
// is un-fused (this file is built with -ffp-contract=off), 1-D `@` and
// np.linalg.norm go through BLAS ddot, which on the reference host is the
// FMA chain fma(x2,y2, fma(x1,y1, x0*y0)).  The result is sorted, so the
// traversal order of the reference's explicit stack does not matter.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <vector>

#include "afam_internal.h"

namespace {

inline double ddot3(const double *a, const double *b) { return std::fma(a[2], b[2], std::fma(a[1], b[1], a[0] * b[0])); }

struct Walker {
    const afam_manifest *m;
    const double *pos;
    std::vector<double> bands;  // upper band boundaries (render.py:249-253) or custom ranges
    std::vector<int32_t> *out;

    int lod_for_distance(double d) const {  // render.py:256-261, searchsorted side='right'
        return (int)(std::upper_bound(bands.begin(), bands.end(), d) - bands.begin()) + 1;
    }

    void walk(int lod, int i, int j, int k) {
        const int b = m->bpa[lod - 1];
        const double *e = m->extents[lod - 1].data() + 6 * (((size_t)i * b + j) * b + k);
        if (std::isnan(e[0])) return;  // block absent from the manifest
        double diff[3];
        for (int a = 0; a < 3; a++) diff[a] = (e[2 * a] + e[2 * a + 1]) / 2.0 - pos[a];  // extent.mean(axis=1)
        const double d = std::sqrt(ddot3(diff, diff));
        if (lod > 1 && lod_for_distance(d) < lod) {  // refine into the 8 children (partition.py:80-91)
            for (int a = 0; a < 2; a++)
                for (int c = 0; c < 2; c++)
                    for (int q = 0; q < 2; q++) walk(lod - 1, 2 * i + a, 2 * j + c, 2 * k + q);
            return;
        }
        out->push_back(lod);
        out->push_back(i);
        out->push_back(j);
        out->push_back(k);
    }
};

}  // namespace

extern "C" {

int afam_manifest_create(afam_manifest **out, int32_t levels, const int32_t *bpa, const double *const *extents) {
    AFAM_CHECK(out && bpa && extents, AFAM_E_VALUE, "NULL argument to afam_manifest_create");
    AFAM_CHECK(levels >= 1 && levels <= 16, AFAM_E_VALUE, "levels %d out of range", levels);
    afam_manifest *m = new afam_manifest();
    m->levels = levels;
    m->bpa.assign(bpa, bpa + levels);
    m->extents.resize(levels);
    for (int l = 0; l < levels; l++) {
        const size_t n = (size_t)bpa[l] * bpa[l] * bpa[l] * 6;
        m->extents[l].assign(extents[l], extents[l] + n);
    }
    *out = m;
    return AFAM_OK;
}

int afam_manifest_destroy(afam_manifest *m) {
    delete m;
    return AFAM_OK;
}

int afam_select_visible(const afam_manifest *m, const double pos[3], const double f[3], const double r[3],
                        const double u[3], double tan_y, double aspect, double near_, const double *ranges,
                        int32_t nranges, int32_t *out, int32_t cap, int32_t *count) {
    AFAM_CHECK(m && pos && f && r && u && count, AFAM_E_VALUE, "NULL argument to afam_select_visible");
    std::vector<int32_t> emitted;
    emitted.reserve(4096);
    Walker w{m, pos, {}, &emitted};
    if (ranges) {
        w.bands.assign(ranges, ranges + nranges);
    } else {
        for (int k = 1; k < m->levels; k++) w.bands.push_back(((double)k * 4.0) / 5.0);  // arange(1,L)*4.0/5.0
    }
    const int c = m->bpa[m->levels - 1];
    for (int i = 0; i < c; i++)
        for (int j = 0; j < c; j++)
            for (int k = 0; k < c; k++) w.walk(m->levels, i, j, k);

    // _frustum_planes (render.py:264-272): inside iff n.x >= offset
    const double tan_x = tan_y * aspect;
    double pn[5][3], po[5];
    for (int a = 0; a < 3; a++) {
        pn[0][a] = f[a];
        pn[1][a] = tan_x * f[a] + r[a];
        pn[2][a] = tan_x * f[a] - r[a];
        pn[3][a] = tan_y * f[a] + u[a];
        pn[4][a] = tan_y * f[a] - u[a];
    }
    po[0] = ddot3(f, pos) + near_;
    for (int p = 1; p < 5; p++) po[p] = ddot3(pn[p], pos);

    std::vector<std::array<int32_t, 4>> vis;
    const size_t ne = emitted.size() / 4;
    vis.reserve(ne);
    for (size_t e = 0; e < ne; e++) {
        const int32_t *a4 = &emitted[4 * e];
        const int b = m->bpa[a4[0] - 1];
        const double *ex = m->extents[a4[0] - 1].data() + 6 * (((size_t)a4[1] * b + a4[2]) * b + a4[3]);
        bool outside = false;
        for (int p = 0; p < 5 && !outside; p++) {  // _box_outside_plane (render.py:275-278)
            double reach[3];
            for (int a = 0; a < 3; a++) reach[a] = pn[p][a] >= 0.0 ? ex[2 * a + 1] : ex[2 * a];
            outside = ddot3(reach, pn[p]) < po[p];
        }
        if (!outside) vis.push_back({a4[0], a4[1], a4[2], a4[3]});
    }
    std::sort(vis.begin(), vis.end());  // sorted(BlockAddress): (lod, ijk) order
    *count = (int32_t)vis.size();
    AFAM_CHECK((int64_t)vis.size() <= cap, AFAM_E_CAPACITY, "visible set of %zu blocks exceeds the output capacity %d",
               vis.size(), cap);
    if (out)
        for (size_t e = 0; e < vis.size(); e++) memcpy(out + 4 * e, vis[e].data(), sizeof(int32_t) * 4);
    return AFAM_OK;
}

}  // extern "C"
