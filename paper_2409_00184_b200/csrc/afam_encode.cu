// Encoder inner loop on the GPU: for a batch of (block, ncp) jobs, the
// endpoint-pinned separable least-squares fit of the block's samples
// (reference bspline.fit_tensor_product / _fit_axis, bspline.py:128-159,
// with the operator of _axis_operator, bspline.py:109-125), the float32
// rounding of the coefficients (model.fit, model.py:96-107), the dense
// decode onto the sample lattice (MicroModel.decode_grid -> bspline.py:162-172)
// and the reconstruction RMSE (encoder.error_rmse, encoder.py:74-78) --
// everything in float64 like the reference.
//
// Each separable contraction is one launch of contract_rotate_kernel over
// all jobs: the slowest axis of the job's [n0][R] input is contracted with a
// dense [nout][n0] operator and the result is written as [R][nout], so the
// contracted axis becomes the fastest.  Three launches contract the three
// axes and restore the axis order ([i][j][k] samples -> [a][b][c]
// coefficients, C order, as bspline.fit_tensor_product returns them); three
// more decode, the last one reducing the squared error against the samples
// instead of storing.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "afam_internal.h"

namespace afam {

constexpr int kFitThreads = 256;
constexpr int kFitRT = 32;     // input columns per CTA tile
constexpr int kFitMaxN = 129;  // operator extents supported (ncp, m <= 129)

// Sample grids are [d0][d1][d2] (C order, bspline.fit_tensor_product's axes
// 0, 1, 2); every axis t has its own operators for its extent d_t.
struct FitJob {
    const float *samples;      // [d0][d1][d2] float32 (block b of the batch)
    const double *op_fit[3];   // axis t: [ncp][d_t]
    const double *op_dec[3];   // axis t: [d_t][ncp]
    const double *opT_fit[3];  // axis t: [d_t][ncp4] transposed, zero-padded
    const double *opT_dec[3];  // axis t: [ncp][d_t4]
    double *buf0, *buf1;       // ping-pong intermediates (>= d0 d1 d2 doubles each)
    float *ctrl;               // nullable: [ncp][ncp][ncp] float32 coefficients out
    double *sse;               // sum of squared errors (accumulated)
    int32_t ncp, pad;
};

struct FitDims {
    int32_t d[3];
};

// element `ax` of a 3-array without a dynamic index (which would copy the
// job / the kernel parameter to local memory)
template <typename T>
__device__ __forceinline__ T sel3(const T (&v)[3], int ax) {
    return ax == 0 ? v[0] : (ax == 1 ? v[1] : v[2]);
}

// Stage s contracts axis s % 3 (fit: d_t -> ncp, decode: ncp -> d_t); R is
// the product of the two other current extents.
__device__ __forceinline__ int fit_R(int stage, const FitDims &D, int ncp) {
    switch (stage) {
        case 0: return D.d[1] * D.d[2];
        case 1: return D.d[2] * ncp;
        case 2: return ncp * ncp;
        case 3: return ncp * ncp;
        case 4: return ncp * D.d[0];
        default: return D.d[0] * D.d[1];
    }
}

// One contraction of every job: in [n0][R] (slowest axis contracted) ->
// out [R][nout].  Stage selects operator and operand types:
//   0: samples (f32) x fit op,  1-2: f64 x fit op (2 rounds the result to
//   float32 and optionally emits it),  3: coefficients x decode op,
//   4: f64 x decode op,  5: f64 x decode op -> squared error vs samples.
__global__ void __launch_bounds__(kFitThreads) contract_rotate_kernel(const FitJob *__restrict__ jobs, FitDims D,
                                                                      int stage) {
    extern __shared__ __align__(16) unsigned char smem[];
    const FitJob J = jobs[blockIdx.y];
    const int ncp = J.ncp;
    const bool dec = stage >= 3;
    const int ax = stage % 3, dt = sel3(D.d, ax);
    const int n0 = dec ? ncp : dt, nout = dec ? dt : ncp;
    const int R = fit_R(stage, D, ncp);
    const int r0 = blockIdx.x * kFitRT;
    if (r0 >= R) return;
    const int rt = min(kFitRT, R - r0);
    const double *op = dec ? sel3(J.op_dec, ax) : sel3(J.op_fit, ax);
    double *sOp = reinterpret_cast<double *>(smem);          // [nout][n0]
    double *sIn = sOp + (size_t)nout * n0;                   // [n0][kFitRT]
    double *sOut = sIn + (size_t)n0 * kFitRT;                // [kFitRT][nout]
    for (int e = threadIdx.x; e < nout * n0; e += blockDim.x) sOp[e] = op[e];
    // ping-pong: stage 0 samples -> buf0; 1: buf0 -> buf1; 2: buf1 -> buf0 (coefficients);
    // 3: buf0 -> buf1; 4: buf1 -> buf0; 5: buf0 -> squared error
    const double *in64 = nullptr;
    switch (stage) {
        case 1: in64 = J.buf0; break;
        case 2: in64 = J.buf1; break;
        case 3: in64 = J.buf0; break;
        case 4: in64 = J.buf1; break;
        case 5: in64 = J.buf0; break;
        default: break;
    }
    for (int e = threadIdx.x; e < n0 * kFitRT; e += blockDim.x) {
        const int k = e / kFitRT, r = e % kFitRT;
        double v = 0.0;
        if (r < rt) {
            const size_t g = (size_t)k * R + r0 + r;
            v = stage == 0 ? (double)J.samples[g] : in64[g];
        }
        sIn[e] = v;
    }
    __syncthreads();
    // thread: column r = lane, output rows a = warp + 8 t
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int a0 = warp; a0 < nout; a0 += 4 * nw) {
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        const int na = min(4, (nout - a0 + nw - 1) / nw);
        for (int k = 0; k < n0; k++) {
            const double x = sIn[k * kFitRT + lane];
#pragma unroll
            for (int t = 0; t < 4; t++)
                if (t < na) acc[t] = fma(sOp[(size_t)(a0 + t * nw) * n0 + k], x, acc[t]);
        }
#pragma unroll
        for (int t = 0; t < 4; t++)
            if (t < na) sOut[lane * nout + a0 + t * nw] = acc[t];
    }
    __syncthreads();
    const int total = rt * nout;
    const size_t obase = (size_t)r0 * nout;
    if (stage == 5) {
        // decoded value at flat index (r0 + r) * m + i == samples flat index: squared error
        double s = 0.0;
        for (int e = threadIdx.x; e < total; e += blockDim.x) {
            const double d = sOut[e] - (double)J.samples[obase + e];
            s = fma(d, d, s);
        }
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        __shared__ double wsum[kFitThreads / 32];
        if (lane == 0) wsum[warp] = s;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int w = 0; w < nw; w++) t += wsum[w];
            atomicAdd(J.sse, t);
        }
        return;
    }
    double *out = stage == 0 ? J.buf0 : (stage == 1 ? J.buf1 : (stage == 2 ? J.buf0 : (stage == 3 ? J.buf1 : J.buf0)));
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
        double v = sOut[e];
        if (stage == 2) {  // model.fit stores float32 coefficients (model.py:103)
            const float f = (float)v;
            if (J.ctrl) J.ctrl[obase + e] = f;
            v = (double)f;
        }
        out[obase + e] = v;
    }
}

// Register-tiled variant for operator extents <= 65 (the 65^3 micro-blocks
// of the configs): a CTA computes all output rows for 64 input columns, each
// thread a 4 x 4 (rows x columns) tile from the transposed operator and the
// input tile in shared memory (16 DFMA per 8 shared loads).
constexpr int kFitRT2 = 64;
constexpr int kFitMaxN2 = 65;

__global__ void __launch_bounds__(kFitThreads, 2) contract_tiled_kernel(const FitJob *__restrict__ jobs, FitDims D,
                                                                       int stage) {
    extern __shared__ __align__(16) unsigned char smem[];
    const FitJob J = jobs[blockIdx.y];
    const int ncp = J.ncp;
    const bool dec = stage >= 3;
    const int ax = stage % 3, dt = sel3(D.d, ax);
    const int n0 = dec ? ncp : dt, nout = dec ? dt : ncp;
    const int R = fit_R(stage, D, ncp);
    const int r0 = blockIdx.x * kFitRT2;
    if (r0 >= R) return;
    const int rt = min(kFitRT2, R - r0);
    const int np = (nout + 3) & ~3;                      // padded row count of the transposed operator
    double *sOpT = reinterpret_cast<double *>(smem);     // [n0][np]
    double *sIn = sOpT + (size_t)n0 * np;                // [n0][kFitRT2]
    double *sOut = sIn + (size_t)n0 * kFitRT2;           // [kFitRT2][nout]
    {  // transposed, padded operator [n0][np]: a straight 16-byte copy
        const double2 *src = reinterpret_cast<const double2 *>(dec ? sel3(J.opT_dec, ax) : sel3(J.opT_fit, ax));
        double2 *dst = reinterpret_cast<double2 *>(sOpT);
        for (int e = threadIdx.x; e < n0 * np / 2; e += blockDim.x) dst[e] = src[e];
    }
    const double *in64 = nullptr;
    switch (stage) {
        case 1: in64 = J.buf0; break;
        case 2: in64 = J.buf1; break;
        case 3: in64 = J.buf0; break;
        case 4: in64 = J.buf1; break;
        case 5: in64 = J.buf0; break;
        default: break;
    }
    for (int e = threadIdx.x; e < n0 * kFitRT2; e += blockDim.x) {
        const int k = e / kFitRT2, r = e % kFitRT2;
        double v = 0.0;
        if (r < rt) {
            const size_t g = (size_t)k * R + r0 + r;
            v = stage == 0 ? (double)J.samples[g] : in64[g];
        }
        sIn[e] = v;
    }
    __syncthreads();
    const int tc = threadIdx.x & 15, tr = threadIdx.x >> 4;  // 4-column group, 4-row group
    for (int ab = 0; ab < nout; ab += 64) {
        const int a0 = ab + 4 * tr;
        if (a0 < np) {
            double acc[4][4];
#pragma unroll
            for (int i = 0; i < 4; i++)
#pragma unroll
                for (int j = 0; j < 4; j++) acc[i][j] = 0.0;
            for (int k = 0; k < n0; k++) {
                const double2 o01 = *reinterpret_cast<const double2 *>(sOpT + (size_t)k * np + a0);
                const double2 o23 = *reinterpret_cast<const double2 *>(sOpT + (size_t)k * np + a0 + 2);
                const double2 x01 = *reinterpret_cast<const double2 *>(sIn + (size_t)k * kFitRT2 + 4 * tc);
                const double2 x23 = *reinterpret_cast<const double2 *>(sIn + (size_t)k * kFitRT2 + 4 * tc + 2);
                const double o[4] = {o01.x, o01.y, o23.x, o23.y}, x[4] = {x01.x, x01.y, x23.x, x23.y};
#pragma unroll
                for (int i = 0; i < 4; i++)
#pragma unroll
                    for (int j = 0; j < 4; j++) acc[i][j] = fma(o[i], x[j], acc[i][j]);
            }
#pragma unroll
            for (int i = 0; i < 4; i++)
#pragma unroll
                for (int j = 0; j < 4; j++)
                    if (a0 + i < nout) sOut[(4 * tc + j) * nout + a0 + i] = acc[i][j];
        }
    }
    __syncthreads();
    const int total = rt * nout;
    const size_t obase = (size_t)r0 * nout;
    if (stage == 5) {
        double sum = 0.0;
        for (int e = threadIdx.x; e < total; e += blockDim.x) {
            const double d = sOut[e] - (double)J.samples[obase + e];
            sum = fma(d, d, sum);
        }
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        __shared__ double wsum[kFitThreads / 32];
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        if (lane == 0) wsum[warp] = sum;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int w = 0; w < kFitThreads / 32; w++) t += wsum[w];
            atomicAdd(J.sse, t);
        }
        return;
    }
    double *out = stage == 0 ? J.buf0 : (stage == 1 ? J.buf1 : (stage == 2 ? J.buf0 : (stage == 3 ? J.buf1 : J.buf0)));
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
        double v = sOut[e];
        if (stage == 2) {  // model.fit stores float32 coefficients (model.py:103)
            const float f = (float)v;
            if (J.ctrl) J.ctrl[obase + e] = f;
            v = (double)f;
        }
        out[obase + e] = v;
    }
}

// Host: _axis_operator (bspline.py:109-125) as an explicit matrix.  With B
// the m x ncp collocation matrix and Bi its interior columns, the pinned fit
// of data d is c_0 = d_0, c_{ncp-1} = d_{m-1}, interior
// (Bi^T Bi)^{-1} Bi^T (d - B[:,0] d_0 - B[:,ncp-1] d_{m-1}) (_fit_axis,
// bspline.py:150-159); returned as F (ncp x m), c = F d.
static void host_fit_operator(int ncp, int deg, int m, std::vector<double> &F, std::vector<double> &Bd) {
    std::vector<double> band;
    std::vector<int32_t> col0;
    host_band(ncp, deg, m, band, col0);
    Bd.assign((size_t)m * ncp, 0.0);
    for (int i = 0; i < m; i++)
        for (int a = 0; a <= deg; a++) Bd[(size_t)i * ncp + col0[i] + a] = band[(size_t)i * band_stride(deg) + a];
    F.assign((size_t)ncp * m, 0.0);
    F[0] = 1.0;                                      // c_0 = d_0
    F[(size_t)(ncp - 1) * m + (m - 1)] = 1.0;        // c_{ncp-1} = d_{m-1}
    const int ni = ncp - 2;
    if (ni <= 0) return;
    // normal matrix N = Bi^T Bi and its Cholesky factor (cho_factor, lower)
    std::vector<double> N((size_t)ni * ni, 0.0);
    for (int p = 0; p < ni; p++)
        for (int q = 0; q < ni; q++) {
            double s = 0.0;
            for (int i = 0; i < m; i++) s += Bd[(size_t)i * ncp + 1 + p] * Bd[(size_t)i * ncp + 1 + q];
            N[(size_t)p * ni + q] = s;
        }
    for (int j = 0; j < ni; j++) {
        double d = N[(size_t)j * ni + j];
        for (int k = 0; k < j; k++) d -= N[(size_t)j * ni + k] * N[(size_t)j * ni + k];
        d = std::sqrt(d);
        N[(size_t)j * ni + j] = d;
        for (int i = j + 1; i < ni; i++) {
            double s = N[(size_t)i * ni + j];
            for (int k = 0; k < j; k++) s -= N[(size_t)i * ni + k] * N[(size_t)j * ni + k];
            N[(size_t)i * ni + j] = s / d;
        }
    }
    // G = Bi^T (I - B[:,0] e_0^T - B[:,ncp-1] e_{m-1}^T): ni x m; solve N X = G column by column
    std::vector<double> col(ni);
    for (int i = 0; i < m; i++) {
        for (int p = 0; p < ni; p++) {
            double g = Bd[(size_t)i * ncp + 1 + p];
            if (i == 0)
                for (int r = 0; r < m; r++) g -= Bd[(size_t)r * ncp + 1 + p] * Bd[(size_t)r * ncp + 0];
            if (i == m - 1)
                for (int r = 0; r < m; r++) g -= Bd[(size_t)r * ncp + 1 + p] * Bd[(size_t)r * ncp + ncp - 1];
            col[p] = g;
        }
        for (int p = 0; p < ni; p++) {  // L y = g
            double s = col[p];
            for (int k = 0; k < p; k++) s -= N[(size_t)p * ni + k] * col[k];
            col[p] = s / N[(size_t)p * ni + p];
        }
        for (int p = ni - 1; p >= 0; p--) {  // L^T x = y
            double s = col[p];
            for (int k = p + 1; k < ni; k++) s -= N[(size_t)k * ni + p] * col[k];
            col[p] = s / N[(size_t)p * ni + p];
        }
        for (int p = 0; p < ni; p++) F[(size_t)(1 + p) * m + i] = col[p];
    }
}

static int get_fit_op(afam_store *s, int ncp, int deg, int m, FitOp **op) {
    auto key = std::make_tuple(ncp, deg, m);
    auto it = s->fit_ops.find(key);
    if (it == s->fit_ops.end()) {
        std::vector<double> F, Bd;
        host_fit_operator(ncp, deg, m, F, Bd);
        FitOp o;
        AFAM_CUDA(cudaMalloc(&o.fit, F.size() * sizeof(double)));
        AFAM_CUDA(cudaMalloc(&o.dec, Bd.size() * sizeof(double)));
        AFAM_CUDA(cudaMemcpy(o.fit, F.data(), F.size() * sizeof(double), cudaMemcpyHostToDevice));
        AFAM_CUDA(cudaMemcpy(o.dec, Bd.data(), Bd.size() * sizeof(double), cudaMemcpyHostToDevice));
        // transposed, zero-padded copies for the tiled kernel
        const int ncp4 = (ncp + 3) & ~3, m4 = (m + 3) & ~3;
        std::vector<double> FT((size_t)m * ncp4, 0.0), BT((size_t)ncp * m4, 0.0);
        for (int a = 0; a < ncp; a++)
            for (int i = 0; i < m; i++) {
                FT[(size_t)i * ncp4 + a] = F[(size_t)a * m + i];
                BT[(size_t)a * m4 + i] = Bd[(size_t)i * ncp + a];
            }
        AFAM_CUDA(cudaMalloc(&o.fitT, FT.size() * sizeof(double)));
        AFAM_CUDA(cudaMalloc(&o.decT, BT.size() * sizeof(double)));
        AFAM_CUDA(cudaMemcpy(o.fitT, FT.data(), FT.size() * sizeof(double), cudaMemcpyHostToDevice));
        AFAM_CUDA(cudaMemcpy(o.decT, BT.data(), BT.size() * sizeof(double), cudaMemcpyHostToDevice));
        it = s->fit_ops.emplace(key, o).first;
    }
    *op = &it->second;
    return AFAM_OK;
}

}  // namespace afam

using namespace afam;

extern "C" int afam_fit_operator(int32_t ncp, int32_t degree, int32_t m, double *fit, double *dec) {
    AFAM_CHECK(degree >= 1 && degree <= AFAM_MAX_DEGREE, AFAM_E_VALUE, "degree %d outside [1, %d]", degree,
               AFAM_MAX_DEGREE);
    AFAM_CHECK(ncp >= degree + 1 && ncp <= m && m <= kFitMaxN, AFAM_E_VALUE,
               "ncp must be in [%d, %d] (m <= %d), got %d", degree + 1, m, kFitMaxN, ncp);
    std::vector<double> F, Bd;
    host_fit_operator(ncp, degree, m, F, Bd);
    if (fit) memcpy(fit, F.data(), F.size() * sizeof(double));
    if (dec) memcpy(dec, Bd.data(), Bd.size() * sizeof(double));
    return AFAM_OK;
}

extern "C" int afam_fit_rmse3(afam_store *s, const float *samples, int32_t nblk, const int32_t *dims,
                              int32_t degree, const int32_t *job_block, const int32_t *job_ncp, int32_t njobs,
                              double *rmse, float *ctrl, const int64_t *ctrl_off, void *stream) {
    AFAM_CHECK(s && samples && dims && job_block && job_ncp && rmse, AFAM_E_VALUE, "NULL argument to afam_fit_rmse");
    AFAM_CHECK(degree >= 1 && degree <= AFAM_MAX_DEGREE, AFAM_E_VALUE, "degree %d outside [1, %d]", degree,
               AFAM_MAX_DEGREE);
    FitDims D;
    int maxd = 0, mind = 1 << 30;
    for (int t = 0; t < 3; t++) {
        D.d[t] = dims[t];
        AFAM_CHECK(dims[t] >= 2 && dims[t] <= kFitMaxN, AFAM_E_VALUE, "block extent %d outside [2, %d]", dims[t],
                   kFitMaxN);
        maxd = std::max(maxd, dims[t]);
        mind = std::min(mind, dims[t]);
    }
    AFAM_CHECK(njobs >= 0 && njobs <= 65535, AFAM_E_VALUE, "at most 65535 jobs per call");
    AFAM_CHECK(!ctrl || ctrl_off, AFAM_E_VALUE, "ctrl needs ctrl_off");
    if (njobs == 0) return AFAM_OK;
    cudaStream_t st = (cudaStream_t)stream;
    AFAM_CUDA(cudaSetDevice(s->device));
    const size_t cube = (size_t)dims[0] * dims[1] * dims[2];
    std::vector<FitJob> jobs(njobs);
    double *work = nullptr, *sse = nullptr;
    AFAM_CUDA(cudaMallocAsync(&work, 2 * cube * sizeof(double) * njobs, st));
    AFAM_CUDA(cudaMallocAsync(&sse, sizeof(double) * njobs, st));
    AFAM_CUDA(cudaMemsetAsync(sse, 0, sizeof(double) * njobs, st));
    int maxncp = 0;
    {
        std::lock_guard<std::mutex> lk(s->mu);
        for (int j = 0; j < njobs; j++) {
            const int b = job_block[j], ncp = job_ncp[j];
            AFAM_CHECK(b >= 0 && b < nblk, AFAM_E_VALUE, "job %d: block %d outside [0, %d)", j, b, nblk);
            // bspline.fit_tensor_product: degree + 1 <= ncp <= m on every axis
            AFAM_CHECK(ncp >= degree + 1 && ncp <= mind, AFAM_E_VALUE, "ncp must be in [%d, %d], got %d",
                       degree + 1, mind, ncp);
            FitJob &J = jobs[j];
            for (int t = 0; t < 3; t++) {
                FitOp *op = nullptr;
                int rc = get_fit_op(s, ncp, degree, dims[t], &op);
                if (rc) return rc;
                J.op_fit[t] = op->fit;
                J.op_dec[t] = op->dec;
                J.opT_fit[t] = op->fitT;
                J.opT_dec[t] = op->decT;
            }
            J.samples = samples + (size_t)b * cube;
            J.buf0 = work + (size_t)j * 2 * cube;
            J.buf1 = J.buf0 + cube;
            J.ctrl = ctrl ? ctrl + ctrl_off[j] : nullptr;
            J.sse = sse + j;
            J.ncp = ncp;
            maxncp = std::max(maxncp, ncp);
        }
    }
    FitJob *d_jobs = nullptr;
    AFAM_CUDA(cudaMallocAsync(&d_jobs, sizeof(FitJob) * njobs, st));
    AFAM_CUDA(cudaMemcpyAsync(d_jobs, jobs.data(), sizeof(FitJob) * njobs, cudaMemcpyHostToDevice, st));
    // the widest R of each stage (over the batch's ncp) sizes the grid; CTAs past a job's R exit
    const int Rmax[6] = {dims[1] * dims[2], dims[2] * maxncp, maxncp * maxncp, maxncp * maxncp, maxncp * dims[0],
                         dims[0] * dims[1]};
    if (maxd <= kFitMaxN2) {
        const int mp = (maxd + 3) & ~3;
        const size_t smem = ((size_t)maxd * mp + (size_t)maxd * kFitRT2 + (size_t)kFitRT2 * maxd) * sizeof(double);
        AFAM_CUDA(cudaFuncSetAttribute(contract_tiled_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
        for (int stage = 0; stage < 6; stage++) {
            dim3 grid((Rmax[stage] + kFitRT2 - 1) / kFitRT2, njobs);
            contract_tiled_kernel<<<grid, kFitThreads, smem, st>>>(d_jobs, D, stage);
        }
    } else {
        const size_t smem =
            ((size_t)maxd * maxd + (size_t)maxd * kFitRT + (size_t)kFitRT * maxd) * sizeof(double);
        AFAM_CUDA(cudaFuncSetAttribute(contract_rotate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
        for (int stage = 0; stage < 6; stage++) {
            dim3 grid((Rmax[stage] + kFitRT - 1) / kFitRT, njobs);
            contract_rotate_kernel<<<grid, kFitThreads, smem, st>>>(d_jobs, D, stage);
        }
    }
    AFAM_CUDA(cudaGetLastError());
    // rmse = sqrt(sse / (d0 d1 d2)) (encoder.error_rmse: sqrt(mean(diff^2)))
    std::vector<double> h(njobs);
    AFAM_CUDA(cudaMemcpyAsync(h.data(), sse, sizeof(double) * njobs, cudaMemcpyDeviceToHost, st));
    AFAM_CUDA(cudaStreamSynchronize(st));
    for (int j = 0; j < njobs; j++) rmse[j] = std::sqrt(h[j] / (double)cube);
    AFAM_CUDA(cudaFreeAsync(d_jobs, st));
    AFAM_CUDA(cudaFreeAsync(sse, st));
    AFAM_CUDA(cudaFreeAsync(work, st));
    return AFAM_OK;
}

extern "C" int afam_fit_rmse(afam_store *s, const float *samples, int32_t nblk, int32_t m, int32_t degree,
                             const int32_t *job_block, const int32_t *job_ncp, int32_t njobs, double *rmse,
                             float *ctrl, const int64_t *ctrl_off, void *stream) {
    const int32_t dims[3] = {m, m, m};
    return afam_fit_rmse3(s, samples, nblk, dims, degree, job_block, job_ncp, njobs, rmse, ctrl, ctrl_off, stream);
}
