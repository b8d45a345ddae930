/*
 * afam.h -- C ABI of the B200-native Adaptive-FAM decode-and-render path.
 *
 * One shared library (libafam.so, sm_100a) exports everything below.  All
 * functions are extern "C", take plain pointers and sizes, return an int
 * status (AFAM_OK == 0) and record a thread-local message readable with
 * afam_last_error().  Every device operation takes a cudaStream_t (passed
 * as void*) and is asynchronous on it unless stated.
 *
 * Each entry point replaces one reference interface of the Python package
 * splinecast (paths relative to /root/reference/pkg/src/splinecast/):
 *
 *   afam_store_put_mfa    store.load_model + model.deserialize   store.py:43-47, model.py:121-148
 *   afam_store_put        MicroModel(...) construction            model.py:27-54
 *   afam_store_evict      ModelCache._evict_one (device side)     runtime.py:104-110
 *   afam_eval_points      MicroModel.values_at / gradients_at,    model.py:64-87,
 *                         bspline.evaluate_points[_with_gradient] bspline.py:206-229
 *   afam_decode_grid      MicroModel.decode_grid,                 model.py:89-93,
 *                         bspline.decode_tensor_product           bspline.py:162-172
 *   afam_select_visible   render.select_visible                   render.py:281-320
 *   afam_fit_rmse         encoder._fit_and_measure / error_rmse   encoder.py:74-83,
 *                         model.fit, bspline.fit_tensor_product   model.py:96-107, bspline.py:109-159
 *   afam_render           render.render                           render.py:398-466
 *
 * Status -> Python exception (reference errors.py:12-25):
 *   1 MissingBlockError, 2 FormatError, 3 CapacityError, 4 ValueError,
 *   5 RuntimeError (CUDA failure).
 */
#ifndef AFAM_H_
#define AFAM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AFAM_OK 0
#define AFAM_E_MISSING_BLOCK 1
#define AFAM_E_FORMAT 2
#define AFAM_E_CAPACITY 3
#define AFAM_E_VALUE 4
#define AFAM_E_CUDA 5

#define AFAM_MAX_DEGREE 15    /* degrees 1..15 are evaluated on device */
#define AFAM_FAST_DEGREE 3    /* degrees 1..3: per-span tables and the float32 kernels;
                                 higher degrees: float64 Cox-de Boor from the knots */
#define AFAM_MAX_TF_POINTS 32  /* inline TF control points in afam_frame; more via color_pts / opacity_pts */

/* Per-slot flags (afam_store_info). */
#define AFAM_SLOT_VALID 1u
#define AFAM_SLOT_FP64 2u     /* ill-conditioned: evaluated in float64 */
#define AFAM_SLOT_DS 4u       /* down-sampled raw block (trilinear), afam_store_put_ds */

const char *afam_last_error(void);
int afam_version(void);
int afam_device_count(void);

/* ------------------------------------------------------------------ store */
typedef struct afam_store afam_store;

/*
 * A device store of `slots` micro-model slots on `device`.  Every slot can
 * hold a model with ncp <= max_ncp and degree <= AFAM_MAX_DEGREE.
 * fp64_ctrl_limit: a slot whose max |control point| exceeds it is flagged
 * AFAM_SLOT_FP64 and decoded in float64 (ill-conditioned
 * endpoint-pinned fits); <= 0 selects the default (4.0).
 */
int afam_store_create(afam_store **out, int device, int32_t slots, int32_t max_ncp,
                      double fp64_ctrl_limit);
int afam_store_destroy(afam_store *s);
int afam_store_slots(const afam_store *s, int32_t *slots, int32_t *max_ncp);

/*
 * Upload one .mfa file image (FORMAT.md:16-70) into `slot`: the raw bytes
 * are copied H2D as-is (pinned host memory makes it truly async) and a
 * device kernel realigns the knots/control points and builds the per-span
 * basis tables.  ncp and extent[6] = {lo_x,hi_x,lo_y,hi_y,lo_z,hi_z} come
 * from the manifest (FORMAT.md:63-70).  Returns AFAM_E_FORMAT for a length
 * or degree-byte mismatch (model.py:123-133).
 */
int afam_store_put_mfa(afam_store *s, int32_t slot, const uint8_t *bytes, uint64_t nbytes, int32_t ncp,
                       const double extent[6], void *stream);

/* Validate one host .mfa image without uploading it (the checks of
 * afam_store_put_mfa: length / degree byte -> AFAM_E_FORMAT, non-finite
 * control points -> AFAM_E_VALUE); *degree (nullable) receives the degree
 * byte.  Replaces the validation half of model.deserialize
 * (model.py:121-148) for loaders that move the bytes by other means. */
int afam_mfa_check(const uint8_t *bytes, uint64_t nbytes, int32_t ncp, int32_t *degree);

/* afam_store_put_mfa from a DEVICE copy of an image already validated by
 * afam_mfa_check (e.g. received over NVLink from the rank that read it from
 * the host: one H2D per cache miss for all ranks): D2D copy
 * into the slot and the same realignment.  Replaces store.load_model +
 * model.deserialize (store.py:43-47, model.py:121-148) on the receiving ranks. */
int afam_store_put_mfa_device(afam_store *s, int32_t slot, const uint8_t *dbytes, uint64_t nbytes, int32_t degree,
                              int32_t ncp, const double extent[6], void *stream);

/* Upload one down-sampled (DS) block file image (reference downsample.py:
 * 16-byte header of uint32 (nx, ny, nz, ghost) then nx*ny*nz float32 LE,
 * x fastest; serialize_ds / deserialize_ds, downsample.py:140-161) into
 * `slot`.  Errors as deserialize_ds / DsBlock: truncated header or length
 * mismatch -> AFAM_E_FORMAT; ghost not 0/1 or dims <= 2*ghost+1 ->
 * AFAM_E_VALUE; larger than a slot -> AFAM_E_CAPACITY.  The device keeps the
 * raw samples and builds the clipped-index central-difference gradient
 * grids (DsBlock._gradient_grids) for the trilinear render path. */
int afam_store_put_ds(afam_store *s, int32_t slot, const uint8_t *bytes, uint64_t nbytes, const double extent[6],
                      void *stream);

/* Upload one .mfa file straight from disk: read into a pinned staging ring
 * (no pageable copy), validate like store.load_model (missing file, length,
 * degree byte: AFAM_E_FORMAT; non-finite control points: AFAM_E_VALUE), then
 * the asynchronous H2D copy and realignment of afam_store_put_mfa.
 * *degree (nullable) receives the file's degree byte.
 * Replaces store.load_model_bytes + model.deserialize (store.py:33-47,
 * model.py:121-148) for the device loader. */
int afam_store_put_file(afam_store *s, int32_t slot, const char *path, int32_t ncp, const double extent[6],
                        int32_t *degree, void *stream);

/* Upload an already-decoded model: knots (3, ncp+degree+1) float32 full
 * clamped vectors, ctrl ncp^3 float32 x-fastest. */
int afam_store_put(afam_store *s, int32_t slot, int32_t degree, int32_t ncp, const float *knots,
                   const float *ctrl, const double extent[6], void *stream);

int afam_store_evict(afam_store *s, int32_t slot);

/* Synchronous query (waits for the slot's upload). */
int afam_store_info(afam_store *s, int32_t slot, int32_t *ncp, int32_t *degree, uint32_t *flags,
                    float *max_abs_ctrl);

/* Device -> host copy of a slot's control points (x-fastest, ncp^3) and
 * knots (3*(ncp+degree+1)); synchronous.  For parity tests. */
int afam_store_read(afam_store *s, int32_t slot, float *ctrl, float *knots);

/* ------------------------------------------------------------ K1: points */
#define AFAM_EVAL_PARAM 1u    /* pts are extent-local parameters u, not world points */
#define AFAM_EVAL_OUT_F64 2u  /* val/grad are float64 buffers (default float32) */

/*
 * Value (and optionally gradient) of the model in slot slots[i] (or
 * `slot` for all points when slots == NULL) at pts[i] (n x 3 float64,
 * device memory).  World points follow MicroModel.values_at/gradients_at
 * (u = clip((p-lo)/(hi-lo), 0, 1), gradient divided by the extent span);
 * with AFAM_EVAL_PARAM the points are parameters (bspline.evaluate_points).
 * val (n) / grad (n x 3) are device buffers of float32 (or float64 with
 * AFAM_EVAL_OUT_F64); grad may be NULL.  AFAM_SLOT_DS slots answer world
 * points with the DS baseline's trilinear queries (DsBlock.values_at /
 * gradients_at, downsample.py:101-138); they have no parameter space.
 */
int afam_eval_points(afam_store *s, const int32_t *slots, int32_t slot, const double *pts, int64_t n,
                     void *val, void *grad, uint32_t flags, void *stream);

/* --------------------------------------------------------- K3: grid decode */
/*
 * Decode blocks slots[0..nblk) on the uniform m^3 lattice (params
 * linspace(0,1,m), fresh float64 clamped knots, bspline.py:109-125).
 * out: nblk * m^3 float32 device buffer, block-major, x fastest within a
 * block.  slots is a host array.
 */
int afam_decode_grid(afam_store *s, const int32_t *slots, int32_t nblk, int32_t m, float *out,
                     void *stream);

/* afam_decode_grid with an explicit kernel choice for the float32 slots:
 * AFAM_DECODE_AUTO (the measured-faster banded CUDA-core kernel unless
 * AFAM_DECODE_TC=1 is set in the environment), AFAM_DECODE_CUDA_CORES, or
 * AFAM_DECODE_TENSOR_CORES (tcgen05 3xTF32 x stage; m == 65 and ncp <= 72,
 * other blocks fall back to the CUDA-core kernel).  Float64 slots always take
 * the float64 CUDA-core kernel.  *ntc (nullable) receives the number of
 * blocks given to the tensor-core kernel. */
#define AFAM_DECODE_AUTO 0
#define AFAM_DECODE_CUDA_CORES 1
#define AFAM_DECODE_TENSOR_CORES 2
int afam_decode_grid_ex(afam_store *s, const int32_t *slots, int32_t nblk, int32_t m, float *out, int32_t path,
                        int32_t *ntc, void *stream);

/* ------------------------------------------------- encoder inner loop */
/*
 * Batched in-level search step (reference encoder.in_level_search /
 * _fit_and_measure, encoder.py:74-156): for job j, fit block job_block[j]
 * of samples (device float32, nblk blocks of m^3, [i][j][k] C order) with
 * job_ncp[j] control points per axis (endpoint-pinned separable least
 * squares, bspline.py:109-159, float64), round the coefficients to float32
 * (model.py:96-107), decode them on the m^3 lattice (bspline.py:162-172,
 * float64) and return the RMSE against the samples in rmse[j] (host array;
 * the call synchronizes).  ctrl (device, nullable): job j's float32
 * coefficients [a][b][c] (C order) at ctrl + ctrl_off[j] (host offsets).
 * The store supplies the device and caches the per-(ncp, degree, m) operators.
 */
int afam_fit_rmse(afam_store *s, const float *samples, int32_t nblk, int32_t m, int32_t degree,
                  const int32_t *job_block, const int32_t *job_ncp, int32_t njobs, double *rmse, float *ctrl,
                  const int64_t *ctrl_off, void *stream);

/* afam_fit_rmse on non-cubic sample grids: samples are nblk blocks of
 * dims[0] x dims[1] x dims[2] ([i][j][k] C order; bspline.fit_tensor_product
 * fits any 3-D grid, one ncp on every axis, degree + 1 <= ncp <= min(dims),
 * bspline.py:128-147; encoder.in_level_search sweeps NCPs up to dims[0],
 * encoder.py:104), decoded back on the same lattice (bspline.py:162-172).
 * afam_fit_rmse(m) is dims = (m, m, m). */
int afam_fit_rmse3(afam_store *s, const float *samples, int32_t nblk, const int32_t *dims, int32_t degree,
                   const int32_t *job_block, const int32_t *job_ncp, int32_t njobs, double *rmse, float *ctrl,
                   const int64_t *ctrl_off, void *stream);

/* The fit operator F (ncp x m: coefficients = F @ samples along one axis) and
 * the dense collocation matrix B (m x ncp) of (ncp, degree, m), host float64
 * (either pointer may be NULL). */
int afam_fit_operator(int32_t ncp, int32_t degree, int32_t m, double *fit, double *dec);

/* ----------------------------------------------------------- frame egress */
/* The deflate stream (one dynamic-Huffman block built from the frame's
 * symbol histogram: per-row PNG filter + literals and distance-1 runs) of
 * the PNG image data of an RGBA8 frame (device, height x width x 4, row 0 at
 * the top); replaces the zlib pass of Frame.to_png_bytes (render.py:216-221).
 * out: device buffer, 4-byte aligned, >= ((4*width+1)*15/8 + 16) * height +
 * 2048 bytes; *out_bytes: the stream
 * length; *adler: Adler-32 of the filtered data (the zlib trailer).  The call
 * synchronizes its stream. */
int afam_png_deflate(const uint8_t *rgba, int32_t width, int32_t height, uint8_t *out, uint64_t out_cap,
                     uint64_t *out_bytes, uint32_t *adler, void *stream);

/* ------------------------------------------------------------ visibility */
typedef struct afam_manifest afam_manifest;

/* Level tables: bpa[l] blocks per axis and extents[l] (bpa^3 * 6 float64,
 * index ((i*bpa+j)*bpa+k)*6) for lod = l+1.  A block missing from the
 * manifest has NaN extents and is never emitted. */
int afam_manifest_create(afam_manifest **out, int32_t levels, const int32_t *bpa,
                         const double *const *extents);
int afam_manifest_destroy(afam_manifest *m);

/*
 * render.select_visible: pos, and the PointOfView.basis() triad f, r, u
 * (render.py:68-73), tan_y = tan(radians(fov_y)/2).  ranges may be NULL
 * (0.8-wide default bands).  Writes sorted (lod,i,j,k) quadruples; returns
 * AFAM_E_CAPACITY if more than cap blocks are visible.
 */
int afam_select_visible(const afam_manifest *m, const double pos[3], const double f[3], const double r[3],
                        const double u[3], double tan_y, double aspect, double near_, const double *ranges,
                        int32_t nranges, int32_t *out, int32_t cap, int32_t *count);

/* --------------------------------------------------------------- K2: render */
typedef struct {
    double origin[3], f[3], r[3], u[3]; /* PointOfView position + basis() */
    double tan_x, tan_y;                /* render.py:330-331 */
    int32_t width, height;              /* full frame */
    /* Rows rendered by this call: bands of band_rows rows, band b handled
     * iff b % nparts == part.  Output rows are packed in band order. */
    int32_t band_rows, nparts, part;
    double sample_distance, power, o_max, near_;     /* RenderParams */
    double ambient, diffuse, specular, shininess;
    /* TransferFunction (render.py:93-124) */
    int32_t ncolor, nopacity;
    double domain_lo, domain_hi;
    double color[AFAM_MAX_TF_POINTS][4];  /* scalar, r, g, b */
    double opacity[AFAM_MAX_TF_POINTS][2];/* scalar, alpha */
    uint32_t flags;                       /* AFAM_RENDER_* */
    /* Optional: when non-NULL, the control points are read from these
     * row-major arrays (ncolor x 4, nopacity x 2) instead of the inline ones,
     * and ncolor / nopacity are unbounded (the reference's TransferFunction
     * takes any number of points, render.py:93-115).  Read only during the
     * afam_render call. */
    const double *color_pts;
    const double *opacity_pts;
} afam_frame;

#define AFAM_RENDER_DEBUG 1u   /* write per-ray sample counts + owner hashes */
#define AFAM_RENDER_FULL_FRAME 2u  /* rgba is the whole height x width frame: this part's rows land
                                      at their frame rows (e.g. another GPU's frame buffer mapped
                                      over NVLink with afam_ipc_open) */

typedef struct {
    uint64_t samples;      /* decoded samples (value+gradient evaluations) */
    int64_t missing_key;   /* (step << 32) | ray of the first sample in an uncovered finest cell, or -1 */
    uint64_t fp64_samples; /* samples decoded on the float64 path */
    uint64_t shaded_samples; /* samples with TF opacity > 0 (gradient + shading evaluated) */
    uint64_t exact_samples;  /* samples decoded from the float64 position (exact span search) */
    uint64_t exact_cells;    /* float64 finest-cell evaluations (ray start, cell crossings, near-face samples) */
    uint64_t clear_samples;  /* AFAM_RENDER_DEBUG only: samples in transparent cells (counted, not decoded) */
} afam_render_stats;

/*
 * render.render for the resident blocks slots[0..nblocks) given in sorted
 * BlockAddress order (host array; the finest-cell owner grid of
 * render.py:357-375 is built from their extents).  rgba: uint8 buffer of
 * (rows rendered) x width x 4, in device memory or in pinned host memory
 * (cudaHostAlloc; the kernel then writes the pixels straight over the host
 * link while it marches, so no separate copy-out follows).  stats: device afam_render_stats
 * (zeroed by this call).  Debug (flags & AFAM_RENDER_DEBUG): nsamp[ray]
 * int32 and ohash[ray] uint64 (FNV-1a over owner indices) device buffers.
 */
int afam_render(afam_store *s, const afam_frame *frame, const int32_t *slots, int32_t nblocks, uint8_t *rgba,
                afam_render_stats *stats, int32_t *nsamp, uint64_t *ohash, void *stream);

/* CUDA IPC of a device buffer between the processes of one node (the fused
 * image-band gather: every rank's render kernel stores its pixels straight
 * into rank 0's frame buffer over NVLink).  handle: 64 bytes.  afam_ipc_open
 * maps a peer's buffer (peer access enabled lazily); afam_ipc_close unmaps. */
int afam_ipc_get_handle(const void *dev_ptr, uint8_t *handle);
int afam_ipc_open(const uint8_t *handle, int32_t device, void **dev_ptr);
int afam_ipc_close(void *dev_ptr);
/* A plain cudaMalloc'ed device buffer (its own allocation, so its IPC handle
 * maps exactly this buffer) and its release. */
int afam_device_alloc(int32_t device, uint64_t bytes, void **dev_ptr);
int afam_device_free(void *dev_ptr);
/* Synchronous device -> host copy (reading such a buffer back). */
int afam_copy_to_host(void *host, const void *dev_ptr, uint64_t bytes);

/* Device time (ms) of the kernels of the last afam_render on this store
 * (CUDA events recorded on its stream around the launches); waits for them. */
int afam_render_elapsed(afam_store *s, float *ms);
/* The calling thread keeps its last 2 afam_render calls in flight-safe
 * state (frame i+1 may be launched before frame i is collected):
 * afam_render_seq gives the number of calls the thread has made on the
 * store's device (the next call's sequence number), afam_render_elapsed_seq
 * the kernel time of call `seq` (one of the last two; waits for it).
 * afam_render_elapsed is the last call's.  (runtime.replay's depth-2
 * pipeline, render.submit) */
int afam_render_seq(afam_store *s, uint64_t *count);
int afam_render_elapsed_seq(afam_store *s, uint64_t seq, float *ms);

/* Rows of the full frame rendered by (band_rows, nparts, part). */
int32_t afam_frame_rows(int32_t height, int32_t band_rows, int32_t nparts, int32_t part);

/* Finest-cell owner grid of render.py:357-375 for the given slots (host). */
int afam_owner_grid(afam_store *s, const int32_t *slots, int32_t nblocks, int32_t *cells, int32_t *grid,
                    int32_t cap);

/* ------------------------------------------------------------ tooling */
/* FP32 FMA throughput probe (the K2 roofline denominator; MEASURED_PEAKS.json
 * has no FP32 figure): independent FFMA chains on every SM; writes the
 * elapsed ms and the FLOPs executed.  out: device float[148*8*256]. */
int afam_bench_fma(float *out, int32_t iters, float *ms, double *flops, void *stream);
/* FP64 twin (the roofline denominator of the float64 decode path of
 * ill-conditioned blocks).  out: device double[148*8*256]. */
int afam_bench_dfma(double *out, int32_t iters, float *ms, double *flops, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* AFAM_H_ */
