/*
 * vrs.h — C ABI of the B200-native VRSplat render path (libvrs.so).
 *
 * Renders 3D Gaussian splats the way VRSplat (arXiv 2505.10144,
 * /root/reference/PAPER.md, cited "P:line") defines its render path:
 *   - Optimal Projection: each Gaussian is projected onto the tangent plane of
 *     the unit sphere at the eye perpendicular to o->mu;
 *   - Optimal-Projection-compatible tile culling, Eq.4 on the per-Gaussian
 *     optimal plane, visibility-mask culling with a summed-area
 *     table;
 *   - StopThePop per-pixel depth resorting along view rays (P:274-275,
 *     P:306-309), with the per-tile sort depth taken at the back-projected
 *     maximum point;
 *   - single-pass foveated rendering: 32x32 coarse tiles, fovea split into
 *     16x16 subtiles, 2x2 pixel groups in the periphery, hybrid tiles blended
 *     with the continuous mask, periphery NN upsample + 3x3 blur.
 * The exact operation-level contract is DESIGN.md "Numerics contract"
 * (SURVEY.md §8(c)); the C++ oracle (oracle/) implements the same function
 * independently and the tests compare the two.
 *
 * Conventions
 *   - All pointers are plain host or device pointers, as stated per argument.
 *     No function takes ownership of a caller pointer.
 *   - The context owns the uploaded scene, the visibility masks and every
 *     scratch buffer; they are sized at vrs_create from vrs_config.max_* and
 *     never reallocated per frame (no per-frame allocation or host sync).
 *   - Errors are returned as vrs_status; vrs_last_error() gives a message.
 *     CUDA errors are sticky per context.  No C++ exception crosses the ABI.
 *   - A context is not thread-safe; use one context per device and thread.
 *   - Rendering is a pure, deterministic function of (scene, cameras,
 *     foveas, masks, config): outputs are bit-identical across runs.
 */
#ifndef VRS_H
#define VRS_H
#include <stdint.h>

#if defined(__GNUC__)
#define VRS_API __attribute__((visibility("default")))
#else
#define VRS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define VRS_ABI_VERSION 1
#define VRS_MAX_VIEWS 8          /* views per vrs_render_views call */
#define VRS_MAX_MASK_SLOTS 8

/* Output pixel formats (vrs_set_output_format). */
#define VRS_OUT_F32 0            /* rgba: float[4] per pixel, depth: float per pixel (default) */
#define VRS_OUT_RGBA8_D16F 1     /* rgba: uint8[4] unorm = round(clamp(v,0,1)*255), depth: IEEE binary16 */
#define VRS_OUT_RGBA16F_D32F 2   /* rgba: IEEE binary16[4] (round to nearest), depth: float */

typedef enum {
    VRS_OK = 0,
    VRS_E_INVALID_ARG = 1, /* bad argument / camera (non-orthonormal R, bad sizes, ...) */
    VRS_E_INGEST = 2,      /* scene ingest failure (all records rejected is NOT an error) */
    VRS_E_CUDA = 3,        /* CUDA runtime error (sticky) */
    VRS_E_OOM = 4,         /* device allocation failed at create */
    VRS_E_CAPACITY = 5,    /* a frame exceeded max_pairs; that frame's output is undefined */
    VRS_E_STATE = 6        /* call out of order (e.g. render before upload) */
} vrs_status;

typedef struct vrs_context vrs_context;

typedef struct {
    int32_t device;          /* CUDA device ordinal */
    int32_t max_views;       /* <= VRS_MAX_VIEWS views per render call */
    int64_t max_gaussians;   /* upper bound on uploaded Gaussians, < 2^24 (16.7 M) */
    int64_t max_pairs;       /* capacity of the Gaussian/tile pair buffers (all views of a call) */
    int32_t max_width;       /* upper bounds on view resolution */
    int32_t max_height;
    int32_t window_k;        /* per-sample StopThePop resort window; only 16 is compiled */
    int32_t assign_tile;     /* 16 or 32: Gaussian/tile assignment size */
    int32_t projection;      /* 0 = Optimal Projection (the method); 1 = EWA local-affine baseline
                                (Eq.3; 3DGS computeCov2D; config C5 comparison) */
    float near_plane;        /* view-space near cull, 0.2 */
    float background[3];     /* composited under residual transmittance; (0,0,0) */
} vrs_config;

/* Pinhole camera, OpenCV axes (x right, y down, z forward).
 * R_wc: world->camera rotation, row-major, orthonormal within 1e-4 with
 * det = +1 (else VRS_E_INVALID_ARG).  Pixel (i,j) has its centre at
 * (i+0.5, j+0.5) and casts the camera-frame ray ((i+0.5-cx)/fx, (j+0.5-cy)/fy, 1).
 * mask_slot: visibility mask slot (vrs_set_visibility_mask) or -1 = all visible. */
typedef struct {
    float R_wc[9];
    float position[3];
    float fx, fy, cx, cy;
    int32_t width, height;
    int32_t mask_slot;
} vrs_camera;

/* Single-pass foveation: full-rate rectangle
 * center +- radius (pixels), linear blend ramp of width ramp*(2*radius)
 * outside it; requires assign_tile = 32. */
typedef struct {
    int32_t enabled;
    float center[2];
    float radius[2];
    float ramp;              /* in [0, 1); paper: 0.10 */
} vrs_fovea;

typedef struct {
    int64_t pairs;               /* Gaussian/tile pairs of the last frame (all views) */
    int64_t samples;             /* rendered samples (pixels + 2x2-group samples) */
    int64_t evaluations;         /* list entries visited by samples before termination */
    int64_t contributions;       /* entries inserted into resort windows */
    int64_t overflow_samples;    /* samples whose window overflowed (approximation events) */
    int64_t terminated_samples;  /* samples that stopped at T < 1e-4 */
    int32_t tiles_by_class[4];   /* HighRes, LowRes, Hybrid, Invisible coarse tiles */
    int64_t work_items;          /* blocks of the single blend launch */
    int64_t visible_splats;      /* (view, Gaussian) with >= 1 pair */
    float stage_ms[8];           /* preprocess, scan, duplicate, sort, ranges, blend, compose, total
                                    (filled only when timing is enabled) */
    int64_t candidates;          /* (view, Gaussian) passing the conservative frustum-cone cull (step 1a) */
    int64_t frustum_gaussians;   /* Gaussians passing it for >= 1 view (read by step 1b) */
    int64_t tile_tests;          /* (Gaussian, tile) candidates of the Eq.4 test (step 3) */
} vrs_frame_stats;

/* Create a context on cfg->device; allocates all device memory.
 * Errors: VRS_E_INVALID_ARG (bad cfg), VRS_E_OOM, VRS_E_CUDA. */
VRS_API vrs_status vrs_create(const vrs_config* cfg, vrs_context** out);
VRS_API void vrs_destroy(vrs_context* ctx);
VRS_API const char* vrs_last_error(const vrs_context* ctx);
VRS_API int32_t vrs_abi_version(void);

/* Upload raw 3DGS attributes (HOST pointers, copied):
 * means n*3, quats_wxyz n*4, log_scales n*3, opacity_logits n,
 * sh n*(deg+1)^2*3 (coefficient-major RGB).  Activation on the host in
 * double (exp / sigmoid / quaternion normalisation, Sigma = R S S^T R^T,
 * Eq.1; q_cut = 2 ln(255 sigma)), rounded once to float.
 * Non-finite records are dropped and counted in *n_rejected (may be NULL);
 * Gaussian indices are those of the kept records in input order.
 * Errors: VRS_E_INVALID_ARG (n > max_gaussians, deg not in 0..3). */
VRS_API vrs_status vrs_upload_gaussians(vrs_context* ctx, int64_t n, int32_t sh_degree, const float* means,
                                const float* quats_wxyz, const float* log_scales, const float* opacity_logits,
                                const float* sh, int64_t* n_rejected);

/* The activated scene as one DEVICE blob, for the multi-GPU setup (SURVEY
 * §8e): rank 0 uploads (host activation, above) and exports; the blob goes
 * device to device to every other rank (an NCCL broadcast); they import it --
 * no host round trip, no second activation.  The blob holds, for the n kept
 * Gaussians: mu + q_cut (16 B), Sigma_w / sigma / s_max / Sigma_w^-1 (64 B),
 * s_max (4 B), SH (16 B per 4 coefficient floats) and the raw parameters the
 * backward needs (32 B), each array 256-B aligned.
 * vrs_scene_blob_bytes: size of the blob of n Gaussians at degree sh_degree.
 * vrs_export_scene: copies the context's scene into `blob` (DEVICE, `bytes`
 * = vrs_scene_blob_bytes of its n and degree), enqueued on `stream`; *n_out
 * and *deg_out (HOST, may be NULL) get n and the degree.
 * vrs_import_scene: replaces the context's scene by a blob exported by a
 * context of the same library (any device), enqueued on `stream`.
 * Errors: VRS_E_STATE (export before any upload), VRS_E_INVALID_ARG (bytes
 * not the blob size, n > max_gaussians, degree not in 0..3). */
VRS_API int64_t vrs_scene_blob_bytes(int64_t n, int32_t sh_degree);
VRS_API vrs_status vrs_export_scene(vrs_context* ctx, void* blob, int64_t bytes, int64_t* n_out, int32_t* deg_out,
                                    void* stream);
VRS_API vrs_status vrs_import_scene(vrs_context* ctx, int64_t n, int32_t sh_degree, const void* blob, int64_t bytes,
                                    void* stream);

/* Visibility mask for a slot (HOST pointer, w*h bytes, row-major, >0 =
 * visible).  mask == NULL clears the slot (all visible). */
VRS_API vrs_status vrs_set_visibility_mask(vrs_context* ctx, int32_t slot, int32_t w, int32_t h, const uint8_t* mask);

/* Backward pass of the last frame (the paper fine-tunes with a
 * differentiable StopThePop + Optimal Projection rasterizer).
 * For L = sum over pixels of grad_rgba . RGBA + grad_depth * Depth, writes
 * dL/d(raw parameters) of the uploaded Gaussians (kept records, upload order):
 * grad_means n*3, grad_quats n*4 (w,x,y,z, through the normalisation),
 * grad_log_scales n*3, grad_logits n, grad_sh n*(deg+1)^2*3 (coefficient-major
 * RGB, like the upload).  rgba/depth: the frame's own F32 outputs (DEVICE);
 * grad_rgba n_px*4, grad_depth n_px (DEVICE, the frame's layout); outputs are
 * DEVICE buffers, overwritten.  The blend order and the blended set are those
 * of the frame; clamps (alpha <= 0.99, tau >= near, colour >= 0) pass no
 * gradient.  Requires the last call to be vrs_render_views of non-foveated
 * views with the Optimal Projection, resort mode 0 and VRS_OUT_F32 (else
 * VRS_E_STATE), and the frame's buffers untouched since.  Enqueued on stream. */
VRS_API vrs_status vrs_backward(vrs_context* ctx, const float* rgba, const float* depth, const float* grad_rgba,
                                const float* grad_depth, float* grad_means, float* grad_quats,
                                float* grad_log_scales, float* grad_logits, float* grad_sh, void* stream);

/* Output format of the final pixels written by vrs_render_views,
 * vrs_render_views_host and vrs_render_views_two_pass (default VRS_OUT_F32).
 * VRS_OUT_RGBA8_D16F is the display format of an HMD compositor: 4 bytes of
 * RGBA (round-to-nearest of clamp(v, 0, 1) * 255 of the same float values)
 * and 2 bytes of depth (binary16, round to nearest) per pixel, 6 B instead of
 * 20 B — what bounds the host path is the device->host copy.  The output
 * pointers keep their float* type in the signatures; with VRS_OUT_RGBA8_D16F
 * they must point to buffers of n_px*4 bytes (rgba) and n_px uint16 (depth),
 * cast to float*.  VRS_OUT_RGBA16F_D32F (the scRGB-style half-float swap-chain
 * format) keeps the frame within the parity tolerances in 12 B instead of
 * 20 B per pixel: RGBA rounded to binary16 (|error| <= 2^-11 |v|, i.e. <= 2e-3
 * for |v| <= 4; no clamp), depth float; rgba then points to n_px*4 binary16
 * (cast to float*), depth to n_px floats.  Errors: VRS_E_INVALID_ARG (unknown
 * format). */
VRS_API vrs_status vrs_set_output_format(vrs_context* ctx, int32_t format);

/* Render n_views views (one frame: all views share one sort and one blend
 * launch).  cams: HOST array of n_views cameras; fovea: HOST array of n_views
 * entries or NULL (no foveation).  rgba: DEVICE float buffer, views
 * concatenated, each H*W*4 (RGB premultiplied = C + T*bg, A = 1 - T);
 * depth: DEVICE float buffer, each H*W (premultiplied expected ray distance,
 * SURVEY L13).  Enqueued on `stream` (a cudaStream_t, NULL = legacy default);
 * returns without synchronising (a per-eye setup cache miss — new
 * resolution, mask or fovea — synchronises once).  Errors: VRS_E_INVALID_ARG,
 * VRS_E_STATE, VRS_E_CUDA.  A frame whose pairs exceed max_pairs is reported
 * as VRS_E_CAPACITY by vrs_get_frame_stats (its output is undefined). */
VRS_API vrs_status vrs_render_views(vrs_context* ctx, int32_t n_views, const vrs_camera* cams, const vrs_fovea* fovea,
                            float* rgba, float* depth, void* stream);

/* Same as vrs_render_views but the outputs are HOST buffers (pinned memory
 * recommended): renders into context-owned device buffers, copies back on
 * `stream` and synchronises the stream before returning (end-to-end path). */
VRS_API vrs_status vrs_render_views_host(vrs_context* ctx, int32_t n_views, const vrs_camera* cams,
                                 const vrs_fovea* fovea, float* rgba_host, float* depth_host, void* stream);

/* Two-pass foveated baseline (App. A), for
 * comparison with the single-pass path.  For every view i (fovea[i] must be
 * enabled): pass 1 renders the pixels with a non-zero fovea blend weight (the
 * rectangle of half-extents radius*(1 + 2*ramp) around the centre, plus one
 * pixel, clipped to the view) at full resolution through a cropped camera
 * (principal point shifted by the integer rectangle origin: identical pixel
 * rays); pass 2 renders the whole view at half resolution (focal lengths and
 * principal point halved, ceil(W/2) x ceil(H/2)) with the view's visibility
 * mask reduced by a 2x2 OR.  Both passes of all views run as ONE frame of
 * 2*n_views views (so max_views >= 2*n_views, and the frame statistics and
 * debug hooks describe that frame).  The output (same layout as
 * vrs_render_views) is up(P2) blended with P1 by the fovea weight w:
 * w*P1 + (1-w)*up(P2) per RGBA and depth channel, up() the bilinear upsample
 * with pixel-centre alignment (full-resolution pixel i samples pass-2
 * coordinate (i - 0.5)/2) and edge clamping.  Errors as vrs_render_views. */
VRS_API vrs_status vrs_render_views_two_pass(vrs_context* ctx, int32_t n_views, const vrs_camera* cams,
                                     const vrs_fovea* fovea, float* rgba, float* depth, void* stream);

/* Detailed counters (evaluations, contributions, overflow) cost atomics;
 * stage timing costs events.  Both off by default. */
/* Resort mode of the blend (DESIGN "N2 hierarchical resort").
 * mode 0 (default): StopThePop per-sample window, K = 16;
 * mode 1: hierarchical -- per 4x4 sample block a queue of block_queue = 8
 * entries ordered by the block-centre depth (entries admitted when a sample
 * of the block passes the membership test), then per 2x2 sample group a queue
 * of 4 entries ordered by the group-centre depth, ahead of a per-sample window
 * of pixel_window = 8 ("hierarchical per-pixel resorting").
 * 0 for a size selects the compiled value.  Takes effect from the next render.
 * Errors: VRS_E_INVALID_ARG (unknown mode, sizes other than the compiled ones,
 * mode 1 with the EWA projection). */
VRS_API vrs_status vrs_set_resort_mode(vrs_context* ctx, int32_t mode, int32_t block_queue, int32_t pixel_window);

/* Sort order: VRS_SORT_STOPTHEPOP (default)
 * = the method -- per-tile key depth at the tile's maximum point and
 * the per-sample K = 16 resort window; VRS_SORT_Z = Mini-Splatting (z): one
 * key depth per Gaussian, its view-space z, blended in list order (no
 * per-sample resort, the 3DGS order that pops under rotation);
 * VRS_SORT_DIST = Mini-Splatting (Dist): key depth |mu - o|, list order
 * (pops under translation).  The per-sample alpha, depth output and
 * termination are those of the method.  Takes effect from the next render.
 * Errors: VRS_E_INVALID_ARG (unknown mode; a global sort with the
 * hierarchical resort mode). */
#define VRS_SORT_STOPTHEPOP 0
#define VRS_SORT_Z 1
#define VRS_SORT_DIST 2
VRS_API vrs_status vrs_set_sort_mode(vrs_context* ctx, int32_t mode);

/* How the blend stages each batch of splat records (the tile list's entries,
 * north_star "Gaussian batches staged into shared memory") -- results are
 * identical, only the staging differs:
 *   VRS_STAGING_THREADS (default): 32-entry batches in a two-stage shared-
 *     memory ring; the block's threads stage the first two, then the warps
 *     consume the stages at their own pace and the last warp done with a
 *     batch refills its stage with the batch two ahead (seven 16-B loads per
 *     entry, one entry per lane), completion on the stage's mbarrier -- no
 *     block barrier inside the blend loop;
 *   VRS_STAGING_TMA: block-synchronous batches of 64 whose records the Tensor
 *     Memory Accelerator copies (cp.async.bulk global -> shared, one 96-B copy
 *     per entry issued by the block's warps, completion on an mbarrier).
 * Applies to the flat (mode 0) blend from the next render.  Errors:
 * VRS_E_INVALID_ARG (unknown mode). */
#define VRS_STAGING_THREADS 0
#define VRS_STAGING_TMA 1
VRS_API vrs_status vrs_set_staging_mode(vrs_context* ctx, int32_t mode);
VRS_API vrs_status vrs_set_instrumentation(vrs_context* ctx, int32_t counters, int32_t timing);

/* Synchronises the last frame's stream and returns its statistics.
 * Returns VRS_E_CAPACITY if that frame overflowed max_pairs. */
VRS_API vrs_status vrs_get_frame_stats(vrs_context* ctx, vrs_frame_stats* out);

/* ---- parity hooks (synchronise; HOST output pointers) ---- */
/* Per-(view, Gaussian) exact pair counts of the last frame, n_views*N u32. */
VRS_API vrs_status vrs_debug_counts(vrs_context* ctx, uint32_t* counts, int64_t capacity, int64_t* n_out);
/* Pair keys ((global tile << 32) | f32 bits of the tile depth) and values
 * (Gaussian index), sorted by (key, value) (sorted=1) or as emitted by the
 * tile test (sorted=0; the emission order is arbitrary). */
VRS_API vrs_status vrs_debug_pairs(vrs_context* ctx, int32_t sorted, uint64_t* keys, uint32_t* vals, int64_t capacity,
                           int64_t* n_out);
/* [start, end) per global tile (views concatenated), 2 u32 per tile. */
VRS_API vrs_status vrs_debug_ranges(vrs_context* ctx, uint32_t* ranges, int64_t capacity, int64_t* n_out);
/* Per-Gaussian projected records of one view in the oracle's 48-float
 * semantic layout. */
VRS_API vrs_status vrs_debug_splats(vrs_context* ctx, int32_t view, float* out, int64_t capacity);
/* Per coarse tile class (0 High, 1 Low, 2 Hybrid, 3 Invisible) and visibility bit. */
VRS_API vrs_status vrs_debug_tile_info(vrs_context* ctx, int32_t view, int32_t* cls, int32_t* vis, int64_t capacity);

/* Largest tile (in pairs) the binned sort sorts in shared memory; larger
 * tiles are sorted in chunks of that size and merged in global memory.  A
 * power of two in [64, 4096] (default 2048: 256-key register runs merged in
 * shared memory; 4096 takes a one-block bitonic sort); lowering it only exercises the
 * merge path (results are identical).  Applies from the next frame. */
VRS_API vrs_status vrs_debug_set_sort_smem_cap(vrs_context* ctx, int32_t cap);

/* ---- primitives exposed for tests (DEVICE pointers, enqueued on stream) ---- */
/* Stable LSD onesweep radix sort of n (key, value) pairs in place by the low
 * key_bits bits of the key (n <= max_pairs).  */
VRS_API vrs_status vrs_sort_pairs(vrs_context* ctx, uint64_t* keys, uint32_t* vals, int64_t n, int32_t key_bits, void* stream);
/* Exclusive prefix sum of n u32 (n <= max_views*max_gaussians); *total (DEVICE) gets the sum. */
VRS_API vrs_status vrs_exclusive_scan(vrs_context* ctx, const uint32_t* in, uint32_t* out, uint32_t* total, int64_t n,
                              void* stream);

#ifdef __cplusplus
}
#endif
#endif /* VRS_H */
