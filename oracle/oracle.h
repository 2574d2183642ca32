/*
 * VRSplat render-path ORACLE — C API (test infrastructure, NOT product code).
 *
 * A plain, slow, single-pass-per-stage CPU implementation of what the paper
 * (arXiv 2505.10144, /root/reference/PAPER.md "P:n") defines for the render
 * path, step by step in the order of SURVEY.md §8(c) O0-O12 and DESIGN.md
 * "Numerics contract".  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no
 * code, header, table or helper with the CUDA path (paper_2505_10144_b200/).
 *
 * Parity pins: see tests/test_oracle_pins.py and DESIGN.md "Pins".  Functions
 * whose output is a contract choice rather than fixed by the paper are marked
 * "parity unpinned" there (off-axis dilation, periphery reconstruction detail).
 */
#ifndef VRS_ORACLE_H
#define VRS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One view: camera (world->camera rotation R row-major, eye centre o,
 * pinhole intrinsics, pixel (i,j) centre at (i+0.5, j+0.5)), optional mask
 * slot (-1 = all visible) and optional fovea. */
typedef struct {
    float R[9];
    float o[3];
    float fx, fy, cx, cy;
    int32_t width, height;
    int32_t mask_slot;
    int32_t fovea_enabled;
    float fovea_center[2];
    float fovea_radius[2];
    float fovea_ramp;
} orc_view;

typedef struct {
    int32_t assign_tile;   /* T_a: 16 or 32 */
    int32_t window_k;      /* per-sample resort window K, any >=1 */
    float near_plane;      /* 0.2 */
    float background[3];   /* black */
    int32_t threads;       /* worker threads over tiles; 0 = hardware concurrency */
    int32_t projection;    /* 0 = Optimal Projection, 1 = EWA baseline (config C5) */
    int32_t resort;        /* 0 = per-sample window of window_k; 1 = hierarchical
                              (DESIGN "N2"): a block queue of block_queue entries per
                              4x4 sample block ahead of a per-sample window of window_k */
    int32_t block_queue;   /* K_B >= 0 (hierarchical mode only) */
    int32_t group_queue;   /* K_G >= 0: per-2x2-group queue between the block queue and the windows */
    int32_t sort_mode;     /* 0 = StopThePop (per-tile key depth + per-sample window);
                              1 = global sort by view-space z of mu, blended in list order
                              (Mini-Splatting (z)); 2 = global sort by |mu - o|,
                              blended in list order (Mini-Splatting (Dist)) */
    int32_t tau_unclamped; /* pin hook (DESIGN R4): 1 = per-sample tau NOT clamped at the near plane
                              (flat window mode only); 0 = the contract's clamp */
} orc_params;

#define ORC_SPLAT_FLOATS 48
#define ORC_STATS 12

void* orc_create(int64_t n, int sh_degree, const float* means, const float* quats_wxyz,
                 const float* log_scales, const float* opacity_logits, const float* sh,
                 int64_t* n_rejected);
void orc_destroy(void* h);
int64_t orc_num_gaussians(void* h);
void orc_get_activated(void* h, float* mu, float* cov, float* icov, float* sigma, float* qcut);
int orc_set_mask(void* h, int slot, int w, int hgt, const uint8_t* mask);

int orc_prepare(void* h, int n_views, const orc_view* views, const orc_params* p);
int64_t orc_num_pairs(void* h);
void orc_get_counts(void* h, uint32_t* out);
void orc_get_pairs(void* h, int sorted, uint64_t* keys, uint32_t* vals);
int64_t orc_num_tiles(void* h);
void orc_get_ranges(void* h, uint32_t* out);
int orc_get_tile_info(void* h, int view, int32_t* cls, int32_t* vis);
void orc_get_splats(void* h, int view, float* out);

int orc_render(void* h, float* rgba, float* depth);
int orc_render_pixels(void* h, int64_t n, const int32_t* vxy, float* rgba, float* depth);
void orc_get_stats(void* h, int64_t* out);
int orc_render_bruteforce(void* h, int view, float* rgba, float* depth);

/* pin helpers */
int orc_tile_test(void* h, int view, int64_t g, int x0, int y0, int x1, int y1, float* out);
void orc_sat(int tw, int th, const uint8_t* bits, uint32_t* sat);
int64_t orc_sat_count(int tw, const uint32_t* sat, int x0, int y0, int x1, int y1);
float orc_eq4_edge(const float* C, const float* p, const float* d, float* xhat);
float orc_sample_depth(void* h, int view, int64_t g, float x, float y);
int64_t orc_blend_orders(void* h, int view, int32_t* counts, uint32_t* seq, int64_t cap);
void orc_sample_alpha_tau(int64_t n, const float* num, const float* ss, const float* den, const float* dtb,
                          const float* sigma, float near_plane, float* alpha, float* tau);
int orc_hier_core(int64_t n, int kb, int kg, int kp, const float* tauB, const float* tauG, const uint32_t* g,
                  const uint32_t* member, const float* tau, const float* alpha, const float* rgb, double* out,
                  int64_t* stats);

#ifdef __cplusplus
}
#endif
#endif
