/* Pure-C use of the VRSplat B200 render library through its C ABI
 * (include/vrs.h): no Python, no PyTorch.  Creates a context, uploads a small
 * procedural scene (raw 3DGS attributes), renders one foveated stereo frame
 * into host buffers and prints a checksum line:
 *   vrs_demo: status=0 pairs=... samples=... mean_rgb=... mean_alpha=...
 * build (the library built in-tree by __graft_entry__.build()):
 *   gcc -O2 -I include examples/vrs_demo.c -L paper_2505_10144_b200 -lvrs \
 *       -Wl,-rpath,$PWD/paper_2505_10144_b200 -lm -o vrs_demo */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "vrs.h"

static uint64_t rng_state = 0x9e3779b97f4a7c15ull;
static double urand(void) { /* SplitMix64 -> [0, 1) */
    uint64_t z = (rng_state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z ^= z >> 31;
    return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

int main(void) {
    const int64_t n = 20000;
    const int W = 320, H = 256, deg = 1, ncoef = (deg + 1) * (deg + 1);
    float* means = malloc(sizeof(float) * 3 * n);
    float* quats = malloc(sizeof(float) * 4 * n);
    float* lsc = malloc(sizeof(float) * 3 * n);
    float* logit = malloc(sizeof(float) * n);
    float* sh = calloc((size_t)n * ncoef * 3, sizeof(float));
    for (int64_t i = 0; i < n; i++) { /* a shell of splats 2-8 m in front of the eyes */
        const double z = 2.0 + 6.0 * urand();
        means[3 * i + 0] = (float)((urand() - 0.5) * 1.6 * z);
        means[3 * i + 1] = (float)((urand() - 0.5) * 1.2 * z);
        means[3 * i + 2] = (float)z;
        for (int k = 0; k < 4; k++) quats[4 * i + k] = (float)(urand() - 0.5);
        for (int k = 0; k < 3; k++) lsc[3 * i + k] = (float)log(0.01 + 0.05 * urand());
        logit[i] = (float)(urand() * 4.0 - 1.0);
        for (int c = 0; c < 3; c++) sh[(size_t)i * ncoef * 3 + c] = (float)(urand() * 2.0 - 1.0);
    }
    vrs_config cfg;
    memset(&cfg, 0, sizeof cfg);
    cfg.device = 0;
    cfg.max_views = 2;
    cfg.max_gaussians = n;
    cfg.max_pairs = 1 << 22;
    cfg.max_width = W;
    cfg.max_height = H;
    cfg.window_k = 16;
    cfg.assign_tile = 32;
    cfg.projection = 0;
    cfg.near_plane = 0.2f;
    vrs_context* ctx = NULL;
    vrs_status st = vrs_create(&cfg, &ctx);
    if (st != VRS_OK) {
        fprintf(stderr, "vrs_create: status %d\n", (int)st);
        return 1;
    }
    int64_t rejected = 0;
    st = vrs_upload_gaussians(ctx, n, deg, means, quats, lsc, logit, sh, &rejected);
    vrs_camera cams[2];
    vrs_fovea fov[2];
    const float f = (float)(W / 2 / tan(55.0 * M_PI / 180.0)); /* 110 deg horizontal */
    for (int e = 0; e < 2; e++) {
        memset(&cams[e], 0, sizeof cams[e]);
        cams[e].R_wc[0] = cams[e].R_wc[4] = cams[e].R_wc[8] = 1.0f;
        cams[e].position[0] = e ? 0.0315f : -0.0315f;
        cams[e].fx = cams[e].fy = f;
        cams[e].cx = W / 2.0f;
        cams[e].cy = H / 2.0f;
        cams[e].width = W;
        cams[e].height = H;
        cams[e].mask_slot = -1;
        fov[e].enabled = 1;
        fov[e].center[0] = W / 2.0f;
        fov[e].center[1] = H / 2.0f;
        fov[e].radius[0] = W / 4.0f;
        fov[e].radius[1] = H / 4.0f;
        fov[e].ramp = 0.1f;
    }
    const size_t px = (size_t)2 * W * H;
    float* rgba = malloc(sizeof(float) * 4 * px);
    float* depth = malloc(sizeof(float) * px);
    if (st == VRS_OK) st = vrs_set_instrumentation(ctx, 1, 0);
    if (st == VRS_OK) st = vrs_render_views_host(ctx, 2, cams, fov, rgba, depth, NULL);
    vrs_frame_stats fs;
    memset(&fs, 0, sizeof fs);
    if (st == VRS_OK) st = vrs_get_frame_stats(ctx, &fs);
    double m[4] = {0, 0, 0, 0};
    for (size_t i = 0; i < px; i++)
        for (int c = 0; c < 4; c++) m[c] += rgba[4 * i + c];
    printf("vrs_demo: status=%d rejected=%lld pairs=%lld samples=%lld mean_rgb=%.6f,%.6f,%.6f mean_alpha=%.6f\n",
           (int)st, (long long)rejected, (long long)fs.pairs, (long long)fs.samples, m[0] / px, m[1] / px,
           m[2] / px, m[3] / px);
    if (st != VRS_OK) fprintf(stderr, "error: %s\n", vrs_last_error(ctx));
    vrs_destroy(ctx);
    free(means); free(quats); free(lsc); free(logit); free(sh); free(rgba); free(depth);
    return st == VRS_OK ? 0 : 1;
}
