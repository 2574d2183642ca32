// C ABI of libvrs (include/vrs.h): context, scene upload (host activation),
// visibility masks, per-eye static setup cache and the per-frame launch
// sequence cull -> preprocess (+ fused candidate scan) -> tile tests into
// per-tile buckets -> binned sort (+ ranges) -> blend -> compose, enqueued on
// the caller's stream (with a fork/join onto the context's side stream for
// the SH colour and the full-rate blend items) with no host sync; the
// two-pass baseline, the output formats, the resort modes and the backward.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "vrs_internal.cuh"

using namespace vrs;

namespace {

struct ViewSetup {
    bool valid = false;
    int W = 0, H = 0, mask_slot = -1, T = 0, fovea = 0;
    uint64_t mask_gen = 0;
    float gx = 0, gy = 0, rx = 0, ry = 0, ramp = 0;
    int32_t n_items = 0, n_low = 0, n_inv = 0;
    int32_t cls_count[4] = {0, 0, 0, 0};
};

template <class T>
cudaError_t dalloc(T** p, size_t count) {
    *p = nullptr;
    if (count == 0) count = 1;
    return cudaMalloc(reinterpret_cast<void**>(p), sizeof(T) * count);
}

}  // namespace

struct vrs_context {
    vrs_config cfg{};
    std::string err;
    vrs_status sticky = VRS_OK;
    // scene
    int64_t N = 0;
    int deg = 0;
    bool uploaded = false;
    float4 *d_mu = nullptr, *d_geo = nullptr, *d_sh = nullptr;
    float* d_smax = nullptr;
    float4* d_raw = nullptr;   // [N][2] raw quaternion (w,x,y,z) and (log-scales, logit): N4 backward
    float* d_gbuf = nullptr;   // [max_views][max_gaussians][24] per-(view, Gaussian) gradient records
    int sh_chunks = 0;
    // frame buffers
    float4* d_rec = nullptr;
    float4* d_col = nullptr;
    uint32_t* d_cand = nullptr;
    uint32_t *d_counts = nullptr, *d_misc = nullptr;  // misc: pairs, overflow, -, candidates, -, ovf, frustum, -
    unsigned long long* d_tv = nullptr;               // tile tests | visible splats << 36
    uint32_t* d_vis_list = nullptr;
    unsigned long long* d_sidk = nullptr;    // [test_cap] candidate map
    int64_t test_cap = 0;
    uint64_t *d_keys = nullptr, *d_keys_alt = nullptr;
    uint32_t *d_vals = nullptr, *d_vals_alt = nullptr;
    uint32_t* d_ranges = nullptr;
    int64_t max_tiles_view = 0, max_items_view = 0, low_px_view = 0;
    float4* d_low_rgba = nullptr;
    float* d_low_depth = nullptr;
    unsigned long long* d_stats = nullptr;
    uint32_t* d_scan_scratch = nullptr;
    SortScratch sort{};
    uint32_t sort_epoch = 0;
    BinScratch bin{};
    // per-view static setup
    int32_t* d_vis = nullptr;     // [V][max_tiles]
    uint32_t* d_sat = nullptr;    // [V][max_sat]
    int32_t* d_cls = nullptr;     // [V][max_tiles]
    uint32_t* d_items = nullptr;  // [V][max_items]
    int32_t* d_nitems = nullptr;  // [V][3]: items, LowRes items, invisible tiles
    uint32_t* d_inv = nullptr;    // [V][max_tiles]: invisible tiles (background-fill items)
    uint32_t* d_lowcnt = nullptr;   // [V][max_tiles]: in-launch compose counters
    float* d_rays = nullptr;        // [V][max_rays_view]: tile-corner ray tables (x then y)
    int64_t max_rays_view = 0;
    uint32_t* d_lowcnt0 = nullptr;  // [V][max_tiles]: their initial values
    int64_t max_sat_view = 0;
    ViewSetup vs[VRS_MAX_VIEWS];
    // masks
    // slots [0, VRS_MAX_MASK_SLOTS): user masks; [VRS_MAX_MASK_SLOTS, 2x): their
    // half-resolution versions for the two-pass baseline (built on demand)
    uint8_t* d_mask[2 * VRS_MAX_MASK_SLOTS] = {};
    int mask_w[2 * VRS_MAX_MASK_SLOTS] = {}, mask_h[2 * VRS_MAX_MASK_SLOTS] = {};
    uint64_t mask_gen[2 * VRS_MAX_MASK_SLOTS] = {};
    uint64_t half_src_gen[VRS_MAX_MASK_SLOTS] = {};  // user generation the half mask was built from
    bool internal_masks = false;                     // validate_camera accepts the half slots
    // two-pass baseline pass images
    float4* d_tp_rgba = nullptr;
    float* d_tp_depth = nullptr;
    size_t tp_px_cap = 0;
    uint64_t gen_counter = 1;
    // last frame
    FrameParams fp{};
    int32_t staging = VRS_STAGING_THREADS;           // blend record staging (vrs_set_staging_mode)
    int32_t sort_mode = VRS_SORT_STOPTHEPOP;         // vrs_set_sort_mode (N3 baselines)
    bool have_frame = false;
    bool last_two_pass = false;                      // last frame = internal 2n-view two-pass frame
    cudaStream_t last_stream = nullptr;
    int64_t last_items = 0, last_tiles = 0;
    int32_t last_cls[4] = {0, 0, 0, 0};
    // host-output path
    float *d_out_rgba = nullptr, *d_out_depth = nullptr;
    size_t out_px_cap = 0;
    // instrumentation
    int counters = 0, timing = 0, no_cull = 0;
    int resort = 0;  // 0 = per-sample window (K = 16); 1 = hierarchical
    int out_fmt = VRS_OUT_F32;  // vrs_set_output_format
    cudaEvent_t ev[8] = {};
    bool ev_created = false;
    // side stream of the frame: SH colour runs beside the tile tests and sort,
    // the periphery compose beside the full-rate blend launch
    cudaStream_t side = nullptr;
    cudaEvent_t fork_ev[4] = {};  // after preprocess, colour done, LowRes blend done, compose done
};

static vrs_status fail(vrs_context* c, vrs_status s, const std::string& msg) {
    if (c) c->err = msg;
    return s;
}

static vrs_status cuda_check(vrs_context* c, cudaError_t e, const char* where) {
    if (e == cudaSuccess) return VRS_OK;
    c->sticky = VRS_E_CUDA;
    c->err = std::string(where) + ": " + cudaGetErrorString(e);
    return VRS_E_CUDA;
}

#define CK(expr)                                                     \
    do {                                                             \
        vrs_status _s = cuda_check(ctx, (expr), #expr);              \
        if (_s != VRS_OK) return _s;                                 \
    } while (0)

static void free_all(vrs_context* c) {
    void* ptrs[] = {c->d_raw, c->d_gbuf, c->d_mu, c->d_geo, c->d_smax, c->d_sh, c->d_rec, c->d_col, c->d_cand, c->d_counts, c->d_misc, c->d_tv, c->d_vis_list,
                    c->d_sidk,
                    c->d_keys, c->d_keys_alt, c->d_vals, c->d_vals_alt, c->d_ranges, c->d_low_rgba, c->d_low_depth,
                    c->d_stats, c->d_scan_scratch, c->sort.hist, c->sort.status, c->sort.counters, c->d_vis,
                    c->bin.tile_cnt, c->bin.rank, c->bin.list, c->bin.list_n, c->bin.scan_stat, c->bin.scan_ctr, c->bin.tbucket, c->bin.ovf_off, c->bin.obucket,
                    c->d_sat, c->d_cls, c->d_items, c->d_nitems, c->d_inv, c->d_lowcnt, c->d_lowcnt0, c->d_rays,
                    c->d_out_rgba, c->d_out_depth};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    for (int i = 0; i < 2 * VRS_MAX_MASK_SLOTS; i++)
        if (c->d_mask[i]) cudaFree(c->d_mask[i]);
    if (c->d_tp_rgba) cudaFree(c->d_tp_rgba);
    if (c->d_tp_depth) cudaFree(c->d_tp_depth);
    if (c->ev_created)
        for (auto& e : c->ev) cudaEventDestroy(e);
    for (auto& e : c->fork_ev)
        if (e) cudaEventDestroy(e);
    if (c->side) cudaStreamDestroy(c->side);
}

extern "C" {

int32_t vrs_abi_version(void) { return VRS_ABI_VERSION; }

const char* vrs_last_error(const vrs_context* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

vrs_status vrs_create(const vrs_config* cfg, vrs_context** out) {
    if (!cfg || !out) return VRS_E_INVALID_ARG;
    *out = nullptr;
    if (cfg->max_views < 1 || cfg->max_views > VRS_MAX_VIEWS || cfg->max_gaussians < 0 || cfg->max_pairs < 1 ||
        cfg->max_pairs >= (int64_t)1 << 30 || cfg->max_width < 1 || cfg->max_height < 1 ||
        (cfg->assign_tile != 16 && cfg->assign_tile != 32) || cfg->window_k != kWindow || (cfg->projection != 0 && cfg->projection != 1) ||
        !(cfg->near_plane > 0.0f) || (int64_t)cfg->max_views * cfg->max_gaussians >= ((int64_t)1 << 32) ||
        cfg->max_gaussians >= ((int64_t)1 << 24))  // the blend stages g in 24 bits beside an 8-warp mask
        return VRS_E_INVALID_ARG;
    vrs_context* ctx = new vrs_context();
    ctx->cfg = *cfg;
    if (cudaSetDevice(cfg->device) != cudaSuccess) {
        delete ctx;
        return VRS_E_CUDA;
    }
    const int64_t V = cfg->max_views, N = std::max<int64_t>(cfg->max_gaussians, 1), P = cfg->max_pairs;
    const int64_t tw16 = (cfg->max_width + 15) / 16, th16 = (cfg->max_height + 15) / 16;
    const int64_t tw = (cfg->max_width + cfg->assign_tile - 1) / cfg->assign_tile;
    const int64_t th = (cfg->max_height + cfg->assign_tile - 1) / cfg->assign_tile;
    ctx->max_tiles_view = tw * th;
    ctx->max_items_view = tw16 * th16 + tw * th;
    ctx->max_sat_view = (tw + 1) * (th + 1);
    ctx->low_px_view = (int64_t)((cfg->max_width + 1) / 2) * ((cfg->max_height + 1) / 2);
    cudaError_t e = cudaSuccess;
    auto A = [&](cudaError_t r) { if (e == cudaSuccess) e = r; };
    A(dalloc(&ctx->d_rec, (size_t)V * N * kRecF4));
    A(dalloc(&ctx->d_col, (size_t)V * N));
    A(dalloc(&ctx->d_cand, (size_t)V * N));
    A(dalloc(&ctx->d_counts, (size_t)V * N));
    A(dalloc(&ctx->d_vis_list, (size_t)V * N));
    ctx->test_cap = 4 * P;
    A(dalloc(&ctx->d_sidk, (size_t)ctx->test_cap));
    A(dalloc(&ctx->d_misc, 8));
    A(dalloc(&ctx->d_tv, 1));  // pairs, overflow, tests, candidates, visible, tile overflow, primitive n, -
    A(dalloc(&ctx->d_keys, (size_t)P));
    A(dalloc(&ctx->d_keys_alt, (size_t)P));
    A(dalloc(&ctx->d_vals, (size_t)P));
    A(dalloc(&ctx->d_vals_alt, (size_t)P));
    A(dalloc(&ctx->d_ranges, (size_t)2 * V * ctx->max_tiles_view));
    A(dalloc(&ctx->d_low_rgba, (size_t)V * ctx->low_px_view));
    A(dalloc(&ctx->d_low_depth, (size_t)V * ctx->low_px_view));
    A(dalloc(&ctx->d_stats, 8));
    A(dalloc(&ctx->d_scan_scratch, 2 * scan_scratch_words(std::max<int64_t>(V * N, ctx->test_cap))));
    A(dalloc(&ctx->sort.hist, 8 * 256));
    A(dalloc(&ctx->sort.status, sort_status_words(P)));
    A(dalloc(&ctx->sort.counters, 8));
    ctx->sort.max_tiles = (P + 4095) / 4096;
    ctx->sort.epoch = &ctx->sort_epoch;
    ctx->bin.max_tiles = V * ctx->max_tiles_view;
    ctx->bin.cap_smem = kBinCap / 2;  // chunks sorted as 256-key runs + shared-memory merges
    A(dalloc(&ctx->bin.tile_cnt, (size_t)ctx->bin.max_tiles));
    A(dalloc(&ctx->bin.rank, (size_t)P));
    A(dalloc(&ctx->bin.tbucket, (size_t)ctx->bin.max_tiles * kTileCap));
    A(dalloc(&ctx->bin.ovf_off, (size_t)ctx->bin.max_tiles));
    A(dalloc(&ctx->bin.obucket, (size_t)P));
    A(dalloc(&ctx->bin.list, (size_t)ctx->bin.max_tiles));
    A(dalloc(&ctx->bin.list_n, 4));
    A(dalloc(&ctx->bin.scan_stat, (size_t)4 * ((ctx->bin.max_tiles + 1023) / 1024)));
    A(dalloc(&ctx->bin.scan_ctr, 2));
    A(dalloc(&ctx->d_vis, (size_t)V * ctx->max_tiles_view));
    A(dalloc(&ctx->d_cls, (size_t)V * ctx->max_tiles_view));
    A(dalloc(&ctx->d_sat, (size_t)V * ctx->max_sat_view));
    A(dalloc(&ctx->d_items, (size_t)V * ctx->max_items_view));
    A(dalloc(&ctx->d_nitems, (size_t)3 * V));
    A(dalloc(&ctx->d_inv, (size_t)V * ctx->max_tiles_view));
    A(dalloc(&ctx->d_lowcnt, (size_t)V * ctx->max_tiles_view));
    A(dalloc(&ctx->d_lowcnt0, (size_t)V * ctx->max_tiles_view));
    ctx->max_rays_view = (tw + 1) + (th + 1);
    A(dalloc(&ctx->d_rays, (size_t)V * ctx->max_rays_view));
    if (e != cudaSuccess) {
        free_all(ctx);
        delete ctx;
        cudaGetLastError();
        return (e == cudaErrorMemoryAllocation) ? VRS_E_OOM : VRS_E_CUDA;
    }
    cudaMemset(ctx->d_misc, 0, 32);
    // colours and records of splats not projected this frame are never blended
    // with a weight, but the window's sentinel (g = 0, alpha = 0) reads a colour:
    // keep it finite
    cudaMemset(ctx->d_col, 0, sizeof(float4) * (size_t)V * N);
    cudaMemset(ctx->d_rec, 0, sizeof(float4) * (size_t)V * N * kRecF4);
    ctx->bin.ovf_count = ctx->d_misc + 5;
    cudaMemset(ctx->bin.tile_cnt, 0, sizeof(uint32_t) * ctx->bin.max_tiles);  // k_tile_scan re-zeroes per frame
    cudaMemset(ctx->bin.scan_stat, 0, sizeof(unsigned long long) * 4 * ((ctx->bin.max_tiles + 1023) / 1024));
    cudaMemset(ctx->bin.scan_ctr, 0, sizeof(uint32_t) * 2);  // (both re-armed by k_tile_scan's last block)
    *out = ctx;
    return VRS_OK;
}

void vrs_destroy(vrs_context* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->cfg.device);
    cudaDeviceSynchronize();
    free_all(ctx);
    delete ctx;
}

/* Host activation (DESIGN "Numerics contract" R2):
 * double precision, rounded once to float. */
vrs_status vrs_upload_gaussians(vrs_context* ctx, int64_t n, int32_t sh_degree, const float* means,
                                const float* quats, const float* log_scales, const float* logits, const float* sh,
                                int64_t* n_rejected) {
    if (!ctx) return VRS_E_INVALID_ARG;
    if (ctx->sticky != VRS_OK) return ctx->sticky;
    if (n < 0 || n > ctx->cfg.max_gaussians || sh_degree < 0 || sh_degree > 3)
        return fail(ctx, VRS_E_INVALID_ARG, "n > max_gaussians or sh_degree not in 0..3");
    if (n > 0 && (!means || !quats || !log_scales || !logits || !sh))
        return fail(ctx, VRS_E_INVALID_ARG, "null attribute pointer");
    CK(cudaSetDevice(ctx->cfg.device));
    const int ncoef = (sh_degree + 1) * (sh_degree + 1);
    const int nfl = ncoef * 3;
    const int chunks = (nfl + 3) / 4;
    std::vector<float4> mu, geo;
    std::vector<float> shh, smaxv;
    mu.reserve(n);
    geo.reserve(4 * n);
    smaxv.reserve(n);
    std::vector<int64_t> keep;
    keep.reserve(n);
    std::vector<float4> rawv;
    rawv.reserve(2 * n);
    for (int64_t i = 0; i < n; i++) {
        const float* m = means + 3 * i;
        const float* q = quats + 4 * i;
        const float* ls = log_scales + 3 * i;
        const float* shc = sh + (size_t)i * nfl;
        bool ok = std::isfinite(m[0]) && std::isfinite(m[1]) && std::isfinite(m[2]) && std::isfinite(ls[0]) &&
                  std::isfinite(ls[1]) && std::isfinite(ls[2]) && std::isfinite(logits[i]);
        for (int k = 0; k < 4; k++) ok = ok && std::isfinite(q[k]);
        for (int k = 0; k < nfl && ok; k++) ok = std::isfinite(shc[k]);
        if (!ok) continue;
        double w = q[0], x = q[1], y = q[2], z = q[3];
        const double nrm = std::sqrt(w * w + x * x + y * y + z * z);
        if (!(nrm > 0.0)) continue;
        w /= nrm; x /= nrm; y /= nrm; z /= nrm;
        const double R[3][3] = {{1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z), 2.0 * (x * z + w * y)},
                                {2.0 * (x * y + w * z), 1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x)},
                                {2.0 * (x * z - w * y), 2.0 * (y * z + w * x), 1.0 - 2.0 * (x * x + y * y)}};
        double s2[3], is2[3];
        for (int k = 0; k < 3; k++) {
            const double s = std::exp((double)ls[k]);
            s2[k] = s * s;
            is2[k] = 1.0 / s2[k];
        }
        float c6[6], i6[6];
        const int I[6] = {0, 0, 0, 1, 1, 2}, J[6] = {0, 1, 2, 1, 2, 2};
        for (int e2 = 0; e2 < 6; e2++) {
            const int a = I[e2], b = J[e2];
            c6[e2] = (float)((R[a][0] * R[b][0]) * s2[0] + (R[a][1] * R[b][1]) * s2[1] + (R[a][2] * R[b][2]) * s2[2]);
            i6[e2] = (float)((R[a][0] * R[b][0]) * is2[0] + (R[a][1] * R[b][1]) * is2[1] +
                             (R[a][2] * R[b][2]) * is2[2]);
            ok = ok && std::isfinite(c6[e2]) && std::isfinite(i6[e2]);
        }
        if (!ok) continue;
        const double smax = std::sqrt(std::max(s2[0], std::max(s2[1], s2[2])));
        const float sg = (float)(1.0 / (1.0 + std::exp(-(double)logits[i])));
        const float qc = (float)(2.0 * std::log(255.0 * (double)sg));
        mu.push_back(make_float4(m[0], m[1], m[2], qc));
        const float smf = (float)(smax * (1.0 + 1e-6));
        geo.push_back(make_float4(c6[0], c6[1], c6[2], c6[3]));
        geo.push_back(make_float4(c6[4], c6[5], sg, smf));
        geo.push_back(make_float4(i6[0], i6[1], i6[2], i6[3]));
        geo.push_back(make_float4(i6[4], i6[5], 0.0f, 0.0f));
        smaxv.push_back(smf);
        rawv.push_back(make_float4(q[0], q[1], q[2], q[3]));
        rawv.push_back(make_float4(ls[0], ls[1], ls[2], logits[i]));
        keep.push_back(i);
    }
    const int64_t nk = (int64_t)keep.size();
    // SH: coefficient-major RGB flattened, [N][chunk] float4 (a visible Gaussian reads its own 48 floats)
    std::vector<float4> shd((size_t)chunks * std::max<int64_t>(nk, 1));
    for (int64_t r = 0; r < nk; r++) {
        const float* shc = sh + (size_t)keep[r] * nfl;
        for (int c = 0; c < chunks; c++) {
            float t[4] = {0, 0, 0, 0};
            for (int k = 0; k < 4; k++)
                if (4 * c + k < nfl) t[k] = shc[4 * c + k];
            shd[(size_t)r * chunks + c] = make_float4(t[0], t[1], t[2], t[3]);
        }
    }
    // (re)allocate scene buffers
    for (float4** p : {&ctx->d_mu, &ctx->d_geo, &ctx->d_sh, &ctx->d_raw})
        if (*p) { cudaFree(*p); *p = nullptr; }
    if (ctx->d_smax) { cudaFree(ctx->d_smax); ctx->d_smax = nullptr; }
    const size_t NN = std::max<int64_t>(nk, 1);
    CK(dalloc(&ctx->d_mu, NN));
    CK(dalloc(&ctx->d_geo, 4 * NN));
    CK(dalloc(&ctx->d_smax, NN));
    CK(dalloc(&ctx->d_sh, (size_t)chunks * NN));
    CK(dalloc(&ctx->d_raw, 2 * NN));
    if (nk > 0) {
        CK(cudaMemcpy(ctx->d_mu, mu.data(), sizeof(float4) * nk, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->d_geo, geo.data(), sizeof(float4) * 4 * nk, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->d_smax, smaxv.data(), sizeof(float) * nk, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->d_sh, shd.data(), sizeof(float4) * chunks * nk, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->d_raw, rawv.data(), sizeof(float4) * 2 * nk, cudaMemcpyHostToDevice));
    }
    ctx->N = nk;
    ctx->have_frame = false;  // the last frame's records refer to the old scene
    ctx->last_items = 0;
    ctx->deg = sh_degree;
    ctx->sh_chunks = chunks;
    ctx->uploaded = true;
    if (n_rejected) *n_rejected = n - nk;
    return VRS_OK;
}

// ---------------------------------------------------------------- scene blob (multi-GPU)
namespace {
inline size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }
struct BlobLayout {
    size_t mu, geo, smax, sh, raw, total;
};
BlobLayout blob_layout(int64_t n, int deg) {
    const size_t N = (size_t)std::max<int64_t>(n, 1);
    const int chunks = ((deg + 1) * (deg + 1) * 3 + 3) / 4;
    BlobLayout L;
    L.mu = 0;
    L.geo = L.mu + align256(16 * N);
    L.smax = L.geo + align256(64 * N);
    L.sh = L.smax + align256(4 * N);
    L.raw = L.sh + align256(16 * (size_t)chunks * N);
    L.total = L.raw + align256(32 * N);
    return L;
}
}  // namespace

int64_t vrs_scene_blob_bytes(int64_t n, int32_t sh_degree) {
    if (n < 0 || sh_degree < 0 || sh_degree > 3) return -1;
    return (int64_t)blob_layout(n, sh_degree).total;
}

vrs_status vrs_export_scene(vrs_context* ctx, void* blob, int64_t bytes, int64_t* n_out, int32_t* deg_out,
                            void* stream) {
    if (!ctx) return VRS_E_INVALID_ARG;
    if (ctx->sticky != VRS_OK) return ctx->sticky;
    if (!ctx->uploaded) return fail(ctx, VRS_E_STATE, "export before vrs_upload_gaussians");
    const BlobLayout L = blob_layout(ctx->N, ctx->deg);
    if (!blob || bytes != (int64_t)L.total) return fail(ctx, VRS_E_INVALID_ARG, "blob size differs from vrs_scene_blob_bytes");
    CK(cudaSetDevice(ctx->cfg.device));
    cudaStream_t st = (cudaStream_t)stream;
    char* b = static_cast<char*>(blob);
    const size_t N = (size_t)ctx->N;
    if (N > 0) {
        CK(cudaMemcpyAsync(b + L.mu, ctx->d_mu, 16 * N, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(b + L.geo, ctx->d_geo, 64 * N, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(b + L.smax, ctx->d_smax, 4 * N, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(b + L.sh, ctx->d_sh, 16 * (size_t)ctx->sh_chunks * N, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(b + L.raw, ctx->d_raw, 32 * N, cudaMemcpyDeviceToDevice, st));
    }
    if (n_out) *n_out = ctx->N;
    if (deg_out) *deg_out = ctx->deg;
    return VRS_OK;
}

vrs_status vrs_import_scene(vrs_context* ctx, int64_t n, int32_t sh_degree, const void* blob, int64_t bytes,
                            void* stream) {
    if (!ctx) return VRS_E_INVALID_ARG;
    if (ctx->sticky != VRS_OK) return ctx->sticky;
    if (n < 0 || n > ctx->cfg.max_gaussians || sh_degree < 0 || sh_degree > 3)
        return fail(ctx, VRS_E_INVALID_ARG, "n / sh_degree");
    const BlobLayout L = blob_layout(n, sh_degree);
    if (!blob || bytes != (int64_t)L.total) return fail(ctx, VRS_E_INVALID_ARG, "blob size differs from vrs_scene_blob_bytes");
    CK(cudaSetDevice(ctx->cfg.device));
    cudaStream_t st = (cudaStream_t)stream;
    const int chunks = ((sh_degree + 1) * (sh_degree + 1) * 3 + 3) / 4;
    for (float4** p : {&ctx->d_mu, &ctx->d_geo, &ctx->d_sh, &ctx->d_raw})
        if (*p) { cudaFree(*p); *p = nullptr; }
    if (ctx->d_smax) { cudaFree(ctx->d_smax); ctx->d_smax = nullptr; }
    const size_t NN = (size_t)std::max<int64_t>(n, 1);
    CK(dalloc(&ctx->d_mu, NN));
    CK(dalloc(&ctx->d_geo, 4 * NN));
    CK(dalloc(&ctx->d_smax, NN));
    CK(dalloc(&ctx->d_sh, (size_t)chunks * NN));
    CK(dalloc(&ctx->d_raw, 2 * NN));
    const char* b = static_cast<const char*>(blob);
    if (n > 0) {
        CK(cudaMemcpyAsync(ctx->d_mu, b + L.mu, 16 * (size_t)n, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(ctx->d_geo, b + L.geo, 64 * (size_t)n, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(ctx->d_smax, b + L.smax, 4 * (size_t)n, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(ctx->d_sh, b + L.sh, 16 * (size_t)chunks * n, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(ctx->d_raw, b + L.raw, 32 * (size_t)n, cudaMemcpyDeviceToDevice, st));
    }
    ctx->N = n;
    ctx->have_frame = false;
    ctx->last_items = 0;
    ctx->deg = sh_degree;
    ctx->sh_chunks = chunks;
    ctx->uploaded = true;
    return VRS_OK;
}

vrs_status vrs_set_visibility_mask(vrs_context* ctx, int32_t slot, int32_t w, int32_t h, const uint8_t* mask) {
    if (!ctx) return VRS_E_INVALID_ARG;
    if (ctx->sticky != VRS_OK) return ctx->sticky;
    if (slot < 0 || slot >= VRS_MAX_MASK_SLOTS) return fail(ctx, VRS_E_INVALID_ARG, "mask slot out of range");
    CK(cudaSetDevice(ctx->cfg.device));
    if (ctx->d_mask[slot]) {
        CK(cudaFree(ctx->d_mask[slot]));
        ctx->d_mask[slot] = nullptr;
    }
    ctx->mask_gen[slot] = ctx->gen_counter++;
    if (!mask) {
        ctx->mask_w[slot] = ctx->mask_h[slot] = 0;
        return VRS_OK;
    }
    if (w < 1 || h < 1 || w > ctx->cfg.max_width || h > ctx->cfg.max_height)
        return fail(ctx, VRS_E_INVALID_ARG, "mask size");
    CK(dalloc(&ctx->d_mask[slot], (size_t)w * h));
    CK(cudaMemcpy(ctx->d_mask[slot], mask, (size_t)w * h, cudaMemcpyHostToDevice));
    ctx->mask_w[slot] = w;
    ctx->mask_h[slot] = h;
    return VRS_OK;
}

vrs_status vrs_set_instrumentation(vrs_context* ctx, int32_t counters, int32_t timing) {
    if (!ctx) return VRS_E_INVALID_ARG;
    ctx->counters = counters & 1;
    ctx->no_cull = (counters >> 8) & 1;  // test hook (P12)
    ctx->timing = timing ? 1 : 0;
    if (ctx->timing && !ctx->ev_created) {
        CK(cudaSetDevice(ctx->cfg.device));
        for (auto& e : ctx->ev) CK(cudaEventCreate(&e));
        ctx->ev_created = true;
    }
    return VRS_OK;
}

static vrs_status validate_camera(vrs_context* ctx, const vrs_camera& c, const vrs_fovea* f) {
    const float* R = c.R_wc;
    for (int i = 0; i < 9; i++)
        if (!std::isfinite(R[i])) return fail(ctx, VRS_E_INVALID_ARG, "non-finite rotation");
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) {
            double d = 0;
            for (int k = 0; k < 3; k++) d += (double)R[3 * i + k] * R[3 * j + k];
            if (std::fabs(d - (i == j ? 1.0 : 0.0)) > 1e-4) return fail(ctx, VRS_E_INVALID_ARG, "R not orthonormal");
        }
    const double det = (double)R[0] * (R[4] * R[8] - R[5] * R[7]) - (double)R[1] * (R[3] * R[8] - R[5] * R[6]) +
                       (double)R[2] * (R[3] * R[7] - R[4] * R[6]);
    if (det < 0) return fail(ctx, VRS_E_INVALID_ARG, "R has det -1");
    if (!(c.fx > 0) || !(c.fy > 0) || !std::isfinite(c.cx) || !std::isfinite(c.cy) || !std::isfinite(c.position[0]) ||
        !std::isfinite(c.position[1]) || !std::isfinite(c.position[2]))
        return fail(ctx, VRS_E_INVALID_ARG, "bad intrinsics / position");
    if (c.width < 1 || c.height < 1 || c.width > ctx->cfg.max_width || c.height > ctx->cfg.max_height)
        return fail(ctx, VRS_E_INVALID_ARG, "view size exceeds max_width/max_height");
    if (c.mask_slot >= (ctx->internal_masks ? 2 * VRS_MAX_MASK_SLOTS : VRS_MAX_MASK_SLOTS))
        return fail(ctx, VRS_E_INVALID_ARG, "mask slot");
    if (c.mask_slot >= 0 && ctx->d_mask[c.mask_slot] &&
        (ctx->mask_w[c.mask_slot] != c.width || ctx->mask_h[c.mask_slot] != c.height))
        return fail(ctx, VRS_E_INVALID_ARG, "mask resolution differs from view resolution");
    if (f && f->enabled) {
        if (ctx->cfg.assign_tile != 32) return fail(ctx, VRS_E_INVALID_ARG, "foveation requires assign_tile 32");
        if (!(f->radius[0] > 0) || !(f->radius[1] > 0) || !(f->ramp >= 0) || !(f->ramp < 1) ||
            !std::isfinite(f->center[0]) || !std::isfinite(f->center[1]))
            return fail(ctx, VRS_E_INVALID_ARG, "bad fovea");
    }
    return VRS_OK;
}

// Build FrameParams for a call and refresh the per-eye setup cache.
static vrs_status prepare_frame(vrs_context* ctx, int nv, const vrs_camera* cams, const vrs_fovea* fov,
                                cudaStream_t st, FrameParams& fp, int& total_items) {
    const int T = ctx->cfg.assign_tile;
    fp = FrameParams{};
    fp.n_views = nv;
    fp.T = T;
    fp.sh_coeffs = (ctx->deg + 1) * (ctx->deg + 1);
    fp.counters = ctx->counters;
    fp.no_cull = ctx->no_cull;
    fp.resort = ctx->resort;
    fp.staging = ctx->staging;
    fp.sort_mode = ctx->sort_mode;
    fp.ewa = ctx->cfg.projection;
    fp.N = ctx->N;
    fp.pair_cap = ctx->cfg.max_pairs;
    fp.near_plane = ctx->cfg.near_plane;
    for (int i = 0; i < 3; i++) fp.bg[i] = ctx->cfg.background[i];
    int64_t tile_base = 0, pix_off = 0;
    total_items = 0;
    for (int k = 0; k < 4; k++) ctx->last_cls[k] = 0;
    for (int vi = 0; vi < nv; vi++) {
        const vrs_camera& c = cams[vi];
        ViewParams& v = fp.v[vi];
        for (int i = 0; i < 9; i++) v.R[i] = c.R_wc[i];
        for (int i = 0; i < 3; i++) v.o[i] = c.position[i];
        v.fx = c.fx; v.fy = c.fy; v.cx = c.cx; v.cy = c.cy;
        v.W = c.width; v.H = c.height;
        v.tw = (c.width + T - 1) / T;
        v.th = (c.height + T - 1) / T;
        v.tile_base = (int32_t)tile_base;
        const bool fe = fov && fov[vi].enabled;
        v.fovea = fe ? 1 : 0;
        if (fe) {
            v.gx = fov[vi].center[0]; v.gy = fov[vi].center[1];
            v.rx = fov[vi].radius[0]; v.ry = fov[vi].radius[1];
            v.ramp = fov[vi].ramp;
        }
        {   // frustum side planes (inward unit normals) and dilation bound, for k_cull
            const double xl = (0.0 - c.cx) / c.fx, xr = ((double)c.width - c.cx) / c.fx;
            const double yt = (0.0 - c.cy) / c.fy, yb = ((double)c.height - c.cy) / c.fy;
            const double Nn[4][3] = {{1.0, 0.0, -xl}, {-1.0, 0.0, xr}, {0.0, 1.0, -yt}, {0.0, -1.0, yb}};
            for (int k = 0; k < 4; k++) {
                const double nn = std::sqrt(Nn[k][0] * Nn[k][0] + Nn[k][1] * Nn[k][1] + Nn[k][2] * Nn[k][2]);
                for (int i = 0; i < 3; i++) {
                    v.plane[k][i] = (float)(Nn[k][i] / nn);
                    v.dplane[k][i] = Nn[k][i] / nn;
                }
            }
            v.kinv[0] = 1.0 / c.fx;
            v.kinv[1] = 1.0 / c.fy;
            v.kinv[2] = -(double)c.cx / c.fx;
            v.kinv[3] = -(double)c.cy / c.fy;
            const double fmin = std::min(c.fx, c.fy);
            v.dil = (float)(0.3 / (fmin * fmin) * 1.01);
        }
        v.pix_off = pix_off;
        v.low_off = (int64_t)vi * ctx->low_px_view;
        v.low_w = (c.width + 1) / 2;
        v.vis = ctx->d_vis + (size_t)vi * ctx->max_tiles_view;
        v.cls = ctx->d_cls + (size_t)vi * ctx->max_tiles_view;
        v.sat = ctx->d_sat + (size_t)vi * ctx->max_sat_view;
        v.items = ctx->d_items + (size_t)vi * ctx->max_items_view;
        v.inv_items = ctx->d_inv + (size_t)vi * ctx->max_tiles_view;
        v.lowcnt = ctx->d_lowcnt + (size_t)vi * ctx->max_tiles_view;
        v.xr = ctx->d_rays + (size_t)vi * ctx->max_rays_view;
        v.yr = v.xr + v.tw + 1;
        v.lowcnt0 = ctx->d_lowcnt0 + (size_t)vi * ctx->max_tiles_view;
        // setup cache (precomputed once per eye)
        const int ms = (c.mask_slot >= 0 && ctx->d_mask[c.mask_slot]) ? c.mask_slot : -1;
        ViewSetup& s = ctx->vs[vi];
        const uint64_t mg = ms >= 0 ? ctx->mask_gen[ms] : 0;
        const bool hit = s.valid && s.W == v.W && s.H == v.H && s.mask_slot == ms && s.mask_gen == mg && s.T == T &&
                         s.fovea == v.fovea && (!v.fovea || (s.gx == v.gx && s.gy == v.gy && s.rx == v.rx &&
                                                              s.ry == v.ry && s.ramp == v.ramp));
        if (!hit) {
            launch_setup_view(ms >= 0 ? ctx->d_mask[ms] : nullptr, v.W, v, T, ctx->d_vis + (size_t)vi * ctx->max_tiles_view,
                              ctx->d_sat + (size_t)vi * ctx->max_sat_view,
                              ctx->d_cls + (size_t)vi * ctx->max_tiles_view,
                              ctx->d_items + (size_t)vi * ctx->max_items_view, ctx->d_nitems + 3 * vi,
                              ctx->d_inv + (size_t)vi * ctx->max_tiles_view,
                              ctx->d_lowcnt + (size_t)vi * ctx->max_tiles_view,
                              ctx->d_lowcnt0 + (size_t)vi * ctx->max_tiles_view, st);
            CK(cudaGetLastError());
            int32_t ni[3] = {0, 0, 0};
            std::vector<int32_t> cls((size_t)v.tw * v.th);
            CK(cudaMemcpyAsync(ni, ctx->d_nitems + 3 * vi, 12, cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(cls.data(), ctx->d_cls + (size_t)vi * ctx->max_tiles_view, 4 * cls.size(),
                               cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            s.valid = true;
            s.W = v.W; s.H = v.H; s.mask_slot = ms; s.mask_gen = mg; s.T = T; s.fovea = v.fovea;
            s.gx = v.gx; s.gy = v.gy; s.rx = v.rx; s.ry = v.ry; s.ramp = v.ramp;
            s.n_items = ni[0];
            s.n_low = ni[1];
            s.n_inv = ni[2];
            for (int k = 0; k < 4; k++) s.cls_count[k] = 0;
            for (int32_t cc : cls) s.cls_count[cc & 3]++;
        }
        for (int k = 0; k < 4; k++) ctx->last_cls[k] += s.cls_count[k];
        v.n_items = s.n_items;
        v.n_low = s.n_low;
        v.item_off = total_items;
        total_items += s.n_items;
        v.n_inv = s.n_inv;
        v.inv_off = fp.n_inv_items;
        fp.n_inv_items += s.n_inv;
        tile_base += (int64_t)v.tw * v.th;
        pix_off += (int64_t)v.W * v.H;
    }
    if (tile_base >= ((int64_t)1 << 20)) return fail(ctx, VRS_E_INVALID_ARG, "too many tiles in one call");
    fp.n_blend_items = total_items;
    ctx->last_tiles = tile_base;
    return VRS_OK;
}

static FrameBufs frame_bufs(vrs_context* ctx) {
    FrameBufs fb{};
    fb.rec = ctx->d_rec;
    fb.col = ctx->d_col;
    fb.cand = ctx->d_cand;
    fb.cand_count = ctx->d_misc + 3;
    fb.frustum_count = ctx->d_misc + 6;
    fb.vis_list = ctx->d_vis_list;
    fb.tv = ctx->d_tv;
    fb.sidk = ctx->d_sidk;
    fb.counts = ctx->d_counts;
    fb.total = ctx->d_misc;
    fb.overflow = ctx->d_misc + 1;
    fb.keys = ctx->d_keys;
    fb.vals = ctx->d_vals;
    fb.keys_alt = ctx->d_keys_alt;
    fb.vals_alt = ctx->d_vals_alt;
    fb.ranges = ctx->d_ranges;
    fb.low_rgba = ctx->d_low_rgba;
    fb.low_depth = ctx->d_low_depth;
    fb.stats = ctx->d_stats;
    return fb;
}

static vrs_status render_impl(vrs_context* ctx, int32_t nv, const vrs_camera* cams, const vrs_fovea* fov, float* rgba,
                              float* depth, cudaStream_t st, int out_fmt) {
    if (!ctx) return VRS_E_INVALID_ARG;
    if (ctx->sticky != VRS_OK) return ctx->sticky;
    if (!ctx->uploaded) return fail(ctx, VRS_E_STATE, "render before vrs_upload_gaussians");
    if (nv < 1 || nv > ctx->cfg.max_views || !cams || !rgba || !depth)
        return fail(ctx, VRS_E_INVALID_ARG, "n_views / null pointer");
    for (int i = 0; i < nv; i++) {
        vrs_status s = validate_camera(ctx, cams[i], fov ? &fov[i] : nullptr);
        if (s != VRS_OK) return s;
    }
    CK(cudaSetDevice(ctx->cfg.device));
    FrameParams fp;
    int total_items = 0;
    {
        vrs_status s = prepare_frame(ctx, nv, cams, fov, st, fp, total_items);
        if (s != VRS_OK) return s;
    }
    fp.out_fmt = out_fmt;
    SceneDev sc{ctx->d_mu, ctx->d_geo, ctx->d_smax, ctx->d_sh, ctx->sh_chunks};
    FrameBufs fb = frame_bufs(ctx);
    const bool tm = ctx->timing && ctx->ev_created;
    if (tm) CK(cudaEventRecord(ctx->ev[0], st));
    CK(cudaMemsetAsync(ctx->d_misc + 1, 0, 4, st));
    if (ctx->counters) CK(cudaMemsetAsync(ctx->d_stats, 0, 8 * sizeof(unsigned long long), st));
    if (!ctx->side) {
        CK(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
        for (auto& e : ctx->fork_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    launch_preprocess(sc, fp, fb, ctx->test_cap, st);  // (the candidate scan is fused into it: "scan" stage ~ 0)
    if (tm) CK(cudaEventRecord(ctx->ev[1], st));
    // SH colour (needed by the blend only) beside the tile tests and the sort
    CK(cudaEventRecord(ctx->fork_ev[0], st));
    CK(cudaStreamWaitEvent(ctx->side, ctx->fork_ev[0], 0));
    launch_color(sc, fp, fb, ctx->side);
    CK(cudaEventRecord(ctx->fork_ev[1], ctx->side));
    if (tm) CK(cudaEventRecord(ctx->ev[2], st));
    launch_tiletest_direct(fp, fb, ctx->test_cap, ctx->bin, st);
    if (tm) CK(cudaEventRecord(ctx->ev[3], st));
    // binned per-tile sort; its tile-count scan also writes the ranges ("ranges" stage ~ 0)
    launch_binsort(fb, fp.pair_cap, ctx->last_tiles, ctx->bin, st);
    if (tm) CK(cudaEventRecord(ctx->ev[4], st));
    CK(cudaStreamWaitEvent(st, ctx->fork_ev[1], 0));
    if (tm) CK(cudaEventRecord(ctx->ev[5], st));
    // blend: ONE launch over every view's items (LowRes first), the invisible
    // tiles' background and the periphery compose (triggered inside the launch)
#if VRS_TWO_LAUNCH  // experiment: round-1 structure (LowRes items + inv ‖ full-rate items on the side stream)
    if (fp.resort == 0) {
        FrameParams fl = fp, ff = fp;
        int n_low = 0, n_full = 0;
        for (int i = 0; i < nv; i++) {
            fl.v[i].item_off = n_low;
            fl.v[i].n_items = fp.v[i].n_low;
            ff.v[i].items = fp.v[i].items + fp.v[i].n_low;
            ff.v[i].item_off = n_full;
            ff.v[i].n_items = fp.v[i].n_items - fp.v[i].n_low;
            n_low += fl.v[i].n_items;
            n_full += ff.v[i].n_items;
        }
        fl.n_blend_items = n_low;
        ff.n_blend_items = n_full;
        ff.n_inv_items = 0;
        CK(cudaEventRecord(ctx->fork_ev[2], st));
        CK(cudaStreamWaitEvent(ctx->side, ctx->fork_ev[2], 0));
        launch_blend(ff, fb, n_full, rgba, depth, ctx->side);
        CK(cudaEventRecord(ctx->fork_ev[3], ctx->side));
        launch_blend(fl, fb, n_low, rgba, depth, st);
        CK(cudaStreamWaitEvent(st, ctx->fork_ev[3], 0));
    } else
#endif
    launch_blend(fp, fb, total_items, rgba, depth, st);
    if (tm) CK(cudaEventRecord(ctx->ev[6], st));
    if (tm) CK(cudaEventRecord(ctx->ev[7], st));
    CK(cudaGetLastError());
    ctx->fp = fp;
    ctx->have_frame = true;
    ctx->last_two_pass = false;
    ctx->last_stream = st;
    ctx->last_items = total_items;
    return VRS_OK;
}

vrs_status vrs_render_views(vrs_context* ctx, int32_t n_views, const vrs_camera* cams, const vrs_fovea* fovea,
                            float* rgba, float* depth, void* stream) {
    if (!ctx) return VRS_E_INVALID_ARG;
    return render_impl(ctx, n_views, cams, fovea, rgba, depth, (cudaStream_t)stream, ctx->out_fmt);
}

vrs_status vrs_render_views_host(vrs_context* ctx, int32_t n_views, const vrs_camera* cams, const vrs_fovea* fovea,
                                 float* rgba_host, float* depth_host, void* stream) {
    if (!ctx) return VRS_E_INVALID_ARG;
    if (!rgba_host || !depth_host || !cams || n_views < 1) return fail(ctx, VRS_E_INVALID_ARG, "null pointer");
    size_t px = 0;
    for (int i = 0; i < n_views; i++) px += (size_t)std::max(cams[i].width, 0) * std::max(cams[i].height, 0);
    CK(cudaSetDevice(ctx->cfg.device));
    if (px > ctx->out_px_cap) {
        if (ctx->d_out_rgba) cudaFree(ctx->d_out_rgba);
        if (ctx->d_out_depth) cudaFree(ctx->d_out_depth);
        ctx->d_out_rgba = ctx->d_out_depth = nullptr;
        CK(dalloc(&ctx->d_out_rgba, 4 * px));
        CK(dalloc(&ctx->d_out_depth, px));
        ctx->out_px_cap = px;
    }
    cudaStream_t st = (cudaStream_t)stream;
    vrs_status s = render_impl(ctx, n_views, cams, fovea, ctx->d_out_rgba, ctx->d_out_depth, st, ctx->out_fmt);
    if (s != VRS_OK) return s;
    // bytes per pixel of the format: RGBA 16 / 8 / 4, depth 4 / 4 / 2
    const size_t rb = ctx->out_fmt == VRS_OUT_F32 ? 16 : (ctx->out_fmt == VRS_OUT_RGBA16F_D32F ? 8 : 4);
    const size_t db = ctx->out_fmt == VRS_OUT_RGBA8_D16F ? 2 : 4;
    CK(cudaMemcpyAsync(rgba_host, ctx->d_out_rgba, rb * px, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(depth_host, ctx->d_out_depth, db * px, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return VRS_OK;
}

/* the two-pass foveated baseline. */
static void two_pass_rect(const vrs_camera& c, const vrs_fovea& f, int& i0, int& j0, int& i1, int& j1) {
    // pixels with a non-zero blend weight lie within radius * (1 + 2 ramp) of
    // the centre (fovea_weight); one pixel of margin on each side
    const double ex = (double)f.radius[0] * (1.0 + 2.0 * (double)f.ramp);
    const double ey = (double)f.radius[1] * (1.0 + 2.0 * (double)f.ramp);
    i0 = (int)std::min(std::max(0.0, std::floor((double)f.center[0] - ex) - 1.0), (double)c.width - 1.0);
    j0 = (int)std::min(std::max(0.0, std::floor((double)f.center[1] - ey) - 1.0), (double)c.height - 1.0);
    i1 = (int)std::max(std::min((double)c.width, std::ceil((double)f.center[0] + ex) + 1.0), (double)i0 + 1.0);
    j1 = (int)std::max(std::min((double)c.height, std::ceil((double)f.center[1] + ey) + 1.0), (double)j0 + 1.0);
}

vrs_status vrs_render_views_two_pass(vrs_context* ctx, int32_t n_views, const vrs_camera* cams,
                                     const vrs_fovea* fovea, float* rgba, float* depth, void* stream) {
    if (!ctx) return VRS_E_INVALID_ARG;
    if (ctx->sticky != VRS_OK) return ctx->sticky;
    if (n_views < 1 || 2 * n_views > ctx->cfg.max_views || !cams || !fovea || !rgba || !depth)
        return fail(ctx, VRS_E_INVALID_ARG, "two-pass needs fovea, outputs and max_views >= 2 * n_views");
    for (int i = 0; i < n_views; i++) {
        if (!fovea[i].enabled) return fail(ctx, VRS_E_INVALID_ARG, "two-pass needs an enabled fovea per view");
        vrs_status s = validate_camera(ctx, cams[i], &fovea[i]);
        if (s != VRS_OK) return s;
    }
    CK(cudaSetDevice(ctx->cfg.device));
    cudaStream_t st = (cudaStream_t)stream;
    vrs_camera pc[VRS_MAX_VIEWS];
    TwoPassParams tp{};
    tp.n = n_views;
    int64_t out_off = 0, p1_px = 0, p2_px = 0;
    for (int i = 0; i < n_views; i++) {
        const vrs_camera& c = cams[i];
        int i0, j0, i1, j1;
        two_pass_rect(c, fovea[i], i0, j0, i1, j1);
        // pass 1: cropped camera, pixel (a, b) = parent pixel (i0 + a, j0 + b)
        vrs_camera c1 = c;
        c1.cx = c.cx - (float)i0;
        c1.cy = c.cy - (float)j0;
        c1.width = i1 - i0;
        c1.height = j1 - j0;
        c1.mask_slot = -1;
        // pass 2: half resolution (sample (a, b) at parent position (2a + 1, 2b + 1)), half mask
        vrs_camera c2 = c;
        c2.fx = c.fx * 0.5f;
        c2.fy = c.fy * 0.5f;
        c2.cx = c.cx * 0.5f;
        c2.cy = c.cy * 0.5f;
        c2.width = (c.width + 1) / 2;
        c2.height = (c.height + 1) / 2;
        c2.mask_slot = -1;
        const int ms = c.mask_slot;
        if (ms >= 0 && ctx->d_mask[ms]) {
            const int hs = VRS_MAX_MASK_SLOTS + ms;
            if (!ctx->d_mask[hs] || ctx->half_src_gen[ms] != ctx->mask_gen[ms] || ctx->mask_w[hs] != c2.width ||
                ctx->mask_h[hs] != c2.height) {
                if (ctx->d_mask[hs]) CK(cudaFree(ctx->d_mask[hs]));
                ctx->d_mask[hs] = nullptr;
                CK(dalloc(&ctx->d_mask[hs], (size_t)c2.width * c2.height));
                launch_mask_half(ctx->d_mask[ms], c.width, c.height, ctx->d_mask[hs], c2.width, c2.height, st);
                CK(cudaGetLastError());
                ctx->mask_w[hs] = c2.width;
                ctx->mask_h[hs] = c2.height;
                ctx->mask_gen[hs] = ctx->gen_counter++;
                ctx->half_src_gen[ms] = ctx->mask_gen[ms];
            }
            c2.mask_slot = hs;
        }
        pc[i] = c1;
        pc[n_views + i] = c2;
        TwoPassView& t = tp.v[i];
        t.W = c.width; t.H = c.height;
        t.i0 = i0; t.j0 = j0; t.w1 = c1.width; t.h1 = c1.height;
        t.W2 = c2.width; t.H2 = c2.height;
        t.out_off = out_off;
        t.p1_off = p1_px;
        t.gx = fovea[i].center[0]; t.gy = fovea[i].center[1];
        t.rx = fovea[i].radius[0]; t.ry = fovea[i].radius[1];
        t.ramp = fovea[i].ramp;
        out_off += (int64_t)c.width * c.height;
        p1_px += (int64_t)c1.width * c1.height;
        p2_px += (int64_t)c2.width * c2.height;
    }
    {   // pass images: all pass-1 views, then all pass-2 views (the render's view order)
        int64_t o = p1_px;
        for (int i = 0; i < n_views; i++) {
            tp.v[i].p2_off = o;
            o += (int64_t)tp.v[i].W2 * tp.v[i].H2;
        }
    }
    const size_t tot = (size_t)(p1_px + p2_px);
    if (tot > ctx->tp_px_cap) {
        if (ctx->d_tp_rgba) cudaFree(ctx->d_tp_rgba);
        if (ctx->d_tp_depth) cudaFree(ctx->d_tp_depth);
        ctx->d_tp_rgba = nullptr;
        ctx->d_tp_depth = nullptr;
        ctx->tp_px_cap = 0;
        CK(dalloc(&ctx->d_tp_rgba, tot));
        CK(dalloc(&ctx->d_tp_depth, tot));
        ctx->tp_px_cap = tot;
    }
    ctx->internal_masks = true;
    vrs_status s = render_impl(ctx, 2 * n_views, pc, nullptr, reinterpret_cast<float*>(ctx->d_tp_rgba),
                               ctx->d_tp_depth, st, VRS_OUT_F32);
    ctx->internal_masks = false;
    if (s != VRS_OK) return s;
    ctx->last_two_pass = true;  // the frame state is the internal 2n-view frame: no backward on it
    tp.out_fmt = ctx->out_fmt;
    launch_two_pass_combine(tp, ctx->d_tp_rgba, ctx->d_tp_depth, rgba, depth, out_off, st);
    CK(cudaGetLastError());
    return VRS_OK;
}

vrs_status vrs_get_frame_stats(vrs_context* ctx, vrs_frame_stats* out) {
    if (!ctx || !out) return VRS_E_INVALID_ARG;
    if (ctx->sticky != VRS_OK) return ctx->sticky;
    if (!ctx->have_frame) return fail(ctx, VRS_E_STATE, "no frame rendered");
    CK(cudaSetDevice(ctx->cfg.device));
    CK(cudaStreamSynchronize(ctx->last_stream));
    std::memset(out, 0, sizeof(*out));
    uint32_t misc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    unsigned long long tv = 0;
    CK(cudaMemcpy(misc, ctx->d_misc, 32, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&tv, ctx->d_tv, 8, cudaMemcpyDeviceToHost));
    out->pairs = misc[0];
    out->candidates = misc[3];
    out->frustum_gaussians = misc[6];
    out->tile_tests = (int64_t)(tv & ((1ull << 36) - 1ull));
    unsigned long long st[8] = {0};
    if (ctx->counters) CK(cudaMemcpy(st, ctx->d_stats, sizeof(st), cudaMemcpyDeviceToHost));
    out->evaluations = (int64_t)st[0];
    out->contributions = (int64_t)st[1];
    out->overflow_samples = (int64_t)st[2];
    out->terminated_samples = (int64_t)st[3];
    int64_t samples = 0;
    for (int vi = 0; vi < ctx->fp.n_views; vi++) {
        const ViewSetup& s = ctx->vs[vi];
        const ViewParams& v = ctx->fp.v[vi];
        // samples = full-rate pixels of High/Hybrid tiles + groups of Low tiles (in image)
        std::vector<int32_t> cls((size_t)v.tw * v.th);
        CK(cudaMemcpy(cls.data(), v.cls, 4 * cls.size(), cudaMemcpyDeviceToHost));
        const int T = ctx->fp.T;
        for (int t = 0; t < (int)cls.size(); t++) {
            const int tx = t % v.tw, ty = t / v.tw;
            const int w = std::min(T, v.W - tx * T), h = std::min(T, v.H - ty * T);
            if (cls[t] == kHigh || cls[t] == kHybrid) samples += (int64_t)w * h;
            else if (cls[t] == kLow) samples += (int64_t)((w + 1) / 2) * ((h + 1) / 2);
        }
        (void)s;
    }
    out->samples = samples;
    for (int k = 0; k < 4; k++) out->tiles_by_class[k] = ctx->last_cls[k];
    out->work_items = ctx->last_items;
    {
        std::vector<uint32_t> cnt((size_t)ctx->fp.n_views * ctx->N);
        launch_counts(ctx->fp, frame_bufs(ctx), ctx->test_cap, ctx->last_stream);
        CK(cudaStreamSynchronize(ctx->last_stream));
        if (!cnt.empty())
            CK(cudaMemcpy(cnt.data(), ctx->d_counts, 4 * cnt.size(), cudaMemcpyDeviceToHost));
        int64_t vsplat = 0;
        for (uint32_t c : cnt) vsplat += c > 0;
        out->visible_splats = vsplat;
    }
    if (ctx->timing && ctx->ev_created) {
        for (int k = 0; k < 7; k++) CK(cudaEventElapsedTime(&out->stage_ms[k], ctx->ev[k], ctx->ev[k + 1]));
        CK(cudaEventElapsedTime(&out->stage_ms[7], ctx->ev[0], ctx->ev[7]));
    }
    if (misc[1] || (int64_t)misc[0] > ctx->cfg.max_pairs || (int64_t)(tv & ((1ull << 36) - 1ull)) > ctx->test_cap)
        return fail(ctx, VRS_E_CAPACITY, "pair buffer overflow (max_pairs too small)");
    return VRS_OK;
}

vrs_status vrs_debug_counts(vrs_context* ctx, uint32_t* counts, int64_t capacity, int64_t* n_out) {
    if (!ctx || !counts) return VRS_E_INVALID_ARG;
    if (!ctx->have_frame) return fail(ctx, VRS_E_STATE, "no frame");
    CK(cudaStreamSynchronize(ctx->last_stream));
    const int64_t n = (int64_t)ctx->fp.n_views * ctx->N;
    if (n_out) *n_out = n;
    if (capacity < n) return fail(ctx, VRS_E_INVALID_ARG, "capacity");
    launch_counts(ctx->fp, frame_bufs(ctx), ctx->test_cap, ctx->last_stream);
    CK(cudaStreamSynchronize(ctx->last_stream));
    if (n) CK(cudaMemcpy(counts, ctx->d_counts, 4 * n, cudaMemcpyDeviceToHost));
    return VRS_OK;
}

/* backward of the last frame (training mode). */
vrs_status vrs_backward(vrs_context* ctx, const float* rgba, const float* depth, const float* grad_rgba,
                        const float* grad_depth, float* grad_means, float* grad_quats, float* grad_log_scales,
                        float* grad_logits, float* grad_sh, void* stream) {
    if (!ctx) return VRS_E_INVALID_ARG;
    if (ctx->sticky != VRS_OK) return ctx->sticky;
    if (!ctx->have_frame) return fail(ctx, VRS_E_STATE, "backward needs a rendered frame");
    if (!rgba || !depth || !grad_rgba || !grad_depth || !grad_means || !grad_quats || !grad_log_scales ||
        !grad_logits || !grad_sh)
        return fail(ctx, VRS_E_INVALID_ARG, "null pointer");
    const FrameParams& fp = ctx->fp;
    if (fp.ewa || fp.resort != 0 || fp.sort_mode != VRS_SORT_STOPTHEPOP || fp.out_fmt != VRS_OUT_F32 ||
        ctx->last_two_pass)
        return fail(ctx, VRS_E_STATE, "backward needs a frame rendered with the Optimal Projection, the K = 16 "
                                      "window and F32 outputs by vrs_render_views");
    for (int i = 0; i < fp.n_views; i++)
        if (fp.v[i].fovea) return fail(ctx, VRS_E_STATE, "backward needs a non-foveated frame");
    CK(cudaSetDevice(ctx->cfg.device));
    cudaStream_t st = (cudaStream_t)stream;
    const size_t gcount = (size_t)ctx->cfg.max_views * (size_t)std::max<int64_t>(ctx->cfg.max_gaussians, 1) * 24;
    if (!ctx->d_gbuf) CK(dalloc(&ctx->d_gbuf, gcount));
    const size_t N = (size_t)ctx->N;
    CK(cudaMemsetAsync(ctx->d_gbuf, 0, sizeof(float) * (size_t)fp.n_views * N * 24, st));
    CK(cudaMemsetAsync(grad_means, 0, sizeof(float) * 3 * N, st));
    CK(cudaMemsetAsync(grad_quats, 0, sizeof(float) * 4 * N, st));
    CK(cudaMemsetAsync(grad_log_scales, 0, sizeof(float) * 3 * N, st));
    CK(cudaMemsetAsync(grad_logits, 0, sizeof(float) * N, st));
    CK(cudaMemsetAsync(grad_sh, 0, sizeof(float) * 3 * (size_t)fp.sh_coeffs * N, st));
    launch_backward(fp, frame_bufs(ctx), ctx->last_items, ctx->d_mu, ctx->d_raw,
                    reinterpret_cast<const float*>(ctx->d_sh), 4 * ctx->sh_chunks, rgba, depth, grad_rgba,
                    grad_depth, ctx->d_gbuf, grad_means, grad_quats, grad_log_scales, grad_logits, grad_sh, st);
    CK(cudaGetLastError());
    return VRS_OK;
}

vrs_status vrs_set_output_format(vrs_context* ctx, int32_t format) {
    if (!ctx) return VRS_E_INVALID_ARG;
    if (format != VRS_OUT_F32 && format != VRS_OUT_RGBA8_D16F && format != VRS_OUT_RGBA16F_D32F)
        return fail(ctx, VRS_E_INVALID_ARG,
                    "output format must be VRS_OUT_F32, VRS_OUT_RGBA8_D16F or VRS_OUT_RGBA16F_D32F");
    ctx->out_fmt = format;
    return VRS_OK;
}

vrs_status vrs_set_resort_mode(vrs_context* ctx, int32_t mode, int32_t block_queue, int32_t pixel_window) {
    if (!ctx) return VRS_E_INVALID_ARG;
    if (mode == 0) {
        if (pixel_window != 0 && pixel_window != kWindow)
            return fail(ctx, VRS_E_INVALID_ARG, "per-sample mode: only K = 16 is compiled");
    } else if (mode == 1) {
        if ((block_queue != 0 && block_queue != kHierQueue) || (pixel_window != 0 && pixel_window != kHierWindow))
            return fail(ctx, VRS_E_INVALID_ARG, "hierarchical mode: only K_B = 8, K_P = 8 are compiled");
        if (ctx->cfg.projection != 0)
            return fail(ctx, VRS_E_INVALID_ARG, "hierarchical mode needs the Optimal Projection");
        if (ctx->sort_mode != VRS_SORT_STOPTHEPOP)
            return fail(ctx, VRS_E_INVALID_ARG, "hierarchical mode needs the StopThePop sort");
    } else {
        return fail(ctx, VRS_E_INVALID_ARG, "resort mode must be 0 or 1");
    }
    ctx->resort = mode;
    return VRS_OK;
}

vrs_status vrs_set_sort_mode(vrs_context* ctx, int32_t mode) {
    if (!ctx) return VRS_E_INVALID_ARG;
    if (mode != VRS_SORT_STOPTHEPOP && mode != VRS_SORT_Z && mode != VRS_SORT_DIST)
        return fail(ctx, VRS_E_INVALID_ARG, "sort mode must be VRS_SORT_STOPTHEPOP, VRS_SORT_Z or VRS_SORT_DIST");
    if (mode != VRS_SORT_STOPTHEPOP && ctx->resort != 0)
        return fail(ctx, VRS_E_INVALID_ARG, "a global sort has no per-sample resort: set resort mode 0 first");
    ctx->sort_mode = mode;
    return VRS_OK;
}

vrs_status vrs_set_staging_mode(vrs_context* ctx, int32_t mode) {
    if (!ctx) return VRS_E_INVALID_ARG;
    if (mode != VRS_STAGING_THREADS && mode != VRS_STAGING_TMA)
        return fail(ctx, VRS_E_INVALID_ARG, "staging mode must be VRS_STAGING_THREADS or VRS_STAGING_TMA");
    ctx->staging = mode;
    return VRS_OK;
}

vrs_status vrs_debug_set_sort_smem_cap(vrs_context* ctx, int32_t cap) {
    if (!ctx) return VRS_E_INVALID_ARG;
    if (cap < 64 || cap > (int32_t)kBinCap || (cap & (cap - 1)))
        return fail(ctx, VRS_E_INVALID_ARG, "sort smem cap must be a power of two in [64, 4096]");
    ctx->bin.cap_smem = (uint32_t)cap;
    return VRS_OK;
}

vrs_status vrs_debug_pairs(vrs_context* ctx, int32_t sorted, uint64_t* keys, uint32_t* vals, int64_t capacity,
                           int64_t* n_out) {
    if (!ctx || !keys || !vals) return VRS_E_INVALID_ARG;
    if (!ctx->have_frame) return fail(ctx, VRS_E_STATE, "no frame");
    cudaStream_t st = ctx->last_stream;
    CK(cudaStreamSynchronize(st));
    uint32_t P = 0;
    CK(cudaMemcpy(&P, ctx->d_misc, 4, cudaMemcpyDeviceToHost));
    const int64_t n = std::min<int64_t>(P, ctx->cfg.max_pairs);
    if (n_out) *n_out = n;
    if (capacity < n) return fail(ctx, VRS_E_INVALID_ARG, "capacity");
    if (sorted) {
        CK(cudaMemcpy(keys, ctx->d_keys, 8 * n, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(vals, ctx->d_vals, 4 * n, cudaMemcpyDeviceToHost));
    } else {
        // re-run the fused tests + compaction (emission order) into the alternate buffers
        FrameBufs fb = frame_bufs(ctx);
        launch_tiletest(ctx->fp, fb, ctx->test_cap, ctx->d_keys_alt, ctx->d_vals_alt, ctx->sort.counters + 7,
                        st);  // (re-derives the same pair total)
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(st));
        CK(cudaMemcpy(keys, ctx->d_keys_alt, 8 * n, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(vals, ctx->d_vals_alt, 4 * n, cudaMemcpyDeviceToHost));
    }
    return VRS_OK;
}

vrs_status vrs_debug_ranges(vrs_context* ctx, uint32_t* ranges, int64_t capacity, int64_t* n_out) {
    if (!ctx || !ranges) return VRS_E_INVALID_ARG;
    if (!ctx->have_frame) return fail(ctx, VRS_E_STATE, "no frame");
    CK(cudaStreamSynchronize(ctx->last_stream));
    if (n_out) *n_out = ctx->last_tiles;
    if (capacity < 2 * ctx->last_tiles) return fail(ctx, VRS_E_INVALID_ARG, "capacity");
    CK(cudaMemcpy(ranges, ctx->d_ranges, 8 * ctx->last_tiles, cudaMemcpyDeviceToHost));
    return VRS_OK;
}

vrs_status vrs_debug_splats(vrs_context* ctx, int32_t view, float* out, int64_t capacity) {
    if (!ctx || !out) return VRS_E_INVALID_ARG;
    if (!ctx->have_frame || view < 0 || view >= ctx->fp.n_views) return fail(ctx, VRS_E_STATE, "no such view");
    if (capacity < 48 * ctx->N) return fail(ctx, VRS_E_INVALID_ARG, "capacity");
    cudaStream_t st = ctx->last_stream;
    CK(cudaStreamSynchronize(st));
    if (ctx->N == 0) return VRS_OK;
    float* d = nullptr;
    CK(dalloc(&d, 48 * (size_t)ctx->N));
    SceneDev sc{ctx->d_mu, ctx->d_geo, ctx->d_smax, ctx->d_sh, ctx->sh_chunks};
    FrameBufs fb = frame_bufs(ctx);
    launch_counts(ctx->fp, fb, ctx->test_cap, st);
    launch_debug_splats(sc, ctx->fp, fb, view, d, st);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = cudaMemcpy(out, d, sizeof(float) * 48 * ctx->N, cudaMemcpyDeviceToHost);
    cudaFree(d);
    CK(e);
    return VRS_OK;
}

vrs_status vrs_debug_tile_info(vrs_context* ctx, int32_t view, int32_t* cls, int32_t* vis, int64_t capacity) {
    if (!ctx) return VRS_E_INVALID_ARG;
    if (!ctx->have_frame || view < 0 || view >= ctx->fp.n_views) return fail(ctx, VRS_E_STATE, "no such view");
    const ViewParams& v = ctx->fp.v[view];
    const int64_t n = (int64_t)v.tw * v.th;
    if (capacity < n) return fail(ctx, VRS_E_INVALID_ARG, "capacity");
    CK(cudaStreamSynchronize(ctx->last_stream));
    if (cls) CK(cudaMemcpy(cls, v.cls, 4 * n, cudaMemcpyDeviceToHost));
    if (vis) CK(cudaMemcpy(vis, v.vis, 4 * n, cudaMemcpyDeviceToHost));
    return VRS_OK;
}

vrs_status vrs_sort_pairs(vrs_context* ctx, uint64_t* keys, uint32_t* vals, int64_t n, int32_t key_bits,
                          void* stream) {
    if (!ctx || (!keys && n > 0) || (!vals && n > 0)) return VRS_E_INVALID_ARG;
    if (n < 0 || n > ctx->cfg.max_pairs || key_bits < 1 || key_bits > 64)
        return fail(ctx, VRS_E_INVALID_ARG, "n or key_bits");
    if (n == 0) return VRS_OK;
    CK(cudaSetDevice(ctx->cfg.device));
    cudaStream_t st = (cudaStream_t)stream;
    uint32_t nn = (uint32_t)n;
    uint32_t* d_n = ctx->d_misc + 6;
    CK(cudaMemcpyAsync(d_n, &nn, 4, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    launch_sort(keys, vals, ctx->d_keys_alt, ctx->d_vals_alt, d_n, n, key_bits, ctx->sort, st, false);
    CK(cudaGetLastError());
    return VRS_OK;
}

vrs_status vrs_exclusive_scan(vrs_context* ctx, const uint32_t* in, uint32_t* out, uint32_t* total, int64_t n,
                              void* stream) {
    if (!ctx || !out || !total || (!in && n > 0)) return VRS_E_INVALID_ARG;
    if (n < 0 || n > (int64_t)ctx->cfg.max_views * std::max<int64_t>(ctx->cfg.max_gaussians, 1))
        return fail(ctx, VRS_E_INVALID_ARG, "n");
    CK(cudaSetDevice(ctx->cfg.device));
    launch_scan(in, out, total, nullptr, n, ctx->d_scan_scratch, (cudaStream_t)stream);
    CK(cudaGetLastError());
    return VRS_OK;
}

}  // extern "C"
