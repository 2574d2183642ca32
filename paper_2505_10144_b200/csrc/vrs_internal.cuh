// Internal definitions of libvrs (CUDA path).  Not shared with the oracle.
//
// Numerics: this library is compiled with -fmad=false and IEEE division /
// square root, so every float expression below rounds exactly like the
// operation order it is written in; FMAs appear only where fmaf() is written.
// That is what makes the decision quantities (culling, tile membership, sort
// keys, per-sample membership and order) bit-identical to the DESIGN.md
// "Numerics contract".
#pragma once
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <mutex>
#include <set>
#include <tuple>

#include "../../include/vrs.h"

namespace vrs {

constexpr int kBlend = 256;        // threads per blend block
constexpr int kWindow = 16;        // StopThePop per-sample resort window K
constexpr int kHierQueue = 8;      // N2 hierarchical mode: block queue K_B per 4x4 sample block
constexpr int kHierWindow = 8;     // N2 hierarchical mode: per-sample window K_P
constexpr int kHierGroup = 4;      // N2 hierarchical mode: queue K_G per 2x2 sample group
constexpr int kRecF4 = 8;          // float4 per projected-splat record (128 B)
constexpr float kO7Margin = 1.001f;  // O7 keep threshold factor (DESIGN R7)
constexpr float kTmin = 1e-4f;     // early termination (L11)
constexpr float kAlphaMax = 0.99f; // alpha clamp (L10)

enum TileClass : int32_t { kHigh = 0, kLow = 1, kHybrid = 2, kInvisible = 3 };
enum ItemKind : uint32_t { kItemFull = 0, kItemHybrid = 1, kItemLow = 2 };

// Per-view parameters, passed by value inside FrameParams.
struct ViewParams {
    float R[9];
    float o[3];
    float fx, fy, cx, cy;
    int32_t W, H;
    int32_t tw, th;          // assignment-tile grid
    int32_t tile_base;       // global tile id offset (views concatenated)
    int32_t fovea;           // foveation on
    float gx, gy, rx, ry, ramp;
    float plane[4][3];       // inward unit normals of the 4 frustum side planes (camera frame)
    double dplane[4][3];     // the same in double (preprocess cone test, O6a)
    double kinv[4];          // 1/fx, 1/fy, -cx/fx, -cy/fy in double (preprocess conic bbox, O6b)
    float dil;               // 0.3 / min(fx, fy)^2: dilation bound for the conservative cull
    int64_t pix_off;         // pixel offset of this view in the output buffers
    int64_t low_off;         // offset of this view in the low-res sample planes
    int32_t low_w;           // low-res plane width ((W+1)/2)
    int32_t n_items;         // blend work items of this view
    int32_t n_low;           // of which LowRes (they come first in items)
    int32_t item_off;        // first item of this view in the launch
    const int32_t* vis;      // [th*tw] visibility bits
    const uint32_t* sat;     // [(th+1)*(tw+1)] summed-area table
    const int32_t* cls;      // [th*tw] tile classes
    const uint32_t* items;   // [n_items] packed work items
    const uint32_t* inv_items;  // [n_inv] invisible coarse tiles (background fill items of the flat blend)
    int32_t n_inv;           // invisible tiles of this view
    int32_t inv_off;         // first invisible item of this view (after all views' blend items)
    float* xr;               // [tw+1] tile-corner rays ((float)min(kT, W) - cx) / fx (filled by k_cull)
    float* yr;               // [th+1] likewise in y
    uint32_t* lowcnt;        // [th*tw] LowRes tiles of the 3x3 neighbourhood still blending (in-launch compose)
    const uint32_t* lowcnt0; // [th*tw] its initial value (counters are re-armed by the composing block)
};

struct FrameParams {
    int32_t n_views;
    int32_t T;               // assignment tile size
    int32_t sh_coeffs;       // (deg+1)^2
    int32_t counters;        // instrumentation on
    int32_t no_cull;         // test hook: disable the warp-block footprint skip (P12)
    int32_t ewa;             // projection: 0 = Optimal Projection, 1 = EWA baseline (config C5)
    int32_t resort;          // 0 = per-sample window K = 16; 1 = hierarchical
    int32_t out_fmt;         // VRS_OUT_F32 or VRS_OUT_RGBA8_D16F (final output pixels)
    int32_t staging;         // blend staging of the splat records: VRS_STAGING_THREADS or VRS_STAGING_TMA
    int32_t sort_mode;       // VRS_SORT_STOPTHEPOP (per-tile key depth + window) or a global-sort baseline (N3)
    int32_t n_blend_items;   // blend items of all views (flat blend grid = n_blend_items + n_inv_items)
    int32_t n_inv_items;     // invisible-tile fill items of all views
    int64_t N;
    int64_t pair_cap;
    float near_plane;
    float bg[3];
    ViewParams v[VRS_MAX_VIEWS];
};

struct SceneDev {
    const float4* mu;        // [N] mu.xyz, q_cut (read for every Gaussian by the cull)
    const float4* geo;       // [N][4] Sigma_w (xx,xy,xz,yy) (yz,zz,sigma,s_max), Sigma_w^-1 (xx,xy,xz,yy)
                             // (yz,zz,0,0): the 64 B a candidate's projection reads, contiguous
    const float* smax;       // [N] largest scale (the cull's cone bound)
    const float4* sh;        // [N][chunks]
    int32_t sh_chunks;
};

struct FrameBufs {
    float4* rec;             // [V][N][8]
    uint32_t* cand;          // [V*N] (view*N + g) passing the conservative cull
    uint32_t* cand_count;    // [1]
    uint32_t* frustum_count; // [1] Gaussians with >= 1 candidate (step 1a statistic)
    unsigned long long* tv;  // [1] expanded tile tests (bits 0-35) | visible splats (bits 36-63), device
    unsigned long long* sidk;  // [test_cap] candidate -> (splat view*N+g) | (rect-local tile index << 32)
    uint32_t* vis_list;      // [V*N] (view*N + g) with >= 1 candidate tile (colour work list)

    uint32_t* counts;        // [V*N] exact pair counts (parity hook only)
    uint32_t* total;         // [1] pair total (device)
    uint32_t* overflow;      // [1] capacity overflow flag
    uint64_t* keys;          // [cap] emission keys
    uint32_t* vals;          // [cap]
    uint64_t* keys_alt;      // [cap] sort ping-pong
    uint32_t* vals_alt;
    uint32_t* ranges;        // [tiles][2]
    float4* col;             // [V][N] view-dependent colour (rgb, 0) of projected splats
    float4* low_rgba;        // low-res samples RGBA
    float* low_depth;        // low-res samples depth
    unsigned long long* stats;  // [8] device counters
};

constexpr int kTvShift = 36;
constexpr unsigned long long kTvMask = (1ull << kTvShift) - 1ull;
__device__ __forceinline__ int64_t fb_tests(const FrameBufs& fb) { return (int64_t)(*fb.tv & kTvMask); }
__device__ __forceinline__ uint32_t fb_visible(const FrameBufs& fb) { return (uint32_t)(*fb.tv >> kTvShift); }

// ----------------------------------------------------------------- device helpers (host side)
// Dynamic shared-memory limit of a kernel, set once per (kernel, device, size):
// the attribute is per device, and contexts on several devices may share a process.
inline void ensure_smem_attr(const void* func, int bytes) {
    static std::mutex mu;
    static std::set<std::tuple<const void*, int, int>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    if (done.insert(std::make_tuple(func, dev, bytes)).second)
        cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}
// SM count of the current device (cached per device).
inline int device_sms() {
    static int cache[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cache[dev]) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        cache[dev] = n > 0 ? n : 148;
    }
    return cache[dev];
}

// ----------------------------------------------------------------- launchers
// n_items_dev[0] = items, n_items_dev[1] = LowRes items (listed first),
// n_items_dev[2] = invisible tiles (listed in inv_items); lowcnt / lowcnt0 get the
// in-launch compose counters (LowRes tiles of each LowRes tile's 3x3 neighbourhood).
void launch_setup_view(const uint8_t* mask, int mask_w, ViewParams vp, int T, int32_t* vis, uint32_t* sat,
                       int32_t* cls, uint32_t* items, int32_t* n_items_dev, uint32_t* inv_items, uint32_t* lowcnt,
                       uint32_t* lowcnt0, cudaStream_t st);
// Cull + preprocess + candidate expansion into fb.sidk (total in fb.tv).
void launch_preprocess(const SceneDev& sc, const FrameParams& fp, FrameBufs fb, int64_t test_cap, cudaStream_t st);
// SH colour of the visible list (after launch_preprocess; needed by the blend only)
void launch_color(const SceneDev& sc, const FrameParams& fp, FrameBufs fb, cudaStream_t st);
// Exclusive scan of n = min(*n_dev, cap) u32 (n_dev may be null: n = cap); *total = sum.
// out may be null.  expand (optional): for element e with count c at offset o,
// expand[o + j] = e | (j << 32) for j < c (and o + j < expand_cap).
void launch_scan(const uint32_t* in, uint32_t* out, uint32_t* total, const uint32_t* n_dev, int64_t cap,
                 uint32_t* scratch, cudaStream_t st, unsigned long long* expand = nullptr,
                 int64_t expand_cap = 0);
size_t scan_scratch_words(int64_t n);
// Binned per-tile sort (k_binsort.cu): tile test -> per-tile buckets (direct
// slots up to kTileCap, overflow list beyond), look-back tile-count scan ->
// ranges (+ overflow offsets, pair total), overflow placement, per-tile sort
// of (depth bits, g) -> sorted (keys, vals).  cap_smem: largest tile sorted in
// shared memory (power of two <= kBinCap); bigger tiles merge in global memory.
constexpr uint32_t kBinCap = 4096;   // shared-memory sort capacity (32 KB of u64 keys)
constexpr uint32_t kTileCap = 1024;  // direct bucket slots per tile
struct BinScratch {
    uint32_t* tile_cnt;      // [max tiles] per-tile pair counters (kept zero between frames)
    uint64_t* tbucket;       // [max tiles][kTileCap] (depth bits << 32 | g) in arrival order
    uint32_t* ovf_off;       // [max tiles] exclusive scan of max(0, count - kTileCap)
    uint64_t* obucket;       // [cap] overflow pairs placed per tile
    uint32_t* ovf_count;     // [1] overflow list length (list in keys_alt / vals_alt / rank)
    uint32_t* rank;          // [cap] overflow entry's rank inside its tile
    uint32_t* list;          // [max tiles] non-empty tiles: big ones from the front, small from the back
    uint32_t* list_n;        // [3] (big, small, small-tile work counter)
    unsigned long long* scan_stat;  // [4 * ceil(max tiles / 1024)] k_tile_scan look-back words (zero between frames)
    uint32_t* scan_ctr;      // [2] k_tile_scan chunk ticket, finished blocks (zero between frames)
    int64_t max_tiles;
    uint32_t cap_smem;
};
// Fused Eq.4 tests + keys: frame path into the per-tile buckets ...
void launch_tiletest_direct(const FrameParams& fp, FrameBufs fb, int64_t test_cap, const BinScratch& bs,
                            cudaStream_t st);
// ... or (parity hook) compacted into (keys, vals) in arbitrary block order.
void launch_tiletest(const FrameParams& fp, FrameBufs fb, int64_t test_cap, uint64_t* keys, uint32_t* vals,
                     uint32_t* counter, cudaStream_t st);
void launch_counts(const FrameParams& fp, FrameBufs fb, int64_t test_cap, cudaStream_t st);
struct SortScratch {
    uint32_t* hist;          // [8][256] digit histograms (may be filled by k_compact)
    uint32_t* status;        // [max_tiles][256] u64 epoch-tagged look-back words
    uint32_t* counters;      // [8]
    uint32_t* epoch;         // host-side pass counter (tags status words; no per-pass memset)
    int64_t max_tiles;
};
size_t sort_status_words(int64_t cap);
// Sort n_dev (device count, capped at cap) pairs by key bits [0, key_bits); result in (keys, vals).
void launch_sort(uint64_t* keys, uint32_t* vals, uint64_t* keys_alt, uint32_t* vals_alt, const uint32_t* n_dev,
                 int64_t cap, int key_bits, SortScratch s, cudaStream_t st, bool hist_ready);
void launch_binsort(FrameBufs fb, int64_t cap, int64_t n_tiles, BinScratch b, cudaStream_t st);
void launch_ranges(const uint64_t* keys, const uint32_t* n_dev, int64_t cap, uint32_t* ranges, int64_t n_tiles,
                   cudaStream_t st);
// Two-pass foveated baseline (k_twopass.cu).
struct TwoPassView {
    int32_t W, H;            // output view
    int32_t i0, j0, w1, h1;  // pass-1 rectangle (full resolution)
    int32_t W2, H2;          // pass-2 (half resolution) size
    int64_t out_off, p1_off, p2_off;  // pixel offsets: output, pass-1 image, pass-2 image
    float gx, gy, rx, ry, ramp;       // fovea (blend weight)
};
struct TwoPassParams {
    int32_t n;
    int32_t out_fmt;
    TwoPassView v[VRS_MAX_VIEWS];
};
void launch_mask_half(const uint8_t* src, int W, int H, uint8_t* dst, int W2, int H2, cudaStream_t st);
void launch_two_pass_combine(const TwoPassParams& tp, const float4* prgba, const float* pdepth, float* rgba,
                             float* depth, int64_t total, cudaStream_t st);  // writes tp.out_fmt
// The whole blend of a frame: flat mode = one k_blend launch (blend items, invisible
// fills and the periphery compose); hierarchical mode = k_blend_hier + k_compose.
void launch_blend(const FrameParams& fp, FrameBufs fb, int total_items, float* rgba, float* depth,
                  cudaStream_t st);
void launch_blend_hier(const FrameParams& fp, FrameBufs fb, int total_items, float* rgba, float* depth,
                       cudaStream_t st);
// N4 backward (k_backward.cu): gbuf [V][N][24] must be zero, outputs zeroed by the caller.
void launch_backward(const FrameParams& fp, FrameBufs fb, int total_items, const float4* mu4, const float4* raw,
                     const float* sh, int sh_stride, const float* f_rgba, const float* f_depth,
                     const float* g_rgba, const float* g_depth, float* gbuf, float* g_means, float* g_quats,
                     float* g_ls, float* g_logits, float* g_sh, cudaStream_t st);
void launch_compose(const FrameParams& fp, FrameBufs fb, float* rgba, float* depth, cudaStream_t st);
void launch_debug_splats(const SceneDev& sc, const FrameParams& fp, FrameBufs fb, int view, float* out,
                         cudaStream_t st);

// ----------------------------------------------------------------- numerics (contract R6)
__device__ __forceinline__ float dot3(float ax, float ay, float az, float bx, float by, float bz) {
    return fmaf(ax, bx, fmaf(ay, by, az * bz));
}
// d^T Q d with pre-doubled coefficients (a,b,c,p,e,f) = (Q00,2Q01,Q11,2Q02,2Q12,Q22)
__device__ __forceinline__ float quad3(float a, float b, float c, float p, float e, float f, float x, float y,
                                       float z) {
    return fmaf(fmaf(a, x, fmaf(b, y, p * z)), x, fmaf(fmaf(c, y, e * z), y, (f * z) * z));
}
// z = 1 specialisation (bit-identical: p*1, e*1, f*1*1 are exact)
// Conservative pixel footprint of a projected splat (record slot 7, written by
// k_preprocess): x = its bounding box's columns as int16 (min | max << 16,
// rounded outward), y = rows likewise, z = a separating axis n across the
// ellipse (binary16 pair: its minor axis), w = binary16 pair (d, hw): the
// offset of the ellipse centre from the box centre along n and the ellipse's
// half-width along n, rounded up, with a 1 px margin (the margin of the box).
// A block of samples whose box or whose extent along n misses it holds no
// member sample (the hierarchical culling of P:431: never changes results).
struct Footprint {
    float bcx, bcy, ex, ey, nx, ny, k, e;
};
// hx, hy: half-extent of the sample blocks it will be tested against
__device__ __forceinline__ Footprint footprint_of(const float4 a7, const float hx, const float hy) {
    const uint32_t bx = __float_as_uint(a7.x), by = __float_as_uint(a7.y);
    const float x0 = (float)(int)(short)(bx & 0xffffu), x1 = (float)(int)(short)(bx >> 16);
    const float y0 = (float)(int)(short)(by & 0xffffu), y1 = (float)(int)(short)(by >> 16);
    const __half2 n = *reinterpret_cast<const __half2*>(&a7.z), dh = *reinterpret_cast<const __half2*>(&a7.w);
    Footprint f;
    f.bcx = 0.5f * (x0 + x1);
    f.bcy = 0.5f * (y0 + y1);
    f.ex = fmaf(0.5f, x1 - x0, hx);
    f.ey = fmaf(0.5f, y1 - y0, hy);
    f.nx = __low2float(n);
    f.ny = __high2float(n);
    f.k = fmaf(f.nx, f.bcx, fmaf(f.ny, f.bcy, __low2float(dh)));
    f.e = __high2float(dh) + fmaf(hx, fabsf(f.nx), hy * fabsf(f.ny));
    return f;
}
// wb = (centre x, centre y, half-extent x, half-extent y) of a sample block
__device__ __forceinline__ bool footprint_hits(const Footprint& f, const float4 wb) {
    return fabsf(f.bcx - wb.x) <= f.ex && fabsf(f.bcy - wb.y) <= f.ey &&
           fabsf(fmaf(f.nx, wb.x, fmaf(f.ny, wb.y, -f.k))) <= f.e;
}
// bit w set iff the footprint meets sample block wblock[w] (all of one size)
template <int kBlocks>
__device__ __forceinline__ uint32_t footprint_mask(const float4 a7, const float4* wblock) {
    const float4 w0 = wblock[0];
    const Footprint f = footprint_of(a7, w0.z, w0.w);
    uint32_t m = 0;
#pragma unroll
    for (int w = 0; w < kBlocks; w++) m |= footprint_hits(f, wblock[w]) ? (1u << w) : 0u;
    return m;
}

__device__ __forceinline__ float quad3z1(float a, float b, float c, float p, float e, float f, float x, float y) {
    return fmaf(fmaf(a, x, fmaf(b, y, p)), x, fmaf(fmaf(c, y, e), y, f));
}

// Final output pixel i in the context's output format (vrs_set_output_format):
// VRS_OUT_F32 = float4 RGBA + float depth; VRS_OUT_RGBA16F_D32F = RGBA IEEE
// binary16 (round to nearest) + float depth; VRS_OUT_RGBA8_D16F = RGBA unorm8
// (round to nearest of clamp(v, 0, 1) * 255) + depth IEEE binary16 (round to
// nearest).  rgba / depth point to the caller's buffers of that format.
__device__ __forceinline__ unsigned char unorm8(float v) {
    return (unsigned char)__float2uint_rn(fminf(fmaxf(v, 0.0f), 1.0f) * 255.0f);
}
__device__ __forceinline__ void store_pixel(int fmt, float* rgba, float* depth, size_t i, float4 c, float d) {
    if (fmt == VRS_OUT_F32) {
        reinterpret_cast<float4*>(rgba)[i] = c;
        depth[i] = d;
    } else if (fmt == VRS_OUT_RGBA16F_D32F) {  // RGBA binary16 + float depth (within the parity tolerances)
        const __half2 rg = __floats2half2_rn(c.x, c.y), ba = __floats2half2_rn(c.z, c.w);
        reinterpret_cast<uint2*>(rgba)[i] =
            make_uint2(*reinterpret_cast<const uint32_t*>(&rg), *reinterpret_cast<const uint32_t*>(&ba));
        depth[i] = d;
    } else {
        reinterpret_cast<uchar4*>(rgba)[i] = make_uchar4(unorm8(c.x), unorm8(c.y), unorm8(c.z), unorm8(c.w));
        reinterpret_cast<__half*>(depth)[i] = __float2half_rn(d);
    }
}

// Blend weight of the fovea ramp at a pixel centre (P:461
// "10% padding of linearly increasing blending weights").
__device__ __forceinline__ float fovea_weight(const ViewParams& v, float px, float py) {
    float ax = fabsf(px - v.gx) - v.rx;
    float ay = fabsf(py - v.gy) - v.ry;
    ax = ax > 0.0f ? ax : 0.0f;
    ay = ay > 0.0f ? ay : 0.0f;
    float dxn = v.ramp * (2.0f * v.rx);
    float dyn = v.ramp * (2.0f * v.ry);
    float wx = dxn > 0.0f ? ax / dxn : (ax > 0.0f ? 1.0f : 0.0f);
    float wy = dyn > 0.0f ? ay / dyn : (ay > 0.0f ? 1.0f : 0.0f);
    float m = wx > wy ? wx : wy;
    float w = 1.0f - m;
    return w < 0.0f ? 0.0f : (w > 1.0f ? 1.0f : w);
}

}  // namespace vrs
