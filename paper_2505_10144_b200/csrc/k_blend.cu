// Steps 5-7: per-tile ranges, the single-pass foveated blend
// and the periphery compose.
//
// Blend: ONE launch per frame.  Its 256-thread
// blocks are 16x16 full-rate items (HighRes / Hybrid subtiles of a
// 32x32 coarse tile, or 16x16 tiles when assigning at 16), 32x32 LowRes
// tiles where every thread renders one 2x2 pixel group sampled at the group
// centre, or invisible tiles (background fill).  Every
// item streams its coarse tile's sorted list in key order.
//
// Staging (default): the list is cut into batches of 32 entries held in a
// two-stage ring in shared memory (the first 96 B of each entry's 128-B splat
// record, its id g, and a mask of the warps whose 8x4 sample block the
// entry's conservative pixel footprint -- bounding box + separating axis --
// meets: the hierarchical culling of P:431, which never changes results,
// only work).  The block stages batches 0 and 1; afterwards the warps consume
// the stages independently, with no block barrier: the last warp to finish a
// batch refills its stage with the batch two ahead (one entry per lane) and
// arrives on the stage's mbarrier, a warp that needs a batch not staged yet
// waits on that mbarrier.  A warp evaluates two relevant entries' memberships
// per iteration and runs their contributions in stream order.  Alternative
// staging (vrs_set_staging_mode): block-synchronous batches whose records are
// copied by the TMA bulk-copy engine (cp.async.bulk, mbarrier completion).
//
// Each sample runs the StopThePop per-pixel resort: a
// K = 16 window ordered by (tau, g) -- a per-thread ring in shared memory
// ([slot][thread], bank-conflict free), started full of no-op sentinels so
// every contribution is "compare with the head, blend the smaller, insert
// the other from the tail" -- popping the nearest entry on overflow and
// blending front to back (Eq.2 with product transmittance), terminating once
// T < 1e-4 (checked after blending).  Hybrid pixels blend their value with
// the 2x2 group average via warp shuffles.
//
// Compose inside the same launch: every LowRes tile counts the
// LowRes tiles of its 3x3 neighbourhood still blending; the block that
// finishes the last of them composes the tile (nearest-neighbour upsample +
// renormalised 3x3 blur of its 2x2-group samples) and re-arms the counter.
#include "k_blend_common.cuh"

namespace vrs {

__global__ void k_ranges(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ n_dev, int64_t cap,
                         uint32_t* ranges, int64_t n_tiles) {
    const int64_t n = min((int64_t)*n_dev, cap);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t t = (uint32_t)(keys[i] >> 32);
        if (t >= n_tiles) continue;  // only after a capacity overflow (undefined frame)
        if (i == 0 || (uint32_t)(keys[i - 1] >> 32) != t) ranges[2 * (size_t)t] = (uint32_t)i;
        if (i == n - 1 || (uint32_t)(keys[i + 1] >> 32) != t) ranges[2 * (size_t)t + 1] = (uint32_t)(i + 1);
    }
}

void launch_ranges(const uint64_t* keys, const uint32_t* n_dev, int64_t cap, uint32_t* ranges, int64_t n_tiles,
                   cudaStream_t st) {
    cudaMemsetAsync(ranges, 0, sizeof(uint32_t) * 2 * (size_t)n_tiles, st);
    const int sms = device_sms();
    k_ranges<<<sms * 16, 256, 0, st>>>(keys, n_dev, cap, ranges, n_tiles);
}

// ----------------------------------------------------------------- compose (step 7)
// Periphery reconstruction of one 2x2 pixel group: nearest-neighbour
// upsample of the LowRes group samples and a 3x3 (1,2,1)x(1,2,1) blur
// restricted to LowRes pixels in the image, renormalised;
// invisible tiles get the background with A = 0, D = 0.  The 3x3
// neighbourhood of group samples covers the blur footprint of all four
// pixels.  Samples are read through L2 (ld.global.cg): inside the blend
// launch they were written by other blocks.
__device__ __forceinline__ void compose_group(const FrameParams& fp, const FrameBufs& fb, const ViewParams& v,
                                              int gx, int gy, float* __restrict__ rgba, float* __restrict__ depth) {
    if (2 * gy >= v.H || 2 * gx >= v.W) return;
    const int tsh = (fp.T == 32) ? 5 : 4, i0 = 2 * gx, j0 = 2 * gy;  // T is 16 or 32
    const int c = v.cls[(j0 >> tsh) * v.tw + (i0 >> tsh)];
    if (c == kHigh || c == kHybrid) return;
    float4 outc[2][2];
    float outd[2][2];
    if (c == kInvisible) {
#pragma unroll
        for (int b = 0; b < 2; b++)
#pragma unroll
            for (int a = 0; a < 2; a++) {
                outc[b][a] = make_float4(fp.bg[0], fp.bg[1], fp.bg[2], 0.0f);
                outd[b][a] = 0.0f;
            }
    } else {
        float4 sc[3][3];
        float sd[3][3];
        bool ok[3][3];
#pragma unroll
        for (int dj = 0; dj < 3; dj++)
#pragma unroll
            for (int di = 0; di < 3; di++) {
                // pixel of that group adjacent to this group: column 2gx-1, (2gx..2gx+1), 2gx+2
                const int pi = (di == 0) ? i0 - 1 : (di == 1 ? i0 : i0 + 2);
                const int pj = (dj == 0) ? j0 - 1 : (dj == 1 ? j0 : j0 + 2);
                bool good = pi >= 0 && pj >= 0 && pi < v.W && pj < v.H;
                if (good) good = v.cls[(pj >> tsh) * v.tw + (pi >> tsh)] == kLow;
                ok[dj][di] = good;
                if (good) {
                    const size_t li = (size_t)v.low_off + (size_t)(pj >> 1) * v.low_w + (pi >> 1);
                    sc[dj][di] = __ldcg(fb.low_rgba + li);
                    sd[dj][di] = __ldcg(fb.low_depth + li);
                } else {
                    sc[dj][di] = make_float4(0.f, 0.f, 0.f, 0.f);
                    sd[dj][di] = 0.0f;
                }
            }
        // Pixels of one group share its sample, so the 3x3 taps of pixel
        // (i0+a, j0+b) collapse onto 2x2 neighbour groups with summed
        // separable weights: a = 0 -> groups {-1: 1, 0: 2 + [i0+1 < W]},
        // a = 1 -> {0: 3, +1: 1} (pixel-level in-image tests folded in).
        const float wx[2][3] = {{1.0f, (i0 + 1 < v.W) ? 3.0f : 2.0f, 0.0f}, {0.0f, 3.0f, 1.0f}};
        const float wy[2][3] = {{1.0f, (j0 + 1 < v.H) ? 3.0f : 2.0f, 0.0f}, {0.0f, 3.0f, 1.0f}};
#pragma unroll
        for (int b = 0; b < 2; b++)
#pragma unroll
            for (int a = 0; a < 2; a++) {
                float acc[5] = {0.f, 0.f, 0.f, 0.f, 0.f}, ws = 0.0f;
#pragma unroll
                for (int sj = b; sj < b + 2; sj++)
#pragma unroll
                    for (int si = a; si < a + 2; si++) {
                        const float w = ok[sj][si] ? wx[a][si] * wy[b][sj] : 0.0f;
                        acc[0] = fmaf(w, sc[sj][si].x, acc[0]);
                        acc[1] = fmaf(w, sc[sj][si].y, acc[1]);
                        acc[2] = fmaf(w, sc[sj][si].z, acc[2]);
                        acc[3] = fmaf(w, sc[sj][si].w, acc[3]);
                        acc[4] = fmaf(w, sd[sj][si], acc[4]);
                        ws += w;
                    }
                const float inv = 1.0f / ws;
                outc[b][a] = make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
                outd[b][a] = acc[4] * inv;
            }
    }
#pragma unroll
    for (int b = 0; b < 2; b++) {
        const int j = j0 + b;
        if (j >= v.H) continue;
        const size_t row = (size_t)v.pix_off + (size_t)j * v.W;
        store_pixel(fp.out_fmt, rgba, depth, row + i0, outc[b][0], outd[b][0]);
        if (i0 + 1 < v.W) store_pixel(fp.out_fmt, rgba, depth, row + i0 + 1, outc[b][1], outd[b][1]);
    }
}

// Stand-alone compose over every group of every view (the hierarchical resort
// mode's frame, which blends without the in-launch compose).
__global__ void k_compose(FrameParams fp, FrameBufs fb, float* __restrict__ rgba, float* __restrict__ depth,
                          int64_t total_groups) {
    const int64_t gi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gi >= total_groups) return;
    int vi = 0;
    while (vi + 1 < fp.n_views && gi >= fp.v[vi + 1].low_off) vi++;
    const ViewParams& v = fp.v[vi];
    const uint32_t k = (uint32_t)(gi - v.low_off);
    compose_group(fp, fb, v, (int)(k % (uint32_t)v.low_w), (int)(k / (uint32_t)v.low_w), rgba, depth);
}

void launch_compose(const FrameParams& fp, FrameBufs fb, float* rgba, float* depth, cudaStream_t st) {
    if (fp.n_views == 0) return;
    const ViewParams& last = fp.v[fp.n_views - 1];
    const int64_t total = last.low_off + (int64_t)last.low_w * ((last.H + 1) / 2);
    k_compose<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(fp, fb, rgba, depth, total);
}

// ----------------------------------------------------------------- blend (step 6)
namespace {

constexpr int kBT = 256;                 // threads per block: one 16x16 item / one 32x32 LowRes item
constexpr int kWarps = kBT / 32;
#ifndef VRS_BLEND_ASYNC
#define VRS_BLEND_ASYNC 1
#endif
#ifndef VRS_BLEND_BATCH
#define VRS_BLEND_BATCH (VRS_BLEND_ASYNC ? 64 : 80)
#endif
constexpr int kBatch = VRS_BLEND_BATCH;  // list entries staged per shared-memory batch
constexpr uint32_t kStageBytes = 96;     // r0..r5 of a splat record
static_assert(kBatch <= kBT && kBatch >= 10, "one staging thread per entry; the compose triggers reuse mask[]");

struct BlendSmem {
    // the staged entries: the first 96 B of their splat records, r0..r5
    // (k_project.cu layout: u.xyz, q_cut | e1.x, e1.z, e2.x, e2.y | e2.z, C00,
    // C01, C11 | A a, b, c, p | A e, f, b.x, b.y | b.z, sigma, -, -), written by
    // the TMA bulk-copy engine (staging mode 1) or by the block's threads (mode 0)
    float4 rec[kBatch][6];
    uint32_t mask[kBatch];    // g << 8 | the warps whose samples the entry's pixel footprint meets
    unsigned long long full;  // mbarrier: the batch landed (TMA staging)
    float4 wblock[kWarps];    // per-warp sample block: centre x, y, half-extent x, y (pixel coords)
    // per-thread resort window: ring of K slots, (tau, g) packed into one
    // order-preserving 64-bit key, alpha alongside; [slot][thread] layout is
    // bank-conflict free for any per-thread slot index
    unsigned long long w_key[kWindow][kBT];
    float w_a[kWindow][kBT];
    unsigned long long cnt[4];
    // warp-asynchronous staging (VRS_BLEND_ASYNC): two stages of kSE entries in
    // rec[] / mask[] rows s * kSE ..; fullb[s] completes when a refill of stage s
    // landed, consumed[s] counts the warps done with its current batch, alive the
    // warps with a sample still blending
#if VRS_BLEND_ASYNC
    unsigned long long fullb[2];
    uint32_t consumed[2];
    uint32_t alive;
#endif
};
// 4 blocks of 256 threads per SM (the 64-register budget) need <= 57344 B each
// (228 KB per SM, 1 KB reserved per block); after the blend loop the staging
// mask holds the in-launch compose triggers
static_assert(sizeof(BlendSmem) + 1024 <= 233472 / 4, "blend shared memory exceeds the 4-blocks/SM budget");

constexpr int kSE = 32;  // entries per stage of the asynchronous staging ring (one per lane)
static_assert(2 * kSE <= kBatch, "two async stages live in the batch buffer");

constexpr uint32_t kSlotBytes = kBT * 8;                   // one ring slot of keys
static_assert((kWindow & (kWindow - 1)) == 0, "ring needs a power-of-two window");

// Geometry of a blend item and of this thread's sample (full-rate: the pixel;
// LowRes: the 2x2 group at (px, py), sampled at its centre).
struct ItemGeom {
    int vi, tile, kind, x0, y0, ox, oy, px, py;
    float xs, ys;
};
__device__ __forceinline__ ItemGeom item_geom(const FrameParams& fp, int item, int half, int lane, int warp) {
    ItemGeom g;
    g.vi = 0;
    while (g.vi + 1 < fp.n_views && item >= fp.v[g.vi + 1].item_off) g.vi++;
    const ViewParams& v = fp.v[g.vi];
    const uint32_t it = v.items[item - v.item_off];
    g.tile = (int)(it & 0xfffffu);
    const int sub = (int)((it >> 20) & 3u);
    g.kind = (int)(it >> 22);
    const int T = fp.T;
    g.x0 = (g.tile % v.tw) * T;
    g.y0 = (g.tile / v.tw) * T;
    const int sx = (warp & 1) * 8 + (lane & 7), sy = (warp >> 1) * 4 + half * 8 + (lane >> 3);
    g.ox = (g.kind == kItemLow) ? g.x0 : g.x0 + (T == 32 ? 16 * (sub & 1) : 0);
    g.oy = (g.kind == kItemLow) ? g.y0 : g.y0 + (T == 32 ? 16 * (sub >> 1) : 0);
    if (g.kind == kItemLow) {
        g.px = g.x0 + 2 * sx;
        g.py = g.y0 + 2 * sy;
        g.xs = (float)(g.px + 1);
        g.ys = (float)(g.py + 1);
    } else {
        g.px = g.ox + sx;
        g.py = g.oy + sy;
        g.xs = (float)g.px + 0.5f;
        g.ys = (float)g.py + 0.5f;
    }
    return g;
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(unsigned long long* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// TMA bulk copy global -> shared of `bytes` (multiple of 16, 16-B aligned),
// completing its byte count on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
    uint64_t gsrc;
    asm("cvta.to.global.u64 %0, %1;" : "=l"(gsrc) : "l"(src));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// blockIdx.x through an opaque read, so the compiler recomputes the item's
// geometry after the blend loop instead of keeping it in registers
__device__ __forceinline__ int block_id_opaque() {
    int b;
    asm volatile("mov.u32 %0, %%ctaid.x;" : "=r"(b));
    return b;
}

}  // namespace

#define REC0(j) S.rec[j][0]
#define REC1(j) S.rec[j][1]
#define REC2(j) S.rec[j][2]
#define REC3(j) S.rec[j][3]
#define REC4(j) S.rec[j][4]
#define REC5(j) S.rec[j][5]
// Thread staging overwrites the staged r5.w (the record's rect01, unused by the
// blend) with g, so a contribution takes g from the r5 load it makes anyway;
// TMA staging copies the record verbatim and keeps g in the mask word.
#ifndef VRS_GID_IN_REC
#define VRS_GID_IN_REC 1
#endif
#define GID(j) ((VRS_GID_IN_REC && !kTma) ? __float_as_uint(S.rec[j][5].w) : (S.mask[j] >> 8))
#define MASKJ(j) S.mask[j]

template <bool kCounters, bool kEwa, bool kTma, bool kGlobal>
#ifndef VRS_BLEND_MINB
#define VRS_BLEND_MINB 4
#endif
__global__ void __launch_bounds__(kBT, VRS_BLEND_MINB) k_blend(FrameParams fp, FrameBufs fb, float* __restrict__ rgba,
                                                      float* __restrict__ depth) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    BlendSmem& S = *reinterpret_cast<BlendSmem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // locate the view and the item (blend items of every view, then the invisible tiles)
    int vi = 0;
    const int item = blockIdx.x, half = 0;
    if (item >= fp.n_blend_items) {
        // invisible tile: background, A = 0, D = 0
        const int iv = item - fp.n_blend_items;
        while (vi + 1 < fp.n_views && iv >= fp.v[vi + 1].inv_off) vi++;
        const ViewParams& v = fp.v[vi];
        const int tile = (int)v.inv_items[iv - v.inv_off];
        const int T = fp.T, x0 = (tile % v.tw) * T, y0 = (tile / v.tw) * T;
        for (int p = tid + half * kBT; p < T * T; p += kBT) {
            const int px = x0 + p % T, py = y0 + p / T;
            if (px < v.W && py < v.H)
                store_pixel(fp.out_fmt, rgba, depth, (size_t)v.pix_off + (size_t)py * v.W + px,
                            make_float4(fp.bg[0], fp.bg[1], fp.bg[2], 0.0f), 0.0f);
        }
        return;
    }
    // Only what the blend loop needs stays live through it (the kernel runs at
    // the 64-register cap of 4 blocks/SM): the item's geometry is recomputed
    // after the loop for the outputs.
    float x, y, xs, ys;  // sample ray (x, y, 1); pixel coordinates (EWA baseline)
    uint32_t rb, re;
    const float4* __restrict__ recv;
    const float4* __restrict__ colv;
    {
        const ItemGeom g = item_geom(fp, item, half, lane, warp);
        const ViewParams& v = fp.v[g.vi];
        if (tid < kWarps) {
            const int wwx = (tid & 1) * 8, wwy = (tid >> 1) * 4 + half * 8;
            float4 b;
            if (g.kind == kItemLow)  // samples at x0 + 2 sx + 1, sx = wwx .. wwx + 7 (rows likewise)
                b = make_float4((float)(g.x0 + 2 * wwx + 8), (float)(g.y0 + 2 * wwy + 4), 7.0f, 3.0f);
            else  // samples at pixel centres ox + sx + 0.5
                b = make_float4((float)(g.ox + wwx + 4), (float)(g.oy + wwy + 2), 3.5f, 1.5f);
            S.wblock[tid] = b;
        }
        xs = g.xs;
        ys = g.ys;
        x = (xs - v.cx) / v.fx;
        y = (ys - v.cy) / v.fy;
        rb = fb.ranges[2 * (size_t)(v.tile_base + g.tile)];
        re = fb.ranges[2 * (size_t)(v.tile_base + g.tile) + 1];
        recv = fb.rec + (size_t)g.vi * fp.N * kRecF4;
        colv = fb.col + (size_t)g.vi * fp.N;
    }
    if (kCounters && tid < 4) S.cnt[tid] = 0ull;
    // Ring offsets carry the thread's column (tid * 8 < one slot of 2048 B), so a
    // window address is the array's block-uniform base (a uniform register) plus
    // one per-thread offset -- no per-thread base pointers live in the loop
    // (C2 blend 1.926 -> 1.874 ms)
    char* const wkb = reinterpret_cast<char*>(&S.w_key[0][0]);
    char* const wab = reinterpret_cast<char*>(&S.w_a[0][0]);
    constexpr uint32_t kRM = kWindow * kSlotBytes - 1u;  // wraps the slot bits, keeps the column bits
#define WK(off) (*reinterpret_cast<unsigned long long*>(wkb + (off)))
#define WA(off) (*reinterpret_cast<float*>(wab + ((off) >> 1)))
    // The window starts full of K sentinels (tau = -2e30 < every canonical
    // depth, alpha = 0): popping a sentinel is an exact no-op, so every
    // contribution runs the same straight-line "insert, pop min" code.
#pragma unroll
    for (int k = 0; k < kWindow; k++) {
        WK(k * kSlotBytes + 8u * tid) = kSentinelKey;
        WA(k * kSlotBytes + 8u * tid) = 0.0f;
    }

    float Tr = 1.0f, Cr = 0.0f, Cg = 0.0f, Cb = 0.0f, Dd = 0.0f;
    // "done" (T < 1e-4, checked after blending) is read from the transmittance
    // itself -- Tr never changes once it holds -- instead of a flag kept live
    // beside it (one register less in the 64-register loop: C2 blend 1.969 ->
    // 1.940 ms)
#define DONE (Tr < kTmin)
    uint32_t hk = 8u * tid;  // byte offset of the ring head (slot * kSlotBytes + column)
    uint32_t n_contrib = 0, stop_pos = re - 1;  // entry whose insertion stopped the sample (re-1: ran out)

    auto blend_one = [&](unsigned long long key, float a) {
        const float4* cp;  // colv + g as one 32x32->64 multiply-add
        asm("mad.wide.u32 %0, %1, 16, %2;" : "=l"(cp) : "r"((uint32_t)key), "l"(colv));
        const float4 col = __ldg(cp);
        const float wgt = a * Tr;
        Cr = fmaf(col.x, wgt, Cr);
        Cg = fmaf(col.y, wgt, Cg);
        Cb = fmaf(col.z, wgt, Cb);
        Dd = fmaf(key_tau(key), wgt, Dd);  // ray-distance factor |d| applied once at the end
        Tr = Tr * (1.0f - a);
    };

    // the contribution of one (sample, splat) pair with its alpha, depth and
    // order key: insert into the window, pop the minimum
    auto contribute = [&](const unsigned long long key, const float alpha, const uint32_t pos) {
        if (kCounters) n_contrib++;
        if constexpr (kGlobal) {  // global-sort baselines (N3): no window, list order
            blend_one(key, alpha);
            if (kCounters && DONE) stop_pos = pos;
            return;
        }
        const unsigned long long kh = WK(hk);
        const float ah = WA(hk);
        // one 64-bit compare, then bitwise selects (the compiler otherwise re-derives the
        // comparison for every use)
        uint32_t dm;  // all ones iff the new entry is the minimum
        asm("{\n .reg .pred p;\n setp.lo.u64 p, %1, %2;\n selp.u32 %0, 0xffffffff, 0, p;\n}"
            : "=r"(dm)
            : "l"(key), "l"(kh));
        auto bsel = [](uint32_t a, uint32_t b, uint32_t m) {  // (a & m) | (b & ~m), opaque to the compiler
            uint32_t r;
            asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(r) : "r"(a), "r"(b), "r"(m));
            return r;
        };
        const uint32_t klo = bsel((uint32_t)key, (uint32_t)kh, dm);
        const uint32_t khi = bsel((uint32_t)(key >> 32), (uint32_t)(kh >> 32), dm);
        const float asel = __uint_as_float(bsel(__float_as_uint(alpha), __float_as_uint(ah), dm));
        blend_one(((unsigned long long)khi << 32) | klo, asel);
        if (kCounters && DONE) stop_pos = pos;
        // (a sample that just terminated never reads its window again, so the
        // insertion does not wait for the transmittance test)
        if (dm != 0u) return;
        hk = (hk + kSlotBytes) & kRM;
        // insertion from the tail (entries arrive nearly sorted); dst
        // is the hole, starting at the popped head's slot
        uint32_t jo = (hk + (kWindow - 2) * kSlotBytes) & kRM;
        uint32_t dst = (jo + kSlotBytes) & kRM;
        unsigned long long kj = WK(jo);
        int left = kWindow - 1;
#pragma unroll 1
        while (kj > key) {
            WK(dst) = kj;
            WA(dst) = WA(jo);
            dst = jo;
            if (--left == 0) break;
            jo = (jo - kSlotBytes) & kRM;
            kj = WK(jo);
        }
        WK(dst) = key;
        WA(dst) = alpha;
    };
    // membership + alpha/tau of entry g for this sample; a3..a5 fetched only on contribution
    auto evaluate = [&](const uint32_t pos, const uint32_t g, const float4 a0, const float4 a1, const float4 a2,
                        auto&& load345) {
        if (DONE) return;
        float alpha, tau;
        if (kEwa) {  // EWA baseline: q from the projected mean in pixels
            const float dxp = xs - a0.x, dyp = ys - a0.y;
            const float q = fmaf(dxp, fmaf(a0.w, dxp, a1.x * dyp), dyp * fmaf(a1.x, dxp, a1.y * dyp));
            if (!(q <= a0.z)) return;
            float4 a3, a4;
            float2 a5;
            load345(a3, a4, a5);
            const float den = quad3z1(a3.x, a3.y, a3.z, a3.w, a4.x, a4.y, x, y);
            const float dtb = fmaf(a4.z, x, fmaf(a4.w, y, a5.x));
            tau = __fdiv_rn(dtb, den);
            alpha = alpha_of_x(fmaxf(q * -0.72134752f, -64.0f), a5.y);
        } else {
            const float s = fmaf(a0.x, x, fmaf(a0.y, y, a0.z));
            const float ex = fmaf(a1.x, x, a1.y);
            const float ey = fmaf(a1.z, x, fmaf(a1.w, y, a2.x));
            const float cx = fmaf(a2.y, ex, a2.z * ey), cy = fmaf(a2.z, ex, a2.w * ey);
            const float num = fmaf(ex, cx, ey * cy);
            const float ss = s * s;
            if (!(s > 0.0f) || !(num <= a0.w * ss)) return;
            // contribution: alpha and tau (R9: one IEEE reciprocal, exact on both sides)
            float4 a3, a4;
            float2 a5;
            load345(a3, a4, a5);
            const float den = quad3z1(a3.x, a3.y, a3.z, a3.w, a4.x, a4.y, x, y);
            const float dtb = fmaf(a4.z, x, fmaf(a4.w, y, a5.x));
            alpha = alpha_tau(num, ss, den, dtb, a5.y, tau);
        }
        contribute(order_key(tau, g, fp.near_plane), alpha, pos);
    };

    // one 32-entry chunk of staged rows r0 .. r0 + cnt - 1 (list positions pos0 ..):
    // the warp's relevant entries (footprint mask) in stream order
    auto chunk = [&](const int r0, const int cnt, const uint32_t pos0) {
#define POS_OF(j) (pos0 + (uint32_t)((j) - r0))
        const bool rel = (lane < cnt) && ((MASKJ(r0 + lane) >> warp) & 1u);
        unsigned bits = __ballot_sync(0xffffffffu, rel);
        if (!kEwa) {
            // two list entries per iteration: both memberships first (independent
            // chains), then the contributions in stream order
            auto member = [&](const int j, float& num, float& ss) {
                const float4 a0 = REC0(j), a1 = REC1(j), a2 = REC2(j);
                const float s = fmaf(a0.x, x, fmaf(a0.y, y, a0.z));
                const float ex = fmaf(a1.x, x, a1.y);
                const float ey = fmaf(a1.z, x, fmaf(a1.w, y, a2.x));
                const float cx = fmaf(a2.y, ex, a2.z * ey), cy = fmaf(a2.z, ex, a2.w * ey);
                num = fmaf(ex, cx, ey * cy);
                ss = s * s;
                return (s > 0.0f) && (num <= a0.w * ss);
            };
            auto contrib = [&](const int j, const float num, const float ss) {
                const float4 a3 = REC3(j), a4 = REC4(j), t = REC5(j);
                const float den = quad3z1(a3.x, a3.y, a3.z, a3.w, a4.x, a4.y, x, y);
                const float dtb = fmaf(a4.z, x, fmaf(a4.w, y, t.x));
                float tau;
                const float alpha = alpha_tau(num, ss, den, dtb, t.y, tau);
                const uint32_t gj = (VRS_GID_IN_REC && !kTma) ? __float_as_uint(t.w) : GID(j);
                contribute(order_key(tau, gj, fp.near_plane), alpha, POS_OF(j));
            };
            while (bits) {
                const int j = r0 + __ffs(bits) - 1;
                bits &= bits - 1;
                float n1, s1;
                const bool m1 = member(j, n1, s1) && !DONE;
                if (bits) {
                    const int j2 = r0 + __ffs(bits) - 1;
                    bits &= bits - 1;
                    float n2, s2;
                    const bool m2 = member(j2, n2, s2);
                    if (m1) contrib(j, n1, s1);
                    if (m2 && !DONE) contrib(j2, n2, s2);
                } else if (m1) {
                    contrib(j, n1, s1);
                }
            }
            return;
        }
        while (bits) {
            const int j = r0 + __ffs(bits) - 1;
            bits &= bits - 1;
            evaluate(POS_OF(j), GID(j), REC0(j), REC1(j), kEwa ? REC1(j) : REC2(j),
                     [&](float4& a3, float4& a4, float2& a5) {
                         a3 = REC3(j);
                         a4 = REC4(j);
                         const float4 t = REC5(j);
                         a5 = make_float2(t.x, t.y);
                     });
        }
#undef POS_OF
    };
    // thread staging of list position pos into row `row`: seven independent LDG.128,
    // the footprint mask against every warp's sample block
    auto fill_row = [&](const uint32_t pos, const int row) {
        uint32_t g = __ldg(fb.vals + pos);
        g = (g < (uint32_t)fp.N) ? g : 0u;  // memory safety after a capacity overflow only
        const float4* rp = recv + (size_t)g * kRecF4;
        const float4 a0 = __ldg(rp + 0), a1 = __ldg(rp + 1), a2 = __ldg(rp + 2), a3 = __ldg(rp + 3),
                     a4 = __ldg(rp + 4), a5 = __ldg(rp + 5), a7 = __ldg(rp + 7);
        S.rec[row][0] = a0; S.rec[row][1] = a1; S.rec[row][2] = a2;
        S.rec[row][3] = a3; S.rec[row][4] = a4;
        S.rec[row][5] = make_float4(a5.x, a5.y, a5.z, VRS_GID_IN_REC ? __uint_as_float(g) : a5.w);
        const uint32_t m = footprint_mask<kWarps>(a7, S.wblock);
        S.mask[row] = (g << 8) | (fp.no_cull ? 0xffu : m);
    };

#if VRS_BLEND_ASYNC
    if constexpr (!kTma) {
        // Warp-asynchronous staging ring: stage s = b & 1 holds batch b (kSE list
        // entries).  The block fills batches 0 and 1; afterwards the last warp to
        // finish a stage's batch refills it with the batch two ahead and arrives on
        // its mbarrier, so a warp never waits for the others at a block barrier --
        // only for a batch that is not staged yet.
        const uint32_t nbat = (re - rb + kSE - 1) / kSE;
        if (tid == 0) {
            mbar_init(&S.fullb[0], 1);
            mbar_init(&S.fullb[1], 1);
            S.consumed[0] = 0;
            S.consumed[1] = 0;
            S.alive = kWarps;
        }
        __syncthreads();  // wblock written
        if (tid < 2 * kSE && rb + (uint32_t)tid < re) fill_row(rb + (uint32_t)tid, tid);
        __syncthreads();  // batches 0 and 1 staged, mbarriers initialised
        bool wdone = false;
        volatile uint32_t* const alive = &S.alive;
        for (uint32_t b = 0; b < nbat; b++) {
            const int st = (int)(b & 1u);
            if (b >= 2) {
                const uint32_t par = ((b >> 1) - 1u) & 1u;
                bool quit = false;
                while (!mbar_try_wait(&S.fullb[st], par)) {
                    if (*alive == 0u) { quit = true; break; }
                }
                if (quit) break;
            }
            const uint32_t base = rb + b * (uint32_t)kSE;
            if (!wdone) chunk(st * kSE, (int)min(re - base, (uint32_t)kSE), base);
            // release the stage; the last warp out refills it with batch b + 2
            if (!wdone && __all_sync(0xffffffffu, DONE)) {
                wdone = true;
                if (lane == 0) atomicSub(&S.alive, 1u);
            }
            __syncwarp();
            // (fence-fence synchronisation through the counter: every warp's reads of
            // the stage are ordered before its increment, the last warp's refill writes
            // after its observation of the full count)
            uint32_t last = 0;
            if (lane == 0) {
                __threadfence_block();
                last = (atomicAdd(&S.consumed[st], 1u) == (uint32_t)kWarps - 1u) ? 1u : 0u;
                if (last) __threadfence_block();
            }
            last = __shfl_sync(0xffffffffu, last, 0);
            if (last) {
                __syncwarp();
                const uint32_t bn = b + 2;
                if (lane == 0) S.consumed[st] = 0;
                if (bn < nbat && *alive != 0u) {
                    const uint32_t pos = rb + bn * (uint32_t)kSE + (uint32_t)lane;
                    if (pos < re) fill_row(pos, st * kSE + lane);
                    __syncwarp();
                    if (lane == 0) {
                        __threadfence_block();
                        mbar_arrive(&S.fullb[st]);
                    }
                }
            }
        }
        __syncthreads();  // every warp is out of the ring (the compose reuses mask[])
    } else
#endif
    {
    uint32_t phase = 0;
    if (kTma && tid == 0) {
        mbar_init(&S.full, kWarps);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (uint32_t base = rb; base < re; base += kBatch) {
        __syncthreads();  // the staging buffer is free again (and the mbarrier initialised)
        const uint32_t n = min(re - base, (uint32_t)kBatch);
        if constexpr (kTma) {
            // every warp stages its share of the batch: one TMA bulk copy of r0..r5
            // of each entry's record, completing on the batch's mbarrier (one
            // arrival per warp, carrying its bytes); the issuing lane tests the
            // entry's pixel footprint (r7) against every warp's samples meanwhile
            constexpr uint32_t kPer = (kBatch + kWarps - 1) / kWarps;
            const uint32_t i = (uint32_t)warp * kPer + (uint32_t)lane;
            const bool mine = (uint32_t)lane < kPer && i < n;
            uint32_t g = 0;
            if (mine) {
                g = __ldg(fb.vals + base + i);
                g = (g < (uint32_t)fp.N) ? g : 0u;  // memory safety after a capacity overflow only
                const uint32_t m = footprint_mask<kWarps>(__ldg(recv + (size_t)g * kRecF4 + 7), S.wblock);
                S.mask[i] = (g << 8) | (fp.no_cull ? 0xffu : m);
            }
            // the previous batch was read through the generic proxy (ordered before
            // this point by the block barrier); the copies write through the async proxy
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                const uint32_t w0 = (uint32_t)warp * kPer;
                const uint32_t cnt = n > w0 ? min(n - w0, kPer) : 0u;
                mbar_arrive_expect_tx(&S.full, cnt * kStageBytes);
            }
            __syncwarp();
            if (mine) bulk_g2s(&S.rec[i][0], recv + (size_t)g * kRecF4, kStageBytes, &S.full);
            while (!mbar_try_wait(&S.full, phase)) {
            }
            phase ^= 1u;
        } else {
            // the block's first n threads load one record each (seven independent LDG.128)
            if ((uint32_t)tid < n) fill_row(base + (uint32_t)tid, tid);
        }
        if (__syncthreads_count(!DONE) == 0) break;
        const int nb = min((int)(re - base), kBatch);
        for (int c = 0; c < nb; c += 32) {
            if (__all_sync(0xffffffffu, DONE)) break;
            chunk(c, min(nb - c, 32), base + (uint32_t)c);
        }
    }
    }
    // drain the window in order (sentinels pop as no-ops)
#pragma unroll 1
    for (int k = 0; k < kWindow && !DONE && !kGlobal; k++) {
        blend_one(WK(hk), WA(hk));
        hk = (hk + kSlotBytes) & kRM;
    }
#undef WK
#undef WA
    // outputs: the item's geometry recomputed from an opaque block index (not live through the loop)
    const ItemGeom g = item_geom(fp, block_id_opaque(), half, lane, warp);
    const ViewParams& v = fp.v[g.vi];
    const int px = g.px, py = g.py, kind = g.kind;
    const int tx = g.tile % v.tw, ty = g.tile / v.tw;
    Dd = Dd * sqrtf(fmaf(x, x, fmaf(y, y, 1.0f)));
    const float oR = Cr + Tr * fp.bg[0], oG = Cg + Tr * fp.bg[1], oB = Cb + Tr * fp.bg[2], oA = 1.0f - Tr;
    if (kind == kItemLow) {
        if (px < v.W && py < v.H) {
            const size_t li = (size_t)v.low_off + (size_t)(py >> 1) * v.low_w + (px >> 1);
            fb.low_rgba[li] = make_float4(oR, oG, oB, oA);
            fb.low_depth[li] = Dd;
        }
    } else if (kind == kItemHybrid) {
        // group (lanes l&~9, |1, |8, |9) average, then w*P + (1-w)*avg
        const int l0 = lane & ~9;
        float vals[5] = {oR, oG, oB, oA, Dd};
        float outv[5];
        const float wgt = fovea_weight(v, (float)px + 0.5f, (float)py + 0.5f);
#pragma unroll
        for (int c = 0; c < 5; c++) {
            const float p00 = __shfl_sync(0xffffffffu, vals[c], l0);
            const float p01 = __shfl_sync(0xffffffffu, vals[c], l0 | 1);
            const float p10 = __shfl_sync(0xffffffffu, vals[c], l0 | 8);
            const float p11 = __shfl_sync(0xffffffffu, vals[c], l0 | 9);
            const float avg = ((p00 + p01) + (p10 + p11)) * 0.25f;
            outv[c] = fmaf(wgt, vals[c] - avg, avg);
        }
        if (px < v.W && py < v.H) {
            const size_t pi = (size_t)v.pix_off + (size_t)py * v.W + px;
            store_pixel(fp.out_fmt, rgba, depth, pi, make_float4(outv[0], outv[1], outv[2], outv[3]), outv[4]);
        }
    } else {
        if (px < v.W && py < v.H) {
            const size_t pi = (size_t)v.pix_off + (size_t)py * v.W + px;
            store_pixel(fp.out_fmt, rgba, depth, pi, make_float4(oR, oG, oB, oA), Dd);
        }
    }
    if (kCounters) {
        // evaluations: list entries visited before termination
        const unsigned long long ev = DONE ? (unsigned long long)(stop_pos - rb + 1) : (unsigned long long)(re - rb);
        const bool in_img = (px < v.W && py < v.H);
        const bool overflowed = !kGlobal && n_contrib > (uint32_t)kWindow;
        unsigned long long c0 = in_img ? ev : 0ull, c1 = in_img ? n_contrib : 0u,
                           c2 = (in_img && overflowed) ? 1u : 0u, c3 = (in_img && DONE) ? 1u : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            c0 += __shfl_xor_sync(0xffffffffu, c0, o);
            c1 += __shfl_xor_sync(0xffffffffu, c1, o);
            c2 += __shfl_xor_sync(0xffffffffu, c2, o);
            c3 += __shfl_xor_sync(0xffffffffu, c3, o);
        }
        __syncthreads();
        if (tid < 4) S.cnt[tid] = 0ull;  // (the staging may have used cnt as scratch)
        __syncthreads();
        if (lane == 0) {
            atomicAdd(&S.cnt[0], c0);
            atomicAdd(&S.cnt[1], c1);
            atomicAdd(&S.cnt[2], c2);
            atomicAdd(&S.cnt[3], c3);
        }
        __syncthreads();
        if (tid == 0) {
            atomicAdd(&fb.stats[0], S.cnt[0]);
            atomicAdd(&fb.stats[1], S.cnt[1]);
            atomicAdd(&fb.stats[2], S.cnt[2]);
            atomicAdd(&fb.stats[3], S.cnt[3]);
        }
    }
    // (the compose triggers live in the staging mask array, free after the loop)
    uint32_t* const TRIG = S.mask;
    // In-launch compose: this LowRes tile's samples are final; count it
    // off the 3x3 neighbourhoods that wait for it and compose the ones it completes
    if (kind != kItemLow) return;
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        uint32_t n = 0;
        for (int dj = -1; dj <= 1; dj++)
            for (int di = -1; di <= 1; di++) {
                const int nx = tx + di, ny = ty + dj;
                if (nx < 0 || ny < 0 || nx >= v.tw || ny >= v.th) continue;
                const int t2 = ny * v.tw + nx;
                if (v.cls[t2] != kLow) continue;
                if (atomicSub(&v.lowcnt[t2], 1u) == 1u) TRIG[1 + n++] = (uint32_t)t2;
            }
        if (n) __threadfence();
        TRIG[0] = n;
    }
    __syncthreads();
    const uint32_t ntrig = TRIG[0];
    for (uint32_t i = 0; i < ntrig; i++) {
        const int t2 = (int)TRIG[1 + i];
        for (int q = tid + half * kBT; q < 256; q += kBT) {  // T = 32: 16 x 16 groups
            const int gx = (t2 % v.tw) * 16 + (q % 16), gy = (t2 / v.tw) * 16 + (q / 16);
            compose_group(fp, fb, v, gx, gy, rgba, depth);
        }
        if (tid == 0 && half == 0) v.lowcnt[t2] = v.lowcnt0[t2];  // re-armed for the next frame
    }
}
#undef DONE

void launch_blend(const FrameParams& fp, FrameBufs fb, int total_items, float* rgba, float* depth,
                  cudaStream_t st) {
    if (fp.resort == 1) {
        if (total_items > 0) launch_blend_hier(fp, fb, total_items, rgba, depth, st);
        launch_compose(fp, fb, rgba, depth, st);
        return;
    }
    const unsigned grid = (unsigned)(fp.n_blend_items + fp.n_inv_items);
    if (grid == 0) return;
    const size_t smem = sizeof(BlendSmem);
    auto go = [&](auto kern) {
        ensure_smem_attr((const void*)kern, (int)smem);
        kern<<<grid, kBT, smem, st>>>(fp, fb, rgba, depth);
    };
    const int sel = (fp.counters ? 8 : 0) | (fp.ewa ? 4 : 0) | (fp.staging == VRS_STAGING_TMA ? 2 : 0) |
                    (fp.sort_mode != VRS_SORT_STOPTHEPOP ? 1 : 0);
    switch (sel) {
        case 0: go(k_blend<false, false, false, false>); break;
        case 1: go(k_blend<false, false, false, true>); break;
        case 2: go(k_blend<false, false, true, false>); break;
        case 3: go(k_blend<false, false, true, true>); break;
        case 4: go(k_blend<false, true, false, false>); break;
        case 5: go(k_blend<false, true, false, true>); break;
        case 6: go(k_blend<false, true, true, false>); break;
        case 7: go(k_blend<false, true, true, true>); break;
        case 8: go(k_blend<true, false, false, false>); break;
        case 9: go(k_blend<true, false, false, true>); break;
        case 10: go(k_blend<true, false, true, false>); break;
        case 11: go(k_blend<true, false, true, true>); break;
        case 12: go(k_blend<true, true, false, false>); break;
        case 13: go(k_blend<true, true, false, true>); break;
        case 14: go(k_blend<true, true, true, false>); break;
        default: go(k_blend<true, true, true, true>); break;
    }
}

}  // namespace vrs
