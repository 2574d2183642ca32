// Per-eye static setup ("precompute this mapping once for each
// eye", P:440-449 visibility culling): visibility bitfield from the HMD mask,
// its summed-area table, coarse-tile classes (HighRes / LowRes / Hybrid /
// Invisible) and the blend work list (16x16 items for HighRes and
// Hybrid tiles, one 32x32 item for LowRes tiles, none for Invisible tiles).
// Runs only when a view's mask / fovea / resolution changes; not per frame.
#include "vrs_internal.cuh"

namespace vrs {

// One block per coarse tile: visibility bit (any mask pixel > 0) and class.
__global__ void k_tile_class(const uint8_t* __restrict__ mask, ViewParams v, int T, int32_t* vis, int32_t* cls) {
    const int tx = blockIdx.x, ty = blockIdx.y;
    const int x0 = tx * T, y0 = ty * T;
    const int x1 = min(x0 + T, v.W), y1 = min(y0 + T, v.H);
    const int w = x1 - x0, npx = w * (y1 - y0);
    int any = (mask == nullptr) ? 1 : 0, all1 = 1, all0 = 1;
    for (int k = threadIdx.x; k < npx; k += blockDim.x) {
        int x = x0 + k % w, y = y0 + k / w;
        if (mask && mask[(size_t)y * v.W + x] > 0) any = 1;
        if (v.fovea) {
            float wt = fovea_weight(v, (float)x + 0.5f, (float)y + 0.5f);
            if (wt != 1.0f) all1 = 0;
            if (wt != 0.0f) all0 = 0;
        }
    }
    any = __syncthreads_or(any);
    all1 = __syncthreads_and(all1);
    all0 = __syncthreads_and(all0);
    if (threadIdx.x == 0) {
        int t = ty * v.tw + tx;
        vis[t] = any;
        int c;
        if (!any) c = kInvisible;
        else if (!v.fovea) c = kHigh;
        else c = all1 ? kHigh : (all0 ? kLow : kHybrid);
        cls[t] = c;
    }
}

// Single block: SAT over the bitfield and the work list.
__global__ void k_sat_items(ViewParams v, int T, const int32_t* __restrict__ vis, const int32_t* __restrict__ cls,
                            uint32_t* sat, uint32_t* items, int32_t* n_items, uint32_t* inv_items) {
    const int tw = v.tw, th = v.th, S = tw + 1;
    __shared__ uint32_t s_scan[1024];
    __shared__ uint32_t s_carry;
    // SAT: row prefix sums then column accumulation
    for (int i = threadIdx.x; i < S; i += blockDim.x) sat[i] = 0;
    for (int y = threadIdx.x; y < th; y += blockDim.x) {
        uint32_t run = 0;
        sat[(size_t)(y + 1) * S] = 0;
        for (int x = 0; x < tw; x++) {
            run += (uint32_t)(vis[y * tw + x] != 0);
            sat[(size_t)(y + 1) * S + x + 1] = run;
        }
    }
    __syncthreads();
    for (int x = threadIdx.x; x < tw; x += blockDim.x) {
        uint32_t col = 0;
        for (int y = 0; y < th; y++) {
            col += sat[(size_t)(y + 1) * S + x + 1];
            sat[(size_t)(y + 1) * S + x + 1] = col;
        }
    }
    // work items in tile row-major order, all LowRes items first (pass 0), then
    // the full-rate ones (pass 1): the LowRes blocks start first, so their
    // in-launch compose runs while the full-rate items are still blending
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    const int ntile = tw * th;
    for (int pass = 0; pass < 2; pass++)
    for (int base = 0; base < ntile; base += blockDim.x) {
        int t = base + threadIdx.x;
        uint32_t cnt = 0;
        int c = kInvisible, tx = 0, ty = 0;
        if (t < ntile) {
            c = cls[t];
            tx = t % tw;
            ty = t / tw;
#ifndef VRS_LOW_LAST
#define VRS_LOW_LAST 0
#endif
            const int plow = VRS_LOW_LAST ? 1 : 0;  // pass of the LowRes items
            if (c == kLow) cnt = pass == plow ? 1u : 0u;
            else if (c != kInvisible && pass == 1 - plow) {
                if (T == 16) cnt = 1;
                else
                    for (int sub = 0; sub < 4; sub++)
                        cnt += (tx * T + 16 * (sub & 1) < v.W && ty * T + 16 * (sub >> 1) < v.H) ? 1u : 0u;
            }
        }
        s_scan[threadIdx.x] = cnt;
        __syncthreads();
        for (int off = 1; off < (int)blockDim.x; off <<= 1) {
            uint32_t add = threadIdx.x >= (unsigned)off ? s_scan[threadIdx.x - off] : 0u;
            __syncthreads();
            s_scan[threadIdx.x] += add;
            __syncthreads();
        }
        uint32_t pos = s_carry + s_scan[threadIdx.x] - cnt;
        if (t < ntile && cnt) {
            if (c == kLow) {
                items[pos] = (uint32_t)t | (kItemLow << 22);
            } else {
                uint32_t kind = (c == kHybrid) ? kItemHybrid : kItemFull;
                if (T == 16) {
                    items[pos] = (uint32_t)t | (kind << 22);
                } else {
                    for (int sub = 0; sub < 4; sub++)
                        if (tx * T + 16 * (sub & 1) < v.W && ty * T + 16 * (sub >> 1) < v.H)
                            items[pos++] = (uint32_t)t | ((uint32_t)sub << 20) | (kind << 22);
                }
            }
        }
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) s_carry += s_scan[threadIdx.x];
        __syncthreads();
        if (pass == 0 && base + (int)blockDim.x >= ntile && threadIdx.x == 0)
            n_items[1] = VRS_LOW_LAST ? 0 : (int32_t)s_carry;  // LowRes items listed first (0 if listed last)
    }
    if (threadIdx.x == 0) n_items[0] = (int32_t)s_carry;
    // invisible tiles: background-fill items of the flat blend launch
    __syncthreads();
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (int base = 0; base < ntile; base += blockDim.x) {
        const int t = base + threadIdx.x;
        const uint32_t cnt = (t < ntile && cls[t] == kInvisible) ? 1u : 0u;
        s_scan[threadIdx.x] = cnt;
        __syncthreads();
        for (int off = 1; off < (int)blockDim.x; off <<= 1) {
            uint32_t add = threadIdx.x >= (unsigned)off ? s_scan[threadIdx.x - off] : 0u;
            __syncthreads();
            s_scan[threadIdx.x] += add;
            __syncthreads();
        }
        if (cnt) inv_items[s_carry + s_scan[threadIdx.x] - 1] = (uint32_t)t;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) s_carry += s_scan[threadIdx.x];
        __syncthreads();
    }
    if (threadIdx.x == 0) n_items[2] = (int32_t)s_carry;
}

// In-launch compose counters (P:438 needs a LowRes tile's 3x3 neighbourhood of
// LowRes samples): a LowRes tile waits for the LowRes tiles around it (itself
// included); other tiles get 0.
__global__ void k_low_counts(ViewParams v, const int32_t* __restrict__ cls, uint32_t* cnt, uint32_t* cnt0) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= v.tw * v.th) return;
    const int tx = t % v.tw, ty = t / v.tw;
    uint32_t n = 0;
    if (cls[t] == kLow)
        for (int dj = -1; dj <= 1; dj++)
            for (int di = -1; di <= 1; di++) {
                const int nx = tx + di, ny = ty + dj;
                if (nx >= 0 && ny >= 0 && nx < v.tw && ny < v.th && cls[ny * v.tw + nx] == kLow) n++;
            }
    cnt[t] = n;
    cnt0[t] = n;
}

void launch_setup_view(const uint8_t* mask, int mask_w, ViewParams vp, int T, int32_t* vis, uint32_t* sat,
                       int32_t* cls, uint32_t* items, int32_t* n_items_dev, uint32_t* inv_items, uint32_t* lowcnt,
                       uint32_t* lowcnt0, cudaStream_t st) {
    (void)mask_w;
    k_tile_class<<<dim3(vp.tw, vp.th), 256, 0, st>>>(mask, vp, T, vis, cls);
    k_sat_items<<<1, 1024, 0, st>>>(vp, T, vis, cls, sat, items, n_items_dev, inv_items);
    k_low_counts<<<(vp.tw * vp.th + 255) / 256, 256, 0, st>>>(vp, cls, lowcnt, lowcnt0);
}

}  // namespace vrs
