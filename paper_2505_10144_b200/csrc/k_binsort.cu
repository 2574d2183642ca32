// Step 4 ("instantiated ... this arrangement is sorted
// ... ranges"): the (tile, depth) sort of the Gaussian/tile pairs as a binned
// per-tile sort instead of a global radix sort.
//
// The tile test (k_project.cu k_tiletest_direct) already knows every pair's
// tile: it takes the pair's arrival rank from the tile's counter and writes
// (depth bits << 32 | g) straight into the tile's bucket slot (tile *
// kTileCap + rank), or onto an overflow list past kTileCap.  Then:
//   k_tile_scan   decoupled look-back scan of the per-tile counts -> ranges
//                 (empty tiles (0, 0), as the oracle reports them; clamped to
//                 the pair capacity), of the overflow counts -> overflow
//                 offsets, the pair total, the list of non-empty tiles, and
//                 the counters zeroed for the next frame;
//   k_ovf_bucket  overflow pairs -> their per-tile overflow slots;
//   k_tile_sort   one warp per tile of <= 256 pairs (keys in registers,
//                 bitonic by shuffles), one block per larger tile (chunks of
//                 <= 2048 keys sorted as 256-key register runs merged along
//                 merge paths in shared memory; chunks merged along merge
//                 paths in global memory), written back as
//                 (tile << 32 | depth, g) at the tile's range.
// (depth bits, g) is unique inside a tile, so the result does not depend on
// the atomic arrival order and equals the stable (tile, depth) sort of the
// (view, g, tile) emission order -- the oracle's order, bit for bit.
#include "vrs_internal.cuh"

namespace vrs {

namespace {
constexpr int kScanT = 256;
#ifndef VRS_TS_GRID
#define VRS_TS_GRID 4
#endif
constexpr int kScanPer = 4;                     // tiles per thread (one 16-B load)
constexpr int kScanChunk = kScanT * kScanPer;   // tiles per look-back chunk
constexpr int kBinT = 256;
// Tiles up to small_max pairs are sorted by one warp, keys in registers (E <=
// 16); small_max is 512 when the frame has enough tiles to keep every warp
// busy (>= 128 per SM: C3's 35.6k tiles, sort 0.285 -> 0.261 ms), else 256
// (C2's 9k tiles: a 512-key register sort is a long serial chain, and the
// block path's eight warps per tile finish sooner: 0.063 vs 0.070 ms).
constexpr int kWarpSortMax = 512;
constexpr int kWarpSortTilesPerSm = 128;

// Ascending bitonic sort of s[0, P), P a power of two >= 64, by a block of NT
// threads.  Compare-exchange i of a stage with distance j <= 32 touches only
// the 64-element block i >> 5, and thread t always owns blocks (t >> 5) + k *
// NT/32, so such stages synchronise the warp only; a block barrier is needed
// when this or the previous stage crosses warps (j > 32, or j = 32 after 64).
template <int NT>
__device__ __forceinline__ void bitonic_sort_smem(uint64_t* s, uint32_t P) {
    const uint32_t tid = threadIdx.x;
    for (uint32_t k = 2; k <= P; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            if (j > 32 || (j == 32 && k > 64)) __syncthreads();
            else __syncwarp();
            for (uint32_t i = tid; i < (P >> 1); i += NT) {
                const uint32_t ix = ((i & ~(j - 1)) << 1) | (i & (j - 1)), iy = ix | j;
                const uint64_t a = s[ix], b = s[iy];
                if ((a > b) == ((ix & k) == 0)) {
                    s[ix] = b;
                    s[iy] = a;
                }
            }
        }
    }
    __syncthreads();
}

// out[0, na+nb) = merge of the sorted (unique-key) runs a and b; each thread
// of the block finds its merge-path split by binary search and merges its
// share serially.
__device__ __forceinline__ void merge_block(const uint64_t* a, uint32_t na, const uint64_t* b, uint32_t nb,
                                            uint64_t* out) {
    const uint32_t m = na + nb;
    const uint32_t d0 = (uint32_t)((uint64_t)m * threadIdx.x / blockDim.x);
    const uint32_t d1 = (uint32_t)((uint64_t)m * (threadIdx.x + 1) / blockDim.x);
    if (d0 >= d1) return;
    uint32_t lo = d0 > nb ? d0 - nb : 0u, hi = min(d0, na);
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (a[mid] < b[d0 - 1 - mid]) lo = mid + 1;
        else hi = mid;
    }
    uint32_t i = lo, j = d0 - lo;
    for (uint32_t d = d0; d < d1; d++) {
        const bool ta = j >= nb || (i < na && a[i] < b[j]);
        out[d] = ta ? a[i++] : b[j++];
    }
}
// One warp sorts the 256-key run r[0, 256) in shared memory in place, in
// registers (blocked layout through the warp's padded scratch sw, the same
// network as warp_sort_tile).
__device__ __forceinline__ void warp_sort_run256(uint64_t* r, uint64_t* sw, int lane) {
    constexpr int E = 8;
    uint64_t x[E];
#pragma unroll
    for (int e = 0; e < E; e++) {
        const uint32_t idx = (uint32_t)(e * 32 + lane);
        sw[(idx / E) * (E + 1) + idx % E] = r[idx];
    }
    __syncwarp();
#pragma unroll
    for (int e = 0; e < E; e++) x[e] = sw[lane * (E + 1) + e];
#pragma unroll
    for (int k = 2; k <= 32 * E; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j < E) {
#pragma unroll
                for (int e = 0; e < E; e++) {
                    if ((e & j) == 0) {
                        const bool asc = ((lane * E + e) & k) == 0;
                        const uint64_t a = x[e], b = x[e | j];
                        const bool sw_ = (a > b) == asc;
                        x[e] = sw_ ? b : a;
                        x[e | j] = sw_ ? a : b;
                    }
                }
            } else {
                const int jl = j / E;
                const bool keep_min = ((lane & jl) == 0) == (((lane * E) & k) == 0);
#pragma unroll
                for (int e = 0; e < E; e++) {
                    const uint64_t y = __shfl_xor_sync(0xffffffffu, x[e], jl);
                    x[e] = keep_min ? (x[e] < y ? x[e] : y) : (x[e] < y ? y : x[e]);
                }
            }
        }
    }
    __syncwarp();
#pragma unroll
    for (int e = 0; e < E; e++) sw[lane * (E + 1) + e] = x[e];
    __syncwarp();
#pragma unroll
    for (int e = 0; e < E; e++) {
        const uint32_t idx = (uint32_t)(e * 32 + lane);
        r[idx] = sw[(idx / E) * (E + 1) + idx % E];
    }
    __syncwarp();
}

// One warp sorts one tile of n <= 32*E keys held in registers (blocked
// layout: lane l holds elements l*E .. l*E+E-1; padding ~0 sorts last):
// bitonic stages with distance j < E are register compare-exchanges, the
// others exchange with lane l ^ (j/E) by shuffles.  No shared memory, no
// barriers.
template <int E>
__device__ __forceinline__ void warp_sort_tile(const uint64_t* __restrict__ bk, uint32_t n, uint64_t tk,
                                               uint64_t* __restrict__ kout, uint32_t* __restrict__ vout,
                                               uint64_t* sw, int lane) {
    // coalesced (striped) global access, transposed through shared memory
    // (row stride E+1 keeps both orders at the 2-wavefront minimum)
    uint64_t x[E];
#pragma unroll
    for (int e = 0; e < E; e++) {
        const uint32_t idx = (uint32_t)(e * 32 + lane);
        sw[(idx / E) * (E + 1) + idx % E] = idx < n ? bk[idx] : ~0ull;
    }
    __syncwarp();
#pragma unroll
    for (int e = 0; e < E; e++) x[e] = sw[lane * (E + 1) + e];
#pragma unroll
    for (int k = 2; k <= 32 * E; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j < E) {
#pragma unroll
                for (int e = 0; e < E; e++) {
                    if ((e & j) == 0) {
                        const bool asc = ((lane * E + e) & k) == 0;
                        const uint64_t a = x[e], b = x[e | j];
                        const bool sw_ = (a > b) == asc;
                        x[e] = sw_ ? b : a;
                        x[e | j] = sw_ ? a : b;
                    }
                }
            } else {
                const int jl = j / E;
                const bool keep_min = ((lane & jl) == 0) == (((lane * E) & k) == 0);
#pragma unroll
                for (int e = 0; e < E; e++) {
                    const uint64_t y = __shfl_xor_sync(0xffffffffu, x[e], jl);
                    x[e] = keep_min ? (x[e] < y ? x[e] : y) : (x[e] < y ? y : x[e]);
                }
            }
        }
    }
    __syncwarp();
#pragma unroll
    for (int e = 0; e < E; e++) sw[lane * (E + 1) + e] = x[e];
    __syncwarp();
#pragma unroll
    for (int e = 0; e < E; e++) {
        const uint32_t idx = (uint32_t)(e * 32 + lane);
        if (idx < n) {
            const uint64_t v = sw[(idx / E) * (E + 1) + idx % E];
            kout[idx] = tk | (v >> 32);
            vout[idx] = (uint32_t)v;
        }
    }
    __syncwarp();
}
}  // namespace

// Status word of a chunk's look-back: flag (1 = chunk aggregate, 2 =
// inclusive prefix) in bits 62-63, value in bits 0-31.  Relaxed GPU-scope
// accesses: a word carries its own flag, so no acquire ordering is needed.
__device__ __forceinline__ void st_status(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_status(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
constexpr unsigned long long kStatAgg = 1ull << 62, kStatInc = 2ull << 62;

// The per-tile counts -> tile ranges, overflow offsets, the pair total and
// the big / small tile lists, as one decoupled look-back scan over chunks of
// kScanChunk tiles (four scanned quantities: pairs, overflow pairs, big
// tiles, small tiles).  Chunks are taken in launch order from a ticket; the
// last block to finish re-arms the ticket and the status words, and every
// block re-zeroes the counts it read, for the next frame.  List positions
// come from the scan, so both lists are in tile order.
__global__ void __launch_bounds__(kScanT) k_tile_scan(uint32_t* __restrict__ cnt, int64_t n_tiles,
                                                      uint32_t* __restrict__ ranges, uint32_t* __restrict__ ovf_off,
                                                      uint32_t* __restrict__ total, uint32_t cap,
                                                      uint32_t* __restrict__ list, uint32_t* __restrict__ list_n,
                                                      int64_t list_cap, uint32_t small_max,
                                                      unsigned long long* __restrict__ stat, uint32_t* __restrict__ ctr) {
    __shared__ uint32_t s_w[4][kScanT / 32];
    __shared__ uint32_t s_pre[4];
    __shared__ uint32_t s_chunk;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_chunk = atomicAdd(&ctr[0], 1u);
    __syncthreads();
    const uint32_t chunk = s_chunk, n_chunks = (uint32_t)((n_tiles + kScanChunk - 1) / kScanChunk);
    const int64_t t0 = (int64_t)chunk * kScanChunk + (int64_t)tid * kScanPer;
    uint32_t v[kScanPer];
    if (t0 + kScanPer <= n_tiles) {
        const uint4 q = *reinterpret_cast<const uint4*>(cnt + t0);
        v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
        *reinterpret_cast<uint4*>(cnt + t0) = make_uint4(0u, 0u, 0u, 0u);
    } else {
#pragma unroll
        for (int k = 0; k < kScanPer; k++) {
            v[k] = t0 + k < n_tiles ? cnt[t0 + k] : 0u;
            if (t0 + k < n_tiles) cnt[t0 + k] = 0u;
        }
    }
    // this thread's sums: pairs, overflow pairs, big tiles, small tiles (sizes as
    // clamped below only differ after a capacity overflow, which the lists tolerate)
    uint32_t q[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int k = 0; k < kScanPer; k++) {
        q[0] += v[k];
        q[1] += v[k] > kTileCap ? v[k] - kTileCap : 0u;
        q[2] += v[k] > small_max ? 1u : 0u;
        q[3] += (v[k] != 0u && v[k] <= small_max) ? 1u : 0u;
    }
    uint32_t inc[4];
#pragma unroll
    for (int c = 0; c < 4; c++) {
        inc[c] = q[c];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc[c], o);
            if (lane >= o) inc[c] += y;
        }
        if (lane == 31) s_w[c][warp] = inc[c];
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int c = 0; c < 4; c++) {
            uint32_t w = lane < kScanT / 32 ? s_w[c][lane] : 0u;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += y;
            }
            if (lane < kScanT / 32) s_w[c][lane] = w;  // inclusive over warps
        }
        __syncwarp();  // (lanes 0-3 read lane 7's totals)
        // look-back: lane c < 4 carries quantity c
        if (lane < 4) {
            const uint32_t agg = s_w[lane][kScanT / 32 - 1];
            unsigned long long* my = stat + 4 * (size_t)chunk + lane;
            uint32_t pre = 0;
            if (chunk == 0) {
                st_status(my, kStatInc | agg);
            } else {
                st_status(my, kStatAgg | agg);
                for (int64_t p = (int64_t)chunk - 1; p >= 0; p--) {
                    unsigned long long w;
                    do {
                        w = ld_status(stat + 4 * (size_t)p + lane);
                    } while ((w >> 62) == 0ull);
                    pre += (uint32_t)w;
                    if ((w >> 62) == 2ull) break;
                }
                st_status(my, kStatInc | (pre + agg));
            }
            s_pre[lane] = pre;
            if (chunk == n_chunks - 1) {  // the last chunk knows the totals
                if (lane == 0) *total = pre + agg;
                if (lane == 2) list_n[0] = pre + agg;
                if (lane == 3) list_n[1] = pre + agg;
                if (lane == 1) list_n[2] = 0u;  // k_tile_sort's small-tile work counter
            }
        }
    }
    __syncthreads();
    uint32_t e[4];
#pragma unroll
    for (int c = 0; c < 4; c++) e[c] = s_pre[c] + (warp ? s_w[c][warp - 1] : 0u) + inc[c] - q[c];
#pragma unroll
    for (int k = 0; k < kScanPer; k++) {
        const int64_t t = t0 + k;
        if (t < n_tiles) {
            // clamped to the pair capacity (only after an overflow, which the stats report)
            const uint32_t a = min(e[0], cap), b = min(e[0] + v[k], cap);
            reinterpret_cast<uint2*>(ranges)[t] = v[k] ? make_uint2(a, b) : make_uint2(0u, 0u);
            ovf_off[t] = e[1];
            if (v[k] > small_max) list[e[2]++] = (uint32_t)t;                                  // big tiles from the front
            else if (v[k] != 0u) list[list_cap - 1 - e[3]++] = (uint32_t)t;                     // small ones from the back
        }
        e[0] += v[k];
        e[1] += v[k] > kTileCap ? v[k] - kTileCap : 0u;
    }
    // the last block to finish re-arms the ticket and the status words
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        s_chunk = atomicAdd(&ctr[1], 1u) == n_chunks - 1 ? 1u : 0u;
    }
    __syncthreads();
    if (s_chunk) {
        for (uint32_t i = tid; i < 4 * n_chunks; i += kScanT) stat[i] = 0ull;
        if (tid == 0) {
            ctr[0] = 0u;
            ctr[1] = 0u;
        }
    }
}

// Overflow pairs (rank >= kTileCap) into their tile's overflow slots.
__global__ void __launch_bounds__(256) k_ovf_bucket(const uint64_t* __restrict__ okeys,
                                                    const uint32_t* __restrict__ ovals,
                                                    const uint32_t* __restrict__ orank,
                                                    const uint32_t* __restrict__ n_dev, uint32_t cap,
                                                    const uint32_t* __restrict__ ovf_off,
                                                    uint64_t* __restrict__ obucket) {
    const uint32_t n = min(*n_dev, cap);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint64_t k = okeys[i];
        const uint32_t pos = ovf_off[(uint32_t)(k >> 32)] + orank[i] - kTileCap;
        if (pos < cap) obucket[pos] = (k << 32) | ovals[i];
    }
}

__global__ void __launch_bounds__(kBinT, 4) k_tile_sort(const uint32_t* __restrict__ list,
                                                     const uint32_t* __restrict__ list_n, int64_t list_cap,
                                                     const uint32_t* __restrict__ ranges,
                                                     const uint64_t* __restrict__ tbucket,
                                                     const uint32_t* __restrict__ ovf_off,
                                                     const uint64_t* __restrict__ obucket, uint64_t* scratch,
                                                     uint64_t* keys, uint32_t* __restrict__ vals, uint32_t cap_smem,
                                                     uint32_t* work) {
    extern __shared__ __align__(16) uint64_t s_k[];
    const uint32_t tid = threadIdx.x;
    const uint32_t nbig = list_n[0], nsmall = list_n[1];
    // big tiles (> kWarpSortMax pairs): one block each, shared memory / merge path
    for (uint32_t w = blockIdx.x; w < nbig; w += gridDim.x) {
        const uint32_t t = list[w];
        const uint32_t off = ranges[2 * (size_t)t], n = ranges[2 * (size_t)t + 1] - off;
        const uint64_t tk = (uint64_t)t << 32;
        const uint64_t* tb = tbucket + (size_t)t * kTileCap;
        const uint64_t* ob = obucket + ovf_off[t];  // element i >= kTileCap is ob[i - kTileCap]
        uint64_t* bk = scratch + off;
        for (uint32_t c0 = 0; c0 < n; c0 += cap_smem) {
            const uint32_t m = min(cap_smem, n - c0);
            uint32_t P = 64;
            while (P < m) P <<= 1;
            __syncthreads();  // the previous tile/chunk is done with s_k
            for (uint32_t i = tid; i < P; i += kBinT) {
                const uint32_t e = c0 + i;
                s_k[i] = i < m ? (e < kTileCap ? tb[e] : ob[e - kTileCap]) : ~0ull;
            }
            __syncthreads();
            const uint64_t* sorted = s_k;
            if (P >= 512 && P <= kBinCap / 2) {
                // runs of 256 sorted by the 8 warps in registers, then merged pairwise in
                // shared memory (ping-pong with the upper half of s_k; the warps' transpose
                // scratch sits past it)
                uint64_t* sw = s_k + kBinCap + (tid >> 5) * (32 * 9);
                for (uint32_t r = tid >> 5; r < P / 256; r += kBinT / 32) warp_sort_run256(s_k + r * 256, sw, (int)(tid & 31u));
                uint64_t* src = s_k;
                uint64_t* dst = s_k + kBinCap / 2;
                for (uint32_t L = 256; L < P; L <<= 1) {
                    __syncthreads();
                    for (uint32_t s0 = 0; s0 < P; s0 += 2 * L) merge_block(src + s0, L, src + s0 + L, L, dst + s0);
                    uint64_t* tmp = src;
                    src = dst;
                    dst = tmp;
                }
                __syncthreads();
                sorted = src;
            } else {
                bitonic_sort_smem<kBinT>(s_k, P);
            }
            if (n <= cap_smem) {
                for (uint32_t i = tid; i < m; i += kBinT) {
                    const uint64_t k = sorted[i];
                    keys[off + i] = tk | (k >> 32);
                    vals[off + i] = (uint32_t)k;
                }
            } else {
                for (uint32_t i = tid; i < m; i += kBinT) bk[c0 + i] = sorted[i];
            }
        }
        if (n > cap_smem) {  // merge the sorted chunks: scratch <-> keys ping-pong over this tile's range
            uint64_t* src = bk;
            uint64_t* dst = keys + off;
            for (uint32_t L = cap_smem; L < n; L <<= 1) {
                __syncthreads();
                for (uint32_t s0 = 0; s0 < n; s0 += 2 * L) {
                    const uint32_t na = min(L, n - s0), nb = min(L, n - s0 - na);
                    merge_block(src + s0, na, src + s0 + na, nb, dst + s0);
                }
                uint64_t* tmp = src;
                src = dst;
                dst = tmp;
            }
            __syncthreads();
            for (uint32_t i = tid; i < n; i += kBinT) {  // (in place when src is keys: same element, same thread)
                const uint64_t k = src[i];
                keys[off + i] = tk | (k >> 32);
                vals[off + i] = (uint32_t)k;
            }
        }
    }
    // small tiles: one warp each, taken dynamically (warp-private slice of s_k)
    const int lane = (int)(tid & 31u);
    __syncthreads();  // the block path is done with s_k
    uint64_t* sw = s_k + (tid >> 5) * (32 * 17);  // 8 x 4.25 KB scratch inside s_k
    while (true) {
        uint32_t w = 0;
        if (lane == 0) w = atomicAdd(work, 1u);
        w = __shfl_sync(0xffffffffu, w, 0);
        if (w >= nsmall) break;
        const uint32_t t = list[list_cap - 1 - w];
        const uint32_t off = ranges[2 * (size_t)t], n = ranges[2 * (size_t)t + 1] - off;
        const uint64_t tk = (uint64_t)t << 32;
        const uint64_t* tb = tbucket + (size_t)t * kTileCap;  // n <= kWarpSortMax <= kTileCap: all direct slots
        if (n <= 64) warp_sort_tile<2>(tb, n, tk, keys + off, vals + off, sw, lane);
        else if (n <= 128) warp_sort_tile<4>(tb, n, tk, keys + off, vals + off, sw, lane);
        else if (n <= 256) warp_sort_tile<8>(tb, n, tk, keys + off, vals + off, sw, lane);
        else warp_sort_tile<16>(tb, n, tk, keys + off, vals + off, sw, lane);
    }
}

static int sms_now() {
    return device_sms();
}

void launch_binsort(FrameBufs fb, int64_t cap, int64_t n_tiles, BinScratch b, cudaStream_t st) {
    if (n_tiles <= 0) {
        cudaMemsetAsync(fb.total, 0, 4, st);
        return;
    }
    const int sort_smem = (int)(kBinCap * 8 + (kBinT / 32) * 32 * 9 * 8);
    static_assert((kBinT / 32) * 32 * 17 <= kBinCap + (kBinT / 32) * 32 * 9, "small-tile scratch inside s_k");
    ensure_smem_attr((const void*)k_tile_sort, sort_smem);
    const int sms = sms_now();
    const uint32_t small_max = n_tiles >= (int64_t)kWarpSortTilesPerSm * sms ? (uint32_t)kWarpSortMax : 256u;
    const unsigned n_chunks = (unsigned)((n_tiles + kScanChunk - 1) / kScanChunk);
    k_tile_scan<<<n_chunks, kScanT, 0, st>>>(b.tile_cnt, n_tiles, fb.ranges, b.ovf_off, fb.total, (uint32_t)cap, b.list,
                                             b.list_n, b.max_tiles, min(b.cap_smem, small_max), b.scan_stat,
                                             b.scan_ctr);
    k_ovf_bucket<<<sms * 2, 256, 0, st>>>(fb.keys_alt, fb.vals_alt, b.rank, b.ovf_count, (uint32_t)cap, b.ovf_off,
                                          b.obucket);
    k_tile_sort<<<sms * VRS_TS_GRID, kBinT, sort_smem, st>>>(b.list, b.list_n, b.max_tiles, fb.ranges, b.tbucket, b.ovf_off,
                                                     b.obucket, fb.keys_alt, fb.keys, fb.vals, b.cap_smem,
                                                     b.list_n + 2);
}

}  // namespace vrs
