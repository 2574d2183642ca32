// Step 4: the global sort of the Gaussian/tile pairs (P:258
// "this arrangement is sorted") — a hand-written stable LSD onesweep radix
// sort (8-bit digits): one histogram kernel for all digits, then one kernel
// per digit whose blocks rank their 4096-key tile with warp-level
// match_any, resolve the global digit offsets by decoupled look-back over
// the preceding tiles, and scatter.  The grid is persistent (a multiple of
// the SM count); blocks acquire tiles in order from an atomic counter and
// stop at the device-resident pair count, so no host sync is needed.
#include <algorithm>
#include <utility>

#include "vrs_internal.cuh"

namespace vrs {

namespace {
constexpr int kSortThreads = 256;
constexpr int kSortItems = 16;
constexpr int kSortTile = kSortThreads * kSortItems;  // 4096
constexpr int kRadix = 256;
constexpr int kWarps = kSortThreads / 32;
constexpr uint32_t kStAgg = 1u << 30, kStPre = 2u << 30, kStMask = (1u << 30) - 1;

// Status words are self-contained (flag + value): relaxed GPU-scope
// accesses suffice and avoid the L1 invalidation an acquire load implies.
__device__ __forceinline__ void st_release32(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
}  // namespace

// Digit histograms of every pass in one read of the keys.  Each thread reads
// 8 consecutive keys and run-length aggregates equal digits in registers
// before touching shared memory (the high digits -- view/tile rows, depth
// exponent -- repeat along the emission order and would serialise atomics).
__global__ void __launch_bounds__(kSortThreads) k_sort_hist(const uint64_t* __restrict__ keys,
                                                            const uint32_t* __restrict__ n_dev, int64_t cap,
                                                            int passes, uint32_t* hist) {
    __shared__ uint32_t s_h[8][kRadix];
    for (int i = threadIdx.x; i < 8 * kRadix; i += blockDim.x) (&s_h[0][0])[i] = 0;
    __syncthreads();
    const int64_t n = min((int64_t)*n_dev, cap);
    constexpr int R = 8;
    for (int64_t base = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * R; base < n;
         base += (int64_t)gridDim.x * blockDim.x * R) {
        uint64_t k[R];
        if (base + R <= n && (reinterpret_cast<uintptr_t>(keys) & 15) == 0) {
            const ulonglong2* p = reinterpret_cast<const ulonglong2*>(keys + base);
#pragma unroll
            for (int i = 0; i < R / 2; i++) {
                const ulonglong2 q = p[i];
                k[2 * i] = q.x;
                k[2 * i + 1] = q.y;
            }
        } else {
#pragma unroll
            for (int i = 0; i < R; i++) k[i] = (base + i < n) ? keys[base + i] : 0ull;
        }
        const int m = (int)min((int64_t)R, n - base);
        for (int p = 0; p < passes; p++) {
            uint32_t cur = (uint32_t)(k[0] >> (8 * p)) & 0xffu, run = 1;
#pragma unroll
            for (int i = 1; i < R; i++) {
                if (i >= m) break;
                const uint32_t d = (uint32_t)(k[i] >> (8 * p)) & 0xffu;
                if (d == cur) {
                    run++;
                } else {
                    atomicAdd(&s_h[p][cur], run);
                    cur = d;
                    run = 1;
                }
            }
            atomicAdd(&s_h[p][cur], run);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < passes * kRadix; i += blockDim.x) {
        const uint32_t c = (&s_h[0][0])[i];
        if (c) atomicAdd(&hist[i], c);
    }
}

struct OnesweepSmem {
    uint32_t wh[kWarps][kRadix];    // per-warp digit counts -> exclusive offsets
    uint32_t tstart[kRadix];        // tile-local exclusive digit offsets
    uint32_t gbase[kRadix];         // global position of the tile's first key of each digit
    uint32_t doff[kRadix];          // global exclusive digit offsets of this pass
    uint64_t k[kSortTile];          // tile keys in digit-sorted order (staged scatter)
    uint32_t v[kSortTile];
    uint32_t tile;
};

// 64-bit look-back status: epoch (frame/pass tag, so no per-pass memset) |
// flag (1 = tile aggregate, 2 = inclusive prefix) | 32-bit count.
__device__ __forceinline__ void st_status(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_status(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__global__ void __launch_bounds__(kSortThreads, 3) k_onesweep(const uint64_t* __restrict__ kin,
                                                              const uint32_t* __restrict__ vin,
                                                              uint64_t* __restrict__ kout, uint32_t* __restrict__ vout,
                                                              const uint32_t* __restrict__ n_dev, int64_t cap,
                                                              int pass, const uint32_t* __restrict__ hist,
                                                              unsigned long long* status, uint32_t* counter,
                                                              uint32_t epoch) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    OnesweepSmem& S = *reinterpret_cast<OnesweepSmem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int shift = 8 * pass;
    const int64_t n = min((int64_t)*n_dev, cap);
    const int64_t ntiles = (n + kSortTile - 1) / kSortTile;
    const uint32_t lt_mask = (1u << lane) - 1u;
    const unsigned long long ep = (unsigned long long)epoch << 34;
    const unsigned long long kAgg = ep | (1ull << 32), kPre = ep | (2ull << 32);
    // global digit offsets of this pass (exclusive scan of the histogram)
    {
        const uint32_t h = hist[pass * kRadix + tid];
        S.doff[tid] = h;
        __syncthreads();
        if (warp == 0) {
            uint32_t run = 0;
            for (int c = 0; c < kRadix; c += 32) {
                const uint32_t v0 = S.doff[c + lane];
                uint32_t inc = v0;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= o) inc += y;
                }
                S.doff[c + lane] = run + inc - v0;
                run += __shfl_sync(0xffffffffu, inc, 31);
            }
        }
    }
    while (true) {
        if (tid == 0) S.tile = atomicAdd(counter, 1u);
        for (int i = tid; i < kWarps * kRadix; i += kSortThreads) (&S.wh[0][0])[i] = 0;
        __syncthreads();
        const int64_t tile = S.tile;
        if (tile >= ntiles) break;
        const int64_t wbase = tile * kSortTile + (int64_t)warp * (kSortItems * 32);
        uint64_t key[kSortItems];
        uint32_t rank[kSortItems];
#pragma unroll
        for (int i = 0; i < kSortItems; i++) {
            const int64_t idx = wbase + i * 32 + lane;
            key[i] = (idx < n) ? kin[idx] : ~0ull;
        }
        // warp-local stable ranking in (item, lane) order
#pragma unroll
        for (int i = 0; i < kSortItems; i++) {
            const int64_t idx = wbase + i * 32 + lane;
            const bool ok = idx < n;
            const uint32_t d = (uint32_t)(key[i] >> shift) & 0xffu;
            const uint32_t peers = __match_any_sync(0xffffffffu, ok ? d : (0x100u + lane));
            const uint32_t old = ok ? S.wh[warp][d] : 0u;
            __syncwarp();
            if (ok && (peers & lt_mask) == 0) S.wh[warp][d] = old + __popc(peers);
            __syncwarp();
            rank[i] = old + __popc(peers & lt_mask);
        }
        __syncthreads();
        // per digit (thread d): exclusive over warps and tile total; publish the aggregate early
        const int d = tid;  // kSortThreads == kRadix
        uint32_t tot = 0;
#pragma unroll
        for (int w = 0; w < kWarps; w++) {
            const uint32_t c = S.wh[w][d];
            S.wh[w][d] = tot;
            tot += c;
        }
        unsigned long long* st = status + (size_t)tile * kRadix + d;
        st_status(st, (tile == 0 ? kPre : kAgg) | tot);
        S.tstart[d] = tot;
        __syncthreads();
        if (warp == 0) {  // tile-local exclusive scan of the digit totals
            uint32_t run = 0;
            for (int c = 0; c < kRadix; c += 32) {
                const uint32_t v0 = S.tstart[c + lane];
                uint32_t inc = v0;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= o) inc += y;
                }
                S.tstart[c + lane] = run + inc - v0;
                run += __shfl_sync(0xffffffffu, inc, 31);
            }
        }
        __syncthreads();
        // stage keys/values in digit-sorted order (frees the registers before the look-back)
#pragma unroll
        for (int i = 0; i < kSortItems; i++) {
            const int64_t idx = wbase + i * 32 + lane;
            if (idx < n) {
                const uint32_t dd = (uint32_t)(key[i] >> shift) & 0xffu;
                const uint32_t lp = S.tstart[dd] + S.wh[warp][dd] + rank[i];
                S.k[lp] = key[i];
                S.v[lp] = vin[idx];
            }
        }
        // decoupled look-back for digit d, kLook predecessors in flight per round trip
        uint32_t excl = 0;
        if (tile > 0) {
            constexpr int kLook = 16;
            int64_t j = tile - 1;
            while (true) {
                unsigned long long sv[kLook];
#pragma unroll
                for (int k = 0; k < kLook; k++)
                    sv[k] = (j - k >= 0) ? ld_status(status + (size_t)(j - k) * kRadix + d) : kPre;
                int k = 0;
                bool fin = false;
#pragma unroll
                for (; k < kLook; k++) {
                    const unsigned long long e = sv[k] & ~0xffffffffull;
                    if (e != kAgg && e != kPre) break;  // not yet published in this epoch
                    excl += (uint32_t)sv[k];
                    if (e == kPre) { fin = true; break; }
                }
                if (fin) break;
                j -= k;
            }
            st_status(st, kPre | (excl + tot));
        }
        S.gbase[d] = S.doff[d] + excl;
        __syncthreads();
        const int cnt = (int)min((int64_t)kSortTile, n - tile * kSortTile);
        for (int i = tid; i < cnt; i += kSortThreads) {
            const uint64_t kk = S.k[i];
            const uint32_t dd = (uint32_t)(kk >> shift) & 0xffu;
            const uint32_t pos = S.gbase[dd] + (uint32_t)i - S.tstart[dd];
            kout[pos] = kk;
            vout[pos] = S.v[i];
        }
        __syncthreads();
    }
}

__global__ void k_copy_pairs(const uint64_t* __restrict__ ks, const uint32_t* __restrict__ vs, uint64_t* kd,
                             uint32_t* vd, const uint32_t* __restrict__ n_dev, int64_t cap) {
    const int64_t n = min((int64_t)*n_dev, cap);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        kd[i] = ks[i];
        vd[i] = vs[i];
    }
}

size_t sort_status_words(int64_t cap) { return 2 * ((size_t)((cap + kSortTile - 1) / kSortTile + 1) * kRadix); }

static int num_sms() { return device_sms(); }

void launch_sort(uint64_t* keys, uint32_t* vals, uint64_t* keys_alt, uint32_t* vals_alt, const uint32_t* n_dev,
                 int64_t cap, int key_bits, SortScratch s, cudaStream_t st, bool hist_ready) {
    const int passes = (key_bits + 7) / 8;
    if (passes <= 0 || cap <= 0) return;
    const int sms = num_sms();
    const int64_t max_tiles = (cap + kSortTile - 1) / kSortTile;
    cudaMemsetAsync(s.counters, 0, sizeof(uint32_t) * 8, st);
    if (!hist_ready) {
        cudaMemsetAsync(s.hist, 0, sizeof(uint32_t) * 8 * kRadix, st);
        k_sort_hist<<<sms * 2, kSortThreads, 0, st>>>(keys, n_dev, cap, passes, s.hist);
    }
    ensure_smem_attr((const void*)k_onesweep, (int)sizeof(OnesweepSmem));
    const unsigned grid = (unsigned)std::min<int64_t>(max_tiles, (int64_t)sms * 3);
    uint64_t *ka = keys, *kb = keys_alt;
    uint32_t *va = vals, *vb = vals_alt;
    unsigned long long* status = reinterpret_cast<unsigned long long*>(s.status);
    for (int p = 0; p < passes; p++) {
        const uint32_t epoch = (++*s.epoch) & 0x3fffffffu;
        if (epoch == 1)  // (re)start of the epoch sequence: clear stale tags once
            cudaMemsetAsync(status, 0, sizeof(unsigned long long) * (size_t)max_tiles * kRadix, st);
        k_onesweep<<<grid, kSortThreads, sizeof(OnesweepSmem), st>>>(ka, va, kb, vb, n_dev, cap, p, s.hist, status,
                                                                      s.counters + p, epoch);
        std::swap(ka, kb);
        std::swap(va, vb);
    }
    if (ka != keys) k_copy_pairs<<<sms * 2, 256, 0, st>>>(ka, va, keys, vals, n_dev, cap);
}

}  // namespace vrs
